"""Seeded synthetic inputs shared by tests, bench and smoke.

This package holds NONE of the method's arithmetic: it only draws seeded
random inputs of the paper's shapes and rounds
them to bf16 where the configuration says so.  Both the CUDA path's callers
and the oracle's callers import it; neither the oracle nor the product
package imports the other.
"""
from .inputs import *  # noqa: F401,F403
from .inputs import __all__  # noqa: F401

"""fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY (see attn_softmax_oracle.py)."""
from .attn_softmax_oracle import *  # noqa: F401,F403
from .attn_softmax_oracle import __all__  # noqa: F401

"""fp64 CPU oracle of the optimizer step that follows the gradient exchange
 -- TEST INFRASTRUCTURE ONLY, like
attn_softmax_oracle.py: imported only by tests/, __graft_entry__.smoke() and
bench.py's baseline legs; the product path never touches it.

The paper trains with Adam (Table 2 "optimizer Adam",
"learning rate 0.001"; "Adam [Kingma:15] of the following
setting: beta_1 = 0.9, beta_2 = 0.999, and epsilon = 1e-8").  Adam itself is
not written out in the paper; this is Algorithm 1 of the cited Kingma & Ba
(2015), step by step:

    m_t = beta1 m_{t-1} + (1 - beta1) g_t
    v_t = beta2 v_{t-1} + (1 - beta2) g_t^2
    mhat_t = m_t / (1 - beta1^t)
    vhat_t = v_t / (1 - beta2^t)
    w_t = w_{t-1} - lr mhat_t / (sqrt(vhat_t) + eps)

Sharded form (the data-parallel update of NEXT-2): the summed gradient is
reduce-scattered so rank r owns the contiguous shard [r S, (r+1) S) of the
parameter vector (length padded with zeros to R S), updates only that shard,
and the updated weights are all-gathered.  Adam is elementwise, so the
sharded update equals the replicated one element by element.

Parity pins: tests/test_adam_oracle.py (torch.optim.Adam, the closed form of
the first step, zero gradient, sharded == replicated under gloo).
"""
from __future__ import annotations

import numpy as np

__all__ = ["ADAM_PAPER", "adam_step", "shard_len", "shard_range"]

# PAPER.md:195-196 (Table 2) and :207
ADAM_PAPER = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8)


def adam_step(w, m, v, g, t, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
    """One Adam step (Kingma & Ba 2015, Algorithm 1) at step t >= 1.
    Returns new (w, m, v) as fp64 arrays; inputs are not modified."""
    if t < 1:
        raise ValueError("Adam step t starts at 1")
    w = np.asarray(w, np.float64)
    m = np.asarray(m, np.float64)
    v = np.asarray(v, np.float64)
    g = np.asarray(g, np.float64)
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    mhat = m / (1.0 - beta1 ** t)
    vhat = v / (1.0 - beta2 ** t)
    w = w - lr * mhat / (np.sqrt(vhat) + eps)
    return w, m, v


def shard_len(n: int, world: int, align: int = 4) -> int:
    """Per-rank shard length S: the smallest multiple of `align` with
    world * S >= n (equal shards, as a NCCL reduce-scatter needs)."""
    per = -(-n // world)
    return -(-per // align) * align


def shard_range(n: int, world: int, rank: int, align: int = 4):
    S = shard_len(n, world, align)
    return rank * S, (rank + 1) * S

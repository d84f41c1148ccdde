"""NEXT-2 on the GPU: the Adam step of libattnsm.so (through the C ABI)
against the fp64 oracle (oracle/adam_oracle.py), and the sharded
reduce-scatter / update / all-gather path on a 1-rank NCCL communicator
(bitwise equal to the replicated update)."""
import numpy as np
import pytest
import torch

from oracle.adam_oracle import ADAM_PAPER, adam_step

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("n", [1, 7, 1003, 4 * 1024 * 1024 + 3])
def test_adam_matches_oracle(cuda_lib, n):
    from paper_1909_00562_b200 import binding
    rng = np.random.default_rng(n)
    w0 = rng.normal(scale=0.1, size=n).astype(np.float32)
    w = torch.tensor(w0, device="cuda")
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    wb = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    wo, mo, vo = w0.astype(np.float64), np.zeros(n), np.zeros(n)
    for t in range(1, 6):
        g = rng.normal(scale=10.0 ** rng.uniform(-4, 0), size=n).astype(np.float32)
        binding.attn_adam_step(binding.adam_params(t, **ADAM_PAPER), w, m, v,
                               torch.tensor(g, device="cuda"), wb)
        wo, mo, vo = adam_step(wo, mo, vo, g, t, **ADAM_PAPER)
    torch.cuda.synchronize()
    assert rel_l2(w.cpu().numpy() - w0, wo - w0) < 1e-5      # the accumulated update
    assert rel_l2(m.cpu().numpy(), mo) < 1e-6
    assert rel_l2(v.cpu().numpy(), vo) < 1e-5
    assert torch.equal(wb, w.bfloat16())                     # RNE copy of the fp32 master


def test_sharded_one_rank_equals_replicated(cuda_lib):
    from paper_1909_00562_b200 import binding
    n = 1000003
    uid = binding.attn_comm_get_unique_id()
    comm = binding.attn_comm_init(uid, 1, 0, torch.cuda.current_device())
    try:
        S = binding.attn_adam_shard_len(comm, n)
        assert S % 4 == 0 and S >= n
        rng = np.random.default_rng(3)
        w0 = torch.tensor(rng.normal(size=n).astype(np.float32), device="cuda")
        g = torch.tensor(rng.normal(size=n).astype(np.float32), device="cuda")
        # replicated reference
        w1, m1, v1 = w0.clone(), torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
        b1 = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        h = binding.adam_params(1)
        binding.attn_adam_step(h, w1, m1, v1, g, b1)
        # sharded
        gs = torch.full((S,), float("nan"), device="cuda")
        gs[:n] = g
        ws = torch.zeros(S, device="cuda")
        ws[:n] = w0
        ms, vs = torch.zeros(S, device="cuda"), torch.zeros(S, device="cuda")
        bs = torch.empty(S, dtype=torch.bfloat16, device="cuda")
        binding.attn_adam_step_sharded(comm, h, n, gs, ws, ms, vs, bs)
        torch.cuda.synchronize()
        assert torch.equal(ws[:n], w1) and torch.equal(ms[:n], m1) and torch.equal(vs[:n], v1)
        assert torch.equal(bs[:n], b1)
        assert torch.all(gs[n:] == 0)            # the padded tail was zeroed
    finally:
        binding.attn_comm_destroy(comm)

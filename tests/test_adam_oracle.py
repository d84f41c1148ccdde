"""Pins for oracle/adam_oracle.py (NEXT-2) against things other than itself:
torch.optim.Adam (a library routine), the closed form of the first step,
the zero-gradient fixed point, and the sharded (reduce-scatter / update /
all-gather) decomposition under a world-size-2 gloo group."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.adam_oracle import ADAM_PAPER, adam_step, shard_len, shard_range


def test_matches_torch_adam_several_steps():
    rng = np.random.default_rng(0)
    n = 1000
    w0 = rng.normal(size=n)
    grads = [rng.normal(scale=s, size=n) for s in (1.0, 0.1, 3.0, 1e-3, 0.5)]
    p = torch.nn.Parameter(torch.tensor(w0, dtype=torch.float64))
    opt = torch.optim.Adam([p], lr=ADAM_PAPER["lr"], betas=(ADAM_PAPER["beta1"], ADAM_PAPER["beta2"]),
                           eps=ADAM_PAPER["eps"])
    w, m, v = w0.copy(), np.zeros(n), np.zeros(n)
    for t, g in enumerate(grads, start=1):
        p.grad = torch.tensor(g)
        opt.step()
        w, m, v = adam_step(w, m, v, g, t, **ADAM_PAPER)
        np.testing.assert_allclose(w, p.detach().numpy(), rtol=1e-13, atol=1e-15)
        st = opt.state[p]
        np.testing.assert_allclose(m, st["exp_avg"].numpy(), rtol=1e-13, atol=1e-18)
        np.testing.assert_allclose(v, st["exp_avg_sq"].numpy(), rtol=1e-13, atol=1e-20)


def test_first_step_closed_form_and_zero_gradient():
    """t = 1 from m = v = 0: mhat = g, vhat = g^2, so w1 = w0 - lr g / (|g| + eps)."""
    g = np.array([2.0, -0.5, 1e-3, 0.0, -7.0])
    w0 = np.array([1.0, 2.0, 3.0, 4.0, 5.0])
    lr, eps = 0.01, 1e-8
    w1, m1, v1 = adam_step(w0, np.zeros(5), np.zeros(5), g, 1, lr=lr, eps=eps)
    np.testing.assert_allclose(w1, w0 - lr * g / (np.abs(g) + eps), rtol=1e-14)
    np.testing.assert_allclose(m1, 0.1 * g, rtol=1e-15)
    np.testing.assert_allclose(v1, 0.001 * g * g, rtol=1e-12)   # 1 - 0.999 rounds in fp64
    # a zero gradient leaves w (and zero moments) unchanged
    w2, m2, v2 = adam_step(w1, np.zeros(5), np.zeros(5), np.zeros(5), 3)
    np.testing.assert_array_equal(w2, w1)
    with pytest.raises(ValueError):
        adam_step(w0, m1, v1, g, 0)


def test_shard_ranges_cover_exactly():
    for n in (1, 7, 1000, 52_430_848):
        for R in (1, 2, 4, 8):
            S = shard_len(n, R)
            assert S % 4 == 0 and R * S >= n and R * (S - 4) < n
            assert shard_range(n, R, R - 1)[1] == R * S


def _sharded_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(1)
    n = 1003
    w0 = rng.normal(size=n)
    local_g = [rng.normal(size=n) for _ in range(world)]      # each rank's local gradient
    S = shard_len(n, world)
    pad = lambda a: np.concatenate([a, np.zeros(world * S - n)])
    g_full = torch.tensor(pad(local_g[rank]))
    shard = torch.zeros(S, dtype=torch.float64)
    dist.reduce_scatter(shard, list(g_full.split(S)), op=dist.ReduceOp.SUM)
    lo, hi = shard_range(n, world, rank)
    w_s, _, _ = adam_step(pad(w0)[lo:hi], np.zeros(S), np.zeros(S), shard.numpy(), 1, **ADAM_PAPER)
    parts = [torch.zeros(S, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.tensor(w_s))
    w_sharded = torch.cat(parts).numpy()[:n]
    w_repl, _, _ = adam_step(w0, np.zeros(n), np.zeros(n), sum(local_g), 1, **ADAM_PAPER)
    q.put((rank, float(np.abs(w_sharded - w_repl).max())))
    dist.destroy_process_group()


def test_sharded_update_equals_replicated_gloo():
    """NEXT-2 decomposition: reduce-scatter of the gradient sum, Adam on the
    owned shard, all-gather of the weights == allreduce + replicated Adam."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, err in res:
        assert err < 1e-12, (rank, err)

"""Data-parallel decomposition on CPU with torch.distributed (gloo, world
size 2): each rank builds its sentence shard exactly as bench.py does
(synthetic.shard_range, global loss scale 1 / global valid tokens), runs the
fp64 oracle on it, and the ranks sum loss and weight gradients with an
all_reduce -- the rootless version of "GPU 0 as the root for accumulating and
synchronizing".  Rank 0 checks the sums against the
full-batch oracle (invariant I7) and that each shard's dH equals the
matching slice."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import attn_softmax_oracle as O
    from synthetic import CONFIGS, global_valid_tokens, make_inputs, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = CONFIGS["small_f32"].with_batch(3)      # 3 sentences per rank (weak scaling)
        B_global = cfg.B * world
        lo, hi = shard_range(B_global, world, rank)
        inp = make_inputs(cfg, sentences=range(lo, hi))
        scale = 1.0 / global_valid_tokens(cfg, B_global)
        f, b = O.fwd_bwd(inp["H_dec"], inp["H_enc"], inp["src_len"], inp["tgt_len"],
                         inp["tgt_ids"], inp["W_c"], inp["W_out"], scale)
        loss = torch.tensor([f["loss"]], dtype=torch.float64)
        dWc = torch.from_numpy(b["dW_c"].copy())
        dWo = torch.from_numpy(b["dW_out"].copy())
        for t in (loss, dWc, dWo):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        if rank == 0:
            full = make_inputs(cfg, sentences=range(B_global))
            F, Bk = O.fwd_bwd(full["H_dec"], full["H_enc"], full["src_len"], full["tgt_len"],
                              full["tgt_ids"], full["W_c"], full["W_out"], scale)
            ok = (abs(loss.item() - F["loss"]) < 1e-12 * abs(F["loss"])
                  and np.allclose(dWc.numpy(), Bk["dW_c"], rtol=1e-10, atol=1e-16)
                  and np.allclose(dWo.numpy(), Bk["dW_out"], rtol=1e-10, atol=1e-16)
                  and np.allclose(b["dH_dec"], Bk["dH_dec"][lo:hi], rtol=1e-10, atol=1e-18))
            q.put(bool(ok))
    finally:
        dist.destroy_process_group()


def test_dp_allreduce_equals_full_batch():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    assert q.get(timeout=5) is True


def test_shard_range_partition():
    from synthetic import shard_range
    for B in (1, 5, 128, 257):
        for world in (1, 2, 3, 8):
            spans = [shard_range(B, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1

"""Data parallelism on >= 2 GPUs through the C ABI (SURVEY.md §8(e)
"distributed equally ... GPU 0 as the root for accumulating and
synchronizing"): two processes, one GPU each, each running its contiguous
sentence shard (synthetic.shard_range) with a 2-rank NCCL communicator
created by the library (attn_comm_get_unique_id / attn_comm_init; the id is
passed over a gloo process group).  Checked per rank:

* the in-flight allreduced dW_out (per V-chunk), dW_c and loss equal, bitwise,
  attn_grad_allreduce applied to the local (comm = NULL) results of the same
  rank -- the exchange inside the stage is exactly a sum over ranks;
* the summed loss / dW_c / dW_out match the FULL-batch fp64 oracle within the
  bf16 tolerances, and each rank's dH_dec / dH_enc match the oracle's slice of
  its sentences (invariant I7, DP additivity).

Needs two visible GPUs; on a one-GPU box the test is skipped (there is no
CPU stand-in: the gloo world-2 test of the decomposition is
tests/test_dp_gloo.py)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = {"loss": 2e-3, "grad": 2e-2}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from oracle import attn_softmax_oracle as O
    from paper_1909_00562_b200 import binding
    from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
    from synthetic import CONFIGS, global_valid_tokens, make_inputs, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {"rank": rank, "ok": False, "msg": ""}
    comm = None
    try:
        torch.cuda.set_device(rank)
        cfg = CONFIGS[name]
        B_global = cfg.B * world                       # per-GPU batch fixed (weak scaling)
        lo, hi = shard_range(B_global, world, rank)
        inp = make_inputs(cfg, sentences=range(lo, hi))
        scale = 1.0 / global_valid_tokens(cfg, B_global)
        uid = [binding.attn_comm_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = binding.attn_comm_init(uid[0], world, rank, rank)
        st = AttnSoftmaxStage(hi - lo, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
        dv = to_device(inp, cfg.dtype)
        args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"],
                dv["W_c"], dv["W_out"], scale)
        local = {k: v.clone() for k, v in st(*args).items()}
        torch.cuda.synchronize()
        for k in ("loss", "dW_c", "dW_out"):
            binding.attn_grad_allreduce(comm, local[k])
        out = st(*args, comm=comm)
        torch.cuda.synchronize()
        msgs = []
        for k in ("loss", "dW_c", "dW_out", "dH_dec", "dH_enc"):
            if not torch.equal(out[k], local[k]):
                msgs.append(f"{k}: in-flight exchange != attn_grad_allreduce of the local result")
        full = make_inputs(cfg, sentences=range(B_global))
        F, Bk = O.fwd_bwd(full["H_dec"], full["H_enc"], full["src_len"], full["tgt_len"],
                          full["tgt_ids"], full["W_c"], full["W_out"], scale)
        loss = float(out["loss"].item())
        if abs(loss - F["loss"]) > TOL["loss"] * abs(F["loss"]):
            msgs.append(f"loss {loss} vs full-batch oracle {F['loss']}")
        for k in ("dW_c", "dW_out"):
            e = _rel_l2(out[k].double().cpu().numpy(), Bk[k])
            if e > TOL["grad"]:
                msgs.append(f"{k} rel-L2 {e:.3e} vs the full-batch oracle")
        for k, sl in (("dH_dec", Bk["dH_dec"][lo:hi]), ("dH_enc", Bk["dH_enc"][lo:hi])):
            e = _rel_l2(out[k].double().cpu().numpy(), sl)
            if e > TOL["grad"]:
                msgs.append(f"{k} rel-L2 {e:.3e} vs the oracle's sentences [{lo}, {hi})")
        res["ok"] = not msgs
        res["msg"] = "; ".join(msgs)
    except Exception as ex:   # reported to the parent, which fails the test
        res["msg"] = f"{type(ex).__name__}: {ex}"
    finally:
        if comm is not None:
            binding.attn_comm_destroy(comm)
        q.put(res)
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["small", "medium"])
def test_two_rank_allreduce_matches_full_batch_oracle(cuda_lib, name):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 visible GPUs (this box has %d)" % torch.cuda.device_count())
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for r in sorted(results, key=lambda x: x["rank"]):
        assert r["ok"], f"rank {r['rank']}: {r['msg']}"

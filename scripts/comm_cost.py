"""C1 step time without a communicator, with a 1-rank NCCL communicator, and
with the communicator's SMs reserved as at N > 1 (comm_reserve_1rank):
what the X step and the SM reservation cost on one GPU (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_00562_b200 import binding
from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
from synthetic import CONFIGS, global_valid_tokens, make_inputs
cfg = CONFIGS["paper"]
inp = make_inputs(cfg)
st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
dv = to_device(inp, cfg.dtype)
args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"], dv["W_out"],
        1.0 / global_valid_tokens(cfg, cfg.B))
out = st.alloc_outputs()
comm = binding.attn_comm_init(binding.attn_comm_get_unique_id(), 1, 0, 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(c, reserve, n=10):
    binding.attn_softmax_set_option("comm_reserve_1rank", reserve)
    binding.attn_softmax_set_option("stage_events", 1)
    for _ in range(3):
        st(*args, out=out, comm=c)
    torch.cuda.synchronize()
    tot = 0.0
    for i in range(n):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st(*args, out=out, comm=c)
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    stg = binding.attn_softmax_stage_times()
    print("   ", "reserve" if reserve else ("comm" if c else "none"),
          " ".join(f"{k}={v:.4f}" for k, v in stg.items()), flush=True)
    return tot / n


for r in range(2):
    print(f"no comm {timed(None, 0):.3f} ms | 1-rank comm {timed(comm, 0):.3f} ms | "
          f"1-rank comm, {binding.attn_comm_nranks(comm)} rank, SMs reserved {timed(comm, 1):.3f} ms", flush=True)
binding.attn_comm_destroy(comm)

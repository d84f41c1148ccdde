"""Development sweep of the persistent vocab kernel's options at C1: one
process, each setting timed with CUDA events over 10 L2-flushed steps (not
the bench).  usage: vb_sweep.py "opt=v,opt=v" "opt=v" ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1909_00562_b200 import binding, build
from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
from synthetic import CONFIGS, global_valid_tokens, make_inputs

DEFAULTS = {"vb_wide": 1, "vb_debug": 0}
build.build()
name = os.environ.get("CFG", "paper")
cfg = CONFIGS[name]
inp = make_inputs(cfg)
scale = 1.0 / global_valid_tokens(cfg, cfg.B)
dv = to_device(inp, cfg.dtype)
args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"],
        dv["W_out"], scale)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tok = int(inp["tgt_len"].sum())


def run(spec, n=10):
    opts = {}
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        opts[k] = int(v)
    for k, v in opts.items():
        binding.attn_softmax_set_option(k, v)
    st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
    out = st.alloc_outputs()
    binding.attn_softmax_set_option("stage_events", 1)
    for _ in range(3):
        st(*args, out=out)
    torch.cuda.synchronize()
    tot, stages = 0.0, {}
    for i in range(n):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st(*args, out=out)
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
        for k, v in binding.attn_softmax_stage_times().items():
            stages[k] = stages.get(k, 0) + v / n
    binding.attn_softmax_set_option("stage_events", 0)
    ms = tot / n
    print(f"{spec or 'default':40s} {ms:.3f} ms {tok / ms * 1e3 / 1e6:.3f} Mtok/s vc "
          f"{st.views()['vocab_chunk']} loss {out['loss'].item():.5f} "
          + " ".join(f"{k}={v:.4f}" for k, v in stages.items()), flush=True)
    for k in opts:   # restore
        binding.attn_softmax_set_option(k, DEFAULTS[k])
    del st, out
    torch.cuda.empty_cache()


DEFAULTS.update({"vb_debug": 0, "dl_budget_mb": 200, "dl_buffers": 3, "vb_l2hints": 3,
                 "vb_pair": 1, "vb_order": 1, "vb_fwd_fused": 0, "vocab_chunk": 0,
                 "store_logits": 0, "vb_last_g2_first": 1, "wide_tiles": 2, "vb_order": 1, "vb_lag": 2, "vb_g2split": 1, "vb_claim": 1, "vb_g1wide": 0, "gemm_claim": 4, "n_fast": 1, "mn_3d_tma": 1, "pdl": 1, "attn_fused": 1, "proj_bn": 256})
for spec in sys.argv[1:]:
    run("" if spec == "default" else spec)

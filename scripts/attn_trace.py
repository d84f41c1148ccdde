"""Per-CTA timeline of the fused attention kernels at C1 (development aid):
globaltimer stamps (us from the kernel's first CTA start).
usage: attn_trace.py [config=paper]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1909_00562_b200 import binding
from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
from synthetic import CONFIGS, global_valid_tokens, make_inputs

opts = dict(a.split("=") for a in sys.argv[1:] if "=" in a)
cfg = CONFIGS[opts.pop("config", "paper")]
for k, v in opts.items():
    binding.attn_softmax_set_option(k, int(v))
inp = make_inputs(cfg)
st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
dv = to_device(inp, cfg.dtype)
out = st.alloc_outputs()
args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"],
        dv["W_out"], 1.0 / global_valid_tokens(cfg, cfg.B))
for _ in range(3):
    st(*args, out=out)
tr = torch.zeros(2 * cfg.B * 16 + cfg.B * 256, dtype=torch.int64, device="cuda")
binding.attn_softmax_set_option("attn_trace", tr.data_ptr())
st(*args, out=out)
torch.cuda.synchronize()
binding.attn_softmax_set_option("attn_trace", 0)
t = tr[:2 * cfg.B * 16].view(2, cfg.B, 16).cpu().numpy()
t2 = tr[2 * cfg.B * 16:].view(cfg.B, 64, 4).cpu().numpy()
names = {0: ["start", "loads1 issued", "score MMAs issued", "sfull seen", "alpha done",
             "ctx MMAs issued", "epilogue done", "-", "sm pass1", "sm pass2", "sm P0", "sm st0", "sm st1"],
         1: ["start", "loads1 issued", "dalpha MMAs issued", "sfull seen", "de done",
             "chunk MMAs issued", "epilogue done", "-", "smb pass1", "smb pass2"]}
for k, nm in enumerate(("forward", "backward")):
    x = t[k].astype(np.float64)
    t0 = x[:, 0].min()
    rel = (x - t0) / 1e3
    print(f"{nm}: span {(x[:, 6].max() - t0) / 1e3:.1f} us, SMs {len(np.unique(t[k][:, 7]))}")
    for i in range(len(names[k])):
        if names[k][i] == "-" or not x[:, i].any():
            continue
        print(f"  {names[k][i]:20s} median {np.median(rel[:, i]):6.2f}  min {rel[:, i].min():6.2f}  max {rel[:, i].max():6.2f}")

x = t[1].astype(np.float64)
t0 = x[:, 0].min()
nk = cfg.d // 64
c2 = (t2[:, :nk].astype(np.float64) - t0) / 1e3
print("backward phase 2 per chunk (median over CTAs, us): MMA tempty-ok / full-ok / epi h0 tfull / epi h1 tfull")
for j in range(nk):
    print(f"  chunk {j:2d}: " + " ".join(f"{np.median(c2[:, j, i]):6.2f}" for i in range(4)))

"""Per-tile trace of the decoding step's top-k vocab GEMM (launch 3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace
import numpy as np
import torch
from paper_1909_00562_b200 import binding
from paper_1909_00562_b200.stage import DecodeStep, to_device
from synthetic import CONFIGS, make_inputs
cfg = replace(CONFIGS["paper"], N=5, lengths="full")
inp = make_inputs(cfg)
dv = to_device(inp, cfg.dtype)
step = DecodeStep(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, 5)
args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["W_c"], dv["W_out"])
for _ in range(3):
    step(*args)
tr = torch.zeros(2000 * 16, dtype=torch.int64, device="cuda")
binding.attn_softmax_set_option("gemm_trace_launch", int(sys.argv[1]) if len(sys.argv) > 1 else 3)
binding.attn_softmax_set_option("gemm_trace", tr.data_ptr())
step(*args)
torch.cuda.synchronize()
binding.attn_softmax_set_option("gemm_trace", 0)
t = tr.view(-1, 16).cpu().numpy()
n = int(np.max(np.nonzero(t[:, 4])[0])) + 1
t = t[:n]
print(f"{n} tiles; MMA span median {np.median(t[:,5]-t[:,4]):.0f}; epilogue median {np.median(t[:,7]-t[:,6]):.0f} p90 {np.percentile(t[:,7]-t[:,6],90):.0f}")
print(f"wall {(t[:,15].max()-t[:,14].min())/1e3:.1f} us")

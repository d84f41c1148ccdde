"""Decoding-step (NEXT-4) timing at the paper shape: 128 sentences x beam 5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace
import torch
from paper_1909_00562_b200.stage import DecodeStep, to_device
from synthetic import CONFIGS, make_inputs
cfg = replace(CONFIGS["paper"], N=int(os.environ.get("BEAM", 5)), lengths="full")
inp = make_inputs(cfg)
dv = to_device(inp, cfg.dtype)
step = DecodeStep(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, 5)
for _ in range(3):
    step(dv["H_dec"], dv["H_enc"], dv["src_len"], dv["W_c"], dv["W_out"])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    step(dv["H_dec"], dv["H_enc"], dv["src_len"], dv["W_c"], dv["W_out"])
e1.record()
torch.cuda.synchronize()
print(f"decode step B={cfg.B} beam={cfg.N}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")

"""Eager vs CUDA-graph replay time of the stage (C1) and the decoding step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace
import torch
from paper_1909_00562_b200 import binding
from paper_1909_00562_b200.stage import AttnSoftmaxStage, DecodeStep, to_device
from synthetic import CONFIGS, make_inputs, global_valid_tokens


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def graphed(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g.replay


cfg = CONFIGS["paper"]
inp = make_inputs(cfg)
dv = to_device(inp, cfg.dtype)
st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
out = st.alloc_outputs()
scale = 1.0 / global_valid_tokens(cfg, cfg.B)
f = lambda: st(dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"],
               dv["W_out"], scale, out=out)
print(f"stage eager {timeit(f):.3f} ms, graph {timeit(graphed(f)):.3f} ms")
dcfg = replace(cfg, N=5, lengths="full")
dinp = make_inputs(dcfg, with_weights=False)
dH = torch.from_numpy(dinp["H_dec"]).cuda().bfloat16()
dS = torch.from_numpy(dinp["H_enc"]).cuda().bfloat16()
step = DecodeStep(cfg.B, 5, cfg.M, cfg.d, cfg.V, 5)
T = cfg.B * 5
ids = torch.empty(T, 5, dtype=torch.int32, device="cuda")
lp = torch.empty(T, 5, device="cuda")
d = lambda: binding.attn_softmax_decode_step(step.shape, dH, dS, dinp["src_len"], dv["W_c"],
                                            dv["W_out"], 5, ids, lp, step.workspace)
print(f"decode eager {timeit(d) * 1e3:.1f} us, graph {timeit(graphed(d)) * 1e3:.1f} us")

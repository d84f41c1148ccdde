"""Time the encoder-decoder forward (NEXT-3) at Table 1 sizes and the C1 batch:
CUDA events over K calls (development; bench.py next_rows carries the number)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1909_00562_b200.stage import EncoderDecoder
from synthetic import CONFIGS, make_lstm_inputs

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "paper"]
L, e = 4, 512
inp = make_lstm_inputs(cfg, layers=L, emb=e)
dev = torch.device("cuda")
bf = lambda a: torch.from_numpy(np.asarray(a, np.float32)).to(dev, torch.bfloat16)
ed = EncoderDecoder(cfg.B, cfg.M, cfg.N, e, cfg.d, L, cfg.V, cfg.V)
ed.set_weights([tuple(bf(w) for w in ws) for ws in inp["enc"]], [tuple(bf(w) for w in ws) for ws in inp["dec"]])
src = torch.from_numpy(inp["src_ids"]).to(dev)
tgt = torch.from_numpy(inp["tgt_ids"]).to(dev)
Es, Et = bf(inp["E_src"]), bf(inp["E_tgt"])
H_enc, H_dec = ed(src, tgt, inp["src_len"], Es, Et)
for _ in range(3):
    ed(src, tgt, inp["src_len"], Es, Et, H_enc, H_dec)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 10
a.record()
for _ in range(K):
    ed(src, tgt, inp["src_len"], Es, Et, H_enc, H_dec)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / K
h = cfg.d
flops = sum(2.0 * cfg.B * T * 4 * h * ((e if l == 0 else h) + h) for T in (cfg.M, cfg.N) for l in range(L))
print(f"encoder-decoder fwd {cfg.name}: {ms:.3f} ms, {flops / ms / 1e9:.1f} TFLOP/s, "
      f"layer-steps {(cfg.M + cfg.N) * L}, {ms * 1e3 / (cfg.M + cfg.N + 2 * (L - 1)):.2f} us per wavefront step")

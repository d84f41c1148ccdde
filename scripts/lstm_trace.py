"""Per-step timeline of the LSTM backward wavefront (development aid): the
globaltimer stamps of option "lstm_trace" for the encoder side of one
hybrid step at C1 / Table 1 sizes, summarised per phase.
stamps: 0 E start, 1 E done, 2 dz wait done (producer), 3 first full stage
(MMA), 4 last commit, 5 accumulator seen (epilogue), 6 outdone published"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1909_00562_b200 import binding
from paper_1909_00562_b200.stage import EncoderDecoderTrainer
from synthetic import CONFIGS, make_lstm_inputs

cfg = CONFIGS["paper"]
L, e = 4, 512
dev = torch.device("cuda")
bf = lambda a: torch.from_numpy(np.asarray(a, np.float32)).to(dev, torch.bfloat16)
li = make_lstm_inputs(cfg, layers=L, emb=e)
tr = EncoderDecoderTrainer(cfg.B, cfg.M, cfg.N, e, cfg.d, L, cfg.V, cfg.V)
tr.set_weights([tuple(bf(w) for w in ws) for ws in li["enc"]], [tuple(bf(w) for w in ws) for ws in li["dec"]])
src, tgt = torch.from_numpy(li["src_ids"]).to(dev), torch.from_numpy(li["tgt_ids"]).to(dev)
Es, Et = bf(li["E_src"]), bf(li["E_tgt"])
dS = torch.randn(cfg.B, cfg.M, cfg.d, device=dev).to(torch.bfloat16) * 1e-4
dH = torch.randn(cfg.B, cfg.N, cfg.d, device=dev).to(torch.bfloat16) * 1e-4
for _ in range(2):
    tr.forward(src, tgt, li["src_len"], Es, Et)
    tr.backward(dS, dH)
G = 32
T = cfg.M
buf = torch.zeros(L * G * T * 8, dtype=torch.int64, device=dev)
binding.attn_softmax_set_option("lstm_trace", buf.data_ptr())
tr.forward(src, tgt, li["src_len"], Es, Et)
tr.backward(dS, dH)
torch.cuda.synchronize()
binding.attn_softmax_set_option("lstm_trace", 0)
x = buf.view(L, G, T, 8).cpu().numpy().astype(np.float64)
t0 = x[x > 0].min()
x = np.where(x > 0, (x - t0) / 1e3, np.nan)   # us
print(f"encoder backward: {np.nanmax(x):.1f} us over {T} steps x {L} layers, G = {G}")
for l in range(L):
    for t in (T - 1, T - 2, T // 2, 1, 0):
        r = x[l, :, t]
        med = np.nanmedian(r, axis=0)
        mx = np.nanmax(r, axis=0)
        print(f"l{l} t{t:2d}  " + "  ".join(f"{med[i]:8.1f}/{mx[i]:8.1f}" for i in range(7)))
# per-phase durations (median over CTAs and middle steps)
for l in range(L):
    m = x[l, :, 5:T - 5]
    d = lambda a, b: np.nanmedian(m[..., b] - m[..., a])
    gap = np.nanmedian(m[:, :-1, 0] - m[:, 1:, 0])   # step t starts after step t+1
    print(f"l{l}: step period {gap:.2f}  E {d(0, 1):.2f}  dgdone->dz wait {d(1, 2):.2f}  "
          f"dz wait->first full {d(2, 3):.2f}  MMA {d(3, 4):.2f}  commit->epi {d(4, 5):.2f}  epi->pub {d(5, 6):.2f}")

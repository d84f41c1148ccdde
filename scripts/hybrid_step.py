"""One HybridNMT training step on one B200 at Table 1 / C1 sizes (development
timing; bench.py next_rows carries the number): the model-parallel forward
(wavefront, keeping activations), the data-parallel attention-softmax stage
(forward + backward), and the model-parallel backward (reverse wavefront +
dW GEMMs), each timed with CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1909_00562_b200.stage import AttnSoftmaxStage, EncoderDecoderTrainer
from synthetic import CONFIGS, global_valid_tokens, make_inputs, make_lstm_inputs

cfg = CONFIGS["paper"]
L, e = 4, 512
dev = torch.device("cuda")
bf = lambda a: torch.from_numpy(np.asarray(a, np.float32)).to(dev, torch.bfloat16)
li = make_lstm_inputs(cfg, layers=L, emb=e)
si = make_inputs(cfg)
tr = EncoderDecoderTrainer(cfg.B, cfg.M, cfg.N, e, cfg.d, L, cfg.V, cfg.V)
tr.set_weights([tuple(bf(w) for w in ws) for ws in li["enc"]], [tuple(bf(w) for w in ws) for ws in li["dec"]])
st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, "bf16")
out = st.alloc_outputs()
src, tgt = torch.from_numpy(li["src_ids"]).to(dev), torch.from_numpy(li["tgt_ids"]).to(dev)
Es, Et = bf(li["E_src"]), bf(li["E_tgt"])
W_c, W_out = bf(si["W_c"]), bf(si["W_out"])
ids = torch.from_numpy(si["tgt_ids"]).to(dev)
scale = 1.0 / global_valid_tokens(cfg, cfg.B)


def step():
    H_enc, H_dec = tr.forward(src, tgt, li["src_len"], Es, Et)
    st(H_dec, H_enc, li["src_len"], si["tgt_len"], ids, W_c, W_out, scale, out=out)
    return tr.backward(out["dH_enc"], out["dH_dec"])


for _ in range(3):
    step()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
K = 10
tot = [0.0, 0.0, 0.0]
for _ in range(K):
    ev[0].record()
    H_enc, H_dec = tr.forward(src, tgt, li["src_len"], Es, Et)
    ev[1].record()
    st(H_dec, H_enc, li["src_len"], si["tgt_len"], ids, W_c, W_out, scale, out=out)
    ev[2].record()
    tr.backward(out["dH_enc"], out["dH_dec"])
    ev[3].record()
    torch.cuda.synchronize()
    for i in range(3):
        tot[i] += ev[i].elapsed_time(ev[i + 1]) / K
tok = int(si["tgt_len"].sum())
print(f"hybrid step: MP fwd {tot[0]:.3f} ms, DP stage {tot[1]:.3f} ms, MP bwd {tot[2]:.3f} ms, "
      f"total {sum(tot):.3f} ms, {tok / (sum(tot) / 1e3) / 1e6:.3f} M target tokens/s")

"""Run the C1 stage a few times (for ncu captures; no timing)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1909_00562_b200 import binding
from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
from synthetic import CONFIGS, global_valid_tokens, make_inputs

opts = dict(a.split("=") for a in sys.argv[1:] if "=" in a)
name = opts.pop("config", "paper")
steps = int(opts.pop("steps", "3"))
for k, v in opts.items():
    binding.attn_softmax_set_option(k, int(v))
cfg = CONFIGS[name]
inp = make_inputs(cfg)
st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
dv = to_device(inp, cfg.dtype)
out = st.alloc_outputs()
scale = 1.0 / global_valid_tokens(cfg, cfg.B)
for _ in range(steps):
    st(dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"],
       dv["W_out"], scale, out=out)
torch.cuda.synchronize()
print("loss", out["loss"].item())

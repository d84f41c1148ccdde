"""Runs warm-up steps then a few steps of the stage (for ncu; no timing)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_00562_b200 import binding
from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
from synthetic import CONFIGS, make_inputs, global_valid_tokens

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "paper"]
for k, opt in (("ATTN_VC", "vocab_chunk"), ("ATTN_PAIR", "cta_pair"), ("ATTN_CTAS", "gemm_ctas"),
               ("ATTN_SL", "store_logits")):
    if os.environ.get(k):
        binding.attn_softmax_set_option(opt, int(os.environ[k]))
inp = make_inputs(cfg)
st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
dv = to_device(inp, cfg.dtype)
out = st.alloc_outputs()
scale = 1.0 / global_valid_tokens(cfg, cfg.B)
for i in range(6):
    st(dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"],
       dv["W_out"], scale, out=out)
    torch.cuda.synchronize()
    if i == 0:
        print("launches per step", binding.attn_softmax_last_launches(), flush=True)
print("loss", out["loss"].item())

"""Timeline (globaltimer ns) of each tcgen05 launch of one C1 step: kernel
span from the first MMA issue to the last commit, per-SM start/end spread,
and the gaps between consecutive launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1909_00562_b200 import binding, build
from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
from synthetic import CONFIGS, make_inputs, global_valid_tokens
build.build()
for k, opt in (("ATTN_VC", "vocab_chunk"), ("ATTN_PAIR", "cta_pair")):
    if os.environ.get(k):
        binding.attn_softmax_set_option(opt, int(os.environ[k]))
cfg = CONFIGS["paper"]
inp = make_inputs(cfg)
st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
dv = to_device(inp, cfg.dtype)
out = st.alloc_outputs()
scale = 1.0 / global_valid_tokens(cfg, cfg.B)
args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"], dv["W_out"], scale)
for _ in range(3):
    st(*args, out=out)
torch.cuda.synchronize()
nl = binding.attn_softmax_last_launches()
bufs = []
res = []
for i in range(nl):
    tr = torch.zeros(20000 * 16, dtype=torch.int64, device="cuda")
    binding.attn_softmax_set_option("gemm_trace_launch", i)
    binding.attn_softmax_set_option("gemm_trace", tr.data_ptr())
    st(*args, out=out)
    torch.cuda.synchronize()
    t = tr.view(-1, 16).cpu().numpy()
    nz = np.nonzero(t[:, 14])[0]
    if len(nz) == 0:
        continue
    t = t[: nz.max() + 1]
    t = t[t[:, 14] > 0]
    start, end = t[:, 14].min(), t[:, 15].max()
    sm_end = [t[t[:, 0] == sm][:, 15].max() for sm in np.unique(t[:, 0])]
    sm_start = [t[t[:, 0] == sm][:, 14].min() for sm in np.unique(t[:, 0])]
    res.append((i, len(t), (end - start) / 1e3, (max(sm_start) - min(sm_start)) / 1e3,
                (max(sm_end) - min(sm_end)) / 1e3, np.median(sm_end - np.min(sm_start)) / 1e3))
binding.attn_softmax_set_option("gemm_trace", 0)
print("launch tiles span_us sm_start_spread_us sm_end_spread_us median_sm_busy_until_us")
for r in res:
    print("%3d %6d %8.1f %8.1f %8.1f %8.1f" % r)
binding.attn_softmax_set_option("stage_events", 1)
st(*args, out=out)
print({k: round(v, 4) for k, v in binding.attn_softmax_stage_times().items()})

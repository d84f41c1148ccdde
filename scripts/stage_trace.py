"""Per-tile trace of one tcgen05 launch inside the real stage (C1).
usage: stage_trace.py <launch index> [cta_pair mask]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1909_00562_b200 import binding, build
from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
from synthetic import CONFIGS, make_inputs, global_valid_tokens
build.build()
idx = int(sys.argv[1])
if len(sys.argv) > 2:
    binding.attn_softmax_set_option("cta_pair", int(sys.argv[2]))
wide = int(os.environ.get("ATTN_WIDE", "0"))
binding.attn_softmax_set_option("wide_tiles", wide)
binding.attn_softmax_set_option("mixed_tiles", int(os.environ.get("ATTN_MIXED", "0")))
binding.attn_softmax_set_option("store_logits", int(os.environ.get("ATTN_SL", "1")))
cfg = CONFIGS["paper"]
inp = make_inputs(cfg)
st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
dv = to_device(inp, cfg.dtype)
out = st.alloc_outputs()
scale = 1.0 / global_valid_tokens(cfg, cfg.B)
args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"], dv["W_out"], scale)
for _ in range(3):
    st(*args, out=out)
tr = torch.zeros(20000 * 16, dtype=torch.int64, device="cuda")
binding.attn_softmax_set_option("gemm_trace_launch", idx)
binding.attn_softmax_set_option("gemm_trace", tr.data_ptr())
st(*args, out=out)
torch.cuda.synchronize()
binding.attn_softmax_set_option("gemm_trace", 0)
t = tr.view(-1, 16).cpu().numpy()
nz = np.nonzero(t[:, 4])[0]
if len(nz) == 0:
    sys.exit(f"launch {idx}: no tcgen05 tiles traced")
n = int(np.max(nz)) + 1
t = t[:n]
kinds = sys.argv[3].split(",") if len(sys.argv) > 3 else None
span = t[:, 5] - t[:, 4]
gt0, gt1 = t[:, 14][t[:, 14] > 0], t[:, 15][t[:, 15] > 0]
print(f"launch {idx}: {n} tiles; first MMA -> last commit {(gt1.max() - gt0.min()) / 1e3:.1f} us (globaltimer)")
# group by span size (problem types have distinct k-block counts)
buckets = (((0, 30000, "short"), (30000, 90000, "mid"), (90000, 10**9, "long")) if wide else
           ((0, 13000, "short"), (13000, 40000, "mid"), (40000, 10**9, "long")))
for lo, hi, name in buckets:
    sel = (span >= lo) & (span < hi)
    if sel.sum():
        print(f"  {name:6s} tiles {sel.sum():5d}: MMA span median {np.median(span[sel]):.0f} p90 {np.percentile(span[sel],90):.0f}; epilogue {np.median((t[:,7]-t[:,6])[sel]):.0f}")
gaps = []
busy = []
for sm in np.unique(t[:, 0]):
    rows = t[t[:, 0] == sm]
    rows = rows[np.argsort(rows[:, 4])]
    busy.append((rows[:, 5] - rows[:, 4]).sum() / max(1, rows[-1, 5] - rows[0, 4]))
    for a, b in zip(rows[:-1], rows[1:]):
        gaps.append(b[4] - a[5])
print("  boundary gaps median %d p90 %d; per-SM MMA-busy fraction median %.3f min %.3f" % (
    np.median(gaps), np.percentile(gaps, 90), np.median(busy), np.min(busy)))
starts = []
for sm in np.unique(t[:, 0]):
    rows = t[t[:, 0] == sm]
    starts.append((rows[:, 4].min(), rows[:, 5].max()))
st_ = np.array(starts)
print("  per-SM first MMA spread %d cycles, last commit spread %d cycles" % (st_[:,0].max()-st_[:,0].min(), st_[:,1].max()-st_[:,1].min()))
# MMA-warp breakdown of the tile boundary (medians, cycles)
prev = []
for sm in np.unique(t[:, 0]):
    rows = t[t[:, 0] == sm]
    rows = rows[np.argsort(rows[:, 4])]
    for a, b in zip(rows[:-1], rows[1:]):
        prev.append((b[3] - a[5], b[8] - b[3], b[9] - b[8], b[10] - b[9], b[4] - b[10],
                     b[11] - a[2], b[4] - b[11]))
pv = np.array(prev)
print("  prev commit->id seen %d | ->decoded %d | ->acc free %d | ->full wait %d | ->first MMA %d" %
      tuple(np.median(pv[:, i]) for i in range(5)))
print("  producer: prev last load -> next first load %d | next first load -> its first MMA %d" %
      tuple(np.median(pv[:, i]) for i in (5, 6)))
# launch-level idle from globaltimer stamps (ns): per SM, start delay after the
# first SM's first MMA and idle after its own last commit until the last one
ends, starts = [], []
for sm in np.unique(t[:, 0]):
    rows = t[(t[:, 0] == sm) & (t[:, 14] > 0)]
    if len(rows):
        starts.append(rows[:, 14].min())
        ends.append(rows[:, 15].max())
starts, ends = np.array(starts), np.array(ends)
span = ends.max() - starts.min()
print("  span %.1f us; mean start delay %.1f us; mean end idle %.1f us (%.1f%% of span)" % (
    span / 1e3, (starts - starts.min()).mean() / 1e3, (ends.max() - ends).mean() / 1e3,
    100 * ((ends.max() - ends).mean() + (starts - starts.min()).mean()) / span))

"""Per-tile trace of the persistent vocab backward at C1 (development aid).
usage: vb_trace.py [option=value ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1909_00562_b200 import binding, build
from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
from synthetic import CONFIGS, global_valid_tokens, make_inputs

build.build()
opts = dict(a.split("=") for a in sys.argv[1:] if "=" in a)
name = opts.pop("config", "paper")
for k, v in opts.items():
    binding.attn_softmax_set_option(k, int(v))
cfg = CONFIGS[name]
inp = make_inputs(cfg)
st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
dv = to_device(inp, cfg.dtype)
out = st.alloc_outputs()
scale = 1.0 / global_valid_tokens(cfg, cfg.B)
args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"],
        dv["W_out"], scale)
for _ in range(3):
    st(*args, out=out)
tr = torch.zeros(400000 * 32, dtype=torch.int64, device="cuda")
binding.attn_softmax_set_option("vb_trace", tr.data_ptr())
st(*args, out=out)
torch.cuda.synchronize()
binding.attn_softmax_set_option("vb_trace", 0)
t = tr.view(-1, 32).cpu().numpy()
t = t[0::2]   # rank 0 of each tile (the pair leader records the MMA stamps)
n = int(np.max(np.nonzero(t[:, 4])[0])) + 1
t = t[:n]
typ = t[:, 1] >> 16
chunk = t[:, 1] & 0xFFFF
names = {0: "G1 dlogits", 1: "G3 dHc", 2: "G2 dW_out", 3: "G0 fwd", 4: "G5 lse"}
mm = typ != 4
gt0 = t[mm, 8].min()
gend = t[:, 11].max()
print(f"{n} tiles, vc={st.views()['vocab_chunk']}, span first MMA -> last epilogue "
      f"{(gend - gt0) / 1e3:.1f} us")
T, d = cfg.B * cfg.N, cfg.d
vc = st.views()["vocab_chunk"]
g5 = typ == 4
if g5.any():
    w = (t[g5, 10] - t[g5, 6]) / 1e3
    wk = (t[g5, 11] - t[g5, 10]) / 1e3
    st = (t[g5, 6] - t[g5, 2]) / 1e3
    print(f"  G5 lse      {g5.sum():5d} tiles: dispatch->epilogue {np.median(st):.1f} us, g0 wait median {np.median(w):.1f} max {w.max():.1f} us, "
          f"work median {np.median(wk):.1f} max {wk.max():.1f} us; ends at {((t[g5, 11] - t[mm, 8].min()) / 1e3).round(0).tolist()}")
g1 = typ == 0
if g1.any():
    lw = (t[g1, 12] - t[g1, 15]) / 1e3
    print(f"  G1 epilogue lse/buffer wait median {np.median(lw):.2f} us p90 {np.percentile(lw, 90):.2f} max {lw.max():.1f}")
for k in (3, 0, 1, 2):
    sel = typ == k
    if not sel.any():
        continue
    kb = {0: d // 64, 1: vc // 64, 2: (T + 63) // 64, 3: d // 64}[k]
    if k in (1, 2) and int(opts.get("vb_wide", 1)) and d % 512 == 0:
        kb *= 2   # a wide k-block is two N = 256 MMAs: count 512-cycle units
    span = (t[sel, 5] - t[sel, 4])
    ghz = np.median(span / np.maximum(t[sel, 9] - t[sel, 8], 1))
    print(f"  {names[k]:11s} {sel.sum():5d} tiles: MMA span/kblock median {np.median(span) / kb:.0f} "
          f"p90 {np.percentile(span, 90) / kb:.0f} cyc (ideal 512); full-wait frac "
          f"{np.median(t[sel, 14] / np.maximum(span, 1)):.2f}; producer dep wait median "
          f"{np.median(t[sel, 3] - t[sel, 2]) / 1e3:.2f} us p90 {np.percentile(t[sel, 3] - t[sel, 2], 90) / 1e3:.2f}; "
          f"epilogue {np.median(t[sel, 7] - t[sel, 6]):.0f} cyc (dep wait {np.median(t[sel, 12] - t[sel, 6]):.0f}, "
          f"p90 {np.percentile(t[sel, 12] - t[sel, 6], 90):.0f}); accumulator held {np.median(t[sel, 16] - t[sel, 6]):.0f} cyc "
          f"after ready, {np.median(t[sel, 16] - t[sel, 5]):.0f} after the last MMA issue; SM clock {ghz:.2f} GHz")
busy, gaps, accw = [], [], []
tm_ = t[mm]
for sm in np.unique(tm_[:, 0]):
    r = tm_[tm_[:, 0] == sm]
    r = r[np.argsort(r[:, 4])]
    busy.append((r[:, 5] - r[:, 4]).sum() / max(1, r[-1, 5] - r[0, 4]))
    for a, b in zip(r[:-1], r[1:]):
        gaps.append(b[4] - a[5])
        accw.append(b[13] - a[5])
print(f"  per-SM MMA-busy fraction median {np.median(busy):.3f} min {np.min(busy):.3f}; "
      f"tile boundary gap median {np.median(gaps):.0f} p90 {np.percentile(gaps, 90):.0f} cyc; "
      f"accumulator-free wait after prev commit median {np.median(accw):.0f}")
# timeline: fraction of SMs in MMA per type over 20 time bins (globaltimer)
bins = np.linspace(gt0, t[:, 9].max(), 21)
print("  timeline (per 5% of the span: SM-equivalents in MMA of G0 / G1 / G3 / G2):")
line = []
for i in range(20):
    a, b = bins[i], bins[i + 1]
    occ = []
    for k in (3, 0, 1, 2):
        sel = typ == k
        s0 = np.clip(t[sel, 8], a, b)
        s1 = np.clip(t[sel, 9], a, b)
        occ.append((s1 - s0).sum() / (b - a))
    line.append("%3.0f/%3.0f/%3.0f/%3.0f" % tuple(occ))
print("   " + " ".join(line[:10]))
print("   " + " ".join(line[10:]))
# last tiles to finish
end = np.where(mm, t[:, 9], 0)
o = np.argsort(end)[-5:]
print("  last commits:", [(names[int(typ[i])], int(chunk[i]), round((end[i] - gt0) / 1e3, 1)) for i in o])

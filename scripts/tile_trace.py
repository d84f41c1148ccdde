"""Per-tile timeline of one tcgen05 GEMM launch (debug trace option)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1909_00562_b200 import binding, build
build.build()
M, N, K, amn, bmn, pair, epi = (int(x) for x in sys.argv[1:8])
binding.attn_softmax_set_option("cta_pair", 8 if pair == 2 else 0)
binding.attn_softmax_set_option("b_multicast", 8 if pair == 3 else 0)
binding.attn_softmax_set_option("wide_tiles", 8 if pair == 4 else 0)
binding.attn_softmax_set_option("debug_epilogue", epi)
A = torch.randn(K, M, device="cuda").bfloat16() if amn else torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(K, N, device="cuda").bfloat16() if bmn else torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda")  # fp32 (bf16 epilogues use its first half)
tm = 128 * (2 if pair >= 2 else 1)
kb_units = 2 if pair == 4 else 1   # MMA work per k-block in 128x256x64 units
tiles = ((M + tm - 1) // tm) * ((N + 255) // 256)
tr = torch.zeros(tiles * 16, dtype=torch.int64, device="cuda")
for _ in range(3):
    binding.attn_debug_gemm_bf16(M, N, K, A, amn, B, bmn, C)
binding.attn_softmax_set_option("gemm_trace", tr.data_ptr())
binding.attn_debug_gemm_bf16(M, N, K, A, amn, B, bmn, C)
torch.cuda.synchronize()
binding.attn_softmax_set_option("gemm_trace", 0)
t = tr.view(tiles, 16).cpu().numpy().astype(np.int64)
kb = (K + 63) // 64
mma = t[:, 5] - t[:, 4]
print(f"tiles {tiles}, k-blocks/tile {kb}, ideal MMA cycles/tile {kb*512*kb_units}")
print("MMA span (first issue -> last commit issue) cycles: median %d p10 %d p90 %d" % tuple(np.percentile(mma, [50, 10, 90])))
# per SM: gap between consecutive tiles' first MMA issues
gaps, stalls, epis, loadlead = [], [], [], []
for sm in np.unique(t[:, 0]):
    rows = t[t[:, 0] == sm]
    rows = rows[np.argsort(rows[:, 4])]
    for a, b in zip(rows[:-1], rows[1:]):
        gaps.append(b[4] - a[4])
        stalls.append(b[4] - a[5])          # last commit of prev -> first MMA of next
    epis.extend(rows[:, 7] - rows[:, 6])
    loadlead.extend(rows[:, 4] - rows[:, 11])
print("tile-to-tile period cycles: median %d p10 %d p90 %d" % tuple(np.percentile(gaps, [50, 10, 90])))
print("boundary gap (prev last commit -> next first MMA): median %d p90 %d" % tuple(np.percentile(stalls, [50, 90])))
print("epilogue time (tfull -> tempty arrive): median %d p90 %d" % tuple(np.percentile(epis, [50, 90])))
print("first load issue -> first MMA: median %d p90 %d" % tuple(np.percentile(loadlead, [50, 90])))
print("MMA-id-seen -> decoded: %d | decoded -> acc free: %d | acc free -> full wait start: %d | full wait -> first MMA: %d" % (
    np.percentile(t[:, 8] - t[:, 3], 50), np.percentile(t[:, 9] - t[:, 8], 50),
    np.percentile(t[:, 10] - t[:, 9], 50), np.percentile(t[:, 4] - t[:, 10], 50)))
prev_commit = []
for sm in np.unique(t[:, 0]):
    rows = t[t[:, 0] == sm]
    rows = rows[np.argsort(rows[:, 4])]
    for a, b in zip(rows[:-1], rows[1:]):
        prev_commit.append((b[3] - a[5], b[11] - a[5]))
pc = np.array(prev_commit)
pp = []
for sm in np.unique(t[:, 0]):
    rows = t[t[:, 0] == sm]
    rows = rows[np.argsort(rows[:, 4])]
    for a, b in zip(rows[:-1], rows[1:]):
        pp.append((b[12] - a[2], b[13] - b[12], b[11] - b[13], 0, b[11] - a[2]))
pp = np.array(pp)
print("producer: prev last-load -> next published %d | publish -> decoded %d | decoded -> first load %d | last empty wait %d | prev last load -> next first load %d" % tuple(np.percentile(pp[:, i], 50) for i in range(5)))
print("prev last commit -> next id seen (MMA): %d | prev last commit -> next first load issue (producer): %d" % (
    np.percentile(pc[:, 0], 50), np.percentile(pc[:, 1], 50)))

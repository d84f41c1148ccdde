"""Turn a gpurun ncu launch list (gpu__time_duration.sum only) and an optional
--set full capture into the tracked summaries under profiles/ (round 2
layout: the persistent vocab kernel).
usage: summarize_r2.py <launches.csv> <out_prefix> [full.ncu-rep] [note]"""
import csv
import io
import subprocess
import sys

src, prefix = sys.argv[1], sys.argv[2]
rep = sys.argv[3] if len(sys.argv) > 3 and sys.argv[3].endswith(".ncu-rep") else None
note = sys.argv[-1] if len(sys.argv) > 3 and not sys.argv[-1].endswith(".ncu-rep") else ""


def rows_of(txt):
    lines = txt.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.reader(io.StringIO("\n".join(lines[start:]))))


r = rows_of(open(src).read())
h = r[0]
ix = {k: i for i, k in enumerate(h)}
launches = []
for row in r[1:]:
    if len(row) < len(h):
        continue
    launches.append((row[ix["Kernel Name"]].split("(")[0].replace("void ", ""),
                     float(row[ix["Metric Value"]].replace(",", ""))))
# one step = from a lens_kernel to the next
starts = [i for i, (k, _) in enumerate(launches) if k.startswith("lens_kernel")]
a, b = starts[0], (starts[1] if len(starts) > 1 else len(launches))
step = launches[a:b]
tot = sum(t for _, t in step)
out = [f"# ncu launch list: one C1 step (launches {a}..{b - 1} of the capture) {note}",
       "# ncu --metrics gpu__time_duration.sum --clock-control none; serialised, cold-cache: compare SHARES",
       "id,step,kernel,time_us,share_pct"]


def step_name(i, k, prev):
    if k.startswith("lens_kernel"):
        return "lengths upload (kernel parameters)"
    if k.startswith("attn_fwd_kernel"):
        return "F1+F2 fused attention fwd (scores, masked softmax, context)"
    if k.startswith("attn_bwd_kernel"):
        return "B3 fused attention bwd (dalpha, softmax bwd, dQ, dH_enc)"
    if k.startswith("lse_reduce"):
        return "F5 lse_reduce (lse, NLL, loss)"
    if k.startswith("vocab_kernel"):
        return "B1 vocab backward, persistent (recompute per V-chunk, dL chunk scratch, dHc, dW_out)"
    if k.startswith("dz_kernel"):
        return "B1' dz = dHc (1 - H_c^2) (+ zero dW_c)"
    if k.startswith("gemm_tc"):
        return {"attn_fwd_kernel": "F3 proj_tanh (Eq. 4)",
                "gemm_tc_kernel": "F4 vocab_fwd (LSE epilogue, no logits stored)",
                "dz_kernel": "B2a {dC = dz W_c[:, d:], dW_c split-K}",
                "attn_bwd_kernel": "B2b dH_dec = dz W_c[:, :d] + dQ"}.get(prev, k)
    return k


prev = ""
for i, (k, t) in enumerate(step):
    nm = step_name(i, k, prev)
    prev = k.split("<")[0]
    out.append(f"{i},{nm},{k.replace(',', ' ')},{t / 1e3:.1f},{100 * t / tot:.1f}")
out.append(f"# total {tot / 1e3:.1f} us")
open(f"{prefix}_launches_paper.csv", "w").write("\n".join(out) + "\n")
print("\n".join(out))

if rep:
    keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "l1tex__m_xbar2l1tex_read_bytes.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__grid_size", "launch__cluster_dim_x"]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(txt)))
    hh, uu = rr[0], rr[1]
    res = [f"# ncu --set full --clock-control none --import-source on ({rep.split('/')[-1]}) {note}",
           "# dram bytes are cold-cache (ncu flushes caches per replayed pass)"]
    for v in rr[2:]:
        res.append("## " + v[hh.index("Kernel Name")])
        for k in keys:
            if k in hh:
                i = hh.index(k)
                res.append(f"{k}: {v[i]} {uu[i]}")
    open(f"{prefix}_ncu_full_paper.txt", "w").write("\n".join(res) + "\n")
    print("\n".join(res))

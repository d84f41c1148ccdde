"""Turn the ncu outputs of scripts/profile.sh into the tracked summaries
under profiles/ (launch list with step names and shares; --set full metrics
of the captured kernels).
usage: summarize_profile.py <tag> <out_prefix> [note]"""
import csv
import io
import sys

tag, prefix = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""


def rows_of(path):
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    return list(csv.reader(io.StringIO("\n".join(txt[start:]))))


# ---- launch list
r = rows_of(f"gpurun_out/launches_{tag}.csv")
h = r[0]
ix = {k: i for i, k in enumerate(h)}
launch = {}
order = []
for row in r[1:]:
    if len(row) < len(h):
        continue
    key = row[ix["ID"]]
    if key not in launch:
        launch[key] = dict(kernel=row[ix["Kernel Name"]].split("(")[0],
                           grid=row[ix["Grid Size"]] if "Grid Size" in ix else "")
        order.append(key)
    launch[key][row[ix["Metric Name"]]] = float(row[ix["Metric Value"]].replace(",", ""))
n = len(order)
# name the launches from their kernels: attention and projection GEMMs, the
# vocab forward, then per V-chunk either (stored logits) the elementwise
# dlogits kernel + the dW_out/dHc launch, or (recompute) the dlogits-0 launch
# + chunk launches that also recompute chunk c+1
names = ["lengths upload (kernel parameters)", "attn scores+masked softmax (batched)",
         "attn context (batched)", "proj_tanh", "vocab_fwd (LSE epilogue)", "lse_reduce"]
stored = any("dlogits_from" in launch[k]["kernel"] for k in order)
if stored:
    names[4] = "vocab_fwd (LSE epilogue + fp16 logits store)"
c = 0
for k in order[6:]:
    kn = launch[k]["kernel"]
    if "dz_kernel" in kn:
        break
    if "dlogits_from" in kn:
        names.append(f"dlogits chunk {c} (elementwise, from the stored logits)")
    elif stored:
        names.append(f"vocab bwd chunk {c} (dW_out+dHc, 256x256 tiles)")
        c += 1
    elif len(names) == 6:
        names.append("dlogits chunk 0 (128x256 tiles)")
    else:
        names.append(f"vocab bwd chunk {c} (dW_out+dHc+dlogits c+1, 256x256 tiles)")
        c += 1
names += ["dz (tanh bwd)", "proj_bwd (dW_c + dH_part + dC)", "attn bwd dA + softmax bwd",
          "attn bwd dH_dec + dH_enc"]
tot = sum(launch[k]["gpu__time_duration.sum"] for k in order)
out = [f"# ncu launch list, build {tag}: one C1 step after 3 warm-up steps {note}",
       f"# cmd: scripts/profile.sh {tag} paper  (ncu --metrics gpu__time_duration.sum,... --clock-control none)",
       "# per-launch times are cold-cache and serialised (caches flushed per launch): compare SHARES, not absolutes",
       "id,step,kernel,time_us,share_pct,tensor_active_pct,dram_read_MB,dram_write_MB"]
vb = 0.0
for i, k in enumerate(order):
    m = launch[k]
    t = m["gpu__time_duration.sum"]
    nm = names[i] if i < len(names) else "?"
    if 6 <= i <= n - 4:
        vb += t
    out.append(f"{i},{nm},{m['kernel'].replace(',', ' ')},{t / 1e3:.1f},{100 * t / tot:.1f},"
               f"{m.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):.2f},"
               f"{m.get('dram__bytes_read.sum', 0) / 1e6:.1f},{m.get('dram__bytes_write.sum', 0) / 1e6:.1f}")
out.append(f"# total {tot / 1e3:.1f} us; vocab backward (ids 6-{n - 4}, incl. dz) = {100 * vb / tot:.1f}% of the step")
open(f"{prefix}_launches_paper.csv", "w").write("\n".join(out) + "\n")
print("\n".join(out))

# ---- full set
r = list(csv.reader(open(f"gpurun_out/prof_{tag}_raw.csv")))
h = r[0]
want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_hit_rate.pct",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size"]
units = r[1]
lab = (["vocab_fwd (LSE epilogue + fp16 logits store)", "dlogits chunk 0 (elementwise)",
        "vocab_bwd chunk 0 (dW_out + dHc)"] if stored else
       ["vocab_fwd (LSE epilogue)", "dlogits chunk 0", "vocab_bwd chunk 0 (dW_out + dHc + dlogits c+1)"])
out = [f"# ncu --set full, build {tag}, C1 paper config, step 2 of scripts/profile_step.py {note}",
       f"# cmd: scripts/profile.sh {tag} paper (ncu --set full --clock-control none --import-source on -k regex:\"gemm_tc|dlogits_from\")",
       "# dram bytes are cold-cache (ncu flushes caches per replayed pass)"]
for j, row in enumerate(r[2:]):
    out.append(f"## {lab[j] if j < len(lab) else j}")
    out.append(f"Kernel Name: {row[h.index('Kernel Name')]}")
    for w in want:
        if w in h:
            out.append(f"{w}: {row[h.index(w)]} {units[h.index(w)]}")
open(f"{prefix}_ncu_full_paper.txt", "w").write("\n".join(out) + "\n")
print("\n".join(out))

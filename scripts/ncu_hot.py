"""Top stall-sampled SASS lines of one kernel in an ncu report (source page, SASS view).
usage: ncu_hot.py <rep> <kernel regex> [n]"""
import csv, io, subprocess, sys
rep, k = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"] + (["-k", k] if k != "-" else []), capture_output=True, text=True).stdout
lines = txt.splitlines()
r = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = r[0]
ci = {x: i for i, x in enumerate(h)}
rows = []
for i, x in enumerate(r[1:]):
    if len(x) < len(h):
        continue
    try:
        s = float(x[ci["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    rows.append((s, i, x[ci["Source"]].strip()))
tot = sum(a for a, _, _ in rows) or 1
for a, i, c in sorted(rows, reverse=True)[:n]:
    ctx = " | ".join(rr[2][:40] for rr in rows[max(0, i - 2):i])
    print(f"{a:6.0f} {100 * a / tot:5.1f}%  [{i:5d}] {c[:70]:70s}  <- {ctx}")

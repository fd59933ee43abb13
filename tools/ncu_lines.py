"""Per-CUDA-line instruction and stall shares of one kernel launch in an ncu report.
usage: python tools/ncu_lines.py <report.ncu-rep> [n lines]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 45
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = next(r for r in rows if "Instructions Executed" in r)
iS = h.index('Warp Stall Sampling (All Samples)'); iI = h.index('Instructions Executed')
agg = []
for r in rows:
    if len(r) == len(h) and r[2] == '-' and r[0].isdigit():
        try:
            agg.append((int(r[0]), int(r[iI] or 0), int(r[iS] or 0), r[1][:90]))
        except ValueError:
            pass
ti = sum(a[1] for a in agg) or 1; ts = sum(a[2] for a in agg) or 1
print("total inst", ti, "samples", ts)
for a in sorted(agg, key=lambda a: -a[1])[:nl]:
    print(f"{a[0]:5d} {100*a[1]/ti:5.1f}%i {100*a[2]/ts:5.1f}%s  {a[3]}")
# stall reasons of the top stalled lines
keys = ['stall_long_sb', 'stall_short_sb', 'stall_mio', 'stall_lg', 'stall_wait', 'stall_math', 'stall_barrier',
        'stall_branch_resolving', 'stall_no_inst', 'stall_not_selected', 'stall_selected', 'stall_dispatch', 'stall_drain', 'stall_membar']
ks = [k for k in keys if k in h]
tot = {k: 0 for k in ks}
lines = []
for r in rows:
    if len(r) == len(h) and r[2] == '-' and r[0].isdigit():
        v = {k: int(r[h.index(k)] or 0) for k in ks}
        for k in ks:
            tot[k] += v[k]
        lines.append((int(r[iS] or 0), r[0], v, r[1][:60]))
print("stall totals:", {k[6:]: round(100 * tot[k] / ts, 1) for k in ks if tot[k]})
for s, ln, v, src in sorted(lines, key=lambda x: -x[0])[:12]:
    top = sorted(((v[k], k[6:]) for k in ks), reverse=True)[:3]
    print(f"{ln:>5} {100*s/ts:5.1f}%s {top} {src}")

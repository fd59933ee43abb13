"""Per-CUDA-line shared-memory wavefronts (actual / ideal / excessive) of one launch in an ncu report.
usage: python tools/ncu_smem.py <report.ncu-rep> [n lines]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = next(r for r in rows if "Instructions Executed" in r)
iW, iI, iE = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal"), h.index("L1 Wavefronts Shared Excessive")
iG = h.index("L1 Tag Requests Global")
agg = []
for r in rows:
    if len(r) == len(h) and r[2] == '-' and r[0].isdigit():
        f = lambda i: int(float(r[i] or 0))  # noqa: E731
        agg.append((f(iW), f(iI), f(iE), f(iG), int(r[0]), r[1][:80]))
tw = sum(a[0] for a in agg) or 1
tg = sum(a[3] for a in agg) or 1
print(f"shared wavefronts {tw}  ideal {sum(a[1] for a in agg)}  excessive {sum(a[2] for a in agg)}  global tag req {tg}")
for a in sorted(agg, key=lambda a: -a[0])[:nl]:
    print(f"{a[4]:5d} wf {100*a[0]/tw:5.1f}% ideal {a[1]:>11d} exc {a[2]:>11d}  {a[5]}")
print("-- global tag requests")
for a in sorted(agg, key=lambda a: -a[3])[:10]:
    print(f"{a[4]:5d} req {100*a[3]/tg:5.1f}%  {a[5]}")

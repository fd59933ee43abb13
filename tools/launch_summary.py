"""Aggregate an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel name.
usage: python tools/launch_summary.py <launches.csv> [title]"""
import collections
import csv
import re
import sys

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else path
rows = [l for l in open(path) if l.startswith('"')]
r = list(csv.reader(rows))
h = r[0]
iN, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for x in r[1:]:
    if x[iM] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", x[iN])
    name = re.sub(r"\(int\)|\(bool\)", "", name).replace("true", "1").replace("false", "0")
    tot[name] += float(x[iV]) / 1e6
    cnt[name] += 1
all_ms = sum(tot.values())
print(title)
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:10.3f} ms {cnt[k]:5d} launches {100 * v / all_ms:5.1f}%  {k[-70:]}")
print(f"{all_ms:10.3f} ms total")

"""Summarise an ncu report: key raw metrics per kernel and the top SASS lines by instructions/stall samples.
usage: python tools/ncu_top.py <report.ncu-rep> [launch index for the source page] [n lines]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
li = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr = r[0]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_sector_hit_rate.pct', 'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'lts__t_bytes.sum']
idx = [hdr.index(w) for w in want if w in hdr]
for row in r[2:]:
    print(" | ".join(f"{hdr[i].split('.')[0][-28:]}={row[i][:38]}" for i in idx))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(li), "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
h = r[1]
iI_ = h.index("Instructions Executed")
rows = [x for x in r[2:] if len(x) == len(h) and x[iI_].isdigit()]
iS = h.index('Warp Stall Sampling (All Samples)')
iI = h.index('Instructions Executed')
iT = h.index('Avg. Threads Executed')
tot = sum(int(x[iI]) for x in rows) or 1
tots = sum(int(x[iS]) for x in rows) or 1
print('kernel', r[0][1][:80], 'inst', tot, 'samples', tots)
for k, x in enumerate(rows):
    x.append(k)
print("-- by stall samples")
for x in sorted(rows, key=lambda x: -int(x[iS]))[:nl]:
    print(str(x[-1]).rjust(5), f"{int(x[iI]) / tot * 100:5.1f}%i {int(x[iS]) / tots * 100:5.1f}%s", x[iT].rjust(4), x[1][:90])

print("-- instruction share by 40-line SASS block")
for b in range(0, len(rows), 40):
    seg = rows[b:b + 40]
    si = sum(int(x[iI]) for x in seg)
    ss = sum(int(x[iS]) for x in seg)
    if si / tot > 0.01:
        print(str(b).rjust(5), f"{si / tot * 100:5.1f}% inst {ss / tots * 100:5.1f}% samples", seg[0][1][:60])

"""For each global load in a kernel's SASS, the distance (in instructions) to the first later
instruction that reads its destination register (address order; a rough check of load hoisting).
usage: python tools/sass_ldg_use.py <mangled-name-substring> [pattern]"""
import re, subprocess, sys
sub = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else r"LDG\.E"
so = "paper_2301_10622_b200/libsinn.so"
names = subprocess.run(["cuobjdump", "-symbols", so], capture_output=True, text=True).stdout
fn = next(l.split()[-1] for l in names.splitlines() if sub in l)
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, so], capture_output=True, text=True).stdout
ins = []
for l in sass.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
for i, (a, t) in enumerate(ins):
    if re.search(pat, t):
        m = re.search(r"(LDG\S*|LDS\S*)\s+(R\d+)", t)
        if not m:
            continue
        r = m.group(2)
        rn = int(r[1:])
        regs = {f"R{rn + k}" for k in range(4 if ".128" in t else (2 if ".64" in t else 1))}
        for j in range(i + 1, min(i + 400, len(ins))):
            body = ins[j][1]
            ops = body.split(None, 1)
            if len(ops) < 2:
                continue
            srcs = ops[1].split(",")[1:] if not ops[0].startswith(("ST", "RED", "ATOM")) else ops[1].split(",")
            if any(re.search(rf"\b{x}\b", s) for s in srcs for x in regs):
                print(f"{a:05x} {t[:60]:60s} -> first use +{j - i:3d}: {body[:50]}")
                break

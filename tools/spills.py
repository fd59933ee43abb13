"""registers/spills of the k_doc_score instantiations (ptxas -v): python tools/spills.py [substring]"""
import re, subprocess, sys
pat = sys.argv[1] if len(sys.argv) > 1 else "k_doc_score"
out = subprocess.run([sys.executable, "paper_2301_10622_b200/_build.py", "--force", "-v"], capture_output=True, text=True).stdout
name = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        continue
    if name and pat in name:
        if "spill" in line or "Used" in line:
            short = re.sub(r".*" + pat, pat, name)[:40]
            print(short, line.split(":", 1)[-1].strip())

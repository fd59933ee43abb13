"""Print value / score ms / threshold ms / recall of bench JSON lines: python tools/show.py gpurun_out/TAG/*.json"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = d.get("kernels", {})
        print(f"{f:40s} {d['value']:12.0f} score {k.get('score', {}).get('ms_per_step', 0):8.3f} "
              f"init {k.get('init', {}).get('ms_per_step', 0):7.3f} step {d['ms_per_step']:8.3f} "
              f"recall {d['recall'].get('vs_gpu_exact')} frac {d['roofline']['frac']:.4f}")
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)

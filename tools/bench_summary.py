"""One-line summary of a bench.py JSON log: step ms, value, clocks, per-GEMM ms."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unparsable", e)
        continue
    k = {n.split("_")[0]: round(v["avg_ms"], 2) for n, v in d.get("kernels", {}).items() if "gemm" in n}
    c = d.get("clocks", {})
    print(f"{path}: {d['ms_per_step']:.2f} ms  {d['value']:.0f} tok/s  sm {c.get('sm_mhz')} MHz  {k}")

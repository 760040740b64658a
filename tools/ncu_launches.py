"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list of bench.py into a
markdown table of librl kernels per step (the last `steps` occurrences of each kernel).

usage: python tools/ncu_launches.py gpurun_out/r02/ncu_launches.csv [steps=2] > profiles/r02/ncu_launches.md
"""
import collections
import csv
import sys


def main(path, steps=2):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    per = collections.defaultdict(list)
    order = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        if not name.startswith(("void rl::", "rl::")):
            continue
        name = name.replace("void ", "").split("(")[0]
        if name not in per:
            order.append(name)
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
        per[name].append(float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1e-6))
    # per-step launches: the bench issues every kernel the same number of times per step
    total = 0.0
    out = []
    for name in order:
        v = per[name]
        n = max(1, len(v) // (steps + 3 + 2))  # warm-up 3 + timed + e2e-less runs: estimate launches per step
        last = v[-steps * n:] if len(v) >= steps * n else v
        ms = sum(last) / steps
        total += ms
        out.append((name, n, ms))
    print("| kernel | launches / step | ms / step | share |")
    print("|---|---|---|---|")
    for name, n, ms in sorted(out, key=lambda x: -x[2]):
        print(f"| `{name}` | {n} | {ms:.3f} | {100 * ms / total:.1f}% |")
    print(f"| total | | {total:.3f} | |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2)

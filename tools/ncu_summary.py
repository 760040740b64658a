"""Summarise an ncu --set full report into a small markdown table (committed under profiles/).

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN/ncu_summary.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % (active)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->SM bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = ["| kernel | " + " | ".join(n for _, n in METRICS) + " |", "|---" * (len(METRICS) + 1) + "|"]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        name = name.split("(")[0].replace("void ", "")
        cells = []
        for m, _ in METRICS:
            if m in hdr:
                i = hdr.index(m)
                cells.append(f"{r[i]} {units[i]}".strip())
            else:
                cells.append("n/a")
        out.append(f"| {name} | " + " | ".join(cells) + " |")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])

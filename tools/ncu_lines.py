"""Aggregate ncu PC-sampling stalls per CUDA source line for one launch of a report.
usage: python tools/ncu_lines.py REPORT.ncu-rep [launch_index] [top_n]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
    agg = collections.defaultdict(lambda: [0.0, "", collections.Counter()])
    hdr = fname = None
    func = ""
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            func = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            wi = hdr.index("Warp Stall Sampling (All Samples)")
            sc = [(i, c) for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
            continue
        if hdr is None or len(r) <= wi or r[2] not in ("-", ""):
            continue
        try:
            w = float(r[wi])
        except ValueError:
            continue
        a = agg[(fname, int(r[0]))]
        a[0] += w
        a[1] = r[1][:80]
        for i, c in sc:
            try:
                a[2][c] += float(r[i])
            except ValueError:
                pass
    tot = sum(v[0] for v in agg.values()) or 1.0
    print(func[:120])
    for (f, ln), (w, src, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        reasons = ", ".join(f"{k[6:]}={v / w * 100:.0f}%" for k, v in st.most_common(2)) if w else ""
        print(f"{w / tot * 100:5.1f}% {f}:{ln:<4} {src:80s} {reasons}")


if __name__ == "__main__":
    main()

"""How many thread-block clusters of the forward GEMM's shared-memory footprint fit on
this B200 at once, per cluster size (the DESIGN.md §5 argument against 4-CTA clusters).
usage: python tools/cluster_occupancy.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_16144_b200 as rl  # noqa: E402

lib = rl.load_library()
f = lib.rl_debug_max_active_clusters
f.restype = ctypes.c_int32
f.argtypes = [ctypes.c_int32]
for c in (1, 2, 4, 8):
    n = f(c)
    print(f"cluster {c}: {n} co-resident clusters = {n * c} of 148 SMs")

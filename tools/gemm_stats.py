"""Where do the step GEMMs lose tensor-pipe cycles? Runs the four GEMMs once at the GLM-16k
shape (as tools/gemm_traffic.py) on the RL_AB_STATS build and prints, per GEMM, the MMA
issuer's waits (on a free accumulator, on a full smem stage), the producer's waits (on a
free stage, in the soft k-barrier) and the epilogue's drain, as a share of the MMA loop.

usage: python paper_2512_16144_b200/_build.py --ab stats -DRL_AB_STATS
       RL_LIBRARY=ab_libs/librl_stats.so python tools/gemm_stats.py
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import runpy  # noqa: E402

import paper_2512_16144_b200 as rl  # noqa: E402

runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gemm_traffic.py"))
lib = rl.load_library()
NAMES = {0: "K1 fwd (LSE)", 1: "K4 dU", 2: "K5 dH", 3: "K6 dW"}
SLOTS = ["mma_wait_tempty", "mma_wait_full", "mma_total", "prod_wait_empty", "prod_kbarrier", "epi_wait_tfull",
         "epi_drain", "tiles"]
for mode, name in NAMES.items():
    buf = (ctypes.c_ulonglong * (512 * 8))()
    assert lib.rl_ab_stats_read(mode, buf) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(512, 8).astype(np.float64)
    alls = a[:148]                      # one CTA per SM
    leaders = alls[alls[:, 2] > 0]      # the MMA issuer runs on the leader CTA of each pair
    tot = leaders[:, 2].mean()
    tiles = leaders[:, 7].mean()
    line = {
        "tiles/pair": round(tiles, 1),
        "mma cycles/tile": round(tot / max(tiles, 1)),
        "wait tempty %": round(100 * leaders[:, 0].mean() / tot, 2),
        "wait full %": round(100 * leaders[:, 1].mean() / tot, 2),
        "wait full max-CTA %": round(100 * (leaders[:, 1] / leaders[:, 2]).max(), 2),
        "prod wait empty %": round(100 * alls[:, 3].mean() / tot, 2),
        "prod k-barrier %": round(100 * alls[:, 4].mean() / tot, 2),
        "epi wait tfull %": round(100 * alls[:, 5].mean() / tot, 2),
        "epi drain cycles/tile": round(alls[:, 6].mean() / max(tiles, 1)),
    }
    print(name, line)

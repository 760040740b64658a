"""Compile librl.so for sm_100a, in-tree (the .so travels with the gpurun snapshot)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librl.so")
SOURCES = ["rl_api.cu"]
# every source and header of the library (the host side is split over several .cuh)
DEPS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh")))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
    "-cudart", "static", "-Xptxas", "-v",
]
# extra -D flags for A/B builds (RL_NVCC_DEFINES="-DFOO=1 ..."); empty for the product build
EXTRA = os.environ.get("RL_NVCC_DEFINES", "").split()


STAMP = LIB + ".flags"   # the nvcc flags the current librl.so was built with


def _flags_text():
    return " ".join(NVCC_FLAGS + EXTRA)


def _stale():
    if not os.path.exists(LIB):
        return True
    # an A/B build (RL_NVCC_DEFINES) and the product build differ only in flags:
    # rebuild whenever the flags differ from the ones recorded next to the library
    try:
        with open(STAMP) as f:
            if f.read().strip() != _flags_text():
                return True
    except OSError:
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(ROOT, "include", "rl.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build_ab(tag: str, defines: list, verbose: bool = False) -> str:
    """An A/B variant with extra -D flags, written to ab_libs/librl_<tag>.so (select it
    with RL_LIBRARY); the product librl.so is left alone."""
    out = os.path.join(ROOT, "ab_libs", f"librl_{tag}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *NVCC_FLAGS, *defines, "-I", os.path.join(ROOT, "include"),
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building " + out)
    if verbose:
        sys.stderr.write(r.stderr)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *NVCC_FLAGS, *EXTRA, "-I", os.path.join(ROOT, "include"),
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", LIB + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building librl.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    with open(STAMP, "w") as f:
        f.write(_flags_text() + "\n")
    return LIB


if __name__ == "__main__":
    # python _build.py [-f]                     product build
    # python _build.py --ab TAG -DFOO=1 ...     A/B variant in ab_libs/
    if "--ab" in sys.argv:
        i = sys.argv.index("--ab")
        print(build_ab(sys.argv[i + 1], sys.argv[i + 2:], verbose=False))
    else:
        print(build(force="-f" in sys.argv, verbose=True))

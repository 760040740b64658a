"""The C ABI used from plain C (examples/c_abi_step.c: gcc, cudart, librl.so — no Python,
no torch on the compute path). CPU: the example compiles and links against include/rl.h
and the built library. GPU (`-m gpu`): it runs one step on an input artifact the fp64
oracle wrote in another process (tests/make_artifact.py) and its outputs match the
oracle's: loss and counters, dH per row, dW."""
import os
import shutil
import subprocess
import sys

import numpy as np
import pytest

import harness

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2512_16144_b200")


def _compile(out):
    gcc = shutil.which("gcc")
    if gcc is None or not os.path.exists(os.path.join(LIBDIR, "librl.so")):
        pytest.skip("gcc or librl.so missing")
    cmd = [gcc, "-std=c11", "-Wall", "-Wextra", "-Werror", "-O2", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "c_abi_step.c"), "-L", LIBDIR,
           "-l:librl.so", "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_example_compiles_and_links(tmp_path):
    _compile(str(tmp_path / "c_abi_step"))


@pytest.mark.gpu
# tiny without band plants (so the whole dW is compared), the small shape with them (dH per row)
@pytest.mark.parametrize("cfg", [("tiny", 0, [], 2, 4), ("small", 1, ["--tokens", "2048", "--plants"], 8, 8)])
def test_example_step_vs_oracle(tmp_path, cfg):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    name, seed, extra, num_prompts, group = cfg
    exe = _compile(str(tmp_path / "c_abi_step"))
    art = str(tmp_path / "art")
    subprocess.run([sys.executable, os.path.join(ROOT, "tests", "make_artifact.py"), "--config", name, "--seed",
                    str(seed), "--out", art, *extra], check=True, timeout=600)
    r = subprocess.run([exe, art, str(num_prompts), str(group)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    print(r.stdout.strip())
    rep = dict(line.split() for line in open(os.path.join(art, "c_report.txt")).read().splitlines())
    import json
    ref_rep = json.load(open(os.path.join(art, "oracle_report.json")))
    keep = np.load(os.path.join(art, "oracle_keep.npy"))
    coef = np.load(os.path.join(art, "oracle_coef.npy"))
    ratio = np.load(os.path.join(art, "oracle_ratio.npy"))
    valid = np.load(os.path.join(art, "oracle_valid.npy"))
    # tokens within 1e-4 of a bound may take either side (R13); a guard-band token may flip
    # its whole rollout; outside those, the counters are exact
    band = valid & ((np.abs(ratio - 0.5) <= harness.BAND) | (np.abs(ratio - 5.0) <= harness.BAND)
                    | (np.abs(ratio / 1e-5 - 1.0) <= harness.BAND))
    gband = valid & (np.abs(ratio / 1e-5 - 1.0) <= harness.BAND)
    for k in ("nonfinite_inputs", "bad_targets", "bad_offsets"):
        assert int(rep[k]) == ref_rep[k], k
    assert abs(int(rep["masked_low"]) - ref_rep["masked_low"]) <= band.sum()
    assert abs(int(rep["guarded_rollouts"]) - ref_rep["guarded_rollouts"]) <= gband.sum()
    assert int(rep["launches"]) >= 5
    T = len(keep)
    offs = np.fromfile(os.path.join(art, "rollout_offsets.i32"), dtype=np.int32)
    rollout_of = np.repeat(np.arange(len(offs) - 1), np.diff(offs))
    unsure = band | np.isin(rollout_of, rollout_of[gband])
    # the loss is unique given the gate: an unsure row moves it by at most its oracle term
    # plus the largest term a kept token can have (k <= beta = 5)
    adv = np.load(os.path.join(art, "oracle_advantages.npy")).astype(np.float64)
    D = float(np.fromfile(os.path.join(art, "loss_mask.u8"), dtype=np.uint8).sum())
    slack = float((np.abs(coef[unsure]) + 5.0 * np.abs(adv[rollout_of[unsure]]) / D).sum())
    assert abs(float(rep["loss"]) - ref_rep["loss"]) <= harness.LOSS_TOL + slack
    dh = np.fromfile(os.path.join(art, "c_d_hidden.f32"), dtype=np.float32).reshape(T, -1).astype(np.float64)
    dh_ref = np.load(os.path.join(art, "oracle_d_hidden.npy"))
    w = np.fromfile(os.path.join(art, "w_vocab.bf16"), dtype=np.uint16)
    w64 = (w.astype(np.uint32) << 16).view(np.float32).astype(np.float64).reshape(-1, dh.shape[1])
    targets = np.fromfile(os.path.join(art, "targets.i32"), dtype=np.int32)
    # rows whose gate is certain (not in a band, not in a rollout a guard-band token may flip)
    sure = ~unsure
    err = harness.dh_row_error(dh[sure], dh_ref[sure], coef[sure], w64, targets[sure])
    assert err <= 1.0, err
    if name == "tiny":
        assert not unsure.any()
        dw = np.fromfile(os.path.join(art, "c_d_w_vocab.f32"), dtype=np.float32).reshape(w64.shape)
        assert harness.rel_fro(dw, np.load(os.path.join(art, "oracle_d_w_vocab.npy"))) <= harness.GRAD_RTOL
    print(name, "d_hidden_row", err, "unsure rows", int(unsure.sum()))

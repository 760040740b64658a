"""The artifact flow of SURVEY.md §8(d): the oracle writes the inputs and its outputs to a
directory in its own process (tests/make_artifact.py), and this GPU process reads the
same bytes back (sha256-checked against meta.json), runs the step through the C ABI and
compares at the north-star tolerances. The oracle and the CUDA path never share a process.
"""
import json
import os
import subprocess
import sys
import types

import numpy as np
import pytest

import harness
import synth
from synth import artifact

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

HERE = os.path.dirname(os.path.abspath(__file__))


def _load(path):
    meta, a = artifact.read(path)
    wl = synth.Workload(meta["config"], meta["num_prompts"], meta["group_size"], 1, meta["H"], meta["V"])
    T = meta["T"]
    b = synth.Batch(wl, meta["seed"], a["hidden.bf16"], a["w_vocab.bf16"], a["targets.i32"], a["rewards.f32"],
                    a["rollout_offsets.i32"], a["loss_mask.u8"], np.zeros(T), np.zeros(T, bool), np.zeros(T))
    R = meta["num_prompts"] * meta["group_size"]
    c = harness.Case(b, None, None, a["infer_logprobs.f32"], np.zeros(R, np.float32), meta["inv_temperature"],
                     alpha=meta["alpha"], beta=meta["beta"], guard=meta["guard"])
    ref = {n: np.load(os.path.join(path, f"oracle_{n}.npy")) for n in
           ("logprob", "entropy", "lse", "ratio", "coef", "keep", "valid", "guarded", "d_hidden", "d_w_vocab")}
    with open(os.path.join(path, "oracle_report.json")) as f:
        ref["report"] = json.load(f)
    return meta, c, ref


@pytest.mark.parametrize("args", [
    ["--config", "tiny", "--seed", "0", "--plants"],                                   # BASELINE configs[0]
    ["--config", "small", "--seed", "1", "--tokens", "2048", "--plants"],              # small shape, 2048-row sample
])
def test_artifact_gpu_vs_oracle_outputs(tmp_path, args):
    out = str(tmp_path / "art")
    subprocess.run([sys.executable, os.path.join(HERE, "make_artifact.py"), "--out", out, *args], check=True,
                   timeout=600)
    meta, c, ref = _load(out)
    gpu = harness.run_gpu_step(c)
    b = c.batch
    r = ref["report"]
    rep = types.SimpleNamespace(keep=ref["keep"].astype(bool), guarded=ref["guarded"].astype(bool),
                                ratio=ref["ratio"], valid=ref["valid"].astype(bool), coef=ref["coef"],
                                **{k: v for k, v in r.items() if k != "plants"})
    oref = types.SimpleNamespace(logp=ref["logprob"], entropy=ref["entropy"], lse=ref["lse"], report=rep)
    c.plants = {int(k): tuple(v) for k, v in r["plants"].items()}
    # forward, gate (bit-exact outside the 1e-4 bands, incl. the guard band's rollouts),
    # counters, loss: the same contract as every other parity test
    err = harness.compare(c, oref, gpu, check_grads=False)
    flips = np.nonzero(gpu["keep"].astype(bool) != rep.keep)[0]
    same = np.ones(b.T, bool)
    same[flips] = False
    # dH_t depends on row t only: every row whose gate agrees, per row
    err["d_hidden_row"] = harness.dh_row_error(gpu["d_hidden"][same], ref["d_hidden"][same], ref["coef"][same],
                                               artifact_w64(c), b.targets[same])
    assert err["d_hidden_row"] <= 1.0, err
    if not len(flips):
        err["d_w_vocab"] = harness.rel_fro(gpu["d_w_vocab"], ref["d_w_vocab"])
        assert err["d_w_vocab"] <= harness.GRAD_RTOL, err
    print(meta["config"], meta["T"], "x", meta["H"], "x", meta["V"], err, "flips", len(flips))


def artifact_w64(c):
    return synth.bf16_bits_to_float32(c.batch.w_vocab).astype(np.float64)

"""The GEMMs' tile order does not change any result (`-m gpu`).

K1 / K4 / Newton-Schulz take their tiles dynamically by default (a global counter, one
pair per tile; rl_gemm.cuh next_tile), K5 / K6 statically with the soft k-barrier. Each
tile still runs all its k-blocks on one CTA pair in a fixed order, so every output must be
bitwise the same under any schedule. librl reads RL_DYN_TILES once per process, so the
same step (dense and sparse backward, a chunked dU buffer) and a Newton-Schulz run are
executed in subprocesses with every GEMM static, every GEMM dynamic and the default, and
the digests of all outputs compared. The shapes give K1 256 and K4 512 tiles (several
waves over the 74 CTA pairs) plus ragged T / V / H tails.
"""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import torch
import harness, synth
import paper_2512_16144_b200 as rl
wl = synth.Workload("order", 4, 8, 130, 520, 8000, ragged=True, prompt_frac=0.1, delta_sigma=0.8, spike_rate=0.01)
c = harness.make_case(wl, 7, targets="sampled", plants=True)
dig = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
out = {{"T": int(c.batch.T)}}
for chunk, dense in ((0, False), (0, True), (1000, False)):
    g = harness.run_gpu_step(c, dz_chunk_rows=chunk, dense_backward=dense)
    for k in ("logprob", "entropy", "lse", "coef", "keep", "guarded", "d_hidden", "d_w_vocab"):
        out[f"{{chunk}}-{{dense}}-{{k}}"] = dig(g[k])
    out[f"{{chunk}}-{{dense}}-loss"] = repr(g["report"]["loss"])
gen = torch.Generator().manual_seed(3)
x = torch.randn(3000, 520, generator=gen).cuda()
out["ns"] = dig(rl.rl_newton_schulz(x, 5).float().cpu().numpy())
torch.cuda.synchronize()
print(json.dumps(out))
"""


def _run(env_update):
    env = dict(os.environ)
    for k in list(env):
        if k.startswith("RL_DYN_TILES"):
            env.pop(k)
    env.update(env_update)
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_outputs_do_not_depend_on_tile_order():
    default = _run({})
    static = _run({"RL_DYN_TILES": "0"})
    dynamic = _run({"RL_DYN_TILES": "1"})
    assert default["T"] > 4 * 1024
    for name, other in (("static", static), ("dynamic", dynamic)):
        diff = sorted(k for k in default if default[k] != other[k])
        assert not diff, f"{name} order differs from the default in {diff}"

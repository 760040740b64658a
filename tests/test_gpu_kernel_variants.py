"""The non-default GEMM variants against the fp64 oracle (`-m gpu`).

librl reads its tile-shape knobs once per process (RL_WIDE[_<K>], RL_SKEW,
RL_CTA_GROUP; rl_api.cu), so each variant runs the full step in a subprocess:
256x256 tiles everywhere, wide tiles for every GEMM (incl. K4), the skewed MMA
order off / at 2 k-blocks, and single-CTA 128x256 tiles. Every variant must meet
the same oracle tolerances as the default, on a case with ragged T/V/H tails
(H = 776: one full and one partial 512-column tile) and a chunked dU buffer.
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
import json, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import harness, synth
wl = synth.Workload("ragged", 3, 4, 28, 200, 1000, ragged=True, prompt_frac=0.1, delta_sigma=0.8, spike_rate=0.02)
out = {{}}
for chunk, dense in ((0, False), (200, False), (0, True)):
    c = harness.make_case(wl, 31, tokens=517, vocab=1300, hidden=776)
    ref = harness.run_oracle(c)
    gpu = harness.run_gpu_step(c, dz_chunk_rows=chunk, dense_backward=dense)
    out[f"{{chunk}}-{{dense}}"] = harness.compare(c, ref, gpu)
print(json.dumps(out))
"""

VARIANTS = {
    "narrow": {"RL_WIDE": "0"},
    "wide_all": {"RL_WIDE": "1"},
    "skew0": {"RL_SKEW": "0"},
    "skew2": {"RL_SKEW": "2"},
    "cta1": {"RL_CTA_GROUP": "1"},
}


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_matches_oracle(name):
    env = dict(os.environ)
    for k in ("RL_WIDE", "RL_SKEW", "RL_CTA_GROUP"):
        env.pop(k, None)
    env.update(VARIANTS[name])
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    errs = json.loads(r.stdout.strip().splitlines()[-1])
    print(name, errs)

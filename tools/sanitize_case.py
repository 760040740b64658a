"""Small end-to-end cases (tiny config, ragged tails, split phases) for compute-sanitizer.
usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import harness  # noqa: E402
import synth  # noqa: E402

for wl, kw in ((synth.CONFIGS["tiny"], {}),
               (synth.Workload("ragged", 3, 4, 28, 200, 1000, ragged=True, prompt_frac=0.1, delta_sigma=0.8,
                               spike_rate=0.02), dict(tokens=333, vocab=1000, hidden=200))):
    c = harness.make_case(wl, 1, **kw)
    ref = harness.run_oracle(c)
    gpu = harness.run_gpu_step(c)
    print(wl.name, harness.compare(c, ref, gpu))
    gpu = harness.run_gpu_step(c, dh_f32=True, accumulate_dw=True, dw_init=None)
print("sanitize cases ok")

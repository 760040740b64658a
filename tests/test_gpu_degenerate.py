"""Degenerate and boundary shapes through the whole step vs the fp64 oracle (`-m gpu`):
one token, a one-word vocabulary (logp = 0, entropy = 0 for every token), the
smallest hidden size (H = 8, below one 64-element TMA box), exact tile multiples
(no tails anywhere), an odd vocabulary (dU row padding), and more rollouts than
tokens (empty rollouts)."""
import numpy as np
import pytest

import harness
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

WL = synth.Workload("deg", 2, 2, 4, 64, 64, ragged=True, delta_sigma=0.5, spike_rate=0.0)


@pytest.mark.parametrize("tokens,vocab,hidden", [
    (1, 64, 64),          # one token (three empty rollouts)
    (37, 1, 64),          # V = 1
    (53, 300, 8),         # H = 8
    (16, 300, 16),        # H = 16
    (512, 512, 128),      # exact multiples of the 256-row / 512-column tiles and BK
    (300, 1001, 72),      # odd V, H not a multiple of 64
    (3, 7, 8),            # everything tiny
])
def test_degenerate_shapes_match_oracle(tokens, vocab, hidden):
    c = harness.make_case(WL, 51, tokens=tokens, vocab=vocab, hidden=hidden)
    ref = harness.run_oracle(c)
    for dense in (False, True):
        gpu = harness.run_gpu_step(c, dense_backward=dense)
        harness.compare(c, ref, gpu)
    if vocab == 1:
        assert np.all(np.abs(gpu["logprob"]) <= 1e-6) and np.all(np.abs(gpu["entropy"]) <= 1e-6)
        # p - onehot = 0 exactly in the oracle; fp32 exp(z - lse) leaves ~1e-7 relative
        assert np.abs(gpu["d_hidden"]).max() <= 1e-6 and np.abs(gpu["d_w_vocab"]).max() <= 1e-6


def test_more_rollouts_than_tokens():
    wl = synth.Workload("many", 4, 4, 1, 64, 128, ragged=False, delta_sigma=0.5)
    c = harness.make_case(wl, 52, tokens=9, vocab=128, hidden=64)
    assert (np.diff(c.batch.rollout_offsets) == 0).any()
    ref = harness.run_oracle(c)
    harness.compare(c, ref, harness.run_gpu_step(c))

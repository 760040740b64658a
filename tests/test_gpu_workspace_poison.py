"""Nothing the step reads from its workspace is left over from an earlier call (`-m gpu`).

The same step (sparse, dense and chunked backward; the probability cache of K1 feeding K4
is on by default) runs once on a zero-filled and once on a NaN-filled (0xFF) workspace:
every output must be bitwise the same, so no kernel reads a workspace byte that this call
did not write (e.g. the padding rows of the last 256-row dU block that K6 reads)."""
import numpy as np
import pytest

import harness
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_16144_b200 as rl  # noqa: E402

WL = synth.Workload("ragged", 3, 4, 28, 200, 1000, ragged=True, prompt_frac=0.1, delta_sigma=0.8, spike_rate=0.02)


def _step(c, fill, dense, chunk):
    b = c.batch
    T, H, V, R = b.T, b.H, b.V, len(c.adv)
    d = harness.to_device(c)
    shape = rl.make_shape(T, H, V)
    params = rl.make_params(R, b.loss_denominator)
    ws = torch.full((rl.rl_workspace_bytes(shape, R, chunk),), fill, dtype=torch.uint8, device="cuda")
    f32 = dict(dtype=torch.float32, device="cuda")
    out = dict(logprob=torch.empty(T, **f32), lse=torch.empty(T, **f32), coef=torch.empty(T, **f32),
               d_hidden=torch.empty(T, H, dtype=torch.bfloat16, device="cuda"), d_w_vocab=torch.empty(V, H, **f32))
    report = rl.new_report()
    rl.rl_policy_loss_fwd_bwd(shape, params, d["hidden"], d["w"], d["targets"], d["infer"], d["adv"], d["offsets"],
                              d["loss_mask"], report=report, logprob=out["logprob"], lse=out["lse"], coef=out["coef"],
                              d_hidden=out["d_hidden"], d_w_vocab=out["d_w_vocab"], dense_backward=dense,
                              dz_chunk_rows=chunk, workspace=ws)
    torch.cuda.synchronize()
    res = {k: v.float().cpu().numpy() for k, v in out.items()}
    res["report"] = rl.read_report(report).as_dict()
    return res


@pytest.mark.parametrize("dense,chunk", [(False, 0), (True, 0), (False, 128)], ids=["sparse", "dense", "chunked"])
def test_outputs_independent_of_workspace_contents(dense, chunk):
    c = harness.make_case(WL, 10, tokens=333, vocab=1000, hidden=200)
    clean = _step(c, 0, dense, chunk)
    poisoned = _step(c, 0xFF, dense, chunk)
    assert np.isfinite(poisoned["d_w_vocab"]).all() and np.isfinite(poisoned["d_hidden"]).all()
    for k in clean:
        if k == "report":
            assert clean[k] == poisoned[k]
        else:
            assert np.array_equal(clean[k], poisoned[k]), k

"""Sparse backward (default) vs dense backward vs the fp64 oracle (`-m gpu`).

The backward GEMMs run over the rows with coef_t != 0 only: a row with coef_t = 0
has an all-zero dU row (the derivative of the loss w.r.t. its log-prob is zero,
PAPER.md L500-504 / Eq.2: masked tokens carry no gradient), so dH of that row is
zero and it adds nothing to dW. Checks: the oracle tolerance for both paths; dH
bitwise equal between them (each dH row is computed from its own dU row in the
same order); dW equal up to fp32 summation order; masked fractions from none to
all; chunked dU buffers whose size is not a multiple of the 256-row tile.
"""
import numpy as np
import pytest

import harness
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_16144_b200 as rl  # noqa: E402

RAGGED = synth.Workload("ragged", 3, 4, 28, 200, 1000, ragged=True, prompt_frac=0.1, delta_sigma=0.8,
                        spike_rate=0.02)
HEAVY = synth.Workload("heavy", 4, 4, 40, 300, 1000, ragged=True, prompt_frac=0.3, delta_sigma=2.0,
                       spike_rate=0.05)


@pytest.mark.parametrize("wl,tokens,alpha,beta,chunk", [
    (RAGGED, 333, synth.ALPHA, synth.BETA, 0),
    (RAGGED, 333, 1e-30, 1e30, 0),            # nothing masked by Eq.2
    (HEAVY, 700, 0.9, 1.1, 0),                # most tokens masked
    (HEAVY, 700, 0.9, 1.1, 100),              # chunk not a multiple of the tile
    (HEAVY, 700, synth.ALPHA, synth.BETA, 256),
])
def test_sparse_matches_dense_and_oracle(wl, tokens, alpha, beta, chunk):
    c = harness.make_case(wl, 21, tokens=tokens, vocab=1000, hidden=200)
    c.alpha, c.beta = alpha, beta
    ref = harness.run_oracle(c)
    sp = harness.run_gpu_step(c, dz_chunk_rows=chunk)
    de = harness.run_gpu_step(c, dz_chunk_rows=chunk, dense_backward=True)
    e1 = harness.compare(c, ref, sp)
    harness.compare(c, ref, de)
    assert np.array_equal(sp["d_hidden"], de["d_hidden"])
    assert harness.rel_fro(sp["d_w_vocab"], de["d_w_vocab"]) <= 1e-5
    kept = int((sp["coef"] != 0).sum())
    print(dict(kept=kept, T=c.batch.T, **e1))
    # skipped rows carry exact zeros
    assert not sp["d_hidden"][sp["coef"] == 0].any()


def test_sparse_fp32_dh_and_accumulate():
    c = harness.make_case(HEAVY, 22, tokens=500, vocab=1000, hidden=200)
    ref = harness.run_oracle(c)
    init = torch.from_numpy(np.random.default_rng(1).standard_normal((1000, 200)).astype(np.float32)).cuda()
    sp = harness.run_gpu_step(c, dh_f32=True, accumulate_dw=True, dw_init=init, dz_chunk_rows=128)
    de = harness.run_gpu_step(c, dh_f32=True, accumulate_dw=True, dw_init=init, dz_chunk_rows=128,
                              dense_backward=True)
    assert np.array_equal(sp["d_hidden"], de["d_hidden"])
    assert harness.rel_fro(sp["d_hidden"], ref.d_hidden) <= harness.GRAD_RTOL
    got = sp["d_w_vocab"] - init.cpu().numpy().astype(np.float64)
    assert harness.rel_fro(got, ref.d_w_vocab) <= 2e-2


@pytest.mark.parametrize("accumulate", [False, True])
def test_all_rows_masked(accumulate):
    """count = 0: no GEMM tile runs; dH is zero, dW is zero (or unchanged)."""
    def corrupt(b, infer):
        b.loss_mask[:] = 0
    c = harness.make_case(RAGGED, 23, tokens=333, vocab=1000, hidden=200, corrupt=corrupt)
    init = torch.full((1000, 200), 3.0, device="cuda")
    g = harness.run_gpu_step(c, accumulate_dw=accumulate, dw_init=init, dz_chunk_rows=128, loss_denominator=1.0)
    assert not g["coef"].any()
    assert not g["d_hidden"].any()
    if accumulate:
        assert np.all(g["d_w_vocab"] == 3.0)
    else:
        assert not g["d_w_vocab"].any()


def test_sparse_split_phases_and_rl_bwd():
    """rl_bwd_ex phase by phase (compaction in the DU phase, reused by DW and DH)
    equals one rl_bwd call, and both equal the dense mask bit up to dW order."""
    c = harness.make_case(HEAVY, 24, tokens=700, vocab=1000, hidden=200)
    ref = harness.run_oracle(c)
    d = harness.to_device(c)
    b = c.batch
    T, H, V = b.T, b.H, b.V
    shape = rl.make_shape(T, H, V, 0, V)
    lse = torch.from_numpy(ref.lse.astype(np.float32)).cuda()
    coef = torch.from_numpy(ref.report.coef.astype(np.float32)).cuda()
    ws = rl.alloc_workspace(rl.rl_workspace_bytes(shape, 1))
    outs = []
    for mode in ("one", "phases", "dense"):
        dh = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
        dw = torch.empty(V, H, device="cuda")
        if mode == "one":
            rl.rl_bwd(shape, d["hidden"], d["w"], d["targets"], lse, coef, d_hidden=dh, d_w_vocab=dw, workspace=ws)
        elif mode == "phases":
            for ph in (rl.RL_BWD_DU, rl.RL_BWD_DW, rl.RL_BWD_DH):
                rl.rl_bwd_ex(shape, d["hidden"], d["w"], d["targets"], lse, coef, d_hidden=dh, d_w_vocab=dw,
                             phases=ph, workspace=ws)
        else:
            rl.rl_bwd_ex(shape, d["hidden"], d["w"], d["targets"], lse, coef, d_hidden=dh, d_w_vocab=dw,
                         phases=rl.RL_BWD_ALL | rl.RL_BWD_DENSE, workspace=ws)
        torch.cuda.synchronize()
        outs.append((dh.float().cpu().numpy(), dw.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert np.array_equal(outs[0][0], outs[2][0])
    assert harness.rel_fro(outs[0][1], outs[2][1]) <= 1e-5
    assert harness.rel_fro(outs[0][0], ref.d_hidden) <= harness.GRAD_RTOL
    assert harness.rel_fro(outs[0][1], ref.d_w_vocab) <= harness.GRAD_RTOL

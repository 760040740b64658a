"""The C-ABI library loads and exports every symbol include/rl.h declares;
host-only entry points validate arguments (CPU, no compute calls)."""
import ctypes
import os
import re

import pytest

import paper_2512_16144_b200 as rl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "rl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rl_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    return rl.load_library()


def test_every_declared_symbol_is_exported(lib):
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(rl.EXPORTED)


def test_struct_layouts_match_header(lib):
    assert ctypes.sizeof(rl.rl_lm_shape) == 56
    assert ctypes.sizeof(rl.rl_loss_params) == 40
    assert ctypes.sizeof(rl.rl_loss_report) == 48
    assert ctypes.sizeof(rl.rl_loss_outputs) == 104
    assert ctypes.sizeof(rl.rl_nvls_reduce) == 96
    assert lib.rl_abi_version() == 3


def test_status_strings(lib):
    assert lib.rl_status_string(0) == b"RL_OK"
    assert lib.rl_status_string(5) == b"RL_ERR_WORKSPACE"


def test_workspace_bytes_host_only(lib):
    s = rl.make_shape(16384, 4096, 151552)
    n = rl.rl_workspace_bytes(s, 16)
    # partials (592 tiles x T x 16 B) + dU (T x V bf16) dominate
    assert n >= 592 * 16384 * 16 + 16384 * 151552 * 2
    assert rl.rl_workspace_bytes(s, 16, 1024) < n
    bad = rl.make_shape(16, 60, 100)
    assert rl.rl_workspace_bytes(bad, 1) == 0


def test_host_validation_before_any_device_work(lib):
    st = lib.rl_group_advantages(ctypes.c_void_p(16), 4, 1, ctypes.c_void_p(16), None)
    assert st == 1 and b"group_size" in lib.rl_last_error_message()
    p = rl.make_params(4, 0.0)
    st = lib.rl_loss_coef(ctypes.byref(p), 10, 100, *([ctypes.c_void_p(16)] * 10), None, 0, None)
    assert st == 1 and b"loss_denominator" in lib.rl_last_error_message()
    p = rl.make_params(4, 10.0, alpha=0.6, beta=0.9)
    st = lib.rl_loss_coef(ctypes.byref(p), 10, 100, *([ctypes.c_void_p(16)] * 10), None, 0, None)
    assert st == 1


def test_fault_counters_raise_on_check():
    """Data faults are counted on the device and neutralised; the binding turns
    non-zero counters into RLDataFault when asked (SURVEY §8(b) error split)."""
    import paper_2512_16144_b200 as rl
    ok = rl.rl_loss_report(loss=-0.5, kept_tokens=10)
    assert rl.check_faults(ok) is ok
    for key in rl.FAULT_COUNTERS:
        bad = rl.rl_loss_report(**{key: 2})
        with pytest.raises(rl.RLDataFault, match=key):
            rl.check_faults(bad)


def test_moe_helpers_validate_on_the_host(lib):
    """rl_fold_gamma / rl_expert_load reject bad sizes and misaligned pointers before any
    device work (include/rl.h), so these run without a GPU."""
    P = ctypes.c_void_p
    assert lib.rl_fold_gamma(P(16), P(16), 4, 12, P(16), None) == 2          # K % 8 != 0
    assert b"multiple of 8" in lib.rl_last_error_message()
    assert lib.rl_fold_gamma(P(16), P(16), -1, 64, P(16), None) == 2         # rows < 0
    assert lib.rl_fold_gamma(P(18), P(16), 4, 64, P(16), None) == 1          # w not 16-byte aligned
    assert b"aligned" in lib.rl_last_error_message()
    assert lib.rl_fold_gamma(None, P(16), 4, 64, P(16), None) != 0           # null pointer
    assert lib.rl_fold_gamma(P(16), P(16), 0, 64, P(16), None) == 0          # nothing to do
    assert lib.rl_expert_load(P(16), 0, 10, P(16), None) == 2                # no groups
    assert lib.rl_expert_load(None, 4, 10, P(16), None) != 0


def test_split_rollout_calls_validate_on_the_host(lib):
    P = ctypes.c_void_p
    p = rl.make_params(4, 10.0, variant="gspo")
    args = [P(16)] * 6   # logprob, infer, targets, adv, offsets, loss_mask
    # GSPO over split rollouts needs the log-ratio sums and counts
    st = lib.rl_loss_coef_ex(ctypes.byref(p), 10, 100, *args, P(16), None, None, P(16), None, None, P(16), P(16),
                             4096, None)
    assert st == 1 and b"GSPO" in lib.rl_last_error_message()
    p = rl.make_params(4, 10.0)
    st = lib.rl_loss_coef_ex(ctypes.byref(p), 10, 100, *args, None, None, None, P(16), None, None, P(16), P(16),
                             4096, None)
    assert st != 0                                                     # rollout_kmin is required
    st = lib.rl_rollout_stats(ctypes.byref(p), 10, 100, P(16), P(16), P(16), P(16), None, None, P(16), P(16), None)
    assert st != 0                                                     # kmin output is required
    p = rl.make_params(4, 0.0)
    st = lib.rl_rollout_stats(ctypes.byref(p), 10, 100, P(16), P(16), P(16), P(16), None, P(16), P(16), P(16), None)
    assert st == 1                                                     # D <= 0

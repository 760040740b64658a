"""Python binding of librl (include/rl.h): argument marshalling only.

Every function keeps the C name and forwards torch tensors' device pointers and
the current CUDA stream to the C ABI; every step of the path runs in librl's
sm_100a kernels. There is no CPU or PyTorch fallback: importing works without a
GPU (so the ABI can be inspected), but every compute call needs the built
librl.so and a B200, and raises RLError otherwise.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RL_LIBRARY") or os.path.join(_HERE, "librl.so")  # RL_LIBRARY: another build (A/B runs)

RL_OK = 0
STATUS_NAMES = {0: "RL_OK", 1: "RL_ERR_INVALID_ARGUMENT", 2: "RL_ERR_SHAPE", 3: "RL_ERR_UNSUPPORTED",
                4: "RL_ERR_CUDA", 5: "RL_ERR_WORKSPACE", 6: "RL_ERR_ALIGNMENT"}

# paper constants
ALPHA, BETA, GUARD = 0.5, 5.0, 1e-5


class RLError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class rl_lm_shape(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int64), ("H", ctypes.c_int64), ("V_local", ctypes.c_int64),
                ("vocab_offset", ctypes.c_int64), ("V_global", ctypes.c_int64),
                ("inv_temperature", ctypes.c_float), ("_pad", ctypes.c_int32),
                ("inv_temperature_rows", ctypes.c_void_p)]


class rl_loss_params(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_float), ("beta", ctypes.c_float), ("guard_threshold", ctypes.c_float),
                ("num_rollouts", ctypes.c_int32), ("loss_denominator", ctypes.c_double),
                ("variant", ctypes.c_int32), ("kl_set", ctypes.c_int32), ("kl_tau", ctypes.c_float),
                ("_pad", ctypes.c_int32)]


LOSS_VARIANTS = {"icepop": 0, "cispo": 1, "gspo": 2}   # rl_loss_variant
KL_SETS = {"masked": 0, "unmasked": 1, "all": 2}        # rl_kl_set


class rl_loss_report(ctypes.Structure):
    _fields_ = [("loss", ctypes.c_double), ("mismatch_kl_sum", ctypes.c_double),
                ("kept_tokens", ctypes.c_uint32), ("masked_low", ctypes.c_uint32),
                ("masked_high", ctypes.c_uint32), ("guarded_rollouts", ctypes.c_uint32),
                ("guarded_tokens", ctypes.c_uint32), ("nonfinite_inputs", ctypes.c_uint32),
                ("bad_targets", ctypes.c_uint32), ("bad_offsets", ctypes.c_uint32)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


NVLS_MAX_RANKS = 8


class rl_nvls_reduce(ctypes.Structure):
    _fields_ = [("multicast", ctypes.c_void_p), ("flags", ctypes.c_void_p * NVLS_MAX_RANKS),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("epoch", ctypes.c_uint32),
                ("lag", ctypes.c_int32), ("mode", ctypes.c_int32), ("_pad", ctypes.c_int32)]


RL_NVLS_ALL_REDUCE, RL_NVLS_REDUCE_SCATTER = 0, 1


class rl_loss_outputs(ctypes.Structure):
    _fields_ = [("report", ctypes.c_void_p), ("logprob", ctypes.c_void_p), ("entropy", ctypes.c_void_p),
                ("lse", ctypes.c_void_p), ("coef", ctypes.c_void_p), ("token_keep", ctypes.c_void_p),
                ("rollout_guarded", ctypes.c_void_p), ("d_hidden", ctypes.c_void_p),
                ("d_hidden_f32", ctypes.c_void_p), ("d_w_vocab", ctypes.c_void_p),
                ("accumulate_dw", ctypes.c_int32), ("dense_backward", ctypes.c_int32),
                ("d_w_vocab_nvls", ctypes.POINTER(rl_nvls_reduce)), ("dz_chunk_rows", ctypes.c_int64)]


class rl_kernel_time(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("ms", ctypes.c_float)]


KERNEL_NAMES = {0: "K0_group_adv", 1: "K1_fwd_gemm_lse", 2: "K2_merge", 3: "K3_loss_coef", 4: "K3b_finalize",
                5: "K4_bwd_dz_gemm", 6: "K5_dh_gemm", 7: "K6_dw_gemm", 8: "memset", 9: "NS_gemm", 10: "NS_aux",
                11: "grouped_gemm", 12: "compact", 13: "K4_dz_from_cache"}

REPORT_BYTES = ctypes.sizeof(rl_loss_report)
assert REPORT_BYTES == 48

_P = ctypes.c_void_p
_SIGS = {
    "rl_group_advantages": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, _P, _P]),
    "rl_logprob_fwd": (ctypes.c_int, [ctypes.POINTER(rl_lm_shape), _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "rl_policy_loss_fwd_bwd": (ctypes.c_int, [ctypes.POINTER(rl_lm_shape), ctypes.POINTER(rl_loss_params), _P, _P,
                                              _P, _P, _P, _P, _P, ctypes.POINTER(rl_loss_outputs), _P,
                                              ctypes.c_size_t, _P]),
    "rl_policy_loss_fwd_bwd_hostio": (ctypes.c_int, [ctypes.POINTER(rl_lm_shape), ctypes.POINTER(rl_loss_params),
                                                     ctypes.c_int32, _P, _P, _P, _P, _P, _P, _P,
                                                     ctypes.POINTER(rl_loss_outputs),
                                                     ctypes.POINTER(rl_loss_report), _P, ctypes.c_size_t, _P]),
    "rl_fwd_partials": (ctypes.c_int, [ctypes.POINTER(rl_lm_shape), _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "rl_fwd_partials_ex": (ctypes.c_int, [ctypes.POINTER(rl_lm_shape), _P, _P, _P, _P, ctypes.c_int32, _P,
                                          ctypes.c_size_t, _P]),
    "rl_merge_partials": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _P, _P, _P, _P]),
    "rl_loss_coef": (ctypes.c_int, [ctypes.POINTER(rl_loss_params), ctypes.c_int64, ctypes.c_int64, _P, _P, _P, _P,
                                    _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "rl_rollout_stats": (ctypes.c_int, [ctypes.POINTER(rl_loss_params), ctypes.c_int64, ctypes.c_int64, _P, _P, _P,
                                        _P, _P, _P, _P, _P, _P]),
    "rl_loss_coef_ex": (ctypes.c_int, [ctypes.POINTER(rl_loss_params), ctypes.c_int64, ctypes.c_int64, _P, _P, _P,
                                       _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "rl_bwd": (ctypes.c_int, [ctypes.POINTER(rl_lm_shape), _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_int32,
                              ctypes.c_int64, _P, ctypes.c_size_t, _P]),
    "rl_bwd_ex": (ctypes.c_int, [ctypes.POINTER(rl_lm_shape), _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_int32,
                                 ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(rl_nvls_reduce),
                                 ctypes.POINTER(rl_nvls_reduce), _P, ctypes.c_size_t, _P]),
    "rl_nvls_flag_count": (ctypes.c_int64, [ctypes.POINTER(rl_lm_shape), ctypes.c_int32]),
    "rl_nvls_shard_rows": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int32]),
    "rl_newton_schulz": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, _P, _P,
                                        ctypes.c_size_t, _P]),
    "rl_newton_schulz_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int64]),
    "rl_ns_shard_sumsq": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_int64, _P, _P, ctypes.c_size_t, _P]),
    "rl_ns_shard_gram": (ctypes.c_int, [ctypes.c_int32, _P, _P, ctypes.c_int64, ctypes.c_int64, _P, _P,
                                        ctypes.c_size_t, _P]),
    "rl_ns_shard_apply": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, _P, ctypes.c_int64, ctypes.c_int64, _P,
                                         _P, ctypes.c_size_t, _P]),
    "rl_muon_step": (ctypes.c_int, [_P, _P, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_float, ctypes.c_float,
                                    ctypes.c_float, ctypes.c_int32, ctypes.c_int32, _P, ctypes.c_size_t, _P]),
    "rl_muon_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int64]),
    "rl_grouped_gemm": (ctypes.c_int, [_P, _P, _P, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                       _P, _P, _P]),
    "rl_rms_inv": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_int64, ctypes.c_float, _P, _P]),
    "rl_fold_gamma": (ctypes.c_int, [_P, _P, ctypes.c_int64, ctypes.c_int64, _P, _P]),
    "rl_expert_load": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _P, _P]),
    "rl_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(rl_lm_shape), ctypes.c_int32, ctypes.c_int64]),
    "rl_workspace_bytes_hostio": (ctypes.c_size_t, [ctypes.POINTER(rl_lm_shape), ctypes.c_int32, ctypes.c_int64]),
    "rl_default_dz_chunk_rows": (ctypes.c_int64, [ctypes.POINTER(rl_lm_shape)]),
    "rl_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "rl_last_error_message": (ctypes.c_char_p, []),
    "rl_abi_version": (ctypes.c_int32, []),
    "rl_last_launch_count": (ctypes.c_int32, []),
    "rl_profile_enable": (ctypes.c_int, [ctypes.c_int32]),
    "rl_profile_read": (ctypes.c_int32, [_P, ctypes.c_int32]),
}
EXPORTED = tuple(_SIGS)

_lib = None


def load_library(path: str | None = None) -> ctypes.CDLL:
    """dlopen librl.so (in-tree). Raises if it has not been built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RLError(3, f"{p} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(p)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def _check(status: int):
    if status != RL_OK:
        msg = load_library().rl_last_error_message().decode(errors="replace")
        raise RLError(status, msg)


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise RLError(1, "expected a CUDA tensor")
    if not t.is_contiguous():
        raise RLError(1, "expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def make_shape(T, H, V_local, vocab_offset=0, V_global=None, inv_temperature=1.0,
               inv_temperature_rows=None) -> rl_lm_shape:
    """`inv_temperature_rows`: optional fp32 CUDA tensor [T] of per-token 1/tau (R20);
    the caller keeps it alive while the shape is in use."""
    if inv_temperature_rows is not None:
        if not inv_temperature_rows.is_cuda or inv_temperature_rows.dtype != torch.float32 \
                or inv_temperature_rows.numel() < int(T) or not inv_temperature_rows.is_contiguous():
            raise RLError(1, "inv_temperature_rows must be a contiguous fp32 CUDA tensor with >= T elements")
    return rl_lm_shape(int(T), int(H), int(V_local), int(vocab_offset),
                       int(V_local + vocab_offset if V_global is None else V_global), float(inv_temperature), 0,
                       inv_temperature_rows.data_ptr() if inv_temperature_rows is not None else None)


def make_params(num_rollouts, loss_denominator, alpha=ALPHA, beta=BETA, guard_threshold=GUARD,
                variant="icepop", kl_tau=0.0, kl_set="masked") -> rl_loss_params:
    v = LOSS_VARIANTS[variant] if isinstance(variant, str) else int(variant)
    ks = KL_SETS[kl_set] if isinstance(kl_set, str) else int(kl_set)
    return rl_loss_params(float(alpha), float(beta), float(guard_threshold), int(num_rollouts),
                          float(loss_denominator), v, ks, float(kl_tau), 0)


def _bf16(t: torch.Tensor | None, name: str) -> torch.Tensor | None:
    if t is not None and t.dtype not in (torch.bfloat16, torch.int16, torch.uint16):
        raise RLError(1, f"{name} must be bf16")
    return t


# ---------------------------------------------------------------- C names
def rl_workspace_bytes(shape: rl_lm_shape, num_rollouts: int = 1, dz_chunk_rows: int = 0) -> int:
    return int(load_library().rl_workspace_bytes(ctypes.byref(shape), int(num_rollouts), int(dz_chunk_rows)))


def rl_workspace_bytes_hostio(shape: rl_lm_shape, num_rollouts: int, dz_chunk_rows: int = 0) -> int:
    return int(load_library().rl_workspace_bytes_hostio(ctypes.byref(shape), int(num_rollouts), int(dz_chunk_rows)))


def alloc_workspace(nbytes: int, device=None) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device or "cuda")


def rl_group_advantages(rewards: torch.Tensor, group_size: int, advantages: torch.Tensor | None = None,
                        stream=None) -> torch.Tensor:
    """S0: A = S - mean_G(S). rewards: [Np*G] fp32 group-major."""
    r = rewards.reshape(-1)
    if advantages is None:
        advantages = torch.empty_like(r)
    if r.numel() % group_size:
        raise RLError(2, "len(rewards) must be a multiple of group_size")
    _check(load_library().rl_group_advantages(_ptr(r), r.numel() // group_size, int(group_size),
                                              _ptr(advantages), _stream(stream)))
    return advantages


def rl_logprob_fwd(shape: rl_lm_shape, hidden, w_vocab, targets, logprob, entropy=None, lse=None,
                   workspace=None, stream=None):
    """S1+S2: logprob/entropy/lse of the targets, logits only in TMEM."""
    ws = workspace if workspace is not None else alloc_workspace(rl_workspace_bytes(shape), hidden.device)
    _check(load_library().rl_logprob_fwd(ctypes.byref(shape), _ptr(_bf16(hidden, "hidden")),
                                         _ptr(_bf16(w_vocab, "w_vocab")), _ptr(targets), _ptr(logprob),
                                         _ptr(entropy), _ptr(lse), _ptr(ws), ws.numel(), _stream(stream)))


def _outputs(report, logprob, entropy=None, lse=None, coef=None, token_keep=None, rollout_guarded=None,
             d_hidden=None, d_hidden_f32=None, d_w_vocab=None, accumulate_dw=False,
             d_w_vocab_nvls=None, dz_chunk_rows=0, dense_backward=False) -> rl_loss_outputs:
    return rl_loss_outputs(_ptr(report), _ptr(logprob), _ptr(entropy), _ptr(lse), _ptr(coef), _ptr(token_keep),
                           _ptr(rollout_guarded), _ptr(d_hidden), _ptr(d_hidden_f32), _ptr(d_w_vocab),
                           1 if accumulate_dw else 0, 1 if dense_backward else 0,
                           ctypes.pointer(d_w_vocab_nvls) if d_w_vocab_nvls is not None else None,
                           int(dz_chunk_rows))


def rl_policy_loss_fwd_bwd(shape: rl_lm_shape, params: rl_loss_params, hidden, w_vocab, targets, infer_logprobs,
                           rollout_adv, rollout_offsets, loss_mask=None, *, report, logprob, entropy=None,
                           lse=None, coef=None, token_keep=None, rollout_guarded=None, d_hidden=None,
                           d_hidden_f32=None, d_w_vocab=None, accumulate_dw=False, d_w_vocab_nvls=None,
                           dz_chunk_rows=0, dense_backward=False, workspace=None, stream=None):
    """S0..S6 on one rank (see include/rl.h). `report` is a [48] uint8 CUDA tensor.
    `d_w_vocab_nvls` (rl_nvls_reduce) all-reduces d_w_vocab over NVLS in the K6 epilogue.
    `dense_backward` runs the backward GEMMs over all rows instead of the coef != 0 rows."""
    ws = workspace if workspace is not None else alloc_workspace(
        rl_workspace_bytes(shape, params.num_rollouts, dz_chunk_rows), w_vocab.device)
    out = _outputs(report, logprob, entropy, lse, coef, token_keep, rollout_guarded, d_hidden, d_hidden_f32,
                   d_w_vocab, accumulate_dw, d_w_vocab_nvls, dz_chunk_rows, dense_backward)
    _check(load_library().rl_policy_loss_fwd_bwd(
        ctypes.byref(shape), ctypes.byref(params), _ptr(_bf16(hidden, "hidden")), _ptr(_bf16(w_vocab, "w_vocab")),
        _ptr(targets), _ptr(infer_logprobs), _ptr(rollout_adv), _ptr(rollout_offsets), _ptr(loss_mask),
        ctypes.byref(out), _ptr(ws), ws.numel(), _stream(stream)))


def rl_policy_loss_fwd_bwd_hostio(shape: rl_lm_shape, params: rl_loss_params, group_size: int, hidden_host,
                                  w_vocab, targets_host, infer_host, rewards_host, offsets_host,
                                  loss_mask_host=None, *, report, d_hidden=None, d_hidden_f32=None,
                                  d_w_vocab=None, accumulate_dw=False, d_w_vocab_nvls=None, dz_chunk_rows=0,
                                  dense_backward=False, workspace=None, stream=None) -> rl_loss_report:
    """The same step with per-step inputs in (pinned) host tensors; returns the report."""
    ws = workspace if workspace is not None else alloc_workspace(
        rl_workspace_bytes_hostio(shape, params.num_rollouts, dz_chunk_rows), w_vocab.device)

    def hp(t):
        if t is None:
            return None
        if t.is_cuda or not t.is_contiguous():
            raise RLError(1, "host inputs must be contiguous CPU tensors")
        return ctypes.c_void_p(t.data_ptr())

    out = _outputs(report, None, d_hidden=d_hidden, d_hidden_f32=d_hidden_f32, d_w_vocab=d_w_vocab,
                   accumulate_dw=accumulate_dw, d_w_vocab_nvls=d_w_vocab_nvls, dz_chunk_rows=dz_chunk_rows,
                   dense_backward=dense_backward)
    rep = rl_loss_report()
    _check(load_library().rl_policy_loss_fwd_bwd_hostio(
        ctypes.byref(shape), ctypes.byref(params), int(group_size), hp(hidden_host), _ptr(w_vocab),
        hp(targets_host), hp(infer_host), hp(rewards_host), hp(offsets_host), hp(loss_mask_host),
        ctypes.byref(out), ctypes.byref(rep), _ptr(ws), ws.numel(), _stream(stream)))
    return rep


def rl_fwd_partials(shape: rl_lm_shape, hidden, w_vocab, targets, partials, workspace=None, stream=None):
    """S1 on a vocab shard -> one (m, s, u, z_target) float4 per row ([T, 4] fp32)."""
    ws = workspace if workspace is not None else alloc_workspace(rl_workspace_bytes(shape), hidden.device)
    _check(load_library().rl_fwd_partials(ctypes.byref(shape), _ptr(_bf16(hidden, "hidden")),
                                          _ptr(_bf16(w_vocab, "w_vocab")), _ptr(targets), _ptr(partials),
                                          _ptr(ws), ws.numel(), _stream(stream)))


def rl_fwd_partials_ex(shape: rl_lm_shape, hidden, w_vocab, targets, partials, flags: int = 0, workspace=None,
                       stream=None):
    """rl_fwd_partials; flags = RL_FWD_CACHE also fills the probability cache in `workspace` for a
    later rl_bwd_ex(phases | RL_BWD_FROM_CACHE) on the same inputs and workspace."""
    ws = workspace if workspace is not None else alloc_workspace(rl_workspace_bytes(shape), hidden.device)
    _check(load_library().rl_fwd_partials_ex(ctypes.byref(shape), _ptr(_bf16(hidden, "hidden")),
                                             _ptr(_bf16(w_vocab, "w_vocab")), _ptr(targets), _ptr(partials),
                                             int(flags), _ptr(ws), ws.numel(), _stream(stream)))


def rl_merge_partials(partials, n_parts: int, T: int, logprob, entropy=None, lse=None, stream=None):
    """S2: merge [n_parts, T, 4] partials (index order) into logprob / entropy / lse."""
    _check(load_library().rl_merge_partials(_ptr(partials), int(n_parts), int(T), _ptr(logprob), _ptr(entropy),
                                            _ptr(lse), _stream(stream)))


def rl_loss_coef(params: rl_loss_params, T: int, V_global: int, logprob, infer_logprobs, targets, rollout_adv,
                 rollout_offsets, loss_mask, coef, token_keep=None, rollout_guarded=None, *, report,
                 workspace=None, stream=None):
    """S3: Eq.1/Eq.2/guard -> coef, keep, guarded, report."""
    ws = workspace if workspace is not None else alloc_workspace(48 * max(1, params.num_rollouts), coef.device)
    _check(load_library().rl_loss_coef(ctypes.byref(params), int(T), int(V_global), _ptr(logprob),
                                       _ptr(infer_logprobs), _ptr(targets), _ptr(rollout_adv),
                                       _ptr(rollout_offsets), _ptr(loss_mask), _ptr(coef), _ptr(token_keep),
                                       _ptr(rollout_guarded), _ptr(report), _ptr(ws), ws.numel(), _stream(stream)))


def rl_rollout_stats(params: rl_loss_params, T: int, V_global: int, logprob, infer_logprobs, targets,
                     rollout_offsets, loss_mask, kmin=None, logratio_sum=None, n_valid=None, stream=None):
    """Per local rollout (min k, sum log k, valid tokens) for rollouts split across ranks;
    reduce them over the ranks (MIN, SUM, SUM), then call rl_loss_coef_ex."""
    R = params.num_rollouts
    dev = rollout_offsets.device
    kmin = kmin if kmin is not None else torch.empty(R, dtype=torch.float32, device=dev)
    logratio_sum = logratio_sum if logratio_sum is not None else torch.empty(R, dtype=torch.float64, device=dev)
    n_valid = n_valid if n_valid is not None else torch.empty(R, dtype=torch.int32, device=dev)
    _check(load_library().rl_rollout_stats(ctypes.byref(params), int(T), int(V_global), _ptr(logprob),
                                           _ptr(infer_logprobs), _ptr(targets), _ptr(rollout_offsets),
                                           _ptr(loss_mask), _ptr(kmin), _ptr(logratio_sum), _ptr(n_valid),
                                           _stream(stream)))
    return kmin, logratio_sum, n_valid


def rl_loss_coef_ex(params: rl_loss_params, T: int, V_global: int, logprob, infer_logprobs, targets, rollout_adv,
                    rollout_offsets, loss_mask, rollout_kmin, rollout_logratio_sum, rollout_n_valid, coef,
                    token_keep=None, rollout_guarded=None, *, report, workspace=None, stream=None):
    """S3 with rollout statistics reduced over the ranks that share split rollouts."""
    ws = workspace if workspace is not None else alloc_workspace(48 * max(1, params.num_rollouts), coef.device)
    _check(load_library().rl_loss_coef_ex(ctypes.byref(params), int(T), int(V_global), _ptr(logprob),
                                          _ptr(infer_logprobs), _ptr(targets), _ptr(rollout_adv),
                                          _ptr(rollout_offsets), _ptr(loss_mask), _ptr(rollout_kmin),
                                          _ptr(rollout_logratio_sum), _ptr(rollout_n_valid), _ptr(coef),
                                          _ptr(token_keep), _ptr(rollout_guarded), _ptr(report), _ptr(ws),
                                          ws.numel(), _stream(stream)))


def rl_bwd(shape: rl_lm_shape, hidden, w_vocab, targets, lse, coef, d_hidden=None, d_hidden_f32=None,
           d_w_vocab=None, accumulate_dw=False, dz_chunk_rows=0, workspace=None, stream=None):
    """S4-S6 on a vocab shard."""
    ws = workspace if workspace is not None else alloc_workspace(
        rl_workspace_bytes(shape, 1, dz_chunk_rows), w_vocab.device)
    _check(load_library().rl_bwd(ctypes.byref(shape), _ptr(hidden), _ptr(w_vocab), _ptr(targets), _ptr(lse),
                                 _ptr(coef), _ptr(d_hidden), _ptr(d_hidden_f32), _ptr(d_w_vocab),
                                 1 if accumulate_dw else 0, int(dz_chunk_rows), _ptr(ws), ws.numel(),
                                 _stream(stream)))


def rl_profile_enable(enable: bool = True):
    load_library().rl_profile_enable(1 if enable else 0)


def rl_profile_read(cap: int = 4096) -> list:
    """[(kernel_name, ms), ...] for launches recorded since the last read (waits on their events)."""
    buf = (rl_kernel_time * cap)()
    n = load_library().rl_profile_read(ctypes.cast(buf, ctypes.c_void_p), cap)
    return [(KERNEL_NAMES.get(buf[i].kernel, str(buf[i].kernel)), float(buf[i].ms)) for i in range(min(n, cap))]


RL_BWD_DU, RL_BWD_DW, RL_BWD_DH, RL_BWD_ALL, RL_BWD_DENSE, RL_BWD_FROM_CACHE = 1, 2, 4, 7, 8, 16
RL_FWD_CACHE = 1


def rl_bwd_ex(shape: rl_lm_shape, hidden, w_vocab, targets, lse, coef, d_hidden=None, d_hidden_f32=None,
              d_w_vocab=None, accumulate_dw=False, dz_chunk_rows=0, phases=RL_BWD_ALL, max_sms=0, dw_nvls=None,
              dh_nvls=None, workspace=None, stream=None):
    """S4-S6 with a phase mask (RL_BWD_DU | RL_BWD_DW | RL_BWD_DH) and an SM budget."""
    ws = workspace if workspace is not None else alloc_workspace(
        rl_workspace_bytes(shape, 1, dz_chunk_rows), w_vocab.device)
    _check(load_library().rl_bwd_ex(ctypes.byref(shape), _ptr(hidden), _ptr(w_vocab), _ptr(targets), _ptr(lse),
                                    _ptr(coef), _ptr(d_hidden), _ptr(d_hidden_f32), _ptr(d_w_vocab),
                                    1 if accumulate_dw else 0, int(dz_chunk_rows), int(phases), int(max_sms),
                                    ctypes.pointer(dw_nvls) if dw_nvls is not None else None,
                                    ctypes.pointer(dh_nvls) if dh_nvls is not None else None,
                                    _ptr(ws), ws.numel(), _stream(stream)))


def rl_nvls_shard_rows(rows: int, world: int) -> int:
    """Rows each rank owns in the reduce-scatter mode (whole 32-row slabs)."""
    return int(load_library().rl_nvls_shard_rows(int(rows), int(world)))


def rl_nvls_flag_count(shape: rl_lm_shape, which: int) -> int:
    """Flag entries for an NVLS reduction of d_w_vocab (0) or d_hidden_f32 (1)."""
    return int(load_library().rl_nvls_flag_count(ctypes.byref(shape), int(which)))


def rl_newton_schulz(g: torch.Tensor, steps: int = 5, out: torch.Tensor | None = None, workspace=None,
                     stream=None) -> torch.Tensor:
    """Muon's Newton-Schulz orthogonalisation of an fp32 [M, N] matrix -> bf16 [M, N]."""
    M, N = g.shape
    if out is None:
        out = torch.empty(M, N, dtype=torch.bfloat16, device=g.device)
    ws = workspace if workspace is not None else alloc_workspace(
        load_library().rl_newton_schulz_workspace_bytes(M, N), g.device)
    _check(load_library().rl_newton_schulz(_ptr(g), M, N, int(steps), _ptr(out), _ptr(ws), ws.numel(),
                                           _stream(stream)))
    return out


def rl_ns_shard_sumsq(g: torch.Tensor, sumsq: torch.Tensor, workspace, stream=None):
    """Row-sharded Newton-Schulz, phase 0: sumsq[0] = sum of g^2 over this shard (fp64)."""
    M, N = g.shape
    _check(load_library().rl_ns_shard_sumsq(_ptr(g), M, N, _ptr(sumsq), _ptr(workspace), workspace.numel(),
                                            _stream(stream)))


def rl_ns_shard_gram(j: int, g: torch.Tensor, sumsq: torch.Tensor, gram: torch.Tensor, workspace, stream=None):
    """Iteration j: (j = 0: X_0 from g and the global sumsq) gram = X_r^T X_r (fp32 [N, N])."""
    M, N = g.shape
    _check(load_library().rl_ns_shard_gram(int(j), _ptr(g), _ptr(sumsq), M, N, _ptr(gram), _ptr(workspace),
                                           workspace.numel(), _stream(stream)))


def rl_ns_shard_apply(j: int, steps: int, gram: torch.Tensor, M_local: int, N: int, out: torch.Tensor | None,
                      workspace, stream=None):
    """Iteration j with the all-reduced gram: X_r <- X_r (aI + bA + cA^2); out on the last j."""
    _check(load_library().rl_ns_shard_apply(int(j), int(steps), _ptr(gram), int(M_local), int(N), _ptr(out),
                                            _ptr(workspace), workspace.numel(), _stream(stream)))


def rl_muon_step(theta: torch.Tensor, grad: torch.Tensor, momentum: torch.Tensor, lr: float, mu: float = 0.95,
                 weight_decay: float = 0.0, nesterov: bool = True, steps: int = 5, workspace=None, stream=None):
    """One Muon update of an fp32 [M, N] parameter (theta and momentum in place)."""
    M, N = theta.shape
    ws = workspace if workspace is not None else alloc_workspace(load_library().rl_muon_workspace_bytes(M, N),
                                                                 theta.device)
    _check(load_library().rl_muon_step(_ptr(theta), _ptr(grad), _ptr(momentum), M, N, float(lr), float(mu),
                                       float(weight_decay), 1 if nesterov else 0, int(steps), _ptr(ws), ws.numel(),
                                       _stream(stream)))


def rl_grouped_gemm(a: torch.Tensor, b: torch.Tensor, offsets: torch.Tensor, out: torch.Tensor | None = None,
                    row_scale: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """MoE grouped GEMM: out[r] = row_scale[r] * (a[r] @ b[g(r)].T), int32 group offsets [G+1] on the device."""
    rows, K = a.shape
    G, N, K2 = b.shape
    if K2 != K or offsets.numel() != G + 1 or offsets.dtype != torch.int32:
        raise RLError(2, "shapes: a [rows, K], b [G, N, K], offsets int32 [G + 1]")
    if out is None:
        out = torch.empty(rows, N, dtype=torch.bfloat16, device=a.device)
    _check(load_library().rl_grouped_gemm(_ptr(_bf16(a, "a")), _ptr(_bf16(b, "b")), _ptr(offsets), G, rows, N, K,
                                          _ptr(row_scale), _ptr(out), _stream(stream)))
    return out


def rl_rms_inv(x: torch.Tensor, eps: float = 1e-6, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """1 / sqrt(mean(x^2) + eps) per row of a bf16 [rows, K] matrix."""
    rows, K = x.shape
    if out is None:
        out = torch.empty(rows, dtype=torch.float32, device=x.device)
    _check(load_library().rl_rms_inv(_ptr(_bf16(x, "x")), rows, K, float(eps), _ptr(out), _stream(stream)))
    return out


def rl_fold_gamma(w: torch.Tensor, gamma: torch.Tensor, out: torch.Tensor | None = None,
                  stream=None) -> torch.Tensor:
    """bf16(w * gamma) along the last dim of a bf16 [..., K] weight (RMSNorm gamma folded in)."""
    K = w.shape[-1]
    if out is None:
        out = torch.empty_like(w)
    if gamma.dtype != torch.float32 or gamma.numel() != K:
        raise RLError(1, "gamma must be fp32 [K]")
    _check(load_library().rl_fold_gamma(_ptr(_bf16(w, "w")), _ptr(gamma), w.numel() // K, K, _ptr(out),
                                        _stream(stream)))
    return out


def rl_expert_load(offsets: torch.Tensor, rows: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """[max load, mean load, MaxViolation] (fp32, device) from int32 group offsets [G + 1]."""
    if offsets.dtype != torch.int32:
        raise RLError(1, "offsets must be int32")
    if out is None:
        out = torch.empty(3, dtype=torch.float32, device=offsets.device)
    _check(load_library().rl_expert_load(_ptr(offsets), offsets.numel() - 1, int(rows), _ptr(out), _stream(stream)))
    return out


def rl_last_launch_count() -> int:
    return int(load_library().rl_last_launch_count())


FAULT_COUNTERS = ("nonfinite_inputs", "bad_targets", "bad_offsets")


class RLDataFault(RuntimeError):
    """Data-dependent input faults that librl counted and neutralised on the device
    (include/rl.h: the token or rollout was treated as masked, coef 0)."""

    def __init__(self, report: "rl_loss_report"):
        self.report = report
        bad = ", ".join(f"{k}={getattr(report, k)}" for k in FAULT_COUNTERS if getattr(report, k))
        super().__init__(f"librl counted input faults: {bad}")


def check_faults(report: "rl_loss_report") -> "rl_loss_report":
    """Raise RLDataFault if any fault counter of a host report is non-zero."""
    if any(getattr(report, k) for k in FAULT_COUNTERS):
        raise RLDataFault(report)
    return report


def read_report(report: torch.Tensor, check: bool = False) -> rl_loss_report:
    """Copy a device report ([48] uint8) to the host (synchronises). With check=True,
    raise RLDataFault if the step counted non-finite log-probs, bad targets or bad
    offsets (they were neutralised, but the batch is malformed)."""
    b = bytes(report.cpu().numpy().tobytes())
    rep = rl_loss_report.from_buffer_copy(b)
    return check_faults(rep) if check else rep


def new_report(device=None) -> torch.Tensor:
    return torch.zeros(REPORT_BYTES, dtype=torch.uint8, device=device or "cuda")

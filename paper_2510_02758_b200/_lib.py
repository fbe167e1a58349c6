"""ctypes binding of the C-ABI library ``_tf_b200.so`` (include/tokenflow_b200.h).

There is no CPU fallback: importing this module fails loudly when the
library is missing, and every entry point raises when the CUDA side reports
an error.  Status codes map to the reference's exceptions:
TF_EINVAL -> ValueError, TF_ENOMEM -> MemoryError (kvstore.py:243),
TF_EIO -> InvariantError (engine.py:91-92).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_tf_b200.so"

TF_OK, TF_EINVAL, TF_ENOMEM, TF_EIO = 0, -22, -12, -5
TIER_GPU, TIER_HOST = 0, 1
ENGINE_SM, ENGINE_CE, ENGINE_AUTO, ENGINE_CE2D = 0, 1, 2, 3


class InvariantError(AssertionError):
    """A runtime invariant or CUDA error (mirrors tokensim.engine.InvariantError)."""


class TfSeg(C.Structure):
    _fields_ = [("gpu_block", C.c_int32), ("host_block", C.c_int32), ("slot_begin", C.c_int32),
                ("n_slots", C.c_int32)]


class TfSpan(C.Structure):
    _fields_ = [("row", C.c_int32), ("rid", C.c_int32), ("pos_begin", C.c_int32), ("pos_end", C.c_int32)]


class TfMember(C.Structure):
    _fields_ = [
        ("request_id", C.c_int32), ("prompt_len", C.c_int32), ("output_len", C.c_int32),
        ("running", C.c_int32), ("pinned", C.c_int32), ("has_tprime", C.c_int32),
        ("generated", C.c_int64), ("consumed", C.c_int64), ("ctx_tokens", C.c_int64),
        ("gpu_resident", C.c_int64),
        ("arrival_time", C.c_double), ("rate", C.c_double), ("busy_since_tick", C.c_double),
        ("t_io", C.c_double), ("t_recompute", C.c_double), ("last_iter_time", C.c_double),
        ("t_prime", C.c_double),
    ]


class TfReqRow(C.Structure):
    _fields_ = [
        ("request_id", C.c_int32), ("status", C.c_int32), ("prompt_len", C.c_int32), ("output_len", C.c_int32),
        ("has_tprime", C.c_int32), ("pad_", C.c_int32),
        ("generated", C.c_int64), ("consumed", C.c_int64), ("total_kv", C.c_int64), ("gpu_resident", C.c_int64),
        ("cpu_synced", C.c_int64), ("inflight_d2h", C.c_int64),
        ("arrival_time", C.c_double), ("rate", C.c_double), ("busy_since_tick", C.c_double),
        ("last_iter_time", C.c_double), ("t_prime", C.c_double),
    ]


class TfSnapGlobals(C.Structure):
    _fields_ = [("q_d2h_tokens", C.c_int64), ("q_h2d_tokens", C.c_int64), ("d2h_rate", C.c_double),
                ("h2d_rate", C.c_double), ("prefill_s_per_token", C.c_double)]


# engine status -> TF_ST_* (include/tokenflow_b200.h)
STATUS_CODES = {"waiting": 1, "prefill_wait": 2, "prefilling": 3, "running": 4, "preempted": 5, "loading": 6,
                "recomputing": 7, "gen_done": 8, "done": 9}


class TfWaiter(C.Structure):
    _fields_ = [("request_id", C.c_int32), ("prompt_len", C.c_int32), ("waited_s", C.c_double)]


class TfTickParams(C.Structure):
    _fields_ = [
        ("n_members", C.c_int32), ("n_waiting", C.c_int32), ("free_slots", C.c_int32),
        ("max_batch", C.c_int32), ("offload_enabled", C.c_int32), ("mode", C.c_int32),
        ("h2d_blocked_tokens", C.c_int64),
        ("now", C.c_double), ("gpu_mem_free", C.c_double), ("gpu_mem_total", C.c_double),
        ("cpu_mem_total", C.c_double), ("gamma", C.c_double),
        ("schedule_interval", C.c_double), ("per_request_mem_estimate", C.c_double),
        ("workingset_adjust_rate", C.c_double), ("buffer_safety_factor", C.c_double),
        ("penalty_weight", C.c_double), ("tau_schedule", C.c_double),
        ("critical_buffer_seconds", C.c_double), ("value_threshold_frac", C.c_double),
        ("value_decay_alpha", C.c_double), ("pacing_buffer_seconds", C.c_double),
        ("ema_factor", C.c_double),
    ]


class TfTickResult(C.Structure):
    _fields_ = [
        ("counts", C.POINTER(C.c_int32)), ("preempt", C.POINTER(C.c_int32)),
        ("resume_ids", C.POINTER(C.c_int32)), ("resume_how", C.POINTER(C.c_int32)),
        ("admitted", C.POINTER(C.c_int32)), ("recomputed", C.POINTER(C.c_int32)),
        ("batch_sizes", C.POINTER(C.c_int32)), ("batch_ids", C.POINTER(C.c_int32)),
        ("t_prime_out", C.POINTER(C.c_double)), ("t_prime_set", C.POINTER(C.c_int32)),
    ]


class TfPrio(C.Structure):
    _fields_ = [("request_id", C.c_int32), ("pad", C.c_int32), ("length", C.c_int64), ("phi", C.c_double),
                ("value", C.c_double), ("t_prime", C.c_double), ("rate", C.c_double), ("utility", C.c_double)]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_PI32 = C.POINTER(C.c_int32)

# name -> (restype, argtypes); must list every symbol in include/tokenflow_b200.h
SIGNATURES = {
    "tf_last_error": (C.c_char_p, []),
    "tf_abi_version": (C.c_int, []),
    "tf_pool_init": (C.c_int, [_P, _I32, _P, _I32, _I32, _I32, _I32, _I32, _I32, C.POINTER(_I64)]),
    "tf_pool_destroy": (C.c_int, [_I64]),
    "tf_pool_block_bytes": (_I64, [_I64]),
    "tf_blocks_alloc": (C.c_int, [_I64, _I32, _I32, _PI32]),
    "tf_blocks_free": (C.c_int, [_I64, _I32, _PI32, _I32]),
    "tf_blocks_free_count": (C.c_int, [_I64, _I32]),
    "tf_table_apply": (C.c_int, [_P, _I32, _PI32, _I32, _P]),
    "tf_kv_gather_d2h": (C.c_int, [_I64, C.POINTER(TfSeg), _I32, _I32, _I32, _I32, _P]),
    "tf_kv_scatter_h2d": (C.c_int, [_I64, C.POINTER(TfSeg), _I32, _I32, _I32, _I32, _P]),
    "tf_copy_small": (C.c_int, [_P, _P, _I64, _P]),
    "tf_launch_count": (_I64, []),
    "tf_launch_floor": (C.c_int, [_P]),
    "tf_rmsnorm": (C.c_int, [_P, _P, _P, _I32, _I32, C.c_float, _P]),
    "tf_silu_mul": (C.c_int, [_P, _P, _I32, _I32, _P]),
    "tf_residual_rmsnorm": (C.c_int, [_P, _P, _P, _P, _I32, _I32, C.c_float, _P]),
    "tf_kv_append": (C.c_int, [_I64, _P, _I32, _P, _P, _I32, _I32, _P, _P, _I64, _P]),
    "tf_rope_kv_append": (C.c_int, [_I64, _P, _I32, _P, _P, _I32, _I32, _P, _I32, _P, _P, _P, _P]),
    "tf_rope_kv_append_wt": (C.c_int, [_I64, _P, _P, _I32, _P, _P, _I32, _I32, _P, _I32, _P, _P, _P, _P]),
    "tf_kv_fill_synthetic": (C.c_int, [_I64, _P, _I32, C.POINTER(TfSpan), _I32, C.c_uint32, _P]),
    "tf_q_fill_synthetic": (C.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, C.c_uint32, _P]),
    "tf_paged_decode_attn": (C.c_int, [_I64, _P, _P, _I32, _P, _P, _I32, _I32, _I32, _I32, C.c_float, _P, _P,
                                       _I64, _P]),
    "tf_paged_decode_attn_workspace": (_I64, [_I64, _I32, _I32, _I32]),
    "tf_paged_decode_attn_impl": (C.c_int, [_I32]),
    "tf_selector_workspace_bytes": (_I64, [_I32, _I32]),
    "tf_selector_init": (C.c_int, [_P, _I64, _P, _I64, _I32, _I32, C.POINTER(_I64)]),
    "tf_selector_destroy": (C.c_int, [_I64]),
    "tf_policy_tick_rows": (C.c_int, [_I64, C.POINTER(TfTickParams), C.POINTER(TfReqRow), _I32,
                                      C.POINTER(TfSnapGlobals), C.POINTER(TfWaiter), C.POINTER(TfTickResult),
                                      _PI32, _PI32, _P]),
    "tf_policy_tick": (C.c_int, [_I64, C.POINTER(TfTickParams), C.POINTER(TfMember), C.POINTER(TfWaiter),
                                 C.POINTER(TfTickResult), _P]),
    "tf_policy_fastpath": (C.c_int, [_I64, C.POINTER(TfTickParams), C.POINTER(TfMember), C.POINTER(TfWaiter),
                                     C.POINTER(TfTickResult), _P]),
    "tf_iteration_batch": (C.c_int, [_I64, _PI32, C.POINTER(C.c_int64), C.POINTER(C.c_double), _I32, _I32, _I32,
                                     C.c_double, _PI32, _PI32, _P]),
    "tf_select_batch": (C.c_int, [_I64, C.POINTER(TfPrio), _I32, C.c_double, _I32, C.POINTER(C.c_uint8), _P]),
    "tf_host_glibc_exp": (C.c_double, [C.c_double]),
    "tf_ar_create": (C.c_int, [_I32, _I32, _I64, _I32, C.POINTER(_I64)]),
    "tf_ar_buffer": (_P, [_I64]),
    "tf_ar_ctl": (_P, [_I64]),
    "tf_ar_export": (C.c_int, [_I64, _P]),
    "tf_ar_open": (C.c_int, [_I64, _P]),
    "tf_ar_set_peers": (C.c_int, [_I64, C.POINTER(_P), C.POINTER(_P)]),
    "tf_ar_residual_rmsnorm": (C.c_int, [_I64, _P, _P, _P, _I32, _I32, C.c_float, _P]),
    "tf_ar_status": (C.c_int, [_I64]),
    "tf_ar_destroy": (C.c_int, [_I64]),
}


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -m paper_2510_02758_b200.build` "
            "(there is no CPU fallback for the KV data plane)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int, what: str = "") -> None:
    if status == TF_OK:
        return
    msg = (lib.tf_last_error() or b"").decode(errors="replace")
    if status == TF_ENOMEM:
        raise MemoryError(f"{what}: {msg}")
    if status == TF_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise InvariantError(f"{what}: status {status}: {msg}")


def stream_ptr(stream) -> int:
    """cudaStream_t of a torch.cuda.Stream (0 = legacy default)."""
    return 0 if stream is None else int(stream.cuda_stream)

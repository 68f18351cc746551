"""ctypes mirror of include/pipespec.h (argument marshalling only).

Loading never falls back to anything: if libpipespec.so is missing the import
raises, and on a machine without an sm_100a GPU every compute call returns
PS_E_CUDA, surfaced as PipeSpecError.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# PS_LIB overrides the library path (A/B timing of kernel variants, or the
# PS_TRACE build libpipespec_trace.so for scripts/timeline.py)
LIB_PATH = os.environ.get("PS_LIB") or os.path.join(PKG, "libpipespec.so")
TEST_LIB_PATH = os.path.join(PKG, "libpipespec_test.so")

PS_OK, PS_E_INVALID, PS_E_CONTRACT, PS_E_CAPACITY, PS_E_CUDA, PS_E_NCCL, PS_E_STALE = 0, -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "PS_OK", -1: "PS_E_INVALID", -2: "PS_E_CONTRACT", -3: "PS_E_CAPACITY", -4: "PS_E_CUDA",
                -5: "PS_E_NCCL", -6: "PS_E_STALE"}
PS_WQ, PS_WK, PS_WV, PS_WO, PS_WG, PS_WU, PS_WD, PS_N_ATTN, PS_N_MLP, PS_LAYER_SLOTS = range(10)
PS_MODE_AR, PS_MODE_SYNC_SD, PS_MODE_PIPESPEC = 0, 1, 2
PS_PREFILL_AUTO, PS_PREFILL_ROWS = 0, 1
PS_EV_DRAFT, PS_EV_VERIFY, PS_EV_AR, PS_EV_RESYNC, PS_EV_STALE = 0, 1, 2, 3, 4
PS_TP_HANDLE_BYTES = 256


class PipeSpecError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class ModelShape(C.Structure):
    _fields_ = [("vocab", C.c_int32), ("d_model", C.c_int32), ("n_layers", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("d_ffn", C.c_int32),
                ("rms_eps", C.c_float), ("rope_theta", C.c_float), ("rope_kind", C.c_int32),
                ("rope_factor", C.c_float), ("lo_ff", C.c_float), ("hi_ff", C.c_float),
                ("rope_orig_max", C.c_int32), ("tied_lm_head", C.c_int32)]


class Weights(C.Structure):
    _fields_ = [("embed", C.c_void_p), ("lm_head", C.c_void_p), ("final_norm", C.c_void_p),
                ("layers", C.POINTER(C.c_void_p))]


class Placement(C.Structure):
    _fields_ = [("device", C.c_int32), ("nccl_comm", C.c_void_p), ("tp_rank", C.c_int32), ("tp_size", C.c_int32)]


class StageOpts(C.Structure):
    _fields_ = [("max_seq", C.c_int32), ("max_window", C.c_int32), ("page_size", C.c_int32),
                ("kv_pool", C.c_void_p), ("kv_pool_bytes", C.c_int64), ("stream", C.c_void_p),
                ("use_graphs", C.c_int32), ("use_megakernel", C.c_int32), ("max_ctas", C.c_int32)]


class StageInfo(C.Structure):
    _fields_ = [("n_tokens", C.c_int64), ("kv_len", C.c_int64), ("pages_in_use", C.c_int64),
                ("pages_total", C.c_int64), ("launches_per_verify", C.c_int64), ("rows_buckets", C.c_int32 * 4),
                ("last_fwd_ms", C.c_double), ("sum_fwd_ms", C.c_double), ("n_fwd", C.c_int64),
                ("max_window", C.c_int32), ("max_seq", C.c_int32), ("attn_sc", C.c_int32)]


class VerifyResult(C.Structure):
    _fields_ = [("a", C.c_int32), ("next", C.c_int32), ("rows", C.c_int32), ("kv_len", C.c_int32),
                ("pred", C.c_int32 * 32)]


class VerifyTicket(C.Structure):
    _fields_ = [("d_result", C.c_void_p), ("h_result", C.POINTER(VerifyResult)), ("event", C.c_void_p)]


class Event(C.Structure):
    _fields_ = [("t_ns", C.c_int64), ("stage", C.c_int32), ("kind", C.c_int32), ("n", C.c_int32),
                ("w", C.c_int32), ("a", C.c_int32), ("next", C.c_int32), ("origin", C.c_int32),
                ("pad", C.c_int32), ("window", C.c_int32 * 32)]


class RunOpts(C.Structure):
    _fields_ = [("mode", C.c_int32), ("max_new_tokens", C.c_int32), ("eos_id", C.c_int32),
                ("gamma", C.POINTER(C.c_int32)), ("lookahead", C.POINTER(C.c_int32)), ("max_lead", C.c_int32),
                ("alpha", C.POINTER(C.c_double)), ("seed", C.c_uint64), ("virtual_ns", C.POINTER(C.c_int64)),
                ("event_log", C.POINTER(Event)), ("event_cap", C.c_int32)]


class RunStats(C.Structure):
    _fields_ = [("tokens", C.c_int64), ("wall_ns", C.c_int64), ("steps", C.c_int64 * 8),
                ("verify_steps", C.c_int64 * 8), ("rollbacks", C.c_int64 * 8), ("busy_ns", C.c_int64 * 8),
                ("accept_hist", C.c_int64 * 64), ("n_events", C.c_int64), ("events_dropped", C.c_int64),
                ("fwd_ns", C.c_int64 * 8), ("n_fwd", C.c_int64 * 8)]


_I32P = C.POINTER(C.c_int32)
_PROTOS = {
    "ps_last_error": (C.c_char_p, []),
    "ps_version": (C.c_int32, []),
    "ps_kernel_launch_count": (C.c_int64, []),
    "ps_kv_pool_bytes": (C.c_int64, [C.POINTER(ModelShape), C.c_int32, C.c_int32]),
    "ps_kv_pool_bytes_tp": (C.c_int64, [C.POINTER(ModelShape), C.c_int32, C.c_int32, C.c_int32]),
    "ps_tp_handle": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "ps_tp_connect": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "ps_tp_connect_local": (C.c_int32, [C.POINTER(C.c_void_p), C.c_int32]),
    "ps_stage_create": (C.c_int32, [C.POINTER(ModelShape), C.POINTER(Weights), C.POINTER(Placement),
                                    C.POINTER(StageOpts), C.POINTER(C.c_void_p)]),
    "ps_stage_destroy": (C.c_int32, [C.c_void_p]),
    "ps_prefill": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int32]),
    "ps_set_prefill_path": (C.c_int32, [C.c_void_p, C.c_int32]),
    "ps_draft": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p]),
    "ps_verify": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int32, _I32P, _I32P, C.c_void_p]),
    "ps_verify_async": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(VerifyTicket)]),
    "ps_verify_wait": (C.c_int32, [C.c_void_p, _I32P, _I32P]),
    "ps_verify_query": (C.c_int32, [C.c_void_p, _I32P]),
    "ps_kv_rollback": (C.c_int32, [C.c_void_p, C.c_int64]),
    "ps_stage_tokens": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]),
    "ps_stage_get_info": (C.c_int32, [C.c_void_p, C.POINTER(StageInfo)]),
    "ps_stage_reset_timers": (C.c_int32, [C.c_void_p]),
    "ps_set_synthetic": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                     C.POINTER(C.c_double), C.c_uint64]),
    "ps_pipeline_run": (C.c_int32, [C.POINTER(C.c_void_p), C.c_int32, C.c_void_p, C.c_int32, C.POINTER(RunOpts),
                                    C.c_void_p, _I32P, C.POINTER(RunStats)]),
    "ps_resync": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int32]),
    "ps_board_create": (C.c_int32, [C.c_char_p, C.c_int32, C.c_int32]),
    "ps_board_unlink": (C.c_int32, [C.c_char_p]),
    "ps_pipeline_run_rank": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_char_p, C.c_void_p, C.c_int32,
                                         C.POINTER(RunOpts), C.c_void_p, _I32P, C.POINTER(RunStats)]),
    "ps_pipeline_run_rank_group": (C.c_int32, [C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_int32, C.c_char_p,
                                               C.c_void_p, C.c_int32, C.POINTER(RunOpts), C.c_void_p, _I32P,
                                               C.POINTER(RunStats)]),
}

# libpipespec_test.so (include/pipespec_test.h): test infrastructure, never
# loaded by the product path
_TEST_PROTOS = {
    "ps_test_last_error": (C.c_char_p, []),
    "ps_test_fake_pipeline": (C.c_int32, [C.c_int32, C.c_void_p, C.c_int32, C.POINTER(RunOpts), C.c_int32,
                                          C.c_double, C.c_uint64, C.c_int32, C.c_void_p, _I32P,
                                          C.POINTER(RunStats)]),
    "ps_test_fake_run_rank": (C.c_int32, [C.c_int32, C.c_int32, C.c_char_p, C.c_void_p, C.c_int32,
                                          C.POINTER(RunOpts), C.c_int32, C.c_double, C.c_uint64, C.c_int32,
                                          C.c_void_p, _I32P, C.POINTER(RunStats)]),
    "ps_test_board_create": (C.c_int32, [C.c_char_p, C.c_int32, C.c_int32]),
    "ps_test_board_unlink": (C.c_int32, [C.c_char_p]),
    "ps_test_launch_overhead": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_float)]),
    "ps_test_tc_probe": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double)]),
    "ps_test_tc_probe2": (C.c_int32, [C.c_int32, C.c_int32, C.POINTER(C.c_double)]),
    "ps_test_hmma_probe": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}
# trace build only (PS_LIB=.../libpipespec_trace.so)
_TRACE_PROTOS = {"ps_trace_read": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64])}

_lib = None
_test_lib = None


def lib():
    """Load libpipespec.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2505_01572_b200._build`")
        L = C.CDLL(LIB_PATH)
        _bind(L, _PROTOS)
        if hasattr(L, "ps_trace_read"):
            _bind(L, _TRACE_PROTOS)
        _lib = L
    return _lib


def _bind(L, protos):
    for name, (res, args) in protos.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def test_lib():
    """Load libpipespec_test.so (tests only)."""
    global _test_lib
    if _test_lib is None:
        if not os.path.exists(TEST_LIB_PATH):
            raise ImportError(f"{TEST_LIB_PATH} not built; run `python -m paper_2505_01572_b200._build`")
        L = C.CDLL(TEST_LIB_PATH)
        _bind(L, _TEST_PROTOS)
        _test_lib = L
    return _test_lib


def test_check(status: int) -> None:
    if status != PS_OK:
        raise PipeSpecError(status, test_lib().ps_test_last_error().decode(errors="replace"))


def check(status: int) -> None:
    if status != PS_OK:
        raise PipeSpecError(status, lib().ps_last_error().decode(errors="replace"))

"""ctypes mirror of include/nest.h.  Argument marshalling only.

Loading fails loudly when libnest.so is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# NEST_LIB: an alternative in-tree build (tuning variants built with
# build.build(out=...)); default: the libnest.so build() writes
LIB_PATH = os.environ.get("NEST_LIB") or os.path.join(HERE, "libnest.so")

NEST_OK = 0
STATUS = {0: "NEST_OK", 1: "NEST_ERR_INVALID", 2: "NEST_ERR_CUDA", 3: "NEST_ERR_NCCL",
          4: "NEST_ERR_CAPACITY", 5: "NEST_ERR_KEY_RANGE", 6: "NEST_ERR_SHARD",
          7: "NEST_ERR_ORDER", 8: "NEST_ERR_DIVISIBILITY"}
POOL_SUM, POOL_NONE = 0, 1
INIT_UNIFORM, INIT_DYADIC, INIT_ZERO = 0, 1, 2
SCHED_SEQUENTIAL, SCHED_CLUSTERED = 0, 1
OPT_SGD, OPT_ROWWISE_ADAGRAD = 0, 1
TABLE_HBM, TABLE_HOST = 0, 1
MAX_MICRO_BATCHES = 8

# every symbol include/nest.h declares (checked by tests/test_abi.py)
SYMBOLS = ["nest_version", "nest_get_unique_id", "nest_workspace_bytes", "nest_shard_rows",
           "nest_create", "nest_destroy", "nest_window_export", "nest_window_connect", "nest_check_guards", "nest_init_tables", "nest_fwp_schedule", "nest_route", "nest_route_begin", "nest_route_end",
           "nest_dbp_refresh", "nest_lookup_prefetch", "nest_lookup_fwd", "nest_lookup_fwd_bf16",
           "nest_grad_bwd_update", "nest_grad_bwd_update_adagrad", "nest_tower_fwd_bwd",
           "nest_tower_fwd_bwd_bf16", "nest_tower_step", "nest_set_streams", "nest_set_zero_copy", "nest_join", "nest_read_state", "nest_tower_read",
           "nest_slot_info", "nest_route_view", "nest_read_rows", "nest_exchange_plan", "nest_profile_enable",
           "nest_profile_read", "nest_profile_records", "nest_last_error"]
PROFILE_STAGES = 16


class NestError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class Config(C.Structure):
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("num_tables", C.c_int32),
                ("dim", C.c_int32), ("table_rows", C.POINTER(C.c_int64)), ("pooling", C.c_int32),
                ("num_features", C.c_int32), ("max_keys", C.c_int64), ("max_batch", C.c_int64),
                ("max_micro_batches", C.c_int32), ("max_recv_keys", C.c_int64),
                ("max_owner_keys", C.c_int64), ("max_mb_rows", C.c_int64),
                ("max_owner_mb_rows", C.c_int64), ("seed", C.c_uint64), ("init_mode", C.c_int32),
                ("tower_layers", C.c_int32), ("tower_hidden", C.c_int32), ("optimizer", C.c_int32),
                ("adagrad_eps", C.c_float), ("table_location", C.c_int32),
                ("tower_train", C.c_int32), ("tower_lr", C.c_float)]


class SlotInfo(C.Structure):
    _fields_ = [("valid", C.c_int32), ("num_micro_batches", C.c_int32), ("batch", C.c_int32),
                ("nnz", C.c_int64), ("uniq", C.c_int64), ("recv", C.c_int64),
                ("mb_uniq", C.c_int64 * MAX_MICRO_BATCHES), ("mb_recv", C.c_int64 * MAX_MICRO_BATCHES),
                ("mb_nnz", C.c_int64 * MAX_MICRO_BATCHES),
                ("mb_out_rows", C.c_int64 * MAX_MICRO_BATCHES)]


class RouteView(C.Structure):
    _fields_ = [("uniq", C.c_void_p), ("inverse", C.c_void_p), ("mask", C.c_void_p),
                ("pos", C.c_void_p), ("send_counts", C.c_void_p), ("all_counts", C.c_void_p),
                ("recv_keys", C.c_void_p), ("owner_rows", C.c_void_p), ("owner_inv", C.c_void_p),
                ("n_owner", C.c_void_p), ("buffer", C.c_void_p)]


MAX_WORLD = 64


class ExchangePlan(C.Structure):
    _fields_ = [("uniq", C.c_int64), ("recv", C.c_int64),
                ("key_send_off", C.c_int64 * (MAX_WORLD + 1)), ("key_recv_off", C.c_int64 * (MAX_WORLD + 1)),
                ("mb_uniq", C.c_int64 * MAX_MICRO_BATCHES), ("mb_recv", C.c_int64 * MAX_MICRO_BATCHES),
                ("src_base", C.c_int64 * (MAX_MICRO_BATCHES + 1)),
                ("own_base", C.c_int64 * (MAX_MICRO_BATCHES + 1))]


class ProfileStage(C.Structure):
    _fields_ = [("name", C.c_char * 24), ("stream", C.c_int32), ("records", C.c_int32),
                ("launches", C.c_int32), ("pad", C.c_int32), ("ms", C.c_double), ("bytes", C.c_double),
                ("units", C.c_double), ("hbm_bytes", C.c_double)]


class ProfileRecord(C.Structure):
    _fields_ = [("stage", C.c_int32), ("stream", C.c_int32), ("t0_ms", C.c_double), ("t1_ms", C.c_double)]


class ProfileSummary(C.Structure):
    _fields_ = [("span_ms", C.c_double), ("a2a_ms", C.c_double), ("a2a_union_ms", C.c_double),
                ("a2a_exposed_ms", C.c_double), ("compute_busy_ms", C.c_double), ("launches", C.c_int64)]


class WindowRec(C.Structure):
    """nest_window_rec_t: one rank's exchange-window record (plain bytes)."""
    _fields_ = [("magic", C.c_uint64), ("pid", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("device", C.c_int32), ("ptr", C.c_uint64), ("ipc", C.c_uint8 * 64),
                ("bytes", C.c_uint64), ("off_own", C.c_uint64), ("off_cnt", C.c_uint64),
                ("off_key", C.c_uint64), ("off_twr", C.c_uint64), ("off_flags", C.c_uint64),
                ("src_stride", C.c_uint64), ("cnt_stride", C.c_uint64), ("key_stride", C.c_uint64),
                ("off_dwb", C.c_uint64), ("dwb_stride", C.c_uint64), ("shard_ptr", C.c_uint64),
                ("shard_off", C.c_uint64), ("shard_ipc", C.c_uint8 * 64), ("dwb_ok", C.c_int32),
                ("dwb_pad", C.c_int32)]


_lib = None


def load() -> C.CDLL:
    """Load libnest.so (build it first with paper_2604_06956_b200.build.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(the CUDA path has no fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
    sig = {
        "nest_version": ([], C.c_char_p),
        "nest_get_unique_id": ([vp], i32),
        "nest_workspace_bytes": ([C.POINTER(Config), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)], i32),
        "nest_shard_rows": ([C.POINTER(Config)], i64),
        "nest_create": ([C.POINTER(Config), vp, vp, vp, vp, C.POINTER(vp)], i32),
        "nest_destroy": ([vp], i32),
        "nest_window_export": ([vp, C.POINTER(WindowRec)], i32),
        "nest_check_guards": ([vp, vp, C.POINTER(i64)], i32),
        "nest_window_connect": ([vp, C.POINTER(WindowRec)], i32),
        "nest_init_tables": ([vp, vp], i32),
        "nest_fwp_schedule": ([vp, vp, vp, i64, i32, i32, i32, vp, vp, vp], i32),
        "nest_route": ([vp, i32, vp, vp, i64, i32, vp, vp, i32, vp], i32),
        "nest_route_begin": ([vp, i32, vp, vp, i64, i32, vp, vp, i32, vp], i32),
        "nest_route_end": ([vp, i32], i32),
        "nest_dbp_refresh": ([vp, i32, i32, vp], i32),
        "nest_lookup_prefetch": ([vp, i32, i32, vp, vp], i32),
        "nest_lookup_fwd": ([vp, i32, i32, vp, vp, vp], i32),
        "nest_lookup_fwd_bf16": ([vp, i32, i32, vp, vp, vp], i32),
        "nest_grad_bwd_update": ([vp, i32, i32, vp, f32, vp, vp], i32),
        "nest_grad_bwd_update_adagrad": ([vp, i32, i32, vp, f32, f32, vp, vp], i32),
        "nest_tower_fwd_bwd": ([vp, vp, i64, vp, vp], i32),
        "nest_tower_fwd_bwd_bf16": ([vp, vp, i64, vp, vp], i32),
        "nest_tower_read": ([vp, i32, i32, vp, vp], i32),
        "nest_tower_step": ([vp, vp], i32),
        "nest_set_streams": ([vp, vp, vp], i32),
        "nest_set_zero_copy": ([vp, i32], i32),
        "nest_join": ([vp, vp], i32),
        "nest_slot_info": ([vp, i32, C.POINTER(SlotInfo)], i32),
        "nest_route_view": ([vp, i32, C.POINTER(RouteView)], i32),
        "nest_read_rows": ([vp, vp, i64, vp, vp], i32),
        "nest_read_state": ([vp, vp, i64, vp, vp], i32),
        "nest_exchange_plan": ([C.POINTER(Config), i32, vp, C.POINTER(ExchangePlan)], i32),
        "nest_profile_enable": ([vp, i32], i32),
        "nest_profile_read": ([vp, C.POINTER(ProfileStage), C.POINTER(ProfileSummary)], i32),
        "nest_profile_records": ([vp, C.POINTER(ProfileRecord), i64, C.POINTER(i64)], i32),
        "nest_last_error": ([vp], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(code: int, ctx=None) -> None:
    if code != NEST_OK:
        msg = load().nest_last_error(ctx)
        raise NestError(code, (msg or b"").decode(errors="replace"))

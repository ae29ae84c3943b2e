"""ctypes binding of libsgm.so (include/sgm.h).

This is exactly the binding a maintainer of the reference would add
(INTEGRATION.md): POD descriptors, raw device pointers, sizes, status codes.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import BackendUnavailable, from_status

MAX_RANK, MAX_GRID, MAX_NODES, MAX_SLOTS = 4, 3, 64, 16
ABI_VERSION = 2

F64, F32, BF16, FF = 0, 1, 2, 3
NUMSYS_NAMES = {F64: "f64", F32: "f32", BF16: "bf16", FF: "ff"}


class SlotDesc(C.Structure):
    _fields_ = [("rank", C.c_int32), ("_pad", C.c_int32), ("dims", C.c_int64 * MAX_RANK)]


class NodeDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("n_inputs", C.c_int32), ("inputs", C.c_int32 * 2),
        ("slot", C.c_int32), ("axis", C.c_int32),
        ("const_num", C.c_int64), ("const_den", C.c_int64),
        ("rank", C.c_int32), ("_pad", C.c_int32),
        ("shape", C.c_int64 * MAX_RANK),
        ("grid_mask", C.c_uint32 * MAX_RANK),
        ("loop_split", C.c_int32 * MAX_RANK),
    ]


class PlanHints(C.Structure):
    _fields_ = [
        ("max_cluster", C.c_int32), ("target_ctas", C.c_int32), ("threads", C.c_int32),
        ("smem_budget", C.c_int32), ("no_loop_split", C.c_int32), ("no_hoist", C.c_int32),
        ("use_tcgen05", C.c_int32), ("no_tma", C.c_int32), ("trace", C.c_int32),
        ("variant", C.c_int32), ("one_cta", C.c_int32), ("max_gsplit", C.c_int32), ("slot_kb", C.c_int32),
        ("wd_test", C.c_int32), ("small_plain", C.c_int32), ("big_first", C.c_int32),
        ("item_cost_ns", C.c_int32), ("min_gsplit", C.c_int32),
        ("no_wd", C.c_int32), ("interleave", C.c_int32),
        ("ff_tma", C.c_int32), ("no_xcache", C.c_int32), ("no_prefetch", C.c_int32),
        ("_reserved", C.c_int32 * 3),
    ]


class PlanDesc(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32), ("numsys", C.c_int32),
        ("n_inputs", C.c_int32), ("n_outputs", C.c_int32),
        ("inputs", SlotDesc * MAX_SLOTS), ("outputs", SlotDesc * MAX_SLOTS),
        ("n_nodes", C.c_int32), ("n_grid", C.c_int32),
        ("grid", C.c_int64 * MAX_GRID), ("n_loop", C.c_int64),
        ("nodes", NodeDesc * MAX_NODES),
        ("hints", PlanHints),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("logical_blocks", C.c_int64), ("ctas", C.c_int64),
        ("cluster", C.c_int32), ("threads", C.c_int32), ("smem_bytes", C.c_int32), ("loop_parts", C.c_int32),
        ("free_parts", C.c_int64), ("scratch_bytes", C.c_int64), ("compile_ms", C.c_double),
        ("cache_hit", C.c_int32), ("n_tcgen05", C.c_int32), ("source_hash", C.c_uint64),
        ("kernel_name", C.c_char * 64), ("plan_summary", C.c_char * 448),
    ]


SYMBOLS = {
    "sgm_abi_version": ([], C.c_int),
    "sgm_last_error": ([], C.c_char_p),
    "sgm_launch_count": ([], C.c_longlong),
    "sgm_init": ([C.c_int], C.c_int),
    "sgm_set_cache_dir": ([C.c_char_p], C.c_int),
    "sgm_plan_create": ([C.POINTER(PlanDesc), C.POINTER(C.c_void_p)], C.c_int),
    "sgm_plan_feasible": ([C.POINTER(PlanDesc), C.POINTER(PlanInfo)], C.c_int),
    "sgm_plan_info_get": ([C.c_void_p, C.POINTER(PlanInfo)], C.c_int),
    "sgm_plan_source": ([C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "sgm_plan_cubin": ([C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "sgm_plan_destroy": ([C.c_void_p], C.c_int),
    "sgm_plan_run": ([C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int, C.c_void_p], C.c_int),
    "sgm_plan_run_host": ([C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_void_p], C.c_int),
    "sgm_plan_time": ([C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int,
                       C.c_void_p, C.POINTER(C.c_double)], C.c_int),
    "sgm_plan_trace": ([C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)], C.c_int),
    "sgm_timer_create": ([C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "sgm_timer_enqueue": ([C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int,
                           C.c_int, C.c_int, C.c_void_p], C.c_int),
    "sgm_timer_read": ([C.c_void_p, C.c_int, C.POINTER(C.c_double)], C.c_int),
    "sgm_timer_destroy": ([C.c_void_p], C.c_int),
    "sgm_compare_u32_acc": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p], C.c_int),
    "sgm_ff_fill": ([C.c_void_p, C.c_int64, C.c_uint64, C.c_uint64, C.c_void_p], C.c_int),
    "sgm_compare_u32": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(C.c_int64)], C.c_int),
    "sgm_rel_err": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.POINTER(C.c_double)], C.c_int),
    "sgm_plan_watchdog": ([C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_int)], C.c_int),
    "sgm_set_pdl": ([C.c_int], C.c_int),
    "sgm_rel_err_acc": ([C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p], C.c_int),
    "sgm_fill_normal": ([C.c_void_p, C.c_int64, C.c_int, C.c_uint64, C.c_void_p], C.c_int),
}

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsgm.so")
_lib = None
_lock = threading.Lock()
_tls = threading.local()


def lib():
    """Load libsgm.so (in-tree build).  Fails loudly: there is no CPU fallback."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise BackendUnavailable(
                        f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
                h = C.CDLL(LIB_PATH)
                for name, (argtypes, restype) in SYMBOLS.items():
                    fn = getattr(h, name)
                    fn.argtypes = argtypes
                    fn.restype = restype
                if h.sgm_abi_version() != ABI_VERSION:
                    raise BackendUnavailable("libsgm ABI mismatch; rebuild")
                _lib = h
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().sgm_last_error()
        raise from_status(status, msg.decode() if msg else "")


def bind_device(device: int) -> None:
    """sgm_init on the calling thread (idempotent and cheap)."""
    if getattr(_tls, "device", None) != device:
        check(lib().sgm_init(int(device)))
        _tls.device = device


def ptr_array(ptrs) -> "C.Array":
    arr = (C.c_void_p * max(1, len(ptrs)))()
    for k, p in enumerate(ptrs):
        arr[k] = p
    return arr


def launch_count() -> int:
    return int(lib().sgm_launch_count())

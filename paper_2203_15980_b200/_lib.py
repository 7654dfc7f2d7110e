"""ctypes binding to libdelta.so (include/delta/delta.h).

No torch types cross this boundary: plain pointers, sizes and POD structs.
The library is built in-tree by `make` (or `__graft_entry__.build()`); if it
is missing, importing this module raises — there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DELTA_LIB: an alternative build of the library (A/B timing of two builds)
LIB_PATH = os.environ.get("DELTA_LIB") or os.path.join(_HERE, "libdelta.so")

u8, u32, u64, i32 = C.c_uint8, C.c_uint32, C.c_uint64, C.c_int32


class DeltaConfig(C.Structure):
    _fields_ = [
        ("budget", u64), ("heuristic", u32), ("policy_mode", u32),
        ("bw_num", u64), ("bw_den", u64), ("eff_num", u64), ("eff_den", u64),
        ("swap_cost_mode", u32), ("prefetch_guard", u32),
        ("watermark_num", u64), ("watermark_den", u64), ("prefetch_limit", u64),
        ("prefetch_enabled", u32), ("overlap_enabled", u32),
        ("scripted_nodes", C.POINTER(u64)), ("scripted_actions", C.POINTER(u32)),
        ("n_scripted", u64),
    ]


class DeltaEvent(C.Structure):
    _fields_ = [("ts", u64), ("node", u64), ("duration", u64), ("bytes", u64),
                ("burst", u32), ("stream", u8), ("kind", u8), ("phase", u8),
                ("prefetch", u8)]


class DeltaDecision(C.Structure):
    _fields_ = [("node", u64), ("action", u32), ("pad", u32)]


class DeltaSummary(C.Structure):
    _fields_ = [
        ("peak_bytes", u64), ("wall_time_us", u64), ("total_stall_us", u64),
        ("copy_busy_us", u64), ("copy_stall_us", u64),
        ("evict", u64), ("offload", u64), ("reload", u64), ("recompute", u64),
        ("prefetch_reload", u64), ("recompute_of_swapout", u64),
        ("infeasible", u32), ("pad", u32),
        ("infeasible_node", u64), ("infeasible_deficit", u64),
        ("n_events", u64), ("n_decisions", u64),
    ]


class DeltaAction(C.Structure):
    _fields_ = [("op", u32), ("stream", u32), ("node", u64), ("offset", u64),
                ("bytes", u64), ("host_offset", u64), ("event", u32),
                ("n_inputs", u32), ("inputs_at", u64), ("plan_event", u64)]


class DeltaProgramInfo(C.Structure):
    _fields_ = [("arena_bytes", u64), ("pool_peak_bytes", u64), ("host_bytes", u64),
                ("n_actions", u64), ("n_inputs", u64), ("n_events", u64)]


STATUS_NAMES = {
    1: "SchemaError", 2: "ValidationErrorEx", 3: "ArgumentError", 4: "StateError",
    5: "IllegalTransition", 6: "UnrecoverableError", 7: "MismatchedTrace",
    8: "TooLarge", 9: "IoError", 10: "InternalError", 20: "CudaError",
    21: "Unsupported", 99: "UnknownError",
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build()")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    sig = {
        "delta_last_error": (C.c_char_p, []),
        "delta_free": (None, [vp]),
        "delta_version": (C.c_char_p, []),
        "delta_trace_new": (i32, [C.c_char_p, P(vp)]),
        "delta_trace_add_node": (i32, [vp, u64, C.c_char_p, u64, u64, P(u64), u64, u32]),
        "delta_trace_add_event": (i32, [vp, u64, u32, u32]),
        "delta_trace_set_cost": (i32, [vp, u64, u64]),
        "delta_trace_parse": (i32, [C.c_char_p, u64, P(vp)]),
        "delta_trace_serialize": (i32, [vp, P(vp), P(u64)]),
        "delta_trace_validate": (i32, [vp, P(u32), P(u32), P(vp)]),
        "delta_trace_num_nodes": (u64, [vp]),
        "delta_trace_num_events": (u64, [vp]),
        "delta_trace_free": (None, [vp]),
        "delta_config_default": (None, [P(DeltaConfig)]),
        "delta_plan": (i32, [vp, P(DeltaConfig), P(vp)]),
        "delta_plan_baseline": (i32, [vp, P(DeltaConfig), P(vp)]),
        "delta_result_summary": (i32, [vp, P(DeltaSummary)]),
        "delta_result_events": (P(DeltaEvent), [vp, P(u64)]),
        "delta_result_decisions": (P(DeltaDecision), [vp, P(u64)]),
        "delta_report_json": (i32, [vp, vp, P(vp), P(u64)]),
        "delta_comparison": (i32, [vp, P(DeltaConfig), P(u64), u64, P(u32), u64, P(u32), u64, i32,
                                   P(vp), P(u64)]),
        "delta_chrome_trace": (i32, [vp, P(vp), P(u64)]),
        "delta_chrome_trace_events": (i32, [vp, u64, P(vp), P(u64)]),
        "delta_result_free": (None, [vp]),
        "delta_plan_time_ns": (i32, [vp, P(DeltaConfig), u32, P(C.c_double)]),
        "delta_transfer_time_us": (i32, [u64, P(DeltaConfig), P(u64)]),
        "delta_lower": (i32, [vp, P(DeltaConfig), u64, P(vp)]),
        "delta_lower_ex": (i32, [vp, P(DeltaConfig), u64, u32, P(vp)]),
        "delta_program_info_get": (i32, [vp, P(DeltaProgramInfo)]),
        "delta_program_actions": (P(DeltaAction), [vp, P(u64)]),
        "delta_program_inputs": (P(u64), [vp, P(u64)]),
        "delta_program_plan": (vp, [vp]),
        "delta_program_free": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


class DeltaError(RuntimeError):
    """A non-zero delta_status; `.kind` is the reference exception class name."""

    def __init__(self, status: int, msg: str):
        self.status = status
        self.kind = STATUS_NAMES.get(status, f"status{status}")
        super().__init__(f"{self.kind}: {msg}")


def check(status: int) -> None:
    if status != 0:
        raise DeltaError(status, lib.delta_last_error().decode(errors="replace"))


def take_string(ptr: C.c_void_p, n: int) -> str:
    try:
        return C.string_at(ptr, n).decode()
    finally:
        lib.delta_free(ptr)


# every symbol include/delta/delta.h declares (checked by the CPU tests)
EXPORTED = None


def header_symbols(header_path: str) -> list[str]:
    import re
    text = open(header_path).read()
    return sorted(set(re.findall(r"\b(delta_[a-z0-9_]+)\s*\(", text)))

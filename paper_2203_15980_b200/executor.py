"""ctypes binding of the step executor (include/delta/delta_rt.h) and the
recipe builder's vocabulary.

A recipe is the list of kernel ops that (re)produce one node; operands are
symbolic arena references (OUT, IN(i)), absolute device pointers, or the
pointer a HOST op of the same recipe returned (SCRATCH(k)).  The executor
(csrc/rt/executor.cu) walks the lowered action program in C++ and launches
them; HOST ops (a plug-in point for caller-supplied work; the built-in
ResNet recipes use none) call back into Python."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from ._lib import check, lib

vp, i32, i64, u32, u64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float

REF_PTR, REF_OUT, REF_IN, REF_SCRATCH = 0, 1, 2, 3
(K_COPY, K_CONV, K_CONV_EX, K_BN_STATS, K_BN_STATS_PARTS, K_BN_APPLY, K_BN_BWD, K_BN_BWD_PARTS,
 K_ADD_GRAD, K_MAXPOOL_FWD, K_MAXPOOL_BWD, K_AVGPOOL, K_SOFTMAX_XENT, K_HOST, K_WGRAD,
 K_XENT_HEAD) = range(1, 17)
(K_LAYERNORM, K_LAYERNORM_BWD, K_GELU, K_ADD_DROPOUT, K_DROPOUT_BWD, K_COLSUM, K_EMBED,
 K_EMBED_GRADS, K_SPAN_HEAD, K_SPAN_HEAD_BWD, K_ATTN, K_ATTN_BWD, K_STATS_SUM,
 K_LAYERNORM_BWD_DROP, K_PARTS_MERGE) = range(17, 32)
FIRST_ONLY, RECOMPUTE_ONLY, SIDE, SIDE_ALWAYS = 1, 2, 4, 8



OBSERVED_DTYPE = np.dtype([("t_ns", np.uint64), ("seq", np.uint64), ("action", np.uint64),
                           ("tail", np.uint8), ("node", np.uint64), ("op", np.uint8)])


class DeltaRef(C.Structure):
    _fields_ = [("kind", u32), ("index", u32), ("ptr", u64)]


class DeltaKop(C.Structure):
    _fields_ = [("kind", u32), ("flags", u32), ("conv", vp), ("i", i64 * 4), ("f", f32 * 2),
                ("pad", u32), ("r", DeltaRef * 14)]


class DeltaRecipe(C.Structure):
    _fields_ = [("node", u64), ("first", u32), ("count", u32)]


HOST_FN = C.CFUNCTYPE(u64, vp, u64, i64, u64, C.POINTER(u64), u32, i32, vp, C.POINTER(i32))
ACTION_FN = C.CFUNCTYPE(None, vp, u64, u64, u64, vp)

_SIGS = {
    "delta_rt_create": (i32, [vp, u64, u64, C.POINTER(vp)]),
    "delta_rt_arena": (vp, [vp]),
    "delta_rt_host_slab": (vp, [vp]),
    "delta_rt_copy_stream": (vp, [vp, i32]),
    "delta_rt_bind": (i32, [vp, vp, C.POINTER(DeltaKop), u64, C.POINTER(DeltaRecipe), u64]),
    "delta_rt_set_callbacks": (i32, [vp, HOST_FN, ACTION_FN, vp]),
    "delta_rt_step": (i32, [vp, vp]),
    "delta_rt_step_timed": (i32, [vp, vp, C.POINTER(f32), C.POINTER(f32), u64]),
    "delta_rt_measure_costs": (i32, [vp, vp, u32, C.POINTER(u64), u64]),
    "delta_rt_step_observed": (i32, [vp, vp, C.POINTER(u64), u64, C.POINTER(u64)]),
    "delta_rt_set_ready_nodes": (i32, [vp, C.POINTER(u64), u32]),
    "delta_rt_wait_ready": (i32, [vp, vp, u32]),
    "delta_rt_destroy": (None, [vp]),
}
for _n, (_r, _a) in _SIGS.items():
    _f = getattr(lib, _n)
    _f.restype = _r
    _f.argtypes = _a


# ------------------------------------------------------------ references
def OUT():
    return (REF_OUT, 0, 0)


def IN(i: int):
    return (REF_IN, i, 0)


def SCRATCH(k: int):
    return (REF_SCRATCH, k, 0)


def PTR(p):
    return (REF_PTR, 0, int(p or 0))


def _ref(r) -> tuple:
    if r is None:
        return (REF_PTR, 0, 0)
    if isinstance(r, tuple):
        return r
    return (REF_PTR, 0, int(r))


def kop(kind: int, refs=(), ints=(), floats=(), conv=None, flags: int = 0) -> DeltaKop:
    k = DeltaKop()
    k.kind = kind
    k.flags = flags
    k.conv = conv
    for j, v in enumerate(ints):
        k.i[j] = int(v)
    for j, v in enumerate(floats):
        k.f[j] = float(v)
    for j, r in enumerate(refs):
        kind_, idx, ptr = _ref(r)
        k.r[j].kind, k.r[j].index, k.r[j].ptr = kind_, idx, ptr
    return k


class Executor:
    """Owned delta_rt: borrows the arena, owns the pinned swap slab and the
    copy-engine streams; binds (program, recipes) and issues steps."""

    def __init__(self, arena_ptr: int, arena_bytes: int, host_bytes: int):
        self._h = vp()
        check(lib.delta_rt_create(arena_ptr, arena_bytes, host_bytes, C.byref(self._h)))
        self.arena_bytes = arena_bytes
        self.host_bytes = host_bytes
        self.host_ptr = lib.delta_rt_host_slab(self._h) or 0
        self.d2h_stream = lib.delta_rt_copy_stream(self._h, 1)
        self.h2d_stream = lib.delta_rt_copy_stream(self._h, 2)
        self._host_ops = []
        self._after = None
        self._error = None
        self._cb_host = HOST_FN(self._on_host)
        self._cb_after = ACTION_FN(self._on_action)
        check(lib.delta_rt_set_callbacks(self._h, self._cb_host, self._cb_after, None))
        self.n_actions = 0
        self.launches_per_step = 0

    # callbacks (run under the GIL; exceptions are carried back as status)
    def _on_host(self, ctx, node, host_op, out, ins, n_ins, recompute, stream, status):
        try:
            r = self._host_ops[host_op](int(out), [int(ins[j]) for j in range(n_ins)],
                                        bool(recompute), int(stream or 0))
            return int(r or 0)
        except BaseException as e:  # noqa: BLE001 - surfaced by step()
            self._error = e
            status[0] = 1
            return 0

    def _on_action(self, ctx, action, node, out, stream):
        if self._after is not None:
            try:
                self._after(int(action), int(node), int(out))
            except BaseException as e:  # noqa: BLE001
                self._error = e

    def bind(self, program, recipes: dict, host_ops: list, launches: dict):
        """recipes: node id -> list of DeltaKop; host_ops: HOST op id -> callable
        (out_ptr, in_ptrs, recompute, stream) -> scratch device pointer or 0;
        launches: node id -> (first-production, recompute) kernel launches of
        OUR kernels in its recipe."""
        kops, table = [], []
        for node, ops in sorted(recipes.items()):
            table.append(DeltaRecipe(node, len(kops), len(ops)))
            kops.extend(ops)
        karr = (DeltaKop * max(1, len(kops)))(*kops)
        tarr = (DeltaRecipe * max(1, len(table)))(*table)
        check(lib.delta_rt_bind(self._h, program._ptr, karr, len(kops), tarr, len(table)))
        self._host_ops = list(host_ops)
        self.n_actions = len(program.actions)
        acts = program.actions
        self.launches_per_step = int(
            sum(launches.get(int(a["node"]), (0, 0))[int(a["op"])] for a in acts
                if int(a["op"]) in (0, 1)))

    def _raise_pending(self):
        if self._error is not None:
            e, self._error = self._error, None
            raise e

    def step(self, stream: int, after=None):
        self._after = after
        try:
            rc = lib.delta_rt_step(self._h, stream)
        finally:
            self._after = None
        self._raise_pending()
        check(rc)

    def step_timed(self, stream: int, after=None):
        """(start_ms, end_ms) per action from the step start (NaN where untimed)."""
        a = np.full(self.n_actions, math.nan, np.float32)
        b = np.full(self.n_actions, math.nan, np.float32)
        self._after = after
        try:
            rc = lib.delta_rt_step_timed(self._h, stream, a.ctypes.data_as(C.POINTER(f32)),
                                         b.ctypes.data_as(C.POINTER(f32)), self.n_actions)
        finally:
            self._after = None
        self._raise_pending()
        check(rc)
        return a, b

    def step_observed(self, stream: int) -> np.ndarray:
        """One step with the device-side action log (delta_rt_step_observed):
        structured array of records in device arrival order."""
        cap = 2 * self.n_actions + 16
        rec = np.zeros((cap, 4), np.uint64)
        n = u64()
        rc = lib.delta_rt_step_observed(self._h, stream, rec.ctypes.data_as(C.POINTER(u64)), cap,
                                        C.byref(n))
        self._raise_pending()
        check(rc)
        rec = rec[:n.value]
        out = np.zeros(n.value, OBSERVED_DTYPE)
        out["t_ns"] = rec[:, 0]
        out["seq"] = rec[:, 1]
        out["action"] = rec[:, 2] >> 1
        out["tail"] = rec[:, 2] & 1
        out["node"] = rec[:, 3] >> 8
        out["op"] = rec[:, 3] & 0xFF
        return out

    def set_ready_nodes(self, nodes: list):
        """event i recorded after the compute action of nodes[i] (every step)"""
        arr = (u64 * max(1, len(nodes)))(*nodes)
        check(lib.delta_rt_set_ready_nodes(self._h, arr, len(nodes)))

    def wait_ready(self, stream: int, i: int):
        check(lib.delta_rt_wait_ready(self._h, stream, i))

    def measure_costs(self, stream: int, iters: int, n_nodes: int) -> np.ndarray:
        out = np.zeros(n_nodes, np.uint64)
        rc = lib.delta_rt_measure_costs(self._h, stream, iters, out.ctypes.data_as(C.POINTER(u64)),
                                        n_nodes)
        self._raise_pending()
        check(rc)
        return out

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.delta_rt_destroy(self._h)
            self._h = None

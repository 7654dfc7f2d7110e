"""ctypes wrappers for the sm_100a kernels and the swap engine
(include/delta/delta_kernels.h).  Arguments are raw device pointers (ints);
torch is only used by callers for allocation and streams.  There is no
fallback: if libdelta or a CUDA launch fails, the call raises."""
from __future__ import annotations

import ctypes as C

from ._lib import check, lib

vp, i32, i64, u32, u64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float
P = C.POINTER
_SIGS = {
    "delta_conv_create": (i32, [i32] * 9 + [vp, P(vp)]),
    "delta_conv_forward": (i32, [vp, vp, vp, vp, vp]),
    "delta_bn_stats_from_partials": (i32, [vp, i64, i32, i32, vp, vp, f32, vp, vp, f32, vp]),
    "delta_conv_geometry": (i32, [vp, P(i32), P(i32), P(i32), P(i32)]),
    "delta_conv_destroy": (None, [vp]),
    "delta_bn_workspace_floats": (i64, [i64, i32]),
    "delta_bn_stats": (i32, [vp, i64, i32, vp, vp, vp, f32, vp, vp, f32, vp]),
    "delta_bn_apply": (i32, [i32, vp, vp, vp, i64, i32] + [vp] * 8 + [vp]),
    "delta_bn_backward": (i32, [vp, i32, vp, vp, vp, i64, i32, vp, vp, vp, vp, vp, vp, vp]),
    "delta_add_grad": (i32, [vp, vp, i32, vp, vp, vp, i64, i32, vp]),
    "delta_maxpool3x3s2_fwd": (i32, [vp, vp, i32, i32, i32, i32, vp]),
    "delta_maxpool_workspace_bytes": (i64, [i32, i32, i32, i32]),
    "delta_maxpool3x3s2_bwd": (i32, [vp, vp, vp, i32, i32, i32, i32, vp, vp]),
    "delta_avgpool_fwd": (i32, [vp, vp, i32, i32, i32, vp]),
    "delta_softmax_xent": (i32, [vp, vp, vp, vp, vp, i32, i32, vp]),
    "delta_swap_create": (i32, [u64, P(vp)]),
    "delta_swap_host_ptr": (vp, [vp]),
    "delta_swap_stream": (vp, [vp, i32]),
    "delta_swap_offload": (i32, [vp, vp, u64, u64, vp]),
    "delta_swap_reload": (i32, [vp, vp, u64, u64, vp]),
    "delta_swap_destroy": (None, [vp]),
    "delta_probe_link": (i32, [u64, i32, P(C.c_double), P(C.c_double), P(C.c_double)]),
    "delta_events_create": (i32, [u32, P(vp)]),
    "delta_event_record": (i32, [vp, u32, vp]),
    "delta_event_wait": (i32, [vp, u32, vp]),
    "delta_events_destroy": (None, [vp]),
}
for _n, (_r, _a) in _SIGS.items():
    _f = getattr(lib, _n)
    _f.restype = _r
    _f.argtypes = _a

# Number of OUR kernel launches issued through this module (the bench reports
# launches per step from the delta across one captured step).
LAUNCHES = [0]


def _count(n: int):
    LAUNCHES[0] += n


class Conv:
    """tcgen05 implicit-GEMM convolution with a cached weight TMA descriptor."""

    def __init__(self, N, H, W, Cin, K, R, S, stride, pad, weight_ptr: int):
        self._h = vp()
        check(lib.delta_conv_create(N, H, W, Cin, K, R, S, stride, pad, weight_ptr,
                                    C.byref(self._h)))
        p, q, kd, tn = i32(), i32(), i32(), i32()
        lib.delta_conv_geometry(self._h, C.byref(p), C.byref(q), C.byref(kd), C.byref(tn))
        self.P, self.Q, self.kdim, self.tile_n = p.value, q.value, kd.value, tn.value
        self.shape = (N, H, W, Cin, K, R, S, stride, pad)

    def __call__(self, x_ptr: int, y_ptr: int, stream: int, stats_ptr: int | None = None):
        """stats_ptr: optional [ceil(M/128)][K] float2 BN-statistics partials."""
        check(lib.delta_conv_forward(self._h, x_ptr, y_ptr, stats_ptr, stream))
        _count(1)

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.delta_conv_destroy(self._h)
            self._h = None


def bn_workspace_floats(M: int, C_: int) -> int:
    return lib.delta_bn_workspace_floats(M, C_)


def bn_stats(x, M, C_, ws, mean, invstd, eps, run_mean, run_var, momentum, stream):
    check(lib.delta_bn_stats(x, M, C_, ws, mean, invstd, eps, run_mean, run_var, momentum, stream))
    _count(2)


def bn_stats_from_partials(partials, M, C_, mean, invstd, eps, run_mean, run_var, momentum,
                           stream, rows_per_part=128):
    check(lib.delta_bn_stats_from_partials(partials, M, C_, rows_per_part, mean, invstd, eps,
                                           run_mean, run_var, momentum, stream))
    _count(1)


def bn_apply(mode, x, res, y, M, C_, mean, invstd, gamma, beta, mean2=None, invstd2=None,
             gamma2=None, beta2=None, stream=None):
    check(lib.delta_bn_apply(mode, x, res, y, M, C_, mean, invstd, gamma, beta, mean2, invstd2,
                             gamma2, beta2, stream))
    _count(1)


def bn_backward(up, pool_hw, mask, x, dx, M, C_, mean, invstd, gamma, dgamma, dbeta, ws, stream):
    check(lib.delta_bn_backward(up, pool_hw, mask, x, dx, M, C_, mean, invstd, gamma, dgamma,
                                dbeta, ws, stream))
    _count(3)


def add_grad(a, up, pool_hw, up_mask, out_mask, out, M, C_, stream):
    """out = (a + up*[up_mask>0]) * [out_mask>0] (None masks skipped)."""
    check(lib.delta_add_grad(a, up, pool_hw, up_mask, out_mask, out, M, C_, stream))
    _count(1)


def maxpool_fwd(x, y, N, H, W, C_, stream):
    check(lib.delta_maxpool3x3s2_fwd(x, y, N, H, W, C_, stream))
    _count(1)


def maxpool_workspace_bytes(N, H, W, C_) -> int:
    return lib.delta_maxpool_workspace_bytes(N, H, W, C_)


def maxpool_bwd(dy, x, dx, N, H, W, C_, ws, stream):
    check(lib.delta_maxpool3x3s2_bwd(dy, x, dx, N, H, W, C_, ws, stream))
    _count(2)


def avgpool_fwd(x, y, N, HW, C_, stream):
    check(lib.delta_avgpool_fwd(x, y, N, HW, C_, stream))
    _count(1)


def softmax_xent(logits, labels, loss, dlogits, row_ws, N, K, stream):
    check(lib.delta_softmax_xent(logits, labels, loss, dlogits, row_ws, N, K, stream))
    _count(2)


class Swap:
    """Pinned host slab + D2H/H2D copy-engine streams (the swap engine)."""

    def __init__(self, host_bytes: int):
        self._h = vp()
        check(lib.delta_swap_create(host_bytes, C.byref(self._h)))
        self.host_ptr = lib.delta_swap_host_ptr(self._h) or 0
        self.d2h_stream = lib.delta_swap_stream(self._h, 1)
        self.h2d_stream = lib.delta_swap_stream(self._h, 2)

    def offload(self, dev_ptr, host_off, nbytes, stream=None):
        check(lib.delta_swap_offload(self._h, dev_ptr, host_off, nbytes, stream or self.d2h_stream))

    def reload(self, dev_ptr, host_off, nbytes, stream=None):
        check(lib.delta_swap_reload(self._h, dev_ptr, host_off, nbytes, stream or self.h2d_stream))

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.delta_swap_destroy(self._h)
            self._h = None


class Events:
    def __init__(self, n: int):
        self._h = vp()
        check(lib.delta_events_create(max(1, n), C.byref(self._h)))

    def record(self, i, stream):
        check(lib.delta_event_record(self._h, i, stream))

    def wait(self, i, stream):
        check(lib.delta_event_wait(self._h, i, stream))

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.delta_events_destroy(self._h)
            self._h = None


def probe_link(nbytes: int = 256 << 20, iters: int = 8):
    """Pinned host<->device bandwidth in GB/s: (h2d, d2h, duplex aggregate)."""
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    check(lib.delta_probe_link(nbytes, iters, C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, c.value

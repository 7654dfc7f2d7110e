"""ctypes wrappers for the sm_100a kernels and the swap engine
(include/delta/delta_kernels.h).  Arguments are raw device pointers (ints);
torch is only used by callers for allocation and streams.  There is no
fallback: if libdelta or a CUDA launch fails, the call raises."""
from __future__ import annotations

import ctypes as C
import os

from ._lib import check, lib

vp, i32, i64, u32, u64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float
P = C.POINTER
_SIGS = {
    "delta_conv_create": (i32, [i32] * 9 + [vp, P(vp)]),
    "delta_conv_create_ex": (i32, [i32] * 11 + [vp, P(vp)]),
    "delta_conv_create_t": (i32, [i32, i32, i32, vp, P(vp)]),
    "delta_softmax_xent_head": (i32, [vp, i32, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp]),
    "delta_conv_forward": (i32, [vp, vp, vp, vp, vp]),
    "delta_stats_parts": (i32, []),
    "delta_stats_partials_floats": (i64, [i32]),
    "delta_bn_stats_from_partials": (i32, [vp, i32, vp, vp, f32, vp, vp, f32, vp]),
    "delta_stats_col_sum": (i32, [vp, i32, vp, i32, vp]),
    "delta_parts_merge": (i32, [vp, i32, i32, vp, vp]),
    "delta_conv_forward_ex": (i32, [vp, vp, vp, vp, vp, vp]),
    "delta_conv_set_tile_n": (i32, [vp, i32]),
    "delta_wgrad_create": (i32, [i32] * 9 + [P(vp)]),
    "delta_wgrad_workspace_bytes": (u64, [vp]),
    "delta_wgrad_launches": (i32, [vp]),
    "delta_wgrad_run": (i32, [vp, vp, vp, vp, vp, vp]),
    "delta_wgrad_destroy": (None, [vp]),
    "delta_bn_backward_from_partials": (i32, [vp, vp, vp, vp, i64, i32, vp, vp, vp, vp, vp, vp]),
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
    "delta_sgd_step": (i32, [vp, vp, vp, vp, i64, i64, f32, f32, f32, vp]),
    "delta_weight_views": (i32, [vp, i32, vp]),
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


EPI_STORE, EPI_ADD_MASK, EPI_BN_BWD, EPI_SCATTER2, EPI_BIAS, EPI_GELU_BWD = 0, 1, 2, 3, 4, 5


class ConvEpilogue(C.Structure):
    """delta_conv_epilogue (include/delta/delta_kernels.h)."""
    _fields_ = [("mode", i32), ("pool_hw", i32), ("add_stride2", i32), ("scatter", i32),
                ("add", vp), ("add_mask", vp), ("out_mask", vp),
                ("xc", vp), ("mean", vp), ("invstd", vp), ("gamma", vp), ("beta", vp)]


class Conv:
    """tcgen05 implicit-GEMM convolution with a cached weight TMA descriptor."""

    def __init__(self, N, H, W, Cin, K, R, S, stride, pad, weight_ptr: int,
                 pad_end: tuple | None = None, weights_ck: bool = False):
        """pad_end = (rows, cols) of padding after the input (default: pad).
        weights_ck: a 1x1 GEMM over N rows whose weights are stored [Cin][K]
        (read MN-major: a linear layer's input gradient from the forward's
        [out][in] weights, no transposed copy)."""
        self._h = vp()
        if weights_ck:
            assert H == W == R == S == stride == 1 and pad == 0
            check(lib.delta_conv_create_t(N, Cin, K, weight_ptr, C.byref(self._h)))
        else:
            pe_h, pe_w = pad_end if pad_end is not None else (-1, -1)
            check(lib.delta_conv_create_ex(N, H, W, Cin, K, R, S, stride, pad, pe_h, pe_w,
                                           weight_ptr, C.byref(self._h)))
        p, q, kd, tn = i32(), i32(), i32(), i32()
        lib.delta_conv_geometry(self._h, C.byref(p), C.byref(q), C.byref(kd), C.byref(tn))
        self.P, self.Q, self.kdim, self.tile_n = p.value, q.value, kd.value, tn.value
        self.shape = (N, H, W, Cin, K, R, S, stride, pad)

    def __call__(self, x_ptr: int, y_ptr: int, stream: int, stats_ptr: int | None = None):
        """stats_ptr: optional BN-statistics partials, stats_partials_floats(K) floats
        (one (count, mean, M2) row per CTA)."""
        check(lib.delta_conv_forward(self._h, x_ptr, y_ptr, stats_ptr, stream))
        _count(1)

    def set_tile_n(self, tile_n: int):
        check(lib.delta_conv_set_tile_n(self._h, tile_n))
        self.tile_n = tile_n

    def add_mask(self, x_ptr, y_ptr, stream, add=None, pool_hw=0, add_mask=None, out_mask=None,
                 add_stride2=False, xc=None, partials_ptr=None):
        """y = (conv(x) + add') * [out_mask > 0]; add' = add, or the pooled add
        / pool_hw * [add_mask > 0] (add_mask is only read with a pooled add),
        or (add_stride2) an [N,P/2,Q/2,K] add placed at the even rows/columns.
        xc + partials_ptr (full add, out_mask, tile_n 64): also the per-CTA
        (sum y, sum y*xc) rows of the BN backward that consumes y."""
        e = ConvEpilogue(EPI_ADD_MASK, pool_hw, int(add_stride2), 0, add, add_mask, out_mask,
                         xc, None, None, None, None)
        check(lib.delta_conv_forward_ex(self._h, x_ptr, y_ptr, partials_ptr, C.byref(e), stream))
        _count(1)

    def scatter2(self, x_ptr, y_ptr, cls: int, stream):
        """parity class `cls` = 2a + b of a stride-2 input gradient: output
        (p, q) written to y[n][2p+a][2q+b] of the [N][2P][2Q][K] tensor."""
        e = ConvEpilogue(EPI_SCATTER2, 0, 0, cls, None, None, None, None, None, None, None, None)
        check(lib.delta_conv_forward_ex(self._h, x_ptr, y_ptr, None, C.byref(e), stream))
        _count(1)

    def bias(self, x_ptr, y_ptr, bias_ptr, stream):
        """linear layer: y = bf16(x W^T + bias) (1x1 over [rows][in])"""
        e = ConvEpilogue(EPI_BIAS, 0, 0, 0, None, None, None, None, None, None, None, bias_ptr)
        check(lib.delta_conv_forward_ex(self._h, x_ptr, y_ptr, None, C.byref(e), stream))
        _count(1)

    def gelu_bwd(self, x_ptr, y_ptr, pre_ptr, stream, stats_ptr=None):
        """y = bf16(conv(x) * gelu'(pre)): an MLP input gradient through the GELU;
        stats_ptr: per-CTA column statistics of y, stats_partials_floats(K)
        floats (stats_col_sum -> its column sums)"""
        e = ConvEpilogue(EPI_GELU_BWD, 0, 0, 0, None, None, None, pre_ptr, None, None, None, None)
        check(lib.delta_conv_forward_ex(self._h, x_ptr, y_ptr, stats_ptr, C.byref(e), stream))
        _count(1)

    def bn_bwd(self, x_ptr, g_ptr, partials_ptr, xc, mean, invstd, gamma, beta, stream):
        """g = bf16(conv(x)) * [relu(bn(xc)) > 0] and per-tile (sum g, sum g*xc)."""
        e = ConvEpilogue(EPI_BN_BWD, 0, 0, 0, None, None, None, xc, mean, invstd, gamma, beta)
        check(lib.delta_conv_forward_ex(self._h, x_ptr, g_ptr, partials_ptr, C.byref(e), stream))
        _count(1)

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.delta_conv_destroy(self._h)
            self._h = None


class Wgrad:
    """tcgen05 convolution weight gradient (fp32 KRSC, deterministic split-K)."""

    def __init__(self, N, H, W, Cin, K, R, S, stride, pad):
        self._h = vp()
        check(lib.delta_wgrad_create(N, H, W, Cin, K, R, S, stride, pad, C.byref(self._h)))
        self.workspace_bytes = int(lib.delta_wgrad_workspace_bytes(self._h))
        self.launches = int(lib.delta_wgrad_launches(self._h))

    def __call__(self, dy_ptr: int, x_ptr: int, dw_ptr: int, ws_ptr: int, stream: int):
        check(lib.delta_wgrad_run(self._h, dy_ptr, x_ptr, dw_ptr, ws_ptr, stream))
        _count(self.launches)

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.delta_wgrad_destroy(self._h)
            self._h = None


STEM_KDIM = 256


def pack_stem_weights(w_krsc, out=None):
    """[K,7,7,4] stem weights -> the pixel-pair layout the C=4 conv path reads
    ([K,256]; column (r*4+j)*8 + e*4 + c = W[k,r,2j+e-1,c], zero elsewhere;
    include/delta/delta_kernels.h).  `w_krsc` and `out` are torch tensors on
    the same device; returns `out`."""
    import torch
    K_ = w_krsc.shape[0]
    if out is None:
        out = torch.zeros(K_, STEM_KDIM, dtype=torch.bfloat16, device=w_krsc.device)
    w8 = torch.zeros(K_, 7, 8, 4, dtype=out.dtype, device=w_krsc.device)
    w8[:, :, 1:] = w_krsc                      # s' = s + 1; s' = 0 is the zero tap
    out[:, :224].copy_(w8.reshape(K_, 224))    # [K,7,4(j),2(e),4(c)] row-major
    out[:, 224:].zero_()
    return out


def bn_workspace_floats(M: int, C_: int) -> int:
    return lib.delta_bn_workspace_floats(M, C_)


# bn_pool.cu bn_bwd_one_launch(): the streaming BN backward as one persistent launch
BN_BWD_ONE_LAUNCH = os.environ.get("DELTA_BN_BWD_GRID", "1") != "0"


def _merge_launches(parts: int) -> int:
    """Launches of a fixed-order partials merge (bn_pool.cu merge_partials /
    bn_backward): a grouping pass above GROUP_ABOVE = 4096 partials."""
    return 2 if parts > 4096 else 1


def _chunks(M: int, C_: int) -> int:
    """Number of reduction chunks of the streaming BN kernels (bn_pool.cu chunk_rows)."""
    rows = (M + 148 * 8 - 1) // (148 * 8)
    rows = max(16, (rows + 15) // 16 * 16)
    return (M + rows - 1) // rows


def bn_stats(x, M, C_, ws, mean, invstd, eps, run_mean, run_var, momentum, stream):
    check(lib.delta_bn_stats(x, M, C_, ws, mean, invstd, eps, run_mean, run_var, momentum, stream))
    _count(1 + _merge_launches(_chunks(M, C_)))


def stats_parts() -> int:
    """Partial rows a conv epilogue writes (one per CTA = one per SM)."""
    return int(lib.delta_stats_parts())


def stats_partials_floats(C_: int) -> int:
    return int(lib.delta_stats_partials_floats(C_))


def parts_merge(ws, parts, cols, out, stream):
    """out[c] = sum_p ws[p*cols + c] in order of p"""
    check(lib.delta_parts_merge(ws, parts, cols, out, stream))
    _count(1)


def stats_col_sum(partials, C_, out, stream, accumulate=False):
    check(lib.delta_stats_col_sum(partials, C_, out, int(accumulate), stream))
    _count(1)


def bn_stats_from_partials(partials, C_, mean, invstd, eps, run_mean, run_var, momentum, stream):
    check(lib.delta_bn_stats_from_partials(partials, C_, mean, invstd, eps, run_mean, run_var,
                                           momentum, stream))
    _count(1)


def bn_apply(mode, x, res, y, M, C_, mean, invstd, gamma, beta, mean2=None, invstd2=None,
             gamma2=None, beta2=None, stream=None):
    check(lib.delta_bn_apply(mode, x, res, y, M, C_, mean, invstd, gamma, beta, mean2, invstd2,
                             gamma2, beta2, stream))
    _count(1)


VIEW_DGRAD, VIEW_STEM, VIEW_DGRAD_S2 = 0, 1, 2


class WeightView(C.Structure):
    """delta_weight_view (include/delta/delta_kernels.h)."""
    _fields_ = [("kind", i32), ("K", i32), ("R", i32), ("S", i32), ("C", i32),
                ("reserved", i32), ("src", vp), ("dst", vp)]


def sgd_step(w, mom, g, wbf, n, n_bf, lr, momentum, weight_decay, stream):
    """One fused SGD pass over the flat fp32 buffers (+ bf16 copy of the first n_bf)."""
    check(lib.delta_sgd_step(w, mom, g, wbf, n, n_bf, lr, momentum, weight_decay, stream))
    _count(1)


def weight_views(table_dev, n, stream):
    """All derived bf16 weight tensors (transposed dgrad / pixel-pair stem) in one launch;
    `table_dev` = device copy of a WeightView array."""
    check(lib.delta_weight_views(table_dev, n, stream))
    _count(1 if n else 0)


def bn_backward(up, pool_hw, mask, x, dx, M, C_, mean, invstd, gamma, dgamma, dbeta, ws, stream):
    check(lib.delta_bn_backward(up, pool_hw, mask, x, dx, M, C_, mean, invstd, gamma, dgamma,
                                dbeta, ws, stream))
    _count(1 if BN_BWD_ONE_LAUNCH else 2 + _merge_launches(_chunks(M, C_)))


def bn_backward_from_partials(partials, g, x, dx, M, C_, mean, invstd, gamma, dgamma, dbeta,
                              stream):
    check(lib.delta_bn_backward_from_partials(partials, g, x, dx, M, C_, mean, invstd, gamma,
                                              dgamma, dbeta, stream))
    _count(2)


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


def softmax_xent_head(logits, ld, bias, labels, loss, dlogits, dl_bf16, dbias, row_ws, N, K,
                      stream):
    check(lib.delta_softmax_xent_head(logits, ld, bias, labels, loss, dlogits, dl_bf16, dbias,
                                      row_ws, N, K, stream))
    _count(3)


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


# ---------------------------------------------------------------- transformer
# (include/delta/delta_xformer.h)
_XSIGS = {
    "delta_layernorm_fwd": (i32, [vp, vp, vp, vp, vp, vp, i64, i32, f32, vp]),
    "delta_layernorm_bwd_workspace_floats": (i64, [i64, i32]),
    "delta_layernorm_bwd": (i32, [vp] * 10 + [i64, i32, vp]),
    "delta_layernorm_bwd_drop": (i32, [vp] * 10 + [i64, i32, vp, vp, f32, vp, u32, vp]),
    "delta_gelu_fwd": (i32, [vp, vp, i64, vp]),
    "delta_add_dropout": (i32, [vp, vp, vp, i64, f32, vp, u32, vp]),
    "delta_dropout_bwd": (i32, [vp, vp, i64, f32, vp, u32, vp]),
    "delta_colsum_workspace_floats": (i64, [i64, i32]),
    "delta_colsum": (i32, [vp, i64, i32, vp, i32, vp, vp, i32, vp]),
    "delta_embed_fwd": (i32, [vp, vp, vp, vp, vp, vp, i32, i32, i32, f32, vp, u32, vp]),
    "delta_embed_grads": (i32, [vp, vp, vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp]),
    "delta_span_head_fwd": (i32, [vp] * 8 + [i32, i32, i32, vp]),
    "delta_span_head_workspace_floats": (i64, [i64, i32]),
    "delta_span_head_bwd": (i32, [vp] * 7 + [i64, i32, vp]),
    "delta_attention_fwd": (i32, [vp, vp, vp, i32, i32, i32, f32, vp, u32, vp]),
    "delta_attention_bwd": (i32, [vp] * 6 + [i32, i32, i32, f32, vp, u32, vp, vp, vp]),
    "delta_adamw_step": (i32, [vp] * 5 + [i64, i64, f32, f32, f32, f32, f32, vp, vp]),
}
for _n, (_r, _a) in _XSIGS.items():
    _f = getattr(lib, _n)
    _f.restype = _r
    _f.argtypes = _a


def layernorm_fwd(x, y, mean, rstd, gamma, beta, rows, H, eps, stream):
    check(lib.delta_layernorm_fwd(x, y, mean, rstd, gamma, beta, rows, H, eps, stream))
    _count(1)


def layernorm_bwd_workspace_floats(rows, H) -> int:
    return int(lib.delta_layernorm_bwd_workspace_floats(rows, H))


def layernorm_bwd(dy, x, dres, dx, mean, rstd, gamma, dgamma, dbeta, ws, rows, H, stream):
    check(lib.delta_layernorm_bwd(dy, x, dres, dx, mean, rstd, gamma, dgamma, dbeta, ws, rows, H,
                                  stream))
    _count(2)


def layernorm_bwd_drop(dy, x, dres, dx, mean, rstd, gamma, dgamma, dbeta, ws, rows, H, dxd, dbias,
                       p, rng, tag, stream):
    """layernorm_bwd + dxd = dropout_bwd(dx; p, tag), dbias = colsum(dxd)"""
    check(lib.delta_layernorm_bwd_drop(dy, x, dres, dx, mean, rstd, gamma, dgamma, dbeta, ws, rows,
                                       H, dxd, dbias, p, rng, tag, stream))
    _count(2)


def gelu_fwd(x, y, n, stream):
    check(lib.delta_gelu_fwd(x, y, n, stream))
    _count(1)


def add_dropout(a, b, y, n, p, rng, tag, stream):
    check(lib.delta_add_dropout(a, b, y, n, p, rng, tag, stream))
    _count(1)


def dropout_bwd(dy, dx, n, p, rng, tag, stream):
    check(lib.delta_dropout_bwd(dy, dx, n, p, rng, tag, stream))
    _count(1)


def colsum_workspace_floats(rows, cols) -> int:
    return int(lib.delta_colsum_workspace_floats(rows, cols))


def colsum(x, rows, cols, out, ws, stream, sel=None, sel_val=0, accumulate=False):
    check(lib.delta_colsum(x, rows, cols, sel, sel_val, out, ws, int(accumulate), stream))
    _count(2)


def embed_fwd(ids, types, word, pos, type_, y, B, S, H, p, rng, tag, stream):
    check(lib.delta_embed_fwd(ids, types, word, pos, type_, y, B, S, H, p, rng, tag, stream))
    _count(1)


def embed_grads(dsum, csr, types, B, S, H, vocab, n_types, dword, dpos, dtype, ws, stream):
    check(lib.delta_embed_grads(dsum, csr, types, B, S, H, vocab, n_types, dword, dpos, dtype, ws,
                                stream))
    _count(2 + 2 * n_types)


def span_head_fwd(h, w, bias, label, logits, dlogits, row_loss, loss, B, S, H, stream):
    check(lib.delta_span_head_fwd(h, w, bias, label, logits, dlogits, row_loss, loss, B, S, H,
                                  stream))
    _count(2)


def span_head_workspace_floats(T, H) -> int:
    return int(lib.delta_span_head_workspace_floats(T, H))


def span_head_bwd(h, dlogits, w, dh, dw, dbias, ws, T, H, stream):
    check(lib.delta_span_head_bwd(h, dlogits, w, dh, dw, dbias, ws, T, H, stream))
    _count(3)


def attention_fwd(qkv, out, lse, B, S, heads, p, rng, tag, stream):
    check(lib.delta_attention_fwd(qkv, out, lse, B, S, heads, p, rng, tag, stream))
    _count(1)


def attention_bwd(qkv, out, dout, lse, D, dqkv, B, S, heads, p, rng, tag, stream, dbias=None,
                  ws=None):
    """dbias (fp32 [3*heads*64]) = column sums of dqkv when given; ws fp32 [B][3*heads*64]"""
    check(lib.delta_attention_bwd(qkv, out, dout, lse, D, dqkv, B, S, heads, p, rng, tag, dbias, ws,
                                  stream))
    _count(2)


def adamw_step(w, m, v, g, wbf, n, n_bf, lr, b1, b2, eps, wd, rng, stream):
    check(lib.delta_adamw_step(w, m, v, g, wbf, n, n_bf, lr, b1, b2, eps, wd, rng, stream))
    _count(2)

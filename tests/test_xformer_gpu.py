"""GPU parity of the transformer (BERT) kernels (include/delta/delta_xformer.h)
against plain PyTorch fp32 references of the same op, with the dropout masks
reconstructed on the host from the same Philox stream (tests/xf_ref.py), and
bitwise determinism (a recompute must reproduce the retained tensor).
Tolerances: bf16 output rounding (2^-8 relative) plus fp32 reduction-order
noise, stated per test."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import xf_ref as R  # noqa: E402  (tests/ is on sys.path via conftest)

pytestmark = pytest.mark.gpu

from paper_2203_15980_b200 import kernels as K  # noqa: E402

dev = "cuda"
SEED, STEP = 0x1234_5678_9ABC, 3


def _st():
    return torch.cuda.current_stream().cuda_stream


def _rng():
    return torch.tensor([SEED, STEP], dtype=torch.int64, device=dev)


def close(got, ref, rel=1e-2, absr=2e-2):
    got, ref = got.float(), ref.float()
    err = (got - ref).abs()
    tol = rel * ref.abs() + absr * ref.pow(2).mean().sqrt() + 1e-6
    assert bool((err <= tol).all()), f"max err {err.max().item():.4g} (rms ref {ref.pow(2).mean().sqrt().item():.4g})"


def rnd(*shape, scale=1.0, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    return (torch.randn(*shape, device=dev, generator=g) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("H,rows", [(256, 1000), (1024, 1000), (1024, 16384)])
def test_layernorm_fwd_bwd(H, rows):
    # 16384 rows: every warp walks several staged rows (stage refills)
    x = rnd(rows, H, scale=2.0)
    gamma = torch.rand(H, device=dev) + 0.5
    beta = torch.randn(H, device=dev) * 0.1
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=dev)
    rstd = torch.empty(rows, device=dev)
    K.layernorm_fwd(x.data_ptr(), y.data_ptr(), mean.data_ptr(), rstd.data_ptr(), gamma.data_ptr(),
                    beta.data_ptr(), rows, H, 1e-12, _st())
    xr = x.float().requires_grad_(True)
    gr = gamma.clone().requires_grad_(True)
    br = beta.clone().requires_grad_(True)
    ref = F.layer_norm(xr, (H,), gr, br, 1e-12)
    close(y, ref)
    close(mean, x.float().mean(-1), 1e-5, 1e-5)
    # backward with a residual gradient added
    dy = rnd(rows, H, seed=1)
    dres = rnd(rows, H, seed=2)
    ref.backward(dy.float())
    dx = torch.empty_like(x)
    dg = torch.empty(H, device=dev)
    db = torch.empty(H, device=dev)
    ws = torch.empty(K.layernorm_bwd_workspace_floats(rows, H), device=dev)
    K.layernorm_bwd(dy.data_ptr(), x.data_ptr(), dres.data_ptr(), dx.data_ptr(), mean.data_ptr(),
                    rstd.data_ptr(), gamma.data_ptr(), dg.data_ptr(), db.data_ptr(), ws.data_ptr(),
                    rows, H, _st())
    close(dx, xr.grad + dres.float())
    close(dg, gr.grad, 1e-3, 1e-3)
    close(db, br.grad, 1e-3, 1e-3)
    # deterministic
    dx2 = torch.empty_like(x)
    dg2 = torch.empty(H, device=dev)
    K.layernorm_bwd(dy.data_ptr(), x.data_ptr(), dres.data_ptr(), dx2.data_ptr(), mean.data_ptr(),
                    rstd.data_ptr(), gamma.data_ptr(), dg2.data_ptr(), db.data_ptr(), ws.data_ptr(),
                    rows, H, _st())
    assert torch.equal(dx, dx2) and torch.equal(dg, dg2)
    # fused with the residual branch's dropout backward and its bias gradient:
    # dx, dgamma, dbeta unchanged; dxd == dropout_bwd(dx) bit for bit; dbias ==
    # the column sums of dxd
    for p in (0.1, 0.0):
        rng = _rng()
        dx3, dxd, dxd_ref = (torch.empty_like(x) for _ in range(3))
        dg3, db3, dbias = (torch.empty(H, device=dev) for _ in range(3))
        K.layernorm_bwd_drop(dy.data_ptr(), x.data_ptr(), dres.data_ptr(), dx3.data_ptr(),
                             mean.data_ptr(), rstd.data_ptr(), gamma.data_ptr(), dg3.data_ptr(),
                             db3.data_ptr(), ws.data_ptr(), rows, H, dxd.data_ptr(),
                             dbias.data_ptr(), p, rng.data_ptr(), 7, _st())
        assert torch.equal(dx3, dx) and torch.equal(dg3, dg) and torch.equal(db3, db)
        K.dropout_bwd(dx.data_ptr(), dxd_ref.data_ptr(), rows * H, p, rng.data_ptr(), 7, _st())
        assert torch.equal(dxd, dxd_ref)
        close(dbias, dxd_ref.double().sum(0).float(), 1e-4, 1e-4)


def test_gelu_fwd():
    x = rnd(4096, 512, scale=3.0)
    y = torch.empty_like(x)
    K.gelu_fwd(x.data_ptr(), y.data_ptr(), x.numel(), _st())
    close(y, F.gelu(x.float()))


@pytest.mark.parametrize("p", [0.0, 0.1])
def test_add_dropout_and_backward_share_the_mask(p):
    n = 64 * 1024
    a, b = rnd(n, seed=3), rnd(n, seed=4)
    y = torch.empty_like(a)
    rng = _rng()
    K.add_dropout(a.data_ptr(), b.data_ptr(), y.data_ptr(), n, p, rng.data_ptr(), 7, _st())
    keep = torch.from_numpy(R.keep_mask(n, p, SEED, STEP, 7)).to(dev)
    sc = R.drop_scale(p)
    ref = a.float() + torch.where(keep, b.float() * sc, torch.zeros_like(b.float()))
    close(y, ref, 1e-2, 1e-3)
    if p:
        assert abs(keep.float().mean().item() - (1 - R.drop_thr(p) / 256)) < 0.01
    dy = rnd(n, seed=5)
    dx = torch.empty_like(dy)
    K.dropout_bwd(dy.data_ptr(), dx.data_ptr(), n, p, rng.data_ptr(), 7, _st())
    close(dx, torch.where(keep, dy.float() * sc, torch.zeros_like(dy.float())), 1e-2, 1e-3)
    # another step draws another mask; the same step redraws the same one
    y2 = torch.empty_like(y)
    K.add_dropout(a.data_ptr(), b.data_ptr(), y2.data_ptr(), n, p, rng.data_ptr(), 7, _st())
    assert torch.equal(y, y2)
    if p:
        rng[1] += 1
        K.add_dropout(a.data_ptr(), b.data_ptr(), y2.data_ptr(), n, p, rng.data_ptr(), 7, _st())
        assert not torch.equal(y, y2)


def test_colsum_with_row_select():
    rows, cols = 3000, 1024
    x = rnd(rows, cols)
    sel = torch.randint(0, 2, (rows,), device=dev, dtype=torch.int32)
    out = torch.empty(cols, device=dev)
    ws = torch.empty(K.colsum_workspace_floats(rows, cols), device=dev)
    K.colsum(x.data_ptr(), rows, cols, out.data_ptr(), ws.data_ptr(), _st())
    close(out, x.float().sum(0), 1e-4, 1e-4)
    K.colsum(x.data_ptr(), rows, cols, out.data_ptr(), ws.data_ptr(), _st(), sel=sel.data_ptr(),
             sel_val=1)
    close(out, x.float()[sel == 1].sum(0), 1e-4, 1e-4)


def _linear(M, Cin, Cout, w):
    return K.Conv(M, 1, 1, Cin, Cout, 1, 1, 1, 0, w.data_ptr())


@pytest.mark.parametrize("shape", [(4096, 1024, 3072), (1000, 1024, 1024), (4096, 4096, 1024)])
def test_linear_bias_epilogue(shape):
    M, Cin, Cout = shape
    x = rnd(M, Cin)
    w = rnd(Cout, Cin, scale=Cin ** -0.5, seed=1)
    b = torch.randn(Cout, device=dev)
    y = torch.empty(M, Cout, device=dev, dtype=torch.bfloat16)
    _linear(M, Cin, Cout, w).bias(x.data_ptr(), y.data_ptr(), b.data_ptr(), _st())
    close(y, x.float() @ w.float().t() + b)


@pytest.mark.parametrize("M,tile_n", [(2048, 128), (256, 128), (2048, 64), (1000, 64)])
def test_linear_gelu_backward_epilogue(M, tile_n):
    # CTA-pair tiles (2048 x 128), single-CTA tiles (few tiles), 64-column
    # tiles; the gelu' operand transform runs in all of them
    Cin, Cout = 1024, 4096   # dgrad of MlpDown: [M][1024] x W2 -> [M][4096]
    dy = rnd(M, Cin)
    wt = rnd(Cout, Cin, scale=Cin ** -0.5, seed=1)     # transposed W2 ([4096][1024])
    pre = rnd(M, Cout, scale=2.0, seed=2)
    conv = _linear(M, Cin, Cout, wt)
    conv.set_tile_n(tile_n)
    y = torch.empty(M, Cout, device=dev, dtype=torch.bfloat16)
    conv.gelu_bwd(dy.data_ptr(), y.data_ptr(), pre.data_ptr(), _st())
    pr = pre.float().requires_grad_(True)
    F.gelu(pr).backward(dy.float() @ wt.float().t())
    close(y, pr.grad)


@pytest.mark.parametrize("mode", ["store", "gelu_bwd"])
def test_linear_input_gradient_from_forward_weights(mode):
    """delta_conv_create_t: the input-gradient GEMM reads the forward weights
    [out][in] through MN-major descriptors — same result as the transposed
    copy, bit for bit, and vs fp32 torch"""
    M, out_f, in_f = 4096, 1024, 4096
    dy = rnd(M, out_f)
    w = rnd(out_f, in_f, scale=out_f ** -0.5, seed=1)          # forward weights [out][in]
    wt = w.t().contiguous()                                      # the transposed copy [in][out]
    pre = rnd(M, in_f, scale=2.0, seed=2)
    c_t = K.Conv(M, 1, 1, out_f, in_f, 1, 1, 1, 0, w.data_ptr(), weights_ck=True)
    c_c = _linear(M, out_f, in_f, wt)
    if mode == "gelu_bwd":
        c_t.set_tile_n(128)
        c_c.set_tile_n(128)
    y_t = torch.empty(M, in_f, device=dev, dtype=torch.bfloat16)
    y_c = torch.empty_like(y_t)
    if mode == "store":
        c_t(dy.data_ptr(), y_t.data_ptr(), _st())
        c_c(dy.data_ptr(), y_c.data_ptr(), _st())
        ref = dy.float() @ w.float()
    else:
        c_t.gelu_bwd(dy.data_ptr(), y_t.data_ptr(), pre.data_ptr(), _st())
        c_c.gelu_bwd(dy.data_ptr(), y_c.data_ptr(), pre.data_ptr(), _st())
        pr = pre.float().requires_grad_(True)
        F.gelu(pr).backward(dy.float() @ w.float())
        ref = pr.grad
    close(y_t, ref)
    assert torch.equal(y_t, y_c)


@pytest.mark.parametrize("M", [4096, 1000])
def test_gelu_bwd_column_statistics(M):
    """EPI_GELU_BWD with per-CTA column statistics: stats_col_sum of them is
    the column sums of the stored output (the up projection's bias
    gradient); the output itself is unchanged by computing them"""
    out_f, in_f = 1024, 4096
    dy = rnd(M, out_f)
    w = rnd(out_f, in_f, scale=out_f ** -0.5, seed=1)
    pre = rnd(M, in_f, scale=2.0, seed=2)
    c = K.Conv(M, 1, 1, out_f, in_f, 1, 1, 1, 0, w.data_ptr(), weights_ck=True)
    c.set_tile_n(128)
    y0 = torch.empty(M, in_f, device=dev, dtype=torch.bfloat16)
    c.gelu_bwd(dy.data_ptr(), y0.data_ptr(), pre.data_ptr(), _st())
    y = torch.empty_like(y0)
    ws = torch.full((K.stats_partials_floats(in_f),), float("nan"), device=dev)
    c.gelu_bwd(dy.data_ptr(), y.data_ptr(), pre.data_ptr(), _st(), stats_ptr=ws.data_ptr())
    assert torch.equal(y, y0)
    out = torch.empty(in_f, device=dev)
    K.stats_col_sum(ws.data_ptr(), in_f, out.data_ptr(), _st())
    close(out, y.double().sum(0).float(), 1e-4, 1e-4)
    out2 = torch.empty_like(out)
    c.gelu_bwd(dy.data_ptr(), y.data_ptr(), pre.data_ptr(), _st(), stats_ptr=ws.data_ptr())
    K.stats_col_sum(ws.data_ptr(), in_f, out2.data_ptr(), _st())
    assert torch.equal(out, out2)


def test_parts_merge():
    """delta_parts_merge: column sums of partial rows in row order"""
    parts, cols = 37, 3000
    ws = torch.randn(parts, cols, device=dev)
    out = torch.empty(cols, device=dev)
    K.parts_merge(ws.data_ptr(), parts, cols, out.data_ptr(), _st())
    close(out, ws.double().sum(0).float(), 1e-5, 1e-5)


def _attn_inputs(B, S, heads, seed=0):
    return rnd(B * S, 3 * heads * 64, seed=seed)


@pytest.mark.parametrize("B,S,heads,p", [(2, 512, 4, 0.0), (2, 256, 3, 0.0), (1, 128, 2, 0.0),
                                         (2, 512, 2, 0.1), (3, 384, 2, 0.1),
                                         # more work items than SMs: the persistent forward
                                         # walks several per CTA (next item prefetched),
                                         # incl. one-tile items (S = 384)
                                         (8, 512, 16, 0.1), (20, 384, 16, 0.1)])
def test_attention_forward_backward(B, S, heads, p):
    Hd = heads * 64
    qkv = _attn_inputs(B, S, heads)
    out = torch.empty(B * S, Hd, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(B * heads * S, device=dev)
    rng = _rng()
    K.attention_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), B, S, heads, p, rng.data_ptr(),
                    11, _st())
    keep = None
    if p:
        keep = torch.from_numpy(R.keep_mask(B * heads * S * S, p, SEED, STEP, 11)).to(dev)
        keep = keep.view(B, heads, S, S).float()
    qr = qkv.float().requires_grad_(True)
    ref = R.attention_ref(qr, B, S, heads, keep, R.drop_scale(p))
    close(out, ref)
    # lse (log2 units of the scaled scores)
    x = qkv.float().view(B, S, 3, heads, 64)
    s = torch.einsum("bqhd,bkhd->bhqk", x[:, :, 0], x[:, :, 1]) / 8.0
    close(lse.view(B, heads, S), torch.logsumexp(s, -1) * 1.4426950408889634, 1e-4, 1e-4)
    # deterministic (the recompute contract)
    out2 = torch.empty_like(out)
    K.attention_fwd(qkv.data_ptr(), out2.data_ptr(), lse.data_ptr(), B, S, heads, p, rng.data_ptr(),
                    11, _st())
    assert torch.equal(out, out2)
    # backward
    dout = rnd(B * S, Hd, seed=9)
    ref.backward(dout.float())
    dqkv = torch.empty_like(qkv)
    D = torch.empty(B * heads * S, device=dev)
    K.attention_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), D.data_ptr(),
                    dqkv.data_ptr(), B, S, heads, p, rng.data_ptr(), 11, _st())
    g = qr.grad.view(B * S, 3, Hd)
    got = dqkv.view(B * S, 3, Hd)
    for i, name in enumerate("qkv"):
        # dQ/dK/dV: bf16 P and dS operands on the tensor cores -> looser tolerance
        close(got[:, i], g[:, i], 3e-2, 3e-2)
    # with the QKV bias gradient reduced in the kernel: dqkv unchanged, the
    # column sums match the fp32 reference's, and are deterministic
    dqkv2 = torch.empty_like(dqkv)
    db = torch.empty(3 * Hd, device=dev)
    ws = torch.empty(B * 3 * Hd, device=dev)
    dbs = []
    for _ in range(2):
        K.attention_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                        D.data_ptr(), dqkv2.data_ptr(), B, S, heads, p, rng.data_ptr(), 11, _st(),
                        db.data_ptr(), ws.data_ptr())
        assert torch.equal(dqkv, dqkv2)
        dbs.append(db.clone())
    assert torch.equal(dbs[0], dbs[1])
    close(db, qr.grad.view(B * S, 3 * Hd).sum(0), 3e-2, 3e-2)


def test_embeddings_forward_and_table_gradients():
    B, S, H, V = 4, 128, 256, 1000
    g = torch.Generator().manual_seed(0)
    ids = torch.randint(0, V, (B * S,), generator=g, dtype=torch.int32)
    ids[:40] = 5  # repeated ids
    types = torch.randint(0, 2, (B * S,), generator=g, dtype=torch.int32)
    word, pos, typ = rnd(V, H, seed=1), rnd(512, H, seed=2), rnd(2, H, seed=3)
    y = torch.empty(B * S, H, device=dev, dtype=torch.bfloat16)
    rng = _rng()
    ids_d, types_d = ids.to(dev), types.to(dev)
    K.embed_fwd(ids_d.data_ptr(), types_d.data_ptr(), word.data_ptr(), pos.data_ptr(), typ.data_ptr(),
                y.data_ptr(), B, S, H, 0.1, rng.data_ptr(), 5, _st())
    keep = torch.from_numpy(R.keep_mask(B * S * H, 0.1, SEED, STEP, 5)).to(dev).view(B * S, H)
    s = word.float()[ids.long()] + pos.float()[torch.arange(B * S) % S] + typ.float()[types.long()]
    close(y, torch.where(keep, s * R.drop_scale(0.1), torch.zeros_like(s)))
    # gradients of the tables from d(sum)
    from paper_2203_15980_b200.bert import token_csr
    csr = torch.from_numpy(token_csr(ids.numpy())).to(dev)
    dsum = rnd(B * S, H, seed=4)
    dword = torch.empty(V, H, device=dev)
    dpos = torch.empty(S, H, device=dev)
    dtyp = torch.empty(2, H, device=dev)
    ws = torch.empty(K.colsum_workspace_floats(B * S, H), device=dev)
    K.embed_grads(dsum.data_ptr(), csr.data_ptr(), types_d.data_ptr(), B, S, H, V, 2,
                  dword.data_ptr(), dpos.data_ptr(), dtyp.data_ptr(), ws.data_ptr(), _st())
    ref_w = torch.zeros(V, H, device=dev).index_add_(0, ids.long().to(dev), dsum.float())
    close(dword, ref_w, 1e-4, 1e-4)
    close(dpos, dsum.float().view(B, S, H).sum(0), 1e-4, 1e-4)
    close(dtyp, torch.stack([dsum.float()[types_d == j].sum(0) for j in range(2)]), 1e-4, 1e-4)


def test_span_head_forward_backward():
    B, S, H = 3, 256, 1024
    h = rnd(B * S, H)
    w = torch.randn(2, H, device=dev) * 0.02
    bias = torch.randn(2, device=dev)
    label = torch.randint(0, S, (B, 2), device=dev, dtype=torch.int32)
    logits = torch.empty(B * S, 2, device=dev)
    dl = torch.empty(B * S, 2, device=dev)
    rl = torch.empty(B, device=dev)
    loss = torch.empty(1, device=dev)
    K.span_head_fwd(h.data_ptr(), w.data_ptr(), bias.data_ptr(), label.data_ptr(), logits.data_ptr(),
                    dl.data_ptr(), rl.data_ptr(), loss.data_ptr(), B, S, H, _st())
    hr = h.float().requires_grad_(True)
    wr = w.clone().requires_grad_(True)
    br = bias.clone().requires_grad_(True)
    z = (hr @ wr.t() + br).view(B, S, 2)
    ref = 0.5 * (F.cross_entropy(z[..., 0], label[:, 0].long()) +
                 F.cross_entropy(z[..., 1], label[:, 1].long()))
    close(logits, z.reshape(-1, 2), 1e-4, 1e-4)
    assert abs(loss.item() - ref.item()) < 1e-4 * max(1.0, abs(ref.item()))
    ref.backward()
    dh = torch.empty_like(h)
    dw = torch.empty(2, H, device=dev)
    db = torch.empty(2, device=dev)
    ws = torch.empty(K.span_head_workspace_floats(B * S, H), device=dev)
    K.span_head_bwd(h.data_ptr(), dl.data_ptr(), w.data_ptr(), dh.data_ptr(), dw.data_ptr(),
                    db.data_ptr(), ws.data_ptr(), B * S, H, _st())
    close(dh, hr.grad)
    close(dw, wr.grad, 1e-3, 1e-3)
    close(db, br.grad, 1e-3, 1e-3)


def test_adamw_step_matches_torch():
    n, n_bf = 10_000, 6_000
    w = torch.randn(n, device=dev)
    g = torch.randn(n, device=dev)
    m, v = torch.zeros(n, device=dev), torch.zeros(n, device=dev)
    wbf = torch.empty(n_bf, device=dev, dtype=torch.bfloat16)
    rng = torch.tensor([1, 0], dtype=torch.int64, device=dev)
    p_ref = [w[:n_bf].clone().requires_grad_(True), w[n_bf:].clone().requires_grad_(True)]
    opt = torch.optim.AdamW([{"params": [p_ref[0]], "weight_decay": 0.01},
                             {"params": [p_ref[1]], "weight_decay": 0.0}], lr=1e-3,
                            betas=(0.9, 0.999), eps=1e-6)
    for _ in range(3):
        K.adamw_step(w.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), wbf.data_ptr(), n, n_bf,
                     1e-3, 0.9, 0.999, 1e-6, 0.01, rng.data_ptr(), _st())
        p_ref[0].grad, p_ref[1].grad = g[:n_bf].clone(), g[n_bf:].clone()
        opt.step()
    assert rng[1].item() == 3
    close(w, torch.cat([p_ref[0].detach(), p_ref[1].detach()]), 1e-5, 1e-5)
    assert torch.equal(wbf, w[:n_bf].to(torch.bfloat16))

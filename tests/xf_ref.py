"""Test-side references for the transformer kernels: a numpy Philox4x32-10
(the dropout masks of include/delta/delta_xformer.h, so the fp32 torch
references can apply exactly the mask the GPU drew) and fp32 torch versions
of the ops."""
from __future__ import annotations

import numpy as np
import torch

M0, M1, W0, W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """vectorised over numpy uint32 arrays (counters); keys scalar"""
    c0, c1, c2, c3 = (np.asarray(c, np.uint64) for c in (c0, c1, c2, c3))
    k0, k1 = np.uint64(k0), np.uint64(k1)
    mask = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = np.uint64(M0) * c0
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & mask
        hi1, lo1 = p1 >> np.uint64(32), p1 & mask
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & mask, lo1, (hi0 ^ c3 ^ k1) & mask, lo0
        k0 = (k0 + np.uint64(W0)) & mask
        k1 = (k1 + np.uint64(W1)) & mask
    return c0, c1, c2, c3


def drop_thr(p: float) -> int:
    return min(255, max(0, int(p * 256.0 + 0.5)))


def keep_mask(n: int, p: float, seed: int, step: int, tag: int) -> np.ndarray:
    """bool keep mask of elements 0..n-1 of dropout site `tag` (philox.cuh)"""
    thr = drop_thr(p)
    if thr == 0:
        return np.ones(n, bool)
    g = np.arange((n + 15) // 16, dtype=np.uint64)
    words = philox4x32_10(g & np.uint64(0xFFFFFFFF), g >> np.uint64(32), np.full_like(g, tag),
                          np.full_like(g, step & 0xFFFFFFFF), seed & 0xFFFFFFFF,
                          ((seed >> 32) ^ (step >> 32)) & 0xFFFFFFFF)
    b = np.stack(words, 1).astype(np.uint32).view(np.uint8).reshape(-1)  # little endian bytes
    return b[:n] >= thr


def drop_scale(p: float) -> float:
    t = drop_thr(p)
    return 256.0 / (256 - t)


def attention_ref(qkv, B, S, heads, keep=None, scale_drop=1.0):
    """fp32 attention of a bf16 qkv [B*S][3*heads*64]; keep: [B, heads, S, S]"""
    Hd = heads * 64
    x = qkv.float().view(B, S, 3, heads, 64)
    q, k, v = (x[:, :, i].permute(0, 2, 1, 3) for i in range(3))  # [B, h, S, 64]
    s = q @ k.transpose(-1, -2) / 8.0
    p = torch.softmax(s, -1)
    if keep is not None:
        p = p * keep * scale_drop
    o = p @ v
    return o.permute(0, 2, 1, 3).reshape(B * S, Hd)


def bert_ref_loss(rt, batch, step: int | None = None):
    """fp32 torch forward of the BertRuntime's model (same fp32 master
    parameters, same dropout masks drawn from the host Philox) -> (loss,
    {param name: leaf tensor with .grad after loss.backward()})."""
    import torch.nn.functional as F
    from paper_2203_15980_b200.bert import EMBED_TAG, drop_tag
    cfg = rt.cfg
    B, S, H, nh = cfg.batch, cfg.seq, cfg.hidden, cfg.heads
    T = B * S
    seed = int(rt.rng[0].item())
    step = int(rt.rng[1].item()) if step is None else step
    dev = rt.params.master.device
    leaves = {n: v.detach().clone().requires_grad_(True) for n, v in rt.params.views.items()}
    ids, types, labels = (t.to(dev).long() for t in batch[:3])

    def mask(n, p, tag, shape):
        return torch.from_numpy(keep_mask(n, p, seed, step, tag)).to(dev).view(shape).float()

    ph, pa = cfg.p_hidden, cfg.p_attn
    x = leaves["word"][ids] + leaves["pos"][torch.arange(T, device=dev) % S] + leaves["type"][types]
    x = x * mask(T * H, ph, EMBED_TAG, (T, H)) * drop_scale(ph)
    lin = lambda name, a: a @ leaves["w:" + name].t() + leaves["b:" + name]
    ln = lambda name, a: F.layer_norm(a, (H,), leaves["ln_g:" + name], leaves["ln_b:" + name],
                                      cfg.ln_eps)
    for l in range(cfg.layers):
        pre = f"layer{l}."
        qkv = lin(pre + "qkv", ln(pre + "ln1", x))
        keep = mask(B * nh * S * S, pa, drop_tag(l, 0), (B, nh, S, S))
        att = attention_ref(qkv, B, S, nh, keep, drop_scale(pa))
        add1 = x + lin(pre + "out", att) * mask(T * H, ph, drop_tag(l, 1), (T, H)) * drop_scale(ph)
        h = F.gelu(lin(pre + "up", ln(pre + "ln2", add1)))
        x = add1 + lin(pre + "down", h) * mask(T * H, ph, drop_tag(l, 2), (T, H)) * drop_scale(ph)
    z = (ln("lnf", x) @ leaves["head_w"].t() + leaves["head_b"]).view(B, S, 2)
    loss = 0.5 * (F.cross_entropy(z[..., 0], labels[:, 0]) + F.cross_entropy(z[..., 1], labels[:, 1]))
    return loss, leaves

"""BERT-large under DELTA on one B200.

The reference's transformer trace (ref src/trace.cpp:422-466,
gen_transformer_like) registers, behind an Embedding, per layer
LayerNorm1 -> QKVProj -> Attention -> OutProj -> AddResid1 -> LayerNorm2 ->
MlpUp -> MlpDown -> AddResid2 (a pre-LN block).  This module registers that
graph for a real BERT (hidden 1024, 16 heads, FFN 4096, 24 layers, erf GELU,
dropout 0.1 on the embeddings, the attention probabilities and both residual
branches, a final LayerNorm and the SQuAD span head the paper trains BERT
with), with one DELTA node per activation and one backward
node per gradient the step writes (the format's backward Produce),
and executes it with this library's kernels:

  linear layers     tcgen05 GEMM (conv_fwd.cu as a 1x1 conv over [tokens][in])
                    with the bias in the epilogue; input gradients with the
                    transposed weights (the MLP's through gelu' in the
                    epilogue), weight gradients on wgrad.cu, bias gradients as
                    column sums
  attention         attention.cu (tcgen05; S <= 512 held on chip)
  the rest          xformer.cu (LayerNorm, GELU, residual add + dropout,
                    embeddings, span head, AdamW)

The GELU is its own node (MlpUp keeps the pre-activation the backward needs):
DELTA can then recompute the cheap GELU output instead of keeping or swapping
both [tokens][4096] tensors — the "attention/GELU recompute vs host swap"
choice of config 5.  Dropout masks are counter-based (philox.cuh), so every
recomputed node is bit-identical to its first production.

Outside the activation budget (as for ResNet): fp32 masters, AdamW moments,
gradients, bf16 weight copies, LayerNorm statistics, attention log-sum-exps,
token ids / labels / the id CSR, and the backward scratch.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import executor as X
from . import graph as G
from . import kernels as K
from . import planner as P
from .runtime import DeltaRuntime, _ptr


@dataclass
class BertConfig:
    layers: int = 24
    hidden: int = 1024
    heads: int = 16
    ffn: int = 4096
    seq: int = 512
    batch: int = 8
    vocab: int = 30522
    types: int = 2
    max_pos: int = 512
    p_hidden: float = 0.1
    p_attn: float = 0.1
    ln_eps: float = 1e-12

    @property
    def tokens(self) -> int:
        return self.batch * self.seq


BERT_LARGE = BertConfig()
EMBED_TAG = 0xE0000


def drop_tag(layer: int, site: int) -> int:
    """dropout site ids: 0 attention probabilities, 1 AddResid1, 2 AddResid2"""
    return 1 + 4 * layer + site


def build_bert(cfg: BertConfig) -> G.Graph:
    """Forward + backward DELTA graph of a pre-LN BERT with a span head."""
    g = G.Graph(f"bert{cfg.layers}_h{cfg.hidden}_bs{cfg.batch}_s{cfg.seq}")
    T, H, F4 = cfg.tokens, cfg.hidden, cfg.ffn
    g.linears = {}   # name -> (in, out)
    g.lns = []       # LayerNorm names
    g.cfg = cfg
    act = lambda n: n.nbytes

    def linear(name, src, out):
        g.linears[name] = (src.shape[-1], out)
        n = g.add(name, "linear", (T, out), [src.id], attrs=dict(lin=name))
        n.flops = 2.0 * T * src.shape[-1] * out
        n.hbm_bytes = act(src) + act(n)
        return n

    def layernorm(name, src):
        g.lns.append(name)
        n = g.add(name, "layernorm", (T, H), [src.id], attrs=dict(ln=name))
        n.hbm_bytes = 2 * act(src)
        return n

    emb = g.add("embedding", "embed", (T, H), [])
    emb.hbm_bytes = 4 * act(emb)
    cur = emb
    layers = []
    for l in range(cfg.layers):
        pre = f"layer{l}."
        ln1 = layernorm(pre + "ln1", cur)
        qkv = linear(pre + "qkv", ln1, 3 * H)
        att = g.add(pre + "attention", "attention", (T, H), [qkv.id],
                    attrs=dict(layer=l, tag=drop_tag(l, 0)))
        att.flops = 4.0 * cfg.batch * cfg.heads * cfg.seq * cfg.seq * 64
        att.hbm_bytes = act(qkv) + act(att)
        proj = linear(pre + "out", att, H)
        add1 = g.add(pre + "add1", "add_dropout", (T, H), [cur.id, proj.id],
                     attrs=dict(tag=drop_tag(l, 1)))
        add1.hbm_bytes = 3 * act(add1)
        ln2 = layernorm(pre + "ln2", add1)
        up = linear(pre + "up", ln2, F4)
        ge = g.add(pre + "gelu", "gelu", (T, F4), [up.id])
        ge.hbm_bytes = 2 * act(ge)
        down = linear(pre + "down", ge, H)
        add2 = g.add(pre + "add2", "add_dropout", (T, H), [add1.id, down.id],
                     attrs=dict(tag=drop_tag(l, 2)))
        add2.hbm_bytes = 3 * act(add2)
        layers.append((pre, cur, ln1, qkv, att, proj, add1, ln2, up, ge, down, add2))
        cur = add2
    lnf = layernorm("lnf", cur)
    head = g.add("head", "span_head", (T, 2), [lnf.id], dtype_bytes=4)
    head.flops = 4.0 * T * H
    head.hbm_bytes = act(lnf)

    # ---- backward ----
    d = g.add("head.bwd", "span_head_bwd", (T, H), [head.id, lnf.id], phase="B")
    d.hbm_bytes = 2 * act(d)
    d = g.add("lnf.bwd", "layernorm_bwd", (T, H), [d.id, cur.id], phase="B",
              attrs=dict(ln="lnf"))
    d.hbm_bytes = 4 * act(d)

    def linear_bwd(name, dy, x, pre_act=None, drop=None, bias_done=False):
        lin = name
        parents = [dy.id, x.id] + ([pre_act.id] if pre_act is not None else [])
        cin, cout = g.linears[lin]
        n = g.add(lin + ".bwd", "linear_bwd", (T, cin), parents, phase="B",
                  attrs=dict(lin=lin, gelu=pre_act is not None, drop=drop, bias_done=bias_done))
        n.flops = 4.0 * T * cin * cout
        n.hbm_bytes = 3 * T * cout * 2 + act(x) + act(n) + (act(n) if pre_act is not None else 0)
        return n

    for (pre, X_, ln1, qkv, att, proj, add1, ln2, up, ge, down, add2), l in zip(
            reversed(layers), reversed(range(cfg.layers))):
        g_out = d                                   # d add2
        # the LayerNorm backward that produced g_out also applies the mask of
        # add2's dropout and reduces the down projection's bias gradient
        g_out.attrs.update(drop=drop_tag(l, 2), drop_lin=pre + "down")
        d_up = linear_bwd(pre + "down", g_out, ge, pre_act=up, drop=drop_tag(l, 2))
        # (its bias gradient comes from the gelu' GEMM's epilogue statistics)
        d_ln2 = linear_bwd(pre + "up", d_up, ln2, bias_done=True)
        d_add1 = g.add(pre + "ln2.bwd", "layernorm_bwd", (T, H), [d_ln2.id, add1.id, g_out.id],
                       phase="B", attrs=dict(ln=pre + "ln2", dres=2))
        d_add1.hbm_bytes = 5 * act(d_add1)
        d_add1.attrs.update(drop=drop_tag(l, 1), drop_lin=pre + "out")
        d_att = linear_bwd(pre + "out", d_add1, att, drop=drop_tag(l, 1))
        d_qkv = g.add(pre + "attention.bwd", "attention_bwd", (T, 3 * H),
                      [d_att.id, qkv.id, att.id], phase="B",
                      attrs=dict(layer=l, tag=drop_tag(l, 0)))
        d_qkv.flops = 2.5 * att.flops + 2 * att.flops  # 5 GEMMs + S/dP recomputed by both roles
        d_qkv.hbm_bytes = 2 * act(qkv) + 3 * act(att)
        # (its bias gradient is reduced inside the attention backward)
        d_ln1 = linear_bwd(pre + "qkv", d_qkv, ln1, bias_done=True)
        d = g.add(pre + "ln1.bwd", "layernorm_bwd", (T, H), [d_ln1.id, X_.id, d_add1.id],
                  phase="B", attrs=dict(ln=pre + "ln1", dres=2))
        d.hbm_bytes = 5 * act(d)
    e = g.add("embedding.bwd", "embed_bwd", (T, H), [d.id], phase="B")
    e.hbm_bytes = 3 * act(e)
    return g


def token_csr(ids: np.ndarray) -> np.ndarray:
    """The batch's token ids grouped by id (host side, with the batch): int32
    [2 + 3T] = U, unique ids (padded to T), segment offsets (T + 1), token
    indices (stable within a segment) — the word-embedding gradient's
    deterministic segmented sum (delta_embed_grads)."""
    ids = np.asarray(ids, np.int64).reshape(-1)
    T = ids.size
    perm = np.argsort(ids, kind="stable")
    sid = ids[perm]
    starts = np.flatnonzero(np.r_[True, sid[1:] != sid[:-1]])
    U = starts.size
    out = np.zeros(2 + 3 * T, np.int32)
    out[0] = U
    out[1:1 + U] = sid[starts]
    seg = np.full(T + 1, T, np.int64)
    seg[:U] = starts
    out[1 + T:2 + 2 * T] = seg
    out[2 + 2 * T:] = perm
    return out


class BertParams:
    """fp32 masters (one flat buffer: embedding tables and weight matrices
    first — their bf16 copy is the GEMM operand — then biases, LayerNorm
    parameters and the head), AdamW moments, flat fp32 gradients."""

    def __init__(self, g: G.Graph, device, seed: int = 0):
        cfg = g.cfg
        H = cfg.hidden
        gen = torch.Generator(device="cpu").manual_seed(seed)
        mats = [("word", (cfg.vocab, H)), ("pos", (cfg.max_pos, H)), ("type", (cfg.types, H))]
        for name, (cin, cout) in g.linears.items():
            mats.append(("w:" + name, (cout, cin)))
        vecs = []
        for name, (cin, cout) in g.linears.items():
            vecs.append(("b:" + name, (cout,), "zeros"))
        for name in g.lns:
            vecs.append(("ln_g:" + name, (H,), "ones"))
            vecs.append(("ln_b:" + name, (H,), "zeros"))
        vecs.append(("head_w", (2, H), "normal"))
        vecs.append(("head_b", (2,), "zeros"))
        specs = [(n, s, "normal") for n, s in mats] + vecs
        sizes = [int(np.prod(s)) for _, s, _ in specs]
        self.numel = sum(sizes)
        self.n_bf = sum(int(np.prod(s)) for _, s in mats)
        self.master = torch.empty(self.numel, dtype=torch.float32, device=device)
        self.grad = torch.zeros(self.numel, dtype=torch.float32, device=device)
        self.m = torch.zeros(self.numel, dtype=torch.float32, device=device)
        self.v = torch.zeros(self.numel, dtype=torch.float32, device=device)
        self.views, self.gviews = {}, {}
        off = 0
        for (name, shape, init), n in zip(specs, sizes):
            host = torch.empty(shape, dtype=torch.float32)
            if init == "normal":
                host.normal_(0.0, 0.02, generator=gen)
            elif init == "ones":
                host.fill_(1.0)
            else:
                host.zero_()
            self.master[off:off + n].copy_(host.reshape(-1))
            self.views[name] = self.master[off:off + n].view(shape)
            self.gviews[name] = self.grad[off:off + n].view(shape)
            off += n
        self.wbf_flat = torch.empty(self.n_bf, dtype=torch.bfloat16, device=device)
        self.wbf = {}
        off = 0
        for name, shape in mats:
            n = int(np.prod(shape))
            self.wbf[name] = self.wbf_flat[off:off + n].view(shape)
            off += n
        # (the input-gradient GEMMs read the forward weights [out][in] through
        # MN-major descriptors: no transposed copies, no per-step view launch)
        T = cfg.tokens
        self.ln_mean = {n: torch.zeros(T, device=device) for n in g.lns}
        self.ln_rstd = {n: torch.ones(T, device=device) for n in g.lns}
        self.lse = [torch.zeros(cfg.batch * cfg.heads * cfg.seq, device=device)
                    for _ in range(cfg.layers)]
        self.bn_rmean = {}  # (DeltaRuntime.measure_costs saves/restores BN running stats)
        self.bn_rvar = {}
        self.refresh_bf16()

    def refresh_bf16(self):
        self.wbf_flat.copy_(self.master[:self.n_bf])

    def adamw_step(self, rng_ptr: int, lr: float, b1=0.9, b2=0.999, eps=1e-6, wd=0.01):
        st = torch.cuda.current_stream().cuda_stream
        K.adamw_step(self.master.data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                     self.grad.data_ptr(), self.wbf_flat.data_ptr(), self.numel, self.n_bf, lr, b1,
                     b2, eps, wd, rng_ptr, st)


class BertRuntime(DeltaRuntime):
    """BERT training step (span head, AdamW) under a DELTA activation budget.

        rt = BertRuntime(BertConfig(batch=8))
        rt.measure_costs(); rt.plan(0.4)
        loss = rt.step(ids, types, labels)      # host int tensors
    """

    # the output projection's weight gradient runs on the side stream during
    # the attention backward (DELTA_BERT_OVERLAP=0: in its own node, serially)
    overlap_attn_wgrad = os.environ.get("DELTA_BERT_OVERLAP", "1") != "0"

    def __init__(self, cfg: BertConfig = BERT_LARGE, device: str = "cuda", seed: int = 0,
                 lr: float = 1e-4, dropout_seed: int = 0x5EED_0F_DE17A):
        self.device = torch.device(device)
        self.cfg = cfg
        self.g = build_bert(cfg)
        self.batch = cfg.batch
        self.lr = lr
        self.anchors = "none"
        G.estimate_costs(self.g)
        self.params = BertParams(self.g, self.device, seed)
        self.nodes = self.g.nodes
        self.stream = torch.cuda.Stream(device=self.device)
        T, H = cfg.tokens, cfg.hidden
        dev = self.device
        self.rng = torch.tensor([dropout_seed, 0], dtype=torch.int64, device=dev)
        # linear layers: forward (bias epilogue), input gradient (transposed
        # weights; the MLP down-projection's through gelu'), weight gradient
        self._lin, self._lin_d, self._lin_w = {}, {}, {}
        wg_ws = 256
        for name, (cin, cout) in self.g.linears.items():
            self._lin[name] = K.Conv(T, 1, 1, cin, cout, 1, 1, 1, 0,
                                     _ptr(self.params.wbf["w:" + name]))
            d = K.Conv(T, 1, 1, cout, cin, 1, 1, 1, 0, _ptr(self.params.wbf["w:" + name]),
                       weights_ck=True)
            if name.endswith("down") and d.tile_n > 128:
                d.set_tile_n(128)  # gelu' epilogue: N tiles <= 128
            self._lin_d[name] = d
            self._lin_w[name] = K.Wgrad(T, 1, 1, cin, cout, 1, 1, 1, 0)
            wg_ws = max(wg_ws, self._lin_w[name].workspace_bytes)
        self.wg_ws = torch.zeros(wg_ws, dtype=torch.uint8, device=dev)  # split counters: zero once
        self.ln_ws = torch.empty(K.layernorm_bwd_workspace_floats(T, H), device=dev)
        self.cs_ws = torch.empty(max(K.colsum_workspace_floats(T, cfg.ffn),
                                     K.span_head_workspace_floats(T, H),
                                     cfg.batch * 3 * H), device=dev)
        self.drop_ws = torch.empty(T, H, dtype=torch.bfloat16, device=dev)  # dropout-bwd scratch
        # per-CTA column statistics of the gelu' input gradient (its column
        # sums are the up-projection's bias gradient: no extra pass over it)
        self.gstats = torch.empty(K.stats_partials_floats(cfg.ffn), device=dev)
        self.attn_D = torch.empty(cfg.batch * cfg.heads * cfg.seq, device=dev)
        self.dlogits = torch.empty(T, 2, device=dev)
        self.row_loss = torch.empty(cfg.batch, device=dev)
        self.loss = torch.zeros(1, device=dev)
        # input staging slots: ids, token types, labels (start, end), id CSR
        self.in_slots = [[torch.zeros(T, dtype=torch.int32, device=dev),
                          torch.zeros(T, dtype=torch.int32, device=dev),
                          torch.zeros(cfg.batch, 2, dtype=torch.int32, device=dev),
                          torch.from_numpy(token_csr(np.zeros(T, np.int64))).to(dev)]
                         for _ in range(2)]
        self._use_slot(0)
        self.graphs = None
        self._h2d = None
        self._loss_host = None
        self.program = None
        self.arena = None
        self.executor = None
        self._bound_slot = None
        self.graph = None
        self.cost_table = None
        self.link_gbs = None
        self.dp = None
        self.buckets = []
        self._comm = None

    # ------------------------------------------------------------ inputs
    def _use_slot(self, slot: int):
        self._slot = slot
        self.ids_dev, self.types_dev, self.labels_dev, self.csr_dev = self.in_slots[slot]

    def _slot_tensors(self, slot: int) -> list:
        return self.in_slots[slot]

    def make_batch(self, ids, types, labels, pin: bool = True) -> tuple:
        """host batch tuple (ids, types, labels, id CSR) for step/train"""
        ids = torch.as_tensor(ids, dtype=torch.int32).reshape(-1)
        types = torch.as_tensor(types, dtype=torch.int32).reshape(-1)
        labels = torch.as_tensor(labels, dtype=torch.int32).reshape(-1, 2)
        csr = torch.from_numpy(token_csr(ids.numpy()))
        b = (ids, types, labels, csr)
        return tuple(t.pin_memory() for t in b) if pin else b

    def step(self, ids, types, labels) -> float:
        """one synchronous step with host inputs (H2D, step, D2H of the loss)"""
        return self._step_host(self.make_batch(ids, types, labels, pin=False))

    def synthetic_batch(self, seed: int = 0, pin: bool = True) -> tuple:
        g = torch.Generator().manual_seed(seed)
        c = self.cfg
        ids = torch.randint(0, c.vocab, (c.tokens,), generator=g, dtype=torch.int32)
        # question | context segments
        types = (torch.arange(c.seq) >= c.seq // 4).to(torch.int32).repeat(c.batch)
        st = torch.randint(c.seq // 4, c.seq - 1, (c.batch,), generator=g)
        en = torch.minimum(st + torch.randint(0, 30, (c.batch,), generator=g),
                           torch.tensor(c.seq - 1))
        labels = torch.stack([st, en], 1).to(torch.int32)
        return self.make_batch(ids, types, labels, pin=pin)

    def _optimizer_step(self):
        self.params.adamw_step(_ptr(self.rng), self.lr)

    # ------------------------------------------------------------ recipes
    def _recipe(self, node: G.Node) -> tuple:
        cfg = self.cfg
        pr = self.params
        T, H = cfg.tokens, cfg.hidden
        op = node.op
        ops = []
        nl = [0, 0]

        def add(k, n=1):
            ops.append(k)
            if not (k.flags & X.RECOMPUTE_ONLY):
                nl[0] += n
            if not (k.flags & X.FIRST_ONLY):
                nl[1] += n

        rng = _ptr(self.rng)
        if op == "embed":
            add(X.kop(X.K_EMBED, (_ptr(self.ids_dev), _ptr(self.types_dev), _ptr(pr.wbf["word"]),
                                  _ptr(pr.wbf["pos"]), _ptr(pr.wbf["type"]), X.OUT(), rng),
                      (cfg.batch, cfg.seq, H, EMBED_TAG), (cfg.p_hidden,)))
        elif op == "layernorm":
            ln = node.attrs["ln"]
            add(X.kop(X.K_LAYERNORM, (X.IN(0), X.OUT(), _ptr(pr.ln_mean[ln]), _ptr(pr.ln_rstd[ln]),
                                      _ptr(pr.views["ln_g:" + ln]), _ptr(pr.views["ln_b:" + ln])),
                      (T, H), (cfg.ln_eps,)))
        elif op == "linear":
            lin = node.attrs["lin"]
            add(X.kop(X.K_CONV_EX, (X.IN(0), X.OUT(), None) + (None,) * 7 +
                      (_ptr(pr.views["b:" + lin]),), (K.EPI_BIAS, 0, 0),
                      conv=self._lin[lin]._h))
        elif op == "attention":
            l = node.attrs["layer"]
            add(X.kop(X.K_ATTN, (X.IN(0), X.OUT(), _ptr(pr.lse[l]), rng),
                      (cfg.batch, cfg.seq, cfg.heads, node.attrs["tag"]), (cfg.p_attn,)))
        elif op == "add_dropout":
            add(X.kop(X.K_ADD_DROPOUT, (X.IN(0), X.IN(1), X.OUT(), rng),
                      (T * H, node.attrs["tag"]), (cfg.p_hidden,)))
        elif op == "gelu":
            add(X.kop(X.K_GELU, (X.IN(0), X.OUT()), (T * cfg.ffn,)))
        elif op == "span_head":
            add(X.kop(X.K_SPAN_HEAD, (X.IN(0), _ptr(pr.views["head_w"]), _ptr(pr.views["head_b"]),
                                      _ptr(self.labels_dev), X.OUT(), _ptr(self.dlogits),
                                      _ptr(self.row_loss), _ptr(self.loss)),
                      (cfg.batch, cfg.seq, H)), 2)
        elif op == "span_head_bwd":
            add(X.kop(X.K_SPAN_HEAD_BWD, (X.IN(1), _ptr(self.dlogits), _ptr(pr.views["head_w"]),
                                          X.OUT(), _ptr(pr.gviews["head_w"]),
                                          _ptr(pr.gviews["head_b"]), _ptr(self.cs_ws)), (T, H)), 3)
        elif op == "layernorm_bwd":
            ln = node.attrs["ln"]
            dres = X.IN(node.attrs["dres"]) if "dres" in node.attrs else None
            refs = (X.IN(0), X.IN(1), dres, X.OUT(), _ptr(pr.ln_mean[ln]), _ptr(pr.ln_rstd[ln]),
                    _ptr(pr.views["ln_g:" + ln]), _ptr(pr.gviews["ln_g:" + ln]),
                    _ptr(pr.gviews["ln_b:" + ln]), _ptr(self.ln_ws))
            if node.attrs.get("drop") is not None:
                # + the gradient through the dropout of the residual branch
                # into drop_ws (read by the very next node, that branch's
                # linear_bwd) and the branch's bias gradient
                add(X.kop(X.K_LAYERNORM_BWD_DROP,
                          refs + (_ptr(self.drop_ws), _ptr(pr.gviews["b:" + node.attrs["drop_lin"]]),
                                  rng),
                          (T, H, node.attrs["drop"]), (cfg.p_hidden,)), 2)
            else:
                add(X.kop(X.K_LAYERNORM_BWD, refs, (T, H)), 2)
        elif op == "linear_bwd":
            lin = node.attrs["lin"]
            cin, cout = self.g.linears[lin]
            dy = X.IN(0)
            fused_drop = False
            if node.attrs.get("drop") is not None:
                # the residual branch's dropout, backward (its mask replayed):
                # done by the LayerNorm backward that produced dy, with the
                # bias gradient, when that node carries it
                fused_drop = self.g.nodes[node.parents[0]].attrs.get("drop_lin") == lin
                if not fused_drop:
                    add(X.kop(X.K_DROPOUT_BWD, (X.IN(0), _ptr(self.drop_ws), rng),
                              (T * cout, node.attrs["drop"]), (cfg.p_hidden,)))
                dy = _ptr(self.drop_ws)
            dconv = self._lin_d[lin]._h
            if node.attrs.get("gelu"):
                # the gelu' input gradient also reduces its per-CTA column
                # statistics: the bias gradient of the up projection (whose
                # output gradient it is) follows from them below
                up = self.g.nodes[node.parents[2]].attrs["lin"]
                add(X.kop(X.K_CONV_EX, (dy, X.OUT(), _ptr(self.gstats), None, None, None, X.IN(2)),
                          (K.EPI_GELU_BWD, 0, 0), conv=dconv))
                add(X.kop(X.K_STATS_SUM, (_ptr(self.gstats), _ptr(pr.gviews["b:" + up])),
                          (self.g.linears[up][1], 0)))
            else:
                add(X.kop(X.K_CONV, (dy, X.OUT(), None), conv=dconv))
            if not (fused_drop and self.g.nodes[node.parents[1]].op == "attention"
                    and self.overlap_attn_wgrad):
                add(X.kop(X.K_WGRAD, (dy, X.IN(1), _ptr(pr.gviews["w:" + lin]), _ptr(self.wg_ws)),
                          conv=self._lin_w[lin]._h), self._lin_w[lin].launches)
            # (else: the attention backward node runs it, see there)
            if not node.attrs.get("bias_done") and not fused_drop:
                add(X.kop(X.K_COLSUM, (dy, None, _ptr(pr.gviews["b:" + lin]), _ptr(self.cs_ws)),
                          (T, cout, 0, 0)), 2)
        elif op == "attention_bwd":
            l = node.attrs["layer"]
            # dqkv and, reduced per sequence inside the kernel, its column
            # sums: the QKV projection's bias gradient
            qkv_lin = self.g.nodes[node.parents[1]].attrs["lin"]
            if self.overlap_attn_wgrad:
                # the output projection's weight gradient (its inputs: the
                # dropout-masked gradient still in drop_ws and this node's
                # input `att`) on the side stream, concurrent with the
                # attention backward: its CTAs fill the SMs the attention
                # kernel's last partial wave leaves idle
                out_lin = self.g.nodes[node.parents[0]].attrs["lin"]
                add(X.kop(X.K_WGRAD, (_ptr(self.drop_ws), X.IN(2), _ptr(pr.gviews["w:" + out_lin]),
                                      _ptr(self.wg_ws)),
                          conv=self._lin_w[out_lin]._h, flags=X.SIDE_ALWAYS),
                    self._lin_w[out_lin].launches)
            add(X.kop(X.K_ATTN_BWD, (X.IN(1), X.IN(2), X.IN(0), _ptr(pr.lse[l]), _ptr(self.attn_D),
                                     X.OUT(), rng, _ptr(pr.gviews["b:" + qkv_lin]),
                                     _ptr(self.cs_ws)),
                      (cfg.batch, cfg.seq, cfg.heads, node.attrs["tag"]), (cfg.p_attn,)), 3)
        elif op == "embed_bwd":
            add(X.kop(X.K_DROPOUT_BWD, (X.IN(0), X.OUT(), rng), (T * H, EMBED_TAG),
                      (cfg.p_hidden,)))
            add(X.kop(X.K_EMBED_GRADS, (X.OUT(), _ptr(self.csr_dev), _ptr(self.types_dev),
                                        _ptr(pr.gviews["word"]), _ptr(pr.gviews["pos"]),
                                        _ptr(pr.gviews["type"]), _ptr(self.cs_ws)),
                      (cfg.batch, cfg.seq, H, cfg.vocab | (cfg.types << 32))), 2 + 2 * cfg.types)
        else:
            raise RuntimeError(f"no kernel for op {op!r} (node {node.name})")
        return ops, tuple(nl)

    def engine_config(self, budget: int, policy=P.PolicyMode.Delta, **kw) -> P.EngineConfig:
        return super().engine_config(budget, policy, **kw)

"""ResNet-50/101 as a DELTA tensor-registration graph.

Every activation the training step keeps is one DELTA node (OpNode), produced
by exactly one forward op; every backward op is a backward-phase node whose
parents are the saved activations (and upstream gradient) it reads and whose
output is the gradient it writes.  This is the trace the runtime plans with
(ref include/deltasim/trace.hpp:14-41; backward Produce nodes as the format
allows, SPEC.md:44 / SURVEY F5), and the same graph drives execution: node
`op` names the kernel that (re)computes it.

Layout: all activations NHWC bf16 in the HBM arena; byte sizes are rounded to
the arena alignment so trace bytes == arena allocation bytes.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

ALIGN = 256
# the shortcut dgrad's epilogue also reduces the next BN3 backward's sums
# (DELTA_FUSE_BN3_SUMS=0: a separate partial pass)
FUSE_BN3_SUMS = os.environ.get("DELTA_FUSE_BN3_SUMS", "1") == "1"


def rnd(b: int) -> int:
    return (b + ALIGN - 1) // ALIGN * ALIGN


@dataclass
class Node:
    id: int
    name: str
    op: str                 # kernel family, see executor.OPS
    shape: tuple            # NHWC (or (N, C)) of the output buffer
    parents: list
    phase: str = "F"        # "F" forward, "B" backward
    attrs: dict = field(default_factory=dict)
    uncomputable: bool = False
    evict_pinned: bool = False
    offload_pinned: bool = False
    dtype_bytes: int = 2
    cost_us: int = 1        # filled by the cost model
    flops: float = 0.0      # algorithmic FLOPs of the op (roofline)
    hbm_bytes: float = 0.0  # algorithmic HBM bytes of the op (roofline)

    @property
    def nbytes(self) -> int:
        n = self.dtype_bytes
        for d in self.shape:
            n *= d
        return rnd(n)


@dataclass
class ConvSpec:
    name: str
    cin: int
    cout: int
    k: int
    stride: int
    pad: int


class Graph:
    def __init__(self, name: str):
        self.name = name
        self.nodes: list[Node] = []
        self.convs: dict[str, ConvSpec] = {}
        self.bns: dict[str, int] = {}          # bn name -> channels
        self.fc = None                         # (cin, cout)

    def add(self, name, op, shape, parents, phase="F", **kw) -> Node:
        n = Node(len(self.nodes), name, op, tuple(shape), list(parents), phase, **kw)
        self.nodes.append(n)
        return n

    def node(self, name) -> Node:
        for n in self.nodes:
            if n.name == name:
                return n
        raise KeyError(name)


BLOCKS = {50: [3, 4, 6, 3], 101: [3, 4, 23, 3]}


def build_resnet(depth: int = 50, batch: int = 256, image: int = 224,
                 num_classes: int = 1000, stem_cin: int = 4) -> Graph:
    """Forward + backward DELTA graph of torchvision-style ResNet (v1.5:
    stride on the 3x3 conv).  `stem_cin` = input channels padded to 4 for the
    8-byte stem gather."""
    g = Graph(f"resnet{depth}_bs{batch}")
    N = batch
    conv_flops = lambda n_out, cin, k: 2.0 * n_out * cin * k * k

    def conv(name, src: Node, cout, k, stride, pad):
        n_, h, w, cin = src.shape
        p = (h + 2 * pad - k) // stride + 1
        q = (w + 2 * pad - k) // stride + 1
        g.convs[name] = ConvSpec(name, cin, cout, k, stride, pad)
        node = g.add(name, "conv", (n_, p, q, cout), [src.id], attrs=dict(conv=name))
        node.flops = conv_flops(n_ * p * q * cout, cin if cin != 4 else 3, k)
        node.hbm_bytes = src.nbytes + node.nbytes
        return node

    def bnrelu(name, src: Node):
        g.bns[name] = src.shape[-1]
        node = g.add(name + "_relu", "bn_relu", src.shape, [src.id], attrs=dict(bn=name))
        node.hbm_bytes = 2 * src.nbytes
        return node

    # ---- forward ----
    x = g.add("input", "input", (N, image, image, stem_cin), [], uncomputable=True,
              evict_pinned=True)
    c0 = conv("conv1", x, 64, 7, 2, 3)
    r0 = bnrelu("bn1", c0)
    n_, h, w, c = r0.shape
    ph, pw = (h + 2 - 3) // 2 + 1, (w + 2 - 3) // 2 + 1
    p0 = g.add("maxpool", "maxpool", (N, ph, pw, c), [r0.id])
    p0.hbm_bytes = r0.nbytes + p0.nbytes

    blocks = []  # (prefix, X, C1, R1, C2, R2, C3, CD or None, O)
    cur = p0
    width = 64
    for li, nblk in enumerate(BLOCKS[depth]):
        for b in range(nblk):
            pre = f"layer{li + 1}.{b}"
            stride = 2 if (b == 0 and li > 0) else 1
            cin = cur.shape[-1]
            c1 = conv(pre + ".conv1", cur, width, 1, 1, 0)
            r1 = bnrelu(pre + ".bn1", c1)
            c2 = conv(pre + ".conv2", r1, width, 3, stride, 1)
            r2 = bnrelu(pre + ".bn2", c2)
            c3 = conv(pre + ".conv3", r2, width * 4, 1, 1, 0)
            g.bns[pre + ".bn3"] = width * 4
            cd = None
            if b == 0:
                cd = conv(pre + ".downsample.0", cur, width * 4, 1, stride, 0)
                g.bns[pre + ".downsample.1"] = width * 4
                o = g.add(pre + ".out", "bn_bn_add_relu", c3.shape, [c3.id, cd.id],
                          attrs=dict(bn=pre + ".bn3", bn2=pre + ".downsample.1"))
                o.hbm_bytes = c3.nbytes + cd.nbytes + o.nbytes
            else:
                o = g.add(pre + ".out", "bn_add_relu", c3.shape, [c3.id, cur.id],
                          attrs=dict(bn=pre + ".bn3"))
                o.hbm_bytes = c3.nbytes + cur.nbytes + o.nbytes
            assert cin == cur.shape[-1]
            blocks.append((pre, cur, c1, r1, c2, r2, c3, cd, o))
            cur = o
        width *= 2
    pooled = g.add("avgpool", "avgpool", (N, cur.shape[-1]), [cur.id])
    pooled.hbm_bytes = cur.nbytes + pooled.nbytes
    g.fc = (cur.shape[-1], num_classes)
    # the classifier GEMM's bf16 logits, classes padded to a multiple of 64
    # (zero weight rows): the tensor-core kernel's N tile; bias and softmax
    # are applied in fp32 by the head kernel
    g.fc_pad = (num_classes + 63) // 64 * 64
    logits = g.add("fc", "fc", (N, g.fc_pad), [pooled.id])
    logits.flops = 2.0 * N * cur.shape[-1] * num_classes
    logits.hbm_bytes = pooled.nbytes + logits.nbytes

    # ---- backward (one node per gradient the step writes) ----
    # head: softmax-xent + fc backward -> dPooled
    d_pool = g.add("fc.bwd", "fc_bwd", pooled.shape, [logits.id, pooled.id], phase="B")
    d_pool.flops = 4.0 * N * cur.shape[-1] * num_classes
    # Gradient nodes carry the gradient w.r.t. a block's PRE-activation (the
    # ReLU mask of the block output is applied once, by the node that writes
    # it), so BN3/downsample backward read no mask.  The exception is the
    # pooled head gradient of the last block, masked where it is consumed.
    upstream = d_pool
    upstream_is_pool = True
    upstream_sums = False
    first = blocks[0][0]
    for bi in reversed(range(len(blocks))):
        (pre, X, C1, R1, C2, R2, C3, CD, O) = blocks[bi]
        bn_parents = (lambda t: [upstream.id, O.id, t.id]) if upstream_is_pool else \
            (lambda t: [upstream.id, t.id])
        extra = dict(from_pool=upstream_is_pool, masked=upstream_is_pool)
        d_c3 = g.add(pre + ".bn3.bwd", "bn_add_relu_bwd", C3.shape, bn_parents(C3), phase="B",
                     attrs=dict(bn=pre + ".bn3", sums_fused=upstream_sums, **extra))
        # sums fused upstream: read g and X, write dX; else a partial pass first
        d_c3.hbm_bytes = (3 if upstream_sums else (6 if upstream_is_pool else 5)) * C3.nbytes
        d_cd = None
        if CD is not None:
            d_cd = g.add(pre + ".downsample.1.bwd", "bn_add_relu_bwd", CD.shape, bn_parents(CD),
                         phase="B", attrs=dict(bn=pre + ".downsample.1", **extra))
            d_cd.hbm_bytes = (6 if upstream_is_pool else 5) * CD.nbytes
        d_c2 = g.add(pre + ".conv3.bwd", "conv_bn_relu_bwd", C2.shape,
                     [d_c3.id, R2.id, C2.id], phase="B",
                     attrs=dict(conv=pre + ".conv3", bn=pre + ".bn2"))
        d_c2.flops = 2 * C3.flops
        # dgrad (read dY, write g) + BN backward (g and BN input twice, write
        # dX) + weight gradient (read dY and the conv input)
        d_c2.hbm_bytes = 2 * d_c3.nbytes + 6 * C2.nbytes
        d_c1 = g.add(pre + ".conv2.bwd", "conv_bn_relu_bwd", C1.shape,
                     [d_c2.id, R1.id, C1.id], phase="B",
                     attrs=dict(conv=pre + ".conv2", bn=pre + ".bn1"))
        d_c1.flops = 2 * C2.flops
        d_c1.hbm_bytes = 2 * d_c2.nbytes + 6 * C1.nbytes
        # output: gradient of the previous block's pre-activation, i.e. masked
        # by X > 0 (X is that block's ReLU output); the first block's input is
        # the maxpool output, whose gradient is left unmasked.
        mask_out = pre != first
        if CD is not None:
            parents = [d_c1.id, X.id, d_cd.id]
            attrs = dict(conv=pre + ".conv1", conv_short=pre + ".downsample.0",
                         mask_out=mask_out)
        elif upstream_is_pool:
            parents = [d_c1.id, X.id, upstream.id, O.id]
            attrs = dict(conv=pre + ".conv1", from_pool=True, mask_out=mask_out)
        else:
            parents = [d_c1.id, X.id, upstream.id]
            attrs = dict(conv=pre + ".conv1", from_pool=False, mask_out=mask_out)
        # The gradient written here is the previous block's BN3 backward input:
        # with a plain (full, stride-1) add and a previous block without a
        # downsample BN, its epilogue also reduces (sum g, sum g*C3) for that
        # BN3 — C3 becomes a parent (read by this node).
        prev = blocks[bi - 1] if bi > 0 else None
        upstream_sums = (FUSE_BN3_SUMS and prev is not None and prev[7] is None and mask_out
                         and CD is None and not upstream_is_pool)
        if upstream_sums:
            attrs["sums_xc"] = len(parents)
            parents = parents + [prev[6].id]
        d_x = g.add(pre + ".conv1.bwd", "conv_shortcut_bwd", X.shape, parents, phase="B",
                    attrs=attrs)
        d_x.flops = 2 * C1.flops + (2 * CD.flops if CD is not None else 0)
        # conv1 dgrad (read dY, write dX) + residual add + ReLU mask reads +
        # weight gradient (dY, X); the downsample's dgrad and wgrad likewise
        d_x.hbm_bytes = 2 * d_c1.nbytes + (5 if upstream_sums else 4) * X.nbytes + \
            (2 * d_cd.nbytes + 2 * X.nbytes if CD is not None else 0)
        upstream = d_x
        upstream_is_pool = False
    # stem: maxpool backward, bn1-relu backward, conv1 weight gradient
    d_r0 = g.add("maxpool.bwd", "maxpool_bwd", r0.shape, [upstream.id, r0.id], phase="B")
    d_r0.hbm_bytes = upstream.nbytes + 2 * r0.nbytes  # argmax pass + gather
    d_c0 = g.add("bn1.bwd", "bn_relu_bwd", c0.shape, [d_r0.id, r0.id, c0.id], phase="B",
                 attrs=dict(bn="bn1"))
    d_c0.hbm_bytes = 7 * c0.nbytes  # masked streaming BN backward: 3 reads, then 3 + 1 write
    # conv1 has no input gradient; its node output is the weight gradient (fp32)
    wg = g.add("conv1.bwd", "conv_wgrad", (64, 7, 7, stem_cin), [d_c0.id, x.id], phase="B",
               attrs=dict(conv="conv1"), dtype_bytes=4)
    wg.flops = c0.flops
    wg.hbm_bytes = d_c0.nbytes + x.nbytes
    return g


def to_trace(g: Graph, name: str | None = None):
    """The DELTA trace of the graph: forward Produce in order, then backward
    Produce in order (ref trace format, README.md 'Trace format')."""
    from .planner import AccessEvent, AccessKind, OpNode, Phase, Trace
    t = Trace(name or g.name)
    for n in g.nodes:
        t.nodes.append(OpNode(n.id, n.name, int(n.cost_us), n.nbytes, list(n.parents),
                              n.uncomputable, n.evict_pinned, n.offload_pinned))
    for n in g.nodes:
        if n.phase == "F":
            t.schedule.append(AccessEvent(n.id, Phase.Forward, AccessKind.Produce))
    for n in g.nodes:
        if n.phase == "B":
            t.schedule.append(AccessEvent(n.id, Phase.Backward, AccessKind.Produce))
    return t


def estimate_costs(g: Graph, tflops: float = 1000.0, gbs: float = 5000.0) -> None:
    """Roofline-estimated op costs (µs) until the GPU cost model measures them."""
    for n in g.nodes:
        t_flop = n.flops / (tflops * 1e6) if n.flops else 0.0
        t_mem = (n.hbm_bytes or 2 * n.nbytes) / (gbs * 1e3)
        n.cost_us = max(1, int(round(max(t_flop, t_mem))) + 2)
    for n in g.nodes:
        if n.uncomputable:
            n.cost_us = max(1, int(n.nbytes / (gbs * 1e3)))

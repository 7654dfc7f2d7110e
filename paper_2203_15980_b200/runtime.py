"""DELTA runtime on B200: plan on the logical clock, execute on the GPU.

    rt = DeltaRuntime(depth=50, batch=256)             # graph + params
    rt.measure_costs()                                  # GPU cost model -> trace costs
    rt.plan(budget_fraction=0.5)                        # libdelta planner + lowering
    loss = rt.step(x, y)                                # one training step

The step replays the lowered action program (csrc/rt/lower.cpp) on three
streams: compute (forward kernels, recompute kernels, backward), D2H and H2D
(copy engines of the swap engine).  Every activation lives at its planned
offset in one HBM arena; nothing else allocates activation memory.  Forward
and recompute of a node run the SAME sm_100a kernel on the same inputs, so a
recomputed tensor is bit-identical to the one it replaces.

Outside the activation budget (as in the paper): fp32 master weights, bf16
weight copies, gradients, optimizer state, BN statistics and the transient
workspace of cuDNN's conv backward (dgrad/wgrad, the one library call on the
backward path).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import graph as G
from . import kernels as K
from . import planner as P

BN_EPS = 1e-5
# BN statistics are reduced in the conv epilogue when the conv's reduction
# length is at least this (the epilogue work hides under the main loop);
# shorter convs get a separate streaming statistics pass.
FUSE_STATS_MIN_KDIM = int(__import__("os").environ.get("DELTA_FUSE_STATS_MIN_KDIM", "384"))
BN_MOMENTUM = 0.1


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


class Params:
    """fp32 master parameters (one flat buffer), bf16 conv weights (KRSC),
    flat fp32 gradients and SGD momentum; BN running/saved statistics."""

    def __init__(self, g: G.Graph, device, seed: int = 0):
        self.g = g
        gen = torch.Generator(device="cpu").manual_seed(seed)
        specs = []  # (name, shape, init)
        for name, cs in g.convs.items():
            specs.append(("conv:" + name, (cs.cout, cs.k, cs.k, cs.cin), "kaiming", cs))
        for name, c in g.bns.items():
            specs.append(("bn_g:" + name, (c,), "ones", None))
            specs.append(("bn_b:" + name, (c,), "zeros", None))
        cin, ncls = g.fc
        specs.append(("fc_w", (ncls, cin), "linear", cin))
        specs.append(("fc_b", (ncls,), "linear_b", cin))
        sizes = [int(np.prod(s[1])) for s in specs]
        total = sum(sizes)
        self.numel = total
        self.master = torch.empty(total, dtype=torch.float32, device=device)
        self.grad = torch.zeros(total, dtype=torch.float32, device=device)
        self.mom = torch.zeros(total, dtype=torch.float32, device=device)
        self.views, self.gviews = {}, {}
        off = 0
        n_conv = 0
        for (name, shape, init, extra), n in zip(specs, sizes):
            host = torch.empty(shape, dtype=torch.float32)
            if init == "kaiming":
                cs = extra
                fan_out = cs.cout * cs.k * cs.k           # torchvision: fan_out, relu
                host.normal_(0.0, math.sqrt(2.0 / fan_out), generator=gen)
                if cs.cin == 4:
                    host[..., 3] = 0.0                    # padded RGB channel
            elif init == "ones":
                host.fill_(1.0)
            elif init == "zeros":
                host.zero_()
            else:
                bound = 1.0 / math.sqrt(extra)
                host.uniform_(-bound, bound, generator=gen)
            self.master[off:off + n].copy_(host.reshape(-1))
            self.views[name] = self.master[off:off + n].view(shape)
            self.gviews[name] = self.grad[off:off + n].view(shape)
            if init == "kaiming":
                n_conv = off + n
            off += n
        self.n_conv = n_conv  # conv weights are the leading slice
        self.conv_bf16 = torch.empty(n_conv, dtype=torch.bfloat16, device=device)
        self.wbf = {}
        off = 0
        for name, cs in g.convs.items():
            n = cs.cout * cs.k * cs.k * cs.cin
            self.wbf[name] = self.conv_bf16[off:off + n].view(cs.cout, cs.k, cs.k, cs.cin)
            off += n
        # the stem kernel reads its weights in the pixel-pair layout
        self.stem_packed = {}
        for name, cs in g.convs.items():
            if cs.cin == 4:
                self.stem_packed[name] = torch.zeros(cs.cout, K.STEM_KDIM, dtype=torch.bfloat16,
                                                     device=device)
        # input-gradient (dgrad) weights of the stride-1 convs, run through our
        # conv kernel: [C][R][S][K], W'[c][r][s][k] = W[k][R-1-r][S-1-s][c]
        self.wd = {}
        for name, cs in g.convs.items():
            if own_dgrad(cs):
                self.wd[name] = torch.empty(cs.cin, cs.k, cs.k, cs.cout, dtype=torch.bfloat16,
                                            device=device)
        self.bn_mean = {n: torch.zeros(c, device=device) for n, c in g.bns.items()}
        self.bn_invstd = {n: torch.ones(c, device=device) for n, c in g.bns.items()}
        self.bn_rmean = {n: torch.zeros(c, device=device) for n, c in g.bns.items()}
        self.bn_rvar = {n: torch.ones(c, device=device) for n, c in g.bns.items()}
        self.refresh_bf16()

    def refresh_bf16(self):
        self.conv_bf16.copy_(self.master[:self.n_conv])
        for name, packed in self.stem_packed.items():
            K.pack_stem_weights(self.wbf[name], packed)
        for name, wd in self.wd.items():
            wd.copy_(self.wbf[name].flip(1, 2).permute(3, 1, 2, 0))

    def sgd_step(self, lr: float, momentum: float = 0.9, weight_decay: float = 1e-4):
        # grads stay untouched (they are what DP all-reduces and tests read)
        self.mom.mul_(momentum).add_(self.grad).add_(self.master, alpha=weight_decay)
        self.master.add_(self.mom, alpha=-lr)
        self.refresh_bf16()


def workspace_plan(g: G.Graph) -> dict:
    """Bytes of every batch-proportional buffer DeltaRuntime allocates outside
    the activation budget (the max-batch search plans with the same numbers).
    'transient' = the largest cuDNN output alive inside one backward node
    (the 3x3 input gradients)."""
    nodes = g.nodes
    M = lambda n: int(np.prod(n.shape[:-1]))
    batch = nodes[0].shape[0]
    ws = {}
    ws["bn_ws"] = 4 * max(K.bn_workspace_floats(M(n), n.shape[-1]) for n in nodes
                          if len(n.shape) == 4 and n.shape[-1] % 64 == 0)
    parts = 4 * max(K.stats_partials_floats(M(n), n.shape[-1]) for n in nodes
                    if n.op in ("conv", "conv_bn_relu_bwd"))
    ws["stats_main"] = ws["stats_ds"] = parts
    short = [nodes[n.parents[2]].nbytes * g.convs[n.attrs["conv_short"]].cin
             // g.convs[n.attrs["conv_short"]].cout for n in nodes
             if n.op == "conv_shortcut_bwd" and "conv_short" in n.attrs
             and g.convs[n.attrs["conv_short"]].stride != 1]
    ws["short_ws"] = max(short + [256])
    mp = next(n for n in nodes if n.op == "maxpool")
    ws["mp_ws"] = K.maxpool_workspace_bytes(*nodes[mp.parents[0]].shape)
    ws["head"] = 4 + batch * g.fc[1] * 4 + batch * 4
    ws["input_slots"] = 2 * (nodes[0].nbytes + batch * 8)
    trans = [0]
    for n in nodes:
        if n.op == "conv_bn_relu_bwd" and not own_dgrad(g.convs[n.attrs["conv"]]):
            trans.append(nodes[n.parents[1]].nbytes)          # cuDNN dgrad output
    ws["transient"] = max(trans)
    return ws


def own_dgrad(cs: G.ConvSpec) -> bool:
    """Input gradients of the 1x1 convs run through our tcgen05 conv kernel
    (transposed weights; fused backward epilogues: residual add + ReLU mask,
    BN-backward reductions; a stride-2 1x1's gradient is computed on its
    sampling grid and scattered by the consumer's epilogue).  3x3 dgrads stay
    with cuDNN for now (our 3x3 kernel is slower than cuDNN's at the narrow
    layer-1/2 widths, scripts/kbench_dgrad.py); the stem has no input gradient."""
    return cs.k == 1 and cs.cin != 4


@dataclass
class StepStats:
    loss: float
    ms: float


class DeltaRuntime:
    """ResNet training step under a DELTA activation budget on one B200."""

    def __init__(self, depth: int = 50, batch: int = 256, image: int = 224,
                 device: str = "cuda", seed: int = 0, anchors: str = "out+narrow",
                 lr: float = 0.1):
        self.device = torch.device(device)
        self.g = G.build_resnet(depth, batch, image)
        self.batch = batch
        self.lr = lr
        self.anchors = anchors
        apply_anchors(self.g, anchors)
        G.estimate_costs(self.g)
        self.params = Params(self.g, self.device, seed)
        self.nodes = self.g.nodes
        self.stream = torch.cuda.Stream(device=self.device)
        self._convs = {}
        self._build_convs()
        ws = workspace_plan(self.g)
        f32 = lambda key: torch.empty(ws[key] // 4, dtype=torch.float32, device=self.device)
        u8 = lambda key: torch.empty(ws[key], dtype=torch.uint8, device=self.device)
        self.bn_ws = f32("bn_ws")
        # BN statistics partials written by the conv epilogue (one 128-row
        # tile per partial); downsample convs use their own scratch because
        # their BN is applied together with the block's bn3.
        self.stats_main = f32("stats_main")
        self.stats_ds = f32("stats_ds")
        # backward scratch outside the budget: the input gradient of a stride-2
        # shortcut conv at its sampling grid
        self.short_ws = u8("short_ws")
        self.mp_ws = u8("mp_ws")
        ncls = self.g.fc[1]
        self.loss = torch.zeros(1, dtype=torch.float32, device=self.device)
        self.dlogits = torch.empty(batch, ncls, dtype=torch.float32, device=self.device)
        self.row_loss = torch.empty(batch, dtype=torch.float32, device=self.device)
        self.x_slots = [torch.zeros(self.g.nodes[0].shape, dtype=torch.bfloat16,
                                    device=self.device) for _ in range(2)]
        self.y_slots = [torch.zeros(batch, dtype=torch.int64, device=self.device)
                        for _ in range(2)]
        self._use_slot(0)
        self.graphs = None
        self._h2d = None
        self._loss_host = None
        self.program = None
        self.arena = None
        self.swap = None
        self.events = None
        self.graph = None
        self.cost_table = None
        self.link_gbs = None
        self.dp = None  # torch.distributed group when running data parallel

    # ------------------------------------------------------------ setup
    def _build_convs(self):
        # epilogue BN statistics cost ~11*BN cycles per tile against ~2*kblocks*BN
        # of MMA: fused only where the main loop hides them (K-dim >= 384)
        self._fuse_stats = {}
        self._dconvs = {}
        for n in self.nodes:
            if n.op == "conv":
                cs = self.g.convs[n.attrs["conv"]]
                src = self.nodes[n.parents[0]]
                Nb, H, W, C = src.shape
                wptr = (_ptr(self.params.stem_packed[cs.name]) if cs.cin == 4
                        else _ptr(self.params.wbf[cs.name]))
                conv = K.Conv(Nb, H, W, C, cs.cout, cs.k, cs.k, cs.stride, cs.pad, wptr)
                assert (conv.P, conv.Q) == n.shape[1:3], (n.name, conv.P, conv.Q, n.shape)
                self._convs[n.name] = conv
                self._fuse_stats[n.name] = conv.kdim >= FUSE_STATS_MIN_KDIM
                if own_dgrad(cs):
                    # on the conv's output grid (a stride-2 1x1's gradient lives at
                    # its sampling points; the consumer scatters it)
                    _, P_, Q_, _ = n.shape
                    dconv = K.Conv(Nb, P_, Q_, cs.cout, cs.cin, cs.k, cs.k, 1, cs.k // 2,
                                   _ptr(self.params.wd[cs.name]))
                    if dconv.tile_n > 128:
                        dconv.set_tile_n(128)  # fused backward epilogues
                    self._dconvs[cs.name] = dconv

    def trace(self) -> P.Trace:
        return G.to_trace(self.g)

    def engine_config(self, budget: int, policy=P.PolicyMode.Delta, **kw) -> P.EngineConfig:
        cm = P.CostModel()
        if self.link_gbs:
            # measured one-way pinned copy bandwidth, bytes/us, exact fraction
            bpus = int(self.link_gbs * 1e3)
            cm = P.CostModel(bandwidth_bytes_per_us=(bpus, 1), effective_fraction=(1, 1))
        return P.EngineConfig(budget=budget, policy_mode=policy, cost_model=cm, **kw)

    def baseline_peak(self) -> int:
        base = P.run_unconstrained_baseline(self.trace(), self.engine_config(0))
        return base.peak_bytes

    def plan(self, budget_fraction: float | None = 0.5, budget: int | None = None,
             policy=P.PolicyMode.Delta, **kw):
        """Plan with libdelta and lower onto the arena.  budget_fraction=None
        plans the no-eviction baseline (Baseline policy, budget = sum)."""
        t = self.trace()
        if budget_fraction is None and budget is None:
            total = sum(n.nbytes for n in self.nodes)
            cfg = self.engine_config(total, P.PolicyMode.Baseline, **kw)
        else:
            if budget is None:
                budget = int(self.baseline_peak() * budget_fraction)
            cfg = self.engine_config(budget, policy, **kw)
        prog = P.Program(t, cfg, align=G.ALIGN)
        if prog.infeasible:
            node, deficit = prog.infeasible
            raise RuntimeError(f"plan infeasible at node {self.nodes[node].name} "
                               f"(deficit {deficit} B, budget {cfg.budget} B)")
        self.program = prog
        self.config = cfg
        self.graph = None
        self.graphs = None
        if self.arena is None or self.arena.numel() < prog.arena_bytes:
            self.arena = None
            torch.cuda.empty_cache()
            self.arena = torch.empty(prog.arena_bytes, dtype=torch.uint8, device=self.device)
        if prog.host_bytes and (self.swap is None or self._swap_bytes < prog.host_bytes):
            self.swap = K.Swap(prog.host_bytes)
            self._swap_bytes = prog.host_bytes
        if self.swap is None:
            self.swap = K.Swap(0)
            self._swap_bytes = 0
        self.events = K.Events(prog.n_events)
        self._base = _ptr(self.arena)
        self._inputs = prog.inputs
        return prog

    # -------------------------------------------------------- tensors
    def _view(self, off: int, node: G.Node) -> torch.Tensor:
        dt = torch.float32 if node.dtype_bytes == 4 else torch.bfloat16
        n = int(np.prod(node.shape))
        return self.arena.narrow(0, off, n * node.dtype_bytes).view(dt).view(node.shape)

    # ------------------------------------------------------------ ops
    def _run_node(self, node: G.Node, out_off: int, in_offs, recompute: bool, st: int):
        base = self._base
        op = node.op
        out = base + out_off
        ins = [base + o for o in in_offs]
        pr = self.params
        if op == "input":
            self._view(out_off, node).copy_(self.x_dev, non_blocking=True)
        elif op == "conv":
            # the first production also emits BN statistics partials from the
            # epilogue; a recompute must not (the scratch may be in use)
            scratch = None
            if not recompute and self._fuse_stats[node.name]:
                scratch = _ptr(self.stats_ds if "downsample" in node.name else self.stats_main)
            self._convs[node.name](ins[0], out, st, scratch)
        elif op in ("bn_relu", "bn_add_relu", "bn_bn_add_relu"):
            bn = node.attrs["bn"]
            M = int(np.prod(node.shape[:-1]))
            C = node.shape[-1]
            if not recompute:  # statistics once per step; recompute reuses them
                self._bn_stats(node.parents[0], ins[0], bn, self.stats_main, M, C, st)
            args = [_ptr(pr.bn_mean[bn]), _ptr(pr.bn_invstd[bn]), _ptr(pr.views["bn_g:" + bn]),
                    _ptr(pr.views["bn_b:" + bn])]
            if op == "bn_relu":
                K.bn_apply(0, ins[0], None, out, M, C, *args, stream=st)
            elif op == "bn_add_relu":
                K.bn_apply(1, ins[0], ins[1], out, M, C, *args, stream=st)
            else:
                bn2 = node.attrs["bn2"]
                if not recompute:
                    self._bn_stats(node.parents[1], ins[1], bn2, self.stats_ds, M, C, st)
                K.bn_apply(2, ins[0], ins[1], out, M, C, *args, _ptr(pr.bn_mean[bn2]),
                           _ptr(pr.bn_invstd[bn2]), _ptr(pr.views["bn_g:" + bn2]),
                           _ptr(pr.views["bn_b:" + bn2]), stream=st)
        elif op == "maxpool":
            src = self.nodes[node.parents[0]]
            Nb, H, W, C = src.shape
            K.maxpool_fwd(ins[0], out, Nb, H, W, C, st)
        elif op == "avgpool":
            src = self.nodes[node.parents[0]]
            Nb, H, W, C = src.shape
            K.avgpool_fwd(ins[0], out, Nb, H * W, C, st)
        elif op == "fc":
            a = self._view(in_offs[0], self.nodes[node.parents[0]])
            torch.addmm(pr.views["fc_b"], a.float(), pr.views["fc_w"].t(),
                        out=self._view(out_off, node))
        elif op == "fc_bwd":
            logits = self._view(in_offs[0], self.nodes[node.parents[0]])
            a = self._view(in_offs[1], self.nodes[node.parents[1]])
            Nb, ncls = logits.shape
            K.softmax_xent(_ptr(logits), _ptr(self.y_dev), _ptr(self.loss), _ptr(self.dlogits),
                           _ptr(self.row_loss), Nb, ncls, st)
            torch.mm(self.dlogits.t(), a.float(), out=pr.gviews["fc_w"])
            torch.sum(self.dlogits, 0, out=pr.gviews["fc_b"])
            self._view(out_off, node).copy_(self.dlogits @ pr.views["fc_w"])
        elif op == "bn_add_relu_bwd":
            # parents: [upstream, (O if masked,) X]; upstream already masked
            # unless it is the pooled head gradient
            bn = node.attrs["bn"]
            M = int(np.prod(node.shape[:-1]))
            C = node.shape[-1]
            pool_hw = int(node.shape[1] * node.shape[2]) if node.attrs.get("from_pool") else 0
            mask = ins[1] if node.attrs.get("masked") else None
            K.bn_backward(ins[0], pool_hw, mask, ins[-1], out, M, C, _ptr(pr.bn_mean[bn]),
                          _ptr(pr.bn_invstd[bn]), _ptr(pr.views["bn_g:" + bn]),
                          _ptr(pr.gviews["bn_g:" + bn]), _ptr(pr.gviews["bn_b:" + bn]),
                          _ptr(self.bn_ws), st)
        elif op == "conv_bn_relu_bwd":
            # parents [dC, R = relu(bn(X)), X]
            conv = node.attrs["conv"]
            bn = node.attrs["bn"]
            dC = self._view(in_offs[0], self.nodes[node.parents[0]])
            R = self._view(in_offs[1], self.nodes[node.parents[1]])
            M = int(np.prod(node.shape[:-1]))
            C = node.shape[-1]
            bnp = (_ptr(pr.bn_mean[bn]), _ptr(pr.bn_invstd[bn]))
            if conv in self._dconvs:
                # dgrad on the tensor cores; the epilogue applies the ReLU mask
                # (recomputed from X) and reduces sum g, sum g*X per tile
                g_ptr = out  # g is written in place of its BN-backward output
                self._dconvs[conv].bn_bwd(ins[0], g_ptr, _ptr(self.stats_main), ins[2], *bnp,
                                          _ptr(pr.views["bn_g:" + bn]), _ptr(pr.views["bn_b:" + bn]),
                                          st)
                K.bn_backward_from_partials(_ptr(self.stats_main), g_ptr, ins[2], out, M, C, *bnp,
                                            _ptr(pr.views["bn_g:" + bn]),
                                            _ptr(pr.gviews["bn_g:" + bn]),
                                            _ptr(pr.gviews["bn_b:" + bn]), st)
                self._conv_bwd(conv, dC, R, need_dx=False)
            else:
                dR = self._conv_bwd(conv, dC, R, need_dx=True)
                K.bn_backward(_ptr(dR), 0, ins[1], ins[2], out, M, C, *bnp,
                              _ptr(pr.views["bn_g:" + bn]), _ptr(pr.gviews["bn_g:" + bn]),
                              _ptr(pr.gviews["bn_b:" + bn]), _ptr(self.bn_ws), st)
        elif op == "conv_shortcut_bwd":
            # out = (dgrad(conv1, dC1) + shortcut gradient) * [X > 0]; the sum
            # and the mask are the dgrad kernel's epilogue
            conv = node.attrs["conv"]
            dC1 = self._view(in_offs[0], self.nodes[node.parents[0]])
            X = self._view(in_offs[1], self.nodes[node.parents[1]])
            out_mask = ins[1] if node.attrs.get("mask_out") else None
            add, pool_hw, add_mask, stride2 = None, 0, None, False
            if "conv_short" in node.attrs:
                short = node.attrs["conv_short"]
                dCD = self._view(in_offs[2], self.nodes[node.parents[2]])
                if short in self._dconvs:
                    if self.g.convs[short].stride == 1:
                        add = out   # summed in place by conv1's dgrad epilogue
                    else:
                        add, stride2 = _ptr(self.short_ws), True  # at its sampling grid
                    self._dconvs[short](ins[2], add, st)
                    self._conv_bwd(short, dCD, X, need_dx=False)
                else:
                    dXs = self._conv_bwd(short, dCD, X, need_dx=True)
                    add = _ptr(dXs)
            elif node.attrs.get("from_pool"):
                add, pool_hw, add_mask = ins[2], int(node.shape[1] * node.shape[2]), ins[3]
            else:
                add = ins[2]
            if conv in self._dconvs:
                self._dconvs[conv].add_mask(ins[0], out, st, add=add, pool_hw=pool_hw,
                                            add_mask=add_mask, out_mask=out_mask,
                                            add_stride2=stride2)
                self._conv_bwd(conv, dC1, X, need_dx=False)
            else:
                dX = self._conv_bwd(conv, dC1, X, need_dx=True)
                M = int(np.prod(node.shape[:-1]))
                K.add_grad(_ptr(dX), add, pool_hw, add_mask, out_mask, out, M, node.shape[-1], st)
        elif op == "maxpool_bwd":
            src = self.nodes[node.parents[1]]
            Nb, H, W, C = src.shape
            K.maxpool_bwd(ins[0], ins[1], out, Nb, H, W, C, _ptr(self.mp_ws), st)
        elif op == "bn_relu_bwd":
            bn = node.attrs["bn"]
            M = int(np.prod(node.shape[:-1]))
            C = node.shape[-1]
            K.bn_backward(ins[0], 0, ins[1], ins[2], out, M, C, _ptr(pr.bn_mean[bn]),
                          _ptr(pr.bn_invstd[bn]), _ptr(pr.views["bn_g:" + bn]),
                          _ptr(pr.gviews["bn_g:" + bn]), _ptr(pr.gviews["bn_b:" + bn]),
                          _ptr(self.bn_ws), st)
        elif op == "conv_wgrad":
            conv = node.attrs["conv"]
            dC = self._view(in_offs[0], self.nodes[node.parents[0]])
            X = self._view(in_offs[1], self.nodes[node.parents[1]])
            self._conv_bwd(conv, dC, X, need_dx=False)
            self._view(out_off, node).copy_(pr.gviews["conv:" + conv])
        else:
            raise RuntimeError(f"no kernel for op {op!r} (node {node.name})")

    def _bn_stats(self, conv_node_id: int, x_ptr: int, bn: str, scratch, M: int, C: int, st):
        """Training-mode BN statistics of a conv output: from the partials the
        conv epilogue wrote when the conv is long enough to hide that work,
        else one streaming pass over the tensor."""
        pr = self.params
        conv = self.nodes[conv_node_id]
        args = (_ptr(pr.bn_mean[bn]), _ptr(pr.bn_invstd[bn]), BN_EPS, _ptr(pr.bn_rmean[bn]),
                _ptr(pr.bn_rvar[bn]), BN_MOMENTUM)
        if self._fuse_stats.get(conv.name):
            K.bn_stats_from_partials(_ptr(scratch), M, C, *args, st)
        else:
            K.bn_stats(x_ptr, M, C, _ptr(self.bn_ws), *args, st)

    def _conv_bwd(self, name: str, dY: torch.Tensor, X: torch.Tensor, need_dx: bool):
        """dgrad/wgrad through cuDNN (channels_last views of arena memory);
        the weight gradient lands in the fp32 grad buffer (KRSC)."""
        cs = self.g.convs[name]
        w = self.params.wbf[name].permute(0, 3, 1, 2)
        gi, gw, _ = torch.ops.aten.convolution_backward(
            dY.permute(0, 3, 1, 2), X.permute(0, 3, 1, 2), w, None, [cs.stride] * 2,
            [cs.pad] * 2, [1, 1], False, [0, 0], 1, [need_dx, True, False])
        self.params.gviews["conv:" + name].copy_(gw.permute(0, 2, 3, 1))
        if need_dx:
            gi = gi.permute(0, 2, 3, 1)
            if not gi.is_contiguous():
                gi = gi.contiguous()
            return gi
        return None

    # -------------------------------------------------------- program
    def run_program(self, timing: dict | None = None, probe: dict | None = None,
                    stamps: list | None = None):
        """Issue one training step: the lowered action program on the three
        streams, then the optimizer.  Returns nothing; loss stays on device.
        `timing`: per-node (and "swap") CUDA event pairs; `stamps`: receives
        (action index, start event, end event) of every compute/recompute/
        offload/reload action (events on the action's own stream)."""
        prog = self.program
        st = self.stream.cuda_stream
        streams = {P.STREAM_COMPUTE: st, P.STREAM_D2H: self.swap.d2h_stream,
                   P.STREAM_H2D: self.swap.h2d_stream}
        nodes = self.nodes
        inputs = self._inputs
        ev = self.events
        base = self._base
        n_timed = 0
        for ai, a in enumerate(prog.actions):
            op = int(a["op"])
            if timing is not None and op in (P.ACT_COMPUTE, P.ACT_RECOMPUTE) and n_timed % 24 == 0:
                # keep the GPU busy while the host queues the next actions, so
                # the event pairs time device execution, not launch latency
                torch.cuda._sleep(int(3e7))
            if op == P.ACT_WAIT:
                ev.wait(int(a["event"]), streams[int(a["stream"])])
            elif op == P.ACT_RECORD:
                ev.record(int(a["event"]), streams[int(a["stream"])])
            elif op in (P.ACT_COMPUTE, P.ACT_RECOMPUTE):
                node = nodes[int(a["node"])]
                at, n_in = int(a["inputs_at"]), int(a["n_inputs"])
                if timing is None and stamps is not None:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(self.stream)
                if timing is not None:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(self.stream)
                self._run_node(node, int(a["offset"]), [int(x) for x in inputs[at:at + n_in]],
                               op == P.ACT_RECOMPUTE, st)
                if probe is not None and node.id in probe:
                    probe[node.id] = self._view(int(a["offset"]), node).clone()
                if timing is not None or stamps is not None:
                    e1.record(self.stream)
                if timing is not None:
                    timing.setdefault(node.id, []).append((e0, e1, op == P.ACT_RECOMPUTE))
                    n_timed += 1
                if stamps is not None:
                    stamps.append((ai, e0, e1))
            elif op in (P.ACT_OFFLOAD, P.ACT_RELOAD):
                sid = streams[int(a["stream"])]
                if timing is not None or stamps is not None:
                    xs = torch.cuda.ExternalStream(sid)
                    c0 = torch.cuda.Event(enable_timing=True)
                    c1 = torch.cuda.Event(enable_timing=True)
                    c0.record(xs)
                if op == P.ACT_OFFLOAD:
                    self.swap.offload(base + int(a["offset"]), int(a["host_offset"]),
                                      int(a["bytes"]), sid)
                else:
                    self.swap.reload(base + int(a["offset"]), int(a["host_offset"]),
                                     int(a["bytes"]), sid)
                if timing is not None or stamps is not None:
                    c1.record(xs)
                if timing is not None:
                    timing.setdefault("swap", []).append((c0, c1, op, int(a["bytes"])))
                if stamps is not None:
                    stamps.append((ai, c0, c1))
        # join the copy streams that carried work back into the compute stream
        used = set(int(x) for x in prog.actions["stream"][np.isin(prog.actions["op"], (P.ACT_OFFLOAD, P.ACT_RELOAD))])
        for sid in sorted(used):
            e = torch.cuda.Event()
            e.record(torch.cuda.ExternalStream(streams[sid]))
            self.stream.wait_event(e)
        if self.dp is not None:
            # data parallel: one DELTA instance per GPU, gradients averaged
            # with NCCL over NVLink (one flat bucket, on the compute stream)
            allreduce_mean(self.params.grad, self.dp)
        self.params.sgd_step(self.lr)

    def capture(self):
        """Capture one full step (program + optimizer) as a CUDA graph per
        input staging slot (two slots let `train` overlap the next batch's
        host->device copy with the current step)."""
        torch.cuda.synchronize()
        graphs = []
        for slot in range(2):
            self._use_slot(slot)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(self.stream):
                with torch.cuda.graph(g, stream=self.stream):
                    self.run_program()
            graphs.append(g)
        self._use_slot(0)
        self.graphs = graphs
        self.graph = graphs[0]
        torch.cuda.synchronize()

    def _use_slot(self, slot: int):
        self._slot = slot
        self.x_dev = self.x_slots[slot]
        self.y_dev = self.y_slots[slot]

    def step_device(self):
        """One step with inputs already resident in the current slot."""
        with torch.cuda.stream(self.stream):
            if self.graph is not None:
                self.graphs[self._slot].replay()
            else:
                self.run_program()

    def step(self, x_host: torch.Tensor, y_host: torch.Tensor) -> float:
        """One synchronous step through the public API with HOST buffers:
        H2D of the batch, the step, D2H of the loss."""
        with torch.cuda.stream(self.stream):
            self.x_dev.copy_(x_host, non_blocking=True)
            self.y_dev.copy_(y_host, non_blocking=True)
        self.step_device()
        with torch.cuda.stream(self.stream):
            loss = self.loss.to("cpu", non_blocking=False)
        return float(loss.item())

    def train(self, batches) -> list:
        """Train on a sequence of (x, y) pinned host batches.  Each step's
        inputs are copied host->device on a copy-engine stream into the
        staging slot the step after next is not using, overlapped with the
        current step; each step's loss is copied device->host right after it.
        Returns the per-step losses."""
        n = len(batches)
        if n == 0:
            return []
        if self._h2d is None:
            self._h2d = torch.cuda.Stream(device=self.device)
            self._loss_host = None
        if self._loss_host is None or self._loss_host.numel() < n:
            self._loss_host = torch.empty(max(n, 64), dtype=torch.float32).pin_memory()
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_done = [torch.cuda.Event(), torch.cuda.Event()]

        def h2d(i):
            slot = i % 2
            with torch.cuda.stream(self._h2d):
                if i >= 2:
                    self._h2d.wait_event(ev_done[slot])  # step i-2 read this slot
                self.x_slots[slot].copy_(batches[i][0], non_blocking=True)
                self.y_slots[slot].copy_(batches[i][1], non_blocking=True)
                ev_in[slot].record(self._h2d)

        h2d(0)
        for i in range(n):
            slot = i % 2
            if i + 1 < n:
                h2d(i + 1)
            self.stream.wait_event(ev_in[slot])
            self._use_slot(slot)
            self.step_device()
            ev_done[slot].record(self.stream)
            with torch.cuda.stream(self.stream):
                self._loss_host[i].copy_(self.loss[0], non_blocking=True)
        self.stream.synchronize()
        self._use_slot(0)
        return self._loss_host[:n].tolist()

    def executed_timeline(self) -> np.ndarray:
        """One eager step with every device action time-stamped; returns the
        plan's timeline (ref Timeline, engine.hpp:44-70) re-stamped with the
        MEASURED device times (µs from the step start): Compute/Recompute/
        Offload/Reload take their kernel's or copy's start and duration;
        zero-duration markers (Use, Free, Evict, Stall) take the end of the
        latest compute-stream action before them.  Feed it to the
        reference's oracle::replay_check (oracle/ref.replay_check) for an
        independent safety certificate of what the GPU actually did."""
        prog = self.program
        stamps = []
        start = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(self.stream):
            start.record(self.stream)
            self.run_program(stamps=stamps)
        torch.cuda.synchronize()
        plan = P.run_iteration(self.trace(), self.config).events
        ev = plan.copy()
        t_of = {}
        for ai, e0, e1 in stamps:
            pe = int(prog.actions[ai]["plan_event"])
            t0 = start.elapsed_time(e0) * 1e3
            t1 = start.elapsed_time(e1) * 1e3
            t_of[pe] = (int(round(t0)), max(0, int(round(t1)) - int(round(t0))))
        now = 0
        for i in range(len(ev)):
            if i in t_of:
                ev[i]["ts"], ev[i]["duration"] = t_of[i]
                if ev[i]["stream"] == P.StreamKind.Compute:
                    now = max(now, int(ev[i]["ts"] + ev[i]["duration"]))
            else:
                ev[i]["ts"] = now
                ev[i]["duration"] = 0
        return ev

    # ----------------------------------------------------- cost model
    def measure_costs(self, iters: int = 3, link: bool = True):
        """GPU-resident cost model: time every node's op on device (CUDA events
        around each action of the no-eviction program, median of `iters`
        steps), quantise to whole microseconds (>= 1) and write them into the
        trace; probe the pinned host link for the swap cost."""
        self.plan(None)
        lr = self.lr
        self.lr = 0.0  # cost probing must not move the weights
        samples: dict[int, list] = {}
        with torch.cuda.stream(self.stream):
            for _ in range(iters + 1):
                timing = {}
                self.run_program(timing)
                torch.cuda.synchronize()
                for nid, lst in timing.items():
                    if nid != "swap":
                        samples.setdefault(nid, []).append(lst[0][0].elapsed_time(lst[0][1]))
        self.lr = lr
        table = {}
        for n in self.nodes:
            ms = sorted(samples[n.id][1:]) if len(samples[n.id]) > 1 else samples[n.id]
            us = ms[len(ms) // 2] * 1e3
            n.cost_us = max(1, int(math.ceil(us)))
            table[n.name] = n.cost_us
        if link:
            h2d, d2h, _ = K.probe_link()
            self.link_gbs = min(h2d, d2h)
        self.cost_table = table
        return table


def apply_anchors(g: G.Graph, anchors: str):
    """Author-specified pins: tensors marked both evict_pinned
    and offload_pinned are never release candidates (ref policy.cpp:111-114)
    and anchor recompute closures.  'out+narrow' anchors every block output and
    the width-channel conv outputs (conv1/conv2 of each bottleneck and the
    stem conv); 'out' anchors block outputs only; 'none' leaves every
    computable activation to the Filter/Director."""
    for n in g.nodes:
        if n.phase != "F" or n.uncomputable:
            continue
        leaf = n.name.split(".")[-1]
        pin = False
        if anchors in ("out", "out+narrow") and leaf == "out":
            pin = True
        if anchors == "out+narrow" and n.op == "conv" and leaf in ("conv1", "conv2"):
            pin = True
        if pin:
            n.evict_pinned = n.offload_pinned = True


# ------------------------------------------------------ data parallelism
def allreduce_mean(t: torch.Tensor, group) -> None:
    """Average `t` across the group in place (NCCL: one AVG all-reduce)."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.AVG, group=group)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        t.div_(dist.get_world_size(group))


def agree_cost_table(g: G.Graph, link_gbs: float | None, group, device="cpu"):
    """Make every rank plan from the same cost table: per-node
    costs are max-reduced and the host-link bandwidth min-reduced, so the
    DELTA plans — a pure function of (trace, config) — are identical."""
    import torch.distributed as dist
    v = torch.tensor([float(n.cost_us) for n in g.nodes] + [-(link_gbs or 0.0)],
                     dtype=torch.float64, device=device)
    dist.all_reduce(v, op=dist.ReduceOp.MAX, group=group)
    for n, c in zip(g.nodes, v[:-1].tolist()):
        n.cost_us = int(c)
    link = -float(v[-1].item())
    return link if link > 0 else None

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
weight copies, gradients, optimizer state, BN statistics and the backward
scratch (the stride-2 input gradients before their BN backward, the weight-
gradient split-K partials).  Every op of the step is one of this library's
sm_100a kernels: no cuDNN, cuBLAS or host callbacks on the step.
"""
from __future__ import annotations

import dataclasses
import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import executor as X
from . import graph as G
from . import kernels as K
from . import planner as P

BN_EPS = 1e-5
# BN statistics are reduced in the conv epilogue when the conv's reduction
# length is at least this; shorter convs get a separate streaming statistics
# pass.  0 = every conv (measured A/B on one box with 8 epilogue warps:
# 11.57k vs 11.44k img/s; with 4 epilogue warps it was a wash, hence the old 384).
DGRAD_BN256 = __import__("os").environ.get("DELTA_DGRAD_BN256", "1") == "1"
FUSE_STATS_MIN_KDIM = int(__import__("os").environ.get("DELTA_FUSE_STATS_MIN_KDIM", "0"))
BN_MOMENTUM = 0.1
_TORCH_OPTIM = __import__("os").environ.get("DELTA_TORCH_OPTIM", "0") == "1"


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
        # the classifier weight right after the conv weights (its bf16 copy is
        # part of the same leading slice), classes padded to the GEMM's tile
        # with zero rows (zero gradient, so they stay zero)
        cin, ncls = g.fc
        self.fc_pad = g.fc_pad
        specs.append(("fc_w_full", (g.fc_pad, cin), "linear", (cin, ncls)))
        for name, c in g.bns.items():
            specs.append(("bn_g:" + name, (c,), "ones", None))
            specs.append(("bn_b:" + name, (c,), "zeros", None))
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
            elif init == "linear":
                fan_in, rows = extra
                host.zero_()
                host[:rows].uniform_(-1.0 / math.sqrt(fan_in), 1.0 / math.sqrt(fan_in), generator=gen)
            else:
                bound = 1.0 / math.sqrt(extra)
                host.uniform_(-bound, bound, generator=gen)
            self.master[off:off + n].copy_(host.reshape(-1))
            self.views[name] = self.master[off:off + n].view(shape)
            self.gviews[name] = self.grad[off:off + n].view(shape)
            if init in ("kaiming", "linear"):
                n_conv = off + n
            off += n
        # the classifier weight as the (ncls, cin) parameter it is
        self.views["fc_w"] = self.views["fc_w_full"][:ncls]
        self.gviews["fc_w"] = self.gviews["fc_w_full"][:ncls]
        self.n_conv = n_conv  # conv + classifier weights are the leading slice (bf16 copy)
        self.conv_bf16 = torch.empty(n_conv, dtype=torch.bfloat16, device=device)
        self.wbf = {}
        off = 0
        for name, cs in g.convs.items():
            n = cs.cout * cs.k * cs.k * cs.cin
            self.wbf[name] = self.conv_bf16[off:off + n].view(cs.cout, cs.k, cs.k, cs.cin)
            off += n
        # classifier GEMM operand: [fc_pad][1][1][cin] (a 1x1 conv's KRSC weights)
        self.wbf["fc"] = self.conv_bf16[off:off + g.fc_pad * cin].view(g.fc_pad, 1, 1, cin)
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
        # the classifier's input gradient: [cin][1][1][fc_pad] (transposed)
        self.wd["fc"] = torch.empty(cin, 1, 1, g.fc_pad, dtype=torch.bfloat16, device=device)
        # stride-2 3x3 input gradients: four sub-pixel parity classes (a, b),
        # each [cin][1+a][1+b][cout]
        self.wd_s2 = {}
        for name, cs in g.convs.items():
            if dgrad_s2(cs):
                self.wd_s2[name] = [torch.empty(cs.cin, 1 + (c >> 1), 1 + (c & 1), cs.cout,
                                                dtype=torch.bfloat16, device=device)
                                    for c in range(4)]
        # every derived weight tensor as one table for the weight-view kernel
        views = []
        for name, packed in self.stem_packed.items():
            cs = g.convs[name]
            views.append(K.WeightView(K.VIEW_STEM, cs.cout, cs.k, cs.k, cs.cin, 0,
                                      self.wbf[name].data_ptr(), packed.data_ptr()))
        for name, wd in self.wd.items():
            if name == "fc":
                views.append(K.WeightView(K.VIEW_DGRAD, g.fc_pad, 1, 1, cin, 0,
                                          self.wbf["fc"].data_ptr(), wd.data_ptr()))
                continue
            cs = g.convs[name]
            views.append(K.WeightView(K.VIEW_DGRAD, cs.cout, cs.k, cs.k, cs.cin, 0,
                                      self.wbf[name].data_ptr(), wd.data_ptr()))
        for name, wds in self.wd_s2.items():
            cs = g.convs[name]
            for c, wd in enumerate(wds):
                views.append(K.WeightView(K.VIEW_DGRAD_S2, cs.cout, cs.k, cs.k, cs.cin, c,
                                          self.wbf[name].data_ptr(), wd.data_ptr()))
        self.n_views = len(views)
        arr = (K.WeightView * max(1, len(views)))(*views)
        self.views_dev = torch.frombuffer(bytearray(arr), dtype=torch.uint8).to(device)
        self.bn_mean = {n: torch.zeros(c, device=device) for n, c in g.bns.items()}
        self.bn_invstd = {n: torch.ones(c, device=device) for n, c in g.bns.items()}
        self.bn_rmean = {n: torch.zeros(c, device=device) for n, c in g.bns.items()}
        self.bn_rvar = {n: torch.ones(c, device=device) for n, c in g.bns.items()}
        self.refresh_bf16()

    def refresh_bf16(self):
        """bf16 conv weights from the fp32 masters, then every derived view."""
        self.conv_bf16.copy_(self.master[:self.n_conv])
        K.weight_views(self.views_dev.data_ptr(), self.n_views,
                       torch.cuda.current_stream().cuda_stream)

    def sgd_step(self, lr: float, momentum: float = 0.9, weight_decay: float = 1e-4):
        """SGD with momentum + weight decay, the bf16 conv weights and their
        derived views: two launches (optim.cu).  Grads stay untouched (they
        are what DP all-reduces and tests read)."""
        st = torch.cuda.current_stream().cuda_stream
        if _TORCH_OPTIM:  # the per-tensor torch sequence the fused kernels replaced (A/B)
            self.mom.mul_(momentum).add_(self.grad).add_(self.master, alpha=weight_decay)
            self.master.add_(self.mom, alpha=-lr)
            self.conv_bf16.copy_(self.master[:self.n_conv])
            for name, packed in self.stem_packed.items():
                K.pack_stem_weights(self.wbf[name], packed)
            for name, wd in self.wd.items():
                wd.copy_(self.wbf[name].flip(1, 2).permute(3, 1, 2, 0))
            K.weight_views(self.views_dev.data_ptr(), self.n_views, st)
            return
        K.sgd_step(self.master.data_ptr(), self.mom.data_ptr(), self.grad.data_ptr(),
                   self.conv_bf16.data_ptr(), self.numel, self.n_conv, lr, momentum,
                   weight_decay, st)
        K.weight_views(self.views_dev.data_ptr(), self.n_views, st)


def workspace_plan(g: G.Graph) -> dict:
    """Bytes of every batch-proportional buffer DeltaRuntime allocates outside
    the activation budget (the max-batch search plans with the same numbers).
    'transient' = the largest stride-2 3x3 input gradient (written by its four
    sub-pixel convs, read by the BN backward of the same node); 'head' = the
    classifier's loss, fp32 / bf16 logit gradients and per-row losses."""
    nodes = g.nodes
    M = lambda n: int(np.prod(n.shape[:-1]))
    batch = nodes[0].shape[0]
    ws = {}
    ws["bn_ws"] = 4 * max(K.bn_workspace_floats(M(n), n.shape[-1]) for n in nodes
                          if len(n.shape) == 4 and n.shape[-1] % 64 == 0)
    # BN-statistics partials: one (count, mean, M2) row per CTA of the conv
    parts = 4 * max(K.stats_partials_floats(n.shape[-1]) for n in nodes
                    if n.op in ("conv", "conv_bn_relu_bwd"))
    ws["stats_main"] = ws["stats_ds"] = ws["stats_sums"] = parts
    short = [nodes[n.parents[2]].nbytes * g.convs[n.attrs["conv_short"]].cin
             // g.convs[n.attrs["conv_short"]].cout for n in nodes
             if n.op == "conv_shortcut_bwd" and "conv_short" in n.attrs
             and g.convs[n.attrs["conv_short"]].stride != 1]
    ws["short_ws"] = max(short + [256])
    ws["mp_ws"] = max([K.maxpool_workspace_bytes(*nodes[n.parents[0]].shape) for n in nodes
                       if n.op == "maxpool"] + [256])
    wg = 0
    for n in nodes:
        if n.op == "conv":
            cs = g.convs[n.attrs["conv"]]
            Nb, H, W, Cin = nodes[n.parents[0]].shape
            wg = max(wg, K.Wgrad(Nb, H, W, Cin, cs.cout, cs.k, cs.k, cs.stride,
                                 cs.pad).workspace_bytes)
    wg = max(wg, K.Wgrad(batch, 1, 1, g.fc[0], g.fc_pad, 1, 1, 1, 0).workspace_bytes)
    ws["wgrad_ws"] = wg
    ws["head"] = 4 + batch * g.fc[1] * 4 + batch * g.fc_pad * 2 + batch * 4
    ws["input_slots"] = 2 * (nodes[0].nbytes + batch * 8)
    trans = [256]
    for n in nodes:
        if n.op == "conv_bn_relu_bwd" and dgrad_s2(g.convs[n.attrs["conv"]]):
            trans.append(nodes[n.parents[1]].nbytes)          # stride-2 input gradient
    ws["transient"] = max(trans)
    return ws


def own_dgrad(cs: G.ConvSpec) -> bool:
    """Input gradients as ONE conv through our tcgen05 kernel (transposed /
    flipped weights; fused backward epilogues: residual add + ReLU mask,
    BN-backward reductions; a stride-2 1x1's gradient is computed on its
    sampling grid and scattered by the consumer's epilogue): every 1x1 and
    every stride-1 3x3.  The stem has no input gradient."""
    return cs.k == 1 or cs.stride == 1


def dgrad_s2(cs: G.ConvSpec) -> bool:
    """The stride-2 3x3 input gradients (conv2 of the first block of layers
    2-4): four sub-pixel stride-1 convs over dY, one per output parity class
    (a, b) — taps {1} or {2, 0} of the flipped weights per dimension, pad 0
    before / 1 after — each writing its class of the gradient directly
    (conv_fwd.cu EV_SCATTER); no zero-inserted upsampling, no wasted MMAs."""
    return cs.k == 3 and cs.stride == 2


@dataclass
class StepStats:
    loss: float
    ms: float


class DeltaRuntime:
    """ResNet training step under a DELTA activation budget on one B200."""

    def __init__(self, depth: int | G.Graph = 50, batch: int = 256, image: int = 224,
                 device: str = "cuda", seed: int = 0, anchors: str = "out+narrow",
                 lr: float = 0.1):
        """depth: 50 / 101 for the built-in ResNets, or a prebuilt graph (e.g.
        importer.graph_from_module of a PyTorch model; batch / image are then
        the graph's)."""
        self.device = torch.device(device)
        if isinstance(depth, G.Graph):
            self.g = depth
            batch = self.g.nodes[0].shape[0]
        else:
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
        # zeroed: the one-launch BN backward keeps its grid-barrier words here
        self.bn_ws = torch.zeros(ws["bn_ws"] // 4, dtype=torch.float32, device=self.device)
        # BN statistics partials written by the conv epilogue (one 128-row
        # tile per partial); downsample convs use their own scratch because
        # their BN is applied together with the block's bn3.
        self.stats_main = f32("stats_main")
        self.stats_ds = f32("stats_ds")
        # the BN3 backward sums reduced by the next block's shortcut dgrad
        self.stats_sums = f32("stats_sums")
        # backward scratch outside the budget: the input gradient of a stride-2
        # shortcut conv at its sampling grid
        self.short_ws = u8("short_ws")
        self.mp_ws = u8("mp_ws")
        # weight-gradient partials + split counters (zeroed once; side stream: serial use)
        self.wg_ws = torch.zeros(ws["wgrad_ws"], dtype=torch.uint8, device=self.device)
        # a stride-2 3x3 input gradient between its sub-pixel convs and its BN backward
        self.dg_ws = u8("transient")
        ncls = self.g.fc[1]
        self.loss = torch.zeros(1, dtype=torch.float32, device=self.device)
        self.dlogits = torch.empty(batch, ncls, dtype=torch.float32, device=self.device)
        self.dlogits_bf16 = torch.empty(batch, self.g.fc_pad, dtype=torch.bfloat16,
                                        device=self.device)
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
        self.executor = None
        self._bound_slot = None
        self.graph = None
        self.cost_table = None
        self.link_gbs = None
        self.dp = None  # torch.distributed group when running data parallel
        self.buckets = []
        self._comm = None

    # ------------------------------------------------------------ setup
    def _build_convs(self):
        # epilogue BN statistics cost ~11*BN cycles per tile against ~2*kblocks*BN
        # of MMA: fused only where the main loop hides them (K-dim >= 384)
        self._fuse_stats = {}
        self._dconvs = {}
        self._dconvs_s2 = {}
        self._wgrads = {}
        bn_bwd_convs = {n.attrs["conv"] for n in self.nodes if n.op == "conv_bn_relu_bwd"}
        sums_convs = {n.attrs["conv"] for n in self.nodes
                      if n.op == "conv_shortcut_bwd" and "sums_xc" in n.attrs}
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
                self._wgrads[cs.name] = K.Wgrad(Nb, H, W, C, cs.cout, cs.k, cs.k, cs.stride,
                                                cs.pad)
                if own_dgrad(cs):
                    # on the conv's output grid (a stride-2 1x1's gradient lives at
                    # its sampling points; the consumer scatters it)
                    _, P_, Q_, _ = n.shape
                    dconv = K.Conv(Nb, P_, Q_, cs.cout, cs.cin, cs.k, cs.k, 1, cs.k // 2,
                                   _ptr(self.params.wd[cs.name]))
                    if dconv.tile_n > 128:
                        # fused backward epilogues run at N tiles of 128, except
                        # the BN-backward one at >= 2 waves of 256-column tiles
                        # (layer 3: 65 -> 52 us per 3x3, 44 -> 40 per 1x1)
                        wide = (DGRAD_BN256 and cs.name in bn_bwd_convs
                                and Nb * P_ * Q_ >= 2 * 148 * 128)
                        dconv.set_tile_n(256 if wide else 128)
                    if cs.name in sums_convs:
                        dconv.set_tile_n(64)  # three epilogue operands: 64-column tiles
                    self._dconvs[cs.name] = dconv
                if dgrad_s2(cs):
                    # four sub-pixel convs over dY [Nb][P][Q][cout], class (a, b):
                    # (1+a) x (1+b) taps, pad 0 before, a / b after
                    _, P_, Q_, _ = n.shape
                    assert (2 * P_, 2 * Q_) == (H, W), (n.name, H, W, P_, Q_)
                    self._dconvs_s2[cs.name] = [
                        K.Conv(Nb, P_, Q_, cs.cout, cs.cin, 1 + (c >> 1), 1 + (c & 1), 1, 0,
                               _ptr(self.params.wd_s2[cs.name][c]), pad_end=(c >> 1, c & 1))
                        for c in range(4)]
            elif n.op == "fc":
                # the classifier as a 1x1 conv over the pooled features (tcgen05):
                # logits [N][fc_pad] bf16; its input gradient likewise over the
                # bf16 logit gradients, and its weight gradient on the wgrad kernel
                Nb, cin = self.nodes[n.parents[0]].shape
                pad = self.g.fc_pad
                self._fc = K.Conv(Nb, 1, 1, cin, pad, 1, 1, 1, 0, _ptr(self.params.wbf["fc"]))
                self._fc_d = K.Conv(Nb, 1, 1, pad, cin, 1, 1, 1, 0, _ptr(self.params.wd["fc"]))
                self._fc_w = K.Wgrad(Nb, 1, 1, cin, pad, 1, 1, 1, 0)

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
             policy=P.PolicyMode.Delta, duplex: bool = False, **kw):
        """Plan with libdelta and lower onto the arena.  budget_fraction=None
        plans the no-eviction baseline (Baseline policy, budget = sum).
        duplex: reloads on a second copy engine (default: one copy stream in
        plan order, the reference's model).  The arena always fits the
        budget: when the offline packing of a plan's lifetimes fragments past
        it, the plan is redone under a budget smaller by the excess
        (self.config = the config actually planned; self.budget_bytes = the
        caller's budget)."""
        t = self.trace()
        if budget_fraction is None and budget is None:
            total = sum(n.nbytes for n in self.nodes)
            cfg = self.engine_config(total, P.PolicyMode.Baseline, **kw)
        else:
            if budget is None:
                budget = int(self.baseline_peak() * budget_fraction)
            cfg = self.engine_config(budget, policy, **kw)
        target = cfg.budget
        for _ in range(16):
            prog = P.Program(t, cfg, align=G.ALIGN, duplex=duplex)
            if prog.infeasible:
                node, deficit = prog.infeasible
                raise RuntimeError(f"plan infeasible at node {self.nodes[node].name} "
                                   f"(deficit {deficit} B, budget {cfg.budget} B)")
            if prog.arena_bytes <= target or cfg.policy_mode == P.PolicyMode.Baseline:
                break
            # the offline packing of this plan's lifetimes fragments past the
            # budget (the reference's pool is a byte counter): plan again under
            # a budget smaller by the excess, so the ARENA fits the caller's
            # budget; the plan is then the reference's plan at that budget
            cfg = dataclasses.replace(
                cfg, budget=cfg.budget - max(prog.arena_bytes - target, target // 256))
        if prog.arena_bytes > target and cfg.policy_mode != P.PolicyMode.Baseline:
            raise RuntimeError(f"arena {prog.arena_bytes} B exceeds the budget {target} B")
        self.budget_bytes = target  # the caller's budget: the arena fits it
        self.program = prog
        self.config = cfg
        self.graph = None
        self.graphs = None
        if self.arena is None or self.arena.numel() < prog.arena_bytes:
            self.executor = None
            self.arena = None
            torch.cuda.empty_cache()
            self.arena = torch.empty(prog.arena_bytes, dtype=torch.uint8, device=self.device)
        if self.executor is None or self.executor.host_bytes < prog.host_bytes:
            host = max(prog.host_bytes, self.executor.host_bytes if self.executor else 0)
            self.executor = X.Executor(_ptr(self.arena), self.arena.numel(), host)
        self._base = _ptr(self.arena)
        self._bound_slot = None
        return prog

    # -------------------------------------------------------- tensors
    def _view(self, off: int, node: G.Node) -> torch.Tensor:
        dt = torch.float32 if node.dtype_bytes == 4 else torch.bfloat16
        n = int(np.prod(node.shape))
        return self.arena.narrow(0, off, n * node.dtype_bytes).view(dt).view(node.shape)

    # ------------------------------------------------------------ ops
    # ------------------------------------------------------------ recipes
    def _recipe(self, node: G.Node) -> tuple:
        """The kernel ops that (re)produce `node` on the executor: symbolic
        arena operands (OUT, IN(i)) and parameter / workspace pointers, every
        one a kernel of this library.  Returns (ops, (launches of our kernels
        on first production, on recompute))."""
        pr = self.params
        op = node.op
        ops = []
        nl = [0, 0]

        def add(k, first=1, rec=1):
            ops.append(k)
            if not (k.flags & X.RECOMPUTE_ONLY):
                nl[0] += first
            if not (k.flags & X.FIRST_ONLY):
                nl[1] += rec

        M = int(np.prod(node.shape[:-1])) if len(node.shape) == 4 else 0
        C = node.shape[-1]
        # streaming BN backward: one persistent launch (bn_pool.cu k_bn_bwd_grid)
        # or partial + merge(s) + apply
        bwd_n = (1 if K.BN_BWD_ONE_LAUNCH else 2 + K._merge_launches(K._chunks(M, C))) if M else 0
        bnp = lambda bn: (_ptr(pr.bn_mean[bn]), _ptr(pr.bn_invstd[bn]))
        gb = lambda bn: (_ptr(pr.views["bn_g:" + bn]), _ptr(pr.views["bn_b:" + bn]))
        dgb = lambda bn: (_ptr(pr.gviews["bn_g:" + bn]), _ptr(pr.gviews["bn_b:" + bn]))

        def stats(conv_node_id, src_ref, bn, scratch):
            """training-mode BN statistics (first production only: a recompute
            reuses them): from the conv epilogue's partials when that conv is
            long enough to hide the work, else one streaming pass."""
            conv = self.nodes[conv_node_id]
            tail = (_ptr(pr.bn_mean[bn]), _ptr(pr.bn_invstd[bn]), _ptr(pr.bn_rmean[bn]),
                    _ptr(pr.bn_rvar[bn]))
            if self._fuse_stats.get(conv.name):
                add(X.kop(X.K_BN_STATS_PARTS, (_ptr(scratch), None) + tail, (M, C, 0),
                          (BN_EPS, BN_MOMENTUM), flags=X.FIRST_ONLY), 1, 0)
            else:
                add(X.kop(X.K_BN_STATS, (src_ref, _ptr(self.bn_ws)) + tail, (M, C),
                          (BN_EPS, BN_MOMENTUM), flags=X.FIRST_ONLY),
                    1 + K._merge_launches(K._chunks(M, C)), 0)

        def wgrad(conv, dy_in, x_in, side=True):
            """our tcgen05 weight gradient straight into the fp32 KRSC grad buffer,
            on the side stream (it only reads the node's inputs: it overlaps the
            input-gradient chain and is joined at the node's end)"""
            return X.kop(X.K_WGRAD, (X.IN(dy_in), X.IN(x_in), _ptr(pr.gviews["conv:" + conv]),
                                     _ptr(self.wg_ws)),
                         conv=self._wgrads[conv]._h, flags=X.SIDE if side else 0)

        if op == "input":
            add(X.kop(X.K_COPY, (X.OUT(), _ptr(self.x_dev)), (self.x_dev.numel() * 2,)))
        elif op == "conv":
            # the first production also emits BN statistics partials from the
            # epilogue; a recompute must not (the scratch may be in use)
            conv = self._convs[node.name]._h
            if self._fuse_stats[node.name]:
                scratch = self.stats_ds if "downsample" in node.name else self.stats_main
                add(X.kop(X.K_CONV, (X.IN(0), X.OUT(), _ptr(scratch)), conv=conv,
                          flags=X.FIRST_ONLY))
                add(X.kop(X.K_CONV, (X.IN(0), X.OUT(), None), conv=conv, flags=X.RECOMPUTE_ONLY))
            else:
                add(X.kop(X.K_CONV, (X.IN(0), X.OUT(), None), conv=conv))
        elif op in ("bn_relu", "bn_add_relu", "bn_bn_add_relu"):
            bn = node.attrs["bn"]
            stats(node.parents[0], X.IN(0), bn, self.stats_main)
            mode = {"bn_relu": 0, "bn_add_relu": 1, "bn_bn_add_relu": 2}[op]
            p2 = (None,) * 4
            if mode == 2:
                bn2 = node.attrs["bn2"]
                stats(node.parents[1], X.IN(1), bn2, self.stats_ds)
                p2 = bnp(bn2) + gb(bn2)
            add(X.kop(X.K_BN_APPLY, (X.IN(0), X.IN(1) if mode else None, X.OUT()) + bnp(bn)
                      + gb(bn) + p2, (mode, M, C)))
        elif op == "maxpool":
            Nb, H, W, Cs = self.nodes[node.parents[0]].shape
            add(X.kop(X.K_MAXPOOL_FWD, (X.IN(0), X.OUT()), (Nb, H, W, Cs)))
        elif op == "avgpool":
            Nb, H, W, Cs = self.nodes[node.parents[0]].shape
            add(X.kop(X.K_AVGPOOL, (X.IN(0), X.OUT()), (Nb, H * W, Cs)))
        elif op == "fc":
            # logits = pooled @ W^T on the tensor cores (bias: in the head kernel)
            add(X.kop(X.K_CONV, (X.IN(0), X.OUT(), None), conv=self._fc._h))
        elif op == "fc_bwd":
            # softmax cross-entropy on logits + bias -> loss, dlogits (fp32 and
            # padded bf16), dbias; then dPooled = dlogits @ W and dW = dlogits^T
            # @ pooled on the tensor cores
            Nb = node.shape[0]
            ncls = self.g.fc[1]
            add(X.kop(X.K_XENT_HEAD, (X.IN(0), _ptr(pr.views["fc_b"]), _ptr(self.y_dev),
                                      _ptr(self.loss), _ptr(self.dlogits),
                                      _ptr(self.dlogits_bf16), _ptr(pr.gviews["fc_b"]),
                                      _ptr(self.row_loss)), (Nb, ncls, self.g.fc_pad)), 3, 3)
            add(X.kop(X.K_CONV, (_ptr(self.dlogits_bf16), X.OUT(), None), conv=self._fc_d._h))
            add(X.kop(X.K_WGRAD, (_ptr(self.dlogits_bf16), X.IN(1),
                                  _ptr(pr.gviews["fc_w_full"]), _ptr(self.wg_ws)),
                      conv=self._fc_w._h), self._fc_w.launches, self._fc_w.launches)
        elif op == "bn_add_relu_bwd":
            # parents: [upstream, (O if masked,) X]; upstream already masked
            # unless it is the pooled head gradient
            bn = node.attrs["bn"]
            pool_hw = int(node.shape[1] * node.shape[2]) if node.attrs.get("from_pool") else 0
            mask = X.IN(1) if node.attrs.get("masked") else None
            if node.attrs.get("sums_fused"):
                # (sum g, sum g*X) came with g from the shortcut dgrad's epilogue
                add(X.kop(X.K_BN_BWD_PARTS, (_ptr(self.stats_sums), X.IN(0), X.IN(1), X.OUT())
                          + bnp(bn) + (gb(bn)[0],) + dgb(bn), (0, M, C)), 2, 2)
            else:
                add(X.kop(X.K_BN_BWD, (X.IN(0), mask, X.IN(len(node.parents) - 1), X.OUT())
                          + bnp(bn) + (gb(bn)[0],) + dgb(bn) + (_ptr(self.bn_ws),),
                          (pool_hw, M, C)), bwd_n, bwd_n)
        elif op == "conv_bn_relu_bwd":
            # parents [dC, R = relu(bn(X)), X]
            conv, bn = node.attrs["conv"], node.attrs["bn"]
            if conv in self._dconvs:
                # dgrad on the tensor cores; its epilogue applies the ReLU mask
                # (recomputed from X) and reduces sum g, sum g*X per tile; g is
                # written in place of its BN-backward output
                add(X.kop(X.K_CONV_EX, (X.IN(0), X.OUT(), _ptr(self.stats_main), None, None, None,
                                        X.IN(2)) + bnp(bn) + gb(bn),
                          (K.EPI_BN_BWD, 0, 0), conv=self._dconvs[conv]._h))
                add(X.kop(X.K_BN_BWD_PARTS, (_ptr(self.stats_main), X.OUT(), X.IN(2), X.OUT())
                          + bnp(bn) + (gb(bn)[0],) + dgb(bn), (0, M, C)), 2, 0)
            elif conv in self._dconvs_s2:
                # stride-2 3x3: the four sub-pixel parity classes write the
                # input gradient into the scratch, then the streaming BN backward
                for cls, dc in enumerate(self._dconvs_s2[conv]):
                    add(X.kop(X.K_CONV_EX, (X.IN(0), _ptr(self.dg_ws), None),
                              (K.EPI_SCATTER2, 0, 0, cls), conv=dc._h))
                add(X.kop(X.K_BN_BWD, (_ptr(self.dg_ws), X.IN(1), X.IN(2), X.OUT()) + bnp(bn)
                          + (gb(bn)[0],) + dgb(bn) + (_ptr(self.bn_ws),), (0, M, C)), bwd_n, bwd_n)
            else:
                raise RuntimeError(f"{node.name}: no input-gradient kernel for conv {conv}")
            add(wgrad(conv, 0, 1), *(self._wgrads[conv].launches,) * 2)
        elif op == "conv_shortcut_bwd":
            # out = (dgrad(conv1, dC1) + shortcut gradient) * [X > 0]; the sum
            # and the mask are the dgrad kernel's epilogue
            conv = node.attrs["conv"]
            out_mask = X.IN(1) if node.attrs.get("mask_out") else None
            add_, pool_hw, add_mask, stride2 = None, 0, None, 0
            if "conv_short" in node.attrs:
                short = node.attrs["conv_short"]
                if short in self._dconvs:
                    if self.g.convs[short].stride == 1:
                        dst = X.OUT()   # summed in place by conv1's dgrad epilogue
                    else:
                        dst, stride2 = _ptr(self.short_ws), 1  # at its sampling grid
                    add(X.kop(X.K_CONV, (X.IN(2), dst, None), conv=self._dconvs[short]._h))
                    add_ = dst
                else:
                    raise RuntimeError(f"{node.name}: shortcut conv {short} must be a 1x1")
                add(wgrad(short, 2, 1), *(self._wgrads[short].launches,) * 2)
            elif node.attrs.get("from_pool"):
                add_, pool_hw, add_mask = X.IN(2), int(node.shape[1] * node.shape[2]), X.IN(3)
            else:
                add_ = X.IN(2)
            if conv not in self._dconvs:
                raise RuntimeError(f"{node.name}: the shortcut's conv1 must be a 1x1 (own dgrad)")
            if "sums_xc" in node.attrs:
                # + the previous block's BN3 backward sums over (g, its C3)
                add(X.kop(X.K_CONV_EX, (X.IN(0), X.OUT(), _ptr(self.stats_sums), add_, add_mask,
                                        out_mask, X.IN(node.attrs["sums_xc"])),
                          (K.EPI_ADD_MASK, pool_hw, stride2), conv=self._dconvs[conv]._h))
            else:
                add(X.kop(X.K_CONV_EX, (X.IN(0), X.OUT(), None, add_, add_mask, out_mask),
                          (K.EPI_ADD_MASK, pool_hw, stride2), conv=self._dconvs[conv]._h))
            add(wgrad(conv, 0, 1), *(self._wgrads[conv].launches,) * 2)
        elif op == "conv_bwd":
            # a conv fed by a maxpool (imported chains): plain input gradient on
            # the tensor cores + weight gradient
            conv = node.attrs["conv"]
            if conv not in self._dconvs:
                raise RuntimeError(f"{node.name}: no input-gradient kernel for conv {conv}")
            add(X.kop(X.K_CONV, (X.IN(0), X.OUT(), None), conv=self._dconvs[conv]._h))
            add(wgrad(conv, 0, 1), *(self._wgrads[conv].launches,) * 2)
        elif op == "maxpool_bwd":
            Nb, H, W, Cs = self.nodes[node.parents[1]].shape
            add(X.kop(X.K_MAXPOOL_BWD, (X.IN(0), X.IN(1), X.OUT(), _ptr(self.mp_ws)),
                      (Nb, H, W, Cs)), 2, 2)
        elif op == "bn_relu_bwd":
            bn = node.attrs["bn"]
            add(X.kop(X.K_BN_BWD, (X.IN(0), X.IN(1), X.IN(2), X.OUT()) + bnp(bn) + (gb(bn)[0],)
                      + dgb(bn) + (_ptr(self.bn_ws),), (0, M, C)), bwd_n, bwd_n)
        elif op == "conv_wgrad":
            # the node's output IS the weight gradient (fp32): written in place,
            # then copied into the flat gradient buffer
            conv = node.attrs["conv"]
            add(X.kop(X.K_WGRAD, (X.IN(0), X.IN(1), X.OUT(), _ptr(self.wg_ws)),
                      conv=self._wgrads[conv]._h), 2, 2)
            add(X.kop(X.K_COPY, (_ptr(pr.gviews["conv:" + conv]), X.OUT()), (node.nbytes,)))
        else:
            raise RuntimeError(f"no kernel for op {op!r} (node {node.name})")
        return ops, tuple(nl)

    def _arena_view(self, ptr: int, node_id: int) -> torch.Tensor:
        return self._view(ptr - self._base, self.nodes[node_id])

    def _bind(self):
        """(Re)build the recipe table for the current input slot and bind it,
        with the current program, to the executor."""
        recipes, launches = {}, {}
        for node in self.nodes:
            ops, nl = self._recipe(node)
            recipes[node.id] = ops
            launches[node.id] = nl
        self.executor.bind(self.program, recipes, [], launches)
        if self.dp is not None:
            # gradient buckets released by ready events of their last writer
            bk = self.grad_buckets()
            nodes = sorted({b[2] for b in bk})
            self.executor.set_ready_nodes(nodes)
            self.ready_nodes = nodes
            self.buckets = [(lo, hi, nodes.index(w)) for lo, hi, w in bk]
        self._bound_slot = self._slot

    # -------------------------------------------------------- program
    def run_program(self, timing: dict | None = None, probe: dict | None = None,
                    stamps: list | None = None, observe: list | None = None):
        """Issue one training step: the lowered action program through the
        C++ executor (csrc/rt/executor.cu) on the compute stream and the two
        copy engines, then the optimizer.  The loss stays on device.
        `timing`: node id -> [(ms, recomputed)], plus "swap" -> [(ms, op,
        bytes)]; `probe`: node id -> a clone of its output after its (last)
        production; `stamps`: receives (action index, start_ms, end_ms) of
        every compute/recompute/offload/reload action; `observe`: receives the
        device-side action log of the step (Executor.step_observed)."""
        st = self.stream.cuda_stream
        if self._bound_slot != self._slot:
            self._bind()
        after = None
        if probe is not None:
            def after(ai, node, out):
                if node in probe:
                    probe[node] = self._arena_view(out, node).clone()
        if observe is not None:
            observe.append(self.executor.step_observed(st))
        elif timing is not None or stamps is not None:
            t0, t1 = self.executor.step_timed(st, after)
            acts = self.program.actions
            for ai, a in enumerate(acts):
                op = int(a["op"])
                if op in (P.ACT_COMPUTE, P.ACT_RECOMPUTE, P.ACT_OFFLOAD, P.ACT_RELOAD):
                    if stamps is not None:
                        stamps.append((ai, float(t0[ai]), float(t1[ai])))
                    if timing is not None:
                        ms = float(t1[ai] - t0[ai])
                        if op in (P.ACT_COMPUTE, P.ACT_RECOMPUTE):
                            timing.setdefault(int(a["node"]), []).append(
                                (ms, op == P.ACT_RECOMPUTE))
                        else:
                            timing.setdefault("swap", []).append((ms, op, int(a["bytes"])))
        else:
            self.executor.step(st, after)
        K._count(self.executor.launches_per_step)
        if self.dp is not None:
            self._allreduce_buckets()
        self._optimizer_step()

    def _optimizer_step(self):
        self.params.sgd_step(self.lr)

    def _slot_tensors(self, slot: int) -> list:
        """the device tensors one staged batch occupies (same order as the
        host tuple a batch is given as)"""
        return [self.x_slots[slot], self.y_slots[slot]]

    def _allreduce_buckets(self):
        """Data parallel: one DELTA instance per GPU; the flat
        fp32 gradient buffer is averaged across ranks in ~25 MB buckets on a
        dedicated communication stream.  Bucket b waits (delta_rt_wait_ready)
        for the event the executor records right after the backward node that
        writes its last gradient, so its all-reduce overlaps the rest of the
        backward pass; the compute stream joins the communication stream
        before the optimizer step.  Capturable into the step's CUDA graph."""
        if self._comm is None:
            self._comm = torch.cuda.Stream(device=self.device)
        cur = torch.cuda.current_stream()
        g = self.params.grad
        for lo, hi, ev in self.buckets:
            self.executor.wait_ready(self._comm.cuda_stream, ev)
            with torch.cuda.stream(self._comm):
                allreduce_mean(g[lo:hi], self.dp)
        cur.wait_stream(self._comm)

    def grad_buckets(self, bucket_bytes: int = 25 * 2**20):
        """Partition the flat gradient buffer into contiguous buckets of about
        `bucket_bytes`, each released by the LAST backward node (in program
        order) that writes a gradient inside it — read off the recipes: every
        kernel operand pointing into the gradient buffer marks its node as a
        writer of the parameter starting there.  Returns [(lo, hi, node)] in
        float elements, ordered by release."""
        g0 = self.params.grad.data_ptr()
        g1 = g0 + self.params.grad.numel() * 4
        writer = {}
        for node in self.nodes:
            ops, _ = self._recipe(node)
            for k in ops:
                for r in k.r:
                    if r.kind == X.REF_PTR and g0 <= r.ptr < g1:
                        writer[r.ptr] = max(writer.get(r.ptr, -1), node.id)
        items = []
        for name, gv in self.params.gviews.items():
            if name == "fc_w":  # a view of fc_w_full
                continue
            p = gv.data_ptr()
            if p not in writer:
                raise RuntimeError(f"no backward node writes the gradient of {name}")
            items.append(((p - g0) // 4, gv.numel(), writer[p]))
        items.sort()
        assert items[0][0] == 0 and all(a[0] + a[1] == b[0] for a, b in zip(items, items[1:]))
        buckets, lo, last = [], 0, -1
        for off, n, w in items:
            last = max(last, w)
            if (off + n - lo) * 4 >= bucket_bytes or off + n == self.params.grad.numel():
                buckets.append((lo, off + n, last))
                lo, last = off + n, -1
        return sorted(buckets, key=lambda b: b[2])


    def capture(self):
        """Capture one full step (program + optimizer) as a CUDA graph per
        input staging slot (two slots let `train` overlap the next batch's
        host->device copy with the current step)."""
        torch.cuda.synchronize()
        graphs = []
        for slot in range(2):
            self._use_slot(slot)
            self._bind()  # the recipe table reads this slot's input buffers
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
        return self._step_host((x_host, y_host))

    def _step_host(self, batch) -> float:
        with torch.cuda.stream(self.stream):
            for dst, src in zip(self._slot_tensors(self._slot), batch):
                dst.copy_(src, non_blocking=True)
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
                for dst, src in zip(self._slot_tensors(slot), batches[i]):
                    dst.copy_(src, non_blocking=True)
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

    def executed_timeline(self, findings: list | None = None) -> np.ndarray:
        """One eager step with a DEVICE-side action log (delta_rt_step_observed:
        a stamp kernel on each action's own stream appends %globaltimer, the
        action and its node/op when the stream reaches it) turned into a
        reference Timeline (engine.hpp:44-70) for oracle::replay_check:

        * Compute / Recompute / Offload / Reload events are the device's
          records: kind and node as the executor ran them, start = head stamp,
          duration = tail - head (µs from the first stamp);
        * the zero-duration markers of the plan (Use, Free, Evict) take the end
          of the latest compute-stream action (or Stall) before them in plan
          order; a Stall spans the measured gap from there to the next
          compute-stream action.

        `findings` (optional list) receives every disagreement between the
        device log and the lowered program: an action missing, duplicated or
        run with another node/op, or a stream that ran its actions out of
        program order.  Empty == the GPU ran exactly the program, in order."""
        recs = []
        with torch.cuda.stream(self.stream):
            self.run_program(observe=recs)
        torch.cuda.synchronize()
        rec = recs[0]
        acts = self.program.actions
        found = [] if findings is None else findings
        work_ops = (P.ACT_COMPUTE, P.ACT_RECOMPUTE, P.ACT_OFFLOAD, P.ACT_RELOAD)
        head, tail = {}, {}
        for r in rec:
            ai = int(r["action"])
            d = tail if r["tail"] else head
            if ai in d:
                found.append(f"action {ai}: duplicate {'tail' if r['tail'] else 'head'} stamp")
            d[ai] = r
            if ai >= len(acts):
                found.append(f"action {ai}: not in the program")
                continue
            a = acts[ai]
            if int(r["node"]) != int(a["node"]) or int(r["op"]) != int(a["op"]):
                found.append(f"action {ai}: device ran op {int(r['op'])} of node {int(r['node'])}, "
                             f"program has op {int(a['op'])} of node {int(a['node'])}")
        last_seq = {}
        for ai, a in enumerate(acts):
            if int(a["op"]) not in work_ops:
                continue
            if ai not in head or ai not in tail:
                found.append(f"action {ai} (op {int(a['op'])}, node {int(a['node'])}) not executed")
                continue
            if int(tail[ai]["seq"]) < int(head[ai]["seq"]) or tail[ai]["t_ns"] < head[ai]["t_ns"]:
                found.append(f"action {ai}: tail stamp before its head")
            s_ = int(a["stream"])
            if s_ in last_seq and int(head[ai]["seq"]) < last_seq[s_]:
                found.append(f"action {ai}: stream {s_} ran it before an earlier program action")
            last_seq[s_] = int(tail[ai]["seq"])
        t0 = int(rec["t_ns"].min()) if len(rec) else 0
        us = lambda t: int(round((int(t) - t0) / 1000.0))
        kind_of = {P.ACT_COMPUTE: P.EventKind.Compute, P.ACT_RECOMPUTE: P.EventKind.Recompute,
                   P.ACT_OFFLOAD: P.EventKind.Offload, P.ACT_RELOAD: P.EventKind.Reload}
        by_event = {}
        for ai, a in enumerate(acts):
            if int(a["op"]) in work_ops and ai in head and ai in tail:
                by_event[int(a["plan_event"])] = ai
        plan = P.run_iteration(self.trace(), self.config).events
        ev = plan.copy()
        # compute-stream work starts in plan order (for Stall spans)
        next_start = [None] * len(ev)
        nxt = None
        for i in range(len(ev) - 1, -1, -1):
            next_start[i] = nxt
            ai = by_event.get(i)
            if ai is not None and int(acts[ai]["stream"]) == P.STREAM_COMPUTE:
                nxt = us(head[ai]["t_ns"])
        now = 0
        for i in range(len(ev)):
            ai = by_event.get(i)
            if ai is not None:
                h, t = head[ai], tail[ai]
                ev[i]["kind"] = kind_of[int(h["op"])]
                ev[i]["node"] = int(h["node"])
                ev[i]["stream"] = (P.StreamKind.Compute if int(h["op"]) in (P.ACT_COMPUTE, P.ACT_RECOMPUTE)
                                   else P.StreamKind.Copy)
                ev[i]["ts"] = us(h["t_ns"])
                ev[i]["duration"] = us(t["t_ns"]) - us(h["t_ns"])
                if ev[i]["stream"] == P.StreamKind.Compute:
                    now = max(now, int(ev[i]["ts"] + ev[i]["duration"]))
            elif int(ev[i]["kind"]) in (P.EventKind.Compute, P.EventKind.Recompute,
                                        P.EventKind.Offload, P.EventKind.Reload):
                found.append(f"plan event {i} ({int(ev[i]['kind'])} of node {int(ev[i]['node'])}) "
                             "has no executed action")
            else:
                ev[i]["ts"] = now
                ev[i]["duration"] = 0
                if int(ev[i]["kind"]) == P.EventKind.Stall and next_start[i] is not None:
                    # the measured wait: up to the next compute-stream start;
                    # later markers of this gap follow the stall
                    ev[i]["duration"] = max(0, next_start[i] - now)
                    now += int(ev[i]["duration"])
        return ev

    # ----------------------------------------------------- cost model
    def measure_costs(self, iters: int = 3, link: bool = True):
        """GPU-resident cost model: time every node's op on device (CUDA events
        around each action of the no-eviction program, median of `iters`
        steps), quantise to whole microseconds (>= 1) and write them into the
        trace; probe the pinned host link for the swap cost."""
        self.plan(None)
        if self._bound_slot != self._slot:
            self._bind()
        # the probe steps run the program only (no optimizer step), but their
        # first productions update the BN running statistics: keep them
        pr = self.params
        saved = {n: (pr.bn_rmean[n].clone(), pr.bn_rvar[n].clone()) for n in pr.bn_rmean}
        with torch.cuda.stream(self.stream):
            costs = self.executor.measure_costs(self.stream.cuda_stream, iters, len(self.nodes))
        torch.cuda.synchronize()
        for n, (m, v) in saved.items():
            pr.bn_rmean[n].copy_(m)
            pr.bn_rvar[n].copy_(v)
        table = {}
        for n in self.nodes:
            n.cost_us = max(1, int(costs[n.id]))
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

"""A PyTorch CNN as a DELTA graph the B200 runtime executes.

`capture.py` records any training step at the ATen level as a trace the
planner (and the reference simulator) accepts, but such a trace names ATen
ops, which the runtime cannot execute.  This module captures a model at the
module level instead — `torch.fx` symbolic tracing of an `nn.Module` — and
registers it with the runtime's own node vocabulary (graph.py), so every node
has a recipe of this library's sm_100a kernels:

  forward   Conv2d(bias=False) -> BatchNorm2d -> ReLU   conv, bn_relu
            MaxPool2d(3, 2, 1)                          maxpool
            AdaptiveAvgPool2d(1) -> Flatten -> Linear   avgpool, fc
  backward  fc_bwd; the last unit's BN-ReLU backward of the pooled gradient
            (bn_add_relu_bwd, from_pool); per conv fed by a BN-ReLU output its
            input gradient fused with that BN-ReLU backward (conv_bn_relu_bwd,
            stride-1 or the stride-2 sub-pixel path); a conv fed by a maxpool
            (conv_bwd) and maxpool_bwd -> bn_relu_bwd; the first conv's
            weight gradient (conv_wgrad)

Supported: a chain of those modules (no residual branches), the first conv
either the 7x7/2 pad-3 stem over a 3-channel image (padded to 4) or any conv
over a multiple of 64 channels; every conv has a multiple of 64 input and a
power-of-two (64..2048) output channels and is 1x1 (stride 1) or 3x3 (pad 1,
stride 1 or 2).  Anything
else raises — there is no fallback path.  `load_weights` copies the module's
parameters and BN buffers into the runtime, so the DELTA step computes the
module's own training step (checked against fp32 autograd in the GPU tests).
"""
from __future__ import annotations

import torch
import torch.fx as fx
import torch.nn as nn

from . import graph as G


class UnsupportedModel(ValueError):
    pass


def _chain(model: nn.Module):
    """The model's modules in call order (a straight chain) from torch.fx."""
    gm = fx.symbolic_trace(model)
    mods = dict(gm.named_modules())
    chain, prev = [], None
    for node in gm.graph.nodes:
        if node.op == "placeholder":
            prev = node
            continue
        if node.op == "output":
            break
        if node.op == "call_module":
            ins = [a for a in node.args if isinstance(a, fx.Node)]
            if ins != [prev]:
                raise UnsupportedModel(f"{node.target}: not a straight chain (branches)")
            chain.append((node.target, mods[node.target]))
            prev = node
        elif node.op == "call_function" and node.target is torch.flatten:
            chain.append(("flatten", nn.Flatten()))
            prev = node
        else:
            raise UnsupportedModel(f"unsupported graph node {node.op} {node.target}")
    return chain


def graph_from_module(model: nn.Module, batch: int, image: int, in_channels: int = 3,
                      name: str = "imported") -> tuple[G.Graph, dict]:
    """(graph, names): names maps graph parameter names (conv / bn / fc) to
    the module's qualified names, for load_weights."""
    chain = _chain(model)
    g = G.Graph(f"{name}_bs{batch}")
    names = {"conv": {}, "bn": {}, "fc": None}
    stem = in_channels == 3
    cin0 = 4 if stem else in_channels
    if not stem and cin0 % 64:
        raise UnsupportedModel("input channels: 3 (stem) or a multiple of 64")
    x = g.add("input", "input", (batch, image, image, cin0), [], uncomputable=True,
              evict_pinned=True)
    cur = x
    units = []        # (conv node, bn-relu node, input node kind)
    i = 0
    pooled = None
    logits = None
    while i < len(chain):
        qn, m = chain[i]
        if isinstance(m, nn.Conv2d):
            if m.bias is not None or m.groups != 1 or m.dilation != (1, 1):
                raise UnsupportedModel(f"{qn}: conv must be bias-free, ungrouped, undilated")
            k, s, p = m.kernel_size[0], m.stride[0], m.padding[0]
            if (m.kernel_size[1], m.stride[1], m.padding[1]) != (k, s, p):
                raise UnsupportedModel(f"{qn}: square kernels only")
            first = cur is x
            if first and stem:
                if (k, s, p, m.in_channels) != (7, 2, 3, 3) or m.out_channels != 64:
                    raise UnsupportedModel(f"{qn}: the 3-channel stem must be 7x7/2 pad 3, 64 out")
            else:
                if m.in_channels % 64 or (k, p) not in ((1, 0), (3, 1)) or \
                        (k == 1 and s != 1) or s not in (1, 2):
                    raise UnsupportedModel(f"{qn}: 1x1/s1 or 3x3/p1 (s1, s2) over 64k channels")
            oc = m.out_channels
            if oc < 64 or oc > 2048 or oc & (oc - 1):
                raise UnsupportedModel(f"{qn}: output channels must be a power of two in [64, 2048]"
                                       " (the BN kernels' channel slices)")
            if i + 2 >= len(chain) or not isinstance(chain[i + 1][1], nn.BatchNorm2d) or \
                    not isinstance(chain[i + 2][1], nn.ReLU):
                raise UnsupportedModel(f"{qn}: a conv must be followed by BatchNorm2d and ReLU")
            cname = f"c{len(units)}"
            n_, h, w, c = cur.shape
            pp = (h + 2 * p - k) // s + 1
            g.convs[cname] = G.ConvSpec(cname, c, m.out_channels, k, s, p)
            cn = g.add(cname, "conv", (n_, pp, pp, m.out_channels), [cur.id], attrs=dict(conv=cname))
            cn.flops = 2.0 * n_ * pp * pp * m.out_channels * (3 if c == 4 else c) * k * k
            cn.hbm_bytes = cur.nbytes + cn.nbytes
            bname = f"bn{len(units)}"
            g.bns[bname] = m.out_channels
            rn = g.add(bname + "_relu", "bn_relu", cn.shape, [cn.id], attrs=dict(bn=bname))
            rn.hbm_bytes = 2 * cn.nbytes
            names["conv"][cname] = qn
            names["bn"][bname] = chain[i + 1][0]
            units.append((cn, rn, cur))
            cur = rn
            i += 3
        elif isinstance(m, nn.MaxPool2d):
            if (m.kernel_size, m.stride, m.padding) not in ((3, 2, 1),) or cur.op != "bn_relu":
                raise UnsupportedModel(f"{qn}: MaxPool2d(3, 2, 1) after a BN-ReLU only")
            n_, h, w, c = cur.shape
            ph = (h + 2 - 3) // 2 + 1
            pn = g.add(f"maxpool{len(units)}", "maxpool", (n_, ph, ph, c), [cur.id])
            pn.hbm_bytes = cur.nbytes + pn.nbytes
            cur = pn
            i += 1
        elif isinstance(m, nn.AdaptiveAvgPool2d):
            if m.output_size not in (1, (1, 1)) or cur.op != "bn_relu":
                raise UnsupportedModel(f"{qn}: global average pooling after a BN-ReLU only")
            if i + 2 >= len(chain) or not isinstance(chain[i + 1][1], nn.Flatten) or \
                    not isinstance(chain[i + 2][1], nn.Linear) or i + 3 != len(chain):
                raise UnsupportedModel("the head must be AdaptiveAvgPool2d(1), Flatten, Linear")
            lin = chain[i + 2][1]
            if lin.in_features != cur.shape[-1] or lin.bias is None:
                raise UnsupportedModel("Linear: in_features = channels, with bias")
            pooled = g.add("avgpool", "avgpool", (batch, cur.shape[-1]), [cur.id])
            pooled.hbm_bytes = cur.nbytes + pooled.nbytes
            g.fc = (cur.shape[-1], lin.out_features)
            g.fc_pad = (lin.out_features + 63) // 64 * 64
            logits = g.add("fc", "fc", (batch, g.fc_pad), [pooled.id])
            logits.flops = 2.0 * batch * lin.in_features * lin.out_features
            logits.hbm_bytes = pooled.nbytes + logits.nbytes
            names["fc"] = chain[i + 2][0]
            i += 3
        else:
            raise UnsupportedModel(f"{qn}: unsupported module {type(m).__name__}")
    if logits is None or not units:
        raise UnsupportedModel("no conv units or no classifier head")

    # ---- backward ----
    d_pool = g.add("fc.bwd", "fc_bwd", pooled.shape, [logits.id, pooled.id], phase="B")
    d_pool.flops = 2.0 * logits.flops
    cl, rl, _ = units[-1]
    up = g.add(f"{rl.attrs['bn']}.bwd", "bn_add_relu_bwd", cl.shape, [d_pool.id, rl.id, cl.id],
               phase="B", attrs=dict(bn=rl.attrs["bn"], from_pool=True, masked=True,
                                     sums_fused=False))
    up.hbm_bytes = 6 * cl.nbytes
    for u in range(len(units) - 1, 0, -1):
        cn, rn, src = units[u]
        pc, pr, _ = units[u - 1]
        if src is pr:
            # the conv's input is the previous BN-ReLU output: dgrad + BN-ReLU backward
            d = g.add(f"{cn.name}.bwd", "conv_bn_relu_bwd", pc.shape, [up.id, pr.id, pc.id],
                      phase="B", attrs=dict(conv=cn.name, bn=pr.attrs["bn"]))
            d.flops = 2 * cn.flops
            d.hbm_bytes = 2 * up.nbytes + 6 * pc.nbytes
            up = d
        else:  # fed by a maxpool of the previous BN-ReLU output
            d = g.add(f"{cn.name}.bwd", "conv_bwd", src.shape, [up.id, src.id], phase="B",
                      attrs=dict(conv=cn.name))
            d.flops = 2 * cn.flops
            d.hbm_bytes = 2 * up.nbytes + 2 * src.nbytes
            dm = g.add(f"{src.name}.bwd", "maxpool_bwd", pr.shape, [d.id, pr.id], phase="B")
            dm.hbm_bytes = d.nbytes + 2 * pr.nbytes
            db = g.add(f"{pr.attrs['bn']}.bwd", "bn_relu_bwd", pc.shape, [dm.id, pr.id, pc.id],
                       phase="B", attrs=dict(bn=pr.attrs["bn"]))
            db.hbm_bytes = 7 * pc.nbytes
            up = db
    c0, _, _ = units[0]
    cs = g.convs[c0.name]
    wg = g.add(f"{c0.name}.bwd", "conv_wgrad", (cs.cout, cs.k, cs.k, cs.cin), [up.id, x.id],
               phase="B", attrs=dict(conv=c0.name), dtype_bytes=4)
    wg.flops = c0.flops
    wg.hbm_bytes = up.nbytes + x.nbytes
    for cs_ in g.convs.values():
        if cs_.k == 1 and cs_.stride != 1:
            raise UnsupportedModel("1x1 stride-2 convs only inside residual blocks")
    G.estimate_costs(g)
    return g, names


@torch.no_grad()
def load_weights(rt, model: nn.Module, names: dict):
    """Copy the module's conv weights (KCRS -> KRSC, a 3-channel stem padded to
    4), BN affine parameters and running statistics, and the classifier into
    the runtime's fp32 masters, then refresh the bf16 copies."""
    pr = rt.params
    mods = dict(model.named_modules())
    for cname, qn in names["conv"].items():
        w = mods[qn].weight.detach().float().permute(0, 2, 3, 1)
        dst = pr.views["conv:" + cname]
        dst.zero_()
        dst[..., :w.shape[-1]].copy_(w)
    for bname, qn in names["bn"].items():
        bn = mods[qn]
        pr.views["bn_g:" + bname].copy_(bn.weight.detach().float())
        pr.views["bn_b:" + bname].copy_(bn.bias.detach().float())
        pr.bn_rmean[bname].copy_(bn.running_mean.detach().float())
        pr.bn_rvar[bname].copy_(bn.running_var.detach().float())
    lin = mods[names["fc"]]
    pr.views["fc_w"].copy_(lin.weight.detach().float())
    pr.views["fc_b"].copy_(lin.bias.detach().float())
    pr.refresh_bf16()
    torch.cuda.synchronize()

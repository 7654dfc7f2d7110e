"""End-to-end GPU parity of the DELTA runtime, at the test batch (16) AND at
the bench configuration (256, every M a multiple of 128, the 256-wide
BN-backward dgrads, the large-grid one-launch BN backward, the bs256 wgrad
splits) and at a batch with partial tiles (250).

* the step through our kernels matches a plain PyTorch fp32 autograd
  reference of the same ResNet (loss within 2e-2 relative — bf16 activations);
* every forward op and every backward node, re-evaluated in fp32 autograd on
  the runtime's own (bf16) inputs, matches ELEMENTWISE within the kernel tests'
  tolerance (|err| <= 1e-2 |ref| + 2e-2 rms(ref));
* under a 50% activation budget (evictions + recomputes, sometimes
  offload/reload) the loss and every parameter gradient are BIT-IDENTICAL to
  the no-eviction run: recomputed activations equal the retained ones;
* the executed plan's decisions equal the reference oracle's on the same
  trace (bit-exact Filter/Director) when oracle/_ref is present;
* the timeline the GPU executed (device-side action log) passes the
  reference's replay_check, unfiltered, for the 50% plan, other budgets and
  policies, and an offload-heavy plan.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu

from paper_2203_15980_b200 import planner as P  # noqa: E402
from paper_2203_15980_b200.runtime import DeltaRuntime  # noqa: E402

BATCH = 16


def make_batch(seed=0, batch=BATCH):
    g = torch.Generator().manual_seed(seed)
    x = torch.zeros(batch, 224, 224, 4, dtype=torch.bfloat16)
    x[..., :3] = torch.randn(batch, 224, 224, 3, generator=g).to(torch.bfloat16)
    y = torch.randint(0, 1000, (batch,), generator=g)
    return x, y


def torch_reference_loss(rt, x, y):
    """fp32 autograd ResNet with the runtime's master weights."""
    pr = rt.params
    params = {k: v.detach().clone().requires_grad_(True) for k, v in pr.views.items()}
    h = x.float().cuda().permute(0, 3, 1, 2)

    def conv(name, t):
        cs = rt.g.convs[name]
        w = params["conv:" + name].permute(0, 3, 1, 2)
        return F.conv2d(t, w, stride=cs.stride, padding=cs.pad)

    def bn(name, t):
        return F.batch_norm(t, None, None, params["bn_g:" + name], params["bn_b:" + name],
                            training=True, eps=1e-5)

    h = F.relu(bn("bn1", conv("conv1", h)))
    h = F.max_pool2d(h, 3, 2, 1)
    for li, nb in enumerate([3, 4, 6, 3]):
        for b in range(nb):
            pre = f"layer{li + 1}.{b}"
            o = F.relu(bn(pre + ".bn1", conv(pre + ".conv1", h)))
            o = F.relu(bn(pre + ".bn2", conv(pre + ".conv2", o)))
            o = bn(pre + ".bn3", conv(pre + ".conv3", o))
            sc = bn(pre + ".downsample.1", conv(pre + ".downsample.0", h)) if b == 0 else h
            h = F.relu(o + sc)
    h = h.mean((2, 3))
    logits = h @ params["fc_w"].t() + params["fc_b"]
    loss = F.cross_entropy(logits, y.cuda())
    loss.backward()
    return loss.item(), {k: v.grad for k, v in params.items()}


def _pair(batch):
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    base = DeltaRuntime(50, batch, seed=0, lr=0.0)
    base.measure_costs(iters=2)
    base.plan(None)
    delta = DeltaRuntime(50, batch, seed=0, lr=0.0)
    for n, m in zip(delta.nodes, base.nodes):
        n.cost_us = m.cost_us
    delta.link_gbs = base.link_gbs
    delta.plan(0.5)
    return base, delta


@pytest.fixture(scope="module")
def rts():
    base, delta = _pair(BATCH)
    yield base, delta
    del base, delta
    torch.cuda.empty_cache()


@pytest.fixture(scope="module", params=[BATCH, 250, 256], ids=lambda b: f"bs{b}")
def rts_any(request):
    """the test batch, a batch with partial 128-row tiles (250) and the bench
    configuration (256)"""
    base, delta = _pair(request.param)
    yield base, delta
    del base, delta
    torch.cuda.empty_cache()


def _probe_all(rt, x, y):
    probe = {n.id: None for n in rt.nodes}
    rt.x_dev.copy_(x)
    rt.y_dev.copy_(y)
    with torch.cuda.stream(rt.stream):
        rt.run_program(probe=probe)
    torch.cuda.synchronize()
    return probe


def _close(ours, ref, what):
    """elementwise, the kernel tests' tolerance (tests/test_kernels_gpu.py _close)"""
    ours = ours.float().reshape(ref.shape)
    ref = ref.float()
    err = (ours - ref).abs()
    tol = 1e-2 * ref.abs() + 2e-2 * ref.pow(2).mean().sqrt() + 1e-6
    bad = err > tol
    assert not bool(bad.any()), (f"{what}: {int(bad.sum())} of {ref.numel()} elements out of "
                                 f"tolerance, max err {err.max().item():.3g} "
                                 f"(rms ref {ref.pow(2).mean().sqrt().item():.3g})")


def test_loss_matches_torch_fp32(rts_any):
    base, _ = rts_any
    x, y = make_batch(0, base.batch)
    loss = base.step(x, y)
    ref_loss, _ = torch_reference_loss(base, x, y)
    assert abs(loss - ref_loss) <= 2e-2 * abs(ref_loss), (loss, ref_loss)


def test_every_op_matches_fp32_autograd_on_its_inputs(rts_any):
    """Each forward op and each backward node of the step, re-evaluated in
    fp32 autograd from the runtime's own (bf16) inputs, elementwise (bf16
    rounding of the stored result is the only expected difference)."""
    base, _ = rts_any
    x, y = make_batch(3, base.batch)
    checked = _check_every_op(base, x, y)
    assert len(checked) >= 260  # 178 nodes + parameter gradients


def _check_every_op(base, x, y):
    pv = _probe_all(base, x, y)
    g = base.g
    pr = base.params
    Pw = {k: v.detach().float() for k, v in pr.views.items()}
    node = {n.name: n for n in g.nodes}

    def T(nid):  # NHWC bf16 -> NCHW fp32 (4-D) / as is
        t = pv[nid].float()
        return t.permute(0, 3, 1, 2).contiguous() if t.dim() == 4 else t

    def nhwc(t):
        return t.permute(0, 2, 3, 1) if t.dim() == 4 else t

    def W(name):
        return Pw["conv:" + name].permute(0, 3, 1, 2).contiguous().requires_grad_(True)

    def conv(name, xin, w):
        cs = g.convs[name]
        return F.conv2d(xin, w, stride=cs.stride, padding=cs.pad)

    def bn(name, t, gam=None, bet=None):
        gam = Pw["bn_g:" + name] if gam is None else gam
        bet = Pw["bn_b:" + name] if bet is None else bet
        return F.batch_norm(t, None, None, gam, bet, training=True, eps=1e-5)

    checked = []

    def expect(what, ours, ref):
        checked.append(what)
        _close(ours, ref, what)

    for n in g.nodes:
        ins = [T(p) for p in n.parents]
        if n.op == "conv":
            expect(n.name, T(n.id), conv(n.attrs["conv"], ins[0], W(n.attrs["conv"])))
        elif n.op == "bn_relu":
            expect(n.name, T(n.id), F.relu(bn(n.attrs["bn"], ins[0])))
        elif n.op == "bn_add_relu":
            expect(n.name, T(n.id), F.relu(bn(n.attrs["bn"], ins[0]) + ins[1]))
        elif n.op == "bn_bn_add_relu":
            expect(n.name, T(n.id), F.relu(bn(n.attrs["bn"], ins[0]) + bn(n.attrs["bn2"], ins[1])))
        elif n.op == "maxpool":
            expect(n.name, T(n.id), F.max_pool2d(ins[0], 3, 2, 1))
        elif n.op == "avgpool":
            expect(n.name, T(n.id), ins[0].mean((2, 3)))
        elif n.op == "fc":
            ncls = g.fc[1]
            out = T(n.id)
            expect(n.name, out[:, :ncls], ins[0] @ Pw["fc_w"].t())   # bias: in the head kernel
            assert bool((out[:, ncls:] == 0).all())                  # zero-padded classes
        elif n.op == "fc_bwd":
            ncls = g.fc[1]
            L = (ins[0][:, :ncls] + Pw["fc_b"]).requires_grad_(True)
            F.cross_entropy(L, y.cuda()).backward()
            expect(n.name, T(n.id), L.grad @ Pw["fc_w"])
            expect("grad fc_w", pr.gviews["fc_w"], L.grad.t() @ ins[1])
            expect("grad fc_b", pr.gviews["fc_b"], L.grad.sum(0))
            assert bool((pr.gviews["fc_w_full"][ncls:] == 0).all())
        elif n.op in ("bn_add_relu_bwd", "bn_relu_bwd"):
            up, xin = ins[0], ins[-1]
            if n.attrs.get("from_pool"):
                up = up[:, :, None, None].expand_as(xin) / (xin.shape[2] * xin.shape[3])
            masked = n.op == "bn_relu_bwd" or n.attrs.get("masked")
            gq = up * (ins[1] > 0) if masked else up
            xr = xin.clone().requires_grad_(True)
            gam = Pw["bn_g:" + n.attrs["bn"]].clone().requires_grad_(True)
            bet = Pw["bn_b:" + n.attrs["bn"]].clone().requires_grad_(True)
            bn(n.attrs["bn"], xr, gam, bet).backward(gq)
            expect(n.name, T(n.id), xr.grad)
            expect("dgamma " + n.name, pr.gviews["bn_g:" + n.attrs["bn"]], gam.grad)
            expect("dbeta " + n.name, pr.gviews["bn_b:" + n.attrs["bn"]], bet.grad)
        elif n.op == "conv_bn_relu_bwd":
            dC, R, Cp = ins
            Rr = R.clone().requires_grad_(True)
            w = W(n.attrs["conv"])
            conv(n.attrs["conv"], Rr, w).backward(dC)
            expect("grad conv:" + n.attrs["conv"], nhwc(pr.gviews["conv:" + n.attrs["conv"]].permute(0, 3, 1, 2)), nhwc(w.grad))
            xr = Cp.clone().requires_grad_(True)
            bn(n.attrs["bn"], xr).backward(Rr.grad * (R > 0))
            expect(n.name, T(n.id), xr.grad)
        elif n.op == "conv_shortcut_bwd":
            Xr = ins[1].clone().requires_grad_(True)
            w = W(n.attrs["conv"])
            conv(n.attrs["conv"], Xr, w).backward(ins[0])
            if "conv_short" in n.attrs:
                wd = W(n.attrs["conv_short"])
                conv(n.attrs["conv_short"], Xr, wd).backward(ins[2])
                ref = Xr.grad
            elif n.attrs.get("from_pool"):
                up, O = ins[2], ins[3]
                up = up[:, :, None, None].expand_as(O) / (O.shape[2] * O.shape[3])
                ref = Xr.grad + up * (O > 0)
            else:
                ref = Xr.grad + ins[2]
            if n.attrs.get("mask_out"):
                ref = ref * (ins[1] > 0)
            expect(n.name, T(n.id), ref)
            expect("grad conv:" + n.attrs["conv"], pr.gviews["conv:" + n.attrs["conv"]].permute(0, 3, 1, 2), w.grad)
        elif n.op == "maxpool_bwd":
            Rr = ins[1].clone().requires_grad_(True)
            F.max_pool2d(Rr, 3, 2, 1).backward(ins[0])
            expect(n.name, T(n.id), Rr.grad)
        elif n.op == "conv_wgrad":
            w = W(n.attrs["conv"])
            conv(n.attrs["conv"], ins[1], w).backward(ins[0])
            expect(n.name, pv[n.id].float().permute(0, 3, 1, 2), w.grad)
        elif n.op == "conv_bwd":
            Xr = ins[1].clone().requires_grad_(True)
            w = W(n.attrs["conv"])
            conv(n.attrs["conv"], Xr, w).backward(ins[0])
            expect(n.name, T(n.id), Xr.grad)
            expect("grad conv:" + n.attrs["conv"],
                   pr.gviews["conv:" + n.attrs["conv"]].permute(0, 3, 1, 2), w.grad)
    return checked


def test_delta_50pct_bit_identical_to_no_eviction(rts_any):
    base, delta = rts_any
    prog = delta.program
    assert prog.plan_counts["evict"] + prog.plan_counts["offload"] > 0
    assert prog.plan_counts["recompute"] > 0
    assert prog.arena_bytes <= base.program.arena_bytes * 0.5 + 1
    x, y = make_batch(1, base.batch)
    l0 = base.step(x, y)
    g0 = base.params.grad.clone()
    l1 = delta.step(x, y)
    g1 = delta.params.grad.clone()
    assert l0 == l1
    assert torch.equal(g0, g1)


def test_plan_decisions_match_reference_oracle(rts):
    _, delta = rts
    oracle_ref = pytest.importorskip("oracle.ref")
    if not oracle_ref.available():
        pytest.skip("oracle/_ref not built")
    t = delta.trace()
    out = oracle_ref.run(t.to_json(), delta.config)
    assert out["ok"], out
    assert out["decisions"] == [[n, int(a)] for n, a in delta.program.decisions]
    mine = P.run_iteration(t, delta.config)
    assert out["chrome"] == mine.chrome_trace()


def test_graph_capture_replay_equals_eager(rts):
    _, delta = rts
    x, y = make_batch(2)
    l_eager = delta.step(x, y)
    g_eager = delta.params.grad.clone()
    delta.capture()
    l_graph = delta.step(x, y)
    assert l_graph == l_eager
    assert torch.equal(delta.params.grad, g_eager)
    # pipelined train(): alternating staging slots, same results per step
    x2, y2 = make_batch(3)
    xp, yp = x.pin_memory(), y.pin_memory()
    x2p, y2p = x2.pin_memory(), y2.pin_memory()
    losses = delta.train([(xp, yp), (x2p, y2p), (xp, yp)])
    assert losses[0] == l_eager and losses[2] == l_eager
    assert losses[1] == delta.step(x2, y2)
    delta.graph = None
    delta.graphs = None


def test_training_under_delta_fits_a_fixed_batch():
    """End-to-end learning check of the whole DELTA step (forward, recompute,
    every backward kernel, SGD): repeated steps on one batch must drive its
    loss well down, at a 50% budget, through the captured CUDA graph."""
    torch.backends.cudnn.deterministic = True
    rt = DeltaRuntime(50, 16, seed=1, lr=0.01)
    rt.measure_costs(iters=1, link=False)
    prog = rt.plan(0.5)
    assert prog.plan_counts["recompute"] > 0
    rt.capture()
    x, y = make_batch(5, 16)
    xp, yp = x.pin_memory(), y.pin_memory()
    losses = rt.train([(xp, yp)] * 25)
    assert all(l == l for l in losses), losses           # no NaN
    assert max(losses[-5:]) < 0.5 * losses[0], losses


def test_bench_paths_are_exercised_at_bs256(rts_any):
    """The code paths only the bench size takes are really in the bs256 step:
    256-wide BN-backward dgrad tiles, M a multiple of 128 everywhere, and the
    one-launch (cooperative, grid-barrier) BN backward."""
    base, _ = rts_any
    from paper_2203_15980_b200 import kernels as K
    widths = {name: d.tile_n for name, d in base._dconvs.items()}
    Ms = {int(np.prod(n.shape[:-1])) for n in base.nodes
          if len(n.shape) == 4 and n.shape[0] == base.batch}
    if base.batch == 256:
        assert 256 in widths.values(), widths
        assert all(m % 128 == 0 for m in Ms)
        assert K.BN_BWD_ONE_LAUNCH
    elif base.batch == 250:
        assert any(m % 128 for m in Ms)  # partial tiles


def _certify(rt, x, y):
    certify = pytest.importorskip("oracle.certify")
    rt.x_dev.copy_(x)
    rt.y_dev.copy_(y)
    out = certify.certify(rt)
    assert out["findings"] == [], out["findings"][:5]
    if out["violations"] is None:
        pytest.skip("oracle/_ref not built")
    assert out["violations"] == [], out["violations"][:5]
    return out


def test_executed_gpu_timeline_passes_reference_replay_check(rts):
    """The timeline the GPU actually executed — the executor's device-side
    action log (kind, node, %globaltimer head/tail per action) — matches the
    lowered program action for action and in per-stream order, and the
    reference's own independent verifier (ref src/oracle.cpp replay_check)
    finds nothing: budget never exceeded, no read of an absent tensor, no
    backward release, monotone non-overlapping streams."""
    _, delta = rts
    x, y = make_batch(4)
    out = _certify(delta, x, y)
    ev = out["events"]
    measured = ev[np.isin(ev["kind"], [P.EventKind.Compute, P.EventKind.Recompute])]
    assert (measured["duration"] > 0).any()


@pytest.mark.parametrize("frac,policy", [(0.55, P.PolicyMode.Delta), (0.7, P.PolicyMode.Delta),
                                         (0.5, P.PolicyMode.OffloadOnly),
                                         (0.5, P.PolicyMode.RecomputeOnly)])
def test_budgets_and_policies_bit_identical_and_certified(rts, frac, policy):
    """Other budgets and the single-mechanism policies (many offloads through
    the swap engine, or recompute only): the step stays bit-identical to the
    no-eviction one and the executed timeline passes the reference verifier
    with no exemption."""
    base, _ = rts
    rt = DeltaRuntime(50, BATCH, seed=0, lr=0.0)
    for n, m in zip(rt.nodes, base.nodes):
        n.cost_us = m.cost_us
    rt.link_gbs = base.link_gbs
    try:
        prog = rt.plan(frac, policy=policy)
    except RuntimeError as e:  # a policy may be infeasible at this budget
        pytest.skip(str(e))
    if policy == P.PolicyMode.OffloadOnly:
        assert prog.plan_counts["offload"] > 1
    x, y = make_batch(6)
    l0 = base.step(x, y)
    g0 = base.params.grad.clone()
    l1 = rt.step(x, y)
    assert l0 == l1
    assert torch.equal(g0, rt.params.grad)
    _certify(rt, x, y)


def test_offload_heavy_plan_certified(rts):
    """A cost table where recomputing is expensive (every cost x50, as a
    profiler-serialised measurement can produce): the Director offloads many
    tensors, prefetches and demand reloads flow through the copy engine, and
    the executed timeline still certifies and the step stays bit-identical."""
    base, _ = rts
    rt = DeltaRuntime(50, BATCH, seed=0, lr=0.0)
    for n, m in zip(rt.nodes, base.nodes):
        n.cost_us = m.cost_us * 50
    rt.link_gbs = base.link_gbs
    prog = rt.plan(0.5)
    assert prog.plan_counts["offload"] > 3 and prog.plan_counts["reload"] > 3, prog.plan_counts
    x, y = make_batch(8)
    l0 = base.step(x, y)
    g0 = base.params.grad.clone()
    assert rt.step(x, y) == l0
    assert torch.equal(g0, rt.params.grad)
    _certify(rt, x, y)


def test_resnet101_step_matches_no_eviction():
    """ResNet-101 (config 3's model) executes under DELTA bit-identically."""
    torch.backends.cudnn.deterministic = True
    base = DeltaRuntime(101, 4, seed=0, lr=0.0)
    base.measure_costs(iters=1, link=False)
    base.plan(None)
    rt = DeltaRuntime(101, 4, seed=0, lr=0.0)
    for n, m in zip(rt.nodes, base.nodes):
        n.cost_us = m.cost_us
    prog = rt.plan(0.5)
    assert prog.plan_counts["recompute"] > 0
    x, y = make_batch(7, 4)
    assert base.step(x, y) == rt.step(x, y)
    assert torch.equal(base.params.grad, rt.params.grad)


def test_executed_comparison_grid(rts):
    """f3: a small budget x policy grid executed on the GPU — the reference's
    comparison CSV header, one row per cell, every feasible cell bit-identical
    to the no-eviction step, the arena within the budget."""
    from paper_2203_15980_b200 import grid as GR
    base, _ = rts
    rt = DeltaRuntime(50, BATCH, seed=0, lr=0.0)
    for n, m in zip(rt.nodes, base.nodes):
        n.cost_us = m.cost_us
    rt.link_gbs = base.link_gbs
    x, y = make_batch(9)
    for s in range(2):
        rt.x_slots[s].copy_(x)
        rt.y_slots[s].copy_(y)
    text, detail = GR.executed_comparison(rt, [0.5, 0.7],
                                          [P.PolicyMode.Delta, P.PolicyMode.OffloadOnly],
                                          [P.Heuristic.Base, P.Heuristic.Greedy], steps=2, warmup=1)
    lines = text.strip().splitlines()
    assert lines[0] == GR.CSV_HEADER
    assert len(lines) == 1 + 2 * 2 * 2
    feasible = [c for c in detail if not c["infeasible"]]
    assert feasible and all(c["bit_identical"] for c in feasible)
    assert all(c["arena_bytes"] <= c["budget"] for c in feasible)


def test_imported_pytorch_cnn_runs_under_delta():
    """f1: a PyTorch nn.Sequential CNN captured by importer.py (torch.fx) runs
    on this library's kernels under a 70% DELTA budget: bit-identical to its
    no-eviction step, and its loss matches the module's own fp32 training
    step with the same weights."""
    import torch.nn as nn
    from paper_2203_15980_b200 import importer as IM
    from test_importer_cpu import small_cnn
    torch.manual_seed(3)
    model = small_cnn().cuda()
    B, H = 32, 224
    runs = []
    for frac in (None, 0.7):
        g, names = IM.graph_from_module(model, batch=B, image=H, name="cnn")
        rt = DeltaRuntime(g, lr=0.0, anchors="none")
        IM.load_weights(rt, model, names)
        rt.measure_costs(iters=1, link=False)
        prog = rt.plan(frac)
        runs.append((rt, prog))
    (base, _), (rt, prog) = runs
    assert prog.plan_counts["recompute"] + prog.plan_counts["offload"] > 0, prog.plan_counts
    gen = torch.Generator().manual_seed(0)
    x = torch.zeros(B, H, H, 4, dtype=torch.bfloat16)
    x[..., :3] = torch.randn(B, H, H, 3, generator=gen).to(torch.bfloat16)
    y = torch.randint(0, 10, (B,), generator=gen)
    l0 = base.step(x, y)
    l1 = rt.step(x, y)
    assert l0 == l1
    assert torch.equal(base.params.grad, rt.params.grad)
    # the module's own training step in fp32 on the same (bf16-rounded) batch
    model.train()
    ref = F.cross_entropy(model(x[..., :3].float().cuda().permute(0, 3, 1, 2)), y.cuda())
    assert abs(l0 - ref.item()) <= 2e-2 * abs(ref.item()), (l0, ref.item())
    ref.backward()
    # every op of the imported graph against fp32 autograd on its own inputs
    # (end-to-end, bf16 activations through ten BN layers drift from the fp32
    # module's gradients; the local checks pin each kernel mapping)
    checked = _check_every_op(base, x, y)
    assert len(checked) >= len(base.nodes) - 2
    cos = F.cosine_similarity(base.params.gviews["fc_w"].flatten(),
                              model[-1].weight.grad.flatten(), dim=0).item()
    assert cos > 0.999, cos

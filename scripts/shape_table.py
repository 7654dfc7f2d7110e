"""Per-shape table of every ResNet-50 convolution the step runs — forward,
input gradient (dgrad) and weight gradient (wgrad) — on OUR sm_100a kernels
(the exact handles/tilings the runtime binds) beside cuDNN on the same shape:
time, TFLOP/s, algorithmic GB/s and the fraction of max(FLOPs / TC peak,
bytes / HBM peak) (MEASURED_PEAKS.json, burst).  CUDA events on the launching
stream, 3 warm-ups, inputs > L2.
    python scripts/shape_table.py [batch] [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2203_15980_b200.runtime import DeltaRuntime, dgrad_s2  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
OUT = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/shape_table.json"
try:
    pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "MEASURED_PEAKS.json")))
    HBM, TC = pk["hbm_gbs"], pk["bf16_tflops"]
except Exception:  # noqa: BLE001
    HBM, TC = 6650.0, 1590.0
st = torch.cuda.current_stream().cuda_stream


def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


rt = DeltaRuntime(50, B, seed=0)
rows = []
seen = set()


def row(kind, name, shape, flops, nbytes, ms, ms_cudnn):
    roof = max(flops / (TC * 1e9), nbytes / (HBM * 1e6))
    r = dict(kind=kind, conv=name, shape=shape, us=round(ms * 1e3, 1),
             tflops=round(flops / ms / 1e9, 1), gbs=round(nbytes / ms / 1e6, 1),
             frac=round(roof / ms, 3), bound="tensor" if flops / (TC * 1e9) >= nbytes / (HBM * 1e6) else "hbm",
             cudnn_us=round(ms_cudnn * 1e3, 1) if ms_cudnn else None,
             cudnn_frac=round(roof / ms_cudnn, 3) if ms_cudnn else None)
    rows.append(r)
    print(json.dumps(r), flush=True)


for n in rt.nodes:
    if n.op != "conv":
        continue
    cs = rt.g.convs[n.attrs["conv"]]
    if cs.name in seen:
        continue
    seen.add(cs.name)
    src = rt.nodes[n.parents[0]]
    Nb, H, W, C = src.shape
    _, P_, Q_, Ko = n.shape
    Creal = 3 if C == 4 else C
    flops = 2.0 * Nb * P_ * Q_ * Ko * Creal * cs.k * cs.k
    shape = f"{H}x{W}x{C}->{P_}x{Q_}x{Ko} k{cs.k}s{cs.stride}"
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(Nb, H, W, C, device="cuda", generator=g).to(torch.bfloat16)
    y = torch.empty(Nb, P_, Q_, Ko, device="cuda", dtype=torch.bfloat16)
    w = rt.params.wbf[cs.name]
    xc, wc = x.permute(0, 3, 1, 2), w.permute(0, 3, 1, 2)
    dy = torch.randn(Nb, P_, Q_, Ko, device="cuda", generator=g).to(torch.bfloat16)
    # forward
    conv = rt._convs[n.name]
    ms = timeit(lambda: conv(x.data_ptr(), y.data_ptr(), st))
    mc = timeit(lambda: F.conv2d(xc, wc, stride=cs.stride, padding=cs.pad))
    row("fwd", cs.name, shape, flops, (x.numel() + y.numel() + w.numel()) * 2, ms, mc)
    # input gradient (the stem has none)
    dyc = dy.permute(0, 3, 1, 2)
    cud = lambda: torch.ops.aten.convolution_backward(dyc, xc, wc, None, [cs.stride] * 2, [cs.pad] * 2,
                                                      [1, 1], False, [0, 0], 1, [True, False, False])
    if cs.name in rt._dconvs:
        dc = rt._dconvs[cs.name]
        dx = torch.empty(Nb, dc.P, dc.Q, C, device="cuda", dtype=torch.bfloat16)
        ms = timeit(lambda: dc(dy.data_ptr(), dx.data_ptr(), st))
        nb = (dy.numel() + dx.numel() + w.numel()) * 2
        # a stride-2 1x1's gradient is computed on its sampling grid (its FLOPs)
        row("dgrad", cs.name, shape, flops, nb, ms, timeit(cud))
    elif dgrad_s2(cs):
        dx = torch.empty(Nb, H, W, C, device="cuda", dtype=torch.bfloat16)
        dcs = rt._dconvs_s2[cs.name]

        def s2():
            for c, d in enumerate(dcs):
                d.scatter2(dy.data_ptr(), dx.data_ptr(), c, st)
        ms = timeit(s2)
        row("dgrad_s2(4 sub-pixel)", cs.name, shape, flops, (dy.numel() + dx.numel() + w.numel()) * 2,
            ms, timeit(cud))
    # weight gradient (fp32 KRSC out)
    wg = rt._wgrads[cs.name]
    dw = torch.empty(Ko, cs.k, cs.k, C, device="cuda")
    ws = torch.empty(max(wg.workspace_bytes, 256), dtype=torch.uint8, device="cuda")
    ms = timeit(lambda: wg(dy.data_ptr(), x.data_ptr(), dw.data_ptr(), ws.data_ptr(), st))
    cuw = lambda: torch.ops.aten.convolution_backward(dyc, xc, wc, None, [cs.stride] * 2, [cs.pad] * 2,
                                                      [1, 1], False, [0, 0], 1, [False, True, False])
    row("wgrad", cs.name, shape, flops, (dy.numel() + x.numel()) * 2 + dw.numel() * 4, ms,
        timeit(cuw))
    del x, y, dy

tot = {}
for r in rows:
    t = tot.setdefault(r["kind"], [0.0, 0.0, 0.0])
    t[0] += r["us"]
    t[1] += r["cudnn_us"] or 0.0
    t[2] += r["us"] * r["frac"]
summary = {k: dict(ours_us=round(v[0], 1), cudnn_us=round(v[1], 1), roofline_us=round(v[2], 1),
                   frac=round(v[2] / v[0], 3)) for k, v in tot.items()}
print(json.dumps({"summary": summary}))
json.dump({"batch": B, "peaks": {"hbm_gbs": HBM, "bf16_tflops": TC}, "rows": rows,
           "summary": summary}, open(OUT, "w"), indent=1)

"""Micro-benchmark of the sm_100a conv kernel on the ResNet-50 bs256 shapes
(CUDA events on the launching stream, inputs > L2), beside cuDNN."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F
from paper_2203_15980_b200 import kernels as K

def timeit(fn, iters=20):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
shapes = [  # H, C, K, R, stride, pad
    (56, 64, 64, 1, 1, 0), (56, 64, 64, 3, 1, 1), (56, 64, 256, 1, 1, 0), (56, 256, 64, 1, 1, 0),
    (56, 256, 128, 1, 1, 0), (56, 128, 128, 3, 2, 1), (28, 128, 512, 1, 1, 0), (56, 256, 512, 1, 2, 0),
    (28, 512, 128, 1, 1, 0), (28, 128, 128, 3, 1, 1), (14, 256, 256, 3, 1, 1), (14, 256, 1024, 1, 1, 0),
    (14, 1024, 256, 1, 1, 0), (7, 512, 512, 3, 1, 1), (7, 512, 2048, 1, 1, 0), (7, 2048, 512, 1, 1, 0),
]
st = torch.cuda.current_stream().cuda_stream
out = []
# stem 7x7/2 over C=4 (pixel-pair TMA im2col path)
x = torch.randn(N, 224, 224, 4, device="cuda").to(torch.bfloat16)
w4 = (torch.randn(64, 7, 7, 4, device="cuda") * 0.05).to(torch.bfloat16)
wp = K.pack_stem_weights(w4)
conv = K.Conv(N, 224, 224, 4, 64, 7, 7, 2, 3, wp.data_ptr())
y = torch.empty(N, 112, 112, 64, device="cuda", dtype=torch.bfloat16)
ms = timeit(lambda: conv(x.data_ptr(), y.data_ptr(), st))
ms_cudnn = timeit(lambda: F.conv2d(x.permute(0, 3, 1, 2), w4.permute(0, 3, 1, 2), stride=2, padding=3))
flops = 2.0 * N * 112 * 112 * 64 * 7 * 7 * 3
print(json.dumps(dict(shape="stem7x7s2", ms=round(ms, 4), tflops_rgb=round(flops / ms / 1e9, 1),
                      gbs=round((x.numel() + y.numel()) * 2 / ms / 1e6, 1), cudnn_ms=round(ms_cudnn, 4))), flush=True)
# BN statistics from the epilogue partials of a 56x56x64 conv (6272 partials)
M = N * 56 * 56
parts = torch.rand(K.stats_partials_floats(64), device="cuda") + 1.0
mean = torch.empty(64, device="cuda"); inv = torch.empty(64, device="cuda")
ms = timeit(lambda: K.bn_stats_from_partials(parts.data_ptr(), 64, mean.data_ptr(), inv.data_ptr(), 1e-5, None, None, 0.1, st))
print(json.dumps(dict(kernel="bn_stats_from_partials_56x56x64", us=round(ms * 1e3, 2))), flush=True)
for (H, C, Ko, R, s, p) in shapes:
    x = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
    w = (torch.randn(Ko, R, R, C, device="cuda") * 0.05).to(torch.bfloat16)
    conv = K.Conv(N, H, H, C, Ko, R, R, s, p, w.data_ptr())
    y = torch.empty(N, conv.P, conv.Q, Ko, device="cuda", dtype=torch.bfloat16)
    ms = timeit(lambda: conv(x.data_ptr(), y.data_ptr(), st))
    xc = x.permute(0, 3, 1, 2)  # channels_last view
    wc = w.permute(0, 3, 1, 2)
    ms_cudnn = timeit(lambda: F.conv2d(xc, wc, stride=s, padding=p))
    flops = 2.0 * N * conv.P * conv.Q * Ko * C * R * R
    byts = x.numel() * 2 + y.numel() * 2
    out.append(dict(shape=[H, C, Ko, R, s], ms=round(ms, 4), tflops=round(flops / ms / 1e9, 1),
                    gbs=round(byts / ms / 1e6, 1), cudnn_ms=round(ms_cudnn, 4),
                    cudnn_tflops=round(flops / ms_cudnn / 1e9, 1)))
    print(json.dumps(out[-1]), flush=True)
h2d, d2h, dup = K.probe_link()
print(json.dumps(dict(link_h2d_gbs=h2d, link_d2h_gbs=d2h, link_duplex_gbs=dup)))

# ---- HBM-bound kernels at layer-1 sizes (bs 256, 56x56) ----
M, C = N * 56 * 56, 256
x = torch.randn(M, C, device="cuda").to(torch.bfloat16)
r = torch.randn(M, C, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
mean = torch.zeros(C, device="cuda"); inv = torch.ones(C, device="cuda")
gam = torch.ones(C, device="cuda"); bet = torch.zeros(C, device="cuda")
ws = torch.zeros(K.bn_workspace_floats(M, C), device="cuda")
dg = torch.empty(C, device="cuda"); db = torch.empty(C, device="cuda")
nb = M * C * 2
res = {}
res["bn_stats"] = (timeit(lambda: K.bn_stats(x.data_ptr(), M, C, ws.data_ptr(), mean.data_ptr(), inv.data_ptr(), 1e-5, 0, 0, 0.1, st)), 1 * nb)
res["bn_apply_relu"] = (timeit(lambda: K.bn_apply(0, x.data_ptr(), None, y.data_ptr(), M, C, mean.data_ptr(), inv.data_ptr(), gam.data_ptr(), bet.data_ptr(), stream=st)), 2 * nb)
res["bn_add_relu"] = (timeit(lambda: K.bn_apply(1, x.data_ptr(), r.data_ptr(), y.data_ptr(), M, C, mean.data_ptr(), inv.data_ptr(), gam.data_ptr(), bet.data_ptr(), stream=st)), 3 * nb)
res["bn_backward"] = (timeit(lambda: K.bn_backward(r.data_ptr(), 0, x.data_ptr(), x.data_ptr(), y.data_ptr(), M, C, mean.data_ptr(), inv.data_ptr(), gam.data_ptr(), dg.data_ptr(), db.data_ptr(), ws.data_ptr(), st)), 7 * nb)
res["bn_backward_nomask"] = (timeit(lambda: K.bn_backward(r.data_ptr(), 0, None, x.data_ptr(), y.data_ptr(), M, C, mean.data_ptr(), inv.data_ptr(), gam.data_ptr(), dg.data_ptr(), db.data_ptr(), ws.data_ptr(), st)), 5 * nb)
res["add_grad_mask"] = (timeit(lambda: K.add_grad(x.data_ptr(), r.data_ptr(), 0, x.data_ptr(), None, y.data_ptr(), M, C, st)), 4 * nb)
for (MM, CC) in [(N * 14 * 14, 1024), (N * 7 * 7, 2048), (N * 56 * 56, 64)]:
    xx = torch.randn(MM, CC, device="cuda").to(torch.bfloat16); rr = torch.randn(MM, CC, device="cuda").to(torch.bfloat16)
    yy = torch.empty_like(xx); m2 = torch.zeros(CC, device="cuda"); i2 = torch.ones(CC, device="cuda"); g2 = torch.ones(CC, device="cuda")
    d1 = torch.empty(CC, device="cuda"); d2 = torch.empty(CC, device="cuda"); w2 = torch.zeros(K.bn_workspace_floats(MM, CC), device="cuda")
    res[f"bn_backward_{MM}x{CC}"] = (timeit(lambda: K.bn_backward(rr.data_ptr(), 0, xx.data_ptr(), xx.data_ptr(), yy.data_ptr(), MM, CC, m2.data_ptr(), i2.data_ptr(), g2.data_ptr(), d1.data_ptr(), d2.data_ptr(), w2.data_ptr(), st)), 7 * MM * CC * 2)
res["torch_copy"] = (timeit(lambda: y.copy_(x)), 2 * nb)
for k, (ms, b) in res.items():
    print(json.dumps(dict(kernel=k, ms=round(ms, 4), gbs=round(b / ms / 1e6, 1))))

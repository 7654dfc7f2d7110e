"""CTA-pair (cta_group::2) 1x1 GEMM tiles vs the 1-CTA kernel: outputs (must be
bit-identical: same K order per output element) and device times.
    DELTA_PAIR=1 python scripts/pair_check.py out.pt   (pair on)
    python scripts/pair_check.py out.pt                (pair off)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_15980_b200 import kernels as K  # noqa: E402

SHAPES = [  # (M, Cin, Cout, mode, stats)
    (16384, 1024, 3072, "bias", False),   # BERT QKV
    (16384, 1024, 4096, "bias", False),   # BERT MlpUp
    (16384, 4096, 1024, "bias", False),   # BERT MlpDown
    (16384, 3072, 1024, "store", False),  # BERT QKV input gradient
    (16384, 1024, 4096, "gelu_bwd", False),  # BERT MlpDown input gradient through gelu'
    (802816, 64, 256, "store", True),     # ResNet layer1 conv3 (BN stats)
    (50176, 1024, 256, "store", True),    # ResNet layer3 conv1
    (12544, 512, 2048, "store", True),    # ResNet layer4 conv3
    (1000, 256, 512, "store", False),     # ragged M
]
CONVS = [  # (N, H, W, C, K, R, stride, pad): the im2col pair path (3x3, strided 1x1)
    (256, 28, 28, 128, 128, 3, 1, 1),
    (256, 14, 14, 256, 256, 3, 1, 1),
    (256, 7, 7, 512, 512, 3, 1, 1),
    (256, 56, 56, 512, 1024, 1, 2, 0),
    (250, 28, 28, 128, 128, 3, 1, 1),
]
dev = "cuda"
out = {}
times = {}
st = torch.cuda.current_stream().cuda_stream
for (M, C, Ko, mode, stats) in SHAPES:
    g = torch.Generator(device=dev).manual_seed(M + C + Ko)
    x = torch.randn(M, C, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(Ko, C, device=dev, generator=g) / C ** 0.5).to(torch.bfloat16)
    b = torch.randn(Ko, device=dev, generator=g)
    y = torch.empty(M, Ko, device=dev, dtype=torch.bfloat16)
    conv = K.Conv(M, 1, 1, C, Ko, 1, 1, 1, 0, w.data_ptr())
    sp = torch.zeros(K.stats_partials_floats(Ko), device=dev) if stats else None

    if mode == "gelu_bwd":
        conv.set_tile_n(128)
        pre = torch.randn(M, Ko, device=dev, generator=g).to(torch.bfloat16)

    def run():
        if mode == "bias":
            conv.bias(x.data_ptr(), y.data_ptr(), b.data_ptr(), st)
        elif mode == "gelu_bwd":
            conv.gelu_bwd(x.data_ptr(), y.data_ptr(), pre.data_ptr(), st)
        else:
            conv(x.data_ptr(), y.data_ptr(), st, sp.data_ptr() if sp is not None else None)
    run()
    torch.cuda.synchronize()
    key = f"{M}x{C}x{Ko}_{mode}"
    out[key] = y.clone().cpu()
    if sp is not None:
        out[key + "_stats"] = sp.clone().cpu()
    ref = x.float() @ w.float().t() + (b if mode == "bias" else 0)
    if mode == "gelu_bwd":
        pr = pre.float().requires_grad_(True)
        torch.nn.functional.gelu(pr).backward(ref)
        ref = pr.grad
    err = ((y.float() - ref).abs() / (ref.abs() + 1e-2 * ref.abs().mean())).max().item()
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    times[key] = {"us": round(ms * 1e3, 1), "tflops": round(2 * M * C * Ko / (ms * 1e-3) / 1e12, 1),
                  "max_rel_err": round(err, 5)}
for (N, H, W, C, Ko, R, st_, pad) in CONVS:
    g = torch.Generator(device=dev).manual_seed(N + H + C)
    x = torch.randn(N, H, W, C, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(Ko, R, R, C, device=dev, generator=g) / (R * R * C) ** 0.5).to(torch.bfloat16)
    conv = K.Conv(N, H, W, C, Ko, R, R, st_, pad, w.data_ptr())
    y = torch.empty(N, conv.P, conv.Q, Ko, device=dev, dtype=torch.bfloat16)
    sp = torch.zeros(K.stats_partials_floats(Ko), device=dev)
    mean, invstd = torch.empty(Ko, device=dev), torch.empty(Ko, device=dev)
    conv(x.data_ptr(), y.data_ptr(), st, sp.data_ptr())
    K.bn_stats_from_partials(sp.data_ptr(), Ko, mean.data_ptr(), invstd.data_ptr(), 1e-5, None, None,
                             0.1, st)
    torch.cuda.synchronize()
    key = f"conv{N}x{H}x{W}x{C}->{Ko}k{R}s{st_}"
    out[key] = y.clone().cpu()
    yf = y.float().reshape(-1, Ko)
    times[key + "_stats_err"] = {"mean": (mean - yf.mean(0)).abs().max().item(),
                                 "invstd_rel": ((invstd - (yf.var(0, unbiased=False) + 1e-5).rsqrt()).abs()
                                                / invstd).max().item()}
    for _ in range(3):
        conv(x.data_ptr(), y.data_ptr(), st, sp.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        conv(x.data_ptr(), y.data_ptr(), st, sp.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    times[key] = {"us": round(ms * 1e3, 1),
                  "tflops": round(2 * N * conv.P * conv.Q * Ko * C * R * R / (ms * 1e-3) / 1e12, 1)}
torch.save(out, sys.argv[1])
print(json.dumps({"pair": os.environ.get("DELTA_PAIR", "1"), "times": times}))

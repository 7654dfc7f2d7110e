"""Forward conv with and without the fused BN-statistics epilogue, ResNet-50
bs256 shapes, 10 launches in a CUDA graph per measurement."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_15980_b200 import kernels as K  # noqa: E402

N = 256
shapes = [  # (H, Cin, K, R, stride)
    (56, 64, 64, 1, 1), (56, 64, 64, 3, 1), (56, 64, 256, 1, 1), (56, 256, 64, 1, 1),
    (28, 128, 128, 3, 1), (28, 128, 512, 1, 1), (28, 512, 128, 1, 1),
    (14, 256, 256, 3, 1), (14, 256, 1024, 1, 1), (14, 1024, 256, 1, 1),
    (7, 512, 512, 3, 1), (7, 512, 2048, 1, 1), (7, 2048, 512, 1, 1)]


def timed(fn, n=10):
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        for _ in range(2):
            fn(cs.cuda_stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            for _ in range(n):
                fn(cs.cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        g.replay()
        e1.record(cs)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for (H, C, Ko, R, st) in shapes:
    P = (H + 2 * (R // 2) - R) // st + 1
    x = torch.randn(N * H * H, C, device="cuda").to(torch.bfloat16)
    w = (torch.randn(Ko, R, R, C, device="cuda") * 0.05).to(torch.bfloat16)
    y = torch.empty(N * P * P, Ko, device="cuda", dtype=torch.bfloat16)
    stats = torch.zeros(K.stats_partials_floats(Ko), device="cuda")
    conv = K.Conv(N, H, H, C, Ko, R, R, st, R // 2, w.data_ptr())
    t0 = timed(lambda s: conv(x.data_ptr(), y.data_ptr(), s))
    t1 = timed(lambda s: conv(x.data_ptr(), y.data_ptr(), s, stats_ptr=stats.data_ptr()))
    print(f"{H}x{H}x{C}->{Ko} k{R}: plain {t0:6.1f} us  +stats {t1:6.1f} us  ({t1 - t0:+.1f})")

"""Maxpool 3x3/2 forward and backward at the ResNet-50 bs256 stem shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_15980_b200 import kernels as K

N, H, W, C = 256, 112, 112, 64
x = torch.randn(N, H, W, C, device="cuda").relu().to(torch.bfloat16)
y = torch.empty(N, 56, 56, C, device="cuda", dtype=torch.bfloat16)
dy = torch.randn(N, 56, 56, C, device="cuda").to(torch.bfloat16)
dx = torch.empty_like(x)
ws = torch.empty(K.maxpool_workspace_bytes(N, H, W, C), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


tf = timeit(lambda: K.maxpool_fwd(x.data_ptr(), y.data_ptr(), N, H, W, C, st))
tb = timeit(lambda: K.maxpool_bwd(dy.data_ptr(), x.data_ptr(), dx.data_ptr(), N, H, W, C,
                                  ws.data_ptr(), st))
fb = (x.numel() + y.numel()) * 2
print(f"maxpool fwd {tf:.1f} us ({fb / tf / 1e3:.0f} GB/s), bwd {tb:.1f} us")

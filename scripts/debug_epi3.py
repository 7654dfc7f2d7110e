import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_15980_b200 import kernels as K
def timeit(fn, iters=20):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3
N, H, C, Ko = 256, 28, 512, 128
w = (torch.randn(Ko, 1, 1, C, device="cuda") * 0.05).to(torch.bfloat16)
wd = w.permute(3, 1, 2, 0).contiguous()
dy = torch.randn(N, H, H, Ko, device="cuda").to(torch.bfloat16)
conv = K.Conv(N, H, H, Ko, C, 1, 1, 1, 0, wd.data_ptr())
conv.set_tile_n(128)
st = torch.cuda.current_stream().cuda_stream
y = torch.empty(N, H, H, C, device="cuda", dtype=torch.bfloat16)
a = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
m = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
print("plain", timeit(lambda: conv(dy.data_ptr(), y.data_ptr(), st)))

print("fused add", timeit(lambda: conv.add_mask(dy.data_ptr(), y.data_ptr(), st, add=a.data_ptr())))
print("fused om", timeit(lambda: conv.add_mask(dy.data_ptr(), y.data_ptr(), st, out_mask=m.data_ptr())))
print("fused add+om", timeit(lambda: conv.add_mask(dy.data_ptr(), y.data_ptr(), st, add=a.data_ptr(), out_mask=m.data_ptr())))

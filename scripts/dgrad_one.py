"""One fused dgrad (add + out-mask epilogue) launch at a ResNet-50 bs256 shape,
for ncu: python scripts/dgrad_one.py H C Ko"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_15980_b200 import kernels as K
H, C, Ko = [int(v) for v in sys.argv[1:4]]
N = 256
w = (torch.randn(Ko, 1, 1, C, device="cuda") * 0.05).to(torch.bfloat16)
wd = w.permute(3, 1, 2, 0).contiguous()
dy = torch.randn(N, H, H, Ko, device="cuda").to(torch.bfloat16)
conv = K.Conv(N, H, H, Ko, C, 1, 1, 1, 0, wd.data_ptr())
if conv.tile_n > 128:
    conv.set_tile_n(128)
y = torch.empty(N, H, H, C, device="cuda", dtype=torch.bfloat16)
a = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
m = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
for _ in range(4):
    conv.add_mask(dy.data_ptr(), y.data_ptr(), st, add=a.data_ptr(), out_mask=m.data_ptr())
torch.cuda.synchronize()

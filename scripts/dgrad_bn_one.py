"""One fused dgrad + BN-backward-epilogue launch at a ResNet-50 bs256 shape,
for ncu: python scripts/dgrad_bn_one.py H C Ko R"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_15980_b200 import kernels as K
H, C, Ko, R = [int(v) for v in sys.argv[1:5]]
N = 256
M = N * H * H
w = (torch.randn(Ko, R, R, C, device="cuda") * 0.05).to(torch.bfloat16)
wd = w.flip(1, 2).permute(3, 1, 2, 0).contiguous()
dy = torch.randn(N, H, H, Ko, device="cuda").to(torch.bfloat16)
conv = K.Conv(N, H, H, Ko, C, R, R, 1, R // 2, wd.data_ptr())
if conv.tile_n > 128:
    conv.set_tile_n(128)
y = torch.empty(N, H, H, C, device="cuda", dtype=torch.bfloat16)
a = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
mean = torch.zeros(C, device="cuda"); inv = torch.ones(C, device="cuda")
gam = torch.ones(C, device="cuda"); bet = torch.zeros(C, device="cuda")
parts = torch.empty(K.stats_partials_floats(C), device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(4):
    conv.bn_bwd(dy.data_ptr(), y.data_ptr(), parts.data_ptr(), a.data_ptr(), mean.data_ptr(),
                inv.data_ptr(), gam.data_ptr(), bet.data_ptr(), st)
torch.cuda.synchronize()

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
conv.set_tile_n(int(os.environ.get("TN", "128")) if conv.tile_n > 128 else conv.tile_n)
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
if os.environ.get("TIME"):
    plain = os.environ.get("PLAIN")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        if plain:
            conv(dy.data_ptr(), y.data_ptr(), st)
        else:
            conv.bn_bwd(dy.data_ptr(), y.data_ptr(), parts.data_ptr(), a.data_ptr(), mean.data_ptr(),
                        inv.data_ptr(), gam.data_ptr(), bet.data_ptr(), st)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    fl = 2 * M * Ko * C * R * R
    print(f"H{H} C{C} K{Ko} R{R} tile_n {conv.tile_n} {'plain' if plain else 'bn_bwd'}: {us:.1f} us  {fl / us / 1e6:.0f} TF/s")
if os.environ.get("CHECK"):
    # same launch at tile_n 128 as reference: g bit-exact, partial sums close
    torch.manual_seed(1)
    mean.normal_(0, 0.1); gam.uniform_(0.5, 1.5); bet.normal_(0, 0.2)
    def run(tn):
        c = K.Conv(N, H, H, Ko, C, R, R, 1, R // 2, wd.data_ptr())
        c.set_tile_n(tn)
        out = torch.zeros_like(y); pp = torch.full_like(parts, float("nan"))
        c.bn_bwd(dy.data_ptr(), out.data_ptr(), pp.data_ptr(), a.data_ptr(), mean.data_ptr(),
                 inv.data_ptr(), gam.data_ptr(), bet.data_ptr(), st)
        torch.cuda.synchronize()
        return out, pp
    o1, p1 = run(128); o2, p2 = run(int(os.environ.get("TN", "256")))
    ns = K.stats_parts()
    s1 = p1[: ns * C * 4].view(ns, C, 4).nansum(0); s2 = p2[: ns * C * 4].view(ns, C, 4).nansum(0)
    print("g bit-exact:", torch.equal(o1, o2), "partials max rel diff:",
          ((s1 - s2).abs() / (s1.abs() + 1)).max().item())

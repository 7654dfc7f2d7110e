import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import test_kernels_gpu as T
from paper_2203_15980_b200 import kernels as K
case = T.DGRAD_CASES[0]
g, w, dy, conv, ref = T._dgrad_setup(case, 7)
N, H, W, Cin = ref.shape
y = torch.empty(N, H, W, Cin, device="cuda", dtype=torch.bfloat16)
conv(dy.data_ptr(), y.data_ptr(), T._stream())
torch.cuda.synchronize()
print("plain err", (y.float() - ref).abs().max().item())
add = torch.randn(N, H, W, Cin, device="cuda", generator=g).to(torch.bfloat16)
am = torch.randn(N, H, W, Cin, device="cuda", generator=g).to(torch.bfloat16)
om = torch.randn(N, H, W, Cin, device="cuda", generator=g).to(torch.bfloat16)
y2 = torch.full_like(y, 7.0)
conv.add_mask(dy.data_ptr(), y2.data_ptr(), T._stream(), add=add.data_ptr(), add_mask=am.data_ptr(), out_mask=om.data_ptr())
torch.cuda.synchronize()
print(y2[0,0,0,:6].tolist()); print(y[0,0,0,:6].tolist()); print(ref[0,0,0,:6].tolist()); print(add[0,0,0,:6].tolist()); print(om[0,0,0,:6].tolist())
print(dy.shape, dy.stride(), y.shape)
ref2 = (ref + add.float()) * (om.float() > 0)
bad = ((y2.float() - ref2).abs() > 0.1).reshape(-1, Cin)
print("bad frac", bad.float().mean().item(), "bad rows", bad.any(1).nonzero()[:10].flatten().tolist(), "n bad rows", bad.any(1).sum().item())
for name, kw in [("add+am", dict(add=add.data_ptr(), add_mask=am.data_ptr())), ("am", dict(add_mask=am.data_ptr())),
                 ("add+om", dict(add=add.data_ptr(), out_mask=om.data_ptr())), ("add", dict(add=add.data_ptr()))]:
    y3 = torch.full_like(y, 7.0)
    conv.add_mask(dy.data_ptr(), y3.data_ptr(), T._stream(), **kw)
    torch.cuda.synchronize()
    print(name, y3[0,0,0,:4].tolist())

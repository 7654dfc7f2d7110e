import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_15980_b200 import kernels as K
N, H, W, Cin, Kout, R = 2, 56, 56, 64, 256, 1
g = torch.Generator(device="cuda").manual_seed(7)
w = (torch.randn(Kout, R, R, Cin, device="cuda", generator=g) / (R * R * Kout) ** 0.5).to(torch.bfloat16)
dy = torch.randn(N, H, W, Kout, device="cuda", generator=g).to(torch.bfloat16)
wd = w.flip(1, 2).permute(3, 1, 2, 0).contiguous()
conv = K.Conv(N, H, W, Kout, Cin, R, R, 1, R // 2, wd.data_ptr())
st = torch.cuda.current_stream().cuda_stream
y = torch.empty(N, H, W, Cin, device="cuda", dtype=torch.bfloat16)
conv(dy.data_ptr(), y.data_ptr(), st)
add = torch.randn(N, H, W, Cin, device="cuda", generator=g).to(torch.bfloat16)
om = torch.randn(N, H, W, Cin, device="cuda", generator=g).to(torch.bfloat16)
for name, kw in [("none", {}), ("add", dict(add=add.data_ptr())), ("om", dict(out_mask=om.data_ptr())),
                 ("add+om", dict(add=add.data_ptr(), out_mask=om.data_ptr()))]:
    y2 = torch.empty_like(y)
    conv.add_mask(dy.data_ptr(), y2.data_ptr(), st, **kw)
    torch.cuda.synchronize()
    d = (y2.float() - y.float())
    print(name, "diff", d.abs().max().item(), "vs add", (d - add.float()).abs().max().item(),
          y2[0, 0, 0, :4].tolist(), y[0, 0, 0, :4].tolist(), add[0, 0, 0, :4].tolist())

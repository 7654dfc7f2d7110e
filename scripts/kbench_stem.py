"""Stem (7x7/2, C=4 NHWC4) forward timing at ResNet-50 bs256; the A-operand
path is chosen by DELTA_STEM_MODE (unset: row tiles; tma; gather).  Saves the output
checksum to compare the two paths bit-for-bit."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_15980_b200 import kernels as K

torch.manual_seed(0)
N = 256
x = torch.randn(N, 224, 224, 4, device="cuda").to(torch.bfloat16)
x[..., 3] = 0
w = (torch.randn(64, 7, 7, 4, device="cuda") * 0.05).to(torch.bfloat16)
w[..., 3] = 0
wp = K.pack_stem_weights(w)
conv = K.Conv(N, 224, 224, 4, 64, 7, 7, 2, 3, wp.data_ptr())
y = torch.empty(N, 112, 112, 64, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    conv(x.data_ptr(), y.data_ptr(), st)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    conv(x.data_ptr(), y.data_ptr(), st)
e.record(); torch.cuda.synchronize()
us = s.elapsed_time(e) / 20 * 1e3
ref = torch.nn.functional.conv2d(x[:8].permute(0, 3, 1, 2).float(), w.permute(0, 3, 1, 2).float(),
                                 stride=2, padding=3).permute(0, 2, 3, 1)
err = (y[:8].float() - ref).abs().max().item()
tag = os.environ.get("DELTA_STEM_MODE") or "rows"
torch.save(y[:16].cpu(), f"/tmp/stem_{tag}.pt")
print(f"stem mode={tag}: {us:.1f} us  max|err| vs fp32 {err:.4f}  "
      f"({411e6 / us / 1e3:.0f} GB/s output write)")

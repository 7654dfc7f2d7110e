import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_15980_b200 import kernels as K
H, C, Ko, R, s, p = [int(v) for v in sys.argv[1:7]]
N = 256
x = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
w = (torch.randn(Ko, R, R, C, device="cuda") * 0.05).to(torch.bfloat16)
conv = K.Conv(N, H, H, C, Ko, R, R, s, p, w.data_ptr())
y = torch.empty(N, conv.P, conv.Q, Ko, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    conv(x.data_ptr(), y.data_ptr(), st)
torch.cuda.synchronize()

"""One weight-gradient launch at a ResNet-50 bs256 shape, for ncu:
python scripts/wgrad_one.py H C K R stride pad"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_15980_b200 import kernels as K
H, C, Ko, R, s, p = [int(v) for v in sys.argv[1:7]]
N = 256
x = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
P_ = (H + 2 * p - R) // s + 1
dy = torch.randn(N, P_, P_, Ko, device="cuda").to(torch.bfloat16)
wg = K.Wgrad(N, H, H, C, Ko, R, R, s, p)
ws = torch.empty(wg.workspace_bytes, dtype=torch.uint8, device="cuda")
dw = torch.empty(Ko, R, R, C, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(4):
    wg(dy.data_ptr(), x.data_ptr(), dw.data_ptr(), ws.data_ptr(), st)
torch.cuda.synchronize()

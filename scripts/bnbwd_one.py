import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_15980_b200 import kernels as K
M, C = 256 * 56 * 56, 256
x = torch.randn(M, C, device="cuda").to(torch.bfloat16)
r = torch.randn(M, C, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
mean = torch.zeros(C, device="cuda"); inv = torch.ones(C, device="cuda"); gam = torch.ones(C, device="cuda")
dg = torch.empty(C, device="cuda"); db = torch.empty(C, device="cuda")
ws = torch.zeros(K.bn_workspace_floats(M, C), device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    K.bn_backward(r.data_ptr(), 0, x.data_ptr(), x.data_ptr(), y.data_ptr(), M, C, mean.data_ptr(), inv.data_ptr(), gam.data_ptr(), dg.data_ptr(), db.data_ptr(), ws.data_ptr(), st)
torch.cuda.synchronize()

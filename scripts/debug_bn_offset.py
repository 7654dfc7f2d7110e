import os, sys
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
st = torch.cuda.current_stream().cuda_stream
for (M, C) in [(802816, 256), (12544, 2048)]:
    nb = M * C * 2
    big = torch.empty(2 * nb + (1 << 20), dtype=torch.uint8, device="cuda")
    mean = torch.zeros(C, device="cuda"); inv = torch.ones(C, device="cuda"); gam = torch.ones(C, device="cuda")
    ws = torch.empty(K.bn_workspace_floats(M, C), device="cuda"); dg = torch.empty(C, device="cuda"); db = torch.empty(C, device="cuda")
    y = torch.empty(M, C, device="cuda", dtype=torch.bfloat16)
    for off in (0, 4096 + 256, 65536 + 2048, 1 << 19):
        x = big[:nb].view(torch.bfloat16)
        u = big[nb + off: 2 * nb + off].view(torch.bfloat16)
        t = timeit(lambda: K.bn_backward(u.data_ptr(), 0, None, x.data_ptr(), y.data_ptr(), M, C, mean.data_ptr(), inv.data_ptr(), gam.data_ptr(), dg.data_ptr(), db.data_ptr(), ws.data_ptr(), st))
        print(M, C, "offset", off, "bwd_nomask total us", round(t, 1), "GB/s(5 passes)", round(5 * nb / t / 1e3, 1))
    torch.cuda.synchronize()
    t = timeit(lambda: y.view(-1).copy_(x))
    print("copy", round(2 * nb / t / 1e3, 1))
    del big

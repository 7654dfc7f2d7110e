"""Per-kernel HBM throughput of the BN kernels at ResNet-50 bs256 sizes (torch
profiler kernel times; algorithmic bytes per kernel)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2203_15980_b200 import kernels as K
N = 256
st = torch.cuda.current_stream().cuda_stream
for (H, C) in [(56, 256), (56, 64), (28, 512), (14, 1024), (7, 2048)]:
    M = N * H * H
    x = torch.randn(M, C, device="cuda").to(torch.bfloat16)
    u = torch.randn(M, C, device="cuda").to(torch.bfloat16)
    mk = torch.randn(M, C, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    mean = torch.zeros(C, device="cuda"); inv = torch.ones(C, device="cuda")
    gam = torch.ones(C, device="cuda"); bet = torch.zeros(C, device="cuda")
    ws = torch.zeros(K.bn_workspace_floats(M, C), device="cuda")
    dg = torch.empty(C, device="cuda"); db = torch.empty(C, device="cuda")
    fns = {"stats": lambda: K.bn_stats(x.data_ptr(), M, C, ws.data_ptr(), mean.data_ptr(), inv.data_ptr(), 1e-5, None, None, 0.1, st),
           "apply0": lambda: K.bn_apply(0, x.data_ptr(), None, y.data_ptr(), M, C, mean.data_ptr(), inv.data_ptr(), gam.data_ptr(), bet.data_ptr(), stream=st),
           "bwd_mask": lambda: K.bn_backward(u.data_ptr(), 0, mk.data_ptr(), x.data_ptr(), y.data_ptr(), M, C, mean.data_ptr(), inv.data_ptr(), gam.data_ptr(), dg.data_ptr(), db.data_ptr(), ws.data_ptr(), st),
           "bwd_nomask": lambda: K.bn_backward(u.data_ptr(), 0, None, x.data_ptr(), y.data_ptr(), M, C, mean.data_ptr(), inv.data_ptr(), gam.data_ptr(), dg.data_ptr(), db.data_ptr(), ws.data_ptr(), st)}
    nb = M * C * 2
    byts = {"k_bn_stats_partial": nb, "k_bn_apply": 2 * nb, "k_bn_bwd_partial_mask": 3 * nb,
            "k_bn_bwd_apply_mask": 4 * nb, "k_bn_bwd_partial": 2 * nb, "k_bn_bwd_apply": 3 * nb}
    out = {"shape": [M, C]}
    for name, fn in fns.items():
        for _ in range(3): fn()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(10): fn()
            torch.cuda.synchronize()
        for ev in prof.key_averages():
            k = ev.key
            for base in ("k_bn_stats_partial", "k_bn_apply", "k_bn_bwd_partial", "k_bn_bwd_apply"):
                if base in k:
                    us = ev.device_time_total / ev.count if hasattr(ev, "device_time_total") else ev.cuda_time_total / ev.count
                    key = base + ("_mask" if name == "bwd_mask" and "bwd" in base else "")
                    out[f"{name}:{base}"] = dict(us=round(us, 1), gbs=round(byts.get(key, 0) / us / 1e3, 1))
    print(json.dumps(out), flush=True)

# max pool 3x3/2 on the stem output (N, 112, 112, 64)
x = torch.relu(torch.randn(N, 112, 112, 64, device="cuda")).to(torch.bfloat16)
y = torch.empty(N, 56, 56, 64, device="cuda", dtype=torch.bfloat16)
dy = torch.randn(N, 56, 56, 64, device="cuda").to(torch.bfloat16)
dx = torch.empty_like(x)
ws = torch.empty(K.maxpool_workspace_bytes(N, 112, 112, 64), dtype=torch.uint8, device="cuda")
def t(fn, iters=10):
    for _ in range(3): fn()
    s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s_.record()
    for _ in range(iters): fn()
    e_.record(); torch.cuda.synchronize()
    return s_.elapsed_time(e_) / iters * 1e3
tf = t(lambda: K.maxpool_fwd(x.data_ptr(), y.data_ptr(), N, 112, 112, 64, st))
tb = t(lambda: K.maxpool_bwd(dy.data_ptr(), x.data_ptr(), dx.data_ptr(), N, 112, 112, 64, ws.data_ptr(), st))
print(json.dumps(dict(maxpool_fwd_us=round(tf, 1), fwd_gbs=round((x.numel() + y.numel()) * 2 / tf / 1e3),
                      maxpool_bwd_us=round(tb, 1),
                      bwd_gbs=round((x.numel() * 2 + dy.numel() * 2 * 2 + ws.numel() * 2 + dx.numel() * 2) / tb / 1e3))))

"""Optimizer step + weight views for ResNet-50: the fused kernels (optim.cu)
vs the per-tensor torch sequence they replaced.  CUDA events, 20 iters."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_15980_b200 import graph as G, kernels as K
from paper_2203_15980_b200.runtime import Params

g = G.build_resnet(50, 256)
p = Params(g, torch.device("cuda"))
p.grad.normal_()


def torch_seq(lr=0.1, m=0.9, wd=1e-4):
    p.mom.mul_(m).add_(p.grad).add_(p.master, alpha=wd)
    p.master.add_(p.mom, alpha=-lr)
    p.conv_bf16.copy_(p.master[:p.n_conv])
    for name, packed in p.stem_packed.items():
        K.pack_stem_weights(p.wbf[name], packed)
    for name, wd_ in p.wd.items():
        wd_.copy_(p.wbf[name].flip(1, 2).permute(3, 1, 2, 0))


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


st = torch.cuda.current_stream().cuda_stream
t_fused = timeit(lambda: p.sgd_step(0.1))
t_sgd = timeit(lambda: K.sgd_step(p.master.data_ptr(), p.mom.data_ptr(), p.grad.data_ptr(),
                                  p.conv_bf16.data_ptr(), p.numel, p.n_conv, 0.1, 0.9, 1e-4, st))
t_views = timeit(lambda: K.weight_views(p.views_dev.data_ptr(), p.n_views, st))
t_torch = timeit(torch_seq)
print(f"params {p.numel}  views {p.n_views}: fused {t_fused:.1f} us (sgd {t_sgd:.1f}, views "
      f"{t_views:.1f}) vs torch sequence {t_torch:.1f} us")

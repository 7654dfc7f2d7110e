"""LayerNorm forward / backward(+dropout) kernel timing on BERT-large shapes
([16384][1024] bf16), CUDA events over 200 launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_15980_b200 import kernels as K  # noqa: E402

rows, H = 16384, 1024
dev = "cuda"
x = torch.randn(rows, H, device=dev).to(torch.bfloat16)
y = torch.empty_like(x)
mean = torch.empty(rows, device=dev)
rstd = torch.empty(rows, device=dev)
g = torch.ones(H, device=dev)
b = torch.zeros(H, device=dev)
st = torch.cuda.current_stream().cuda_stream
# L2 flush by READING 256 MB (writing it would leave dirty lines the timed
# kernel would pay to write back)
flush = torch.ones(64 * 2**20, device=dev)


def timed(fn, n=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(n):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / n * 1e3


us = timed(lambda: K.layernorm_fwd(x.data_ptr(), y.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                                   g.data_ptr(), b.data_ptr(), rows, H, 1e-12, st))
print(f"layernorm_fwd {us:.1f} us  {2 * rows * H * 2 / us / 1e3:.0f} GB/s "
      f"lib={os.environ.get('DELTA_LIB', '')} ctas={os.environ.get('DELTA_LNF_CTAS', '')}")

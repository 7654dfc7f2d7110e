"""Micro-benchmark: input-gradient (dgrad) convolutions of ResNet-50 bs256 through
our tcgen05 kernel (plain / add+mask / BN-backward epilogues) beside cuDNN's
dgrad (aten convolution_backward, input gradient only).  CUDA events, inputs > L2."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_15980_b200 import kernels as K


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
# H, C (fwd in = dgrad out), K (fwd out), R
shapes = [(56, 64, 256, 1), (56, 256, 64, 1), (56, 64, 64, 3), (28, 128, 512, 1), (28, 512, 128, 1),
          (28, 128, 128, 3), (14, 256, 1024, 1), (14, 1024, 256, 1), (14, 256, 256, 3),
          (7, 512, 2048, 1), (7, 2048, 512, 1), (7, 512, 512, 3)]
st = torch.cuda.current_stream().cuda_stream
for (H, C, Ko, R) in shapes:
    M = N * H * H
    w = (torch.randn(Ko, R, R, C, device="cuda") * 0.05).to(torch.bfloat16)
    wd = w.flip(1, 2).permute(3, 1, 2, 0).contiguous()
    dy = torch.randn(N, H, H, Ko, device="cuda").to(torch.bfloat16)
    conv = K.Conv(N, H, H, Ko, C, R, R, 1, R // 2, wd.data_ptr())
    y = torch.empty(N, H, H, C, device="cuda", dtype=torch.bfloat16)
    t_plain256 = timeit(lambda: conv(dy.data_ptr(), y.data_ptr(), st))
    if conv.tile_n > 128:
        conv.set_tile_n(128)
    a = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
    m = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
    mean = torch.zeros(C, device="cuda"); inv = torch.ones(C, device="cuda")
    gam = torch.ones(C, device="cuda"); bet = torch.zeros(C, device="cuda")
    parts = torch.empty(K.stats_partials_floats(C), device="cuda")
    t_plain = timeit(lambda: conv(dy.data_ptr(), y.data_ptr(), st))
    t_add = timeit(lambda: conv.add_mask(dy.data_ptr(), y.data_ptr(), st, add=a.data_ptr(), out_mask=m.data_ptr()))
    t_bn = timeit(lambda: conv.bn_bwd(dy.data_ptr(), y.data_ptr(), parts.data_ptr(), a.data_ptr(), mean.data_ptr(), inv.data_ptr(), gam.data_ptr(), bet.data_ptr(), st))
    xt = torch.empty(N, C, H, H, device="cuda", dtype=torch.bfloat16, memory_format=torch.channels_last)
    wt = w.permute(0, 3, 1, 2)
    t_cudnn = timeit(lambda: torch.ops.aten.convolution_backward(dy.permute(0, 3, 1, 2), xt, wt, None, [1, 1], [R // 2] * 2, [1, 1], False, [0, 0], 1, [True, False, False]))
    flops = 2.0 * M * C * Ko * R * R
    print(json.dumps(dict(shape=[H, C, Ko, R], plain_us=round(t_plain * 1e3, 1), plain_default_tile_us=round(t_plain256 * 1e3, 1), add_mask_us=round(t_add * 1e3, 1),
                          bn_bwd_us=round(t_bn * 1e3, 1), cudnn_us=round(t_cudnn * 1e3, 1),
                          plain_tflops=round(flops / t_plain / 1e9, 1),
                          min_hbm_us=round((M * C + M * Ko) * 2 / 6.5e6, 1))), flush=True)

# stride-2 shortcut: conv1 dgrad + the downsample's gradient at its sampling grid
for (H, C, Ko) in [(56, 256, 128), (28, 512, 256), (14, 1024, 512)]:
    M = N * H * H
    w = (torch.randn(Ko, 1, 1, C, device="cuda") * 0.05).to(torch.bfloat16)
    wd = w.permute(3, 1, 2, 0).contiguous()
    dy = torch.randn(N, H, H, Ko, device="cuda").to(torch.bfloat16)
    conv = K.Conv(N, H, H, Ko, C, 1, 1, 1, 0, wd.data_ptr())
    if conv.tile_n > 128:
        conv.set_tile_n(128)
    y = torch.empty(N, H, H, C, device="cuda", dtype=torch.bfloat16)
    sub = torch.randn(N, H // 2, H // 2, C, device="cuda").to(torch.bfloat16)
    m = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
    full = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
    t_s2 = timeit(lambda: conv.add_mask(dy.data_ptr(), y.data_ptr(), st, add=sub.data_ptr(), out_mask=m.data_ptr(), add_stride2=True))
    t_full = timeit(lambda: conv.add_mask(dy.data_ptr(), y.data_ptr(), st, add=full.data_ptr(), out_mask=m.data_ptr()))
    print(json.dumps(dict(shape=[H, C, Ko], add_stride2_us=round(t_s2 * 1e3, 1), add_full_us=round(t_full * 1e3, 1))), flush=True)

"""Weight-gradient micro-benchmark at ResNet-50 bs256 shapes: our tcgen05
split-K kernel (+ its reduce) vs cuDNN's wgrad (aten convolution_backward,
weight only) + the fp32 KRSC copy the runtime needs after it."""
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
    return s.elapsed_time(e) / iters * 1e3


N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
st = torch.cuda.current_stream().cuda_stream
shapes = [  # H, C, K, R, stride, pad
    (224, 4, 64, 7, 2, 3),
    (56, 64, 64, 1, 1, 0), (56, 64, 64, 3, 1, 1), (56, 64, 256, 1, 1, 0), (56, 256, 64, 1, 1, 0),
    (56, 256, 128, 1, 1, 0), (56, 128, 128, 3, 2, 1), (56, 256, 512, 1, 2, 0),
    (28, 128, 512, 1, 1, 0), (28, 512, 128, 1, 1, 0), (28, 128, 128, 3, 1, 1),
    (14, 256, 1024, 1, 1, 0), (14, 1024, 256, 1, 1, 0), (14, 256, 256, 3, 1, 1),
    (7, 512, 2048, 1, 1, 0), (7, 2048, 512, 1, 1, 0), (7, 512, 512, 3, 1, 1)]
tot_ours = tot_cudnn = 0.0
for (H, C, Ko, R, s, p) in shapes:
    x = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
    if C == 4:
        x[..., 3] = 0
    P_ = (H + 2 * p - R) // s + 1
    dy = torch.randn(N, P_, P_, Ko, device="cuda").to(torch.bfloat16)
    w = torch.randn(Ko, R, R, C, device="cuda").to(torch.bfloat16)
    wg = K.Wgrad(N, H, H, C, Ko, R, R, s, p)
    ws = torch.empty(wg.workspace_bytes, dtype=torch.uint8, device="cuda")
    dw = torch.empty(Ko, R, R, C, device="cuda")
    t_ours = timeit(lambda: wg(dy.data_ptr(), x.data_ptr(), dw.data_ptr(), ws.data_ptr(), st))

    def cudnn():
        _, gw, _ = torch.ops.aten.convolution_backward(
            dy.permute(0, 3, 1, 2), x.permute(0, 3, 1, 2), w.permute(0, 3, 1, 2), None, [s, s],
            [p, p], [1, 1], False, [0, 0], 1, [False, True, False])
        dw.copy_(gw.permute(0, 2, 3, 1))
    t_cudnn = timeit(cudnn)
    flops = 2.0 * N * P_ * P_ * Ko * C * R * R
    tot_ours += t_ours
    tot_cudnn += t_cudnn
    print(json.dumps(dict(shape=[H, C, Ko, R, s], ours_us=round(t_ours, 1), cudnn_us=round(t_cudnn, 1),
                          ours_tflops=round(flops / t_ours / 1e6, 1), splits_ws_mb=round(wg.workspace_bytes / 2**20, 1))), flush=True)
print(json.dumps(dict(total_ours_us=round(tot_ours, 1), total_cudnn_us=round(tot_cudnn, 1))))

"""Per-launch cost of dependent kernels inside a CUDA graph on this GPU:
N back-to-back tiny kernels (each 148 blocks) captured once, replayed."""
import torch
x = torch.zeros(148 * 256, device="cuda")
s = torch.cuda.Stream()
for n in (100, 1000):
    with torch.cuda.stream(s):
        for _ in range(3):
            for _ in range(n):
                x.add_(1.0)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                x.add_(1.0)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
    torch.cuda.synchronize()
    print(f"{n} dependent launches in a graph: {e0.elapsed_time(e1) / 10 / n * 1e3:.2f} us each "
          f"(kernel alone: 148 blocks x 256 threads, 150 KB)")

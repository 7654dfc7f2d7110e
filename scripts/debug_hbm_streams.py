import torch
def timeit(fn, iters=20):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3
n = 802816 * 256
a = torch.randn(n, device="cuda").to(torch.bfloat16)
b = torch.randn(n, device="cuda").to(torch.bfloat16)
c = torch.empty_like(a)
d = torch.randn(n, device="cuda").to(torch.bfloat16)
nb = n * 2
t = timeit(lambda: c.copy_(a)); print("copy 1R1W", round(2 * nb / t / 1e3))
t = timeit(lambda: torch.add(a, b, out=c)); print("add 2R1W", round(3 * nb / t / 1e3))
t = timeit(lambda: torch.addcmul(a, b, d, out=c)); print("addcmul 3R1W", round(4 * nb / t / 1e3))
t = timeit(lambda: a.sum()); print("sum 1R", round(nb / t / 1e3))
af = a.view(802816, 256); bf = b.view(802816, 256)
t = timeit(lambda: (af * bf).sum(0)); print("mul+sum (2R + 1W + 1R)", round(4 * nb / t / 1e3))

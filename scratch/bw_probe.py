import torch
x = torch.randn(1 << 28, device="cuda")   # 1 GiB
y = torch.empty_like(x)
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return best
b = x.numel() * 4
print("copy   GB/s", 2 * b / t(lambda: y.copy_(x)) / 1e9)
print("read   GB/s (sum)", b / t(lambda: x.sum()) / 1e9)
print("read   GB/s (amax)", b / t(lambda: x.abs().max()) / 1e9 * 0 + b / t(lambda: torch.amax(x)) / 1e9)
print("write  GB/s (fill)", b / t(lambda: y.fill_(1.0)) / 1e9)
h = torch.empty(x.numel() // 8, dtype=torch.int32, device="cuda")
print("read 4B + write 0.5B (x -> x[::8] int)", (b + h.numel() * 4) / t(lambda: h.copy_(x[::8])) / 1e9)

import torch
x = torch.empty(1 << 27, dtype=torch.float64, device='cuda')  # 1 GiB
y = torch.empty_like(x)
def t(f, n=10):
    f(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
    return best
g = 1 << 30
print('fill  GB/s', g / t(lambda: x.fill_(1.0)) / 1e6)
print('copy  GB/s (r+w)', 2 * g / t(lambda: y.copy_(x)) / 1e6)
print('sum   GB/s', g / t(lambda: x.sum()) / 1e6)

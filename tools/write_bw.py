"""Pure-write HBM bandwidth on this GPU (ceiling for write-dominated kernels such as s2_out)."""
import torch

n = 5_000_000_000 // 2
x = torch.empty(n, dtype=torch.int16, device="cuda")
y = torch.empty(n, dtype=torch.int16, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]))
    return best


for name, fn, rb in (("fill_", lambda: x.fill_(7), 0), ("zero_", lambda: x.zero_(), 0),
                     ("copy_", lambda: y.copy_(x), 1)):
    ms = t(fn)
    wb = 2 * n
    print(f"{name}: {ms:.3f} ms  write {wb / ms / 1e6:.0f} GB/s  total {(wb * (1 + rb)) / ms / 1e6:.0f} GB/s")

"""PCIe copy rates on this box: H2D, D2H, both directions at once (pinned)."""
import torch

n = 2 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        torch.cuda.synchronize()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: h.copy_(d, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


bi = t(both)
print(f"H2D {n / h2d / 1e6:.1f} GB/s  D2H {n / d2h / 1e6:.1f} GB/s  both-directions {2 * n / bi / 1e6:.1f} GB/s total")

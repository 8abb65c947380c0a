"""Per-build time with and without per-kernel event profiling (small trees)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2401_06089_b200 import DendrogramBuilder, synth  # noqa: E402
for shape, n in (("blobs1m", 999_999), ("random", 100_000), ("tied", 128_000_000)):
    nv, u, v, w = synth.GENERATORS[shape](n, seed=0)
    b = DendrogramBuilder("cuda:0")
    du, dv, dw = (torch.from_numpy(x).cuda() for x in (u, v, w))
    r = b.build(nv, du, dv, dw)
    for prof in (False, True, False, True):
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = 20 if n < 10_000_000 else 3
        a.record()
        for _ in range(k):
            b.build(nv, du, dv, dw, out=r, profile=prof)
        z.record()
        torch.cuda.synchronize()
        print(f"{shape} n={n} profile={prof}: {a.elapsed_time(z) / k:.3f} ms/build")

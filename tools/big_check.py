"""Largest-size sanity: build a 300M-edge random tree (tied weights, or
uniform weights with `random`) and check the size-independent dendrogram
properties of tests/test_parity_gpu.py.  python tools/big_check.py [n] [shape]"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2401_06089_b200 import DendrogramBuilder, synth  # noqa: E402
from tests.test_parity_gpu import check_dendrogram_properties  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000_000
shape = sys.argv[2] if len(sys.argv) > 2 else "tied"
t = time.time()
nv, u, v, w = synth.GENERATORS[shape](n, seed=0)
print(f"generated n={n} in {time.time() - t:.1f}s", flush=True)
b = DendrogramBuilder("cuda:0")
du, dv, dw = (torch.from_numpy(x).cuda() for x in (u, v, w))
r = b.build(nv, du, dv, dw)
torch.cuda.synchronize()
a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
r = b.build(nv, du, dv, dw, out=r)
z.record()
torch.cuda.synchronize()
print(f"build {a.elapsed_time(z):.1f} ms, levels {r.num_levels}, workspace {b._ws.numel() / 1e9:.1f} GB, "
      f"paths {r.stats.path_info()}", flush=True)
del du, dv, dw
torch.cuda.empty_cache()
check_dendrogram_properties(nv, u, v, w, r)
print("properties ok")

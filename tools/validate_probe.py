"""Time device validation (weighted_tree_b200's dmst_validate) at 128M."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2401_06089_b200 import synth, validate_b200  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128_000_000
nv, u, v, w = synth.GENERATORS["tied"](n, seed=0)
du, dv, dw = (torch.from_numpy(x).cuda() for x in (u, v, w))
validate_b200(nv, du, dv, dw)
torch.cuda.synchronize()
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    validate_b200(nv, du, dv, dw)
    b.record()
    torch.cuda.synchronize()
    print(f"validate n={n}: {a.elapsed_time(b):.2f} ms")
dv2 = dv.clone()
dv2[n - 1] = du[0]  # likely duplicate or cycle -> slow path (sort)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
try:
    validate_b200(nv, du, dv2, dw)
except ValueError as e:
    msg = str(e)
b.record()
torch.cuda.synchronize()
print(f"invalid tree ({msg}): {a.elapsed_time(b):.2f} ms")

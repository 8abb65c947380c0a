"""Where does the host-buffer build spend its time?  Serial build_host vs
its parts (H2D alone, device build, D2H alone), config-4 shape."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_06089_b200 import DendrogramBuilder, HostBuildResult, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128_000_000
nv, u, v, w = synth.GENERATORS["tied"](n, seed=0)
hu, hv, hw = (torch.from_numpy(x).pin_memory() for x in (u, v, w))
b = DendrogramBuilder("cuda:0")
out = HostBuildResult.empty(n, nv)


def ev_time(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        t0 = time.perf_counter()
        fn()
        z.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(z))
        wall = (time.perf_counter() - t0) * 1e3
    return best, wall


print("build_host serial: %.1f ms (wall %.1f)" % ev_time(lambda: b.build_host(nv, hu, hv, hw, out=out)))
du, dv, dw = (torch.empty_like(x, device="cuda") for x in (hu, hv, hw))


def h2d():
    du.copy_(hu, non_blocking=True)
    dv.copy_(hv, non_blocking=True)
    dw.copy_(hw, non_blocking=True)


print("H2D only: %.1f ms (wall %.1f)" % ev_time(h2d))
r = b.build(nv, du, dv, dw)
print("device build: %.1f ms (wall %.1f)" % ev_time(lambda: b.build(nv, du, dv, dw, out=r)))


def d2h():
    out.orig_of.copy_(r.orig_of, non_blocking=True)
    out.heights.copy_(r.heights, non_blocking=True)
    out.edge_parent.copy_(r.edge_parent, non_blocking=True)
    out.vertex_parent.copy_(r.vertex_parent, non_blocking=True)


print("D2H only: %.1f ms (wall %.1f)" % ev_time(d2h))
st = b.build_host(nv, hu, hv, hw, out=out, profile=True).stats
prof = st.kernel_profile()
print("build_host kernel sum %.1f ms" % sum(v[0] for v in prof.values()))

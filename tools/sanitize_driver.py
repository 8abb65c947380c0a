"""Small builds for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every entry point (device build incl. the cooperative tail, host-buffer build,
validation incl. the duplicate-sort path, dendrogram height) on small trees,
each checked against the CPU oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import dendro_oracle as O  # noqa: E402
from paper_2401_06089_b200 import (DendrogramBuilder, dendrogram_height_b200, synth,  # noqa: E402
                                   validate_b200)
from paper_2401_06089_b200.api import _tree_format_error  # noqa: E402

b = DendrogramBuilder("cuda:0")
bad = 0
for shape in ("random", "tied", "path", "caterpillar"):
    for n in (1, 5, 1000, 70_000):
        nv, u, v, w = synth.GENERATORS[shape](n, seed=n)
        r = b.build(nv, u, v, w, debug=True, want_chains=True)
        e = O.build(nv, u, v, w)
        ok = (np.array_equal(r.edge_parent.cpu().numpy(), e.edge_parent)
              and np.array_equal(r.vertex_parent.cpu().numpy(), e.vertex_parent)
              and np.array_equal(r.orig_of.cpu().numpy(), e.orig_of))
        hb = b.build_host(nv, u, v, w)
        ok &= np.array_equal(hb.edge_parent.numpy(), e.edge_parent)
        ok &= dendrogram_height_b200(r.edge_parent) == O.dendrogram_height(e.edge_parent, e.vertex_parent)
        bad += not ok
# validation: valid, duplicate (sort path), cycle (sort path, no duplicate), self-loop
nv, u, v, w = synth.random_attach(50_000, seed=3)
u = u.astype(np.int64)
v = v.astype(np.int64)
cases = {"valid": (u, v)}
u2, v2 = u.copy(), v.copy()
u2[-1], v2[-1] = v[0], u[0]
cases["duplicate"] = (u2, v2)
u3, v3 = u.copy(), v.copy()
u3[7] = v3[7]
cases["self_loop"] = (u3, v3)
for name, (uu, vv) in cases.items():
    def verdict(fn, err):
        try:
            fn(nv, uu, vv, w)
            return ""
        except err as exc:
            return str(exc)
    bad += verdict(validate_b200, _tree_format_error()) != verdict(O.weighted_tree, O.TreeFormatError)
print("sanitize driver done, mismatches:", bad)

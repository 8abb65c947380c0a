"""Small builds for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import dendro_oracle as O  # noqa: E402
from paper_2401_06089_b200 import DendrogramBuilder, synth  # noqa: E402

b = DendrogramBuilder("cuda:0")
bad = 0
for shape in ("random", "tied", "path", "caterpillar"):
    for n in (1, 5, 1000, 70_000):
        nv, u, v, w = synth.GENERATORS[shape](n, seed=n)
        r = b.build(nv, u, v, w, debug=True)
        e = O.build(nv, u, v, w)
        ok = (np.array_equal(r.edge_parent.cpu().numpy(), e.edge_parent)
              and np.array_equal(r.vertex_parent.cpu().numpy(), e.vertex_parent)
              and np.array_equal(r.orig_of.cpu().numpy(), e.orig_of))
        bad += not ok
print("sanitize driver done, mismatches:", bad)

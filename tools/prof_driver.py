"""One dendrogram build for profiling (ncu / compute-sanitizer).

    python tools/prof_driver.py [--n N] [--shape tied|random|path|caterpillar] [--repeat R]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2401_06089_b200 import DendrogramBuilder, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16_000_000)
ap.add_argument("--shape", default="tied")
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--paths", default="", help="JSON dmst_stats path overrides")
a = ap.parse_args()
nv, u, v, w = synth.GENERATORS[a.shape](a.n, seed=0)
b = DendrogramBuilder("cuda:0")
du, dv, dw = (torch.from_numpy(x).cuda() for x in (u, v, w))
for _ in range(a.repeat):
    r = b.build(nv, du, dv, dw, paths=json.loads(a.paths) if a.paths else None)
torch.cuda.synchronize()
print("levels", r.num_levels, "launches", r.stats.kernel_launches, "sort1", r.stats.sort1_passes,
      "sort2", r.stats.sort2_passes)

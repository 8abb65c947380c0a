"""Per-kernel timeline of one build (DMST_TIMELINE=1): python tools/timeline.py [n] [shape]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DMST_TIMELINE"] = "1"
import torch  # noqa: E402
from paper_2401_06089_b200 import DendrogramBuilder, synth  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
shape = sys.argv[2] if len(sys.argv) > 2 else "tied"
import json  # noqa: E402
paths = json.loads(sys.argv[3]) if len(sys.argv) > 3 else None
nv, u, v, w = synth.GENERATORS[shape](n, seed=0)
b = DendrogramBuilder("cuda:0")
du, dv, dw = (torch.from_numpy(x).cuda() for x in (u, v, w))
for _ in range(2):
    r = b.build(nv, du, dv, dw, profile=True, paths=paths)
torch.cuda.synchronize()
print(r.stats.path_info())

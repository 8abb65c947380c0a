"""Statistics of the chain keys (sort #2 input) of one build: how sorted is
the key sequence in rank order?  python tools/key_stats.py [n] [shape]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2401_06089_b200 import DendrogramBuilder, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
shape = sys.argv[2] if len(sys.argv) > 2 else "tied"
nv, u, v, w = synth.GENERATORS[shape](n, seed=0)
b = DendrogramBuilder("cuda:0")
r = b.build(nv, u, v, w, debug=True)
key = r.debug["chain_key"].cpu().numpy().astype(np.int64)
ret = r.debug["retirement"].cpu().numpy().astype(np.int64)
lvl = r.debug["chain_level"].cpu().numpy().astype(np.int64)
print("n", n, "levels", r.num_levels, "distinct keys", len(np.unique(key)), "max key", key.max())
print("root frac", np.mean(key == 0))
nz = key[key > 0]
asc = np.mean(np.diff(nz) > 0)
print("nonzero ascending steps", asc, "runs", int(np.sum(np.diff(nz) <= 0)) + 1)
# greedy increasing subsequence
last = -1; keep = 0
for k in nz[: 2_000_000]:
    if k > last:
        keep += 1; last = k
print("greedy ascending keep frac (first 2M)", keep / min(len(nz), 2_000_000))
for L in range(0, r.num_levels + 1):
    m = lvl == L
    print("chain level", L, "frac", m.mean(), "ret0 frac", np.mean(ret[m] == 0) if m.any() else 0)
# how far is each item from its sorted position (displacement)
order = np.argsort(key, kind="stable")
pos = np.empty_like(order); pos[order] = np.arange(len(order))
disp = np.abs(pos - np.arange(len(order)))
print("median displacement", np.median(disp), "p90", np.percentile(disp, 90))

"""Time the device mutual-reachability MST (config 2 shape: 1M 3-D blobs)."""
import sys
import time

import numpy as np
import torch

from paper_2401_06089_b200 import mutual_reachability_mst_b200

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rng = np.random.default_rng(0)
centers = rng.uniform(-10.0, 10.0, (10, 3))
coords = centers[rng.integers(0, 10, n)] + rng.standard_normal((n, 3))
x = torch.from_numpy(coords).cuda()
mutual_reachability_mst_b200(x[:5000], 2)
torch.cuda.synchronize()
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t = mutual_reachability_mst_b200(x, 2)
    e1.record()
    torch.cuda.synchronize()
    print(f"n={n}: {e0.elapsed_time(e1):.1f} ms", flush=True)

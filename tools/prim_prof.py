"""One device mreach MST (for ncu captures of k_prim / k_core_sq)."""
import sys

import numpy as np
import torch

from paper_2401_06089_b200 import mutual_reachability_mst_b200

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((n, 3))).cuda()
mutual_reachability_mst_b200(x, 2)
torch.cuda.synchronize()

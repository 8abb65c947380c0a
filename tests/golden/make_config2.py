"""Generate the config-2 fixture: the reference's own mutual-reachability MST
of 1,000,000 3-D Gaussian-blob points (min_pts = 2).

Config 2 (BASELINE.json configs[1]):
  rng = numpy.random.default_rng(0)
  centers = rng.uniform(-10, 10, (10, 3))
  labels  = rng.integers(0, 10, n)
  coords  = centers[labels] + rng.standard_normal((n, 3))
  tree    = dendromst.pointgen.mutual_reachability_mst(PointCloud(coords, "blobs", 0), min_pts=2)
            (/root/reference/pkg/src/dendromst/pointgen.py:158-178, dense numba Prim)

The tree is produced by the UNMODIFIED reference, imported from
/root/reference/pkg/src (read-only; NUMBA_CACHE_DIR must point somewhere
writable).  It takes ~50 min on one core, so the result is committed as
tests/golden/config2_blobs1m.npz (u, v int32; w float64; original-id order
= Prim discovery order, exactly as the reference emits it).

Usage: NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_config2.py [n]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from dendromst.pointgen import PointCloud, mutual_reachability_mst  # noqa: E402


def blobs(n: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-10.0, 10.0, (10, 3))
    labels = rng.integers(0, 10, n)
    return centers[labels] + rng.standard_normal((n, 3))


def main() -> None:
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                       "config2_blobs1m.npz" if n == 1_000_000 else f"config2_blobs{n}.npz")
    coords = blobs(n, 0)
    t0 = time.perf_counter()
    tree = mutual_reachability_mst(PointCloud(coords, "blobs", 0), min_pts=2)
    dt = time.perf_counter() - t0
    np.savez_compressed(out, u=tree.u.astype(np.int32), v=tree.v.astype(np.int32),
                        w=tree.w, num_vertices=np.int64(tree.num_vertices))
    print(f"wrote {out}: {tree.num_edges} edges in {dt:.1f}s")


if __name__ == "__main__":
    main()

"""Golden vectors for the device mutual-reachability MST producer (SURVEY.md
8f rank 4): the UNMODIFIED reference's `mutual_reachability_mst` and
`core_distances` (/root/reference/pkg/src/dendromst/pointgen.py:56-178) on
small point clouds -- both Prim engines, ties (integer grids with duplicate
points), dims 2..8, min_pts 2..5.  Written to tests/golden/mreach_small.npz
(coords, core_sq, u, v, w per case) + mreach_small.json (the case list).

Usage: NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_mreach.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from dendromst.pointgen import PointCloud, core_distances, gen_points, mutual_reachability_mst  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [
    # name, kind, n, dim, min_pts, engine, seed
    ("normal3_numba", "normal", 3000, 3, 2, "numba", 1),
    ("uniform2_numpy", "uniform", 2000, 2, 4, "numpy", 2),
    ("normal8_numpy", "normal", 1500, 8, 3, "numpy", 3),
    ("normal8_numba", "normal", 1500, 8, 5, "numba", 4),
    ("normal5_numba", "normal", 1200, 5, 2, "numba", 5),
    ("blobs3_auto", "blobs", 5000, 3, 2, "auto", 6),
    ("grid2_numba", "grid", 1000, 2, 2, "numba", 7),
    ("grid2_numpy", "grid", 1000, 2, 2, "numpy", 7),
    ("grid3_numba_k3", "grid", 800, 3, 3, "numba", 8),
    ("tiny_auto", "normal", 5, 2, 2, "auto", 9),
]


def coords_for(kind, n, dim, seed):
    if kind in ("normal", "uniform"):
        return gen_points(kind, n, dim, seed).coords
    rng = np.random.default_rng(seed)
    if kind == "blobs":
        centers = rng.uniform(-10.0, 10.0, (10, dim))
        return centers[rng.integers(0, 10, n)] + rng.standard_normal((n, dim))
    if kind == "grid":  # integer lattice: duplicate points and tied distances
        return rng.integers(0, 12, (n, dim)).astype(np.float64)
    raise ValueError(kind)


def main() -> None:
    arrays, meta = {}, []
    for name, kind, n, dim, k, engine, seed in CASES:
        x = np.ascontiguousarray(coords_for(kind, n, dim, seed), dtype=np.float64)
        t = mutual_reachability_mst(PointCloud(x, kind, seed), min_pts=k, engine=engine)
        arrays[f"{name}_coords"] = x
        arrays[f"{name}_core_sq"] = core_distances(x, k) ** 2
        arrays[f"{name}_u"] = t.u.astype(np.int32)
        arrays[f"{name}_v"] = t.v.astype(np.int32)
        arrays[f"{name}_w"] = t.w
        meta.append({"name": name, "kind": kind, "n": n, "dim": dim, "min_pts": k, "engine": engine, "seed": seed})
    np.savez_compressed(os.path.join(HERE, "mreach_small.npz"), **arrays)
    with open(os.path.join(HERE, "mreach_small.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(f"wrote {len(meta)} cases")


if __name__ == "__main__":
    main()

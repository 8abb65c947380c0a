"""Golden verdicts of the reference's input validation (`weighted_tree`,
/root/reference/pkg/src/dendromst/tree_core.py:110-139) on valid and invalid
trees: the reference's own test cases (tests/test_tree_core.py:41-68) plus
larger and combined defects.  Records the exact TreeFormatError message (""
for a valid tree).  Run in the development container (the reference cannot
travel to the GPU box):

    NUMBA_CACHE_DIR=/tmp/nb PYTHONPATH=/root/reference/pkg/src python tests/golden/make_invalid.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("DENDROMST_SRC", "/root/reference/pkg/src"))
from dendromst.tree_core import TreeFormatError, weighted_tree  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    rng = np.random.default_rng(7)
    yield "kat_edge_count", 4, [0, 1], [1, 2], [1.0, 2.0]                  # test_tree_core.py:42-44
    yield "kat_too_few_vertices", 1, [], [], []                             # :46-48
    yield "kat_self_loop", 3, [0, 1], [1, 1], [1.0, 2.0]                    # :50-52
    yield "kat_duplicate", 3, [0, 1], [1, 0], [1.0, 2.0]                    # :54-56
    yield "kat_cycle", 4, [0, 1, 2], [1, 2, 0], [1.0, 2.0, 3.0]             # :58-60
    yield "kat_out_of_range", 3, [0, 1], [1, 3], [1.0, 2.0]                 # :62-64
    yield "kat_non_finite", 3, [0, 1], [1, 2], [1.0, float("nan")]          # :66-68
    yield "negative_id", 3, [0, -1], [1, 2], [1.0, 2.0]
    yield "valid_pair", 2, [0], [1], [0.5]
    for n in (1000, 20_000):
        nv = n + 1
        child = np.arange(1, nv)
        par = rng.integers(0, child)
        perm = rng.permutation(n)
        u, v, w = par[perm], child[perm], rng.random(n)
        yield f"valid_{n}", nv, u, v, w
        w2 = w.copy(); w2[[n // 3, n // 2]] = [np.inf, np.nan]
        yield f"inf_nan_{n}", nv, u, v, w2
        u2 = u.copy(); u2[n // 4] = v[n // 4]; u2[n // 5] = v[n // 5]
        yield f"self_loops_{n}", nv, u2, v, w
        u3 = u.copy(); v3 = v.copy(); u3[n - 1], v3[n - 1] = v[0], u[0]   # duplicate of edge 0, reversed
        yield f"duplicate_{n}", nv, u3, v3, w
        # cut a leaf off and add a chord between two far vertices: same edge
        # count, no duplicate, one cycle + an isolated vertex
        leaf = np.setdiff1d(v, u)[0]
        e = int(np.nonzero(v == leaf)[0][0])
        a, b = int(v[(e + 1) % n]), int(v[(e + n // 2) % n])
        u5 = u.copy(); v5 = v.copy(); u5[e], v5[e] = a, b
        yield f"cycle_isolated_{n}", nv, u5, v5, w
        # two isolated leaves and a doubled chord elsewhere -> still "not a tree"
        u6 = u5.copy(); v6 = v5.copy()
        leaf2 = [x for x in np.setdiff1d(v, u)[1:4] if x not in (a, b)][0]
        e2 = int(np.nonzero(v == leaf2)[0][0])
        u6[e2], v6[e2] = int(v[(e2 + 3) % n]), int(v[(e2 + n // 3) % n])
        yield f"two_cycles_{n}", nv, u6, v6, w
        yield f"out_of_range_{n}", nv, u, np.where(np.arange(n) == 7, nv, v), w
        yield f"nan_and_self_loop_{n}", nv, u2, v, w2                         # first check wins


def main():
    out = {}
    arrays = {}
    for name, nv, u, v, w in cases():
        u = np.asarray(u, np.int64); v = np.asarray(v, np.int64); w = np.asarray(w, np.float64)
        try:
            weighted_tree(nv, u, v, w)
            msg = ""
        except TreeFormatError as exc:
            msg = str(exc)
        out[name] = {"num_vertices": int(nv), "message": msg}
        arrays[f"{name}/u"] = u
        arrays[f"{name}/v"] = v
        arrays[f"{name}/w"] = w
        print(f"{name:28s} {msg!r}")
    np.savez_compressed(os.path.join(HERE, "invalid_trees.npz"), **arrays)
    with open(os.path.join(HERE, "invalid_trees.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

"""Generate golden vectors from the UNMODIFIED reference (dendromst 0.1.0).

Imports /root/reference/pkg/src (read-only; only available in the build
container, never on the GPU box) and records, for a corpus of small trees,
the reference's own outputs of the hot path:

  rank_edges   (tree_core.py:174-190)  -> orig_of, heights (RankedTree.w)
  pandora      (expansion.py:148-153)  -> edge_parent, vertex_parent
  build_hierarchy (contraction.py:186-219) -> retirement_level, view_kind_counts
  assign_chains   (expansion.py:97-128)    -> terminal, level

Corpus: the reference's known-answer trees (tests/test_expansion.py:23-63,
tests/test_classify.py:18-38, tests/test_tree_core.py:71-82), trees from the
reference's own generators (tests/conftest.py:18-47: star, path, caterpillar,
attach; distinct or all-equal weights; shuffled input order), signed-zero
and negative-weight cases, and small mutual-reachability MSTs
(pointgen.mutual_reachability_mst).  Output: tests/golden/golden_small.npz
(ragged arrays concatenated, with offsets).

Usage: NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import dendromst as R  # noqa: E402
from dendromst.pointgen import gen_points, mutual_reachability_mst  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def make_weights(m, rng, equal=False):          # tests/conftest.py:18-21
    if equal:
        return np.full(m, 1.0)
    return rng.permutation(m).astype(np.float64) + 1.0


def topology_edges(topology, nv, rng):          # tests/conftest.py:24-39
    v = np.arange(1, nv, dtype=np.int64)
    if topology == "star":
        u = np.zeros(nv - 1, dtype=np.int64)
    elif topology == "path":
        u = np.arange(nv - 1, dtype=np.int64)
    elif topology == "caterpillar":
        spine = max(2, nv // 2)
        u = np.concatenate([np.arange(spine - 1, dtype=np.int64), rng.integers(0, spine, nv - spine)])
    elif topology == "attach":
        u = rng.integers(0, np.maximum(v, 1))
    else:
        raise ValueError(topology)
    return u, v


def make_tree(topology, nv, rng, equal=False):  # tests/conftest.py:42-47
    u, v = topology_edges(topology, nv, rng)
    w = make_weights(nv - 1, rng, equal)
    perm = rng.permutation(nv - 1)
    return R.weighted_tree(nv, u[perm], v[perm], w[perm])


def corpus():
    trees = []
    add = lambda name, t: trees.append((name, t))
    # known-answer trees from the reference's tests
    add("kat_path_132", R.weighted_tree(4, [0, 1, 2], [1, 2, 3], [1.0, 3.0, 2.0]))
    add("kat_hub", R.weighted_tree(7, [0, 0, 0, 0, 1, 2], [1, 2, 3, 4, 5, 6],
                                  [7.0, 5.0, 4.0, 2.0, 6.0, 3.0]))
    add("kat_single_edge", R.weighted_tree(2, [0], [1], [1.0]))
    add("kat_ties_path", R.weighted_tree(4, [0, 1, 2], [1, 2, 3], [5.0, 5.0, 5.0]))
    add("kat_star12", make_tree("star", 12, np.random.default_rng(0)))
    add("kat_star65", make_tree("star", 65, np.random.default_rng(5)))
    # signed zeros / negative weights (validation only checks isfinite)
    add("signed_zero", R.weighted_tree(6, [0, 1, 2, 3, 4], [1, 2, 3, 4, 5],
                                       [0.0, -0.0, 1.0, -0.0, 0.0]))
    add("negative_mixed", R.weighted_tree(6, [0, 0, 1, 1, 2], [1, 2, 3, 4, 5],
                                          [-1.5, 2.0, -0.0, 0.0, -1.5]))
    rng = np.random.default_rng(2024)
    for topo in ("star", "path", "caterpillar", "attach"):
        for nv in (2, 3, 4, 5, 8, 17, 33, 64, 100, 257, 512, 1000):
            add(f"{topo}_{nv}", make_tree(topo, nv, rng))
        for nv in (2, 5, 64, 300):
            add(f"{topo}_{nv}_eq", make_tree(topo, nv, rng, equal=True))
    for i in range(8):
        nv = int(rng.integers(2, 600))
        u, v = topology_edges("attach", nv, rng)
        w = np.round(rng.random(nv - 1) * 8) / 8 - 0.5  # many ties, negatives, +-0
        w[rng.random(nv - 1) < 0.1] = -0.0
        perm = rng.permutation(nv - 1)
        add(f"attach_tied_{i}", R.weighted_tree(nv, u[perm], v[perm], w[perm]))
    for i, (dist, n) in enumerate([("normal", 50), ("uniform", 200), ("normal", 513), ("uniform", 1000)]):
        add(f"mreach_{dist}_{n}", mutual_reachability_mst(gen_points(dist, n, 2 + i % 2, 100 + i)))
    return trees


def main():
    cols = {k: [] for k in ("u", "v", "w", "orig_of", "heights", "edge_parent", "vertex_parent",
                            "retirement", "terminal", "level", "counts")}
    names, nvs, ns, nls = [], [], [], []
    for name, tree in corpus():
        ranked = R.rank_edges(tree)
        d = R.pandora(ranked)
        inc = R.build_incidence(ranked)
        h = R.build_hierarchy(ranked, inc)
        a = R.assign_chains(h)
        names.append(name)
        nvs.append(tree.num_vertices)
        ns.append(tree.num_edges)
        nls.append(h.num_levels)
        cols["u"].append(tree.u); cols["v"].append(tree.v); cols["w"].append(tree.w)
        cols["orig_of"].append(ranked.orig_of); cols["heights"].append(ranked.w)
        cols["edge_parent"].append(d.edge_parent); cols["vertex_parent"].append(d.vertex_parent)
        cols["retirement"].append(h.retirement_level)
        cols["terminal"].append(a.terminal); cols["level"].append(a.level)
        cols["counts"].append(np.asarray(h.view_kind_counts, dtype=np.int64).reshape(-1))
    out = {k: np.concatenate(v) for k, v in cols.items()}
    out["names"] = np.asarray(names)
    out["num_vertices"] = np.asarray(nvs, dtype=np.int64)
    out["num_edges"] = np.asarray(ns, dtype=np.int64)
    out["num_levels"] = np.asarray(nls, dtype=np.int64)
    path = os.path.join(HERE, "golden_small.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(names)} trees, {sum(ns)} edges")


if __name__ == "__main__":
    main()

"""Reference digests at the BASELINE.json config sizes.

Runs the UNMODIFIED reference (imported from /root/reference/pkg/src) exactly
as `dendromst build` scopes it (cli.py:82-85): rank_edges (tree_core.py:174-190)
then pandora's composition (expansion.py:148-153: build_incidence,
vertex_parents, build_hierarchy, assign_chains, stitch_chains -- spelled out
so the hierarchy's view_kind_counts come from the same run).  The inputs are
trees by construction (paper_2401_06089_b200.synth), so WeightedTree is built
directly; validation (weighted_tree, 357 s at 128M) is the caller's
precondition and is pinned separately (invalid_trees.*).

For every case it records sha256 digests of the reference outputs as the
device produces them (int32 orig_of / edge_parent / vertex_parent, float64
heights = w by rank), the per-view kind counts, the level count, the input
digest (so the GPU box can assert it regenerated the same input) and the
reference's own wall time on this container (informational only).

Output: tests/golden/ref_digests/<case>.json (one file per case).
Usage:
  NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_digests.py CASE [CASE ...]
  cases: config4_tied config4_uniform random16M path16M caterpillar16M
         config2 config5_<seed> (8M, uniform, seed 0..63)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import dendromst as R  # noqa: E402
from dendromst.classify import vertex_parents  # noqa: E402
from dendromst.expansion import assign_chains, stitch_chains  # noqa: E402
from paper_2401_06089_b200 import synth  # noqa: E402


def case_input(name):
    if name == "config4_tied":
        return synth.random_attach(128_000_000, seed=0, tied=True), dict(gen="tied", n=128_000_000, seed=0)
    if name == "config4_uniform":
        return synth.random_attach(128_000_000, seed=0), dict(gen="random", n=128_000_000, seed=0)
    if name == "random16M":
        return synth.random_attach(16_000_000, seed=0), dict(gen="random", n=16_000_000, seed=0)
    if name == "path16M":
        return synth.path(16_000_000, seed=0), dict(gen="path", n=16_000_000, seed=0)
    if name == "caterpillar16M":
        return synth.caterpillar(16_000_000, seed=0), dict(gen="caterpillar", n=16_000_000, seed=0)
    if name == "config2":
        return synth.blobs1m(), dict(gen="blobs1m", n=999_999, seed=0)
    if name.startswith("config5_"):
        sd = int(name.split("_")[1])
        return synth.random_attach(8_000_000, seed=sd), dict(gen="random", n=8_000_000, seed=sd)
    raise SystemExit(f"unknown case {name}")


def sha(a, dtype):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a).astype(dtype)).tobytes()).hexdigest()


def run(name):
    (nv, u, v, w), meta = case_input(name)
    digest_in = synth.input_digest(u, v, w)
    n = u.shape[0]
    tree = R.WeightedTree(nv, np.asarray(u, np.int64), np.asarray(v, np.int64), np.asarray(w, np.float64),
                          np.arange(n, dtype=np.int64))
    del u, v, w
    t0 = time.perf_counter()
    ranked = R.rank_edges(tree)
    t1 = time.perf_counter()
    inc = R.build_incidence(ranked)
    vp = vertex_parents(inc)
    h = R.build_hierarchy(ranked, inc)
    d = stitch_chains(assign_chains(h), vp)
    t2 = time.perf_counter()
    out = dict(case=name, **meta, num_vertices=int(nv), input_digest=digest_in,
               orig_of=sha(ranked.orig_of, np.int32), heights=sha(ranked.w, np.float64),
               edge_parent=sha(d.edge_parent, np.int32), vertex_parent=sha(d.vertex_parent, np.int32),
               view_kind_counts=[[int(x) for x in c] for c in h.view_kind_counts],
               num_levels=int(h.num_levels),
               reference_seconds=dict(rank_edges=round(t1 - t0, 2), pandora=round(t2 - t1, 2),
                                      where="build container (8 vCPU Xeon, 1 core used), not the B200 host"))
    os.makedirs(os.path.join(HERE, "ref_digests"), exist_ok=True)
    with open(os.path.join(HERE, "ref_digests", f"{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(name, "levels", h.num_levels, f"rank {t1 - t0:.1f}s pandora {t2 - t1:.1f}s", flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:]:
        run(c)

"""Config-1 golden (BASELINE.json configs[0]): the reference's own
rank_edges + pandora on the random-attachment tree n = 100,000,
w = rng.random, seed 0 (paper_2401_06089_b200.synth.random_attach).

Stores the reference outputs (int32) plus an input checksum so the GPU-box
test can assert it regenerated the same input.
Usage: NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_config1.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import dendromst as R  # noqa: E402
from paper_2401_06089_b200 import synth  # noqa: E402


def main():
    nv, u, v, w = synth.random_attach(100_000, seed=0)
    tree = R.weighted_tree(nv, u, v, w)
    ranked = R.rank_edges(tree)
    d = R.pandora(ranked)
    h = R.build_hierarchy(ranked, R.build_incidence(ranked))
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config1_100k.npz")
    np.savez_compressed(out, orig_of=ranked.orig_of.astype(np.int32),
                        edge_parent=d.edge_parent.astype(np.int32),
                        vertex_parent=d.vertex_parent.astype(np.int32),
                        counts=np.asarray(h.view_kind_counts, dtype=np.int64),
                        digest=np.asarray(synth.input_digest(u, v, w)))
    print("wrote", out, "levels", h.num_levels)


if __name__ == "__main__":
    main()

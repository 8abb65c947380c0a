"""Golden `dendromst stats` reports (cli.py:97-135) computed by the
unmodified reference for seeded synthetic trees (inputs regenerated from
paper_2401_06089_b200.synth, so only the reports are stored).

    NUMBA_CACHE_DIR=/tmp/nb PYTHONPATH=/root/reference/pkg/src python tests/golden/make_stats.py
"""
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("DENDROMST_SRC", "/root/reference/pkg/src"))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from dendromst.analysis import dendrogram_height, level_stats  # noqa: E402
from dendromst.classify import vertex_parents  # noqa: E402
from dendromst.contraction import build_hierarchy  # noqa: E402
from dendromst.expansion import assign_chains, stitch_chains  # noqa: E402
from dendromst.tree_core import build_incidence, rank_edges, weighted_tree  # noqa: E402

from paper_2401_06089_b200 import synth  # noqa: E402

CASES = [("random", 1000, 1), ("tied", 1000, 2), ("path", 1000, 3), ("caterpillar", 1000, 4),
         ("random", 20000, 5), ("tied", 20000, 6), ("caterpillar", 20000, 7), ("random", 100000, 8)]


def report(nv, u, v, w):
    ranked = rank_edges(weighted_tree(nv, u, v, w))          # cli.py:98 (_load_ranked)
    inc = build_incidence(ranked)                             # :99
    hierarchy = build_hierarchy(ranked, inc)                  # :100
    assignment = assign_chains(hierarchy)                     # :101
    dendrogram = stitch_chains(assignment, vertex_parents(inc))  # :108
    n = ranked.num_edges
    height = dendrogram_height(dendrogram)                    # :110
    per_level = level_stats(hierarchy)                        # :111
    return {"edges": n, "vertices": ranked.num_vertices, "levels": hierarchy.num_levels, "height": height,
            "chains": assignment.num_chains(),
            "skewness_log2_edges": height / math.log2(n) if n >= 2 else 0.0,
            "skewness_log2_points": height / math.log2(n + 1),
            "per_level": [list(map(int, c)) for c in per_level]}


def main():
    out = []
    for shape, n, seed in CASES:
        nv, u, v, w = synth.GENERATORS[shape](n, seed=seed)
        r = report(nv, u.astype(np.int64), v.astype(np.int64), w)
        out.append({"shape": shape, "n": n, "seed": seed, "report": r})
        print(shape, n, seed, r["height"], r["chains"], r["levels"])
    with open(os.path.join(HERE, "stats_golden.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

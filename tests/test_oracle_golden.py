"""Pin the CPU oracle (oracle/dendro_oracle.py) to the reference.

Golden vectors were produced by the unmodified reference
(tests/golden/make_golden.py); the explicit known-answer tests restate the
reference's own tests (file:line cited per test).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import dendro_oracle as O
from tests.conftest import TOPOLOGIES, golden_trees, make_tree

GOLDEN = list(golden_trees())


@pytest.mark.parametrize("t", GOLDEN, ids=[t["name"] for t in GOLDEN])
def test_oracle_matches_reference_golden(t):
    res = O.build(t["num_vertices"], t["u"], t["v"], t["w"])
    assert np.array_equal(res.orig_of, t["orig_of"])
    assert np.array_equal(res.heights.view(np.uint64), t["heights"].view(np.uint64))
    assert np.array_equal(res.edge_parent, t["edge_parent"])
    assert np.array_equal(res.vertex_parent, t["vertex_parent"])
    assert res.num_levels == t["num_levels"]
    assert res.view_kind_counts == t["counts"]
    assert np.array_equal(res.hierarchy.retirement_level, t["retirement"])
    chains = O.assign_chains(res.hierarchy)
    assert np.array_equal(chains.terminal, t["terminal"])
    assert np.array_equal(chains.level, t["level"])


def test_kat_path_example():
    # tests/test_expansion.py:23-47, tests/test_contraction.py:75-86, tests/test_classify.py:31-38
    r = O.rank_edges(4, [0, 1, 2], [1, 2, 3], [1.0, 3.0, 2.0])
    assert r.rank_of.tolist() == [2, 0, 1] and r.orig_of.tolist() == [1, 2, 0]
    ep, vp, h = O.pandora(r)
    assert ep.tolist() == [O.ROOT, 0, 0] and vp.tolist() == [2, 2, 1, 1]
    assert h.retirement_level.tolist() == [1, 0, 0]
    assert h.view_kind_counts == [(1, 2, 0, 3), (0, 1, 0, 1)]
    assert h.levels[0].vertex_map.tolist() == [0, 0, 1, 1]
    assert h.levels[0].super_max_incident.tolist() == [0, 0]
    c = O.assign_chains(h)
    assert c.terminal.tolist() == [O.ROOT, 0, 0]
    assert c.anchor.tolist() == [0, 1, 0] and c.level.tolist() == [0, 1, 1]


def test_kat_ties_by_original_id():
    # tests/test_tree_core.py:79-82
    r = O.rank_edges(4, [0, 1, 2], [1, 2, 3], [5.0, 5.0, 5.0])
    assert r.rank_of.tolist() == [0, 1, 2]


def test_kat_hub_vertex_parent():
    # tests/test_classify.py:18-28
    r = O.rank_edges(7, [0, 0, 0, 0, 1, 2], [1, 2, 3, 4, 5, 6], [7.0, 5.0, 4.0, 2.0, 6.0, 3.0])
    _, vp, _ = O.pandora(r)
    assert int(vp[0]) == 5


def test_kat_star_single_chain():
    # tests/test_expansion.py:50-57, tests/test_acceptance.py:248-259
    nv, u, v, w = make_tree("star", 12, np.random.default_rng(0))
    ep, _, _ = O.pandora(O.rank_edges(nv, u, v, w))
    assert ep.tolist() == [O.ROOT] + list(range(nv - 2))


def test_kat_single_edge():
    # tests/test_expansion.py:60-63
    ep, vp, _ = O.pandora(O.rank_edges(2, [0], [1], [1.0]))
    assert ep.tolist() == [O.ROOT] and vp.tolist() == [0, 0]


def test_component_labels_canonical():
    # tests/test_contraction.py:56-62
    assert O.component_labels(6, np.array([0, 4]), np.array([1, 5])).tolist() == [0, 0, 1, 2, 3, 3]
    assert O.component_labels(3, np.array([], dtype=np.int64),
                              np.array([], dtype=np.int64)).tolist() == [0, 1, 2]


def test_signed_zero_ties_with_positive_zero():
    # numpy semantics (-0.0 == +0.0) pinned: SURVEY.md §8c "parity unpinned by reference tests"
    r = O.rank_edges(4, [0, 1, 2], [1, 2, 3], [-0.0, 0.0, -0.0])
    assert r.orig_of.tolist() == [0, 1, 2]
    assert np.signbit(r.w).tolist() == [True, False, True]


@pytest.mark.parametrize("topology", TOPOLOGIES)
@pytest.mark.parametrize("equal", [False, True])
def test_oracle_equals_sequential_bottom_up(topology, equal):
    # tests/test_expansion.py:65-70, tests/test_acceptance.py:123-145 (criterion 1)
    rng = np.random.default_rng(17)
    for nv in (2, 3, 9, 50, 200):
        nv, u, v, w = make_tree(topology, nv, rng, equal)
        r = O.rank_edges(nv, u, v, w)
        ep, vp, _ = O.pandora(r)
        bep, bvp = O.dendrogram_bottom_up(r)
        assert np.array_equal(ep, bep) and np.array_equal(vp, bvp)

"""GPU parity: the CUDA path (through the C ABI) vs the reference.

Small and medium trees: bit-exact equality with the reference's golden
vectors (tests/golden/, produced by the unmodified reference) and with the
CPU oracle (oracle/dendro_oracle.py, itself pinned to those goldens).
Full sizes (BASELINE.json configs 3 and 4): size-independent properties of a
single-linkage dendrogram plus agreement with the oracle on prefixes the
oracle finishes in seconds.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import dendro_oracle as O
from paper_2401_06089_b200 import synth
from tests.conftest import TOPOLOGIES, golden_trees, has_gpu, make_tree

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

GOLDEN = list(golden_trees())
ROOT_DIR = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def builder():
    from paper_2401_06089_b200.build import build
    from paper_2401_06089_b200 import DendrogramBuilder
    build()
    return DendrogramBuilder("cuda:0")


def _np(t):
    return t.cpu().numpy()


def assert_matches(res, orig_of, heights, edge_parent, vertex_parent, counts=None):
    assert np.array_equal(_np(res.orig_of), orig_of)
    assert np.array_equal(_np(res.heights).view(np.uint64), np.asarray(heights).view(np.uint64))
    assert np.array_equal(_np(res.edge_parent), edge_parent)
    assert np.array_equal(_np(res.vertex_parent), vertex_parent)
    if counts is not None:
        assert res.view_kind_counts == list(counts)


@pytest.mark.parametrize("t", GOLDEN, ids=[t["name"] for t in GOLDEN])
def test_golden_corpus(builder, t):
    res = builder.build(t["num_vertices"], t["u"], t["v"], t["w"], debug=True)
    assert_matches(res, t["orig_of"], t["heights"], t["edge_parent"], t["vertex_parent"], t["counts"])
    assert res.num_levels == t["num_levels"]
    # per-stage parity: ContractionHierarchy.retirement_level, ChainAssignment.terminal/.level
    assert np.array_equal(_np(res.debug["retirement"]).astype(np.int64), t["retirement"])
    assert np.array_equal(_np(res.debug["chain_terminal"]), t["terminal"])
    assert np.array_equal(_np(res.debug["chain_level"]), t["level"])


@pytest.mark.parametrize("topology", TOPOLOGIES)
@pytest.mark.parametrize("equal", [False, True])
def test_reference_generators_vs_oracle(builder, topology, equal):
    # tests/conftest.py generators, many sizes incl. the smallest
    rng = np.random.default_rng(1000 + TOPOLOGIES.index(topology) + 10 * equal)
    for nv in [2, 3, 4, 5, 7, 16, 31, 32, 33, 100, 255, 256, 257, 1000, 4097, 20000]:
        nv, u, v, w = make_tree(topology, nv, rng, equal)
        exp = O.build(nv, u, v, w)
        res = builder.build(nv, u, v, w)
        assert_matches(res, exp.orig_of, exp.heights, exp.edge_parent, exp.vertex_parent,
                       exp.view_kind_counts)


@pytest.mark.parametrize("shape", ["random", "tied", "path", "caterpillar"])
@pytest.mark.parametrize("n", [1, 2, 1000, 4095, 4096, 4097, 65537, 300_000])
def test_synthetic_shapes_vs_oracle(builder, shape, n):
    nv, u, v, w = synth.GENERATORS[shape](n, seed=n)
    exp = O.build(nv, u, v, w)
    res = builder.build(nv, u, v, w)
    assert_matches(res, exp.orig_of, exp.heights, exp.edge_parent, exp.vertex_parent,
                   exp.view_kind_counts)


def test_heavy_ties_negative_and_signed_zero(builder):
    rng = np.random.default_rng(7)
    for n in (10, 1000, 100_000):
        nv, u, v, _ = synth.random_attach(n, seed=n)
        w = rng.integers(-3, 4, n).astype(np.float64)
        w[w == 0] = np.where(rng.random(int((w == 0).sum())) < 0.5, -0.0, 0.0)
        exp = O.build(nv, u, v, w)
        res = builder.build(nv, u, v, w)
        assert_matches(res, exp.orig_of, exp.heights, exp.edge_parent, exp.vertex_parent)


def _compaction_weights(kind, n, rng):
    """Weight sets that exercise the edge sort's top-field compaction (few
    distinct sign + exponent fields): rare outliers the key sample misses,
    both signs, signed zeros, subnormals, and more fields than a code holds."""
    if kind == "int4096":                      # config 4's weights
        return rng.integers(0, 4096, n).astype(np.float64)
    if kind == "rare_outliers":                # [1, 2) plus a handful far away
        w = 1.0 + rng.random(n)
        idx = rng.choice(n, 5, replace=False)
        w[idx] = [1e-200, -1e300, 5e-324, -0.0, 3e250]
        return w
    if kind == "signed_scaled":                # +-k * 2^e over 6 exponents
        return rng.choice([-1.0, 1.0], n) * rng.integers(1, 64, n) * np.exp2(rng.integers(-3, 3, n))
    if kind == "many_fields":                  # > 256 exponents: no compaction
        return np.exp2(rng.integers(-400, 400, n).astype(np.float64)) * (1 + rng.integers(0, 8, n) / 8)
    if kind == "one_field":                    # all in [1, 2): nothing to compact
        return 1.0 + rng.integers(0, 1 << 20, n) / float(1 << 20)
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["int4096", "rare_outliers", "signed_scaled", "many_fields", "one_field"])
@pytest.mark.parametrize("n", [1000, 600_000])
def test_sort_key_compaction_vs_oracle(builder, kind, n):
    rng = np.random.default_rng(n + len(kind))
    nv, u, v, _ = synth.random_attach(n, seed=11)
    w = _compaction_weights(kind, n, rng)
    exp = O.build(nv, u, v, w)
    res = builder.build(nv, u, v, w)
    assert_matches(res, exp.orig_of, exp.heights, exp.edge_parent, exp.vertex_parent)
    orig_of, heights, _, _ = builder.rank_edges(nv, u, v, w)
    assert np.array_equal(_np(orig_of), exp.orig_of)
    assert np.array_equal(_np(heights).view(np.uint64), np.asarray(exp.heights).view(np.uint64))


def test_reversed_path_orientation(builder):
    # deep in-trees pointing to HIGHER vertex ids (the pointer-jumping worst case)
    n = 200_000
    u = np.arange(n)
    nv, uu, vv, w = n + 1, u, u + 1, (n - u).astype(np.float64)
    perm = np.random.default_rng(3).permutation(n)
    exp = O.build(nv, uu[perm], vv[perm], w[perm])
    res = builder.build(nv, uu[perm], vv[perm], w[perm])
    assert_matches(res, exp.orig_of, exp.heights, exp.edge_parent, exp.vertex_parent)


def test_permuted_vertex_ids(builder):
    # relabelled vertices: random-access pointer chains (tests/test_tree_core.py:118-124 spirit)
    rng = np.random.default_rng(11)
    for shape in ("path", "caterpillar", "random"):
        nv, u, v, w = synth.GENERATORS[shape](100_000, seed=5)
        relabel = rng.permutation(nv).astype(np.int32)
        u, v = relabel[u], relabel[v]
        exp = O.build(nv, u, v, w)
        res = builder.build(nv, u, v, w)
        assert_matches(res, exp.orig_of, exp.heights, exp.edge_parent, exp.vertex_parent)


def test_config1_reference_golden(builder):
    # BASELINE.json configs[0]: random tree n=100k, uniform weights, seed 0
    g = np.load(os.path.join(ROOT_DIR, "tests", "golden", "config1_100k.npz"))
    nv, u, v, w = synth.random_attach(100_000, seed=0)
    assert synth.input_digest(u, v, w) == str(g["digest"])
    res = builder.build(nv, u, v, w)
    assert np.array_equal(_np(res.orig_of), g["orig_of"])
    assert np.array_equal(_np(res.edge_parent), g["edge_parent"])
    assert np.array_equal(_np(res.vertex_parent), g["vertex_parent"])
    assert res.view_kind_counts == [tuple(c) for c in g["counts"].tolist()]


def test_config2_mreach_blobs(builder):
    # BASELINE.json configs[1]: reference-computed MST of 1M 3-D blob points
    path = os.path.join(ROOT_DIR, "tests", "golden", "config2_blobs1m.npz")
    if not os.path.exists(path):
        pytest.skip("config-2 fixture not generated yet (tests/golden/make_config2.py)")
    g = np.load(path)
    nv, u, v, w = int(g["num_vertices"]), g["u"], g["v"], g["w"]
    exp = O.build(nv, u, v, w)
    res = builder.build(nv, u, v, w)
    assert_matches(res, exp.orig_of, exp.heights, exp.edge_parent, exp.vertex_parent,
                   exp.view_kind_counts)


def test_split_entry_points_equal_fused(builder):
    nv, u, v, w = synth.random_attach(50_000, seed=9, tied=True)
    fused = builder.build(nv, u, v, w)
    orig_of, heights, ru, rv = builder.rank_edges(nv, u, v, w)
    assert np.array_equal(_np(orig_of), _np(fused.orig_of))
    assert np.array_equal(_np(heights).view(np.uint64), _np(fused.heights).view(np.uint64))
    exp = O.rank_edges(nv, u, v, w)
    assert np.array_equal(_np(ru), exp.u) and np.array_equal(_np(rv), exp.v)
    ep, vp, st = builder.pandora(nv, ru, rv)
    assert np.array_equal(_np(ep), _np(fused.edge_parent))
    assert np.array_equal(_np(vp), _np(fused.vertex_parent))
    assert st.view_kind_counts() == fused.view_kind_counts


@pytest.mark.parametrize("shape,n", [("tied", 1), ("random", 5000), ("tied", 300_000), ("path", 70_000)])
def test_host_buffer_entry_point(builder, shape, n):
    # dmst_build_host: host inputs/outputs, copies overlapped with the pipeline
    import torch
    from paper_2401_06089_b200 import HostBuildResult
    nv, u, v, w = synth.GENERATORS[shape](n, seed=7)
    exp = O.build(nv, u, v, w)
    for pinned in (True, False):
        out = HostBuildResult.empty(n, nv, pin=pinned)
        hu, hv, hw = (torch.from_numpy(x) for x in (u, v, w))
        if pinned:
            hu, hv, hw = hu.pin_memory(), hv.pin_memory(), hw.pin_memory()
        res = builder.build_host(nv, hu, hv, hw, out=out)
        assert_matches(res, exp.orig_of, exp.heights, exp.edge_parent, exp.vertex_parent)
        assert res.stats.view_kind_counts() == list(exp.view_kind_counts)


def _stress_tree(kind: str, n: int, seed: int):
    """Shapes that stress the bucketed / chased / sorted stages at scale."""
    rng = np.random.default_rng(seed)
    nv = n + 1
    ids = rng.permutation(nv).astype(np.int64)          # scatter vertex ids
    child = np.arange(1, nv, dtype=np.int64)
    if kind == "star":                                  # one hub: every record in one vertex bucket
        par = np.zeros(n, np.int64)
    elif kind == "hubs":                                # 16 hubs
        par = rng.integers(0, np.minimum(child, 16))
    elif kind == "binary":                              # balanced binary tree
        par = (child - 1) // 2
    elif kind == "broom":                               # long handle + bristles
        h = nv // 2
        par = np.where(child < h, child - 1, rng.integers(h - 64, h, n))
    else:                                               # random attachment
        par = rng.integers(0, child)
    u, v = ids[par], ids[child]
    if kind in ("binary", "star"):
        w = rng.integers(0, 7, n).astype(np.float64)      # heavy ties
    elif kind == "equal":
        w = np.full(n, 2.5)
    else:
        w = rng.random(n)
    perm = rng.permutation(n)
    return nv, u[perm].astype(np.int32), v[perm].astype(np.int32), w[perm]


@pytest.mark.parametrize("kind", ["star", "hubs", "binary", "broom", "equal"])
def test_stress_shapes_vs_oracle(builder, kind):
    nv, u, v, w = _stress_tree(kind, 1_500_000, seed=11)
    exp = O.build(nv, u, v, w)
    res = builder.build(nv, u, v, w)
    assert_matches(res, exp.orig_of, exp.heights, exp.edge_parent, exp.vertex_parent,
                   exp.view_kind_counts)


def test_drop_in_functions():
    from paper_2401_06089_b200 import pandora_b200, rank_edges_b200, Dendrogram
    from types import SimpleNamespace
    nv, u, v, w = make_tree("attach", 500, np.random.default_rng(4))
    tree = SimpleNamespace(num_vertices=nv, u=u, v=v, w=w)
    ranked = rank_edges_b200(tree)
    exp = O.rank_edges(nv, u, v, w)
    assert np.array_equal(ranked.orig_of, exp.orig_of) and np.array_equal(ranked.rank_of, exp.rank_of)
    assert np.array_equal(ranked.u, exp.u) and np.array_equal(ranked.w, exp.w)
    d = pandora_b200(ranked)
    ep, vp, _ = O.pandora(exp)
    assert d == Dendrogram(ep, vp)
    assert d.edge_parent.dtype == np.int64


def test_register_algorithm_into_registry():
    from paper_2401_06089_b200 import pandora_b200, register_algorithm
    reg = {"pandora": None}
    register_algorithm(reg)
    assert reg["pandora_b200"] is pandora_b200


def test_deterministic_across_runs(builder):
    nv, u, v, w = synth.random_attach(1_000_000, seed=3, tied=True)
    a = builder.build(nv, u, v, w)
    a = [x.clone() for x in (a.orig_of, a.heights, a.edge_parent, a.vertex_parent)]
    b = builder.build(nv, u, v, w)
    for x, y in zip(a, (b.orig_of, b.heights, b.edge_parent, b.vertex_parent)):
        assert bool((x == y).all())


def test_invalid_input_raises(builder):
    with pytest.raises(ValueError):
        builder.build(5, np.zeros(3, np.int32), np.ones(3, np.int32), np.ones(3))


# ------------------------------------------------------------- full sizes

def check_dendrogram_properties(nv, u, v, w, res):
    """Size-independent properties, on the device (torch), of the outputs of
    rank_edges + pandora (criteria 4/5 of tests/test_acceptance.py:163-197)."""
    import torch
    dev = res.orig_of.device
    n = res.orig_of.shape[0]
    ut = torch.from_numpy(np.asarray(u, np.int64)).to(dev)
    vt = torch.from_numpy(np.asarray(v, np.int64)).to(dev)
    wt = torch.from_numpy(np.asarray(w, np.float64)).to(dev)
    orig = res.orig_of.long()
    # orig_of is a permutation
    seen = torch.zeros(n, dtype=torch.int32, device=dev)
    seen.index_add_(0, orig, torch.ones(n, dtype=torch.int32, device=dev))
    assert bool((seen == 1).all())
    # heights = w[orig_of] bitwise; non-increasing; ties by ascending original id
    h = res.heights
    assert bool((h.view(torch.int64) == wt[orig].view(torch.int64)).all())
    assert bool((h[1:] <= h[:-1]).all())
    tie = h[1:] == h[:-1]
    assert bool((orig[1:][tie] > orig[:-1][tie]).all())
    # vertex_parent = largest incident rank
    ranks = torch.arange(n, device=dev)
    ru, rv = ut[orig], vt[orig]
    mi = torch.full((nv,), -1, dtype=torch.int64, device=dev)
    mi.scatter_reduce_(0, ru, ranks, reduce="amax")
    mi.scatter_reduce_(0, rv, ranks, reduce="amax")
    assert bool((res.vertex_parent.long() == mi).all())
    # edge_parent: root at rank 0, parents heavier, every edge node binary
    ep = res.edge_parent.long()
    assert int(ep[0]) == -1
    assert bool((ep[1:] >= 0).all()) and bool((ep[1:] < ranks[1:]).all())
    children = torch.zeros(n, dtype=torch.int64, device=dev)
    children.index_add_(0, ep[1:], torch.ones(n - 1, dtype=torch.int64, device=dev))
    children.index_add_(0, mi, torch.ones(nv, dtype=torch.int64, device=dev))
    assert bool((children == 2).all())
    # kind-count identities per view (classify.py, criterion 4)
    for a, l, c, s in res.view_kind_counts:
        if s:
            assert a + l + c == s and a == l - 1 and 2 * a <= s


@pytest.mark.parametrize("shape", ["path", "caterpillar", "random"])
def test_config3_skewed_16M(builder, shape):
    # BASELINE.json configs[2]: maximally skewed chain/caterpillar, n = 16M
    n = 16_000_000
    nv, u, v, w = synth.GENERATORS[shape](n, seed=0)
    res = builder.build(nv, u, v, w)
    check_dendrogram_properties(nv, u, v, w, res)
    if shape != "random":
        ep = _np(res.edge_parent)
        assert np.array_equal(ep, np.arange(-1, n - 1))  # a single sorted root chain
        assert res.num_levels == 1


@pytest.mark.parametrize("tied", [True, False])
def test_config4_128M(builder, tied):
    # BASELINE.json configs[3]: random tree n = 128M with tied weights (+ untied companion)
    n = 128_000_000
    nv, u, v, w = synth.random_attach(n, seed=0, tied=tied)
    res = builder.build(nv, u, v, w)
    check_dendrogram_properties(nv, u, v, w, res)
    a = [x.clone() for x in (res.orig_of, res.edge_parent, res.vertex_parent)]
    res2 = builder.build(nv, u, v, w)
    for x, y in zip(a, (res2.orig_of, res2.edge_parent, res2.vertex_parent)):
        assert bool((x == y).all())

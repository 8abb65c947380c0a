"""GPU parity of every size-gated code path, forced at sizes the oracle checks.

A 128M-edge build takes paths a small tree never reaches by default: views
>= 1 too big for the cooperative tail (host level loop: k_v1, stride-2 k_v2 +
k_jump, k_select_edges with direct or bucketed maxIncident), bucketed
maxIncident on views >= 1, the 256 x 20 chain-sort geometry, wide (64-bit)
edge-sort keys without top-field compaction.  dmst_stats' path fields
(include/dmst.h) force each of them per call, so the reference's 84-tree
golden corpus, its generators, the synthetic config shapes and the 1.5M
stress shapes run bit-exact through every combination.  Reference:
build_hierarchy / contract_level / view_max_incident (contraction.py:149-219),
assign_chains / stitch_chains (expansion.py:97-145), rank_edges
(tree_core.py:174-190) -- paths under /root/reference/pkg/src/dendromst/.

The last test asserts that every kernel kind the library has launched inside
a bit-exact comparison of this module (accumulated from the per-call
kernel profiles), i.e. no kernel on the 128M path goes unchecked.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import dendro_oracle as O
from paper_2401_06089_b200 import synth
from tests.conftest import TOPOLOGIES, golden_trees, has_gpu, make_tree
from tests.test_parity_gpu import _stress_tree

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

# name -> dmst_stats path overrides
PATHS = {
    "default": {},
    # host level loop for every view; views >= 1 whose mi64 <= 64 MB direct
    "no_tail": {"tail_edges": -1},
    # every view >= 1 bucketed (multisplit + shared-memory apply); no tail
    "bucketed": {"direct_mi_bytes": -1},
    # host loop down to tiny views, then the tail; views of <= 2048 vertices direct
    "late_tail": {"tail_edges": 64, "direct_mi_bytes": 16384},
    # wide 64-bit edge-sort keys, no compaction; 256 x 20 chain-sort tiles
    "wide_sort_large_s2": {"sort1_mode": 3, "sort2_geometry": 2},
    # narrow keys without compaction; 512 x 16 chain-sort tiles; no tail, bucketed
    "nocompact_bucketed": {"sort1_mode": 2, "sort2_geometry": 1, "direct_mi_bytes": -1, "tail_edges": -1},
    # wide keys always sorted by the full LSD (no shared-memory finish)
    "no_local": {"sort1_mode": 4},
    # bucketed maxIncident by 4M-vertex slices + L2 atomics on every view >= 0; no tail
    "sliced": {"mi_apply_mode": 2, "direct_mi_bytes": -1, "tail_edges": -1},
    # the shared-memory apply forced
    "smem_apply": {"mi_apply_mode": 1},
    # view 0's labels: always V2 + vertex map / always chased in the select (long
    # chases deferred to k_select_fix after V2 + pointer jumping); no tail
    "v0_vertex_map": {"v0_select": 1},
    "v0_chase": {"v0_select": 2, "tail_edges": -1},
}

SEEN_KINDS: dict[str, int] = {}   # kernel kind -> launches inside checked builds


@pytest.fixture(scope="module")
def builder():
    from paper_2401_06089_b200.build import build
    from paper_2401_06089_b200 import DendrogramBuilder
    build()
    return DendrogramBuilder("cuda:0")


def _np(t):
    return t.cpu().numpy()


def _oracle_full(nv, u, v, w):
    """Oracle outputs plus the per-stage arrays the debug entry point exposes."""
    r = O.rank_edges(nv, u, v, w)
    ep, vp, h = O.pandora(r)
    ch = O.assign_chains(h)
    return dict(orig_of=r.orig_of, heights=r.w, edge_parent=ep, vertex_parent=vp,
                counts=list(h.view_kind_counts), levels=h.num_levels,
                retirement=h.retirement_level, terminal=ch.terminal, level=ch.level)


def _check(builder, nv, u, v, w, exp, paths, debug=True):
    res = builder.build(nv, u, v, w, paths=PATHS[paths], debug=debug, profile=True)
    assert np.array_equal(_np(res.orig_of), exp["orig_of"])
    assert np.array_equal(_np(res.heights).view(np.uint64), np.asarray(exp["heights"]).view(np.uint64))
    assert np.array_equal(_np(res.edge_parent), exp["edge_parent"])
    assert np.array_equal(_np(res.vertex_parent), exp["vertex_parent"])
    assert res.view_kind_counts == [tuple(c) for c in exp["counts"]]
    assert res.num_levels == exp["levels"]
    if debug:
        assert np.array_equal(_np(res.debug["retirement"]).astype(np.int64), exp["retirement"])
        assert np.array_equal(_np(res.debug["chain_terminal"]), exp["terminal"])
        assert np.array_equal(_np(res.debug["chain_level"]), exp["level"])
    for k, (_, calls) in res.stats.kernel_profile().items():
        SEEN_KINDS[k] = SEEN_KINDS.get(k, 0) + calls
    return res


def _assert_path_taken(res, paths):
    """The override really changed the path (when the tree has the views for it)."""
    info = res.stats.path_info()
    L = res.num_levels
    views = [c[3] for c in res.view_kind_counts]
    has_later = [k for k in range(1, L + 1) if views[k] > 0]
    p = PATHS[paths]
    if p.get("tail_edges") == -1:
        assert info["tail_level"] == -1
    if p.get("direct_mi_bytes") == -1:
        assert not info["mi_direct_views"]
        assert set(has_later) <= set(info["mi_bucketed_views"])
        # the tail needs a direct view: only an edgeless last view can reach it
        assert info["tail_level"] == -1 or views[info["tail_level"]] == 0
    if p.get("sort1_mode", 0) & 1:
        assert not info["sort1_narrow"]
    if p.get("sort1_mode", 0) & 2:
        assert not info["sort1_compacted"]
    if p.get("sort1_mode", 0) & 4:
        assert info["sort1_local"] is None
    if p.get("mi_apply_mode") == 2:
        assert info["mi_sliced"]
    if p.get("mi_apply_mode") == 1:
        assert not info["mi_sliced"]
    if p.get("v0_select") == 1:
        assert info["v0_chase"] is None
    if p.get("v0_select") == 2:
        assert info["v0_chase"] in ("chase", "chase+fix")
    if p.get("sort2_geometry") and info["sort2_passes"]:
        from paper_2401_06089_b200._lib import SORT2_GEOMETRIES
        assert info["sort2_geometry"] == SORT2_GEOMETRIES[p["sort2_geometry"]]


GOLDEN = list(golden_trees())


@pytest.mark.parametrize("paths", [p for p in PATHS if p != "default"])
def test_golden_corpus_all_paths(builder, paths):
    # the unmodified reference's outputs (tests/golden/make_golden.py), per-stage arrays included
    for t in GOLDEN:
        exp = dict(orig_of=t["orig_of"], heights=t["heights"], edge_parent=t["edge_parent"],
                   vertex_parent=t["vertex_parent"], counts=t["counts"], levels=t["num_levels"],
                   retirement=t["retirement"], terminal=t["terminal"], level=t["level"])
        res = _check(builder, t["num_vertices"], t["u"], t["v"], t["w"], exp, paths)
        _assert_path_taken(res, paths)


@pytest.mark.parametrize("paths", list(PATHS))
@pytest.mark.parametrize("topology", TOPOLOGIES)
def test_reference_generators_all_paths(builder, paths, topology):
    rng = np.random.default_rng(77 + TOPOLOGIES.index(topology))
    for nv in [2, 3, 17, 257, 4097, 60_000]:
        for equal in (False, True):
            nv2, u, v, w = make_tree(topology, nv, rng, equal)
            _check(builder, nv2, u, v, w, _oracle_full(nv2, u, v, w), paths)


@pytest.mark.parametrize("paths", list(PATHS))
@pytest.mark.parametrize("shape", ["random", "tied", "path", "caterpillar"])
def test_synthetic_shapes_all_paths(builder, paths, shape):
    for n in (5000, 400_000):
        nv, u, v, w = synth.GENERATORS[shape](n, seed=n + 1)
        res = _check(builder, nv, u, v, w, _oracle_full(nv, u, v, w), paths)
        _assert_path_taken(res, paths)


@pytest.mark.parametrize("paths", [p for p in PATHS if p != "default"])
@pytest.mark.parametrize("kind", ["star", "hubs", "binary", "broom", "equal", "random"])
def test_stress_shapes_all_paths(builder, paths, kind):
    nv, u, v, w = _stress_tree(kind, 1_500_000, seed=12)
    res = _check(builder, nv, u, v, w, _oracle_full(nv, u, v, w), paths, debug=False)
    _assert_path_taken(res, paths)


@pytest.mark.parametrize("paths", ["no_tail", "bucketed", "late_tail", "v0_chase"])
def test_deep_in_trees_all_paths(builder, paths):
    # reversed path (in-trees towards higher ids: pointer jumping on every view)
    # and relabelled vertex ids (random-access chases) through the host loop
    n = 200_000
    a = np.arange(n)
    perm = np.random.default_rng(5).permutation(n)
    nv, u, v, w = n + 1, a[perm], a[perm] + 1, (n - a[perm]).astype(np.float64)
    _check(builder, nv, u, v, w, _oracle_full(nv, u, v, w), paths)
    rng = np.random.default_rng(6)
    for shape in ("random", "tied"):
        nv, u, v, w = synth.GENERATORS[shape](300_000, seed=8)
        relabel = rng.permutation(nv).astype(np.int32)
        u, v = relabel[u], relabel[v]
        _check(builder, nv, u, v, w, _oracle_full(nv, u, v, w), paths)


def _local_weights(kind: str, n: int, rng):
    """Weight sets for the wide-key edge sort that finishes in shared memory
    (>= 5 active 8-bit digits) and for its fallback (a run of equal top
    digits longer than one window)."""
    if kind == "uniform":
        return rng.random(n)
    if kind == "spread":          # both signs, 40 binades: long compacted codes, many digits
        return rng.standard_normal(n) * np.exp2(rng.integers(-20, 20, n))
    if kind == "clustered":       # 1% of the weights in a band 2^-30 wide: runs of ~1000 items
        w = rng.random(n)
        m = rng.random(n) < 0.01
        w[m] = 0.5 + rng.random(int(m.sum())) * 2.0 ** -30
        return w
    if kind == "overflow":        # 30% equal weights among uniform ones: one run >> a window
        w = rng.random(n)
        w[rng.random(n) < 0.3] = 0.25
        return w
    if kind == "near_cap":        # runs just below / above the 8192-item window
        w = rng.random(n)
        for c, size in enumerate((1900, 4000, 4500)):
            size = min(size, n // 4)
            idx = rng.choice(n, size, replace=False)
            w[idx] = 0.125 * (c + 1) + rng.random(size) * 2.0 ** -40
        return w
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["uniform", "spread", "clustered", "overflow", "near_cap"])
@pytest.mark.parametrize("n", [3000, 70_000, 1_000_000])
def test_wide_key_local_sort(builder, kind, n):
    # the wide-key edge sort that finishes per window in shared memory
    # (local_sort.cuh) and its fallback, against the oracle and against the
    # forced full LSD sort (sort1_mode bit 2): same bits either way
    rng = np.random.default_rng(n + len(kind))
    nv, u, v, _ = synth.random_attach(n, seed=n % 97)
    w = _local_weights(kind, n, rng)
    exp = _oracle_full(nv, u, v, w)
    res = _check(builder, nv, u, v, w, exp, "default", debug=False)
    full = _check(builder, nv, u, v, w, exp, "no_local", debug=False)
    info, finfo = res.stats.path_info(), full.stats.path_info()
    assert finfo["sort1_local"] is None
    if res.stats.sort1_passes >= 5 or info["sort1_local"]:
        assert info["sort1_local"] in ("smem", "fallback")
    if kind == "overflow" and n >= 70_000:
        assert info["sort1_local"] == "fallback"
    if kind in ("uniform", "spread") and n >= 70_000:
        assert info["sort1_local"] == "smem"


@pytest.mark.parametrize("shape", ["path", "caterpillar", "random"])
def test_v0_chase_defers_long_chases(builder, shape):
    # single sorted chains chase O(n) steps from every endpoint: forced into the
    # chasing select, every such edge is deferred and finished from V2's vertex
    # map; random trees (max chase ~7) finish in the select itself.
    nv, u, v, w = synth.GENERATORS[shape](300_000, seed=3)
    exp = _oracle_full(nv, u, v, w)
    forced = _check(builder, nv, u, v, w, exp, "v0_chase")
    default = _check(builder, nv, u, v, w, exp, "default")
    assert forced.stats.path_info()["v0_chase"] == ("chase" if shape == "random" else "chase+fix")
    assert default.stats.path_info()["v0_chase"] is None  # the default chases only views of >= 64M edges


def test_rejects_bad_path_options(builder):
    nv, u, v, w = synth.random_attach(100, seed=1)
    with pytest.raises(ValueError):
        builder.build(nv, u, v, w, paths={"sort2_geometry": 3})
    with pytest.raises(ValueError):
        builder.build(nv, u, v, w, paths={"sort1_mode": 8})
    with pytest.raises(ValueError):
        builder.build(nv, u, v, w, paths={"v0_select": 3})
    with pytest.raises(ValueError):
        builder.build(nv, u, v, w, paths={"no_such_option": 1})


def test_every_kernel_kind_was_checked():
    # every kernel kind the 128M headline build launches (profiles/launches_r*_summary.csv)
    # has run inside a bit-exact comparison above; "other" (memset-like helpers) aside
    need = {"sort1_hist", "sort1_pass_first", "sort1_pass_mid", "sort1_pass_final", "sort1_local", "mi_hist",
            "mi_split_a", "mi_split_b", "mi_apply", "v1", "leafscan", "v2", "jump", "select_edges",
            "walk", "sort2_pass", "link_split", "link_apply", "upsweep_scan", "tail"}
    if not SEEN_KINDS:
        pytest.skip("run together with the path tests above")
    missing = need - set(SEEN_KINDS)
    assert not missing, f"kernel kinds never checked bit-exact: {sorted(missing)}"

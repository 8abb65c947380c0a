"""Upstream producer: the mutual-reachability MST.

CPU: the oracle restatement (oracle/dendro_oracle.py) against the
reference's own outputs (tests/golden/mreach_small.*, made by
tests/golden/make_mreach.py from the unmodified reference).  GPU: the device
producer (dmst_mreach_mst) against the same goldens -- bit-exact core
distances, edge order, endpoints and weights, both Prim engines, ties --
and against the config-2 fixture (1M points, the reference's ~50 min run)
at full size; then the produced tree through the dendrogram build.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from oracle import dendro_oracle as O
from tests.conftest import has_gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = json.load(open(os.path.join(HERE, "mreach_small.json")))
GOLD = np.load(os.path.join(HERE, "mreach_small.npz"))


def _case(c):
    g = {k: GOLD[f"{c['name']}_{k}"] for k in ("coords", "core_sq", "u", "v", "w")}
    return g


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference_goldens(c):
    g = _case(c)
    if c["n"] > 3000:
        pytest.skip("oracle Prim is O(n^2) numpy steps; covered on the GPU")
    cs = O.core_sq(g["coords"], c["min_pts"])
    assert np.array_equal(cs.view(np.uint64), g["core_sq"].view(np.uint64))
    nv, u, v, w = O.mutual_reachability_mst(g["coords"], c["min_pts"], c["engine"])
    assert nv == c["n"]
    assert np.array_equal(u, g["u"]) and np.array_equal(v, g["v"])
    assert np.array_equal(w.view(np.uint64), g["w"].view(np.uint64))


def test_argument_errors_match_reference():
    from paper_2401_06089_b200 import mutual_reachability_mst_b200
    x = np.zeros((4, 2))
    with pytest.raises(ValueError, match=r"min_pts must be in \[2, 4\]"):
        mutual_reachability_mst_b200(x, min_pts=5)
    with pytest.raises(ValueError, match="unknown engine 'fast'"):
        mutual_reachability_mst_b200(x, engine="fast")


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_device_mreach_matches_reference(c):
    import torch
    from paper_2401_06089_b200 import mutual_reachability_mst_b200
    g = _case(c)
    t, core = mutual_reachability_mst_b200(g["coords"], c["min_pts"], c["engine"], return_core_sq=True)
    torch.cuda.synchronize()
    assert np.array_equal(core.cpu().numpy().view(np.uint64), g["core_sq"].view(np.uint64))
    assert t.num_vertices == c["n"]
    assert np.array_equal(t.u.cpu().numpy(), g["u"]) and np.array_equal(t.v.cpu().numpy(), g["v"])
    assert np.array_equal(t.w.cpu().numpy().view(np.uint64), g["w"].view(np.uint64))


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_device_mreach_config2_full_size():
    """BASELINE.json configs[1]: 1M 3-D blob points, min_pts = 2 (the fixture
    is the reference's own tree, tests/golden/make_config2.py)."""
    import torch
    from paper_2401_06089_b200 import DendrogramBuilder, mutual_reachability_mst_b200, synth
    rng = np.random.default_rng(0)
    n = 1_000_000
    centers = rng.uniform(-10.0, 10.0, (10, 3))
    labels = rng.integers(0, 10, n)
    coords = centers[labels] + rng.standard_normal((n, 3))
    t = mutual_reachability_mst_b200(coords, 2)
    nv, u, v, w = synth.blobs1m()
    assert t.num_vertices == nv
    assert np.array_equal(t.u.cpu().numpy(), u) and np.array_equal(t.v.cpu().numpy(), v)
    assert np.array_equal(t.w.cpu().numpy().view(np.uint64), w.view(np.uint64))
    # straight into the dendrogram build, device to device
    r = DendrogramBuilder("cuda:0").build(t.num_vertices, t.u, t.v, t.w)
    ref = DendrogramBuilder("cuda:0").build(nv, u, v, w)
    torch.cuda.synchronize()
    assert bool((r.edge_parent == ref.edge_parent).all()) and bool((r.vertex_parent == ref.vertex_parent).all())

"""Input validation (`weighted_tree`, tree_core.py:110-139 of the reference):
the oracle restatement pinned to the reference's own verdicts
(tests/golden/invalid_trees.*, made by tests/golden/make_invalid.py with the
unmodified reference), and the device path (dmst_validate via
weighted_tree_b200) against the same verdicts and at scale."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from oracle import dendro_oracle as O
from tests.conftest import has_gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def invalid_cases():
    meta = json.load(open(os.path.join(GOLD, "invalid_trees.json")))
    arr = np.load(os.path.join(GOLD, "invalid_trees.npz"))
    for name, m in meta.items():
        yield name, m["num_vertices"], arr[f"{name}/u"], arr[f"{name}/v"], arr[f"{name}/w"], m["message"]


CASES = list(invalid_cases())


def _verdict(fn, nv, u, v, w, err):
    try:
        fn(nv, u, v, w)
        return ""
    except err as exc:
        return str(exc)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_oracle_matches_reference_verdicts(case):
    name, nv, u, v, w, msg = case
    assert _verdict(O.weighted_tree, nv, u, v, w, O.TreeFormatError) == msg


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_device_validation_matches_reference_verdicts(case):
    from paper_2401_06089_b200 import weighted_tree_b200
    from paper_2401_06089_b200.api import _tree_format_error
    name, nv, u, v, w, msg = case
    got = _verdict(weighted_tree_b200, nv, u, v, w, _tree_format_error())
    assert got == msg
    if not msg:
        t = weighted_tree_b200(nv, u.astype(np.int32), v.astype(np.int32), w)
        assert t.u.dtype == np.int64 and np.array_equal(t.u, u) and np.array_equal(t.original_id, np.arange(len(u)))


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("defect", ["none", "nan", "self_loop", "duplicate", "cycle", "range", "int64_range"])
def test_device_validation_at_scale(defect):
    # 4M-edge random tree with one defect, device verdict vs the oracle restatement
    from paper_2401_06089_b200 import synth, weighted_tree_b200
    from paper_2401_06089_b200.api import _tree_format_error
    n = 4_000_000
    nv, u, v, w = synth.random_attach(n, seed=5)
    u = u.astype(np.int64)
    v = v.astype(np.int64)
    w = w.copy()
    if defect == "nan":
        w[n - 3] = np.nan
    elif defect == "self_loop":
        u[n // 2] = v[n // 2]
    elif defect == "duplicate":
        u[n - 1], v[n - 1] = v[5], u[5]
    elif defect == "cycle":
        leaf = int(np.setdiff1d(v, u)[0])
        e = int(np.nonzero(v == leaf)[0][0])
        u[e], v[e] = v[(e + 1) % n], v[(e + n // 2) % n]
    elif defect == "range":
        v[123] = nv
    elif defect == "int64_range":
        v[123] = 1 << 40
    exp = _verdict(O.weighted_tree, nv, u, v, w, O.TreeFormatError)
    got = _verdict(weighted_tree_b200, nv, u, v, w, _tree_format_error())
    assert got == exp
    assert (got == "") == (defect == "none")

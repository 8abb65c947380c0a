"""Dendrogram statistics (`dendromst stats`, cli.py:97-135; analysis.py:21-52):
the oracle restatement pinned to the reference's reports
(tests/golden/stats_golden.json, made by tests/golden/make_stats.py), and the
device path (stats_b200 / dendrogram_height_b200) against the same reports
and, at 16M, against the known heights of single-chain trees."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from oracle import dendro_oracle as O
from paper_2401_06089_b200 import synth
from tests.conftest import has_gpu

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "stats_golden.json")))
IDS = [f"{g['shape']}_{g['n']}" for g in GOLD]


def _norm(r):
    r = dict(r)
    r["per_level"] = [list(map(int, c)) for c in r["per_level"]]
    return r


@pytest.mark.parametrize("g", GOLD, ids=IDS)
def test_oracle_stats_match_reference(g):
    nv, u, v, w = synth.GENERATORS[g["shape"]](g["n"], seed=g["seed"])
    assert _norm(O.stats_report(nv, u, v, w)) == g["report"]


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("g", GOLD, ids=IDS)
def test_device_stats_match_reference(g):
    from paper_2401_06089_b200 import stats_b200
    nv, u, v, w = synth.GENERATORS[g["shape"]](g["n"], seed=g["seed"])
    assert _norm(stats_b200(nv, u, v, w)) == g["report"]


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("shape", ["path", "caterpillar"])
def test_device_height_single_chain_16M(shape):
    # one chain of all n edges: height n, one chain
    from paper_2401_06089_b200 import stats_b200
    n = 16_000_000
    nv, u, v, w = synth.GENERATORS[shape](n, seed=0)
    r = stats_b200(nv, u, v, w)
    assert r["height"] == n and r["chains"] == 1 and r["levels"] == 1


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_device_height_vs_oracle_random_1M():
    from paper_2401_06089_b200 import stats_b200
    nv, u, v, w = synth.GENERATORS["tied"](1_000_000, seed=12)
    assert _norm(stats_b200(nv, u, v, w)) == _norm(O.stats_report(nv, u, v, w))

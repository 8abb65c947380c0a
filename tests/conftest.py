"""Test configuration: the `gpu` marker and shared generators.

Generators restate the reference's fixtures (/root/reference/pkg/tests/conftest.py:15-82)
so the parity tests read like the reference's own tests.
"""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

TOPOLOGIES = ("star", "path", "caterpillar", "attach")  # conftest.py:15


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: large-size tests")


def make_weights(m: int, rng, equal: bool = False) -> np.ndarray:   # conftest.py:18-21
    if equal:
        return np.full(m, 1.0)
    return rng.permutation(m).astype(np.float64) + 1.0


def topology_edges(topology: str, nv: int, rng):                     # conftest.py:24-39
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
        raise ValueError(f"unknown topology {topology!r}")
    return u, v


def make_tree(topology: str, nv: int, rng, equal_weights: bool = False):  # conftest.py:42-47
    """-> (nv, u, v, w) with input order shuffled."""
    u, v = topology_edges(topology, nv, rng)
    w = make_weights(nv - 1, rng, equal_weights)
    perm = rng.permutation(nv - 1)
    return nv, u[perm], v[perm], w[perm]


def golden_trees(path=None):
    """Yield dicts of the golden corpus made by tests/golden/make_golden.py."""
    path = path or os.path.join(ROOT, "tests", "golden", "golden_small.npz")
    g = np.load(path)
    off = 0
    coff = 0
    for i, name in enumerate(g["names"]):
        n = int(g["num_edges"][i])
        nv = int(g["num_vertices"][i])
        L = int(g["num_levels"][i])
        sl = slice(off, off + n)
        t = {"name": str(name), "num_vertices": nv, "num_levels": L,
             "u": g["u"][sl], "v": g["v"][sl], "w": g["w"][sl],
             "orig_of": g["orig_of"][sl], "heights": g["heights"][sl],
             "edge_parent": g["edge_parent"][sl],
             "vertex_parent": g["vertex_parent"][off + i: off + i + nv],
             "retirement": g["retirement"][sl], "terminal": g["terminal"][sl],
             "level": g["level"][sl],
             "counts": [tuple(int(x) for x in c) for c in
                        g["counts"][coff: coff + 4 * (L + 1)].reshape(-1, 4)]}
        off += n
        coff += 4 * (L + 1)
        yield t


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


REF_SITE = os.path.join(ROOT, "baseline", "_ref")


def reference_package():
    """The unmodified reference package `dendromst`, pip-installed into
    baseline/_ref (`pip install --no-deps --target baseline/_ref`
    of /root/reference/pkg; it travels to the GPU box with the repo
    snapshot), or None when it is not installed."""
    if not os.path.isdir(os.path.join(REF_SITE, "dendromst")):
        return None
    if REF_SITE not in sys.path:
        sys.path.insert(0, REF_SITE)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/dmst_numba_cache")
    try:
        import dendromst  # noqa: F401
        import dendromst.cli  # noqa: F401
        return dendromst
    except Exception:
        return None

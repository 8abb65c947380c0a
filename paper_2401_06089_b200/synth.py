"""Seeded synthetic MSTs of the shapes BASELINE.json names.

All generators return (num_vertices, u int32, v int32, w float64) with the
input order shuffled by ``rng.permutation`` so input order != construction
order, as the reference's fixtures do (/root/reference/pkg/tests/conftest.py:42-47).

* ``random_attach``: v = 1..nv-1 attaches to u = rng.integers(0, v)
  (conftest.py:35-36); w = rng.random(n), or float64(rng.integers(0, 4096, n))
  when ``tied`` (config 4's ~31k edges per tied weight).   Configs 1, 4, 5.
* ``path`` / ``caterpillar``: maximally skewed single-chain trees with
  monotone weights (config 3): path u=i, v=i+1, w=i; caterpillar spine of
  nv//2 vertices (conftest.py:31-34) with w = arange(n) in construction order,
  so every leg is lighter... (heavier weight, lower rank) than every spine edge.
"""
from __future__ import annotations

import hashlib

import numpy as np


def _shuffle(rng, u, v, w):
    perm = rng.permutation(u.shape[0])
    return (np.ascontiguousarray(u[perm], dtype=np.int32),
            np.ascontiguousarray(v[perm], dtype=np.int32),
            np.ascontiguousarray(w[perm], dtype=np.float64))


def random_attach(n: int, seed: int = 0, tied: bool = False):
    rng = np.random.default_rng(seed)
    nv = n + 1
    v = np.arange(1, nv, dtype=np.int64)
    u = rng.integers(0, v)
    if tied:
        w = rng.integers(0, 4096, n).astype(np.float64)
    else:
        w = rng.random(n)
    return (nv, *_shuffle(rng, u, v, w))


def path(n: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    u = np.arange(n, dtype=np.int64)
    return (n + 1, *_shuffle(rng, u, u + 1, u.astype(np.float64)))


def caterpillar(n: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    nv = n + 1
    spine = max(2, nv // 2)
    u = np.concatenate([np.arange(spine - 1, dtype=np.int64),
                        rng.integers(0, spine, nv - spine)])
    v = np.arange(1, nv, dtype=np.int64)
    return (nv, *_shuffle(rng, u, v, np.arange(n, dtype=np.float64)))


def blobs1m(n: int = 999_999, seed: int = 0):
    """Config 2: the reference's mutual-reachability MST (min_samples=2) of 1M
    3-D Gaussian-blob points, computed once by the unmodified reference
    (tests/golden/make_config2.py) and committed as a fixture; n and seed are
    fixed by the fixture."""
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                        "config2_blobs1m.npz")
    g = np.load(path)
    return (int(g["num_vertices"]), np.ascontiguousarray(g["u"], np.int32), np.ascontiguousarray(g["v"], np.int32),
            np.ascontiguousarray(g["w"], np.float64))


GENERATORS = {
    "random": lambda n, seed=0: random_attach(n, seed, tied=False),
    "tied": lambda n, seed=0: random_attach(n, seed, tied=True),
    "path": path,
    "blobs1m": blobs1m,
    "caterpillar": caterpillar,
}


def input_digest(u, v, w) -> str:
    """sha256 of (u, v as int64; w as float64): pins regenerated inputs."""
    h = hashlib.sha256()
    for a in (np.asarray(u).astype(np.int64), np.asarray(v).astype(np.int64),
              np.asarray(w).astype(np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()

"""ORACLE / TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference hot path (`rank_edges` + `pandora`) of
arxiv/paper_2401_06089's `dendromst` package, written from the reference's
behaviour, numpy for the array work and C (oracle/uf_roots.c, the numba
union-find's twin) for the one sequential loop.  Every function cites the
reference file:line it restates; paths are relative to
/root/reference/pkg/src/dendromst/.

Who may import this module: tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline / `--impl reference` legs - and only as the checker or the
timed CPU baseline.  The product path (paper_2401_06089_b200) never imports
it and has no CPU fallback.

Pinning: tests/test_oracle_golden.py checks this module against golden
vectors produced by the UNMODIFIED reference (tests/golden/make_golden.py
imports /root/reference/pkg/src) and against the reference's own
known-answer tests (tests/test_*.py KATs).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import math

import numpy as np

ROOT = -1  # expansion.py:20

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    """Load (building on first use) the C union-find, oracle/_build/liboracle.so."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_build", "liboracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(path)
        p64 = ctypes.POINTER(ctypes.c_int64)
        lib.oracle_uf_roots.argtypes = [ctypes.c_int64, ctypes.c_int64, p64, p64, p64]
        lib.oracle_uf_roots.restype = None
        _LIB = lib
    return _LIB


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


# ----------------------------------------------------------------- tree_core

@dataclass(frozen=True)
class Ranked:
    """RankedTree (tree_core.py:39-56) without the frozen base object."""
    num_vertices: int
    rank_of: np.ndarray
    orig_of: np.ndarray
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray

    @property
    def num_edges(self) -> int:
        return int(self.u.shape[0])


def rank_edges(num_vertices: int, u, v, w) -> Ranked:
    """tree_core.py:174-190: stable argsort of -w; ties by ascending original id."""
    u = np.ascontiguousarray(u, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.int64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    order = np.argsort(-w, kind="stable")                      # :180
    rank_of = np.empty(w.shape[0], dtype=np.int64)
    rank_of[order] = np.arange(w.shape[0])                     # :181-182
    return Ranked(num_vertices, rank_of, order, u[order], v[order], w[order])  # :186-189


def max_incident(num_vertices: int, u: np.ndarray, v: np.ndarray,
                 rank: np.ndarray) -> np.ndarray:
    """tree_core.py:193-199 / contraction.py:149-154: scatter-max of ranks, -1 init."""
    mi = np.full(num_vertices, -1, dtype=np.int64)
    np.maximum.at(mi, u, rank)
    np.maximum.at(mi, v, rank)
    return mi


# ------------------------------------------------------------------ classify

LEAF, CHAIN, ALPHA = 0, 1, 2  # classify.py:17-20


def edge_kinds_from_ends(at_u: np.ndarray, at_v: np.ndarray) -> np.ndarray:
    """classify.py:37-42."""
    kinds = np.full(at_u.shape[0], CHAIN, dtype=np.int8)
    kinds[at_u & at_v] = LEAF
    kinds[~at_u & ~at_v] = ALPHA
    return kinds


def kind_counts(kinds: np.ndarray) -> tuple[int, int, int]:
    """classify.py:45-50: (n_alpha, n_leaf, n_chain)."""
    return (int(np.count_nonzero(kinds == ALPHA)),
            int(np.count_nonzero(kinds == LEAF)),
            int(np.count_nonzero(kinds == CHAIN)))


# --------------------------------------------------------------- contraction

def uf_roots(num_vertices: int, cu: np.ndarray, cv: np.ndarray) -> np.ndarray:
    """contraction.py:53-79 (`_uf_roots`): C twin of the numba loop."""
    cu = np.ascontiguousarray(cu, dtype=np.int64)
    cv = np.ascontiguousarray(cv, dtype=np.int64)
    parent = np.empty(num_vertices, dtype=np.int64)
    _lib().oracle_uf_roots(num_vertices, cu.shape[0], _ptr(cu), _ptr(cv), _ptr(parent))
    return parent


def component_labels(num_vertices: int, u, v) -> np.ndarray:
    """contraction.py:82-93: canonical labels ordered by smallest member."""
    roots = uf_roots(num_vertices, u, v)
    is_root = roots == np.arange(num_vertices)
    ids = np.cumsum(is_root) - 1
    return ids[roots]


@dataclass
class Level:
    """ContractionLevel (contraction.py:106-120)."""
    surviving_edges: np.ndarray
    vertex_map: np.ndarray
    super_max_incident: np.ndarray
    super_count: int
    edge_u: np.ndarray
    edge_v: np.ndarray


@dataclass
class Hierarchy:
    """ContractionHierarchy (contraction.py:123-146)."""
    levels: list
    retirement_level: np.ndarray
    view_kind_counts: list
    edge_u: np.ndarray
    edge_v: np.ndarray
    num_vertices: int

    @property
    def num_levels(self) -> int:
        return len(self.levels)


def contract_level(nv: int, u, v, rank, alpha: np.ndarray) -> Level:
    """contraction.py:165-183."""
    keep = alpha
    vertex_map = component_labels(nv, u[~keep], v[~keep])       # :168
    super_count = int(vertex_map.max()) + 1                     # :169
    edge_u = vertex_map[u[keep]]                                # :170
    edge_v = vertex_map[v[keep]]                                # :171
    surviving = rank[keep]                                      # :172
    smi = max_incident(super_count, edge_u, edge_v, surviving)  # :173-175
    return Level(surviving, vertex_map, smi, super_count, edge_u, edge_v)


def build_hierarchy(r: Ranked, mi: np.ndarray) -> Hierarchy:
    """contraction.py:186-219: classify -> contract until a view has no alpha."""
    n = r.num_edges
    nv, vu, vv, vrank = r.num_vertices, r.u, r.v, np.arange(n)  # :193
    cur_mi = mi
    levels: list[Level] = []
    counts: list[tuple[int, int, int, int]] = []
    retirement = np.full(n, -1, dtype=np.int64)                 # :197
    while True:
        at_u = vrank == cur_mi[vu]                              # view_kinds :157-162
        at_v = vrank == cur_mi[vv]
        kinds = edge_kinds_from_ends(at_u, at_v)
        counts.append((*kind_counts(kinds), int(vrank.shape[0])))  # :201
        alpha = kinds == ALPHA
        if levels and not alpha.any():                          # :203-205
            retirement[vrank] = len(levels)
            break
        level = contract_level(nv, vu, vv, vrank, alpha)        # :206
        retirement[vrank[~alpha]] = len(levels)                 # :207
        levels.append(level)
        nv, vu, vv, vrank = level.super_count, level.edge_u, level.edge_v, level.surviving_edges
        cur_mi = level.super_max_incident                       # :210
    return Hierarchy(levels, retirement, counts, r.u, r.v, r.num_vertices)


# ----------------------------------------------------------------- expansion

@dataclass
class Chains:
    """ChainAssignment (expansion.py:38-53)."""
    terminal: np.ndarray
    anchor: np.ndarray
    level: np.ndarray


def assign_chains(h: Hierarchy) -> Chains:
    """expansion.py:97-128: earliest level whose supervertex parent is heavier."""
    n = int(h.retirement_level.shape[0])
    terminal = np.full(n, ROOT, dtype=np.int64)
    anchor = np.zeros(n, dtype=np.int64)
    level_arr = np.zeros(n, dtype=np.int64)
    retirement = h.retirement_level
    pending = np.arange(n)
    comp = None
    for k, lvl in enumerate(h.levels, start=1):
        comp = lvl.vertex_map if comp is None else lvl.vertex_map[comp]   # :114
        eligible = retirement[pending] < k                                # :115
        cand = pending[eligible]
        if cand.shape[0] == 0:
            pending = pending[~eligible] if eligible.any() else pending
            continue
        sv = comp[h.edge_u[cand]]                                         # :120
        p = lvl.super_max_incident[sv]                                    # :121
        hit = (p >= 0) & (p < cand)                                       # :122
        matched = cand[hit]
        terminal[matched] = p[hit]
        anchor[matched] = sv[hit]
        level_arr[matched] = k
        pending = np.concatenate([pending[~eligible], cand[~hit]])        # :127
    return Chains(terminal, anchor, level_arr)


def stitch_chains(c: Chains, vertex_parent: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """expansion.py:131-145: lexsort (terminal, anchor, rank); link to predecessor."""
    n = c.terminal.shape[0]
    ranks = np.arange(n)
    order = np.lexsort((ranks, c.anchor, c.terminal))          # :135
    t_s = c.terminal[order]
    a_s = c.anchor[order]
    head = np.ones(n, dtype=bool)
    head[1:] = (t_s[1:] != t_s[:-1]) | (a_s[1:] != a_s[:-1])   # :138-139
    prev = np.concatenate(([ROOT], order[:-1]))                # :140
    parent_sorted = np.where(head, t_s, prev)                   # :141
    edge_parent = np.empty(n, dtype=np.int64)
    edge_parent[order] = parent_sorted                         # :142-143
    return edge_parent, np.asarray(vertex_parent, dtype=np.int64).copy()


def pandora(r: Ranked):
    """expansion.py:148-153: returns (edge_parent, vertex_parent, hierarchy)."""
    mi = max_incident(r.num_vertices, r.u, r.v, np.arange(r.num_edges))  # build_incidence
    vp = mi.copy()                                                         # classify.py:23-25
    h = build_hierarchy(r, mi)
    ep, vp = stitch_chains(assign_chains(h), vp)
    return ep, vp, h


@dataclass
class BuildResult:
    orig_of: np.ndarray
    heights: np.ndarray
    edge_parent: np.ndarray
    vertex_parent: np.ndarray
    view_kind_counts: list
    num_levels: int
    hierarchy: Hierarchy


def build(num_vertices: int, u, v, w) -> BuildResult:
    """The timed scope of `dendromst build` (cli.py:82-85 in the survey's
    numbering; /root/reference/pkg/src/dendromst/cli.py `_cmd_build`):
    rank_edges then pandora."""
    r = rank_edges(num_vertices, u, v, w)
    ep, vp, h = pandora(r)
    return BuildResult(r.orig_of, r.w, ep, vp, h.view_kind_counts, h.num_levels, h)


# ------------------------------------------------------- sequential oracles

def dendrogram_bottom_up(r: Ranked) -> tuple[np.ndarray, np.ndarray]:
    """oracles.py:63-85: sequential union-find from lightest to heaviest edge
    (the reference's second, independent ground truth)."""
    n = r.num_edges
    edge_parent = np.full(n, ROOT, dtype=np.int64)
    vertex_parent = np.full(r.num_vertices, ROOT, dtype=np.int64)
    parent = list(range(r.num_vertices))

    def find(x):
        root = x
        while parent[root] != root:
            root = parent[root]
        while parent[x] != root:
            parent[x], x = root, parent[x]
        return root

    latest = [ROOT] * r.num_vertices
    u, v = r.u.tolist(), r.v.tolist()
    for rank in range(n - 1, -1, -1):
        for x in (u[rank], v[rank]):
            rr = latest[find(x)]
            if rr != ROOT:
                edge_parent[rr] = rank
            else:
                vertex_parent[x] = rank
        a, b = find(u[rank]), find(v[rank])
        if a > b:
            a, b = b, a
        parent[b] = a
        latest[find(u[rank])] = rank
    return edge_parent, vertex_parent


# ------------------------------------------------------------ validation
class TreeFormatError(ValueError):
    pass


def weighted_tree(num_vertices: int, u, v, w):
    """Restates weighted_tree (tree_core.py:110-139): the same checks in the
    same order with the same messages; returns (num_vertices, u, v, w) with
    the reference's dtypes.  Connectivity by the C union-find (uf_roots)."""
    u = np.ascontiguousarray(u, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.int64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    n = u.shape[0]
    if num_vertices < 2:                                              # :116-117
        raise TreeFormatError("a tree needs at least 2 vertices")
    if n != num_vertices - 1:                                         # :118-121
        raise TreeFormatError(f"edge count {n} != numVertices - 1 = {num_vertices - 1}")
    if v.shape[0] != n or w.shape[0] != n:                            # :122-123
        raise TreeFormatError("edge arrays have mismatched lengths")
    if not np.all(np.isfinite(w)):                                    # :124-126
        bad = int(np.nonzero(~np.isfinite(w))[0][0])
        raise TreeFormatError(f"non-finite weight on edge {bad}")
    if u.min(initial=0) < 0 or v.min(initial=0) < 0:                  # :127-128
        raise TreeFormatError("negative vertex id")
    if max(u.max(initial=-1), v.max(initial=-1)) >= num_vertices:     # :129-130
        raise TreeFormatError("vertex id out of range")
    if np.any(u == v):                                                # :131-133
        bad = int(np.nonzero(u == v)[0][0])
        raise TreeFormatError(f"self-loop on edge {bad}")
    key = np.minimum(u, v) * np.int64(num_vertices) + np.maximum(u, v)  # :134-136
    if np.unique(key).shape[0] != n:
        raise TreeFormatError("duplicate undirected edge")
    roots = uf_roots(num_vertices, u, v)                              # :137-138 (_connected, :102-107)
    if int(np.count_nonzero(roots == np.arange(num_vertices))) != 1:
        raise TreeFormatError("input is disconnected or cyclic, not a tree")
    return num_vertices, u, v, w


# ------------------------------------------------------------- statistics
def dendrogram_height(edge_parent: np.ndarray, vertex_parent: np.ndarray) -> int:
    """analysis.py:21-33: edge depths in one ascending-rank pass (parents are
    heavier, i.e. smaller rank); height = max depth over vertex parents."""
    n = int(edge_parent.shape[0])
    depth = np.empty(n, dtype=np.int64)
    ep = np.asarray(edge_parent, dtype=np.int64)
    for e in range(n):
        p = ep[e]
        depth[e] = 1 if p == ROOT else depth[p] + 1
    return int(depth[np.asarray(vertex_parent, dtype=np.int64)].max())


def num_chains(c: Chains) -> int:
    """expansion.py:52-54: distinct (terminal, anchor) pairs."""
    return int(np.unique(np.stack([c.terminal, c.anchor], axis=1), axis=0).shape[0])


def stats_report(num_vertices: int, u, v, w) -> dict:
    """The numbers `dendromst stats` prints (cli.py:97-135), per_level as tuples."""
    r = rank_edges(num_vertices, u, v, w)
    ep, vp, h = pandora(r)
    n = r.num_edges
    height = dendrogram_height(ep, vp)
    return {"edges": n, "vertices": num_vertices, "levels": h.num_levels, "height": height,
            "chains": num_chains(assign_chains(h)),
            "skewness_log2_edges": height / math.log2(n) if n >= 2 else 0.0,
            "skewness_log2_points": height / math.log2(n + 1),
            "per_level": [tuple(int(x) for x in c) for c in h.view_kind_counts]}


# -------------------------------------------------------------- file format
def dendrogram_text(edge_parent, vertex_parent) -> bytes:
    """Restates write_dendrogram (dendro_io.py:28-38): the bytes of the v1 file."""
    ep = np.asarray(edge_parent, dtype=np.int64).tolist()
    vp = np.asarray(vertex_parent, dtype=np.int64).tolist()
    head = f"#dendrogram v1 n={len(ep)} nv={len(vp)}\n"
    body = "".join(f"E {r} {p}\n" for r, p in enumerate(ep)) + "".join(f"V {x} {p}\n" for x, p in enumerate(vp))
    return (head + body).encode()


def verify_text(a: bytes, b: bytes) -> tuple[int, str]:
    """Restates `dendromst verify` (cli.py:138-155) on two v1 files' bytes
    (read_dendrogram, dendro_io.py:41-75, for well-formed files)."""
    def parse(data):
        lines = data.decode().splitlines()
        parts = lines[0].split()
        n, nv = int(parts[2][2:]), int(parts[3][3:])
        ep = np.full(n, ROOT, dtype=np.int64)
        vp = np.full(nv, ROOT, dtype=np.int64)
        for line in lines[1:]:
            if not line or line.startswith("#"):
                continue
            kind, idx, parent = line.split()
            (ep if kind == "E" else vp)[int(idx)] = int(parent)
        return ep, vp
    (ea, va), (eb, vb) = parse(a), parse(b)
    for label, pa, pb in (("edge", ea, eb), ("vertex", va, vb)):
        if pa.shape != pb.shape:
            return 1, f"size mismatch: {pa.shape[0]} vs {pb.shape[0]} {label} nodes"
        diff = np.nonzero(pa != pb)[0]
        if diff.shape[0]:
            i = int(diff[0])
            return 1, f"first divergence: {label} {i}: {int(pa[i])} != {int(pb[i])}"
    return 0, "identical"


# ---------------------------------------------------------------- upstream producer
# Mutual-reachability MST, restating
# /root/reference/pkg/src/dendromst/pointgen.py:56-178 for small clouds.

def _kdtree_sqdist(diff: np.ndarray) -> np.ndarray:
    """Squared distances in scipy cKDTree's p = 2 summation order (checked
    bitwise against cKDTree.query): four strided accumulators over the full
    blocks of 4 dimensions, combined left to right, then the rest."""
    q = diff * diff
    dim = q.shape[-1]
    acc = [np.zeros(q.shape[:-1]) for _ in range(4)]
    full = dim // 4 * 4
    for i in range(0, full, 4):
        for j in range(4):
            acc[j] = acc[j] + q[..., i + j]
    s = ((acc[0] + acc[1]) + acc[2]) + acc[3]
    for i in range(full, dim):
        s = s + q[..., i]
    return s


def core_sq(coords: np.ndarray, min_pts: int) -> np.ndarray:
    """core_distances(coords, min_pts) ** 2 (pointgen.py:56-61): the
    min_pts-th smallest distance (self included), by brute force."""
    x = np.asarray(coords, np.float64)
    out = np.empty(x.shape[0])
    for lo in range(0, x.shape[0], 512):
        d = _kdtree_sqdist(x[lo:lo + 512, None, :] - x[None, :, :])
        kth = np.partition(d, min_pts - 1, axis=1)[:, min_pts - 1]
        out[lo:lo + 512] = np.sqrt(kth) ** 2
    return out


def _prim_sqdist(x: np.ndarray, c: np.ndarray, numpy_engine: bool) -> np.ndarray:
    q = (x - c) ** 2
    dim = q.shape[1]
    if numpy_engine and dim == 8:   # numpy's pairwise row sum at 8 columns
        return ((q[:, 0] + q[:, 1]) + (q[:, 2] + q[:, 3])) + ((q[:, 4] + q[:, 5]) + (q[:, 6] + q[:, 7]))
    s = q[:, 0] if numpy_engine else 0.0 + q[:, 0]
    for t in range(1, dim):
        s = s + q[:, t]
    return s


def prim_mst(coords: np.ndarray, core_sq_: np.ndarray, engine: str = "auto"):
    """Dense Prim (pointgen.py:71-148): (u, v, w_sq) in discovery order.
    numba engine (:91-148): compacted arrays, swap-with-last removal, first
    minimum in compacted order; numpy engine (:71-88): first minimum by
    point id.  Both update with strict `<`."""
    x = np.asarray(coords, np.float64)
    n = x.shape[0]
    if engine == "auto":
        engine = "numba" if n >= 4096 else "numpy"
    numpy_engine = engine == "numpy"
    idx = np.arange(1, n, dtype=np.int64)
    acoord = x[1:].copy()
    acore = np.asarray(core_sq_, np.float64)[1:].copy()
    abest = np.full(n - 1, np.inf)
    afrom = np.zeros(n - 1, np.int64)
    out_u = np.empty(n - 1, np.int64)
    out_v = np.empty(n - 1, np.int64)
    out_w = np.empty(n - 1)
    cur = 0
    m = n - 1
    for it in range(n - 1):
        d = _prim_sqdist(acoord[:m], x[cur], numpy_engine)
        d = np.where(acore[:m] > d, acore[:m], d)
        cc = core_sq_[cur]
        d = np.where(cc > d, cc, d)
        upd = d < abest[:m]
        abest[:m][upd] = d[upd]
        afrom[:m][upd] = cur
        if numpy_engine:
            mn = abest[:m].min()
            cand = np.nonzero(abest[:m] == mn)[0]
            bk = int(cand[np.argmin(idx[cand])])
        else:
            bk = int(np.argmin(abest[:m]))
        cur = int(idx[bk])
        out_u[it], out_v[it], out_w[it] = afrom[bk], cur, abest[bk]
        m -= 1
        for arr in (idx, acore, abest, afrom):
            arr[bk] = arr[m]
        acoord[bk] = acoord[m]
    return out_u, out_v, out_w


def mutual_reachability_mst(coords: np.ndarray, min_pts: int = 2, engine: str = "auto"):
    """(num_vertices, u, v, w) of mutual_reachability_mst (pointgen.py:158-178)."""
    x = np.asarray(coords, np.float64)
    u, v, w_sq = prim_mst(x, core_sq(x, min_pts), engine)
    return x.shape[0], u, v, np.sqrt(w_sq)

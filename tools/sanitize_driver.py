"""Small builds for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every entry point (device build incl. the cooperative tail, host-buffer build,
validation incl. the duplicate-sort path, dendrogram height, the v1 text
writer / reader / verify, the mutual-reachability MST producer) on small
inputs, each checked against the CPU oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import dendro_oracle as O  # noqa: E402
from paper_2401_06089_b200 import (DendrogramBuilder, dendrogram_height_b200, synth,  # noqa: E402
                                   validate_b200)
from paper_2401_06089_b200.api import _tree_format_error  # noqa: E402

b = DendrogramBuilder("cuda:0")
bad = 0
for shape in ("random", "tied", "path", "caterpillar"):
    for n in (1, 5, 1000, 70_000):
        nv, u, v, w = synth.GENERATORS[shape](n, seed=n)
        r = b.build(nv, u, v, w, debug=True, want_chains=True)
        e = O.build(nv, u, v, w)
        ok = (np.array_equal(r.edge_parent.cpu().numpy(), e.edge_parent)
              and np.array_equal(r.vertex_parent.cpu().numpy(), e.vertex_parent)
              and np.array_equal(r.orig_of.cpu().numpy(), e.orig_of))
        hb = b.build_host(nv, u, v, w)
        ok &= np.array_equal(hb.edge_parent.numpy(), e.edge_parent)
        ok &= dendrogram_height_b200(r.edge_parent) == O.dendrogram_height(e.edge_parent, e.vertex_parent)
        bad += not ok
# forced code paths a 128M build takes: view 0 chased in the select (random:
# no deferral; path: every edge deferred to k_select_fix), the host level loop,
# sliced maxIncident on every view
for shape, paths in (("random", {"v0_select": 2, "tail_edges": -1}), ("path", {"v0_select": 2}),
                     ("tied", {"mi_apply_mode": 2, "direct_mi_bytes": -1, "tail_edges": -1})):
    nv, u, v, w = synth.GENERATORS[shape](60_000, seed=4)
    r = b.build(nv, u, v, w, paths=paths)
    e = O.build(nv, u, v, w)
    bad += not (np.array_equal(r.edge_parent.cpu().numpy(), e.edge_parent)
                and np.array_equal(r.vertex_parent.cpu().numpy(), e.vertex_parent))
# validation: valid, duplicate (sort path), cycle (sort path, no duplicate), self-loop
nv, u, v, w = synth.random_attach(50_000, seed=3)
u = u.astype(np.int64)
v = v.astype(np.int64)
cases = {"valid": (u, v)}
u2, v2 = u.copy(), v.copy()
u2[-1], v2[-1] = v[0], u[0]
cases["duplicate"] = (u2, v2)
u3, v3 = u.copy(), v.copy()
u3[7] = v3[7]
cases["self_loop"] = (u3, v3)
for name, (uu, vv) in cases.items():
    def verdict(fn, err):
        try:
            fn(nv, uu, vv, w)
            return ""
        except err as exc:
            return str(exc)
    bad += verdict(validate_b200, _tree_format_error()) != verdict(O.weighted_tree, O.TreeFormatError)
# edge sort key transforms: top-field compaction + narrow 32-bit keys
rng = np.random.default_rng(5)
nv, u, v, _ = synth.random_attach(20_000, seed=5)
for w in (rng.integers(0, 4096, nv - 1).astype(np.float64),
          rng.choice([-1.0, 1.0], nv - 1) * rng.integers(1, 64, nv - 1) * np.exp2(rng.integers(-3, 3, nv - 1))):
    r = b.build(nv, u, v, w)
    e = O.build(nv, u, v, w)
    bad += not (np.array_equal(r.orig_of.cpu().numpy(), e.orig_of)
                and np.array_equal(r.edge_parent.cpu().numpy(), e.edge_parent))
# wide-key edge sort finished in shared memory: uniform, clustered (window LSD
# passes) and a long tied run (overflow -> full LSD fallback)
nv, u, v, _ = synth.random_attach(30_000, seed=9)
wu = rng.random(nv - 1)
wc = wu.copy()
wc[rng.random(nv - 1) < 0.05] = 0.5 + rng.random() * 2.0 ** -30
wo = wu.copy()
wo[rng.random(nv - 1) < 0.3] = 0.25
for w in (wu, wc, wo):
    r = b.build(nv, u, v, w)
    e = O.build(nv, u, v, w)
    bad += not (np.array_equal(r.orig_of.cpu().numpy(), e.orig_of)
                and np.array_equal(r.edge_parent.cpu().numpy(), e.edge_parent))
# v1 text format: device writer -> device reader -> verify
import tempfile  # noqa: E402
from paper_2401_06089_b200 import read_dendrogram_b200, verify_b200, write_dendrogram_b200  # noqa: E402
with tempfile.TemporaryDirectory() as d:
    pa, pb = os.path.join(d, "a"), os.path.join(d, "b")
    write_dendrogram_b200(pa, r.edge_parent, r.vertex_parent)
    write_dendrogram_b200(pb, r.edge_parent, r.vertex_parent, sidecar=True)
    back = read_dendrogram_b200(pa)
    bad += not bool((back.edge_parent == r.edge_parent).all())
    bad += verify_b200(pa, pb) != (0, "identical")
# upstream producer: core distances + both Prim engines
from paper_2401_06089_b200 import mutual_reachability_mst_b200  # noqa: E402
for dim, engine in ((3, "numba"), (8, "numpy"), (2, "numba")):
    x = rng.standard_normal((300, dim))
    if dim == 2:
        x = np.round(x * 3)  # ties
    t = mutual_reachability_mst_b200(x, 3, engine)
    _, eu, ev, ew = O.mutual_reachability_mst(x, 3, engine)
    bad += not (np.array_equal(t.u.cpu().numpy(), eu) and np.array_equal(t.v.cpu().numpy(), ev)
                and np.array_equal(t.w.cpu().numpy(), ew))
print("sanitize driver done, mismatches:", bad)

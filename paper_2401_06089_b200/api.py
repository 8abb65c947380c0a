"""Host-side mirror of the reference hot-path interface, on the B200 path.

Reference interface (paths under /root/reference/pkg/src/dendromst/):

* ``rank_edges(tree: WeightedTree) -> RankedTree``      tree_core.py:174-190
* ``pandora(tree: RankedTree) -> Dendrogram``           expansion.py:148-153
* ``_ALGOS: dict[str, Callable[[RankedTree], Dendrogram]]``   cli.py:27-31
* ``Dendrogram(edge_parent, vertex_parent)`` with array equality  expansion.py:56-80

This module provides the same entry points running on the GPU through the
C ABI (include/dmst.h):

* :func:`rank_edges_b200` / :func:`pandora_b200` — same arguments, same
  results, drop-in for the reference functions; :func:`pandora_b200` has
  the ``_ALGOS`` signature and :func:`register_algorithm` installs it.
* :func:`build_b200` — both fused, the timed scope of ``dendromst build``.
* :class:`DendrogramBuilder` — device-resident API (torch tensors in/out,
  reusable workspace) for callers that keep the MST in HBM.

Device buffers are torch tensors (PyTorch is the allocator and stream
provider only).  There is no CPU fallback: without a CUDA device or
without the built library these functions raise.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

ROOT = -1  # expansion.py:20


def _reference_dendrogram_type():
    try:  # if the reference package is importable, return ITS type so == works both ways
        from dendromst.expansion import Dendrogram as RefDendrogram  # type: ignore
        return RefDendrogram
    except Exception:
        return None


@dataclass
class Dendrogram:
    """Mirror of ``dendromst.expansion.Dendrogram`` (expansion.py:56-80)."""
    edge_parent: np.ndarray
    vertex_parent: np.ndarray

    @property
    def num_edges(self) -> int:
        return int(self.edge_parent.shape[0])

    @property
    def num_vertices(self) -> int:
        return int(self.vertex_parent.shape[0])

    def __eq__(self, other) -> bool:
        if not hasattr(other, "edge_parent") or not hasattr(other, "vertex_parent"):
            return NotImplemented
        return (np.array_equal(self.edge_parent, other.edge_parent)
                and np.array_equal(self.vertex_parent, other.vertex_parent))


class TreeFormatError(ValueError):
    """Mirror of ``dendromst.tree_core.TreeFormatError`` (raised by
    :func:`weighted_tree_b200`; the reference's own class when importable)."""


def _tree_format_error():
    try:
        from dendromst.tree_core import TreeFormatError as Ref  # type: ignore
        return Ref
    except Exception:
        return TreeFormatError


@dataclass(frozen=True)
class WeightedTree:
    """Mirror of ``dendromst.tree_core.WeightedTree`` (tree_core.py:20-36)."""
    num_vertices: int
    u: object
    v: object
    w: object
    original_id: object

    @property
    def num_edges(self) -> int:
        return int(self.u.shape[0])


@dataclass(frozen=True)
class RankedTree:
    """Mirror of ``dendromst.tree_core.RankedTree`` (tree_core.py:39-56)."""
    base: object
    rank_of: np.ndarray
    orig_of: np.ndarray
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray

    @property
    def num_vertices(self) -> int:
        return int(self.base.num_vertices)

    @property
    def num_edges(self) -> int:
        return int(self.u.shape[0])


@dataclass
class BuildResult:
    """Device-resident outputs of one build (rank space, like the reference)."""
    orig_of: torch.Tensor        # int32[n]   RankedTree.orig_of
    heights: torch.Tensor        # float64[n] RankedTree.w (merge heights)
    edge_parent: torch.Tensor    # int32[n]   Dendrogram.edge_parent
    vertex_parent: torch.Tensor  # int32[nv]  Dendrogram.vertex_parent
    stats: _lib.DmstStats = field(repr=False, default=None)
    debug: dict = field(default_factory=dict, repr=False)

    @property
    def num_levels(self) -> int:
        return int(self.stats.num_levels)

    @property
    def view_kind_counts(self) -> list[tuple[int, int, int, int]]:
        return self.stats.view_kind_counts()

    def dendrogram(self) -> Dendrogram:
        """Host Dendrogram with the reference's int64 dtype."""
        return Dendrogram(self.edge_parent.cpu().numpy().astype(np.int64),
                          self.vertex_parent.cpu().numpy().astype(np.int64))


@dataclass
class HostBuildResult:
    """Host-resident outputs of :meth:`DendrogramBuilder.build_host`."""
    orig_of: torch.Tensor        # int32[n]   (CPU)
    heights: torch.Tensor        # float64[n]
    edge_parent: torch.Tensor    # int32[n]
    vertex_parent: torch.Tensor  # int32[nv]
    stats: _lib.DmstStats = field(repr=False, default=None)

    @property
    def num_levels(self) -> int:
        return int(self.stats.num_levels)

    @property
    def view_kind_counts(self) -> list[tuple[int, int, int, int]]:
        return self.stats.view_kind_counts()

    @classmethod
    def empty(cls, n: int, nv: int, pin: bool = True) -> "HostBuildResult":
        def mk(k, dt):
            t = torch.empty(k, dtype=dt)
            return t.pin_memory() if pin else t
        return cls(mk(n, torch.int32), mk(n, torch.float64), mk(n, torch.int32), mk(nv, torch.int32))

    def dendrogram(self) -> Dendrogram:
        return Dendrogram(self.edge_parent.numpy().astype(np.int64), self.vertex_parent.numpy().astype(np.int64))


def _as_host(x, dtype: torch.dtype) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    if t.device.type != "cpu":
        raise ValueError("build_host takes host (CPU) arrays")
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _device_of(device) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2401_06089_b200 needs a CUDA device (no CPU fallback)")
    d = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if d.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {d}")
    if d.index is None:
        d = torch.device("cuda", torch.cuda.current_device())
    return d


def _as_dev(x, dtype: torch.dtype, dev: torch.device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(device=dev, non_blocking=True)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x)).to(device=dev)
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


class DendrogramBuilder:
    """Reusable workspace + entry points on one device.

    ``build`` takes (num_vertices, u, v, w) as torch tensors (ideally
    int32/int32/float64 already on the device) or numpy arrays.
    """

    def __init__(self, device=None):
        self.lib = _lib.load()
        self.device = _device_of(device)
        self._ws: torch.Tensor | None = None

    def workspace(self, n: int, nv: int) -> torch.Tensor:
        need = int(self.lib.dmst_workspace_bytes(n, nv))
        if need == 0:
            raise ValueError(f"bad sizes n={n} nv={nv}")
        if self._ws is None or self._ws.numel() < need:
            self._ws = None
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def host_workspace(self, n: int, nv: int) -> torch.Tensor:
        need = int(self.lib.dmst_host_workspace_bytes(n, nv))
        if need == 0:
            raise ValueError(f"bad sizes n={n} nv={nv}")
        if getattr(self, "_hws", None) is None or self._hws.numel() < need:
            self._hws = None
            self._hws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._hws

    def build_host(self, num_vertices: int, u, v, w, *, out: HostBuildResult | None = None,
                   profile: bool = False, paths: dict | None = None) -> HostBuildResult:
        """rank_edges + pandora on HOST arrays (dmst_build_host): inputs are
        copied in and every output copied back as soon as its stage is done,
        overlapped with the remaining kernels.  Page-locked (pinned) inputs
        and outputs make the copies asynchronous; ``out`` defaults to pinned
        buffers.  Returns after the results have landed in host memory."""
        dev = self.device
        u = _as_host(u, torch.int32)
        v = _as_host(v, torch.int32)
        w = _as_host(w, torch.float64)
        n, nv = int(u.shape[0]), int(num_vertices)
        if v.shape[0] != n or w.shape[0] != n:
            raise ValueError("edge arrays have mismatched lengths")
        if out is None:
            out = HostBuildResult.empty(n, nv)
        with torch.cuda.device(dev):
            ws = self.host_workspace(n, nv) if n >= 1 and nv >= 2 else torch.empty(1, dtype=torch.uint8, device=dev)
            st = _lib.DmstStats()
            st.profile = 1 if profile else 0
            st.set_paths(paths)
            _lib.check(self.lib.dmst_build_host(
                _ptr(u), _ptr(v), _ptr(w), n, nv, _ptr(out.orig_of), _ptr(out.heights),
                _ptr(out.edge_parent), _ptr(out.vertex_parent), ctypes.byref(st),
                _ptr(ws), ws.numel(), self._stream()))
        out.stats = st
        return out

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def build(self, num_vertices: int, u, v, w, *, out: BuildResult | None = None,
              debug: bool = False, profile: bool = False, want_chains: bool = False,
              paths: dict | None = None) -> BuildResult:
        """rank_edges + pandora on device tensors (dmst_build).  ``paths``
        overrides the size-based code-path choices (dmst_stats in-fields:
        tail_edges, direct_mi_bytes, sort1_mode, sort2_geometry); results are
        identical for every setting, the path taken is in ``stats.path_info()``."""
        dev = self.device
        with torch.cuda.device(dev):
            u = _as_dev(u, torch.int32, dev)
            v = _as_dev(v, torch.int32, dev)
            w = _as_dev(w, torch.float64, dev)
            n = int(u.shape[0])
            nv = int(num_vertices)
            if v.shape[0] != n or w.shape[0] != n:
                raise ValueError("edge arrays have mismatched lengths")
            if out is None:
                out = BuildResult(
                    orig_of=torch.empty(n, dtype=torch.int32, device=dev),
                    heights=torch.empty(n, dtype=torch.float64, device=dev),
                    edge_parent=torch.empty(n, dtype=torch.int32, device=dev),
                    vertex_parent=torch.empty(max(nv, 0), dtype=torch.int32, device=dev))
            ws = self.workspace(n, nv) if n >= 1 and nv >= 2 else torch.empty(1, dtype=torch.uint8, device=dev)
            st = _lib.DmstStats()
            st.profile = 1 if profile else 0
            st.want_chains = 1 if want_chains else 0
            st.set_paths(paths)
            if debug:
                dbg = {"retirement": torch.empty(n, dtype=torch.int8, device=dev),
                       "chain_key": torch.empty(n, dtype=torch.int32, device=dev),
                       "chain_terminal": torch.empty(n, dtype=torch.int32, device=dev),
                       "chain_level": torch.empty(n, dtype=torch.int32, device=dev)}
                rc = self.lib.dmst_build_debug(
                    _ptr(u), _ptr(v), _ptr(w), n, nv, _ptr(out.orig_of), _ptr(out.heights),
                    _ptr(out.edge_parent), _ptr(out.vertex_parent), ctypes.byref(st),
                    _ptr(dbg["retirement"]), _ptr(dbg["chain_key"]), _ptr(dbg["chain_terminal"]),
                    _ptr(dbg["chain_level"]), _ptr(ws), ws.numel(), self._stream())
                out.debug = dbg
            else:
                rc = self.lib.dmst_build(
                    _ptr(u), _ptr(v), _ptr(w), n, nv, _ptr(out.orig_of), _ptr(out.heights),
                    _ptr(out.edge_parent), _ptr(out.vertex_parent), ctypes.byref(st),
                    _ptr(ws), ws.numel(), self._stream())
            _lib.check(rc)
            out.stats = st
            return out

    def rank_edges(self, num_vertices: int, u, v, w):
        """-> (orig_of, heights, ru, rv) device int32/float64 tensors."""
        dev = self.device
        with torch.cuda.device(dev):
            u = _as_dev(u, torch.int32, dev)
            v = _as_dev(v, torch.int32, dev)
            w = _as_dev(w, torch.float64, dev)
            n = int(u.shape[0])
            orig_of = torch.empty(n, dtype=torch.int32, device=dev)
            heights = torch.empty(n, dtype=torch.float64, device=dev)
            ru = torch.empty(n, dtype=torch.int32, device=dev)
            rv = torch.empty(n, dtype=torch.int32, device=dev)
            ws = self.workspace(n, int(num_vertices))
            _lib.check(self.lib.dmst_rank_edges(
                _ptr(u), _ptr(v), _ptr(w), n, int(num_vertices), _ptr(orig_of), _ptr(heights),
                _ptr(ru), _ptr(rv), _ptr(ws), ws.numel(), self._stream()))
            return orig_of, heights, ru, rv

    def pandora(self, num_vertices: int, ru, rv, paths: dict | None = None):
        """-> (edge_parent, vertex_parent, stats) from rank-order endpoints."""
        dev = self.device
        with torch.cuda.device(dev):
            ru = _as_dev(ru, torch.int32, dev)
            rv = _as_dev(rv, torch.int32, dev)
            n = int(ru.shape[0])
            nv = int(num_vertices)
            ep = torch.empty(n, dtype=torch.int32, device=dev)
            vp = torch.empty(nv, dtype=torch.int32, device=dev)
            ws = self.workspace(n, nv)
            st = _lib.DmstStats()
            st.set_paths(paths)
            _lib.check(self.lib.dmst_pandora(_ptr(ru), _ptr(rv), n, nv, _ptr(ep), _ptr(vp),
                                             ctypes.byref(st), _ptr(ws), ws.numel(), self._stream()))
            return ep, vp, st


_TREE_MESSAGES = {  # tree_core.py:116-138, verbatim
    1: "a tree needs at least 2 vertices",
    2: "edge count {n} != numVertices - 1 = {nv1}",
    3: "non-finite weight on edge {bad}",
    4: "negative vertex id",
    5: "vertex id out of range",
    6: "self-loop on edge {bad}",
    7: "duplicate undirected edge",
    8: "input is disconnected or cyclic, not a tree",
}


def _validate(builder: "DendrogramBuilder", num_vertices: int, u, v, w) -> None:
    """Raise the reference's TreeFormatError (same message) if (u, v, w) is
    not a valid spanning tree on num_vertices vertices (weighted_tree,
    tree_core.py:110-139), checked on the device by dmst_validate."""
    err = _tree_format_error()
    n, nv = int(u.shape[0]), int(num_vertices)
    if nv < 2:
        raise err(_TREE_MESSAGES[1])
    if n != nv - 1:
        raise err(_TREE_MESSAGES[2].format(n=n, nv1=nv - 1))
    if v.shape[0] != n or w.shape[0] != n:
        raise err("edge arrays have mismatched lengths")
    dev = builder.device
    wt = _as_dev(w, torch.float64, dev)
    ids = []
    for a in (u, v):  # int64 ids outside int32 are range errors decided on the host
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        if t.dtype != torch.int32:
            lo, hi = (int(t.min()), int(t.max())) if n else (0, -1)
            if lo < -(1 << 31) or hi >= (1 << 31):
                ids = None
                break
        ids.append(_as_dev(t, torch.int32, dev))
    kind = ctypes.c_int32(0)
    bad = ctypes.c_int64(-1)
    with torch.cuda.device(dev):
        if ids is None:  # ids that do not fit int32: negative or out of range, after the weight check
            finite = torch.isfinite(wt)
            if not bool(finite.all()):
                raise err(_TREE_MESSAGES[3].format(bad=int((~finite).nonzero()[0, 0])))
            neg = any(int(torch.as_tensor(a).min()) < 0 for a in (u, v))
            raise err(_TREE_MESSAGES[4] if neg else _TREE_MESSAGES[5])
        ws = builder.workspace(n, nv)
        _lib.check(builder.lib.dmst_validate(_ptr(ids[0]), _ptr(ids[1]), _ptr(wt), n, nv, ctypes.byref(kind),
                                             ctypes.byref(bad), _ptr(ws), ws.numel(), builder._stream()))
    if kind.value:
        raise err(_TREE_MESSAGES[kind.value].format(n=n, nv1=nv - 1, bad=bad.value))


_builders: dict[tuple[int, int], DendrogramBuilder] = {}


def _builder(device=None) -> DendrogramBuilder:
    """The module-level helpers' builder: one per (device, host thread), so
    concurrent callers never share a workspace (dmst.h: concurrent calls need
    different workspaces and streams)."""
    dev = _device_of(device)
    key = (dev.index, threading.get_ident())
    b = _builders.get(key)
    if b is None:
        b = _builders[key] = DendrogramBuilder(dev)
    return b


def weighted_tree_b200(num_vertices: int, u, v, w, device=None) -> WeightedTree:
    """Drop-in for ``weighted_tree`` (tree_core.py:110-139): validate on the
    GPU, raise ``TreeFormatError`` with the reference's message, return the
    tree with the reference's dtypes (int64 ids, float64 weights)."""
    _validate(_builder(device), num_vertices, u, v, w)
    n = int(u.shape[0])
    cpu = lambda a, dt: (a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)).astype(dt)  # noqa: E731
    return WeightedTree(int(num_vertices), cpu(u, np.int64), cpu(v, np.int64), cpu(w, np.float64),
                        np.arange(n, dtype=np.int64))


def validate_b200(num_vertices: int, u, v, w, device=None) -> None:
    """Validation only (no host copies of the arrays)."""
    _validate(_builder(device), num_vertices, u, v, w)


def dendrogram_height_b200(edge_parent: torch.Tensor, device=None) -> int:
    """Drop-in for ``dendrogram_height`` (analysis.py:21-33) on a device
    edge_parent tensor (int32, rank space, ROOT = -1): pointer jumping."""
    b = _builder(device)
    ep = _as_dev(edge_parent, torch.int32, b.device)
    n = int(ep.shape[0])
    ws = b.workspace(max(n, 1), max(n, 1) + 1)
    h = ctypes.c_int64(0)
    with torch.cuda.device(b.device):
        _lib.check(b.lib.dmst_dendrogram_height(_ptr(ep), n, ctypes.byref(h), _ptr(ws), ws.numel(), b._stream()))
    return int(h.value)


def stats_b200(num_vertices: int, u, v, w, device=None) -> dict:
    """The report of ``dendromst stats`` (cli.py:97-135) for (u, v, w):
    edges, vertices, levels, height, chains, both skewness figures and the
    per-level kind counts, computed on the GPU (build with chain counting,
    then dendrogram_height on the device edge_parent)."""
    import math
    b = _builder(device)
    res = b.build(num_vertices, u, v, w, want_chains=True)
    n = int(res.edge_parent.shape[0])
    height = dendrogram_height_b200(res.edge_parent, device=b.device)
    return {"edges": n, "vertices": int(num_vertices), "levels": res.num_levels, "height": height,
            "chains": int(res.stats.num_chains),
            "skewness_log2_edges": height / math.log2(n) if n >= 2 else 0.0,
            "skewness_log2_points": height / math.log2(n + 1),
            "per_level": res.view_kind_counts}


def format_dendrogram_b200(edge_parent, vertex_parent, device=None) -> torch.Tensor:
    """The dendrogram text format v1 file (write_dendrogram, dendro_io.py:28-38)
    formatted on the GPU: header + "E <rank> <parent>" / "V <id> <parent>"
    lines, as a uint8 DEVICE tensor (byte-identical to the reference's file)."""
    b = _builder(device)
    dev = b.device
    ep = _as_dev(edge_parent, torch.int32, dev)
    vp = _as_dev(vertex_parent, torch.int32, dev)
    n, nv = int(ep.shape[0]), int(vp.shape[0])
    head = f"#dendrogram v1 n={n} nv={nv}\n".encode()
    lines = n + nv
    ws = torch.empty(8 * ((lines + 2047) // 2048 + 2), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        size = int(b.lib.dmst_format_dendrogram(_ptr(ep), _ptr(vp), n, nv, None, 0, _ptr(ws), ws.numel(),
                                                b._stream()))
        if size < 0:
            _lib.check(-1)
        out = torch.empty(len(head) + size, dtype=torch.uint8, device=dev)
        out[:len(head)] = torch.frombuffer(bytearray(head), dtype=torch.uint8).to(dev)
        body = out[len(head):]
        got = int(b.lib.dmst_format_dendrogram(_ptr(ep), _ptr(vp), n, nv, _ptr(body) if size else None, size,
                                               _ptr(ws), ws.numel(), b._stream()))
        if got != size:
            _lib.check(-1)
    return out


_STAGE: dict[tuple[int, int], list] = {}  # pinned staging buffers per (device, host thread)


def sidecar_path(path) -> str:
    """Binary sidecar of a v1 dendrogram file: ``<path>.npy``, one int32
    array = edge_parent, then vertex_parent, then an 8-word binding to the
    text file it was written with."""
    return os.fspath(path) + ".npy"


_SIDECAR_MAGIC = 0x31524344  # "DCR1"


def _text_binding(path) -> np.ndarray:
    """(magic, size, mtime_ns, inode) of the text file as 4 int64 = 8 int32:
    a sidecar is used only while the text file is exactly the one it was
    written beside (a rewrite by any writer changes mtime_ns, and usually size)."""
    st = os.stat(path)
    return np.array([_SIDECAR_MAGIC, st.st_size, st.st_mtime_ns, st.st_ino], dtype=np.int64).view(np.int32)


def write_dendrogram_b200(path, edge_parent, vertex_parent, device=None, chunk_bytes: int = 64 << 20,
                          sidecar: bool = False) -> int:
    """Drop-in for ``write_dendrogram`` (dendro_io.py:28-38): the same bytes,
    formatted on the GPU and streamed to the file through two reusable pinned
    host buffers (the copy of chunk k + 1 overlaps the write of chunk k).
    With ``sidecar`` the parent arrays are also saved as ``<path>.npy``
    (4 B per node instead of ~20 B of text), which ``read_dendrogram_b200``
    loads instead of parsing when it is at least as new as the text file.
    Returns the text file size."""
    dev_bytes = format_dendrogram_b200(edge_parent, vertex_parent, device=device)
    total = int(dev_bytes.numel())
    dev = dev_bytes.device
    key = (dev.index, threading.get_ident())
    bufs = _STAGE.get(key)
    if bufs is None or bufs[0].numel() < chunk_bytes:
        bufs = _STAGE[key] = [torch.empty(chunk_bytes, dtype=torch.uint8).pin_memory() for _ in range(2)]
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    stream = torch.cuda.current_stream(dev)
    with open(path, "wb") as f:
        offs = list(range(0, total, chunk_bytes))

        def issue(k):
            lo = offs[k]
            hi = min(total, lo + chunk_bytes)
            bufs[k & 1][:hi - lo].copy_(dev_bytes[lo:hi], non_blocking=True)
            evs[k & 1].record(stream)
        if offs:
            issue(0)
        for k, lo in enumerate(offs):
            if k + 1 < len(offs):
                issue(k + 1)
            evs[k & 1].synchronize()
            hi = min(total, lo + chunk_bytes)
            f.write(memoryview(bufs[k & 1].numpy())[:hi - lo])
    side = sidecar_path(path)
    if sidecar:
        both = torch.cat([torch.as_tensor(edge_parent).reshape(-1).to(dev, torch.int32),
                          torch.as_tensor(vertex_parent).reshape(-1).to(dev, torch.int32)]).cpu().numpy()
        with open(side, "wb") as f:
            np.save(f, np.concatenate([both, _text_binding(path)]))
    elif os.path.exists(side):
        os.remove(side)  # a sidecar of an older file must not outlive it
    return total


class DendrogramFormatError(ValueError):
    """Mirror of ``dendromst.dendro_io.DendrogramFormatError`` (the reference's
    own class is raised when it is importable)."""


def _format_error():
    try:
        from dendromst.dendro_io import DendrogramFormatError as Ref  # type: ignore
        return Ref
    except Exception:
        return DendrogramFormatError


def read_dendrogram_b200(path, device=None, use_sidecar: bool = True) -> BuildResult:
    """Drop-in for ``read_dendrogram`` (dendro_io.py:41-75): the header is
    checked on the host (same messages), the body is parsed on the GPU
    (dmst_parse_dendrogram) straight into device edge_parent / vertex_parent
    tensors (returned in a BuildResult with orig_of / heights = None).
    Lines must use single spaces and '\\n' endings (what write_dendrogram and
    write_dendrogram_b200 produce); a malformed line raises
    DendrogramFormatError("bad line: ...").  A ``<path>.npy`` sidecar
    (write_dendrogram_b200(sidecar=True)) is loaded instead of parsing the
    body when its size matches the header and its binding (size, mtime_ns,
    inode of the text file when the sidecar was written) matches the text
    file as it is now."""
    err = _format_error()
    b = _builder(device)
    dev = b.device
    side = sidecar_path(path)
    if use_sidecar and os.path.exists(side):
        with open(path, "rb") as f:
            first = f.readline()
        parts = first.decode(errors="replace").split()
        if len(parts) == 4 and parts[0] == "#dendrogram" and parts[1] == "v1":
            try:
                n, nv = int(parts[2][2:]), int(parts[3][3:])
                arr = np.load(side, mmap_mode="r")
            except (ValueError, OSError):
                arr = None
            if (arr is not None and arr.dtype == np.int32 and arr.shape == (n + nv + 8,)
                    and np.array_equal(arr[n + nv:], _text_binding(path))):
                both = torch.from_numpy(np.array(arr[:n + nv])).to(dev)
                return BuildResult(orig_of=None, heights=None, edge_parent=both[:n], vertex_parent=both[n:])
    with open(path, "rb") as f:
        data = f.read()
    nl = data.find(b"\n")
    header = (data if nl < 0 else data[:nl]).decode(errors="replace").strip()
    parts = header.split()
    if (len(parts) != 4 or parts[0] != "#dendrogram" or parts[1] != "v1"
            or not parts[2].startswith("n=") or not parts[3].startswith("nv=")):
        raise err(f"bad header: {header!r}")
    try:
        n = int(parts[2][2:])
        nv = int(parts[3][3:])
    except ValueError:
        raise err(f"bad header: {header!r}") from None
    body = memoryview(data)[nl + 1:] if nl >= 0 else memoryview(b"")
    blen = len(body)
    host = torch.frombuffer(bytearray(body), dtype=torch.uint8) if blen else torch.empty(0, dtype=torch.uint8)
    with torch.cuda.device(dev):
        dbody = host.to(dev)
        ep = torch.empty(max(n, 0), dtype=torch.int32, device=dev)
        vp = torch.empty(max(nv, 0), dtype=torch.int32, device=dev)
        ws = torch.empty(int(b.lib.dmst_parse_workspace_bytes(blen, max(n, 0), max(nv, 0))) or 64,
                         dtype=torch.uint8, device=dev)
        bad, ne, nvl = ctypes.c_int64(-1), ctypes.c_int64(0), ctypes.c_int64(0)
        _lib.check(b.lib.dmst_parse_dendrogram(_ptr(dbody) if blen else None, blen, n, nv, _ptr(ep), _ptr(vp),
                                               ctypes.byref(bad), ctypes.byref(ne), ctypes.byref(nvl),
                                               _ptr(ws), ws.numel(), b._stream()))
    if bad.value >= 0:
        line = bytes(body).split(b"\n")[bad.value].decode(errors="replace")
        raise err(f"bad line: {line!r}")
    if ne.value != n or nvl.value != nv:
        raise err(f"expected {n} edge and {nv} vertex lines, got {ne.value} and {nvl.value}")
    return BuildResult(orig_of=None, heights=None, edge_parent=ep, vertex_parent=vp)


def verify_b200(path_a, path_b, device=None, use_sidecar: bool = False) -> tuple[int, str]:
    """``dendromst verify a b`` (cli.py:138-155) with the files parsed and
    compared on the GPU: returns (exit code, the line the reference prints).
    The text files themselves are compared unless ``use_sidecar``."""
    da = read_dendrogram_b200(path_a, device=device, use_sidecar=use_sidecar)
    db = read_dendrogram_b200(path_b, device=device, use_sidecar=use_sidecar)
    b = _builder(device)
    ws = torch.empty(64, dtype=torch.uint8, device=b.device)
    for label, pa, pb in (("edge", da.edge_parent, db.edge_parent),
                          ("vertex", da.vertex_parent, db.vertex_parent)):
        if pa.shape != pb.shape:
            return 1, f"size mismatch: {pa.shape[0]} vs {pb.shape[0]} {label} nodes"
        first = ctypes.c_int64(-1)
        with torch.cuda.device(b.device):
            _lib.check(b.lib.dmst_first_difference(_ptr(pa), _ptr(pb), int(pa.shape[0]), ctypes.byref(first),
                                                   _ptr(ws), ws.numel(), b._stream()))
        if first.value >= 0:
            i = first.value
            return 1, f"first divergence: {label} {i}: {int(pa[i])} != {int(pb[i])}"
    return 0, "identical"


_ENGINES = {"auto": 0, "numba": 1, "numpy": 2}


def mutual_reachability_mst_b200(coords, min_pts: int = 2, engine: str = "auto", device=None,
                                 return_core_sq: bool = False):
    """Drop-in for ``mutual_reachability_mst`` (pointgen.py:158-178) on the
    GPU: core distances by brute-force k-NN in cKDTree's summation order,
    then the dense Prim scan of the chosen engine (same tie-breaking, same
    discovery order = original edge ids).  ``coords``: (n, dim) float64
    array or tensor, dim <= 8, min_pts <= 16 on the device.  Returns a
    WeightedTree whose u, v (int32) and w (float64) are DEVICE tensors, the
    input of DendrogramBuilder.build (+ core_sq with return_core_sq)."""
    x = torch.as_tensor(coords)
    if x.dim() != 2:
        raise ValueError("coords must be (n, dim)")
    n, dim = int(x.shape[0]), int(x.shape[1])
    if not 2 <= min_pts <= n:
        raise ValueError(f"min_pts must be in [2, {n}]")
    if engine not in _ENGINES:
        raise ValueError(f"unknown engine {engine!r}")
    if min_pts > 16 or not 1 <= dim <= 8:
        raise ValueError("the device producer supports min_pts <= 16 and 1 <= dim <= 8")
    b = _builder(device)
    dev = b.device
    with torch.cuda.device(dev):
        x = x.to(dev, torch.float64).contiguous()
        u = torch.empty(n - 1, dtype=torch.int32, device=dev)
        v = torch.empty(n - 1, dtype=torch.int32, device=dev)
        w = torch.empty(n - 1, dtype=torch.float64, device=dev)
        core = torch.empty(n, dtype=torch.float64, device=dev)
        ws = torch.empty(int(b.lib.dmst_mreach_workspace_bytes(n, dim)), dtype=torch.uint8, device=dev)
        _lib.check(b.lib.dmst_mreach_mst(_ptr(x), n, dim, int(min_pts), _ENGINES[engine], _ptr(u), _ptr(v), _ptr(w),
                                         _ptr(core), _ptr(ws), ws.numel(), b._stream()))
    tree = WeightedTree(n, u, v, w, torch.arange(n - 1, device=dev))
    return (tree, core) if return_core_sq else tree


def build_b200(num_vertices: int, u, v, w, device=None, debug: bool = False) -> BuildResult:
    """rank_edges + pandora on the GPU (the timed scope of `dendromst build`)."""
    return _builder(device).build(num_vertices, u, v, w, debug=debug)


def rank_edges_b200(tree, device=None) -> RankedTree:
    """Drop-in for ``rank_edges`` (tree_core.py:174-190) on a WeightedTree-like
    object (``num_vertices``, ``u``, ``v``, ``w``)."""
    orig_of, heights, ru, rv = _builder(device).rank_edges(tree.num_vertices, tree.u, tree.v, tree.w)
    order = orig_of.cpu().numpy().astype(np.int64)
    rank_of = np.empty_like(order)
    rank_of[order] = np.arange(order.shape[0])
    return RankedTree(base=tree, rank_of=rank_of, orig_of=order,
                      u=ru.cpu().numpy().astype(np.int64), v=rv.cpu().numpy().astype(np.int64),
                      w=heights.cpu().numpy())


def pandora_b200(tree, device=None):
    """Drop-in for ``pandora`` (expansion.py:148-153) with the ``_ALGOS``
    signature: RankedTree-like (``num_vertices``, rank-order ``u``, ``v``)
    -> Dendrogram (the reference's own class when it is importable)."""
    ep, vp, _ = _builder(device).pandora(tree.num_vertices, tree.u, tree.v)
    cls = _reference_dendrogram_type() or Dendrogram
    return cls(edge_parent=ep.cpu().numpy().astype(np.int64),
               vertex_parent=vp.cpu().numpy().astype(np.int64))


def register_algorithm(registry: dict | None = None, name: str = "pandora_b200") -> dict:
    """Install :func:`pandora_b200` into the reference's algorithm registry
    (``dendromst.cli._ALGOS``, cli.py:27-31) so ``dendromst build/bench
    --algo pandora_b200`` runs on the GPU.  The CLI builds its choices from
    ``_ALGOS`` at parse time (cli.py:200, :218)."""
    if registry is None:
        from dendromst import cli  # type: ignore
        registry = cli._ALGOS
    registry[name] = pandora_b200
    return registry

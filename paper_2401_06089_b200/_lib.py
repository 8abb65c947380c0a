"""ctypes binding of the C ABI declared in include/dmst.h.

The shared library is built in-tree (paper_2401_06089_b200/libdmst.so, by
__graft_entry__.build() or `python -m paper_2401_06089_b200.build`).  There
is deliberately no CPU fallback: if the library is missing this module
raises, loudly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdmst.so")

DMST_EINVAL = 22
DMST_ECUDA = -1
DMST_MAX_LEVELS = 64
DMST_MAX_KERNELS = 24
SORT2_GEOMETRIES = {0: None, 1: "512x16", 2: "256x20"}

# every symbol include/dmst.h declares
EXPORTS = (
    "dmst_workspace_bytes",
    "dmst_host_workspace_bytes",
    "dmst_build",
    "dmst_build_host",
    "dmst_rank_edges",
    "dmst_pandora",
    "dmst_build_debug",
    "dmst_validate",
    "dmst_dendrogram_height",
    "dmst_format_dendrogram",
    "dmst_parse_workspace_bytes",
    "dmst_parse_dendrogram",
    "dmst_first_difference",
    "dmst_mreach_workspace_bytes",
    "dmst_mreach_mst",
    "dmst_last_error",
    "dmst_kernel_name",
    "dmst_version",
)


class DmstStats(ctypes.Structure):
    _fields_ = [
        ("profile", ctypes.c_int32),
        ("num_levels", ctypes.c_int32),
        ("level_counts", (ctypes.c_int32 * 4) * (DMST_MAX_LEVELS + 1)),
        ("view_vertices", ctypes.c_int32 * (DMST_MAX_LEVELS + 1)),
        ("sort1_passes", ctypes.c_int32),
        ("sort2_passes", ctypes.c_int32),
        ("jump_rounds", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int32),
        ("want_chains", ctypes.c_int32),
        ("num_chains", ctypes.c_int32),
        ("kernel_ms", ctypes.c_float * DMST_MAX_KERNELS),
        ("kernel_calls", ctypes.c_int32 * DMST_MAX_KERNELS),
        ("tail_edges", ctypes.c_int64),
        ("direct_mi_bytes", ctypes.c_int64),
        ("sort1_mode", ctypes.c_int32),
        ("sort2_geometry", ctypes.c_int32),
        ("mi_apply_mode", ctypes.c_int32),
        ("sort1_narrow", ctypes.c_int32),
        ("sort1_compacted", ctypes.c_int32),
        ("sort2_geometry_used", ctypes.c_int32),
        ("tail_level", ctypes.c_int32),
        ("sort1_local", ctypes.c_int32),
        ("mi_sliced", ctypes.c_int32),
        ("mi_bucketed", ctypes.c_uint64),
        ("mi_direct", ctypes.c_uint64),
        ("v0_select", ctypes.c_int32),
        ("v0_chase", ctypes.c_int32),
    ]

    # code-path overrides accepted by DendrogramBuilder.build(paths=...)
    PATH_OPTIONS = ("tail_edges", "direct_mi_bytes", "sort1_mode", "sort2_geometry", "mi_apply_mode",
                    "v0_select")

    def set_paths(self, paths: dict | None) -> None:
        for k, v in (paths or {}).items():
            if k not in self.PATH_OPTIONS:
                raise ValueError(f"unknown path option {k!r} (have {self.PATH_OPTIONS})")
            setattr(self, k, int(v))

    def path_info(self) -> dict:
        """Which code path each stage took (bench.py's byte model reads this)."""
        L = int(self.num_levels)
        return {"sort1_passes": int(self.sort1_passes), "sort1_narrow": bool(self.sort1_narrow),
                "sort1_compacted": bool(self.sort1_compacted),
                "sort1_local": {0: None, 1: "smem", 2: "fallback"}[int(self.sort1_local)],
                "mi_sliced": bool(self.mi_sliced),
                "v0_chase": {0: None, 1: "chase", 2: "chase+fix"}[int(self.v0_chase)],
                "sort2_passes": int(self.sort2_passes),
                "sort2_geometry": SORT2_GEOMETRIES[int(self.sort2_geometry_used)],
                "tail_level": int(self.tail_level),
                "mi_bucketed_views": [k for k in range(L + 1) if (int(self.mi_bucketed) >> k) & 1],
                "mi_direct_views": [k for k in range(L + 1) if (int(self.mi_direct) >> k) & 1]}

    def kernel_profile(self) -> dict[str, tuple[float, int]]:
        """{kernel kind: (device ms, launches)} when profile=1 was set."""
        lib = load()
        out = {}
        for i in range(DMST_MAX_KERNELS):
            if self.kernel_calls[i]:
                out[lib.dmst_kernel_name(i).decode()] = (float(self.kernel_ms[i]), int(self.kernel_calls[i]))
        return out

    def view_kind_counts(self) -> list[tuple[int, int, int, int]]:
        """ContractionHierarchy.view_kind_counts (contraction.py:127-131)."""
        return [tuple(int(x) for x in self.level_counts[k])
                for k in range(self.num_levels + 1)]


class DmstError(RuntimeError):
    pass


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t
    lib.dmst_workspace_bytes.argtypes = [i64, i64]
    lib.dmst_workspace_bytes.restype = sz
    lib.dmst_build.argtypes = [vp, vp, vp, i64, i64, vp, vp, vp, vp,
                               ctypes.POINTER(DmstStats), vp, sz, vp]
    lib.dmst_build.restype = ctypes.c_int
    lib.dmst_host_workspace_bytes.argtypes = [i64, i64]
    lib.dmst_host_workspace_bytes.restype = sz
    lib.dmst_build_host.argtypes = [vp, vp, vp, i64, i64, vp, vp, vp, vp,
                                    ctypes.POINTER(DmstStats), vp, sz, vp]
    lib.dmst_build_host.restype = ctypes.c_int
    lib.dmst_build_debug.argtypes = [vp, vp, vp, i64, i64, vp, vp, vp, vp,
                                     ctypes.POINTER(DmstStats), vp, vp, vp, vp, vp, sz, vp]
    lib.dmst_build_debug.restype = ctypes.c_int
    lib.dmst_rank_edges.argtypes = [vp, vp, vp, i64, i64, vp, vp, vp, vp, vp, sz, vp]
    lib.dmst_rank_edges.restype = ctypes.c_int
    lib.dmst_pandora.argtypes = [vp, vp, i64, i64, vp, vp, ctypes.POINTER(DmstStats), vp, sz, vp]
    lib.dmst_pandora.restype = ctypes.c_int
    lib.dmst_validate.argtypes = [vp, vp, vp, i64, i64, ctypes.POINTER(ctypes.c_int32),
                                  ctypes.POINTER(ctypes.c_int64), vp, sz, vp]
    lib.dmst_validate.restype = ctypes.c_int
    lib.dmst_dendrogram_height.argtypes = [vp, i64, ctypes.POINTER(ctypes.c_int64), vp, sz, vp]
    lib.dmst_dendrogram_height.restype = ctypes.c_int
    lib.dmst_format_dendrogram.argtypes = [vp, vp, i64, i64, vp, sz, vp, sz, vp]
    lib.dmst_format_dendrogram.restype = ctypes.c_int64
    p64 = ctypes.POINTER(ctypes.c_int64)
    lib.dmst_parse_workspace_bytes.argtypes = [i64, i64, i64]
    lib.dmst_parse_workspace_bytes.restype = sz
    lib.dmst_parse_dendrogram.argtypes = [vp, i64, i64, i64, vp, vp, p64, p64, p64, vp, sz, vp]
    lib.dmst_parse_dendrogram.restype = ctypes.c_int
    lib.dmst_first_difference.argtypes = [vp, vp, i64, p64, vp, sz, vp]
    lib.dmst_first_difference.restype = ctypes.c_int
    lib.dmst_mreach_workspace_bytes.argtypes = [i64, ctypes.c_int32]
    lib.dmst_mreach_workspace_bytes.restype = sz
    i32 = ctypes.c_int32
    lib.dmst_mreach_mst.argtypes = [vp, i64, i32, i32, i32, vp, vp, vp, vp, vp, sz, vp]
    lib.dmst_mreach_mst.restype = ctypes.c_int
    lib.dmst_last_error.argtypes = []
    lib.dmst_last_error.restype = ctypes.c_char_p
    lib.dmst_kernel_name.argtypes = [ctypes.c_int32]
    lib.dmst_kernel_name.restype = ctypes.c_char_p
    lib.dmst_version.argtypes = []
    lib.dmst_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().dmst_last_error().decode(errors="replace")
        if rc == DMST_EINVAL:
            raise ValueError(msg)
        raise DmstError(f"dmst error {rc}: {msg}")

"""B200-native PANDORA dendrogram construction (arXiv 2401.06089).

MST edge arrays (u, v, w) -> rank-space dendrogram (edge_parent,
vertex_parent) + merge heights, bit-identical to the reference
`dendromst` package, on hand-written sm_100a CUDA kernels behind a C ABI
(include/dmst.h).  See DESIGN.md.
"""
from .api import (ROOT, BuildResult, Dendrogram, DendrogramBuilder, HostBuildResult, RankedTree,
                  TreeFormatError, WeightedTree, build_b200, pandora_b200, rank_edges_b200,
                  dendrogram_height_b200, format_dendrogram_b200, register_algorithm, stats_b200,
                  mutual_reachability_mst_b200, read_dendrogram_b200, sidecar_path, validate_b200, verify_b200, weighted_tree_b200,
                  write_dendrogram_b200)

__all__ = ["ROOT", "BuildResult", "Dendrogram", "DendrogramBuilder", "HostBuildResult", "RankedTree",
           "TreeFormatError", "WeightedTree", "validate_b200", "weighted_tree_b200",
           "dendrogram_height_b200", "stats_b200", "format_dendrogram_b200", "write_dendrogram_b200",
           "read_dendrogram_b200", "verify_b200", "sidecar_path", "mutual_reachability_mst_b200",
           "build_b200", "pandora_b200", "rank_edges_b200", "register_algorithm"]
__version__ = "0.1.0"

/*
 * dmst — B200-native PANDORA dendrogram construction, C ABI.
 *
 * Drop-in boundary for the reference hot path of arxiv/paper_2401_06089's
 * `dendromst` package (paths relative to /root/reference/pkg/src/dendromst/):
 *
 *   dmst_rank_edges  replaces  rank_edges(tree) -> RankedTree     tree_core.py:174-190
 *   dmst_pandora     replaces  pandora(ranked) -> Dendrogram      expansion.py:148-153
 *                              (build_incidence tree_core.py:193-199, vertex_parents
 *                               classify.py:23-25, build_hierarchy contraction.py:186-219,
 *                               assign_chains expansion.py:97-128, stitch_chains :131-145)
 *   dmst_build       replaces  the timed scope of `dendromst build`:
 *                              rank_edges + _ALGOS["pandora"]      cli.py:82-85 (`_cmd_build`)
 *
 * Conventions (all identical to the reference):
 *   - rank r = position after a stable descending-weight sort; ties by
 *     ascending original id; -0.0 ties with +0.0 (numpy `<` semantics).
 *   - orig_of[r]       = original edge id of rank r      (RankedTree.orig_of)
 *   - heights[r]       = w[orig_of[r]], bitwise copy      (RankedTree.w)
 *   - edge_parent[r]   in [-1, r-1], -1 = ROOT            (Dendrogram.edge_parent)
 *   - vertex_parent[x] = largest incident rank            (Dendrogram.vertex_parent)
 *   Device dtypes are int32 ids/ranks and float64 weights; the Python
 *   wrapper widens to the reference's int64.
 *
 * Every pointer except `stats` is a DEVICE pointer (dmst_build_host takes
 * HOST buffers instead).  The caller allocates every device buffer, including
 * the workspace (size from dmst_workspace_bytes); the library never allocates
 * device memory and keeps no data between calls (it caches CUDA events, and
 * for dmst_build_host one side stream, per host thread).  Inputs are read-only.  Work is
 * enqueued on `stream`; the call returns after the stream has drained
 * (the contraction level loop sizes each level from device counts).
 * Calls on different streams with different workspaces may run
 * concurrently; results are bit-identical across runs and streams.
 *
 * Return value: 0 on success, DMST_EINVAL (22) on bad sizes/pointers,
 * DMST_ECUDA (-1) on a CUDA error; the message is in dmst_last_error()
 * (thread-local).  The input must already be a valid spanning tree
 * (validation is the caller's, tree_core.py:110-139, as in the reference,
 * whose `pandora` raises nothing itself — SPEC.md:265).
 * Limits: 1 <= n_edges < 2^29, n_vertices == n_edges + 1.
 */
#ifndef DMST_H
#define DMST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DMST_EINVAL 22
#define DMST_ECUDA (-1)
#define DMST_MAX_LEVELS 64

#define DMST_MAX_KERNELS 24

/* Per-call diagnostics (host memory, optional).  Set `profile` = 1 before
 * the call to have every kernel bracketed by CUDA events on `stream`;
 * kernel_ms / kernel_calls then hold per-kernel-kind device time and launch
 * counts (names from dmst_kernel_name). */
typedef struct dmst_stats {
  int32_t profile;                           /* in: 1 = record per-kernel events */
  int32_t num_levels;                        /* ContractionHierarchy.num_levels */
  int32_t level_counts[DMST_MAX_LEVELS + 1][4]; /* view_kind_counts: (n_alpha, n_leaf, n_chain, n_k) per view 0..L */
  int32_t view_vertices[DMST_MAX_LEVELS + 1];   /* supervertex count of every view */
  int32_t sort1_passes;                      /* non-constant 8-bit digits sorted in the edge sort */
  int32_t sort2_passes;                      /* digits sorted in the chain sort */
  int32_t jump_rounds;                       /* pointer-jumping rounds over all levels */
  int32_t kernel_launches;                   /* kernels this call enqueued */
  int32_t want_chains;                       /* in: 1 = count the dendrogram chains */
  int32_t num_chains;                        /* out: ChainAssignment.num_chains() (want_chains = 1) */
  float kernel_ms[DMST_MAX_KERNELS];         /* out (profile=1): device ms per kernel kind */
  int32_t kernel_calls[DMST_MAX_KERNELS];    /* out: launches per kernel kind */
  /* in: code-path overrides (0 = the library's size-based default).  They
   * choose WHICH kernels run, never the result: every setting gives the same
   * bits (tests/test_paths_gpu.py), so tests can drive the paths a 128M-edge
   * build takes on trees the oracle checks in seconds. */
  int64_t tail_edges;       /* views >= 1 of at most this many edges finish inside the
                               cooperative k_tail (default and maximum 4M); -1 = never */
  int64_t direct_mi_bytes;  /* views >= 1 whose packed maxIncident (8 B per vertex) is at
                               most this large take direct atomics in k_select_edges + k_v1
                               (default 64 MB); -1 = always bucketed (multisplit + apply) */
  int32_t sort1_mode;       /* bit 0: no narrow 32-bit keys; bit 1: no top-field compaction;
                               bit 2: wide keys never finish in shared memory (full LSD sort) */
  int32_t sort2_geometry;   /* chain-sort tiles: 1 = 512 x 16, 2 = 256 x 20 (two CTAs per SM);
                               0 = by size (2 from 32M edges) */
  int32_t mi_apply_mode;    /* bucketed maxIncident: 1 = two multisplit passes + shared-memory
                               apply per 8192-vertex bucket, 2 = one pass into 4M-vertex slices
                               + L2-resident 64-bit atomics + k_v1; 0 = the library's choice.
                               The link stage follows it: 1 = two passes + shared-memory
                               apply, 2 = one pass into 2M-rank slices + L2-resident stores */
  /* out: the path this call took (what bench.py's byte model reads) */
  int32_t sort1_narrow;     /* 1 = the edge sort ran on 32-bit keys */
  int32_t sort1_compacted;  /* 1 = the sign/exponent field was replaced by its dense code */
  int32_t sort2_geometry_used; /* 0 = no chain sort (a single chain), else as sort2_geometry */
  int32_t tail_level;       /* first view finished inside k_tail, -1 = none */
  int32_t sort1_local;      /* 1 = wide keys: top three digits sorted globally, the rest per
                               window in shared memory; 2 = a window overflowed, full LSD ran */
  int32_t mi_sliced;        /* 1 = some view's maxIncident took the sliced L2-atomic apply */
  uint64_t mi_bucketed;     /* bit k: view k's maxIncident was bucketed */
  uint64_t mi_direct;       /* bit k: view k's maxIncident took direct atomics */
  int32_t v0_select;        /* in: view 0's supervertex labels: 1 = V2 writes the vertex map, the
                               select gathers from it; 2 = the select chases maxIncident from the
                               endpoints it needs (no V2; edges with chases over 16 steps are
                               finished from a V2 vertex map); 0 = by the view's kind counts */
  int32_t v0_chase;         /* out: 1 = view 0's select chased, 2 = and deferred some edges */
} dmst_stats;

/* Workspace size for a tree with n_edges edges. */
size_t dmst_workspace_bytes(int64_t n_edges, int64_t n_vertices);

/* rank_edges + pandora, fused (what `dendromst build` times). */
int dmst_build(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges,
               int64_t n_vertices, int32_t* orig_of, double* heights, int32_t* edge_parent,
               int32_t* vertex_parent, dmst_stats* stats, void* workspace,
               size_t workspace_bytes, void* stream);

/* Device workspace for dmst_build_host (pipeline workspace + device copies
 * of the inputs and outputs). */
size_t dmst_host_workspace_bytes(int64_t n_edges, int64_t n_vertices);

/* dmst_build with HOST buffers: u, v, w, orig_of, heights, edge_parent and
 * vertex_parent are host pointers (page-locked memory gives asynchronous,
 * overlapped copies; pageable memory works but serialises).  The inputs are
 * copied in on a per-thread side stream; each output is copied out as soon
 * as the stage producing it completes (orig_of/heights after the edge sort,
 * vertex_parent after maxIncident, edge_parent at the end), overlapping the
 * copies with the remaining kernels.  Returns when every copy has landed.
 * This is the call a host-side binding of the reference's `dendromst build`
 * path (cli.py:82-85: rank_edges + pandora on numpy arrays) makes. */
int dmst_build_host(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges,
                    int64_t n_vertices, int32_t* orig_of, double* heights, int32_t* edge_parent,
                    int32_t* vertex_parent, dmst_stats* stats, void* workspace,
                    size_t workspace_bytes, void* stream);

/* rank_edges only: orig_of, heights and rank-order endpoints ru/rv. */
int dmst_rank_edges(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges,
                    int64_t n_vertices, int32_t* orig_of, double* heights, int32_t* ru,
                    int32_t* rv, void* workspace, size_t workspace_bytes, void* stream);

/* pandora on an already ranked tree (ru/rv = RankedTree.u/.v). */
int dmst_pandora(const int32_t* ru, const int32_t* rv, int64_t n_edges, int64_t n_vertices,
                 int32_t* edge_parent, int32_t* vertex_parent, dmst_stats* stats,
                 void* workspace, size_t workspace_bytes, void* stream);

/* Debug/introspection variant of dmst_build for per-stage parity tests:
 * additionally copies (device -> the given DEVICE buffers, each nullable)
 *   retirement[n]  ContractionHierarchy.retirement_level (int8 values)
 *   chain_key[n]   dense chain id per edge: 0 = root chain, else
 *                  1 + (offset of view `level`) + anchor supervertex
 *   chain_terminal[n], chain_level[n]  ChainAssignment.terminal / .level
 */
int dmst_build_debug(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges,
                     int64_t n_vertices, int32_t* orig_of, double* heights,
                     int32_t* edge_parent, int32_t* vertex_parent, dmst_stats* stats,
                     int8_t* retirement, int32_t* chain_key, int32_t* chain_terminal,
                     int32_t* chain_level, void* workspace, size_t workspace_bytes,
                     void* stream);

/* Tree validation: the checks of the reference's `weighted_tree`
 * (tree_core.py:110-139), on the device, in the same order:
 *   DMST_TREE_TOO_SMALL   n_vertices < 2                       (:116-117)
 *   DMST_TREE_EDGE_COUNT  n_edges != n_vertices - 1            (:118-121)
 *   DMST_TREE_NONFINITE   non-finite weight; *bad_edge = first (:124-126)
 *   DMST_TREE_NEGATIVE_ID negative vertex id                   (:127-128)
 *   DMST_TREE_ID_RANGE    vertex id >= n_vertices              (:129-130)
 *   DMST_TREE_SELF_LOOP   u == v; *bad_edge = first            (:131-133)
 *   DMST_TREE_DUPLICATE   duplicate undirected edge            (:134-136)
 *   DMST_TREE_NOT_A_TREE  disconnected or cyclic               (:137-138)
 * *error_kind = DMST_TREE_OK (0) for a valid tree.  u, v, w are DEVICE
 * pointers, error_kind / bad_edge HOST pointers; workspace as for
 * dmst_build.  Returns 0 when the check ran (whatever its verdict),
 * DMST_EINVAL / DMST_ECUDA otherwise. */
#define DMST_TREE_OK 0
#define DMST_TREE_TOO_SMALL 1
#define DMST_TREE_EDGE_COUNT 2
#define DMST_TREE_NONFINITE 3
#define DMST_TREE_NEGATIVE_ID 4
#define DMST_TREE_ID_RANGE 5
#define DMST_TREE_SELF_LOOP 6
#define DMST_TREE_DUPLICATE 7
#define DMST_TREE_NOT_A_TREE 8
int dmst_validate(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges, int64_t n_vertices,
                  int32_t* error_kind, int64_t* bad_edge, void* workspace, size_t workspace_bytes,
                  void* stream);

/* dendrogram_height (analysis.py:21-33) of a rank-space edge_parent array
 * (DEVICE pointer, n_edges entries, ROOT = -1): the largest number of edge
 * ancestors of a vertex, by pointer jumping.  *height is a HOST pointer.
 * Workspace: any buffer of at least 16 n_edges + 4096 bytes (e.g. the
 * dmst_build workspace).  Returns DMST_EINVAL when a parent is neither ROOT
 * nor a smaller (heavier) rank, i.e. the array is not a dendrogram. */
int dmst_dendrogram_height(const int32_t* edge_parent, int64_t n_edges, int64_t* height, void* workspace,
                           size_t workspace_bytes, void* stream);

/* Dendrogram text format v1 body (write_dendrogram, dendro_io.py:28-38):
 * "E <rank> <parent>\n" per edge then "V <id> <parent>\n" per vertex,
 * formatted on the device into `out` (DEVICE buffer of out_capacity bytes;
 * NULL = size query).  The header line "#dendrogram v1 n=.. nv=..\n" is the
 * caller's.  Workspace: >= 8 * (ceil((n_edges + n_vertices) / 2048) + 1)
 * bytes.  Returns the body size in bytes, or -1 on error (dmst_last_error). */
int64_t dmst_format_dendrogram(const int32_t* edge_parent, const int32_t* vertex_parent, int64_t n_edges,
                               int64_t n_vertices, char* out, size_t out_capacity, void* workspace,
                               size_t workspace_bytes, void* stream);

/* read_dendrogram (dendro_io.py:41-75) of the body after the header line:
 * `body` (DEVICE, body_len bytes) holds "E <rank> <parent>" / "V <id>
 * <parent>" lines ('#' and blank lines skipped; single spaces, '\n'
 * endings); edge_parent / vertex_parent (DEVICE, n_edges / n_vertices)
 * start at ROOT (-1) and receive every line; an id given on several lines
 * takes the last one's parent, as the reference's in-order assignment does
 * (dendro_io.py:60-66).  HOST outputs: *bad_line = 0-based body line of the
 * first malformed line (-1 if none), and the numbers of E and V lines.
 * Workspace: dmst_parse_workspace_bytes(body_len, n_edges, n_vertices). */
size_t dmst_parse_workspace_bytes(int64_t body_len, int64_t n_edges, int64_t n_vertices);
int dmst_parse_dendrogram(const char* body, int64_t body_len, int64_t n_edges, int64_t n_vertices,
                          int32_t* edge_parent, int32_t* vertex_parent, int64_t* bad_line, int64_t* edge_lines,
                          int64_t* vertex_lines, void* workspace, size_t workspace_bytes, void* stream);

/* First index where two DEVICE int32 arrays of n entries differ (-1: none;
 * `dendromst verify`, cli.py:138-155).  Workspace: 8 bytes. */
int dmst_first_difference(const int32_t* a, const int32_t* b, int64_t n, int64_t* first, void* workspace,
                          size_t workspace_bytes, void* stream);

/* Upstream producer: replaces
 * dendromst.pointgen.mutual_reachability_mst (pointgen.py:158-178) with
 * core_distances (:56-61) and the dense Prim scans (:71-148).
 * coords: DEVICE float64 [n_points][dim] (row-major, 1 <= dim <= 8);
 * min_pts in [1, min(n_points, 16)]; engine 0 = "auto" (numba scan order for
 * n_points >= 4096, else numpy), 1 = "numba", 2 = "numpy" -- the engines
 * break ties differently and are reproduced bit-exactly.  Outputs (DEVICE,
 * n_points - 1 entries, Prim discovery order = original edge id): u, v,
 * w = sqrt(w_sq); core_sq (nullable, n_points) = core_distances ** 2.
 * Workspace: dmst_mreach_workspace_bytes(n_points, dim). */
size_t dmst_mreach_workspace_bytes(int64_t n_points, int32_t dim);
int dmst_mreach_mst(const double* coords, int64_t n_points, int32_t dim, int32_t min_pts, int32_t engine,
                    int32_t* u, int32_t* v, double* w, double* core_sq, void* workspace, size_t workspace_bytes,
                    void* stream);

/* Message for the last non-zero return on this thread ("" if none). */
const char* dmst_last_error(void);

/* Name of kernel kind `id` (0 <= id < DMST_MAX_KERNELS), "" if unused. */
const char* dmst_kernel_name(int32_t id);

/* Library version string. */
const char* dmst_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DMST_H */

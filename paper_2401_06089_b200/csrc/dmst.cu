// B200-native PANDORA dendrogram construction: kernels + C ABI.
//
// Pipeline (one stream, all buffers caller-owned), with the reference
// symbol each stage replaces (paths under /root/reference/pkg/src/dendromst/):
//
//  1. edge sort        rank_edges            tree_core.py:174-190
//     k_sort1_hist -> k_digit_scan -> k_onesweep x (non-constant digits);
//     key = order-preserving uint64 of (w + 0.0), descending; payload =
//     original id.  Last pass writes orig_of, heights (decoded from the
//     key), rank-order endpoints, and scatter-maxes ranks into
//     vertex_parent (build_incidence, tree_core.py:193-199).
//  2. contraction      build_hierarchy       contraction.py:186-219
//     per view k: k_vertex (maxIncident pointer + child count per edge),
//     k_break_cycles, k_root_walk (+ k_jump rounds for deep in-trees),
//     k_select<RootSel> (supervertex ids), k_map (vertex_map),
//     k_select<EdgeSel> (classify, retirement, alpha-edge compaction with
//     remapped endpoints and super maxIncident).
//  3. expansion        assign_chains         expansion.py:97-128
//     k_walk: per edge, the level walk -> dense chain key (+ digit histogram)
//  4. chain sort+link  stitch_chains         expansion.py:131-145
//     stable onesweep on the chain key (payload = rank), k_link.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dmst.h"
#include "common.cuh"
#include "onesweep.cuh"

namespace dmst {

// ----------------------------------------------------------------- config
constexpr int S1_BLOCK = 256, S1_ITEMS = 16;   // edge sort: u64 key, u32 payload
constexpr int S2_BLOCK = 256, S2_ITEMS = 16;   // chain sort: u32 key, u32 payload
constexpr int S1_TILE = S1_BLOCK * S1_ITEMS;
constexpr int S2_TILE = S2_BLOCK * S2_ITEMS;
constexpr int SEL_BLOCK = 256, SEL_ITEMS = 8;  // select-scan tiles
constexpr int SEL_TILE = SEL_BLOCK * SEL_ITEMS;
constexpr int EW_BLOCK = 256;                  // elementwise kernels
constexpr int ROOT_WALK_STEPS = 32;

// Kernel kinds for the optional per-kernel event profile (dmst_stats.profile).
enum KernelKind {
  KK_SORT1_HIST, KK_SORT1_FIRST, KK_SORT1_MID, KK_SORT1_FINAL, KK_DIGIT_SCAN, KK_VERTEX,
  KK_BREAK_CYCLES, KK_ROOT_WALK, KK_JUMP, KK_SELECT_ROOTS, KK_MAP, KK_SELECT_EDGES, KK_WALK,
  KK_SORT2_PASS, KK_LINK, KK_OTHER, KK_COUNT
};
static_assert(KK_COUNT <= DMST_MAX_KERNELS, "kernel kinds");
const char* const kKernelNames[KK_COUNT] = {
    "sort1_hist", "sort1_pass_first", "sort1_pass_mid", "sort1_pass_final", "digit_scan",
    "vertex", "break_cycles", "root_walk", "jump", "select_roots", "map", "select_edges",
    "walk", "sort2_pass", "link", "other"};

// ------------------------------------------------------------ key codec
__device__ __forceinline__ uint64_t desc_key(double w) {
  uint64_t b = (uint64_t)__double_as_longlong(w);
  if (b == 0x8000000000000000ull) b = 0;  // -0.0 == +0.0 (numpy compare)
  uint64_t asc = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  return ~asc;
}
__device__ __forceinline__ double key_to_double(uint64_t key) {
  uint64_t asc = ~key;
  uint64_t b = (asc >> 63) ? (asc & 0x7fffffffffffffffull) : ~asc;
  return __longlong_as_double((long long)b);
}

// ------------------------------------------------ 1. edge sort (sort #1)
// One read of w: all eight digit histograms + the "-0.0 present" flag.
__global__ void __launch_bounds__(256) k_sort1_hist(const double* __restrict__ w, int64_t n,
                                                    uint32_t* __restrict__ hist,
                                                    uint32_t* __restrict__ negzero) {
  __shared__ uint32_t sh[8][kRadix];
  for (int i = threadIdx.x; i < 8 * kRadix; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  bool nz = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    const bool ok = i < n;
    uint64_t key = 0;
    if (ok) {
      double x = ld_stream(w + i);
      nz |= (uint64_t)__double_as_longlong(x) == 0x8000000000000000ull;
      key = desc_key(x);
    }
    const uint32_t act = __ballot_sync(kFull, ok);
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      uint32_t d = (uint32_t)(key >> (8 * p)) & 0xff;
      uint32_t d0 = __shfl_sync(kFull, d, 0);
      if (__all_sync(kFull, !ok || d == d0)) {
        if (threadIdx.x % 32 == 0) atomicAdd(&sh[p][d0], __popc(act));
      } else if (ok) {
        atomicAdd(&sh[p][d], 1u);
      }
    }
  }
  if (__any_sync(kFull, nz) && threadIdx.x % 32 == 0) atomicOr(negzero, 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * kRadix; i += blockDim.x) {
    uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

struct Sort1FirstLoader {
  const double* __restrict__ w;
  __device__ __forceinline__ void load(int64_t i, uint64_t& k, uint32_t& v) const {
    k = desc_key(ld_stream(w + i));
    v = (uint32_t)i;
  }
};

// Final pass of the edge sort: outputs of rank_edges + maxIncident.
struct Sort1FinalEmitter {
  const int32_t* __restrict__ u;
  const int32_t* __restrict__ v;
  int32_t* __restrict__ orig_of;
  double* __restrict__ heights;
  int2* __restrict__ euv;        // rank-order endpoints
  int32_t* __restrict__ ru;      // optional split copies (dmst_rank_edges)
  int32_t* __restrict__ rv;
  int32_t* __restrict__ mi;      // maxIncident (= vertex_parent), -1 init; may be null
  template <int N>
  __device__ __forceinline__ void emit(const uint32_t (&dst)[N], const uint64_t (&k)[N],
                                       const uint32_t (&id)[N], const bool (&ok)[N]) const {
    int32_t a[N], b[N];
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (ok[i]) {
        a[i] = __ldg(u + id[i]);
        b[i] = __ldg(v + id[i]);
      }
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (ok[i]) {
        const uint32_t r = dst[i];
        orig_of[r] = (int32_t)id[i];
        heights[r] = key_to_double(k[i]);
        if (euv) euv[r] = make_int2(a[i], b[i]);
        if (ru) { ru[r] = a[i]; rv[r] = b[i]; }
        if (mi) {
          atomicMax(mi + a[i], (int32_t)r);
          atomicMax(mi + b[i], (int32_t)r);
        }
      }
  }
};

// heights were decoded from canonicalised keys; restore -0.0 bit patterns.
__global__ void k_fix_negzero(const double* __restrict__ w, const int32_t* __restrict__ orig_of,
                              double* __restrict__ heights, int64_t n) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n && heights[r] == 0.0) heights[r] = w[orig_of[r]];
}

// dmst_pandora entry: already-ranked endpoints -> euv + maxIncident.
__global__ void k_incidence(const int32_t* __restrict__ ru, const int32_t* __restrict__ rv,
                            int64_t n, int2* __restrict__ euv, int32_t* __restrict__ mi) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) {
    int32_t a = ru[r], b = rv[r];
    euv[r] = make_int2(a, b);
    atomicMax(mi + a, (int32_t)r);
    atomicMax(mi + b, (int32_t)r);
  }
}

// --------------------------------------------- 2. contraction (per view)
// View k: nv vertices, ne edges; euv[j] endpoints; grank[j] global rank
// (null => identity, view 0); smi[x] = local index of x's largest incident
// edge (maxIncident, contraction.py:149-154), -1 if x is isolated.
//
// k_vertex: x points across its maxIncident edge (that edge is never alpha,
// so these pointers form a functional graph whose in-trees are exactly the
// contraction components; the only cycles are 2-cycles on leaf edges).  It
// also counts, per edge, how many endpoints it is maxIncident at
// (2 = leaf, 1 = chain, 0 = alpha: classify.py:37-42) in a 2-bit field.
__global__ void k_vertex(int64_t nv, const int32_t* __restrict__ smi, const int2* __restrict__ euv,
                         const int32_t* __restrict__ grank, int32_t* __restrict__ ptr,
                         uint32_t* __restrict__ cnt2, int32_t* __restrict__ smi_global) {
  int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nv) return;
  int32_t j = smi[x];
  int32_t y = (int32_t)x;
  if (j >= 0) {
    int2 e = euv[j];
    y = e.x ^ e.y ^ (int32_t)x;
    atomicAdd(cnt2 + (j >> 4), 1u << ((j & 15) * 2));
  }
  ptr[x] = y;
  if (smi_global) smi_global[x] = j < 0 ? -1 : (grank ? grank[j] : j);
}

// Break each leaf 2-cycle at its smaller endpoint (the component root).
__global__ void k_break_cycles(int64_t nv, const int32_t* __restrict__ ptr, int32_t* __restrict__ q) {
  int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nv) return;
  int32_t y = ptr[x];
  q[x] = (ptr[y] == (int32_t)x) ? min((int32_t)x, y) : y;
}

// Bounded walk to the root; unresolved vertices (deep in-trees, e.g. the
// single chain of a path) get a shortcut pointer and go to the jump list.
__global__ void k_root_walk(int64_t nv, int32_t* __restrict__ q, int32_t* __restrict__ active,
                            uint32_t* __restrict__ active_cnt) {
  int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool unresolved = false;
  if (x < nv) {
    int32_t r = q[x];
    int s = 0;
    for (; s < ROOT_WALK_STEPS; ++s) {
      int32_t nr = q[r];
      if (nr == r) break;
      r = nr;
    }
    unresolved = q[r] != r;
    if (r != q[x]) q[x] = r;
  }
  uint32_t m = __ballot_sync(kFull, unresolved);
  if (m) {
    uint32_t lead = __ffs(m) - 1, base = 0;
    if (lane_id() == lead) base = atomicAdd(active_cnt, __popc(m));
    base = __shfl_sync(kFull, base, lead);
    if (unresolved) active[base + __popc(m & lanemask_lt())] = (int32_t)x;
  }
}

// One pointer-jumping round over the unresolved list (in place: every
// pointer only ever moves to an ancestor, so concurrent updates are safe).
__global__ void k_jump(const int32_t* __restrict__ in, const uint32_t* __restrict__ in_cnt,
                       int32_t* __restrict__ out, uint32_t* __restrict__ out_cnt, int32_t* q) {
  const uint32_t cnt = *in_cnt;
  for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x; t0 < cnt; t0 += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = t0 + threadIdx.x;
    bool again = false;
    int32_t x = 0;
    if (t < cnt) {
      x = in[t];
      int32_t r = q[x];
      int32_t nr = q[r];
      if (nr != r) {
        q[x] = nr;
        again = q[nr] != nr;
      }
    }
    uint32_t m = __ballot_sync(kFull, again);
    if (m) {
      uint32_t lead = __ffs(m) - 1, base = 0;
      if (lane_id() == lead) base = atomicAdd(out_cnt, __popc(m));
      base = __shfl_sync(kFull, base, lead);
      if (again) out[base + __popc(m & lanemask_lt())] = x;
    }
  }
}

// Order-preserving select: single pass, decoupled look-back over tiles.
// Items are warp-striped (coalesced); rank order = index order.
template <class Sel>
__global__ void __launch_bounds__(SEL_BLOCK)
k_select(int64_t n, uint32_t* __restrict__ status, uint32_t* __restrict__ tile_ctr,
         uint32_t* __restrict__ totals, Sel sel) {
  constexpr int NW = SEL_BLOCK / 32;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[NW + 1];
  __shared__ uint32_t s_excl;
  __shared__ uint32_t s_aux[2][NW];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t wbase = (int64_t)tile * SEL_TILE + (int64_t)warp * SEL_ITEMS * 32 + lane;
  const uint32_t lt = lanemask_lt();

  typename Sel::Item it[SEL_ITEMS];
  uint32_t wpos[SEL_ITEMS];
  bool flag[SEL_ITEMS];
  uint32_t run = 0, aux0 = 0, aux1 = 0;
#pragma unroll
  for (int i = 0; i < SEL_ITEMS; ++i) {
    int64_t idx = wbase + (int64_t)i * 32;
    flag[i] = idx < n ? sel.flag(idx, it[i], aux0, aux1) : false;
    uint32_t b = __ballot_sync(kFull, flag[i]);
    wpos[i] = run + __popc(b & lt);
    run += __popc(b);
  }
  // per-block aux sums (one global atomic per block)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    aux0 += __shfl_xor_sync(kFull, aux0, o);
    aux1 += __shfl_xor_sync(kFull, aux1, o);
  }
  if (lane == 0) {
    s_warp[warp] = run;
    s_aux[0][warp] = aux0;
    s_aux[1][warp] = aux1;
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t c = lane < NW ? s_warp[lane] : 0;
    uint32_t incl = warp_incl_sum(c);
    if (lane < NW) s_warp[lane] = incl - c;
    uint32_t total = __shfl_sync(kFull, incl, NW - 1);
    uint32_t a0 = lane < NW ? s_aux[0][lane] : 0, a1 = lane < NW ? s_aux[1][lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(kFull, a0, o);
      a1 += __shfl_xor_sync(kFull, a1, o);
    }
    if (lane == 0) {
      uint32_t excl = 0;
      if (tile == 0) {
        st_relaxed(status, kFlagPrefix | total);
      } else {
        st_relaxed(status + tile, kFlagAgg | total);
        excl = lookback(status, tile, 1);
        st_relaxed(status + tile, kFlagPrefix | (excl + total));
      }
      s_excl = excl;
      if (tile == gridDim.x - 1) totals[0] = excl + total;
      if (a0) atomicAdd(totals + 1, a0);
      if (a1) atomicAdd(totals + 2, a1);
    }
  }
  __syncthreads();
  const uint32_t base = s_excl + s_warp[warp];
#pragma unroll
  for (int i = 0; i < SEL_ITEMS; ++i) {
    int64_t idx = wbase + (int64_t)i * 32;
    if (idx < n) sel.emit(idx, flag[i], base + wpos[i], it[i]);
  }
}

// Supervertex ids: roots in vertex order get consecutive ids.
struct RootSel {
  const int32_t* __restrict__ q;
  int32_t* __restrict__ newid;
  struct Item {};
  __device__ __forceinline__ bool flag(int64_t x, Item&, uint32_t&, uint32_t&) const {
    return q[x] == (int32_t)x;
  }
  __device__ __forceinline__ void emit(int64_t x, bool f, uint32_t pos, const Item&) const {
    if (f) newid[x] = (int32_t)pos;
  }
};

// vertex_map (contraction.py:168) and reset of the next view's maxIncident.
__global__ void k_map(int64_t nv, const int32_t* __restrict__ q, const int32_t* __restrict__ newid,
                      int32_t* __restrict__ vm, const uint32_t* __restrict__ super_count,
                      int32_t* __restrict__ smi_next) {
  int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nv) return;
  vm[x] = newid[q[x]];
  if (x < *super_count) smi_next[x] = -1;
}

// Classify edges of view k (classify.py:37-50), retire non-alpha edges at
// level k (contraction.py:207), and compact alpha edges in rank order into
// view k+1 with remapped endpoints (:170-172) and super maxIncident (:173-175).
struct EdgeSel {
  const uint32_t* __restrict__ cnt2_in;
  uint32_t* __restrict__ cnt2;       // zeroed after reading (for the next view)
  const int2* __restrict__ euv;
  const int32_t* __restrict__ grank; // null => identity (view 0)
  const int32_t* __restrict__ vm;
  int8_t* __restrict__ ret;
  int2* __restrict__ euv_next;
  int32_t* __restrict__ grank_next;
  int32_t* __restrict__ smi_next;
  int8_t level;
  struct Item {
    int32_t g;
  };
  __device__ __forceinline__ bool flag(int64_t j, Item& it, uint32_t& n_leaf, uint32_t& n_chain) const {
    uint32_t c = (cnt2_in[j >> 4] >> ((j & 15) * 2)) & 3u;
    n_leaf += c == 2;
    n_chain += c == 1;
    it.g = grank ? grank[j] : (int32_t)j;
    return c == 0;
  }
  __device__ __forceinline__ void emit(int64_t j, bool alpha, uint32_t pos, const Item& it) const {
    if ((j & 15) == 0) cnt2[j >> 4] = 0u;
    if (!alpha) {
      ret[it.g] = level;
    } else {
      int2 e = euv[j];
      int32_t a = vm[e.x], b = vm[e.y];
      euv_next[pos] = make_int2(a, b);
      grank_next[pos] = it.g;
      atomicMax(smi_next + a, (int32_t)pos);
      atomicMax(smi_next + b, (int32_t)pos);
    }
  }
};

// ------------------------------------------------------ 3. expansion walk
struct LevelTable {
  int64_t voff[DMST_MAX_LEVELS + 1];  // offset of vertex_map of view k in vm_all
  int64_t soff[DMST_MAX_LEVELS + 2];  // offset of maxIncident (global ranks) of view k in smi_all
  int32_t L;
};

// assign_chains (expansion.py:97-128): an edge retired at view r is tried
// at views r+1..L; the first whose supervertex parent p satisfies
// 0 <= p < e wins.  The chain (terminal, anchor) is encoded as the dense key
// 1 + soff[k] + anchor (a terminal edge is only ever a terminal at the one
// level it retires at, so (level, anchor) identifies the chain); 0 = root.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
k_walk(int64_t n, const int8_t* __restrict__ ret, const int2* __restrict__ euv,
       const int32_t* __restrict__ vm_all, const int32_t* __restrict__ smi_all,
       const __grid_constant__ LevelTable lt, uint32_t* __restrict__ keys,
       uint32_t* __restrict__ hist, int digits) {
  __shared__ uint32_t sh[4][kRadix];
  for (int i = threadIdx.x; i < 4 * kRadix; i += BLOCK) (&sh[0][0])[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * BLOCK;
  for (int64_t e0 = (int64_t)blockIdx.x * BLOCK; e0 < n; e0 += stride) {
    const int64_t e = e0 + threadIdx.x;
    const bool ok = e < n;
    uint32_t key = 0;
    if (ok) {
      const int r = ret[e];
      if (r < lt.L) {
        int32_t x = euv[e].x;
        for (int k = 0; k < r; ++k) x = vm_all[lt.voff[k] + x];
        for (int k = r + 1; k <= lt.L; ++k) {
          x = vm_all[lt.voff[k - 1] + x];
          int32_t p = smi_all[lt.soff[k] + x];
          if (p >= 0 && p < (int32_t)e) {
            key = (uint32_t)(1 + lt.soff[k] + x);
            break;
          }
        }
      }
      keys[e] = key;
    }
    const uint32_t act = __ballot_sync(kFull, ok);
    for (int p = 0; p < digits; ++p) {
      uint32_t d = (key >> (8 * p)) & 0xff;
      uint32_t d0 = __shfl_sync(kFull, d, 0);
      if (__all_sync(kFull, !ok || d == d0)) {
        if (threadIdx.x % 32 == 0) atomicAdd(&sh[p][d0], __popc(act));
      } else if (ok) {
        atomicAdd(&sh[p][d], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < digits * kRadix; i += BLOCK) {
    uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

struct Sort2FirstLoader {
  const uint32_t* __restrict__ keys;
  __device__ __forceinline__ void load(int64_t i, uint32_t& k, uint32_t& v) const {
    k = ld_stream(keys + i);
    v = (uint32_t)i;
  }
};

// stitch_chains (expansion.py:131-145): in (key, rank) order the parent of
// an edge is its predecessor in the same chain, or the chain's terminal.
__global__ void k_link(int64_t n, const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ svals,
                       const int32_t* __restrict__ smi_all, int32_t* __restrict__ edge_parent) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t key = skeys[i];
  uint32_t e = svals ? svals[i] : (uint32_t)i;
  int32_t parent;
  if (i > 0 && skeys[i - 1] == key)
    parent = svals ? (int32_t)svals[i - 1] : (int32_t)(i - 1);
  else
    parent = key == 0 ? -1 : smi_all[key - 1];
  edge_parent[e] = parent;
}

// Debug: ChainAssignment.terminal / .level from the dense key.
__global__ void k_debug_chain(int64_t n, const uint32_t* __restrict__ keys,
                              const int32_t* __restrict__ smi_all, const __grid_constant__ LevelTable lt,
                              int32_t* __restrict__ key_out, int32_t* __restrict__ term,
                              int32_t* __restrict__ lvl) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  uint32_t key = keys[e];
  if (key_out) key_out[e] = (int32_t)key;
  int32_t t = -1, l = 0;
  if (key) {
    t = smi_all[key - 1];
    l = 1;
    while (l < lt.L && (int64_t)(key - 1) >= lt.soff[l + 1]) ++l;
  }
  if (term) term[e] = t;
  if (lvl) lvl[e] = l;
}

// =================================================================== host
namespace {

thread_local std::string g_err;

struct Fail {
  int code;
};

#define DMST_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      g_err = std::string(#call) + ": " + cudaGetErrorString(e_);                    \
      throw Fail{DMST_ECUDA};                                                        \
    }                                                                                \
  } while (0)

#define DMST_CHECK_LAUNCH() DMST_CUDA(cudaGetLastError())

[[noreturn]] void invalid(const std::string& m) {
  g_err = m;
  throw Fail{DMST_EINVAL};
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Workspace carve-up; the same code sizes and assigns it.
struct Workspace {
  // edge sort (sort #1); region later reused by the chain sort and jump lists
  uint64_t* keysA;
  uint64_t* keysB;
  uint32_t* valsA;
  uint32_t* valsB;
  uint32_t* status[2];    // look-back words, max(tiles) * 256 each
  uint32_t* small;        // counters/histograms (zeroed per use)
  // pipeline
  int2* euv0;             // rank-order endpoints
  int32_t* ptr;           // pointers / newid
  int32_t* q;             // root pointers
  uint32_t* cnt2;         // 2-bit child counts per edge
  int8_t* ret;            // retirement level per edge
  int2* euv[2];           // view edges (ping-pong)
  int32_t* grank[2];
  int32_t* smi[2];
  int32_t* vm_all;        // vertex maps of views 0..L-1
  int32_t* smi_all;       // maxIncident (global ranks) of views 1..L
  uint32_t* sel_status;   // select-scan look-back words
  size_t bytes;
};

constexpr int kSmallWords = 8 * kRadix /*hist1*/ + 8 * kRadix /*gbase1*/ + 4 * kRadix /*hist2*/ +
                            4 * kRadix /*gbase2*/ + 64 /*tile ctrs*/ + 64 /*misc*/;
// small layout offsets
constexpr int SM_HIST1 = 0, SM_GBASE1 = SM_HIST1 + 8 * kRadix, SM_HIST2 = SM_GBASE1 + 8 * kRadix,
              SM_GBASE2 = SM_HIST2 + 4 * kRadix, SM_TILECTR = SM_GBASE2 + 4 * kRadix,
              SM_MISC = SM_TILECTR + 64;
// misc words
constexpr int MISC_NEGZERO = 0, MISC_ACTIVE0 = 1, MISC_ACTIVE1 = 2, MISC_ROOTS = 4 /*3 words*/,
              MISC_EDGES = 8 /*3 words*/, MISC_SELCTR = 12 /*2 words*/;

Workspace carve(int64_t n, int64_t nv, char* base) {
  Workspace w{};
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  const int64_t half = n / 2 + 1;
  const int64_t tiles = std::max(cdiv(n, S1_TILE), cdiv(n, S2_TILE));
  w.keysA = (uint64_t*)take(8 * n);
  w.keysB = (uint64_t*)take(8 * n);
  w.valsA = (uint32_t*)take(4 * n);
  w.valsB = (uint32_t*)take(4 * n);
  w.status[0] = (uint32_t*)take(4 * tiles * kRadix);
  w.status[1] = (uint32_t*)take(4 * tiles * kRadix);
  w.small = (uint32_t*)take(4 * kSmallWords);
  w.euv0 = (int2*)take(8 * n);
  w.ptr = (int32_t*)take(4 * nv);
  w.q = (int32_t*)take(4 * nv);
  w.cnt2 = (uint32_t*)take(4 * (n / 16 + 1));
  w.ret = (int8_t*)take(n);
  for (int i = 0; i < 2; ++i) {
    w.euv[i] = (int2*)take(8 * half);
    w.grank[i] = (int32_t*)take(4 * half);
    w.smi[i] = (int32_t*)take(4 * (half + 1));
  }
  w.vm_all = (int32_t*)take(4 * (2 * nv + DMST_MAX_LEVELS + 2));
  w.smi_all = (int32_t*)take(4 * (nv + DMST_MAX_LEVELS + 2));
  w.sel_status = (uint32_t*)take(4 * (cdiv(nv, SEL_TILE) + 1));
  w.bytes = off + 256;
  return w;
}

void check_args(int64_t n, int64_t nv, const void* ws, size_t ws_bytes) {
  if (n < 1) invalid("n_edges must be >= 1");
  if (n >= (int64_t(1) << 30) - 1) invalid("n_edges must be < 2^30 - 1");
  if (nv != n + 1) invalid("n_vertices must equal n_edges + 1 (a spanning tree)");
  if (!ws) invalid("workspace is null");
  if (ws_bytes < carve(n, nv, nullptr).bytes) invalid("workspace too small");
}

inline unsigned grid_for(int64_t n, int block) { return (unsigned)std::max<int64_t>(1, cdiv(n, block)); }

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

struct Ctx {
  cudaStream_t s;
  Workspace w;
  int launches = 0;
  bool profile = false;
  struct Ev {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Ev> ev;
  void begin(int kind) {
    if (!profile) return;
    Ev e{kind, nullptr, nullptr};
    DMST_CUDA(cudaEventCreate(&e.a));
    DMST_CUDA(cudaEventCreate(&e.b));
    DMST_CUDA(cudaEventRecord(e.a, s));
    ev.push_back(e);
  }
  void launched() {
    ++launches;
    DMST_CHECK_LAUNCH();
    if (profile) DMST_CUDA(cudaEventRecord(ev.back().b, s));
  }
  // After the final stream sync: fold event pairs into stats.
  void collect(dmst_stats* st) {
    for (Ev& e : ev) {
      float ms = 0.f;
      if (st && cudaEventElapsedTime(&ms, e.a, e.b) == cudaSuccess) {
        st->kernel_ms[e.kind] += ms;
        st->kernel_calls[e.kind] += 1;
      }
    }
    release();
  }
  void release() {
    for (Ev& e : ev) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    ev.clear();
  }
  ~Ctx() { release(); }
  template <typename T>
  T read_dev(const T* p) {
    T h;
    DMST_CUDA(cudaMemcpyAsync(&h, p, sizeof(T), cudaMemcpyDeviceToHost, s));
    DMST_CUDA(cudaStreamSynchronize(s));
    return h;
  }
  void read_words(uint32_t* h, const uint32_t* d, size_t count) {
    DMST_CUDA(cudaMemcpyAsync(h, d, count * 4, cudaMemcpyDeviceToHost, s));
    DMST_CUDA(cudaStreamSynchronize(s));
  }
};

template <typename K, typename V, int BLOCK, int ITEMS, class Loader, class Emitter>
void launch_pass(Ctx& c, int kind, int64_t n, int shift, const uint32_t* gbase, int pass_idx,
                 Loader ld, Emitter em) {
  using S = OnesweepSmem<K, V, BLOCK, ITEMS>;
  auto kern = k_onesweep<K, V, BLOCK, ITEMS, Loader, Emitter>;
  DMST_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(S)));
  PassArgs a;
  a.n = n;
  a.shift = shift;
  a.gbase = gbase;
  a.num_tiles = (uint32_t)cdiv(n, S::TILE);
  a.status = c.w.status[pass_idx & 1];
  a.status_next = c.w.status[(pass_idx + 1) & 1];
  a.tile_ctr = c.w.small + SM_TILECTR + pass_idx;
  c.begin(kind);
  kern<<<a.num_tiles, BLOCK, sizeof(S), c.s>>>(a, ld, em);
  c.launched();
}

// Generic multi-pass driver.  `active` lists the digit indices to sort
// (constant digits skipped).  first/last passes use the given loader/emitter.
template <typename K, int BLOCK, int ITEMS, class FirstLoader, class FinalEmitter>
void run_sort(Ctx& c, const int (&kinds)[3], int64_t n, const std::vector<int>& active,
              const uint32_t* gbase, K* bufA, K* bufB, uint32_t* valA, uint32_t* valB,
              FirstLoader first, FinalEmitter final_em) {
  using S = OnesweepSmem<K, uint32_t, BLOCK, ITEMS>;
  const int64_t tiles = cdiv(n, S::TILE);
  DMST_CUDA(cudaMemsetAsync(c.w.status[0], 0, 4 * tiles * kRadix, c.s));
  DMST_CUDA(cudaMemsetAsync(c.w.small + SM_TILECTR, 0, 64 * 4, c.s));
  if (active.empty()) {
    k_identity_pass<K, uint32_t><<<grid_for(n, EW_BLOCK), EW_BLOCK, 0, c.s>>>(n, first, final_em);
    c.launched();
    return;
  }
  K* kin = nullptr;
  uint32_t* vin = nullptr;
  const int P = (int)active.size();
  for (int p = 0; p < P; ++p) {
    const int d = active[p];
    const uint32_t* gb = gbase + d * kRadix;
    K* kout = (p % 2 == 0) ? bufA : bufB;
    uint32_t* vout = (p % 2 == 0) ? valA : valB;
    ArrayEmitter<K, uint32_t> mid{kout, vout};
    ArrayLoader<K, uint32_t> ldr{kin, vin};
    if (P == 1)
      launch_pass<K, uint32_t, BLOCK, ITEMS>(c, kinds[2], n, 8 * d, gb, p, first, final_em);
    else if (p == 0)
      launch_pass<K, uint32_t, BLOCK, ITEMS>(c, kinds[0], n, 8 * d, gb, p, first, mid);
    else if (p == P - 1)
      launch_pass<K, uint32_t, BLOCK, ITEMS>(c, kinds[2], n, 8 * d, gb, p, ldr, final_em);
    else
      launch_pass<K, uint32_t, BLOCK, ITEMS>(c, kinds[1], n, 8 * d, gb, p, ldr, mid);
    kin = kout;
    vin = vout;
  }
}

// Sort #1 (rank_edges).  Writes orig_of/heights and, via `em`, the rest.
void edge_sort(Ctx& c, const double* w, int64_t n, Sort1FinalEmitter em, int* passes_out) {
  uint32_t* hist = c.w.small + SM_HIST1;
  uint32_t* gbase = c.w.small + SM_GBASE1;
  uint32_t* negzero = c.w.small + SM_MISC + MISC_NEGZERO;
  DMST_CUDA(cudaMemsetAsync(hist, 0, 8 * kRadix * 4, c.s));
  DMST_CUDA(cudaMemsetAsync(negzero, 0, 4, c.s));
  const unsigned hgrid = (unsigned)std::min<int64_t>(grid_for(n, 256), (int64_t)num_sms() * 8);
  c.begin(KK_SORT1_HIST);
  k_sort1_hist<<<hgrid, 256, 0, c.s>>>(w, n, hist, negzero);
  c.launched();
  c.begin(KK_DIGIT_SCAN);
  k_digit_scan<<<1, kRadix, 0, c.s>>>(hist, gbase, 8);
  c.launched();
  std::vector<uint32_t> h(8 * kRadix + 1);
  DMST_CUDA(cudaMemcpyAsync(h.data(), hist, 8 * kRadix * 4, cudaMemcpyDeviceToHost, c.s));
  DMST_CUDA(cudaMemcpyAsync(h.data() + 8 * kRadix, negzero, 4, cudaMemcpyDeviceToHost, c.s));
  DMST_CUDA(cudaStreamSynchronize(c.s));
  std::vector<int> active;
  for (int d = 0; d < 8; ++d) {
    bool constant = false;
    for (int b = 0; b < kRadix; ++b)
      if (h[d * kRadix + b] == (uint32_t)n) constant = true;
    if (!constant) active.push_back(d);
  }
  if (passes_out) *passes_out = (int)active.size();
  run_sort<uint64_t, S1_BLOCK, S1_ITEMS>(c, {KK_SORT1_FIRST, KK_SORT1_MID, KK_SORT1_FINAL}, n, active, gbase, c.w.keysA, c.w.keysB, c.w.valsA,
                                         c.w.valsB, Sort1FirstLoader{w}, em);
  if (h[8 * kRadix]) {
    c.begin(KK_OTHER);
    k_fix_negzero<<<grid_for(n, EW_BLOCK), EW_BLOCK, 0, c.s>>>(w, em.orig_of, em.heights, n);
    c.launched();
  }
}

struct SelCounts {
  uint32_t total, aux0, aux1;
};

template <class Sel>
SelCounts run_select(Ctx& c, int kind, int64_t n, Sel sel, uint32_t* totals, bool read_back) {
  const int64_t tiles = cdiv(n, SEL_TILE);
  uint32_t* ctr = c.w.small + SM_MISC + MISC_SELCTR;
  DMST_CUDA(cudaMemsetAsync(c.w.sel_status, 0, 4 * tiles, c.s));
  DMST_CUDA(cudaMemsetAsync(ctr, 0, 4, c.s));
  DMST_CUDA(cudaMemsetAsync(totals, 0, 12, c.s));
  if (n == 0) return SelCounts{0, 0, 0};
  c.begin(kind);
  k_select<Sel><<<(unsigned)tiles, SEL_BLOCK, 0, c.s>>>(n, c.w.sel_status, ctr, totals, sel);
  c.launched();
  SelCounts r{0, 0, 0};
  if (read_back) {
    uint32_t h[3];
    c.read_words(h, totals, 3);
    r = {h[0], h[1], h[2]};
  }
  return r;
}

// Full pipeline after the edge sort: euv0 and mi (= vertex_parent) ready.
void pandora_core(Ctx& c, int64_t n, int64_t nv, int32_t* mi, int32_t* edge_parent, dmst_stats* st,
                  int8_t* dbg_ret, int32_t* dbg_key, int32_t* dbg_term, int32_t* dbg_lvl) {
  Workspace& w = c.w;
  LevelTable lt{};
  uint32_t* misc = w.small + SM_MISC;
  DMST_CUDA(cudaMemsetAsync(w.cnt2, 0, 4 * (n / 16 + 1), c.s));

  int64_t nv_k = nv, n_k = n;
  const int2* euv_k = w.euv0;
  const int32_t* grank_k = nullptr;
  const int32_t* smi_k = mi;
  int cur = 0;
  int level = 0;
  int jump_rounds = 0;
  int64_t voff = 0, soff = 0;
  if (st) memset(st->level_counts, 0, sizeof(st->level_counts));
  while (true) {
    if (level > DMST_MAX_LEVELS) invalid("too many contraction levels");
    // view `level`: pointers + child counts (+ global maxIncident for views >= 1)
    int32_t* smi_global = nullptr;
    if (level >= 1) {
      lt.soff[level] = soff;
      smi_global = w.smi_all + soff;
      soff += nv_k;
    }
    c.begin(KK_VERTEX);
    k_vertex<<<grid_for(nv_k, EW_BLOCK), EW_BLOCK, 0, c.s>>>(nv_k, smi_k, euv_k, grank_k, w.ptr, w.cnt2, smi_global);
    c.launched();
    c.begin(KK_BREAK_CYCLES);
    k_break_cycles<<<grid_for(nv_k, EW_BLOCK), EW_BLOCK, 0, c.s>>>(nv_k, w.ptr, w.q);
    c.launched();
    // roots
    int32_t* act[2] = {(int32_t*)w.keysA, (int32_t*)w.keysB};
    uint32_t* act_cnt[2] = {misc + MISC_ACTIVE0, misc + MISC_ACTIVE1};
    DMST_CUDA(cudaMemsetAsync(misc + MISC_ACTIVE0, 0, 8, c.s));
    c.begin(KK_ROOT_WALK);
    k_root_walk<<<grid_for(nv_k, EW_BLOCK), EW_BLOCK, 0, c.s>>>(nv_k, w.q, act[0], act_cnt[0]);
    c.launched();
    uint32_t pending = c.read_dev(act_cnt[0]);
    int a = 0;
    while (pending) {
      DMST_CUDA(cudaMemsetAsync(act_cnt[a ^ 1], 0, 4, c.s));
      unsigned g = (unsigned)std::min<int64_t>(grid_for(pending, EW_BLOCK), (int64_t)num_sms() * 16);
      c.begin(KK_JUMP);
      k_jump<<<g, EW_BLOCK, 0, c.s>>>(act[a], act_cnt[a], act[a ^ 1], act_cnt[a ^ 1], w.q);
      c.launched();
      ++jump_rounds;
      a ^= 1;
      pending = c.read_dev(act_cnt[a]);
    }
    // supervertex ids + vertex_map
    uint32_t* root_tot = misc + MISC_ROOTS;
    run_select(c, KK_SELECT_ROOTS, nv_k, RootSel{w.q, w.ptr}, root_tot, false);
    int32_t* vm = w.vm_all + voff;
    lt.voff[level] = voff;
    voff += nv_k;
    int32_t* smi_next = w.smi[cur ^ 1];
    c.begin(KK_MAP);
    k_map<<<grid_for(nv_k, EW_BLOCK), EW_BLOCK, 0, c.s>>>(nv_k, w.q, w.ptr, vm, root_tot, smi_next);
    c.launched();
    // classify + retire + compact alpha edges into view level+1
    EdgeSel es{w.cnt2, w.cnt2, euv_k, grank_k, vm, w.ret, w.euv[cur ^ 1], w.grank[cur ^ 1], smi_next,
               (int8_t)level};
    SelCounts ec = run_select(c, KK_SELECT_EDGES, n_k, es, misc + MISC_EDGES, true);
    const uint32_t super_count = c.read_dev(root_tot);
    const int64_t n_alpha = ec.total;
    if (st) {
      st->level_counts[level][0] = (int32_t)n_alpha;
      st->level_counts[level][1] = (int32_t)ec.aux0;
      st->level_counts[level][2] = (int32_t)ec.aux1;
      st->level_counts[level][3] = (int32_t)n_k;
      st->view_vertices[level] = (int32_t)nv_k;
    }
    if (level >= 1 && n_alpha == 0) break;  // contraction.py:203-205
    // next view
    euv_k = w.euv[cur ^ 1];
    grank_k = w.grank[cur ^ 1];
    smi_k = smi_next;
    cur ^= 1;
    nv_k = super_count;
    n_k = n_alpha;
    ++level;
  }
  const int L = level;
  lt.L = L;
  lt.soff[L + 1] = soff;
  if (st) {
    st->num_levels = L;
    st->jump_rounds = jump_rounds;
  }

  // expansion walk -> chain keys (+ digit histograms)
  const uint64_t max_key = (uint64_t)soff;  // keys in [0, soff]
  int digits = 1;
  while (digits < 4 && (max_key >> (8 * digits))) ++digits;
  uint32_t* hist2 = w.small + SM_HIST2;
  uint32_t* gbase2 = w.small + SM_GBASE2;
  uint32_t* keys = (uint32_t*)w.keysA;
  DMST_CUDA(cudaMemsetAsync(hist2, 0, 4 * kRadix * 4, c.s));
  {
    const unsigned g = (unsigned)std::min<int64_t>(grid_for(n, 256), (int64_t)num_sms() * 8);
    c.begin(KK_WALK);
    k_walk<256><<<g, 256, 0, c.s>>>(n, w.ret, w.euv0, w.vm_all, w.smi_all, lt, keys, hist2, digits);
    c.launched();
  }
  c.begin(KK_DIGIT_SCAN);
  k_digit_scan<<<1, kRadix, 0, c.s>>>(hist2, gbase2, digits);
  c.launched();
  if (dbg_ret) DMST_CUDA(cudaMemcpyAsync(dbg_ret, w.ret, n, cudaMemcpyDeviceToDevice, c.s));
  if (dbg_key || dbg_term || dbg_lvl) {
    c.begin(KK_OTHER);
    k_debug_chain<<<grid_for(n, EW_BLOCK), EW_BLOCK, 0, c.s>>>(n, keys, w.smi_all, lt, dbg_key, dbg_term, dbg_lvl);
    c.launched();
  }
  std::vector<uint32_t> h(4 * kRadix);
  c.read_words(h.data(), hist2, 4 * kRadix);
  std::vector<int> active;
  for (int d = 0; d < digits; ++d) {
    bool constant = false;
    for (int b = 0; b < kRadix; ++b)
      if (h[d * kRadix + b] == (uint32_t)n) constant = true;
    if (!constant) active.push_back(d);
  }
  if (st) st->sort2_passes = (int)active.size();
  // chain sort: keys at keysA[0, 4n); ping-pong A = (keysA[4n, 8n), valsA),
  // B = (keysB[0, 4n), keysB[4n, 8n)); the last pass lands in A or B.
  const uint32_t* skeys = keys;
  const uint32_t* svals = nullptr;
  if (!active.empty()) {
    uint32_t* kA = keys + n;
    uint32_t* vA = w.valsA;
    uint32_t* kB = (uint32_t*)w.keysB;
    uint32_t* vB = (uint32_t*)w.keysB + n;
    const bool lastA = ((active.size() - 1) % 2) == 0;
    ArrayEmitter<uint32_t, uint32_t> fin{lastA ? kA : kB, lastA ? vA : vB};
    run_sort<uint32_t, S2_BLOCK, S2_ITEMS>(c, {KK_SORT2_PASS, KK_SORT2_PASS, KK_SORT2_PASS}, n, active, gbase2, kA, kB, vA, vB, Sort2FirstLoader{keys}, fin);
    skeys = fin.keys;
    svals = fin.vals;
  }
  c.begin(KK_LINK);
  k_link<<<grid_for(n, EW_BLOCK), EW_BLOCK, 0, c.s>>>(n, skeys, svals, w.smi_all, edge_parent);
  c.launched();
}

template <class F>
int guarded(F&& f) {
  g_err.clear();
  try {
    f();
    return 0;
  } catch (const Fail& e) {
    return e.code;
  }
}

}  // namespace
}  // namespace dmst

using namespace dmst;

extern "C" {

size_t dmst_workspace_bytes(int64_t n_edges, int64_t n_vertices) {
  if (n_edges < 1 || n_vertices < 2) return 0;
  return carve(n_edges, n_vertices, nullptr).bytes;
}

static int build_impl(const int32_t* u, const int32_t* v, const double* w, int64_t n, int64_t nv,
                      int32_t* orig_of, double* heights, int32_t* edge_parent, int32_t* vertex_parent,
                      dmst_stats* st, int8_t* dbg_ret, int32_t* dbg_key, int32_t* dbg_term,
                      int32_t* dbg_lvl, void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    check_args(n, nv, ws, ws_bytes);
    if (!u || !v || !w || !orig_of || !heights || !edge_parent || !vertex_parent)
      invalid("null input/output pointer");
    Ctx c;
    c.s = (cudaStream_t)stream;
    char* base = (char*)(((uintptr_t)ws + 255) & ~uintptr_t(255));
    c.w = carve(n, nv, base);
    if (st) {
      const int32_t prof = st->profile;
      memset(st, 0, sizeof(*st));
      st->profile = prof;
      c.profile = prof != 0;
    }
    DMST_CUDA(cudaMemsetAsync(vertex_parent, 0xff, 4 * nv, c.s));
    Sort1FinalEmitter em{u, v, orig_of, heights, c.w.euv0, nullptr, nullptr, vertex_parent};
    int p1 = 0;
    edge_sort(c, w, n, em, &p1);
    pandora_core(c, n, nv, vertex_parent, edge_parent, st, dbg_ret, dbg_key, dbg_term, dbg_lvl);
    DMST_CUDA(cudaStreamSynchronize(c.s));
    c.collect(st);
    if (st) {
      st->sort1_passes = p1;
      st->kernel_launches = c.launches;
    }
  });
}

int dmst_build(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges,
               int64_t n_vertices, int32_t* orig_of, double* heights, int32_t* edge_parent,
               int32_t* vertex_parent, dmst_stats* stats, void* workspace, size_t workspace_bytes,
               void* stream) {
  return build_impl(u, v, w, n_edges, n_vertices, orig_of, heights, edge_parent, vertex_parent, stats,
                    nullptr, nullptr, nullptr, nullptr, workspace, workspace_bytes, stream);
}

int dmst_build_debug(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges,
                     int64_t n_vertices, int32_t* orig_of, double* heights, int32_t* edge_parent,
                     int32_t* vertex_parent, dmst_stats* stats, int8_t* retirement,
                     int32_t* chain_key, int32_t* chain_terminal, int32_t* chain_level,
                     void* workspace, size_t workspace_bytes, void* stream) {
  return build_impl(u, v, w, n_edges, n_vertices, orig_of, heights, edge_parent, vertex_parent, stats,
                    retirement, chain_key, chain_terminal, chain_level, workspace, workspace_bytes,
                    stream);
}

int dmst_rank_edges(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges,
                    int64_t n_vertices, int32_t* orig_of, double* heights, int32_t* ru, int32_t* rv,
                    void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    check_args(n_edges, n_vertices, workspace, workspace_bytes);
    if (!u || !v || !w || !orig_of || !heights || !ru || !rv) invalid("null input/output pointer");
    Ctx c;
    c.s = (cudaStream_t)stream;
    char* base = (char*)(((uintptr_t)workspace + 255) & ~uintptr_t(255));
    c.w = carve(n_edges, n_vertices, base);
    Sort1FinalEmitter em{u, v, orig_of, heights, nullptr, ru, rv, nullptr};
    edge_sort(c, w, n_edges, em, nullptr);
    DMST_CUDA(cudaStreamSynchronize(c.s));
  });
}

int dmst_pandora(const int32_t* ru, const int32_t* rv, int64_t n_edges, int64_t n_vertices,
                 int32_t* edge_parent, int32_t* vertex_parent, dmst_stats* stats, void* workspace,
                 size_t workspace_bytes, void* stream) {
  return guarded([&] {
    check_args(n_edges, n_vertices, workspace, workspace_bytes);
    if (!ru || !rv || !edge_parent || !vertex_parent) invalid("null input/output pointer");
    Ctx c;
    c.s = (cudaStream_t)stream;
    char* base = (char*)(((uintptr_t)workspace + 255) & ~uintptr_t(255));
    c.w = carve(n_edges, n_vertices, base);
    if (stats) {
      const int32_t prof = stats->profile;
      memset(stats, 0, sizeof(*stats));
      stats->profile = prof;
      c.profile = prof != 0;
    }
    DMST_CUDA(cudaMemsetAsync(vertex_parent, 0xff, 4 * n_vertices, c.s));
    c.begin(KK_OTHER);
    k_incidence<<<grid_for(n_edges, EW_BLOCK), EW_BLOCK, 0, c.s>>>(ru, rv, n_edges, c.w.euv0, vertex_parent);
    c.launched();
    pandora_core(c, n_edges, n_vertices, vertex_parent, edge_parent, stats, nullptr, nullptr, nullptr,
                 nullptr);
    DMST_CUDA(cudaStreamSynchronize(c.s));
    c.collect(stats);
    if (stats) stats->kernel_launches = c.launches;
  });
}

const char* dmst_last_error(void) { return dmst::g_err.c_str(); }

const char* dmst_kernel_name(int32_t id) {
  return (id >= 0 && id < KK_COUNT) ? kKernelNames[id] : "";
}

const char* dmst_version(void) { return "dmst 0.1.0 sm_100a"; }

}  // extern "C"

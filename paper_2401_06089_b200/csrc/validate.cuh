// Device input validation: the checks of the reference's `weighted_tree`
// (/root/reference/pkg/src/dendromst/tree_core.py:110-139), SURVEY.md §8f
// rank 1.  On the CPU that validation costs more than the whole timed build
// (357 s vs 279 s at 128M); here it is one streaming pass, a lock-free
// union-find and (only for inputs that fail connectivity) a sort of the
// undirected edge keys to tell duplicates from other non-trees.
#pragma once
#include "common.cuh"

namespace dmst {

// Per-edge scan, in the reference's order of checks:
//   r[0] = first edge with a non-finite weight (:124-126)
//   r[1] = any negative vertex id (:127-128)
//   r[2] = any vertex id >= num_vertices (:129-130)
//   r[3] = first self-loop edge (:131-133)
// plus the AND / OR of the undirected keys (min << 32 | max) for the
// duplicate sort's digit skipping.  r[0], r[3] start at 0xffffffff.
__global__ void __launch_bounds__(256) k_validate_scan(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                                                       const double* __restrict__ w, int64_t n, int64_t nv,
                                                       uint32_t* __restrict__ r, unsigned long long* __restrict__ ao) {
  uint32_t first_nf = 0xffffffffu, first_sl = 0xffffffffu, neg = 0, rng = 0;
  unsigned long long ka = ~0ull, ko = 0ull;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int32_t a = ld_stream(u + i), b = ld_stream(v + i);
    const double x = ld_stream(w + i);
    if (!isfinite(x) && first_nf == 0xffffffffu) first_nf = (uint32_t)i;
    neg |= (a < 0 || b < 0) ? 1u : 0u;
    rng |= ((int64_t)a >= nv || (int64_t)b >= nv) ? 1u : 0u;
    if (a == b && first_sl == 0xffffffffu) first_sl = (uint32_t)i;
    const uint32_t lo = (uint32_t)min(a, b), hi = (uint32_t)max(a, b);
    const unsigned long long k = ((unsigned long long)lo << 32) | hi;
    ka &= k;
    ko |= k;
  }
  first_nf = __reduce_min_sync(kFull, first_nf);
  first_sl = __reduce_min_sync(kFull, first_sl);
  neg = __reduce_or_sync(kFull, neg);
  rng = __reduce_or_sync(kFull, rng);
  const uint32_t alo = __reduce_and_sync(kFull, (uint32_t)ka), ahi = __reduce_and_sync(kFull, (uint32_t)(ka >> 32));
  const uint32_t olo = __reduce_or_sync(kFull, (uint32_t)ko), ohi = __reduce_or_sync(kFull, (uint32_t)(ko >> 32));
  if (lane_id() == 0) {
    if (first_nf != 0xffffffffu) atomicMin(r + 0, first_nf);
    if (neg) atomicOr(r + 1, 1u);
    if (rng) atomicOr(r + 2, 1u);
    if (first_sl != 0xffffffffu) atomicMin(r + 3, first_sl);
    atomicAnd(ao, ((unsigned long long)ahi << 32) | alo);
    atomicOr(ao + 1, ((unsigned long long)ohi << 32) | olo);
  }
}

__global__ void k_cc_init(int32_t* __restrict__ p, int64_t nv) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x < nv) p[x] = (int32_t)x;
}

__device__ __forceinline__ int32_t cc_find(int32_t* p, int32_t x) {
  // path halving; concurrent hooks only ever point roots to smaller roots
  int32_t q = p[x];
  while (q != x) {
    const int32_t g = p[q];
    if (g != q) p[x] = g;  // benign race: g is an ancestor of x
    x = q;
    q = g;
  }
  return x;
}

// Lock-free union of every edge's endpoints (connectivity, tree_core.py:102-107
// / contraction.py:53-79 component_labels): the larger root is hooked under
// the smaller with a CAS, retried from the new roots on contention.
__global__ void __launch_bounds__(256) k_cc_hook(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                                                 int64_t n, int32_t* p) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    int32_t a = cc_find(p, ld_stream(u + i)), b = cc_find(p, ld_stream(v + i));
    while (a != b) {
      if (a > b) {
        const int32_t t = a;
        a = b;
        b = t;
      }
      const int32_t old = atomicCAS(p + b, b, a);
      if (old == b) break;
      b = cc_find(p, old);
      a = cc_find(p, a);
    }
  }
}

// Number of roots (p[x] == x): 1 iff the graph is connected.
__global__ void __launch_bounds__(256) k_cc_roots(const int32_t* __restrict__ p, int64_t nv, uint32_t* __restrict__ cnt) {
  uint32_t c = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nv; x += stride) c += p[x] == (int32_t)x;
  c = __reduce_add_sync(kFull, c);
  if (lane_id() == 0 && c) atomicAdd(cnt, c);
}

// Undirected edge keys (min << 32 | max) for the duplicate check
// (tree_core.py:134-136: np.unique on min * nv + max).
struct DupKeyLoader {
  static constexpr int NS = 2;
  __host__ __device__ static constexpr int sb(int) { return 4; }
  const int32_t* __restrict__ u;
  const int32_t* __restrict__ v;
  __device__ __forceinline__ const void* ptr(int s) const { return s == 0 ? (const void*)u : (const void*)v; }
  __device__ __forceinline__ static uint64_t mk(int32_t a, int32_t b) {
    return ((uint64_t)(uint32_t)min(a, b) << 32) | (uint32_t)max(a, b);
  }
  __device__ __forceinline__ uint64_t key(int64_t i) const { return mk(ld_stream(u + i), ld_stream(v + i)); }
  __device__ __forceinline__ void load(int64_t i, uint64_t& k, Vals<0>&) const { k = key(i); }
  __device__ __forceinline__ void get(char* const* st, int li, int64_t, uint64_t& k, Vals<0>&) const {
    k = mk(reinterpret_cast<const int32_t*>(st[0])[li], reinterpret_cast<const int32_t*>(st[1])[li]);
  }
};

__global__ void k_adjacent_equal(const unsigned long long* __restrict__ k, int64_t n, uint32_t* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool dup = i > 0 && i < n && k[i] == k[i - 1];
  if (__any_sync(kFull, dup) && lane_id() == 0) atomicOr(flag, 1u);
}

}  // namespace dmst

namespace dmst {

// ------------------------------------------------ dendrogram statistics
// dendrogram_height (analysis.py:21-33): depth(e) = depth(parent(e)) + 1,
// depth 1 at the root; the height is the largest depth (the deepest edge
// node has two vertex children, so it is some vertex's parent).  Pointer
// jumping over (ancestor, distance) pairs packed in 8 B: one random probe
// per live edge per round, ceil(log2(height)) rounds.
__global__ void k_depth_init(const int32_t* __restrict__ parent, int64_t n, int2* __restrict__ ad) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) ad[e] = make_int2(parent[e], 1);
}

__global__ void __launch_bounds__(256) k_depth_jump(const int2* __restrict__ in, int2* __restrict__ out, int64_t n,
                                                    uint32_t* __restrict__ live) {
  uint32_t any = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
    int2 a = in[e];
    if (a.x >= 0) {
      const int2 b = in[a.x];
      a = make_int2(b.x, a.y + b.y);
      any |= a.x >= 0;
    }
    out[e] = a;
  }
  if (__any_sync(kFull, any != 0) && lane_id() == 0) atomicOr(live, 1u);
}

__global__ void __launch_bounds__(256) k_depth_max(const int2* __restrict__ ad, int64_t n, uint32_t* __restrict__ mx) {
  int32_t m = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) m = max(m, ad[e].y);
  m = __reduce_max_sync(kFull, m);
  if (lane_id() == 0) atomicMax(mx, (uint32_t)m);
}

// Chain count (ChainAssignment.num_chains, expansion.py:52-54): distinct
// chain keys = heads of the (key, rank)-sorted items.
__global__ void __launch_bounds__(256) k_count_heads(const unsigned long long* __restrict__ items, int64_t n,
                                                     uint32_t* __restrict__ cnt) {
  uint32_t c = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    c += (i == 0 || (items[i] >> 32) != (items[i - 1] >> 32)) ? 1u : 0u;
  c = __reduce_add_sync(kFull, c);
  if (lane_id() == 0 && c) atomicAdd(cnt, c);
}

}  // namespace dmst

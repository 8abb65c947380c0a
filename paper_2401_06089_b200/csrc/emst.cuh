// Upstream producer: the mutual-reachability MST of a
// point cloud, bit-identical to the reference's
// `mutual_reachability_mst` (pointgen.py:158-178):
//   core_sq = core_distances(coords, min_pts) ** 2      (pointgen.py:56-61)
//   dense Prim over max(|x_i - x_j|^2, core_sq_i, core_sq_j) (pointgen.py:71-148)
//   w = sqrt(w_sq), edges in Prim discovery order.
// Device layout: points SoA in HBM (L2-resident up to ~2M points), one
// cooperative kernel runs every Prim step (one grid barrier per step).
#pragma once
#include <cooperative_groups.h>

#include "radix.cuh"

namespace dmst {

constexpr int EMST_MAX_DIM = 8;
constexpr int KNN_MAX_K = 16;

// |a - b|^2 in the summation order of scipy's cKDTree for p = 2 (verified
// bitwise against cKDTree.query here): four strided accumulators over the
// full blocks of 4 dimensions, combined left to right, then the remaining
// dimensions one by one.
template <int DIM>
__device__ __forceinline__ double sqdist_kdtree(const double* a, const double* b) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  constexpr int FULL = DIM / 4 * 4;
#pragma unroll
  for (int i = 0; i < FULL; i += 4)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double d = __dsub_rn(a[i + j], b[i + j]);
      acc[j] = __dadd_rn(acc[j], __dmul_rn(d, d));
    }
  double s = __dadd_rn(__dadd_rn(__dadd_rn(acc[0], acc[1]), acc[2]), acc[3]);
#pragma unroll
  for (int i = FULL; i < DIM; ++i) {
    const double d = __dsub_rn(a[i], b[i]);
    s = __dadd_rn(s, __dmul_rn(d, d));
  }
  return s;
}

// numba engine (pointgen.py:117-121): d = 0; d += diff * diff, no FMA.
// numpy engine (pointgen.py:82): ((pts - pts[cur]) ** 2).sum(axis=1) -- a
// plain left-to-right row sum below 8 columns, numpy's pairwise block of 8
// accumulators at exactly 8.
template <int DIM, bool NUMPY>
__device__ __forceinline__ double sqdist_prim(const double (&x)[DIM], const double (&c)[DIM]) {
  double q[DIM];
#pragma unroll
  for (int t = 0; t < DIM; ++t) {
    const double d = __dsub_rn(x[t], c[t]);
    q[t] = __dmul_rn(d, d);
  }
  if constexpr (NUMPY && DIM == 8) {
    return __dadd_rn(__dadd_rn(__dadd_rn(q[0], q[1]), __dadd_rn(q[2], q[3])),
                     __dadd_rn(__dadd_rn(q[4], q[5]), __dadd_rn(q[6], q[7])));
  } else {
    double s = NUMPY ? q[0] : __dadd_rn(0.0, q[0]);
#pragma unroll
    for (int t = 1; t < DIM; ++t) s = __dadd_rn(s, q[t]);
    return s;
  }
}

// ---------------------------------------------------------------- core distances
// Brute force: every point against every point (tiles staged in shared
// memory, broadcast reads), the k smallest squared distances kept sorted in
// registers.  core = sqrt(k-th smallest) as cKDTree reports it, squared
// again as the reference does (core_distances(...) ** 2).
constexpr int KNN_BLOCK = 256, KNN_TILE = 512;
template <int DIM>
__global__ void __launch_bounds__(KNN_BLOCK) k_core_sq(const double* __restrict__ pts, int64_t n, int k,
                                                      double* __restrict__ core_sq) {
  __shared__ double tile[KNN_TILE * DIM];
  const int64_t i = (int64_t)blockIdx.x * KNN_BLOCK + threadIdx.x;
  double q[DIM];
#pragma unroll
  for (int t = 0; t < DIM; ++t) q[t] = i < n ? pts[i * DIM + t] : 0.0;
  double best[KNN_MAX_K];
#pragma unroll
  for (int s = 0; s < KNN_MAX_K; ++s) best[s] = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  double thr = best[0];
  for (int64_t j0 = 0; j0 < n; j0 += KNN_TILE) {
    const int cnt = n - j0 < KNN_TILE ? (int)(n - j0) : KNN_TILE;
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * DIM; e += KNN_BLOCK) tile[e] = pts[j0 * DIM + e];
    __syncthreads();
    for (int jj = 0; jj < cnt; ++jj) {
      const double d = sqdist_kdtree<DIM>(q, tile + jj * DIM);
      if (d < thr) {  // insert into the sorted list (static indexing)
        double x = d;
#pragma unroll
        for (int s = 0; s < KNN_MAX_K; ++s)
          if (s < k && x < best[s]) {
            const double y = best[s];
            best[s] = x;
            x = y;
          }
#pragma unroll
        for (int s = 0; s < KNN_MAX_K; ++s)
          if (s == k - 1) thr = best[s];
      }
    }
  }
  if (i < n) {
    const double core = sqrt(thr);
    core_sq[i] = __dmul_rn(core, core);
  }
}

// ---------------------------------------------------------------- dense Prim
// State of the unvisited points in the numba engine's compacted order
// (pointgen.py:100-110; swap-with-last removal, :141-148), SoA.
struct PrimState {
  double* acoord;   // [DIM][cap]
  double* acore;
  double* abest;
  int32_t* afrom;
  int32_t* idx;
  int64_t cap;
};

struct PrimSlot {  // one block's candidate of one step
  double bv;
  int32_t key;    // tie-break key: compacted position (numba) or point id (numpy)
  int32_t k;      // compacted position
  int32_t id;     // point id
  int32_t from;
};

__device__ __forceinline__ bool slot_less(double b, int32_t key, double bv, int32_t bkey) {
  return b < bv || (b == bv && key < bkey);
}

template <int DIM>
__global__ void k_prim_init(const double* __restrict__ pts, const double* __restrict__ core_sq, int64_t n,
                            PrimState st) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n - 1) return;
#pragma unroll
  for (int t = 0; t < DIM; ++t) st.acoord[t * st.cap + k] = pts[(k + 1) * DIM + t];
  st.acore[k] = core_sq[k + 1];
  st.abest[k] = __longlong_as_double(0x7ff0000000000000ll);
  st.afrom[k] = 0;
  st.idx[k] = (int32_t)(k + 1);
}

constexpr int PRIM_BLOCK = 512;
struct PrimArgs {
  const double* pts;
  const double* core_sq;
  int64_t n;
  PrimState st;
  PrimSlot* slots;  // [2][gridDim.x]
  int32_t* out_u;
  int32_t* out_v;
  double* out_w;    // w_sq until the final sqrt
};

// One cooperative launch for all n - 1 steps.  Step: every thread updates
// best/from of its compacted positions (k = gtid + j * T) against the
// current point and keeps its lexicographic minimum (best, key); block
// minimum -> slot; grid barrier; every block reduces all slots to the same
// winner; the owner thread of the winner's position moves the last element
// into it (so the next step's reads of that position are its own writes).
template <int DIM, bool NUMPY>
__global__ void __launch_bounds__(PRIM_BLOCK) k_prim(PrimArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ PrimSlot wbest[PRIM_BLOCK / 32];
  __shared__ PrimSlot win;
  const int64_t T = (int64_t)gridDim.x * PRIM_BLOCK;
  const int64_t gtid = (int64_t)blockIdx.x * PRIM_BLOCK + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const PrimState& st = a.st;
  int32_t cur = 0;
  double cc, curc[DIM];
#pragma unroll
  for (int t = 0; t < DIM; ++t) curc[t] = a.pts[t];
  cc = a.core_sq[0];
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  for (int64_t it = 0; it < a.n - 1; ++it) {
    const int64_t m = a.n - 1 - it;
    double bv = INF;
    int32_t bkey = 0x7fffffff, bk = -1, bid = 0, bfrom = 0;
    for (int64_t k = gtid; k < m; k += T) {
      double x[DIM];
#pragma unroll
      for (int t = 0; t < DIM; ++t) x[t] = st.acoord[t * st.cap + k];
      double d = sqdist_prim<DIM, NUMPY>(x, curc);
      const double ck = st.acore[k];
      if (ck > d) d = ck;
      if (cc > d) d = cc;
      double b = st.abest[k];
      int32_t fr = st.afrom[k];
      if (d < b) {
        b = d;
        fr = cur;
        st.abest[k] = b;
        st.afrom[k] = fr;
      }
      const int32_t id = st.idx[k];
      const int32_t key = NUMPY ? id : (int32_t)k;
      if (slot_less(b, key, bv, bkey)) {
        bv = b;
        bkey = key;
        bk = (int32_t)k;
        bid = id;
        bfrom = fr;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(kFull, bv, o);
      const int32_t okey = __shfl_xor_sync(kFull, bkey, o), ok = __shfl_xor_sync(kFull, bk, o),
                    oid = __shfl_xor_sync(kFull, bid, o), ofr = __shfl_xor_sync(kFull, bfrom, o);
      if (slot_less(ov, okey, bv, bkey)) {
        bv = ov;
        bkey = okey;
        bk = ok;
        bid = oid;
        bfrom = ofr;
      }
    }
    if (lane == 0) wbest[wid] = PrimSlot{bv, bkey, bk, bid, bfrom};
    __syncthreads();
    PrimSlot* slots = a.slots + (it & 1) * gridDim.x;
    if (wid == 0) {
      PrimSlot s = lane < PRIM_BLOCK / 32 ? wbest[lane] : PrimSlot{INF, 0x7fffffff, -1, 0, 0};
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(kFull, s.bv, o);
        const int32_t okey = __shfl_xor_sync(kFull, s.key, o), ok = __shfl_xor_sync(kFull, s.k, o),
                      oid = __shfl_xor_sync(kFull, s.id, o), ofr = __shfl_xor_sync(kFull, s.from, o);
        if (slot_less(ov, okey, s.bv, s.key)) s = PrimSlot{ov, okey, ok, oid, ofr};
      }
      if (lane == 0) slots[blockIdx.x] = s;
    }
    grid.sync();
    if (wid == 0) {
      PrimSlot s{INF, 0x7fffffff, -1, 0, 0};
      for (uint32_t b = lane; b < gridDim.x; b += 32) {
        const PrimSlot o = slots[b];
        if (slot_less(o.bv, o.key, s.bv, s.key)) s = o;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(kFull, s.bv, o);
        const int32_t okey = __shfl_xor_sync(kFull, s.key, o), ok = __shfl_xor_sync(kFull, s.k, o),
                      oid = __shfl_xor_sync(kFull, s.id, o), ofr = __shfl_xor_sync(kFull, s.from, o);
        if (slot_less(ov, okey, s.bv, s.key)) s = PrimSlot{ov, okey, ok, oid, ofr};
      }
      if (lane == 0) win = s;
    }
    __syncthreads();
    const PrimSlot w = win;
    if (gtid == 0) {
      a.out_u[it] = w.from;
      a.out_v[it] = w.id;
      a.out_w[it] = w.bv;
    }
    if (w.k != m - 1 && gtid == w.k % T) {  // swap-with-last (pointgen.py:141-148)
      const int64_t l = m - 1, bk = w.k;
      st.idx[bk] = st.idx[l];
      st.acore[bk] = st.acore[l];
      st.abest[bk] = st.abest[l];
      st.afrom[bk] = st.afrom[l];
#pragma unroll
      for (int t = 0; t < DIM; ++t) st.acoord[t * st.cap + bk] = st.acoord[t * st.cap + l];
    }
    cur = w.id;
#pragma unroll
    for (int t = 0; t < DIM; ++t) curc[t] = a.pts[(int64_t)cur * DIM + t];
    cc = a.core_sq[cur];
    __syncthreads();  // `win` / `wbest` reused by the next step
  }
}

__global__ void k_sqrt_inplace(double* __restrict__ w, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = sqrt(w[i]);
}

}  // namespace dmst

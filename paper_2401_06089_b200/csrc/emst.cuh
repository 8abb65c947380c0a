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

struct PrimSlot {  // one block's candidate of one step (+ the candidate point, so the
                   // next step needs no dependent load of its coordinates)
  double bv;
  int32_t key;    // tie-break key: compacted position (numba) or point id (numpy)
  int32_t k;      // compacted position
  int32_t id;     // point id
  int32_t from;
  double core;
  double x[EMST_MAX_DIM];
};

// slots are rewritten every other step by other SMs: read them from L2
__device__ __forceinline__ PrimSlot ldcg_slot(const PrimSlot* p) {
  PrimSlot s;
  s.bv = __ldcg(&p->bv);
  s.key = __ldcg(&p->key);
  s.k = __ldcg(&p->k);
  s.id = __ldcg(&p->id);
  s.from = __ldcg(&p->from);
  s.core = __ldcg(&p->core);
#pragma unroll
  for (int t = 0; t < EMST_MAX_DIM; ++t) s.x[t] = __ldcg(&p->x[t]);
  return s;
}

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

constexpr int PRIM_BLOCK = 512, PRIM_U = 4, PRIM_MAX_GRID = 296;
// positions per thread staged in shared memory after the register-resident
// ones: ~200 KB per CTA (8 B per coordinate + core + best, 4 B from + id)
template <int DIM>
__host__ __device__ constexpr int prim_smem_slots() {
  return (200 * 1024) / (PRIM_BLOCK * (8 * DIM + 24));
}
template <int DIM>
__host__ __device__ constexpr size_t prim_smem_bytes() {
  return (size_t)prim_smem_slots<DIM>() * PRIM_BLOCK * (8 * DIM + 24);
}
struct PrimArgs {
  const double* pts;
  const double* core_sq;
  int64_t n;
  PrimState st;
  PrimSlot* slots;          // [2][gridDim.x + 1]: block candidates, then the last element
  unsigned long long* bar;  // grid barrier counter (zeroed before the launch)
  int32_t* out_u;
  int32_t* out_v;
  double* out_w;            // w_sq until the final sqrt
};

template <int DIM>
struct PrimCand {
  double bv, core;
  int32_t key, k, id, from;
  double x[DIM];
  __device__ __forceinline__ void reset() {
    bv = __longlong_as_double(0x7ff0000000000000ll);
    key = 0x7fffffff;
    k = -1;
    id = from = 0;
    core = 0.0;
#pragma unroll
    for (int t = 0; t < DIM; ++t) x[t] = 0.0;
  }
  __device__ __forceinline__ void take(const PrimCand& q) {
    if (slot_less(q.bv, q.key, bv, key)) *this = q;
  }
  __device__ __forceinline__ void warp_min() {  // butterfly: every lane ends with the minimum
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      PrimCand q;
      q.bv = __shfl_xor_sync(kFull, bv, o);
      q.key = __shfl_xor_sync(kFull, key, o);
      q.k = __shfl_xor_sync(kFull, k, o);
      q.id = __shfl_xor_sync(kFull, id, o);
      q.from = __shfl_xor_sync(kFull, from, o);
      q.core = __shfl_xor_sync(kFull, core, o);
#pragma unroll
      for (int t = 0; t < DIM; ++t) q.x[t] = __shfl_xor_sync(kFull, x[t], o);
      take(q);
    }
  }
  __device__ __forceinline__ void store(PrimSlot& s) const {
    s.bv = bv;
    s.key = key;
    s.k = k;
    s.id = id;
    s.from = from;
    s.core = core;
#pragma unroll
    for (int t = 0; t < DIM; ++t) s.x[t] = x[t];
  }
  __device__ __forceinline__ void load(const PrimSlot& s) {
    bv = s.bv;
    key = s.key;
    k = s.k;
    id = s.id;
    from = s.from;
    core = s.core;
#pragma unroll
    for (int t = 0; t < DIM; ++t) x[t] = s.x[t];
  }
};

__device__ __forceinline__ void bar_arrive(unsigned long long* p) {
  asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ unsigned long long bar_poll(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// One cooperative launch for all n - 1 steps.  Step: every thread updates
// best/from of its compacted positions (k = gtid + j * T, U loads in flight)
// against the current point and keeps its lexicographic minimum (best,
// key); the owner of the last position publishes that element (the
// swap-with-last source); per-warp minima -> shared memory -> warp 0: block
// minimum -> slot, release-arrive on the grid counter, acquire-spin, then
// all slots (loads in flight together) -> the winner, which carries the
// next current point; one block barrier releases the other warps.  The
// owner thread of the winner's position moves the published last element
// into it, so the next step's reads of that position are its own writes.
template <int DIM, bool NUMPY>
__global__ void __launch_bounds__(PRIM_BLOCK) k_prim(PrimArgs a) {
  constexpr int NW = PRIM_BLOCK / 32;
  constexpr int SPL = (PRIM_MAX_GRID + 31) / 32;  // slots per lane (upper bound)
  __shared__ PrimSlot wbest[NW];
  __shared__ PrimSlot win, last;
  const uint32_t G = gridDim.x;
  const int64_t T = (int64_t)G * PRIM_BLOCK;
  const int64_t gtid = (int64_t)blockIdx.x * PRIM_BLOCK + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const PrimState& st = a.st;
  constexpr int U = DIM <= 3 ? PRIM_U : DIM <= 6 ? 2 : 1;  // register-resident positions
  int32_t cur = 0;
  double cc, curc[DIM];
#pragma unroll
  for (int t = 0; t < DIM; ++t) curc[t] = a.pts[t];
  cc = a.core_sq[0];
  // the thread's first U positions (k = gtid + q * T) live in registers for
  // the whole kernel: only the owner ever reads or writes a position, the
  // swap source is published from registers and the swap target is patched
  // in registers, so those positions never go back to memory; positions
  // beyond them are read and written in HBM / L2 as before.
  double rx[U][DIM], rck[U], rbb[U];
  int32_t rfr[U], rid[U];
#pragma unroll
  for (int q = 0; q < U; ++q) {
    const int64_t k = gtid + q * T;
    const bool ok = k < a.n - 1;
#pragma unroll
    for (int t = 0; t < DIM; ++t) rx[q][t] = ok ? st.acoord[t * st.cap + k] : 0.0;
    rck[q] = ok ? st.acore[k] : 0.0;
    rbb[q] = ok ? st.abest[k] : -1.0;
    rfr[q] = ok ? st.afrom[k] : 0;
    rid[q] = ok ? st.idx[k] : 0;
  }
  // the next S positions live in this CTA's shared memory (owner-only
  // slots, SoA per position index j: no bank conflicts, no barriers)
  constexpr int S = prim_smem_slots<DIM>();
  extern __shared__ __align__(16) unsigned char prim_sm[];
  double* sx = reinterpret_cast<double*>(prim_sm);          // [DIM][S][BLOCK]
  double* sck = sx + DIM * S * PRIM_BLOCK;                   // [S][BLOCK]
  double* sbb = sck + S * PRIM_BLOCK;                        // [S][BLOCK]
  int32_t* sfr = reinterpret_cast<int32_t*>(sbb + S * PRIM_BLOCK);
  int32_t* sid = sfr + S * PRIM_BLOCK;
  const int tid = threadIdx.x;
  for (int j = 0; j < S; ++j) {
    const int64_t k = gtid + (int64_t)(U + j) * T;
    const bool ok = k < a.n - 1;
#pragma unroll
    for (int t = 0; t < DIM; ++t) sx[(t * S + j) * PRIM_BLOCK + tid] = ok ? st.acoord[t * st.cap + k] : 0.0;
    sck[j * PRIM_BLOCK + tid] = ok ? st.acore[k] : 0.0;
    sbb[j * PRIM_BLOCK + tid] = ok ? st.abest[k] : -1.0;
    sfr[j * PRIM_BLOCK + tid] = ok ? st.afrom[k] : 0;
    sid[j * PRIM_BLOCK + tid] = ok ? st.idx[k] : 0;
  }
  for (int64_t it = 0; it < a.n - 1; ++it) {
    const int64_t m = a.n - 1 - it;
    PrimSlot* slots = a.slots + (it & 1) * (G + 1);
    PrimCand<DIM> best;
    best.reset();
    auto visit = [&](int64_t k, const double (&x)[DIM], double ck, double& bb, int32_t& fr, int32_t id,
                     bool in_memory) {
      double d = sqdist_prim<DIM, NUMPY>(x, curc);
      if (ck > d) d = ck;
      if (cc > d) d = cc;
      if (d < bb) {
        bb = d;
        fr = cur;
        if (in_memory) {
          st.abest[k] = d;
          st.afrom[k] = cur;
        }
      }
      const int32_t key = NUMPY ? id : (int32_t)k;
      if (k == m - 1) {  // publish the swap-with-last source (post-update)
        PrimSlot& l = slots[G];
        l.bv = bb;
        l.from = fr;
        l.id = id;
        l.core = ck;
#pragma unroll
        for (int t = 0; t < DIM; ++t) l.x[t] = x[t];
      }
      if (slot_less(bb, key, best.bv, best.key)) {
        best.bv = bb;
        best.key = key;
        best.k = (int32_t)k;
        best.id = id;
        best.from = fr;
        best.core = ck;
#pragma unroll
        for (int t = 0; t < DIM; ++t) best.x[t] = x[t];
      }
    };
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int64_t k = gtid + q * T;
      if (k < m) visit(k, rx[q], rck[q], rbb[q], rfr[q], rid[q], false);
    }
    for (int j = 0; j < S; ++j) {
      const int64_t k = gtid + (int64_t)(U + j) * T;
      if (k >= m) break;  // positions grow with j
      double x[DIM];
#pragma unroll
      for (int t = 0; t < DIM; ++t) x[t] = sx[(t * S + j) * PRIM_BLOCK + tid];
      double bb = sbb[j * PRIM_BLOCK + tid];
      int32_t fr = sfr[j * PRIM_BLOCK + tid];
      const double bb0 = bb;
      visit(k, x, sck[j * PRIM_BLOCK + tid], bb, fr, sid[j * PRIM_BLOCK + tid], false);
      if (bb != bb0) {
        sbb[j * PRIM_BLOCK + tid] = bb;
        sfr[j * PRIM_BLOCK + tid] = fr;
      }
    }
    constexpr int UM = DIM <= 4 ? 2 : 1;  // memory-resident positions in flight
    for (int64_t k0 = gtid + (int64_t)(U + S) * T; k0 < m; k0 += T * UM) {
      double x[UM][DIM], ck[UM], bb[UM];
      int32_t fr[UM], id[UM];
#pragma unroll
      for (int q = 0; q < UM; ++q) {
        const int64_t k = k0 + q * T;
        const bool ok = k < m;
#pragma unroll
        for (int t = 0; t < DIM; ++t) x[q][t] = ok ? st.acoord[t * st.cap + k] : 0.0;
        ck[q] = ok ? st.acore[k] : 0.0;
        bb[q] = ok ? st.abest[k] : -1.0;
        fr[q] = ok ? st.afrom[k] : 0;
        id[q] = ok ? st.idx[k] : 0;
      }
#pragma unroll
      for (int q = 0; q < UM; ++q) {
        const int64_t k = k0 + q * T;
        if (k < m) visit(k, x[q], ck[q], bb[q], fr[q], id[q], true);
      }
    }
    best.warp_min();
    if (lane == 0) best.store(wbest[wid]);
    __syncthreads();
    if (wid == 0) {
      PrimCand<DIM> c;
      if (lane < NW)
        c.load(wbest[lane]);
      else
        c.reset();
      c.warp_min();
      if (lane == 0) {
        c.store(slots[blockIdx.x]);
        bar_arrive(a.bar);
        const unsigned long long target = (unsigned long long)(it + 1) * G;
        while (bar_poll(a.bar) < target) {
        }
      }
      __syncwarp();
      // (best, key) of every slot at once (loads in flight together), the
      // minimum's slot index, then that slot and the published last element
      double sb[SPL];
      int32_t sk[SPL];
#pragma unroll
      for (int q = 0; q < SPL; ++q) {
        const uint32_t b = lane + 32u * q;
        sb[q] = b < G ? __ldcg(&slots[b].bv) : __longlong_as_double(0x7ff0000000000000ll);
        sk[q] = b < G ? __ldcg(&slots[b].key) : 0x7fffffff;
      }
      double bv = sb[0];
      int32_t bkey = sk[0], bslot = lane;
#pragma unroll
      for (int q = 1; q < SPL; ++q)
        if (slot_less(sb[q], sk[q], bv, bkey)) {
          bv = sb[q];
          bkey = sk[q];
          bslot = lane + 32 * q;
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(kFull, bv, o);
        const int32_t ok = __shfl_xor_sync(kFull, bkey, o), os = __shfl_xor_sync(kFull, bslot, o);
        if (slot_less(ov, ok, bv, bkey)) {
          bv = ov;
          bkey = ok;
          bslot = os;
        }
      }
      if (lane == 0) win = ldcg_slot(&slots[bslot]);
      if (lane == 1) last = ldcg_slot(&slots[G]);
    }
    __syncthreads();
    PrimCand<DIM> w;
    w.load(win);
    if (gtid == 0) {
      a.out_u[it] = w.from;
      a.out_v[it] = w.id;
      a.out_w[it] = w.bv;
    }
    if (w.k != m - 1 && gtid == (int64_t)w.k % T) {  // swap-with-last (pointgen.py:141-148)
      const int64_t bk = w.k;
      const PrimSlot& l = last;
      const int64_t q0 = bk / T;
      if (q0 >= U && q0 < U + S) {
        const int j = (int)(q0 - U);
#pragma unroll
        for (int t = 0; t < DIM; ++t) sx[(t * S + j) * PRIM_BLOCK + tid] = l.x[t];
        sck[j * PRIM_BLOCK + tid] = l.core;
        sbb[j * PRIM_BLOCK + tid] = l.bv;
        sfr[j * PRIM_BLOCK + tid] = l.from;
        sid[j * PRIM_BLOCK + tid] = l.id;
      } else if (q0 < U) {
#pragma unroll
        for (int q = 0; q < U; ++q)
          if (q == q0) {
            rid[q] = l.id;
            rck[q] = l.core;
            rbb[q] = l.bv;
            rfr[q] = l.from;
#pragma unroll
            for (int t = 0; t < DIM; ++t) rx[q][t] = l.x[t];
          }
      } else {
        st.idx[bk] = l.id;
        st.acore[bk] = l.core;
        st.abest[bk] = l.bv;
        st.afrom[bk] = l.from;
#pragma unroll
        for (int t = 0; t < DIM; ++t) st.acoord[t * st.cap + bk] = l.x[t];
      }
    }
    cur = w.id;
#pragma unroll
    for (int t = 0; t < DIM; ++t) curc[t] = w.x[t];
    cc = w.core;
    __syncthreads();  // win / last / wbest read before the next step rewrites them
  }
}

__global__ void k_sqrt_inplace(double* __restrict__ w, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = sqrt(w[i]);
}

}  // namespace dmst

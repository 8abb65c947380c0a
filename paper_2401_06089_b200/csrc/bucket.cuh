// Unstable bucketing of scatter-max records + shared-memory apply.
//
// maxIncident (tree_core.py:193-199; contraction.py:149-154, 173-175 of
// /root/reference/pkg/src/dendromst/) is a scatter-max of 2 records per edge
// (vertex x, rank j, other endpoint) into a per-vertex array.  Done with
// global atomics it is one random DRAM read-modify-write per record.  Here
// the records are instead grouped by "fine bucket" (FB = 8192 consecutive
// vertices) with two order-free multisplit passes (coarse then fine; no
// ranking, a shared-memory atomic per record assigns its slot), after which
// one CTA per fine bucket reduces its records in shared memory and writes
// the bucket's slice of mi64 (and V1's outputs) with coalesced stores.
#pragma once
#include "common.cuh"

namespace dmst {

constexpr int FB_BITS = 13;                  // fine bucket = 8192 vertices (64 KB of smem state)
constexpr int FB = 1 << FB_BITS;
constexpr int BK_BLOCK = 256, BK_ITEMS = 16;  // bucketing sub-tile = 4096 records
constexpr int BK_T = BK_BLOCK * BK_ITEMS;
constexpr int BK_SPAN = 4096;                 // max fine buckets one pass-B sub-tile may touch

struct Recs {  // SoA records (vertex, j + 1, other end)
  uint32_t* x;
  uint32_t* j1;
  uint32_t* o;
};

// Record i of edge i >> 1 of a view (endpoints euv).
struct EdgeRecSrc {
  const int2* __restrict__ euv;
  __device__ __forceinline__ void load(int64_t i, uint32_t& x, uint32_t& j1, uint32_t& o) const {
    const int2 e = __ldg(euv + (i >> 1));
    const bool second = i & 1;
    x = (uint32_t)(second ? e.y : e.x);
    o = (uint32_t)(second ? e.x : e.y);
    j1 = (uint32_t)(i >> 1) + 1u;
  }
  __device__ __forceinline__ uint32_t vertex(int64_t i) const {
    const int2 e = __ldg(euv + (i >> 1));
    return (uint32_t)((i & 1) ? e.y : e.x);
  }
};

struct SoaRecSrc {
  const uint32_t* __restrict__ x;
  const uint32_t* __restrict__ j1;
  const uint32_t* __restrict__ o;
  __device__ __forceinline__ void load(int64_t i, uint32_t& xx, uint32_t& jj, uint32_t& oo) const {
    xx = ld_stream(x + i);
    jj = ld_stream(j1 + i);
    oo = ld_stream(o + i);
  }
  __device__ __forceinline__ uint32_t vertex(int64_t i) const { return ld_stream(x + i); }
};

// counts[f] += number of records whose vertex is in fine bucket f, for
// f in [flo, flo + 16384) (windowed: very large views run several windows).
constexpr int FH_WINDOW = 16384;
template <class Src>
__global__ void __launch_bounds__(256) k_fine_hist(Src src, int64_t m, uint32_t flo, uint32_t nf,
                                                   uint32_t* __restrict__ counts) {
  constexpr int W = FH_WINDOW;
  extern __shared__ uint32_t h[];  // [W]
  for (int i = threadIdx.x; i < W; i += 256) h[i] = 0;
  __syncthreads();
  constexpr int U = 8;
  const int64_t stride = (int64_t)gridDim.x * 256 * U;
  for (int64_t b = (int64_t)blockIdx.x * 256 * U + threadIdx.x; b < m; b += stride) {
    uint32_t f[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int64_t i = b + q * 256;
      f[q] = i < m ? (src.vertex(i) >> FB_BITS) - flo : 0xffffffffu;
    }
#pragma unroll
    for (int q = 0; q < U; ++q)
      if (f[q] < (uint32_t)W) atomicAdd(&h[f[q]], 1u);
  }
  __syncthreads();
  const uint32_t lim = min((uint32_t)W, nf - flo);
  for (uint32_t i = threadIdx.x; i < lim; i += 256)
    if (h[i]) atomicAdd(counts + flo + i, h[i]);
}

// Single CTA: fine_base = exclusive scan of counts (nf + 1 entries), fine
// cursors, coarse bases/cursors (coarse bucket c = fine buckets
// [c << gshift, (c + 1) << gshift)).
__global__ void __launch_bounds__(1024) k_fine_scan(const uint32_t* __restrict__ counts, uint32_t nf,
                                                    uint32_t gshift, uint32_t* __restrict__ fine_base,
                                                    uint32_t* __restrict__ fine_cur,
                                                    uint32_t* __restrict__ coarse_cur) {
  __shared__ uint32_t scratch[1024 / 32 + 1];
  const uint32_t per = (nf + 1023) / 1024;
  const uint32_t b = threadIdx.x * per, e = min(nf, b + per);
  uint32_t s = 0;
  for (uint32_t i = b; i < e; ++i) s += counts[i];
  uint32_t tot;
  uint32_t run = block_excl_sum<1024>(s, scratch, &tot);
  for (uint32_t i = b; i < e; ++i) {
    fine_base[i] = run;
    fine_cur[i] = run;
    if ((i & ((1u << gshift) - 1)) == 0) coarse_cur[i >> gshift] = run;
    run += counts[i];
  }
  if (threadIdx.x == 0) fine_base[nf] = tot;
}

// One order-free multisplit pass.  Pass A (FINE = false): bucket = fine >> gshift
// (< 256 buckets).  Pass B (FINE = true): bucket = fine bucket, input already
// grouped by coarse bucket so a sub-tile touches a narrow fine range.
// Persistent CTAs, grid-stride over sub-tiles of BK_T records.
template <bool FINE>
constexpr size_t bucket_smem_bytes() { return 4 * (2 * (FINE ? BK_SPAN : 256) + 3 * BK_T); }

template <bool FINE, class Src>
__global__ void __launch_bounds__(BK_BLOCK) k_bucket(Src src, int64_t m, uint32_t gshift,
                                                     uint32_t* __restrict__ cursor, Recs out) {
  constexpr int NC = FINE ? BK_SPAN : 256;
  extern __shared__ uint32_t bsm[];
  uint32_t* cnt = bsm;            // [NC]
  uint32_t* gofs = bsm + NC;      // [NC]
  uint32_t* stx = bsm + 2 * NC;   // [BK_T]
  uint32_t* stj = stx + BK_T;
  uint32_t* sto = stj + BK_T;
  __shared__ uint32_t scratch[BK_BLOCK / 32 + 1];
  __shared__ uint32_t s_lo, s_span;
  const uint32_t tid = threadIdx.x;
  for (int64_t t0 = (int64_t)blockIdx.x * BK_T; t0 < m; t0 += (int64_t)gridDim.x * BK_T) {
    const int64_t rem = m - t0;
    const int count = rem < BK_T ? (int)rem : BK_T;
    if (tid == 0) {
      uint32_t lo = 0, span = NC;
      if (FINE) {
        const uint32_t c0 = src.vertex(t0) >> (FB_BITS + gshift);
        const uint32_t c1 = src.vertex(t0 + count - 1) >> (FB_BITS + gshift);
        lo = c0 << gshift;
        span = (c1 + 1 - c0) << gshift;
      }
      s_lo = lo;
      s_span = span;
    }
    for (int i = tid; i < NC; i += BK_BLOCK) cnt[i] = 0;
    __syncthreads();
    const uint32_t lo = s_lo;
    const bool smem_path = s_span <= (uint32_t)NC;
    uint32_t x[BK_ITEMS], j1[BK_ITEMS], o[BK_ITEMS], bk[BK_ITEMS], slot[BK_ITEMS];
#pragma unroll
    for (int i = 0; i < BK_ITEMS; ++i) {
      const int li = i * BK_BLOCK + tid;
      if (li < count) src.load(t0 + li, x[i], j1[i], o[i]);
    }
    if (!smem_path) {
      // rare: a sub-tile spanning more fine buckets than the shared counters
      // hold (heavily skewed vertex ids) -> one global atomic per record
#pragma unroll
      for (int i = 0; i < BK_ITEMS; ++i) {
        const int li = i * BK_BLOCK + tid;
        if (li < count) {
          const uint32_t f = x[i] >> FB_BITS;
          const uint32_t d = atomicAdd(cursor + f, 1u);
          out.x[d] = x[i];
          out.j1[d] = j1[i];
          out.o[d] = o[i];
        }
      }
      __syncthreads();
      continue;
    }
#pragma unroll
    for (int i = 0; i < BK_ITEMS; ++i) {
      const int li = i * BK_BLOCK + tid;
      if (li < count) {
        const uint32_t f = x[i] >> FB_BITS;
        bk[i] = FINE ? f - lo : f >> gshift;
        slot[i] = atomicAdd(&cnt[bk[i]], 1u);
      }
    }
    __syncthreads();
    // local exclusive scan of the counters + global reservation; thread t owns
    // counters [t * per, (t + 1) * per) of the active span (per = 1 unless a
    // sub-tile straddles many buckets), so reservations go out in parallel
    const uint32_t span = FINE ? s_span : (uint32_t)NC;
    const uint32_t per = (span + BK_BLOCK - 1) / BK_BLOCK;
    constexpr int PMAX = NC / BK_BLOCK;
    uint32_t c[PMAX], s = 0;
#pragma unroll
    for (int q = 0; q < PMAX; ++q) {
      c[q] = (uint32_t)q < per ? cnt[tid * per + q] : 0u;
      s += c[q];
    }
    uint32_t tot;
    uint32_t run = block_excl_sum<BK_BLOCK>(s, scratch, &tot);
    uint32_t g[PMAX];
#pragma unroll
    for (int q = 0; q < PMAX; ++q) {
      const uint32_t b = tid * per + q;
      g[q] = ((uint32_t)q < per && c[q]) ? atomicAdd(cursor + (FINE ? lo + b : b), c[q]) : 0u;
    }
#pragma unroll
    for (int q = 0; q < PMAX; ++q) {
      if ((uint32_t)q < per) {
        const uint32_t b = tid * per + q;
        if (c[q]) gofs[b] = g[q] - run;
        cnt[b] = run;  // becomes the local start of bucket b
        run += c[q];
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < BK_ITEMS; ++i) {
      const int li = i * BK_BLOCK + tid;
      if (li < count) {
        const uint32_t p = cnt[bk[i]] + slot[i];
        stx[p] = x[i];
        stj[p] = j1[i];
        sto[p] = o[i];
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < BK_ITEMS; ++i) {
      const int sidx = i * BK_BLOCK + tid;
      if (sidx < count) {
        const uint32_t xx = stx[sidx];
        const uint32_t f = xx >> FB_BITS;
        const uint32_t b = FINE ? f - lo : f >> gshift;
        const uint32_t d = gofs[b] + sidx;
        out.x[d] = xx;
        out.j1[d] = stj[sidx];
        out.o[d] = sto[sidx];
      }
    }
    __syncthreads();
  }
}

// One CTA per fine bucket: reduce its records in shared memory (max rank,
// then the winning record's other end) and write, for every vertex x of the
// bucket: mi64[x] = ((j + 1) << 32) | other (0 if isolated), V1's parent
// output (vertex_parent for view 0, super maxIncident in global ranks for
// later views) and the per-edge child count (2-bit field, L2-resident).
struct MiApplyOut {
  unsigned long long* mi64;
  int32_t* parent_out;
  const int32_t* grank;  // null => identity (view 0)
  uint32_t* cnt2;
};

__global__ void __launch_bounds__(512) k_mi_apply_smem(Recs rec, const uint32_t* __restrict__ fine_base,
                                                       int64_t nv, MiApplyOut out) {
  extern __shared__ unsigned long long smi[];  // [FB] max ((j + 1) << 32 | other)
  const uint32_t f = blockIdx.x;
  const int64_t v0 = (int64_t)f << FB_BITS;
  for (int i = threadIdx.x; i < FB; i += blockDim.x) smi[i] = 0ull;
  __syncthreads();
  const uint32_t rb = fine_base[f], re = fine_base[f + 1];
  constexpr int U = 8;
  const uint32_t step = blockDim.x * U;
  for (uint32_t b = rb + threadIdx.x; b < re; b += step) {
    uint32_t xl[U];
    unsigned long long pk[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const uint32_t i = b + q * blockDim.x;
      xl[q] = i < re ? ld_stream(rec.x + i) - (uint32_t)v0 : 0u;
      pk[q] = i < re ? ((unsigned long long)ld_stream(rec.j1 + i) << 32) | ld_stream(rec.o + i) : 0ull;
    }
#pragma unroll
    for (int q = 0; q < U; ++q)
      if (pk[q]) atomicMax(&smi[xl[q]], pk[q]);
  }
  __syncthreads();
  const int lim = nv - v0 < FB ? (int)(nv - v0) : FB;
  for (int i = threadIdx.x; i < lim; i += blockDim.x) {
    const unsigned long long m = smi[i];
    const uint32_t b = (uint32_t)(m >> 32);
    int32_t par = -1;
    if (b) {
      const uint32_t j = b - 1;
      par = out.grank ? __ldg(out.grank + j) : (int32_t)j;
      atomicAdd(out.cnt2 + (j >> 4), 1u << ((j & 15) * 2));
    }
    out.mi64[v0 + i] = m;
    out.parent_out[v0 + i] = par;
  }
}

}  // namespace dmst

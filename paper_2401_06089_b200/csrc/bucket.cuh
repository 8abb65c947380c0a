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
#include <type_traits>

#include "common.cuh"
#include "radix.cuh"  // TMA bulk-copy / mbarrier helpers

namespace dmst {

constexpr int FB_BITS = 13;                  // fine bucket = 8192 vertices (64 KB of smem state)
constexpr int FB = 1 << FB_BITS;
// multisplit geometry: pass A (coarse, <= 256 buckets) and pass B (fine)
constexpr int BKA_BLOCK = 512, BKA_ITEMS = 8;   // 4096 records per sub-tile
constexpr int BKA_PER_SM = 2;                   // pass-A CTAs per SM
constexpr int BKB_BLOCK = 512, BKB_ITEMS = 4;   // 2048 records per sub-tile
constexpr int BKB_SPAN = 1024;                  // max fine buckets a pass-B sub-tile may touch
constexpr int BKB_PER_SM = 4;                   // pass-B CTAs per SM (in-place regrouping: ~56 KB smem)

// Records are AoS tuples of RW words whose first word is the bucketing key
// (maxIncident: (vertex, j + 1, other end), RW = 3; chain links: (rank,
// parent), RW = 2): a bucket run of m records is one contiguous run of
// 4 RW m bytes.
struct Recs {
  uint32_t* r;  // [RW m]
};

// Record sources.  Besides global loads (load / vertex) a source describes
// its staged form: NS streams of sb(s) bytes per record, contiguous from
// ptr(s), fetched per sub-tile with TMA bulk copies; get() / staged_vertex()
// then read the stage (st[s] = stream s of the sub-tile).
//
// Record i of edge i >> 1 of a view (endpoints euv).
struct EdgeRecSrc {
  static constexpr int RW = 3, NS = 1;
  __host__ __device__ static constexpr int sb(int) { return 4; }  // 8 B per edge = 2 records
  const int2* __restrict__ euv;
  __device__ __forceinline__ const void* ptr(int) const { return euv; }
  __device__ __forceinline__ void get(const unsigned char* const* st, int li, int64_t i, uint32_t (&r)[3]) const {
    const int2 e = reinterpret_cast<const int2*>(st[0])[li >> 1];
    const bool second = i & 1;
    r[0] = (uint32_t)(second ? e.y : e.x);
    r[2] = (uint32_t)(second ? e.x : e.y);
    r[1] = (uint32_t)(i >> 1) + 1u;
  }
  __device__ __forceinline__ uint32_t staged_vertex(const unsigned char* const* st, int li, int64_t i) const {
    const int2 e = reinterpret_cast<const int2*>(st[0])[li >> 1];
    return (uint32_t)((i & 1) ? e.y : e.x);
  }
  __device__ __forceinline__ void load(int64_t i, uint32_t (&r)[3]) const {
    const int2 e = __ldg(euv + (i >> 1));
    const bool second = i & 1;
    r[0] = (uint32_t)(second ? e.y : e.x);
    r[2] = (uint32_t)(second ? e.x : e.y);
    r[1] = (uint32_t)(i >> 1) + 1u;
  }
  __device__ __forceinline__ uint32_t vertex(int64_t i) const {
    const int2 e = __ldg(euv + (i >> 1));
    return (uint32_t)((i & 1) ? e.y : e.x);
  }
};

// Materialised records (RW words each).
template <int RW_>
struct AosRecSrc {
  static constexpr int RW = RW_, NS = 1;
  __host__ __device__ static constexpr int sb(int) { return 4 * RW; }
  const uint32_t* __restrict__ r;
  __device__ __forceinline__ const void* ptr(int) const { return r; }
  __device__ __forceinline__ void get(const unsigned char* const* st, int li, int64_t, uint32_t (&o)[RW]) const {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(st[0]) + RW * li;
#pragma unroll
    for (int q = 0; q < RW; ++q) o[q] = p[q];
  }
  __device__ __forceinline__ uint32_t staged_vertex(const unsigned char* const* st, int li, int64_t) const {
    return reinterpret_cast<const uint32_t*>(st[0])[RW * li];
  }
  __device__ __forceinline__ void load(int64_t i, uint32_t (&o)[RW]) const {
#pragma unroll
    for (int q = 0; q < RW; ++q) o[q] = ld_stream(r + RW * i + q);
  }
  __device__ __forceinline__ uint32_t vertex(int64_t i) const { return __ldg(r + RW * i); }
};

template <class Src>
__device__ __forceinline__ const int2* edge_ptr(const Src& src) {
  if constexpr (std::is_same<Src, EdgeRecSrc>::value) return src.euv;
  else return nullptr;
}

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
  bool vec = false;
  if constexpr (std::is_same<Src, EdgeRecSrc>::value) vec = aligned16(src.euv);
  if (vec) {
    // two edges (four records) per 16-B load, four loads in flight per thread
    constexpr int U = 4;
    const int64_t ne = m >> 1, np = ne >> 1;  // edges, edge pairs
    const int4* pairs = reinterpret_cast<const int4*>(edge_ptr(src));
    const int64_t stride = (int64_t)gridDim.x * 256 * U;
    for (int64_t b = (int64_t)blockIdx.x * 256 * U + threadIdx.x; b < np; b += stride) {
      int4 e[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int64_t i = b + q * 256;
        e[q] = i < np ? ld_stream(pairs + i) : make_int4(-1, -1, -1, -1);
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const uint32_t f0 = ((uint32_t)e[q].x >> FB_BITS) - flo, f1 = ((uint32_t)e[q].y >> FB_BITS) - flo;
        const uint32_t f2 = ((uint32_t)e[q].z >> FB_BITS) - flo, f3 = ((uint32_t)e[q].w >> FB_BITS) - flo;
        if (e[q].x >= 0) {
          if (f0 < (uint32_t)W) atomicAdd(&h[f0], 1u);
          if (f1 < (uint32_t)W) atomicAdd(&h[f1], 1u);
          if (f2 < (uint32_t)W) atomicAdd(&h[f2], 1u);
          if (f3 < (uint32_t)W) atomicAdd(&h[f3], 1u);
        }
      }
    }
    if ((ne & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd edge count: the last edge
      const int2 e = edge_ptr(src)[ne - 1];
      const uint32_t f0 = ((uint32_t)e.x >> FB_BITS) - flo, f1 = ((uint32_t)e.y >> FB_BITS) - flo;
      if (f0 < (uint32_t)W) atomicAdd(&h[f0], 1u);
      if (f1 < (uint32_t)W) atomicAdd(&h[f1], 1u);
    }
  } else {
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
// (<= 256 buckets).  Pass B (FINE = true): bucket = fine bucket, input already
// grouped by coarse bucket so a sub-tile touches a narrow fine range.
// Persistent CTAs take sub-tiles round-robin; sub-tile k + 2 is fetched by a
// TMA bulk copy (mbarrier completion) while sub-tile k is grouped, so DRAM
// latency stays off the critical path.  Per sub-tile: a shared-memory atomic
// per record gives its slot within its bucket, one global atomic per
// non-empty bucket reserves the output range, the records are regrouped in
// shared memory and written out as one word stream (consecutive threads ->
// consecutive words of a bucket run).  Only the slots live in registers.
// INPLACE (AoS sources whose staged record is the output record): the
// regrouped sub-tile is written into the consumed stage buffer, so no
// separate staging area and ~2x the CTAs per SM.
template <class Src, int BLOCK, int ITEMS, int NC>
struct SplitSmem {
  static constexpr int T = BLOCK * ITEMS;
  static constexpr bool INPLACE = Src::NS == 1 && Src::sb(0) == 4 * Src::RW;
  __host__ __device__ static constexpr size_t stream_bytes(int s) { return ((size_t)T * Src::sb(s) + 127) & ~size_t(127); }
  __host__ __device__ static constexpr size_t stream_off(int s) {
    size_t b = 0;
    for (int q = 0; q < s; ++q) b += stream_bytes(q);
    return b;
  }
  __host__ __device__ static constexpr size_t in_bytes() { return stream_off(Src::NS); }
  __host__ __device__ static constexpr size_t off_st() { return 2 * in_bytes(); }
  __host__ __device__ static constexpr size_t off_cnt() { return off_st() + (INPLACE ? 0 : 4 * Src::RW * (size_t)T); }
  __host__ __device__ static constexpr size_t bytes() { return off_cnt() + 8 * (size_t)NC; }
};

// Write-out: one record per thread (8-B records, and the 12-B records of
// pass A: 1.71 -> 1.67 ms, link splits 1.28 -> 1.18 ms at 128M) or, for pass B's
// in-place 12-B records, one word stream (per-record there: 1.83 -> 2.11 ms).
template <bool FINE, class Src, int BLOCK, int ITEMS, int NC, bool PERREC = (Src::RW == 2 || !FINE)>
__global__ void __launch_bounds__(BLOCK) k_split(Src src, int64_t m, uint32_t gshift,
                                                 uint32_t* __restrict__ cursor, Recs out) {
  using S = SplitSmem<Src, BLOCK, ITEMS, NC>;
  constexpr int T = S::T, RW = Src::RW, NS = Src::NS;
  extern __shared__ __align__(128) unsigned char sm[];
  uint32_t* st = reinterpret_cast<uint32_t*>(sm + S::off_st());    // [RW T] grouped records
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sm + S::off_cnt());  // [NC]
  uint32_t* gofs = cnt + NC;                                       // [NC]
  __shared__ uint32_t scratch[BLOCK / 32 + 1];
  __shared__ uint32_t s_lo, s_span;
  __shared__ __align__(8) uint64_t bar[2];
  const uint32_t tid = threadIdx.x;
  const int64_t ntiles = (m + T - 1) / T;
  bool tma = true;
#pragma unroll
  for (int q = 0; q < NS; ++q) tma &= aligned16(src.ptr(q));

  auto issue = [&](int64_t tile, int buf) {
    const int64_t t0 = tile * T;
    if (!tma || tile >= ntiles || t0 + T > m) return;
    fence_proxy_async();
    uint32_t bytes = 0;
#pragma unroll
    for (int q = 0; q < NS; ++q) bytes += (uint32_t)(T * Src::sb(q));
    mbar_expect_tx(&bar[buf], bytes);
#pragma unroll
    for (int q = 0; q < NS; ++q)
      bulk_g2s(sm + buf * S::in_bytes() + S::stream_off(q), (const char*)src.ptr(q) + t0 * Src::sb(q),
               (uint32_t)(T * Src::sb(q)), &bar[buf]);
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
    issue(blockIdx.x, 0);
    issue(blockIdx.x + gridDim.x, 1);
  }

  int k = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
    const int buf = k & 1;
    const unsigned char* stage[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) stage[q] = sm + buf * S::in_bytes() + S::stream_off(q);
    const int64_t t0 = tile * T;
    const int count = m - t0 < T ? (int)(m - t0) : T;
    const bool staged = tma && count == T;
    if (staged) mbar_wait(&bar[buf], (uint32_t)(k >> 1) & 1u);
    auto rec = [&](int li, uint32_t (&r)[RW]) {
      if (staged)
        src.get(stage, li, t0 + li, r);
      else
        src.load(t0 + li, r);
    };
    auto vtx = [&](int li) { return staged ? src.staged_vertex(stage, li, t0 + li) : src.vertex(t0 + li); };
    if (tid == 0) {
      uint32_t lo = 0, span = NC;
      if (FINE) {
        const uint32_t c0 = vtx(0) >> (FB_BITS + gshift);
        const uint32_t c1 = vtx(count - 1) >> (FB_BITS + gshift);
        lo = c0 << gshift;
        span = (c1 + 1 - c0) << gshift;
      }
      s_lo = lo;
      s_span = span;
    }
    for (int i = tid; i < NC; i += BLOCK) cnt[i] = 0;
    __syncthreads();
    const uint32_t lo = s_lo;
    if (s_span > (uint32_t)NC) {
      // rare: a sub-tile spanning more fine buckets than the shared counters
      // hold (heavily skewed vertex ids) -> one global atomic per record
      for (int li = tid; li < count; li += BLOCK) {
        uint32_t r[RW];
        rec(li, r);
        const uint64_t d = atomicAdd(cursor + (r[0] >> FB_BITS), 1u);
#pragma unroll
        for (int q = 0; q < RW; ++q) out.r[RW * d + q] = r[q];
      }
      __syncthreads();
      if (tid == 0) issue(tile + 2 * (int64_t)gridDim.x, buf);
      continue;
    }
    auto bucket = [&](uint32_t x) { return FINE ? (x >> FB_BITS) - lo : (x >> FB_BITS) >> gshift; };
    uint32_t slot[ITEMS];
    uint32_t keep[S::INPLACE ? ITEMS : 1][RW];  // in-place: records held across the regrouping
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int li = i * BLOCK + tid;
      if (li < count) {
        if constexpr (S::INPLACE) {
          rec(li, keep[i]);
          slot[i] = atomicAdd(&cnt[bucket(keep[i][0])], 1u);
        } else {
          slot[i] = atomicAdd(&cnt[bucket(vtx(li))], 1u);
        }
      }
    }
    __syncthreads();
    // exclusive scan of the counters + global reservation; thread t owns
    // counters [t * PER, (t + 1) * PER)
    constexpr int PER = (NC + BLOCK - 1) / BLOCK;
    uint32_t c[PER], sum = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const uint32_t b = tid * PER + q;
      c[q] = b < (uint32_t)NC ? cnt[b] : 0u;
      sum += c[q];
    }
    uint32_t tot;
    uint32_t run = block_excl_sum<BLOCK>(sum, scratch, &tot);
    // the reservations' round trip overlaps the regrouping below: their
    // results are only needed for the write-out
    uint32_t g[PER], lst[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const uint32_t b = tid * PER + q;
      g[q] = 0;
      lst[q] = run;
      if (b < (uint32_t)NC) {
        if (c[q]) g[q] = atomicAdd(cursor + (FINE ? lo + b : b), c[q]);
        cnt[b] = run;  // local start of bucket b
        run += c[q];
      }
    }
    __syncthreads();
    uint32_t* stg = S::INPLACE ? reinterpret_cast<uint32_t*>(const_cast<unsigned char*>(stage[0])) : st;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int li = i * BLOCK + tid;
      if (li < count) {
        uint32_t r[RW];
        if constexpr (S::INPLACE) {
#pragma unroll
          for (int q = 0; q < RW; ++q) r[q] = keep[i][q];
        } else {
          rec(li, r);
        }
        const uint32_t p = cnt[bucket(r[0])] + slot[i];
#pragma unroll
        for (int q = 0; q < RW; ++q) stg[RW * p + q] = r[q];
      }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const uint32_t b = tid * PER + q;
      if (b < (uint32_t)NC && c[q]) gofs[b] = g[q] - lst[q];
    }
    __syncthreads();
    if (!S::INPLACE && tid == 0) issue(tile + 2 * (int64_t)gridDim.x, buf);  // stage buffer consumed
    if constexpr (PERREC) {
      // one record per thread: its bucket's offset is looked up once and the
      // record leaves as RW-word (8-B for RW = 2) stores
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int p = i * BLOCK + tid;
        if (p < count) {
          uint32_t r[RW];
          if constexpr (RW == 2) {
            const uint2 x = reinterpret_cast<const uint2*>(stg)[p];
            r[0] = x.x;
            r[1] = x.y;
          } else {
#pragma unroll
            for (int q = 0; q < RW; ++q) r[q] = stg[RW * p + q];
          }
          const uint64_t d = (uint64_t)gofs[bucket(r[0])] + (uint32_t)p;
          if constexpr (RW == 2) {
            reinterpret_cast<uint2*>(out.r)[d] = make_uint2(r[0], r[1]);
          } else {
#pragma unroll
            for (int q = 0; q < RW; ++q) out.r[RW * d + q] = r[q];
          }
        }
      }
    } else {
      for (int s_ = tid; s_ < RW * count; s_ += BLOCK) {
        const int it = s_ / RW;
        out.r[RW * (uint64_t)gofs[bucket(stg[RW * it])] + s_] = stg[s_];
      }
    }
    __syncthreads();
    if (S::INPLACE && tid == 0) issue(tile + 2 * (int64_t)gridDim.x, buf);  // regrouped tile written out
  }
}

// Alternative apply for records grouped by 4M-vertex SLICE (pass A only,
// coarse bucket = slice): one 64-bit atomicMax per record into mi64, which
// was zeroed; CTAs run in record order, so the slice being updated (32 MB of
// mi64) stays L2-resident (L2 atomics: ~210 G/s vs ~30 G/s DRAM-resident,
// tools/randbench.cu).  V1 (parents, child counts) then runs as k_v1.
#ifndef DMST_SLICE_BITS
#define DMST_SLICE_BITS 21
#endif
constexpr int kSliceBits = DMST_SLICE_BITS;  // 2M vertices = 16 MB of mi64 per slice (22: 32 MB, 21.64 vs 21.59 ms; 23: 22.6 ms)
// Coarse cursors of the sliced split from per-slice counts (<= 256 slices).
__global__ void __launch_bounds__(256) k_slice_scan(const uint32_t* __restrict__ counts, uint32_t ns,
                                                    uint32_t* __restrict__ coarse_cur) {
  __shared__ uint32_t scratch[256 / 32 + 1];
  const uint32_t c = threadIdx.x < ns ? counts[threadIdx.x] : 0u;
  uint32_t tot;
  const uint32_t run = block_excl_sum<256>(c, scratch, &tot);
  if (threadIdx.x < ns) coarse_cur[threadIdx.x] = run;
}

#ifndef DMST_MI_ATOMIC_G
#define DMST_MI_ATOMIC_G 4
#endif
constexpr int kMiAtomicGroups = DMST_MI_ATOMIC_G;  // groups of 4 records (48 B = three 16-B loads) per thread
__global__ void __launch_bounds__(256) k_mi_atomic(Recs rec, int64_t m, unsigned long long* __restrict__ mi64) {
  constexpr int G = kMiAtomicGroups;
  const int64_t g0 = (int64_t)blockIdx.x * 256 * G + threadIdx.x;  // group index
  const int64_t ng = m / 4;
  const uint4* r4 = reinterpret_cast<const uint4*>(rec.r);
  uint4 a[G][3];
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int64_t g = g0 + q * 256;
#pragma unroll
    for (int t = 0; t < 3; ++t) a[q][t] = g < ng ? ld_stream(r4 + 3 * g + t) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const uint32_t w[12] = {a[q][0].x, a[q][0].y, a[q][0].z, a[q][0].w, a[q][1].x, a[q][1].y,
                            a[q][1].z, a[q][1].w, a[q][2].x, a[q][2].y, a[q][2].z, a[q][2].w};
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const unsigned long long pk = ((unsigned long long)w[3 * r + 1] << 32) | w[3 * r + 2];
      if (pk) atomicMax(mi64 + w[3 * r], pk);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (m & 3)) {  // the last m % 4 records
    const int64_t i = (m & ~int64_t(3)) + threadIdx.x;
    const unsigned long long pk = ((unsigned long long)ld_stream(rec.r + 3 * i + 1) << 32) | ld_stream(rec.r + 3 * i + 2);
    if (pk) atomicMax(mi64 + ld_stream(rec.r + 3 * i), pk);
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
      xl[q] = i < re ? ld_stream(rec.r + 3 * (uint64_t)i) - (uint32_t)v0 : 0u;
      pk[q] = i < re ? ((unsigned long long)ld_stream(rec.r + 3 * (uint64_t)i + 1) << 32) |
                           ld_stream(rec.r + 3 * (uint64_t)i + 2)
                     : 0ull;
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

// Stable LSD radix sort passes, reduce-then-scan, with TMA-staged input.
//
// One 8-bit digit per pass, three kernels:
//   k_upsweep    each CTA counts the digits of its contiguous chunk of the
//                input (keys only) -> counts[digit][chunk];
//   k_chunk_scan one CTA: exclusive scan of counts in digit-major order ->
//                the global output offset of every (digit, chunk);
//   k_downsweep  persistent: CTA c walks its chunk in sub-tiles of T items,
//                keeps a running output offset per digit in shared memory
//                (no inter-CTA look-back, no spinning), ranks each sub-tile
//                in shared memory and writes every digit run contiguously.
// The next sub-tile's input is fetched by cp.async.bulk (TMA bulk copy,
// completion on an mbarrier) into a second staging buffer while the
// current one is ranked, so DRAM latency is off the critical path.
//
// Loaders describe the input streams (staged) and how a (key, payload)
// item is formed from them, so the first pass of a sort can build keys on
// the fly from the caller's arrays and the last pass (Emitter) can write
// final outputs.  Payloads are VW 32-bit words (SoA in shared memory).
//
// Replaces `np.argsort(-w, kind="stable")` (tree_core.py:180) and
// `np.lexsort` (expansion.py:135) of /root/reference/pkg/src/dendromst/,
// and partitions the scatter-max records of np.maximum.at
// (tree_core.py:197-198) so their updates stay in L2 / shared memory.
#pragma once
#include "common.cuh"

namespace dmst {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;

template <int VW>
struct Vals {
  uint32_t w[VW];
};

template <int BITS = kRadixBits, typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift) {
  return (uint32_t)(key >> shift) & ((1u << BITS) - 1u);
}

// ----------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %0;" ::"r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Global -> shared bulk copy (bytes % 16 == 0, both addresses 16-B aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// ------------------------------------------------------------- loaders
// A Loader has NS input streams; stream s holds elements of sb(s) bytes and
// item i of the sort uses element i / IPE of every stream.  It provides
//   ptr(s)                      stream base pointer
//   key(i)                      key of item i from global memory (upsweep)
//   load(i, k, v)               item i from global memory (partial tiles)
//   get(stage, li, i, k, v)     item i (local index li) from staged streams
template <typename K, int VW>
struct ArrayLoader {
  static constexpr int NS = 1 + VW, IPE = 1;
  __host__ __device__ static constexpr int sb(int s) { return s == 0 ? (int)sizeof(K) : 4; }
  const K* __restrict__ keys;
  const uint32_t* __restrict__ vals[VW];
  __device__ __forceinline__ const void* ptr(int s) const { return s == 0 ? (const void*)keys : (const void*)vals[s - 1]; }
  __device__ __forceinline__ K key(int64_t i) const { return ld_stream(keys + i); }
  __device__ __forceinline__ void load(int64_t i, K& k, Vals<VW>& v) const {
    k = ld_stream(keys + i);
#pragma unroll
    for (int q = 0; q < VW; ++q) v.w[q] = ld_stream(vals[q] + i);
  }
  __device__ __forceinline__ void get(char* const* st, int li, int64_t, K& k, Vals<VW>& v) const {
    k = reinterpret_cast<const K*>(st[0])[li];
#pragma unroll
    for (int q = 0; q < VW; ++q) v.w[q] = reinterpret_cast<const uint32_t*>(st[1 + q])[li];
  }
};

template <typename K, int VW>
struct ArrayEmitter {
  K* __restrict__ keys;
  uint32_t* __restrict__ vals[VW];
  template <int N>
  __device__ __forceinline__ void emit(const uint32_t (&dst)[N], const K (&k)[N], const Vals<VW> (&v)[N],
                                       const bool (&ok)[N]) const {
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (ok[i]) {
        keys[dst[i]] = k[i];
#pragma unroll
        for (int q = 0; q < VW; ++q) vals[q][dst[i]] = v[i].w[q];
      }
  }
};

template <class L>
__device__ __forceinline__ bool loader_tma_ok(const L& ld) {
  bool ok = true;
#pragma unroll
  for (int s = 0; s < L::NS; ++s) ok &= aligned16(ld.ptr(s));
  return ok;
}

// --------------------------------------------------------------- upsweep
struct SweepArgs {
  int64_t n;
  int64_t chunk;          // items per CTA (multiple of the downsweep sub-tile)
  int shift;              // digit bit offset
  uint32_t G;             // number of chunks (= CTAs)
  uint32_t GS;            // row stride of counts (G rounded up to a multiple of 4)
  uint32_t* counts;       // [256][GS] digit-major (upsweep out, scan in/out)
  unsigned long long* prof;  // optional: per-CTA phase time sums [G][8] (tools/sortbench)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kMaxChunks = 148 * 4;  // downsweep CTAs (chunks) per pass, upper bound
constexpr int kUpSplit = 4;  // upsweep CTAs per chunk (counts accumulate atomically)

template <int BITS, class Loader>
__global__ void __launch_bounds__(256) k_upsweep(SweepArgs a, Loader ld) {
  constexpr int R = 1 << BITS, BPT = R / 256;
  __shared__ uint32_t h[8][R];  // per-warp histograms
  const uint32_t warp = threadIdx.x >> 5;
#pragma unroll
  for (int w = 0; w < 8; ++w)
#pragma unroll
    for (int q = 0; q < BPT; ++q) h[w][q * 256 + threadIdx.x] = 0;
  __syncthreads();
  const uint32_t chunk_id = blockIdx.x / kUpSplit, part = blockIdx.x % kUpSplit;
  const int64_t cbeg = (int64_t)chunk_id * a.chunk;
  const int64_t plen = (a.chunk / kUpSplit + 1023) & ~int64_t(1023);
  const int64_t begin = cbeg + part * plen;
  const int64_t end = min(min(a.n, cbeg + a.chunk), begin + plen);
  constexpr int U = 8;
  for (int64_t i0 = begin; i0 < end; i0 += 256 * U) {
    uint32_t d[U];
    bool ok[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int64_t i = i0 + q * 256 + threadIdx.x;
      ok[q] = i < end;
      d[q] = ok[q] ? digit_of<BITS>(ld.key(i), a.shift) : 0u;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const uint32_t act = __ballot_sync(kFull, ok[q]);
      const uint32_t d0 = __shfl_sync(kFull, d[q], 0);
      if (__all_sync(kFull, !ok[q] || d[q] == d0)) {
        if (lane_id() == 0 && act) atomicAdd(&h[warp][d0], __popc(act));
      } else if (ok[q]) {
        atomicAdd(&h[warp][d[q]], 1u);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    const uint32_t b = q * 256 + threadIdx.x;
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) c += h[w][b];
    if (c) atomicAdd(a.counts + (uint64_t)b * a.GS + chunk_id, c);
  }
}

// Exclusive scan of counts[R][GS] in place, digit-major => the global
// output offset of every (digit, chunk).  Thread t owns rows t*BPT.. (vector loads).
template <int BITS>
__global__ void __launch_bounds__(256) k_chunk_scan(uint32_t* counts, uint32_t GS) {
  constexpr int BPT = (1 << BITS) / 256;
  __shared__ uint32_t scratch[256 / 32 + 1];
  const uint32_t nq = GS / 4;
  uint32_t s = 0;
#pragma unroll
  for (int r = 0; r < BPT; ++r) {
    const uint4* row = reinterpret_cast<const uint4*>(counts + (uint64_t)(threadIdx.x * BPT + r) * GS);
#pragma unroll 8
    for (uint32_t q = 0; q < nq; ++q) {
      const uint4 v = row[q];
      s += v.x + v.y + v.z + v.w;
    }
  }
  uint32_t tot;
  uint32_t run = block_excl_sum<256>(s, scratch, &tot);
#pragma unroll
  for (int r = 0; r < BPT; ++r) {
    uint4* row = reinterpret_cast<uint4*>(counts + (uint64_t)(threadIdx.x * BPT + r) * GS);
#pragma unroll 8
    for (uint32_t q = 0; q < nq; ++q) {
      const uint4 v = row[q];
      uint4 o;
      o.x = run;
      o.y = o.x + v.x;
      o.z = o.y + v.y;
      o.w = o.z + v.z;
      run = o.w + v.w;
      row[q] = o;
    }
  }
}

// ------------------------------------------------------------- downsweep
template <typename K, int VW, int BLOCK, int ITEMS, class Loader, int BITS = kRadixBits>
struct DownSmem {
  static constexpr int R = 1 << BITS;
  static constexpr int T = BLOCK * ITEMS;
  static constexpr int NW = BLOCK / 32;
  static constexpr int NS = Loader::NS;
  __host__ __device__ static constexpr size_t stream_bytes(int s) {
    return ((size_t)T / Loader::IPE * Loader::sb(s) + 127) & ~size_t(127);
  }
  __host__ __device__ static constexpr size_t stream_off(int s) {
    size_t b = 0;
    for (int q = 0; q < s; ++q) b += stream_bytes(q);
    return b;
  }
  // sorted sub-tile (keys, then VW value rows) is scattered in place into the
  // stage buffer it was read from, so a buffer holds max(staged, sorted).
  __host__ __device__ static constexpr size_t keys_bytes() { return ((size_t)T * sizeof(K) + 127) & ~size_t(127); }
  __host__ __device__ static constexpr size_t stage_bytes() {
    const size_t staged = stream_off(NS);
    const size_t sorted = keys_bytes() + (size_t)VW * T * 4;
    return staged > sorted ? staged : sorted;
  }
  __host__ __device__ static constexpr size_t off_stage(int st) { return st * stage_bytes(); }
  __host__ __device__ static constexpr size_t off_misc() { return 2 * stage_bytes(); }
  struct Misc {
    uint32_t whist[NW][R];
    uint32_t run[R];     // running global offset per digit
    uint32_t lstart[R];
    uint32_t gofs[R];
    uint32_t scan[NW + 1];
    uint64_t bar[2];
  };
  __host__ __device__ static constexpr size_t bytes() { return off_misc() + sizeof(Misc); }
};

// Stable rank of item i within its warp's items of equal digit.  Peers by
// __match_any_sync (DMST_RANK_BALLOT selects 8 ballots instead); all peers
// read the warp counter (broadcast), the lowest peer advances it.
template <bool FULL>
__device__ __forceinline__ uint32_t warp_rank(uint32_t* whist, uint32_t d, bool valid, uint32_t lane,
                                              uint32_t lt) {
#ifdef DMST_RANK_BALLOT
  uint32_t peers = FULL ? kFull : (valid ? __ballot_sync(kFull, valid) : ~__ballot_sync(kFull, valid));
#pragma unroll
  for (int b = 0; b < kRadixBits; ++b) {
    const uint32_t bit = (d >> b) & 1u;
    peers &= __ballot_sync(kFull, bit) ^ (bit - 1u);
  }
#else
  const uint32_t peers = __match_any_sync(kFull, FULL ? d : (valid ? d : 0xffffu));
#endif
  uint32_t old = 0;
  if (FULL || valid) old = whist[d];
  const uint32_t below = __popc(peers & lt);
  __syncwarp();  // order all peers' reads of the counter before the leader's write
  if ((FULL || valid) && below == 0) whist[d] = old + __popc(peers);
  __syncwarp();
  return old + below;
}

// Rank, scatter (in place, into stage buffer `buf`) and write out one sub-tile.
template <bool FULL, typename K, int VW, int BLOCK, int ITEMS, class S, class Emitter>
__device__ __forceinline__ void down_subtile(const SweepArgs& a, const Emitter& em, typename S::Misc& m,
                                             unsigned char* buf, K (&k)[ITEMS], Vals<VW> (&v)[ITEMS],
                                             int cnt_items) {
  constexpr int T = S::T, NW = S::NW, R = S::R, BPT = R / BLOCK;
  constexpr int BITS = R == 256 ? 8 : R == 512 ? 9 : 10;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t lt = lanemask_lt();
  const int lbase = warp * ITEMS * 32 + lane;
  uint32_t rk[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const bool valid = FULL || lbase + i * 32 < cnt_items;
    rk[i] = warp_rank<FULL>(m.whist[warp], digit_of<BITS>(k[i], a.shift), valid, lane, lt);
  }
  __syncthreads();  // (also: every thread has finished reading `buf`)

  // thread t owns digits t*BPT .. t*BPT+BPT-1 (consecutive, for the block scan)
  uint32_t cb[BPT], csum = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    const uint32_t b = tid * BPT + q;
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t x = m.whist[w][b];
      m.whist[w][b] = c;
      c += x;
    }
    cb[q] = c;
    csum += c;
  }
  uint32_t total;
  uint32_t lstart = block_excl_sum<BLOCK>(csum, m.scan, &total);
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    const uint32_t b = tid * BPT + q;
    m.lstart[b] = lstart;
    m.gofs[b] = m.run[b] - lstart;
    m.run[b] += cb[q];
    lstart += cb[q];
  }
  __syncthreads();

  K* skeys = reinterpret_cast<K*>(buf);
  uint32_t* svals = reinterpret_cast<uint32_t*>(buf + S::keys_bytes());
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (FULL || lbase + i * 32 < cnt_items) {
      const uint32_t d = digit_of<BITS>(k[i], a.shift);
      const uint32_t pos = m.lstart[d] + m.whist[warp][d] + rk[i];
      skeys[pos] = k[i];
#pragma unroll
      for (int q = 0; q < VW; ++q) svals[q * T + pos] = v[i].w[q];
    }
  }
  __syncthreads();

  uint32_t dst[ITEMS];
  bool ok[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int sidx = i * BLOCK + tid;
    ok[i] = FULL || sidx < cnt_items;
    if (ok[i]) {
      k[i] = skeys[sidx];
#pragma unroll
      for (int q = 0; q < VW; ++q) v[i].w[q] = svals[q * T + sidx];
      dst[i] = m.gofs[digit_of<BITS>(k[i], a.shift)] + sidx;
    }
  }
#pragma unroll
  for (int w = 0; w < NW; ++w)
#pragma unroll
    for (int q = 0; q < BPT; ++q) m.whist[w][tid * BPT + q] = 0;
  em.template emit<ITEMS>(dst, k, v, ok);
  __syncthreads();
}

template <typename K, int VW, int BLOCK, int ITEMS, int MINB, class Loader, class Emitter, int BITS = kRadixBits>
__global__ void __launch_bounds__(BLOCK, MINB)
k_downsweep(SweepArgs a, Loader ld, Emitter em) {
  static_assert(BLOCK == 256 && (1 << BITS) % BLOCK == 0, "digit bins are owned by threads");
  using S = DownSmem<K, VW, BLOCK, ITEMS, Loader, BITS>;
  constexpr int T = S::T, NW = S::NW, NS = S::NS, BPT = S::R / BLOCK;
  extern __shared__ __align__(128) unsigned char smem[];
  typename S::Misc& m = *reinterpret_cast<typename S::Misc*>(smem + S::off_misc());

  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t begin = (int64_t)blockIdx.x * a.chunk;
  const int64_t end = min(a.n, begin + a.chunk);
  if (begin >= end) return;
  const int nsub = (int)((end - begin + T - 1) / T);
  const bool tma = loader_tma_ok(ld);

#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    const uint32_t b = tid * BPT + q;
    m.run[b] = a.counts[(uint64_t)b * a.GS + blockIdx.x];
#pragma unroll
    for (int w = 0; w < NW; ++w) m.whist[w][b] = 0;
  }
  if (tid == 0) {
    mbar_init(&m.bar[0], 1);
    mbar_init(&m.bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();

  // issue the bulk copies of sub-tile `sub` into stage buffer sub & 1
  auto issue = [&](int sub) {
    const int64_t i0 = begin + (int64_t)sub * T;
    if (!tma || i0 + T > end) return;  // partial / unaligned: direct loads later
    fence_proxy_async();
    uint32_t bytes = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) bytes += (uint32_t)(T / Loader::IPE * Loader::sb(s));
    uint64_t* bar = &m.bar[sub & 1];
    mbar_expect_tx(bar, bytes);
#pragma unroll
    for (int s = 0; s < NS; ++s)
      bulk_g2s(smem + S::off_stage(sub & 1) + S::stream_off(s),
               (const char*)ld.ptr(s) + (i0 / Loader::IPE) * Loader::sb(s),
               (uint32_t)(T / Loader::IPE * Loader::sb(s)), bar);
  };
  if (tid == 0) issue(0);

  for (int sub = 0; sub < nsub; ++sub) {
    if (tid == 0 && sub + 1 < nsub) issue(sub + 1);
    const int64_t i0 = begin + (int64_t)sub * T;
    const int64_t rem_items = end - i0;
    const int cnt_items = rem_items < T ? (int)rem_items : T;
    unsigned char* buf = smem + S::off_stage(sub & 1);
    K k[ITEMS];
    Vals<VW> v[ITEMS];
    const int lbase = warp * ITEMS * 32 + lane;
    if (tma && cnt_items == T) {
      mbar_wait(&m.bar[sub & 1], (uint32_t)(sub >> 1) & 1u);
      char* st[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) st[s] = (char*)buf + S::stream_off(s);
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int li = lbase + i * 32;
        ld.get(st, li, i0 + li, k[i], v[i]);
      }
      down_subtile<true, K, VW, BLOCK, ITEMS, S>(a, em, m, buf, k, v, T);
    } else {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int li = lbase + i * 32;
        if (li < cnt_items) ld.load(i0 + li, k[i], v[i]);
      }
      if (cnt_items == T)
        down_subtile<true, K, VW, BLOCK, ITEMS, S>(a, em, m, buf, k, v, T);
      else
        down_subtile<false, K, VW, BLOCK, ITEMS, S>(a, em, m, buf, k, v, cnt_items);
    }
  }
}

// Every digit was constant: the stable order is the identity.
template <typename K, int VW, class Loader, class Emitter>
__global__ void k_identity_pass(int64_t n, Loader ld, Emitter em) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t dst[1];
  K k[1];
  Vals<VW> v[1];
  bool ok[1];
  ok[0] = i < n;
  if (ok[0]) {
    ld.load(i, k[0], v[0]);
    dst[0] = (uint32_t)i;
  }
  em.template emit<1>(dst, k, v, ok);
}

// Exclusive scan of per-digit global histograms: hist[p][256] -> gbase[p][256].
__global__ void k_digit_scan(const uint32_t* __restrict__ hist, uint32_t* __restrict__ gbase, int passes) {
  __shared__ uint32_t scratch[kRadix / 32 + 1];
  for (int p = 0; p < passes; ++p) {
    uint32_t total;
    uint32_t x = hist[p * kRadix + threadIdx.x];
    gbase[p * kRadix + threadIdx.x] = block_excl_sum<kRadix>(x, scratch, &total);
  }
}

}  // namespace dmst

// Stable LSD radix sort passes, reduce-then-scan, with TMA-staged input.
//
// One digit (8 or 9 bits) per pass, three kernels:
//   k_upsweep    each CTA counts the digits of its contiguous chunk of the
//                input (keys only) -> counts[digit][chunk]; for the edge
//                sort's first pass it also reduces all keys (KEYRED);
//   k_row_scan + k_row_total_scan: exclusive scan of counts in digit-major
//                order -> the global output offset of every (digit, chunk),
//                and the pass's warp-ranking method (match_any or ballots);
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
// final outputs.  Between passes an item is a key array plus an AoS
// payload array (PW 32-bit words per item; PW = 0: key only), so a digit
// run is at most two contiguous runs in memory.
//
// Replaces `np.argsort(-w, kind="stable")` (tree_core.py:180) and
// `np.lexsort` (expansion.py:135) of /root/reference/pkg/src/dendromst/.
#pragma once
#include "common.cuh"

namespace dmst {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;

template <int VW>
struct Vals {
  uint32_t w[VW];
};
template <>
struct Vals<0> {  // key-only items
  uint32_t w[1];
};

// Order-preserving map of (w + 0.0) to uint64, inverted so that ascending
// key order is descending weight; -0.0 is canonicalised to +0.0 so the two
// tie, as numpy's comparison does (tree_core.py:180).
__device__ __forceinline__ uint64_t desc_key_of(double w) {
  uint64_t b = (uint64_t)__double_as_longlong(w);
  if (b == 0x8000000000000000ull) b = 0;
  uint64_t asc = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  return ~asc;
}

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
// A Loader has NS input streams; stream s holds sb(s) bytes per item.  It
// provides
//   ptr(s)                      stream base pointer
//   key(i)                      key of item i from global memory (upsweep)
//   load(i, k, v)               item i from global memory (partial tiles)
//   get(stage, li, i, k, v)     item i (local index li) from staged streams
//
// Between passes an item is a key array (K) plus an AoS payload array of PW
// 32-bit words per item: a digit run of m items is then one contiguous run
// of m * 4 * PW payload bytes instead of PW runs of 4 m bytes, which keeps
// the scattered writes of uniformly distributed digits sector-efficient.
template <typename K, int PW>
struct ArrayLoader {
  static constexpr int NS = PW > 0 ? 2 : 1;
  __host__ __device__ static constexpr int sb(int s) { return s == 0 ? (int)sizeof(K) : 4 * PW; }
  const K* __restrict__ keys;
  const uint32_t* __restrict__ pay;
  // the upsweep may read the keys as 16-B vectors (raw key = sort key)
  using RawKey = K;
  static constexpr bool VEC = true;
  __device__ __forceinline__ const K* raw_keys() const { return keys; }
  __device__ __forceinline__ K key_of_raw(K r, int64_t) const { return r; }
  __device__ __forceinline__ const void* ptr(int s) const { return s == 0 ? (const void*)keys : (const void*)pay; }
  __device__ __forceinline__ K key(int64_t i) const { return ld_stream(keys + i); }
  __device__ __forceinline__ void load(int64_t i, K& k, Vals<PW>& v) const {
    k = ld_stream(keys + i);
#pragma unroll
    for (int q = 0; q < PW; ++q) v.w[q] = ld_stream(pay + i * PW + q);
  }
  __device__ __forceinline__ void get(char* const* st, int li, int64_t, K& k, Vals<PW>& v) const {
    k = reinterpret_cast<const K*>(st[0])[li];
    if constexpr (PW > 0) {
      const uint32_t* p = reinterpret_cast<const uint32_t*>(st[1]) + li * PW;
      if constexpr (PW == 2) {
        const uint2 x = *reinterpret_cast<const uint2*>(p);
        v.w[0] = x.x;
        v.w[1] = x.y;
      } else {
#pragma unroll
        for (int q = 0; q < PW; ++q) v.w[q] = p[q];
      }
    }
  }
};

// A sorted sub-tile in shared memory: item s (0 <= s < cnt) has key
// skeys[s], payload words spay[s * PW ..], and goes to global index
// gofs[digit] + s; digit d's run is [lstart[d], lstart[d + 1]).  Emitters
// write it out with coalesced per-digit runs.
template <typename K, int PW, int BITS>
struct TileView {
  const K* skeys;
  const uint32_t* spay;
  const uint32_t* gofs;
  const uint32_t* lstart;  // [R + 1]
  int cnt;
  int shift;
  __device__ __forceinline__ uint32_t digit(int s) const { return digit_of<BITS>(skeys[s], shift); }
  __device__ __forceinline__ uint32_t dst(int s) const { return gofs[digit(s)] + (uint32_t)s; }
};

// Emitters may keep per-CTA state across the sub-tiles of a pass (State,
// in shared memory): init() before the first sub-tile, finish() after the last.
struct NoEmitState {};

template <typename K, int PW>
struct ArrayEmitter {
  using State = NoEmitState;
  K* __restrict__ keys;
  uint32_t* __restrict__ pay;
  template <int BLOCK, int R>
  __device__ __forceinline__ void init(State&) const {}
  template <int BLOCK, int R>
  __device__ __forceinline__ void finish(State&) const {}
  template <int BLOCK, class Tile>
  __device__ __forceinline__ void emit(const Tile& t, State&) const {
    for (int s = threadIdx.x; s < t.cnt; s += BLOCK) {
      const uint32_t d = t.dst(s);
      keys[d] = t.skeys[s];
      if constexpr (PW == 1) pay[d] = t.spay[s];
    }
    if constexpr (PW > 1) {
      // payload as one word stream: word s of the sorted tile goes to
      // global word gofs[digit] * PW + s (consecutive threads -> consecutive words)
      for (int s = threadIdx.x; s < t.cnt * PW; s += BLOCK) {
        const int it = s / PW;
        pay[(uint64_t)t.gofs[t.digit(it)] * PW + s] = t.spay[s];
      }
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
};

constexpr int kMaxChunks = 148 * 4;  // downsweep CTAs (chunks) per pass, upper bound
constexpr int kUpSplit = 4;  // upsweep CTAs per chunk (counts accumulate atomically)

// KEYRED (edge sort, first pass): the same read of w also produces the
// AND / OR of all keys (digit skipping) and the "-0.0 present" flag, so the
// edge sort has no separate reduction pass; the digit counted was predicted
// from a sample of the keys (k_key_sample) and is re-checked on the host.
struct KeyRed {
  const double* w;
  unsigned long long* and_or;
  uint32_t* negzero;
  uint32_t* top_bits;  // presence bitmap of the top fields (key >> 52), 4096 bits
  // the sample (k_key_sample): AND / OR of its keys and its smallest top field
  // (the base of the in-register 32-field window); the digit this upsweep
  // counts is predicted from it on the device (no host round trip) and
  // written to d0_out for the host
  const unsigned long long* sample_ao;
  const uint32_t* sample_tmin;
  uint32_t* d0_out;
  int allow_local;  // 0: never predict the shared-memory finish (sort1_mode bit 2)
};

// The first pass's digit, predicted from the sample's varying bits: >= 5
// active 8-bit digits predicts the wide-key shared-memory finish
// (local_sort.cuh), whose first global digit is the lowest of the 24 highest
// varying bits, one bit above the sample's top varying bit (the full data
// often varies one bit higher); otherwise the lowest active digit.
__host__ __device__ inline int predict_first_digit(unsigned long long sand, unsigned long long sor, int allow_local) {
  const unsigned long long var = sand ^ sor;
  int nd = 0, lo = -1;
  for (int sft = 0; sft < 64; sft += 8)
    if ((var >> sft) & 0xffull) {
      ++nd;
      if (lo < 0) lo = sft;
    }
  if (nd == 0) return 0;
  if (nd >= 5 && allow_local) {
    int hb = 63;
    while (!((var >> hb) & 1ull)) --hb;
    return hb + 1 - 23 > 0 ? hb + 1 - 23 : 0;
  }
  return lo;
}

template <class L, class = void>
struct HasVec {
  static constexpr bool value = false;
};
template <class L>
struct HasVec<L, decltype(void(L::VEC))> {
  static constexpr bool value = L::VEC;
};
template <class L>
__host__ __device__ constexpr bool loader_vec() { return HasVec<L>::value; }
template <class L, bool = HasVec<L>::value>
struct LoaderRawKey {
  using type = uint32_t;  // unused
};
template <class L>
struct LoaderRawKey<L, true> {
  using type = typename L::RawKey;
};

template <int BITS, class Loader, bool KEYRED = false>
__global__ void __launch_bounds__(256) k_upsweep(SweepArgs a, Loader ld, KeyRed kr = KeyRed{}) {
  constexpr int R = 1 << BITS, BPT = R / 256;
  __shared__ uint32_t h[8][R];  // per-warp histograms
  __shared__ uint32_t tbits[KEYRED ? 128 : 1];
  const uint32_t warp = threadIdx.x >> 5;
#pragma unroll
  for (int w = 0; w < 8; ++w)
#pragma unroll
    for (int q = 0; q < BPT; ++q) h[w][q * 256 + threadIdx.x] = 0;
  if constexpr (KEYRED) {
    if (threadIdx.x < 128) tbits[threadIdx.x] = 0;
  }
  __syncthreads();
  int shift = a.shift;
  uint32_t top_base = 0;
  if constexpr (KEYRED) {
    shift = predict_first_digit(kr.sample_ao[0], kr.sample_ao[1], kr.allow_local);
    top_base = min(*kr.sample_tmin, 4095u);
    if (blockIdx.x == 0 && threadIdx.x == 0) *kr.d0_out = (uint32_t)shift;
  }
  const uint32_t chunk_id = blockIdx.x / kUpSplit, part = blockIdx.x % kUpSplit;
  const int64_t cbeg = (int64_t)chunk_id * a.chunk;
  const int64_t plen = (a.chunk / kUpSplit + 1023) & ~int64_t(1023);
  const int64_t begin = cbeg + part * plen;
  const int64_t end = min(min(a.n, cbeg + a.chunk), begin + plen);
  if constexpr (!KEYRED && loader_vec<Loader>()) {
    if (aligned16(ld.raw_keys())) {  // uniform across the grid
    // keys as 16-B vectors: 2-4 keys per load, 4 loads in flight per thread
    using RK = typename LoaderRawKey<Loader>::type;
    constexpr int PER = 16 / (int)sizeof(RK), UV = 4;
    const RK* kp = ld.raw_keys();
    const int64_t vend = begin + ((end - begin) / PER) * PER;
    // (the loop bound is uniform across the warp: the ballots below need every lane)
    for (int64_t i0 = begin; i0 < vend; i0 += (int64_t)256 * PER * UV) {
      uint4 xv[UV];
#pragma unroll
      for (int q = 0; q < UV; ++q) {
        const int64_t i = i0 + ((int64_t)q * 256 + threadIdx.x) * PER;
        xv[q] = i < vend ? ld_stream(reinterpret_cast<const uint4*>(kp + i)) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int q = 0; q < UV; ++q) {
        const int64_t i = i0 + ((int64_t)q * 256 + threadIdx.x) * PER;
        const bool ok = i < vend;
        const RK* e = reinterpret_cast<const RK*>(&xv[q]);
#pragma unroll
        for (int t = 0; t < PER; ++t) {
          const uint32_t dd = ok ? digit_of<BITS>(ld.key_of_raw(e[t], i + t), a.shift) : 0u;
          const uint32_t act = __ballot_sync(kFull, ok);
          const uint32_t d0 = __shfl_sync(kFull, dd, 0);
          if (__all_sync(kFull, !ok || dd == d0)) {  // one digit across the warp (skewed keys)
            if (lane_id() == 0 && act) atomicAdd(&h[warp][d0], __popc(act));
          } else if (ok) {
            atomicAdd(&h[warp][dd], 1u);
          }
        }
      }
    }
    for (int64_t i = vend + threadIdx.x; i < end; i += 256) atomicAdd(&h[warp][digit_of<BITS>(ld.key(i), a.shift)], 1u);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      const uint32_t b = q * 256 + threadIdx.x;
      uint32_t c = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) c += h[w][b];
      if (c) atomicAdd(a.counts + (uint64_t)b * a.GS + chunk_id, c);
    }
    return;
    }
  }
  constexpr int U = KEYRED ? 16 : 8;  // the fused pass over w is load-latency-bound at 8
  uint64_t ka = ~0ull, ko = 0ull;
  uint32_t tw = 0;
  bool nz = false;
  for (int64_t i0 = begin; i0 < end; i0 += 256 * U) {
    uint32_t d[U];
    bool ok[U];
    double x[U];
    if constexpr (KEYRED) {
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int64_t i = i0 + q * 256 + threadIdx.x;
        x[q] = i < end ? ld_stream(kr.w + i) : kr.w[begin];
      }
    }
    uint32_t far = 0, tq[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int64_t i = i0 + q * 256 + threadIdx.x;
      ok[q] = i < end;
      if constexpr (KEYRED) {
        const uint64_t k = desc_key_of(x[q]);
        nz |= (uint64_t)__double_as_longlong(x[q]) == 0x8000000000000000ull;
        ka &= k;
        ko |= k;
        tq[q] = (uint32_t)(k >> 52);
        const uint32_t dt = tq[q] - top_base;
        tw |= dt < 32 ? 1u << dt : 0u;
        far |= dt < 32 ? 0u : 1u << q;
        d[q] = digit_of<BITS>(k, shift);
      } else {
        d[q] = ok[q] ? digit_of<BITS>(ld.key(i), shift) : 0u;
      }
    }
    if constexpr (KEYRED) {
      if (far) {  // top fields outside the window (rare): straight to the bitmap
#pragma unroll
        for (int q = 0; q < U; ++q)
          if ((far >> q) & 1u) atomicOr(&tbits[tq[q] >> 5], 1u << (tq[q] & 31));
      }
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
  if constexpr (KEYRED) {
    const uint32_t alo = __reduce_and_sync(kFull, (uint32_t)ka), ahi = __reduce_and_sync(kFull, (uint32_t)(ka >> 32));
    const uint32_t olo = __reduce_or_sync(kFull, (uint32_t)ko), ohi = __reduce_or_sync(kFull, (uint32_t)(ko >> 32));
    const bool anz = __any_sync(kFull, nz);
    if (lane_id() == 0 && begin < end) {
      atomicAnd(kr.and_or, ((unsigned long long)ahi << 32) | alo);
      atomicOr(kr.and_or + 1, ((unsigned long long)ohi << 32) | olo);
      if (anz) atomicOr(kr.negzero, 1u);
    }
    tw = __reduce_or_sync(kFull, tw);
    if (lane_id() == 0 && tw) {  // window bits base.. base+31 -> two aligned words
      const uint32_t wb = top_base >> 5, sh = top_base & 31;
      atomicOr(&tbits[wb], tw << sh);
      if (sh && wb + 1 < 128) atomicOr(&tbits[wb + 1], tw >> (32 - sh));
    }
  }
  __syncthreads();
  if constexpr (KEYRED) {
    if (threadIdx.x < 128 && tbits[threadIdx.x]) atomicOr(kr.top_bits + threadIdx.x, tbits[threadIdx.x]);
  }
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    const uint32_t b = q * 256 + threadIdx.x;
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) c += h[w][b];
    if (c) atomicAdd(a.counts + (uint64_t)b * a.GS + chunk_id, c);
  }
}

// Exclusive scan of counts[R][GS] digit-major => the global output offset of
// every (digit, chunk), in two small kernels instead of one serial CTA:
//   k_row_scan        one warp per digit row: the row becomes its exclusive
//                     in-row offsets, the row total goes to rowsum[r];
//   k_row_total_scan  one CTA: exclusive scan of the R row totals -> rowstart
//                     (the downsweep adds rowstart[d] to its row entry), and
//                     the pass's warp-ranking method: with digit frequencies
//                     p_d, a warp of 32 items holds E = sum_d 1 - (1 - p_d)^32
//                     distinct digits on average; __match_any_sync is cheaper
//                     below ~kBallotE, ballots above (ballot word = 1).
// Layout behind the R * GS counts: [ballot word, pad x3, rowsum[R], rowstart[R]].
constexpr float kBallotE = 12.0f;
constexpr int kRowScanWarps = 8;
__host__ __device__ constexpr uint64_t scan_ballot_off(int R, uint32_t GS) { return (uint64_t)R * GS; }
__host__ __device__ constexpr uint64_t scan_rowsum_off(int R, uint32_t GS) { return (uint64_t)R * GS + 4; }
__host__ __device__ constexpr uint64_t scan_rowstart_off(int R, uint32_t GS) { return (uint64_t)R * GS + 4 + R; }

template <int BITS>
__global__ void __launch_bounds__(32 * kRowScanWarps) k_row_scan(uint32_t* counts, uint32_t GS) {
  constexpr int R = 1 << BITS;
  const uint32_t lane = threadIdx.x & 31;
  const int r = blockIdx.x * kRowScanWarps + (threadIdx.x >> 5);
  if (r >= R) return;
  uint32_t* row = counts + (uint64_t)r * GS;
  uint32_t base = 0;
  for (uint32_t q0 = 0; q0 < GS; q0 += 64) {  // two loads in flight per lane
    const uint32_t qa = q0 + lane, qb = q0 + 32 + lane;
    const uint32_t xa = qa < GS ? row[qa] : 0u, xb = qb < GS ? row[qb] : 0u;
    const uint32_t ia = warp_incl_sum(xa), ib = warp_incl_sum(xb);
    const uint32_t ta = __shfl_sync(kFull, ia, 31);
    if (qa < GS) row[qa] = base + ia - xa;
    if (qb < GS) row[qb] = base + ta + ib - xb;
    base += ta + __shfl_sync(kFull, ib, 31);
  }
  if (lane == 0) counts[scan_rowsum_off(R, GS) + r] = base;
}

template <int BITS>
__global__ void __launch_bounds__(1 << BITS) k_row_total_scan(uint32_t* counts, uint32_t GS) {
  constexpr int R = 1 << BITS;
  __shared__ uint32_t scratch[R / 32 + 1];
  __shared__ float fscr[R / 32];
  const uint32_t r = threadIdx.x;
  const uint32_t v = counts[scan_rowsum_off(R, GS) + r];
  uint32_t tot;
  const uint32_t start = block_excl_sum<R>(v, scratch, &tot);
  counts[scan_rowstart_off(R, GS) + r] = start;
  float e = 1.f - __powf(1.f - (float)v / (float)max(tot, 1u), 32.f);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(kFull, e, o);
  if (lane_id() == 0) fscr[r >> 5] = e;
  __syncthreads();
  if (r == 0) {
    float E = 0.f;
    for (int w = 0; w < R / 32; ++w) E += fscr[w];
    counts[scan_ballot_off(R, GS)] = E > kBallotE ? 1u : 0u;
  }
}

// ------------------------------------------------------------- downsweep
template <typename K, int PW, int BLOCK, int ITEMS, class Loader, class Emitter, int BITS = kRadixBits>
struct DownSmem {
  static constexpr int R = 1 << BITS;
  static constexpr int T = BLOCK * ITEMS;
  static constexpr int NW = BLOCK / 32;
  static constexpr int NS = Loader::NS;
  __host__ __device__ static constexpr size_t stream_bytes(int s) {
    return ((size_t)T * Loader::sb(s) + 127) & ~size_t(127);
  }
  __host__ __device__ static constexpr size_t stream_off(int s) {
    size_t b = 0;
    for (int q = 0; q < s; ++q) b += stream_bytes(q);
    return b;
  }
  // sorted sub-tile (keys, then the AoS payload) is scattered in place into
  // the stage buffer it was read from, so a buffer holds max(staged, sorted).
  __host__ __device__ static constexpr size_t keys_bytes() { return ((size_t)T * sizeof(K) + 127) & ~size_t(127); }
  __host__ __device__ static constexpr size_t stage_bytes() {
    const size_t staged = stream_off(NS);
    const size_t sorted = keys_bytes() + (size_t)PW * T * 4;
    return staged > sorted ? staged : sorted;
  }
  __host__ __device__ static constexpr size_t off_stage(int st) { return st * stage_bytes(); }
  __host__ __device__ static constexpr size_t off_misc() { return 2 * stage_bytes(); }
  struct Misc {
    uint32_t whist[NW][R];
    uint32_t run[R];     // running global offset per digit
    uint32_t lstart[R + 1];
    uint32_t gofs[R];
    typename Emitter::State est;
    uint32_t scan[NW + 1];
    uint32_t ballot;     // ranking method of this pass
    uint64_t bar[2];
  };
  __host__ __device__ static constexpr size_t bytes() { return off_misc() + sizeof(Misc); }
};

// Stable rank of item i within its warp's items of equal digit.  Peers come
// from __match_any_sync (cost grows with the number of distinct digits in
// the warp) or from BITS ballots (constant cost); `ballot` is chosen per
// pass from the digit distribution (k_row_total_scan).  All peers read the warp
// counter (broadcast), the lowest peer advances it.
template <bool FULL, int BITS>
__device__ __forceinline__ uint32_t warp_rank(uint32_t* whist, uint32_t d, bool valid, uint32_t lane,
                                              uint32_t lt, bool ballot) {
  uint32_t peers;
  if (ballot) {
    peers = FULL ? kFull : (valid ? __ballot_sync(kFull, valid) : ~__ballot_sync(kFull, valid));
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
      // s = bit b of d sign-extended (all ones / zero): peers keep the lanes
      // whose bit b equals ours, ~(ballot ^ s), one LOP3 per bit
      int32_t sb;
      asm("bfe.s32 %0, %1, %2, 1;" : "=r"(sb) : "r"(d), "r"(b));
      const uint32_t m = __ballot_sync(kFull, sb != 0);
      peers &= ~(m ^ (uint32_t)sb);
    }
  } else {
    peers = __match_any_sync(kFull, FULL ? d : (valid ? d : 0xffffu));
  }
  uint32_t old = 0;
  if (FULL || valid) old = whist[d];
  const uint32_t below = __popc(peers & lt);
  __syncwarp();  // order all peers' reads of the counter before the leader's write
  if ((FULL || valid) && below == 0) whist[d] = old + __popc(peers);
  __syncwarp();
  return old + below;
}

// Rank, scatter (in place, into stage buffer `buf`) and write out one sub-tile.
template <bool FULL, typename K, int PW, int BLOCK, int ITEMS, int BITS, class S, class Emitter>
__device__ __forceinline__ void down_subtile(const SweepArgs& a, const Emitter& em, typename S::Misc& m,
                                             unsigned char* buf, K (&k)[ITEMS], Vals<PW> (&v)[ITEMS],
                                             int cnt_items) {
  constexpr int T = S::T, NW = S::NW, R = S::R;
  constexpr int BPT = R >= BLOCK ? R / BLOCK : 1;  // digits owned per thread
  constexpr int OWNERS = R / BPT;                  // threads owning digits
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t lt = lanemask_lt();
  const int lbase = warp * ITEMS * 32 + lane;
  uint32_t rk[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const bool valid = FULL || lbase + i * 32 < cnt_items;
    rk[i] = warp_rank<FULL, BITS>(m.whist[warp], digit_of<BITS>(k[i], a.shift), valid, lane, lt, m.ballot);
  }
  __syncthreads();  // (also: every thread has finished reading `buf`)

  // thread t < OWNERS owns digits t*BPT .. t*BPT+BPT-1 (consecutive, for the block scan)
  const bool owner = (int)tid < OWNERS;
  uint32_t cb[BPT], csum = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    cb[q] = 0;
    if (owner) {
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
  }
  uint32_t total;
  uint32_t lstart = block_excl_sum<BLOCK>(csum, m.scan, &total);
  if (owner) {
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      const uint32_t b = tid * BPT + q;
      m.lstart[b] = lstart;
      m.gofs[b] = m.run[b] - lstart;
      m.run[b] += cb[q];
      lstart += cb[q];
    }
  }
  if (tid == 0) m.lstart[R] = FULL ? T : cnt_items;
  __syncthreads();

  K* skeys = reinterpret_cast<K*>(buf);
  uint32_t* spay = reinterpret_cast<uint32_t*>(buf + S::keys_bytes());
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (FULL || lbase + i * 32 < cnt_items) {
      const uint32_t d = digit_of<BITS>(k[i], a.shift);
      const uint32_t pos = m.lstart[d] + m.whist[warp][d] + rk[i];
      skeys[pos] = k[i];
      if constexpr (PW == 2) {
        *reinterpret_cast<uint2*>(spay + pos * 2) = make_uint2(v[i].w[0], v[i].w[1]);
      } else {
#pragma unroll
        for (int q = 0; q < PW; ++q) spay[pos * PW + q] = v[i].w[q];
      }
    }
  }
  __syncthreads();
  if (owner) {
#pragma unroll
    for (int w = 0; w < NW; ++w)
#pragma unroll
      for (int q = 0; q < BPT; ++q) m.whist[w][tid * BPT + q] = 0;
  }
  TileView<K, PW, BITS> t{skeys, spay, m.gofs, m.lstart, FULL ? T : cnt_items, a.shift};
  em.template emit<BLOCK>(t, m.est);
  __syncthreads();
}

template <typename K, int PW, int BLOCK, int ITEMS, int MINB, class Loader, class Emitter, int BITS = kRadixBits>
__global__ void __launch_bounds__(BLOCK, MINB)
k_downsweep(SweepArgs a, Loader ld, Emitter em) {
  static_assert(BLOCK % 32 == 0 && ((1 << BITS) % BLOCK == 0 || BLOCK % (1 << BITS) == 0), "digit ownership");
  using S = DownSmem<K, PW, BLOCK, ITEMS, Loader, Emitter, BITS>;
  constexpr int T = S::T, NW = S::NW, NS = S::NS, R = S::R;
  extern __shared__ __align__(128) unsigned char smem[];
  typename S::Misc& m = *reinterpret_cast<typename S::Misc*>(smem + S::off_misc());

  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t begin = (int64_t)blockIdx.x * a.chunk;
  const int64_t end = min(a.n, begin + a.chunk);
  if (begin >= end) return;
  const int nsub = (int)((end - begin + T - 1) / T);
  const bool tma = loader_tma_ok(ld);

  for (int b = tid; b < R; b += BLOCK) {
    m.run[b] = a.counts[(uint64_t)b * a.GS + blockIdx.x] + a.counts[scan_rowstart_off(R, a.GS) + b];
#pragma unroll
    for (int w = 0; w < NW; ++w) m.whist[w][b] = 0;
  }
  if (tid == 0) {
    mbar_init(&m.bar[0], 1);
    mbar_init(&m.bar[1], 1);
    mbar_fence_init();
    m.ballot = a.counts[scan_ballot_off(R, a.GS)];
  }
  em.template init<BLOCK, R>(m.est);
  __syncthreads();

  // issue the bulk copies of sub-tile `sub` into stage buffer sub & 1
  auto issue = [&](int sub) {
    const int64_t i0 = begin + (int64_t)sub * T;
    if (!tma || i0 + T > end) return;  // partial / unaligned: direct loads later
    fence_proxy_async();
    uint32_t bytes = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) bytes += (uint32_t)(T * Loader::sb(s));
    uint64_t* bar = &m.bar[sub & 1];
    mbar_expect_tx(bar, bytes);
#pragma unroll
    for (int s = 0; s < NS; ++s)
      bulk_g2s(smem + S::off_stage(sub & 1) + S::stream_off(s), (const char*)ld.ptr(s) + i0 * Loader::sb(s),
               (uint32_t)(T * Loader::sb(s)), bar);
  };
  if (tid == 0) issue(0);

  for (int sub = 0; sub < nsub; ++sub) {
    if (tid == 0 && sub + 1 < nsub) issue(sub + 1);
    const int64_t i0 = begin + (int64_t)sub * T;
    const int64_t rem_items = end - i0;
    const int cnt_items = rem_items < T ? (int)rem_items : T;
    unsigned char* buf = smem + S::off_stage(sub & 1);
    K k[ITEMS];
    Vals<PW> v[ITEMS];
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
      down_subtile<true, K, PW, BLOCK, ITEMS, BITS, S>(a, em, m, buf, k, v, T);
    } else {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int li = lbase + i * 32;
        if (li < cnt_items) ld.load(i0 + li, k[i], v[i]);
      }
      if (cnt_items == T)
        down_subtile<true, K, PW, BLOCK, ITEMS, BITS, S>(a, em, m, buf, k, v, T);
      else
        down_subtile<false, K, PW, BLOCK, ITEMS, BITS, S>(a, em, m, buf, k, v, cnt_items);
    }
  }
  __syncthreads();
  em.template finish<BLOCK, R>(m.est);
}


// Every digit was constant: the stable order is the identity.  Items go
// through a shared-memory tile with gofs = tile base, so emitters see the
// same interface as in a sort pass.
template <typename K, int PW, int BLOCK, class Loader, class Emitter>
__global__ void __launch_bounds__(BLOCK) k_identity_pass(int64_t n, Loader ld, Emitter em) {
  __shared__ K skeys[BLOCK];
  __shared__ uint32_t spay[BLOCK * (PW > 0 ? PW : 1)];
  __shared__ uint32_t gofs[kRadix];
  __shared__ uint32_t lstart[kRadix + 1];
  __shared__ typename Emitter::State est;
  const int64_t i0 = (int64_t)blockIdx.x * BLOCK;
  const int64_t i = i0 + threadIdx.x;
  const int cnt = n - i0 < BLOCK ? (int)(n - i0) : BLOCK;
  if (i < n) {
    K k;
    Vals<PW> v;
    ld.load(i, k, v);
    skeys[threadIdx.x] = k;
#pragma unroll
    for (int q = 0; q < PW; ++q) spay[threadIdx.x * PW + q] = v.w[q];
  }
  __syncthreads();
  const uint32_t d0 = digit_of<kRadixBits>(skeys[0], 0);  // every key is the same
  for (int b = threadIdx.x; b <= kRadix; b += BLOCK) {
    if (b < kRadix) gofs[b] = (uint32_t)i0;
    lstart[b] = (uint32_t)b <= d0 ? 0u : (uint32_t)cnt;  // one run, of digit d0
  }
  em.template init<BLOCK, kRadix>(est);
  __syncthreads();
  TileView<K, PW, kRadixBits> t{skeys, spay, gofs, lstart, cnt, 0};
  em.template emit<BLOCK>(t, est);
  __syncthreads();
  em.template finish<BLOCK, kRadix>(est);
}


}  // namespace dmst

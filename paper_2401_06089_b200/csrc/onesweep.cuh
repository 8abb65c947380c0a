// Stable LSD radix sort, one 8-bit digit per pass, "onesweep" style:
// a single kernel per pass ranks a tile in shared memory, obtains the
// tile's global per-digit offsets by decoupled look-back over the preceding
// tiles, and scatters through shared memory so that each digit run of a
// tile is written contiguously.  The per-pass global digit offsets come
// from one up-front histogram (computed by the producer kernel of the keys,
// so no extra read pass).  Loader/emitter functors let the first pass build
// keys on the fly (no materialised key array) and the last pass write the
// final outputs directly.
//
// This replaces the reference's `np.argsort(-w, kind="stable")`
// (/root/reference/pkg/src/dendromst/tree_core.py:180) and
// `np.lexsort((rank, anchor, terminal))` (expansion.py:135).
#pragma once
#include "common.cuh"

namespace dmst {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;

struct PassArgs {
  int64_t n;
  int shift;                 // bit offset of this pass's digit
  const uint32_t* gbase;     // [256] exclusive global start of each digit
  uint32_t* status;          // [num_tiles * 256] look-back words (zeroed)
  uint32_t* status_next;     // zeroed here for the following pass (may be null)
  uint32_t* tile_ctr;        // dynamic tile counter (zeroed)
  uint32_t num_tiles;
};

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift) {
  return (uint32_t)(key >> shift) & (kRadix - 1);
}

template <typename K, typename V, int BLOCK, int ITEMS>
struct OnesweepSmem {
  static constexpr int TILE = BLOCK * ITEMS;
  static constexpr int NW = BLOCK / 32;
  K keys[TILE];
  V vals[TILE];
  uint32_t whist[NW][kRadix];
  uint32_t lstart[kRadix];
  uint32_t gofs[kRadix];
  uint32_t scan[NW + 1];
  uint32_t tile;
};

template <typename K, typename V, int BLOCK, int ITEMS, class Loader, class Emitter>
__global__ void __launch_bounds__(BLOCK)
k_onesweep(PassArgs a, Loader ld, Emitter em) {
  static_assert(BLOCK == kRadix, "one thread per digit bin");
  using S = OnesweepSmem<K, V, BLOCK, ITEMS>;
  constexpr int TILE = S::TILE;
  constexpr int NW = S::NW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);

  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) sm.tile = atomicAdd(a.tile_ctr, 1u);
#pragma unroll
  for (int w = 0; w < NW; ++w) sm.whist[w][tid] = 0;
  __syncthreads();
  const uint32_t tile = sm.tile;
  const int64_t base = (int64_t)tile * TILE;

  // Reset the next pass's look-back words for this tile (ping-pong buffers).
  if (a.status_next) a.status_next[(uint64_t)tile * kRadix + tid] = 0u;

  // ---- load (warp-striped: warp w owns a contiguous ITEMS*32 slice) ----
  K k[ITEMS];
  V v[ITEMS];
  uint32_t rk[ITEMS];
  const int64_t wbase = base + (int64_t)warp * ITEMS * 32 + lane;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    int64_t idx = wbase + (int64_t)i * 32;
    if (idx < a.n) ld.load(idx, k[i], v[i]);
  }

  // ---- warp-level stable ranking by digit (match-any multisplit) ----
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    int64_t idx = wbase + (int64_t)i * 32;
    uint32_t d = idx < a.n ? digit_of(k[i], a.shift) : 0x100u;
    uint32_t peers = __match_any_sync(kFull, d);
    uint32_t lead = __ffs(peers) - 1;
    uint32_t old = 0;
    if (lane == lead && d < 0x100u) {
      old = sm.whist[warp][d];
      sm.whist[warp][d] = old + __popc(peers);
    }
    old = __shfl_sync(kFull, old, lead);
    rk[i] = old + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();

  // ---- per-digit: cross-warp exclusive scan, tile count, look-back ----
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    uint32_t c = sm.whist[w][tid];
    sm.whist[w][tid] = cnt;
    cnt += c;
  }
  uint32_t* my_status = a.status + (uint64_t)tile * kRadix + tid;
  if (tile == 0) {
    st_relaxed(my_status, kFlagPrefix | (a.gbase[tid] + cnt));
  } else {
    st_relaxed(my_status, kFlagAgg | cnt);
  }
  uint32_t total;
  uint32_t lstart = block_excl_sum<BLOCK>(cnt, sm.scan, &total);
  uint32_t excl;
  if (tile == 0) {
    excl = a.gbase[tid];
  } else {
    excl = lookback(a.status + tid, tile, kRadix);
    st_relaxed(my_status, kFlagPrefix | (excl + cnt));
  }
  sm.lstart[tid] = lstart;
  sm.gofs[tid] = excl - lstart;  // global dst = gofs[d] + tile-local sorted position
  __syncthreads();

  // ---- scatter into shared memory in digit order ----
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    int64_t idx = wbase + (int64_t)i * 32;
    if (idx < a.n) {
      uint32_t d = digit_of(k[i], a.shift);
      uint32_t pos = sm.lstart[d] + sm.whist[warp][d] + rk[i];
      sm.keys[pos] = k[i];
      sm.vals[pos] = v[i];
    }
  }
  __syncthreads();

  // ---- coalesced write-out: consecutive threads -> consecutive positions ----
  const int64_t rem = a.n - base;
  const uint32_t tcount = rem < TILE ? (uint32_t)rem : (uint32_t)TILE;
  uint32_t dst[ITEMS];
  bool ok[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    uint32_t s = i * BLOCK + tid;
    ok[i] = s < tcount;
    if (ok[i]) {
      k[i] = sm.keys[s];
      v[i] = sm.vals[s];
      dst[i] = sm.gofs[digit_of(k[i], a.shift)] + s;
    }
  }
  em.template emit<ITEMS>(dst, k, v, ok);
}

// Every digit was constant: the stable order is the identity.
template <typename K, typename V, class Loader, class Emitter>
__global__ void k_identity_pass(int64_t n, Loader ld, Emitter em) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t dst[1];
  K k[1];
  V v[1];
  bool ok[1];
  ok[0] = i < n;
  if (ok[0]) {
    ld.load(i, k[0], v[0]);
    dst[0] = (uint32_t)i;
  }
  em.template emit<1>(dst, k, v, ok);
}

// Plain array loader / emitter for the middle passes.
template <typename K, typename V>
struct ArrayLoader {
  const K* __restrict__ keys;
  const V* __restrict__ vals;
  __device__ __forceinline__ void load(int64_t i, K& k, V& v) const {
    k = ld_stream(keys + i);
    v = ld_stream(vals + i);
  }
};

template <typename K, typename V>
struct ArrayEmitter {
  K* __restrict__ keys;
  V* __restrict__ vals;
  template <int N>
  __device__ __forceinline__ void emit(const uint32_t (&dst)[N], const K (&k)[N], const V (&v)[N],
                                       const bool (&ok)[N]) const {
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (ok[i]) {
        keys[dst[i]] = k[i];
        vals[dst[i]] = v[i];
      }
  }
};

// Exclusive scan of the per-pass digit histograms: hist[p][256] -> gbase[p][256].
__global__ void k_digit_scan(const uint32_t* __restrict__ hist, uint32_t* __restrict__ gbase, int passes) {
  __shared__ uint32_t scratch[kRadix / 32 + 1];
  for (int p = 0; p < passes; ++p) {
    uint32_t total;
    uint32_t x = hist[p * kRadix + threadIdx.x];
    gbase[p * kRadix + threadIdx.x] = block_excl_sum<kRadix>(x, scratch, &total);
  }
}

}  // namespace dmst

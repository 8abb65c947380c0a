// Device kernels of the dendrogram pipeline (sm_100a).  Host orchestration
// and the C ABI are in dmst.cu.  Reference symbols are cited as
// file:line under /root/reference/pkg/src/dendromst/.
#pragma once
#include "../../include/dmst.h"
#include "common.cuh"
#include "radix.cuh"
#include "bucket.cuh"

namespace dmst {

constexpr int EW_BLOCK = 256;                  // elementwise kernels
constexpr int SEL_BLOCK = 256;                 // k_select_edges
#ifndef DMST_LS_TILE
#define DMST_LS_TILE 2048
#endif
constexpr int LS_TILE = DMST_LS_TILE;          // k_leafscan words per tile
constexpr int CHASE_FREE = 8;    // V2 chase steps before rulers may end a chase
constexpr int CHASE_CAP = 512;   // hard bound on one V2 chase

// ~1/32 of vertices are "rulers": a long chase stops at the first ruler it
// reaches, so pointer jumping only runs over rulers (deep in-trees: chains).
__device__ __forceinline__ bool is_ruler(uint32_t v) { return ((v * 0x9E3779B1u) >> 27) == 0; }

// ------------------------------------------------------------ key codec
__device__ __forceinline__ uint64_t desc_key(double w) { return desc_key_of(w); }
__device__ __forceinline__ double key_to_double(uint64_t key) {
  uint64_t asc = ~key;
  uint64_t b = (asc >> 63) ? (asc & 0x7fffffffffffffffull) : ~asc;
  return __longlong_as_double((long long)b);
}

// ------------------------------------------------ 1. edge sort (sort #1)
// AND / OR of the keys of a strided sample (<= 65536 keys): predicts the
// edge sort's first active digit so its upsweep can also do the full key
// reduction (k_upsweep<KEYRED>).
// Also the smallest top field (key >> 52: sign + exponent) of the sample,
// the base of the upsweep's in-register top-field presence window.
__global__ void __launch_bounds__(1024) k_key_sample(const double* __restrict__ w, int64_t n,
                                                     unsigned long long* __restrict__ and_or,
                                                     uint32_t* __restrict__ top_min) {
  const int64_t stride = n > 65536 ? n / 65536 : 1;
  uint64_t a = ~0ull, o = 0ull;
  uint32_t tmin = 0xfffu;
#pragma unroll 8
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * stride; i < n;
       i += (int64_t)gridDim.x * blockDim.x * stride) {
    const uint64_t k = desc_key(w[i]);
    a &= k;
    o |= k;
    tmin = min(tmin, (uint32_t)(k >> 52));
  }
  tmin = __reduce_min_sync(kFull, tmin);
  if (lane_id() == 0) atomicMin(top_min, tmin);
  const uint32_t alo = __reduce_and_sync(kFull, (uint32_t)a), ahi = __reduce_and_sync(kFull, (uint32_t)(a >> 32));
  const uint32_t olo = __reduce_or_sync(kFull, (uint32_t)o), ohi = __reduce_or_sync(kFull, (uint32_t)(o >> 32));
  if (lane_id() == 0) {
    atomicAnd(and_or, ((unsigned long long)ahi << 32) | alo);
    atomicOr(and_or + 1, ((unsigned long long)ohi << 32) | olo);
  }
}

// One read of w: bitwise AND / OR of all sort keys (a digit is constant
// iff AND and OR agree on its bits -> that radix pass is skipped) and the
// "-0.0 present" flag.
__global__ void __launch_bounds__(256) k_key_reduce(const double* __restrict__ w, int64_t n,
                                                    unsigned long long* __restrict__ and_or,
                                                    uint32_t* __restrict__ negzero) {
  uint64_t a = ~0ull, o = 0ull;
  bool nz = false;
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; b < n; b += stride) {
    double x[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int64_t i = b + (int64_t)q * blockDim.x;
      x[q] = i < n ? ld_stream(w + i) : w[0];
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      nz |= (uint64_t)__double_as_longlong(x[q]) == 0x8000000000000000ull;
      const uint64_t k = desc_key(x[q]);
      a &= k;
      o |= k;
    }
  }
  const uint32_t alo = __reduce_and_sync(kFull, (uint32_t)a), ahi = __reduce_and_sync(kFull, (uint32_t)(a >> 32));
  const uint32_t olo = __reduce_or_sync(kFull, (uint32_t)o), ohi = __reduce_or_sync(kFull, (uint32_t)(o >> 32));
  const bool anz = __any_sync(kFull, nz);
  if (lane_id() == 0) {
    atomicAnd(and_or, ((unsigned long long)ahi << 32) | alo);
    atomicOr(and_or + 1, ((unsigned long long)ohi << 32) | olo);
    if (anz) atomicOr(negzero, 1u);
  }
}

// First pass: key from w; payload (original id, u, v) carried through the
// sort so the final pass needs no random gathers.
// Top-field compaction: when the keys hold few distinct top fields
// (sign + exponent, key >> 52), `code` maps each present top field to its
// order-preserving dense rank, so the radix passes over the (code, mantissa)
// key skip the exponent's unused bits (tied or integral weights: 3 -> 2
// passes); `inv` maps the codes back for the heights.
constexpr int kTopShift = 52;
constexpr uint64_t kMantMask = (1ull << kTopShift) - 1;
__device__ __forceinline__ uint64_t compact_key(uint64_t k, const uint8_t* code) {
  return code ? ((uint64_t)__ldg(code + (k >> kTopShift)) << kTopShift) | (k & kMantMask) : k;
}

// K = uint64_t: the (compacted) 64-bit key.  K = uint32_t ("narrow keys"):
// when every varying key bit lies in [lo, lo + 32), the passes carry only
// those 32 bits (4 B less per item each way); the final pass restores the
// constant bits from the AND of all keys.
template <typename K>
struct Sort1Loader {
  static constexpr int NS = 3;
  __host__ __device__ static constexpr int sb(int s) { return s == 0 ? 8 : 4; }
  const double* __restrict__ w;
  const int32_t* __restrict__ u;
  const int32_t* __restrict__ v;
  const uint8_t* __restrict__ code;  // top-field compaction table or nullptr
  uint32_t lo;                       // narrow keys: lowest carried bit
  __device__ __forceinline__ const void* ptr(int s) const {
    return s == 0 ? (const void*)w : s == 1 ? (const void*)u : (const void*)v;
  }
  __device__ __forceinline__ K make(double x) const { return (K)(compact_key(desc_key(x), code) >> lo); }
  __device__ __forceinline__ K key(int64_t i) const { return make(ld_stream(w + i)); }
  __device__ __forceinline__ void load(int64_t i, K& k, Vals<3>& p) const {
    k = make(ld_stream(w + i));
    p.w[0] = (uint32_t)i;
    p.w[1] = (uint32_t)ld_stream(u + i);
    p.w[2] = (uint32_t)ld_stream(v + i);
  }
  __device__ __forceinline__ void get(char* const* st, int li, int64_t i, K& k, Vals<3>& p) const {
    k = make(reinterpret_cast<const double*>(st[0])[li]);
    p.w[0] = (uint32_t)i;
    p.w[1] = reinterpret_cast<const uint32_t*>(st[1])[li];
    p.w[2] = reinterpret_cast<const uint32_t*>(st[2])[li];
  }
};
using Sort1FirstLoader = Sort1Loader<uint64_t>;

// Final pass: RankedTree outputs (orig_of, w by rank) + rank-order endpoints,
// written from the sorted sub-tile (payload = (original id, u, v)).
// With `scount` set it also counts the endpoints per maxIncident slice
// (vertex >> sshift, <= 256 slices) in shared memory and adds the counts to
// scount[] at the end: the sliced maxIncident of view 0 then needs no
// histogram pass over the rank-order endpoints.
struct SliceCountState {
  uint32_t h[256];
};
template <typename K>
struct Sort1Emitter {
  using State = SliceCountState;
  template <int BLOCK, int R>
  __device__ __forceinline__ void init(State& st) const {
    if (scount)
      for (int b = threadIdx.x; b < 256; b += BLOCK) st.h[b] = 0;
  }
  template <int BLOCK, int R>
  __device__ __forceinline__ void finish(State& st) const {
    if (scount)
      for (int b = threadIdx.x; b < 256; b += BLOCK)
        if (st.h[b]) atomicAdd(scount + b, st.h[b]);
  }
  int32_t* __restrict__ orig_of;
  double* __restrict__ heights;
  int2* __restrict__ euv;        // rank-order endpoints (pipeline)
  int32_t* __restrict__ ru;      // optional split copies (dmst_rank_edges)
  int32_t* __restrict__ rv;
  const uint16_t* __restrict__ inv;  // top-field compaction: code -> top field (or nullptr)
  uint64_t base;                     // narrow keys: the constant bits outside [lo, lo + 32)
  uint32_t lo;
  uint32_t* __restrict__ scount = nullptr;  // per-slice endpoint counts (or null)
  uint32_t sshift = 0;
  // rank r <- item (key kn, original id, u, v)
  __device__ __forceinline__ void put(uint32_t r, K kn, uint32_t id, uint32_t eu, uint32_t ev) const {
    const uint64_t k = base | ((uint64_t)kn << lo);
    orig_of[r] = (int32_t)id;
    heights[r] = key_to_double(inv ? ((uint64_t)__ldg(inv + (k >> kTopShift)) << kTopShift) | (k & kMantMask) : k);
    if (euv) euv[r] = make_int2((int)eu, (int)ev);
    if (ru) {
      ru[r] = (int32_t)eu;
      rv[r] = (int32_t)ev;
    }
  }
  template <int BLOCK, class Tile>
  __device__ __forceinline__ void emit(const Tile& t, State& st) const {
    for (int s = threadIdx.x; s < t.cnt; s += BLOCK) {
      const K kn = t.skeys[s];
      const uint32_t* p = t.spay + 3 * s;
      put(t.gofs[digit_of<kRadixBits>(kn, t.shift)] + (uint32_t)s, kn, p[0], p[1], p[2]);
      if (scount) {
        atomicAdd(&st.h[p[1] >> sshift], 1u);
        atomicAdd(&st.h[p[2] >> sshift], 1u);
      }
    }
  }
};
using Sort1FinalEmitter = Sort1Emitter<uint64_t>;
}  // namespace dmst
#include "local_sort.cuh"
namespace dmst {

// Compaction tables from the top-field presence bitmap (128 words, 4096
// bits): code[t] = number of present top fields below t, inv[code] = t.
// One block of 128 threads.
__global__ void __launch_bounds__(128) k_top_codes(const uint32_t* __restrict__ bits, uint8_t* __restrict__ code,
                                                   uint16_t* __restrict__ inv) {
  __shared__ uint32_t wsum[4];
  const uint32_t i = threadIdx.x, word = bits[i], pc = __popc(word);
  uint32_t x = pc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane_id() >= (uint32_t)o) x += y;
  }
  if (lane_id() == 31) wsum[i >> 5] = x;
  __syncthreads();
  uint32_t base = x - pc;
  for (uint32_t q = 0; q < (i >> 5); ++q) base += wsum[q];
  for (int j = 0; j < 32; ++j) {
    const uint32_t c = base + __popc(word & ((1u << j) - 1u));
    code[32 * i + j] = (uint8_t)c;
    if ((word >> j) & 1u) inv[c] = (uint16_t)(32 * i + j);
  }
}

// heights were decoded from canonicalised keys; restore -0.0 bit patterns.
__global__ void k_fix_negzero(const double* __restrict__ w, const int32_t* __restrict__ orig_of,
                              double* __restrict__ heights, int64_t n) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n && heights[r] == 0.0) heights[r] = w[orig_of[r]];
}

// Copy a few words into host-mapped memory (small readbacks without the copy engines).
__global__ void k_readback(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, uint32_t words) {
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}

// dmst_pandora entry: already-ranked endpoints -> packed euv.
__global__ void k_pack_euv(const int32_t* __restrict__ ru, const int32_t* __restrict__ rv, int64_t n,
                           int2* __restrict__ euv) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) euv[r] = make_int2(ru[r], rv[r]);
}

// ------------------------------------------ 2. maxIncident (scatter-max)
// mi64[x] = max over edges j incident to x of ((j + 1) << 32 | other end):
// the largest incident rank (maxIncident, tree_core.py:193-199 /
// contraction.py:149-154) packed with the vertex across that edge, 0 for
// an isolated vertex.  Large views group their records by vertex bucket
// first (bucket.cuh); small views scatter-max directly (L2-resident).

__device__ __forceinline__ unsigned long long pack_mi(uint32_t j1, uint32_t other) {
  return ((unsigned long long)j1 << 32) | other;
}

// --------------------------------------------- 3. contraction (per view)
// View k: nv vertices, ne edges (local index j, ascending global rank
// grank[j]; view 0: grank = identity), mi64 as above.
//
// V1: per vertex, the maxIncident edge j (vertex_parent for view 0,
// classify.py:23-25; super_max_incident in global ranks for views >= 1,
// contraction.py:173-175) and the per-edge count of endpoints at which the
// edge is maxIncident, as a 2-bit field: 2 = leaf, 1 = chain, 0 = alpha
// (edge_kinds_from_ends, classify.py:37-42).
__global__ void k_v1(int64_t nv, const unsigned long long* __restrict__ mi64,
                     const int32_t* __restrict__ grank, int32_t* __restrict__ parent_out,
                     uint32_t* __restrict__ cnt2) {
  int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nv) return;
  const unsigned long long m = ld_stream(mi64 + x);
  const uint32_t j1 = (uint32_t)(m >> 32);
  int32_t out = -1;
  if (j1) {
    const uint32_t j = j1 - 1;
    out = grank ? __ldg(grank + j) : (int32_t)j;
    atomicAdd(cnt2 + (j >> 4), 1u << ((j & 15) * 2));
  }
  parent_out[x] = out;
}

// Exclusive prefixes of leaf-edge and alpha-edge counts per 16-edge word
// (single pass, decoupled look-back: warp 0 resolves the leaf prefix, warp 1
// the alpha prefix) + view totals (n_leaf, n_chain).  A supervertex is
// numbered by the rank order of its component's leaf edge, so
// label(leaf j) = kw[j >> 4].y + leaves below j in its word; an alpha edge's
// slot in the next view is apre[j >> 4] + alphas below j in its word.  Both
// are lookups into L2-resident arrays instead of scans.
// kw[w] = (cnt2[w], exclusive count of leaf edges before edge 16w).
__device__ __forceinline__ uint32_t leaf_bits(uint32_t w) { return (w >> 1) & 0x55555555u; }
__device__ __forceinline__ uint32_t chain_bits(uint32_t w) { return w & 0x55555555u; }
// one bit (at even positions) per edge whose 2-bit count is 0 and which exists (< ne)
__device__ __forceinline__ uint32_t alpha_bits(uint32_t w, int64_t word, int64_t ne) {
  uint32_t a = ~(w | (w >> 1)) & 0x55555555u;
  const int64_t valid = ne - word * 16;
  if (valid < 16) a &= valid <= 0 ? 0u : (1u << (2 * valid)) - 1u;
  return a;
}

// Even bits of x (one per 2-bit field) compressed into the low 16 bits.
__device__ __forceinline__ uint32_t even_bits16(uint32_t x) {
  x &= 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0F0F0F0Fu;
  x = (x | (x >> 4)) & 0x00FF00FFu;
  return (x | (x >> 8)) & 0x0000FFFFu;
}

__global__ void __launch_bounds__(256) k_leafscan(int64_t words, int64_t ne, const uint32_t* __restrict__ cnt2,
                                                  uint2* __restrict__ kw, uint2* __restrict__ lw,
                                                  uint32_t* __restrict__ apre,
                                                  uint32_t* __restrict__ status, uint32_t* __restrict__ tile_ctr,
                                                  uint32_t* __restrict__ counts) {
  constexpr int ITEMS = LS_TILE / 256, TILE = LS_TILE;
  __shared__ uint32_t s_tile, s_excl[2];
  __shared__ uint32_t scratch[256 / 32 + 1];
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t ntiles = gridDim.x;
  const int64_t base = (int64_t)tile * TILE + (int64_t)threadIdx.x * ITEMS;
  uint32_t cw[ITEMS], lsum = 0, asum = 0, chains = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t w = base + i < words ? cnt2[base + i] : 0u;
    cw[i] = w;
    lsum += __popc(leaf_bits(w));
    asum += __popc(alpha_bits(w, base + i, ne));
    chains += __popc(chain_bits(w));
  }
  uint32_t ltot, atot, ctot;
  const uint32_t lex = block_excl_sum<256>(lsum, scratch, &ltot);
  const uint32_t aex = block_excl_sum<256>(asum, scratch, &atot);
  block_excl_sum<256>(chains, scratch, &ctot);
  const uint32_t warp = threadIdx.x >> 5;
  if (warp < 2) {
    uint32_t* st = status + warp * ntiles;
    const uint32_t tot = warp == 0 ? ltot : atot;
    if (lane_id() == 0) st_relaxed(st + tile, (tile == 0 ? kFlagPrefix : kFlagAgg) | tot);
    const uint32_t prev = tile == 0 ? 0u : warp_lookback(st, tile);
    if (lane_id() == 0) {
      if (tile) st_relaxed(st + tile, kFlagPrefix | (prev + tot));
      s_excl[warp] = prev;
    }
  }
  if (threadIdx.x == 0) {
    atomicAdd(counts + 0, ltot);
    atomicAdd(counts + 1, ctot);
  }
  __syncthreads();
  uint32_t lrun = s_excl[0] + lex, arun = s_excl[1] + aex;
  static_assert(ITEMS % 2 == 0 && (256 * ITEMS) % 2 == 0, "word pairs stay in one thread");
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (base + i < words) {
      kw[base + i] = make_uint2(cw[i], lrun);
      apre[base + i] = arun;
    }
    if ((i & 1) == 0 && base + i < words) {  // 32-edge leaf bitmap word + leaf prefix (k_v2)
      const uint32_t lo = even_bits16(leaf_bits(cw[i]));
      const uint32_t hi = i + 1 < ITEMS ? even_bits16(leaf_bits(cw[i + 1])) : 0u;
      lw[(base + i) >> 1] = make_uint2(lo | (hi << 16), lrun);
    }
    lrun += __popc(leaf_bits(cw[i]));
    arun += __popc(alpha_bits(cw[i], base + i, ne));
  }
}

// The same leaf / alpha numbering as k_leafscan, reduce-then-scan in three
// short kernels (no tile-to-tile look-back chain, whose propagation bounds
// the single-pass scan at ~38 ns per tile): per-tile totals, one scan of the
// totals, per-tile local scan + writes (the 2-bit counts are re-read from L2).
__global__ void __launch_bounds__(256) k_ls_reduce(int64_t words, int64_t ne, const uint32_t* __restrict__ cnt2,
                                                   uint32_t* __restrict__ tile_tot, uint32_t* __restrict__ counts) {
  constexpr int ITEMS = LS_TILE / 256;
  __shared__ uint32_t scratch[256 / 32 + 1];
  const int64_t base = (int64_t)blockIdx.x * LS_TILE + (int64_t)threadIdx.x * ITEMS;
  uint32_t lsum = 0, asum = 0, chains = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t w = base + i < words ? cnt2[base + i] : 0u;
    lsum += __popc(leaf_bits(w));
    asum += __popc(alpha_bits(w, base + i, ne));
    chains += __popc(chain_bits(w));
  }
  uint32_t ltot, atot, ctot;
  block_excl_sum<256>(lsum, scratch, &ltot);
  block_excl_sum<256>(asum, scratch, &atot);
  block_excl_sum<256>(chains, scratch, &ctot);
  if (threadIdx.x == 0) {
    tile_tot[2 * blockIdx.x] = ltot;
    tile_tot[2 * blockIdx.x + 1] = atot;
    atomicAdd(counts + 0, ltot);
    atomicAdd(counts + 1, ctot);
  }
}
// exclusive scan of the (leaf, alpha) tile totals in place; one CTA
__global__ void __launch_bounds__(1024) k_ls_scan(uint32_t* __restrict__ tile_tot, uint32_t ntiles) {
  __shared__ uint32_t scratch[1024 / 32 + 1];
  const uint32_t per = (ntiles + 1023) / 1024, b = threadIdx.x * per, e = min(ntiles, b + per);
  uint32_t sl = 0, sa = 0;
  for (uint32_t t = b; t < e; ++t) {
    sl += tile_tot[2 * t];
    sa += tile_tot[2 * t + 1];
  }
  uint32_t tl, ta;
  uint32_t rl = block_excl_sum<1024>(sl, scratch, &tl);
  uint32_t ra = block_excl_sum<1024>(sa, scratch, &ta);
  for (uint32_t t = b; t < e; ++t) {
    const uint32_t xl = tile_tot[2 * t], xa = tile_tot[2 * t + 1];
    tile_tot[2 * t] = rl;
    tile_tot[2 * t + 1] = ra;
    rl += xl;
    ra += xa;
  }
}
__global__ void __launch_bounds__(256) k_ls_apply(int64_t words, int64_t ne, const uint32_t* __restrict__ cnt2,
                                                  const uint32_t* __restrict__ tile_pre, uint2* __restrict__ kw,
                                                  uint2* __restrict__ lw, uint32_t* __restrict__ apre) {
  constexpr int ITEMS = LS_TILE / 256;
  __shared__ uint32_t scratch[256 / 32 + 1];
  const int64_t base = (int64_t)blockIdx.x * LS_TILE + (int64_t)threadIdx.x * ITEMS;
  uint32_t cw[ITEMS], lsum = 0, asum = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t w = base + i < words ? cnt2[base + i] : 0u;
    cw[i] = w;
    lsum += __popc(leaf_bits(w));
    asum += __popc(alpha_bits(w, base + i, ne));
  }
  uint32_t tot;
  const uint32_t lex = block_excl_sum<256>(lsum, scratch, &tot);
  const uint32_t aex = block_excl_sum<256>(asum, scratch, &tot);
  uint32_t lrun = tile_pre[2 * blockIdx.x] + lex, arun = tile_pre[2 * blockIdx.x + 1] + aex;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (base + i < words) {
      kw[base + i] = make_uint2(cw[i], lrun);
      apre[base + i] = arun;
    }
    if ((i & 1) == 0 && base + i < words) {  // 32-edge leaf bitmap word + leaf prefix (k_v2)
      const uint32_t lo = even_bits16(leaf_bits(cw[i]));
      const uint32_t hi = i + 1 < ITEMS ? even_bits16(leaf_bits(cw[i + 1])) : 0u;
      lw[(base + i) >> 1] = make_uint2(lo | (hi << 16), lrun);
    }
    lrun += __popc(leaf_bits(cw[i]));
    arun += __popc(alpha_bits(cw[i], base + i, ne));
  }
}

__device__ __forceinline__ uint32_t leaf_label(uint2 w, uint32_t j) {
  const uint32_t below = (1u << ((j & 15) * 2)) - 1u;
  return w.y + __popc(leaf_bits(w.x) & below);
}

// V2: chase maxIncident pointers to the component's leaf edge (ranks grow
// strictly along the chase; the leaf edge is the component's lightest
// edge) and label the vertex with that leaf's number: vertex_map
// (component_labels + contract_level, contraction.py:82-93, :165-169).
// A chase longer than CHASE_FREE steps stops at the first ruler vertex (or
// after CHASE_CAP steps) and stores ~y (y = where it stopped); rulers and
// non-rulers go to separate lists for pointer jumping.
// Views >= 1 (smi != null) store the vertex map interleaved with the view's
// maxIncident as (vm[x], smi[x]) pairs: the chain walk then gets both from
// one random 8-B probe (one DRAM sector) per level; vm has stride 2 there.
__global__ void k_v2(int64_t nv, const unsigned long long* __restrict__ mi64, const uint2* __restrict__ lw,
                     int32_t* __restrict__ vm, const int32_t* __restrict__ smi, int32_t* __restrict__ rul,
                     uint32_t* __restrict__ rul_cnt, int32_t* __restrict__ non, uint32_t* __restrict__ non_cnt,
                     bool keep) {
  // lw[j >> 5] = (leaf bitmap of edges 32w..32w+31, leaf count before 32w):
  // half the footprint of kw, so the chase's kind tests stay L2-resident
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t pol = l2_keep_policy();
  bool unresolved = false;
  if (x < nv) {
    unsigned long long m = ld_stream(mi64 + x);
    uint32_t j = (uint32_t)(m >> 32) - 1u;
    uint32_t y = (uint32_t)m;
    int s = 0;
    uint2 lwj = make_uint2(0, 0);
    while (m != 0ull) {  // m == 0: isolated vertex (single-vertex view), label 0
      lwj = ld_keep2(lw + (j >> 5), pol);
      if ((lwj.x >> (j & 31)) & 1u) break;  // leaf edge
      if (++s > CHASE_CAP || (s > CHASE_FREE && is_ruler(y))) {
        unresolved = true;
        break;
      }
      // a table within ~4x of L2 keeps its hops (normal policy: 0.81 -> 0.69
      // ms for views 1-2 at 128M); a larger one streams them (evict-first)
      m = keep ? mi64[y] : __ldcs(mi64 + y);
      j = (uint32_t)(m >> 32) - 1u;
      y = (uint32_t)m;
    }
    const int32_t lab = unresolved ? ~(int32_t)y
                                   : (m ? (int32_t)(lwj.y + __popc(lwj.x & ((1u << (j & 31)) - 1u))) : 0);
    if (smi)
      __stcs(reinterpret_cast<int2*>(vm) + x, make_int2(lab, __ldcs(smi + x)));
    else
      __stcs(vm + x, lab);
  }
  const bool ruler = unresolved && is_ruler((uint32_t)x);
  const bool plain = unresolved && !ruler;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const bool mine = t == 0 ? ruler : plain;
    const uint32_t msk = __ballot_sync(kFull, mine);
    if (msk) {
      uint32_t lead = __ffs(msk) - 1, b = 0;
      if (lane_id() == lead) b = atomicAdd(t == 0 ? rul_cnt : non_cnt, __popc(msk));
      b = __shfl_sync(kFull, b, lead);
      if (mine) (t == 0 ? rul : non)[b + __popc(msk & lanemask_lt())] = (int32_t)x;
    }
  }
}

// One pointer-jumping round over unresolved vertices: vm[x] >= 0 is a label,
// vm[x] < 0 is ~(a vertex further along the chase).  Pointers only ever
// move forward along the chase, so in-place updates are safe.
__global__ void k_jump(const int32_t* __restrict__ in, const uint32_t* __restrict__ in_cnt,
                       int32_t* __restrict__ out, uint32_t* __restrict__ out_cnt, int32_t* vm, int vs) {
  const uint32_t cnt = *in_cnt;
  for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x; t0 < cnt; t0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = t0 + threadIdx.x;
    bool again = false;
    int32_t x = 0;
    if (t < cnt) {
      x = in[t];
      const int32_t q = vm[(int64_t)~vm[(int64_t)x * vs] * vs];
      vm[(int64_t)x * vs] = q;
      again = q < 0;
    }
    const uint32_t m = __ballot_sync(kFull, again);
    if (m) {
      uint32_t lead = __ffs(m) - 1, b = 0;
      if (lane_id() == lead) b = atomicAdd(out_cnt, __popc(m));
      b = __shfl_sync(kFull, b, lead);
      if (again) out[b + __popc(m & lanemask_lt())] = x;
    }
  }
}

// Retire non-alpha edges of view k at level k (contraction.py:207) and
// compact alpha edges, in rank order, into view k+1 with endpoints remapped
// to supervertices (:170-172).  An alpha edge's slot comes from the alpha
// prefix of its 16-edge word (k_leafscan), so this is a plain elementwise
// pass with no inter-CTA scan.  The next view's maxIncident is scatter-maxed
// here for small views (L2-resident), else bucketed afterwards from
// euv_next (bucket.cuh).  View 0 also writes x1[j] = view-1 supervertex of
// every edge (the chain walk's starting point).
struct EdgeSel {
  uint32_t* __restrict__ cnt2;       // zeroed for the next view
  const uint2* __restrict__ kw;      // (child counts, leaf prefix) per 16 edges
  const uint32_t* __restrict__ apre; // alpha prefix per 16 edges
  const int2* __restrict__ euv;
  const int32_t* __restrict__ grank; // null => identity (view 0)
  const int32_t* __restrict__ vm;    // vertex map, stride vs (2 = packed walk table)
  int vs;
  int8_t* __restrict__ ret;
  int2* __restrict__ euv_next;
  int32_t* __restrict__ grank_next;
  unsigned long long* __restrict__ mi64_next;  // direct mode (null => bucketed from euv_next)
  int32_t* __restrict__ x1;          // view 0 only
  int8_t level;
  uint32_t* __restrict__ reset_misc;   // level counters (15 words) zeroed for the next view
  uint32_t* __restrict__ reset_status; // leafscan look-back words zeroed for the next view
  int64_t n_status;
  uint32_t* __restrict__ scount;     // next view sliced: its endpoints counted per slice (or null)
  uint32_t sshift;
  // CHASE select (view 0): labels by chasing maxIncident instead of a vertex map
  const unsigned long long* __restrict__ mi0;
  const uint2* __restrict__ lw;      // (leaf bitmap, leaf prefix) per 32 edges
  int32_t* __restrict__ defer;       // edges whose chase ran over CHASE_FUSED steps
  uint32_t* __restrict__ defer_cnt;
};

constexpr int SEL_U = 4;  // edges per thread per iteration (gathers in flight together)
constexpr int CHASE_FUSED = 16;
#ifndef DMST_SEL_CHASE_U
#define DMST_SEL_CHASE_U 2
#endif  // view-0 select: chase steps before an edge is deferred

// Per-edge inputs of the select: 2-bit count -> kind, leaf label, alpha slot,
// global rank, endpoints (only when a label must be looked up).
struct SelEdge {
  bool in, alpha, need;
  int32_t lab, g;
  uint32_t pos;
  int2 e;
};
__device__ __forceinline__ SelEdge sel_load(const EdgeSel& es, int64_t j, int64_t n) {
  SelEdge r;
  r.in = j < n;
  const uint2 w = r.in ? es.kw[j >> 4] : make_uint2(0, 0);
  const uint32_t sh = (uint32_t)(j & 15) * 2;
  const uint32_t c = (w.x >> sh) & 3u;
  r.alpha = r.in && c == 0u;
  r.lab = c == 2u ? (int32_t)leaf_label(w, (uint32_t)j) : -1;
  r.pos = r.alpha ? es.apre[j >> 4] + __popc(alpha_bits(w.x, 0, 16) & ((1u << sh) - 1u)) : 0u;
  r.g = r.in ? (es.grank ? __ldcs(es.grank + j) : (int32_t)j) : 0;
  r.need = r.alpha || (r.in && es.x1 != nullptr && r.lab < 0);
  r.e = r.need ? __ldcs(es.euv + j) : make_int2(0, 0);
  return r;
}

// Per-edge outputs: the view-1 supervertex (view 0), retirement of a
// non-alpha edge, or the alpha edge's slot in the next view (+ its slice
// counts / direct maxIncident).
__device__ __forceinline__ void sel_emit(const EdgeSel& es, int64_t j, const SelEdge& d, int32_t a, int32_t b,
                                         uint32_t* shist) {
  // a leaf edge's component is labelled by the edge itself; a chain or
  // alpha edge's by its first endpoint
  if (es.x1) __stcs(es.x1 + j, a);
  if (!d.alpha) {
    es.ret[d.g] = es.level;
  } else {
    __stcs(es.euv_next + d.pos, make_int2(a, b));
    __stcs(es.grank_next + d.pos, d.g);
    if (es.scount) {
      atomicAdd(&shist[(uint32_t)a >> es.sshift], 1u);
      atomicAdd(&shist[(uint32_t)b >> es.sshift], 1u);
    }
    if (es.mi64_next) {
      atomicMax(es.mi64_next + a, pack_mi(d.pos + 1u, (uint32_t)b));
      atomicMax(es.mi64_next + b, pack_mi(d.pos + 1u, (uint32_t)a));
    }
  }
}

// CHASE (view 0 only): no vertex map.  A label is found by chasing view 0's
// maxIncident pointers from the endpoint to its component's leaf edge, as
// k_v2 would (contraction.py:82-93), but only for the endpoints the select
// needs (the first endpoint of chain edges, both ends of alpha edges: ~1.36
// random reads per edge on random trees instead of V2's 0.64 per vertex +
// the select's 1.0 per edge + V2's streaming pass).  An edge with a chase
// longer than CHASE_FUSED steps is deferred (es.defer) and finished by
// k_select_fix after V2 + pointer jumping.
template <bool CHASE, int U = (CHASE ? DMST_SEL_CHASE_U : SEL_U)>
__global__ void __launch_bounds__(SEL_BLOCK) k_select_edges(int64_t n, EdgeSel es) {
  __shared__ uint32_t shist[256];  // per-slice endpoint counts of the next view (es.scount)
  if (es.scount) {
    for (int b = threadIdx.x; b < 256; b += SEL_BLOCK) shist[b] = 0;
    __syncthreads();
  }
  {  // the host has read this view's counters: clear them for the next view
    const int64_t g = (int64_t)blockIdx.x * SEL_BLOCK + threadIdx.x;
    for (int64_t i = g; i < es.n_status; i += (int64_t)gridDim.x * SEL_BLOCK) es.reset_status[i] = 0u;
    if (g < 15) es.reset_misc[g] = 0u;
  }
  const uint64_t pol = l2_keep_policy();
  const int64_t stride = (int64_t)gridDim.x * SEL_BLOCK * U;
  for (int64_t b0 = (int64_t)blockIdx.x * SEL_BLOCK * U + threadIdx.x; b0 < n; b0 += stride) {
    SelEdge d[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int64_t j = b0 + (int64_t)q * SEL_BLOCK;
      d[q] = sel_load(es, j, n);
      if (d[q].in && (j & 15) == 0) es.cnt2[j >> 4] = 0u;
    }
    int32_t a[U], bb[U];
    if constexpr (!CHASE) {
#pragma unroll
      for (int q = 0; q < U; ++q) {
        a[q] = d[q].need ? es.vm[(int64_t)d[q].e.x * es.vs] : d[q].lab;
        bb[q] = d[q].alpha ? es.vm[(int64_t)d[q].e.y * es.vs] : 0;
      }
    } else {
      unsigned long long ma[U], mb[U];
      bool pa[U], pb[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        pa[q] = d[q].need;
        pb[q] = d[q].alpha;
        ma[q] = pa[q] ? __ldcs(es.mi0 + d[q].e.x) : 0ull;
        mb[q] = pb[q] ? __ldcs(es.mi0 + d[q].e.y) : 0ull;
        a[q] = d[q].lab;
        bb[q] = 0;
      }
      for (int s = 0;; ++s) {
        uint2 la[U], lb[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {  // kind tests: the leaf bitmap is L2-resident
          if (pa[q]) la[q] = ld_keep2(es.lw + (((uint32_t)(ma[q] >> 32) - 1u) >> 5), pol);
          if (pb[q]) lb[q] = ld_keep2(es.lw + (((uint32_t)(mb[q] >> 32) - 1u) >> 5), pol);
        }
        bool more = false;
#pragma unroll
        for (int q = 0; q < U; ++q) {
          if (pa[q]) {
            const uint32_t jj = (uint32_t)(ma[q] >> 32) - 1u;
            if ((la[q].x >> (jj & 31)) & 1u) {
              a[q] = (int32_t)(la[q].y + __popc(la[q].x & ((1u << (jj & 31)) - 1u)));
              pa[q] = false;
            } else if (s == CHASE_FUSED) {
              a[q] = -1;
              pa[q] = false;
            } else {
              more = true;
            }
          }
          if (pb[q]) {
            const uint32_t jj = (uint32_t)(mb[q] >> 32) - 1u;
            if ((lb[q].x >> (jj & 31)) & 1u) {
              bb[q] = (int32_t)(lb[q].y + __popc(lb[q].x & ((1u << (jj & 31)) - 1u)));
              pb[q] = false;
            } else if (s == CHASE_FUSED) {
              bb[q] = -1;
              pb[q] = false;
            } else {
              more = true;
            }
          }
        }
        if (!more) break;
#pragma unroll
        for (int q = 0; q < U; ++q) {
          // chase hops with the normal policy (evict-first: +0.13 ms at 128M)
          if (pa[q]) ma[q] = es.mi0[(uint32_t)ma[q]];
          if (pb[q]) mb[q] = es.mi0[(uint32_t)mb[q]];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      if (!d[q].in) continue;
      const int64_t j = b0 + (int64_t)q * SEL_BLOCK;
      if (CHASE && (a[q] < 0 || bb[q] < 0)) {  // chase too long: finished by k_select_fix
        es.defer[atomicAdd(es.defer_cnt, 1u)] = (int32_t)j;
        continue;
      }
      sel_emit(es, j, d[q], a[q], bb[q], shist);
    }
  }
  if (es.scount) {
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += SEL_BLOCK)
      if (shist[b]) atomicAdd(es.scount + b, shist[b]);
  }
}

// The deferred edges of a CHASE select, once V2 + pointer jumping have
// written view 0's vertex map (es.vm).
__global__ void __launch_bounds__(SEL_BLOCK) k_select_fix(const int32_t* __restrict__ list,
                                                          const uint32_t* __restrict__ cnt, EdgeSel es) {
  __shared__ uint32_t shist[256];
  if (es.scount) {
    for (int b = threadIdx.x; b < 256; b += SEL_BLOCK) shist[b] = 0;
    __syncthreads();
  }
  const uint32_t m = *cnt;
  for (int64_t t = (int64_t)blockIdx.x * SEL_BLOCK + threadIdx.x; t < m; t += (int64_t)gridDim.x * SEL_BLOCK) {
    const int64_t j = list[t];
    const SelEdge d = sel_load(es, j, INT64_MAX);
    const int32_t a = d.need ? es.vm[(int64_t)d.e.x * es.vs] : d.lab;
    const int32_t b = d.alpha ? es.vm[(int64_t)d.e.y * es.vs] : 0;
    sel_emit(es, j, d, a, b, shist);
  }
  if (es.scount) {
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += SEL_BLOCK)
      if (shist[b]) atomicAdd(es.scount + b, shist[b]);
  }
}

// Final view (no alpha edges, contraction.py:203-205): every edge retires at L.
__global__ void k_retire_all(int64_t n, const int32_t* __restrict__ grank, int8_t* __restrict__ ret, int8_t L) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) ret[grank ? grank[j] : j] = L;
}

// ------------------------------------------------------ 4. expansion walk
struct LevelTable {
  int64_t soff[DMST_MAX_LEVELS + 2];  // offset of maxIncident (global ranks) of view k in smi_all
  int32_t L;
};

// assign_chains (expansion.py:97-128): an edge retired at view r is tried
// at views r+1..L; the first whose supervertex parent p satisfies
// 0 <= p < e wins.  The chain (terminal, anchor) is encoded as the dense key
// 1 + soff[k] + anchor (a terminal edge is a terminal only at the one level
// it retires at, so (level, anchor) identifies the chain); 0 = root chain.
// The walk starts at the edge's view-1 supervertex x1[e] (written by the
// view-0 select); per level one 8-B probe of the packed walk table
// lvl[soff[k] + x] = (vm_k[x], smi_k[x]) (maxIncident of view k in global
// ranks, and the supervertex of x in view k + 1).
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
k_walk(int64_t n, const int8_t* __restrict__ ret, const int32_t* __restrict__ x1, const int2* __restrict__ lvl,
       const __grid_constant__ LevelTable lt, uint32_t* __restrict__ keys, uint32_t* __restrict__ and_or) {
  uint32_t ka = ~0u, ko = 0u;
  const uint64_t pol = l2_keep_policy();
  const int64_t stride = (int64_t)gridDim.x * BLOCK;
  for (int64_t e0 = (int64_t)blockIdx.x * BLOCK; e0 < n; e0 += stride) {
    const int64_t e = e0 + threadIdx.x;
    if (e < n) {
      uint32_t key = 0;
      const int r = __ldcs(ret + e);
      if (r < lt.L) {
        int32_t x = __ldcs(x1 + e);  // view-1 supervertex
        for (int k = 1;; ++k) {
          // view 1's table is larger than L2 (evict-first); the deeper,
          // smaller tables are kept resident (evict_last)
          const int2* pt = lvl + lt.soff[k] + x;
          int2 t;
          if (k == 1) {
            t = __ldcs(pt);  // evict-first: leave L2 to the deeper tables (walk -0.08 ms)
          } else {
            const uint2 q = ld_keep2(reinterpret_cast<const uint2*>(pt), pol);
            t = make_int2((int)q.x, (int)q.y);
          }
          if (k > r && t.y >= 0 && t.y < (int32_t)e) {
            key = (uint32_t)(1 + lt.soff[k] + x);
            break;
          }
          if (k >= lt.L) break;
          x = t.x;
        }
      }
      __stcs(keys + e, key);
      ka &= key;
      ko |= key;
    }
  }
  ka = __reduce_and_sync(kFull, ka);
  ko = __reduce_or_sync(kFull, ko);
  if (lane_id() == 0) {
    atomicAnd(and_or, ka);
    atomicOr(and_or + 1, ko);
  }
}

// Chain sort items are packed 64-bit (chain key << 32 | rank): one array, so
// a digit run of m items is one contiguous 8 m-byte run; the radix digits
// sit at bit 32 + (chain-key digit offset).
struct Sort2FirstLoader {
  static constexpr int NS = 1;
  __host__ __device__ static constexpr int sb(int) { return 4; }
  const uint32_t* __restrict__ keys;
  using RawKey = uint32_t;
  static constexpr bool VEC = true;
  __device__ __forceinline__ const uint32_t* raw_keys() const { return keys; }
  __device__ __forceinline__ uint64_t key_of_raw(uint32_t r, int64_t i) const {
    return ((uint64_t)r << 32) | (uint32_t)i;
  }
  __device__ __forceinline__ const void* ptr(int) const { return keys; }
  __device__ __forceinline__ uint64_t key(int64_t i) const {
    return ((uint64_t)ld_stream(keys + i) << 32) | (uint32_t)i;
  }
  __device__ __forceinline__ void load(int64_t i, uint64_t& k, Vals<0>&) const { k = key(i); }
  __device__ __forceinline__ void get(char* const* st, int li, int64_t i, uint64_t& k, Vals<0>&) const {
    k = ((uint64_t)reinterpret_cast<const uint32_t*>(st[0])[li] << 32) | (uint32_t)i;
  }
};

// stitch_chains (expansion.py:131-145): in (key, rank) order the parent of
// an edge is its predecessor in the same chain, or the chain's terminal
// (-1 = ROOT for the root chain, key 0).  Writing edge_parent[e] straight
// from chain order is a random 4-B store per edge (~1.3 ms per 128M even
// into an L2-resident window, 3 ms into DRAM; tools/winscatter), so the
// (rank, parent) records are grouped by 8192-rank window with the two
// multisplit passes of bucket.cuh (this source feeds the first one, reading
// the sorted chain keys / ranks) and k_link_apply writes every window from
// shared memory with coalesced stores.  Window f holds exactly the ranks
// [8192 f, 8192 (f + 1)), so all bucket offsets are static.
struct LinkSortedSrc {
  static constexpr int RW = 2, NS = 1;
  __host__ __device__ static constexpr int sb(int) { return 8; }  // one sorted 8-B item per record
  const unsigned long long* __restrict__ items;  // sorted (chain key << 32 | rank)
  const int32_t* __restrict__ smi_all;
  __device__ __forceinline__ const void* ptr(int) const { return items; }
  __device__ __forceinline__ uint32_t parent(uint32_t key, uint32_t pkey, uint32_t pval, bool first) const {
    if (!first && pkey == key) return pval;
    return key == 0 ? 0xffffffffu : (uint32_t)smi_all[key - 1];
  }
  __device__ __forceinline__ void get(const unsigned char* const* st, int li, int64_t i, uint32_t (&r)[2]) const {
    const unsigned long long* k = reinterpret_cast<const unsigned long long*>(st[0]);
    const unsigned long long it = k[li];
    const unsigned long long pv = li > 0 ? k[li - 1] : (i > 0 ? __ldg(items + i - 1) : 0ull);
    r[0] = (uint32_t)it;
    r[1] = parent((uint32_t)(it >> 32), (uint32_t)(pv >> 32), (uint32_t)pv, i == 0);
  }
  __device__ __forceinline__ uint32_t staged_vertex(const unsigned char* const* st, int li, int64_t) const {
    return (uint32_t)reinterpret_cast<const unsigned long long*>(st[0])[li];
  }
  __device__ __forceinline__ void load(int64_t i, uint32_t (&r)[2]) const {
    const unsigned long long it = __ldg(items + i);
    const unsigned long long pv = i > 0 ? __ldg(items + i - 1) : 0ull;
    r[0] = (uint32_t)it;
    r[1] = parent((uint32_t)(it >> 32), (uint32_t)(pv >> 32), (uint32_t)pv, i == 0);
  }
  __device__ __forceinline__ uint32_t vertex(int64_t i) const { return (uint32_t)__ldg(items + i); }
};

// Static bucket starts: coarse bucket c = [c << (FB_BITS + gshift)), fine f = [f << FB_BITS).
__global__ void k_link_cursors(uint32_t* __restrict__ coarse, uint32_t nc, uint32_t* __restrict__ fine, uint32_t nf,
                               uint32_t gshift) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
    fine[i] = i << FB_BITS;
    if (i < nc) coarse[i] = i << (FB_BITS + gshift);
  }
}

// Sliced link: (rank, parent) records grouped by 2M-rank slice (one
// multisplit pass); plain 4-B stores into edge_parent in record order, so the
// slice being written (8 MB) stays L2-resident and its partial sectors merge
// there (random stores into an L2-resident table: ~210 G/s, tools/randbench.cu).
__global__ void __launch_bounds__(256) k_link_scatter(const uint2* __restrict__ recs, int64_t n,
                                                      int32_t* __restrict__ edge_parent) {
  constexpr int G = 4;  // 16-B loads (two records) in flight per thread
  const int64_t p0 = (int64_t)blockIdx.x * 256 * G + threadIdx.x;
  const uint4* r4 = reinterpret_cast<const uint4*>(recs);
  const int64_t np = n / 2;
  uint4 a[G];
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int64_t p = p0 + q * 256;
    a[q] = p < np ? __ldcs(r4 + p) : make_uint4(0xffffffffu, 0, 0xffffffffu, 0);
  }
#pragma unroll
  for (int q = 0; q < G; ++q) {
    if (a[q].x != 0xffffffffu) edge_parent[a[q].x] = (int32_t)a[q].y;
    if (a[q].z != 0xffffffffu) edge_parent[a[q].z] = (int32_t)a[q].w;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) {
    const uint2 r = __ldcs(recs + n - 1);
    edge_parent[r.x] = (int32_t)r.y;
  }
}

// One CTA per 8192-rank window: place its (rank, parent) records in shared
// memory, then store the window's edge_parent slice coalesced.
__global__ void __launch_bounds__(512) k_link_apply(const uint2* __restrict__ recs, int64_t n,
                                                    int32_t* __restrict__ edge_parent) {
  __shared__ int32_t sp[FB];
  const int64_t base = (int64_t)blockIdx.x << FB_BITS;
  const int cnt = n - base < FB ? (int)(n - base) : FB;
  if (cnt == FB) {
    // full window: all 16 records of a thread in flight at once (two per 16-B load)
    constexpr int V = FB / 2 / 512;
    const uint4* r4 = reinterpret_cast<const uint4*>(recs + base);
    uint4 x[V];
#pragma unroll
    for (int q = 0; q < V; ++q) x[q] = __ldcs(r4 + q * 512 + threadIdx.x);
#pragma unroll
    for (int q = 0; q < V; ++q) {
      sp[x[q].x - (uint32_t)base] = (int32_t)x[q].y;
      sp[x[q].z - (uint32_t)base] = (int32_t)x[q].w;
    }
  } else {
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const uint2 r = __ldcs(recs + base + i);
      sp[r.x - (uint32_t)base] = (int32_t)r.y;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) __stcs(edge_parent + base + i, sp[i]);
}

// Single-chain trees (every chain key equal, chain sort skipped): rank order
// is chain order.
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

}  // namespace dmst

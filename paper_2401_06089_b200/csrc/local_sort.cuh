// Edge sort, wide keys: finish the sort inside shared memory.
//
// A 64-bit-key edge sort (uniform float64 weights: 8 active digits) runs only
// its three TOP active digits as global LSD passes; the items are then
// ordered by `key >> pshift` (pshift = the lowest of those digits), with the
// original id order inside every run of equal prefix (stable passes).  Runs
// are short for spread-out weights (~250 items per run at 128M uniform
// weights), so one kernel finishes the sort: each CTA takes the runs that
// START in its 2048-item tile (the window must end within kLocalCap items of
// the tile start) and sorts
// the window by (key, position in window) — the position breaks ties exactly
// as the original id does — then writes the RankedTree outputs for its window
// directly (orig_of, heights, rank-order endpoints).  Five global passes
// over 20-B items become one read, one write and on-chip work.
//
// In-window sort: a counting sort on (key - window base) >> shift (4096
// buckets over the key range of the window's runs) scatters the keys into ~1-item buckets (shared-memory atomics,
// order-free), then every item's final slot is its bucket start plus the
// number of bucket members below it in (key, position) order (one thread per
// item, no dependent chains).  A window whose largest bucket exceeds kLocalBucketMax
// (clustered keys) is sorted instead by stable 8-bit LSD passes over its
// varying bits (ranking as in k_downsweep).  A window longer than kLocalCap
// (a run of equal top bits that large: heavily tied or clustered weights)
// sets `overflow`; the host then re-runs the plain LSD sort, which produces
// the same bits.
//
// Replaces `np.argsort(-w, kind="stable")` (tree_core.py:180 of
// /root/reference/pkg/src/dendromst/) together with radix.cuh.
#pragma once
#include "common.cuh"
#include "radix.cuh"

namespace dmst {

// Geometry: BLOCK threads x ITEMS items = the window capacity; windows start
// at the first run start of each TILE-item tile; 2^BBITS counting-sort buckets.
constexpr int kLocalBucketMax = 24;             // larger bucket -> LSD passes for the window
template <int BLOCK_, int ITEMS_, int TILE_, int BBITS_>
struct LocalGeom {
  static constexpr int LF_BLOCK = BLOCK_, LF_ITEMS = ITEMS_, kLocalTile = TILE_, kLocalBucketBits = BBITS_;
  static constexpr int kLocalCap = BLOCK_ * ITEMS_;
};
using LocalGeomDefault = LocalGeom<512, 8, 2048, 11>;

struct LocalSortArgs {
  const uint64_t* __restrict__ keys;  // [n], sorted by key >> pshift (stable)
  const uint32_t* __restrict__ pay;   // [3 n] (original id, u, v)
  int64_t n;
  int pshift;
  uint32_t* __restrict__ overflow;    // set to 1 when a window exceeds kLocalCap
};

template <class G>
struct LocalSmem {
  static constexpr int LF_BLOCK = G::LF_BLOCK, kLocalCap = G::kLocalCap, kLocalBucketBits = G::kLocalBucketBits;
  uint64_t okey[kLocalCap];
  uint16_t oidx[kLocalCap];
  union {
    struct {
      uint32_t cnt[1 << kLocalBucketBits];
      uint32_t cur[1 << kLocalBucketBits];
    } cs;
    struct {
      uint32_t whist[LF_BLOCK / 32][kRadix];
      uint32_t lstart[kRadix + 1];
    } lsd;
  } u;
  uint32_t scan[LF_BLOCK / 32 + 1];
  unsigned long long red[2][LF_BLOCK / 32];
  unsigned long long found[2];
  uint32_t maxb;
  uint32_t shist[256];  // per-slice endpoint counts (em.scount)
};

template <class Emitter, class G = LocalGeomDefault>
__global__ void __launch_bounds__(G::LF_BLOCK, 1024 / G::LF_BLOCK) k_local_final(LocalSortArgs a, Emitter em) {
  constexpr int LF_BLOCK = G::LF_BLOCK, LF_ITEMS = G::LF_ITEMS, kLocalTile = G::kLocalTile;
  constexpr int kLocalCap = G::kLocalCap, kLocalBucketBits = G::kLocalBucketBits;
  constexpr int NW = LF_BLOCK / 32, R = kRadix, NB = 1 << kLocalBucketBits;
  static_assert(NB % LF_BLOCK == 0 && LF_BLOCK >= R, "geometry");
  extern __shared__ __align__(16) unsigned char lsm[];
  LocalSmem<G>& s = *reinterpret_cast<LocalSmem<G>*>(lsm);
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t lo = (int64_t)blockIdx.x * kLocalTile;
  const int64_t hi = min(a.n, lo + kLocalTile);

  // ---- window [start, end): the runs starting in [lo, hi), found from the
  // keys [lo - 1, lo + kLocalCap) staged once in shared memory (the window
  // must end by lo + kLocalCap; a run start is where key >> pshift changes).
  // Prefixes compare on the high words when pshift >= 32.
  const int64_t stage_end = min(a.n, lo + kLocalCap);
  const int nst = (int)(stage_end - lo);
  for (int i = tid; i < nst; i += LF_BLOCK) s.okey[i] = ld_stream(a.keys + lo + i);
  const uint64_t before = lo > 0 ? ld_stream(a.keys + lo - 1) : 0ull;
  if (tid < 2) s.found[tid] = ~0ull;
  if (tid == 0) s.maxb = 0;
  __syncthreads();
  const int psh = a.pshift;
  auto differ = [&](uint64_t x, uint64_t y) {
    return psh >= 32 ? ((uint32_t)((x ^ y) >> 32) >> (psh - 32)) != 0u : ((x ^ y) >> psh) != 0ull;
  };
  {
    // runs are short: look at the first LF_BLOCK / 2 positions after lo and
    // after hi (one per thread), the rest of the staged keys only if needed
    const int tile = (int)(hi - lo);
    const int half = (int)(tid >= LF_BLOCK / 2);
    const int hb0 = half ? tile : 0, hb1 = half ? nst : tile;  // positions [hb0, hb1) of this half
    for (int i0 = hb0;; i0 += LF_BLOCK / 2) {
      const int i = i0 + (int)(tid % (LF_BLOCK / 2));
      uint32_t f = 0xffffffffu;
      if (i < hb1 && ((lo + i == 0) || differ(s.okey[i], i ? s.okey[i - 1] : before))) f = (uint32_t)i;
      f = __reduce_min_sync(kFull, f);
      if (lane == 0 && f != 0xffffffffu) atomicMin(&s.found[half], (unsigned long long)f);
      __syncthreads();
      const bool more = (s.found[0] == ~0ull && i0 - hb0 + LF_BLOCK / 2 < tile - 0) ||
                        (s.found[1] == ~0ull && (i0 - hb0) + LF_BLOCK / 2 < nst - tile);
      __syncthreads();  // every thread has read `found` before the next step may update it
      if (!more) break;
    }
  }
  for (int b = tid; b < NB; b += LF_BLOCK) s.u.cs.cnt[b] = 0;
  __syncthreads();
  if (s.found[0] == ~0ull) return;  // no run starts in this tile
  const int64_t start = lo + (int64_t)s.found[0];
  const int64_t end = s.found[1] != ~0ull ? lo + (int64_t)s.found[1] : (stage_end == a.n ? a.n : -1);
  if (end < 0) {  // the window runs past the staged keys: over capacity
    if (tid == 0) atomicOr(a.overflow, 1u);
    return;
  }
  const int W = (int)(end - start);
  const int woff = (int)(start - lo);
  const int ipw = (W + NW * 32 - 1) / (NW * 32);  // items per lane actually used (<= LF_ITEMS)
  const int wbase = warp * ipw * 32 + lane;

  // ---- keys -> registers (blocked by warp).  The window's keys lie in
  // [first prefix << pshift, (last prefix + 1) << pshift): the counting sort
  // spreads 2^BBITS buckets over that range (a monotone map of the key).
  const uint64_t kfirst = s.okey[woff] >> psh << psh;
  const uint64_t klast = s.okey[woff + W - 1] | ((1ull << psh) - 1ull);
  const uint64_t span = klast - kfirst;
  const int sbits = span ? 64 - __clzll((long long)span) : 0;
  const int s0 = max(sbits - 32, 0);                          // (key - kfirst) >> s0 fits 32 bits
  const int bsh = max(min(sbits, 32) - kLocalBucketBits, 0);  // then >> bsh: the bucket
  // (an item's window position wbase + 32 q and its bucket are recomputed
  // where needed instead of held in registers: 64 registers at 2 CTAs / SM)
  uint64_t k[LF_ITEMS];
  uint32_t x[LF_ITEMS];
  auto bucket_of = [&](uint64_t key) { return (uint32_t)((key - kfirst) >> s0) >> bsh; };
#pragma unroll
  for (int q = 0; q < LF_ITEMS; ++q) {
    const int idx = wbase + q * 32;
    k[q] = ~0ull;
    if (q < ipw && idx < W) {
      k[q] = s.okey[woff + idx];
      atomicAdd(&s.u.cs.cnt[bucket_of(k[q])], 1u);
    }
  }
  __syncthreads();
  constexpr int BPT = NB / LF_BLOCK;  // buckets per thread (consecutive)
  uint32_t c[BPT], sum = 0, mx = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    c[q] = s.u.cs.cnt[tid * BPT + q];
    sum += c[q];
    mx = max(mx, c[q]);
  }
  mx = __reduce_max_sync(kFull, mx);
  if (lane == 0 && mx > (uint32_t)kLocalBucketMax) atomicMax(&s.maxb, mx);
  uint32_t tot;
  uint32_t run = block_excl_sum<LF_BLOCK>(sum, s.scan, &tot);
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    s.u.cs.cnt[tid * BPT + q] = run;  // bucket start
    s.u.cs.cur[tid * BPT + q] = run;
    run += c[q];
  }
  __syncthreads();
  if (s.maxb == 0) {
    // ---- scatter into the buckets (order-free), then every item's slot is
    // its bucket start + the bucket members below it in (key, position) order
#pragma unroll
    for (int q = 0; q < LF_ITEMS; ++q) {
      if (q < ipw && wbase + q * 32 < W) {
        const uint32_t p = atomicAdd(&s.u.cs.cur[bucket_of(k[q])], 1u);
        s.okey[p] = k[q];
        s.oidx[p] = (uint16_t)(wbase + q * 32);
      }
    }
    __syncthreads();
    uint32_t pos[LF_ITEMS];
#pragma unroll
    for (int q = 0; q < LF_ITEMS; ++q) {
      if (q < ipw && wbase + q * 32 < W) {
        const uint32_t bq = bucket_of(k[q]), xq = (uint32_t)(wbase + q * 32);
        const int b0 = (int)s.u.cs.cnt[bq], b1 = (int)s.u.cs.cur[bq];
        uint32_t r = 0;
        if (b1 - b0 > 1) {
          for (int j = b0; j < b1; ++j) {
            const uint64_t kj = s.okey[j];
            r += kj < k[q] || (kj == k[q] && s.oidx[j] < xq);
          }
        }
        pos[q] = (uint32_t)b0 + r;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < LF_ITEMS; ++q) {
      if (q < ipw && wbase + q * 32 < W) {
        s.okey[pos[q]] = k[q];
        s.oidx[pos[q]] = (uint16_t)(wbase + q * 32);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < LF_ITEMS; ++q) {
      const int idx = wbase + q * 32;
      if (q < ipw) {
        k[q] = s.okey[idx];
        x[q] = s.oidx[idx];
      }
    }
  } else {
    // ---- clustered window: stable 8-bit LSD passes over the bits that
    // vary in it; padding keys (all ones) stay behind the window's items
#pragma unroll
    for (int q = 0; q < LF_ITEMS; ++q) x[q] = (uint32_t)(wbase + q * 32);
    uint64_t ka = ~0ull, ko = 0ull;
#pragma unroll
    for (int q = 0; q < LF_ITEMS; ++q) {
      if (q < ipw && wbase + q * 32 < W) {
        ka &= k[q];
        ko |= k[q];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ka &= __shfl_xor_sync(kFull, ka, o);
      ko |= __shfl_xor_sync(kFull, ko, o);
    }
    if (lane == 0) {
      s.red[0][warp] = ka;
      s.red[1][warp] = ko;
    }
    for (int b = tid; b < NW * R; b += LF_BLOCK) (&s.u.lsd.whist[0][0])[b] = 0;
    __syncthreads();
    uint64_t va = ~0ull, vo = 0ull;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      va &= s.red[0][w];
      vo |= s.red[1][w];
    }
    const uint64_t var = va ^ vo;
    const int lob = var ? __ffsll((long long)var) - 1 : 64;
    const int hib = var ? 63 - __clzll((long long)var) : -1;
    const uint32_t lt = lanemask_lt();
    for (int sh = lob; sh <= hib; sh += kRadixBits) {
      uint32_t rk[LF_ITEMS];
#pragma unroll
      for (int q = 0; q < LF_ITEMS; ++q)
        if (q < ipw)
          rk[q] = warp_rank<true, kRadixBits>(s.u.lsd.whist[warp], digit_of(k[q], sh), true, lane, lt, true);
      __syncthreads();
      uint32_t cc = 0;
      if (tid < R) {
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const uint32_t y = s.u.lsd.whist[w][tid];
          s.u.lsd.whist[w][tid] = cc;
          cc += y;
        }
      }
      uint32_t t2;
      const uint32_t ls = block_excl_sum<LF_BLOCK>(tid < R ? cc : 0u, s.scan, &t2);
      if (tid < R) s.u.lsd.lstart[tid] = ls;
      __syncthreads();
#pragma unroll
      for (int q = 0; q < LF_ITEMS; ++q) {
        if (q < ipw) {
          const uint32_t d = digit_of(k[q], sh);
          const uint32_t p = s.u.lsd.lstart[d] + s.u.lsd.whist[warp][d] + rk[q];
          s.okey[p] = k[q];
          s.oidx[p] = (uint16_t)x[q];
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < LF_ITEMS; ++q) {
        if (q < ipw) {
          const int idx = wbase + q * 32;
          k[q] = s.okey[idx];
          x[q] = s.oidx[idx];
        }
      }
      for (int b = tid; b < NW * R; b += LF_BLOCK) (&s.u.lsd.whist[0][0])[b] = 0;
      __syncthreads();
    }
  }
  // ---- window position idx -> global rank start + idx (payload from the
  // window's 12-B records, L2-resident)
  const uint32_t* pw = a.pay + 3 * start;
  if (em.scount) {
    for (int b = tid; b < 256; b += LF_BLOCK) s.shist[b] = 0;
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < LF_ITEMS; ++q) {
    const int idx = wbase + q * 32;
    if (q < ipw && idx < W) {
      const uint32_t* p = pw + 3 * x[q];
      const uint32_t eu = __ldg(p + 1), ev = __ldg(p + 2);
      em.put((uint32_t)(start + idx), k[q], __ldg(p), eu, ev);
      if (em.scount) {
        atomicAdd(&s.shist[eu >> em.sshift], 1u);
        atomicAdd(&s.shist[ev >> em.sshift], 1u);
      }
    }
  }
  if (em.scount) {  // the sliced maxIncident of view 0 needs no histogram pass
    __syncthreads();
    for (int b = tid; b < 256; b += LF_BLOCK)
      if (s.shist[b]) atomicAdd(em.scount + b, s.shist[b]);
  }
}

}  // namespace dmst

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
// A dendrogram's parents are heavier edges (smaller ranks) or ROOT; anything
// else (a corrupt file) is flagged instead of being followed out of bounds.
__global__ void k_depth_init(const int32_t* __restrict__ parent, int64_t n, int2* __restrict__ ad,
                             uint32_t* __restrict__ bad) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  int32_t p = parent[e];
  if (p < -1 || p >= e) {
    atomicOr(bad, 1u);
    p = -1;
  }
  ad[e] = make_int2(p, 1);
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

namespace dmst {

// ------------------------------------------ dendrogram text format v1
// write_dendrogram (dendro_io.py:28-38): "E <rank> <parent>\n" for every
// edge, then "V <id> <parent>\n" for every vertex, formatted on the device:
// line lengths -> per-block totals -> one scan of the block totals -> every
// block re-derives its lines' offsets and writes them into a byte buffer.
constexpr int FMT_BLOCK = 256, FMT_ITEMS = 8, FMT_TILE = FMT_BLOCK * FMT_ITEMS;
constexpr int FMT_MAXLINE = 24;  // "E 536870911 536870910\n" is 22 bytes (ids < 2^29)

__device__ __forceinline__ int dec_len(int64_t x) {  // characters of %d
  int len = x < 0 ? 2 : 1;
  uint64_t a = x < 0 ? (uint64_t)(-x) : (uint64_t)x;
  while (a >= 10) {
    a /= 10;
    ++len;
  }
  return len;
}

__device__ __forceinline__ char* put_dec(char* p, int64_t x) {
  if (x < 0) {
    *p++ = '-';
    x = -x;
  }
  char tmp[20];
  int k = 0;
  uint64_t a = (uint64_t)x;
  do {
    tmp[k++] = (char)('0' + a % 10);
    a /= 10;
  } while (a);
  while (k) *p++ = tmp[--k];
  return p;
}

// line i < n: edge i; else vertex i - n
__device__ __forceinline__ int fmt_line_len(int64_t i, int64_t n, const int32_t* ep, const int32_t* vp) {
  const bool edge = i < n;
  const int64_t id = edge ? i : i - n;
  const int32_t par = edge ? ep[id] : vp[id];
  return 2 + dec_len(id) + 1 + dec_len(par) + 1;  // "E " id " " parent "\n"
}

__global__ void __launch_bounds__(FMT_BLOCK) k_fmt_count(int64_t n, int64_t nv, const int32_t* __restrict__ ep,
                                                         const int32_t* __restrict__ vp,
                                                         unsigned long long* __restrict__ block_len) {
  const int64_t lines = n + nv;
  const int64_t base = (int64_t)blockIdx.x * FMT_TILE;
  uint32_t s = 0;
  for (int q = 0; q < FMT_ITEMS; ++q) {
    const int64_t i = base + (int64_t)q * FMT_BLOCK + threadIdx.x;
    if (i < lines) s += fmt_line_len(i, n, ep, vp);
  }
  s = __reduce_add_sync(kFull, s);
  __shared__ uint32_t ws[FMT_BLOCK / 32];
  if (lane_id() == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < FMT_BLOCK / 32; ++w) t += ws[w];
    block_len[blockIdx.x] = t;
  }
}

// One block: exclusive scan of the block totals (64-bit), in place; the
// grand total goes to block_len[nb].
__global__ void __launch_bounds__(1024) k_fmt_scan(unsigned long long* block_len, int64_t nb) {
  __shared__ unsigned long long carry;
  __shared__ unsigned long long wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
    const int64_t b = b0 + threadIdx.x;
    const unsigned long long x = b < nb ? block_len[b] : 0ull;
    unsigned long long incl = x;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(kFull, incl, o);
      if ((int)lane_id() >= o) incl += y;
    }
    if (lane_id() == 31) wsum[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
      unsigned long long v = wsum[threadIdx.x], iv = v;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(kFull, iv, o);
        if ((int)threadIdx.x >= o) iv += y;
      }
      wsum[threadIdx.x] = iv - v;
    }
    __syncthreads();
    const unsigned long long excl = carry + wsum[threadIdx.x >> 5] + incl - x;
    if (b < nb) block_len[b] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) block_len[nb] = carry;
}

__global__ void __launch_bounds__(FMT_BLOCK) k_fmt_write(int64_t n, int64_t nv, const int32_t* __restrict__ ep,
                                                         const int32_t* __restrict__ vp,
                                                         const unsigned long long* __restrict__ block_off,
                                                         char* __restrict__ out) {
  // the block's lines are formatted into shared memory, then copied out as
  // one contiguous byte run (consecutive threads -> consecutive bytes)
  extern __shared__ char txt[];  // [FMT_TILE * FMT_MAXLINE]
  const int64_t lines = n + nv;
  const int64_t base = (int64_t)blockIdx.x * FMT_TILE;
  const int64_t first = base + (int64_t)threadIdx.x * FMT_ITEMS;  // contiguous lines per thread
  uint32_t mine = 0;
  for (int q = 0; q < FMT_ITEMS; ++q)
    if (first + q < lines) mine += fmt_line_len(first + q, n, ep, vp);
  __shared__ uint32_t scratch[FMT_BLOCK / 32 + 1];
  uint32_t tot;
  const uint32_t excl = block_excl_sum<FMT_BLOCK>(mine, scratch, &tot);
  char* p = txt + excl;
  for (int q = 0; q < FMT_ITEMS; ++q) {
    const int64_t i = first + q;
    if (i >= lines) break;
    const bool edge = i < n;
    const int64_t id = edge ? i : i - n;
    *p++ = edge ? 'E' : 'V';
    *p++ = ' ';
    p = put_dec(p, id);
    *p++ = ' ';
    p = put_dec(p, edge ? ep[id] : vp[id]);
    *p++ = '\n';
  }
  __syncthreads();
  char* dst = out + block_off[blockIdx.x];
  for (uint32_t b = threadIdx.x; b < tot; b += FMT_BLOCK) dst[b] = txt[b];
}

}  // namespace dmst

namespace dmst {

// --------------------------------------- dendrogram text format v1 reader
// read_dendrogram (dendro_io.py:41-75) for the body after the header line:
// one thread per 32-byte chunk finds the line starts inside it (a line
// starts after each '\n'), counts them per block, and after one scan of the
// block counts every block parses its lines ("E <rank> <parent>" /
// "V <id> <parent>", blank and '#' lines skipped) straight into the arrays.
// err[0] = 0-based line number of the first malformed line (+1), err[1..2]
// = E / V line counts.
constexpr int PARSE_BLOCK = 256, PARSE_CHUNK = 32, PARSE_TILE = PARSE_BLOCK * PARSE_CHUNK;

__device__ __forceinline__ bool line_start(const char* b, int64_t i) { return i == 0 || b[i - 1] == '\n'; }

__global__ void __launch_bounds__(PARSE_BLOCK) k_parse_count(const char* __restrict__ body, int64_t len,
                                                             unsigned long long* __restrict__ block_lines) {
  const int64_t beg = (int64_t)blockIdx.x * PARSE_TILE + (int64_t)threadIdx.x * PARSE_CHUNK;
  uint32_t c = 0;
  for (int q = 0; q < PARSE_CHUNK; ++q) {
    const int64_t i = beg + q;
    if (i < len && line_start(body, i)) ++c;
  }
  c = __reduce_add_sync(kFull, c);
  __shared__ uint32_t ws[PARSE_BLOCK / 32];
  if (lane_id() == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < PARSE_BLOCK / 32; ++w) t += ws[w];
    block_lines[blockIdx.x] = t;
  }
}

__device__ __forceinline__ bool parse_int(const char* b, int64_t len, int64_t& i, int64_t& v) {
  bool neg = false;
  if (i < len && b[i] == '-') {
    neg = true;
    ++i;
  }
  const int64_t s = i;
  int64_t x = 0;
  while (i < len && b[i] >= '0' && b[i] <= '9' && i - s < 18) x = x * 10 + (b[i++] - '0');
  if (i == s) return false;
  v = neg ? -x : x;
  return true;
}

__global__ void __launch_bounds__(PARSE_BLOCK) k_parse_lines(const char* __restrict__ body, int64_t len,
                                                             const unsigned long long* __restrict__ block_off,
                                                             int64_t n, int64_t nv,
                                                             unsigned long long* __restrict__ last,
                                                             unsigned long long* __restrict__ err) {
  const int64_t beg = (int64_t)blockIdx.x * PARSE_TILE + (int64_t)threadIdx.x * PARSE_CHUNK;
  uint32_t mine = 0;
  for (int q = 0; q < PARSE_CHUNK; ++q) {
    const int64_t i = beg + q;
    if (i < len && line_start(body, i)) ++mine;
  }
  __shared__ uint32_t scratch[PARSE_BLOCK / 32 + 1];
  uint32_t tot;
  uint64_t line = block_off[blockIdx.x] + block_excl_sum<PARSE_BLOCK>(mine, scratch, &tot);
  uint32_t ne = 0, nvv = 0;
  unsigned long long bad = ~0ull;
  for (int q = 0; q < PARSE_CHUNK; ++q) {
    int64_t i = beg + q;
    if (i >= len || !line_start(body, i)) continue;
    const uint64_t ln = line++;
    const char k = body[i];
    if (k == '\n' || k == '#') continue;  // blank / comment line
    bool ok = (k == 'E' || k == 'V') && i + 1 < len && body[i + 1] == ' ';
    int64_t id = 0, par = 0;
    if (ok) {
      i += 2;
      ok = parse_int(body, len, i, id) && i < len && body[i] == ' ';
    }
    if (ok) {
      ++i;
      ok = parse_int(body, len, i, par) && (i == len || body[i] == '\n');
    }
    if (ok) ok = id >= 0 && id < (k == 'E' ? n : nv) && par >= INT32_MIN && par <= INT32_MAX;
    if (!ok) {
      bad = min(bad, (unsigned long long)ln);
      continue;
    }
    // duplicate ids: the last line wins, as in the reference's sequential
    // assignment (dendro_io.py:60-66): keep the max of (line, parent)
    atomicMax(&last[k == 'E' ? id : n + id], ((ln + 1) << 32) | (uint32_t)(int32_t)par);
    if (k == 'E')
      ++ne;
    else
      ++nvv;
  }
  if (bad != ~0ull) atomicMin(err, bad + 1);
  ne = __reduce_add_sync(kFull, ne);
  nvv = __reduce_add_sync(kFull, nvv);
  if (lane_id() == 0) {
    if (ne) atomicAdd(err + 1, (unsigned long long)ne);
    if (nvv) atomicAdd(err + 2, (unsigned long long)nvv);
  }
}

// (line + 1, parent) of the last line per id -> parents (ROOT where none).
__global__ void k_parse_finish(const unsigned long long* __restrict__ last, int64_t n, int64_t nv,
                               int32_t* __restrict__ ep, int32_t* __restrict__ vp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n + nv) return;
  const unsigned long long x = last[i];
  const int32_t p = x ? (int32_t)(uint32_t)x : -1;
  if (i < n)
    ep[i] = p;
  else
    vp[i - n] = p;
}

// First index where two int32 arrays differ (atomicMin), for `verify`.
__global__ void k_first_diff(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n,
                             unsigned long long* __restrict__ first) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool d = i < n && a[i] != b[i];
  const uint32_t m = __ballot_sync(kFull, d);
  if (m && lane_id() == (uint32_t)(__ffs(m) - 1)) atomicMin(first, (unsigned long long)i);
}

}  // namespace dmst

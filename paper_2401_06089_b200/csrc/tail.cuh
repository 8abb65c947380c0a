// Device-resident tail of the contraction level loop.  Once a view is small
// (<= kTailEdges edges) every remaining level runs inside ONE cooperative
// kernel with grid-wide barriers between its phases, instead of ~8 launches,
// a few memsets and a host synchronisation per level (~55 us per level of
// launch and sync latency on views whose work is a few microseconds).  The
// phases are the same computations as the big-view kernels (k_v1,
// k_leafscan, k_v2 + k_jump, k_select_edges, k_retire_all), restated for a
// grid-stride cooperative grid.  Reference: build_hierarchy and friends,
// contraction.py:149-219 (paths under /root/reference/pkg/src/dendromst/).
#pragma once
#include <cooperative_groups.h>
#include "kernels.cuh"

namespace dmst {

constexpr int64_t kTailEdges = 1 << 22;  // views at most this large run in k_tail
constexpr int TAIL_BLOCK = 512;
constexpr int TAIL_CAP = 64;             // chase steps before pointer jumping takes over

struct TailArgs {
  uint32_t* cnt2;
  uint2* kw;
  uint32_t* apre;
  int2* euv[2];
  int32_t* grank[2];
  unsigned long long* mi64[2];
  int32_t* smi_all;
  int2* lvl_all;
  int8_t* ret;
  uint32_t* scratch;      // [3 * gridDim + 8]: per-block sums, round counters
  int64_t* soff_out;      // [DMST_MAX_LEVELS + 2] soff of views level0 + 1 .. L + 1
  int32_t* counts_out;    // [DMST_MAX_LEVELS + 1][5]: (n_alpha, n_leaf, n_chain, n_k, nv_k)
  int32_t* result;        // [0] = L, [1] = pointer-jumping rounds
  int level0, cur0;
  int64_t n0, nv0, soff_k0, soff0;  // first view: sizes, its table offset, next free offset
};

// Block-wide sum (all threads get the total).
__device__ __forceinline__ uint32_t tail_block_sum(uint32_t x, uint32_t* sh) {
  x = __reduce_add_sync(kFull, x);
  __syncthreads();
  if (lane_id() == 0) sh[threadIdx.x >> 5] = x;
  __syncthreads();
  uint32_t t = 0;
  for (int i = 0; i < TAIL_BLOCK / 32; ++i) t += sh[i];
  return t;
}

__global__ void __launch_bounds__(TAIL_BLOCK) k_tail(const __grid_constant__ TailArgs t) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t sh[TAIL_BLOCK / 32];
  __shared__ uint32_t sh2w[TAIL_BLOCK / 32 + 1];
  const int64_t gtid = (int64_t)blockIdx.x * TAIL_BLOCK + threadIdx.x;
  const int64_t gsz = (int64_t)gridDim.x * TAIL_BLOCK;
  const uint32_t G = gridDim.x;
  uint32_t* bs = t.scratch;                // [3][G]
  uint32_t* rounds = t.scratch + 3 * G;    // [4] rotating unresolved counters
  int cur = t.cur0, level = t.level0, jumps = 0;
  int64_t n_k = t.n0, nv_k = t.nv0, soff_k = t.soff_k0, soff = t.soff0;
  const uint64_t pol = l2_keep_policy();
  while (true) {
    const int2* euv = t.euv[cur];
    const int32_t* grank = t.grank[cur];
    const unsigned long long* mi = t.mi64[cur];
    int32_t* smi = t.smi_all + soff_k;
    int2* lvl = t.lvl_all + soff_k;
    int32_t* vm = reinterpret_cast<int32_t*>(lvl);  // stride 2
    // ---- V1 (k_v1): maxIncident in global ranks + 2-bit child counts
    for (int64_t x = gtid; x < nv_k; x += gsz) {
      const unsigned long long m = mi[x];
      const uint32_t j1 = (uint32_t)(m >> 32);
      int32_t par = -1;
      if (j1) {
        const uint32_t j = j1 - 1;
        par = grank[j];
        atomicAdd(t.cnt2 + (j >> 4), 1u << ((j & 15) * 2));
      }
      smi[x] = par;
    }
    if (gtid < 4) rounds[gtid] = 0;
    grid.sync();
    // ---- leafscan (k_leafscan): per-block sums, then per-block prefixes
    const int64_t words = n_k / 16 + 1;
    const int64_t per = (words + G - 1) / G;
    const int64_t wb = (int64_t)blockIdx.x * per, we = min(words, wb + per);
    const int64_t tper = (per + TAIL_BLOCK - 1) / TAIL_BLOCK;
    const int64_t tb = wb + (int64_t)threadIdx.x * tper, te = min(we, tb + tper);
    uint32_t ls = 0, as = 0, cs = 0;
    for (int64_t wd = tb; wd < te; ++wd) {
      const uint32_t w = t.cnt2[wd];
      ls += __popc(leaf_bits(w));
      as += __popc(alpha_bits(w, wd, n_k));
      cs += __popc(chain_bits(w));
    }
    {
      const uint32_t bl = tail_block_sum(ls, sh), ba = tail_block_sum(as, sh), bc = tail_block_sum(cs, sh);
      if (threadIdx.x == 0) {
        bs[blockIdx.x] = bl;
        bs[G + blockIdx.x] = ba;
        bs[2 * G + blockIdx.x] = bc;
      }
    }
    grid.sync();
    uint32_t lpre = 0, apre = 0, n_leaf = 0, n_chain = 0;
    {
      uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      for (uint32_t b = threadIdx.x; b < G; b += TAIL_BLOCK) {
        if (b < blockIdx.x) {
          a0 += bs[b];
          a1 += bs[G + b];
        }
        a2 += bs[b];
        a3 += bs[2 * G + b];
      }
      lpre = tail_block_sum(a0, sh);
      apre = tail_block_sum(a1, sh);
      n_leaf = tail_block_sum(a2, sh);
      n_chain = tail_block_sum(a3, sh);
    }
    // exclusive scan of the per-thread (leaf, alpha) sums inside the block
    {
      uint32_t tot;
      uint32_t lr = lpre + block_excl_sum<TAIL_BLOCK>(ls, sh2w, &tot);
      uint32_t ar = apre + block_excl_sum<TAIL_BLOCK>(as, sh2w, &tot);
      for (int64_t wd = tb; wd < te; ++wd) {
        const uint32_t w = t.cnt2[wd];
        t.kw[wd] = make_uint2(w, lr);
        t.apre[wd] = ar;
        lr += __popc(leaf_bits(w));
        ar += __popc(alpha_bits(w, wd, n_k));
      }
    }
    grid.sync();
    // ---- V2 (k_v2): chase to the leaf edge; long chases left as ~vertex
    for (int64_t x = gtid; x < nv_k; x += gsz) {
      unsigned long long m = mi[x];
      uint32_t j = (uint32_t)(m >> 32) - 1u, y = (uint32_t)m;
      uint2 kwj = make_uint2(0, 0);
      bool unres = false;
      int s = 0;
      while (m != 0ull) {
        kwj = ld_keep2(t.kw + (j >> 4), pol);
        if (((kwj.x >> ((j & 15) * 2)) & 3u) == 2u) break;
        if (++s > TAIL_CAP) {
          unres = true;
          break;
        }
        m = mi[y];
        j = (uint32_t)(m >> 32) - 1u;
        y = (uint32_t)m;
      }
      const int32_t lab = unres ? ~(int32_t)y : (m ? (int32_t)leaf_label(kwj, j) : 0);
      lvl[x] = make_int2(lab, smi[x]);
      if (unres) atomicAdd(rounds, 1u);
    }
    grid.sync();
    // ---- pointer jumping (k_jump) until every vertex has a label
    for (int r = 0; *(volatile uint32_t*)(rounds + (r & 3)) != 0; ++r) {
      if (gtid == 0) rounds[(r + 2) & 3] = 0;
      for (int64_t x = gtid; x < nv_k; x += gsz) {
        const int32_t p = vm[2 * x];
        if (p < 0) {
          const int32_t q = vm[2 * (int64_t)~p];
          vm[2 * x] = q;
          if (q < 0) atomicAdd(rounds + ((r + 1) & 3), 1u);
        }
      }
      ++jumps;
      grid.sync();
    }
    const int64_t n_alpha = n_k - (int64_t)n_leaf - (int64_t)n_chain;
    if (gtid == 0) {
      int32_t* co = t.counts_out + 5 * level;
      co[0] = (int32_t)n_alpha;
      co[1] = (int32_t)n_leaf;
      co[2] = (int32_t)n_chain;
      co[3] = (int32_t)n_k;
      co[4] = (int32_t)nv_k;
    }
    if (level >= 1 && n_alpha == 0) {  // contraction.py:203-205
      for (int64_t j = gtid; j < n_k; j += gsz) t.ret[grank[j]] = (int8_t)level;
      if (gtid == 0) {
        t.result[0] = level;
        t.result[1] = jumps;
        t.soff_out[level + 1] = soff;
      }
      return;
    }
    // ---- next view (k_select_edges, direct maxIncident)
    const int64_t nv_next = n_leaf, n_next = n_alpha;
    unsigned long long* mi_next = t.mi64[cur ^ 1];
    int2* euv_next = t.euv[cur ^ 1];
    int32_t* grank_next = t.grank[cur ^ 1];
    for (int64_t x = gtid; x < nv_next; x += gsz) mi_next[x] = 0ull;
    const int64_t soff_next = soff;
    soff += nv_next;
    if (gtid == 0) t.soff_out[level + 1] = soff_next;
    grid.sync();
    for (int64_t j = gtid; j < n_k; j += gsz) {
      const uint2 w = t.kw[j >> 4];
      const uint32_t sh2 = (uint32_t)(j & 15) * 2;
      const uint32_t c = (w.x >> sh2) & 3u;
      const int32_t g = grank[j];
      if ((j & 15) == 0) t.cnt2[j >> 4] = 0u;
      if (c != 0u) {
        t.ret[g] = (int8_t)level;
      } else {
        const uint32_t pos = t.apre[j >> 4] + __popc(alpha_bits(w.x, 0, 16) & ((1u << sh2) - 1u));
        const int2 e = euv[j];
        const int32_t a = vm[2 * (int64_t)e.x], b = vm[2 * (int64_t)e.y];
        euv_next[pos] = make_int2(a, b);
        grank_next[pos] = g;
        atomicMax(mi_next + a, pack_mi(pos + 1u, (uint32_t)b));
        atomicMax(mi_next + b, pack_mi(pos + 1u, (uint32_t)a));
      }
    }
    grid.sync();
    cur ^= 1;
    n_k = n_next;
    nv_k = nv_next;
    soff_k = soff_next;
    ++level;
    if (level >= DMST_MAX_LEVELS) {
      if (gtid == 0) t.result[0] = -1;
      return;
    }
  }
}

}  // namespace dmst

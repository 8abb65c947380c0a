// B200-native PANDORA dendrogram construction: host orchestration + C ABI.
//
// Pipeline (one stream, all buffers caller-owned), with the reference
// symbol each stage replaces (paths under /root/reference/pkg/src/dendromst/):
//
//  1. edge sort        rank_edges            tree_core.py:174-190
//     k_sort1_hist, then per non-constant digit k_upsweep -> row scans ->
//     k_downsweep (radix.cuh).
//     Key = order-preserving uint64 of (w + 0.0), descending; payload =
//     (original id, u, v) so the last pass writes orig_of, heights (decoded
//     from the key) and rank-order endpoints without random gathers.
//  2. maxIncident      build_incidence       tree_core.py:193-199
//     records (x, rank, other end) grouped by 8192-vertex bucket with two
//     order-free multisplit passes (bucket.cuh), then reduced per bucket in
//     shared memory (k_mi_apply_smem, fused with V1).
//  3. contraction      build_hierarchy       contraction.py:186-219
//     per view k: k_v1 (maxIncident + 2-bit child counts), k_leafscan
//     (leaf-edge numbering = supervertex ids), k_v2 (chase to the leaf
//     edge; k_jump rounds for deep in-trees), k_select_edges
//     (retirement, alpha-edge compaction into view k+1).
//  4. expansion        assign_chains         expansion.py:97-128
//     k_walk: per edge, the level walk -> dense chain key (+ digit histogram)
//  5. chain sort+link  stitch_chains         expansion.py:131-145
//     stable radix sort on the chain key (payload = rank), k_link.
#include <algorithm>
#include <cstdio>
#include <mutex>
#include <unordered_map>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "validate.cuh"
#include "tail.cuh"
#include "emst.cuh"

namespace dmst {

// ----------------------------------------------------------------- config
// Radix sort geometry (sub-tile = BLOCK x ITEMS items; MINB CTAs per SM).
// Edge sort: u64 key + 3-word payload.
constexpr int S1_BLOCK = 512, S1_ITEMS = 8, S1_MINB = 1;
// narrow (32-bit) keys: 256-thread CTAs, two per SM, 12-item tiles
constexpr int S1N_BLOCK = 256, S1N_MINB = 2;
constexpr int S1N_ITEMS = 12;
// the fused first upsweep counts before the key width is known: its chunk
// geometry (S1N_MINB chunks per SM, multiples of S1_ALIGN) is shared by the
// first pass of either width (the wide one then runs in two waves)
constexpr int64_t S1_ALIGN = 12288;
static_assert(S1_ALIGN % (S1_BLOCK * S1_ITEMS) == 0 && S1_ALIGN % (S1N_BLOCK * S1N_ITEMS) == 0, "S1_ALIGN");
// Chain sort: u32 key + 1-word payload.
constexpr int S2_BLOCK = 512, S2_ITEMS = 16, S2_MINB = 1, S2_BITS = 9;
// large trees: 256-thread CTAs, two per SM, 20-item tiles (2.36 -> 2.25 ms at
// 128M); small trees, often several per GPU on concurrent streams, keep the
// fewer, larger chunks of one CTA per SM (config 5: 129 -> 124 ms)
constexpr int S2L_BLOCK = 256, S2L_ITEMS = 20, S2L_MINB = 2;
constexpr int64_t kS2LargeEdges = 32ll << 20;
constexpr int64_t kDirectMiBytes = 64ll << 20;  // direct scatter-max below this mi64 size

#ifndef DMST_LINK_SLICE_BITS
#define DMST_LINK_SLICE_BITS kSliceBits  // link: ranks per L2-resident slice of edge_parent (2M = 8 MB; 4M / 8M: +0.1-0.2 ms)
#endif
#ifndef DMST_V2_KEEP_BYTES
// V2 chase hops keep the maxIncident table in L2 (normal policy) up to this
// size, ~4x L2 (measured: config 4's view 1, 268 MB, and every config-5 view
// gain; view 0 of config 4, 1 GB, is chased in the select instead)
#define DMST_V2_KEEP_BYTES (512ll << 20)
#endif

enum KernelKind {
  KK_SORT1_HIST, KK_SORT1_FIRST, KK_SORT1_MID, KK_SORT1_FINAL, KK_MI_HIST, KK_MI_SPLIT_A, KK_MI_SPLIT_B,
  KK_MI_APPLY, KK_V1, KK_LEAFSCAN, KK_V2, KK_JUMP, KK_SELECT_EDGES, KK_WALK, KK_SORT2_PASS, KK_LINK_SPLIT,
  KK_LINK_APPLY, KK_UPSWEEP, KK_TAIL, KK_SORT1_LOCAL, KK_OTHER, KK_COUNT
};
static_assert(KK_COUNT <= DMST_MAX_KERNELS, "kernel kinds");
const char* const kKernelNames[KK_COUNT] = {
    "sort1_hist", "sort1_pass_first", "sort1_pass_mid", "sort1_pass_final", "mi_hist", "mi_split_a",
    "mi_split_b", "mi_apply", "v1", "leafscan", "v2", "jump", "select_edges", "walk", "sort2_pass",
    "link_split", "link_apply", "upsweep_scan", "tail", "sort1_local", "other"};

namespace {

thread_local std::string g_err;

struct Fail {
  int code;
};

#define DMST_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      g_err = std::string(#call) + ": " + cudaGetErrorString(e_);                    \
      throw Fail{DMST_ECUDA};                                                        \
    }                                                                                \
  } while (0)

[[noreturn]] void invalid(const std::string& m) {
  g_err = m;
  throw Fail{DMST_EINVAL};
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }
inline unsigned grid_for(int64_t n, int block) { return (unsigned)std::max<int64_t>(1, cdiv(n, block)); }


// Workspace carve-up; the same code sizes and assigns it.
//  R (48n B): edge sort ping-pong (keys 2x8n, payload 2x3x4n); later
//             maxIncident records (2 x 24n), jump lists, chain-sort buffers.
struct Workspace {
  char* R;
  uint32_t* counts;       // radix per-chunk digit counts [256][kMaxChunks]
  uint32_t* fine;         // bucketing: counts, base, cursors (fine), cursors (coarse)
  uint32_t* small;        // counters/histograms (zeroed per use)
  int2* euv0;             // rank-order endpoints
  unsigned long long* mi64_0;
  unsigned long long* mi64[2];  // views >= 1 (ping-pong)
  uint32_t* cnt2;         // 2-bit child counts per edge (16 per word)
  uint2* kw;              // (cnt2 word, leaf prefix) per 16 edges, for V2
  int8_t* ret;            // retirement level per edge
  int2* euv[2];           // view edges (ping-pong)
  int32_t* grank[2];
  int32_t* vm_all;        // vertex map of view 0
  int2* lvl_all;          // walk table of views 1..L: (vertex map, maxIncident) at soff[k] + x
  int32_t* smi_all;       // maxIncident (global ranks) of views 1..L
  int32_t* x1;            // view-1 supervertex of every edge (walk start)
  uint32_t* sel_status;   // leafscan look-back words (leaf, alpha)
  uint32_t* apre;         // alpha prefix per 16 edges
  uint2* lw;              // (leaf bitmap, leaf prefix) per 32 edges (k_v2)
  size_t bytes;
};

constexpr int kSmallWords = 8 * kRadix /*hist1*/ + 8 * kRadix /*gbase1*/ + 4 * kRadix /*hist2*/ +
                            4 * kRadix /*gbase2*/ + kRadix /*vhist*/ + kRadix /*vbase*/ + 64 /*tile ctrs*/ +
                            256 /*misc*/;
constexpr int SM_HIST1 = 0, SM_GBASE1 = SM_HIST1 + 8 * kRadix, SM_HIST2 = SM_GBASE1 + 8 * kRadix,  // NOLINT
              SM_GBASE2 = SM_HIST2 + 4 * kRadix, SM_VHIST = SM_GBASE2 + 4 * kRadix,
              SM_VBASE = SM_VHIST + kRadix, SM_TILECTR = SM_VBASE + kRadix, SM_MISC = SM_TILECTR + 64;
constexpr int MISC_NEGZERO = 0, MISC_ACTIVE0 = 1, MISC_ACTIVE1 = 2, MISC_ACTIVE2 = 3, MISC_COUNTS = 4 /*2*/,
              MISC_NONRUL = 6, MISC_LSCTR = 13, MISC_LOCALOVF = 16, MISC_SORT1D0 = 17,
              MISC_DEFER = 20;

Workspace carve(int64_t n, int64_t nv, char* base) {
  Workspace w{};
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  const int64_t half = n / 2 + 1;
  w.R = take(48 * n + 4096);
  w.counts = (uint32_t*)take(4 * 1024 * (kMaxChunks + 4));
  w.fine = (uint32_t*)take(4 * (4 * (nv / FB + 2) + 512));
  w.small = (uint32_t*)take(4 * kSmallWords);
  w.euv0 = (int2*)take(8 * n);
  w.mi64_0 = (unsigned long long*)take(8 * nv);
  for (int i = 0; i < 2; ++i) w.mi64[i] = (unsigned long long*)take(8 * (half + 1));
  w.cnt2 = (uint32_t*)take(4 * (n / 16 + 2));
  w.kw = (uint2*)take(8 * (n / 16 + 2));
  w.ret = (int8_t*)take(n);
  for (int i = 0; i < 2; ++i) {
    w.euv[i] = (int2*)take(8 * half);
    w.grank[i] = (int32_t*)take(4 * half);
  }
  w.vm_all = (int32_t*)take(4 * (nv + 2));
  w.lvl_all = (int2*)take(8 * (nv + DMST_MAX_LEVELS + 2));
  w.smi_all = (int32_t*)take(4 * (nv + DMST_MAX_LEVELS + 2));
  w.x1 = (int32_t*)take(4 * (n + 2));
  w.sel_status = (uint32_t*)take(8 * (cdiv(n / 16 + 1, LS_TILE) + 2));
  w.apre = (uint32_t*)take(4 * (n / 16 + 2));
  w.lw = (uint2*)take(8 * (n / 32 + 2));
  w.bytes = off + 256;
  return w;
}

void check_args(int64_t n, int64_t nv, const void* ws, size_t ws_bytes) {
  if (n < 1) invalid("n_edges must be >= 1");
  if (n >= (int64_t(1) << 29)) invalid("n_edges must be < 2^29");
  if (nv != n + 1) invalid("n_vertices must equal n_edges + 1 (a spanning tree)");
  if (!ws) invalid("workspace is null");
  if (ws_bytes < carve(n, nv, nullptr).bytes) invalid("workspace too small");
}

int num_sms() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

// Host-mapped pinned buffer for small readbacks (Ctx::to_host), one per
// (host thread, device): kept for the thread's lifetime, so a thread that
// alternates devices reuses its buffers instead of reallocating them.
struct MappedBuf {
  static constexpr uint32_t kWords = 2048;
  volatile uint32_t* host = nullptr;
  uint32_t* dev = nullptr;
};
MappedBuf& mapped_buf() {
  thread_local std::unordered_map<int, MappedBuf> bufs;
  int dev = 0;
  DMST_CUDA(cudaGetDevice(&dev));
  MappedBuf& mb = bufs[dev];
  if (mb.host == nullptr) {
    void* h = nullptr;
    DMST_CUDA(cudaHostAlloc(&h, 4 * MappedBuf::kWords, cudaHostAllocMapped | cudaHostAllocPortable));
    void* d = nullptr;
    DMST_CUDA(cudaHostGetDevicePointer(&d, h, 0));
    mb.host = (volatile uint32_t*)h;
    mb.dev = (uint32_t*)d;
  }
  return mb;
}

// Thread-local pool of timing events (profiling creates two per launch).
std::vector<cudaEvent_t>& event_pool() {
  thread_local std::vector<cudaEvent_t> pool;
  return pool;
}
cudaEvent_t pooled_event() {
  auto& p = event_pool();
  if (!p.empty()) {
    cudaEvent_t e = p.back();
    p.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  DMST_CUDA(cudaEventCreate(&e));
  return e;
}

// Copies between caller host buffers and the device, overlapped with the
// pipeline on a side stream (dmst_build_host).  Stages signal readiness of
// their outputs with events; the side stream waits on them and copies out.
struct HostIO {
  cudaStream_t side = nullptr;
  int32_t* h_orig = nullptr;
  double* h_heights = nullptr;
  int32_t* h_ep = nullptr;
  int32_t* h_vp = nullptr;
  const int32_t* d_orig = nullptr;
  const double* d_heights = nullptr;
  const int32_t* d_vp = nullptr;
  int64_t n = 0, nv = 0;
  cudaEvent_t ev[4] = {};
};

// Per-call code-path choices (dmst_stats in-fields; 0 there = these defaults)
// and a record of the path taken (dmst_stats out-fields).
struct Paths {
  int64_t tail_edges = kTailEdges;
  int64_t direct_mi_bytes = kDirectMiBytes;
  int sort1_mode = 0;
  int sort2_geometry = 0;
  int mi_apply_mode = 0;  // 0 / 1: shared-memory apply per fine bucket; 2: slices + L2 atomics
  int v0_select = 0;      // 0: by the view's kind counts; 1: V2 + vertex map; 2: chase in the select
  // out
  int v0_chase = 0;       // 1 = view 0's select chased maxIncident (no V2), 2 = and deferred edges
  int sort1_narrow = 0, sort1_compacted = 0, sort2_geometry_used = 0, tail_level = -1;
  int sort1_local = 0;  // 1 = wide keys finished in shared memory, 2 = tried, fell back to full LSD
  int mi_sliced_used = 0;
  uint64_t mi_bucketed = 0, mi_direct = 0;
};

// Per host thread (and device): an auxiliary stream and two events, so a
// table the sliced maxIncident will update can be zeroed while the edge sort
// runs (the sort is bound by shared-memory work, not DRAM).
struct AuxStream {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[3] = {};  // ev[0]: the build's start on the main stream; ev[1], ev[2]: prezero slots done
};
AuxStream& aux_stream() {
  thread_local std::unordered_map<int, AuxStream> m;
  int dev = 0;
  DMST_CUDA(cudaGetDevice(&dev));
  AuxStream& a = m[dev];
  if (!a.s) {
    DMST_CUDA(cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking));
    for (auto& e : a.ev) DMST_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  return a;
}

struct Ctx {
  cudaStream_t s;
  Workspace w;
  struct Prezero {  // a table zeroed on the aux stream (ready after aux ev[1 + slot])
    const void* p = nullptr;
    size_t bytes = 0;
  } pz[2], pz_next;  // pz_next: issue during the next multisplit pass A
  bool aux_marked = false;
  bool slices_counted = false;      // the edge sort counted view 0's endpoints per slice (w.fine)
  int launches = 0;
  int sms = 148;
  bool profile = false;
  HostIO* io = nullptr;
  Paths paths;
  struct Ev {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Ev> ev;
  void begin(int kind) {
    if (!profile) return;
    Ev e{kind, pooled_event(), pooled_event()};
    DMST_CUDA(cudaEventRecord(e.a, s));
    ev.push_back(e);
  }
  void launched() {
    ++launches;
    DMST_CUDA(cudaGetLastError());
    if (profile) DMST_CUDA(cudaEventRecord(ev.back().b, s));
  }
  void collect(dmst_stats* st) {
    if (getenv("DMST_TIMELINE") && !ev.empty()) {  // debugging aid: kernel start/end vs the first event
      float prev_end = 0.f;
      for (Ev& e : ev) {
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, ev[0].a, e.a);
        cudaEventElapsedTime(&b, ev[0].a, e.b);
        fprintf(stderr, "TL %-18s start %9.3f end %9.3f dur %8.3f gap %8.3f\n", kKernelNames[e.kind], a, b, b - a,
                a - prev_end);
        prev_end = b;
      }
    }
    for (Ev& e : ev) {
      float ms = 0.f;
      if (st && cudaEventElapsedTime(&ms, e.a, e.b) == cudaSuccess) {
        st->kernel_ms[e.kind] += ms;
        st->kernel_calls[e.kind] += 1;
      }
    }
    release();
  }
  void release() {
    auto& p = event_pool();
    for (Ev& e : ev) {
      p.push_back(e.a);
      p.push_back(e.b);
    }
    ev.clear();
  }
  ~Ctx() { release(); }
  // host copy-out of an output that is complete on `s` (no-op without HostIO)
  void copy_out(int slot, void* h, const void* d, size_t bytes) {
    if (!io || !h) return;
    DMST_CUDA(cudaEventRecord(io->ev[slot], s));
    DMST_CUDA(cudaStreamWaitEvent(io->side, io->ev[slot], 0));
    DMST_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, io->side));
  }
  // Small device->host reads (level counts, digit masks) go through a
  // host-mapped pinned buffer written by a tiny kernel, not the copy
  // engines: dmst_build_host's multi-GB output copies occupy those, and a
  // queued 8-byte cudaMemcpy would wait behind them.
  struct Pending {
    void* h;
    uint32_t off, bytes;
  };
  std::vector<Pending> pend;
  uint32_t mapped_used = 0;
  void to_host(void* h, const void* d, size_t bytes) {
    MappedBuf& mb = mapped_buf();
    const uint32_t words = (uint32_t)((bytes + 3) / 4);
    if (mapped_used + words > MappedBuf::kWords) invalid("readback buffer overflow");
    k_readback<<<1, 32, 0, s>>>(mb.dev + mapped_used, (const uint32_t*)d, words);
    DMST_CUDA(cudaGetLastError());
    pend.push_back({h, mapped_used, (uint32_t)bytes});
    mapped_used += words;
  }
  void sync() {
    DMST_CUDA(cudaStreamSynchronize(s));
    MappedBuf& mb = mapped_buf();
    for (const Pending& p : pend) memcpy(p.h, (const void*)(mb.host + p.off), p.bytes);
    pend.clear();
    mapped_used = 0;
  }
  void zero(void* d, size_t bytes) { DMST_CUDA(cudaMemsetAsync(d, 0, bytes, s)); }
  void ones(void* d, size_t bytes) { DMST_CUDA(cudaMemsetAsync(d, 0xff, bytes, s)); }
  unsigned persistent_grid(int64_t work, int block, int per_sm) {
    return (unsigned)std::min<int64_t>(grid_for(work, block), (int64_t)sms * per_sm);
  }
};

// Tables a later stage needs zeroed are cleared on the aux stream while the
// main stream runs shared-memory-bound kernels.  mark_aux() records the
// build's start (their last use was in an earlier call on this stream);
// prezero() may then be issued any time later in the build (issue it after a
// long kernel's launch so the memset's blocks share SMs with that kernel, not
// with a tiny one).
void mark_aux(Ctx& c) {
  DMST_CUDA(cudaEventRecord(aux_stream().ev[0], c.s));
  c.aux_marked = true;
}
void prezero(Ctx& c, int slot, void* p, size_t bytes) {
  if (!c.aux_marked) return;  // (zero_for_atomics then memsets in stream order)
  AuxStream& a = aux_stream();
  DMST_CUDA(cudaStreamWaitEvent(a.s, a.ev[0], 0));
  DMST_CUDA(cudaMemsetAsync(p, 0, bytes, a.s));
  DMST_CUDA(cudaEventRecord(a.ev[1 + slot], a.s));
  c.pz[slot].p = p;
  c.pz[slot].bytes = bytes;
}
// c.s waits for every pending prezero (before memory one touched may be reused).
void join_aux(Ctx& c) {
  for (int slot = 0; slot < 2; ++slot)
    if (c.pz[slot].p) {
      DMST_CUDA(cudaStreamWaitEvent(c.s, aux_stream().ev[1 + slot], 0));
      c.pz[slot].p = nullptr;
    }
}
// `bytes` at `p` are zero once c.s reaches this point (prezeroed or memset now).
void zero_for_atomics(Ctx& c, void* p, size_t bytes) {
  for (int slot = 0; slot < 2; ++slot)
    if (c.pz[slot].p == p && bytes <= c.pz[slot].bytes) {
      DMST_CUDA(cudaStreamWaitEvent(c.s, aux_stream().ev[1 + slot], 0));
      c.pz[slot].p = nullptr;
      return;
    }
  c.zero(p, bytes);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and device
// (a host API call per launch would add latency inside the level loop).
template <typename K>
void smem_attr(K* kernel, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> done[64];
  int dev = 0;
  DMST_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = done[dev & 63][(const void*)kernel];
  if (cur < bytes) {
    DMST_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    cur = bytes;
  }
}

// Radix pass geometry: G persistent CTAs, one contiguous chunk each.
struct SweepGeom {
  int64_t G, chunk;
  uint32_t GS;
};
// chunks are multiples of `align` (default T): passes with different tile
// sizes over the same keys then share one chunk geometry
SweepGeom sweep_geom(const Ctx& c, int64_t n, int T, int minb, int64_t align = 0) {
  SweepGeom g;
  const int64_t A = align ? align : T;
  int64_t G = std::min<int64_t>(cdiv(n, A), std::min<int64_t>((int64_t)c.sms * minb, kMaxChunks));
  g.chunk = cdiv(cdiv(n, G), A) * A;
  g.G = cdiv(n, g.chunk);
  g.GS = (uint32_t)((g.G + 3) & ~int64_t(3));
  return g;
}

// One radix pass: upsweep (per-chunk digit counts; skipped when a fused
// upsweep already produced them), chunk scan, downsweep.
template <typename K, int PW, int BLOCK, int ITEMS, int MINB, int BITS, class Loader, class Emitter>
int64_t radix_pass(Ctx& c, int kind, int64_t n, int shift, Loader ld, Emitter em, bool counts_ready = false,
                   int64_t align = 0, int geom_minb = 0) {
  using S = DownSmem<K, PW, BLOCK, ITEMS, Loader, Emitter, BITS>;
  constexpr int T = S::T;
  auto kern = k_downsweep<K, PW, BLOCK, ITEMS, MINB, Loader, Emitter, BITS>;
  smem_attr(kern, (int)S::bytes());
  const SweepGeom g = sweep_geom(c, n, T, geom_minb ? geom_minb : MINB, align);
  SweepArgs a{};
  a.n = n;
  a.shift = shift;
  a.chunk = g.chunk;
  a.G = (uint32_t)g.G;
  a.GS = g.GS;
  a.counts = c.w.counts;
  if (!counts_ready) {
    c.zero(a.counts, 4 * (size_t(1) << BITS) * a.GS);
    c.begin(KK_UPSWEEP);
    k_upsweep<BITS, Loader><<<(unsigned)(g.G * kUpSplit), 256, 0, c.s>>>(a, ld);
    c.launched();
  }
  c.begin(KK_UPSWEEP);
  k_row_scan<BITS><<<(1u << BITS) / kRowScanWarps, 32 * kRowScanWarps, 0, c.s>>>(a.counts, a.GS);
  c.launched();
  c.begin(KK_UPSWEEP);
  k_row_total_scan<BITS><<<1, 1u << BITS, 0, c.s>>>(a.counts, a.GS);
  c.launched();
  c.begin(kind);
  kern<<<(unsigned)g.G, BLOCK, S::bytes(), c.s>>>(a, ld, em);
  c.launched();
  return g.G;
}

// Multi-pass driver over the non-constant digits (bit offsets `shifts`).
// Ping-pong buffers: keys bufK[2], AoS payload bufP[2] (PW words per item);
// first/last passes use the given loader/emitter.
template <typename K, int PW, int BLOCK, int ITEMS, int MINB, int BITS, class FirstLoader, class FinalEmitter>
int64_t run_sort(Ctx& c, const int (&kinds)[3], int64_t n, const std::vector<int>& shifts,
              K* const (&bufK)[2], uint32_t* const (&bufP)[2], FirstLoader first, FinalEmitter final_em,
              int ready_shift = -1, int64_t align = 0, int first_minb = 0) {
  const int P = (int)shifts.size();
  if (P == 0) {
    c.begin(KK_OTHER);
    k_identity_pass<K, PW, EW_BLOCK><<<grid_for(n, EW_BLOCK), EW_BLOCK, 0, c.s>>>(n, first, final_em);
    c.launched();
    return grid_for(n, EW_BLOCK);
  }
  int64_t G = 0;
  for (int p = 0; p < P; ++p) {
    const int o = p % 2, in = o ^ 1;
    ArrayEmitter<K, PW> mid{bufK[o], bufP[o]};
    ArrayLoader<K, PW> ldr{bufK[in], bufP[in]};
    const bool ready = p == 0 && shifts[0] == ready_shift;
    if (P == 1)
      G = radix_pass<K, PW, BLOCK, ITEMS, MINB, BITS>(c, kinds[2], n, shifts[p], first, final_em, ready, align,
                                                      first_minb);
    else if (p == 0)
      G = radix_pass<K, PW, BLOCK, ITEMS, MINB, BITS>(c, kinds[0], n, shifts[p], first, mid, ready, align,
                                                      first_minb);
    else if (p == P - 1)
      G = radix_pass<K, PW, BLOCK, ITEMS, MINB, BITS>(c, kinds[2], n, shifts[p], ldr, final_em, false, align);
    else
      G = radix_pass<K, PW, BLOCK, ITEMS, MINB, BITS>(c, kinds[1], n, shifts[p], ldr, mid, false, align);
  }
  return G;
}

// Radix digits (BITS wide, at bit offsets 0, BITS, ...) that are not
// constant across all keys, from the AND / OR of every key.
std::vector<int> active_digits(uint64_t key_and, uint64_t key_or, int bits, int key_bits) {
  std::vector<int> shifts;
  const uint64_t mask = (1ull << bits) - 1;
  for (int sft = 0; sft < key_bits; sft += bits)
    if (((key_and ^ key_or) >> sft) & mask) shifts.push_back(sft);
  return shifts;
}

// Varying bits of the (compacted) keys: XOR of AND / OR, with the dense
// top-field code's bits when compaction applies.
uint64_t var_of(const unsigned long long (&ao)[2], const uint8_t* code, int ncodes) {
  if (!code) return ao[0] ^ ao[1];
  int cbits = 0;
  while ((1 << cbits) < ncodes) ++cbits;
  return ((ao[0] ^ ao[1]) & kMantMask) | (((1ull << cbits) - 1) << kTopShift);
}

// Sort #1 (rank_edges): orig_of, heights, euv (and/or ru, rv).
void edge_sort(Ctx& c, const int32_t* u, const int32_t* v, const double* w, int64_t n,
               Sort1FinalEmitter em, int* passes_out, void* zero_ptr = nullptr, size_t zero_bytes = 0) {
  unsigned long long* sample_ao = (unsigned long long*)(c.w.small + SM_HIST1);
  unsigned long long* and_or = sample_ao + 2;
  uint32_t* top_min = c.w.small + SM_HIST1 + 8;
  uint32_t* top_bits = c.w.small + SM_HIST1 + 16;                    // 128 words
  uint16_t* top_inv = (uint16_t*)(c.w.small + SM_HIST1 + 144);       // 256 codes
  uint8_t* top_code = (uint8_t*)(c.w.small + SM_HIST1 + 272);        // 4096 fields
  uint32_t* negzero = c.w.small + SM_MISC + MISC_NEGZERO;
  c.ones(sample_ao, 8);  // AND starts all-ones, OR all-zeros (memsets: no pageable copies)
  c.zero(sample_ao + 1, 8);
  c.ones(and_or, 8);
  c.zero(and_or + 1, 8);
  c.ones(top_min, 4);
  c.zero(top_bits, 4 * 128);
  c.zero(negzero, 4);
  // predict the first active digit from a sample, then count it in the same
  // read of w that reduces all keys (k_upsweep<KEYRED>)
  c.begin(KK_SORT1_HIST);
  k_key_sample<<<64, 1024, 0, c.s>>>(w, n, sample_ao, top_min);  // one sample per thread
  c.launched();
  uint32_t* d0_dev = c.w.small + SM_MISC + MISC_SORT1D0;
  const SweepGeom g = sweep_geom(c, n, S1_BLOCK * S1_ITEMS, S1N_MINB, S1_ALIGN);
  SweepArgs a{};
  a.n = n;
  a.shift = 0;  // the KEYRED upsweep predicts its digit from the sample on the device
  a.chunk = g.chunk;
  a.G = (uint32_t)g.G;
  a.GS = g.GS;
  a.counts = c.w.counts;
  c.zero(a.counts, 4 * kRadix * (size_t)a.GS);
  c.begin(KK_SORT1_HIST);
  k_upsweep<8, Sort1FirstLoader, true><<<(unsigned)(g.G * kUpSplit), 256, 0, c.s>>>(
      a, Sort1FirstLoader{w, u, v, nullptr},
      KeyRed{w, and_or, negzero, top_bits, sample_ao, top_min, d0_dev, (c.paths.sort1_mode & 4) ? 0 : 1});
  c.launched();
  unsigned long long ao[2];
  uint32_t nz = 0, tb[128], d0u = 0;
  unsigned long long sao[2];
  c.to_host(&d0u, d0_dev, 4);
  c.to_host(sao, sample_ao, 16);
  c.to_host(ao, and_or, 16);
  c.to_host(&nz, negzero, 4);
  c.to_host(tb, top_bits, sizeof(tb));
  c.sync();
  const int d0 = (int)d0u;  // = predict_first_digit(sample AND, OR)
  const bool local_guess = !(c.paths.sort1_mode & 4) && active_digits(sao[0], sao[1], 8, 64).size() >= 5;
  std::vector<int> shifts = active_digits(ao[0], ao[1], 8, 64);
  // top-field compaction when it saves a pass: (code, mantissa) keys
  int ncodes = 0;
  for (uint32_t x : tb) ncodes += __builtin_popcount(x);
  const uint8_t* code = nullptr;
  if (ncodes > 1 && ncodes <= 256 && !(c.paths.sort1_mode & 2)) {
    int cbits = 0;
    while ((1 << cbits) < ncodes) ++cbits;
    const uint64_t cand = ao[0] & kMantMask, cor = (ao[1] & kMantMask) | (((1ull << cbits) - 1) << kTopShift);
    std::vector<int> cs = active_digits(cand, cor, 8, 64);
    if (cs.size() < shifts.size()) {
      c.begin(KK_OTHER);
      k_top_codes<<<1, 128, 0, c.s>>>(top_bits, top_code, top_inv);
      c.launched();
      code = top_code;
      em.inv = top_inv;
      shifts = cs;
      c.paths.sort1_compacted = 1;
    }
  }
  // the upsweep counted digit d0 of the raw keys: valid for the compacted
  // keys only below the top field
  const bool local = shifts.size() >= 5 && !(c.paths.sort1_mode & 4);
  // (local: the three global digits [t0, t0 + 24) must cover the highest
  // varying bit; t0 = the fused upsweep's digit when it does)
  const int hb_full = shifts.empty() ? 0 : 63 - __builtin_clzll(var_of(ao, code, ncodes));
  const int first_shift = shifts.empty() ? -1
                          : local        ? (local_guess && hb_full <= d0 + 23 ? d0 : std::max(hb_full - 23, 0))
                                         : shifts[0];
  const int ready = first_shift >= 0 && first_shift == d0 && (!code || d0 + 8 <= kTopShift) ? d0 : -1;
  if (passes_out) *passes_out = (int)shifts.size();
  char* R = c.w.R;
  uint32_t* vb = (uint32_t*)(R + 16 * n);
  uint32_t* const bufP[2] = {vb, vb + 3 * n};
  // narrow keys: every varying bit of the (compacted) key within 32 bits
  // from lo (= the first digit, so the fused upsweep's counts stay valid)
  const uint64_t kand = code ? ao[0] & kMantMask : ao[0];
  const uint64_t kvar = code ? (ao[0] ^ ao[1]) & kMantMask : ao[0] ^ ao[1];
  const uint64_t cvar = code ? ((1ull << ([&] { int b = 0; while ((1 << b) < ncodes) ++b; return b; })()) - 1) << kTopShift
                             : 0ull;
  const uint64_t var = kvar | cvar;
  const int lo = shifts.empty() ? 0 : shifts[0];
  const bool narrow = !shifts.empty() && (var >> lo) < (1ull << 32) && !(c.paths.sort1_mode & 1);
  c.paths.sort1_narrow = narrow;
  if (narrow) {
    std::vector<int> s32(shifts);
    for (int& x : s32) x -= lo;
    uint32_t* const bufK[2] = {(uint32_t*)R, (uint32_t*)(R + 8 * n)};
    Sort1Emitter<uint32_t> em32{em.orig_of, em.heights, em.euv, em.ru, em.rv, em.inv,
                                lo ? kand & ((1ull << lo) - 1) : 0ull, (uint32_t)lo};
    em32.base |= lo + 32 < 64 ? kand & ~((1ull << (lo + 32)) - 1) : 0ull;
    em32.scount = em.scount;
    em32.sshift = em.sshift;
    run_sort<uint32_t, 3, S1N_BLOCK, S1N_ITEMS, S1N_MINB, 8>(
        c, {KK_SORT1_FIRST, KK_SORT1_MID, KK_SORT1_FINAL}, n, s32, bufK, bufP,
        Sort1Loader<uint32_t>{w, u, v, code, (uint32_t)lo}, em32, ready >= 0 ? 0 : -1, S1_ALIGN);
  } else {
    uint64_t* const bufK[2] = {(uint64_t*)R, (uint64_t*)(R + 8 * n)};
    bool done = false;
    if (local && !narrow) {
      // top three active digits as global LSD passes, the rest per window in
      // shared memory; a window over capacity falls back to the full LSD sort
      // the three global digits cover the 24 highest VARYING key bits
      // (unaligned: sign/exponent bits that never vary are not spent on them)
      const int t0 = first_shift;
      const std::vector<int> top3 = {t0, t0 + 8, t0 + 16};
      ArrayEmitter<uint64_t, 3> tmp{bufK[0], bufP[0]};  // the third pass (p = 2) writes buffer 0
      run_sort<uint64_t, 3, S1_BLOCK, S1_ITEMS, S1_MINB, 8>(c, {KK_SORT1_FIRST, KK_SORT1_MID, KK_SORT1_MID}, n,
                                                         top3, bufK, bufP, Sort1FirstLoader{w, u, v, code}, tmp,
                                                         ready, S1_ALIGN, S1N_MINB);
      uint32_t* ovf = c.w.small + SM_MISC + MISC_LOCALOVF;
      c.zero(ovf, 4);
      LocalSortArgs la{bufK[0], bufP[0], n, top3[0], ovf};
      auto launch_local = [&](auto geom) {
        using G = decltype(geom);
        auto kern = k_local_final<Sort1FinalEmitter, G>;
        smem_attr(kern, sizeof(LocalSmem<G>));
        c.begin(KK_SORT1_LOCAL);
        kern<<<grid_for(n, G::kLocalTile), G::LF_BLOCK, sizeof(LocalSmem<G>), c.s>>>(la, em);
        c.launched();
      };
      launch_local(LocalGeomDefault{});
      uint32_t over = 0;
      c.to_host(&over, ovf, 4);
      c.sync();
      done = over == 0;
      c.paths.sort1_local = done ? 1 : 2;
      if (passes_out) *passes_out = done ? 3 : (int)shifts.size();
    }
    if (!done && local && em.scount) c.zero(em.scount, 4 * 256);  // windows that finished counted already
    if (!done)
      run_sort<uint64_t, 3, S1_BLOCK, S1_ITEMS, S1_MINB, 8>(c, {KK_SORT1_FIRST, KK_SORT1_MID, KK_SORT1_FINAL}, n,
                                                         shifts, bufK, bufP, Sort1FirstLoader{w, u, v, code}, em,
                                                         local ? -1 : ready, S1_ALIGN, S1N_MINB);
  }
  // a table a later stage needs zeroed: cleared on the aux stream while the
  // (shared-memory-bound) radix passes just launched run
  if (zero_ptr) prezero(c, 0, zero_ptr, zero_bytes);
  // whichever kernel wrote the final output (radix pass, identity pass or the
  // shared-memory finish) counted the slices
  c.slices_counted = em.scount != nullptr;
  if (nz) {
    c.begin(KK_OTHER);
    k_fix_negzero<<<grid_for(n, EW_BLOCK), EW_BLOCK, 0, c.s>>>(w, em.orig_of, em.heights, n);
    c.launched();
  }
}

// maxIncident of a view from m records: fine-bucket histogram, two
// order-free multisplit passes (coarse, fine) and the per-bucket shared-memory
// reduction, which also performs V1 for the view.  `in`/`mid`/`fin` are
// record buffers (mid and fin must not overlap the source).
// coarse bucket = 2^gshift fine buckets: about sqrt(nf) coarse buckets (at
// most 256) so both multisplit passes write runs of similar length
uint32_t coarse_shift(uint32_t nf) {
  uint32_t gshift = 0;
  while ((int64_t(nf) >> gshift) > 255 || (int64_t(nf) >> gshift) > (1ll << (gshift + 1))) ++gshift;
  return gshift;
}

bool mi_sliced(const Ctx& c, int64_t nv) {
  return c.paths.mi_apply_mode ? c.paths.mi_apply_mode == 2 : (nv >= (16 << 20) || nv <= (1 << 20));
}

template <class Src>
void mi_buckets(Ctx& c, Src src, int64_t m, int64_t nv, Recs mid, Recs fin, MiApplyOut out,
                bool counted = false) {
  const uint32_t nf = (uint32_t)cdiv(nv, FB);
  // sliced: one multisplit pass into 2M-vertex slices, then L2-resident
  // atomics (config 4: 22.1 -> 21.6 ms; config 1: 0.72 -> 0.57 ms).  Default
  // for views of >= 16M or <= 1M vertices; in between (8M-edge trees, built
  // several per GPU at once, whose slices contend for L2: config 5 100.7 vs
  // 101.7 ms) the shared-memory apply
  const bool sliced = mi_sliced(c, nv);
  const uint32_t gshift = sliced ? (uint32_t)(kSliceBits - FB_BITS) : coarse_shift(nf);
  uint32_t* counts = c.w.fine;
  uint32_t* fine_base = counts + (nf + 2);
  uint32_t* fine_cur = fine_base + (nf + 2);
  uint32_t* coarse_cur = fine_cur + (nf + 2);
  if (sliced && counted) {
    // per-slice endpoint counts came with the edge sort's final pass (w.fine[0, 256))
    c.begin(KK_MI_HIST);
    k_slice_scan<<<1, 256, 0, c.s>>>(counts, (uint32_t)cdiv(nv, int64_t(1) << kSliceBits), coarse_cur);
    c.launched();
  } else {
    c.zero(counts, 4 * (nf + 1));
    smem_attr(k_fine_hist<Src>, 4 * FH_WINDOW);
    for (uint32_t flo = 0; flo < nf; flo += FH_WINDOW) {
      c.begin(KK_MI_HIST);
      k_fine_hist<Src><<<c.persistent_grid(m, 256, 3), 256, 4 * FH_WINDOW, c.s>>>(src, m, flo, nf, counts);
      c.launched();
    }
    c.begin(KK_MI_HIST);
    k_fine_scan<<<1, 1024, 0, c.s>>>(counts, nf, gshift, fine_base, fine_cur, coarse_cur);
    c.launched();
  }
  using SA = SplitSmem<Src, BKA_BLOCK, BKA_ITEMS, 256>;
  using SB = SplitSmem<AosRecSrc<3>, BKB_BLOCK, BKB_ITEMS, BKB_SPAN>;
  auto kA = k_split<false, Src, BKA_BLOCK, BKA_ITEMS, 256>;
  auto kB = k_split<true, AosRecSrc<3>, BKB_BLOCK, BKB_ITEMS, BKB_SPAN>;
  smem_attr(kA, (int)SA::bytes());
  smem_attr(kB, (int)SB::bytes());
  if (sliced) zero_for_atomics(c, out.mi64, 8 * (size_t)nv);  // the atomics' starting point
  c.begin(KK_MI_SPLIT_A);
  kA<<<c.persistent_grid(m, SA::T, BKA_PER_SM), BKA_BLOCK, SA::bytes(), c.s>>>(src, m, gshift, coarse_cur, mid);
  c.launched();
  if (c.pz_next.p) {  // the next view's table, zeroed while this (shared-memory-bound) pass runs
    prezero(c, 1, const_cast<void*>(c.pz_next.p), c.pz_next.bytes);
    c.pz_next = Ctx::Prezero{};
  }
  if (sliced) {
    c.paths.mi_sliced_used = 1;
    c.begin(KK_MI_APPLY);
    k_mi_atomic<<<(unsigned)std::max<int64_t>(1, cdiv(m / 4, 256 * kMiAtomicGroups)), 256, 0, c.s>>>(mid, m,
                                                                                                   out.mi64);
    c.launched();
    c.begin(KK_MI_APPLY);
    k_v1<<<grid_for(nv, EW_BLOCK), EW_BLOCK, 0, c.s>>>(nv, out.mi64, out.grank, out.parent_out, out.cnt2);
    c.launched();
    return;
  }
  c.begin(KK_MI_SPLIT_B);
  kB<<<c.persistent_grid(m, SB::T, BKB_PER_SM), BKB_BLOCK, SB::bytes(), c.s>>>(AosRecSrc<3>{mid.r}, m, gshift,
                                                                                 fine_cur, fin);
  c.launched();
  smem_attr(k_mi_apply_smem, 8 * FB);  // 64 KB
  c.begin(KK_MI_APPLY);
  k_mi_apply_smem<<<nf, 512, 8 * FB, c.s>>>(fin, fine_base, nv, out);
  c.launched();
}

Recs recs_at(char* base, int64_t) {
  return Recs{(uint32_t*)base};
}

// Run levels level0..L of the contraction in k_tail; fills lt.soff / lt.L,
// the per-view stats and the running soff exactly as the host loop would.
void run_tail(Ctx& c, int level0, int cur, int64_t n_k, int64_t nv_k, LevelTable& lt, int64_t& soff,
              dmst_stats* st, int& jump_rounds) {
  Workspace& w = c.w;
  int blocks_per_sm = 0;  // queried per call (host-side occupancy calculation, no device round trip)
  DMST_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_tail, TAIL_BLOCK, 0));
  if (blocks_per_sm < 1) invalid("k_tail cannot be co-resident");
  c.paths.tail_level = level0;
  const int64_t want = cdiv(std::max(n_k, nv_k), TAIL_BLOCK);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)c.sms * blocks_per_sm));
  // scratch / outputs in the radix counts area (idle during the level loop)
  uint32_t* scratch = w.counts;
  int64_t* soff_out = (int64_t*)(w.counts + align_up(4 * (3 * (size_t)grid + 8)) / 4);
  int32_t* counts_out = (int32_t*)(soff_out + DMST_MAX_LEVELS + 2);
  int32_t* result = counts_out + 5 * (DMST_MAX_LEVELS + 1);
  TailArgs ta{};
  ta.cnt2 = w.cnt2;
  ta.kw = w.kw;
  ta.apre = w.apre;
  for (int i = 0; i < 2; ++i) {
    ta.euv[i] = w.euv[i];
    ta.grank[i] = w.grank[i];
    ta.mi64[i] = w.mi64[i];
  }
  ta.smi_all = w.smi_all;
  ta.lvl_all = w.lvl_all;
  ta.ret = w.ret;
  ta.scratch = scratch;
  ta.soff_out = soff_out;
  ta.counts_out = counts_out;
  ta.result = result;
  ta.level0 = level0;
  ta.cur0 = cur;
  ta.n0 = n_k;
  ta.nv0 = nv_k;
  ta.soff_k0 = lt.soff[level0];
  ta.soff0 = soff;
  // zeroed so the single readback below never reads unwritten words
  c.zero(counts_out, 4 * 5 * (size_t)(DMST_MAX_LEVELS + 1));
  c.zero(soff_out, 8 * (size_t)(DMST_MAX_LEVELS + 2));
  void* args[] = {&ta};
  c.begin(KK_TAIL);
  DMST_CUDA(cudaLaunchCooperativeKernel((const void*)k_tail, dim3(grid), dim3(TAIL_BLOCK), args, 0, c.s));
  c.launched();
  // one readback for the level count and every view's counts / offsets
  int32_t res[2];
  std::vector<int32_t> co(5 * (size_t)(DMST_MAX_LEVELS + 1));
  std::vector<int64_t> so(DMST_MAX_LEVELS + 2);
  c.to_host(res, result, 8);
  c.to_host(co.data(), counts_out, 4 * co.size());
  c.to_host(so.data(), soff_out, 8 * so.size());
  c.sync();
  const int L = res[0];
  if (L < level0 || L > DMST_MAX_LEVELS) invalid("too many contraction levels");
  for (int k = level0; k <= L; ++k) {
    if (st) {
      for (int q = 0; q < 4; ++q) st->level_counts[k][q] = co[5 * k + q];
      st->view_vertices[k] = co[5 * k + 4];
    }
    lt.soff[k + 1] = so[k + 1];
  }
  soff = so[L + 1];
  lt.L = L;
  jump_rounds += res[1];
}

// Full pipeline after the edge sort: euv0 (rank-order endpoints) ready.
void pandora_core(Ctx& c, int64_t n, int64_t nv, int32_t* vertex_parent, int32_t* edge_parent,
                  dmst_stats* st, int8_t* dbg_ret, int32_t* dbg_key, int32_t* dbg_term, int32_t* dbg_lvl) {
  Workspace& w = c.w;
  uint32_t* misc = w.small + SM_MISC;

  // level-loop counters and look-back words start at zero (later views: reset
  // by k_select_edges once the host has read them)
  c.zero(misc + 1, 4 * 15);
  c.zero(w.sel_status, 8 * (cdiv(n / 16 + 1, LS_TILE) + 2));
  // maxIncident + V1 of the input view: 2n records generated from euv0
  c.zero(w.cnt2, 4 * (n / 16 + 2));
  // view 1's table (<= n/2 + 1 vertices; ~0.26 n on random trees) zeroed
  // during view 0's pass A when view 1 will take the sliced apply
  if (mi_sliced(c, n / 4) && n / 4 > (1 << 20)) c.pz_next = Ctx::Prezero{w.mi64[1], 8 * (size_t)(n / 2 + 2)};
  mi_buckets(c, EdgeRecSrc{w.euv0}, 2 * n, nv, recs_at(w.R, 2 * n), recs_at(w.R + 24 * n, 2 * n),
             MiApplyOut{w.mi64_0, vertex_parent, nullptr, w.cnt2}, c.slices_counted);
  c.pz_next = Ctx::Prezero{};
  c.slices_counted = false;

  c.paths.mi_bucketed |= 1;
  if (c.io) c.copy_out(2, c.io->h_vp, vertex_parent, 4 * (size_t)nv);
  bool v1_done = true;

  LevelTable lt{};
  int64_t nv_k = nv, n_k = n;
  const int2* euv_k = w.euv0;
  const int32_t* grank_k = nullptr;
  const unsigned long long* mi_k = w.mi64_0;
  int cur = 0, level = 0, jump_rounds = 0;
  int64_t soff = 0;
  // jump lists in R: rulers (+ 2 ping-pong) and non-rulers
  int32_t* lists[4] = {(int32_t*)w.R, (int32_t*)w.R + nv, (int32_t*)w.R + 2 * nv, (int32_t*)w.R + 3 * nv};
  uint32_t* lcnt[4] = {misc + MISC_ACTIVE0, misc + MISC_ACTIVE1, misc + MISC_ACTIVE2, misc + MISC_NONRUL};
  while (true) {
    if (level >= DMST_MAX_LEVELS) invalid("too many contraction levels");
    if (level >= 2) join_aux(c);  // view 1's prezero never outlives view 1
    // small view: every remaining level in one cooperative kernel (tail.cuh)
    if (level >= 1 && !v1_done && n_k <= std::min<int64_t>(c.paths.tail_edges, kTailEdges)) {
      join_aux(c);
      run_tail(c, level, cur, n_k, nv_k, lt, soff, st, jump_rounds);
      level = lt.L;
      break;
    }
    // V1: maxIncident edge per vertex + child counts per edge (already done
    // by the bucketed apply unless the view was small enough for direct atomics)
    if (!v1_done) {
      int32_t* parent_out = w.smi_all + lt.soff[level];
      c.begin(KK_V1);
      k_v1<<<grid_for(nv_k, EW_BLOCK), EW_BLOCK, 0, c.s>>>(nv_k, mi_k, grank_k, parent_out, w.cnt2);
      c.launched();
    }
    // leaf numbering + kind counts
    const int64_t words = n_k / 16 + 1;
    const unsigned ls_tiles = grid_for(words, LS_TILE);
    // look-back words and level counters were zeroed before the loop (view 0)
    // or by the previous view's k_select_edges
    if (ls_tiles >= 64) {  // large views: reduce-then-scan (no look-back chain)
      c.begin(KK_LEAFSCAN);
      k_ls_reduce<<<ls_tiles, 256, 0, c.s>>>(words, n_k, w.cnt2, w.sel_status, misc + MISC_COUNTS);
      c.launched();
      c.begin(KK_LEAFSCAN);
      k_ls_scan<<<1, 1024, 0, c.s>>>(w.sel_status, ls_tiles);
      c.launched();
      c.begin(KK_LEAFSCAN);
      k_ls_apply<<<ls_tiles, 256, 0, c.s>>>(words, n_k, w.cnt2, w.sel_status, w.kw, w.lw, w.apre);
      c.launched();
    } else {
      c.begin(KK_LEAFSCAN);
      k_leafscan<<<ls_tiles, 256, 0, c.s>>>(words, n_k, w.cnt2, w.kw, w.lw, w.apre, w.sel_status,
                                           misc + MISC_LSCTR, misc + MISC_COUNTS);
      c.launched();
    }
    // V2: supervertex labels (vertex_map).  Runs before the host reads the
    // counts (one sync per level); on the final view its result is unused.
    // view 0: plain vertex map; views >= 1: packed walk table (stride 2)
    int32_t* vm = level == 0 ? w.vm_all : (int32_t*)(w.lvl_all + lt.soff[level]);
    const int vs = level == 0 ? 1 : 2;
    auto launch_v2 = [&] {
      c.begin(KK_V2);
      k_v2<<<grid_for(nv_k, EW_BLOCK), EW_BLOCK, 0, c.s>>>(nv_k, mi_k, w.lw, vm,
                                                           level == 0 ? nullptr : w.smi_all + lt.soff[level],
                                                           lists[0], lcnt[0], lists[3], lcnt[3],
                                                           8 * nv_k <= (int64_t)DMST_V2_KEEP_BYTES);
      c.launched();
    };
    // view 0's vertex map is read only by its select: the select may find the
    // labels itself by chasing maxIncident from the endpoints it needs
    // (decided below from the view's kind counts), so V2 waits for them
    const bool chase_cand = level == 0 && c.paths.v0_select != 1;
    if (!chase_cand) launch_v2();
    uint32_t mw[6];  // misc words 1..6: ACTIVE0, ACTIVE1, ACTIVE2, COUNTS[2], NONRUL
    static_assert(MISC_ACTIVE0 == 1 && MISC_COUNTS == 4 && MISC_NONRUL == 6, "readback layout");
    c.to_host(mw, misc + 1, sizeof(mw));
    c.sync();
    uint32_t counts[4] = {mw[3], mw[4], mw[0], mw[5]};
    const int64_t n_leaf = counts[0], n_chain = counts[1];
    const int64_t n_alpha = n_k - n_leaf - n_chain;
    if (st) {
      st->level_counts[level][0] = (int32_t)n_alpha;
      st->level_counts[level][1] = (int32_t)n_leaf;
      st->level_counts[level][2] = (int32_t)n_chain;
      st->level_counts[level][3] = (int32_t)n_k;
      st->view_vertices[level] = (int32_t)nv_k;
    }
    if (level >= 1 && n_alpha == 0) {  // contraction.py:203-205
      if (n_k > 0) {
        c.begin(KK_OTHER);
        k_retire_all<<<grid_for(n_k, EW_BLOCK), EW_BLOCK, 0, c.s>>>(n_k, grank_k, w.ret, (int8_t)level);
        c.launched();
      }
      break;
    }
    // Chasing in the select reads ~(chain + 2 alpha) (1 + chase) sectors
    // against V2's ~0.64 per vertex + one per needed endpoint (random trees:
    // 1.36 vs 1.64 per edge + V2's stream; ncu at 128M: 23.3 vs 24.9 GB of
    // DRAM traffic) but its dependent chase steps run at a lower rate:
    // measured 21.13-21.18 vs 21.21-21.30 ms at 128M, 100.8-101.2 vs 100.5 ms
    // on config 5 (8 trees of 8M at once).  So: only views of >= 64M edges,
    // and not when alpha edges are many or chains long (a chain-dominated
    // view: one long sorted chain chases O(n) steps per endpoint)
    const bool chase = chase_cand && (c.paths.v0_select == 2 || (n_k >= (int64_t(64) << 20) && 4 * n_chain <= 3 * n_k &&
                                                                 10 * n_alpha <= 3 * n_k));
    auto v2_sync = [&] {  // V2 after the counts were read: read its ruler / non-ruler counts
      launch_v2();
      c.to_host(mw, misc + 1, sizeof(mw));
      c.sync();
      counts[2] = mw[0];
      counts[3] = mw[5];
    };
    if (chase_cand && !chase) v2_sync();
    // pointer jumping: rulers first (a chain of rulers ~1/32 as long as the
    // in-tree), then the non-rulers, whose targets are then resolved rulers
    auto run_jumps = [&] {
      for (int phase = 0; phase < 2; ++phase) {
        uint32_t pending = counts[phase == 0 ? 2 : 3];
        const int32_t* in = lists[phase == 0 ? 0 : 3];
        const uint32_t* in_cnt = lcnt[phase == 0 ? 0 : 3];
        int a = 1;
        while (pending) {
          c.zero(lcnt[a], 4);
          c.begin(KK_JUMP);
          k_jump<<<c.persistent_grid(pending, EW_BLOCK, 16), EW_BLOCK, 0, c.s>>>(in, in_cnt, lists[a], lcnt[a], vm,
                                                                                 vs);
          c.launched();
          ++jump_rounds;
          c.to_host(&pending, lcnt[a], 4);
          c.sync();
          in = lists[a];
          in_cnt = lcnt[a];
          a = a == 1 ? 2 : 1;
        }
      }
    };
    if (!chase) run_jumps();
    // retire + compact alpha edges into view level+1
    const int64_t nv_next = n_leaf, n_next = n_alpha;
    // (a view without edges has an all-zero maxIncident: nothing to bucket)
    const bool direct = n_next == 0 || (c.paths.direct_mi_bytes >= 0 && nv_next * 8 <= c.paths.direct_mi_bytes);
    if (n_next > 0 && level + 1 <= 63) (direct ? c.paths.mi_direct : c.paths.mi_bucketed) |= 1ull << (level + 1);
    unsigned long long* mi_next = w.mi64[cur ^ 1];
    // records of view level+1: R[24n, 36n); bucketing mid buffer R[0, 12n)
    uint32_t* rec = (uint32_t*)(w.R + 24 * n);
    lt.soff[level + 1] = soff;
    soff += nv_next;
    if (direct) {
      join_aux(c);  // a prezero of this table must land first
      c.zero(mi_next, 8 * nv_next);
    }
    EdgeSel es;
    es.cnt2 = w.cnt2;
    es.kw = w.kw;
    es.apre = w.apre;
    es.euv = euv_k;
    es.grank = grank_k;
    es.vm = vm;
    es.vs = vs;
    es.ret = w.ret;
    es.euv_next = w.euv[cur ^ 1];
    es.grank_next = w.grank[cur ^ 1];
    es.mi64_next = direct ? mi_next : nullptr;
    es.x1 = level == 0 ? w.x1 : nullptr;
    es.level = (int8_t)level;
    es.reset_misc = misc + 1;
    es.reset_status = w.sel_status;
    es.n_status = 2 * (int64_t)ls_tiles;
    // a sliced next view gets its per-slice endpoint counts from this pass
    const bool count_next = !direct && n_next > 0 && mi_sliced(c, nv_next);
    es.scount = count_next ? w.fine : nullptr;
    es.sshift = kSliceBits;
    if (count_next) c.zero(w.fine, 4 * 256);
    if (!chase) {
      c.begin(KK_SELECT_EDGES);
      k_select_edges<false><<<c.persistent_grid(n_k, SEL_BLOCK * SEL_U, 8), SEL_BLOCK, 0, c.s>>>(n_k, es);
      c.launched();
    } else {
      es.mi0 = mi_k;
      es.lw = w.lw;
      es.defer = lists[3] + nv_k;  // R[16 nv, 20 nv): after the four jump lists
      es.defer_cnt = misc + MISC_DEFER;
      c.zero(es.defer_cnt, 4);
      c.begin(KK_SELECT_EDGES);
      k_select_edges<true><<<c.persistent_grid(n_k, SEL_BLOCK * DMST_SEL_CHASE_U, 8), SEL_BLOCK, 0, c.s>>>(n_k, es);
      c.launched();
      uint32_t n_defer = 0;
      c.to_host(&n_defer, es.defer_cnt, 4);
      c.sync();
      c.paths.v0_chase = n_defer ? 2 : 1;
      if (n_defer) {  // long chases: V2 + pointer jumping, then the deferred edges from the vertex map
        v2_sync();
        run_jumps();
        c.begin(KK_SELECT_EDGES);
        k_select_fix<<<c.persistent_grid(n_defer, SEL_BLOCK, 8), SEL_BLOCK, 0, c.s>>>(es.defer, es.defer_cnt, es);
        c.launched();
        c.zero(misc + 1, 4 * 15);  // V2 / jumps used the counters the select had cleared
      }
    }
    v1_done = false;
    if (!direct && n_next > 0) {
      const int64_t m = 2 * n_next;
      mi_buckets(c, EdgeRecSrc{es.euv_next}, m, nv_next, recs_at(w.R, m), Recs{rec},
                 MiApplyOut{mi_next, w.smi_all + lt.soff[level + 1], w.grank[cur ^ 1], w.cnt2}, count_next);
      v1_done = true;
    }
    // next view
    euv_k = w.euv[cur ^ 1];
    grank_k = w.grank[cur ^ 1];
    mi_k = mi_next;
    cur ^= 1;
    nv_k = nv_next;
    n_k = n_next;
    ++level;
  }
  join_aux(c);
  const int L = level;
  lt.L = L;
  lt.soff[L + 1] = soff;
  if (st) {
    st->num_levels = L;
    st->jump_rounds = jump_rounds;
  }

  // expansion walk -> chain keys (+ AND / OR of all keys for digit skipping)
  uint32_t* key_ao = w.small + SM_HIST2;
  uint32_t* keys = (uint32_t*)w.R;
  c.ones(key_ao, 4);
  c.zero(key_ao + 1, 4);
  c.begin(KK_WALK);
  k_walk<256><<<c.persistent_grid(n, 256, 8), 256, 0, c.s>>>(n, w.ret, w.x1, w.lvl_all, lt, keys,
                                                              key_ao);
  c.launched();
  if (dbg_ret) DMST_CUDA(cudaMemcpyAsync(dbg_ret, w.ret, n, cudaMemcpyDeviceToDevice, c.s));
  if (dbg_key || dbg_term || dbg_lvl) {
    c.begin(KK_OTHER);
    k_debug_chain<<<grid_for(n, EW_BLOCK), EW_BLOCK, 0, c.s>>>(n, keys, w.smi_all, lt, dbg_key, dbg_term, dbg_lvl);
    c.launched();
  }
  // keys are <= soff[L + 1]: a key range of >= 3 digits (every tree of more
  // than a few hundred thousand edges) sorts every digit of the range without
  // reading the keys' AND / OR back (a constant digit would only cost a pass);
  // smaller ranges read it to skip constant digits and catch single chains
  std::vector<int> shifts;
  const int64_t kmax = lt.soff[L + 1];
  if (kmax >= (int64_t(1) << (2 * S2_BITS))) {
    for (int sft = 0; sft < 32 && (kmax >> sft) > 0; sft += S2_BITS) shifts.push_back(sft);
  } else {
    uint32_t kao[2];
    c.to_host(kao, key_ao, 8);
    c.sync();
    shifts = active_digits(kao[0], kao[1], S2_BITS, 32);
  }
  if (st) st->sort2_passes = (int)shifts.size();
  // chain sort: keys at R[0, 4n); ping-pong A = R[4n, 12n), B = R[12n, 20n);
  if (shifts.empty()) {  // one chain (all keys equal): rank order is chain order
    if (st) st->num_chains = 1;
    c.begin(KK_LINK_APPLY);
    k_link<<<grid_for(n, EW_BLOCK), EW_BLOCK, 0, c.s>>>(n, keys, nullptr, w.smi_all, edge_parent);
    c.launched();
  } else {
    // packed (chain key << 32 | rank) items: ping-pong R[4n, 12n) / R[12n, 20n)
    uint64_t* const bufK[2] = {(uint64_t*)(w.R + align_up(4 * n)), (uint64_t*)(w.R + align_up(12 * n))};
    uint32_t* const bufP[2] = {nullptr, nullptr};
    const int lastb = ((int)shifts.size() - 1) % 2;
    ArrayEmitter<uint64_t, 0> fin{bufK[lastb], nullptr};
    std::vector<int> shifts64(shifts);
    for (int& x : shifts64) x += 32;
    const bool large = c.paths.sort2_geometry ? c.paths.sort2_geometry == 2 : n >= kS2LargeEdges;
    c.paths.sort2_geometry_used = large ? 2 : 1;
    const int kinds2[3] = {KK_SORT2_PASS, KK_SORT2_PASS, KK_SORT2_PASS};
    if (large)
      run_sort<uint64_t, 0, S2L_BLOCK, S2L_ITEMS, S2L_MINB, S2_BITS>(c, kinds2, n, shifts64, bufK, bufP,
                                                                    Sort2FirstLoader{keys}, fin);
    else
      run_sort<uint64_t, 0, S2_BLOCK, S2_ITEMS, S2_MINB, S2_BITS>(c, kinds2, n, shifts64, bufK, bufP,
                                                                 Sort2FirstLoader{keys}, fin);
    if (st && st->want_chains) {
      uint32_t* cnt = w.small + SM_MISC + 60;
      c.zero(cnt, 4);
      c.begin(KK_OTHER);
      k_count_heads<<<c.persistent_grid(n, 256, 8), 256, 0, c.s>>>((const unsigned long long*)fin.keys, n, cnt);
      c.launched();
      uint32_t h = 0;
      c.to_host(&h, cnt, 4);
      c.sync();
      st->num_chains = (int32_t)h;
    }
    // (rank, parent) records grouped by 8192-rank window: R[20n, 28n) -> R[28n, 36n)
    uint32_t* recA = (uint32_t*)(w.R + align_up(20 * n));
    uint32_t* recB = (uint32_t*)(w.R + align_up(28 * n));
    // sliced (as the maxIncident apply): one multisplit pass into 2M-rank
    // slices + L2-resident scatter, instead of two passes + a shared-memory apply
    const bool lsl = mi_sliced(c, n);
    const uint32_t nf = (uint32_t)cdiv(n, FB), gshift = lsl ? (uint32_t)(DMST_LINK_SLICE_BITS - FB_BITS) : coarse_shift(nf);
    const uint32_t nc = (uint32_t)cdiv(nf, 1u << gshift);
    uint32_t* fine_cur = w.fine;
    uint32_t* coarse_cur = w.fine + (nf + 2);
    c.begin(KK_LINK_SPLIT);
    k_link_cursors<<<grid_for(nf, EW_BLOCK), EW_BLOCK, 0, c.s>>>(coarse_cur, nc, fine_cur, nf, gshift);
    c.launched();
    using LA = SplitSmem<LinkSortedSrc, BKA_BLOCK, BKA_ITEMS, 256>;
    using LB = SplitSmem<AosRecSrc<2>, BKB_BLOCK, BKB_ITEMS, BKB_SPAN>;
    auto kA = k_split<false, LinkSortedSrc, BKA_BLOCK, BKA_ITEMS, 256>;
    auto kB = k_split<true, AosRecSrc<2>, BKB_BLOCK, BKB_ITEMS, BKB_SPAN>;
    smem_attr(kA, (int)LA::bytes());
    smem_attr(kB, (int)LB::bytes());
    c.begin(KK_LINK_SPLIT);
    kA<<<c.persistent_grid(n, LA::T, BKA_PER_SM), BKA_BLOCK, LA::bytes(), c.s>>>(
        LinkSortedSrc{(const unsigned long long*)fin.keys, w.smi_all}, n, gshift, coarse_cur, Recs{recA});
    c.launched();
    if (lsl) {
      c.begin(KK_LINK_APPLY);
      k_link_scatter<<<(unsigned)std::max<int64_t>(1, cdiv(n / 2, 256 * 4)), 256, 0, c.s>>>((const uint2*)recA, n,
                                                                                          edge_parent);
      c.launched();
      return;
    }
    c.begin(KK_LINK_SPLIT);
    kB<<<c.persistent_grid(n, LB::T, BKB_PER_SM), BKB_BLOCK, LB::bytes(), c.s>>>(AosRecSrc<2>{recA}, n, gshift,
                                                                                 fine_cur, Recs{recB});
    c.launched();
    c.begin(KK_LINK_APPLY);
    k_link_apply<<<nf, 512, 0, c.s>>>((const uint2*)recB, n, edge_parent);
    c.launched();
  }
}

template <class F>
int guarded(F&& f) {
  g_err.clear();
  try {
    f();
    return 0;
  } catch (const Fail& e) {
    return e.code;
  }
}

void init_ctx(Ctx& c, int64_t n, int64_t nv, void* ws, void* stream, dmst_stats* st) {
  c.s = (cudaStream_t)stream;
  c.sms = num_sms();
  char* base = (char*)(((uintptr_t)ws + 255) & ~uintptr_t(255));
  c.w = carve(n, nv, base);
  if (st) {
    const int32_t prof = st->profile, wc = st->want_chains;
    const int64_t te = st->tail_edges, dm = st->direct_mi_bytes;
    const int32_t s1 = st->sort1_mode, s2 = st->sort2_geometry, ma = st->mi_apply_mode, vsel = st->v0_select;
    if (ma < 0 || ma > 2) invalid("mi_apply_mode must be 0, 1 or 2");
    if (vsel < 0 || vsel > 2) invalid("v0_select must be 0, 1 or 2");
    if (s1 < 0 || s1 > 7) invalid("sort1_mode must be in [0, 7]");
    if (s2 < 0 || s2 > 2) invalid("sort2_geometry must be 0, 1 or 2");
    if (te < -1 || dm < -1) invalid("tail_edges / direct_mi_bytes must be >= -1");
    memset(st, 0, sizeof(*st));
    st->profile = prof;
    st->want_chains = wc;
    st->tail_edges = te;
    st->direct_mi_bytes = dm;
    st->sort1_mode = s1;
    st->sort2_geometry = s2;
    st->mi_apply_mode = ma;
    st->v0_select = vsel;
    c.profile = prof != 0;
    if (te) c.paths.tail_edges = te;  // -1: n_k <= -1 never holds
    if (dm) c.paths.direct_mi_bytes = dm;
    c.paths.sort1_mode = s1;
    c.paths.sort2_geometry = s2;
    c.paths.mi_apply_mode = ma;
    c.paths.v0_select = vsel;
  }
}

void report_paths(const Ctx& c, dmst_stats* st) {
  if (!st) return;
  st->sort1_narrow = c.paths.sort1_narrow;
  st->sort1_compacted = c.paths.sort1_compacted;
  st->sort1_local = c.paths.sort1_local;
  st->mi_sliced = c.paths.mi_sliced_used;
  st->sort2_geometry_used = c.paths.sort2_geometry_used;
  st->tail_level = c.paths.tail_level;
  st->mi_bucketed = c.paths.mi_bucketed;
  st->mi_direct = c.paths.mi_direct;
  st->v0_chase = c.paths.v0_chase;
}

static int build_impl(const int32_t* u, const int32_t* v, const double* w, int64_t n, int64_t nv,
                      int32_t* orig_of, double* heights, int32_t* edge_parent, int32_t* vertex_parent,
                      dmst_stats* st, int8_t* dbg_ret, int32_t* dbg_key, int32_t* dbg_term,
                      int32_t* dbg_lvl, void* ws, size_t ws_bytes, void* stream, HostIO* io = nullptr,
                      cudaEvent_t inputs_ready = nullptr) {
  return guarded([&] {
    check_args(n, nv, ws, ws_bytes);
    if (!u || !v || !w || !orig_of || !heights || !edge_parent || !vertex_parent)
      invalid("null input/output pointer");
    Ctx c;
    init_ctx(c, n, nv, ws, stream, st);
    c.io = io;
    if (inputs_ready) DMST_CUDA(cudaStreamWaitEvent(c.s, inputs_ready, 0));
    mark_aux(c);
    Sort1FinalEmitter em{orig_of, heights, c.w.euv0, nullptr, nullptr};
    int p1 = 0;
    const bool sl = mi_sliced(c, nv);  // view 0's table, zeroed during the edge sort's passes
    if (sl) {  // and view 0's endpoints counted per slice by the final pass
      c.zero(c.w.fine, 4 * 256);
      em.scount = c.w.fine;
      em.sshift = kSliceBits;
    }
    edge_sort(c, u, v, w, n, em, &p1, sl ? c.w.mi64_0 : nullptr, sl ? 8 * (size_t)nv : 0);
    if (io) {
      c.copy_out(0, io->h_orig, orig_of, 4 * (size_t)n);
      c.copy_out(1, io->h_heights, heights, 8 * (size_t)n);
    }
    pandora_core(c, n, nv, vertex_parent, edge_parent, st, dbg_ret, dbg_key, dbg_term, dbg_lvl);
    if (io) c.copy_out(3, io->h_ep, edge_parent, 4 * (size_t)n);
    c.sync();
    if (io) DMST_CUDA(cudaStreamSynchronize(io->side));
    c.collect(st);
    report_paths(c, st);
    if (st) {
      st->sort1_passes = p1;
      st->kernel_launches = c.launches;
    }
  });
}

// Device buffers of dmst_build_host behind the pipeline workspace.
struct HostBufs {
  int32_t *u, *v, *orig, *ep, *vp;
  double *w, *heights;
  size_t bytes;
};
HostBufs host_bufs(int64_t n, int64_t nv, char* base) {
  HostBufs b{};
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  b.w = (double*)take(8 * n);
  b.u = (int32_t*)take(4 * n);
  b.v = (int32_t*)take(4 * n);
  b.orig = (int32_t*)take(4 * n);
  b.heights = (double*)take(8 * n);
  b.ep = (int32_t*)take(4 * n);
  b.vp = (int32_t*)take(4 * nv);
  b.bytes = off;
  return b;
}


// ------------------------------------------------ mutual-reachability MST
// (pointgen.py:56-178)
size_t mreach_ws_bytes(int64_t n, int dim) {
  const int64_t cap = n;
  return align_up(8 * (size_t)n)                     // core_sq
         + align_up(8 * (size_t)dim * cap)           // acoord
         + 2 * align_up(8 * (size_t)cap)             // acore, abest
         + 2 * align_up(4 * (size_t)cap)             // afrom, idx
         + align_up(sizeof(PrimSlot) * 2 * (PRIM_MAX_GRID + 1)) + 1024;
}

template <int DIM>
void mreach_impl(Ctx& c, const double* pts, int64_t n, int k, int engine, int32_t* u, int32_t* v, double* w,
                 double* core_sq_out, char* ws) {
  char* p = (char*)(((uintptr_t)ws + 255) & ~uintptr_t(255));
  double* core_sq = (double*)p;
  p += align_up(8 * (size_t)n);
  PrimState st{};
  st.cap = n;
  st.acoord = (double*)p;
  p += align_up(8 * (size_t)DIM * n);
  st.acore = (double*)p;
  p += align_up(8 * (size_t)n);
  st.abest = (double*)p;
  p += align_up(8 * (size_t)n);
  st.afrom = (int32_t*)p;
  p += align_up(4 * (size_t)n);
  st.idx = (int32_t*)p;
  p += align_up(4 * (size_t)n);
  PrimSlot* slots = (PrimSlot*)p;
  p += align_up(sizeof(PrimSlot) * 2 * (PRIM_MAX_GRID + 1));
  unsigned long long* bar = (unsigned long long*)p;
  c.zero(bar, 8);
  c.begin(KK_OTHER);
  k_core_sq<DIM><<<grid_for(n, KNN_BLOCK), KNN_BLOCK, 0, c.s>>>(pts, n, k, core_sq);
  c.launched();
  if (core_sq_out)
    DMST_CUDA(cudaMemcpyAsync(core_sq_out, core_sq, 8 * (size_t)n, cudaMemcpyDeviceToDevice, c.s));
  if (n < 2) return;
  c.begin(KK_OTHER);
  k_prim_init<DIM><<<grid_for(n, EW_BLOCK), EW_BLOCK, 0, c.s>>>(pts, core_sq, n, st);
  c.launched();
  const bool numpy = engine == 2 || (engine == 0 && n < 4096);  // "auto" (pointgen.py:170-171)
  const void* kern = numpy ? (const void*)k_prim<DIM, true> : (const void*)k_prim<DIM, false>;
  constexpr size_t psm = prim_smem_bytes<DIM>();
  if (numpy)
    smem_attr(k_prim<DIM, true>, (int)psm);
  else
    smem_attr(k_prim<DIM, false>, (int)psm);
  int per_sm = 0;
  DMST_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PRIM_BLOCK, psm));
  if (per_sm < 1) invalid("k_prim cannot be co-resident");
  // at most PRIM_MAX_GRID blocks: warp 0 reduces all block slots after the barrier
  const int64_t grid = std::max<int64_t>(
      1, std::min<int64_t>({cdiv(n - 1, 2 * PRIM_BLOCK), (int64_t)c.sms * per_sm, (int64_t)PRIM_MAX_GRID}));
  PrimArgs a{pts, core_sq, n, st, slots, bar, u, v, w};
  void* args[] = {&a};
  c.begin(KK_OTHER);
  DMST_CUDA(cudaLaunchCooperativeKernel(kern, dim3((unsigned)grid), dim3(PRIM_BLOCK), args, psm, c.s));
  c.launched();
  c.begin(KK_OTHER);
  k_sqrt_inplace<<<grid_for(n - 1, EW_BLOCK), EW_BLOCK, 0, c.s>>>(w, n - 1);
  c.launched();
}
}  // namespace
}  // namespace dmst

using namespace dmst;

extern "C" {

size_t dmst_workspace_bytes(int64_t n_edges, int64_t n_vertices) {
  if (n_edges < 1 || n_vertices < 2) return 0;
  return carve(n_edges, n_vertices, nullptr).bytes;
}

size_t dmst_host_workspace_bytes(int64_t n_edges, int64_t n_vertices) {
  if (n_edges < 1 || n_vertices < 2) return 0;
  return carve(n_edges, n_vertices, nullptr).bytes + host_bufs(n_edges, n_vertices, nullptr).bytes + 256;
}

int dmst_build_host(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges,
                    int64_t n_vertices, int32_t* orig_of, double* heights, int32_t* edge_parent,
                    int32_t* vertex_parent, dmst_stats* stats, void* workspace, size_t workspace_bytes,
                    void* stream) {
  // side stream + events are per host thread and reused across calls
  thread_local cudaStream_t side = nullptr;
  thread_local cudaEvent_t evs[6] = {};
  thread_local int side_dev = -1;
  int rc = guarded([&] {
    if (n_edges < 1 || n_vertices != n_edges + 1) invalid("n_vertices must equal n_edges + 1 (a spanning tree)");
    if (!u || !v || !w || !orig_of || !heights || !edge_parent || !vertex_parent)
      invalid("null input/output pointer");
    if (!workspace || workspace_bytes < dmst_host_workspace_bytes(n_edges, n_vertices))
      invalid("workspace too small (dmst_host_workspace_bytes)");
    int dev = 0;
    DMST_CUDA(cudaGetDevice(&dev));
    if (side == nullptr || side_dev != dev) {
      DMST_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
      for (auto& e : evs) DMST_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      side_dev = dev;
    }
  });
  if (rc) return rc;
  const int64_t n = n_edges, nv = n_vertices;
  char* base = (char*)(((uintptr_t)workspace + 255) & ~uintptr_t(255));
  const size_t pipe = carve(n, nv, nullptr).bytes;
  HostBufs b = host_bufs(n, nv, base + pipe);
  rc = guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    // inputs: H2D on the side stream, ordered after work already on `stream`
    DMST_CUDA(cudaEventRecord(evs[4], s));
    DMST_CUDA(cudaStreamWaitEvent(side, evs[4], 0));
    DMST_CUDA(cudaMemcpyAsync(b.w, w, 8 * (size_t)n, cudaMemcpyHostToDevice, side));
    DMST_CUDA(cudaMemcpyAsync(b.u, u, 4 * (size_t)n, cudaMemcpyHostToDevice, side));
    DMST_CUDA(cudaMemcpyAsync(b.v, v, 4 * (size_t)n, cudaMemcpyHostToDevice, side));
    DMST_CUDA(cudaEventRecord(evs[5], side));
  });
  if (rc) return rc;
  HostIO io;
  io.side = side;
  io.h_orig = orig_of;
  io.h_heights = heights;
  io.h_ep = edge_parent;
  io.h_vp = vertex_parent;
  io.n = n;
  io.nv = nv;
  for (int i = 0; i < 4; ++i) io.ev[i] = evs[i];
  return build_impl(b.u, b.v, b.w, n, nv, b.orig, b.heights, b.ep, b.vp, stats, nullptr, nullptr, nullptr,
                    nullptr, base, pipe, stream, &io, evs[5]);
}

int dmst_build(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges,
               int64_t n_vertices, int32_t* orig_of, double* heights, int32_t* edge_parent,
               int32_t* vertex_parent, dmst_stats* stats, void* workspace, size_t workspace_bytes,
               void* stream) {
  return build_impl(u, v, w, n_edges, n_vertices, orig_of, heights, edge_parent, vertex_parent, stats,
                    nullptr, nullptr, nullptr, nullptr, workspace, workspace_bytes, stream);
}

int dmst_build_debug(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges,
                     int64_t n_vertices, int32_t* orig_of, double* heights, int32_t* edge_parent,
                     int32_t* vertex_parent, dmst_stats* stats, int8_t* retirement,
                     int32_t* chain_key, int32_t* chain_terminal, int32_t* chain_level,
                     void* workspace, size_t workspace_bytes, void* stream) {
  return build_impl(u, v, w, n_edges, n_vertices, orig_of, heights, edge_parent, vertex_parent, stats,
                    retirement, chain_key, chain_terminal, chain_level, workspace, workspace_bytes,
                    stream);
}

int dmst_rank_edges(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges,
                    int64_t n_vertices, int32_t* orig_of, double* heights, int32_t* ru, int32_t* rv,
                    void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    check_args(n_edges, n_vertices, workspace, workspace_bytes);
    if (!u || !v || !w || !orig_of || !heights || !ru || !rv) invalid("null input/output pointer");
    Ctx c;
    init_ctx(c, n_edges, n_vertices, workspace, stream, nullptr);
    Sort1FinalEmitter em{orig_of, heights, nullptr, ru, rv};
    edge_sort(c, u, v, w, n_edges, em, nullptr);
    c.sync();
  });
}

int dmst_pandora(const int32_t* ru, const int32_t* rv, int64_t n_edges, int64_t n_vertices,
                 int32_t* edge_parent, int32_t* vertex_parent, dmst_stats* stats, void* workspace,
                 size_t workspace_bytes, void* stream) {
  return guarded([&] {
    check_args(n_edges, n_vertices, workspace, workspace_bytes);
    if (!ru || !rv || !edge_parent || !vertex_parent) invalid("null input/output pointer");
    Ctx c;
    init_ctx(c, n_edges, n_vertices, workspace, stream, stats);
    c.begin(KK_OTHER);
    k_pack_euv<<<grid_for(n_edges, EW_BLOCK), EW_BLOCK, 0, c.s>>>(ru, rv, n_edges, c.w.euv0);
    c.launched();
    pandora_core(c, n_edges, n_vertices, vertex_parent, edge_parent, stats, nullptr, nullptr, nullptr,
                 nullptr);
    c.sync();
    c.collect(stats);
    report_paths(c, stats);
    if (stats) stats->kernel_launches = c.launches;
  });
}

int dmst_validate(const int32_t* u, const int32_t* v, const double* w, int64_t n_edges, int64_t n_vertices,
                  int32_t* error_kind, int64_t* bad_edge, void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    if (!error_kind || !bad_edge) invalid("error_kind / bad_edge must be host pointers");
    *error_kind = DMST_TREE_OK;
    *bad_edge = -1;
    // tree_core.py:116-121: sizes first
    if (n_vertices < 2) {
      *error_kind = DMST_TREE_TOO_SMALL;
      return;
    }
    if (n_edges != n_vertices - 1) {
      *error_kind = DMST_TREE_EDGE_COUNT;
      return;
    }
    if (n_edges >= (int64_t(1) << 29)) invalid("n_edges must be < 2^29");
    if (!u || !v || !w) invalid("null input pointer");
    if (!workspace || workspace_bytes < carve(n_edges, n_vertices, nullptr).bytes) invalid("workspace too small");
    const int64_t n = n_edges, nv = n_vertices;
    Ctx c;
    init_ctx(c, n, nv, workspace, stream, nullptr);
    uint32_t* r = c.w.small + SM_MISC + 32;  // [0..3] checks, [4] roots, [5] duplicate flag
    unsigned long long* ao = (unsigned long long*)(c.w.small + SM_MISC + 48);
    c.zero(r, 24);
    c.ones(r, 4);      // r[0]: first non-finite edge
    c.ones(r + 3, 4);  // r[3]: first self-loop
    c.ones(ao, 8);
    c.zero(ao + 1, 8);
    c.begin(KK_OTHER);
    k_validate_scan<<<c.persistent_grid(n, 256, 8), 256, 0, c.s>>>(u, v, w, n, nv, r, ao);
    c.launched();
    uint32_t h[4];
    c.to_host(h, r, sizeof(h));
    c.sync();
    if (h[0] != 0xffffffffu) {  // :124-126
      *error_kind = DMST_TREE_NONFINITE;
      *bad_edge = h[0];
      return;
    }
    if (h[1]) {  // :127-128
      *error_kind = DMST_TREE_NEGATIVE_ID;
      return;
    }
    if (h[2]) {  // :129-130
      *error_kind = DMST_TREE_ID_RANGE;
      return;
    }
    if (h[3] != 0xffffffffu) {  // :131-133
      *error_kind = DMST_TREE_SELF_LOOP;
      *bad_edge = h[3];
      return;
    }
    // connectivity (:137-138).  n = nv - 1 edges and connected => a tree, so
    // the duplicate check (:134-136) only has to run when this fails.
    int32_t* p = c.w.vm_all;
    c.begin(KK_OTHER);
    k_cc_init<<<grid_for(nv, EW_BLOCK), EW_BLOCK, 0, c.s>>>(p, nv);
    c.launched();
    c.begin(KK_OTHER);
    k_cc_hook<<<c.persistent_grid(n, 256, 8), 256, 0, c.s>>>(u, v, n, p);
    c.launched();
    c.begin(KK_OTHER);
    k_cc_roots<<<c.persistent_grid(nv, 256, 8), 256, 0, c.s>>>(p, nv, r + 4);
    c.launched();
    uint32_t roots = 0;
    c.to_host(&roots, r + 4, 4);
    unsigned long long hao[2];
    c.to_host(hao, ao, 16);
    c.sync();
    if (roots == 1) return;
    // not a tree: duplicates first, as the reference reports them first
    const std::vector<int> shifts = active_digits(hao[0], hao[1], 8, 64);
    if (shifts.empty()) {  // every undirected key equal (n >= 2 edges => duplicate)
      if (n >= 2) *error_kind = DMST_TREE_DUPLICATE;
      else *error_kind = DMST_TREE_NOT_A_TREE;
      return;
    }
    uint64_t* const bufK[2] = {(uint64_t*)c.w.R, (uint64_t*)(c.w.R + align_up(8 * n))};
    uint32_t* const bufP[2] = {nullptr, nullptr};
    const int lastb = ((int)shifts.size() - 1) % 2;
    ArrayEmitter<uint64_t, 0> fin{bufK[lastb], nullptr};
    run_sort<uint64_t, 0, S1_BLOCK, S1_ITEMS, S1_MINB, 8>(c, {KK_OTHER, KK_OTHER, KK_OTHER}, n, shifts, bufK, bufP,
                                                         DupKeyLoader{u, v}, fin);
    c.begin(KK_OTHER);
    k_adjacent_equal<<<grid_for(n, EW_BLOCK), EW_BLOCK, 0, c.s>>>((const unsigned long long*)fin.keys, n, r + 5);
    c.launched();
    uint32_t dup = 0;
    c.to_host(&dup, r + 5, 4);
    c.sync();
    *error_kind = dup ? DMST_TREE_DUPLICATE : DMST_TREE_NOT_A_TREE;
  });
}

int dmst_dendrogram_height(const int32_t* edge_parent, int64_t n_edges, int64_t* height, void* workspace,
                           size_t workspace_bytes, void* stream) {
  return guarded([&] {
    if (!height) invalid("height must be a host pointer");
    *height = 0;
    if (n_edges < 1) return;
    if (!edge_parent || !workspace || workspace_bytes < (size_t)(16 * n_edges + 4096)) invalid("bad pointers / workspace");
    const int64_t n = n_edges;
    Ctx c;
    c.s = (cudaStream_t)stream;
    c.sms = num_sms();
    char* base = (char*)(((uintptr_t)workspace + 255) & ~uintptr_t(255));
    int2* buf[2] = {(int2*)base, (int2*)(base + align_up(8 * n))};
    uint32_t* flag = (uint32_t*)(base + align_up(8 * n) + align_up(8 * n));
    if ((size_t)((char*)flag - (char*)workspace) + 16 > workspace_bytes) invalid("workspace too small");
    c.zero(flag + 2, 4);
    c.begin(KK_OTHER);
    k_depth_init<<<grid_for(n, EW_BLOCK), EW_BLOCK, 0, c.s>>>(edge_parent, n, buf[0], flag + 2);
    c.launched();
    uint32_t bad = 0;
    c.to_host(&bad, flag + 2, 4);
    c.sync();
    if (bad) invalid("edge_parent[e] must be ROOT (-1) or a heavier edge's rank in [0, e)");
    int cur = 0;
    bool live_left = true;
    // parents are strictly smaller ranks, so ceil(log2 n) <= 29 rounds resolve every edge
    for (int round = 0; round < 64 && live_left; ++round) {
      c.zero(flag, 4);
      c.begin(KK_OTHER);
      k_depth_jump<<<c.persistent_grid(n, 256, 8), 256, 0, c.s>>>(buf[cur], buf[cur ^ 1], n, flag);
      c.launched();
      cur ^= 1;
      uint32_t live = 0;
      c.to_host(&live, flag, 4);
      c.sync();
      live_left = live != 0;
    }
    if (live_left) invalid("edge_parent does not resolve to ROOT within 64 pointer-jumping rounds");
    c.zero(flag + 1, 4);
    c.begin(KK_OTHER);
    k_depth_max<<<c.persistent_grid(n, 256, 8), 256, 0, c.s>>>(buf[cur], n, flag + 1);
    c.launched();
    uint32_t mx = 0;
    c.to_host(&mx, flag + 1, 4);
    c.sync();
    *height = mx;
  });
}

int64_t dmst_format_dendrogram(const int32_t* edge_parent, const int32_t* vertex_parent, int64_t n_edges,
                               int64_t n_vertices, char* out, size_t out_capacity, void* workspace,
                               size_t workspace_bytes, void* stream) {
  int64_t total = -1;
  const int rc = guarded([&] {
    if (n_edges < 0 || n_vertices < 0) invalid("negative sizes");
    if (n_edges >= (int64_t(1) << 29) || n_vertices > (int64_t(1) << 29)) invalid("ids must be < 2^29");
    const int64_t lines = n_edges + n_vertices;
    if (lines == 0) {
      total = 0;
      return;
    }
    if (!edge_parent && n_edges) invalid("null edge_parent");
    if (!vertex_parent && n_vertices) invalid("null vertex_parent");
    const int64_t nb = cdiv(lines, FMT_TILE);
    if (!workspace || workspace_bytes < (size_t)(8 * (nb + 1))) invalid("workspace too small");
    Ctx c;
    c.s = (cudaStream_t)stream;
    c.sms = num_sms();
    unsigned long long* bl = (unsigned long long*)workspace;
    c.begin(KK_OTHER);
    k_fmt_count<<<(unsigned)nb, FMT_BLOCK, 0, c.s>>>(n_edges, n_vertices, edge_parent, vertex_parent, bl);
    c.launched();
    c.begin(KK_OTHER);
    k_fmt_scan<<<1, 1024, 0, c.s>>>(bl, nb);
    c.launched();
    unsigned long long t = 0;
    c.to_host(&t, bl + nb, 8);
    c.sync();
    total = (int64_t)t;
    if (!out) return;  // size query
    if (out_capacity < t) invalid("output buffer too small");
    smem_attr(k_fmt_write, (size_t)FMT_TILE * FMT_MAXLINE);
    c.begin(KK_OTHER);
    k_fmt_write<<<(unsigned)nb, FMT_BLOCK, (size_t)FMT_TILE * FMT_MAXLINE, c.s>>>(n_edges, n_vertices, edge_parent,
                                                                               vertex_parent, bl, out);
    c.launched();
    c.sync();
  });
  return rc ? -1 : total;
}

size_t dmst_parse_workspace_bytes(int64_t body_len, int64_t n_edges, int64_t n_vertices) {
  if (body_len < 0 || n_edges < 0 || n_vertices < 0) return 0;
  return (size_t)(8 * (cdiv(body_len, PARSE_TILE) + 1) + 32 + 8 * (n_edges + n_vertices) + 64);
}

int dmst_parse_dendrogram(const char* body, int64_t body_len, int64_t n_edges, int64_t n_vertices,
                          int32_t* edge_parent, int32_t* vertex_parent, int64_t* bad_line, int64_t* edge_lines,
                          int64_t* vertex_lines, void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    if (!bad_line || !edge_lines || !vertex_lines) invalid("result pointers must be host pointers");
    *bad_line = -1;
    *edge_lines = *vertex_lines = 0;
    if (n_edges < 0 || n_vertices < 0 || body_len < 0) invalid("negative sizes");
    Ctx c;
    c.s = (cudaStream_t)stream;
    c.sms = num_sms();
    if (n_edges) DMST_CUDA(cudaMemsetAsync(edge_parent, 0xff, 4 * (size_t)n_edges, c.s));  // ROOT
    if (n_vertices) DMST_CUDA(cudaMemsetAsync(vertex_parent, 0xff, 4 * (size_t)n_vertices, c.s));
    if (body_len == 0) {
      c.sync();
      return;
    }
    if (!body) invalid("null body");
    const int64_t nb = cdiv(body_len, PARSE_TILE);
    if (!workspace || workspace_bytes < dmst_parse_workspace_bytes(body_len, n_edges, n_vertices))
      invalid("workspace too small (dmst_parse_workspace_bytes)");
    unsigned long long* bl = (unsigned long long*)workspace;
    unsigned long long* err = bl + nb + 1;
    unsigned long long* last = err + 4;
    c.ones(err, 8);
    c.zero(err + 1, 16);
    c.zero(last, 8 * (size_t)(n_edges + n_vertices));
    c.begin(KK_OTHER);
    k_parse_count<<<(unsigned)nb, PARSE_BLOCK, 0, c.s>>>(body, body_len, bl);
    c.launched();
    c.begin(KK_OTHER);
    k_fmt_scan<<<1, 1024, 0, c.s>>>(bl, nb);
    c.launched();
    c.begin(KK_OTHER);
    k_parse_lines<<<(unsigned)nb, PARSE_BLOCK, 0, c.s>>>(body, body_len, bl, n_edges, n_vertices, last, err);
    c.launched();
    if (n_edges + n_vertices) {
      c.begin(KK_OTHER);
      k_parse_finish<<<grid_for(n_edges + n_vertices, EW_BLOCK), EW_BLOCK, 0, c.s>>>(last, n_edges, n_vertices,
                                                                                    edge_parent, vertex_parent);
      c.launched();
    }
    unsigned long long h[3];
    c.to_host(h, err, 24);
    c.sync();
    *bad_line = h[0] == ~0ull ? -1 : (int64_t)h[0] - 1;
    *edge_lines = (int64_t)h[1];
    *vertex_lines = (int64_t)h[2];
  });
}

int dmst_first_difference(const int32_t* a, const int32_t* b, int64_t n, int64_t* first, void* workspace,
                          size_t workspace_bytes, void* stream) {
  return guarded([&] {
    if (!first) invalid("first must be a host pointer");
    *first = -1;
    if (n <= 0) return;
    if (!a || !b || !workspace || workspace_bytes < 8) invalid("bad pointers / workspace");
    Ctx c;
    c.s = (cudaStream_t)stream;
    c.sms = num_sms();
    unsigned long long* f = (unsigned long long*)workspace;
    c.ones(f, 8);
    c.begin(KK_OTHER);
    k_first_diff<<<grid_for(n, EW_BLOCK), EW_BLOCK, 0, c.s>>>(a, b, n, f);
    c.launched();
    unsigned long long h = 0;
    c.to_host(&h, f, 8);
    c.sync();
    *first = h == ~0ull ? -1 : (int64_t)h;
  });
}

size_t dmst_mreach_workspace_bytes(int64_t n_points, int32_t dim) {
  return n_points < 1 || dim < 1 ? 0 : mreach_ws_bytes(n_points, dim);
}

int dmst_mreach_mst(const double* coords, int64_t n_points, int32_t dim, int32_t min_pts, int32_t engine,
                    int32_t* u, int32_t* v, double* w, double* core_sq, void* workspace, size_t workspace_bytes,
                    void* stream) {
  return guarded([&] {
    const int64_t n = n_points;
    if (n < 2 || n > INT32_MAX) invalid("need 2 <= n_points < 2^31");
    if (dim < 1 || dim > EMST_MAX_DIM) invalid("dim must be in [1, 8]");
    if (min_pts < 1 || min_pts > n || min_pts > KNN_MAX_K) invalid("min_pts must be in [1, min(n, 16)]");
    if (engine < 0 || engine > 2) invalid("engine must be 0 (auto), 1 (numba) or 2 (numpy)");
    if (!coords || !u || !v || !w || !workspace) invalid("null pointer");
    if (workspace_bytes < mreach_ws_bytes(n, dim)) invalid("workspace too small");
    Ctx c;
    c.s = (cudaStream_t)stream;
    c.sms = num_sms();
    switch (dim) {
#define DMST_DIM(D) \
  case D:           \
    mreach_impl<D>(c, coords, n, min_pts, engine, u, v, w, core_sq, (char*)workspace); \
    break;
      DMST_DIM(1) DMST_DIM(2) DMST_DIM(3) DMST_DIM(4) DMST_DIM(5) DMST_DIM(6) DMST_DIM(7) DMST_DIM(8)
#undef DMST_DIM
    }
  });
}

const char* dmst_last_error(void) { return dmst::g_err.c_str(); }

const char* dmst_kernel_name(int32_t id) {
  return (id >= 0 && id < KK_COUNT) ? kKernelNames[id] : "";
}

const char* dmst_version(void) { return "dmst 0.2.0 sm_100a"; }

}  // extern "C"

// gim_api.cu — C-ABI entry points, device memory management and the host IMM driver of
// libgim (declared in include/gim.h). Host code is compiled with -ffp-contract=off so that the
// IMM doubles follow the evaluation order fixed in DESIGN.md (reading R21).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gim.h"
#include "gim_device.cuh"
#include "gim_internal.h"

using namespace gim;

namespace {

struct DevBuf {
  void* p = nullptr;
  uint64_t bytes = 0;
  template <class T> T* as() const { return static_cast<T*>(p); }
};

struct Seg {
  uint64_t gstart, lstart, count;   // global id range [gstart, gstart+count) at local index lstart
};

enum { CLS_RR = 0, CLS_GIANT, CLS_STORE, CLS_INV, CLS_SELECT, CLS_N };

#ifndef GIM_CHUNK_LOG2
#define GIM_CHUNK_LOG2 25
#endif
// RR ids per generation chunk (bounds the per-chunk buffers: ~3.5 GB at 2^25). Every chunk pays
// the K-RR / K-GIANT launch tails and one host sync: C5 (37.9M sets per IMM) 31.7 / 29.1 / 27.5 /
// 26.7 ms at 2^22 / 2^23 / 2^24 / 2^25; C3/C4 (rounds below 2^22 ids) unchanged
constexpr uint32_t kChunk = 1u << GIM_CHUNK_LOG2;
#ifndef GIM_ARGMAX_CTAS
#define GIM_ARGMAX_CTAS 4
#endif
constexpr int kArgmaxCtasPerSM = GIM_ARGMAX_CTAS;   // k_argmax grid = this x #SMs (256 threads each)
constexpr uint32_t kSelHead = 8;   // greedy steps before a bounded greedy's host stop check
// candidate argmax grid: one CTA per SM (measured 32 / 64 / 148 / 296 CTAs: C5 selection 4.29 /
// 3.97 / 3.75 / 4.05 ms, C3 1.80 / 1.75 / 1.71 / 1.70 ms)
#ifndef GIM_LOOK_SAFETY
#define GIM_LOOK_SAFETY 1.2
#endif
// lookahead: rounds m with u_prev < kLookSafety * (1 + eps') / 2^m are sampled together. Below 2,
// only the LAST merged round can fall in the band u in [thr_m, kLookSafety thr_m) where the probe
// may not settle it, and that round holds exactly its own T_m sets (no prefix, no drop); if it
// passes, its sets are the ones the round needs anyway. Measured 0.8 / 1.2 / 1.6: C3 18.18 /
// 17.49 / 17.42 ms, C5 23.01 / 22.26 / 22.68 ms, C4 4.44 / 4.11 / 4.10 ms.
constexpr double kLookSafety = GIM_LOOK_SAFETY;
#ifndef GIM_COVER_CTAS
#define GIM_COVER_CTAS 8
#endif
constexpr int kCoverCtasPerSM = GIM_COVER_CTAS;     // k_cover grid = this x #SMs (256 threads each)


}  // namespace

struct gim_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;   // speculative sampling overlapping a NodeSelection (gim_imm)
  bool own_stream = false;
  int speculate = 0;                // GIM_OPT_SPECULATE (measured: no gain)
  cudaEvent_t ev_cnt_copied = nullptr, ev_sel_done = nullptr;
  bool sel_pending = false;         // a selection is in flight on `stream`
  uint64_t set_limit = ~0ull;       // cover skips local sets >= this (after a tail truncation)
  bool truncated = false;
  int num_sms = 148;
  std::string err;
  gim_alloc_fn afn = nullptr;
  gim_free_fn ffn = nullptr;
  void* auser = nullptr;
  // graph (O1)
  bool graph = false;
  uint32_t n = 0;
  uint64_t m = 0;
  int model = 0, scheme = 0;
  float p_uniform = 0.f;
  uint64_t thr_uniform = 0;
  DevBuf row_ptr, src, thr_edge;   // row_ptr holds [n + 1] row pointers, then (WC) [n + 1] thresholds
  uint32_t* thr_node = nullptr;     // WC threshold per node: row_ptr + n + 1 (one L2 window covers both)
  int l2_persist = 0;               // GIM_OPT_L2_PERSIST (measured: C5 store 3.8 -> 5.9 ms, index 6.2 -> 10.5 ms with it)
  DevBuf out_ptr, out_dst, out_in, thr_wc;   // out-CSR for gim_mc_spread (built on first use)
  bool out_valid = false;
  // MRIM (readings R26-R28): rounds T; pair ids t*n + u index the count / index / selection
  // arrays (n*T of them); the T rounds of MRIM set i are the consecutive standard ids i*T + t
  uint32_t rounds = 1;
  // sharding
  int rank = 0, world = 1;
  void* nccl = nullptr;              // communicator owned by the ctx (gim_set_nccl)
  gim_allreduce_fn arfn = nullptr;
  void* aruser = nullptr;
  gim_allgather_fn agfn = nullptr;   // set: replicated-pool protocol (no per-step collectives)
  void* aguser = nullptr;
  gim_reducescatter_fn rsfn = nullptr;   // set (with arfn, no agfn): node-sharded selection
  void* rsuser = nullptr;
  DevBuf rs_gcnt, rs_dshard, rs_keys, rs_kx;   // node-sharded selection: shard counts/decrements, keys
  int force_coll = 0;                  // GIM_OPT_FORCE_COLLECTIVES: world-1 runs the P > 1 protocol
  DevBuf ag_small, ag_send, ag_recv;
  // pool (O6)
  bool have_seed = false;
  uint64_t seed = 0, T_global = 0, nsets = 0, pool_len = 0;
  std::vector<Seg> segs;
  DevBuf pool, offsets, count_total;
  // generation scratch
  DevBuf giant2_list;             // sets the shared-memory giant pass hands to the global pass
  DevBuf sizes, soff, giant_list, retry_list, item_list, scan_out, scan_tmp, staging, ctr, dump, lt_spill, esc_list;
  DevBuf bitmaps, gqueues;
  DevBuf spill;                   // per-warp global queue + hash of the warp kernels' spill tier (kEmpty when unused)
  DevBuf lane_spill;              // R31 lane kernel: per-lane members beyond the shared 32
  uint32_t skip_lane_cap = 32;    // R31 lane kernel: set size limit (GIM_OPT_SKIP_LANE_CAP)
  uint32_t giant_slots = 0;
  uint32_t giant_n = 0;             // n the giant slots were sized for (reused while n <= giant_n)
  int giant_nt_opt = 0;             // GIM_OPT_GIANT_NT: 0 auto, else threads per giant CTA
  int fresh_final = 0;              // GIM_OPT_FRESH_FINAL (reading R29)
  int sel_persistent = 0;           // GIM_OPT_SELECT_PERSISTENT: k steps in one cooperative launch
  DevBuf sel_bar;
  double giant_per_slot = 0.0;      // giant sets per default slot in the previous chunk
  bool dense_sets = false;          // some chunk had >= 12 giant sets per slot (sticky: spill tier on)
  bool giant_cap_reached = false;
  uint64_t stage_cap = 0;
  int lt_bps = 0;                  // resident K-LT CTAs per SM on this context's device
  int giant_sq = 0;                // GIM_OPT_GIANT_SHARED: shared-memory first giant pass (measured neutral: off)
  int skip = 0;                    // geometric-skip RNG contract (GIM_OPT_SKIP, reading R31)
  int skip_bps = 0;                // resident k_skip_lane CTAs per SM
  int skip_lane = -1;              // skip: -1 auto (lane kernel first for big chunks), 0 / 1
  int64_t spill_cap = -1;          // spill-tier set size limit (GIM_OPT_SPILL; -1 = auto)
  uint32_t spill_cap_eff = 0;      // the cap of the current generate call (<= qcap: no spill)
  uint32_t max_deg = 0;            // largest in-degree of the loaded graph
  DevBuf skip_tab;                 // skip: log centers L_k, R_k (2 x 184 doubles) + inv per in-degree
  bool skip_tab_valid = false;
  GenCounters* h_ctr = nullptr;   // pinned
  uint64_t* h_u64 = nullptr;      // pinned scratch
  unsigned long long* h_keys = nullptr;   // pinned selection keys
  uint32_t h_keys_cap = 0;
  // selection scratch
  DevBuf cnt, covered, keys, dec;
  // segmented inverted index (one segment per generation chunk; rebuilt whole when invalid)
  struct InvSeg {
    DevBuf off, inv;
  };
  std::vector<InvSeg> iseg;
  bool inv_valid = true;
  // lazy segments: sets [pend_set0, nsets) (elements [pend_e0, pool_len)) are not indexed yet;
  // the next selection indexes them as ONE segment (several IMM rounds whose selections stopped
  // at their first step share one O(n) histogram/scan pass)
  bool inv_pending = false;
  uint64_t pend_set0 = 0, pend_e0 = 0;
  int inv_segmented = 1;        // GIM_OPT_INV_SEGMENTS
  DevBuf cnt_snap;              // count_total at the last indexed chunk
  DevBuf seg_desc;              // device InvSegDev[kMaxInvSeg] + uint32 nseg
  DevBuf cand;                  // argmax candidates + hist[33] + tau_p1 + ncand
  int use_cand = 1;             // GIM_OPT_ARGMAX_CAND
  uint32_t sel_fused = 0;       // GIM_OPT_SELECT_FUSED: candidate cap of the fused steps (0 = off)
  bool force_unfused = false;   // the fused selection failed its certificate: redo unfused
  bool sel_fused_used = false;  // the pending selection ran fused
  bool sel_cand_used = false;   // the pending selection took candidate argmaxes (certificate checked)
  DevBuf sel_done;              // fused steps: per-step completion tickets + the fail flag
  int fused_ctas = 2;           // fused cover grid = this x #SMs (fewer tickets per step)
  uint32_t sel_coop = 0;        // GIM_OPT_SELECT_COOP: candidate cap of the cooperative selection (0 = off)
  DevBuf cmap, cdec;            // cooperative selection: node -> candidate index (kEmpty), decrement rings
  DevBuf sel_ctl;               // SelCtl of the bounded greedy (IMM estimation rounds)
  DevBuf probe;                 // first-step argmax key of gim_imm's probe
  uint64_t sel_cstar = 0;       // smallest passing covered count of the running round (0 = off)
  uint32_t last_sel_steps = 0;  // greedy steps the last selection ran
  int inv_passes = 0;           // GIM_OPT_INV_PASSES: node-range passes of the index scatter (0 = auto)
  int inv_sort = -1;            // GIM_OPT_INV_SORT: -1 auto (n * 4 > 64 MB), 0 scatter, 1 sort
  uint32_t chunk = 0;           // GIM_OPT_CHUNK: RR ids per generation chunk (0 = kChunk)
  DevBuf isort_keys, isort_vals, isort_tmp;   // sort-based segments: sorted keys, set ids, CUB scratch
  int imm_early_exit = 1;       // GIM_OPT_IMM_EARLY_EXIT
  int imm_lookahead = 1;        // GIM_OPT_IMM_LOOKAHEAD
  int sel_small = 1;            // GIM_OPT_SELECT_CTA: single-CTA selection when the counts fit in shared memory
  int sel_cluster = 0;          // GIM_OPT_SELECT_CLUSTER: the cluster version for n up to 8x that (measured slower)
  uint64_t cmap_n = 0;          // nodes covered by cmap (kEmpty-initialised)
  // options
  int force_giant = 0, profile = 0;
  int mb_chains = 8;            // GIM_OPT_MB_CHAINS: Philox chains per thread in the microbenchmark
  int ic_lane = -1;             // GIM_OPT_IC_LANE: -1 auto (mean coins per set), 0 off, 1 on
  double coins_per_set = 0.0;   // running estimate from previous chunks
  uint32_t qcap = kQMax;
  uint64_t staging_init = 0;
  gim_stats st{};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[CLS_N];
  std::vector<cudaEvent_t> ev_free;   // recycled timing events
  // CUDA graph of the k-step selection loop (P = 1), valid while its key is unchanged
  cudaGraphExec_t sel_exec = nullptr;    // fused selection graph
  std::vector<cudaGraphExec_t> sel_parts;   // default selection: consecutive graphs of greedy steps
  cudaGraphExec_t p_exec = nullptr;      // P > 1 selection loop with the native NCCL exchange
  std::vector<uintptr_t> p_key;
  std::vector<uintptr_t> sel_key;
  int use_graph = 1;
};

namespace {

uint64_t nsp(const gim_ctx* c) { return (uint64_t)c->n * c->rounds; }   // counted elements

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

gim_status fail(gim_ctx* c, gim_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

gim_status fail_cuda(gim_ctx* c, const char* what, cudaError_t e) {
  cudaGetLastError();
  return fail(c, GIM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                          \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return fail_cuda(c, #call, _e); \
  } while (0)
#define TRY(call)                      \
  do {                                 \
    gim_status _s = (call);            \
    if (_s != GIM_OK) return _s;       \
  } while (0)

void dfree(gim_ctx* c, DevBuf& b) {
  if (b.p) {
    if (c->ffn) c->ffn(b.p, c->stream, c->auser);
    else cudaFreeAsync(b.p, c->stream);
  }
  b = DevBuf{};
}

gim_status dalloc(gim_ctx* c, DevBuf& b, uint64_t bytes) {
  dfree(c, b);
  bytes = std::max<uint64_t>((bytes + 255) & ~uint64_t(255), 256);
  void* p = nullptr;
  if (c->afn) {
    p = c->afn(bytes, c->stream, c->auser);
    if (!p) return fail(c, GIM_ENOMEM, "allocator callback failed for " + std::to_string(bytes) + " bytes");
  } else {
    cudaError_t e = cudaMallocAsync(&p, bytes, c->stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(c, GIM_ENOMEM, "cudaMallocAsync(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    }
  }
  b.p = p;
  b.bytes = bytes;
  c->st.n_allocs++;
  return GIM_OK;
}

// Capacity >= bytes; contents are NOT preserved.
gim_status ensure(gim_ctx* c, DevBuf& b, uint64_t bytes) {
  if (b.bytes >= bytes && b.p) return GIM_OK;
  return dalloc(c, b, std::max<uint64_t>(bytes, b.bytes + b.bytes / 2));
}

// Capacity >= bytes; the first `keep` bytes are preserved.
gim_status grow_keep(gim_ctx* c, DevBuf& b, uint64_t bytes, uint64_t keep) {
  if (b.bytes >= bytes && b.p) return GIM_OK;
  DevBuf nb;
  TRY(dalloc(c, nb, std::max<uint64_t>(bytes, b.bytes * 2)));
  if (keep && b.p) CK(cudaMemcpyAsync(nb.p, b.p, keep, cudaMemcpyDeviceToDevice, c->stream));
  dfree(c, b);
  b = nb;
  return GIM_OK;
}

// ---- profiling (CUDA events on the ctx stream, resolved at sync points) ----------------------
struct Prof {
  gim_ctx* c;
  int cls;
  cudaEvent_t a = nullptr, b = nullptr;
  static cudaEvent_t take(gim_ctx* c) {
    cudaEvent_t e = nullptr;
    if (!c->ev_free.empty()) {
      e = c->ev_free.back();
      c->ev_free.pop_back();
    } else {
      cudaEventCreate(&e);
    }
    return e;
  }
  Prof(gim_ctx* c_, int cls_) : c(c_), cls(cls_) {
    if (c->profile) {
      a = take(c);
      b = take(c);
      cudaEventRecord(a, c->stream);
    }
  }
  ~Prof() {
    if (a) {
      cudaEventRecord(b, c->stream);
      c->ev[cls].emplace_back(a, b);
    }
  }
};

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

gim_status sync(gim_ctx* c) {
  const double t0 = now_ms();
  const cudaError_t se = cudaStreamSynchronize(c->stream);
  c->st.host_ms_sync += now_ms() - t0;
  c->st.n_syncs++;
  CK(se);
  double* acc[CLS_N] = {&c->st.ms_rr, &c->st.ms_giant, &c->st.ms_store, &c->st.ms_inv, &c->st.ms_select};
  for (int k = 0; k < CLS_N; ++k) {
    for (auto& pr : c->ev[k]) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) *acc[k] += ms;
      c->ev_free.push_back(pr.first);
      c->ev_free.push_back(pr.second);
    }
    c->ev[k].clear();
  }
  cudaGetLastError();
  return GIM_OK;
}

gim_status launched(gim_ctx* c, cudaError_t e, const char* what, int n = 1) {
  c->st.launches += n;
  if (e != cudaSuccess) return fail_cuda(c, what, e);
  return GIM_OK;
}

// ---- segmented inverted index ----------------------------------------------------------------
void drop_inv(gim_ctx* c) {
  for (auto& sg : c->iseg) {
    dfree(c, sg.off);
    dfree(c, sg.inv);
  }
  c->iseg.clear();
}

// Index local sets [set0, set1) (pool elements [e0, e1)) as a new segment; the per-node
// histogram is count_total - cnt_snap (no extra atomics), then scan + cursor scatter.
gim_status build_inv_segment(gim_ctx* c, uint64_t set0, uint64_t set1, uint64_t e0, uint64_t e1) {
  const uint64_t n = nsp(c);
  if (e1 - e0 >= 0xFFFFFFFFull) return fail(c, GIM_ENOMEM, "an index segment must hold < 2^32 RR elements");
  gim_ctx::InvSeg sg;
  TRY(dalloc(c, sg.off, (n + 1) * 4));
  TRY(dalloc(c, sg.inv, std::max<uint64_t>(e1 - e0, 1) * 4));
  TRY(ensure(c, c->scan_tmp, (scan_tiles(n) + 2) * 8));
  Prof pf(c, CLS_INV);
  // sort-based segment (GIM_OPT_INV_SORT; auto: when the per-node cursors exceed 64 MB, i.e. far
  // beyond the L2, so that each scatter step would be a random DRAM read-modify-write)
  const bool sort_mode = set1 > set0 && (c->inv_sort == 1 || (c->inv_sort == -1 && n * 4 > (64ull << 20)));
  int nl = 0;
  // histogram count_total - snap and its scan in one pass pair: list starts (scatter: advanced to
  // the list ends by the scatter's atomics) or list ends (sorted segment)
  cudaError_t e = launch_seg_scan(c->count_total.as<uint32_t>(), c->cnt_snap.as<uint32_t>(), n, sg.off.as<uint32_t>(),
                                  sort_mode, c->scan_tmp.as<uint64_t>(), c->scan_tmp.as<uint64_t>() + scan_tiles(n) + 1,
                                  c->stream, &nl);
  TRY(launched(c, e, "segment scan", nl));
  if (sort_mode) {
    const uint64_t E = e1 - e0;
    uint32_t nbits = 1;
    while (nbits < 32 && (1ull << nbits) < n) ++nbits;
    const size_t cub_bytes = inv_sort_tmp_bytes(E, nbits);
    TRY(ensure(c, c->isort_keys, E * 4));
    TRY(ensure(c, c->isort_vals, E * 4));
    TRY(ensure(c, c->isort_tmp, cub_bytes + 256));
    e = launch_inv_sort(c->offsets.as<uint64_t>(), c->pool.as<uint32_t>(), (uint32_t)set0, (uint32_t)set1, e0, E, nbits,
                        c->isort_keys.as<uint32_t>(), c->isort_vals.as<uint32_t>(), c->isort_tmp.p, cub_bytes,
                        sg.inv.as<uint32_t>(), c->num_sms * 8, c->stream, &nl);
    TRY(launched(c, e, "inv sort", nl));
  } else if (set1 > set0) {
    // node-range passes (GIM_OPT_INV_PASSES; default 1: measured C5 index 5.66 ms with one pass
    // vs 6.19 ms with one pass per 32 MB of cursors — the re-reads of the pool cost more than the
    // L2-resident atomics save)
    const int passes = c->inv_passes > 0 ? c->inv_passes : 1;
    e = launch_inv_scatter(c->offsets.as<uint64_t>(), c->pool.as<uint32_t>(), (uint32_t)set0, (uint32_t)set1,
                           sg.off.as<uint32_t>(), sg.inv.as<uint32_t>(), c->num_sms * 8, c->stream, (uint32_t)n,
                           passes, &nl);
    TRY(launched(c, e, "k_inv_scatter", nl));
  }
  c->iseg.push_back(std::move(sg));
  return GIM_OK;
}

// Index the pending (unindexed) sets as one new segment, or rebuild the whole index as one
// segment when it is invalid or a new segment would not fit (kMaxInvSeg, 2^32 elements).
gim_status flush_inv(gim_ctx* c) {
  if (c->inv_valid && c->inv_pending) {
    if (c->iseg.size() < (size_t)kMaxInvSeg && c->pool_len - c->pend_e0 < 0xFFFFFFFFull)
      TRY(build_inv_segment(c, c->pend_set0, c->nsets, c->pend_e0, c->pool_len));
    else
      c->inv_valid = false;
  }
  c->inv_pending = false;
  if (!c->inv_valid) {                          // one segment over the whole local pool
    drop_inv(c);
    CK(cudaMemsetAsync(c->cnt_snap.p, 0, nsp(c) * 4, c->stream));
    TRY(build_inv_segment(c, 0, c->nsets, 0, c->pool_len));
    c->inv_valid = true;
    c->set_limit = ~0ull;
    c->truncated = false;
  }
  return GIM_OK;
}

// ---- pool management ------------------------------------------------------------------------
gim_status reset_pool(gim_ctx* c, uint64_t seed) {
  c->have_seed = true;
  c->seed = seed;
  c->T_global = 0;
  c->nsets = 0;
  c->pool_len = 0;
  c->segs.clear();
  TRY(ensure(c, c->count_total, nsp(c) * 4));
  CK(cudaMemsetAsync(c->count_total.p, 0, nsp(c) * 4, c->stream));
  TRY(ensure(c, c->offsets, 8 * 1024));
  CK(cudaMemsetAsync(c->offsets.p, 0, 8, c->stream));
  drop_inv(c);
  c->inv_valid = true;
  c->inv_pending = false;
  c->set_limit = ~0ull;
  c->truncated = false;
  TRY(ensure(c, c->cnt_snap, nsp(c) * 4));
  CK(cudaMemsetAsync(c->cnt_snap.p, 0, nsp(c) * 4, c->stream));
  return GIM_OK;
}

gim_status ensure_giant_slots(gim_ctx* c, uint32_t want) {
  if (c->giant_slots >= want || c->giant_cap_reached) return GIM_OK;
  const uint64_t words = ((uint64_t)c->n + 31) / 32;
  const uint64_t per_slot = words * 4 + (uint64_t)c->n * 4;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  uint64_t cap = std::max<uint64_t>(1, (uint64_t)(free_b / 8) / std::max<uint64_t>(per_slot, 1));
  uint32_t slots = (uint32_t)std::min<uint64_t>({(uint64_t)want, cap});
  if (slots < want) c->giant_cap_reached = true;
  if (slots <= c->giant_slots) return GIM_OK;
  TRY(dalloc(c, c->bitmaps, words * 4 * slots));
  CK(cudaMemsetAsync(c->bitmaps.p, 0, words * 4 * slots, c->stream));
  TRY(dalloc(c, c->gqueues, (uint64_t)c->n * 4 * slots));
  CK(cudaMemsetAsync(c->gqueues.p, 0xFF, (uint64_t)c->n * 4 * slots, c->stream));   // kEmpty
  c->giant_slots = slots;
  c->giant_n = c->n;
  return GIM_OK;
}

// L2 persisting window over the row pointers (+ WC thresholds): every BFS level of every RR set
// starts with these loads, on the critical path of deep sets; src (read only for live edges) and
// the pool stream through the rest of the L2. Window and set-aside capped by the device limits;
// hitRatio scales down when the rows exceed the set-aside (C5: 333 MB).
void set_l2_window(gim_ctx* c) {
  cudaStreamAttrValue v{};
  if (c->l2_persist && c->graph) {
    int max_win = 0, max_persist = 0;
    cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, c->device);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c->device);
    const size_t bytes = std::min<size_t>(c->row_ptr.bytes, (size_t)std::max(max_win, 0));
    if (bytes > 0 && max_persist > 0) {
      const size_t persist = std::min<size_t>(bytes, (size_t)max_persist);
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist);
      v.accessPolicyWindow.base_ptr = c->row_ptr.p;
      v.accessPolicyWindow.num_bytes = bytes;
      v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)persist / (double)bytes);
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    }
  }
  cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &v);   // num_bytes 0: off
  cudaGetLastError();
}

RRParams base_params(gim_ctx* c) {
  RRParams p{};
  p.n = c->n;
  p.row_ptr = c->row_ptr.as<uint32_t>();
  p.src = c->src.as<uint32_t>();
  p.thr_node = c->thr_node;
  p.thr_edge = c->thr_edge.as<uint64_t>();
  p.thr_uniform = c->thr_uniform;
  p.p_uniform = c->p_uniform;
  p.skip_tab = c->skip_tab.as<double>();
  p.spill = c->spill.as<uint32_t>();
  p.spill_cap = c->spill_cap_eff;
  p.seed = c->seed;
  {
    uint32_t k0 = (uint32_t)c->seed, k1 = (uint32_t)(c->seed >> 32);
    for (int r = 0; r < 10; ++r) {
      p.rk[2 * r] = k0;
      p.rk[2 * r + 1] = k1;
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
  }
  p.sizes = c->sizes.as<uint32_t>();
  p.soff = c->soff.as<uint64_t>();
  p.staging = c->staging.as<uint32_t>();
  p.stage_cap = c->stage_cap;
  p.ctr = c->ctr.as<GenCounters>();
  p.giant_recs = c->giant_list.as<GiantRec>();
  p.giant2_recs = c->giant2_list.as<GiantRec>();
  p.dump = c->dump.as<uint32_t>();
  p.dump_cap = c->dump.bytes / 4;
  p.retry_list = c->retry_list.as<uint32_t>();
  p.qcap = c->qcap;
  p.lt_spill = c->lt_spill.as<uint32_t>();
  p.force_giant = c->force_giant;
  p.rounds = c->rounds;
  return p;
}

gim_status read_ctr(gim_ctx* c) {
  CK(cudaMemcpyAsync(c->h_ctr, c->ctr.p, sizeof(GenCounters), cudaMemcpyDeviceToHost, c->stream));
  return sync(c);
}

// Generate local RR sets for global ids [gstart, gstart + cnt) and append them to the pool.
gim_status gen_chunk(gim_ctx* c, uint64_t gstart, uint32_t cnt) {
  TRY(ensure(c, c->sizes, (uint64_t)cnt * 4));
  TRY(ensure(c, c->soff, (uint64_t)cnt * 8));
  TRY(ensure(c, c->giant_list, (uint64_t)cnt * sizeof(GiantRec)));
  TRY(ensure(c, c->giant2_list, (uint64_t)cnt * sizeof(GiantRec)));
  TRY(ensure(c, c->dump, std::max<uint64_t>((uint64_t)cnt * 8, 1u << 20) * 4));
  TRY(ensure(c, c->retry_list, (uint64_t)cnt * 4));
  TRY(ensure(c, c->item_list, (uint64_t)cnt * 4));
  TRY(ensure(c, c->esc_list, (uint64_t)cnt * 4));
  TRY(ensure(c, c->scan_out, ((uint64_t)cnt + 1) * 8));
  TRY(ensure(c, c->scan_tmp, (scan_tiles(cnt) + 2) * 8));
  TRY(ensure(c, c->ctr, sizeof(GenCounters)));
  if (c->stage_cap == 0 && c->staging_init) {
    TRY(dalloc(c, c->staging, c->staging_init * 4));
    c->stage_cap = c->staging_init;
  } else {
    const double mean = c->nsets ? (double)c->pool_len / (double)c->nsets : 32.0;
    const uint64_t want = (uint64_t)(mean * (double)cnt * 1.25) + (1u << 20) +
                          (uint64_t)c->num_sms * 64 * kStageChunk;   // per-warp chunk slack
    if (c->stage_cap < want && !c->staging_init) {
      TRY(dalloc(c, c->staging, want * 4));
      c->stage_cap = c->staging.bytes / 4;
    }
  }
  CK(cudaMemsetAsync(c->ctr.p, 0, sizeof(GenCounters), c->stream));
  if (c->model == MODEL_IC) {
    // spill tier of the warp kernels. Auto: WC sets grow by ~1 live in-edge per node (deep,
    // narrow: kept in flight beside the small ones in the warp's spill tier); uniform-p sets
    // become big through hubs of thousands of live in-edges (wide: better spread over a CTA)
    // (per-edge coins: no spill when giant sets are rare — a giant set's ~10^5 coins on one warp
    // finish after the rest of the launch; measured C3 sampling 16.5 vs 14.4 ms with K-GIANT;
    // spill up to 2048 nodes when the previous chunk had many giant sets per K-GIANT slot, the
    // dense graphs where K-GIANT is throughput-bound: B32 sampling + giant 76.8 vs 79.7 ms)
    const uint32_t coin_cap = c->dense_sets ? 2048u : 0u;
    uint32_t cap = c->spill_cap >= 0 ? (uint32_t)c->spill_cap
                                     : (!c->skip ? coin_cap : (c->scheme == W_WC ? kSpillQ : 2048u));
    cap = std::min<uint32_t>(cap, kSpillQ);
    c->spill_cap_eff = cap;
    if (cap > c->qcap) {
      const uint64_t need = (uint64_t)c->num_sms * kRRBlocksPerSM * kRRWarps * spill_words_per_warp() * 4;
      if (c->spill.bytes < need) {             // hash halves must start (and stay) empty
        TRY(dalloc(c, c->spill, need));
        CK(cudaMemsetAsync(c->spill.p, 0xFF, need, c->stream));
      }
    }
  } else {
    c->spill_cap_eff = 0;
  }
  if (c->skip && !c->skip_tab_valid) {         // R31: log-center tables + 1/ln(1-p) per in-degree
    const uint64_t nd = (c->scheme == W_WC ? (uint64_t)c->max_deg : 0) + 2;
    TRY(ensure(c, c->skip_tab, (2 * kSkipTabK + nd) * 8));
    TRY(launched(c, launch_skip_tables(c->scheme, c->p_uniform, c->max_deg, c->skip_tab.as<double>(),
                                       c->stream), "k_skip_tables"));
    c->skip_tab_valid = true;
  }
  RRParams p = base_params(c);
  p.id_base = gstart;
  p.count = cnt;
  p.item_list = nullptr;
  int rr_grid = c->num_sms * kRRBlocksPerSM;   // persistent CTAs, 8 warps each
  if (c->model == MODEL_LT) {
    if (!c->lt_bps) c->lt_bps = lt_blocks_per_sm();   // per context (= per device)
    rr_grid = c->num_sms * c->lt_bps;
    TRY(ensure(c, c->lt_spill, (uint64_t)rr_grid * kLtWarps * (kLtCap2 - kLtCap) * 32 * 4));
    p.lt_spill = c->lt_spill.as<uint32_t>();
  }
  // giant CTA width: narrow (more sets in flight) when the previous chunk had many giant sets
  // per default slot — dense graphs, where K-GIANT otherwise dominates
  const int giant_nt = c->giant_nt_opt ? c->giant_nt_opt
                                       : (c->giant_per_slot >= 12.0 ? kGiantThreadsNarrow : kGiantThreads);
  const uint32_t giant_grid = (uint32_t)(1024 / giant_nt) * (uint32_t)c->num_sms;
  TRY(ensure_giant_slots(c, giant_grid));
  const uint64_t bm_words = ((uint64_t)c->n + 31) / 32;
  // warp kernel, then the giant kernel unconditionally (it reads the giant count on the device
  // and exits at once when there is none), then the size scan: one host sync per chunk.
  // IC with tiny sets: the lane kernel runs first and escalates big sets to the warp kernel
  // (small chunks stay on the warp path: with few sets in flight, one lane per set exposes each
  // set's whole chain of dependent loads)
  const bool lane_first = c->model == MODEL_IC &&
                          (c->ic_lane == 1 || (c->ic_lane == -1 && c->coins_per_set > 0.0 &&
                                               c->coins_per_set < 160.0 && cnt >= (1u << 17)));
  auto run_pass = [&](const RRParams& pp) -> gim_status {
    if (c->skip) {                             // R31: lane kernel -> warp kernel -> giant kernel
      const bool sl = c->skip_lane == 1 || (c->skip_lane == -1 && cnt >= (1u << 15));
      RRParams pw = pp;
      if (sl) {
        if (!c->skip_bps) c->skip_bps = skip_lane_blocks_per_sm();
        RRParams pl = pp;
        pl.esc_list = c->esc_list.as<uint32_t>();
        pl.lane_cap = c->skip_lane_cap;
        if (c->skip_lane_cap > 32) {
          TRY(ensure(c, c->lane_spill, skip_lane_spill_words(c->num_sms * c->skip_bps) * 4));
          pl.lane_spill = c->lane_spill.as<uint32_t>();
        }
        {
          Prof pf(c, CLS_RR);
          TRY(launched(c, launch_skip_lane(c->scheme, pl, c->num_sms * c->skip_bps, c->stream), "k_skip_lane"));
          c->st.n_rr_launches++;
        }
        pw.item_list = c->esc_list.as<uint32_t>();
        pw.count_ptr = &c->ctr.as<GenCounters>()->esc_count;
      }
      {
        Prof pf(c, CLS_RR);
        TRY(launched(c, launch_skip_warp(c->scheme, pw, c->num_sms * kRRBlocksPerSM, c->stream), "k_skip_warp"));
        c->st.n_rr_launches++;
      }
      {
        Prof pf(c, CLS_GIANT);
        TRY(launched(c, launch_skip_giant(c->scheme, pp, (int)c->giant_slots, c->bitmaps.as<uint32_t>(),
                                          c->gqueues.as<uint32_t>(), bm_words, c->stream), "k_skip_giant"));
        c->st.n_giant_launches++;
      }
      return GIM_OK;
    }
    if (lane_first) {
      RRParams pl = pp;
      pl.esc_list = c->esc_list.as<uint32_t>();
      {
        Prof pf(c, CLS_RR);
        TRY(launched(c, launch_rr_ic_lane(c->scheme, pl, c->num_sms * kIcLaneBlocksPerSM, c->stream), "k_rr_ic_lane"));
        c->st.n_rr_launches++;
      }
      RRParams pw = pp;                        // the warp kernel replays the escalated items
      pw.item_list = c->esc_list.as<uint32_t>();
      pw.count_ptr = &c->ctr.as<GenCounters>()->esc_count;
      Prof pf(c, CLS_RR);
      TRY(launched(c, launch_rr_warp(c->model, c->scheme, pw, rr_grid, c->stream), "k_rr_warp(escalated)"));
      c->st.n_rr_launches++;
    } else {
      Prof pf(c, CLS_RR);
      TRY(launched(c, launch_rr_warp(c->model, c->scheme, pp, rr_grid, c->stream), "k_rr_warp"));
      c->st.n_rr_launches++;
    }
    {
      Prof pf(c, CLS_GIANT);
      // wide CTAs: a shared-memory pass first (sets up to kGQS nodes), the global-bitmap pass
      // for the sets it hands over; narrow CTAs (many giant sets): the global pass directly
      const bool sq = c->giant_sq && giant_nt == kGiantThreads;
      if (sq) {
        TRY(launched(c, launch_rr_giant(c->model, c->scheme, pp, c->num_sms * kGiantBlocksPerSM, nullptr, nullptr, 0,
                                        c->stream, giant_nt, true), "k_rr_giant(shared)"));
        c->st.n_giant_launches++;
      }
      RRParams pg = pp;
      pg.giant_pass2 = sq ? 1 : 0;               // else the global pass reads the first list
      TRY(launched(c, launch_rr_giant(c->model, c->scheme, pg, (int)std::min(c->giant_slots, giant_grid),
                                      c->bitmaps.as<uint32_t>(), c->gqueues.as<uint32_t>(), bm_words,
                                      c->stream, giant_nt, false), "k_rr_giant"));
      c->st.n_giant_launches++;
    }
    return GIM_OK;
  };
  TRY(run_pass(p));
  {
    Prof pf(c, CLS_STORE);
    int nl = 0;
    cudaError_t e = launch_scan_u32(c->sizes.as<uint32_t>(), cnt, c->scan_out.as<uint64_t>(),
                                    c->scan_tmp.as<uint64_t>(), c->scan_tmp.as<uint64_t>() + scan_tiles(cnt) + 1,
                                    c->stream, &nl);
    TRY(launched(c, e, "scan(sizes)", nl));
  }
  CK(cudaMemcpyAsync(c->h_u64, c->scan_out.as<uint64_t>() + cnt, 8, cudaMemcpyDeviceToHost, c->stream));
  TRY(read_ctr(c));
  c->st.giant_sets += c->h_ctr->giant_count;
  if (cnt >= 4096)
    c->giant_per_slot = (double)c->h_ctr->giant_count / ((double)kGiantBlocksPerSM * (double)c->num_sms);
  if (c->giant_per_slot >= 12.0) c->dense_sets = true;
  for (int iter = 0; c->h_ctr->retry_count; ++iter) {
    if (iter > 40) return fail(c, GIM_ENOMEM, "staging retry loop did not converge");
    // staging overflow: grow (keep the part already written) and redo the failed items
    const uint32_t retries = c->h_ctr->retry_count;
    const uint64_t old_cap = c->stage_cap;
    TRY(grow_keep(c, c->staging, old_cap * 4 * 2, old_cap * 4));
    c->stage_cap = c->staging.bytes / 4;
    CK(cudaMemcpyAsync(c->item_list.p, c->retry_list.p, (uint64_t)retries * 4, cudaMemcpyDeviceToDevice, c->stream));
    GenCounters h = *c->h_ctr;
    h.stage_tail = old_cap;
    h.claim = h.claim_giant = h.giant_count = h.retry_count = 0;
    h.giant2_count = h.claim_giant2 = 0;
    h.claim_lane = h.esc_count = 0;
    h.dump_tail = 0;
    *c->h_ctr = h;
    CK(cudaMemcpyAsync(c->ctr.p, c->h_ctr, sizeof(GenCounters), cudaMemcpyHostToDevice, c->stream));
    RRParams pr = base_params(c);
    pr.lt_spill = c->lt_spill.as<uint32_t>();
    pr.id_base = gstart;
    pr.count = retries;
    pr.item_list = c->item_list.as<uint32_t>();
    TRY(run_pass(pr));
    TRY(read_ctr(c));
    c->st.giant_sets += c->h_ctr->giant_count;
    if (!c->h_ctr->retry_count) {             // sizes complete: redo the scan
      Prof pf(c, CLS_STORE);
      int nl = 0;
      cudaError_t e = launch_scan_u32(c->sizes.as<uint32_t>(), cnt, c->scan_out.as<uint64_t>(),
                                      c->scan_tmp.as<uint64_t>(), c->scan_tmp.as<uint64_t>() + scan_tiles(cnt) + 1,
                                      c->stream, &nl);
      TRY(launched(c, e, "scan(sizes)", nl));
      CK(cudaMemcpyAsync(c->h_u64, c->scan_out.as<uint64_t>() + cnt, 8, cudaMemcpyDeviceToHost, c->stream));
      TRY(sync(c));
    }
  }
#ifdef GIM_GIANT_TRACE
  giant_trace_dump(c->stream);
#endif
#ifdef GIM_WINSTAT
  fprintf(stderr, "WINSTAT sets=%u windows=%llu valid_groups=%llu hub_steps=%llu coins=%llu\n", cnt,
          c->h_ctr->dbg[0], c->h_ctr->dbg[1], c->h_ctr->dbg[2], c->h_ctr->coins);
#endif
  c->st.coins += c->h_ctr->coins;
  c->st.live_edges += c->h_ctr->live;
  if (cnt >= 4096)   // running mean coins per set drives the lane/warp choice of later chunks
    c->coins_per_set = (double)(c->h_ctr->coins + c->h_ctr->coins_giant) / (double)cnt;
  c->st.coins_giant += c->h_ctr->coins_giant;
  c->st.live_giant += c->h_ctr->live_giant;
  // two-pass storage: sizes were scanned above; compacting copy + count_total
  const uint64_t total = c->h_u64[0];
  // k_store totals the members of 32 consecutive sets in uint32 (a window lies inside the chunk)
  if (total >= 0xFFFFFFFFull) return fail(c, GIM_ENOMEM, "a generate chunk must hold < 2^32 RR elements");
  if (c->sel_pending && (c->pool.bytes < (c->pool_len + total) * 4 || c->offsets.bytes < (c->nsets + cnt + 1) * 8))
    CK(cudaEventSynchronize(c->ev_sel_done));   // the running selection reads pool/offsets
  TRY(grow_keep(c, c->pool, (c->pool_len + total) * 4, c->pool_len * 4));
  TRY(grow_keep(c, c->offsets, (c->nsets + cnt + 1) * 8, (c->nsets + 1) * 8));
  {
    Prof pf(c, CLS_STORE);
    TRY(launched(c, launch_store(c->staging.as<uint32_t>(), c->sizes.as<uint32_t>(), c->soff.as<uint64_t>(),
                                 c->scan_out.as<uint64_t>(), cnt, c->pool_len, c->pool.as<uint32_t>(),
                                 c->offsets.as<uint64_t>() + c->nsets, c->count_total.as<uint32_t>(),
                                 c->rounds, (uint32_t)(gstart % c->rounds), c->n, c->num_sms * 8, c->stream),
                    "k_store"));
  }
  c->segs.push_back(Seg{gstart, c->nsets, cnt});
  c->nsets += cnt;
  c->pool_len += total;
  c->st.rr_sets += cnt;
  c->st.rr_elements += total;
  return GIM_OK;
}

gim_status truncate_pool(gim_ctx* c, uint64_t theta) {
  uint64_t keep_sets = 0;
  std::vector<Seg> kept;
  for (const Seg& s : c->segs) {
    if (s.gstart >= theta) break;
    const uint64_t k = std::min<uint64_t>(s.count, theta - s.gstart);
    kept.push_back(Seg{s.gstart, s.lstart, k});
    keep_sets = s.lstart + k;
    if (k < s.count) break;
  }
  CK(cudaMemcpyAsync(c->h_u64, c->offsets.as<uint64_t>() + keep_sets, 8, cudaMemcpyDeviceToHost, c->stream));
  TRY(sync(c));
  const uint64_t e0 = c->h_u64[0];
  if (c->pool_len > e0)
    TRY(launched(c, launch_count_sub(c->pool.as<uint32_t>(), e0, c->pool_len, c->count_total.as<uint32_t>(),
                                     c->num_sms * 8, c->stream), "k_count_sub"));
  c->segs = kept;
  if (c->inv_pending && keep_sets <= c->pend_set0) c->inv_pending = false;   // the unindexed sets are gone
  c->nsets = keep_sets;
  c->pool_len = e0;
  c->T_global = theta;
  c->set_limit = keep_sets;          // the index segments stay valid: cover skips cut sets
  c->truncated = true;
  return GIM_OK;
}

// Replicated-pool protocol (world > 1 with an all-gather hook, include/gim.h gim_set_allgather):
// this rank generated its slice of the new global ids [a, theta) as local sets [set0, nsets) /
// elements [e0, pool_len); exchange element counts, all-gather the slices' sizes and elements
// (padded to the largest slice), and rebuild [set0, ...) as ALL new sets in global id order
// (rank slices are contiguous and rank-ordered), with count_total updated to the global counts.
gim_status replicate_round(gim_ctx* c, uint64_t a, uint64_t theta, uint64_t set0, uint64_t e0, size_t seg0) {
  const int W = c->world;
  const uint64_t Tr = c->rounds, len = (theta - a) / Tr;
  const uint64_t Ls = c->pool_len - e0, Ss = c->nsets - set0;
  std::vector<uint64_t> S(W), L(W);
  uint64_t maxS = 1, totS = 0;
  for (int r = 0; r < W; ++r) {
    S[r] = Tr * ((uint64_t)((unsigned __int128)len * (r + 1) / W) - (uint64_t)((unsigned __int128)len * r / W));
    maxS = std::max(maxS, S[r]);
    totS += S[r];
  }
  if (S[c->rank] != Ss) return fail(c, GIM_ESTATE, "replicated pool: local slice size mismatch");
  // 1. element counts of every rank
  TRY(ensure(c, c->ag_small, 8 * (uint64_t)(W + 1)));
  c->h_u64[0] = Ls;
  CK(cudaMemcpyAsync(c->ag_small.p, c->h_u64, 8, cudaMemcpyHostToDevice, c->stream));
  c->st.allreduces++;
  if (c->agfn(c->ag_small.p, 8, c->ag_small.as<uint64_t>() + 1, c->stream, c->aguser))
    return fail(c, GIM_ECOLL, "all-gather(element counts) failed");
  std::vector<uint64_t> hL(W);
  CK(cudaMemcpyAsync(hL.data(), c->ag_small.as<uint64_t>() + 1, 8 * (uint64_t)W, cudaMemcpyDeviceToHost, c->stream));
  TRY(sync(c));
  uint64_t maxL = 1, totL = 0;
  for (int r = 0; r < W; ++r) {
    L[r] = hL[r];
    maxL = std::max(maxL, L[r]);
    totL += L[r];
  }
  if (hL[c->rank] != Ls) return fail(c, GIM_ECOLL, "all-gather returned a wrong own element count");
  // 2. sizes of the local sets, padded to maxS; elements padded to maxL (pool capacity)
  TRY(ensure(c, c->ag_send, std::max(maxS * 4, maxL * 4)));
  TRY(ensure(c, c->ag_recv, (uint64_t)W * std::max(maxS * 4, maxL * 4)));
  TRY(launched(c, launch_sizes_of(c->offsets.as<uint64_t>() + set0, Ss, maxS, c->ag_send.as<uint32_t>(),
                                  c->num_sms * 4, c->stream), "k_sizes_of"));
  c->st.allreduces++;
  if (c->agfn(c->ag_send.p, maxS * 4, c->ag_recv.p, c->stream, c->aguser))
    return fail(c, GIM_ECOLL, "all-gather(set sizes) failed");
  // compact the gathered sizes in rank order into the scan input
  TRY(ensure(c, c->sizes, (totS + 1) * 4));
  TRY(ensure(c, c->scan_out, (totS + 1) * 8));
  TRY(ensure(c, c->scan_tmp, (scan_tiles(totS) + 2) * 8));
  for (uint64_t r = 0, o = 0; r < (uint64_t)W; o += S[r], ++r)
    if (S[r]) CK(cudaMemcpyAsync(c->sizes.as<uint32_t>() + o, c->ag_recv.as<uint32_t>() + (uint64_t)r * maxS, S[r] * 4,
                                 cudaMemcpyDeviceToDevice, c->stream));
  // elements: undo the local counts, gather, write back in rank order, count globally
  if (Ls) TRY(launched(c, launch_count_sub(c->pool.as<uint32_t>(), e0, e0 + Ls, c->count_total.as<uint32_t>(),
                                           c->num_sms * 8, c->stream), "k_count_sub"));
  CK(cudaMemcpyAsync(c->ag_send.p, c->pool.as<uint32_t>() + e0, Ls * 4, cudaMemcpyDeviceToDevice, c->stream));
  c->st.allreduces++;
  if (c->agfn(c->ag_send.p, maxL * 4, c->ag_recv.p, c->stream, c->aguser))
    return fail(c, GIM_ECOLL, "all-gather(set elements) failed");
  TRY(grow_keep(c, c->pool, (e0 + totL) * 4, e0 * 4));
  TRY(grow_keep(c, c->offsets, (set0 + totS + 1) * 8, (set0 + 1) * 8));
  for (uint64_t r = 0, o = 0; r < (uint64_t)W; o += L[r], ++r)
    if (L[r]) CK(cudaMemcpyAsync(c->pool.as<uint32_t>() + e0 + o, c->ag_recv.as<uint32_t>() + r * maxL, L[r] * 4,
                                 cudaMemcpyDeviceToDevice, c->stream));
  if (totL) TRY(launched(c, launch_count_add(c->pool.as<uint32_t>(), e0, e0 + totL, c->count_total.as<uint32_t>(),
                                             c->num_sms * 8, c->stream), "k_count_add"));
  {
    int nl = 0;
    cudaError_t e = launch_scan_u32(c->sizes.as<uint32_t>(), totS, c->scan_out.as<uint64_t>(),
                                    c->scan_tmp.as<uint64_t>(), c->scan_tmp.as<uint64_t>() + scan_tiles(totS) + 1,
                                    c->stream, &nl);
    TRY(launched(c, e, "scan(gathered sizes)", nl));
  }
  TRY(launched(c, launch_offsets_of(c->scan_out.as<uint64_t>(), totS, e0, c->offsets.as<uint64_t>() + set0,
                                    c->num_sms * 4, c->stream), "k_offsets_of"));
  c->nsets = set0 + totS;
  c->pool_len = e0 + totL;
  c->segs.resize(seg0);
  c->segs.push_back(Seg{a, set0, totS});
  return GIM_OK;
}

// theta counts sets in API units: RR sets, or MRIM sets of `rounds` standard ids each (R26).
// host_sync = false (inside gim_imm): the selection that follows is enqueued behind the index
// build without a host round trip; errors surface at its completion sync.
gim_status generate(gim_ctx* c, uint64_t theta_sets, uint64_t seed, bool host_sync = true) {
  if (!c->graph) return fail(c, GIM_ESTATE, "no graph loaded");
  if (theta_sets >= (1ull << 32) / c->rounds) return fail(c, GIM_EINVAL, "theta * rounds must be < 2^32");
  const uint64_t theta = theta_sets * c->rounds;
  if (!c->have_seed || c->seed != seed) TRY(reset_pool(c, seed));
  if (theta < c->T_global) {
    TRY(truncate_pool(c, theta));
  } else if (theta > c->T_global) {
    if (c->truncated) {                // segment deltas no longer match: rebuild at the next select
      c->inv_valid = false;
      c->truncated = false;
      c->set_limit = ~0ull;
    }
    // the rank's slice of the new sets (whole MRIM sets: the T rounds of a set stay together)
    const uint64_t a = c->T_global, len = (theta - a) / c->rounds, Tr = c->rounds;
    const uint64_t lo = a + Tr * (uint64_t)((unsigned __int128)len * c->rank / c->world);
    const uint64_t hi = a + Tr * (uint64_t)((unsigned __int128)len * (c->rank + 1) / c->world);
    const uint64_t set0 = c->nsets, e0 = c->pool_len;
    const size_t seg0 = c->segs.size();
    const uint64_t ch = c->chunk ? c->chunk : kChunk;
    for (uint64_t s = lo; s < hi; s += ch) TRY(gen_chunk(c, s, (uint32_t)std::min<uint64_t>(ch, hi - s)));
    if ((c->world > 1 || c->force_coll) && c->agfn) TRY(replicate_round(c, a, theta, set0, e0, seg0));
    // the new sets join the unindexed range; the next selection indexes it as one segment (its
    // O(n) count scan is paid once per selection that needs it, not per 2^22-id chunk or round)
    if (c->nsets > set0) {
      if (c->inv_segmented && c->inv_valid) {
        if (!c->inv_pending) {
          c->inv_pending = true;
          c->pend_set0 = set0;
          c->pend_e0 = e0;
        }
      } else {
        c->inv_valid = false;                  // rebuilt as one segment at the next selection
      }
    }
    c->T_global = theta;
  }
  return host_sync ? sync(c) : GIM_OK;
}

// ---- NodeSelection (O7) ---------------------------------------------------------------------
// Replays the enqueue sequence `body` (kernels + the library's own NCCL collectives, which stream
// capture supports) from a CUDA graph cached under `key`: the k-step loops of the P > 1
// protocols then cost one graph launch instead of a host round of launches per step.
template <class Body>
gim_status replay_captured(gim_ctx* c, const std::vector<uintptr_t>& key, Body body, int launches) {
  if (!c->p_exec || key != c->p_key) {
    if (c->p_exec) cudaGraphExecDestroy(c->p_exec);
    c->p_exec = nullptr;
    c->p_key.clear();
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const gim_status st = body();
    const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (st != GIM_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (e != cudaSuccess) return fail_cuda(c, "stream capture (P > 1 selection)", e);
    const cudaError_t ie = cudaGraphInstantiate(&c->p_exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) return fail_cuda(c, "cudaGraphInstantiate (P > 1 selection)", ie);
    c->p_key = key;
  }
  return launched(c, cudaGraphLaunch(c->p_exec, c->stream), "selection graph (P > 1)", launches);
}

gim_status read_keys(gim_ctx* c, uint32_t kk) {
  if (c->h_keys_cap < kk + 1) {
    if (c->h_keys) cudaFreeHost(c->h_keys);
    c->h_keys = nullptr;
    CK(cudaMallocHost(&c->h_keys, ((uint64_t)kk + 1) * 8));
    c->h_keys_cap = kk + 1;
  }
  CK(cudaMemcpyAsync(c->h_keys, c->keys.p, (uint64_t)kk * 8, cudaMemcpyDeviceToHost, c->stream));
  c->h_keys[kk] = 0;
  return GIM_OK;
}

// Node-sharded selection (world > 1, gim_set_reducescatter + gim_set_allreduce): rank r owns the
// global counts of nodes [r ns, (r+1) ns), ns = ceil(n / world). Counts are reduce-scattered
// once; per greedy step (Alg. 1 l.6-10, Alg. 7): the argmax of the own shard (the
// previous step's reduce-scattered decrements applied first), the keys of all ranks exchanged
// by a SUM all-reduce of one slot per rank, the global pick (largest key: lowest id on ties,
// R10) retired by its owner and covered in the local pool, the local decrements
// reduce-scattered to the owners.
gim_status select_launch_rs(gim_ctx* c, uint32_t k, const InvSegDev* segd, SelCtl* ctl, bool limited) {
  const uint64_t n = c->n;
  const uint32_t W = (uint32_t)c->world, r = (uint32_t)c->rank;
  const uint64_t ns = (n + W - 1) / W, npad = ns * W;
  const uint32_t id_base = (uint32_t)(ns * r);
  const uint32_t ns_valid = n > id_base ? (uint32_t)std::min<uint64_t>(ns, n - id_base) : 0u;
  const uint32_t kk = k;
  TRY(ensure(c, c->cnt, npad * 4));
  TRY(ensure(c, c->dec, npad * 4));
  TRY(ensure(c, c->rs_gcnt, ns * 4 + 16));
  TRY(ensure(c, c->rs_dshard, ns * 4 + 16));
  TRY(ensure(c, c->rs_keys, (uint64_t)kk * 8));
  TRY(ensure(c, c->rs_kx, (uint64_t)W * 8));
  auto* keys = reinterpret_cast<unsigned long long*>(c->keys.p);
  auto* lkeys = reinterpret_cast<unsigned long long*>(c->rs_keys.p);
  auto* kx = reinterpret_cast<unsigned long long*>(c->rs_kx.p);
  uint32_t* gcnt = c->rs_gcnt.as<uint32_t>();
  int32_t* dshard = c->rs_dshard.as<int32_t>();
  int32_t* dec = c->dec.as<int32_t>();
  CK(cudaMemcpyAsync(c->cnt.p, c->count_total.p, n * 4, cudaMemcpyDeviceToDevice, c->stream));
  if (npad > n) CK(cudaMemsetAsync(c->cnt.as<uint32_t>() + n, 0, (npad - n) * 4, c->stream));
  CK(cudaEventRecord(c->ev_cnt_copied, c->stream));
  CK(cudaMemsetAsync(c->covered.p, 0, std::max<uint64_t>(c->nsets, 1), c->stream));
  CK(cudaMemsetAsync(keys, 0, (uint64_t)kk * 8, c->stream));
  CK(cudaMemsetAsync(lkeys, 0, (uint64_t)kk * 8, c->stream));
  TRY(launched(c, launch_sel_ctl(ctl, c->sel_cstar, kk, nullptr, c->stream), "k_sel_ctl"));
  CK(cudaMemsetAsync(dec, 0, npad * 4, c->stream));
  CK(cudaMemsetAsync(dshard, 0, ns * 4, c->stream));
  c->st.allreduces++;
  if (c->rsfn(c->cnt.p, gcnt, ns, c->stream, c->rsuser)) return fail(c, GIM_ECOLL, "reduce-scatter(count) failed");
  Prof pf(c, CLS_SELECT);
  auto loop = [&]() -> gim_status {
    for (uint32_t j = 0; j < kk; ++j) {
      TRY(launched(c, launch_argmax(gcnt, dshard, ns_valid, lkeys, (int)j, nullptr, c->num_sms * kArgmaxCtasPerSM,
                                    c->stream, false, id_base, ctl), "k_argmax(shard)"));
      TRY(launched(c, launch_rs_pack(lkeys, (int)j, r, W, kx, c->stream), "k_rs_pack"));
      c->st.allreduces++;
      if (c->arfn(kx, 2ull * W, c->stream, c->aruser)) return fail(c, GIM_ECOLL, "all-reduce(keys) failed");
      TRY(launched(c, launch_rs_pick(kx, W, keys, (int)j, gcnt, id_base, ns_valid, c->stream), "k_rs_pick"));
      TRY(launched(c, launch_cover(keys, (int)j, segd, ctl, c->offsets.as<uint64_t>(), c->pool.as<uint32_t>(),
                                   c->covered.as<uint8_t>(), c->cnt.as<uint32_t>(), dec, c->num_sms * kCoverCtasPerSM,
                                   c->stream, limited, nullptr), "k_cover"));
      if (j + 1 < kk) {
        c->st.allreduces++;
        if (c->rsfn(dec, dshard, ns, c->stream, c->rsuser)) return fail(c, GIM_ECOLL, "reduce-scatter(dec) failed");
        CK(cudaMemsetAsync(dec, 0, npad * 4, c->stream));
      }
    }
    return GIM_OK;
  };
  if (c->nccl && c->use_graph) {
    const std::vector<uintptr_t> key = {1, (uintptr_t)c->nccl, (uintptr_t)gcnt, (uintptr_t)dshard, (uintptr_t)lkeys,
                                        (uintptr_t)kx, (uintptr_t)keys, (uintptr_t)segd, (uintptr_t)c->offsets.p,
                                        (uintptr_t)c->pool.p, (uintptr_t)c->covered.p, (uintptr_t)c->cnt.p,
                                        (uintptr_t)dec, (uintptr_t)ctl, kk, (uintptr_t)n, (uintptr_t)limited};
    TRY(replay_captured(c, key, loop, 4 * (int)kk));
  } else {
    TRY(loop());
  }
  c->sel_fused_used = false;
  TRY(read_keys(c, kk));
  CK(cudaEventRecord(c->ev_sel_done, c->stream));
  c->sel_pending = true;
  return GIM_OK;
}

gim_status select_launch(gim_ctx* c, uint32_t k) {
  c->sel_cand_used = false;
  if (!c->graph) return fail(c, GIM_ESTATE, "no graph loaded");
  if (k < 1 || k > c->n) return fail(c, GIM_EINVAL, "k must satisfy 1 <= k <= n");
  if (!c->have_seed || c->T_global == 0) return fail(c, GIM_ESTATE, "RR pool is empty");
  const bool sharded = (c->world > 1 || c->force_coll) && !c->agfn;   // replicated pool: select as P = 1
  if (sharded && !c->arfn) return fail(c, GIM_ESTATE, "world > 1 requires gim_set_allreduce or gim_set_allgather");
  const uint64_t n = nsp(c);                        // counted elements (nodes, or MRIM pairs)
  const uint32_t kk = k * c->rounds;                // picks: k per round (R27)
  const MrimSel mrs{c->rounds, c->n, k};
  const MrimSel* mr = c->rounds > 1 ? &mrs : nullptr;
  TRY(ensure(c, c->cnt, n * 4));
  TRY(ensure(c, c->covered, std::max<uint64_t>(c->nsets / c->rounds, 1)));
  TRY(ensure(c, c->keys, (uint64_t)kk * 8));
  if (sharded) TRY(ensure(c, c->dec, n * 4));
  int32_t* dec = sharded ? c->dec.as<int32_t>() : nullptr;
  TRY(flush_inv(c));
  TRY(ensure(c, c->seg_desc, sizeof(InvSegDev) * kMaxInvSeg + 16));
  {
    InvSegDev tab[kMaxInvSeg];
    for (size_t q = 0; q < c->iseg.size(); ++q)
      tab[q] = InvSegDev{c->iseg[q].off.as<uint32_t>(), c->iseg[q].inv.as<uint32_t>()};
    TRY(launched(c, launch_set_segs(tab, (uint32_t)c->iseg.size(),
                                    (uint32_t)std::min<uint64_t>(c->set_limit, 0xFFFFFFFFull),
                                    c->seg_desc.as<InvSegDev>(),
                                    reinterpret_cast<uint32_t*>(c->seg_desc.as<InvSegDev>() + kMaxInvSeg),
                                    c->stream), "k_set_segs"));
  }
  const bool limited = c->set_limit != ~0ull;     // cover must skip truncated sets
  const InvSegDev* segd = c->seg_desc.as<InvSegDev>();
  TRY(ensure(c, c->sel_ctl, sizeof(SelCtl)));
  SelCtl* ctl = c->sel_ctl.as<SelCtl>();
  if (sharded && c->rsfn && c->rounds == 1) return select_launch_rs(c, k, segd, ctl, limited);
  CK(cudaMemcpyAsync(c->cnt.p, c->count_total.p, n * 4, cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaEventRecord(c->ev_cnt_copied, c->stream));
  CK(cudaMemsetAsync(c->covered.p, 0, std::max<uint64_t>(c->nsets / c->rounds, 1), c->stream));
  CK(cudaMemsetAsync(c->keys.p, 0, (uint64_t)kk * 8, c->stream));
  if (dec) {
    CK(cudaMemsetAsync(dec, 0, n * 4, c->stream));
    c->st.allreduces++;
    if (c->arfn(c->cnt.p, n, c->stream, c->aruser)) return fail(c, GIM_ECOLL, "all-reduce(count) failed");
  }
  auto* keys = reinterpret_cast<unsigned long long*>(c->keys.p);
  // P = 1: candidate list for the argmax (at most kMaxCand nodes whose initial count reaches
  // tau_p1; counts only decrease, so a pick >= tau_p1 is the argmax over all nodes)
  const uint32_t kMaxCand = 1u << 16;
  uint32_t* cand = nullptr;
  unsigned int *hist = nullptr, *ncand = nullptr;
  uint32_t* tau_p1 = nullptr;
  const bool fused_mode = !dec && c->rounds == 1 && (c->sel_fused || c->sel_coop) && !c->force_unfused &&
                          !c->speculate && !c->sel_persistent;
  if (!fused_mode && !dec && c->rounds == 1 && !c->force_unfused &&
      (c->use_cand == 2 || (c->use_cand == 1 && n >= (1u << 20)))) {   // small n: full scan is cheaper
    // (measured with the per-step backup scan gone: C3 selection 1.95 vs 2.19 ms with full scans,
    // C2 1.29 vs 1.14 ms — the candidate list pays from ~10^6 nodes)
    TRY(ensure(c, c->cand, (uint64_t)kMaxCand * 4 + 64 * 4));
    cand = c->cand.as<uint32_t>();
    hist = reinterpret_cast<unsigned int*>(cand + kMaxCand);
    tau_p1 = reinterpret_cast<uint32_t*>(hist + 40);
    ncand = reinterpret_cast<unsigned int*>(hist + 41);
    TRY(launched(c, launch_cand_setup(c->cnt.as<uint32_t>(), (uint32_t)n, kMaxCand, hist, tau_p1, cand, ncand,
                                      c->num_sms * 4, c->stream), "candidate setup", 3));
  }
  // candidate argmax: each step is argmax over the list + cover; an uncertified pick makes the
  // cover fail the selection, which select_finish redoes with full scans (no per-step backup scan)
  TRY(launched(c, launch_sel_ctl(ctl, c->sel_cstar, kk, cand ? tau_p1 : nullptr, c->stream), "k_sel_ctl"));
  c->sel_cand_used = cand != nullptr;
  // cooperative selection (P = 1, standard IM): one cooperative launch, one grid barrier per
  // step, redundant per-CTA candidate argmax; certificate failures are redone by select_finish
  const bool coop = !dec && c->rounds == 1 && c->sel_coop && !c->force_unfused && !c->speculate &&
                    !c->sel_persistent;
  if (coop) {
    const uint32_t cap = std::min<uint32_t>(c->sel_coop, kCoopCands);
    TRY(ensure(c, c->cand, (uint64_t)kCoopCands * 4 + 64 * 4));
    uint32_t* cnd = c->cand.as<uint32_t>();
    unsigned int* hst = reinterpret_cast<unsigned int*>(cnd + kCoopCands);
    uint32_t* tau = reinterpret_cast<uint32_t*>(hst + 40);
    unsigned int* ncd = reinterpret_cast<unsigned int*>(hst + 41);
    TRY(launched(c, launch_cand_setup(c->cnt.as<uint32_t>(), (uint32_t)n, cap, hst, tau, cnd, ncd,
                                      c->num_sms * 4, c->stream), "candidate setup", 3));
    if (c->cmap_n < n || !c->cmap.p) {
      TRY(dalloc(c, c->cmap, n * 4));
      CK(cudaMemsetAsync(c->cmap.p, 0xFF, n * 4, c->stream));
      c->cmap_n = n;
    }
    TRY(ensure(c, c->cdec, 3ull * kCoopCands * 4));
    CK(cudaMemsetAsync(c->cdec.p, 0, 3ull * kCoopCands * 4, c->stream));
    TRY(ensure(c, c->sel_bar, 64));
    CK(cudaMemsetAsync(c->sel_bar.p, 0, 8, c->stream));
    TRY(ensure(c, c->sel_done, ((uint64_t)kk + 2) * 4));
    uint32_t* ff = c->sel_done.as<uint32_t>() + kk;
    CK(cudaMemsetAsync(ff, 0, 4, c->stream));
    {
      Prof pf(c, CLS_SELECT);
      TRY(launched(c, launch_select_coop(c->cnt.as<uint32_t>(), cnd, ncd, tau, c->cmap.as<uint32_t>(),
                                         c->cdec.as<int32_t>(), keys, (int)kk, segd, c->offsets.as<uint64_t>(),
                                         c->pool.as<uint32_t>(), c->covered.as<uint8_t>(),
                                         c->sel_bar.as<unsigned int>(), ff, c->num_sms, limited, c->stream),
                   "k_select_coop", 3));
    }
    c->sel_fused_used = true;
    TRY(read_keys(c, kk));
    CK(cudaMemcpyAsync(c->h_keys + kk, ff, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaEventRecord(c->ev_sel_done, c->stream));
    c->sel_pending = true;
    return GIM_OK;
  }
  // fused greedy steps (P = 1, standard IM): one launch per step, candidate argmax in the last
  // CTA of each cover; certificate failures are redone unfused by select_finish
  const bool fused = !dec && c->rounds == 1 && c->sel_fused && !c->force_unfused && !c->speculate &&
                     !c->sel_persistent;
  c->sel_fused_used = fused;
  uint32_t* fflag = nullptr;
  unsigned int* done = nullptr;
  if (fused) {
    const uint32_t cap = c->sel_fused;
    TRY(ensure(c, c->cand, (uint64_t)cap * 4 + 64 * 4));
    cand = c->cand.as<uint32_t>();
    hist = reinterpret_cast<unsigned int*>(cand + cap);
    tau_p1 = reinterpret_cast<uint32_t*>(hist + 40);
    ncand = reinterpret_cast<unsigned int*>(hist + 41);
    TRY(launched(c, launch_cand_setup(c->cnt.as<uint32_t>(), (uint32_t)n, cap, hist, tau_p1, cand, ncand,
                                      c->num_sms * 4, c->stream), "candidate setup", 3));
    TRY(ensure(c, c->sel_done, ((uint64_t)kk + 2) * 4));
    done = c->sel_done.as<unsigned int>();
    fflag = reinterpret_cast<uint32_t*>(done + kk);
    CK(cudaMemsetAsync(done, 0, ((uint64_t)kk + 2) * 4, c->stream));
  }
  if (fused) {
    const std::vector<uintptr_t> key = {(uintptr_t)c->cnt.p, (uintptr_t)segd, (uintptr_t)cand,
                                        (uintptr_t)c->offsets.p, (uintptr_t)c->pool.p, (uintptr_t)c->covered.p,
                                        (uintptr_t)c->keys.p, (uintptr_t)k, (uintptr_t)n, (uintptr_t)limited,
                                        (uintptr_t)c->rounds, (uintptr_t)done, (uintptr_t)c->fused_ctas};
    int nl = 0;
    if (c->use_graph) {
      if (!c->sel_exec || key != c->sel_key) {
        if (c->sel_exec) cudaGraphExecDestroy(c->sel_exec);
        for (cudaGraphExec_t& ex : c->sel_parts) cudaGraphExecDestroy(ex);
        c->sel_parts.clear();
        c->sel_exec = nullptr;
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        launch_select_fused(keys, (int)kk, segd, c->offsets.as<uint64_t>(), c->pool.as<uint32_t>(),
                            c->covered.as<uint8_t>(), c->cnt.as<uint32_t>(), cand, ncand, tau_p1, done, fflag,
                            c->num_sms * c->fused_ctas, c->stream, limited, &nl);
        CK(cudaStreamEndCapture(c->stream, &graph));
        const cudaError_t ie = cudaGraphInstantiate(&c->sel_exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) return fail_cuda(c, "cudaGraphInstantiate", ie);
        c->sel_key = key;
      }
      Prof pf(c, CLS_SELECT);
      TRY(launched(c, cudaGraphLaunch(c->sel_exec, c->stream), "selection graph (fused)", (int)kk + 1));
    } else {
      Prof pf(c, CLS_SELECT);
      TRY(launched(c, launch_select_fused(keys, (int)kk, segd, c->offsets.as<uint64_t>(), c->pool.as<uint32_t>(),
                                          c->covered.as<uint8_t>(), c->cnt.as<uint32_t>(), cand, ncand, tau_p1, done,
                                          fflag, c->num_sms * c->fused_ctas, c->stream, limited, &nl),
                   "fused selection", (int)kk + 1));
    }
  } else if (!dec && !cand && c->sel_persistent) {
    // P = 1: the k greedy steps in one cooperative launch, grid barriers between the phases
    TRY(ensure(c, c->sel_bar, 64));
    CK(cudaMemsetAsync(c->sel_bar.p, 0, 8, c->stream));
    Prof pf(c, CLS_SELECT);
    TRY(launched(c, launch_select_persistent(c->cnt.as<uint32_t>(), (uint32_t)n, keys, (int)kk, segd,
                                             c->offsets.as<uint64_t>(), c->pool.as<uint32_t>(),
                                             c->covered.as<uint8_t>(), mr, limited, c->sel_bar.as<unsigned int>(),
                                             c->num_sms, c->stream), "k_select_persistent"));
  } else if (!dec && !cand && c->rounds == 1 && c->sel_small && n <= select_cta_max_n() && !c->speculate) {
    // small graphs: every greedy step in one CTA, counts in shared memory (no launch per step)
    Prof pf(c, CLS_SELECT);
    TRY(launched(c, launch_select_cta(c->count_total.as<uint32_t>(), (uint32_t)n, keys, (int)kk, segd,
                                      c->offsets.as<uint64_t>(), c->pool.as<uint32_t>(), c->covered.as<uint8_t>(),
                                      ctl, limited, c->stream), "k_select_cta"));
  } else if (!dec && !cand && c->rounds == 1 && c->sel_small && c->sel_cluster && n <= select_cluster_max_n() &&
             !c->speculate) {
    // mid-size graphs: the same on a thread-block cluster, counts in the CTAs' shared memories
    Prof pf(c, CLS_SELECT);
    TRY(launched(c, launch_select_cluster(c->count_total.as<uint32_t>(), (uint32_t)n, keys, (int)kk, segd,
                                          c->offsets.as<uint64_t>(), c->pool.as<uint32_t>(), c->covered.as<uint8_t>(),
                                          ctl, limited, c->stream), "k_select_cluster"));
  } else if (!dec && c->use_graph) {
    // P = 1: the 2k argmax/cover launches replayed from a CUDA graph (captured once per set of
    // buffer pointers; steady-state IMM runs reuse it), so the GPU runs them back to back.
    const std::vector<uintptr_t> key = {(uintptr_t)c->cnt.p, (uintptr_t)segd, (uintptr_t)cand,
                                        (uintptr_t)c->offsets.p, (uintptr_t)c->pool.p, (uintptr_t)c->covered.p,
                                        (uintptr_t)c->keys.p, (uintptr_t)k, (uintptr_t)n, (uintptr_t)limited,
                                        (uintptr_t)c->rounds, (uintptr_t)ctl};
    auto step = [&](uint32_t j) {
      if (cand)
        launch_argmax_cand(c->cnt.as<uint32_t>(), cand, ncand, keys, (int)j, c->num_sms, c->stream, ctl);
      else
        launch_argmax(c->cnt.as<uint32_t>(), nullptr, (uint32_t)n, keys, (int)j, nullptr,
                      c->num_sms * kArgmaxCtasPerSM, c->stream, mr != nullptr, 0u, ctl);
      launch_cover(keys, (int)j, segd, ctl, c->offsets.as<uint64_t>(), c->pool.as<uint32_t>(),
                   c->covered.as<uint8_t>(), c->cnt.as<uint32_t>(), nullptr, c->num_sms * kCoverCtasPerSM, c->stream,
                   limited, mr);
    };
    // the steps as consecutive graphs [0, 8), [8, 32), [32, kk): a bounded greedy (IMM estimation
    // round) checks its stop flag on the host between them, so a selection that stops early does
    // not replay the no-op launches of the remaining steps (C3 round 3 stops at step 2 of 50,
    // C5 round 6 at step 10 of 100); a full selection replays them back to back
    std::vector<uint32_t> cuts = {0};
    for (uint32_t b : {kSelHead, 4 * kSelHead})
      if (b < kk) cuts.push_back(b);
    cuts.push_back(kk);
    const size_t parts = cuts.size() - 1;
    if (c->sel_exec || c->sel_parts.size() != parts || key != c->sel_key) {
      for (cudaGraphExec_t& ex : c->sel_parts)
        if (ex) cudaGraphExecDestroy(ex);
      c->sel_parts.assign(parts, nullptr);
      if (c->sel_exec) cudaGraphExecDestroy(c->sel_exec);   // a fused selection's graph
      c->sel_exec = nullptr;
      c->sel_key.clear();
      for (size_t q = 0; q < parts; ++q) {
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        for (uint32_t j = cuts[q]; j < cuts[q + 1]; ++j) step(j);
        CK(cudaStreamEndCapture(c->stream, &graph));
        const cudaError_t ie = cudaGraphInstantiate(&c->sel_parts[q], graph, 0);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) return fail_cuda(c, "cudaGraphInstantiate", ie);
      }
      c->sel_key = key;
    }
    Prof pf(c, CLS_SELECT);
    for (size_t q = 0; q < parts; ++q) {
      if (q > 0 && c->sel_cstar) {
        CK(cudaMemcpyAsync(c->h_u64 + 4, &ctl->stop, 4, cudaMemcpyDeviceToHost, c->stream));
        TRY(sync(c));
        if ((uint32_t)c->h_u64[4] != 0u) break;
      }
      TRY(launched(c, cudaGraphLaunch(c->sel_parts[q], c->stream), "selection graph",
                   2 * (int)(cuts[q + 1] - cuts[q])));
    }
  } else {
    auto loop = [&]() -> gim_status {
      for (uint32_t j = 0; j < kk; ++j) {
        {
          Prof pf(c, CLS_SELECT);
          if (cand)
            TRY(launched(c, launch_argmax_cand(c->cnt.as<uint32_t>(), cand, ncand, keys, (int)j, c->num_sms, c->stream, ctl),
                         "k_argmax_cand"));
          else
            TRY(launched(c, launch_argmax(c->cnt.as<uint32_t>(), dec, (uint32_t)n, keys, (int)j, nullptr,
                                          c->num_sms * kArgmaxCtasPerSM, c->stream, mr != nullptr, 0u, ctl), "k_argmax"));
          TRY(launched(c, launch_cover(keys, (int)j, segd, ctl, c->offsets.as<uint64_t>(), c->pool.as<uint32_t>(),
                                       c->covered.as<uint8_t>(), c->cnt.as<uint32_t>(), dec, c->num_sms * kCoverCtasPerSM,
                                       c->stream, limited, mr), "k_cover"));
        }
        if (dec && j + 1 < kk) {
          c->st.allreduces++;
          if (c->arfn(dec, n, c->stream, c->aruser)) return fail(c, GIM_ECOLL, "all-reduce(dec) failed");
        }
      }
      return GIM_OK;
    };
    if (dec && c->nccl && c->use_graph && !c->profile) {
      // dense all-reduce protocol with the native exchange: the whole k-step loop as one graph
      const std::vector<uintptr_t> key = {2, (uintptr_t)c->nccl, (uintptr_t)c->cnt.p, (uintptr_t)dec, (uintptr_t)keys,
                                          (uintptr_t)segd, (uintptr_t)c->offsets.p, (uintptr_t)c->pool.p,
                                          (uintptr_t)c->covered.p, (uintptr_t)ctl, kk, (uintptr_t)n, (uintptr_t)limited,
                                          (uintptr_t)c->rounds};
      Prof pf(c, CLS_SELECT);
      TRY(replay_captured(c, key, loop, 3 * (int)kk));
    } else {
      TRY(loop());
    }
  }
  if (c->h_keys_cap < kk + 1) {
    if (c->h_keys) cudaFreeHost(c->h_keys);
    c->h_keys = nullptr;
    CK(cudaMallocHost(&c->h_keys, ((uint64_t)kk + 1) * 8));
    c->h_keys_cap = kk + 1;
  }
  CK(cudaMemcpyAsync(c->h_keys, keys, (uint64_t)kk * 8, cudaMemcpyDeviceToHost, c->stream));
  c->h_keys[kk] = 0;
  if (fused) CK(cudaMemcpyAsync(c->h_keys + kk, fflag, 4, cudaMemcpyDeviceToHost, c->stream));
  else if (c->sel_cand_used) CK(cudaMemcpyAsync(c->h_keys + kk, &ctl->fail, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaEventRecord(c->ev_sel_done, c->stream));
  c->sel_pending = true;
  return GIM_OK;
}

gim_status select_finish(gim_ctx* c, uint32_t k, uint32_t* seeds, uint64_t* gains, uint64_t* covered) {
  TRY(sync(c));
  c->sel_pending = false;
  if ((c->sel_fused_used || c->sel_cand_used) && c->h_keys[(uint64_t)k * c->rounds]) {
    // a candidate argmax could not be certified (best candidate below tau): redo with full scans
    c->st.fused_fallbacks++;
    c->force_unfused = true;
    const gim_status st = select_launch(c, k);
    c->force_unfused = false;
    TRY(st);
    TRY(sync(c));
    c->sel_pending = false;
  }
  uint64_t cov = 0;
  uint32_t steps = 0;                   // a step that ran has a nonzero key (k <= n: a pick exists)
  for (uint32_t j = 0; j < k * c->rounds; ++j) {
    steps += c->h_keys[j] != 0ull;
    seeds[j] = ~(uint32_t)(c->h_keys[j] & 0xFFFFFFFFull);
    const uint64_t g = c->h_keys[j] >> 32;
    if (gains) gains[j] = g;
    cov += g;
  }
  if (covered) *covered = cov;
  c->last_sel_steps = steps;
  c->st.selects++;
  return GIM_OK;
}

gim_status select_impl(gim_ctx* c, uint32_t k, uint32_t* seeds, uint64_t* gains, uint64_t* covered) {
  TRY(select_launch(c, k));
  return select_finish(c, k, seeds, gains, covered);
}

// Speculative sampling on stream2 while the selection launched on `stream` runs: the library's
// generation code runs unchanged with the two streams swapped. stream2 first waits until the
// selection has copied count_total (which k_store updates).
gim_status generate_speculative(gim_ctx* c, uint64_t theta, uint64_t seed) {
  CK(cudaStreamWaitEvent(c->stream2, c->ev_cnt_copied, 0));
  std::swap(c->stream, c->stream2);
  const gim_status st = generate(c, theta, seed);
  std::swap(c->stream, c->stream2);
  return st;
}

// ---- IMM constants (O8; readings R1-R3, R21) -----------------------------------------------
struct ImmConst {
  double ell_eff, eps_p, lnC, lambda_p, alpha, beta, lambda_s;
};

// ln C(N, K) in lambda', lambda*: N = n, K = k for IMM; MRIM (R28) N = n*T pairs, K = k*T picks
ImmConst imm_constants(uint32_t n_, uint32_t k, double eps, double ell, uint32_t T = 1) {
  ImmConst K;
  const double n = (double)n_;
  const double ln_n = std::log(n);
  const double log2n = std::log2(n);
  K.ell_eff = ell * (1.0 + std::log(2.0) / ln_n);
  K.eps_p = std::sqrt(2.0) * eps;
  K.lnC = 0.0;
  const uint64_t NN = (uint64_t)n_ * T, KK = (uint64_t)k * T;
  for (uint64_t t = 1; t <= KK; ++t) K.lnC += std::log((double)(NN - KK + t)) - std::log((double)t);
  K.lambda_p = (2.0 + 2.0 / 3.0 * K.eps_p) * (K.lnC + K.ell_eff * ln_n + std::log(log2n)) * n / (K.eps_p * K.eps_p);
  K.alpha = std::sqrt(K.ell_eff * ln_n + std::log(2.0));
  K.beta = std::sqrt((1.0 - 1.0 / M_E) * (K.lnC + K.ell_eff * ln_n + std::log(2.0)));
  const double s = (1.0 - 1.0 / M_E) * K.alpha + K.beta;
  K.lambda_s = 2.0 * n * (s * s) / (eps * eps);
  return K;
}

}  // namespace

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

gim_status gim_create(int device, void* cuda_stream, gim_ctx** out) {
  if (!out) return GIM_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return GIM_ECUDA;
  }
  if (device < 0 || device >= ndev) return GIM_ECUDA;
  DeviceGuard g(device);
  gim_ctx* c = new gim_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cuda_stream) {
    c->stream = static_cast<cudaStream_t>(cuda_stream);
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      return GIM_ECUDA;
    }
    c->own_stream = true;
  }
  if (cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_cnt_copied, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_sel_done, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return GIM_ECUDA;
  }
  cudaMemPool_t mp;
  if (cudaDeviceGetDefaultMemPool(&mp, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (cudaMallocHost(&c->h_ctr, sizeof(GenCounters)) != cudaSuccess ||
      cudaMallocHost(&c->h_u64, 64) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return GIM_ECUDA;
  }
  *out = c;
  return GIM_OK;
}

void gim_destroy(gim_ctx* c) {
  if (!c) return;
  DeviceGuard g(c->device);
  cudaStreamSynchronize(c->stream);
  DevBuf* bufs[] = {&c->row_ptr, &c->src, &c->thr_edge, &c->pool, &c->offsets, &c->count_total,
                    &c->sizes, &c->soff, &c->giant_list, &c->giant2_list, &c->retry_list, &c->item_list, &c->scan_out,
                    &c->scan_tmp, &c->staging, &c->ctr, &c->dump, &c->lt_spill, &c->spill, &c->lane_spill, &c->skip_tab, &c->esc_list, &c->bitmaps, &c->gqueues, &c->cnt,
                    &c->covered, &c->keys, &c->dec, &c->cnt_snap, &c->seg_desc, &c->cand,
                    &c->out_ptr, &c->out_dst, &c->out_in, &c->thr_wc, &c->ag_small,
                    &c->ag_send, &c->ag_recv, &c->sel_bar, &c->rs_gcnt, &c->rs_dshard, &c->rs_keys, &c->rs_kx,
                    &c->sel_ctl, &c->cmap, &c->cdec, &c->sel_done, &c->probe, &c->isort_keys, &c->isort_vals,
                    &c->isort_tmp};
  for (auto& sg : c->iseg) {
    dfree(c, sg.off);
    dfree(c, sg.inv);
  }
  for (DevBuf* b : bufs) dfree(c, *b);
  cudaStreamSynchronize(c->stream);
  for (auto& v : c->ev)
    for (auto& pr : v) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  for (cudaEvent_t e : c->ev_free) cudaEventDestroy(e);
  if (c->sel_exec) cudaGraphExecDestroy(c->sel_exec);
  for (cudaGraphExec_t& ex : c->sel_parts) cudaGraphExecDestroy(ex);
  c->sel_parts.clear();
  if (c->p_exec) cudaGraphExecDestroy(c->p_exec);
  if (c->h_ctr) cudaFreeHost(c->h_ctr);
  if (c->h_u64) cudaFreeHost(c->h_u64);
  if (c->h_keys) cudaFreeHost(c->h_keys);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  cudaStreamSynchronize(c->stream2);
  cudaStreamDestroy(c->stream2);
  cudaEventDestroy(c->ev_cnt_copied);
  cudaEventDestroy(c->ev_sel_done);
  if (c->nccl) nccl_comm_destroy(c->nccl);
  // the default pool keeps freed memory (release threshold = max, set in gim_create): hand the
  // unused part back so other processes on this GPU can use it
  cudaMemPool_t mp;
  if (cudaDeviceGetDefaultMemPool(&mp, c->device) == cudaSuccess) cudaMemPoolTrimTo(mp, 0);
  cudaGetLastError();
  delete c;
}

const char* gim_last_error(const gim_ctx* c) { return c ? c->err.c_str() : "null context"; }

gim_status gim_set_allocator(gim_ctx* c, gim_alloc_fn a, gim_free_fn f, void* user) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  if (c->graph) return fail(c, GIM_ESTATE, "gim_set_allocator must precede gim_load_graph");
  if ((a == nullptr) != (f == nullptr)) return fail(c, GIM_EINVAL, "alloc and free must both be set");
  c->afn = a;
  c->ffn = f;
  c->auser = user;
  return GIM_OK;
}

gim_status gim_load_graph(gim_ctx* c, uint32_t n, uint64_t m, const uint64_t* rp, const uint32_t* src,
                          const float* w, gim_model model, gim_weights scheme, float p_uniform) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  DeviceGuard g(c->device);
  if (n < 1 || n == 0xFFFFFFFFu) return fail(c, GIM_EINVAL, "n must be in [1, 2^32-2]");
  if (m >= 0xFFFFFF00ull) return fail(c, GIM_EINVAL, "m must be < 2^32 - 256");
  if (!rp || (m && !src)) return fail(c, GIM_EINVAL, "row_ptr/src missing");
  if (model != GIM_IC && model != GIM_LT) return fail(c, GIM_EINVAL, "bad model");
  if (scheme != GIM_W_EXPLICIT && scheme != GIM_W_WC && scheme != GIM_W_UNIFORM) return fail(c, GIM_EINVAL, "bad scheme");
  if (scheme == GIM_W_EXPLICIT && m && !w) return fail(c, GIM_EINVAL, "explicit weights required");
  if (model == GIM_LT && scheme == GIM_W_UNIFORM) return fail(c, GIM_EINVAL, "LT with uniform p is not supported (reading R23)");
  if (scheme == GIM_W_UNIFORM && !(p_uniform >= 0.f && p_uniform <= 1.f)) return fail(c, GIM_EINVAL, "p_uniform must be in [0,1]");
  // canonical in-CSR (reading R15): the end points here, everything else on the device below
  if (rp[0] != 0 || rp[n] != m) return fail(c, GIM_EINVAL, "row_ptr[0] must be 0 and row_ptr[n] must be m");
  if ((uint64_t)n * c->rounds >= 0xFFFFFFFFull) return fail(c, GIM_EINVAL, "n * rounds must be < 2^32 - 1");
  // release the previous graph and pool
  dfree(c, c->row_ptr);
  dfree(c, c->src);
  dfree(c, c->thr_edge);
  // giant slots (bitmaps all zero, queues all kEmpty: K-GIANT restores both after every set) are
  // kept for a graph that is not larger, so reloading a graph does not re-clear gigabytes
  if (n > c->giant_n) {
    dfree(c, c->bitmaps);
    dfree(c, c->gqueues);
    c->giant_slots = 0;
    c->giant_n = 0;
    c->giant_cap_reached = false;
  }
  c->graph = false;
  c->out_valid = false;
  dfree(c, c->out_ptr);
  dfree(c, c->out_dst);
  dfree(c, c->out_in);
  dfree(c, c->thr_wc);
  c->n = n;
  c->m = m;
  c->model = model;
  c->scheme = scheme;
  if (c->skip && ((int)model != MODEL_IC || (int)scheme == W_EXPLICIT)) c->skip = 0;   // R31 needs IC + WC/uniform
  c->p_uniform = p_uniform;
  c->thr_uniform = (uint64_t)std::ceil((double)p_uniform * 4294967296.0);
  TRY(dalloc(c, c->row_ptr, ((uint64_t)n + 1) * 4 * (scheme == GIM_W_WC ? 2 : 1)));
  TRY(dalloc(c, c->src, std::max<uint64_t>(m, 1) * 4));
  c->thr_node = scheme == GIM_W_WC ? c->row_ptr.as<uint32_t>() + n + 1 : nullptr;
  {
    // upload (pinned host buffers DMA directly), validate + convert row pointers on the device
    DevBuf rp64;
    TRY(dalloc(c, rp64, ((uint64_t)n + 1) * 8 + 16));
    uint32_t* flags = reinterpret_cast<uint32_t*>(rp64.as<uint64_t>() + n + 1);
    CK(cudaMemcpyAsync(rp64.p, rp, ((uint64_t)n + 1) * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(flags, 0, 4, c->stream));
    CK(cudaMemsetAsync(flags + 1, 0xFF, 4, c->stream));
    CK(cudaMemsetAsync(flags + 2, 0, 8, c->stream));                 // max in-degree
    // src arrives in row-aligned slices on `stream`; each slice's rows are validated on stream2
    // as soon as it has landed, so the validation overlaps the rest of the PCIe upload. The row
    // pointers are read on the host only where they are monotone (a bad row_ptr is reported by
    // the validation itself and the slicing falls back to one slice).
    const int K = m >= (1u << 23) ? 8 : 1;
    std::vector<uint32_t> cut = {0};
    bool mono = true;
    for (int k = 1; k < K; ++k) {
      const uint64_t target = m * (uint64_t)k / K;
      uint32_t lo = cut.back(), hi = n;                  // first row with rp >= target
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (rp[mid] >= target) hi = mid; else lo = mid + 1;
      }
      if (lo > cut.back() && lo < n) cut.push_back(lo);
    }
    cut.push_back(n);
    for (size_t q = 1; q < cut.size(); ++q) mono = mono && rp[cut[q - 1]] <= rp[cut[q]] && rp[cut[q]] <= m;
    if (!mono) cut = {0, n};
    struct Events {                                    // destroyed on every exit path
      std::vector<cudaEvent_t> v;
      ~Events() {
        for (cudaEvent_t e : v) cudaEventDestroy(e);
      }
    } ev_guard;
    std::vector<cudaEvent_t>& evs = ev_guard.v;
    for (size_t q = 0; q + 1 < cut.size(); ++q) {
      const uint64_t e0 = rp[cut[q]], e1 = (q + 2 == cut.size()) ? m : rp[cut[q + 1]];
      if (e1 > e0) CK(cudaMemcpyAsync(c->src.as<uint32_t>() + e0, src + e0, (e1 - e0) * 4, cudaMemcpyHostToDevice, c->stream));
      cudaEvent_t ev;
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      evs.push_back(ev);
      CK(cudaEventRecord(ev, c->stream));
      CK(cudaStreamWaitEvent(c->stream2, ev, 0));
      TRY(launched(c, launch_validate_csr(rp64.as<uint64_t>(), n, m, c->src.as<uint32_t>(), c->row_ptr.as<uint32_t>(),
                                          flags, flags + 1, c->thr_node, c->num_sms * 8, c->stream2, cut[q],
                                          cut[q + 1]), "k_validate_csr"));
    }
    {
      cudaEvent_t ev;
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      evs.push_back(ev);
      CK(cudaEventRecord(ev, c->stream2));
      CK(cudaStreamWaitEvent(c->stream, ev, 0));
    }
    CK(cudaMemcpyAsync(c->h_u64, flags, 16, cudaMemcpyDeviceToHost, c->stream));
    TRY(sync(c));
    dfree(c, rp64);
    c->max_deg = (uint32_t)c->h_u64[1];
    c->skip_tab_valid = false;
    const uint32_t err = (uint32_t)c->h_u64[0], row = (uint32_t)(c->h_u64[0] >> 32);
    if (err) {
      dfree(c, c->row_ptr);
      dfree(c, c->src);
      const char* what = (err & 1) ? "row_ptr must be non-decreasing and <= m"
                         : (err & 2) ? "src out of range"
                         : (err & 4) ? "self-loop"
                                     : "row not strictly ascending";
      return fail(c, GIM_EINVAL, std::string(what) + " (row " + std::to_string(row) + ")");
    }
  }
  // explicit weights: thresholds on the host, rows now known to be valid
  std::vector<uint64_t> thr;
  if (scheme == GIM_W_EXPLICIT) {
    thr.resize(std::max<uint64_t>(m, 1));
    for (uint32_t v = 0; v < n; ++v) {
      uint64_t acc = 0;
      for (uint64_t e = rp[v]; e < rp[v + 1]; ++e) {
        const float x = w[e];
        if (!(x >= 0.f && x <= 1.f)) { dfree(c, c->row_ptr); dfree(c, c->src); return fail(c, GIM_EINVAL, "weights must be in [0,1]"); }
        const double t = (double)x * 4294967296.0;   // exact for float32
        thr[e] = (model == GIM_LT) ? (uint64_t)std::floor(t) : (uint64_t)std::ceil(t);
        acc += thr[e];
      }
      if (model == GIM_LT && acc > 4294967296ull)
      {
        dfree(c, c->row_ptr);
        dfree(c, c->src);
        return fail(c, GIM_ELTWEIGHT, "LT in-weights of node " + std::to_string(v) + " sum above 1");
      }
    }
  }
  if (scheme == GIM_W_EXPLICIT) {
    TRY(dalloc(c, c->thr_edge, thr.size() * 8));
    CK(cudaMemcpyAsync(c->thr_edge.p, thr.data(), thr.size() * 8, cudaMemcpyHostToDevice, c->stream));
  }
  c->graph = true;
  set_l2_window(c);
  c->have_seed = false;
  TRY(reset_pool(c, 0));
  c->have_seed = false;
  return sync(c);
}

gim_status gim_set_shard(gim_ctx* c, int rank, int world) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  if (world < 1 || rank < 0 || rank >= world) return fail(c, GIM_EINVAL, "need 0 <= rank < world");
  c->rank = rank;
  c->world = world;
  c->have_seed = false;
  c->T_global = c->nsets = c->pool_len = 0;
  c->segs.clear();
  return GIM_OK;
}

gim_status gim_set_allgather(gim_ctx* c, gim_allgather_fn fn, void* user) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  c->agfn = fn;
  c->aguser = user;
  c->have_seed = false;                        // the pool layout changes: regenerate
  return GIM_OK;
}

gim_status gim_set_reducescatter(gim_ctx* c, gim_reducescatter_fn fn, void* user) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  c->rsfn = fn;
  c->rsuser = user;
  return GIM_OK;
}

gim_status gim_nccl_unique_id(void* id_out) {
  if (!id_out) return GIM_EINVAL;
  return nccl_unique_id(id_out) ? GIM_ECOLL : GIM_OK;
}

gim_status gim_set_nccl(gim_ctx* c, const void* id, int rank, int world, int protocol) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  if (!id || protocol < 0 || protocol > 2) return fail(c, GIM_EINVAL, "id required; protocol 0 (all-reduce), 1 (replicated), 2 (node-sharded)");
  if (rank != c->rank || world != c->world) return fail(c, GIM_EINVAL, "rank / world must match gim_set_shard");
  if (!nccl_available()) return fail(c, GIM_ECOLL, "libnccl.so.2 not found");
  DeviceGuard g(c->device);
  if (c->nccl) nccl_comm_destroy(c->nccl);
  c->nccl = nullptr;
  if (nccl_comm_init(&c->nccl, id, rank, world)) return fail(c, GIM_ECOLL, "ncclCommInitRank failed");
  c->arfn = nccl_allreduce_i32;
  c->aruser = c->nccl;
  c->agfn = protocol == 1 ? nccl_allgather_bytes : nullptr;
  c->aguser = protocol == 1 ? c->nccl : nullptr;
  c->rsfn = protocol == 2 ? nccl_reducescatter_i32 : nullptr;
  c->rsuser = protocol == 2 ? c->nccl : nullptr;
  return GIM_OK;
}

gim_status gim_set_allreduce(gim_ctx* c, gim_allreduce_fn fn, void* user) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  c->arfn = fn;
  c->aruser = user;
  return GIM_OK;
}

gim_status gim_generate_rr(gim_ctx* c, uint64_t theta, uint64_t seed) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  DeviceGuard g(c->device);
  const double t0 = now_ms();
  const gim_status s = generate(c, theta, seed);
  c->st.host_ms_api += now_ms() - t0;
  return s;
}

gim_status gim_select(gim_ctx* c, uint32_t k, uint32_t* seeds, uint64_t* gains, uint64_t* covered) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  if (!seeds) return fail(c, GIM_EINVAL, "seeds_out required");
  DeviceGuard g(c->device);
  const double t0 = now_ms();
  const gim_status s = select_impl(c, k, seeds, gains, covered);
  c->st.host_ms_api += now_ms() - t0;
  return s;
}

gim_status gim_imm(gim_ctx* c, uint32_t k, double eps, double ell, uint64_t seed, uint32_t* seeds,
                   gim_imm_result* res) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  if (!seeds) return fail(c, GIM_EINVAL, "seeds_out required");
  if (!c->graph) return fail(c, GIM_ESTATE, "no graph loaded");
  if (c->n < 2) return fail(c, GIM_EINVAL, "IMM needs n >= 2 (reading R25)");
  if (k < 1 || k > c->n) return fail(c, GIM_EINVAL, "k must satisfy 1 <= k <= n");
  if (!(eps > 0.0 && eps < 1.0)) return fail(c, GIM_EINVAL, "eps must be in (0,1)");
  if (!(ell > 0.0)) return fail(c, GIM_EINVAL, "ell must be > 0");
  DeviceGuard g(c->device);
  const double t_api = now_ms();
  const ImmConst K = imm_constants(c->n, k, eps, ell, c->rounds);
  gim_imm_result r;
  std::memset(&r, 0, sizeof(r));
  r.ell_eff = K.ell_eff;
  r.eps_prime = K.eps_p;
  r.lambda_prime = K.lambda_p;
  r.lambda_star = K.lambda_s;
  const double n = (double)c->n;
  c->have_seed = false;                                      // IMM starts from R = {}
  TRY(generate(c, 0, seed));
  double LB = 1.0;                                           // reading R6
  uint64_t cov = 0;
  std::vector<uint32_t> tmp((size_t)k * c->rounds);
  auto R_sets = [c]() { return c->T_global / c->rounds; };     // sets in API units
  const int i_max = (int)std::floor(std::log2(n)) - 1;       // reading R5
  const bool global_counts = !(c->world > 1 || c->force_coll) || c->agfn;
  // lookahead sampling (GIM_OPT_IMM_LOOKAHEAD): after a round the probe settled with
  // k * gain_0 / T = u_prev, the next rounds whose passing fraction (1 + eps') / 2^m is well above
  // u_prev are sampled in the same generate call (one sampling pass instead of several); each of
  // them then probes the counts of its own prefix of T_m sets. A round the probe does not settle
  // truncates the pool back to its T_m (the extra sets are dropped) and continues as usual.
  const bool can_look = c->imm_lookahead && c->imm_early_exit && c->rounds == 1 && c->world == 1 &&
                        !c->force_coll && !c->speculate;
  double u_prev = -1.0;
  uint64_t la_end = 0;                                       // pool size sampled ahead (0: none)
  // the probe's bound fraction u is about the same from round to round while the passing
  // fraction halves: once a probe did not settle its round, later ones will not either
  bool probe_on = true;
  for (int i = 1; i <= i_max && i <= 64; ++i) {              // Alg. 2 l.2
    const double x = n / std::ldexp(1.0, i);                 // l.3
    const double theta_i = K.lambda_p / x;                   // l.4 (f = lambda', reading R1)
    const uint64_t T = (uint64_t)std::ceil(theta_i);
    uint64_t R;
    if (la_end > T) {
      R = T;                                                 // this round's prefix of the pool
    } else {
      la_end = 0;
      R = std::max<uint64_t>(R_sets(), T);                   // l.5 (reading R4)
      uint64_t target = R;
      if (can_look && u_prev >= 0.0 && R_sets() < T)
        for (int m = i + 1; m <= i_max; ++m) {
          // (GIM_OPT_IMM_LOOKAHEAD = 2, tests: two rounds ahead whatever u_prev, to exercise drops)
          const bool ahead = c->imm_lookahead == 2 ? m <= i + 2
                                                   : u_prev < kLookSafety * (1.0 + K.eps_p) / std::ldexp(1.0, m);
          if (!ahead) break;
          target = (uint64_t)std::ceil(K.lambda_p / (n / std::ldexp(1.0, m)));
        }
      TRY(generate(c, target, seed, false));
      if (target > R) la_end = target;
      else if (R_sets() > R) TRY(truncate_pool(c, R * c->rounds));   // drop excess speculation
    }
    // speculative target while this round's selection runs: the next round's T if the test
    // fails, capped by ceil(lambda*/x), the largest theta a passing test can produce
    const uint64_t spec = std::min<uint64_t>(
        (i < i_max) ? (uint64_t)std::ceil(K.lambda_p / (x / 2.0)) : 0ull, (uint64_t)std::ceil(K.lambda_s / x));
    // bounded greedy: the smallest covered count c* that passes l.7 in the same double
    // arithmetic (the test is monotone in cov); a selection whose bound cov_j + (k - j) gain_j
    // drops below c* stops there, and the test below then fails as it would after k steps
    c->sel_cstar = 0;
    if (c->imm_early_exit) {
      auto passes = [&](uint64_t cv) { return (n * (double)cv) / (double)R >= (1.0 + K.eps_p) * x; };
      uint64_t lo = 0, hi = R + 1;             // passes(hi) assumed; c* = R + 1 if nothing passes
      while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (passes(mid)) hi = mid; else lo = mid + 1;
      }
      c->sel_cstar = lo;                       // >= 1 since R >= 1 (0 would disable the bound)
    }
    // probe: the first greedy pick is the argmax of count_total itself; when already
    // k * gain_0 < c* the bounded greedy would stop at its first cover, so the round's result
    // (one pick, cov = gain_0) is known without indexing the new sets or launching the
    // selection — their index segment is built later, merged with the next rounds' sets
    bool probed = false;
    const bool prefix = la_end > R;                          // the pool holds sets beyond this round
    if (c->sel_cstar && (c->inv_pending || prefix) && global_counts && !c->speculate && (probe_on || prefix)) {
      TRY(ensure(c, c->probe, 8));
      CK(cudaMemsetAsync(c->probe.p, 0, 8, c->stream));
      const uint32_t* counts = c->count_total.as<uint32_t>();
      if (prefix) {                                          // counts of the first R sets only
        TRY(ensure(c, c->cnt, nsp(c) * 4));
        CK(cudaMemcpyAsync(c->cnt.p, c->count_total.p, nsp(c) * 4, cudaMemcpyDeviceToDevice, c->stream));
        TRY(launched(c, launch_count_sub_range(c->pool.as<uint32_t>(), c->offsets.as<uint64_t>() + R,
                                               c->offsets.as<uint64_t>() + c->nsets, c->cnt.as<uint32_t>(),
                                               c->num_sms * 8, c->stream), "k_count_sub_range"));
        counts = c->cnt.as<uint32_t>();
      }
      {
        Prof pf(c, CLS_SELECT);
        TRY(launched(c, launch_argmax(const_cast<uint32_t*>(counts), nullptr, (uint32_t)nsp(c),
                                      c->probe.as<unsigned long long>(), 0, nullptr, c->num_sms * kArgmaxCtasPerSM,
                                      c->stream, c->rounds > 1), "k_argmax(probe)"));
      }
      CK(cudaMemcpyAsync(c->h_u64, c->probe.p, 8, cudaMemcpyDeviceToHost, c->stream));
      TRY(sync(c));
      const uint64_t g0 = c->h_u64[0] >> 32;
      if ((uint64_t)k * c->rounds * g0 < c->sel_cstar) {
        probed = true;
        cov = g0;
        c->last_sel_steps = 1;
        c->st.probe_stops++;
      }
      u_prev = probed ? (double)((uint64_t)k * c->rounds * g0) / (double)R : -1.0;
      if (!probed) probe_on = false;
    } else {
      u_prev = -1.0;
    }
    if (!probed && prefix) {                                 // lookahead mispredicted: back to T
      TRY(truncate_pool(c, R * c->rounds));
      la_end = 0;
      c->st.lookahead_drops++;
    }
    if (!probed) {
      const gim_status sst = select_launch(c, k);             // l.6 (reading R9)
      c->sel_cstar = 0;
      TRY(sst);
      if (c->speculate && spec > R) TRY(generate_speculative(c, spec, seed));
      TRY(select_finish(c, k, tmp.data(), nullptr, &cov));
    }
    c->sel_cstar = 0;
    r.theta_i[i - 1] = T;
    r.theta_i_real[i - 1] = theta_i;
    r.cov_i[i - 1] = cov;
    r.sel_steps_i[i - 1] = c->last_sel_steps;
    r.rounds = (uint32_t)i;
    if ((n * (double)cov) / (double)R >= (1.0 + K.eps_p) * x) {   // l.7 (reading R7)
      LB = (n * (double)cov) / (double)R / (1.0 + K.eps_p);       // l.8
      break;
    }
  }
  const double theta = K.lambda_s / LB;                      // reading R2
  const uint64_t T = (uint64_t)std::ceil(theta);
  uint64_t R_last = 0;
  for (uint32_t q = 0; q < r.rounds; ++q) R_last = std::max<uint64_t>(R_last, r.theta_i[q]);
  if (c->fresh_final) {
    // reading R29: the final phase on a fresh pool of ceil(theta) sets of a second key (the
    // different seed makes generate discard the estimation pool)
    TRY(generate(c, T, seed ^ 0x9E3779B97F4A7C15ull, false));
  } else {
    const uint64_t R_final = std::max<uint64_t>(R_last, T);   // reading R8
    TRY(generate(c, R_final, seed, false));                  // extends or truncates speculation
  }
  std::vector<uint64_t> gains((size_t)k * c->rounds);
  TRY(select_impl(c, k, seeds, gains.data(), &cov));
  r.LB = LB;
  r.theta = theta;
  r.R_final = R_sets();
  r.covered = cov;
  r.spread_est = n * (double)cov / (double)R_sets();        // Eq. 3
  if (res) *res = r;
  c->st.host_ms_api += now_ms() - t_api;
  return GIM_OK;
}

gim_status gim_rr_export(gim_ctx* c, uint64_t* n_sets, uint64_t* pool_len, uint64_t* ids, uint64_t* offs,
                         uint32_t* nodes, int sort_each_set) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  DeviceGuard g(c->device);
  if (n_sets) *n_sets = c->nsets;
  if (pool_len) *pool_len = c->pool_len;
  if (ids)
    for (const Seg& s : c->segs)
      for (uint64_t i = 0; i < s.count; ++i) ids[s.lstart + i] = s.gstart + i;
  std::vector<uint64_t> tmp;
  uint64_t* o = offs;
  if (!o && nodes && sort_each_set) {
    tmp.resize(c->nsets + 1);
    o = tmp.data();
  }
  if (o) {
    if (c->nsets == 0) o[0] = 0;
    else CK(cudaMemcpyAsync(o, c->offsets.p, (c->nsets + 1) * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  if (nodes && c->pool_len) CK(cudaMemcpyAsync(nodes, c->pool.p, c->pool_len * 4, cudaMemcpyDeviceToHost, c->stream));
  TRY(sync(c));
  if (nodes && sort_each_set)
    for (uint64_t i = 0; i < c->nsets; ++i) std::sort(nodes + o[i], nodes + o[i + 1]);
  return GIM_OK;
}

gim_status gim_set_rounds(gim_ctx* c, uint32_t rounds) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  if (rounds == 0) return fail(c, GIM_EINVAL, "rounds must be >= 1");
  if (c->graph && (uint64_t)c->n * rounds >= 0xFFFFFFFFull)
    return fail(c, GIM_EINVAL, "n * rounds must be < 2^32 - 1 (uint32 pair ids)");
  if (rounds != c->rounds) {
    c->rounds = rounds;
    if (c->graph) {                            // empty pool; count vectors sized n * rounds
      DeviceGuard g(c->device);
      TRY(reset_pool(c, c->seed));
    }
    c->have_seed = false;                      // the pool (and its index) is regenerated
  }
  return GIM_OK;
}

gim_status gim_mc_spread(gim_ctx* c, const uint32_t* seeds, uint32_t k, uint64_t trials, uint64_t mc_seed,
                         double* mean_out, double* stderr_out, uint32_t* sizes_out) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  if (!c->graph) return fail(c, GIM_ESTATE, "no graph loaded");
  if (c->model == GIM_LT && trials >= 0xFFFFFFull) return fail(c, GIM_EINVAL, "LT forward MC: trials < 2^24 - 1");
  if (!seeds || k < 1 || trials < 1 || !mean_out) return fail(c, GIM_EINVAL, "seeds, k >= 1, trials >= 1, mean_out required");
  for (uint32_t i = 0; i < k; ++i)
    if (seeds[i] >= c->n) return fail(c, GIM_EINVAL, "seed id out of range");
  DeviceGuard g(c->device);
  const uint64_t n = c->n, m = c->m;
  const int grid = c->num_sms * 8;
  if (!c->out_valid) {                          // out-CSR: once per graph
    TRY(dalloc(c, c->out_ptr, (n + 1) * 4));
    TRY(dalloc(c, c->out_dst, (m + 4) * 4));
    TRY(dalloc(c, c->out_in, (m + 4) * 4));
    TRY(dalloc(c, c->thr_wc, (m + 4) * 4));    // groups of 4 are read as one uint4
    TRY(ensure(c, c->scan_tmp, (scan_tiles(n) + 2) * 8));
    size_t tb = 0;
    CK(build_out_csr(nullptr, nullptr, c->n, m, c->scheme, nullptr, nullptr, nullptr, nullptr, nullptr, &tb,
                     nullptr, grid, c->stream));
    DevBuf tmp;
    TRY(dalloc(c, tmp, tb));
    const cudaError_t e = build_out_csr(c->row_ptr.as<uint32_t>(), c->src.as<uint32_t>(), c->n, m, c->scheme,
                                        c->out_ptr.as<uint32_t>(), c->out_dst.as<uint32_t>(), c->out_in.as<uint32_t>(),
                                        c->thr_wc.as<uint32_t>(), tmp.p, &tb, c->scan_tmp.as<uint64_t>(), grid,
                                        c->stream);
    dfree(c, tmp);
    if (e != cudaSuccess) return fail_cuda(c, "build_out_csr", e);
    c->out_valid = true;
  }
  TRY(ensure_giant_slots(c, 2u * (uint32_t)c->num_sms));   // one MC trial per slot at a time
  uint32_t mc_grid = std::min<uint32_t>(c->giant_slots, 2u * (uint32_t)c->num_sms);
  DevBuf lt_acc;                                   // LT: per-slot 64-bit (trial tag | accumulator)
  if (c->model == GIM_LT) {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    mc_grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(mc_grid, (free_b / 4) / (n * 8 + 1)));
    TRY(dalloc(c, lt_acc, (uint64_t)mc_grid * n * 8));
    CK(cudaMemsetAsync(lt_acc.p, 0, (uint64_t)mc_grid * n * 8, c->stream));
  }
  DevBuf dseeds, dsizes, dclaim;
  TRY(dalloc(c, dseeds, (uint64_t)k * 4));
  TRY(dalloc(c, dsizes, trials * 4));
  TRY(dalloc(c, dclaim, 8));
  CK(cudaMemcpyAsync(dseeds.p, seeds, (uint64_t)k * 4, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(dclaim.p, 0, 8, c->stream));
  const uint64_t bm_words = (n + 31) / 32;
  TRY(launched(c, launch_mc_ic(c->scheme, c->n, c->out_ptr.as<uint32_t>(), c->out_dst.as<uint32_t>(),
                               c->out_in.as<uint32_t>(), c->thr_wc.as<uint32_t>(), c->thr_edge.as<uint64_t>(),
                               c->thr_uniform, dseeds.as<uint32_t>(), k, trials, mc_seed,
                               dclaim.as<unsigned long long>(), dsizes.as<uint32_t>(), c->bitmaps.as<uint32_t>(),
                               c->gqueues.as<uint32_t>(), bm_words, (int)mc_grid, c->stream,
                               c->row_ptr.as<uint32_t>(),
                               c->model == GIM_LT ? lt_acc.as<unsigned long long>() : nullptr),
               c->model == GIM_LT ? "k_mc_lt" : "k_mc_ic"));
  std::vector<uint32_t> sz(trials);
  CK(cudaMemcpyAsync(sz.data(), dsizes.p, trials * 4, cudaMemcpyDeviceToHost, c->stream));
  TRY(sync(c));
  dfree(c, lt_acc);
  dfree(c, dseeds);
  dfree(c, dsizes);
  dfree(c, dclaim);
  // mean and standard error in trial order, the oracle's expressions (og_mc_spread)
  double sum = 0.0, sum2 = 0.0;
  for (uint64_t t = 0; t < trials; ++t) {
    sum += (double)sz[t];
    sum2 += (double)sz[t] * (double)sz[t];
  }
  const double mean = sum / (double)trials;
  const double var = sum2 / (double)trials - mean * mean;
  *mean_out = mean;
  if (stderr_out) *stderr_out = std::sqrt((var > 0 ? var : 0) / (double)trials);
  if (sizes_out) std::memcpy(sizes_out, sz.data(), trials * 4);
  return GIM_OK;
}

gim_status gim_counts_export(gim_ctx* c, uint32_t* count_out) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  if (!count_out) return fail(c, GIM_EINVAL, "count_out required");
  if (!c->graph) return fail(c, GIM_ESTATE, "no graph loaded");
  DeviceGuard g(c->device);
  // rounds may have been raised since the last generate (gim_set_rounds): the device vector
  // then has fewer than n * rounds entries
  if (c->count_total.bytes < nsp(c) * 4)
    return fail(c, GIM_ESTATE, "count vector does not match the MRIM rounds: generate first");
  CK(cudaMemcpyAsync(count_out, c->count_total.p, nsp(c) * 4, cudaMemcpyDeviceToHost, c->stream));
  return sync(c);
}

gim_status gim_set_option(gim_ctx* c, gim_option opt, int64_t value) {
  if (!c) return GIM_EINVAL;
  c->err.clear();
  switch (opt) {
    case GIM_OPT_FORCE_GIANT: c->force_giant = value ? 1 : 0; return GIM_OK;
    case GIM_OPT_QUEUE_CAP:
      if (value < 1 || value > kQMax) return fail(c, GIM_EINVAL, "queue cap must be in [1, kQMax]");
      c->qcap = (uint32_t)value;
      return GIM_OK;
    case GIM_OPT_PROFILE: c->profile = value ? 1 : 0; return GIM_OK;
    case GIM_OPT_SELECT_GRAPH: c->use_graph = value ? 1 : 0; return GIM_OK;
    case GIM_OPT_INV_SEGMENTS: c->inv_segmented = value ? 1 : 0; return GIM_OK;
    case GIM_OPT_MB_CHAINS: c->mb_chains = (int)value; return GIM_OK;
    case GIM_OPT_SPECULATE: c->speculate = value ? 1 : 0; return GIM_OK;
    case GIM_OPT_FRESH_FINAL: c->fresh_final = value ? 1 : 0; return GIM_OK;
    case GIM_OPT_SPILL:
      if (value < -1 || value > (int64_t)kSpillQ) return fail(c, GIM_EINVAL, "spill cap must be in [-1 (auto), 16384]");
      c->spill_cap = value;
      return GIM_OK;
    case GIM_OPT_SKIP: {
      const int on = value ? 1 : 0;
      if (on && c->graph && (c->model != MODEL_IC || c->scheme == W_EXPLICIT))
        return fail(c, GIM_EINVAL, "the geometric-skip contract needs IC with WC or uniform weights");
      if (on != c->skip) {
        c->skip = on;
        c->have_seed = false;                  // different RR sets: the pool restarts
      }
      if (value == 2 || value == 3) c->skip_lane = value - 2;   // test hook: 2 = warp only, 3 = lane first
      return GIM_OK;
    }
    case GIM_OPT_SELECT_PERSISTENT: c->sel_persistent = value ? 1 : 0; return GIM_OK;
    case GIM_OPT_IMM_EARLY_EXIT: c->imm_early_exit = value ? 1 : 0; return GIM_OK;
    case GIM_OPT_SELECT_CTA: c->sel_small = value ? 1 : 0; return GIM_OK;
    case GIM_OPT_IMM_LOOKAHEAD: c->imm_lookahead = (value < 0 || value > 2) ? 1 : (int)value; return GIM_OK;
    case GIM_OPT_SELECT_CLUSTER: c->sel_cluster = value ? 1 : 0; return GIM_OK;
    case GIM_OPT_INV_SORT: c->inv_sort = (value < -1 || value > 1) ? -1 : (int)value; return GIM_OK;
    case GIM_OPT_CHUNK:
      if (value != 0 && (value < 1024 || value > (int64_t)kChunk)) return fail(c, GIM_EINVAL, "chunk must be 0 or in [1024, 2^25]");
      c->chunk = (uint32_t)value;
      return GIM_OK;
    case GIM_OPT_L2_PERSIST:
      c->l2_persist = value ? 1 : 0;
      set_l2_window(c);
      return GIM_OK;
    case GIM_OPT_INV_PASSES: c->inv_passes = (value < 0 || value > 64) ? 0 : (int)value; return GIM_OK;
    case GIM_OPT_GIANT_NT:
      if (value != 0 && value != kGiantThreads && value != kGiantThreadsNarrow)
        return fail(c, GIM_EINVAL, "giant CTA width must be 0 (auto), 256 or 128");
      c->giant_nt_opt = (int)value;
      return GIM_OK;
    case GIM_OPT_PDL:
      set_pdl((int)value);
      if (c->sel_exec) cudaGraphExecDestroy(c->sel_exec);   // recapture with the new launch mode
      for (cudaGraphExec_t& ex : c->sel_parts) cudaGraphExecDestroy(ex);
      c->sel_parts.clear();
      c->sel_exec = nullptr;
      return GIM_OK;
    case GIM_OPT_IC_LANE: c->ic_lane = (value < -1 || value > 1) ? -1 : (int)value; return GIM_OK;
    case GIM_OPT_FUSED_CTAS:
      if (value < 1 || value > 16) return fail(c, GIM_EINVAL, "fused CTAs per SM must be in [1, 16]");
      c->fused_ctas = (int)value;
      if (c->sel_exec) cudaGraphExecDestroy(c->sel_exec);
      for (cudaGraphExec_t& ex : c->sel_parts) cudaGraphExecDestroy(ex);
      c->sel_parts.clear();
      c->sel_exec = nullptr;
      return GIM_OK;
    case GIM_OPT_SKIP_LANE_CAP:
      if (value < 1 || value > 512) return fail(c, GIM_EINVAL, "lane cap must be in [1, 512]");
      c->skip_lane_cap = (uint32_t)value;
      return GIM_OK;
    case GIM_OPT_GIANT_SHARED: c->giant_sq = value ? 1 : 0; return GIM_OK;
    case GIM_OPT_SELECT_COOP:
      if (value < 0 || value > (int64_t)kCoopCands) return fail(c, GIM_EINVAL, "coop candidate cap must be in [0, 8192]");
      c->sel_coop = (uint32_t)value;
      return GIM_OK;
    case GIM_OPT_FORCE_COLLECTIVES:
      c->force_coll = value ? 1 : 0;
      c->have_seed = false;
      return GIM_OK;
    case GIM_OPT_SELECT_FUSED:
      if (value < 0 || value > (1 << 16)) return fail(c, GIM_EINVAL, "fused candidate cap must be in [0, 65536]");
      c->sel_fused = (uint32_t)value;
      return GIM_OK;
    case GIM_OPT_ARGMAX_CAND: c->use_cand = (value < 0 || value > 2) ? 1 : (int)value; return GIM_OK;
    case GIM_OPT_STAGING_CAP:
      if (value < 0) return fail(c, GIM_EINVAL, "staging cap must be >= 0");
      c->staging_init = (uint64_t)value;
      c->stage_cap = 0;
      return GIM_OK;
  }
  return fail(c, GIM_EINVAL, "unknown option");
}

gim_status gim_get_stats(gim_ctx* c, gim_stats* out) {
  if (!c || !out) return GIM_EINVAL;
  *out = c->st;
  return GIM_OK;
}

gim_status gim_reset_stats(gim_ctx* c) {
  if (!c) return GIM_EINVAL;
  c->st = gim_stats{};
  return GIM_OK;
}

gim_status gim_microbench_philox(gim_ctx* c, uint64_t groups, double* ms) {
  if (!c || !ms || groups == 0) return GIM_EINVAL;
  const int chains = c->mb_chains;
  c->err.clear();
  DeviceGuard g(c->device);
  const int grid = c->num_sms * 8;
  const uint64_t threads = (uint64_t)grid * 256;
  const uint32_t per = (uint32_t)std::max<uint64_t>(1, groups / threads);
  DevBuf sink;
  TRY(dalloc(c, sink, 256));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(launch_philox_bench(1, per, sink.as<uint32_t>(), grid, c->stream, chains));   // warm-up
  CK(cudaEventRecord(a, c->stream));
  CK(launch_philox_bench(2, per, sink.as<uint32_t>(), grid, c->stream, chains));
  CK(cudaEventRecord(b, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  float t = 0.f;
  CK(cudaEventElapsedTime(&t, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  dfree(c, sink);
  c->st.launches += 2;
  *ms = (double)t * ((double)groups / (double)(threads * per));   // normalised to `groups`
  return sync(c);
}

}  // extern "C"

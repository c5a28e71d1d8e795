// rr.cu — RR-set generation kernels (K-IC/K-LT warp kernel, K-GIANT fallback, K-STORE).
//
// What they compute: RR_i = {u : u reaches root_i in the instance graph g_i}
// by a randomized reverse BFS over the in-CSR (Alg. 3), IC coin per in-edge
// slot, LT one in-edge per node (§3.7). B200 design:
//  * persistent warps claim RR ids dynamically (Alg. 6's N_b persistent blocks, P:449-478,
//    with ids pre-assigned instead of the N_RR/tail_RR mutex, reading R20);
//  * one warp per RR set (N_th = 32), frontier queue + visited hash in shared memory
//    (Q_shr; Visited as an exact-set hash, readings R12-R13);
//  * coins are drawn BEFORE the source column is loaded: lane l evaluates one Philox call = the
//    4 coins of slot group g = e >> 2, and only live edges read src[e];
//  * ballot/scan compaction of newly visited nodes into the append-only queue, which is also
//    the RR buffer (replaces RR_tmp);
//  * a set that outgrows the queue is aborted and replayed exactly by the block-per-RR giant
//    kernel with a global bitmap (replaces offloadQueue/reloadQueue, Alg. 4/5: the
//    keyed RNG makes the replay draw the same coins);
//  * two-pass storage: bump-allocated staging + sizes, then exclusive scan and a compacting
//    copy that also builds count_total (Occur; Alg. 6 l.4-11).
#include <atomic>
#ifdef GIM_GIANT_TRACE
#include <algorithm>
#include <cstdio>
#include <vector>
#endif
#include "gim_device.cuh"
#include "gim_internal.h"

namespace gim {

__device__ __forceinline__ uint32_t hash_slot(uint32_t u) { return __umulhi(u * 0x9E3779B1u, (uint32_t)kHSize); }

// Exact-set test-and-set in the shared-memory visited hash. Returns true iff u was absent.
__device__ __forceinline__ bool hash_insert(uint32_t* h, uint32_t u) {
  uint32_t s = hash_slot(u);
  while (true) {
    const uint32_t old = atomicCAS(&h[s], kEmpty, u);
    if (old == kEmpty) return true;
    if (old == u) return false;
    s = (s + 1 == (uint32_t)kHSize) ? 0u : s + 1;
  }
}

// Asynchronous 4-byte global -> shared copy (completion: cp_async_wait_all, then __syncwarp).
// dst: shared-space byte address (__cvta_generic_to_shared of the buffer, computed once)
__device__ __forceinline__ void cp_async4(uint32_t dst, const uint32_t* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }



// LT: index of the chosen in-edge of v (0..d-1) or d if none (reading R18). Warp-collective.
template <int SCHEME>
__device__ __forceinline__ uint32_t lt_choose(const RRParams& p, uint64_t id, uint32_t v,
                                              uint32_t a, uint32_t d, int lane) {
  const uint4 o = philox4x32_10(make_uint4((uint32_t)id, (uint32_t)(id >> 32), v, kSlotLtHi),
                                (uint32_t)p.seed, (uint32_t)(p.seed >> 32));
  const uint32_t r = o.x;
  if (SCHEME == W_WC) return __umulhi(r, d);            // floor(r * d / 2^32): uniform in-neighbour
  // explicit weights: first t with r < sum_{s<=t} W_s, warp prefix scan
  uint64_t carry = 0;
  for (uint32_t base = 0; base < d; base += 32) {
    const uint32_t t = base + lane;
    uint64_t x = (t < d) ? p.thr_edge[a + t] : 0ull;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, x, off);
      if (lane >= off) x += y;
    }
    x += carry;
    const uint32_t hit = __ballot_sync(kFull, t < d && (uint64_t)r < x);
    if (hit) return base + (__ffs(hit) - 1);
    carry = __shfl_sync(kFull, x, 31);
  }
  return d;
}


// Live-slot mask of slot group g from its 4 coins w: bit j set iff slot e = 4g + j lies in
// [a, b) and is live. WC: coin <= floor((2^32-1)/d) <=> coin * d < 2^32; UNIFORM: coin <=
// ceil(p 2^32) - 1; EXPLICIT: coin < ceil(w_e 2^32).
template <int SCHEME>
__device__ __forceinline__ uint32_t live_mask_words(const RRParams& p, uint4 w, uint32_t g, uint32_t a,
                                                    uint32_t b, uint32_t thr) {
  const uint32_t e0 = g << 2;
  uint32_t m;
  if (SCHEME == W_EXPLICIT) {
    m = 0;
    const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (e0 + j >= a && e0 + j < b && (uint64_t)words[j] < p.thr_edge[e0 + j]) m |= 1u << j;
    return m;
  }
  m = (uint32_t)(w.x <= thr) | ((uint32_t)(w.y <= thr) << 1) | ((uint32_t)(w.z <= thr) << 2) |
      ((uint32_t)(w.w <= thr) << 3);
  const uint32_t lo = a > e0 ? a - e0 : 0u;          // first valid word (group g_lo)
  const uint32_t hi = (b - e0) < 4u ? b - e0 : 4u;   // one past the last valid word (group g_hi)
  return m & (0xFFFFFFFFu << lo) & (0xFu >> (4u - hi));
}

// One lane's coins of slot group g (one Philox call) as a live mask. No memory is touched.
template <int SCHEME>
__device__ __forceinline__ uint32_t ic_live_mask(const RRParams& p, uint32_t id_lo, uint32_t id_hi,
                                                 uint32_t k0, uint32_t k1, uint32_t g, uint32_t a,
                                                 uint32_t b, uint32_t thr) {
  (void)k0; (void)k1;
  return live_mask_words<SCHEME>(p, philox4x32_10_rk(make_uint4(id_lo, id_hi, g, 0u), p.rk), g, a, b, thr);
}

// Slow path (some lane of the warp has a live slot): load src[e] for live slots only and
// test-and-set them in the visited structure; uu[j] = newly visited node or kEmpty.
template <class Visit>
__device__ __forceinline__ void ic_take_live(const RRParams& p, uint32_t g, uint32_t m,
                                             uint32_t (&uu)[4], Visit visit) {
  const uint32_t e0 = g << 2;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (m & (1u << j)) {
      const uint32_t u = __ldg(p.src + e0 + j);
      if (visit(u)) uu[j] = u;
    }
  }
}

// Per-node live threshold of the 32-bit fast test (WC and UNIFORM).
template <int SCHEME>
__device__ __forceinline__ uint32_t node_thr(const RRParams& p, uint32_t d) {
  if (SCHEME == W_WC) return 0xFFFFFFFFu / d;
  if (SCHEME == W_UNIFORM) return p.thr_uniform ? (uint32_t)(p.thr_uniform - 1) : 0u;
  return 0u;
}

// Warp-inclusive scan of the number of new nodes per lane; returns (exclusive offset, total).
__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t cnt, int lane, uint32_t& total) {
  uint32_t incl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, off);
    if (lane >= off) incl += y;
  }
  total = __shfl_sync(kFull, incl, 31);
  return incl - cnt;
}

// Flattened sweep of a batch's short slot-group ranges. Lane i of the batch
// brings node i's remaining groups [gs, gs + ngf) with its row range [a, b) and live threshold.
// The non-empty ranges are compacted into lanes 0..nne-1 once per batch; the owner of flattened
// group gi of a 32-group window is then one ballot + one redux away (the starts of non-empty
// ranges are distinct), instead of a 5-step dependent shuffle search per window.
struct Flat {
  uint32_t a, b, thr, gofs, start;   // compacted lane r: the r-th non-empty range; gofs = gs - start
  uint32_t nne, total;               // non-empty ranges, total flattened groups
};

__device__ __forceinline__ Flat flat_setup(uint32_t a, uint32_t b, uint32_t thr, uint32_t gs, uint32_t ngf,
                                           int lane) {
  Flat f;
  const uint32_t ne = __ballot_sync(kFull, ngf != 0u);
  f.nne = __popc(ne);
  const uint32_t E = warp_excl_scan(ngf, lane, f.total);
  // src = position of the (lane+1)-th set bit of ne (lanes >= nne get junk); usually every
  // node of the batch has a range (ne is a prefix mask) and src = lane
  uint32_t src = (uint32_t)lane;
  if (ne & (ne + 1u)) {                        // warp-uniform: some range is empty
    uint32_t r = (uint32_t)lane;
    src = 0;
#pragma unroll
    for (uint32_t w = 16; w >= 1; w >>= 1) {
      const uint32_t c = __popc((ne >> src) & ((1u << w) - 1u));
      if (c <= r) { r -= c; src += w; }
    }
    src &= 31u;
  }
  f.a = __shfl_sync(kFull, a, src);
  f.b = __shfl_sync(kFull, b, src);
  f.thr = __shfl_sync(kFull, thr, src);
  f.start = __shfl_sync(kFull, E, src);
  f.gofs = __shfl_sync(kFull, gs - E, src);
  return f;
}

// Compacted lane owning flattened group base + lane (any lane in [0, nne) if past the total).
__device__ __forceinline__ uint32_t flat_owner(const Flat& f, uint32_t base, int lane) {
  if (f.nne <= 1u) return 0u;                  // warp-uniform: a single range
  const bool ok = (uint32_t)lane < f.nne;
  const uint32_t before = __popc(__ballot_sync(kFull, ok && f.start < base));
  const uint32_t d = f.start - base;
  const uint32_t starts = __reduce_or_sync(kFull, (ok && f.start >= base && d < 32u) ? (1u << d) : 0u);
  const uint32_t cnt = before + __popc(starts & (0xFFFFFFFFu >> (31 - lane)));
  return cnt ? cnt - 1u : 0u;
}


// Slow path of the warp kernel: load src[e] for this lane's live slots of group g, test-and-set
// them in the smem visited hash and append the new nodes to the queue (warp-collective).
// Returns false (nothing appended) if the queue would overflow.
template <class Visit>
__device__ __forceinline__ bool append_live(const RRParams& p, uint32_t g, uint32_t m, uint32_t* q,
                                            uint32_t& tail, int lane, Visit vis) {
  uint32_t uu[4] = {kEmpty, kEmpty, kEmpty, kEmpty};
  if (m) ic_take_live(p, g, m, uu, vis);
  const uint32_t cnt = (uu[0] != kEmpty) + (uu[1] != kEmpty) + (uu[2] != kEmpty) + (uu[3] != kEmpty);
  uint32_t total;
  if (!__any_sync(kFull, cnt > 1u)) {
    // common case (WC: ~one live in-edge per node): at most one new node per lane, so the
    // append offsets are a ballot prefix instead of a warp scan
    const uint32_t has = __ballot_sync(kFull, cnt != 0u);
    total = __popc(has);
    if (tail + total > p.qcap) return false;
    if (cnt) q[tail + __popc(has & ((1u << lane) - 1u))] = min(min(uu[0], uu[1]), min(uu[2], uu[3]));
  } else {
    uint32_t pos = tail + warp_excl_scan(cnt, lane, total);
    if (tail + total > p.qcap) return false;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (uu[j] != kEmpty) q[pos++] = uu[j];
  }
  tail += total;
  return true;
}


// Sweep of whole hub steps: groups [g0, g0 + steps * kHubGroups) of a node with in-edge range
// [a, b), all inside [a>>2, (b-1)>>2] (the node's remaining groups, fewer than one step, are
// swept by the flattened batch). kHubIlp independent Philox chains per lane, interleaved round
// by round. Fast path: only "could any coin be live?" — the minimum of a lane's 4*kHubIlp coins
// against the node threshold — then one warp vote; exact masks (packed 4 bits per chain) are
// built from the same registers only when some lane may hold a live slot.
template <int SCHEME, class OnLive>
__device__ __forceinline__ bool hub_sweep_whole(const RRParams& p, uint32_t id_lo, uint32_t id_hi,
                                                uint32_t a, uint32_t b, uint32_t g0, uint32_t steps,
                                                uint32_t thr, bool never, int lane, uint32_t& lives,
                                                OnLive on_live) {
  if (never) return true;
  for (uint32_t gb = g0, s = 0; s < steps; ++s, gb += kHubGroups) {
    uint4 w[kHubIlp];
#pragma unroll
    for (int r = 0; r < kHubIlp; ++r) w[r] = make_uint4(id_lo, id_hi, gb + 32u * r + lane, 0u);
    philox4x32_10_rk_xn<kHubIlp>(w, p.rk);
    uint32_t mn = 0xFFFFFFFFu;
#pragma unroll
    for (int r = 0; r < kHubIlp; ++r) mn = min(mn, min(min(w[r].x, w[r].y), min(w[r].z, w[r].w)));
    if (!__any_sync(kFull, SCHEME == W_EXPLICIT || mn <= thr)) continue;
    uint32_t packed = 0;
    if (SCHEME != W_EXPLICIT) {
#pragma unroll
      for (int r = 0; r < kHubIlp; ++r)
        packed |= live_mask_words<SCHEME>(p, w[r], gb + 32u * r + lane, a, b, thr) << (4 * r);
      if (!__any_sync(kFull, packed)) continue;
    }
#pragma unroll 1
    for (int r = 0; r < kHubIlp; ++r) {
      uint32_t m;
      if (SCHEME != W_EXPLICIT) {
        m = (packed >> (4 * r)) & 0xFu;
      } else {   // per-edge thresholds: one chain's mask at a time (register pressure)
        uint4 wr = w[0];
#pragma unroll
        for (int t = 1; t < kHubIlp; ++t) wr = (t == r) ? w[t] : wr;
        m = live_mask_words<SCHEME>(p, wr, gb + 32u * r + lane, a, b, thr);
      }
      if (!__any_sync(kFull, m)) continue;
      lives += __popc(m);
      if (!on_live(gb + 32u * r + lane, m)) return false;
    }
  }
  return true;
}

// Sweep of one node's slot groups [a>>2, (b-1)>>2] with kHubIlp independent Philox chains per
// lane (128 x kHubIlp slots per warp step). Fast path: only "could any coin be live?" — the
// minimum of a lane's 4*kHubIlp coins against the node threshold — then one warp vote; the
// exact masks are built from the same registers only when some lane may hold a live slot.
// on_live(g, mask) is warp-collective and returns false to abort the sweep.
template <int SCHEME, class OnLive>
__device__ __forceinline__ bool hub_sweep(const RRParams& p, uint32_t id_lo, uint32_t id_hi, uint32_t a,
                                          uint32_t b, uint32_t thr, bool never, int lane,
                                          uint32_t& lives, OnLive on_live) {
  const uint32_t g_lo = a >> 2, g_hi = (b - 1) >> 2;
  for (uint32_t gb = g_lo; gb <= g_hi; gb += kHubGroups) {
    uint4 w[kHubIlp];
#pragma unroll
    for (int r = 0; r < kHubIlp; ++r) w[r] = make_uint4(id_lo, id_hi, gb + 32u * r + lane, 0u);
    philox4x32_10_rk_xn<kHubIlp>(w, p.rk);        // groups past g_hi are computed and ignored
    uint32_t mn = 0xFFFFFFFFu;
#pragma unroll
    for (int r = 0; r < kHubIlp; ++r) {
      if (gb + 32u * r + lane > g_hi) w[r] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
      mn = min(mn, min(min(w[r].x, w[r].y), min(w[r].z, w[r].w)));
    }
    const bool maybe = !never && (SCHEME == W_EXPLICIT || mn <= thr || (g_hi - gb) < 32u * kHubIlp);
    if (!__any_sync(kFull, maybe)) continue;
#pragma unroll 1
    for (int r = 0; r < kHubIlp; ++r) {
      uint4 wr = w[0];
#pragma unroll
      for (int t = 1; t < kHubIlp; ++t) wr = (t == r) ? w[t] : wr;
      const uint32_t g = gb + 32u * r + lane;
      const uint32_t m = (g <= g_hi && !never) ? live_mask_words<SCHEME>(p, wr, g, a, b, thr) : 0u;
      if (!__any_sync(kFull, m)) continue;
      lives += __popc(m);
      if (!on_live(g, m)) return false;
    }
  }
  return true;
}

// ------------------------------------------------------------------------------------------
// K-RR: warp-per-RR persistent kernel.
// ------------------------------------------------------------------------------------------
template <int MODEL, int SCHEME>
__global__ void __launch_bounds__(kRRWarps * 32, kRRBlocksPerSM) k_rr_warp(RRParams p) {
  extern __shared__ uint32_t smem[];
  const int lane = threadIdx.x & 31;
  uint32_t* q = smem + (threadIdx.x >> 5) * (kQMax + kHSize + kPend);
  uint32_t* h = q + kQMax;
  uint32_t* pend = h + kHSize;
  const uint32_t pend_s = (uint32_t)__cvta_generic_to_shared(pend);
  for (int i = lane; i < kHSize; i += 32) h[i] = kEmpty;
  __syncwarp();
  // spill tier (p.spill_cap > p.qcap): this warp's global queue + hash for sets > qcap
  const uint64_t gwarp = (uint64_t)blockIdx.x * kRRWarps + (threadIdx.x >> 5);
  uint32_t* gq = p.spill + gwarp * (uint64_t)(kSpillQ + kSpillH);
  uint32_t* gh = gq + kSpillQ;
  const bool can_spill = p.spill_cap > p.qcap;
  const uint32_t k0 = (uint32_t)p.seed, k1 = (uint32_t)(p.seed >> 32);
  unsigned long long coins = 0;     // per-lane counters (statistics only)
  uint32_t lives = 0;

  const uint32_t count = p.count_ptr ? *p.count_ptr : p.count;
  uint32_t claim_next = 0, claim_end = 0;            // ids claimed kClaimBatch at a time
  unsigned long long chunk_off = 0;                  // this warp's staging chunk
  uint32_t chunk_left = 0;
  while (true) {
    if (claim_next == claim_end) {
      // batches amortise the shared counter (tiny sets); single ids near the end keep the
      // heavy-tailed last sets from piling up on one warp
      const uint32_t batch = (claim_end < count - count / kClaimTailDiv) ? kClaimBatch : 1u;
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&p.ctr->claim, batch);
      claim_next = __shfl_sync(kFull, base, 0);
      claim_end = claim_next + batch;
    }
    const uint32_t i = claim_next++;
    if (i >= count) break;
    const uint32_t item = p.item_list ? p.item_list[i] : i;
    if (p.force_giant) {
      if (lane == 0) p.giant_recs[atomicAdd(&p.ctr->giant_count, 1u)] = GiantRec{item, 0u, 0u, 0u, 0ull};
      continue;
    }
    const uint64_t id = p.id_base + item;
    const uint32_t id_lo = (uint32_t)id, id_hi = (uint32_t)(id >> 32);
    const uint32_t root = rr_root_of(p.seed, id, p.n, p.rounds);
    if (lane == 0) {
      q[0] = root;
      h[hash_slot(root)] = root;     // table is empty here
    }
    __syncwarp();
    uint32_t head = 0, tail = 1, resume = 0;
    bool overflow = false;
    bool spilled = false;                              // warp-uniform: members in gq / gh
    if (MODEL == MODEL_IC) {
      const bool never = (SCHEME == W_UNIFORM) && p.thr_uniform == 0;
      // Live in-edges found during a batch are not resolved on the spot: each lane starts an
      // asynchronous copy of src[e] into pend[] and the sweep goes on, so the batch's source
      // loads overlap its remaining coin work and each other. flush() waits once, then
      // test-and-sets the sources in the visited hash and appends the new ones to the queue.
      uint32_t npend = 0;                                // warp-uniform
      auto flush = [&]() -> bool {
        cp_async_wait_all();
        __syncwarp();
        bool ok = true;
        for (uint32_t base = 0; base < npend; base += 32) {
          const uint32_t i = base + lane;
          uint32_t u = 0;
          bool isnew = false;
          if (i < npend) {
            u = pend[i];
            isnew = spilled ? spill_hash_insert(gh, u) : hash_insert(h, u);
          }
          const uint32_t has = __ballot_sync(kFull, isnew);
          const uint32_t total = __popc(has);
          if (!spilled && can_spill && tail + total > p.qcap) {
            // move the set to the spill tier: queue copied, members re-inserted in gh
            for (uint32_t t = lane; t < tail; t += 32) {
              const uint32_t x = q[t];
              gq[t] = x;
              spill_hash_insert(gh, x);
            }
            if (isnew) spill_hash_insert(gh, u);
            spilled = true;
            __syncwarp();
          }
          if (tail + total > (spilled ? p.spill_cap : p.qcap)) { ok = false; break; }
          if (isnew) (spilled ? gq : q)[tail + __popc(has & ((1u << lane) - 1u))] = u;
          tail += total;
        }
        npend = 0;
        __syncwarp();
        return ok;
      };
      auto pend_add = [&](uint32_t g, uint32_t m) -> bool {
        const uint32_t cnt = __popc(m);
        uint32_t total, off;
        if (!__any_sync(kFull, cnt > 1u)) {            // usual case: <= 1 live slot per lane
          const uint32_t has = __ballot_sync(kFull, cnt != 0u);
          total = __popc(has);
          off = __popc(has & ((1u << lane) - 1u));
        } else {
          off = warp_excl_scan(cnt, lane, total);
        }
        if (npend + total > (uint32_t)kPend && !flush()) return false;
        uint32_t pos = pend_s + 4u * (npend + off);
        const uint32_t* sp = p.src + (g << 2);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (m & (1u << j)) { cp_async4(pos, sp + j); pos += 4u; }
        npend += total;
        return true;
      };
      // Expand every pending frontier node of this RR set together: lane i holds node
      // q[head + i] of the batch (row range, live threshold, group count), the warp sweeps the
      // concatenation of their slot-group ranges 32 groups at a time, and live in-edges found
      // anywhere in a sweep step are appended in one warp-wide step.
      while (head < tail) {
        const uint32_t nb = min(tail - head, 32u);
        uint32_t a = 0, b = 0, thr = 0, ng = 0;
        if (lane < nb) {
          const uint32_t v = spilled ? gq[head + lane] : q[head + lane];
          const uint32_t tv = (SCHEME == W_WC) ? __ldg(p.thr_node + v) : 0u;   // loads in parallel
          a = __ldg(p.row_ptr + v);
          b = __ldg(p.row_ptr + v + 1);
          if (b > a) {
            ng = ((b - 1) >> 2) - (a >> 2) + 1;
            thr = (SCHEME == W_WC) ? tv : node_thr<SCHEME>(p, b - a);
          }
        }
        coins += b - a;
        resume = head;                                  // batch start: re-expanded on overflow
        head += nb;
        // a hub (>= kHubGroups slot groups) sweeps its whole kHubGroups-steps alone below; the
        // remaining < kHubGroups groups of every node are flattened here
        const uint32_t hub_full = ng & ~(kHubGroups - 1u);
        const uint32_t hubs = __ballot_sync(kFull, hub_full != 0u);
        const uint32_t ngf = ng - hub_full;
        const uint32_t gs = (a >> 2) + hub_full;        // first flattened group of this node
        const Flat f = flat_setup(a, b, thr, gs, ngf, lane);
        const uint32_t total_g = f.total;
        for (uint32_t base = 0; base < total_g; base += 32) {
          const uint32_t gi = base + lane;
          const uint32_t k = flat_owner(f, base, lane);   // compacted range of flattened group gi
          const uint32_t ak = __shfl_sync(kFull, f.a, k), bk = __shfl_sync(kFull, f.b, k);
          const uint32_t tk = __shfl_sync(kFull, f.thr, k), gk = __shfl_sync(kFull, f.gofs, k);
          const uint32_t g = gk + gi;
          uint32_t m = 0;
          if (gi < total_g && !never) m = ic_live_mask<SCHEME>(p, id_lo, id_hi, k0, k1, g, ak, bk, tk);
#ifdef GIM_WINSTAT
          if (lane == 0) {
            atomicAdd(&p.ctr->dbg[0], 1ull);
            atomicAdd(&p.ctr->dbg[1], (unsigned long long)min(32u, total_g - base));
          }
#endif
          if (!__any_sync(kFull, m)) continue;          // no live in-edge in these 128 slots
          lives += __popc(m);
          if (!pend_add(g, m)) { overflow = true; break; }
        }
        // hub sweep: kHubIlp independent Philox chains per lane, 128 x kHubIlp slots per step
        for (uint32_t hm = overflow ? 0u : hubs; hm; hm &= hm - 1) {
          const uint32_t k = __ffs(hm) - 1;
          const uint32_t ak = __shfl_sync(kFull, a, k), bk = __shfl_sync(kFull, b, k);
          const uint32_t tk = __shfl_sync(kFull, thr, k), hk = __shfl_sync(kFull, hub_full, k);
#ifdef GIM_WINSTAT
          if (lane == 0) atomicAdd(&p.ctr->dbg[2], (unsigned long long)(hk / kHubGroups));
#endif
          if (!hub_sweep_whole<SCHEME>(p, id_lo, id_hi, ak, bk, ak >> 2, hk / kHubGroups, tk, never, lane,
                                       lives, pend_add))
            overflow = true;
        }
        if (!overflow && !flush()) overflow = true;
        __syncwarp();
        if (overflow) break;
      }
    } else {  // LT: frontier <= 1
      while (head < tail) {
        const uint32_t v = q[head++];
        const uint32_t a = __ldg(p.row_ptr + v), b = __ldg(p.row_ptr + v + 1);
        if (b <= a) continue;
        resume = head - 1;
        const uint32_t d = b - a;
        const uint32_t j = lt_choose<SCHEME>(p, id, v, a, d, lane);
        if (lane == 0) { coins += 1; lives += (j < d); }
        if (j < d) {
          uint32_t isnew = 0, u = 0;
          if (lane == 0) {
            u = __ldg(p.src + a + j);
            isnew = hash_insert(h, u);
          }
          isnew = __shfl_sync(kFull, isnew, 0);
          u = __shfl_sync(kFull, u, 0);
          if (isnew) {
            if (tail + 1 > p.qcap) { overflow = true; }
            else {
              if (lane == 0) q[tail] = u;
              tail += 1;
            }
          }
        }
        __syncwarp();
        if (overflow) break;
      }
    }
    if (overflow) {
      // hand the partial BFS to the giant kernel: q[0..tail) are visited and q[0..resume) are
      // fully expanded; the batch being expanded (q[resume..]) is re-expanded there with the
      // same coins, so the continuation is exact.
      unsigned long long off = 0;
      if (lane == 0) off = atomicAdd(&p.ctr->dump_tail, (unsigned long long)tail);
      off = __shfl_sync(kFull, off, 0);
      const bool fits = off + tail <= p.dump_cap;
      if (fits)
        for (uint32_t t = lane; t < tail; t += 32) p.dump[off + t] = spilled ? gq[t] : q[t];
      if (lane == 0)
        p.giant_recs[atomicAdd(&p.ctr->giant_count, 1u)] =
            fits ? GiantRec{item, tail, resume, 0u, off} : GiantRec{item, 0u, 0u, 0u, 0ull};
    } else {
      if (tail > chunk_left) {                       // reserve a new staging chunk
        const uint32_t want = max(tail, kStageChunk);
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&p.ctr->stage_tail, (unsigned long long)want);
        chunk_off = __shfl_sync(kFull, base, 0);
        chunk_left = want;
      }
      const unsigned long long off = chunk_off;
      chunk_off += tail;
      chunk_left -= tail;
      if (off + tail > p.stage_cap) {
        if (lane == 0) p.retry_list[atomicAdd(&p.ctr->retry_count, 1u)] = item;
      } else {
        for (uint32_t t = lane; t < tail; t += 32) p.staging[off + t] = spilled ? gq[t] : q[t];
        if (lane == 0) { p.sizes[item] = tail; p.soff[item] = off; }
      }
    }
    // clear the visited structures: the shared hash as a whole (vectorised, 4 KB: measured
    // faster than erasing by member list, 11.41 vs 11.71 ms C3 sampling); the spill hash by
    // member list, or wholly after an overflow (nodes hashed but never queued)
    if (overflow) cp_async_wait_all();
    uint4* h4 = reinterpret_cast<uint4*>(h);
    for (int t = lane; t < kHSize / 4; t += 32) h4[t] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    if (spilled && overflow) {
      uint4* gh4 = reinterpret_cast<uint4*>(gh);
      for (uint32_t t = lane; t < kSpillH / 4; t += 32) gh4[t] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    } else if (spilled) {
      for (uint32_t t = lane; t < tail; t += 32) spill_hash_erase(gh, gq[t]);
    }
    __syncwarp();
  }
  // per-warp statistics
  unsigned long long c64 = coins, l64 = lives;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    c64 += __shfl_xor_sync(kFull, c64, off);
    l64 += __shfl_xor_sync(kFull, l64, off);
  }
  if (lane == 0) {
    atomicAdd(&p.ctr->coins, c64);
    atomicAdd(&p.ctr->live, l64);
  }
}

// Lane-per-set kernels: refill the lanes that want a new set (mask `need`) from the warp's pool of
// claimed ids [pool_next, pool_end) (warp-uniform); one global atomic per kLaneClaim sets instead
// of one per refill — with 1.5-node sets a refill happens almost every iteration, and the
// returning atomic on the shared counter was the top stall of K-IC-lane on C5 (35% of ncu
// samples). Returns this lane's id (meaningful for the lanes in `need`). Warp-collective.
#ifndef GIM_LANE_CLAIM
#define GIM_LANE_CLAIM 64
#endif
constexpr uint32_t kLaneClaim = GIM_LANE_CLAIM;
static_assert(kLaneClaim >= 32, "one claim must cover a full warp refill");
__device__ __forceinline__ uint32_t lane_claim(unsigned int* ctr, uint32_t need, uint32_t& pool_next,
                                               uint32_t& pool_end, int lane) {
  const uint32_t nneed = __popc(need), avail = pool_end - pool_next;
  uint32_t base = 0;
  if (avail < nneed) {
    if (lane == 0) base = atomicAdd(ctr, kLaneClaim);
    base = __shfl_sync(kFull, base, 0);
  }
  const uint32_t r = __popc(need & ((1u << lane) - 1u));
  const uint32_t i = r < avail ? pool_next + r : base + (r - avail);
  if (avail < nneed) {
    pool_next = base + (nneed - avail);
    pool_end = base + kLaneClaim;
  } else {
    pool_next += nneed;
  }
  return i;
}

// ------------------------------------------------------------------------------------------
// K-IC lane kernel (tiny RR sets, e.g. uniform p = 0.01 on C5: ~1.5 nodes and ~56 coins per
// set): each lane owns one RR set with a 32-node queue in shared memory (lane-interleaved) that is
// also its visited set; every iteration each lane evaluates ONE slot group (one Philox = 4 coins)
// of its current node, so the warp's Philox work stays lane-parallel across 32 independent sets.
// A set that reaches a node with > kIcLaneMaxDeg in-edges or more than kIcLaneCap nodes is
// escalated: its id goes to esc_list and the warp kernel replays it exactly (same coins).
// ------------------------------------------------------------------------------------------
template <int SCHEME>
__global__ void __launch_bounds__(kIcLaneWarps * 32, kIcLaneBlocksPerSM) k_rr_ic_lane(RRParams p) {
  extern __shared__ uint32_t smem[];
  const int lane = threadIdx.x & 31;
  uint32_t* qv = smem + (threadIdx.x >> 5) * (kIcLaneCap * 32);     // qv[i * 32 + lane]
  const bool never = (SCHEME == W_UNIFORM) && p.thr_uniform == 0;
  uint32_t item = 0, head = 0, tail = 0, a = 0, b = 0, g = 0, g_hi = 0, thr = 0;
  uint64_t id = 0;
  bool active = false, want = true, on_node = false;
  uint32_t coins = 0, lives = 0;
  unsigned long long chunk_off = 0;
  uint32_t chunk_left = 0;
  uint32_t pool_next = 0, pool_end = 0;      // warp-uniform pool of claimed ids
  while (true) {
    const uint32_t need = __ballot_sync(kFull, want);
    if (need) {                              // refill finished lanes from the warp's id pool
      const uint32_t i = lane_claim(&p.ctr->claim_lane, need, pool_next, pool_end, lane);
      if (want) {
        want = false;
        active = i < p.count;
        if (active) {
          item = p.item_list ? p.item_list[i] : i;
          id = p.id_base + item;
          qv[lane] = rr_root_of(p.seed, id, p.n, p.rounds);
          head = 0;
          tail = 1;
          on_node = false;
          if (p.force_giant) {                 // forced fallback: everything via the warp kernel
            p.esc_list[atomicAdd(&p.ctr->esc_count, 1u)] = item;
            active = false;
            want = true;
          }
        }
      }
    }
    if (!__any_sync(kFull, active)) {
      if (!__any_sync(kFull, want)) break;
      continue;
    }
    bool finish = false, escalate = false;
    if (active && !on_node) {                // next node of this lane's BFS
      if (head == tail) {
        finish = true;
      } else {
        const uint32_t v = qv[head * 32 + lane];
        ++head;
        a = __ldg(p.row_ptr + v);
        b = __ldg(p.row_ptr + v + 1);
        if (b - a > kIcLaneMaxDeg) {
          escalate = true;
        } else if (b > a) {
          on_node = true;
          g = a >> 2;
          g_hi = (b - 1) >> 2;
          thr = node_thr<SCHEME>(p, b - a);
          coins += b - a;
        }
      }
    }
    if (active && on_node) {                 // one slot group of the current node
      const uint4 w = philox4x32_10_rk(make_uint4((uint32_t)id, (uint32_t)(id >> 32), g, 0u), p.rk);
      uint32_t m = never ? 0u : live_mask_words<SCHEME>(p, w, g, a, b, thr);
      lives += __popc(m);
      while (m) {
        const uint32_t j = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t u = __ldg(p.src + (g << 2) + j);
        bool seen = false;
        for (uint32_t t = 0; t < tail; ++t) seen |= (qv[t * 32 + lane] == u);
        if (!seen) {
          if (tail == (uint32_t)kIcLaneCap) { escalate = true; break; }
          qv[tail * 32 + lane] = u;
          ++tail;
        }
      }
      if (++g > g_hi) on_node = false;
    }
    if (escalate) {
      p.esc_list[atomicAdd(&p.ctr->esc_count, 1u)] = item;
      active = false;
      want = true;
    }
    // finished sets: warp-aggregated staging (per-warp chunk), then per-lane copy
    const uint32_t fin = __ballot_sync(kFull, finish);
    if (fin) {
      uint32_t incl = finish ? tail : 0u;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, off);
        if (lane >= off) incl += y;
      }
      const uint32_t tot = __shfl_sync(kFull, incl, 31);
      if (tot > chunk_left) {
        const uint32_t want_el = max(tot, kStageChunk);
        unsigned long long b0 = 0;
        if (lane == 0) b0 = atomicAdd(&p.ctr->stage_tail, (unsigned long long)want_el);
        chunk_off = __shfl_sync(kFull, b0, 0);
        chunk_left = want_el;
      }
      const unsigned long long base = chunk_off;
      chunk_off += tot;
      chunk_left -= tot;
      if (finish) {
        const unsigned long long off = base + incl - tail;
        if (off + tail > p.stage_cap) {
          p.retry_list[atomicAdd(&p.ctr->retry_count, 1u)] = item;
        } else {
          for (uint32_t t = 0; t < tail; ++t) p.staging[off + t] = qv[t * 32 + lane];
          p.sizes[item] = tail;
          p.soff[item] = off;
        }
        active = false;
        want = true;
      }
    }
  }
  unsigned long long c64 = coins, l64 = lives;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    c64 += __shfl_xor_sync(kFull, c64, off);
    l64 += __shfl_xor_sync(kFull, l64, off);
  }
  if (lane == 0) {
    atomicAdd(&p.ctr->coins, c64);
    atomicAdd(&p.ctr->live, l64);
  }
}

cudaError_t launch_rr_ic_lane(int scheme, const RRParams& p, int grid, cudaStream_t s) {
  const int smem = kIcLaneWarps * kIcLaneCap * 32 * 4;
  if (scheme == W_WC) k_rr_ic_lane<W_WC><<<grid, kIcLaneWarps * 32, smem, s>>>(p);
  else if (scheme == W_UNIFORM) k_rr_ic_lane<W_UNIFORM><<<grid, kIcLaneWarps * 32, smem, s>>>(p);
  else k_rr_ic_lane<W_EXPLICIT><<<grid, kIcLaneWarps * 32, smem, s>>>(p);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K-LT: lane-per-walk LT sampling (§3.7: at most one live in-edge per node, so the
// "frontier" is one node and the RR set is a reverse walk). Each lane owns one RR set; 32 walks
// per warp hide each other's dependent-load latency (row_ptr -> draw -> src -> membership).
// The lane's path sits in shared memory (lane-interleaved, conflict-free) and is also the
// membership set: a walk stops at a node with no chosen in-edge or at a node already on the
// path (R19). Walks longer than kLtCap hand their path to K-GIANT (exact resume at the last
// node: same draw, same chosen edge).
// ------------------------------------------------------------------------------------------

template <int SCHEME>
__device__ __forceinline__ uint32_t lt_choose_lane(const RRParams& p, uint64_t id, uint32_t v, uint32_t a,
                                                   uint32_t d) {
  const uint4 o = philox4x32_10_rk(make_uint4((uint32_t)id, (uint32_t)(id >> 32), v, kSlotLtHi), p.rk);
  const uint32_t r = o.x;
  if (SCHEME == W_WC) return __umulhi(r, d);           // floor(r * d / 2^32)
  uint64_t acc = 0;                                      // explicit: half-open fixed-point intervals
  for (uint32_t t = 0; t < d; ++t) {
    acc += p.thr_edge[a + t];
    if ((uint64_t)r < acc) return t;
  }
  return d;
}

template <int SCHEME>
__global__ void __launch_bounds__(kLtWarps * 32) k_rr_lt_lane(RRParams p) {
  extern __shared__ uint32_t smem[];
  const int lane = threadIdx.x & 31;
  uint32_t* path = smem + (threadIdx.x >> 5) * (kLtCap * 32);   // path[i * 32 + lane]
  const uint64_t gwarp = (uint64_t)blockIdx.x * kLtWarps + (threadIdx.x >> 5);
  uint32_t* spill = p.lt_spill + gwarp * (uint64_t)((kLtCap2 - kLtCap) * 32);   // entries >= kLtCap
  auto at = [&](uint32_t t) -> uint32_t& {
    return t < (uint32_t)kLtCap ? path[t * 32 + lane] : spill[(t - kLtCap) * 32 + lane];
  };
  uint32_t item = 0, v = 0, len = 0;
  uint64_t id = 0;
  bool active = false, want = true;       // want: lane needs a new walk
  uint32_t coins = 0, lives = 0;
  const uint32_t cap = min((uint32_t)kLtCap2, p.qcap);
  // 128-bit Bloom filter of the lane's path (one hashed bit per member): a next node whose bit is
  // clear is certainly new, so the O(len) membership scan runs only on a possible revisit
  uint32_t bl0 = 0, bl1 = 0, bl2 = 0, bl3 = 0;
  auto bloom_bit = [](uint32_t u) { return (u * 0x9E3779B1u) >> 25; };   // 0..127
  auto bloom_test = [&](uint32_t h) {
    const uint32_t w = (h & 64u) ? ((h & 32u) ? bl3 : bl2) : ((h & 32u) ? bl1 : bl0);
    return (w >> (h & 31u)) & 1u;
  };
  auto bloom_set = [&](uint32_t h) {
    const uint32_t b = 1u << (h & 31u);
    if (h < 32u) bl0 |= b; else if (h < 64u) bl1 |= b; else if (h < 96u) bl2 |= b; else bl3 |= b;
  };
  unsigned long long chunk_off = 0;                  // this warp's staging chunk
  uint32_t chunk_left = 0;
  while (true) {
    // refill lanes that finished (one claim per warp)
    const uint32_t need = __ballot_sync(kFull, want);
    if (need) {                              // refill finished lanes from the warp's id pool
      // LT walks are long (≈ 18 nodes on C4): refills are rare and a warp-local id pool only
      // delays the tail (measured 2.61 vs 2.48 ms) — one claim per refill
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&p.ctr->claim, (uint32_t)__popc(need));
      base = __shfl_sync(kFull, base, 0);
      const uint32_t i = base + __popc(need & ((1u << lane) - 1u));
      if (want) {
        want = false;
        active = i < p.count;
        if (active) {
          item = p.item_list ? p.item_list[i] : i;
          id = p.id_base + item;
          v = rr_root_of(p.seed, id, p.n, p.rounds);
          path[lane] = v;
          len = 1;
          bl0 = bl1 = bl2 = bl3 = 0;
          bloom_set(bloom_bit(v));
          if (p.force_giant) {
            p.giant_recs[atomicAdd(&p.ctr->giant_count, 1u)] = GiantRec{item, 0u, 0u, 0u, 0ull};
            active = false;
            want = true;
          }
        }
      }
    }
    if (!__any_sync(kFull, active)) {
      if (!__any_sync(kFull, want)) break;      // claims exhausted and no walk in flight
      continue;
    }
    bool finish = false, overflow = false;
    if (active) {
      const uint32_t a = __ldg(p.row_ptr + v), b = __ldg(p.row_ptr + v + 1);
      const uint32_t d = b - a;
      if (d == 0) {
        finish = true;
      } else {
        const uint32_t j = lt_choose_lane<SCHEME>(p, id, v, a, d);
        ++coins;
        if (j >= d) {
          finish = true;                       // r beyond the total weight: no live in-edge
        } else {
          ++lives;
          const uint32_t u = __ldg(p.src + a + j);
          bool seen = false;
          const uint32_t hb = bloom_bit(u);
          if (bloom_test(hb)) {                 // possible revisit: scan the path
            const uint32_t ls = min(len, (uint32_t)kLtCap);
            for (uint32_t t = 0; t < ls; ++t) seen |= (path[t * 32 + lane] == u);
            for (uint32_t t = kLtCap; t < len; ++t) seen |= (spill[(t - kLtCap) * 32 + lane] == u);
          }
          if (seen) finish = true;
          else if (len == cap) overflow = true;
          else { at(len) = u; ++len; v = u; bloom_set(hb); }
        }
      }
    }
    // finished walks: warp-aggregated staging reservation, then per-lane copy
    const uint32_t fin = __ballot_sync(kFull, finish);
    if (fin) {
      uint32_t incl = finish ? len : 0u;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, off);
        if (lane >= off) incl += y;
      }
      const uint32_t tot = __shfl_sync(kFull, incl, 31);
      if (tot > chunk_left) {                        // reserve a new staging chunk
        const uint32_t want = max(tot, kStageChunk);
        unsigned long long b0 = 0;
        if (lane == 0) b0 = atomicAdd(&p.ctr->stage_tail, (unsigned long long)want);
        chunk_off = __shfl_sync(kFull, b0, 0);
        chunk_left = want;
      }
      const unsigned long long base = chunk_off;
      chunk_off += tot;
      chunk_left -= tot;
      unsigned long long off = 0;
      bool ok = false;
      if (finish) {
        off = base + incl - len;
        ok = off + len <= p.stage_cap;
        if (!ok) {
          p.retry_list[atomicAdd(&p.ctr->retry_count, 1u)] = item;
        } else {
          p.sizes[item] = len;
          p.soff[item] = off;
        }
      }
      // the whole warp copies each finished walk in turn: 32 coalesced elements per step
      // instead of one lane writing its path element by element
      __syncwarp();
      for (uint32_t cm = __ballot_sync(kFull, finish && ok); cm; cm &= cm - 1) {
        const int k = __ffs(cm) - 1;
        const uint32_t lk = __shfl_sync(kFull, len, k);
        const unsigned long long ok_off = __shfl_sync(kFull, off, k);
        for (uint32_t t = lane; t < lk; t += 32)
          p.staging[ok_off + t] = t < (uint32_t)kLtCap ? path[t * 32 + k] : spill[(t - kLtCap) * 32 + k];
      }
      if (finish) {
        active = false;
        want = true;
      }
    }
    if (overflow) {                          // rare: hand the path to the giant kernel
      const unsigned long long off = atomicAdd(&p.ctr->dump_tail, (unsigned long long)len);
      const bool fits = off + len <= p.dump_cap;
      if (fits)
        for (uint32_t t = 0; t < len; ++t) p.dump[off + t] = at(t);
      p.giant_recs[atomicAdd(&p.ctr->giant_count, 1u)] =
          fits ? GiantRec{item, len, len - 1, 0u, off} : GiantRec{item, 0u, 0u, 0u, 0ull};
      active = false;
      want = true;
    }
  }
  unsigned long long c64 = coins, l64 = lives;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    c64 += __shfl_xor_sync(kFull, c64, off);
    l64 += __shfl_xor_sync(kFull, l64, off);
  }
  if (lane == 0) {
    atomicAdd(&p.ctr->coins, c64);
    atomicAdd(&p.ctr->live, l64);
  }
}

// ------------------------------------------------------------------------------------------
// K-GIANT: block-per-RR continuation for sets that outgrew the warp queue (the role of the
// paper's reservoir queue Q_res, Alg. 4/5). Per-block global bitmap (Visited[n])
// and global queue (capacity n, entries kEmpty when unused). No level barriers: the 16 warps
// of the block claim queued nodes from a shared head counter, expand each with the 4-chain
// sweep of the hub path, and append new nodes with an atomic tail; the set is complete when no
// node is pending and no warp is busy (the order of expansion cannot change the set).
// ------------------------------------------------------------------------------------------
#ifndef GIM_SPLIT_GROUPS
#define GIM_SPLIT_GROUPS 2048
#endif
constexpr uint32_t kSplitGroups = GIM_SPLIT_GROUPS;   // hub nodes above this are split across warps
constexpr uint32_t kChunkRing = 128;      // shared ring of published hub chunks
constexpr uint32_t kBusySlot = 0xFFFFFFFEu; // ring slot being written (node ids are < 2^32 - 2)
#ifndef GIM_GIANT_DIV
#define GIM_GIANT_DIV 2
#endif
constexpr uint32_t kGiantClaimDiv = GIM_GIANT_DIV;   // batch = pending / this, clamped to [1, 32]
#ifndef GIM_GIANT_FLAT_MIN
#define GIM_GIANT_FLAT_MIN 8
#endif
constexpr uint32_t kGiantFlatMin = GIM_GIANT_FLAT_MIN;   // batches of >= this many nodes: ballot/redux owner lookup
static_assert(kSplitGroups % kHubGroups == 0, "hub chunks are whole hub steps");

// Relaxed load at gpu scope (not hoisted out of spin loops, not served from a stale L1 line).
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* ptr) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}

#ifdef GIM_GIANT_TRACE
// diagnostic build: per giant set {cycles in K-GIANT, final size, dumped size, claimed batches}
constexpr unsigned int kGTrace = 1u << 16;
__device__ uint4 g_gtrace[kGTrace];
__device__ unsigned int g_gtrace_n;
void giant_trace_dump(cudaStream_t s) {
  unsigned int n = 0;
  cudaStreamSynchronize(s);
  cudaMemcpyFromSymbol(&n, g_gtrace_n, 4);
  n = n < kGTrace ? n : kGTrace;
  std::vector<uint4> v(n);
  if (n) cudaMemcpyFromSymbol(v.data(), g_gtrace, n * sizeof(uint4));
  const unsigned int zero = 0;
  cudaMemcpyToSymbol(g_gtrace_n, &zero, 4);
  std::sort(v.begin(), v.end(), [](const uint4& a, const uint4& b) { return a.x > b.x; });
  unsigned long long sum = 0;
  for (const uint4& e : v) sum += e.x;
  fprintf(stderr, "GTRACE sets=%u mean_us=%.1f\n", n, n ? sum / 1965.0 / n : 0.0);
  for (unsigned int i = 0; i < n && i < 8; ++i)
    fprintf(stderr, "GTRACE top%u us=%.1f size=%u dumped=%u claims=%u\n", i, v[i].x / 1965.0, v[i].y, v[i].z, v[i].w);
}
#endif

// SQ = true (the first pass): queue and visited hash in shared memory (kGQS entries, kGHS slots)
// — every claim, visit and queue read is a shared-memory access, not an L2 round trip; a set
// that outgrows kGQS is aborted and handed to the second pass (SQ = false: per-CTA global
// bitmap Visited[n], and global queue), which resumes it from its original record.
constexpr uint32_t kGQS = 4096;
constexpr uint32_t kGHS = 8192;              // power of two, load <= 1/2
template <int MODEL, int SCHEME, int kGiantThreads, bool SQ>
__global__ void __launch_bounds__(kGiantThreads, 1024 / kGiantThreads) k_rr_giant(RRParams p, uint32_t* bitmaps,
                                                               uint32_t* gqueues, uint64_t bm_words) {
  __shared__ uint32_t s_head, s_tail, s_busy, s_r, s_abort;
  __shared__ uint32_t s_chead, s_cres;           // hub-chunk ring: claimed / reserved counters
  __shared__ uint4 s_ring[kChunkRing];           // {node, a, b, thr}; .x == kEmpty: not yet written
  __shared__ unsigned long long s_off;
  extern __shared__ uint32_t dsm[];              // SQ: queue [kGQS] + hash [kGHS]
  const int lane = threadIdx.x & 31;
  uint32_t* bm = SQ ? nullptr : bitmaps + (uint64_t)blockIdx.x * bm_words;
  uint32_t* Q = SQ ? dsm : gqueues + (uint64_t)blockIdx.x * p.n;     // entries are kEmpty when unused
  uint32_t* Hs = dsm + kGQS;
  const uint32_t cap = SQ ? kGQS : p.n;
  const bool second = !SQ && p.giant_pass2;     // the global pass after the shared one
  const GiantRec* recs = second ? p.giant2_recs : p.giant_recs;
  unsigned int* claim_ctr = second ? &p.ctr->claim_giant2 : &p.ctr->claim_giant;
  const uint32_t giant_count = second ? *(volatile unsigned int*)&p.ctr->giant2_count
                                      : *(volatile unsigned int*)&p.ctr->giant_count;
  const bool never = (SCHEME == W_UNIFORM) && p.thr_uniform == 0;
  uint32_t coins = 0, lives = 0;
  for (uint32_t i = threadIdx.x; i < kChunkRing; i += kGiantThreads) s_ring[i].x = kEmpty;
  if (SQ) {
    for (uint32_t i = threadIdx.x; i < kGQS + kGHS; i += kGiantThreads) dsm[i] = kEmpty;
    if (threadIdx.x == 0) s_abort = 0;
  }
  auto visit = [&](uint32_t u) -> bool {
    if (SQ) {
      uint32_t sl = (u * 0x9E3779B1u) >> 19;     // top 13 bits: kGHS = 2^13 slots
      while (true) {
        const uint32_t old = atomicCAS(&Hs[sl], kEmpty, u);
        if (old == kEmpty) return true;
        if (old == u) return false;
        sl = (sl + 1) & (kGHS - 1u);
      }
    }
    const uint32_t bit = 1u << (u & 31);
    return !(atomicOr(&bm[u >> 5], bit) & bit);
  };
  // read queue entry i, written by another warp possibly still in flight (kEmpty until then)
  auto qread = [&](uint32_t i) -> uint32_t {
    if (SQ) {                                  // atomic reads: the writer is another warp
      uint32_t v = atomicOr(&Q[i], 0u);
      while (v == kEmpty && !atomicOr(&s_abort, 0u)) {
        __nanosleep(32);
        v = atomicOr(&Q[i], 0u);
      }
      return v == kEmpty ? 0u : v;             // aborted: any node (the set is discarded)
    }
    uint32_t v = ld_relaxed_gpu(Q + i);
    while (v == kEmpty) {
      __nanosleep(32);
      v = ld_relaxed_gpu(Q + i);
    }
    return v;
  };
  auto qwrite = [&](uint32_t pos, uint32_t u) {
    if (SQ) {
      if (pos < cap) atomicExch(&Q[pos], u);
      else atomicExch(&s_abort, 1u);           // the set outgrows the shared queue
    } else {
      Q[pos] = u;
    }
  };
  // append this lane's new nodes uu[] to the block queue (warp-collective)
  auto append = [&](const uint32_t (&uu)[4]) {
    const uint32_t cnt = (uu[0] != kEmpty) + (uu[1] != kEmpty) + (uu[2] != kEmpty) + (uu[3] != kEmpty);
    uint32_t tot;
    const uint32_t excl = warp_excl_scan(cnt, lane, tot);
    uint32_t base = 0;
    if (lane == 0 && tot) base = atomicAdd(&s_tail, tot);
    uint32_t pos = __shfl_sync(kFull, base, 0) + excl;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (uu[j] != kEmpty) qwrite(pos++, uu[j]);
  };
  // IC: live in-edges of a claimed batch, resolved together (as in K-RR): cp.async of src[e]
  // into pend[], then one wait, bitmap test-and-set and append per 32 entries
  constexpr uint32_t kGiantWarps = kGiantThreads / 32;
  __shared__ uint32_t s_pend[kGiantWarps][kPend];
  uint32_t* pend = s_pend[threadIdx.x >> 5];
  const uint32_t pend_s = (uint32_t)__cvta_generic_to_shared(pend);
  uint32_t npend = 0;                                  // warp-uniform
  auto flush = [&]() {
    cp_async_wait_all();
    __syncwarp();
    for (uint32_t base = 0; base < npend; base += 32) {
      const uint32_t i = base + lane;
      uint32_t u = 0;
      bool isnew = false;
      if (i < npend) {
        u = pend[i];
        isnew = visit(u);
      }
      const uint32_t has = __ballot_sync(kFull, isnew);
      const uint32_t total = __popc(has);
      uint32_t b0 = 0;
      if (lane == 0 && total) b0 = atomicAdd(&s_tail, total);
      b0 = __shfl_sync(kFull, b0, 0);
      if (isnew) qwrite(b0 + __popc(has & ((1u << lane) - 1u)), u);
    }
    npend = 0;
    __syncwarp();
  };
  auto pend_add = [&](uint32_t g, uint32_t m) -> bool {
    const uint32_t cnt = __popc(m);
    uint32_t total, off;
    if (!__any_sync(kFull, cnt > 1u)) {
      const uint32_t has = __ballot_sync(kFull, cnt != 0u);
      total = __popc(has);
      off = __popc(has & ((1u << lane) - 1u));
    } else {
      off = warp_excl_scan(cnt, lane, total);
    }
    if (npend + total > (uint32_t)kPend) flush();
    uint32_t pos = pend_s + 4u * (npend + off);
    const uint32_t* sp = p.src + (g << 2);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (m & (1u << j)) { cp_async4(pos, sp + j); pos += 4u; }
    npend += total;
    return true;
  };

  while (true) {
    if (threadIdx.x == 0) s_r = atomicAdd(claim_ctr, 1u);
    __syncthreads();
    const uint32_t r = s_r;
    if (r >= giant_count) break;
    const GiantRec rec = recs[r];
#ifdef GIM_GIANT_TRACE
    __shared__ unsigned long long s_t0;
    __shared__ unsigned int s_claims;
    if (threadIdx.x == 0) { s_t0 = clock64(); s_claims = 0; }
#endif
    const uint64_t id = p.id_base + rec.item;
    const uint32_t id_lo = (uint32_t)id, id_hi = (uint32_t)(id >> 32);
    if (rec.qlen == 0) {
      if (threadIdx.x == 0) {
        const uint32_t root = rr_root_of(p.seed, id, p.n, p.rounds);
        Q[0] = root;
        visit(root);
        s_tail = 1;
        s_head = 0;
      }
    } else if (SQ && rec.qlen > kGQS) {        // the dump alone outgrows the shared queue
      if (threadIdx.x == 0) {
        s_abort = 1u;
        s_tail = 0;
        s_head = 0;
      }
    } else {                                   // resume the warp kernel's partial BFS
      for (uint32_t t = threadIdx.x; t < rec.qlen; t += kGiantThreads) {
        const uint32_t u = p.dump[rec.dump_off + t];
        Q[t] = u;
        visit(u);
      }
      if (threadIdx.x == 0) {
        s_tail = rec.qlen;
        s_head = rec.head;
      }
    }
    if (threadIdx.x == 0) {
      s_busy = 0;
      s_chead = 0;
      s_cres = 0;
    }
    __syncthreads();
    // asynchronous expansion: warps claim published hub chunks first, then batches of queued
    // nodes, until nothing is pending and no warp is busy
    while (true) {
      uint32_t f = 0, state = 0, c = 1;          // 1 = nodes Q[f, f+c), 3 = ring entry f, 2 = done
      if (lane == 0) {
        atomicAdd(&s_busy, 1u);
        while (true) {
          if (SQ && atomicOr(&s_abort, 0u)) {          // the set moves to the global pass
            atomicSub(&s_busy, 1u);
            state = 2;
            break;
          }
          const uint32_t ch = *(volatile uint32_t*)&s_chead;
          const uint32_t cr = *(volatile uint32_t*)&s_cres;
          if (ch < cr) {
            if (atomicCAS(&s_chead, ch, ch + 1) == ch) { f = ch; state = 3; break; }
            continue;
          }
          const uint32_t h = *(volatile uint32_t*)&s_head;
          const uint32_t t = min(*(volatile uint32_t*)&s_tail, cap);
          if (h < t) {
            // IC: a batch of up to 32 nodes, smaller while the frontier is narrow so that
            // every warp of the block gets work; LT: one node (its walk is a single path)
            const uint32_t want = (MODEL == MODEL_IC) ? min(32u, max(1u, (t - h) / kGiantClaimDiv)) : 1u;
            if (atomicCAS(&s_head, h, h + want) == h) {
              f = h; c = want; state = 1;
#ifdef GIM_GIANT_TRACE
              atomicAdd(&s_claims, 1u);
#endif
              break;
            }
            continue;
          }
          atomicSub(&s_busy, 1u);
          while (true) {                        // idle: wait for work or global quiescence
            const uint32_t b0 = *(volatile uint32_t*)&s_busy;
            __threadfence_block();
            const uint32_t h2 = *(volatile uint32_t*)&s_head;
            const uint32_t t2 = min(*(volatile uint32_t*)&s_tail, cap);
            const uint32_t ch2 = *(volatile uint32_t*)&s_chead;
            const uint32_t cr2 = *(volatile uint32_t*)&s_cres;
            if (SQ && atomicOr(&s_abort, 0u)) { state = 2; break; }
            if (h2 < t2 || ch2 < cr2) { atomicAdd(&s_busy, 1u); break; }
            if (b0 == 0) { state = 2; break; }
            __nanosleep(64);
          }
          if (state == 2) break;
        }
      }
      state = __shfl_sync(kFull, state, 0);
      if (state == 2) break;
      f = __shfl_sync(kFull, f, 0);
      c = __shfl_sync(kFull, c, 0);
      if (MODEL == MODEL_IC) {
        if (state == 3) {                        // a published chunk [a, b) of a hub node
          uint4 e;
          if (lane == 0) {
            volatile uint4* slot = &s_ring[f % kChunkRing];
            while ((e.x = slot->x) == kEmpty || e.x == kBusySlot) __nanosleep(32);
            __threadfence_block();
            e.y = slot->y; e.z = slot->z; e.w = slot->w;
            __threadfence_block();
            slot->x = kEmpty;                    // consumed
          }
          const uint32_t a = __shfl_sync(kFull, e.y, 0), b = __shfl_sync(kFull, e.z, 0);
          const uint32_t thr = __shfl_sync(kFull, e.w, 0);
          hub_sweep<SCHEME>(p, id_lo, id_hi, a, b, thr, never, lane, lives, pend_add);
        } else {
          // a batch of c queued nodes, expanded like a K-RR batch: lane i holds node Q[f+i]
          uint32_t a = 0, b = 0, thr = 0, ng = 0;
          if ((uint32_t)lane < c) {
            // the appender may still be writing the entry: sleep while empty
            const uint32_t v = qread(f + lane);
            const uint32_t tv = (SCHEME == W_WC) ? __ldg(p.thr_node + v) : 0u;
            a = __ldg(p.row_ptr + v);
            b = __ldg(p.row_ptr + v + 1);
            if (b > a) {
              ng = ((b - 1) >> 2) - (a >> 2) + 1;
              thr = (SCHEME == W_WC) ? tv : node_thr<SCHEME>(p, b - a);
              coins += b - a;
            }
          }
          const uint32_t hub_full = ng & ~(kHubGroups - 1u);
          const uint32_t hubs = __ballot_sync(kFull, hub_full != 0u);
          const uint32_t ngf = ng - hub_full;
          const uint32_t gs = (a >> 2) + hub_full;
          // node of flattened group gi: for small batches (often a few nodes while the frontier
          // is narrow) a shuffle search 0-2 steps deep; for wide ones (dense graphs) the
          // ballot/redux lookup of K-RR over the compacted ranges (one step per window)
          const bool wide = c >= kGiantFlatMin;
          uint32_t total_g;
          const uint32_t E = warp_excl_scan(ngf, lane, total_g);
          const uint32_t P = E + ngf;
          Flat f{};
          if (wide) f = flat_setup(a, b, thr, gs, ngf, lane);
          const uint32_t top = c > 1 ? 1u << (31 - __clz(c - 1)) : 0u;
          for (uint32_t base = 0; base < total_g; base += 32) {
            const uint32_t gi = base + lane;
            uint32_t ak, bk, tk, gk;
            if (wide) {
              const uint32_t k = flat_owner(f, base, lane);
              ak = __shfl_sync(kFull, f.a, k);
              bk = __shfl_sync(kFull, f.b, k);
              tk = __shfl_sync(kFull, f.thr, k);
              gk = __shfl_sync(kFull, f.gofs, k);
            } else {
              uint32_t k = 0;
#pragma unroll
              for (uint32_t step = 16; step >= 1; step >>= 1) {
                if (step <= top) {
                  const uint32_t pv = __shfl_sync(kFull, P, k + step - 1);
                  if (pv <= gi) k += step;
                }
              }
              ak = __shfl_sync(kFull, a, k);
              bk = __shfl_sync(kFull, b, k);
              tk = __shfl_sync(kFull, thr, k);
              gk = __shfl_sync(kFull, gs - E, k);
            }
            const uint32_t g = gk + gi;
            uint32_t m = 0;
            if (gi < total_g && !never) m = ic_live_mask<SCHEME>(p, id_lo, id_hi, 0u, 0u, g, ak, bk, tk);
            if (!__any_sync(kFull, m)) continue;
            lives += __popc(m);
            pend_add(g, m);
          }
          for (uint32_t hm = hubs; hm; hm &= hm - 1) {
            const uint32_t k = __ffs(hm) - 1;
            const uint32_t ak = __shfl_sync(kFull, a, k), bk = __shfl_sync(kFull, b, k);
            const uint32_t tk = __shfl_sync(kFull, thr, k), hk = __shfl_sync(kFull, hub_full, k);
            const uint32_t g_lo = ak >> 2;
            uint32_t kept = hk;                  // whole-step groups this warp sweeps itself
            if (hk > kSplitGroups) {
              // big hub: publish its groups [g_lo + kSplitGroups, g_lo + hk) as chunks of
              // kSplitGroups for idle warps (ring room permitting); sweep the rest here
              const uint32_t nch = (hk - 1) / kSplitGroups;   // chunks after the first
              uint32_t pushed = 0, rbase = 0;
              if (lane == 0) {                   // reserve ring room: outstanding <= kChunkRing
                while (true) {
                  const uint32_t cr = *(volatile uint32_t*)&s_cres;
                  const uint32_t ch = *(volatile uint32_t*)&s_chead;
                  const uint32_t mm = min(nch, kChunkRing - (cr - ch));
                  if (mm == 0) break;
                  if (atomicCAS(&s_cres, cr, cr + mm) == cr) { pushed = mm; rbase = cr; break; }
                }
              }
              pushed = __shfl_sync(kFull, pushed, 0);
              rbase = __shfl_sync(kFull, rbase, 0);
              const uint32_t g_end = g_lo + hk;
              for (uint32_t cc = lane; cc < pushed; cc += 32) {
                const uint32_t cs = g_lo + (cc + 1) * kSplitGroups;
                const uint32_t ce = min(g_end, cs + kSplitGroups);
                uint4* slot = &s_ring[(rbase + cc) % kChunkRing];
                while (atomicCAS(&slot->x, kEmpty, kBusySlot) != kEmpty) __nanosleep(32);
                volatile uint4* vs = slot;
                vs->y = cs << 2;                 // cs > g_lo: past a
                vs->z = min(bk, ce << 2);
                vs->w = tk;
                __threadfence_block();
                vs->x = 0u;                      // publish (any value but kEmpty / kBusySlot)
              }
              kept = kSplitGroups;
              const uint32_t rs = g_lo + (pushed + 1) * kSplitGroups;   // unpushed chunks
              if (rs < g_end)
                hub_sweep<SCHEME>(p, id_lo, id_hi, rs << 2, min(bk, g_end << 2), tk, never, lane, lives,
                                  pend_add);
            }
            hub_sweep_whole<SCHEME>(p, id_lo, id_hi, ak, bk, g_lo, kept / kHubGroups, tk, never, lane, lives,
                                    pend_add);
          }
        }
        flush();
      } else {                                   // LT: one node, one draw
        const uint32_t v = qread(f);
        const uint32_t a = __ldg(p.row_ptr + v), b = __ldg(p.row_ptr + v + 1);
        if (b > a) {
          const uint32_t d = b - a;
          const uint32_t j = lt_choose<SCHEME>(p, id, v, a, d, lane);
          uint32_t uu[4] = {kEmpty, kEmpty, kEmpty, kEmpty};
          if (lane == 0) {
            coins += 1;
            if (j < d) {
              ++lives;
              const uint32_t u = __ldg(p.src + a + j);
              if (visit(u)) uu[0] = u;
            }
          }
          append(uu);
        }
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        atomicSub(&s_busy, 1u);
      }
    }
    __syncthreads();
    if (SQ && s_abort) {                       // hand the set to the global pass, restore state
      const uint32_t used = min(s_tail, cap);
      if (threadIdx.x == 0) p.giant2_recs[atomicAdd(&p.ctr->giant2_count, 1u)] = rec;
      for (uint32_t t = threadIdx.x; t < used; t += kGiantThreads) Q[t] = kEmpty;
      uint4* h4 = reinterpret_cast<uint4*>(Hs);
      for (uint32_t t = threadIdx.x; t < kGHS / 4; t += kGiantThreads) h4[t] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
      for (uint32_t i = threadIdx.x; i < kChunkRing; i += kGiantThreads) s_ring[i].x = kEmpty;
      __syncthreads();
      if (threadIdx.x == 0) s_abort = 0;
      continue;
    }
    const uint32_t size = s_tail;
#ifdef GIM_GIANT_TRACE
    if (threadIdx.x == 0) {
      const unsigned int t = atomicAdd(&g_gtrace_n, 1u);
      if (t < kGTrace) g_gtrace[t] = make_uint4((uint32_t)(clock64() - s_t0), size, rec.qlen, s_claims);
    }
#endif
    if (threadIdx.x == 0) s_off = atomicAdd(&p.ctr->stage_tail, (unsigned long long)size);
    __syncthreads();
    const unsigned long long off = s_off;
    const bool fits = off + size <= p.stage_cap;
    if (!fits && threadIdx.x == 0) p.retry_list[atomicAdd(&p.ctr->retry_count, 1u)] = rec.item;
    if (fits && threadIdx.x == 0) { p.sizes[rec.item] = size; p.soff[rec.item] = off; }
    for (uint32_t t = threadIdx.x; t < size; t += kGiantThreads) {
      const uint32_t u = Q[t];
      if (fits) p.staging[off + t] = u;
      if (!SQ) bm[u >> 5] = 0u;
      Q[t] = kEmpty;
    }
    if (SQ) {
      uint4* h4 = reinterpret_cast<uint4*>(Hs);
      for (uint32_t t = threadIdx.x; t < kGHS / 4; t += kGiantThreads) h4[t] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    }
    __syncthreads();
  }
  unsigned long long c64 = coins, l64 = lives;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    c64 += __shfl_xor_sync(kFull, c64, off);
    l64 += __shfl_xor_sync(kFull, l64, off);
  }
  if (lane == 0) {
    atomicAdd(&p.ctr->coins_giant, c64);
    atomicAdd(&p.ctr->live_giant, l64);
  }
}

// ------------------------------------------------------------------------------------------
// K-STORE: compacting copy staging -> pool in item order + count_total histogram.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_store(const uint32_t* __restrict__ staging,
                                               const uint32_t* __restrict__ sizes,
                                               const uint64_t* __restrict__ soff,
                                               const uint64_t* __restrict__ scan, uint32_t count,
                                               uint64_t pool_base, uint32_t* __restrict__ pool,
                                               uint64_t* __restrict__ offsets_out,
                                               uint32_t* __restrict__ count_total, uint32_t rounds,
                                               uint32_t round0, uint32_t n) {
  // A warp takes 32 consecutive sets (contiguous in the pool) and copies their concatenated
  // members 32 at a time: lane k holds set r0+k (size, staging offset, inclusive end), each
  // element finds its set by a warp binary search. Pool writes are coalesced; tiny sets (C5:
  // 1.5 members on average) no longer leave most lanes idle.
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t r0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32u; r0 < count;
       r0 += nwarps * 32u) {
    const uint32_t nr = min(32u, count - r0);
    const uint64_t base = scan[r0];
    uint32_t sz = 0, roff = 0;
    uint64_t from = 0;
    if ((uint32_t)lane < nr) {
      sz = sizes[r0 + lane];
      from = soff[r0 + lane];
      offsets_out[r0 + lane] = pool_base + scan[r0 + lane];
      // MRIM (R26): element (u, t) of round t = id mod T is stored as the pair id t*n + u
      if (rounds > 1u) roff = ((round0 + r0 + lane) % rounds) * n;
    }
    uint32_t total;
    const uint32_t E = warp_excl_scan(sz, lane, total);
    const uint32_t P = E + sz;
    for (uint32_t i0 = 0; i0 < total; i0 += 32) {       // warp-uniform trip count
      const uint32_t i = i0 + lane;
      const uint32_t k = warp_owner(P, i);
      const uint64_t fk = __shfl_sync(kFull, from, k);
      const uint32_t ek = __shfl_sync(kFull, E, k);
      const uint32_t ok = rounds > 1u ? __shfl_sync(kFull, roff, k) : 0u;
      if (i < total) {
        const uint32_t v = staging[fk + (i - ek)] + ok;
        pool[pool_base + base + i] = v;
#ifndef GIM_AB_NOCOUNT
        atomicAdd(count_total + v, 1u);
#endif
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) offsets_out[count] = pool_base + scan[count];
}

// cnt[v] -= 1 for every element of pool[*e0, *e1) (bounds read on the device: the prefix counts
// of a lookahead round, gim_imm).
__global__ void k_count_sub_range(const uint32_t* __restrict__ pool, const uint64_t* __restrict__ e0p,
                                  const uint64_t* __restrict__ e1p, uint32_t* __restrict__ cnt) {
  const uint64_t e0 = *e0p, e1 = *e1p;
  for (uint64_t t = e0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < e1; t += (uint64_t)gridDim.x * blockDim.x)
    atomicSub(cnt + pool[t], 1u);
}
cudaError_t launch_count_sub_range(const uint32_t* pool, const uint64_t* e0p, const uint64_t* e1p, uint32_t* cnt,
                                   int grid, cudaStream_t s) {
  k_count_sub_range<<<grid, 256, 0, s>>>(pool, e0p, e1p, cnt);
  return cudaGetLastError();
}

// count_total[v] += 1 for every element of pool[e0, e1) (replicated pool: the gathered round).
__global__ void k_count_add(const uint32_t* __restrict__ pool, uint64_t e0, uint64_t e1,
                            uint32_t* __restrict__ count_total) {
  for (uint64_t t = e0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < e1;
       t += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(count_total + pool[t], 1u);
}

// sizes[j] = offsets[j+1] - offsets[j] (j < cnt), zero-padded to `padded` entries.
__global__ void k_sizes_of(const uint64_t* __restrict__ offsets, uint64_t cnt, uint64_t padded,
                           uint32_t* __restrict__ sizes) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < padded; j += (uint64_t)gridDim.x * blockDim.x)
    sizes[j] = j < cnt ? (uint32_t)(offsets[j + 1] - offsets[j]) : 0u;
}

// offsets_out[j] = base + scan[j] for j <= cnt (scan = exclusive prefix of sizes, scan[cnt] = total).
__global__ void k_offsets_of(const uint64_t* __restrict__ scan, uint64_t cnt, uint64_t base,
                             uint64_t* __restrict__ offsets_out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j <= cnt; j += (uint64_t)gridDim.x * blockDim.x)
    offsets_out[j] = base + scan[j];
}

// count_total[v] -= 1 for every member of local sets [s0, s1) (pool truncation).
__global__ void k_count_sub(const uint32_t* __restrict__ pool, uint64_t e0, uint64_t e1,
                            uint32_t* __restrict__ count_total) {
  for (uint64_t t = e0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < e1;
       t += (uint64_t)gridDim.x * blockDim.x)
    atomicSub(count_total + pool[t], 1u);
}

// ------------------------------------------------------------------------------------------
// Host launch wrappers
// ------------------------------------------------------------------------------------------
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): `done` holds one
// bit per device ordinal (contexts on several devices in one process each need their own).
static cudaError_t set_smem_once(std::atomic<uint64_t>& done, const void* fn, int smem) {
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  if (cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) return e;
  done.fetch_or(bit, std::memory_order_acq_rel);
  return cudaSuccess;
}

template <int MODEL, int SCHEME>
static cudaError_t launch_rr_t(const RRParams& p, int grid, cudaStream_t s) {
  const int smem = kRRWarps * kRRSmemPerWarp;
  static std::atomic<uint64_t> attr{0};        // the attribute is per device: one bit each
  if (cudaError_t e = set_smem_once(attr, (const void*)k_rr_warp<MODEL, SCHEME>, smem)) return e;
  k_rr_warp<MODEL, SCHEME><<<grid, kRRWarps * 32, smem, s>>>(p);
  return cudaGetLastError();
}

template <int SCHEME>
static cudaError_t launch_lt_t(const RRParams& p, int grid, cudaStream_t s) {
  const int smem = kLtWarps * kLtCap * 32 * 4;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = set_smem_once(attr, (const void*)k_rr_lt_lane<SCHEME>, smem)) return e;
  k_rr_lt_lane<SCHEME><<<grid, kLtWarps * 32, smem, s>>>(p);
  return cudaGetLastError();
}

static cudaError_t launch_rr_lt(int scheme, const RRParams& p, int grid, cudaStream_t s) {
  if (scheme == W_WC) return launch_lt_t<W_WC>(p, grid, s);
  return launch_lt_t<W_EXPLICIT>(p, grid, s);
}

// resident CTAs per SM of the LT lane kernel (the host sizes the spill buffer from it)
int lt_blocks_per_sm() {
  int bps = 1;
  const int smem = kLtWarps * kLtCap * 32 * 4;
  cudaFuncSetAttribute(k_rr_lt_lane<W_WC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_rr_lt_lane<W_WC>, kLtWarps * 32, smem);
  return bps > 0 ? bps : 1;
}

cudaError_t launch_rr_warp(int model, int scheme, const RRParams& p, int grid, cudaStream_t s) {
  if (model == MODEL_IC) {
    if (scheme == W_WC) return launch_rr_t<MODEL_IC, W_WC>(p, grid, s);
    if (scheme == W_UNIFORM) return launch_rr_t<MODEL_IC, W_UNIFORM>(p, grid, s);
    return launch_rr_t<MODEL_IC, W_EXPLICIT>(p, grid, s);
  }
  return launch_rr_lt(scheme, p, grid, s);
}

template <int MODEL, int SCHEME, int NT, bool SQ>
static cudaError_t giant_attr() {
  if (!SQ) return cudaSuccess;
  static std::atomic<uint64_t> done{0};
  return set_smem_once(done, (const void*)k_rr_giant<MODEL, SCHEME, NT, SQ>, (int)((kGQS + kGHS) * 4));
}

template <int NT, bool SQ>
cudaError_t launch_rr_giant_nt(int model, int scheme, const RRParams& p, int grid, uint32_t* bitmaps,
                               uint32_t* gqueues, uint64_t bm_words, cudaStream_t s) {
  const int smem = SQ ? (int)((kGQS + kGHS) * 4) : 0;
  cudaError_t e = cudaSuccess;
  if (model == MODEL_IC) {
    e = scheme == W_WC ? giant_attr<MODEL_IC, W_WC, NT, SQ>()
        : scheme == W_UNIFORM ? giant_attr<MODEL_IC, W_UNIFORM, NT, SQ>() : giant_attr<MODEL_IC, W_EXPLICIT, NT, SQ>();
  } else {
    e = scheme == W_WC ? giant_attr<MODEL_LT, W_WC, NT, SQ>() : giant_attr<MODEL_LT, W_EXPLICIT, NT, SQ>();
  }
  if (e != cudaSuccess) return e;
  if (model == MODEL_IC) {
    if (scheme == W_WC) k_rr_giant<MODEL_IC, W_WC, NT, SQ><<<grid, NT, smem, s>>>(p, bitmaps, gqueues, bm_words);
    else if (scheme == W_UNIFORM) k_rr_giant<MODEL_IC, W_UNIFORM, NT, SQ><<<grid, NT, smem, s>>>(p, bitmaps, gqueues, bm_words);
    else k_rr_giant<MODEL_IC, W_EXPLICIT, NT, SQ><<<grid, NT, smem, s>>>(p, bitmaps, gqueues, bm_words);
  } else {
    if (scheme == W_WC) k_rr_giant<MODEL_LT, W_WC, NT, SQ><<<grid, NT, smem, s>>>(p, bitmaps, gqueues, bm_words);
    else k_rr_giant<MODEL_LT, W_EXPLICIT, NT, SQ><<<grid, NT, smem, s>>>(p, bitmaps, gqueues, bm_words);
  }
  return cudaGetLastError();
}

// nt = threads per giant set: kGiantThreads (default) or kGiantThreadsNarrow (many giant sets).
// sq: the shared-memory first pass over giant_recs (then call again with sq = false for the
// sets it hands over in giant2_recs); !sq alone: the global pass over giant_recs directly.
cudaError_t launch_rr_giant(int model, int scheme, const RRParams& p, int grid, uint32_t* bitmaps,
                            uint32_t* gqueues, uint64_t bm_words, cudaStream_t s, int nt, bool sq) {
  if (sq) return launch_rr_giant_nt<kGiantThreads, true>(model, scheme, p, grid, bitmaps, gqueues, bm_words, s);
  if (nt == kGiantThreadsNarrow)
    return launch_rr_giant_nt<kGiantThreadsNarrow, false>(model, scheme, p, grid, bitmaps, gqueues, bm_words, s);
  return launch_rr_giant_nt<kGiantThreads, false>(model, scheme, p, grid, bitmaps, gqueues, bm_words, s);
}

cudaError_t launch_store(const uint32_t* staging, const uint32_t* sizes, const uint64_t* soff,
                         const uint64_t* scan, uint32_t count, uint64_t pool_base, uint32_t* pool,
                         uint64_t* offsets_out, uint32_t* count_total, uint32_t rounds, uint32_t round0, uint32_t n, int grid, cudaStream_t s) {
  k_store<<<grid, 256, 0, s>>>(staging, sizes, soff, scan, count, pool_base, pool, offsets_out,
                               count_total, rounds, round0, n);
  return cudaGetLastError();
}

// Philox microbenchmark (diagnostic, gim_microbench_philox): each thread evaluates `per_thread`
// slot groups of one RR id, exactly the per-group work of the IC kernel without memory traffic.
template <int NCH>
__global__ void __launch_bounds__(256) k_philox_bench(RRParams p, uint32_t per_thread, uint32_t* sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (uint32_t i = 0; i < per_thread; i += NCH) {
    uint4 w[NCH];
#pragma unroll
    for (int r = 0; r < NCH; ++r) w[r] = make_uint4(tid, 0u, i + r, 0u);
    philox4x32_10_rk_xn<NCH>(w, p.rk);           // NCH interleaved chains (the hub sweep uses 4)
#pragma unroll
    for (int r = 0; r < NCH; ++r) acc += (min(min(w[r].x, w[r].y), min(w[r].z, w[r].w)) <= 0x1000u);
  }
  if (acc == 0xFFFFFFFFu) sink[0] = acc;
}

cudaError_t launch_philox_bench(uint64_t seed, uint32_t per_thread, uint32_t* sink, int grid, cudaStream_t s,
                                int chains) {
  RRParams p{};
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    p.rk[2 * r] = k0;
    p.rk[2 * r + 1] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  if (chains >= 8) k_philox_bench<8><<<grid, 256, 0, s>>>(p, (per_thread + 7) & ~7u, sink);
  else if (chains >= 4) k_philox_bench<4><<<grid, 256, 0, s>>>(p, (per_thread + 3) & ~3u, sink);
  else k_philox_bench<1><<<grid, 256, 0, s>>>(p, per_thread, sink);
  return cudaGetLastError();
}

cudaError_t launch_count_add(const uint32_t* pool, uint64_t e0, uint64_t e1, uint32_t* count_total, int grid,
                             cudaStream_t s) {
  k_count_add<<<grid, 256, 0, s>>>(pool, e0, e1, count_total);
  return cudaGetLastError();
}
cudaError_t launch_sizes_of(const uint64_t* offsets, uint64_t cnt, uint64_t padded, uint32_t* sizes, int grid,
                            cudaStream_t s) {
  k_sizes_of<<<grid, 256, 0, s>>>(offsets, cnt, padded, sizes);
  return cudaGetLastError();
}
cudaError_t launch_offsets_of(const uint64_t* scan, uint64_t cnt, uint64_t base, uint64_t* offsets_out, int grid,
                              cudaStream_t s) {
  k_offsets_of<<<grid, 256, 0, s>>>(scan, cnt, base, offsets_out);
  return cudaGetLastError();
}
cudaError_t launch_count_sub(const uint32_t* pool, uint64_t e0, uint64_t e1, uint32_t* count_total,
                             int grid, cudaStream_t s) {
  k_count_sub<<<grid, 256, 0, s>>>(pool, e0, e1, count_total);
  return cudaGetLastError();
}

}  // namespace gim

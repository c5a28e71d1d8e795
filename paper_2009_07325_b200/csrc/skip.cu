// skip.cu — IC RR sampling under the geometric-skip RNG contract (reading R31, DESIGN.md;
// option GIM_OPT_SKIP).
//
// Alg. 3 l.18 flips one U(0,1) coin per in-edge. Where every in-edge of a node v
// has the same probability — weighted cascade p = 1/d_in(v) and uniform p — the live
// in-edges of v are i.i.d. Bernoulli(p) slots, so the gaps between live slots are geometric
// (Pr[gap >= g] = (1-p)^g) and can be drawn directly: about 1 + d·p draws per node instead of d
// coins (C3: ~2 draws per visited node against ~365 coins). The contract, restated from
// DESIGN.md R31:
//  * in-edge offsets of v are cut into blocks of kSkipBlock = 1024: block b = [1024b, min(1024(b+1), d));
//  * draw j of block b is word (j & 3) of Philox(seed; id_lo, 2^31 | b, v, j >> 2);
//  * gap = floor(ln((r + 1/2) 2^-32) * inv_v), inv_v = 1 / ln(1 - p); from pos = 1024b, while
//    pos + gap < end: offset pos + gap is live and pos += gap + 1;
//  * p = 1 (WC d = 1, uniform p = 1): every slot live, no draw; uniform p = 0: none.
// ln is evaluated by skip_ln: the same fixed sequence of correctly rounded IEEE-754 operations
// as the oracle's (written separately there), with explicit _rn intrinsics so that nvcc never
// contracts a multiply-add — the device reproduces the host's doubles bit for bit.
//
// Kernels (the same three-tier shape as the per-edge-coin path in rr.cu):
//  * k_skip_lane   lane-per-set for the many small sets (32-node queue per lane in shared
//                  memory); a set that outgrows it is escalated to
//  * k_skip_warp   warp-per-set: the pending frontier (up to 32 nodes) is flattened into
//                  (node, block) items that lanes pull dynamically, one draw per lane per step;
//                  live sources are fetched by cp.async into a pending buffer and resolved per
//                  batch against the shared-memory visited hash (as K-RR); a set that outgrows
//                  the queue is restarted by
//  * k_skip_giant  CTA per set: the warps of the CTA pull batches of queued nodes from a shared
//                  head and expand them with the same batch routine; global queue + visited
//                  bitmap (the giant slots of K-GIANT), restored by member list afterwards.
#include <algorithm>
#include "gim_device.cuh"
#include "gim_internal.h"

namespace gim {

constexpr uint32_t kSkipBlock = 1024;
constexpr int kSkipLaneWarps = 8;
constexpr int kSkipLaneCap = 32;             // lane kernel: members per lane in shared memory
constexpr uint32_t kSkipLaneCap2 = 512;      // lane kernel: most members per lane (shared + global spill)
constexpr uint32_t kSkipLaneMaxBlk = 8;      // lane kernel: blocks per node limit (then escalate)
constexpr uint32_t kSkipTag = 0x80000000u;   // counter word 1 of a skip draw: 2^31 | block

// The series form of ln (reading R31): x = m 2^e, m in [sqrt(1/2), sqrt(2)), ln x = e ln2 +
// 2 atanh(y), y = (m - 1)/(m + 1), atanh(y)/y = sum_{k<=9} y^2k / (2k+1). Only used to build the
// table of centers below (it divides).
__device__ __forceinline__ double skip_ln_series(double x) {
  unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  int e = (int)((bits >> 52) & 0x7FFull) - 1023;
  double m = __longlong_as_double((long long)((bits & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
  if (m > 1.4142135623730951) {
    m = __dmul_rn(m, 0.5);
    e += 1;
  }
  const double y = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0));
  const double y2 = __dmul_rn(y, y);
  double s = 1.0 / 19.0;
  s = __fma_rn(s, y2, 1.0 / 17.0);
  s = __fma_rn(s, y2, 1.0 / 15.0);
  s = __fma_rn(s, y2, 1.0 / 13.0);
  s = __fma_rn(s, y2, 1.0 / 11.0);
  s = __fma_rn(s, y2, 1.0 / 9.0);
  s = __fma_rn(s, y2, 1.0 / 7.0);
  s = __fma_rn(s, y2, 1.0 / 5.0);
  s = __fma_rn(s, y2, 1.0 / 3.0);
  s = __fma_rn(s, y2, 1.0);
  const double de = (double)e;
  return __dadd_rn(__dmul_rn(de, 6.93147180369123816490e-01),
                   __dadd_rn(__dmul_rn(de, 1.90821492927058770002e-10), __dmul_rn(__dmul_rn(2.0, y), s)));
}

// The ln of the contract, division-free: m in [sqrt(1/2), sqrt(2)) as above, nearest center
// c_k = 1 + k/256 (k = floor((m - 1) 256 + 1/2) in [-75, 106]), t = (m - c_k) R_k, R_k = 1/c_k,
// ln m = L_k + ln(1 + t) with L_k = ln c_k (series form, tabulated) and ln(1 + t) by its Taylor
// polynomial of degree 7 (|t| <= 1/512). Center k = 0 is exactly 1 (L = 0, R = 1).
constexpr int kSkipK0 = 75;
__device__ __forceinline__ double skip_ln(double x, const double* tab) {
  unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  int e = (int)((bits >> 52) & 0x7FFull) - 1023;
  double m = __longlong_as_double((long long)((bits & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
  if (m > 1.4142135623730951) {
    m = __dmul_rn(m, 0.5);
    e += 1;
  }
  const int k = (int)floor(__dadd_rn(__dmul_rn(__dsub_rn(m, 1.0), 256.0), 0.5));
  const double c = __dadd_rn(1.0, __dmul_rn((double)k, 0.00390625));
  const double L = tab[k + kSkipK0], R = tab[kSkipTabK + k + kSkipK0];
  const double t = __dmul_rn(__dsub_rn(m, c), R);
  double s = 1.0 / 7.0;
  s = __fma_rn(s, t, -1.0 / 6.0);
  s = __fma_rn(s, t, 1.0 / 5.0);
  s = __fma_rn(s, t, -1.0 / 4.0);
  s = __fma_rn(s, t, 1.0 / 3.0);
  s = __fma_rn(s, t, -1.0 / 2.0);
  s = __fma_rn(s, t, 1.0);
  const double de = (double)e;
  return __dadd_rn(__dmul_rn(de, 6.93147180369123816490e-01),
                   __dadd_rn(__dmul_rn(de, 1.90821492927058770002e-10), __dadd_rn(L, __dmul_rn(t, s))));
}

// inv_v = 1 / ln(1 - p) (< 0), or 0 when every in-edge is live (p = 1): WC q = (d-1)/d,
// uniform q = 1 - p. Tabulated per in-degree by k_skip_inv (WC) — read, not recomputed, per node.
template <int SCHEME>
__device__ __forceinline__ double skip_inv_of(float p_uniform, uint32_t d, const double* tab) {
  double q;
  if (SCHEME == W_WC) {
    if (d <= 1u) return 0.0;
    q = __ddiv_rn((double)(d - 1u), (double)d);
  } else {
    q = __dsub_rn(1.0, (double)p_uniform);
    if (!(q > 0.0)) return 0.0;
  }
  return __ddiv_rn(1.0, skip_ln(q, tab));
}

template <int SCHEME>
__device__ __forceinline__ double skip_inv(const RRParams& p, uint32_t d) {
  return __ldg(p.skip_tab + 2 * kSkipTabK + (SCHEME == W_WC ? d : 0u));
}

__global__ void k_skip_centers(double* tab) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < kSkipTabK) {
    const int k = i - kSkipK0;
    const double c = __dadd_rn(1.0, __dmul_rn((double)k, 0.00390625));
    tab[i] = skip_ln_series(c);
    tab[kSkipTabK + i] = __ddiv_rn(1.0, c);
  }
}

template <int SCHEME>
__global__ void k_skip_inv(double* tab, float p_uniform, uint32_t max_deg) {
  const uint32_t nd = SCHEME == W_WC ? max_deg + 1u : 1u;
  for (uint32_t d = blockIdx.x * blockDim.x + threadIdx.x; d < nd; d += gridDim.x * blockDim.x)
    tab[2 * kSkipTabK + d] = skip_inv_of<SCHEME>(p_uniform, d, tab);
}

cudaError_t launch_skip_tables(int scheme, float p_uniform, uint32_t max_deg, double* tab, cudaStream_t s) {
  k_skip_centers<<<1, 192, 0, s>>>(tab);
  const int grid = (int)std::min<uint64_t>(1024, ((uint64_t)max_deg + 256) / 256);
  if (scheme == W_WC) k_skip_inv<W_WC><<<grid, 256, 0, s>>>(tab, p_uniform, max_deg);
  else k_skip_inv<W_UNIFORM><<<1, 32, 0, s>>>(tab, p_uniform, max_deg);
  return cudaGetLastError();
}

// One lane's position in one block of one node.
struct SkipCur {
  double inv;
  uint4 w;          // words of draw group j >> 2
  uint32_t a;       // global slot of the node's local offset 0
  uint32_t v;
  uint32_t d;
  uint32_t blk;
  uint32_t pos;     // next local offset
  uint32_t end;     // end of the block (local)
  uint32_t j;       // next draw of the block
};

__device__ __forceinline__ void skip_block(SkipCur& c, uint32_t blk) {
  c.blk = blk;
  c.pos = blk * kSkipBlock;
  c.end = min(c.pos + kSkipBlock, c.d);
  c.j = 0;
}

// Next live slot of the block: returns true with e = its global slot, false when the block is
// exhausted (no draw is taken once pos reaches the end, as in the oracle's loop).
__device__ __forceinline__ bool skip_step(SkipCur& c, uint32_t id_lo, const uint32_t* rk,
                                          const double* tab, uint32_t& e, uint32_t& draws) {
  if (c.pos >= c.end) return false;
  if (c.inv != 0.0) {
    const uint32_t jj = c.j & 3u;
    if (jj == 0u) c.w = philox4x32_10_rk(make_uint4(id_lo, kSkipTag | c.blk, c.v, c.j >> 2), rk);
    const uint32_t r = jj == 0u ? c.w.x : jj == 1u ? c.w.y : jj == 2u ? c.w.z : c.w.w;
    ++c.j;
    ++draws;
    const double u = __dmul_rn(__dadd_rn((double)r, 0.5), 0x1p-32);
    const double g = floor(__dmul_rn(skip_ln(u, tab), c.inv));
    if (g >= (double)(c.end - c.pos)) {
      c.pos = c.end;
      return false;
    }
    c.pos += (uint32_t)g;
  }
  e = c.a + c.pos;
  ++c.pos;
  return true;
}

// ------------------------------------------------------------------------------------------
// k_skip_lane: lane-per-set. Each iteration every active lane either starts its next queued node
// (row-pointer loads, per-node inverse) or takes one draw of its current block; a live slot's
// source is loaded and tested against the lane's queue (linear scan, <= 32 entries).
// ------------------------------------------------------------------------------------------
template <int SCHEME>
__global__ void __launch_bounds__(kSkipLaneWarps * 32) k_skip_lane(RRParams p) {
  extern __shared__ uint32_t smem[];
  __shared__ double s_tab[2 * kSkipTabK];        // log centers, read per draw
  for (int i = threadIdx.x; i < 2 * kSkipTabK; i += blockDim.x) s_tab[i] = p.skip_tab[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t* qv = smem + (threadIdx.x >> 5) * (kSkipLaneCap * 32);     // qv[i * 32 + lane]
  // members beyond kSkipLaneCap continue in this warp's global spill region (lane-interleaved,
  // L1-resident while the warp works on it), up to p.lane_cap; beyond that the set escalates
  const uint64_t gwarp = (uint64_t)blockIdx.x * kSkipLaneWarps + (threadIdx.x >> 5);
  uint32_t* lsp = p.lane_spill + gwarp * (uint64_t)((kSkipLaneCap2 - kSkipLaneCap) * 32);
  const uint32_t lcap = min(p.lane_cap, kSkipLaneCap2);
  auto at = [&](uint32_t t) -> uint32_t& {
    return t < (uint32_t)kSkipLaneCap ? qv[t * 32 + lane] : lsp[(t - kSkipLaneCap) * 32 + lane];
  };
  const bool never = (SCHEME == W_UNIFORM) && p.thr_uniform == 0;
  uint32_t item = 0, head = 0, tail = 0, draws = 0, lives = 0;
  uint32_t id_lo = 0;
  uint64_t id = 0;
  SkipCur cur{};
  bool active = false, want = true, on_node = false;
  unsigned long long chunk_off = 0;
  uint32_t chunk_left = 0;
  uint32_t pool_next = 0, pool_end = 0;
  const uint32_t count = p.count;
  while (true) {
    const uint32_t need = __ballot_sync(kFull, want);
    if (need) {
      // refill from a warp-local pool of claimed ids (one atomic per 64 sets)
      const uint32_t nneed = __popc(need), avail = pool_end - pool_next;
      uint32_t base = 0;
      if (avail < nneed) {
        if (lane == 0) base = atomicAdd(&p.ctr->claim_lane, 64u);
        base = __shfl_sync(kFull, base, 0);
      }
      const uint32_t rnk = __popc(need & ((1u << lane) - 1u));
      const uint32_t i = rnk < avail ? pool_next + rnk : base + (rnk - avail);
      if (avail < nneed) {
        pool_next = base + (nneed - avail);
        pool_end = base + 64u;
      } else {
        pool_next += nneed;
      }
      if (want) {
        want = false;
        active = i < count;
        if (active) {
          item = p.item_list ? p.item_list[i] : i;
          id = p.id_base + item;
          id_lo = (uint32_t)id;
          qv[lane] = rr_root_of(p.seed, id, p.n, p.rounds);
          head = 0;
          tail = 1;
          on_node = false;
          if (p.force_giant) {
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
    if (active && !on_node) {
      if (head == tail) {
        finish = true;
      } else {
        const uint32_t v = at(head);
        ++head;
        const uint32_t a = __ldg(p.row_ptr + v), b = __ldg(p.row_ptr + v + 1);
        const uint32_t d = b - a;
        if (d > 0u && !never) {
          // a node whose expected draws (blocks + d p live slots) would serialise this lane
          const bool heavy = (d + kSkipBlock - 1u) / kSkipBlock > kSkipLaneMaxBlk ||
                             (SCHEME == W_UNIFORM && p.p_uniform * (float)d > 24.f);
          if (heavy) {
            escalate = true;
          } else {
            cur.a = a;
            cur.v = v;
            cur.d = d;
            cur.inv = skip_inv<SCHEME>(p, d);
            skip_block(cur, 0u);
            on_node = true;
          }
        }
      }
    } else if (active) {
      uint32_t e;
      if (skip_step(cur, id_lo, p.rk, s_tab, e, draws)) {
        ++lives;
        const uint32_t u = __ldg(p.src + e);
        bool seen = false;
        const uint32_t ts = min(tail, (uint32_t)kSkipLaneCap);
        for (uint32_t t = 0; t < ts; ++t) seen |= (qv[t * 32 + lane] == u);
        for (uint32_t t = kSkipLaneCap; t < tail; ++t) seen |= (lsp[(t - kSkipLaneCap) * 32 + lane] == u);
        if (!seen) {
          if (tail >= lcap) escalate = true;
          else { at(tail) = u; ++tail; }
        }
      } else if ((cur.blk + 1u) * kSkipBlock < cur.d) {
        skip_block(cur, cur.blk + 1u);
      } else {
        on_node = false;
      }
    }
    if (escalate) {
      p.esc_list[atomicAdd(&p.ctr->esc_count, 1u)] = item;
      active = false;
      want = true;
    }
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
          for (uint32_t t = 0; t < tail; ++t) p.staging[off + t] = at(t);
          p.sizes[item] = tail;
          p.soff[item] = off;
        }
        active = false;
        want = true;
      }
    }
  }
  unsigned long long c64 = draws, l64 = lives;
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

__device__ __forceinline__ bool skip_hash_insert(uint32_t* h, uint32_t u) {
  uint32_t s = __umulhi(u * 0x9E3779B1u, (uint32_t)kHSize);
  while (true) {
    const uint32_t old = atomicCAS(&h[s], kEmpty, u);
    if (old == kEmpty) return true;
    if (old == u) return false;
    s = (s + 1 == (uint32_t)kHSize) ? 0u : s + 1;
  }
}

// clear member u from the hash: walk from its home slot to the slot holding it (holes left by
// members cleared before cannot stop the walk: it compares against u, not against empty). The
// lanes of a warp erase concurrently, so every probe is one atomic compare-and-swap.
__device__ __forceinline__ void skip_hash_erase(uint32_t* h, uint32_t u) {
  uint32_t s = __umulhi(u * 0x9E3779B1u, (uint32_t)kHSize);
  while (atomicCAS(&h[s], u, kEmpty) != u) s = (s + 1 == (uint32_t)kHSize) ? 0u : s + 1;
}

__device__ __forceinline__ void cp_async4_skip(uint32_t dst, const uint32_t* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src) : "memory");
}

// Expand one batch of frontier nodes (warp-collective): lane i < nb holds node v. The batch's
// (node, block) items are flattened and pulled by lanes dynamically, one draw per lane per step;
// a live slot's source is copied asynchronously into pend[] (cp.async) and flush() resolves the
// pending sources against the visited structure when pend is full and at the end. Returns false
// when flush() reports a queue overflow.
template <int SCHEME, class Flush>
__device__ __forceinline__ bool skip_expand_batch(const RRParams& p, const double* s_tab, uint32_t id_lo,
                                                  bool has_node, uint32_t v, uint32_t pend_s, uint32_t& npend,
                                                  Flush flush, uint32_t& draws, uint32_t& lives, int lane) {
  const bool never = (SCHEME == W_UNIFORM) && p.thr_uniform == 0;
  uint32_t a = 0, d = 0, nblk = 0;
  double inv = 0.0;
  if (has_node) {
    a = __ldg(p.row_ptr + v);
    d = __ldg(p.row_ptr + v + 1) - a;
    if (d > 0u && !never) {
      nblk = (d + kSkipBlock - 1u) / kSkipBlock;
      inv = skip_inv<SCHEME>(p, d);
    }
  }
  uint32_t incl = nblk;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, off);
    if (lane >= off) incl += y;
  }
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  const uint32_t E = incl - nblk;
  SkipCur cur{};
  bool has_cur = false;
  uint32_t next = 0;                              // items handed out (warp-uniform)
  while (true) {
    const uint32_t need = __ballot_sync(kFull, !has_cur);
    if (need && next < total) {
      const uint32_t idx = next + __popc(need & ((1u << lane) - 1u));
      const uint32_t k = warp_owner(incl, min(idx, total - 1u));
      const uint32_t ak = __shfl_sync(kFull, a, k), dk = __shfl_sync(kFull, d, k);
      const uint32_t vk = __shfl_sync(kFull, v, k), ek = __shfl_sync(kFull, E, k);
      const double ik = __shfl_sync(kFull, inv, k);
      if (!has_cur && idx < total) {
        cur.a = ak;
        cur.d = dk;
        cur.v = vk;
        cur.inv = ik;
        skip_block(cur, idx - ek);
        has_cur = true;
      }
      next = min(total, next + __popc(need));
    }
    if (!__any_sync(kFull, has_cur)) break;
    uint32_t e = 0;
    bool live = false;
    if (has_cur) {
      live = skip_step(cur, id_lo, p.rk, s_tab, e, draws);
      if (!live) has_cur = false;
    }
    const uint32_t lm = __ballot_sync(kFull, live);
    if (lm) {
      const uint32_t nl = __popc(lm);
      if (npend + nl > (uint32_t)kPend && !flush()) return false;
      if (live) cp_async4_skip(pend_s + 4u * (npend + __popc(lm & ((1u << lane) - 1u))), p.src + e);
      npend += nl;
      lives += live;
    }
  }
  return flush();
}

// ------------------------------------------------------------------------------------------
// k_skip_warp: warp per set, queue + visited hash in shared memory (the K-RR layout); items from
// the escalation list (or all items). A set that outgrows the queue continues in the warp's
// global spill tier; one that outgrows that too becomes a giant record (restarted from its
// root by k_skip_giant: the draws are keyed, so the replay is exact).
// ------------------------------------------------------------------------------------------
uint64_t spill_words_per_warp() { return kSpillQ + kSpillH; }

template <int SCHEME>
__global__ void __launch_bounds__(kRRWarps * 32, kRRBlocksPerSM) k_skip_warp(RRParams p) {
  extern __shared__ uint32_t smem[];
  __shared__ double s_tab[2 * kSkipTabK];
  for (int i = threadIdx.x; i < 2 * kSkipTabK; i += blockDim.x) s_tab[i] = p.skip_tab[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t* q = smem + (threadIdx.x >> 5) * (kQMax + kHSize + kPend);
  uint32_t* h = q + kQMax;
  uint32_t* pend = h + kHSize;
  // spill tier: a set that outgrows the shared-memory queue continues in this warp's global
  // queue gq (kSpillQ) + hash gh (kSpillH, L2-resident) instead of being restarted elsewhere —
  // giant sets then run concurrently with (and hidden behind) the small ones
  const uint64_t gwarp = (uint64_t)blockIdx.x * kRRWarps + (threadIdx.x >> 5);
  uint32_t* gq = p.spill + gwarp * (uint64_t)(kSpillQ + kSpillH);
  uint32_t* gh = gq + kSpillQ;
  for (int i = lane; i < kHSize; i += 32) h[i] = kEmpty;
  __syncwarp();
  const uint32_t pend_s = (uint32_t)__cvta_generic_to_shared(pend);
  uint32_t draws = 0, lives = 0;
  const uint32_t count = p.count_ptr ? *p.count_ptr : p.count;
  unsigned long long chunk_off = 0;
  uint32_t chunk_left = 0;
  while (true) {
    uint32_t i = 0;
    if (lane == 0) i = atomicAdd(&p.ctr->claim, 1u);
    i = __shfl_sync(kFull, i, 0);
    if (i >= count) break;
    const uint32_t item = p.item_list ? p.item_list[i] : i;
    if (p.force_giant) {
      if (lane == 0) p.giant_recs[atomicAdd(&p.ctr->giant_count, 1u)] = GiantRec{item, 0u, 0u, 0u, 0ull};
      continue;
    }
    const uint64_t id = p.id_base + item;
    const uint32_t id_lo = (uint32_t)id;
    const uint32_t root = rr_root_of(p.seed, id, p.n, p.rounds);
    if (lane == 0) {
      q[0] = root;
      skip_hash_insert(h, root);
    }
    __syncwarp();
    uint32_t head = 0, tail = 1, npend = 0;
    bool spilled = false;                         // warp-uniform: members live in gq / gh
    auto flush = [&]() -> bool {
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncwarp();
      bool ok = true;
      for (uint32_t base = 0; base < npend; base += 32) {
        const uint32_t t = base + lane;
        uint32_t u = 0;
        bool isnew = false;
        if (t < npend) {
          u = pend[t];
          isnew = spilled ? spill_hash_insert(gh, u) : skip_hash_insert(h, u);
        }
        const uint32_t has = __ballot_sync(kFull, isnew);
        const uint32_t total = __popc(has);
        if (!spilled && tail + total > p.qcap) {
          // move the set to the spill tier: queue copied, members re-inserted in gh
          for (uint32_t i = lane; i < tail; i += 32) {
            const uint32_t x = q[i];
            gq[i] = x;
            spill_hash_insert(gh, x);
          }
          if (isnew) spill_hash_insert(gh, u);
          spilled = true;
          __syncwarp();
        }
        if (spilled && tail + total > p.spill_cap) { ok = false; break; }
        if (isnew) (spilled ? gq : q)[tail + __popc(has & ((1u << lane) - 1u))] = u;
        tail += total;
      }
      npend = 0;
      __syncwarp();
      return ok;
    };
    bool overflow = false;
    while (head < tail) {
      const uint32_t nb = min(tail - head, 32u);
      const uint32_t v = (uint32_t)lane < nb ? (spilled ? gq[head + lane] : q[head + lane]) : 0u;
      head += nb;
      if (!skip_expand_batch<SCHEME>(p, s_tab, id_lo, (uint32_t)lane < nb, v, pend_s, npend, flush, draws, lives,
                                     lane)) {
        overflow = true;
        break;
      }
    }
    if (spilled || overflow) {                    // the smem hash holds a stale prefix: wipe it
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      uint4* h4 = reinterpret_cast<uint4*>(h);
      for (int t = lane; t < kHSize / 4; t += 32) h4[t] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
      __syncwarp();
    }
    if (overflow) {                               // beyond the spill tier: restart as a giant set
      if (lane == 0) p.giant_recs[atomicAdd(&p.ctr->giant_count, 1u)] = GiantRec{item, 0u, 0u, 0u, 0ull};
      uint4* gh4 = reinterpret_cast<uint4*>(gh);  // gh may hold nodes that are not queued
      for (uint32_t t = lane; t < kSpillH / 4; t += 32) gh4[t] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
      __syncwarp();
      continue;
    }
    if (tail > chunk_left) {
      const uint32_t want = max(tail, kStageChunk);
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(&p.ctr->stage_tail, (unsigned long long)want);
      chunk_off = __shfl_sync(kFull, base, 0);
      chunk_left = want;
    }
    const unsigned long long off = chunk_off;
    chunk_off += tail;
    chunk_left -= tail;
    const bool fits = off + tail <= p.stage_cap;
    if (!fits && lane == 0) p.retry_list[atomicAdd(&p.ctr->retry_count, 1u)] = item;
    if (fits && lane == 0) { p.sizes[item] = tail; p.soff[item] = off; }
    for (uint32_t t = lane; t < tail; t += 32) {
      const uint32_t u = spilled ? gq[t] : q[t];
      if (fits) p.staging[off + t] = u;
      if (spilled) spill_hash_erase(gh, u);
      else skip_hash_erase(h, u);                 // O(|RR|) clear instead of the whole table
    }
    __syncwarp();
  }
  unsigned long long c64 = draws, l64 = lives;
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

__device__ __forceinline__ uint32_t ld_relaxed_gpu_skip(const uint32_t* ptr) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}

// ------------------------------------------------------------------------------------------
// k_skip_giant: CTA per giant set (kSkipGiantWarps warps), giant slot blockIdx.x: a global queue
// Q of n entries (kEmpty when unused) and an n-bit visited bitmap (Visited[n]; 0 when
// unused), both restored by member list after the set. No level barriers: warps claim batches
// of queued nodes from a shared head (fewer than 32 while the frontier is narrow, so that every
// warp gets work), expand them with skip_expand_batch and append with an atomic tail; the set is
// complete when nothing is pending and no warp holds a batch (the order cannot change the set).
// ------------------------------------------------------------------------------------------
constexpr int kSkipGiantWarps = 8;
template <int SCHEME>
__global__ void __launch_bounds__(kSkipGiantWarps * 32) k_skip_giant(RRParams p, uint32_t* bitmaps,
                                                                     uint32_t* gqueues, uint64_t bm_words) {
  __shared__ uint32_t s_head, s_tail, s_busy, s_r;
  __shared__ unsigned long long s_off;
  __shared__ uint32_t s_pend[kSkipGiantWarps][kPend];
  __shared__ double s_tab[2 * kSkipTabK];
  for (int i = threadIdx.x; i < 2 * kSkipTabK; i += blockDim.x) s_tab[i] = p.skip_tab[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t* Q = gqueues + (uint64_t)blockIdx.x * p.n;
  uint32_t* bm = bitmaps + (uint64_t)blockIdx.x * bm_words;
  uint32_t* pend = s_pend[threadIdx.x >> 5];
  const uint32_t pend_s = (uint32_t)__cvta_generic_to_shared(pend);
  const uint32_t count = *(volatile unsigned int*)&p.ctr->giant_count;
  uint32_t draws = 0, lives = 0;
  auto visit = [bm](uint32_t u) {
    const uint32_t bit = 1u << (u & 31);
    return !(atomicOr(&bm[u >> 5], bit) & bit);
  };
  while (true) {
    if (threadIdx.x == 0) s_r = atomicAdd(&p.ctr->claim_giant, 1u);
    __syncthreads();
    const uint32_t r = s_r;
    if (r >= count) break;
    const uint32_t item = p.giant_recs[r].item;
    const uint64_t id = p.id_base + item;
    const uint32_t id_lo = (uint32_t)id;
    if (threadIdx.x == 0) {
      const uint32_t root = rr_root_of(p.seed, id, p.n, p.rounds);
      Q[0] = root;
      visit(root);
      s_head = 0;
      s_tail = 1;
      s_busy = 0;
    }
    __syncthreads();
    uint32_t npend = 0;
    auto flush = [&]() -> bool {
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncwarp();
      for (uint32_t base = 0; base < npend; base += 32) {
        const uint32_t t = base + lane;
        uint32_t u = 0;
        bool isnew = false;
        if (t < npend) {
          u = pend[t];
          isnew = visit(u);
        }
        const uint32_t has = __ballot_sync(kFull, isnew);
        uint32_t b0 = 0;
        if (lane == 0 && has) b0 = atomicAdd(&s_tail, (uint32_t)__popc(has));
        b0 = __shfl_sync(kFull, b0, 0);
        if (isnew) Q[b0 + __popc(has & ((1u << lane) - 1u))] = u;
      }
      npend = 0;
      __syncwarp();
      return true;
    };
    while (true) {
      uint32_t f = 0, c = 0, state = 0;            // 1: nodes Q[f, f + c); 2: done
      if (lane == 0) {
        atomicAdd(&s_busy, 1u);
        while (true) {
          const uint32_t hh = *(volatile uint32_t*)&s_head;
          const uint32_t tt = *(volatile uint32_t*)&s_tail;
          if (hh < tt) {
            const uint32_t want = min(32u, max(1u, (tt - hh) / 2u));
            if (atomicCAS(&s_head, hh, hh + want) == hh) { f = hh; c = want; state = 1; break; }
            continue;
          }
          atomicSub(&s_busy, 1u);
          while (true) {                            // idle: new work or quiescence
            const uint32_t b0 = *(volatile uint32_t*)&s_busy;
            __threadfence_block();
            const uint32_t h2 = *(volatile uint32_t*)&s_head;
            const uint32_t t2 = *(volatile uint32_t*)&s_tail;
            if (h2 < t2) { atomicAdd(&s_busy, 1u); break; }
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
      uint32_t v = 0;
      if ((uint32_t)lane < c) {                     // the appender may still be writing the entry
        v = ld_relaxed_gpu_skip(Q + f + lane);
        while (v == kEmpty) {
          __nanosleep(32);
          v = ld_relaxed_gpu_skip(Q + f + lane);
        }
      }
      skip_expand_batch<SCHEME>(p, s_tab, id_lo, (uint32_t)lane < c, v, pend_s, npend, flush, draws, lives, lane);
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        atomicSub(&s_busy, 1u);
      }
    }
    __syncthreads();
    const uint32_t size = s_tail;
    if (threadIdx.x == 0) s_off = atomicAdd(&p.ctr->stage_tail, (unsigned long long)size);
    __syncthreads();
    const unsigned long long off = s_off;
    const bool fits = off + size <= p.stage_cap;
    if (!fits && threadIdx.x == 0) p.retry_list[atomicAdd(&p.ctr->retry_count, 1u)] = item;
    if (fits && threadIdx.x == 0) { p.sizes[item] = size; p.soff[item] = off; }
    for (uint32_t t = threadIdx.x; t < size; t += kSkipGiantWarps * 32) {
      const uint32_t u = Q[t];
      if (fits) p.staging[off + t] = u;
      bm[u >> 5] = 0u;                              // every set bit of the word is a member
      Q[t] = kEmpty;
    }
    __syncthreads();
  }
  unsigned long long c64 = draws, l64 = lives;
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
// launch wrappers
// ------------------------------------------------------------------------------------------
static cudaError_t smem_attr(const void* fn, int smem) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

cudaError_t launch_skip_lane(int scheme, const RRParams& p, int grid, cudaStream_t s) {
  const int smem = kSkipLaneWarps * kSkipLaneCap * 32 * 4;
  if (scheme == W_WC) k_skip_lane<W_WC><<<grid, kSkipLaneWarps * 32, smem, s>>>(p);
  else k_skip_lane<W_UNIFORM><<<grid, kSkipLaneWarps * 32, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_skip_warp(int scheme, const RRParams& p, int grid, cudaStream_t s) {
  const int smem = kRRWarps * kRRSmemPerWarp;
  cudaError_t e = scheme == W_WC ? smem_attr((const void*)k_skip_warp<W_WC>, smem)
                                 : smem_attr((const void*)k_skip_warp<W_UNIFORM>, smem);
  if (e != cudaSuccess) return e;
  if (scheme == W_WC) k_skip_warp<W_WC><<<grid, kRRWarps * 32, smem, s>>>(p);
  else k_skip_warp<W_UNIFORM><<<grid, kRRWarps * 32, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_skip_giant(int scheme, const RRParams& p, int grid, uint32_t* bitmaps, uint32_t* gqueues,
                              uint64_t bm_words, cudaStream_t s) {
  if (scheme == W_WC) k_skip_giant<W_WC><<<grid, kSkipGiantWarps * 32, 0, s>>>(p, bitmaps, gqueues, bm_words);
  else k_skip_giant<W_UNIFORM><<<grid, kSkipGiantWarps * 32, 0, s>>>(p, bitmaps, gqueues, bm_words);
  return cudaGetLastError();
}

uint64_t skip_lane_spill_words(int grid) { return (uint64_t)grid * kSkipLaneWarps * 32 * (kSkipLaneCap2 - kSkipLaneCap); }

int skip_lane_blocks_per_sm() {
  int bps = 1;
  const int smem = kSkipLaneWarps * kSkipLaneCap * 32 * 4;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_skip_lane<W_WC>, kSkipLaneWarps * 32, smem);
  return bps > 0 ? bps : 1;
}

}  // namespace gim

// select.cu — NodeSelection kernels: exclusive scan, inverted index (K-INV), argmax (K-ARGMAX),
// covered-set retirement (K-COVER).
//
// What they compute (Alg. 1 l.6-10; §3.8; Alg. 7):
// u_j = argmax_{v not in S} count[v] by a max-reduction over Occur, ties -> lowest
// id (reading R10); then every uncovered RR set containing u_j is flagged covered and
// count[w] -= 1 for each member w (Alg. 7 l.11-16; reading R11). B200 design (DESIGN.md
// "NodeSelection"): Alg. 7 scans every RR set per step; here an inverted node -> RR index
// (histogram = count_total, exclusive scan, scatter) gives the sets containing u_j directly,
// so a selection touches each pool element at most once for decrements. The argmax is one
// streaming pass with a packed 64-bit key (count << 32 | ~v) reduced by warp shuffles and one
// atomicMax per CTA; the previous pick is retired inside the same pass (count = sentinel).
#include <atomic>
#include <algorithm>
#include <cooperative_groups.h>

#include "gim_device.cuh"
#include "gim_internal.h"

namespace gim {

constexpr int kScanThreads = 1024;
constexpr int kScanPerThread = 4;
constexpr int kScanTile = kScanThreads * kScanPerThread;

__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t x, int lane) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint64_t y = __shfl_up_sync(kFull, x, off);
    if (lane >= off) x += y;
  }
  return x;
}

// Block-wide exclusive scan of one value per thread (1024 threads); returns the exclusive
// prefix and writes the block total to *total.
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t x, uint64_t* total) {
  __shared__ uint64_t s_w[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t incl = warp_incl_scan_u64(x, lane);
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint64_t w = s_w[lane];
    const uint64_t wi = warp_incl_scan_u64(w, lane);
    s_w[lane] = wi - w;
    if (lane == 31) s_w[31] = wi - w, *total = wi;   // keep exclusive; publish total via arg
  }
  __syncthreads();
  const uint64_t r = s_w[warp] + incl - x;
  __syncthreads();
  return r;
}

// Phase 1: per-tile sums.
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(const uint32_t* __restrict__ in,
                                                            uint64_t count, uint64_t* __restrict__ tile_sums) {
  __shared__ uint64_t s_total;
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanPerThread;
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanPerThread; ++j)
    if (base + j < count) s += in[base + j];
  block_excl_scan(s, &s_total);
  __syncthreads();
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = s_total;
}

// Index segment histogram + scan in one pass pair (no separate delta array): the segment's count
// of node v is cnt[v] - snap[v] (count_total minus its value at the previous segment); phase 1
// sums it per tile, phase 3 writes the exclusive (scatter: list starts) or inclusive (sorted
// segment: list ends) prefix and sets snap := cnt.
__global__ void __launch_bounds__(kScanThreads) k_seg_sums(const uint32_t* __restrict__ cnt,
                                                           const uint32_t* __restrict__ snap, uint64_t count,
                                                           uint64_t* __restrict__ tile_sums) {
  __shared__ uint64_t s_total;
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanPerThread;
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanPerThread; ++j)
    if (base + j < count) s += cnt[base + j] - snap[base + j];
  block_excl_scan(s, &s_total);
  __syncthreads();
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = s_total;
}
__global__ void __launch_bounds__(kScanThreads) k_seg_apply(const uint32_t* __restrict__ cnt,
                                                            uint32_t* __restrict__ snap, uint64_t count,
                                                            const uint64_t* __restrict__ tile_sums,
                                                            const uint64_t* __restrict__ grand_total,
                                                            uint32_t* __restrict__ out, int inclusive) {
  __shared__ uint64_t s_total;
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanPerThread;
  uint32_t v[kScanPerThread], c[kScanPerThread];
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanPerThread; ++j) {
    c[j] = (base + j < count) ? cnt[base + j] : 0u;
    v[j] = (base + j < count) ? c[j] - snap[base + j] : 0u;
    s += v[j];
  }
  uint64_t ex = block_excl_scan(s, &s_total) + tile_sums[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanPerThread; ++j) {
    if (base + j < count) {
      out[base + j] = (uint32_t)(inclusive ? ex + v[j] : ex);
      snap[base + j] = c[j];
    }
    ex += v[j];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[count] = (uint32_t)*grand_total;
}

// Phase 2: exclusive scan of the tile sums by one CTA (loops over chunks of 1024).
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(uint64_t* __restrict__ tile_sums, uint64_t ntiles,
                                                             uint64_t* __restrict__ grand_total) {
  __shared__ uint64_t s_total;
  uint64_t carry = 0;
  for (uint64_t b = 0; b < ntiles; b += kScanThreads) {
    const uint64_t i = b + threadIdx.x;
    const uint64_t x = (i < ntiles) ? tile_sums[i] : 0;
    const uint64_t ex = block_excl_scan(x, &s_total);
    __syncthreads();
    if (i < ntiles) tile_sums[i] = carry + ex;
    carry += s_total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *grand_total = carry;
}

// Phase 3: out[i] = exclusive prefix (uint64); out[count] = total.
template <class OutT>
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const uint32_t* __restrict__ in, uint64_t count,
                                                             const uint64_t* __restrict__ tile_sums,
                                                             const uint64_t* __restrict__ grand_total,
                                                             OutT* __restrict__ out) {
  __shared__ uint64_t s_total;
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanPerThread;
  uint32_t v[kScanPerThread];
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanPerThread; ++j) {
    v[j] = (base + j < count) ? in[base + j] : 0u;
    s += v[j];
  }
  uint64_t ex = block_excl_scan(s, &s_total) + tile_sums[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanPerThread; ++j) {
    if (base + j < count) out[base + j] = (OutT)ex;
    ex += v[j];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[count] = (OutT)*grand_total;
}

// Warp-level helpers: exclusive scan of one value per lane, and the lane (0..31) whose
// half-open range [E_k, E_k + len_k) contains i, given inclusive prefixes P_k held per lane.
__device__ __forceinline__ uint32_t warp_excl_scan_u32(uint32_t x, int lane, uint32_t& total) {
  uint32_t incl = x;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, off);
    if (lane >= off) incl += y;
  }
  total = __shfl_sync(kFull, incl, 31);
  return incl - x;
}

// ------------------------------------------------------------------------------------------
// K-INV scatter: inv[inv_off[v] + cursor[v]++] = local set index r, for every member v of r.
// A warp takes 32 consecutive sets (contiguous in the pool) and sweeps their members 32 at a
// time; the owning set of a member is found with a 5-step shuffle search. Only members in the
// node range [vlo, vlo + vspan) are scattered: when the cursor array is larger than the L2
// (C5: 166 MB), the host runs one pass per node range so the cursor atomics and the inv writes
// of a pass stay L2-resident instead of each being a random DRAM read-modify-write.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_inv_scatter(const uint64_t* __restrict__ offsets,
                                                     const uint32_t* __restrict__ pool, uint32_t set0,
                                                     uint32_t nsets_end,
                                                     uint32_t* __restrict__ end,
                                                     uint32_t* __restrict__ inv, uint32_t vlo, uint32_t vspan) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  const uint32_t nsets = nsets_end;
  for (uint32_t r0 = set0 + (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32u; r0 < nsets;
       r0 += nwarps * 32u) {
    const uint32_t nr = min(32u, nsets - r0);
    const uint64_t base = offsets[r0];
    const uint32_t hi_rel = (uint32_t)(offsets[r0 + nr] - base);
    // inclusive end (relative) of the set held by this lane
    const uint32_t P = (lane < nr) ? (uint32_t)(offsets[r0 + lane + 1] - base) : hi_rel;
    for (uint32_t i0 = 0; i0 < hi_rel; i0 += 32) {      // warp-uniform trip count
      const uint32_t i = i0 + lane;
      const uint32_t k = warp_owner(P, i);
      if (i < hi_rel) {
        const uint32_t v = pool[base + i];
        if (v - vlo < vspan) inv[atomicAdd(end + v, 1u)] = r0 + k;   // end[v]: list start, advanced to its end
      }
    }
  }
}


// ------------------------------------------------------------------------------------------
// K-ARGMAX: keys[j] = max over v of (selected ? 0 : count[v] << 32 | ~v). Applies the
// all-reduced decrements of the previous step first (P > 1) and retires the previous pick.
// Streams count as uint4 (4 nodes per load) with 4 independent loads in flight per thread.
// ------------------------------------------------------------------------------------------
// Programmatic dependent launch (the greedy steps' argmax/cover chain): a kernel lets the next
// one in the stream launch at once (its CTAs become resident and wait) and itself waits for the
// previous kernel's results before touching them, so the 2k dependent launches of a selection
// do not pay a launch gap each. Both are no-ops without a programmatic predecessor/successor.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// excl = 0x80000000 in MRIM mode: pairs of a round that already has its k seeds carry the high
// bit (set by k_cover) and are skipped like selected ones; 0 otherwise.
__device__ __forceinline__ void argmax_one(uint32_t c, uint32_t v, unsigned long long& best, uint32_t excl) {
  const unsigned long long key = (c == kSent || (c & excl)) ? 0ull : (((unsigned long long)c << 32) | (unsigned long long)(~v));
  best = key > best ? key : best;
}

__device__ __forceinline__ void argmax_step(uint32_t* __restrict__ cnt, int32_t* __restrict__ dec,
                                            uint32_t n, unsigned long long* __restrict__ keys, int j,
                                            const uint32_t* __restrict__ tau_p1, uint32_t excl,
                                            uint32_t id_base = 0, const SelCtl* ctl = nullptr) {
  // bounded greedy stopped (SelCtl): no pick from here on, keys[j] stays 0. Large n: test first
  // and skip the scan; small n: the flag load overlaps the (cheap) scan and only the final
  // atomicMax is skipped — no serial load at the head of every greedy step
  const bool test_first = ctl != nullptr && n >= (1u << 20);
  if (test_first && *(volatile const uint32_t*)&ctl->stop) return;
  const uint32_t stopped = (ctl != nullptr && !test_first) ? *(volatile const uint32_t*)&ctl->stop : 0u;
  // candidate mode: the candidate argmax already found a count >= tau_p1, which no node outside
  // the candidate list can reach (their counts started below it and only decrease)
  if (tau_p1 != nullptr && (uint32_t)(keys[j] >> 32) >= *tau_p1 && keys[j] != 0ull) return;
  __shared__ unsigned long long s_best[32];   // up to 1024 threads per CTA
  unsigned long long best = 0;
  const uint32_t n4 = n >> 2;
  const uint32_t stride = gridDim.x * blockDim.x;
  uint4* c4 = reinterpret_cast<uint4*>(cnt);
  int4* d4 = reinterpret_cast<int4*>(dec);
  for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += 4 * stride) {
    uint4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = i0 + u * stride;
      x[u] = (i < n4) ? c4[i] : make_uint4(kSent, kSent, kSent, kSent);
    }
    if (dec != nullptr) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = i0 + u * stride;
        if (i < n4) {
          const int4 d = d4[i];
          if (d.x | d.y | d.z | d.w) {
            if (x[u].x != kSent) x[u].x -= (uint32_t)d.x;
            if (x[u].y != kSent) x[u].y -= (uint32_t)d.y;
            if (x[u].z != kSent) x[u].z -= (uint32_t)d.z;
            if (x[u].w != kSent) x[u].w -= (uint32_t)d.w;
            c4[i] = x[u];
            d4[i] = make_int4(0, 0, 0, 0);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t v = id_base + ((i0 + u * stride) << 2);
      argmax_one(x[u].x, v, best, excl);
      argmax_one(x[u].y, v + 1, best, excl);
      argmax_one(x[u].z, v + 2, best, excl);
      argmax_one(x[u].w, v + 3, best, excl);
    }
  }
  // tail (n % 4 nodes)
  for (uint32_t v = (n4 << 2) + blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    uint32_t c = cnt[v];
    if (dec != nullptr && c != kSent && dec[v]) { c -= (uint32_t)dec[v]; dec[v] = 0; cnt[v] = c; }
    argmax_one(c, id_base + v, best, excl);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(kFull, best, off);
    best = o > best ? o : best;
  }
  if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = (threadIdx.x < (blockDim.x >> 5)) ? s_best[threadIdx.x] : 0ull;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(kFull, best, off);
      best = o > best ? o : best;
    }
    if (threadIdx.x == 0 && best && !stopped) atomicMax(keys + j, best);
  }
}

__global__ void __launch_bounds__(256) k_argmax(uint32_t* __restrict__ cnt, int32_t* __restrict__ dec,
                                                uint32_t n, unsigned long long* __restrict__ keys, int j,
                                                const uint32_t* __restrict__ tau_p1, uint32_t excl,
                                                uint32_t id_base, const SelCtl* ctl) {
  pdl_wait();
  pdl_trigger();
  argmax_step(cnt, dec, n, keys, j, tau_p1, excl, id_base, ctl);
}

// Node-sharded selection (include/gim.h gim_set_reducescatter): this rank's best key of step j
// goes to its slot of the exchange buffer (2 int32 per rank, the other slots zero, so a SUM
// all-reduce gathers them); after the exchange the largest key is the global pick, which the
// owner of its shard retires.
__global__ void k_rs_pack(const unsigned long long* __restrict__ local_keys, int j, uint32_t rank, uint32_t world,
                          unsigned long long* __restrict__ kx) {
  for (uint32_t r = threadIdx.x; r < world; r += blockDim.x) kx[r] = (r == rank) ? local_keys[j] : 0ull;
}
__global__ void k_rs_pick(const unsigned long long* __restrict__ kx, uint32_t world, unsigned long long* keys, int j,
                          uint32_t* __restrict__ gshard, uint32_t id_base, uint32_t ns_valid) {
  if (threadIdx.x == 0) {
    unsigned long long best = 0;
    for (uint32_t r = 0; r < world; ++r) best = kx[r] > best ? kx[r] : best;
    keys[j] = best;
    const uint32_t u = ~(uint32_t)best;
    if (best && u - id_base < ns_valid) gshard[u - id_base] = kSent;
  }
}

// ------------------------------------------------------------------------------------------
// Candidate list for the argmax (P = 1): tau_p1 = 2^B - 1 for the smallest B such that at most
// kMaxCand nodes have count >= 2^B - 1 (log2-bucket histogram), and cand = those nodes.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_cnt_hist(const uint32_t* __restrict__ cnt, uint32_t n,
                                                  unsigned int* __restrict__ hist) {
  // bucket floor(log2(c + 1)), 0..32. Streams cnt as uint4 (4 loads in flight per thread); the
  // common small buckets 0..7 are counted in registers (a shared atomic per count serialises
  // when nearly every node falls in the same bucket), the rest with shared atomics.
  __shared__ unsigned int h[33];
  if (threadIdx.x < 33) h[threadIdx.x] = 0;
  __syncthreads();
  uint32_t r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto add = [&](uint32_t c) {
    const uint32_t b = 31 - __clz(c + 1u);
    if (b < 8) {
#pragma unroll
      for (uint32_t j = 0; j < 8; ++j) r[j] += (b == j);
    } else {
      atomicAdd(&h[b], 1u);
    }
  };
  const uint32_t n4 = n >> 2;
  const uint4* c4 = reinterpret_cast<const uint4*>(cnt);
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += 4 * stride) {
    uint4 w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = i0 + u * stride;
      w[u] = (i < n4) ? __ldcs(c4 + i) : make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i0 + u * stride >= n4) continue;             // past the end
      add(w[u].x); add(w[u].y); add(w[u].z); add(w[u].w);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3u)) add(cnt[(n4 << 2) + threadIdx.x]);
#pragma unroll
  for (uint32_t j = 0; j < 8; ++j) {
    const uint32_t t = __reduce_add_sync(kFull, r[j]);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(&h[j], t);
  }
  __syncthreads();
  if (threadIdx.x < 33 && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

__global__ void k_pick_tau(const unsigned int* __restrict__ hist, uint32_t kmax, uint32_t* tau_p1,
                           unsigned int* ncand) {
  unsigned long long cum = 0;
  uint32_t B = 33;
  for (int b = 32; b >= 0; --b) {
    cum += hist[b];
    if (cum > kmax) break;
    B = (uint32_t)b;
  }
  // nodes in buckets >= B are candidates: count >= 2^B - 1 (B = 0: every node)
  *tau_p1 = (B >= 32) ? 0xFFFFFFFFu : ((1u << B) - 1u);
  *ncand = 0;
}

__global__ void __launch_bounds__(256) k_cand_compact(const uint32_t* __restrict__ cnt, uint32_t n,
                                                      const uint32_t* __restrict__ tau_p1,
                                                      uint32_t* __restrict__ cand, unsigned int* ncand) {
  const uint32_t t = *tau_p1;
  if (t == 0xFFFFFFFFu) return;
  const int lane = threadIdx.x & 31;
  const uint32_t n4 = (n + 3) >> 2;                    // uint4 groups; the ragged tail is masked
  const uint4* c4 = reinterpret_cast<const uint4*>(cnt);
  const uint32_t stride = gridDim.x * blockDim.x;
  // warp-uniform trip count: every lane of a warp runs the same iterations (ballots below)
  for (uint32_t b0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); b0 < n4; b0 += 4 * stride) {
    uint4 w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = b0 + u * stride + lane;
      if (i + 1 < n4 || (i + 1 == n4 && (n & 3u) == 0)) w[u] = __ldcs(c4 + i);
      else if (i + 1 == n4) {                          // last group, partly past n
        const uint32_t v = i << 2;
        w[u] = make_uint4(cnt[v], v + 1 < n ? cnt[v + 1] : 0u, v + 2 < n ? cnt[v + 2] : 0u, 0u);
      } else {
        w[u] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = b0 + u * stride + lane;
      const uint32_t v = i << 2;
      const uint32_t m = (uint32_t)(w[u].x >= t && v < n) | ((uint32_t)(w[u].y >= t && v + 1 < n) << 1) |
                         ((uint32_t)(w[u].z >= t && v + 2 < n) << 2) | ((uint32_t)(w[u].w >= t && v + 3 < n) << 3);
      if (!__any_sync(kFull, m)) continue;             // usual: no candidate in these 128 nodes
      uint32_t total;
      const uint32_t off = warp_excl_scan_u32(__popc(m), lane, total);
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(ncand, total);
      uint32_t pos = __shfl_sync(kFull, base, 0) + off;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (m & (1u << j)) cand[pos++] = v + j;
    }
  }
}

__global__ void __launch_bounds__(256) k_argmax_cand(const uint32_t* __restrict__ cnt,
                                                     const uint32_t* __restrict__ cand,
                                                     const unsigned int* __restrict__ ncand,
                                                     unsigned long long* __restrict__ keys, int j,
                                                     const SelCtl* ctl) {
  __shared__ unsigned long long s_best[8];
  pdl_wait();
  pdl_trigger();
  if (ctl != nullptr && *(volatile const uint32_t*)&ctl->stop) return;   // large n only (C5)
  const uint32_t nc = *ncand;
  unsigned long long best = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    const uint32_t v = cand[i];
    argmax_one(cnt[v], v, best, 0u);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(kFull, best, off);
    best = o > best ? o : best;
  }
  if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = (threadIdx.x < (blockDim.x >> 5)) ? s_best[threadIdx.x] : 0ull;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(kFull, best, off);
      best = o > best ? o : best;
    }
    if (threadIdx.x == 0 && best) atomicMax(keys + j, best);
  }
}

// ------------------------------------------------------------------------------------------
// K-COVER: for every local set r in inv[u_j] not yet covered: covered[r] = 1 and, for each
// member w != u_j, count[w] -= 1 (P = 1) or dec[w] += 1 (P > 1, all-reduced before the next
// argmax). One 8-lane group per inverted-index entry: after the first greedy steps the lists are
// short and mostly covered, so spreading entries over many groups (latency hiding) beats
// flattening members within a warp (measured 19 vs 94 us per step on C3).
// ------------------------------------------------------------------------------------------
#ifndef GIM_COVER_ILP
#define GIM_COVER_ILP 16
#endif
constexpr int kCoverIlp = GIM_COVER_ILP;
#ifndef GIM_COVER_BIG
#define GIM_COVER_BIG 256
#endif
constexpr uint32_t kCoverBig = 32;                  // big sets queued per CTA (more: the group does it)
constexpr uint64_t kCoverBigMin = GIM_COVER_BIG;    // members above which the whole CTA decrements

template <bool LIMIT>
__device__ __forceinline__ void cover_step(const unsigned long long* __restrict__ keys, int j,
                                           const InvSegDev* __restrict__ segs,
                                           const uint64_t* __restrict__ offsets,
                                           const uint32_t* __restrict__ pool,
                                           uint8_t* __restrict__ covered, uint32_t* __restrict__ cnt,
                                           int32_t* __restrict__ dec, MrimSel mr,
                                           uint32_t u_known = kEmpty, const uint32_t* __restrict__ cmap = nullptr,
                                           int32_t* __restrict__ cdec = nullptr, SelCtl* ctl = nullptr) {
  __shared__ uint64_t s_lo[kMaxInvSeg], s_end[kMaxInvSeg];   // list start, inclusive prefix end
  __shared__ const uint32_t* s_inv[kMaxInvSeg];
  __shared__ uint32_t s_nseg, s_limit, s_stop;
  const uint32_t sub = threadIdx.x & 7;
  // bounded greedy (IMM estimation rounds, SelCtl): gains never increase, so after the argmax of
  // step j the final covered count is at most cov_j + (kk - j) * gain_j with cov_j = the gains of
  // steps < j. Below cstar the round's test (Alg. 2 l.7) fails whatever the remaining steps pick:
  // the selection stops here (every CTA evaluates the same bound from the same keys).
  // u_known: the pick computed by this CTA itself (cooperative selection; the pick is excluded
  // from later argmaxes there, not retired in cnt, which other CTAs may still be reading).
  // keys[j] == 0: the selection stopped at an earlier step (its argmax made no pick)
  const unsigned long long kj = u_known != kEmpty ? 0ull : keys[j];
  const bool dead = u_known == kEmpty && kj == 0ull;
  const uint32_t u = u_known != kEmpty ? u_known : ~(uint32_t)kj;
  if (!dead && u_known == kEmpty && blockIdx.x == 0 && threadIdx.x == 0) cnt[u] = kSent;   // retire the pick
  uint32_t stop_now = dead ? 1u : 0u;
  if (threadIdx.x < 32) {                     // lanes load the segments' list bounds in parallel
    const uint32_t l = threadIdx.x;
    InvSegDev sg{nullptr, nullptr};
    if (l < (uint32_t)kMaxInvSeg && !dead) sg = segs[l];  // unused slots are null: no dependency on nseg
    uint32_t uncertified = 0;
    if (ctl != nullptr && !dead) {             // bound: loads in parallel with the list bounds
      const unsigned long long cstar = ctl->cstar;
      const uint32_t* tau = ctl->tau;
      unsigned long long sum = 0;
      for (int t = (int)l; t < j; t += 32) sum += keys[t] >> 32;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(kFull, sum, off);
      const unsigned long long bound = sum + (unsigned long long)(ctl->kk - (uint32_t)j) * (kj >> 32);
      // candidate argmax: a pick below tau is not certified (a node outside the list may beat it)
      uncertified = (tau != nullptr && (uint32_t)(kj >> 32) < *tau) ? 1u : 0u;
      stop_now = ((cstar != 0ull && bound < cstar) || uncertified) ? 1u : 0u;
    } else if (ctl != nullptr && dead && ctl->tau != nullptr && *(volatile const uint32_t*)&ctl->stop == 0u) {
      uncertified = 1u;                        // no candidate at all (empty list): not certified either
    }
    // set-id limit (only after a tail truncation), loaded alongside the descriptors
    const uint32_t lim = (LIMIT && l == 0) ? reinterpret_cast<const uint32_t*>(segs + kMaxInvSeg)[1] : 0u;
    uint64_t lo = 0, len = 0;
    if (sg.end) {
      lo = u ? sg.end[u - 1] : 0u;
      len = sg.end[u] - lo;
    }
    uint64_t incl = len;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, incl, off);
      if (l >= (uint32_t)off) incl += y;
    }
    if (l < (uint32_t)kMaxInvSeg) {
      s_lo[l] = lo;
      s_end[l] = incl;
      s_inv[l] = sg.inv;
    }
    const uint32_t used = __ballot_sync(kFull, sg.end != nullptr);   // warp-wide vote
    if (l == 0) {
      s_nseg = __popc(used);
      s_limit = lim;
      s_stop = stop_now;
      if (stop_now && (!dead || uncertified) && blockIdx.x == 0) {
        if (uncertified) ctl->fail = 1u;
        ctl->stop = 1u;
      }
    }
  }
  // MRIM (R27): the pick that gives round t = u / n its k-th seed closes the round: every pair of
  // the round gets the high bit (atomicOr commutes with this kernel's decrements; counts stay
  // < 2^31), so the argmax skips it from now on
  __shared__ uint32_t s_close;
  if (mr.rounds > 1u && threadIdx.x < 32) {
    const uint32_t t = u / mr.n;
    uint32_t picks = 0;
    for (int q = (int)threadIdx.x; q <= j; q += 32) picks += (~(uint32_t)keys[q]) / mr.n == t;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) picks += __shfl_xor_sync(kFull, picks, off);
    if (threadIdx.x == 0) s_close = picks == mr.k ? 1u : 0u;
  }
  __syncthreads();
  if (s_stop) return;
  if (mr.rounds > 1u && s_close) {
    const uint32_t t = u / mr.n;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < mr.n; v += gridDim.x * blockDim.x)
      atomicOr(cnt + (uint64_t)t * mr.n + v, 0x80000000u);
  }
  const uint32_t ns = s_nseg, limit = LIMIT ? s_limit : 0xFFFFFFFFu;
  const uint64_t total = (ns && limit) ? s_end[kMaxInvSeg - 1] : 0;   // limit 0: every set cut
  const uint64_t ngroups = (uint64_t)gridDim.x * (blockDim.x >> 3);
  // big covered sets (the first greedy steps cover hub-rich sets of up to thousands of members):
  // their members are decremented by the whole CTA after its entries, not by one 8-lane group —
  // a 2,793-member set was 22 dependent load rounds of one group
  __shared__ uint64_t s_big_a[kCoverBig], s_big_b[kCoverBig];
  __shared__ uint32_t s_nbig;
  if (threadIdx.x == 0) s_nbig = 0;
  __syncthreads();
  uint32_t q = 0;
  for (uint64_t t = blockIdx.x * (blockDim.x >> 3) + (threadIdx.x >> 3); t < total; t += ngroups) {
    while (t >= s_end[q]) ++q;                 // t increases monotonically per group
    const uint64_t pos = s_lo[q] + (t - (q ? s_end[q - 1] : 0));
    const uint32_t r0 = s_inv[q][pos];
    const uint32_t r = LIMIT ? min(r0, limit - 1u) : r0;   // sets >= limit were truncated away
    // MRIM: entry r is round r mod T of MRIM set r / T, whose T rounds are consecutive sets
    const uint32_t ci = mr.rounds > 1u ? r / mr.rounds : r;
    const uint8_t cov = covered[ci];           // flag and offsets loaded together
    const uint64_t a = offsets[mr.rounds > 1u ? ci * mr.rounds : r];
    const uint64_t b = offsets[mr.rounds > 1u ? ci * mr.rounds + mr.rounds : r + 1];
    if (cov || (LIMIT && r0 != r)) continue;
    if (sub == 0) covered[ci] = 1;     // each set appears once across the lists of u: no race
    if (cmap == nullptr && b - a > kCoverBigMin) {
      uint32_t slot = kCoverBig;
      if (sub == 0) slot = atomicAdd(&s_nbig, 1u);
      slot = __shfl_sync(0xFFu << (threadIdx.x & 24), slot, threadIdx.x & 24);
      if (slot < kCoverBig) {
        if (sub == 0) { s_big_a[slot] = a; s_big_b[slot] = b; }
        continue;
      }
    }
    // members: kCoverIlp loads in flight per lane (big sets would otherwise serialise one L2
    // round trip per 8 members), then fire-and-forget decrements; u itself is skipped
    for (uint64_t e = a + sub; e < b; e += 8 * kCoverIlp) {
      uint32_t w[kCoverIlp];
#pragma unroll
      for (int t = 0; t < kCoverIlp; ++t) w[t] = (e + 8 * t < b) ? pool[e + 8 * t] : u;
      if (cmap != nullptr) {                   // cooperative selection: candidates only
        uint32_t ci[kCoverIlp];
#pragma unroll
        for (int t = 0; t < kCoverIlp; ++t) ci[t] = (w[t] == u) ? kEmpty : __ldg(cmap + w[t]);
#pragma unroll
        for (int t = 0; t < kCoverIlp; ++t)
          if (ci[t] != kEmpty) atomicAdd(cdec + ci[t], 1);
        continue;
      }
#pragma unroll
      for (int t = 0; t < kCoverIlp; ++t) {
        if (w[t] == u) continue;
        if (dec == nullptr) atomicSub(cnt + w[t], 1u);
        else atomicAdd(dec + w[t], 1);
      }
    }
  }
  __syncthreads();
  const uint32_t nbig = min(s_nbig, (uint32_t)kCoverBig);
  for (uint32_t i = 0; i < nbig; ++i) {
    const uint64_t a = s_big_a[i], b = s_big_b[i];
    for (uint64_t e = a + threadIdx.x; e < b; e += (uint64_t)blockDim.x * 4) {
      uint32_t w[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) w[t] = (e + (uint64_t)blockDim.x * t < b) ? pool[e + (uint64_t)blockDim.x * t] : u;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (w[t] == u) continue;
        if (dec == nullptr) atomicSub(cnt + w[t], 1u);
        else atomicAdd(dec + w[t], 1);
      }
    }
  }
}

template <bool LIMIT>
__global__ void __launch_bounds__(256) k_cover(const unsigned long long* __restrict__ keys, int j,
                                               const InvSegDev* __restrict__ segs, SelCtl* ctl,
                                               const uint64_t* __restrict__ offsets,
                                               const uint32_t* __restrict__ pool,
                                               uint8_t* __restrict__ covered, uint32_t* __restrict__ cnt,
                                               int32_t* __restrict__ dec, MrimSel mr) {
  pdl_wait();
  pdl_trigger();
  cover_step<LIMIT>(keys, j, segs, offsets, pool, covered, cnt, dec, mr, kEmpty, nullptr, nullptr, ctl);
}

// ------------------------------------------------------------------------------------------
// Fused greedy step (P = 1): k_cover_next(j) retires pick j and decrements (cover_step), then the
// last CTA to finish — a completion ticket per step — computes pick j + 1 over the candidate
// list: the nodes whose initial count reaches tau (at most a few thousand). Counts only
// decrease, so a best candidate count >= tau certifies the argmax over all nodes (every other
// node started below tau); otherwise *fail is set and the host redoes the selection with the
// full-scan argmax. One launch and one dependency chain per greedy step instead of two.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void cand_argmax_cta(const uint32_t* cnt, const uint32_t* __restrict__ cand,
                                                uint32_t nc, uint32_t tau_p1, unsigned long long* keys, int j,
                                                uint32_t* fail) {
  __shared__ unsigned long long s_cbest[32];
  unsigned long long best = 0;
  for (uint32_t i0 = threadIdx.x; i0 < nc; i0 += 4 * blockDim.x) {
    uint32_t v[4], c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = i0 + u * blockDim.x;
      v[u] = i < nc ? cand[i] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) c[u] = (i0 + u * blockDim.x < nc) ? __ldcg(cnt + v[u]) : kSent;   // L2: atomics land there
#pragma unroll
    for (int u = 0; u < 4; ++u) argmax_one(c[u], v[u], best, 0u);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(kFull, best, off);
    best = o > best ? o : best;
  }
  if ((threadIdx.x & 31) == 0) s_cbest[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = (threadIdx.x < (blockDim.x >> 5)) ? s_cbest[threadIdx.x] : 0ull;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(kFull, best, off);
      best = o > best ? o : best;
    }
    if (threadIdx.x == 0) {
      keys[j] = best;
      if (best == 0ull || (uint32_t)(best >> 32) < tau_p1) atomicExch(fail, 1u);   // not certified
    }
  }
}

__global__ void __launch_bounds__(256) k_cand_argmax0(const uint32_t* cnt, const uint32_t* __restrict__ cand,
                                                      const unsigned int* __restrict__ ncand,
                                                      const uint32_t* __restrict__ tau_p1,
                                                      unsigned long long* keys, uint32_t* fail) {
  cand_argmax_cta(cnt, cand, *ncand, *tau_p1, keys, 0, fail);
}

template <bool LIMIT>
__global__ void __launch_bounds__(256) k_cover_next(unsigned long long* __restrict__ keys, int j, int kk,
                                                    const InvSegDev* __restrict__ segs,
                                                    const uint64_t* __restrict__ offsets,
                                                    const uint32_t* __restrict__ pool,
                                                    uint8_t* __restrict__ covered, uint32_t* __restrict__ cnt,
                                                    const uint32_t* __restrict__ cand,
                                                    const unsigned int* __restrict__ ncand,
                                                    const uint32_t* __restrict__ tau_p1,
                                                    unsigned int* __restrict__ done, uint32_t* fail) {
  if (keys[j] == 0ull) return;                 // no candidate left (already failed): the rest no-ops
  cover_step<LIMIT>(keys, j, segs, offsets, pool, covered, cnt, nullptr, MrimSel{1u, 0u, 0u});
  if (j + 1 >= kk) return;
  __shared__ uint32_t s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();                            // this CTA's decrements before its ticket
    s_last = atomicAdd(done + j, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  cand_argmax_cta(cnt, cand, *ncand, *tau_p1, keys, j + 1, fail);
}

// Grid-wide barrier of a co-resident (cooperatively launched) grid: generation counter; the
// arriving CTA reads the generation before arriving, the last arrival resets the count and bumps
// the generation; fences order every CTA's writes of the phase before the next phase's reads.
__device__ __forceinline__ void grid_barrier(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = bar + 1;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------------------
// Cooperative selection (P = 1, GIM_OPT_SELECT_COOP): the k greedy steps in ONE cooperative
// launch with ONE grid barrier per step. The argmax only ever looks at the candidate list (the
// <= C nodes whose initial count reaches tau; counts only decrease, so a best candidate count
// >= tau certifies the global argmax), and every CTA computes it redundantly from a private
// copy of the candidates' counts in shared memory — no cross-CTA reduction, hence no barrier
// between the argmax and the cover of a step. The cover of step j adds the decrements of
// CANDIDATE members to buffer B[j % 3] (indexed through cmap: node -> candidate index);
// after the step's barrier every CTA subtracts B[j % 3] from its copy. Three rotating buffers
// make a buffer's reuse safe with one barrier per step: B[(j+1) % 3] (read in step j-1's
// argmax, by every CTA before barrier j-1) is zeroed by block 0 during step j, and its next
// writer is step j+1's cover, after barrier j. Non-candidate counts are never read again. An
// uncertified step makes every CTA (all compute the same best) stop and sets *fail: the host
// redoes the selection with the full-scan kernels.
// ------------------------------------------------------------------------------------------
constexpr uint32_t kCoopCandMax = 8192;
template <bool LIMIT>
__global__ void __launch_bounds__(1024, 1) k_select_coop(const uint32_t* __restrict__ cnt,
                                                         const uint32_t* __restrict__ cand,
                                                         const unsigned int* __restrict__ ncand,
                                                         const uint32_t* __restrict__ tau_p1,
                                                         const uint32_t* __restrict__ cmap, int32_t* cdec,
                                                         unsigned long long* __restrict__ keys, int kk,
                                                         const InvSegDev* __restrict__ segs,
                                                         const uint64_t* __restrict__ offsets,
                                                         const uint32_t* __restrict__ pool,
                                                         uint8_t* __restrict__ covered, unsigned int* bar,
                                                         uint32_t* fail) {
  extern __shared__ uint32_t s_coop[];               // [kCoopCandMax] counts + [kCoopCandMax] node ids
  uint32_t* s_cnt = s_coop;                          // this CTA's copy of the candidates' counts
  uint32_t* s_v = s_coop + kCoopCandMax;
  __shared__ unsigned long long s_red[32];
  __shared__ uint32_t s_idx[32];
  const uint32_t nc = min(*ncand, kCoopCandMax), tau = *tau_p1;
  for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
    const uint32_t v = cand[i];
    s_v[i] = v;
    s_cnt[i] = cnt[v];
  }
  __syncthreads();
  for (int j = 0; j < kk; ++j) {
    if (j > 0) {                                          // the previous step's decrements
      const int32_t* bj = cdec + (uint64_t)((j - 1) % 3) * kCoopCandMax;
      for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x)
        if (s_cnt[i] != kSent) s_cnt[i] -= (uint32_t)__ldcg(bj + i);
    }
    if (blockIdx.x == 0) {                                // zero the buffer step j+1 will fill
      int32_t* bz = cdec + (uint64_t)((j + 1) % 3) * kCoopCandMax;
      for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) bz[i] = 0;
    }
    __syncthreads();
    unsigned long long best = 0;                          // key = count << 32 | ~v (R10)
    uint32_t bidx = 0;
    for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
      const uint32_t c = s_cnt[i];
      if (c == kSent) continue;
      const unsigned long long key = ((unsigned long long)c << 32) | (unsigned long long)(~s_v[i]);
      if (key > best) { best = key; bidx = i; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(kFull, best, off);
      const uint32_t oi = __shfl_xor_sync(kFull, bidx, off);
      if (o > best) { best = o; bidx = oi; }
    }
    if ((threadIdx.x & 31) == 0) { s_red[threadIdx.x >> 5] = best; s_idx[threadIdx.x >> 5] = bidx; }
    __syncthreads();
    if (threadIdx.x < 32) {
      best = (threadIdx.x < (blockDim.x >> 5)) ? s_red[threadIdx.x] : 0ull;
      bidx = (threadIdx.x < (blockDim.x >> 5)) ? s_idx[threadIdx.x] : 0u;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(kFull, best, off);
        const uint32_t oi = __shfl_xor_sync(kFull, bidx, off);
        if (o > best) { best = o; bidx = oi; }
      }
      if (threadIdx.x == 0) {
        s_red[0] = best;
        s_idx[0] = bidx;
        if (best != 0ull) s_cnt[bidx] = kSent;            // excluded from later steps
      }
    }
    __syncthreads();
    best = s_red[0];
    __syncthreads();                                      // s_red is rewritten next step
    if (best == 0ull || (uint32_t)(best >> 32) < tau) {   // not certified: every CTA stops
      if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(fail, 1u);
      return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) keys[j] = best;
    cover_step<LIMIT>(keys, j, segs, offsets, pool, covered, nullptr, nullptr, MrimSel{1u, 0u, 0u},
                      ~(uint32_t)best, cmap, cdec + (uint64_t)(j % 3) * kCoopCandMax);
    grid_barrier(bar);
  }
}

// The k greedy steps of one NodeSelection in ONE cooperative launch (P = 1): per step the argmax
// phase and the cover phase of the kernels above, separated by grid barriers instead of kernel
// boundaries (GIM_OPT_SELECT_PERSISTENT).
template <bool LIMIT>
__global__ void __launch_bounds__(1024, 1) k_select_persistent(uint32_t* __restrict__ cnt, uint32_t n,
                                                           unsigned long long* __restrict__ keys, int kk,
                                                           const InvSegDev* __restrict__ segs,
                                                           const uint64_t* __restrict__ offsets,
                                                           const uint32_t* __restrict__ pool,
                                                           uint8_t* __restrict__ covered, MrimSel mr,
                                                           uint32_t excl, unsigned int* bar) {
  for (int j = 0; j < kk; ++j) {
    argmax_step(cnt, nullptr, n, keys, j, nullptr, excl, 0u);
    grid_barrier(bar);
    cover_step<LIMIT>(keys, j, segs, offsets, pool, covered, cnt, nullptr, mr);
    grid_barrier(bar);
  }
}

// ------------------------------------------------------------------------------------------
// Small-graph NodeSelection (P = 1, standard IM, n counts fit in shared memory): all k greedy
// steps in ONE CTA of 1024 threads — the count vector lives in shared memory (argmax = a scan of
// shared memory, decrements = shared atomics), the covered flags / inverted lists / pool in
// global memory (L2-resident at these sizes). Between argmax and cover only __syncthreads: no
// kernel boundary and no grid barrier per step (Alg. 1 l.6-10, Alg. 7; bounded greedy
// of SelCtl as in cover_step).
// ------------------------------------------------------------------------------------------
constexpr int kSmallSelThreads = 1024;
template <bool LIMIT>
__global__ void __launch_bounds__(kSmallSelThreads, 1) k_select_cta(const uint32_t* __restrict__ count_total,
                                                                   uint32_t n, unsigned long long* __restrict__ keys,
                                                                   int kk, const InvSegDev* __restrict__ segs,
                                                                   const uint64_t* __restrict__ offsets,
                                                                   const uint32_t* __restrict__ pool,
                                                                   uint8_t* __restrict__ covered, SelCtl* ctl) {
  extern __shared__ uint32_t s_cnt[];                 // [n]
  __shared__ unsigned long long s_wbest[kSmallSelThreads / 32];
  __shared__ uint64_t s_lo[kMaxInvSeg], s_end[kMaxInvSeg];
  __shared__ const uint32_t* s_inv[kMaxInvSeg];
  __shared__ const uint32_t* s_endp[kMaxInvSeg];
  __shared__ uint32_t s_u, s_stop, s_nseg, s_limit;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t v = tid; v < n; v += kSmallSelThreads) s_cnt[v] = count_total[v];
  if (tid < 32) {
    InvSegDev sg{nullptr, nullptr};
    if (tid < kMaxInvSeg) sg = segs[tid];
    if (tid < kMaxInvSeg) {
      s_inv[tid] = sg.inv;
      s_endp[tid] = sg.end;
    }
    const uint32_t used = __ballot_sync(kFull, sg.end != nullptr);
    if (tid == 0) {
      s_nseg = __popc(used);
      s_limit = LIMIT ? reinterpret_cast<const uint32_t*>(segs + kMaxInvSeg)[1] : 0xFFFFFFFFu;
    }
  }
  const unsigned long long cstar = ctl ? ctl->cstar : 0ull;
  unsigned long long cov = 0;                         // thread 0: gains of the steps so far
  __syncthreads();
  const uint32_t nseg = s_nseg, limit = s_limit;
  const uint32_t sub = tid & 7;
  for (int j = 0; j < kk; ++j) {
    // argmax over the shared counts (4 independent loads per thread per round)
    unsigned long long best = 0;
    for (uint32_t v = tid; v < n; v += kSmallSelThreads) argmax_one(s_cnt[v], v, best, 0u);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(kFull, best, off);
      best = o > best ? o : best;
    }
    if (lane == 0) s_wbest[warp] = best;
    __syncthreads();
    if (warp == 0) {
      best = s_wbest[lane];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(kFull, best, off);
        best = o > best ? o : best;
      }
      const uint32_t u = ~(uint32_t)best;
      // lane q < nseg: list bounds of u in segment q, inclusive prefix over the segments
      uint64_t lo = 0, len = 0;
      if ((uint32_t)lane < nseg) {
        const uint32_t* e = s_endp[lane];
        lo = u ? e[u - 1] : 0u;
        len = e[u] - lo;
      }
      uint64_t incl = len;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint64_t y = __shfl_up_sync(kFull, incl, off);
        if (lane >= off) incl += y;
      }
      if (lane < kMaxInvSeg) {
        s_lo[lane] = lo;
        s_end[lane] = (uint32_t)lane < nseg ? incl : ~0ull;
      }
      if (lane == 0) {
        keys[j] = best;
        const unsigned long long g = best >> 32;
        // bounded greedy: the remaining kk - j steps gain at most g each
        const bool stop = cstar != 0ull && cov + (unsigned long long)(kk - j) * g < cstar;
        cov += g;
        s_stop = stop ? 1u : 0u;
        if (stop) ctl->stop = 1u;
        s_u = u;
        s_cnt[u] = kSent;                             // retire the pick
      }
    }
    __syncthreads();
    if (s_stop) break;
    const uint32_t u = s_u;
    const uint64_t total = (nseg && limit) ? s_end[nseg - 1] : 0ull;
    // cover: one 8-lane group per inverted-list entry of u (as cover_step)
    uint32_t q = 0;
    for (uint64_t t = tid >> 3; t < total; t += kSmallSelThreads / 8) {
      while (t >= s_end[q]) ++q;
      const uint64_t pos = s_lo[q] + (t - (q ? s_end[q - 1] : 0));
      const uint32_t r0 = s_inv[q][pos];
      const uint32_t r = LIMIT ? min(r0, limit - 1u) : r0;
      const uint8_t cv = covered[r];
      const uint64_t a = offsets[r], b = offsets[r + 1];
      if (cv || (LIMIT && r0 != r)) continue;
      if (sub == 0) covered[r] = 1;
      for (uint64_t e = a + sub; e < b; e += 8 * 8) {
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = (e + 8 * i < b) ? pool[e + 8 * i] : u;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (w[i] != u) atomicSub(&s_cnt[w[i]], 1u);
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------
// Mid-size graphs (n <= 8 x 51,200): the same single-launch selection on a thread-block CLUSTER
// of CS CTAs (one per SM): CTA r keeps the counts of nodes [r ns, (r+1) ns) in its shared memory;
// the argmax is a local scan + an exchange of the CS partial bests through distributed shared
// memory, the cover is split over all CTAs of the cluster and decrements a member's count with an
// atomic on its owner's shared memory (DSMEM); two cluster barriers per greedy step, no launch.
// ------------------------------------------------------------------------------------------
template <bool LIMIT>
__global__ void __launch_bounds__(kSmallSelThreads, 1) k_select_cluster(const uint32_t* __restrict__ count_total,
                                                                       uint32_t n, uint32_t ns,
                                                                       unsigned long long* __restrict__ keys, int kk,
                                                                       const InvSegDev* __restrict__ segs,
                                                                       const uint64_t* __restrict__ offsets,
                                                                       const uint32_t* __restrict__ pool,
                                                                       uint8_t* __restrict__ covered, SelCtl* ctl) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ uint32_t s_cnt[];                 // [ns]: counts of this CTA's node range
  __shared__ unsigned long long s_wbest[kSmallSelThreads / 32];
  __shared__ unsigned long long s_mybest;             // read by every CTA of the cluster
  __shared__ uint64_t s_lo[kMaxInvSeg], s_end[kMaxInvSeg];
  __shared__ const uint32_t* s_inv[kMaxInvSeg];
  __shared__ const uint32_t* s_endp[kMaxInvSeg];
  __shared__ uint32_t s_u, s_stop, s_nseg, s_limit;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster.block_rank(), cs = cluster.num_blocks();
  const uint32_t v0 = rank * ns, v1 = min(n, v0 + ns);
  for (uint32_t i = tid; i < ns; i += kSmallSelThreads) s_cnt[i] = (v0 + i < v1) ? count_total[v0 + i] : kSent;
  if (tid < 32) {
    InvSegDev sg{nullptr, nullptr};
    if (tid < kMaxInvSeg) sg = segs[tid];
    if (tid < kMaxInvSeg) {
      s_inv[tid] = sg.inv;
      s_endp[tid] = sg.end;
    }
    const uint32_t used = __ballot_sync(kFull, sg.end != nullptr);
    if (tid == 0) {
      s_nseg = __popc(used);
      s_limit = LIMIT ? reinterpret_cast<const uint32_t*>(segs + kMaxInvSeg)[1] : 0xFFFFFFFFu;
    }
  }
  const unsigned long long cstar = ctl ? ctl->cstar : 0ull;
  unsigned long long cov = 0;                         // thread 0: gains of the steps so far
  cluster.sync();                                     // every CTA's counts are in place
  const uint32_t nseg = s_nseg, limit = s_limit;
  const uint32_t sub = tid & 7;
  for (int j = 0; j < kk; ++j) {
    unsigned long long best = 0;
    for (uint32_t i = tid; i < v1 - v0; i += kSmallSelThreads) argmax_one(s_cnt[i], v0 + i, best, 0u);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(kFull, best, off);
      best = o > best ? o : best;
    }
    if (lane == 0) s_wbest[warp] = best;
    __syncthreads();
    if (warp == 0) {
      best = s_wbest[lane];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(kFull, best, off);
        best = o > best ? o : best;
      }
      if (lane == 0) s_mybest = best;
    }
    cluster.sync();                                   // partial bests published
    if (warp == 0) {
      best = 0;
      if ((uint32_t)lane < cs) best = *cluster.map_shared_rank(&s_mybest, (unsigned)lane);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(kFull, best, off);
        best = o > best ? o : best;
      }
      const uint32_t u = ~(uint32_t)best;
      uint64_t lo = 0, len = 0;
      if ((uint32_t)lane < nseg) {
        const uint32_t* e = s_endp[lane];
        lo = u ? e[u - 1] : 0u;
        len = e[u] - lo;
      }
      uint64_t incl = len;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint64_t y = __shfl_up_sync(kFull, incl, off);
        if (lane >= off) incl += y;
      }
      if (lane < kMaxInvSeg) {
        s_lo[lane] = lo;
        s_end[lane] = (uint32_t)lane < nseg ? incl : ~0ull;
      }
      if (lane == 0) {
        const unsigned long long g = best >> 32;
        const bool stop = cstar != 0ull && cov + (unsigned long long)(kk - j) * g < cstar;
        cov += g;
        s_stop = stop ? 1u : 0u;
        s_u = u;
        if (rank == 0) {
          keys[j] = best;
          if (stop) ctl->stop = 1u;
        }
        if (u - v0 < v1 - v0) s_cnt[u - v0] = kSent;   // the owner retires the pick
      }
    }
    __syncthreads();
    if (s_stop) break;                                // the same decision in every CTA
    const uint32_t u = s_u;
    const uint64_t total = (nseg && limit) ? s_end[nseg - 1] : 0ull;
    uint32_t q = 0;
    const uint64_t gstride = (uint64_t)cs * (kSmallSelThreads / 8);
    for (uint64_t t = (uint64_t)rank * (kSmallSelThreads / 8) + (tid >> 3); t < total; t += gstride) {
      while (t >= s_end[q]) ++q;
      const uint64_t pos = s_lo[q] + (t - (q ? s_end[q - 1] : 0));
      const uint32_t r0 = s_inv[q][pos];
      const uint32_t r = LIMIT ? min(r0, limit - 1u) : r0;
      const uint8_t cv = covered[r];
      const uint64_t a = offsets[r], b = offsets[r + 1];
      if (cv || (LIMIT && r0 != r)) continue;
      if (sub == 0) covered[r] = 1;
      for (uint64_t e = a + sub; e < b; e += 8 * 8) {
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = (e + 8 * i < b) ? pool[e + 8 * i] : u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (w[i] == u) continue;
          const uint32_t owner = w[i] / ns;
          atomicSub(cluster.map_shared_rank(s_cnt, owner) + (w[i] - owner * ns), 1u);
        }
      }
    }
    cluster.sync();                                   // every decrement landed before the next argmax
  }
  cluster.sync();                                     // no CTA leaves while others may touch its smem
}

// ------------------------------------------------------------------------------------------
// Host launch wrappers
// ------------------------------------------------------------------------------------------
int g_pdl = 0;   // GIM_OPT_PDL (process-wide: the launch wrappers carry no ctx)
void set_pdl(int on) { g_pdl = on ? 1 : 0; }

uint64_t scan_tiles(uint64_t count) { return (count + kScanTile - 1) / kScanTile; }

template <class OutT>
cudaError_t launch_scan_impl(const uint32_t* in, uint64_t count, OutT* out, uint64_t* tile_tmp,
                             uint64_t* total_tmp, cudaStream_t s, int* launches) {
  const uint64_t nt = scan_tiles(count);
  if (nt > 0) {
    k_scan_sums<<<(unsigned)nt, kScanThreads, 0, s>>>(in, count, tile_tmp);
    ++*launches;
  }
  k_scan_tiles<<<1, kScanThreads, 0, s>>>(tile_tmp, nt, total_tmp);
  ++*launches;
  k_scan_apply<OutT><<<(unsigned)(nt > 0 ? nt : 1), kScanThreads, 0, s>>>(in, count, tile_tmp, total_tmp, out);
  ++*launches;
  return cudaGetLastError();
}
cudaError_t launch_scan_u32(const uint32_t* in, uint64_t count, uint64_t* out, uint64_t* tile_tmp,
                            uint64_t* total_tmp, cudaStream_t s, int* launches) {
  return launch_scan_impl<uint64_t>(in, count, out, tile_tmp, total_tmp, s, launches);
}
cudaError_t launch_scan_u32_to32(const uint32_t* in, uint64_t count, uint32_t* out, uint64_t* tile_tmp,
                                 uint64_t* total_tmp, cudaStream_t s, int* launches) {
  return launch_scan_impl<uint32_t>(in, count, out, tile_tmp, total_tmp, s, launches);
}
cudaError_t launch_seg_scan(const uint32_t* cnt, uint32_t* snap, uint64_t count, uint32_t* out, bool inclusive,
                            uint64_t* tile_tmp, uint64_t* total_tmp, cudaStream_t s, int* launches) {
  const uint64_t nt = scan_tiles(count);
  if (nt > 0) k_seg_sums<<<(unsigned)nt, kScanThreads, 0, s>>>(cnt, snap, count, tile_tmp);
  k_scan_tiles<<<1, kScanThreads, 0, s>>>(tile_tmp, nt, total_tmp);
  k_seg_apply<<<(unsigned)(nt > 0 ? nt : 1), kScanThreads, 0, s>>>(cnt, snap, count, tile_tmp, total_tmp, out,
                                                                    inclusive ? 1 : 0);
  *launches = nt > 0 ? 3 : 2;
  return cudaGetLastError();
}

cudaError_t launch_inv_scatter(const uint64_t* offsets, const uint32_t* pool, uint32_t set0, uint32_t set1,
                               uint32_t* end, uint32_t* inv, int grid, cudaStream_t s, uint32_t n, int passes,
                               int* launches) {
  const uint32_t span = (uint32_t)(((uint64_t)n + passes - 1) / passes);
  *launches = 0;
  for (int q = 0; q < passes; ++q) {
    const uint32_t lo = (uint32_t)std::min<uint64_t>((uint64_t)q * span, n);
    const uint32_t len = (uint32_t)std::min<uint64_t>(span, (uint64_t)n - lo);
    if (len == 0) break;
    k_inv_scatter<<<grid, 256, 0, s>>>(offsets, pool, set0, set1, end, inv, lo, len);
    ++*launches;
  }
  return cudaGetLastError();
}

// Writes the segment descriptor table from a by-value parameter (no host staging buffer).
struct SegTable {
  InvSegDev seg[kMaxInvSeg];
  uint32_t nseg, limit;
};
__global__ void k_set_segs(SegTable t, InvSegDev* out, uint32_t* nseg_out) {
  if (threadIdx.x < kMaxInvSeg) out[threadIdx.x] = t.seg[threadIdx.x];
  if (threadIdx.x == 0) {
    nseg_out[0] = t.nseg;
    nseg_out[1] = t.limit;            // local sets >= limit were truncated away
  }
}

cudaError_t launch_set_segs(const InvSegDev* segs, uint32_t nseg, uint32_t limit, InvSegDev* out,
                            uint32_t* nseg_out, cudaStream_t s) {
  SegTable t;
  for (int q = 0; q < kMaxInvSeg; ++q) t.seg[q] = (q < (int)nseg) ? segs[q] : InvSegDev{nullptr, nullptr};
  t.nseg = nseg;
  t.limit = limit;
  k_set_segs<<<1, 32, 0, s>>>(t, out, nseg_out);
  return cudaGetLastError();
}


// Launch with programmatic stream serialization (see pdl_wait / pdl_trigger).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

cudaError_t launch_argmax(uint32_t* cnt, int32_t* dec, uint32_t n, unsigned long long* keys, int j,
                          const uint32_t* tau_p1, int grid, cudaStream_t s, bool excl, uint32_t id_base,
                          const SelCtl* ctl) {
  return launch_pdl(k_argmax, grid, 256, s, cnt, dec, n, keys, j, tau_p1, excl ? 0x80000000u : 0u, id_base, ctl);
}

__global__ void k_sel_ctl(SelCtl* ctl, unsigned long long cstar, uint32_t kk, const uint32_t* tau) {
  ctl->cstar = cstar;
  ctl->stop = 0u;
  ctl->kk = kk;
  ctl->fail = 0u;
  ctl->tau = tau;
}
cudaError_t launch_sel_ctl(SelCtl* ctl, unsigned long long cstar, uint32_t kk, const uint32_t* tau, cudaStream_t s) {
  k_sel_ctl<<<1, 1, 0, s>>>(ctl, cstar, kk, tau);
  return cudaGetLastError();
}

cudaError_t launch_rs_pack(const unsigned long long* local_keys, int j, uint32_t rank, uint32_t world,
                           unsigned long long* kx, cudaStream_t s) {
  k_rs_pack<<<1, 64, 0, s>>>(local_keys, j, rank, world, kx);
  return cudaGetLastError();
}
cudaError_t launch_rs_pick(const unsigned long long* kx, uint32_t world, unsigned long long* keys, int j,
                           uint32_t* gshard, uint32_t id_base, uint32_t ns_valid, cudaStream_t s) {
  k_rs_pick<<<1, 32, 0, s>>>(kx, world, keys, j, gshard, id_base, ns_valid);
  return cudaGetLastError();
}

cudaError_t launch_cand_setup(const uint32_t* cnt, uint32_t n, uint32_t kmax, unsigned int* hist,
                              uint32_t* tau_p1, uint32_t* cand, unsigned int* ncand, int grid, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(hist, 0, 33 * sizeof(unsigned int), s);
  if (e != cudaSuccess) return e;
  k_cnt_hist<<<grid, 256, 0, s>>>(cnt, n, hist);
  k_pick_tau<<<1, 1, 0, s>>>(hist, kmax, tau_p1, ncand);
  k_cand_compact<<<grid, 256, 0, s>>>(cnt, n, tau_p1, cand, ncand);
  return cudaGetLastError();
}

cudaError_t launch_argmax_cand(const uint32_t* cnt, const uint32_t* cand, const unsigned int* ncand,
                               unsigned long long* keys, int j, int grid, cudaStream_t s, const SelCtl* ctl) {
  return launch_pdl(k_argmax_cand, grid, 256, s, cnt, cand, ncand, keys, j, ctl);
}

cudaError_t launch_select_persistent(uint32_t* cnt, uint32_t n, unsigned long long* keys, int kk,
                                     const InvSegDev* segs, const uint64_t* offsets, const uint32_t* pool,
                                     uint8_t* covered, const MrimSel* mr, bool limit, unsigned int* bar,
                                     int num_sms, cudaStream_t s) {
  const MrimSel m = mr ? *mr : MrimSel{1u, 0u, 0u};
  const uint32_t excl = mr ? 0x80000000u : 0u;
  void* kern = limit ? (void*)k_select_persistent<true> : (void*)k_select_persistent<false>;
  // one 1024-thread CTA per SM: the grid barrier's arrival counter sees #SM atomics, not 4-8x more
  const int grid = num_sms;
  void* args[] = {&cnt, &n, &keys, &kk, &segs, &offsets, &pool, &covered, (void*)&m, (void*)&excl, &bar};
  return cudaLaunchCooperativeKernel(kern, dim3((unsigned)grid), dim3(1024), args, 0, s);
}

cudaError_t launch_select_fused(unsigned long long* keys, int kk, const InvSegDev* segs, const uint64_t* offsets,
                                const uint32_t* pool, uint8_t* covered, uint32_t* cnt, const uint32_t* cand,
                                const unsigned int* ncand, const uint32_t* tau_p1, unsigned int* done,
                                uint32_t* fail, int grid, cudaStream_t s, bool limit, int* launches) {
  k_cand_argmax0<<<1, 256, 0, s>>>(cnt, cand, ncand, tau_p1, keys, fail);
  for (int j = 0; j < kk; ++j) {
    if (limit)
      k_cover_next<true><<<grid, 256, 0, s>>>(keys, j, kk, segs, offsets, pool, covered, cnt, cand, ncand, tau_p1,
                                              done, fail);
    else
      k_cover_next<false><<<grid, 256, 0, s>>>(keys, j, kk, segs, offsets, pool, covered, cnt, cand, ncand, tau_p1,
                                               done, fail);
  }
  *launches = kk + 1;
  return cudaGetLastError();
}

// cmap[v] = candidate index of node v, kEmpty otherwise (filled by k_cand_map after a kEmpty memset)
__global__ void k_cand_map(const uint32_t* __restrict__ cand, const unsigned int* __restrict__ ncand,
                           uint32_t* __restrict__ cmap, int unmap) {
  const uint32_t nc = min(*ncand, kCoopCandMax);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x)
    cmap[cand[i]] = unmap ? kEmpty : i;
}

cudaError_t launch_select_coop(const uint32_t* cnt, const uint32_t* cand, const unsigned int* ncand,
                               const uint32_t* tau_p1, uint32_t* cmap, int32_t* cdec, unsigned long long* keys,
                               int kk, const InvSegDev* segs, const uint64_t* offsets, const uint32_t* pool,
                               uint8_t* covered, unsigned int* bar, uint32_t* fail, int num_sms, bool limit,
                               cudaStream_t s) {
  const int smem = (int)(2 * kCoopCandMax * 4);
  void* kern = limit ? (void*)k_select_coop<true> : (void*)k_select_coop<false>;
  static std::atomic<uint64_t> attr{0};
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  if (!(attr.load() & (1ull << (dev & 63)))) {
    if (cudaError_t e = cudaFuncSetAttribute((const void*)k_select_coop<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) return e;
    if (cudaError_t e = cudaFuncSetAttribute((const void*)k_select_coop<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) return e;
    attr.fetch_or(1ull << (dev & 63));
  }
  k_cand_map<<<64, 256, 0, s>>>(cand, ncand, cmap, 0);
  void* args[] = {&cnt, &cand, &ncand, &tau_p1, &cmap, &cdec, &keys, &kk, &segs, &offsets, &pool, &covered, &bar, &fail};
  cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3((unsigned)num_sms), dim3(1024), args, (size_t)smem, s);
  if (e != cudaSuccess) return e;
  k_cand_map<<<64, 256, 0, s>>>(cand, ncand, cmap, 1);   // restore cmap to all-kEmpty
  return cudaGetLastError();
}

uint32_t select_cta_max_n() { return (uint32_t)((200u << 10) / 4); }   // counts in <= 200 KB of shared memory

cudaError_t launch_select_cta(const uint32_t* count_total, uint32_t n, unsigned long long* keys, int kk,
                              const InvSegDev* segs, const uint64_t* offsets, const uint32_t* pool,
                              uint8_t* covered, SelCtl* ctl, bool limit, cudaStream_t s) {
  const int smem = (int)(n * 4u);
  static std::atomic<uint64_t> attr{0};
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  if (!(attr.load() & (1ull << (dev & 63)))) {
    const int cap = (int)(select_cta_max_n() * 4u);
    if (cudaError_t e = cudaFuncSetAttribute((const void*)k_select_cta<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap)) return e;
    if (cudaError_t e = cudaFuncSetAttribute((const void*)k_select_cta<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap)) return e;
    attr.fetch_or(1ull << (dev & 63));
  }
  if (limit) k_select_cta<true><<<1, kSmallSelThreads, smem, s>>>(count_total, n, keys, kk, segs, offsets, pool, covered, ctl);
  else k_select_cta<false><<<1, kSmallSelThreads, smem, s>>>(count_total, n, keys, kk, segs, offsets, pool, covered, ctl);
  return cudaGetLastError();
}

uint32_t select_cluster_max_n() { return 8u * select_cta_max_n(); }

cudaError_t launch_select_cluster(const uint32_t* count_total, uint32_t n, unsigned long long* keys, int kk,
                                  const InvSegDev* segs, const uint64_t* offsets, const uint32_t* pool,
                                  uint8_t* covered, SelCtl* ctl, bool limit, cudaStream_t s) {
  const uint32_t cs = (n + select_cta_max_n() - 1) / select_cta_max_n();   // 2..8 CTAs
  const uint32_t ns = (n + cs - 1) / cs;
  const int smem = (int)(ns * 4u);
  static std::atomic<uint64_t> attr{0};
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  if (!(attr.load() & (1ull << (dev & 63)))) {
    const int cap = (int)(select_cta_max_n() * 4u);
    for (const void* f : {(const void*)k_select_cluster<true>, (const void*)k_select_cluster<false>}) {
      if (cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, cap)) return e;
      if (cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 0)) return e;
    }
    attr.fetch_or(1ull << (dev & 63));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(kSmallSelThreads);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (limit)
    return cudaLaunchKernelEx(&cfg, k_select_cluster<true>, count_total, n, ns, keys, kk, segs, offsets, pool, covered, ctl);
  return cudaLaunchKernelEx(&cfg, k_select_cluster<false>, count_total, n, ns, keys, kk, segs, offsets, pool, covered, ctl);
}

cudaError_t launch_cover(const unsigned long long* keys, int j, const InvSegDev* segs, SelCtl* ctl,
                         const uint64_t* offsets, const uint32_t* pool,
                         uint8_t* covered, uint32_t* cnt, int32_t* dec, int grid, cudaStream_t s, bool limit,
                         const MrimSel* mr) {
  const MrimSel m = mr ? *mr : MrimSel{1u, 0u, 0u};
  if (limit) return launch_pdl(k_cover<true>, grid, 256, s, keys, j, segs, ctl, offsets, pool, covered, cnt, dec, m);
  return launch_pdl(k_cover<false>, grid, 256, s, keys, j, segs, ctl, offsets, pool, covered, cnt, dec, m);
}

}  // namespace gim

// mc.cu — forward Monte-Carlo spread under IC (verification at scale).
//
// What it computes: I(S) in one sampled instance graph, the number of nodes a seed set S
// activates when every newly active node u tries each out-edge (u, v) once, succeeding with
// probability p_uv (the IC process, §2.2), averaged over `trials` instance
// graphs. It uses none of the reverse (RR) machinery, so comparing it with n * F_R'(S) on an
// independent RR pool checks Eq. 3 at full size (north_star: "Monte-Carlo-verified
// spread within 1%").
//
// Randomness (tag 11): the coin of out-edge slot e in trial t is word
// (e & 3) of Philox4x32-10 with key (mc_seed_lo, mc_seed_hi) and counter (t_lo, t_hi, e >> 2,
// 0xC0000000); out-slots are the rows of the out-CSR sorted by (source, in-slot). Each edge is
// tried at most once, so the activated set is the forward closure of S over live out-edges and
// does not depend on the order of expansion: every trial's size is exact, and equals the oracle's
// (oracle/gim_oracle.c og_mc_spread) trial by trial.
//
// B200 shape: the out-CSR (uint32 offsets, destination and per-slot WC threshold) is built once
// on the device (CUB stable radix sort of the in-slots by source). The MC kernel runs one trial
// per CTA at a time (persistent CTAs claim trials), level-synchronous BFS with a global visited
// bitmap and queue per CTA slot; within a level a warp expands a batch of up to 32 frontier
// nodes by sweeping their concatenated slot groups (one Philox per lane per step, coins before
// any load of the destination).
#include <cub/device/device_radix_sort.cuh>

#include "gim_device.cuh"
#include "gim_internal.h"

namespace gim {

namespace {

constexpr uint32_t kSlotMcHi = 0xC0000000u;   // tag 11
constexpr int kMcThreads = 512;

__global__ void k_out_deg(const uint32_t* __restrict__ src, uint64_t m, uint32_t* __restrict__ odeg) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(odeg + src[e], 1u);
}

__global__ void k_iota(uint32_t* __restrict__ a, uint64_t m) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
    a[e] = (uint32_t)e;
}

// in_dst[e] = v for every in-slot e of row v (a warp per row)
__global__ void k_in_dst(const uint32_t* __restrict__ row_ptr, uint32_t n, uint32_t* __restrict__ in_dst) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += (gridDim.x * blockDim.x) >> 5)
    for (uint32_t e = row_ptr[v] + lane; e < row_ptr[v + 1]; e += 32) in_dst[e] = v;
}

// out-slot j (sorted by (source, in-slot)): destination and the live threshold of the scheme
__global__ void k_out_fill(const uint32_t* __restrict__ sorted_in_slot, const uint32_t* __restrict__ in_dst,
                           uint64_t m, uint32_t* __restrict__ out_dst, uint32_t* __restrict__ out_in) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < m; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = sorted_in_slot[j];
    out_dst[j] = in_dst[e];
    out_in[j] = e;
  }
}

__global__ void k_out_thr_wc(const uint32_t* __restrict__ out_dst, const uint32_t* __restrict__ row_ptr, uint64_t m,
                             uint32_t* __restrict__ thr) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < m; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = out_dst[j];
    thr[j] = 0xFFFFFFFFu / (row_ptr[v + 1] - row_ptr[v]);   // coin <= thr <=> coin * d_in(v) < 2^32
  }
}

struct McParams {
  uint32_t n;
  const uint32_t* out_ptr;     // [n+1]
  const uint32_t* out_dst;     // [m]
  const uint32_t* out_in;      // [m] in-slot of each out-slot (explicit weights)
  const uint32_t* thr_wc;      // [m] WC: live iff coin <= thr_wc[j]
  const uint64_t* thr_edge;    // explicit: live iff coin < thr_edge[in-slot]
  uint64_t thr_uniform;        // uniform: live iff coin < thr_uniform
  const uint32_t* seeds;
  uint32_t k;
  uint64_t trials;
  uint32_t rk[20];             // round keys of mc_seed
  unsigned long long* claim;
  uint32_t* sizes;             // [trials]
};

template <int SCHEME>
__device__ __forceinline__ uint32_t mc_live_mask(const McParams& p, uint4 w, uint32_t g, uint32_t a, uint32_t b) {
  const uint32_t e0 = g << 2;
  const uint32_t words[4] = {w.x, w.y, w.z, w.w};
  uint32_t m = 0;
  if (SCHEME == W_WC) {
    const uint4 t = *reinterpret_cast<const uint4*>(p.thr_wc + e0);   // 16-B aligned group
    const uint32_t th[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) m |= (uint32_t)(words[j] <= th[j]) << j;
  } else if (SCHEME == W_UNIFORM) {
#pragma unroll
    for (int j = 0; j < 4; ++j) m |= (uint32_t)((uint64_t)words[j] < p.thr_uniform) << j;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (e0 + j >= a && e0 + j < b) m |= (uint32_t)((uint64_t)words[j] < p.thr_edge[p.out_in[e0 + j]]) << j;
  }
  const uint32_t lo = a > e0 ? a - e0 : 0u;
  const uint32_t hi = (b - e0) < 4u ? b - e0 : 4u;
  return m & (0xFFFFFFFFu << lo) & (0xFu >> (4u - hi));
}

template <int SCHEME>
__global__ void __launch_bounds__(kMcThreads, 2) k_mc_ic(McParams p, uint32_t* bitmaps, uint32_t* queues,
                                                        uint64_t bm_words) {
  __shared__ unsigned long long s_t;
  __shared__ uint32_t s_head, s_tail;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t* bm = bitmaps + (uint64_t)blockIdx.x * bm_words;
  uint32_t* Q = queues + (uint64_t)blockIdx.x * p.n;
  while (true) {
    if (threadIdx.x == 0) {
      s_t = atomicAdd(p.claim, 1ull);
      s_tail = 0;
    }
    __syncthreads();
    const unsigned long long t = s_t;
    if (t >= p.trials) break;
    // S activates first (duplicates once)
    for (uint32_t i = threadIdx.x; i < p.k; i += blockDim.x) {
      const uint32_t u = p.seeds[i];
      const uint32_t bit = 1u << (u & 31);
      if (!(atomicOr(bm + (u >> 5), bit) & bit)) Q[atomicAdd(&s_tail, 1u)] = u;
    }
    __syncthreads();
    uint32_t lo = 0, hi = s_tail;
    while (lo < hi) {                          // level-synchronous: expand Q[lo, hi)
      if (threadIdx.x == 0) s_head = lo;
      __syncthreads();
      while (true) {
        uint32_t f = 0;
        if (lane == 0) f = atomicAdd(&s_head, 32u);
        f = __shfl_sync(kFull, f, 0);
        if (f >= hi) break;
        const uint32_t c = min(32u, hi - f);
        uint32_t a = 0, b = 0, ng = 0;
        if (lane < c) {
          const uint32_t u = Q[f + lane];
          a = p.out_ptr[u];
          b = p.out_ptr[u + 1];
          if (b > a) ng = ((b - 1) >> 2) - (a >> 2) + 1;
        }
        // flattened sweep over the batch's slot groups (inclusive prefix P per lane)
        uint32_t P = ng;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, P, off);
          if ((int)lane >= off) P += y;
        }
        const uint32_t total = __shfl_sync(kFull, P, 31);
        const uint32_t E = P - ng;
        for (uint32_t base = 0; base < total; base += 32) {
          const uint32_t gi = base + lane;
          const uint32_t kk = warp_owner(P, gi < total ? gi : total - 1);
          const uint32_t ak = __shfl_sync(kFull, a, kk), bk = __shfl_sync(kFull, b, kk);
          const uint32_t gk = __shfl_sync(kFull, (a >> 2) - E, kk);
          uint32_t m = 0, g = 0;
          if (gi < total) {
            g = gk + gi;
            const uint4 w = philox4x32_10_rk(make_uint4((uint32_t)t, (uint32_t)(t >> 32), g, kSlotMcHi), p.rk);
            m = mc_live_mask<SCHEME>(p, w, g, ak, bk);
          }
          while (m) {
            const uint32_t j = __ffs(m) - 1;
            m &= m - 1;
            const uint32_t v = p.out_dst[(g << 2) + j];
            const uint32_t bit = 1u << (v & 31);
            if (!(atomicOr(bm + (v >> 5), bit) & bit)) Q[atomicAdd(&s_tail, 1u)] = v;
          }
        }
      }
      __syncthreads();
      lo = hi;
      hi = s_tail;
      __syncthreads();
    }
    const uint32_t size = hi;
    if (threadIdx.x == 0) p.sizes[t] = size;
    // restore the slot (shared with K-GIANT: bitmap all zero, queue all kEmpty); whole bitmap
    // words can be cleared since every set bit belongs to a member
    for (uint32_t i = threadIdx.x; i < size; i += blockDim.x) {
      bm[Q[i] >> 5] = 0u;
      Q[i] = kEmpty;
    }
    __syncthreads();
  }
}

// LT forward process (Eq. 1) with the exact threshold comparison of reading R30:
// tau_v = (o + 1/2) / 2^32, o = word 0 of Philox(mc_seed; t, tag 11 | 2^40 | v); v activates when
// its active in-neighbours reach it — WC: cnt * 2^33 >= (2o + 1) * d_in(v); explicit: sum of
// W = floor(w 2^32) >= o + 1. Per slot and node a 64-bit accumulator (trial tag << 40 | acc),
// updated by CAS: the update that crosses the threshold activates v (exactly once), so the
// activated set is the order-free fixpoint, trial by trial equal to the oracle's.
template <int SCHEME>
__device__ __forceinline__ bool lt_met(uint64_t acc, uint32_t o, uint32_t d) {
  if (SCHEME == W_WC) return ((unsigned __int128)acc << 33) >= (unsigned __int128)(2ull * o + 1ull) * d;
  return acc >= (uint64_t)o + 1ull;
}

template <int SCHEME>
__global__ void __launch_bounds__(kMcThreads, 2) k_mc_lt(McParams p, const uint32_t* __restrict__ row_ptr,
                                                        uint32_t* bitmaps, uint32_t* queues, uint64_t bm_words,
                                                        unsigned long long* accs) {
  __shared__ unsigned long long s_t;
  __shared__ uint32_t s_head, s_tail;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t* bm = bitmaps + (uint64_t)blockIdx.x * bm_words;
  uint32_t* Q = queues + (uint64_t)blockIdx.x * p.n;
  unsigned long long* acc = accs + (uint64_t)blockIdx.x * p.n;
  while (true) {
    if (threadIdx.x == 0) {
      s_t = atomicAdd(p.claim, 1ull);
      s_tail = 0;
    }
    __syncthreads();
    const unsigned long long t = s_t;
    if (t >= p.trials) break;
    const unsigned long long tag = (t % 0xFFFFFFull) + 1ull;   // 24-bit, never 0 (= untouched)
    for (uint32_t i = threadIdx.x; i < p.k; i += blockDim.x) {
      const uint32_t u = p.seeds[i];
      const uint32_t bit = 1u << (u & 31);
      if (!(atomicOr(bm + (u >> 5), bit) & bit)) Q[atomicAdd(&s_tail, 1u)] = u;
    }
    __syncthreads();
    uint32_t lo = 0, hi = s_tail;
    while (lo < hi) {
      if (threadIdx.x == 0) s_head = lo;
      __syncthreads();
      while (true) {
        uint32_t f = 0;
        if (lane == 0) f = atomicAdd(&s_head, 32u);
        f = __shfl_sync(kFull, f, 0);
        if (f >= hi) break;
        const uint32_t c = min(32u, hi - f);
        uint32_t a = 0, b = 0, nv = 0;
        if (lane < c) {
          const uint32_t u = Q[f + lane];
          a = p.out_ptr[u];
          b = p.out_ptr[u + 1];
          nv = b - a;
        }
        // flattened sweep over the batch's out-slots, one slot per lane
        uint32_t P = nv;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, P, off);
          if ((int)lane >= off) P += y;
        }
        const uint32_t total = __shfl_sync(kFull, P, 31);
        const uint32_t E = P - nv;
        for (uint32_t base = 0; base < total; base += 32) {
          const uint32_t gi = base + lane;
          const uint32_t kk = warp_owner(P, gi < total ? gi : total - 1);
          const uint32_t ek = __shfl_sync(kFull, a - E, kk);
          if (gi >= total) continue;
          const uint32_t e = ek + gi;
          const uint32_t v = p.out_dst[e];
          const uint32_t bit = 1u << (v & 31);
          if (bm[v >> 5] & bit) continue;                   // already active
          const uint64_t inc = (SCHEME == W_WC) ? 1ull : p.thr_edge[p.out_in[e]];
          unsigned long long old = acc[v], prev, nw;
          uint64_t cur;
          while (true) {
            cur = ((old >> 40) == tag) ? (old & ((1ull << 40) - 1ull)) : 0ull;
            nw = (tag << 40) | (cur + inc);
            prev = atomicCAS(acc + v, old, nw);
            if (prev == old) break;
            old = prev;
          }
          const uint32_t o = philox4x32_10_rk(make_uint4((uint32_t)t, (uint32_t)(t >> 32), v, kSlotMcHi | 0x100u), p.rk).x;
          const uint32_t d = (SCHEME == W_WC) ? row_ptr[v + 1] - row_ptr[v] : 0u;
          if (lt_met<SCHEME>(cur + inc, o, d) && !lt_met<SCHEME>(cur, o, d) &&
              !(atomicOr(bm + (v >> 5), bit) & bit))
            Q[atomicAdd(&s_tail, 1u)] = v;
        }
      }
      __syncthreads();
      lo = hi;
      hi = s_tail;
      __syncthreads();
    }
    const uint32_t size = hi;
    if (threadIdx.x == 0) p.sizes[t] = size;
    for (uint32_t i = threadIdx.x; i < size; i += blockDim.x) {
      bm[Q[i] >> 5] = 0u;
      Q[i] = kEmpty;
    }
    __syncthreads();
  }
}

}  // namespace

// Out-CSR of the in-CSR: out_ptr[n+1], out_dst[m], out_in[m] (in-slot of each out-slot, rows
// sorted by (source, in-slot): CUB's radix sort is stable), thr_wc[m] for WC. tmp = scratch
// provided by the caller (query its size with tmp == nullptr -> *tmp_bytes).
cudaError_t build_out_csr(const uint32_t* row_ptr, const uint32_t* src, uint32_t n, uint64_t m, int scheme,
                          uint32_t* out_ptr, uint32_t* out_dst, uint32_t* out_in, uint32_t* thr_wc,
                          void* tmp, size_t* tmp_bytes, uint64_t* scan_tmp, int grid, cudaStream_t s) {
  size_t cub_bytes = 0;
  cub::DoubleBuffer<uint32_t> dk(nullptr, nullptr), dv(nullptr, nullptr);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, dk, dv, (int64_t)m, 0, 32, s);
  if (e != cudaSuccess) return e;
  const size_t need = 4 * (m + 1) * 4 + ((uint64_t)n + 1) * 4 + cub_bytes + 256;
  if (!tmp) {
    *tmp_bytes = need;
    return cudaSuccess;
  }
  uint32_t* k0 = static_cast<uint32_t*>(tmp);
  uint32_t* k1 = k0 + (m + 1);
  uint32_t* v0 = k1 + (m + 1);
  uint32_t* v1 = v0 + (m + 1);
  uint32_t* deg = v1 + (m + 1);                       // n + 1
  void* cub_tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(deg + n + 1) + 255) & ~uintptr_t(255));
  // keys = source of each in-slot, values = in-slot
  if ((e = cudaMemcpyAsync(k0, src, m * 4, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
  k_iota<<<grid, 256, 0, s>>>(v0, m);
  cub::DoubleBuffer<uint32_t> keys(k0, k1), vals(v0, v1);
  int end_bit = 1;
  while (end_bit < 32 && (1ull << end_bit) < n) ++end_bit;
  if ((e = cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, keys, vals, (int64_t)m, 0, end_bit, s)) != cudaSuccess)
    return e;
  // out-degrees -> out_ptr (exclusive prefix; m < 2^32)
  if ((e = cudaMemsetAsync(deg, 0, (uint64_t)n * 4, s)) != cudaSuccess) return e;
  k_out_deg<<<grid, 256, 0, s>>>(src, m, deg);
  int nl = 0;
  if ((e = launch_scan_u32_to32(deg, n, out_ptr, scan_tmp, scan_tmp + scan_tiles(n) + 1, s, &nl)) != cudaSuccess)
    return e;
  // out_ptr[n] = m
  const uint32_t m32 = (uint32_t)m;
  if ((e = cudaMemcpyAsync(out_ptr + n, &m32, 4, cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
  // in_dst into the other spare buffer
  uint32_t* in_dst = (vals.Current() == v0) ? v1 : v0;
  k_in_dst<<<grid, 256, 0, s>>>(row_ptr, n, in_dst);
  k_out_fill<<<grid, 256, 0, s>>>(vals.Current(), in_dst, m, out_dst, out_in);
  if (scheme == W_WC) k_out_thr_wc<<<grid, 256, 0, s>>>(out_dst, row_ptr, m, thr_wc);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;   // m32 is a stack value
  return cudaGetLastError();
}

cudaError_t launch_mc_ic(int scheme, uint32_t n, const uint32_t* out_ptr, const uint32_t* out_dst,
                         const uint32_t* out_in, const uint32_t* thr_wc, const uint64_t* thr_edge,
                         uint64_t thr_uniform, const uint32_t* seeds, uint32_t k, uint64_t trials, uint64_t mc_seed,
                         unsigned long long* claim, uint32_t* sizes, uint32_t* bitmaps, uint32_t* queues,
                         uint64_t bm_words, int grid, cudaStream_t s, const uint32_t* row_ptr,
                         unsigned long long* lt_accs) {
  McParams p{};
  p.n = n;
  p.out_ptr = out_ptr;
  p.out_dst = out_dst;
  p.out_in = out_in;
  p.thr_wc = thr_wc;
  p.thr_edge = thr_edge;
  p.thr_uniform = thr_uniform;
  p.seeds = seeds;
  p.k = k;
  p.trials = trials;
  uint32_t k0 = (uint32_t)mc_seed, k1 = (uint32_t)(mc_seed >> 32);
  for (int r = 0; r < 10; ++r) {
    p.rk[2 * r] = k0;
    p.rk[2 * r + 1] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  p.claim = claim;
  p.sizes = sizes;
  if (lt_accs) {
    if (scheme == W_WC) k_mc_lt<W_WC><<<grid, kMcThreads, 0, s>>>(p, row_ptr, bitmaps, queues, bm_words, lt_accs);
    else k_mc_lt<W_EXPLICIT><<<grid, kMcThreads, 0, s>>>(p, row_ptr, bitmaps, queues, bm_words, lt_accs);
    return cudaGetLastError();
  }
  if (scheme == W_WC) k_mc_ic<W_WC><<<grid, kMcThreads, 0, s>>>(p, bitmaps, queues, bm_words);
  else if (scheme == W_UNIFORM) k_mc_ic<W_UNIFORM><<<grid, kMcThreads, 0, s>>>(p, bitmaps, queues, bm_words);
  else k_mc_ic<W_EXPLICIT><<<grid, kMcThreads, 0, s>>>(p, bitmaps, queues, bm_words);
  return cudaGetLastError();
}

}  // namespace gim

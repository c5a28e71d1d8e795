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
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const uint32_t* __restrict__ in, uint64_t count,
                                                             const uint64_t* __restrict__ tile_sums,
                                                             const uint64_t* __restrict__ grand_total,
                                                             uint64_t* __restrict__ out) {
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
    if (base + j < count) out[base + j] = ex;
    ex += v[j];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[count] = *grand_total;
}

// ------------------------------------------------------------------------------------------
// K-INV scatter: inv[inv_off[v] + cursor[v]++] = local set index r, for every member v of r.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_inv_scatter(const uint64_t* __restrict__ offsets,
                                                     const uint32_t* __restrict__ pool, uint32_t nsets,
                                                     const uint64_t* __restrict__ inv_off,
                                                     uint32_t* __restrict__ cursor,
                                                     uint32_t* __restrict__ inv) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nsets; r += nwarps) {
    const uint64_t a = offsets[r], b = offsets[r + 1];
    for (uint64_t t = a + lane; t < b; t += 32) {
      const uint32_t v = pool[t];
      const uint32_t pos = atomicAdd(cursor + v, 1u);
      inv[inv_off[v] + pos] = r;
    }
  }
}

// ------------------------------------------------------------------------------------------
// K-ARGMAX: keys[j] = max over v of (selected ? 0 : count[v] << 32 | ~v). Applies the
// all-reduced decrements of the previous step first (P > 1) and retires the previous pick.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_argmax(uint32_t* __restrict__ cnt, int32_t* __restrict__ dec,
                                                uint32_t n, unsigned long long* __restrict__ keys, int j) {
  __shared__ unsigned long long s_best[8];
  const uint32_t uprev = (j > 0) ? ~(uint32_t)keys[j - 1] : kEmpty;
  unsigned long long best = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    uint32_t c = cnt[v];
    bool dirty = false;
    if (dec != nullptr) {
      const int32_t d = dec[v];
      if (d) { c -= (uint32_t)d; dec[v] = 0; dirty = true; }
    }
    if (v == uprev) { c = kSent; dirty = true; }
    if (dirty) cnt[v] = c;
    const unsigned long long key = (c == kSent) ? 0ull : (((unsigned long long)c << 32) | (unsigned long long)(~v));
    best = key > best ? key : best;
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
// member w, count[w] -= 1 (P = 1) or dec[w] += 1 (P > 1, all-reduced before the next argmax).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_cover(const unsigned long long* __restrict__ keys, int j,
                                               const uint64_t* __restrict__ inv_off,
                                               const uint32_t* __restrict__ inv,
                                               const uint64_t* __restrict__ offsets,
                                               const uint32_t* __restrict__ pool,
                                               uint8_t* __restrict__ covered, uint32_t* __restrict__ cnt,
                                               int32_t* __restrict__ dec) {
  const int lane = threadIdx.x & 31;
  const uint32_t u = ~(uint32_t)keys[j];
  const uint64_t lo = inv_off[u], hi = inv_off[u + 1];
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t t = lo + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < hi; t += nwarps) {
    const uint32_t r = inv[t];
    if (covered[r]) continue;
    __syncwarp();
    if (lane == 0) covered[r] = 1;
    const uint64_t a = offsets[r], b = offsets[r + 1];
    if (dec == nullptr) {
      for (uint64_t e = a + lane; e < b; e += 32) atomicSub(cnt + pool[e], 1u);
    } else {
      for (uint64_t e = a + lane; e < b; e += 32) atomicAdd(dec + pool[e], 1);
    }
  }
}

// ------------------------------------------------------------------------------------------
// Host launch wrappers
// ------------------------------------------------------------------------------------------
uint64_t scan_tiles(uint64_t count) { return (count + kScanTile - 1) / kScanTile; }

cudaError_t launch_scan_u32(const uint32_t* in, uint64_t count, uint64_t* out, uint64_t* tile_tmp,
                            uint64_t* total_tmp, cudaStream_t s, int* launches) {
  const uint64_t nt = scan_tiles(count);
  if (nt > 0) {
    k_scan_sums<<<(unsigned)nt, kScanThreads, 0, s>>>(in, count, tile_tmp);
    ++*launches;
  }
  k_scan_tiles<<<1, kScanThreads, 0, s>>>(tile_tmp, nt, total_tmp);
  ++*launches;
  k_scan_apply<<<(unsigned)(nt > 0 ? nt : 1), kScanThreads, 0, s>>>(in, count, tile_tmp, total_tmp, out);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_inv_scatter(const uint64_t* offsets, const uint32_t* pool, uint32_t nsets,
                               const uint64_t* inv_off, uint32_t* cursor, uint32_t* inv, int grid,
                               cudaStream_t s) {
  k_inv_scatter<<<grid, 256, 0, s>>>(offsets, pool, nsets, inv_off, cursor, inv);
  return cudaGetLastError();
}

cudaError_t launch_argmax(uint32_t* cnt, int32_t* dec, uint32_t n, unsigned long long* keys, int j,
                          int grid, cudaStream_t s) {
  k_argmax<<<grid, 256, 0, s>>>(cnt, dec, n, keys, j);
  return cudaGetLastError();
}

cudaError_t launch_cover(const unsigned long long* keys, int j, const uint64_t* inv_off,
                         const uint32_t* inv, const uint64_t* offsets, const uint32_t* pool,
                         uint8_t* covered, uint32_t* cnt, int32_t* dec, int grid, cudaStream_t s) {
  k_cover<<<grid, 256, 0, s>>>(keys, j, inv_off, inv, offsets, pool, covered, cnt, dec);
  return cudaGetLastError();
}

}  // namespace gim

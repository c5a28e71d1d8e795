// inv_sort.cu — sort-based inverted-index segment (K-INV, large n).
//
// The node -> RR-set index (Alg. 7's "sets containing u", built once per segment as
// DESIGN.md §9 "Inverted index" describes) is normally scattered: inv[cursor[v]++] = r for every
// element (v in RR set r). When the per-node cursor array is far larger than the L2 (C5: 41.6M
// nodes, 166 MB) and the sets are tiny, every scatter step is a random DRAM read-modify-write.
// Here the same segment is produced by a stable radix sort of the segment's (node, set) pairs by
// node instead: keys = the pool slice itself (nodes), values = the local set index of each
// element, written in pool order, so the sorted values ARE the lists, each in ascending set order
// (a deterministic layout; the scatter's order within a list is arbitrary, and the cover does not
// depend on it). The per-node list ends come from the same count scan as the scatter's (its
// inclusive form). cub::DeviceRadixSort is a library primitive (like the sort mc.cu uses for the
// out-CSR).
#include <cub/device/device_radix_sort.cuh>
#include "gim_device.cuh"
#include "gim_internal.h"

namespace gim {

// vals[e - e0] = local set index r of element e, for the sets [set0, set1) (pool-contiguous).
// A warp takes 32 consecutive sets and writes their members' set indices 32 at a time.
__global__ void __launch_bounds__(256) k_set_ids(const uint64_t* __restrict__ offsets, uint32_t set0, uint32_t set1,
                                                 uint64_t e0, uint32_t* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t r0 = set0 + (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32u; r0 < set1;
       r0 += nwarps * 32u) {
    const uint32_t nr = min(32u, set1 - r0);
    const uint64_t base = offsets[r0];
    const uint32_t hi_rel = (uint32_t)(offsets[r0 + nr] - base);
    const uint32_t P = (lane < nr) ? (uint32_t)(offsets[r0 + lane + 1] - base) : hi_rel;
    for (uint32_t i0 = 0; i0 < hi_rel; i0 += 32) {
      const uint32_t i = i0 + lane;
      const uint32_t k = warp_owner(P, i);
      if (i < hi_rel) vals[base - e0 + i] = r0 + k;
    }
  }
}

size_t inv_sort_tmp_bytes(uint64_t elements, uint32_t nbits) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)elements, 0, (int)nbits);
  return bytes;
}

cudaError_t launch_inv_sort(const uint64_t* offsets, const uint32_t* pool, uint32_t set0, uint32_t set1, uint64_t e0,
                            uint64_t elements, uint32_t nbits, uint32_t* keys_tmp, uint32_t* vals_tmp, void* cub_tmp,
                            size_t cub_bytes, uint32_t* inv, int grid, cudaStream_t s, int* launches) {
  *launches = 0;
  k_set_ids<<<grid, 256, 0, s>>>(offsets, set0, set1, e0, vals_tmp);
  ++*launches;
  if (cudaError_t e = cudaGetLastError()) return e;
  size_t bytes = cub_bytes;
  if (cudaError_t e = cub::DeviceRadixSort::SortPairs(cub_tmp, bytes, pool + e0, keys_tmp, vals_tmp, inv,
                                                      (int64_t)elements, 0, (int)nbits, s))
    return e;
  *launches += 4;                                        // onesweep passes (launch accounting only)
  return cudaGetLastError();
}

}  // namespace gim

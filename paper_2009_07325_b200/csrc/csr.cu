// csr.cu — on-device validation of the canonical in-CSR (reading R15) and conversion of the
// uint64 row pointers of the C ABI to the uint32 row pointers the kernels read (§8(a) row a1).
// One warp per row: monotone row pointers within [0, m], sources < n, no self-loop, sources
// strictly ascending. Violations set bits in *err and the lowest offending row in *bad_row;
// err[2] receives the largest in-degree (the geometric-skip contract tabulates 1/ln(1 - 1/d)).
#include "gim_device.cuh"
#include "gim_internal.h"

namespace gim {

__global__ void __launch_bounds__(256) k_validate_csr(const uint64_t* __restrict__ rp64, uint32_t n,
                                                      uint64_t m, const uint32_t* __restrict__ src,
                                                      uint32_t* __restrict__ rp32, uint32_t* err,
                                                      uint32_t* bad_row, uint32_t* __restrict__ thr_node,
                                                      uint32_t v0, uint32_t v1) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t v = v0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); v < v1; v += nwarps) {
    const uint64_t a = rp64[v], b = rp64[v + 1];
    uint32_t e_bits = 0;
    if (b < a || b > m) {
      e_bits = 1u;
    } else {
      for (uint64_t e = a + lane; e < b; e += 32) {
        const uint32_t u = src[e];
        if (u >= n) e_bits |= 2u;
        if (u == v) e_bits |= 4u;
        if (e > a && src[e - 1] >= u) e_bits |= 8u;
      }
    }
    e_bits = __reduce_or_sync(kFull, e_bits);
    if (lane == 0 && b > a && b - a > *(volatile uint32_t*)(err + 2)) atomicMax(err + 2, (uint32_t)(b - a));
    if (lane == 0) {
      rp32[v] = (uint32_t)a;
      // WC live threshold of row v (p = 1/d_in(v): coin <= thr <=> coin * d < 2^32), read by the
      // RR kernels in parallel with the row pointers instead of a division per expanded node
      if (thr_node) thr_node[v] = (b > a) ? (uint32_t)(0xFFFFFFFFull / (b - a)) : 0u;
      if (e_bits) {
        atomicOr(err, e_bits);
        atomicMin(bad_row, v);
      }
    }
  }
  if (v1 == n && blockIdx.x == 0 && threadIdx.x == 0) rp32[n] = (uint32_t)m;
}

// Rows [v0, v1) (their sources must be resident: gim_load_graph validates each row range as soon
// as its slice of src has arrived, overlapping the rest of the upload).
cudaError_t launch_validate_csr(const uint64_t* rp64, uint32_t n, uint64_t m, const uint32_t* src,
                                uint32_t* rp32, uint32_t* err, uint32_t* bad_row, uint32_t* thr_node, int grid,
                                cudaStream_t s, uint32_t v0, uint32_t v1) {
  k_validate_csr<<<grid, 256, 0, s>>>(rp64, n, m, src, rp32, err, bad_row, thr_node, v0, v1);
  return cudaGetLastError();
}

}  // namespace gim

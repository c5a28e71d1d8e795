// gim_internal.h — host-side declarations of the kernel launch wrappers (libgim internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gim {
struct RRParams;

int lt_blocks_per_sm();
// native NCCL exchange (nccl_ex.cu): dlopen'ed NCCL; hooks with the gim_*_fn signatures
bool nccl_available();
int nccl_unique_id(void* out128);
int nccl_comm_init(void** comm, const void* id128, int rank, int world);
void nccl_comm_destroy(void* comm);
int nccl_allreduce_i32(void* buf, uint64_t count, void* stream, void* comm);
int nccl_allgather_bytes(const void* send, uint64_t bytes, void* recv, void* stream, void* comm);
int nccl_reducescatter_i32(void* send, void* recv, uint64_t recv_count, void* stream, void* comm);
#ifdef GIM_GIANT_TRACE
void giant_trace_dump(cudaStream_t s);   // diagnostic build: per-set K-GIANT timing to stderr
#endif
cudaError_t launch_rr_ic_lane(int scheme, const RRParams& p, int grid, cudaStream_t s);
cudaError_t launch_rr_warp(int model, int scheme, const RRParams& p, int grid, cudaStream_t s);
cudaError_t launch_rr_giant(int model, int scheme, const RRParams& p, int grid, uint32_t* bitmaps,
                            uint32_t* gqueues, uint64_t bm_words, cudaStream_t s, int nt, bool sq);
// geometric-skip contract (skip.cu, reading R31)
cudaError_t launch_skip_lane(int scheme, const RRParams& p, int grid, cudaStream_t s);
cudaError_t launch_skip_warp(int scheme, const RRParams& p, int grid, cudaStream_t s);
cudaError_t launch_skip_giant(int scheme, const RRParams& p, int grid, uint32_t* bitmaps, uint32_t* gqueues,
                              uint64_t bm_words, cudaStream_t s);
int skip_lane_blocks_per_sm();
uint64_t skip_lane_spill_words(int grid);   // lane kernel's global member spill, words
uint64_t spill_words_per_warp();   // spill tier of the warp kernels: words per warp
constexpr int kSkipTabK = 184;   // log centers k = -75..106 (+ padding) of the R31 ln
cudaError_t launch_skip_tables(int scheme, float p_uniform, uint32_t max_deg, double* tab, cudaStream_t s);
cudaError_t launch_store(const uint32_t* staging, const uint32_t* sizes, const uint64_t* soff,
                         const uint64_t* scan, uint32_t count, uint64_t pool_base, uint32_t* pool,
                         uint64_t* offsets_out, uint32_t* count_total, uint32_t rounds, uint32_t round0,
                         uint32_t n, int grid, cudaStream_t s);
cudaError_t launch_count_add(const uint32_t* pool, uint64_t e0, uint64_t e1, uint32_t* count_total, int grid,
                             cudaStream_t s);
cudaError_t launch_sizes_of(const uint64_t* offsets, uint64_t cnt, uint64_t padded, uint32_t* sizes, int grid,
                            cudaStream_t s);
cudaError_t launch_offsets_of(const uint64_t* scan, uint64_t cnt, uint64_t base, uint64_t* offsets_out, int grid,
                              cudaStream_t s);
cudaError_t launch_count_sub(const uint32_t* pool, uint64_t e0, uint64_t e1, uint32_t* count_total,
                             int grid, cudaStream_t s);
cudaError_t launch_count_sub_range(const uint32_t* pool, const uint64_t* e0p, const uint64_t* e1p, uint32_t* cnt,
                                   int grid, cudaStream_t s);

cudaError_t launch_philox_bench(uint64_t seed, uint32_t per_thread, uint32_t* sink, int grid, cudaStream_t s,
                                int chains);

uint64_t scan_tiles(uint64_t count);
void set_pdl(int on);   // programmatic dependent launch of the selection kernels (GIM_OPT_PDL)
cudaError_t launch_scan_u32(const uint32_t* in, uint64_t count, uint64_t* out, uint64_t* tile_tmp,
                            uint64_t* total_tmp, cudaStream_t s, int* launches);
// same, 32-bit output (the caller guarantees the total is < 2^32)
cudaError_t launch_scan_u32_to32(const uint32_t* in, uint64_t count, uint32_t* out, uint64_t* tile_tmp,
                                 uint64_t* total_tmp, cudaStream_t s, int* launches);
// index segment histogram (count_total - snap) + scan, snap := count_total; out = list starts
// (exclusive) or list ends (inclusive), out[count] = total
cudaError_t launch_seg_scan(const uint32_t* cnt, uint32_t* snap, uint64_t count, uint32_t* out, bool inclusive,
                            uint64_t* tile_tmp, uint64_t* total_tmp, cudaStream_t s, int* launches);
cudaError_t launch_inv_scatter(const uint64_t* offsets, const uint32_t* pool, uint32_t set0, uint32_t set1,
                               uint32_t* end, uint32_t* inv, int grid, cudaStream_t s, uint32_t n, int passes,
                               int* launches);
// sort-based index segment (inv_sort.cu): inv = set indices sorted by node (list ends: the
// inclusive segment scan)
size_t inv_sort_tmp_bytes(uint64_t elements, uint32_t nbits);
cudaError_t launch_inv_sort(const uint64_t* offsets, const uint32_t* pool, uint32_t set0, uint32_t set1, uint64_t e0,
                            uint64_t elements, uint32_t nbits, uint32_t* keys_tmp, uint32_t* vals_tmp, void* cub_tmp,
                            size_t cub_bytes, uint32_t* inv, int grid, cudaStream_t s, int* launches);
struct InvSegDev;
cudaError_t launch_set_segs(const InvSegDev* segs, uint32_t nseg, uint32_t limit, InvSegDev* out,
                            uint32_t* nseg_out, cudaStream_t s);
struct SelCtl;
cudaError_t launch_argmax(uint32_t* cnt, int32_t* dec, uint32_t n, unsigned long long* keys, int j,
                          const uint32_t* tau_p1, int grid, cudaStream_t s, bool excl = false,
                          uint32_t id_base = 0, const SelCtl* ctl = nullptr);
// node-sharded selection (gim_set_reducescatter): key exchange pack / global pick
cudaError_t launch_rs_pack(const unsigned long long* local_keys, int j, uint32_t rank, uint32_t world,
                           unsigned long long* kx, cudaStream_t s);
cudaError_t launch_rs_pick(const unsigned long long* kx, uint32_t world, unsigned long long* keys, int j,
                           uint32_t* gshard, uint32_t id_base, uint32_t ns_valid, cudaStream_t s);
cudaError_t launch_cand_setup(const uint32_t* cnt, uint32_t n, uint32_t kmax, unsigned int* hist,
                              uint32_t* tau_p1, uint32_t* cand, unsigned int* ncand, int grid, cudaStream_t s);
cudaError_t launch_argmax_cand(const uint32_t* cnt, const uint32_t* cand, const unsigned int* ncand,
                               unsigned long long* keys, int j, int grid, cudaStream_t s,
                               const SelCtl* ctl = nullptr);
struct InvSegDev;
// Bounded greedy of an IMM estimation round (gim_imm): cstar = the
// smallest covered count that passes the round's test (Alg. 2 l.7); 0 disables. stop is set by
// the cover of the first step whose bound cov_j + (kk - j) * gain_j falls below cstar, and every
// later argmax / cover of the selection returns at once.
// Candidate argmax (large n): tau points at the certificate threshold; a pick below it is not
// certified — the cover sets fail (and stop) and the host redoes the selection with full scans.
struct SelCtl {
  unsigned long long cstar;
  uint32_t stop, kk;
  uint32_t fail, pad;
  const uint32_t* tau;
};
cudaError_t launch_sel_ctl(SelCtl* ctl, unsigned long long cstar, uint32_t kk, const uint32_t* tau, cudaStream_t s);
// MRIM selection (R27): pair ids t*n + u over `rounds` rounds, at most k picks per round
struct MrimSel {
  uint32_t rounds, n, k;
};
cudaError_t launch_select_persistent(uint32_t* cnt, uint32_t n, unsigned long long* keys, int kk,
                                     const InvSegDev* segs, const uint64_t* offsets, const uint32_t* pool,
                                     uint8_t* covered, const MrimSel* mr, bool limit, unsigned int* bar,
                                     int num_sms, cudaStream_t s);
cudaError_t launch_cover(const unsigned long long* keys, int j, const InvSegDev* segs, SelCtl* ctl,
                         const uint64_t* offsets, const uint32_t* pool,
                         uint8_t* covered, uint32_t* cnt, int32_t* dec, int grid, cudaStream_t s,
                         bool limit, const MrimSel* mr = nullptr);
// small graphs (P = 1): all k steps in one CTA, counts in shared memory (n <= select_cta_max_n())
uint32_t select_cta_max_n();
cudaError_t launch_select_cta(const uint32_t* count_total, uint32_t n, unsigned long long* keys, int kk,
                              const InvSegDev* segs, const uint64_t* offsets, const uint32_t* pool,
                              uint8_t* covered, SelCtl* ctl, bool limit, cudaStream_t s);
// mid-size graphs (P = 1): the same on a cluster of 2..8 CTAs, counts split over their shared
// memories (DSMEM atomics for the decrements)
uint32_t select_cluster_max_n();
cudaError_t launch_select_cluster(const uint32_t* count_total, uint32_t n, unsigned long long* keys, int kk,
                                  const InvSegDev* segs, const uint64_t* offsets, const uint32_t* pool,
                                  uint8_t* covered, SelCtl* ctl, bool limit, cudaStream_t s);
// fused greedy steps (P = 1): candidate argmax of step 0, then per step cover + next argmax
cudaError_t launch_select_fused(unsigned long long* keys, int kk, const InvSegDev* segs, const uint64_t* offsets,
                                const uint32_t* pool, uint8_t* covered, uint32_t* cnt, const uint32_t* cand,
                                const unsigned int* ncand, const uint32_t* tau_p1, unsigned int* done,
                                uint32_t* fail, int grid, cudaStream_t s, bool limit, int* launches);
// cooperative selection: one launch, one grid barrier per greedy step, redundant candidate argmax
constexpr uint32_t kCoopCands = 8192;   // most candidates of the cooperative selection
cudaError_t launch_select_coop(const uint32_t* cnt, const uint32_t* cand, const unsigned int* ncand,
                               const uint32_t* tau_p1, uint32_t* cmap, int32_t* cdec, unsigned long long* keys,
                               int kk, const InvSegDev* segs, const uint64_t* offsets, const uint32_t* pool,
                               uint8_t* covered, unsigned int* bar, uint32_t* fail, int num_sms, bool limit,
                               cudaStream_t s);
cudaError_t launch_validate_csr(const uint64_t* rp64, uint32_t n, uint64_t m, const uint32_t* src,
                                uint32_t* rp32, uint32_t* err, uint32_t* bad_row, uint32_t* thr_node, int grid,
                                cudaStream_t s, uint32_t v0, uint32_t v1);
// forward Monte-Carlo (mc.cu)
cudaError_t build_out_csr(const uint32_t* row_ptr, const uint32_t* src, uint32_t n, uint64_t m, int scheme,
                          uint32_t* out_ptr, uint32_t* out_dst, uint32_t* out_in, uint32_t* thr_wc,
                          void* tmp, size_t* tmp_bytes, uint64_t* scan_tmp, int grid, cudaStream_t s);
cudaError_t launch_mc_ic(int scheme, uint32_t n, const uint32_t* out_ptr, const uint32_t* out_dst,
                         const uint32_t* out_in, const uint32_t* thr_wc, const uint64_t* thr_edge,
                         uint64_t thr_uniform, const uint32_t* seeds, uint32_t k, uint64_t trials, uint64_t mc_seed,
                         unsigned long long* claim, uint32_t* sizes, uint32_t* bitmaps, uint32_t* queues,
                         uint64_t bm_words, int grid, cudaStream_t s, const uint32_t* row_ptr = nullptr,
                         unsigned long long* lt_accs = nullptr);   // lt_accs set: LT forward process
}  // namespace gim

/* gim.h — C ABI of the B200-native gIM/IMM hot path (libgim.so, sm_100a).
 *
 * The calls follow the problem statement of the paper (§2.3, Eq. 2): given
 * a graph G, influence probabilities p_uv, a diffusion model and k, find a seed set S with
 * |S| = k maximising E[I(S)]. The method is IMM's two steps as gIM accelerates them (Alg. 1,
 * P:178-198; Alg. 2): RR-set sampling (Alg. 3/6) and greedy
 * max-coverage NodeSelection (§3.8, Alg. 7). "P:n" = line n of the paper
 * (/root/reference/PAPER.md); "R1..R25" = readings of the paper listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Every call returns gim_status (GIM_OK = 0). On error gim_last_error(ctx) returns a
 *    NUL-terminated message owned by ctx, valid until the next call on ctx. No exceptions
 *    cross the ABI; no CPU fallback exists: without a usable CUDA device gim_create fails with
 *    GIM_ECUDA.
 *  - Node ids are dense uint32 in [0, n). Host arrays passed in are copied; the caller keeps
 *    ownership. Output arrays are caller-allocated host memory.
 *  - A ctx is bound to one device and one CUDA stream; it is not thread-safe. All device work
 *    is enqueued on the ctx stream, and every call returns after its results are host-visible.
 *  - The RR-set randomness is a pure function of (seed, RR id): Philox4x32-10 with key
 *    (seed_lo, seed_hi) and counter (id_lo, id_hi, slot_lo, slot_hi) (reading R16; DESIGN.md
 *    "RNG contract"), so every RR set is reproducible bit for bit on any number of GPUs.
 */
#ifndef GIM_H_
#define GIM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GIM_OK = 0,
  GIM_EINVAL = 1,      /* invalid argument (sizes, ranges, non-canonical CSR, k, eps, ell) */
  GIM_ESTATE = 2,      /* call not valid in the current state (no graph, empty pool)     */
  GIM_ENOMEM = 3,      /* device allocation failed                                        */
  GIM_ECUDA = 4,       /* CUDA runtime / kernel error, or no device                       */
  GIM_ECOLL = 5,       /* the all-reduce callback returned non-zero                       */
  GIM_ELTWEIGHT = 6    /* LT with explicit weights whose in-sum exceeds 1 at some node    */
} gim_status;

typedef enum { GIM_IC = 0, GIM_LT = 1 } gim_model;          /* PAPER.md §2.2 */
typedef enum { GIM_W_EXPLICIT = 0, GIM_W_WC = 1, GIM_W_UNIFORM = 2 } gim_weights;

typedef struct gim_ctx gim_ctx;   /* opaque; one per (process, device) */

/* Create a context on CUDA device `device`. cuda_stream is a cudaStream_t (may be NULL: the
 * library creates its own non-blocking stream). Errors: GIM_ECUDA (no device / bad id). */
gim_status gim_create(int device, void* cuda_stream, gim_ctx** out);

/* Free every device allocation of ctx and ctx itself. NULL is a no-op. */
void gim_destroy(gim_ctx* ctx);

/* Last error message of ctx (never NULL; "" after success). */
const char* gim_last_error(const gim_ctx* ctx);

/* Load the graph (§3.2 "Graph Representation", as an in-CSR: reading R14).
 *  in_row_ptr[n+1], in_src[m]: row v lists the sources u of edges u->v; canonical form is
 *    required — in_row_ptr[0] = 0, in_row_ptr[n] = m, non-decreasing; each row strictly
 *    ascending, every u < n, no u == v (reading R15). Violations: GIM_EINVAL.
 *  weights[m] (float32 in [0,1], slot-aligned with in_src) is required iff scheme ==
 *    GIM_W_EXPLICIT, else ignored. GIM_W_WC: p_uv = 1/d_in(v) (weighted cascade).
 *    GIM_W_UNIFORM: p_uv = p_uniform in [0,1] (IC only).
 *  model GIM_LT requires GIM_W_WC or GIM_W_EXPLICIT with sum_u w_uv <= 1 at every v
 *    (P:125), else GIM_ELTWEIGHT (or GIM_EINVAL for LT + uniform, reading R23).
 *  Limits: 1 <= n < 2^32 - 1, m < 2^32 - 256 (row pointers are held as uint32 on the device).
 * Replaces any previous graph and clears the RR pool; after an error no graph is loaded.
 * Validation and the row-pointer conversion run on the device (pinned host arrays are DMA'd). */
gim_status gim_load_graph(gim_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* in_row_ptr,
                          const uint32_t* in_src, const float* weights, gim_model model,
                          gim_weights scheme, float p_uniform);

/* Data-parallel sharding of RR ids (default rank 0 of 1). For any id range [a, b) this rank
 * generates and holds the contiguous slice [a + r(b-a)/P, a + (r+1)(b-a)/P) (integer floor).
 * Must be called before gim_generate_rr / gim_imm; clears the pool. GIM_EINVAL unless
 * 0 <= rank < world. */
gim_status gim_set_shard(gim_ctx* ctx, int rank, int world);

/* In-place SUM all-reduce over the world of int32 (two's complement) elements living in device
 * memory on the ctx device, enqueued on / ordered with cuda_stream. Returns 0 on success. Used
 * by gim_select when world > 1 (the count vector once, then one decrement
 * vector per greedy step). Required before gim_select/gim_imm when world > 1. */
typedef int (*gim_allreduce_fn)(void* dev_buf, uint64_t count, void* cuda_stream, void* user);
gim_status gim_set_allreduce(gim_ctx* ctx, gim_allreduce_fn fn, void* user);

/* All-gather over the world: every rank contributes `bytes` bytes of device memory at dev_send;
 * dev_recv (world * bytes, device) receives them in rank order; enqueued on / ordered with
 * cuda_stream; returns 0 on success. With world > 1 and an all-gather set, the library runs the
 * REPLICATED-POOL protocol (SURVEY.md §8(e) mitigation): each rank samples its slice of every
 * round's new RR ids, then the round's sets are all-gathered (one size exchange + two padded
 * all-gathers per generate call) so every rank holds the global pool in global id order, and
 * NodeSelection runs locally and identically on every rank with no per-step collective
 * (gim_set_allreduce is then unused). Without it, the per-step count/decrement all-reduce
 * protocol is used. gim_rr_export / gim_counts_export then return the global pool. */
typedef int (*gim_allgather_fn)(const void* dev_send, uint64_t bytes, void* dev_recv, void* cuda_stream,
                                void* user);
gim_status gim_set_allgather(gim_ctx* ctx, gim_allgather_fn fn, void* user);

/* Reduce-scatter over the world of int32 elements in device memory: dev_recv[recv_count] =
 * SUM over ranks r of their dev_send[rank * recv_count .. (rank + 1) * recv_count) for THIS
 * rank; enqueued on / ordered with cuda_stream; returns 0 on success. With world > 1, a
 * reduce-scatter and an all-reduce (and no all-gather) set, NodeSelection runs the
 * NODE-SHARDED protocol: nodes are split into world contiguous shards of
 * ceil(n / world); the local counts are reduce-scattered once, then per greedy step every rank
 * takes the argmax of its shard's global counts, the world's candidate keys are exchanged with
 * a 2*world-int32 SUM all-reduce (each rank fills only its own slot), the winner is covered in
 * the rank's local pool and its decrements are reduce-scattered to the shard owners — about
 * half the per-step bytes of the dense all-reduce protocol and no replicated pool. */
typedef int (*gim_reducescatter_fn)(void* dev_send, void* dev_recv, uint64_t recv_count, void* cuda_stream,
                                    void* user);
gim_status gim_set_reducescatter(gim_ctx* ctx, gim_reducescatter_fn fn, void* user);

/* Native NCCL exchange: instead of callbacks, the library issues the protocol's collectives
 * itself on its stream through an NCCL communicator it creates and owns (NCCL over NVLink /
 * NVSwitch; the libnccl.so.2 already loaded in the process, e.g. torch's, else the system's).
 * gim_nccl_unique_id fills a 128-byte ncclUniqueId on one rank; the caller broadcasts it; every
 * rank then calls gim_set_nccl collectively (after gim_set_shard; rank / world must match).
 * protocol: 0 = dense per-step all-reduce, 1 = replicated pool (all-gather), 2 = node-sharded
 * (reduce-scatter + all-reduce) — the same protocols as the callback hooks, same results.
 * GIM_ECOLL when NCCL cannot be loaded or the communicator cannot be created. */
gim_status gim_nccl_unique_id(void* id_out);
gim_status gim_set_nccl(gim_ctx* ctx, const void* id, int rank, int world, int protocol);

/* Route every device allocation of ctx through the caller (e.g. torch's caching allocator).
 * Must be called before gim_load_graph. alloc_fn returns NULL on failure. */
typedef void* (*gim_alloc_fn)(uint64_t bytes, void* cuda_stream, void* user);
typedef void (*gim_free_fn)(void* ptr, void* cuda_stream, void* user);
gim_status gim_set_allocator(gim_ctx* ctx, gim_alloc_fn alloc_fn, gim_free_fn free_fn,
                             void* user);

/* RR-set sampling (Alg. 1 l.3-4; Alg. 3/6). Afterwards the global pool is exactly
 * { RR(seed, i) : 0 <= i < theta } (reading R20), this rank holding its slices. Same seed and a
 * larger theta extends the pool (Alg. 2 reuses sets, reading R8); a smaller theta truncates;
 * a different seed discards and regenerates. RR(seed, i): root = floor(u64 * n / 2^64) with
 * u64 from Philox slot 2^63 (R17); IC keeps in-edge slot e iff coin(i, e) * 2^-32 < p_e where
 * coin = word (e & 3) of Philox slot (e >> 2) (R16); LT walks one in-edge per node chosen by
 * Philox slot 2^62 | v (R18-R19). Also maintains count[v] = #{local i : v in RR_i}
 * (Occur). Errors: GIM_ESTATE (no graph), GIM_ENOMEM, GIM_ECUDA. */
gim_status gim_generate_rr(gim_ctx* ctx, uint64_t theta, uint64_t seed);

/* Greedy max coverage over the current (global) pool, non-destructive (reading R9): k steps of
 * u_j = argmax_{v not in S} count[v] (ties -> lowest id, zero maximum allowed: R10), then
 * every uncovered RR set containing u_j is covered and count[w] -= 1 for each member (Alg. 7,
 * P:541-561; R11). seeds_out[k] required; gains_out[k] (marginal coverage) and covered_out
 * (sum of gains = |{i : S cap RR_i != {}}|) may be NULL. Errors: GIM_EINVAL (k < 1 or k > n),
 * GIM_ESTATE (empty pool / missing all-reduce), GIM_ENOMEM (also: the node -> RR index holds
 * 32-bit positions, so a rank's pool must stay below 2^32 - 1 elements), GIM_ECOLL, GIM_ECUDA. */
gim_status gim_select(gim_ctx* ctx, uint32_t k, uint32_t* seeds_out, uint64_t* gains_out,
                      uint64_t* covered_out);

/* IMM result / trace (reading R1-R8, R21). theta_i[r] are the round targets ceil(theta_i)
 * actually sampled, cov_i[r] the covered count of round r's selection over its sel_steps_i[r]
 * greedy steps. With GIM_OPT_IMM_EARLY_EXIT (default on) an estimation round's selection stops
 * at the first step j whose bound cov_j + (k - j) * gain_j (gains never increase) falls below
 * the smallest count that passes the round's test (Alg. 2 l.7): the round fails either way, so
 * LB, theta, R_final and the seeds are unchanged; then sel_steps_i[r] < k (k * T in MRIM mode)
 * and cov_i[r] is the covered count of those steps. */
typedef struct {
  double ell_eff, eps_prime, lambda_prime, lambda_star, LB, theta;
  uint32_t rounds;
  uint64_t theta_i[64], cov_i[64];
  double theta_i_real[64];
  uint64_t R_final;
  uint64_t covered;
  double spread_est;   /* n * covered / R_final (Eq. 3) */
  uint32_t sel_steps_i[64];
} gim_imm_result;

/* Full IMM (Alg. 2 bootstrap of LB, then theta = lambda_star / LB and the final NodeSelection):
 * starts from an empty pool. seeds_out[k] required; res may be NULL. GIM_EINVAL unless n >= 2,
 * 1 <= k <= n, 0 < eps < 1, ell > 0 (reading R25). */
gim_status gim_imm(gim_ctx* ctx, uint32_t k, double eps, double ell, uint64_t seed,
                   uint32_t* seeds_out, gim_imm_result* res);

/* Parity/debug export of this rank's local slice (caller-allocated; pass NULL buffers to query
 * n_sets / pool_len only). ids_out[n_sets]: global RR id of each local set; offsets_out
 * [n_sets+1]: local offsets into nodes_out[pool_len]. sort_each_set != 0 sorts every set
 * ascending (the device stores sets in discovery order, which is not part of the contract). */
gim_status gim_rr_export(gim_ctx* ctx, uint64_t* n_sets, uint64_t* pool_len, uint64_t* ids_out,
                         uint64_t* offsets_out, uint32_t* nodes_out, int sort_each_set);

/* count_out[n] (n*T in MRIM mode, indexed by pair id): this rank's local occurrence counts
 * (Occur). */
gim_status gim_counts_export(gim_ctx* ctx, uint32_t* count_out);

/* Forward Monte-Carlo spread (verification at scale): `trials` independent runs of the
 * diffusion. IC: each newly active node tries each out-edge once; the coin of
 * out-slot e (out-CSR rows sorted by (source, in-slot)) in trial t is word (e & 3) of
 * Philox(mc_seed; t, tag 11 | e >> 2). LT (Eq. 1; reading R30): tau_v = (o + 1/2)/2^32
 * with o = word 0 of Philox(mc_seed; t, tag 11 | 2^40 | v), compared exactly (WC: active
 * in-neighbours * 2^33 >= (2o + 1) d_in(v); explicit: sum of floor(w 2^32) >= o + 1); trials <
 * 2^24 - 1. Both are independent of every RR stream. mean_out = mean number
 * of activated nodes (seeds included, duplicates once), stderr_out (nullable) its standard error,
 * sizes_out[trials] (nullable) the per-trial counts. Builds the out-CSR on first use. Compared
 * with n * F_R'(S) on an independent RR pool it checks Eq. 3 at full size.
 * Errors: GIM_ESTATE (no graph), GIM_EINVAL (k == 0, trials == 0, seed >= n). */
gim_status gim_mc_spread(gim_ctx* ctx, const uint32_t* seeds, uint32_t k, uint64_t trials, uint64_t mc_seed,
                         double* mean_out, double* stderr_out, uint32_t* sizes_out);

/* Multi-round IM (MRIM), the CR-NAIMM algorithm as gIM adapts it (§4.8: "after
 * selecting a random node, we initiate a random BFS originating from the selected node as many
 * times as the number of rounds. Also, each element in a random RR set is a tuple of node-id and
 * round number"). rounds = T >= 1 (T = 1, the default, is standard IM); discards the pool.
 * Readings:
 *  R26 MRIM set i = {(u, t) : 0 <= t < T, u in RR^t_i}: the T rounds share root(seed, i) and
 *      round t draws the coins of standard RR id i*T + t; the pair (u, t) is the element id
 *      t*n + u. In MRIM mode theta (gim_generate_rr) counts MRIM sets; gim_rr_export returns the
 *      T*theta per-round sets (ids i*T + t) whose members are pair ids.
 *  R27 gim_select(k): k seeds PER ROUND, k*T picks in greedy order: the unselected pair of a
 *      round with fewer than k seeds with the largest count, ties -> lowest pair id;
 *      seeds_out[k*T] / gains_out[k*T] hold pair ids (round = id / n, node = id % n).
 *  R28 gim_imm(k): IMM with ln C(n*T, k*T) in lambda' and lambda*; seeds_out[k*T] pair ids;
 *      R_final / theta count MRIM sets.
 * GIM_EINVAL if T == 0 or n*T >= 2^32 - 1 (pair ids are uint32, 2^32 - 1 is a sentinel). */
gim_status gim_set_rounds(gim_ctx* ctx, uint32_t rounds);

/* Tunables (test / ablation hooks; the defaults are the tuned configuration):
 *  GIM_OPT_FORCE_GIANT  = 1: every RR set goes through the block-per-RR giant kernel.
 *  GIM_OPT_QUEUE_CAP    = Q: shared-memory queue capacity per RR (power of two, 32..1024);
 *                          sets larger than Q are replayed by the giant kernel.
 *  GIM_OPT_PROFILE      = 1: time every kernel class with CUDA events (see gim_get_stats).
 *  GIM_OPT_STAGING_CAP  = elements of staging memory to start from (forces retries if tiny).
 *  GIM_OPT_SELECT_GRAPH = 1 (default): for P = 1 replay the 2k argmax/cover launches of a
 *                          NodeSelection from captured CUDA graphs of consecutive steps ([0, 8),
 *                          [8, 32), [32, k); a bounded greedy checks its stop flag between them;
 *                          with gim_set_nccl also the P > 1 step loops); 0: launch them one by one.
 *  GIM_OPT_INV_SEGMENTS = 1 (default): the sets generated since the last selection are indexed
 *                          as one new inverted-index segment when a selection needs them (rounds
 *                          settled by gim_imm's probe are merged into the next segment); 0:
 *                          rebuild one index over the whole pool at every selection (ablation).
 *  GIM_OPT_ARGMAX_CAND  = 1 (default): for P = 1 and n >= 2^20 the per-step argmax scans a candidate list of
 *                          <= 65536 nodes (count >= a power-of-two threshold tau; counts only
 *                          decrease, so a best candidate >= tau is the argmax over all nodes); a
 *                          step whose best candidate is below tau fails the selection, which is
 *                          redone with full scans (gim_stats.fused_fallbacks); 0: always full;
 *                          2: candidates whatever n (tests).
 *  GIM_OPT_IC_LANE      = -1 (default): IC sampling starts with the lane-per-set kernel when the
 *                          running mean of coins per set is below 160 (tiny sets) and the chunk
 *                          has >= 131072 sets, else the warp kernel; 1: always lane-first;
 *                          0: never. Results are identical.
 *  GIM_OPT_SPECULATE    = 0 (default) / 1: inside gim_imm, sample the next round's RR ids on a
 *                          second stream while a round's NodeSelection runs (capped at the
 *                          largest theta the LB test can yield; excess is truncated). Results
 *                          are identical; measured slower on C4 and neutral on C3.
 *  GIM_OPT_PDL          = 0 (default) / 1: launch the argmax / cover kernels of the greedy steps
 *                         with programmatic dependent launch (each kernel's CTAs become resident
 *                         while its predecessor runs and wait for its results). Process-wide.
 *  GIM_OPT_GIANT_NT     = 0 (default, auto) / 256 / 128: threads per giant-set CTA of the
 *                         block-per-RR fallback (auto: 128 when the previous chunk produced >= 12
 *                         giant sets per 256-thread slot, else 256).
 *  GIM_OPT_FRESH_FINAL  = 0 (default: IMM's published reuse of the estimation sets, R8) / 1:
 *                         gim_imm's final phase samples a fresh pool of ceil(theta) sets with the
 *                         key seed ^ 0x9E3779B97F4A7C15 (reading R29; the Chen 2018 fix [EXT]).
 *  GIM_OPT_SELECT_PERSISTENT = 0 (default) / 1: for P = 1 (or a replicated pool) run the k
 *                         greedy steps of a selection in one cooperative launch with grid
 *                         barriers between the argmax and cover phases (no candidate list).
 *  GIM_OPT_MB_CHAINS    = 1 / 4 / 8 (default 8): interleaved Philox chains per thread in
 *                          gim_microbench_philox.
 *  GIM_OPT_SKIP         = 0 (default: one Philox coin per in-edge, reading R16) / 1: the
 *                         geometric-skip RNG contract (reading R31): the live in-edges
 *                         of a visited node v are drawn as geometric gaps, blocks of 1024 in-edge
 *                         offsets, draw j of block b = word (j & 3) of Philox(seed; id_lo, 2^31|b,
 *                         v, j >> 2), gap = floor(ln((r + 1/2) 2^-32) / ln(1 - p)). Same
 *                         distribution of RR sets (Bernoulli(p) per in-edge), different sets: the
 *                         pool restarts. IC with WC or uniform weights only (GIM_EINVAL otherwise;
 *                         a later gim_load_graph of another model/scheme turns it off).
 *  GIM_OPT_SPILL        = S (-1 = auto: under GIM_OPT_SKIP 16384 for WC and 2048 for uniform p,
 *                         0 with per-edge coins; else 0..16384): IC sets that outgrow the warp
 *                         kernel's shared queue continue in the warp's global spill tier up to
 *                         S nodes (S <= the queue capacity: no spill tier), beyond that in the
 *                         CTA-per-set giant kernel. Results are identical.
 *  GIM_OPT_SELECT_FUSED = C (default 0 = off; e.g. 2048): for P = 1 (standard IM, no speculation),
 *                         each greedy step is ONE launch: the cover of pick j, then the last CTA
 *                         to finish computes pick j+1 over the <= C nodes whose initial count
 *                         reaches a threshold tau (counts only decrease, so a best candidate
 *                         count >= tau certifies the global argmax); an uncertified step makes
 *                         the selection rerun unfused (gim_stats.fused_fallbacks). Results are
 *                         identical; measured 4.48 vs 4.23 ms per C3 selection set (off).
 *  GIM_OPT_FUSED_CTAS   = c (default 2, 1..16): CTAs per SM of the fused step kernel.
 *  GIM_OPT_FORCE_COLLECTIVES = 1: run the world > 1 exchange protocol selected by the hooks even
 *                         at world = 1 (test hook: drives the NCCL callbacks on one GPU).
 *  GIM_OPT_GIANT_SHARED = 0 (default) / 1: giant sets (outgrowing the warp queue) first go through
 *                         a block-per-set pass with the queue and visited hash in shared memory
 *                         (sets up to 4096 nodes); larger ones continue in the global-bitmap pass.
 *                         Results are identical; measured neutral on C3 (giant 3.07 vs 3.03 ms).
 *  GIM_OPT_SKIP_LANE_CAP = L (default 32, 1..512): under GIM_OPT_SKIP, the lane-per-set kernel keeps
 *                         sets of up to L nodes (32 in shared memory, the rest in a per-lane
 *                         global spill); larger sets escalate to the warp kernel. Results are
 *                         identical; measured C3 sampling 7.5 / 11.7 / 18.4 / 29.6 / 61.9 ms at
 *                         L = 32 / 96 / 160 / 256 / 512 (a long set holds its whole warp).
 *  GIM_OPT_SELECT_COOP  = C (0 = off; 1..8192): for P = 1 (standard IM, no speculation) run the k
 *                         greedy steps of a selection in ONE cooperative launch with one grid
 *                         barrier per step: every CTA takes the argmax redundantly over the <= C
 *                         candidates whose initial count reaches tau (certified: counts only
 *                         decrease), and the cover accumulates only the candidates' decrements;
 *                         an uncertified step makes the selection rerun with the default
 *                         kernels (gim_stats.fused_fallbacks). Results are identical; measured
 *                         slower (C3 selection 5.85 / 6.87 ms at C = 2048 / 8192 vs 4.28 ms, no
 *                         fallbacks): the grid barrier costs more than the launch it replaces.
 *  GIM_OPT_IMM_EARLY_EXIT = 1 (default) / 0: bounded greedy in gim_imm's estimation rounds (see
 *                         gim_imm_result.sel_steps_i); 0 runs every round's k steps.
 *  GIM_OPT_INV_PASSES   = P (0 = default 1, 1..64): the inverted-index scatter runs P node-range
 *                         passes over the new sets so each pass's cursor atomics stay in the L2
 *                         (results identical; measured slower on C5: 6.19 vs 5.66 ms at P = 6).
 *  GIM_OPT_L2_PERSIST   = 0 (default) / 1: an L2 persisting access-policy window on the library
 *                         stream over the row pointers (+ WC thresholds), read at every BFS level
 *                         (measured: C3 neutral; C5 store 3.8 -> 5.9 ms, index 6.2 -> 10.5 ms).
 *  GIM_OPT_SELECT_CTA   = 1 (default) / 0: for P = 1 (or a replicated pool), standard IM and
 *                         n <= 51,200 (the counts fit in 200 KB of shared memory), the k greedy
 *                         steps run in ONE 1024-thread CTA: argmax over shared counts, decrements
 *                         as shared atomics, no launch or grid barrier per step.
 *  GIM_OPT_INV_SORT     = -1 (default: auto, when n * 4 > 64 MB) / 0 / 1: build each index
 *                         segment by a stable radix sort of its (node, set) pairs by node instead
 *                         of the cursor scatter (lists in ascending set order; same lists).
 *  GIM_OPT_CHUNK        = ids (0 = default 2^25; 1024..2^25): RR ids sampled per generation chunk
 *                         (one K-RR / K-GIANT / store pass each; results identical).
 *  GIM_OPT_SELECT_CLUSTER = 0 (default) / 1: with GIM_OPT_SELECT_CTA, graphs of 51,200 < n <=
 *                         409,600 run the k greedy steps in one launch on a thread-block cluster of
 *                         2..8 CTAs whose shared memories hold the counts (DSMEM exchange of the
 *                         partial argmaxes, DSMEM atomics for the decrements). Results identical;
 *                         measured slower on C2 (selection 5.31 vs 1.16 ms): a few SMs cannot
 *                         carry the covers of a 358K-set pool, which the graph path spreads over
 *                         all 148.
 *  GIM_OPT_IMM_LOOKAHEAD = 1 (default) / 0: in gim_imm, after a round the probe settled (bound
 *                         fraction u = k gain_0 / T_i), the following rounds whose passing fraction
 *                         (1 + eps') / 2^m exceeds u / 1.2 are sampled in the same generate call and
 *                         probed on the counts of their own prefix of T_m sets; a round the probe
 *                         does not settle truncates the pool to its T_m (gim_stats.lookahead_drops).
 *                         The trace, LB, theta, R_final and the seeds are unchanged. 2: two rounds
 *                         ahead whatever u (tests: exercises the drop path). */
typedef enum {
  GIM_OPT_FORCE_GIANT = 1,
  GIM_OPT_QUEUE_CAP = 2,
  GIM_OPT_PROFILE = 3,
  GIM_OPT_STAGING_CAP = 4,
  GIM_OPT_SELECT_GRAPH = 6,
  GIM_OPT_INV_SEGMENTS = 7,
  GIM_OPT_ARGMAX_CAND = 8,
  GIM_OPT_IC_LANE = 9,
  GIM_OPT_SPECULATE = 10,
  GIM_OPT_MB_CHAINS = 11,
  GIM_OPT_PDL = 12,
  GIM_OPT_GIANT_NT = 13,
  GIM_OPT_FRESH_FINAL = 14,
  GIM_OPT_SELECT_PERSISTENT = 15,
  GIM_OPT_SKIP = 16,
  GIM_OPT_SPILL = 17,
  GIM_OPT_SELECT_FUSED = 18,
  GIM_OPT_FUSED_CTAS = 19,
  GIM_OPT_FORCE_COLLECTIVES = 20,
  GIM_OPT_GIANT_SHARED = 21,
  GIM_OPT_SKIP_LANE_CAP = 22,
  GIM_OPT_SELECT_COOP = 23,
  GIM_OPT_IMM_EARLY_EXIT = 24,
  /* 25: retired (conditional IF-node selection graph; measured slower) */
  GIM_OPT_INV_PASSES = 26,
  GIM_OPT_L2_PERSIST = 27,
  GIM_OPT_SELECT_CTA = 28,
  GIM_OPT_INV_SORT = 29,
  GIM_OPT_CHUNK = 30,
  GIM_OPT_SELECT_CLUSTER = 31,
  GIM_OPT_IMM_LOOKAHEAD = 32
} gim_option;
gim_status gim_set_option(gim_ctx* ctx, gim_option opt, int64_t value);

/* Counters since the last gim_reset_stats. Kernel times (ms, CUDA events on the ctx stream)
 * are only collected with GIM_OPT_PROFILE = 1. gim_imm time counts once (its inner
 * generate/select calls are internal). */
typedef struct {
  uint64_t launches;          /* kernels launched by the library                      */
  uint64_t rr_sets;           /* RR sets generated (local)                             */
  uint64_t rr_elements;       /* pool elements appended (local)                        */
  uint64_t giant_sets;        /* sets replayed by the giant kernel                     */
  uint64_t coins;             /* in-edge slots examined (IC) / draws (LT), warp kernel */
  uint64_t live_edges;        /* live in-edges found, warp kernel                      */
  uint64_t coins_giant;       /* same, giant kernel                                    */
  uint64_t live_giant;
  uint64_t selects;           /* NodeSelection calls                                   */
  uint64_t allreduces;        /* all-reduce callback invocations                       */
  double ms_rr, ms_giant, ms_store, ms_inv, ms_select; /* kernel time per class        */
  uint64_t n_rr_launches, n_giant_launches;
  uint64_t n_syncs, n_allocs;   /* host<->device syncs, device allocations                */
  double host_ms_sync;          /* host wall time blocked in stream synchronisation       */
  double host_ms_api;           /* host wall time inside gim_generate_rr/select/imm       */
  uint64_t fused_fallbacks;     /* fused selections redone unfused (uncertified argmax)   */
  uint64_t probe_stops;         /* gim_imm rounds settled by the first-step probe alone   */
  uint64_t lookahead_drops;     /* lookahead sets dropped because a round needed selection */
} gim_stats;
gim_status gim_get_stats(gim_ctx* ctx, gim_stats* out);
gim_status gim_reset_stats(gim_ctx* ctx);

/* Diagnostic: time `groups` Philox4x32-10 slot-group evaluations (4 coins each, the per-group
 * ALU work of the IC kernel without memory traffic) on the ctx stream; *ms = kernel time. Used
 * to check the ALU roofline of the sampling kernel. */
gim_status gim_microbench_philox(gim_ctx* ctx, uint64_t groups, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* GIM_H_ */

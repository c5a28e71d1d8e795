// gim_device.cuh — device-side building blocks of libgim (sm_100a).
//
// Philox4x32-10 and the (seed; RR id, slot) key scheme (reading R16, DESIGN.md "RNG
// contract"), kernel parameter blocks and launch wrappers shared by rr.cu / select.cu /
// gim_api.cu. Independent of oracle/ (no shared code; both sides are pinned separately to the
// Random123 known-answer vectors).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gim {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr uint32_t kEmpty = 0xFFFFFFFFu;   // empty hash slot / "no node"
constexpr uint32_t kSent = 0xFFFFFFFFu;    // count sentinel of an already-selected node

enum { MODEL_IC = 0, MODEL_LT = 1 };
enum { W_EXPLICIT = 0, W_WC = 1, W_UNIFORM = 2 };

// Slot tags of the counter's high word.
constexpr uint32_t kSlotRootHi = 0x80000000u;   // 2^63: root draw
constexpr uint32_t kSlotLtHi = 0x40000000u;     // 2^62 | v: LT in-edge draw at node v

// Philox4x32-10 (Salmon et al. SC'11): 10 rounds, key bumped after every round.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Same, with the 20 round keys precomputed (rk[2r], rk[2r+1] = key of round r): kernels pass
// them in the parameter (constant) bank so every key XOR is one LOP3 with a constant operand.
__device__ __forceinline__ uint4 philox4x32_10_rk(uint4 c, const uint32_t* rk) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ rk[2 * r], lo1, hi0 ^ c.w ^ rk[2 * r + 1], lo0);
  }
  return c;
}

// N independent Philox4x32-10 evaluations interleaved round by round (same key): each round key
// is fetched once for all N states and the N dependency chains give the scheduler ILP.
template <int N>
__device__ __forceinline__ void philox4x32_10_rk_xn(uint4 (&c)[N], const uint32_t* rk) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t ka = rk[2 * r], kb = rk[2 * r + 1];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const uint32_t lo0 = 0xD2511F53u * c[i].x, hi0 = __umulhi(0xD2511F53u, c[i].x);
      const uint32_t lo1 = 0xCD9E8D57u * c[i].z, hi1 = __umulhi(0xCD9E8D57u, c[i].z);
      c[i] = make_uint4(hi1 ^ c[i].y ^ ka, lo1, hi0 ^ c[i].w ^ kb, lo0);
    }
  }
}

// Lane k (0..31) whose half-open range [P_{k-1}, P_k) contains i, given inclusive prefixes
// P_k held per lane (non-decreasing; i < P_31). Warp-collective.
__device__ __forceinline__ uint32_t warp_owner(uint32_t P, uint32_t i) {
  uint32_t k = 0;
#pragma unroll
  for (uint32_t step = 16; step >= 1; step >>= 1) {
    const uint32_t pv = __shfl_sync(kFull, P, k + step - 1);
    if (pv <= i) k += step;
  }
  return k;
}

// Root of RR set `id`: floor(u64 * n / 2^64), u64 = out0 | out1 << 32 of slot 2^63
// ("u = randSelect(V)", Alg. 3 l.5; reading R17).
__device__ __forceinline__ uint32_t rr_root(uint64_t seed, uint64_t id, uint32_t n) {
  const uint4 o = philox4x32_10(make_uint4((uint32_t)id, (uint32_t)(id >> 32), 0u, kSlotRootHi),
                                (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint64_t u64 = (uint64_t)o.x | ((uint64_t)o.y << 32);
  return (uint32_t)__umul64hi(u64, (uint64_t)n);
}

// MRIM (reading R26, §4.8): the T rounds of MRIM set i are standard RR ids i*T + t that
// share the root of id i ("after selecting a random node, we initiate a random BFS originating
// from the selected node as many times as the number of rounds"). rounds = 1: standard IM.
__device__ __forceinline__ uint32_t rr_root_of(uint64_t seed, uint64_t id, uint32_t n, uint32_t rounds) {
  return rr_root(seed, rounds > 1u ? id / rounds : id, n);
}

// Device counters of one generation launch sequence (zeroed by the host per chunk).
struct GenCounters {
  unsigned long long stage_tail;   // staging bump allocator (elements)
  unsigned long long coins;        // in-edge slots examined / LT draws
  unsigned long long live;         // live in-edges found
  unsigned long long coins_giant;  // same, giant kernel
  unsigned long long live_giant;
  unsigned long long dump_tail;    // partial-BFS dump allocator (elements)
  unsigned int claim;              // warp-kernel work claim
  unsigned int claim_lane;         // lane-kernel work claim
  unsigned int esc_count;          // sets escalated by the lane kernel to the warp kernel
  unsigned int claim_giant;        // giant-kernel work claim
  unsigned int giant_count;        // ids pushed to the giant list
  unsigned int retry_count;        // ids whose staging write did not fit
  unsigned int giant2_count;       // sets the shared-memory giant pass handed to the global pass
  unsigned int claim_giant2;       // global giant pass work claim
  unsigned long long dbg[4];       // GIM_WINSTAT builds: K-RR flattened windows / valid groups / hub steps
};

// A set handed from the warp kernel to the giant kernel: the warp's partial BFS (queue
// q[0..qlen) of which q[0..head) are fully expanded) is dumped at dump[dump_off..] so the giant
// kernel resumes instead of replaying. qlen == 0: start from the root.
struct GiantRec {
  uint32_t item, qlen, head, pad;
  unsigned long long dump_off;
};

// One segment of the inverted node -> RR index (built per generate call): the local set ids
// containing v are inv[end[v-1] .. end[v]) (end[-1] = 0). 32-bit: a segment holds < 2^32 elements.
struct InvSegDev {
  const uint32_t* end;
  const uint32_t* inv;
};
constexpr int kMaxInvSeg = 16;

// Parameters of the RR-generation kernels.
struct RRParams {
  uint32_t n;
  const uint32_t* row_ptr;     // in-CSR row pointers (uint32, m < 2^32)
  const uint32_t* src;         // in-CSR sources
  const uint32_t* thr_node;    // WC: per-node live threshold floor((2^32-1)/d_in(v))
  const uint64_t* thr_edge;    // explicit weights: IC ceil(w*2^32), LT floor(w*2^32)
  uint64_t thr_uniform;        // uniform p: ceil(p*2^32)
  float p_uniform;             // uniform p itself (geometric-skip contract, R31)
  const double* skip_tab;      // R31: L_k[184], R_k[184], then inv[d] (WC: d = 0..max_deg; uniform: inv[0])
  uint64_t seed;
  uint32_t rk[20];             // Philox round keys of `seed` (host-computed)
  uint64_t id_base;            // global RR id = id_base + item
  uint32_t count;              // items to process
  const unsigned int* count_ptr;   // if set, the item count is read here (device-produced lists)
  uint32_t* esc_list;          // IC lane kernel: items escalated to the warp kernel
  const uint32_t* item_list;   // nullptr: items are 0..count-1; else item = item_list[i]
  uint32_t* sizes;             // [chunk] RR size per item
  uint64_t* soff;              // [chunk] staging offset per item
  uint32_t* staging;
  uint64_t stage_cap;
  GenCounters* ctr;
  GiantRec* giant_recs;        // sets handed to the giant kernel
  GiantRec* giant2_recs;       // sets the shared-memory giant pass hands to the global pass
  int giant_pass2;             // the global giant pass reads giant2_recs (after the shared pass)
  uint32_t* dump;              // partial-BFS dumps
  uint64_t dump_cap;
  uint32_t* retry_list;        // items whose staging write failed
  uint32_t qcap;               // shared-memory queue capacity (<= kQMax)
  uint32_t* lt_spill;          // LT: per-warp spill of walks longer than kLtCap (lane-interleaved)
  uint32_t* spill;             // warp kernels: per-warp global queue + hash for sets > qcap
  uint32_t spill_cap;          // sets beyond this many nodes go to the CTA giant kernel (<= qcap: no spill)
  uint32_t* lane_spill;        // R31 lane kernel: per-lane global members beyond the shared 32
  uint32_t lane_cap;           // R31 lane kernel: set size limit (then escalate to the warp kernel)
  int force_giant;
  uint32_t rounds;             // MRIM rounds T (1 = standard IM): root of id = root(id / T)
};

// Shared-memory layout of the warp-per-RR kernel.
constexpr int kRRWarps = 8;          // warps per CTA
#ifndef GIM_QMAX
#define GIM_QMAX 512
#endif
#ifndef GIM_HSIZE
#define GIM_HSIZE 1024
#endif
constexpr int kQMax = GIM_QMAX;      // queue capacity (the queue doubles as the RR buffer)
constexpr int kHSize = GIM_HSIZE;    // visited hash slots (load <= (Q + 128) / H)
#ifndef GIM_PEND
#define GIM_PEND 128
#endif
// pending live in-edges of the batch being expanded (their src copies in flight, cp.async);
// >= 128 = the most one warp step can find (32 lanes x 4 slots)
constexpr int kPend = GIM_PEND;
static_assert(kPend >= 128, "one warp step can find 128 live slots");
constexpr int kRRSmemPerWarp = (kQMax + kHSize + kPend) * 4;   // 6.5 KB -> 4 CTAs x 8 warps per SM
#ifndef GIM_RR_BLOCKS
#define GIM_RR_BLOCKS 4
#endif
constexpr int kRRBlocksPerSM = GIM_RR_BLOCKS;
#ifndef GIM_HUB_ILP
#define GIM_HUB_ILP 2
#endif
constexpr int kHubIlp = GIM_HUB_ILP;  // Philox chains per lane per step on a hub node
constexpr uint32_t kHubGroups = 32u * GIM_HUB_ILP;   // nodes with >= this many slot groups are hubs
static_assert((kHubGroups & (kHubGroups - 1u)) == 0u, "hub steps are split off with a mask");
#ifndef GIM_GIANT_THREADS
#define GIM_GIANT_THREADS 256
#endif
constexpr int kGiantThreads = GIM_GIANT_THREADS;              // warps of one giant set = this / 32
constexpr int kGiantBlocksPerSM = 1024 / GIM_GIANT_THREADS;   // giant sets in flight per SM
// Narrow giant CTAs (8 giant sets in flight per SM, 4 warps each) for chunks with many giant sets
// per slot (dense graphs: BA r >= 16); chosen per chunk from the previous chunk's giant count.
constexpr int kGiantThreadsNarrow = 128;
#ifndef GIM_CLAIM_BATCH
#define GIM_CLAIM_BATCH 1
#endif
#ifndef GIM_CLAIM_TAIL_DIV
#define GIM_CLAIM_TAIL_DIV 4
#endif
constexpr uint32_t kClaimBatch = GIM_CLAIM_BATCH;       // RR ids claimed per warp per atomic
constexpr uint32_t kClaimTailDiv = GIM_CLAIM_TAIL_DIV;  // last count/div ids claimed one by one
constexpr uint32_t kStageChunk = 1024;    // staging elements reserved per warp per atomic
constexpr int kLtWarps = 8;          // K-LT: warps per CTA
#ifndef GIM_LT_CAP
#define GIM_LT_CAP 64
#endif
constexpr int kLtCap = GIM_LT_CAP;   // K-LT: path entries per lane in shared memory
constexpr int kLtCap2 = 512;         // K-LT: max path per lane (shared + global spill)
constexpr int kIcLaneWarps = 8;      // K-IC lane kernel: warps per CTA
#ifndef GIM_LANE_BLOCKS
#define GIM_LANE_BLOCKS 5   // C5 lane sampling 10.12 / 9.67 / 9.63 ms at 4 / 5 / 6 (latency-bound: more sets in flight)
#endif
constexpr int kIcLaneBlocksPerSM = GIM_LANE_BLOCKS;   // K-IC lane kernel: resident CTAs per SM
constexpr int kIcLaneCap = 32;       // K-IC lane kernel: set size limit (then escalate)
constexpr uint32_t kIcLaneMaxDeg = 256;   // K-IC lane kernel: in-degree limit (then escalate)
constexpr int kGiantWin = 2048;      // frontier window of the giant kernel (smem)

// Spill tier of the warp-per-set kernels (K-RR and the R31 warp kernel): a set that outgrows the
// shared-memory queue continues in its warp's global queue gq (kSpillQ entries) and open-
// addressing hash gh (kSpillH slots, kEmpty when unused, L2-resident) instead of being handed to
// the CTA-per-set giant kernel: giant sets then run beside the small ones.
constexpr uint32_t kSpillQ = 16384;
constexpr uint32_t kSpillH = 32768;          // power of two
__device__ __forceinline__ bool spill_hash_insert(uint32_t* gh, uint32_t u) {
  uint32_t s = (u * 0x9E3779B1u) >> 17;       // top 15 bits: kSpillH = 2^15 slots
  while (true) {
    const uint32_t old = atomicCAS(&gh[s], kEmpty, u);
    if (old == kEmpty) return true;
    if (old == u) return false;
    s = (s + 1) & (kSpillH - 1u);
  }
}
// walk from u's home slot to the slot holding it (holes left by members erased before cannot
// stop the walk: it compares against u, not against empty)
__device__ __forceinline__ void spill_hash_erase(uint32_t* gh, uint32_t u) {
  uint32_t s = (u * 0x9E3779B1u) >> 17;
  while (atomicCAS(&gh[s], u, kEmpty) != u) s = (s + 1) & (kSpillH - 1u);
}

}  // namespace gim

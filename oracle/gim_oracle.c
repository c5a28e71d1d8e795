/* oracle/gim_oracle.c — the parity ORACLE for the gIM / IMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing outside tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this code. It shares no code, header,
 * table or constant generator with the CUDA library (paper_2009_07325_b200/); neither side
 * includes or links the other. Inputs come from gim_inputs/ (graph generator, no method
 * arithmetic).
 *
 * A plain, slow, obviously-correct, single-threaded implementation of what the GPU path must
 * reproduce bit for bit. Citations: "P:n" = /root/reference/PAPER.md line n (gIM paper,
 * arXiv 2009.07325); "O1..O9" and "R1..R25" = SURVEY.md §8(c) oracle steps and readings
 * (restated in DESIGN.md). Parity status of every function: pinned (see tests/test_oracle_*.py
 * and DESIGN.md "Oracle pins"); none is "parity unpinned".
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared gim_oracle.c -lm  (no -ffast-math)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------
 * O2. Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as 1, 2, 3").
 * The paper only says "p = U(0,1)" (Alg. 3 l.18) — reading R16 fixes the generator.
 * ------------------------------------------------------------------------------------------ */
void og_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  int r;
  for (r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Key scheme (O2): key = (seed_lo, seed_hi); counter = (id_lo, id_hi, s_lo, s_hi). */
static void keyed(uint64_t seed, uint64_t id, uint64_t slot, uint32_t out[4]) {
  uint32_t ctr[4], key[2];
  ctr[0] = (uint32_t)id;   ctr[1] = (uint32_t)(id >> 32);
  ctr[2] = (uint32_t)slot; ctr[3] = (uint32_t)(slot >> 32);
  key[0] = (uint32_t)seed; key[1] = (uint32_t)(seed >> 32);
  og_philox(ctr, key, out);
}

#define SLOT_ROOT (((uint64_t)1) << 63)          /* tag 10 */
#define SLOT_LT (((uint64_t)1) << 62)            /* tag 01 */
#define SLOT_MC (((uint64_t)3) << 62)            /* tag 11: oracle-only forward Monte-Carlo */

/* O3. root_i = floor(u64 * n / 2^64) — "u = randSelect(V)" (Alg. 3 l.5; reading R17). */
uint32_t og_root(uint64_t seed, uint64_t id, uint32_t n) {
  uint32_t o[4];
  uint64_t u64;
  keyed(seed, id, SLOT_ROOT, o);
  u64 = (uint64_t)o[0] | ((uint64_t)o[1] << 32);
  return (uint32_t)(((unsigned __int128)u64 * (unsigned __int128)n) >> 64);
}

/* O4. coin(i, e) = word (e & 3) of Philox(seed; i, e >> 2). */
uint32_t og_coin(uint64_t seed, uint64_t id, uint64_t e) {
  uint32_t o[4];
  keyed(seed, id, e >> 2, o);
  return o[e & 3];
}

/* LT draw at node v (O5). */
uint32_t og_lt_draw(uint64_t seed, uint64_t id, uint32_t v) {
  uint32_t o[4];
  keyed(seed, id, SLOT_LT | (uint64_t)v, o);
  return o[0];
}

/* ------------------------------------------------------------------------------------------
 * Context: graph (O1) + pool (O6).
 * ------------------------------------------------------------------------------------------ */
enum { OG_IC = 0, OG_LT = 1 };
enum { OG_W_EXPLICIT = 0, OG_W_WC = 1, OG_W_UNIFORM = 2 };

typedef struct og_ctx {
  uint32_t n;
  uint64_t m;
  uint64_t* row_ptr;      /* in-CSR, n+1 */
  uint32_t* src;          /* m */
  float* w;               /* m or NULL */
  int model, scheme;
  float p_uniform;
  uint64_t thr_uniform;   /* ceil(p * 2^32) */
  uint64_t* thr_edge;     /* explicit IC: ceil(w_e * 2^32); explicit LT: floor(w_e * 2^32) */
  /* out-CSR for the forward Monte-Carlo check only */
  uint64_t* out_ptr;
  uint32_t* out_dst;
  uint64_t* out_in_slot;  /* in-CSR slot of each out-edge (to read its weight) */
  /* scratch */
  uint8_t* visited;
  uint32_t* queue;
  /* pool (O6) */
  uint64_t seed;
  int have_seed;
  uint64_t nsets, pool_len, cap_sets, cap_pool;
  uint64_t* offsets;      /* nsets+1 */
  uint32_t* nodes;
  uint32_t* count;        /* n */
  /* workload statistics */
  uint64_t stat_coins, stat_live;
  /* MRIM pool (R26): mr_nsets sets of (node, round) pair ids, count over n*T pairs */
  uint32_t mr_T;
  uint64_t mr_seed;
  int mr_have;
  uint64_t mr_nsets, mr_len, mr_cap_sets, mr_cap_pool;
  uint64_t* mr_offsets;
  uint32_t* mr_nodes;
  uint32_t* mr_count;
  uint32_t* mr_tmp;
  int fresh_final;          /* R29: final phase on a fresh pool (og_set_fresh_final) */
  int skip;                 /* R31: geometric-skip RNG contract (og_set_skip) */
} og_ctx;

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

void og_destroy(og_ctx* c) {
  if (!c) return;
  free(c->row_ptr); free(c->src); free(c->w); free(c->thr_edge);
  free(c->out_ptr); free(c->out_dst); free(c->out_in_slot);
  free(c->visited); free(c->queue);
  free(c->offsets); free(c->nodes); free(c->count);
  free(c->mr_offsets); free(c->mr_nodes); free(c->mr_count); free(c->mr_tmp);
  free(c);
}

/* Graph arrays are copied. Returns NULL on invalid input. */
og_ctx* og_create(uint32_t n, uint64_t m, const uint64_t* row_ptr, const uint32_t* src,
                  const float* w, int model, int scheme, float p_uniform) {
  og_ctx* c;
  uint64_t e;
  uint32_t v;
  if (n < 1) return NULL;
  if (scheme == OG_W_EXPLICIT && !w) return NULL;
  c = (og_ctx*)calloc(1, sizeof(og_ctx));
  c->n = n; c->m = m; c->model = model; c->scheme = scheme; c->p_uniform = p_uniform;
  c->row_ptr = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
  c->src = (uint32_t*)malloc(sizeof(uint32_t) * (m ? m : 1));
  memcpy(c->row_ptr, row_ptr, sizeof(uint64_t) * (n + 1));
  if (m) memcpy(c->src, src, sizeof(uint32_t) * m);
  /* O4: live iff coin * 2^-32 < p, exactly: coin < ceil(p * 2^32). p*2^32 is exact in double
   * for a float32 p. */
  c->thr_uniform = (uint64_t)ceil((double)p_uniform * 4294967296.0);
  if (scheme == OG_W_EXPLICIT) {
    c->w = (float*)malloc(sizeof(float) * (m ? m : 1));
    c->thr_edge = (uint64_t*)malloc(sizeof(uint64_t) * (m ? m : 1));
    if (m) memcpy(c->w, w, sizeof(float) * m);
    for (e = 0; e < m; ++e) {
      double x = (double)w[e] * 4294967296.0;
      c->thr_edge[e] = (model == OG_LT) ? (uint64_t)floor(x) : (uint64_t)ceil(x);
    }
  }
  /* the out-CSR (transpose) used by og_mc_spread is built on first use */
  c->visited = (uint8_t*)calloc(n, 1);
  c->queue = (uint32_t*)malloc(sizeof(uint32_t) * n);
  c->cap_sets = 1024;
  c->offsets = (uint64_t*)calloc(c->cap_sets + 1, sizeof(uint64_t));
  c->cap_pool = 4096;
  c->nodes = (uint32_t*)malloc(sizeof(uint32_t) * c->cap_pool);
  c->count = (uint32_t*)calloc(n, sizeof(uint32_t));
  return c;
}

static uint64_t deg_in(const og_ctx* c, uint32_t v) { return c->row_ptr[v + 1] - c->row_ptr[v]; }

/* O4: edge e (an in-edge of v) is live in RR set `id`. */
static int ic_live(og_ctx* c, uint64_t seed, uint64_t id, uint64_t e, uint32_t v) {
  uint64_t coin = og_coin(seed, id, e);
  c->stat_coins++;
  if (c->scheme == OG_W_WC) return coin * deg_in(c, v) < ((uint64_t)1 << 32);   /* p = 1/d_in(v) */
  if (c->scheme == OG_W_UNIFORM) return coin < c->thr_uniform;
  return coin < c->thr_edge[e];
}

/* ------------------------------------------------------------------------------------------
 * R31 (option, off by default; SURVEY.md §8(f) NEXT "geometric skip sampling"). Alg. 3 l.18
 * draws one U(0,1) per in-edge. Where every in-edge of v has the same probability p —
 * weighted cascade p = 1/d_in(v) and uniform p — the live in-edges of v are i.i.d.
 * Bernoulli(p) slots, so the gaps between consecutive live slots are geometric:
 * Pr[gap >= g] = (1-p)^g. This contract draws the gaps instead of the coins:
 *  * the in-edge offsets of v are cut into blocks of SKIP_BLOCK: block b = offsets
 *    [b*1024, min((b+1)*1024, d));
 *  * draw j (j = 0, 1, ...) of block b is word (j & 3) of Philox(seed; id_lo, 2^31 | b, v,
 *    j >> 2) — counter word 1 carries the tag bit (RR ids are < 2^32, so that word is 0 in every
 *    other draw of the key scheme);
 *  * gap = floor(ln(U) * inv_v), U = (r + 1/2) 2^-32, inv_v = 1 / ln(1 - p) — inversion of the
 *    geometric CDF; starting at pos = b*1024: while pos + gap < end of block, offset pos + gap
 *    is live and pos += gap + 1;
 *  * p = 1 (WC with d = 1, uniform p >= 1): every in-edge is live, no draw; p = 0: none is.
 * ln is og_skip_ln below: a fixed sequence of correctly rounded IEEE-754 double operations
 * (a 182-entry table of centers, itself built by the same kind of sequence), so every machine
 * evaluates it (and the gap) identically. Pins: skip_ln against mpmath; the exact
 * gap distribution (counted over all 2^32 words) against (1-p)^g; per-slot live rates and the
 * Eq. 3 estimator against exact enumeration (tests/test_oracle_skip.py).
 * ------------------------------------------------------------------------------------------ */
#define SKIP_BLOCK 1024u
#define SKIP_LN2_HI 6.93147180369123816490e-01   /* ln 2 = HI + LO, HI with 21 trailing zero bits */
#define SKIP_LN2_LO 1.90821492927058770002e-10

/* The series form: ln x for a positive normal double, x = m 2^e with m in [sqrt(1/2), sqrt(2)),
 * ln x = e ln2 + 2 atanh(y), y = (m-1)/(m+1) (|y| <= 0.1716), atanh(y)/y = sum_k y^2k/(2k+1)
 * up to k = 9 (remainder < 1e-17 relative), Horner with fma. Used to tabulate ln(c_k) below. */
double og_skip_ln_series(double x) {
  uint64_t bits;
  double m, y, y2, s;
  int e;
  memcpy(&bits, &x, 8);
  e = (int)((bits >> 52) & 0x7FF) - 1023;
  bits = (bits & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
  memcpy(&m, &bits, 8);                          /* m in [1, 2) */
  if (m > 1.4142135623730951) { m = m * 0.5; e += 1; }
  y = (m - 1.0) / (m + 1.0);
  y2 = y * y;
  s = 1.0 / 19.0;
  s = fma(s, y2, 1.0 / 17.0);
  s = fma(s, y2, 1.0 / 15.0);
  s = fma(s, y2, 1.0 / 13.0);
  s = fma(s, y2, 1.0 / 11.0);
  s = fma(s, y2, 1.0 / 9.0);
  s = fma(s, y2, 1.0 / 7.0);
  s = fma(s, y2, 1.0 / 5.0);
  s = fma(s, y2, 1.0 / 3.0);
  s = fma(s, y2, 1.0);
  return (double)e * SKIP_LN2_HI + ((double)e * SKIP_LN2_LO + (2.0 * y) * s);
}

/* The ln of the contract (division-free per call): m in [sqrt(1/2), sqrt(2)) as above, nearest
 * center c_k = 1 + k/256 (k = floor((m - 1) 256 + 1/2), -75 <= k <= 106), t = (m - c_k) R_k with
 * R_k = 1/c_k, ln m = L_k + ln(1 + t), L_k = ln c_k (the series form), ln(1 + t) by its Taylor
 * polynomial of degree 7 (|t| <= 1/512: remainder < 1e-19 relative). Center 0 is exactly 1
 * (L = 0, R = 1), so x near 1 keeps its relative accuracy. */
#define SKIP_K0 75
static double skip_L[SKIP_K0 + 107], skip_R[SKIP_K0 + 107];
static int skip_tab_ready;
static void skip_tables(void) {
  int k;
  for (k = -SKIP_K0; k <= 106; ++k) {
    double c = 1.0 + (double)k / 256.0;
    skip_R[k + SKIP_K0] = 1.0 / c;
    skip_L[k + SKIP_K0] = og_skip_ln_series(c);
  }
  skip_tab_ready = 1;
}

double og_skip_ln(double x) {
  uint64_t bits;
  double m, c, t, s;
  int e, k;
  if (!skip_tab_ready) skip_tables();
  memcpy(&bits, &x, 8);
  e = (int)((bits >> 52) & 0x7FF) - 1023;
  bits = (bits & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
  memcpy(&m, &bits, 8);                          /* m in [1, 2) */
  if (m > 1.4142135623730951) { m = m * 0.5; e += 1; }
  k = (int)floor((m - 1.0) * 256.0 + 0.5);
  c = 1.0 + (double)k / 256.0;
  t = (m - c) * skip_R[k + SKIP_K0];
  s = 1.0 / 7.0;
  s = fma(s, t, -1.0 / 6.0);
  s = fma(s, t, 1.0 / 5.0);
  s = fma(s, t, -1.0 / 4.0);
  s = fma(s, t, 1.0 / 3.0);
  s = fma(s, t, -1.0 / 2.0);
  s = fma(s, t, 1.0);
  return (double)e * SKIP_LN2_HI + ((double)e * SKIP_LN2_LO + (skip_L[k + SKIP_K0] + t * s));
}

/* inv_v = 1 / ln(1 - p) < 0; 0 when p = 1 (every in-edge live, no draws). WC: 1 - 1/d as
 * (d-1)/d (one rounding). Uniform: 1 - p exact for a float32 p. */
double og_skip_inv(int scheme, uint64_t d, float p_uniform) {
  double q;
  if (scheme == OG_W_WC) {
    if (d <= 1) return 0.0;
    q = (double)(d - 1) / (double)d;
  } else {
    q = 1.0 - (double)p_uniform;
    if (!(q > 0.0)) return 0.0;
  }
  return 1.0 / og_skip_ln(q);
}

/* gap of word r: floor(ln((r + 1/2) 2^-32) * inv), returned as a double (>= 0; compare before
 * converting: it may exceed any block) */
double og_skip_gap(double inv, uint32_t r) {
  return floor(og_skip_ln(((double)r + 0.5) * 0x1p-32) * inv);
}

uint32_t og_skip_word(uint64_t seed, uint64_t id, uint32_t v, uint32_t b, uint32_t j) {
  uint32_t o[4], ctr[4], key[2];
  ctr[0] = (uint32_t)id; ctr[1] = 0x80000000u | b; ctr[2] = v; ctr[3] = j >> 2;
  key[0] = (uint32_t)seed; key[1] = (uint32_t)(seed >> 32);
  og_philox(ctr, key, o);
  return o[j & 3];
}

/* R31 selects the skip contract (IC with WC or uniform weights only); the pool restarts. */
int og_set_skip(og_ctx* c, int on) {
  if (on && (c->model != OG_IC || c->scheme == OG_W_EXPLICIT)) return 1;
  if ((on ? 1 : 0) != c->skip) { c->skip = on ? 1 : 0; c->have_seed = 0; c->mr_have = 0; }
  return 0;
}

/* O4. IC RR set: reverse BFS over live in-edges from a uniform root — the RR set definition of
 * P:166-168 realised as the randomized BFS of P:260 / Alg. 3 l.8-22, with the root
 * marked visited (R12) and exact set semantics (R13). Writes the set, ascending, to out[];
 * returns its size. */
static uint32_t rr_ic(og_ctx* c, uint64_t seed, uint64_t id, uint32_t root, uint32_t* out) {
  uint32_t head = 0, tail = 0, i;
  c->visited[root] = 1;
  c->queue[tail++] = root;
  while (head < tail) {
    uint32_t v = c->queue[head++];
    uint64_t e;
    if (c->skip) {                                    /* R31: the same BFS, live slots by gaps */
      uint64_t a = c->row_ptr[v], d = c->row_ptr[v + 1] - a, b;
      double inv;
      if (d == 0 || (c->scheme == OG_W_UNIFORM && c->thr_uniform == 0)) continue;
      inv = og_skip_inv(c->scheme, d, c->p_uniform);
      for (b = 0; b * SKIP_BLOCK < d; ++b) {
        uint64_t pos = b * SKIP_BLOCK, end = pos + SKIP_BLOCK < d ? pos + SKIP_BLOCK : d;
        uint32_t j;
        for (j = 0; pos < end; ++j) {
          if (inv != 0.0) {
            double g = og_skip_gap(inv, og_skip_word(seed, id, v, (uint32_t)b, j));
            c->stat_coins++;
            if (g >= (double)(end - pos)) break;
            pos += (uint64_t)g;
          }
          c->stat_live++;
          {
            uint32_t u = c->src[a + pos];
            if (!c->visited[u]) {
              c->visited[u] = 1;
              c->queue[tail++] = u;
            }
          }
          pos += 1;
        }
      }
      continue;
    }
    for (e = c->row_ptr[v]; e < c->row_ptr[v + 1]; ++e) {
      if (ic_live(c, seed, id, e, v)) {
        uint32_t u = c->src[e];
        c->stat_live++;
        if (!c->visited[u]) {
          c->visited[u] = 1;
          c->queue[tail++] = u;
        }
      }
    }
  }
  for (i = 0; i < tail; ++i) { c->visited[c->queue[i]] = 0; out[i] = c->queue[i]; }
  qsort(out, tail, sizeof(uint32_t), cmp_u32);
  return tail;
}

/* O5. LT RR set: reverse random walk choosing at most one in-edge per node according to the
 * edge weights, frontier <= 1, stopping at a node with no chosen edge or at an
 * already-visited node (R19). Half-open fixed-point intervals (R18). */
static uint32_t rr_lt(og_ctx* c, uint64_t seed, uint64_t id, uint32_t root, uint32_t* out) {
  uint32_t len = 0, i;
  uint32_t v = root;
  c->visited[v] = 1;
  c->queue[len++] = v;
  for (;;) {
    uint64_t d = deg_in(c, v);
    uint64_t r, j;
    uint32_t u;
    if (d == 0) break;
    r = og_lt_draw(seed, id, v);
    c->stat_coins++;
    if (c->scheme == OG_W_WC) {
      j = (r * d) >> 32;                     /* uniform in-neighbour: weights 1/d */
    } else {
      uint64_t acc = 0, t;
      j = d;
      for (t = 0; t < d; ++t) {
        acc += c->thr_edge[c->row_ptr[v] + t];
        if (r < acc) { j = t; break; }
      }
      if (j == d) break;                     /* r beyond the total weight: no live in-edge */
    }
    c->stat_live++;
    u = c->src[c->row_ptr[v] + j];
    if (c->visited[u]) break;
    c->visited[u] = 1;
    c->queue[len++] = u;
    v = u;
  }
  for (i = 0; i < len; ++i) { c->visited[c->queue[i]] = 0; out[i] = c->queue[i]; }
  qsort(out, len, sizeof(uint32_t), cmp_u32);
  return len;
}

/* the RR set of id `id` grown from `root` (og_rr_set: root = og_root(seed, id), O3) */
static uint32_t rr_from(og_ctx* c, uint64_t seed, uint64_t id, uint32_t root, uint32_t* out) {
  return (c->model == OG_LT) ? rr_lt(c, seed, id, root, out) : rr_ic(c, seed, id, root, out);
}

uint32_t og_rr_set(og_ctx* c, uint64_t seed, uint64_t id, uint32_t* out) {
  return rr_from(c, seed, id, og_root(seed, id, c->n), out);
}

/* O6. Extend (or truncate) the pool to exactly { RR(seed, i) : 0 <= i < T } in id order, with
 * count[v] = #{i : v in RR_i} — Occur of P:285 / Alg. 3 l.13, RR + Offsets_RR of Alg. 6
 * (P:435-445), except that sets are stored in id order (R20). A different seed restarts. */
int og_generate(og_ctx* c, uint64_t T, uint64_t seed) {
  uint64_t i, j;
  if (!c->have_seed || c->seed != seed) {
    c->nsets = 0; c->pool_len = 0; c->offsets[0] = 0;
    memset(c->count, 0, sizeof(uint32_t) * c->n);
    c->seed = seed; c->have_seed = 1;
  }
  while (c->nsets > T) {                      /* truncate */
    uint64_t a = c->offsets[c->nsets - 1], b = c->offsets[c->nsets];
    for (j = a; j < b; ++j) c->count[c->nodes[j]]--;
    c->nsets--; c->pool_len = a;
  }
  for (i = c->nsets; i < T; ++i) {
    uint32_t len;
    if (c->nsets + 1 > c->cap_sets) {
      c->cap_sets *= 2;
      c->offsets = (uint64_t*)realloc(c->offsets, sizeof(uint64_t) * (c->cap_sets + 1));
    }
    if (c->pool_len + c->n > c->cap_pool) {
      while (c->pool_len + c->n > c->cap_pool) c->cap_pool *= 2;
      c->nodes = (uint32_t*)realloc(c->nodes, sizeof(uint32_t) * c->cap_pool);
    }
    len = og_rr_set(c, seed, i, c->nodes + c->pool_len);
    for (j = 0; j < len; ++j) c->count[c->nodes[c->pool_len + j]]++;
    c->pool_len += len;
    c->nsets++;
    c->offsets[c->nsets] = c->pool_len;
  }
  return 0;
}

uint64_t og_num_sets(const og_ctx* c) { return c->nsets; }
uint64_t og_pool_len(const og_ctx* c) { return c->pool_len; }
void og_export(const og_ctx* c, uint64_t* offsets_out, uint32_t* nodes_out, uint32_t* count_out) {
  if (offsets_out) memcpy(offsets_out, c->offsets, sizeof(uint64_t) * (c->nsets + 1));
  if (nodes_out && c->pool_len) memcpy(nodes_out, c->nodes, sizeof(uint32_t) * c->pool_len);
  if (count_out) memcpy(count_out, c->count, sizeof(uint32_t) * c->n);
}
void og_stats(const og_ctx* c, uint64_t out[2]) { out[0] = c->stat_coins; out[1] = c->stat_live; }

/* ------------------------------------------------------------------------------------------
 * O7. NodeSelection: greedy max coverage over a pool of ascending sets — Alg. 1 l.6-10
 * with the counter method of §3.8 and Alg. 7 literally:
 * for each pick, scan every uncovered set for u; if found, flag it covered and decrement the
 * counter of every member (u included, R11). Argmax over unselected nodes, ties -> lowest id,
 * zero maximum allowed (R10). Non-destructive (R9): starts from the given counts.
 * ------------------------------------------------------------------------------------------ */
static int contains_sorted(const uint32_t* a, uint64_t len, uint32_t u) {
  uint64_t lo = 0, hi = len;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < u) lo = mid + 1; else hi = mid;
  }
  return lo < len && a[lo] == u;
}

int og_select_pool(uint32_t n, uint64_t nsets, const uint64_t* offsets, const uint32_t* nodes,
                   const uint32_t* count, uint32_t k, uint32_t* seeds_out, uint64_t* gains_out,
                   uint64_t* cov_out) {
  int64_t* cnt;
  uint8_t *covered, *selected;
  uint64_t i, w, cov = 0;
  uint32_t j, v;
  if (k < 1 || k > n) return 1;
  cnt = (int64_t*)malloc(sizeof(int64_t) * n);
  covered = (uint8_t*)calloc(nsets ? nsets : 1, 1);
  selected = (uint8_t*)calloc(n, 1);
  for (v = 0; v < n; ++v) cnt[v] = count[v];
  for (j = 0; j < k; ++j) {
    int64_t best = -1;
    uint32_t u = 0;
    for (v = 0; v < n; ++v)
      if (!selected[v] && cnt[v] > best) { best = cnt[v]; u = v; }
    selected[u] = 1;
    seeds_out[j] = u;
    if (gains_out) gains_out[j] = (uint64_t)best;
    cov += (uint64_t)best;
    for (i = 0; i < nsets; ++i) {                       /* Alg. 7 l.1 */
      uint64_t off = offsets[i], len = offsets[i + 1] - offsets[i];
      if (covered[i]) continue;                          /* l.2 */
      if (!contains_sorted(nodes + off, len, u)) continue;  /* l.3-10 */
      covered[i] = 1;                                    /* l.12 */
      for (w = 0; w < len; ++w) cnt[nodes[off + w]]--;   /* l.13-15 */
    }
  }
  if (cov_out) *cov_out = cov;
  free(cnt); free(covered); free(selected);
  return 0;
}

int og_select(og_ctx* c, uint32_t k, uint32_t* seeds_out, uint64_t* gains_out, uint64_t* cov_out) {
  if (c->nsets == 0) return 2;
  return og_select_pool(c->n, c->nsets, c->offsets, c->nodes, c->count, k, seeds_out, gains_out,
                        cov_out);
}

/* ------------------------------------------------------------------------------------------
 * O8. IMM constants. The paper defers f(n, eps, k) and lambda to IMM (
 * readings R1-R3): lambda' and lambda* of Tang, Shi, Xiao (SIGMOD'15). Double, contraction off,
 * expression order fixed.
 * out = { ell_eff, eps_prime, lnC, lambda_prime, alpha, beta, lambda_star }
 * ------------------------------------------------------------------------------------------ */
/* lnC = ln C(N, K) (the union bound over candidate seed sets); N = n, K = k for IMM; MRIM
 * (R28) takes N = n*T pairs and K = k*T picks. */
static int imm_constants_g(uint32_t n, uint64_t N, uint64_t K, double eps, double ell, double out[7]) {
  double ln_n, log2n, ell_eff, eps_p, lnC = 0.0, lambda_p, alpha, beta, lambda_s, e = M_E;
  uint64_t t;
  if (n < 2 || K < 1 || K > N || !(eps > 0.0 && eps < 1.0) || !(ell > 0.0)) return 1;
  ln_n = log((double)n);
  log2n = log2((double)n);
  ell_eff = ell * (1.0 + log(2.0) / ln_n);
  eps_p = sqrt(2.0) * eps;
  for (t = 1; t <= K; ++t) lnC += log((double)(N - K + t)) - log((double)t);
  lambda_p = (2.0 + 2.0 / 3.0 * eps_p) * (lnC + ell_eff * ln_n + log(log2n)) * (double)n / (eps_p * eps_p);
  alpha = sqrt(ell_eff * ln_n + log(2.0));
  beta = sqrt((1.0 - 1.0 / e) * (lnC + ell_eff * ln_n + log(2.0)));
  {
    double s = (1.0 - 1.0 / e) * alpha + beta;
    lambda_s = 2.0 * (double)n * (s * s) / (eps * eps);
  }
  out[0] = ell_eff; out[1] = eps_p; out[2] = lnC; out[3] = lambda_p;
  out[4] = alpha; out[5] = beta; out[6] = lambda_s;
  return 0;
}

int og_imm_constants(uint32_t n, uint32_t k, double eps, double ell, double out[7]) {
  if (k > n) return 1;
  return imm_constants_g(n, n, k, eps, ell, out);
}

/* R29 (SURVEY R8's NEXT variant; Chen 2018 [EXT] on IMM's martingale analysis): the final phase
 * draws a fresh pool, independent of the sets that produced LB — the sets of a second key,
 * seed ^ 0x9E3779B97F4A7C15: R_final = ceil(theta) sets RR(seed_f, i). Off by default (IMM's
 * published reuse, R8). */
#define OG_FRESH_KEY 0x9E3779B97F4A7C15ull
void og_set_fresh_final(og_ctx* c, int on) { c->fresh_final = on ? 1 : 0; }

/* O8 driver: Alg. 2 rounds, then theta = lambda_star / LB and the final selection
 * (Alg. 1). Readings R4-R8. Cumulative pool (IMM reuses the estimation sets).
 * dres = { LB, theta, spread_est, ell_eff, eps_prime, lambda_prime, lambda_star }
 * tr_theta[i] = theta_i (double), tr_T[i] = ceil(theta_i), tr_cov[i] = covered count of round i.
 * ures = { rounds, R_final, cov_final }. */
int og_imm(og_ctx* c, uint32_t k, double eps, double ell, uint64_t seed, uint32_t* seeds_out,
           uint64_t* gains_out, double dres[7], double tr_theta[64], uint64_t tr_T[64],
           uint64_t tr_cov[64], uint64_t ures[3]) {
  double K[7], n = (double)c->n, LB = 1.0, theta, log2n;
  uint64_t cov = 0, T, R;
  int i, i_max, rounds = 0;
  uint32_t* tmp_seeds;
  if (og_imm_constants(c->n, k, eps, ell, K)) return 1;
  tmp_seeds = (uint32_t*)malloc(sizeof(uint32_t) * k);
  c->have_seed = 0;                                      /* IMM starts from R = {} */
  og_generate(c, 0, seed);
  log2n = log2(n);
  i_max = (int)floor(log2n) - 1;                         /* R5 */
  for (i = 1; i <= i_max && i <= 64; ++i) {
    double x = n / ldexp(1.0, i);                        /* Alg. 2 l.3 */
    double theta_i = K[3] / x;                           /* l.4 */
    T = (uint64_t)ceil(theta_i);
    R = c->nsets > T ? c->nsets : T;                     /* l.5, R4 */
    og_generate(c, R, seed);
    og_select(c, k, tmp_seeds, NULL, &cov);              /* l.6, R9 */
    tr_theta[i - 1] = theta_i; tr_T[i - 1] = T; tr_cov[i - 1] = cov;
    rounds = i;
    if ((n * (double)cov) / (double)c->nsets >= (1.0 + K[1]) * x) {   /* l.7, R7 */
      LB = (n * (double)cov) / (double)c->nsets / (1.0 + K[1]);       /* l.8 */
      break;
    }
  }
  theta = K[6] / LB;                                     /* R2 */
  T = (uint64_t)ceil(theta);
  if (c->fresh_final) {
    og_generate(c, T, seed ^ OG_FRESH_KEY);              /* R29: a different key discards R */
  } else {
    R = c->nsets > T ? c->nsets : T;                     /* R8: reuse, no truncation */
    og_generate(c, R, seed);
  }
  og_select(c, k, seeds_out, gains_out, &cov);
  dres[0] = LB; dres[1] = theta; dres[2] = n * (double)cov / (double)c->nsets;   /* Eq. 3 */
  dres[3] = K[0]; dres[4] = K[1]; dres[5] = K[3]; dres[6] = K[6];
  ures[0] = (uint64_t)rounds; ures[1] = c->nsets; ures[2] = cov;
  free(tmp_seeds);
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * Forward Monte-Carlo spread (verification only; uses none of the reverse machinery).
 * IC per P:120: each newly active u tries each out-edge once with probability p_uv.
 * LT per Eq. 1: thresholds tau_v ~ U(0,1); v activates when the summed weight of
 * its active in-neighbours reaches tau_v (iterated to the fixpoint, which is order-free).
 * Reading R30: tau_v = (o + 1/2) / 2^32 (o = the tag-11 draw of v) is compared EXACTLY — WC
 * (w = 1/d_in(v)): cnt * 2^33 >= (2o + 1) * d_in(v); explicit weights in the fixed point of R18
 * (W = floor(w 2^32)): sum W >= o + 1 — so the activated set has no rounding-order dependence.
 * Randomness: Philox keyed (mc_seed; trial, tag-11 slot), independent of any RR stream.
 * ------------------------------------------------------------------------------------------ */
static void build_out_csr(og_ctx* c) {
  uint64_t e, *cur;
  uint32_t v, n = c->n;
  if (c->out_ptr) return;
  c->out_ptr = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  c->out_dst = (uint32_t*)malloc(sizeof(uint32_t) * (c->m ? c->m : 1));
  c->out_in_slot = (uint64_t*)malloc(sizeof(uint64_t) * (c->m ? c->m : 1));
  for (e = 0; e < c->m; ++e) c->out_ptr[c->src[e] + 1]++;
  for (v = 0; v < n; ++v) c->out_ptr[v + 1] += c->out_ptr[v];
  cur = (uint64_t*)malloc(sizeof(uint64_t) * n);
  memcpy(cur, c->out_ptr, sizeof(uint64_t) * n);
  for (v = 0; v < n; ++v)
    for (e = c->row_ptr[v]; e < c->row_ptr[v + 1]; ++e) {
      uint64_t pos = cur[c->src[e]]++;
      c->out_dst[pos] = v;
      c->out_in_slot[pos] = e;
    }
  free(cur);
}

static double edge_p(const og_ctx* c, uint64_t in_slot, uint32_t v) {
  if (c->scheme == OG_W_WC) return 1.0 / (double)deg_in(c, v);
  if (c->scheme == OG_W_UNIFORM) return (double)c->p_uniform;
  return (double)c->w[in_slot];
}

int og_mc_spread(og_ctx* c, const uint32_t* S, uint32_t k, uint64_t trials, uint64_t mc_seed,
                 double* mean_out, double* stderr_out) {
  uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * c->n);
  uint8_t* act = (uint8_t*)calloc(c->n, 1);
  uint64_t* acc = (uint64_t*)calloc(c->n, sizeof(uint64_t));
  uint32_t* touched = (uint32_t*)malloc(sizeof(uint32_t) * (c->m + c->n + 1));
  double sum = 0.0, sum2 = 0.0;
  uint64_t t;
  build_out_csr(c);
  for (t = 0; t < trials; ++t) {
    uint32_t head = 0, tail = 0, ntouch = 0, i;
    for (i = 0; i < k; ++i)
      if (!act[S[i]]) { act[S[i]] = 1; q[tail++] = S[i]; }
    while (head < tail) {
      uint32_t u = q[head++];
      uint64_t e;
      for (e = c->out_ptr[u]; e < c->out_ptr[u + 1]; ++e) {
        uint32_t v = c->out_dst[e];
        if (act[v]) continue;
        if (c->model == OG_IC) {
          double p = edge_p(c, c->out_in_slot[e], v);
          uint32_t o[4];
          keyed(mc_seed, t, SLOT_MC | (e >> 2), o);
          if ((double)o[e & 3] < p * 4294967296.0) { act[v] = 1; q[tail++] = v; }
        } else {
          uint32_t o[4];
          int met;
          keyed(mc_seed, t, SLOT_MC | (((uint64_t)1) << 40) | (uint64_t)v, o);   /* tau_v */
          if (acc[v] == 0) touched[ntouch++] = v;
          if (c->scheme == OG_W_WC) {
            acc[v] += 1;                                   /* active in-neighbours */
            met = ((unsigned __int128)acc[v] << 33) >= (unsigned __int128)(2 * (uint64_t)o[0] + 1) * deg_in(c, v);
          } else {
            acc[v] += c->thr_edge[c->out_in_slot[e]];     /* LT: floor(w 2^32) */
            met = acc[v] >= (uint64_t)o[0] + 1;
          }
          if (met) { act[v] = 1; q[tail++] = v; }
        }
      }
    }
    sum += (double)tail;
    sum2 += (double)tail * (double)tail;
    for (i = 0; i < tail; ++i) act[q[i]] = 0;
    for (i = 0; i < ntouch; ++i) acc[touched[i]] = 0;
  }
  *mean_out = sum / (double)trials;
  {
    double var = sum2 / (double)trials - (*mean_out) * (*mean_out);
    *stderr_out = sqrt((var > 0 ? var : 0) / (double)trials);
  }
  free(q); free(act); free(acc); free(touched);
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * MRIM: multi-round influence maximization, the CR-NAIMM algorithm of Sun et al. (KDD'18) as
 * gIM adapts it (§4.8): "after selecting a random node, we initiate a random BFS
 * originating from the selected node as many times as the number of rounds. Also, each element
 * in a random RR set is a tuple of node-id and round number. The rest of our algorithm remains
 * almost intact." The goal: a seed set per round maximizing the number of nodes
 * influenced at least once. Readings R26-R28:
 * R26  MRR_i = {(u, t) : 0 <= t < T, u in RR^t_i}: root_i = og_root(seed, i) is shared by the T
 *      rounds; round t's BFS (IC coins / LT draws, O4/O5) is keyed by the standard RR id
 *      i*T + t, so the rounds are independent and T = 1 is exactly the standard RR set i.
 *      The pair (u, t) is the id t*n + u; a set is stored ascending (rounds, then nodes).
 * R27  selection: greedy max coverage over pairs (Alg. 1 l.6-10, Alg. 7 with pair counters)
 *      where a round accepts at most k seeds: each of the k*T picks is the unselected pair of a
 *      not-yet-full round with the largest count, ties -> lowest pair id.
 * R28  theta: IMM's lambda', lambda* (R1, R2) with ln C(n*T, k*T) for ln C(n, k) (the pairs are
 *      the ground set, k*T picks); n, ell_eff and the rounds x = n / 2^i unchanged (the
 *      objective counts nodes, at most n).
 * ------------------------------------------------------------------------------------------ */
int og_mrim_generate(og_ctx* c, uint64_t N, uint32_t T, uint64_t seed) {
  uint64_t i, j;
  uint32_t t;
  const uint64_t nT = (uint64_t)c->n * T;
  if (T < 1 || nT >= 0xFFFFFFFFull) return 1;
  if (!c->mr_have || c->mr_seed != seed || c->mr_T != T) {
    free(c->mr_offsets); free(c->mr_nodes); free(c->mr_count);
    c->mr_T = T; c->mr_seed = seed; c->mr_have = 1;
    c->mr_nsets = 0; c->mr_len = 0;
    c->mr_cap_sets = 1024;
    c->mr_offsets = (uint64_t*)calloc(c->mr_cap_sets + 1, sizeof(uint64_t));
    c->mr_cap_pool = 4096;
    c->mr_nodes = (uint32_t*)malloc(sizeof(uint32_t) * c->mr_cap_pool);
    c->mr_count = (uint32_t*)calloc(nT, sizeof(uint32_t));
    if (!c->mr_tmp) c->mr_tmp = (uint32_t*)malloc(sizeof(uint32_t) * c->n);
  }
  while (c->mr_nsets > N) {                   /* truncate */
    uint64_t a = c->mr_offsets[c->mr_nsets - 1], b = c->mr_offsets[c->mr_nsets];
    for (j = a; j < b; ++j) c->mr_count[c->mr_nodes[j]]--;
    c->mr_nsets--; c->mr_len = a;
  }
  for (i = c->mr_nsets; i < N; ++i) {
    uint32_t root = og_root(seed, i, c->n);   /* "selecting a random node" */
    if (c->mr_nsets + 1 > c->mr_cap_sets) {
      c->mr_cap_sets *= 2;
      c->mr_offsets = (uint64_t*)realloc(c->mr_offsets, sizeof(uint64_t) * (c->mr_cap_sets + 1));
    }
    if (c->mr_len + nT > c->mr_cap_pool) {
      while (c->mr_len + nT > c->mr_cap_pool) c->mr_cap_pool *= 2;
      c->mr_nodes = (uint32_t*)realloc(c->mr_nodes, sizeof(uint32_t) * c->mr_cap_pool);
    }
    for (t = 0; t < T; ++t) {                 /* "as many times as the number of rounds" */
      uint32_t len = rr_from(c, seed, i * (uint64_t)T + t, root, c->mr_tmp), q;
      for (q = 0; q < len; ++q) {
        uint32_t pr = t * c->n + c->mr_tmp[q];   /* (node-id, round) tuple */
        c->mr_nodes[c->mr_len++] = pr;
        c->mr_count[pr]++;
      }
    }
    c->mr_nsets++;
    c->mr_offsets[c->mr_nsets] = c->mr_len;
  }
  return 0;
}

/* One MRIM set (R26) by itself, ascending pair ids; returns its size (out: n*T entries). */
uint32_t og_mrim_set(og_ctx* c, uint64_t seed, uint64_t i, uint32_t T, uint32_t* out) {
  uint32_t root = og_root(seed, i, c->n), len = 0, t, q;
  if (!c->mr_tmp) c->mr_tmp = (uint32_t*)malloc(sizeof(uint32_t) * c->n);
  for (t = 0; t < T; ++t) {
    uint32_t l = rr_from(c, seed, i * (uint64_t)T + t, root, c->mr_tmp);
    for (q = 0; q < l; ++q) out[len++] = t * c->n + c->mr_tmp[q];
  }
  return len;
}

uint64_t og_mrim_num_sets(const og_ctx* c) { return c->mr_have ? c->mr_nsets : 0; }
uint64_t og_mrim_pool_len(const og_ctx* c) { return c->mr_have ? c->mr_len : 0; }
void og_mrim_export(const og_ctx* c, uint64_t* offsets_out, uint32_t* pairs_out, uint32_t* count_out) {
  if (!c->mr_have) return;
  if (offsets_out) memcpy(offsets_out, c->mr_offsets, sizeof(uint64_t) * (c->mr_nsets + 1));
  if (pairs_out && c->mr_len) memcpy(pairs_out, c->mr_nodes, sizeof(uint32_t) * c->mr_len);
  if (count_out) memcpy(count_out, c->mr_count, sizeof(uint32_t) * (uint64_t)c->n * c->mr_T);
}

/* R27 over a pool of ascending pair sets: n nodes, T rounds, k seeds per round; seeds_out and
 * gains_out hold the k*T picks (pair ids) in pick order. */
int og_mrim_select_pool(uint32_t n, uint32_t T, uint64_t nsets, const uint64_t* offsets,
                        const uint32_t* pairs, const uint32_t* count, uint32_t k, uint32_t* seeds_out,
                        uint64_t* gains_out, uint64_t* cov_out) {
  const uint64_t nT = (uint64_t)n * T;
  int64_t* cnt;
  uint8_t *covered, *selected;
  uint32_t* picks;
  uint64_t i, w, v, cov = 0;
  uint32_t j;
  if (T < 1 || k < 1 || k > n) return 1;
  cnt = (int64_t*)malloc(sizeof(int64_t) * nT);
  covered = (uint8_t*)calloc(nsets ? nsets : 1, 1);
  selected = (uint8_t*)calloc(nT, 1);
  picks = (uint32_t*)calloc(T, sizeof(uint32_t));
  for (v = 0; v < nT; ++v) cnt[v] = count[v];
  for (j = 0; j < k * T; ++j) {
    int64_t best = -1;
    uint32_t u = 0;
    for (v = 0; v < nT; ++v)
      if (!selected[v] && picks[v / n] < k && cnt[v] > best) { best = cnt[v]; u = (uint32_t)v; }
    selected[u] = 1;
    picks[u / n]++;
    seeds_out[j] = u;
    if (gains_out) gains_out[j] = (uint64_t)best;
    cov += (uint64_t)best;
    for (i = 0; i < nsets; ++i) {                        /* Alg. 7 with pair counters */
      uint64_t off = offsets[i], len = offsets[i + 1] - offsets[i];
      if (covered[i]) continue;
      if (!contains_sorted(pairs + off, len, u)) continue;
      covered[i] = 1;
      for (w = 0; w < len; ++w) cnt[pairs[off + w]]--;
    }
  }
  if (cov_out) *cov_out = cov;
  free(cnt); free(covered); free(selected); free(picks);
  return 0;
}

int og_mrim_select(og_ctx* c, uint32_t k, uint32_t* seeds_out, uint64_t* gains_out, uint64_t* cov_out) {
  if (!c->mr_have || c->mr_nsets == 0) return 2;
  return og_mrim_select_pool(c->n, c->mr_T, c->mr_nsets, c->mr_offsets, c->mr_nodes, c->mr_count, k,
                             seeds_out, gains_out, cov_out);
}

int og_mrim_constants(uint32_t n, uint32_t k, uint32_t T, double eps, double ell, double out[7]) {
  if (T < 1 || k > n) return 1;
  return imm_constants_g(n, (uint64_t)n * T, (uint64_t)k * T, eps, ell, out);
}

/* Alg. 2 over MRIM sets (R26-R28), exactly as og_imm: LB rounds on x = n / 2^i,
 * theta = lambda* / LB, cumulative pool, final selection of k*T pairs. Outputs as og_imm. */
int og_mrim(og_ctx* c, uint32_t k, uint32_t T, double eps, double ell, uint64_t seed,
            uint32_t* seeds_out, uint64_t* gains_out, double dres[7], double tr_theta[64],
            uint64_t tr_T[64], uint64_t tr_cov[64], uint64_t ures[3]) {
  double K[7], n = (double)c->n, LB = 1.0, theta, log2n;
  uint64_t cov = 0, Tn, R;
  int i, i_max, rounds = 0;
  uint32_t* tmp_seeds;
  if (og_mrim_constants(c->n, k, T, eps, ell, K)) return 1;
  tmp_seeds = (uint32_t*)malloc(sizeof(uint32_t) * k * T);
  c->mr_have = 0;                                        /* R = {} */
  if (og_mrim_generate(c, 0, T, seed)) { free(tmp_seeds); return 1; }
  log2n = log2(n);
  i_max = (int)floor(log2n) - 1;
  for (i = 1; i <= i_max && i <= 64; ++i) {
    double x = n / ldexp(1.0, i);
    double theta_i = K[3] / x;
    Tn = (uint64_t)ceil(theta_i);
    R = c->mr_nsets > Tn ? c->mr_nsets : Tn;
    og_mrim_generate(c, R, T, seed);
    og_mrim_select(c, k, tmp_seeds, NULL, &cov);
    tr_theta[i - 1] = theta_i; tr_T[i - 1] = Tn; tr_cov[i - 1] = cov;
    rounds = i;
    if ((n * (double)cov) / (double)c->mr_nsets >= (1.0 + K[1]) * x) {
      LB = (n * (double)cov) / (double)c->mr_nsets / (1.0 + K[1]);
      break;
    }
  }
  theta = K[6] / LB;
  Tn = (uint64_t)ceil(theta);
  if (c->fresh_final) {
    og_mrim_generate(c, Tn, T, seed ^ OG_FRESH_KEY);     /* R29 */
  } else {
    R = c->mr_nsets > Tn ? c->mr_nsets : Tn;
    og_mrim_generate(c, R, T, seed);
  }
  og_mrim_select(c, k, seeds_out, gains_out, &cov);
  dres[0] = LB; dres[1] = theta; dres[2] = n * (double)cov / (double)c->mr_nsets;
  dres[3] = K[0]; dres[4] = K[1]; dres[5] = K[3]; dres[6] = K[6];
  ures[0] = (uint64_t)rounds; ures[1] = c->mr_nsets; ures[2] = cov;
  free(tmp_seeds);
  return 0;
}

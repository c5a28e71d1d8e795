// gim_inputs/plg.cpp — seeded synthetic INPUT generator shared by the oracle and the CUDA path.
//
// Directed Chung-Lu power-law graph ("plg") + canonical in-CSR builder.
// This module holds NONE of the method's arithmetic: no Philox, no coins, no influence
// probabilities. Its RNG is a splitmix64 counter hash (deliberately NOT the method's
// Philox4x32-10) so that nothing here can mask a bug on either side of the parity test.
//
// Recipe (stated in DESIGN.md "Input recipe"):
//   * rank weights w(i) = (i + i0)^(-1/(gamma-1)), i = 0..n-1; i0 solved so that the expected
//     number of draws landing on rank 0 equals d_cap (per direction, before dedup);
//   * two independent random permutations map out-ranks and in-ranks to node ids;
//   * draw t picks an out-rank a and an in-rank b from one Vose alias table; candidate edge
//     (perm_out[a] -> perm_in[b]) gets index 2t; with probability rho the reverse edge
//     (perm_in[b] -> perm_out[a]) is also a candidate with index 2t+1;
//   * self-loops are dropped, duplicates keep their smallest index, and the graph is exactly
//     the first m distinct candidate edges in index order (draws are topped up until m exist);
//   * output is the canonical in-CSR: row v lists the sources u of edges u->v, strictly
//     ascending (SURVEY.md §8(c) O1 / reading R15).
//
// Build: g++ -O3 -fopenmp -shared -fPIC plg.cpp -o libplg.so   (see Makefile)
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <omp.h>

namespace {

inline uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
// Counter-based stream: word j of draw t under base key.
inline uint64_t rnd(uint64_t base, uint64_t t, uint64_t j) {
  return fmix64(base + (t * 4 + j) * 0x9E3779B97F4A7C15ULL);
}
inline uint64_t mulhi64(uint64_t a, uint64_t b) {
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
}

struct Alias {
  std::vector<uint64_t> thr;   // accept threshold in [0, 2^32]
  std::vector<uint32_t> alias;
  uint32_t n = 0;
  uint32_t sample(uint64_t w_col, uint32_t w_acc) const {
    uint32_t c = (uint32_t)mulhi64(w_col, n);
    return ((uint64_t)w_acc < thr[c]) ? c : alias[c];
  }
};

// Vose's alias method over rank weights (i + i0)^-a.
Alias build_alias(uint32_t n, double i0, double a) {
  Alias t;
  t.n = n;
  t.thr.assign(n, 0);
  t.alias.assign(n, 0);
  std::vector<double> p(n);
  double sum = 0.0;
  for (uint32_t i = 0; i < n; ++i) { p[i] = std::pow((double)i + i0, -a); sum += p[i]; }
  std::vector<uint32_t> small, large;
  small.reserve(n); large.reserve(n);
  for (uint32_t i = 0; i < n; ++i) {
    p[i] = p[i] * (double)n / sum;
    if (p[i] < 1.0) small.push_back(i); else large.push_back(i);
  }
  while (!small.empty() && !large.empty()) {
    uint32_t s = small.back(); small.pop_back();
    uint32_t l = large.back();
    t.thr[s] = (uint64_t)std::floor(p[s] * 4294967296.0);
    t.alias[s] = l;
    p[l] = (p[l] + p[s]) - 1.0;
    if (p[l] < 1.0) { large.pop_back(); small.push_back(l); }
  }
  for (uint32_t l : large) { t.thr[l] = 4294967296ULL; t.alias[l] = l; }
  for (uint32_t s : small) { t.thr[s] = 4294967296ULL; t.alias[s] = s; }
  return t;
}

// Sum of w(i) over i < n in a fixed order (256 fixed chunks summed in order), so the result —
// and through solve_i0 the alias tables and the graph — does not depend on the thread count.
double sum_weights(uint32_t n, double i0, double a) {
  constexpr int64_t C = 256;
  double part[C];
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < C; ++c) {
    const int64_t lo = (int64_t)n * c / C, hi = (int64_t)n * (c + 1) / C;
    double s = 0.0;
    for (int64_t i = lo; i < hi; ++i) s += std::pow((double)i + i0, -a);
    part[c] = s;
  }
  double s = 0.0;
  for (int64_t c = 0; c < C; ++c) s += part[c];
  return s;
}

// Solve i0 so that draws * w(0)/sum(w) == d_cap (bisection on log i0).
double solve_i0(uint32_t n, double draws, double a, double d_cap) {
  if (d_cap <= 0.0) return 1.0;
  double lo = std::log(1e-3), hi = std::log(1e9);
  for (int it = 0; it < 48; ++it) {
    double mid = 0.5 * (lo + hi);
    double i0 = std::exp(mid);
    double top = draws * std::pow(i0, -a) / sum_weights(n, i0, a);
    if (top > d_cap) lo = mid; else hi = mid;   // larger i0 -> flatter -> smaller top
  }
  return std::exp(0.5 * (lo + hi));
}

void permutation(uint32_t n, uint64_t base, std::vector<uint32_t>& perm) {
  perm.resize(n);
  for (uint32_t i = 0; i < n; ++i) perm[i] = i;
  for (uint32_t i = n; i > 1; --i) {
    uint32_t j = (uint32_t)mulhi64(rnd(base, i, 0), i);
    std::swap(perm[i - 1], perm[j]);
  }
}

}  // namespace

extern "C" {

// OpenMP threads of the generator (torchrun sets OMP_NUM_THREADS=1 per rank; the output does
// not depend on the thread count).
void plg_set_threads(int k) {
  if (k > 0) omp_set_num_threads(k);
}

// Generates the canonical in-CSR. Caller provides row_ptr[n+1] and src[m].
// Returns 0 on success, <0 on invalid arguments, -4 if the edge budget cannot be met
// (m too close to n*(n-1)).
int plg_generate(uint32_t n, uint64_t m, double gamma, double rho, double d_cap,
                 uint64_t graph_seed, uint64_t* row_ptr, uint32_t* src, double* i0_out) {
  if (n < 2 || gamma <= 1.0 || rho < 0.0 || rho > 1.0) return -1;
  if ((double)m > 0.5 * (double)n * (double)(n - 1)) return -2;
  const double a = 1.0 / (gamma - 1.0);
  const uint64_t base_draw = fmix64(graph_seed ^ 0x243F6A8885A308D3ULL);
  const uint64_t base_pout = fmix64(graph_seed ^ 0x13198A2E03707344ULL);
  const uint64_t base_pin = fmix64(graph_seed ^ 0xA4093822299F31D0ULL);
  const uint64_t rho_thr = (rho >= 1.0) ? ~0ULL : (uint64_t)std::ldexp(rho, 64);

  const double draws_est = (double)m / (1.0 + rho);
  const double i0 = solve_i0(n, draws_est, a, d_cap);
  if (i0_out) *i0_out = i0;
  const Alias al = build_alias(n, i0, a);
  std::vector<uint32_t> perm_out, perm_in;
  permutation(n, base_pout, perm_out);
  permutation(n, base_pin, perm_in);

  auto draw = [&](uint64_t t, uint32_t& u, uint32_t& v, bool& rev) {
    uint64_t w0 = rnd(base_draw, t, 0), w1 = rnd(base_draw, t, 1);
    uint64_t w2 = rnd(base_draw, t, 2), w3 = rnd(base_draw, t, 3);
    u = perm_out[al.sample(w0, (uint32_t)w1)];
    v = perm_in[al.sample(w2, (uint32_t)(w1 >> 32))];
    rev = (rho_thr == ~0ULL) ? true : (w3 < rho_thr);
  };

  uint64_t T = (uint64_t)(draws_est * 1.03) + 64;
  std::vector<uint64_t> cnt;     // per-destination candidate counts -> offsets
  std::vector<uint64_t> cell;    // (src << 32 | idx) per candidate, grouped by destination
  std::vector<uint32_t> keep;    // kept per row after dedup
  for (int attempt = 0; attempt < 64; ++attempt) {
    if (2 * T >= (1ULL << 32)) return -3;
    // pass 1: count candidates per destination
    std::vector<std::atomic<uint64_t>> c(n + 1);
    for (uint32_t i = 0; i <= n; ++i) c[i].store(0, std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (int64_t)T; ++t) {
      uint32_t u, v; bool rev;
      draw((uint64_t)t, u, v, rev);
      if (u == v) continue;
      c[v].fetch_add(1, std::memory_order_relaxed);
      if (rev) c[u].fetch_add(1, std::memory_order_relaxed);
    }
    cnt.assign(n + 1, 0);
    for (uint32_t i = 0; i < n; ++i) cnt[i + 1] = cnt[i] + c[i].load();
    const uint64_t C = cnt[n];
    cell.assign(C, 0);
    std::vector<std::atomic<uint64_t>> cur(n);
    for (uint32_t i = 0; i < n; ++i) cur[i].store(cnt[i], std::memory_order_relaxed);
    // pass 2: scatter (src, idx)
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (int64_t)T; ++t) {
      uint32_t u, v; bool rev;
      draw((uint64_t)t, u, v, rev);
      if (u == v) continue;
      cell[cur[v].fetch_add(1, std::memory_order_relaxed)] = ((uint64_t)u << 32) | (uint64_t)(2 * t);
      if (rev) cell[cur[u].fetch_add(1, std::memory_order_relaxed)] = ((uint64_t)v << 32) | (uint64_t)(2 * t + 1);
    }
    // per-row sort by (src, idx); dedup keeping the smallest idx
    keep.assign(n, 0);
    uint64_t U = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : U)
    for (int64_t v = 0; v < (int64_t)n; ++v) {
      uint64_t b = cnt[v], e = cnt[v + 1];
      std::sort(cell.begin() + b, cell.begin() + e);
      uint64_t w = b;
      for (uint64_t j = b; j < e; ++j) {
        if (w > b && (cell[w - 1] >> 32) == (cell[j] >> 32)) continue;
        cell[w++] = cell[j];
      }
      keep[v] = (uint32_t)(w - b);
      U += w - b;
    }
    if (U < m) {
      T = T + (uint64_t)((double)(m - U) * (double)T / (double)std::max<uint64_t>(U, 1) * 1.1) + 64;
      continue;
    }
    // keep exactly the m distinct edges with the smallest first index
    uint32_t thr_idx = 0xFFFFFFFFu;
    if (U > m) {
      std::vector<uint32_t> idx;
      idx.reserve(U);
      for (uint32_t v = 0; v < n; ++v)
        for (uint64_t j = cnt[v]; j < cnt[v] + keep[v]; ++j) idx.push_back((uint32_t)cell[j]);
      std::nth_element(idx.begin(), idx.begin() + (m - 1), idx.end());
      thr_idx = idx[m - 1];
    }
    row_ptr[0] = 0;
    uint64_t out = 0;
    for (uint32_t v = 0; v < n; ++v) {
      for (uint64_t j = cnt[v]; j < cnt[v] + keep[v]; ++j) {
        if ((uint32_t)cell[j] <= thr_idx) src[out++] = (uint32_t)(cell[j] >> 32);
      }
      row_ptr[v + 1] = out;
    }
    return (out == m) ? 0 : -5;
  }
  return -4;
}


// Barabasi-Albert scale-free graph (the paper's density experiment): a clique of r0
// nodes, then nodes v = r0..n-1 arrive one by one and attach to r distinct existing nodes, each
// drawn with probability d_i / sum_j d_j (uniform pick from the endpoint list, redrawn on a
// repeat). Undirected: every edge {a, b} becomes a->b and b->a. Output: canonical in-CSR
// (sources ascending). m = 2 * (r0 (r0 - 1) / 2 + r (n - r0)). Draw t uses rnd(base, t, 0).
// Returns 0, or -1 on invalid arguments (need 1 <= r <= r0, 2 <= r0 <= n), -2 if m != m_expect.
int ba_generate(uint32_t n, uint32_t r, uint32_t r0, uint64_t graph_seed, uint64_t m_expect,
                uint64_t* row_ptr, uint32_t* src) {
  if (r < 1 || r0 < r || r0 < 2 || n < r0) return -1;
  const uint64_t m_und = (uint64_t)r0 * (r0 - 1) / 2 + (uint64_t)r * (n - r0);
  if (2 * m_und != m_expect) return -2;
  std::vector<uint32_t> ea(m_und), eb(m_und);
  std::vector<uint32_t> ends;
  ends.reserve(2 * m_und);
  uint64_t k = 0;
  for (uint32_t i = 0; i < r0; ++i)
    for (uint32_t j = 0; j < i; ++j) {
      ea[k] = j; eb[k] = i; ++k;
      ends.push_back(i); ends.push_back(j);
    }
  const uint64_t base = fmix64(graph_seed ^ 0x452821E638D01377ULL);
  std::vector<uint32_t> tg(r);
  uint64_t t = 0;
  for (uint32_t v = r0; v < n; ++v) {
    uint32_t got = 0;
    while (got < r) {
      const uint32_t u = ends[(size_t)mulhi64(rnd(base, t++, 0), ends.size())];
      bool dup = false;
      for (uint32_t q = 0; q < got; ++q) dup |= (tg[q] == u);
      if (!dup) tg[got++] = u;
    }
    for (uint32_t q = 0; q < r; ++q) {
      ea[k] = tg[q]; eb[k] = v; ++k;
      ends.push_back(tg[q]); ends.push_back(v);
    }
  }
  // in-CSR of both directions: counting sort by destination, then sort each row
  std::vector<uint64_t> deg(n + 1, 0);
  for (uint64_t e = 0; e < m_und; ++e) { ++deg[ea[e]]; ++deg[eb[e]]; }
  row_ptr[0] = 0;
  for (uint32_t v = 0; v < n; ++v) row_ptr[v + 1] = row_ptr[v] + deg[v];
  std::vector<uint64_t> cur(row_ptr, row_ptr + n);
  for (uint64_t e = 0; e < m_und; ++e) {
    src[cur[eb[e]]++] = ea[e];          // ea -> eb
    src[cur[ea[e]]++] = eb[e];          // eb -> ea
  }
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < (int64_t)n; ++v) std::sort(src + row_ptr[v], src + row_ptr[v + 1]);
  return 0;
}

}  // extern "C"

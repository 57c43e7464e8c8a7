// Seeded synthetic edge-list generators (see include/bbtc_gen.h).
//
// Inputs only: this file holds no triangle-counting arithmetic.  The CUDA path
// and the oracle each canonicalise these raw samples on their own.
#include "bbtc_gen.h"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <omp.h>

static thread_local std::string g_err;
static int fail(const std::string& m) { g_err = m; return -1; }
extern "C" const char* bbtcgen_last_error(void) { return g_err.c_str(); }

static inline uint64_t fmix64(uint64_t z) {
  // SplitMix64 finaliser (Steele, Lea, Flood 2014).
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

extern "C" uint64_t bbtcgen_u64(uint64_t seed, uint64_t counter) {
  return fmix64(counter * 0x9E3779B97F4A7C15ull + fmix64(seed + 0x632BE59BD9B4E019ull));
}

static inline double unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }  // [0,1)
static inline uint64_t below(uint64_t h, uint64_t n) {                         // [0,n)
  return (uint64_t)(((unsigned __int128)h * n) >> 64);
}
static inline int nthreads(int t) { return t > 0 ? t : omp_get_max_threads(); }

// Samples [start, start + count) of the R-MAT sequence (src/dst hold count entries):
// each sample is a pure function of (seed, e), so ranks can generate their shards.
extern "C" int bbtcgen_rmat_range(uint32_t scale, uint32_t ef, double a, double b, double c, uint64_t seed,
                                  uint64_t start, uint64_t count, uint32_t* src, uint32_t* dst, int threads) {
  if (scale == 0 || scale > 32) return fail("rmat: scale must be in 1..32");
  double d = 1.0 - a - b - c;
  if (a <= 0 || b < 0 || c < 0 || d < 0) return fail("rmat: need a>0, b,c,d>=0, a+b+c<=1");
  if (!src || !dst) return fail("rmat: null output");
  const uint64_t ns = (uint64_t)ef << scale;
  if (start > ns || count > ns - start) return fail("rmat: sample range past the end");
  const double ab = a + b, a_norm = a / ab, c_norm = c / (c + d);
  src -= start;
  dst -= start;
#pragma omp parallel for schedule(static) num_threads(nthreads(threads))
  for (int64_t e = (int64_t)start; e < (int64_t)(start + count); ++e) {
    uint64_t s = 0, t = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      uint64_t ctr = (((uint64_t)e << 6) | l) << 1;
      uint64_t ii = unit(bbtcgen_u64(seed, ctr)) > ab;
      uint64_t jj = unit(bbtcgen_u64(seed, ctr | 1)) > (ii ? c_norm : a_norm);
      s |= ii << l;
      t |= jj << l;
    }
    src[e] = (uint32_t)s;
    dst[e] = (uint32_t)t;
  }
  return 0;
}

extern "C" int bbtcgen_rmat(uint32_t scale, uint32_t ef, double a, double b, double c, uint64_t seed,
                            uint32_t* src, uint32_t* dst, int threads) {
  if (scale == 0 || scale > 32) return fail("rmat: scale must be in 1..32");
  return bbtcgen_rmat_range(scale, ef, a, b, c, seed, 0, (uint64_t)ef << scale, src, dst, threads);
}

// Mean of a Pareto(gamma) truncated to [lo, hi].
static double trunc_pareto_mean(double g, double lo, double hi) {
  if (std::fabs(g - 2.0) < 1e-12) return std::log(hi / lo) / (1.0 / lo - 1.0 / hi);
  return ((g - 1.0) / (g - 2.0)) * (std::pow(lo, 2.0 - g) - std::pow(hi, 2.0 - g)) /
         (std::pow(lo, 1.0 - g) - std::pow(hi, 1.0 - g));
}

extern "C" int bbtcgen_chunglu_range(uint32_t n, uint64_t m, double g, double dmax, uint64_t seed, uint64_t start,
                                     uint64_t count, uint32_t* src, uint32_t* dst, double* dmin_out, int threads) {
  if (start > m || count > m - start) return fail("chunglu: sample range past the end");
  if (n < 2) return fail("chunglu: n must be >= 2");
  if (!(g > 1.0)) return fail("chunglu: gamma must be > 1");
  const double target = 2.0 * (double)m / (double)n;
  if (!(dmax > target)) return fail("chunglu: dmax must exceed the mean degree 2m/n");
  if (!src || !dst) return fail("chunglu: null output");
  // Solve dmin: the truncated mean increases with the lower bound.
  double lo = 1e-9, hi = dmax;
  for (int it = 0; it < 300; ++it) {
    double mid = 0.5 * (lo + hi);
    if (trunc_pareto_mean(g, mid, dmax) < target) lo = mid; else hi = mid;
  }
  const double dmin = 0.5 * (lo + hi);
  if (dmin_out) *dmin_out = dmin;
  // Weights at the quantiles (r+1/2)/n of the truncated Pareto, rescaled to the exact mean.
  std::vector<double> w(n);
  const double A = std::pow(dmin, 1.0 - g), B = std::pow(dmax, 1.0 - g);
  double sum = 0;
  for (uint32_t r = 0; r < n; ++r) {
    double q = ((double)r + 0.5) / (double)n;
    w[r] = std::pow(A - q * (A - B), 1.0 / (1.0 - g));
    sum += w[r];
  }
  // Walker/Vose alias table over w (sequential => deterministic).
  std::vector<double> prob(n);
  std::vector<uint32_t> alias(n);
  {
    std::vector<uint32_t> small, large;
    small.reserve(n); large.reserve(n);
    for (uint32_t r = 0; r < n; ++r) {
      prob[r] = w[r] * (double)n / sum;
      (prob[r] < 1.0 ? small : large).push_back(r);
    }
    while (!small.empty() && !large.empty()) {
      uint32_t s = small.back(); small.pop_back();
      uint32_t l = large.back();
      alias[s] = l;
      prob[l] = (prob[l] + prob[s]) - 1.0;
      if (prob[l] < 1.0) { large.pop_back(); small.push_back(l); }
    }
    for (uint32_t r : large) { prob[r] = 1.0; alias[r] = r; }
    for (uint32_t r : small) { prob[r] = 1.0; alias[r] = r; }
  }
  std::vector<double>().swap(w);
  // Seeded relabelling so ids carry no degree order (Fisher-Yates).
  std::vector<uint32_t> perm(n);
  for (uint32_t r = 0; r < n; ++r) perm[r] = r;
  const uint64_t pseed = bbtcgen_u64(seed, 0xC4A7E5ull << 40);
  for (uint32_t i = n - 1; i > 0; --i) {
    uint32_t j = (uint32_t)below(bbtcgen_u64(pseed, i), (uint64_t)i + 1);
    uint32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
  src -= start;
  dst -= start;
#pragma omp parallel for schedule(static) num_threads(nthreads(threads))
  for (int64_t e = (int64_t)start; e < (int64_t)(start + count); ++e) {
    uint32_t ends[2];
    for (int side = 0; side < 2; ++side) {
      uint64_t ctr = (((uint64_t)e << 1) | side) << 1;
      uint32_t r = (uint32_t)below(bbtcgen_u64(seed, ctr), n);
      ends[side] = unit(bbtcgen_u64(seed, ctr | 1)) < prob[r] ? r : alias[r];
    }
    src[e] = perm[ends[0]];
    dst[e] = perm[ends[1]];
  }
  return 0;
}

extern "C" int bbtcgen_chunglu(uint32_t n, uint64_t m, double g, double dmax, uint64_t seed,
                               uint32_t* src, uint32_t* dst, double* dmin_out, int threads) {
  return bbtcgen_chunglu_range(n, m, g, dmax, seed, 0, m, src, dst, dmin_out, threads);
}

extern "C" int bbtcgen_gnp(uint32_t n, double q, uint64_t seed, uint32_t* src, uint32_t* dst,
                           uint64_t cap, uint64_t* count) {
  if (!count) return fail("gnp: null count");
  uint64_t k = 0;
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t v = u + 1; v < n; ++v)
      if (unit(bbtcgen_u64(seed, u * n + v)) < q) {
        if (k < cap) { src[k] = (uint32_t)u; dst[k] = (uint32_t)v; }
        ++k;
      }
  *count = k;
  return 0;
}

extern "C" int bbtcgen_uniform_pairs(uint32_t n, uint64_t count, uint64_t seed, uint32_t* src,
                                     uint32_t* dst) {
  if (n == 0 && count) return fail("uniform_pairs: n must be > 0");
  for (uint64_t e = 0; e < count; ++e) {
    src[e] = (uint32_t)below(bbtcgen_u64(seed, 2 * e), n);
    dst[e] = (uint32_t)below(bbtcgen_u64(seed, 2 * e + 1), n);
  }
  return 0;
}

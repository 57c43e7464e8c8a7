/* bbtc_gen.h — seeded synthetic edge-list generators (inputs only).
 *
 * This library produces RAW edge samples: it may emit self-loops, duplicates
 * and both orientations.  It contains none of the triangle-counting method's
 * arithmetic (no canonicalisation, ordering, partitioning or counting); both
 * the CUDA path and the CPU oracle consume its output and canonicalise it
 * independently (§2 "Problem Formulation").
 *
 * Every generator is counter-based: sample e draws its random numbers from
 * bbtcgen_u64(seed, stream(e, …)), so the output is a pure function of the
 * arguments and identical for any thread count.
 *
 * Ownership: the caller allocates src/dst (host memory, length as documented
 * per call) and keeps ownership.  Return value: 0 on success, -1 on an invalid
 * argument (message via bbtcgen_last_error()).
 */
#ifndef BBTC_GEN_H
#define BBTC_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* SplitMix64-finalised hash of (seed, counter): the single RNG primitive. */
uint64_t bbtcgen_u64(uint64_t seed, uint64_t counter);

/* Graph500 R-MAT (the paper's RMAT rows, Table 3; parameters
 * a,b,c from BASELINE.json configs): n_samples = edgefactor << scale pairs,
 * ids in [0, 2^scale).  For each sample and level l = 0..scale-1:
 *   ii = r1 > a+b;  jj = r2 > (ii ? c/(c+d) : a/(a+b));  src |= ii<<l; dst |= jj<<l
 * with d = 1-a-b-c.  src/dst: length edgefactor<<scale. */
int bbtcgen_rmat(uint32_t scale, uint32_t edgefactor, double a, double b, double c,
                 uint64_t seed, uint32_t* src, uint32_t* dst, int threads);

/* Chung-Lu power law (SURVEY.md §8(d) "Chung-Lu"): expected weights follow a
 * truncated Pareto(gamma) on [dmin, dmax], dmin solved so that the mean weight
 * is 2m/n; n_samples = m pairs, both endpoints i.i.d. proportional to weight
 * (Walker alias table), then a seeded random relabelling of ids.
 * src/dst: length m.  *dmin_out (may be NULL) receives the solved dmin. */
int bbtcgen_chunglu(uint32_t n, uint64_t m, double gamma, double dmax, uint64_t seed,
                    uint32_t* src, uint32_t* dst, double* dmin_out, int threads);

/* Erdős–Rényi G(n, q) over unordered pairs u<v (O(n^2); small n only).
 * Writes at most cap pairs; returns the number of pairs via *count
 * (which may exceed cap, in which case only cap were written). */
int bbtcgen_gnp(uint32_t n, double q, uint64_t seed, uint32_t* src, uint32_t* dst,
                uint64_t cap, uint64_t* count);

/* Uniform random pairs in [0,n)^2 (may include self-loops and duplicates). */
int bbtcgen_uniform_pairs(uint32_t n, uint64_t count, uint64_t seed, uint32_t* src, uint32_t* dst);

/* Samples [start, start + count) of the same sequences (src/dst hold count entries):
 * a rank generates its shard of the raw edge list without the rest. */
int bbtcgen_rmat_range(uint32_t scale, uint32_t edgefactor, double a, double b, double c, uint64_t seed,
                       uint64_t start, uint64_t count, uint32_t* src, uint32_t* dst, int threads);
int bbtcgen_chunglu_range(uint32_t n, uint64_t m, double gamma, double dmax, uint64_t seed, uint64_t start,
                          uint64_t count, uint32_t* src, uint32_t* dst, double* dmin_out, int threads);
const char* bbtcgen_last_error(void);

#ifdef __cplusplus
}
#endif
#endif

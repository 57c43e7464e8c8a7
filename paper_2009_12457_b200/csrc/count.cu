// count.cu — the hot path's intersection kernel (step a7) and plan statistics.
//
// Alg. 5 BB-TC-LIST: for task t = (i,j,k) and every edge (u,v) of
// G_ij, count |N(G_ik,u) ∩ N(G_jk,v)|, summed into the task's uint64 counter.
//
// B200 design: one persistent grid, one warp per work item (task t,
// a range of consecutive edges of G_ij sized to equal estimated work), items
// claimed from a global atomic cursor.  A warp takes 32 consecutive edges of G_ij
// in its walk order (column order by default), so one of the two lists of an edge
// repeats across neighbouring lanes: that "staged" list S (N(G_jk,v) by column,
// N(G_ik,u) by row) is inserted once into a per-warp shared-memory hash table, and
// every word w of the other, "probe" list P is looked up in it: w ∈ S  <=>  w is a
// common neighbour, i.e. one triangle.  This computes exactly Σ_(u,v) |S ∩ P|,
// what Alg. 1's merge returns per edge, with every lane busy whatever the skew of
// the list lengths, and needs no order inside the lists.
#include <cub/cub.cuh>

#include <cstring>

#include "internal.h"

namespace bbtc {
namespace {

constexpr int kWarps = 8;            // warps per CTA
constexpr int kTable = 1024;         // per-warp shared words: one hash table of 4-word buckets (4 KiB)
#ifndef BBTC_HASH_LOAD_HALF
#define BBTC_HASH_LOAD_HALF 0
#endif
constexpr bool kLoadHalf = BBTC_HASH_LOAD_HALF;   // shared multi-list tables at load <= 1/2 (else 1/4)
constexpr int kHashCap = kLoadHalf ? kTable / 2 : kTable / 4;   // staged words of a shared (multi-list) table
constexpr int kChunk = kTable / 2;   // staged words of a single-list table fill (load <= 1/2)
constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr unsigned kFull = 0xffffffffu;
constexpr size_t kSmemBytes = (size_t)kWarps * (kTable * 4 + 32 * 16);   // table + payload (uint2[32]) + spare
static_assert(32 * 16 >= 32 * 8 + 8, "the payload area's spare half holds a warp's study-mode clock");
constexpr int kCtasPerSm = 8;        // cap on resident CTAs per SM (BBTC_CTAS_PER_SM overrides)
#ifndef BBTC_MIN_CTAS
#define BBTC_MIN_CTAS 5
#endif
constexpr int kMinCtas = BBTC_MIN_CTAS;   // register budget: >= 5 CTAs (40 warps) resident per SM
#ifndef BBTC_PREFETCH
#define BBTC_PREFETCH 0
#endif
constexpr bool kPrefetch = BBTC_PREFETCH;   // L2 prefetch of a batch's probe lists
#ifndef BBTC_BITMAP
#define BBTC_BITMAP 1
#endif
constexpr bool kBitmap = BBTC_BITMAP;   // single-list batches over a small V_k use a bitmap
static_assert(kBitmapMaxWords == (uint32_t)kTable, "a bitmap over V_k must fit the per-warp table");
#ifndef BBTC_RUN_PIPE
#define BBTC_RUN_PIPE 1
#endif
constexpr bool kRunPipe = BBTC_RUN_PIPE;   // pipelined column runs (hash-only variant)
#ifndef BBTC_RUN_PIPE_BM
#define BBTC_RUN_PIPE_BM 0
#endif
#ifndef BBTC_LANEWALK
// Lanes walk their own < 32-word probe remainders when the lengths are even enough
// (instead of the flattened walk): rmat24 p=10 list kernel 33.1 -> 32.2 ms, orkut and
// friendster unchanged (profiles/r02/ab5; K = 3 / always: no better, friendster worse).
#define BBTC_LANEWALK 1
#endif
#ifndef BBTC_STREAM_HINT
#define BBTC_STREAM_HINT 0   // A/B: evict-first (ld.global.cs) loads for the walked edges and staged lists
#endif
// Loads of data read once in order (the walk arrays, the staged lists): with the hint
// they are marked evict-first so the L2 keeps the randomly gathered probe lists.
template <class T>
__device__ __forceinline__ T ld_stream(const T* p) {
#if BBTC_STREAM_HINT
  return __ldcs(p);
#else
  return *p;
#endif
}
#ifndef BBTC_DEBUG_BOUNDS
#define BBTC_DEBUG_BOUNDS 0   // debug builds: bounds checks in the list kernel (report via mapped host memory)
#endif
#if BBTC_DEBUG_BOUNDS
// [0] = failing check id (first one wins), [1..7] = its values; [8] = m, [9] = row-offset words.
__device__ unsigned long long* g_dbg;
__device__ __noinline__ void dbg_fail(unsigned long long code, unsigned long long a, unsigned long long b,
                                      unsigned long long c, unsigned long long d, unsigned long long e,
                                      unsigned long long f, unsigned long long g) {
  if (atomicCAS(g_dbg, 0ull, code) == 0ull) {
    g_dbg[1] = a; g_dbg[2] = b; g_dbg[3] = c; g_dbg[4] = d; g_dbg[5] = e; g_dbg[6] = f; g_dbg[7] = g;
    __threadfence_system();
  }
  __trap();
}
#define DBG_CHECK(cond, code, a, b, c, d, e, f, g) \
  do {                                             \
    if (!(cond)) dbg_fail(code, a, b, c, d, e, f, g); \
  } while (0)
#else
#define DBG_CHECK(cond, code, a, b, c, d, e, f, g) do { } while (0)
#endif
#ifndef BBTC_P1_UNIFIED
#define BBTC_P1_UNIFIED 1   // phase 1: the last < 4 rounds of a long list in one predicated round
#endif
constexpr bool kP1Unified = BBTC_P1_UNIFIED;
#ifndef BBTC_LANEWALK_K
#define BBTC_LANEWALK_K 2  // lane walk when 32 * max remainder <= K * sum of remainders + 64
#endif
constexpr int kCarveoutPct = 0;      // shared-memory carveout in percent (0 = driver default)

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x += y;
  }
  return x;
}

// Length of the run of set bits from lane 0: a batch or run takes only the leading
// lanes of its key (equal keys are contiguous in a column-ordered block; the prefix
// rule keeps the kernel correct for any walk order).
__device__ __forceinline__ int lane_prefix(uint32_t b) { return b == kFull ? 32 : __ffs(~b) - 1; }

__device__ __forceinline__ uint32_t lanemask_le(int lane) { return 0xffffffffu >> (31 - lane); }
__device__ __forceinline__ uint32_t lanemask_lt(int lane) { return (1u << lane) - 1u; }

__device__ __forceinline__ uint32_t hbucket(uint32_t key, int shift) { return (key * 0x9E3779B1u) >> shift; }

// Segmented flatten: the warp walks the concatenation of per-lane segments
// [start, start+len) (start = exclusive prefix of len over lanes) 32 positions at a
// time.  Non-empty segments are compacted into `pay` (one uint4 payload each); the
// owner of each position is found with one redux.or of the segment starts falling in
// the current window plus a popc.  `load(f, P)` fetches the position's word two
// windows ahead of `use(f, P, w)` (software pipelining of the gather).
template <class Ld, class Use>
__device__ __forceinline__ void flatten(uint2* pay, int lane, bool nonempty, uint32_t start, uint2 payload,
                                        uint32_t total, Ld load, Use use) {
  const uint32_t nmask = __ballot_sync(kFull, nonempty);
  if (nonempty) pay[__popc(nmask & lanemask_lt(lane))] = payload;
  __syncwarp();
  if (total == 0) return;
  uint32_t before = 0;   // segment starts < the next window to be resolved
  auto owner = [&](uint32_t f0) {
    const uint32_t d = start - f0;
    const uint32_t starts = __reduce_or_sync(kFull, (nonempty && d < 32) ? (1u << d) : 0u);
    const uint32_t idx = before + __popc(starts & lanemask_le(lane)) - 1;
    DBG_CHECK(f0 + lane >= total || idx < 32, 4, f0, idx, before, starts, total, start, 0);
    before += __popc(starts);
    return idx;
  };
  uint2 P0 = pay[owner(0)], P1 = P0;
  uint32_t w0 = lane < total ? load(lane, P0) : 0, w1 = 0;
  if (32 < total) {
    P1 = pay[owner(32)];
    if (32 + lane < total) w1 = load(32 + lane, P1);
  }
  for (uint32_t f0 = 0; f0 < total; f0 += 32) {
    uint2 P2 = P1;
    uint32_t w2 = 0;
    const uint32_t f2 = f0 + 64 + lane;
    if (f0 + 64 < total) {
      P2 = pay[owner(f0 + 64)];
      if (f2 < total) w2 = load(f2, P2);
    }
    if (f0 + lane < total) use(f0 + lane, P0, w0);
    P0 = P1; w0 = w1;
    P1 = P2; w1 = w2;
  }
  __syncwarp();
}

// Hash tables of buckets of BW words, linear probing over buckets; a table is sized in
// 4-word units (nb4 of them) and addressed in buckets of BW words.  4-word buckets take
// one LDS.128 per probe; 2-word buckets (LDS.64) measured faster in the bitmap kernel
// variant (rmat24 list kernel 31.9 -> 31.2 ms, orkut 11.76 -> 11.47) and slower in the
// hash-only one (friendster 333 -> 351 ms; 1-word buckets slower everywhere:
// profiles/r02/r02m), so the width follows the variant (BBTC_BUCKET_WORDS[_BM]).
#ifndef BBTC_BUCKET_WORDS
#define BBTC_BUCKET_WORDS 4
#endif
#ifndef BBTC_BUCKET_WORDS_BM
#define BBTC_BUCKET_WORDS_BM 2
#endif
struct TabGeom {
  uint32_t bmask;
  int shift;
};
template <int BW>
__device__ __forceinline__ TabGeom tab_geom(uint32_t nb4) {
  static_assert(BW == 1 || BW == 2 || BW == 4, "bucket width");
  const uint32_t nb = nb4 * (4 / BW);
  return {nb - 1, 32 - (__ffs(nb) - 1)};
}

// Inserts key hk into the table.
template <int BW>
__device__ __forceinline__ void table_insert(uint32_t* tab, uint32_t hk, TabGeom G) {
  uint32_t h = hbucket(hk, G.shift);
  for (;;) {
    uint32_t* bk = tab + BW * h;
#pragma unroll
    for (int x = 0; x < BW; ++x)
      if (atomicCAS(bk + x, kEmpty, hk) == kEmpty) return;
    h = (h + 1) & G.bmask;
  }
}

template <int BW>
__device__ __forceinline__ uint32_t table_probe(const uint32_t* tab, uint32_t hk, TabGeom G) {
  uint32_t h = hbucket(hk, G.shift);
  if constexpr (BW == 4) {
    const uint4* tab4 = reinterpret_cast<const uint4*>(tab);
    uint4 q = tab4[h];
    bool hit = (q.x == hk) | (q.y == hk) | (q.z == hk) | (q.w == hk);
    while (!hit && q.w != kEmpty) {   // full bucket: next one (rare at these loads)
      h = (h + 1) & G.bmask;
      q = tab4[h];
      hit = (q.x == hk) | (q.y == hk) | (q.z == hk) | (q.w == hk);
    }
    return hit;
  } else if constexpr (BW == 2) {
    const uint2* tab2 = reinterpret_cast<const uint2*>(tab);
    uint2 q = tab2[h];
    bool hit = (q.x == hk) | (q.y == hk);
    while (!hit && q.y != kEmpty) {
      h = (h + 1) & G.bmask;
      q = tab2[h];
      hit = (q.x == hk) | (q.y == hk);
    }
    return hit;
  } else {
    uint32_t q = tab[h];
    while (q != hk && q != kEmpty) {
      h = (h + 1) & G.bmask;
      q = tab[h];
    }
    return q == hk;
  }
}

// Probe lists of lanes: P = cols[bx .. bx + bl).  Phase 1 walks the long lists one at
// a time in whole 32-word rounds (all lanes on consecutive words of one list, four
// loads in flight); phase 2 flattens the < 32-word remainders across the lanes.
// test(w, slot) = 1 if probe word w of a lane whose staged list has slot `slot` is in it.
template <bool kUnified, class Test>
__device__ __forceinline__ uint32_t probe_lists(const uint32_t* __restrict__ cols, uint2* pay, int lane, uint32_t bx,
                                                uint32_t bl, uint32_t slot, Test test) {
  uint32_t hits = 0;
#if BBTC_DEBUG_BOUNDS
  DBG_CHECK((unsigned long long)bx + bl <= g_dbg[8], 3, bx, bl, slot, g_dbg[8], 0, 0, 0);
#endif
  uint32_t longs = __ballot_sync(kFull, bl >= 32);
  while (longs) {
    const int src = __ffs(longs) - 1;
    longs &= longs - 1;
    const uint32_t* B = cols + __shfl_sync(kFull, bx, src) + lane;
    const uint32_t nfull = __shfl_sync(kFull, bl, src) & ~31u;
    const uint32_t sl = __shfl_sync(kFull, slot, src);
    uint32_t off = 0;
    // kUnified: rounds of up to four 32-word loads in flight, the last one predicated —
    // a list of 32-127 words costs one load latency instead of one per round.  In the
    // hash-only kernel variant (friendster 336.4 -> 331.4 ms); the bitmap variant, tighter
    // on registers, measured slower with it (rmat24 31.9 -> 32.2, orkut 11.89 -> 12.11;
    // profiles/r02/r02w).
    if constexpr (kUnified) {
      for (; off < nfull; off += 128) {
        const bool h2 = off + 32 < nfull, h3 = off + 64 < nfull, h4 = off + 96 < nfull;
        const uint32_t w1 = B[off], w2 = h2 ? B[off + 32] : 0u, w3 = h3 ? B[off + 64] : 0u;
        const uint32_t w4 = h4 ? B[off + 96] : 0u;
        hits += test(w1, sl) + (h2 ? test(w2, sl) : 0u) + (h3 ? test(w3, sl) : 0u) + (h4 ? test(w4, sl) : 0u);
      }
    } else {
      for (; off + 128 <= nfull; off += 128) {
        const uint32_t w1 = B[off], w2 = B[off + 32], w3 = B[off + 64], w4 = B[off + 96];
        hits += test(w1, sl) + test(w2, sl) + test(w3, sl) + test(w4, sl);
      }
      for (; off < nfull; off += 32) hits += test(B[off], sl);
    }
  }
  const uint32_t rem = bl & 31u;
#if BBTC_LANEWALK
  // Remainders of similar length: every lane walks its own (4 loads in flight) instead
  // of the flattened walk, whose per-window owner search costs ~10 instructions.
  const uint32_t rmax = __reduce_max_sync(kFull, rem);
  const uint32_t rsum = __reduce_add_sync(kFull, rem);
  if (rmax * 32 <= BBTC_LANEWALK_K * rsum + 64) {
    const uint32_t* B = cols + bx + (bl & ~31u);
    uint32_t x = 0;
    for (; x + 4 <= rmax; x += 4) {
      const uint32_t w0 = x < rem ? B[x] : 0u, w1 = x + 1 < rem ? B[x + 1] : 0u;
      const uint32_t w2 = x + 2 < rem ? B[x + 2] : 0u, w3 = x + 3 < rem ? B[x + 3] : 0u;
      if (x < rem) hits += test(w0, slot);
      if (x + 1 < rem) hits += test(w1, slot);
      if (x + 2 < rem) hits += test(w2, slot);
      if (x + 3 < rem) hits += test(w3, slot);
    }
    for (; x < rmax; ++x)
      if (x < rem) hits += test(B[x], slot);
    return hits;
  }
#endif
  const uint32_t rinc = warp_incl_scan(rem, lane);
  const uint32_t total_r = __shfl_sync(kFull, rinc, 31);
  const uint32_t rstart = rinc - rem;
  flatten(pay, lane, rem > 0, rstart, make_uint2(bx + (bl & ~31u) - rstart, slot), total_r,
          [&](uint32_t f, uint2 P) { return cols[P.x + f]; },
          [&](uint32_t, uint2 P, uint32_t w) { hits += test(w, P.y); });
  return hits;
}

// The rare path, kept out of line so it does not weigh on the main loop's code: one
// staged list S = cS[s0 .. s0+total_a) longer than a shared table (or any list
// when slot tags do not fit in 32 bits), hashed alone with untagged keys in chunks
// of kChunk words.  |S ∩ P| is additive over a partition of S, so every probe list
// is probed once per chunk.  Returns this lane's hits.
template <bool kUnified>
__device__ __noinline__ uint32_t long_list(const uint32_t* __restrict__ cols, const uint32_t* __restrict__ cS,
                                           uint32_t s0, uint32_t total_a, uint32_t bx, uint32_t bl, uint32_t* tab,
                                           uint2* pay, int lane) {
  uint4* tab4 = reinterpret_cast<uint4*>(tab);
  uint32_t hits = 0;
  for (uint32_t c0 = 0; c0 < total_a; c0 += kChunk) {
    const uint32_t cn = min((uint32_t)kChunk, total_a - c0);
    uint32_t nb = 16;
    while (2 * nb < cn) nb <<= 1;
    const TabGeom G = tab_geom<4>(nb);
    for (uint32_t x = lane; x < nb; x += 32) tab4[x] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    __syncwarp();
    for (uint32_t x = lane; x < cn; x += 32) table_insert<4>(tab, ld_stream(cS + s0 + c0 + x), G);
    __syncwarp();
    hits += probe_lists<kUnified>(cols, pay, lane, bx, bl, 0,
                        [&](uint32_t w, uint32_t) { return table_probe<4>(tab, w, G); });
  }
  return hits;
}

// Streamed column-major blocks carry column offsets cp[0..nc] (block-local edge
// offsets, cp[nc] = nnz) instead of a column id per edge.  col_search: the largest
// c in [lo, hi) with cp[c] <= x, i.e. the column of edge x (empty columns share the
// offset of the next one and are skipped), given cp[lo] <= x.  32-ary warp search:
// one coalesced probe of 32 offsets per step.
__device__ __forceinline__ uint32_t col_search(const uint32_t* __restrict__ cp, uint32_t lo, uint32_t hi, uint32_t x,
                                               int lane) {
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo + 31) >> 5;
    const uint32_t idx = lo + lane * step;
    const uint32_t m = __ballot_sync(kFull, idx < hi && cp[idx] <= x);
    lo += (31 - __clz(m)) * step;
    hi = min(lo + step, hi);
  }
  const uint32_t idx = lo + lane;
  const uint32_t m = __ballot_sync(kFull, idx < hi && cp[idx] <= x);
  return lo + 31 - __clz(m);
}

// Column of every lane's edge (local offset x, `valid` lanes) from column offsets,
// given a column c with cp[c] <= every lane's x: one coalesced window of the next 32
// column ends per round, a 5-step shuffle search per lane; lanes past the window
// restart from the column of the first of them (col_search).  Returns the column
// (0xFFFFFFFF for invalid lanes).
__device__ __forceinline__ uint32_t col_of(const uint32_t* __restrict__ cp, uint32_t nc, uint32_t c, uint32_t x,
                                           bool valid, int lane) {
  uint32_t v = 0xFFFFFFFFu;
  bool need = valid;
  for (;;) {
    const uint32_t w = cp[min(c + 1 + lane, nc)];   // end of column c + lane
    uint32_t pos = 0;
#pragma unroll
    for (int st = 16; st >= 1; st >>= 1) {
      const uint32_t t = __shfl_sync(kFull, w, pos + st - 1);
      if (t <= x) pos += st;
    }
    const uint32_t w31 = __shfl_sync(kFull, w, 31);   // (every lane: a warp-wide shuffle)
    if (pos == 31 && w31 <= x) pos = 32;
    if (need && pos < 32) {
      v = c + pos;
      need = false;
    }
    const uint32_t un = __ballot_sync(kFull, need);
    if (!un) break;
    // Past the window: gallop — lane l probes column c + 32*2^l (one load per lane), the
    // first probe past the first unresolved edge bounds a col_search over that octave.
    const uint32_t xf = __shfl_sync(kFull, x, __ffs(un) - 1);
    typedef unsigned long long u64;
    const u64 at = min((u64)c + (32ull << lane), (u64)nc);
    const uint32_t t = __popc(__ballot_sync(kFull, at < nc && cp[at] <= xf));   // >= 1: cp[c+32] <= xf
    const uint32_t lo = (uint32_t)((u64)c + (32ull << (t - 1)));
    c = col_search(cp, lo, (uint32_t)min((u64)c + (32ull << t), (u64)nc), xf, lane);
  }
  return v;
}

// Alg. 5 over work items.  kSlots: batches of several staged lists share one table
// with slot-tagged keys (w << 5 | slot), which needs |V_k| < 2^27; otherwise every
// batch takes one staged list at a time (long_list).  kCol: walk G_ij by column
// (ccu/ccv arrays, stage N(G_jk,v)) or by row (rows/cols, stage N(G_ik,u)).  kCP
// (streamed column-major blocks): the column of an edge comes from the block's column
// offsets (colptr + BlockDesc.co) instead of a ccv array.
template <bool kSlots, bool kCol, bool kBm, bool kCP>
__global__ void __launch_bounds__(kWarps * 32, kMinCtas)
k_count(const uint32_t* __restrict__ cols, const uint32_t* __restrict__ it_u, const uint32_t* __restrict__ it_v,
        const uint32_t* __restrict__ rowptr, const BlockDesc* __restrict__ blocks, const TaskDesc* __restrict__ tasks,
        const uint64_t* __restrict__ item_start, uint32_t n_exec, uint64_t item_lo, uint64_t n_items,
        uint32_t rank, uint32_t world, unsigned long long* __restrict__ cursor,
        unsigned long long* __restrict__ counts, uint32_t n_tasks, const uint32_t* ready, uint32_t epoch,
        const uint32_t* __restrict__ colptr, const uint32_t* __restrict__ item_col,
        unsigned long long* __restrict__ task_cycles, const uint32_t* __restrict__ slot_of) {
  static_assert(!kCP || kCol, "column offsets replace the column ids of a column-major walk");
  extern __shared__ __align__(16) uint32_t smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  uint32_t* tab = smem + wid * kTable;
  uint4* tab4 = reinterpret_cast<uint4*>(tab);
  uint2* pay = reinterpret_cast<uint2*>(smem + kWarps * kTable) + wid * 32;

  for (;;) {
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(cursor, 1ull);
    it = __shfl_sync(kFull, it, 0);
    const uint64_t g = item_lo + it * world + rank;
    if (g >= n_items) break;
    // study mode (bbtc_task_times): the item's start clock in the spare half of the warp's
    // payload area (shared memory, so the main loop carries no extra live register)
    auto t_slot = [&]() {
      return reinterpret_cast<long long*>(reinterpret_cast<uint2*>(smem + kWarps * kTable) + kWarps * 32) + wid;
    };
    if (task_cycles && lane == 0) *t_slot() = clock64();
    // task of item g: last t with item_start[t] <= g
    uint32_t lo = 0, hi = n_exec - 1;
    while (lo < hi) {
      uint32_t mid = (lo + hi + 1) >> 1;
      if (item_start[mid] <= g) lo = mid; else hi = mid - 1;
    }
    DBG_CHECK(lo < n_exec, 6, lo, n_exec, g, 0, 0, 0, 0);
    const TaskDesc T = tasks[lo];
    DBG_CHECK(T.ij < g_dbg[10] && T.ik < g_dbg[10] && T.jk < g_dbg[10] && T.idx < n_tasks, 7, T.ij, T.ik, T.jk, T.idx,
              g_dbg[10], n_tasks, 0);
    if (ready) {
      // Streaming (a6): wait until the copy engine has delivered the task's blocks.
      if (lane == 0) {
        const uint32_t need[3] = {T.ij, T.ik, T.jk};
        for (int x = 0; x < 3; ++x) {
          uint32_t rv;
          uint64_t spins = 0;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(rv) : "l"(ready + need[x]) : "memory");
            if (rv != epoch) {
              __nanosleep(1000);
              if (++spins > (1ull << 25)) __trap();   // ~30 s without the copy: fail, never hang
            }
          } while (rv != epoch);
        }
      }
      __syncwarp();
    }
    const BlockDesc Bij = blocks[T.ij];
    const BlockDesc BS = blocks[kCol ? T.jk : T.ik];   // block of the staged lists
    const BlockDesc BP = blocks[kCol ? T.ik : T.jk];   // block of the probe lists
    const uint64_t e_begin = Bij.e0 + (g - item_start[lo]) * T.chunk;
    const uint64_t e_end = min(e_begin + T.chunk, Bij.e0 + Bij.nnz);
    const uint32_t* rpS = rowptr + BS.ro;
    const uint32_t* cS = cols + BS.e0;
    const uint32_t* rpP = rowptr + BP.ro;
    // Probe slots (resident plans): the probe block's row r at cols[so + 8r] = {len,
    // CSR offset, first 6 ids}; rows of <= 6 entries are probed in the slot itself.
    const uint32_t so = slot_of ? slot_of[kCol ? T.ik : T.jk] : 0u;
    // probe list of row r of the probe block: its index in the cols arena and length
    auto probe_of = [&](uint32_t r, uint32_t& x, uint32_t& len) {
      if (so) {
        const uint2 h = *reinterpret_cast<const uint2*>(cols + so + 8 * r);
        len = h.x;
        x = h.x <= 6 ? so + 8 * r + 2 : (uint32_t)BP.e0 + h.y;
      } else {
        const uint32_t b0 = rpP[r];
        len = rpP[r + 1] - b0;
        x = (uint32_t)BP.e0 + b0;
      }
    };
    // kCP: G_ij's column offsets, unless the block ships its column ids (kNoColptr)
    const bool cpm = kCP && Bij.co != kNoColptr;
    const uint32_t* cpb = cpm ? colptr + Bij.co : nullptr;
    uint32_t ccol = 0;                                        // a column with cpb[ccol] <= next edge
    if (cpm) ccol = item_col[T.icol + (g - item_start[lo])];  // (k_item_cols, plan time)

    uint32_t hits = 0;
    uint64_t base = e_begin;
    while (base < e_end) {
      // ---- 32 edges (u,v) of G_ij; key = the staged side's row (v by column, u by row)
      const uint64_t e = base + lane;
      const bool valid = e < e_end;
      const uint32_t u = valid ? ld_stream(it_u + e) : 0xFFFFFFFFu;
      uint32_t v;
      if (cpm) v = col_of(cpb, Bij.nc, ccol, (uint32_t)(e - Bij.e0), valid, lane);
      else v = valid ? ld_stream(it_v + e) : 0xFFFFFFFFu;
      const uint32_t key = kCol ? v : u;
      const uint32_t pid = kCol ? u : v;
      uint32_t a0 = 0, alen = 0, bx = 0, blen = 0;   // a: staged list, b: probe list (bx: index in cols)
      DBG_CHECK(!valid || ((!kCol || key < Bij.nc) && BS.ro + key + 1 < g_dbg[9] && BP.ro + pid + 1 < g_dbg[9]), 5,
                T.idx, e, u, v, BS.ro, BP.ro, Bij.nc);
      if (valid) {
        a0 = rpS[key];
        alen = rpS[key + 1] - a0;
        probe_of(pid, bx, blen);
      }
      DBG_CHECK(!valid || ((!kCol || v < Bij.nc) && a0 + alen <= BS.nnz && blen <= BP.nnz && alen <= BS.nnz &&
                           e < Bij.e0 + Bij.nnz),
                1, T.idx, e, u, v, ((unsigned long long)a0 << 32) | alen, ((unsigned long long)bx << 32) | blen,
                ((unsigned long long)BS.nnz << 32) | BP.nnz);
      const uint32_t kprev = __shfl_up_sync(kFull, key, 1);
      const bool leader = valid && (lane == 0 || key != kprev);
      const uint32_t lmask = __ballot_sync(kFull, leader);
      const uint32_t le = lmask & lanemask_le(lane);
      const int my_leader = le ? 31 - __clz(le) : 0;
      const uint32_t slot = __popc(lmask & lanemask_lt(my_leader));   // staged-list slot 0..31
      const uint32_t lead_len = leader ? alen : 0;
      const uint32_t incl = warp_incl_scan(lead_len, lane);
      const uint32_t aoff = __shfl_sync(kFull, incl - lead_len, my_leader);
      const uint32_t aend = aoff + alen;
      // Small V_k and few distinct staged lists in the batch (all of them fit the table
      // as bitmaps over V_k, T.bmw words each): bitmaps instead of a hash table (one
      // LDS + a bit test per probe word, any list length).
      const bool bm_path = kBm && T.bmw != 0 && __popc(lmask) * T.bmw <= (uint32_t)kTable;
      // lanes [0,L) whose staged lists fit one shared table (load <= 1/4)
      int L = bm_path ? __popc(__ballot_sync(kFull, valid))
                      : kSlots ? __popc(__ballot_sync(kFull, valid && aend <= kHashCap)) : 0;
      bool dense = false;   // one list of kHashCap..kChunk words: a table of its own, load <= 1/2
      bool longl = false;   // longer (or untaggable): the out-of-line chunked path
      if (L == 0) {
        const uint32_t k0 = __shfl_sync(kFull, key, 0);
        const uint32_t a_first = __shfl_sync(kFull, alen, 0);
        L = lane_prefix(__ballot_sync(kFull, valid && key == k0));
        if (kSlots && a_first <= kChunk) dense = true;
        else longl = true;
      }
      const bool in = lane < L;
      // edges whose staged list is empty cannot close a triangle: no probes for them
      const uint32_t bl = (in && alen > 0) ? blen : 0;
      // Ask L2 for every lane's probe list now (fire-and-forget, no registers): the
      // 32 random gathers of the batch then overlap the staging of S instead of each
      // list's first round waiting out a full DRAM latency in turn.
      if (kPrefetch && bl > 0) {
        const uint32_t* pf = cols + bx;
        const uint32_t lines = min((bl + 31) >> 5, 4u);
        for (uint32_t x = 0; x < lines; ++x) asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + 32 * x));
      }
      // A staged list that fills the whole batch usually continues (a column with many
      // edges): keep its table and probe the run's next edges against it, instead of
      // re-reading and re-hashing the list for every 32 edges.
      auto continue_run = [&](auto test) {
        const uint32_t k0 = __shfl_sync(kFull, key, 0);
        if (L == 32 && __all_sync(kFull, valid && key == k0)) {
          // kCP: the run's edges end where column k0 ends
          const uint64_t run_end = cpm ? Bij.e0 + cpb[k0 + 1] : 0;
          auto same = [&](uint64_t e) { return cpm ? e < run_end : ld_stream((kCol ? it_v : it_u) + e) == k0; };
          if constexpr (kRunPipe && (!kBm || BBTC_RUN_PIPE_BM)) {
            // Two-stage pipeline over the run's batches: while batch t is probed, the row
            // offsets of batch t+1 (whose edge ids arrived during batch t-1) and the edge
            // ids of batch t+2 are in flight.  Only in the hash-only variant: measured
            // friendster -2%, while the bitmap variant (tighter on registers) lost 1.6% on
            // rmat24 (profiles/r01c/ab_run_pipe.jsonl).
            auto edge = [&](uint64_t e, uint32_t& pid2) {
              const bool ok = e < e_end && same(e);
              pid2 = ok ? ld_stream((kCol ? it_u : it_v) + e) : 0u;
              return ok;
            };
            uint64_t e2 = base + L + lane;
            uint32_t p_cur, p_nxt;
            bool ok_cur = edge(e2, p_cur);
            bool ok_nxt = edge(e2 + 32, p_nxt);
            uint32_t x2 = 0, bl2 = 0;
            if (ok_cur && alen > 0) probe_of(p_cur, x2, bl2);
            for (;;) {
              const int L2 = lane_prefix(__ballot_sync(kFull, ok_cur));   // the run's edges
              if (L2 == 0) break;
              uint32_t xn = 0, bln = 0, p_nn = 0;
              bool ok_nn = false;
              if (L2 == 32) {
                if (ok_nxt && alen > 0) probe_of(p_nxt, xn, bln);
                ok_nn = edge(e2 + 64, p_nn);
              }
              hits += probe_lists<kP1Unified && !kBm>(cols, pay, lane, x2, lane < L2 ? bl2 : 0u, 0, test);
              L += L2;
              if (L2 < 32) break;
              e2 += 32;
              ok_cur = ok_nxt;
              x2 = xn;
              bl2 = bln;
              ok_nxt = ok_nn;
              p_nxt = p_nn;
            }
          } else {
            for (;;) {
              const uint64_t e2 = base + L + lane;
              const bool ok = e2 < e_end && same(e2);
              const int L2 = lane_prefix(__ballot_sync(kFull, ok));   // the run's edges
              if (L2 == 0) break;
              uint32_t x2 = 0, bl2 = 0;
              if (ok && alen > 0) probe_of(kCol ? it_u[e2] : it_v[e2], x2, bl2);
              hits += probe_lists<kP1Unified && !kBm>(cols, pay, lane, x2, lane < L2 ? bl2 : 0u, 0, test);
              L += L2;
              if (L2 < 32) break;
          }
          }
        }
      };
      if (__any_sync(kFull, bl > 0)) {
        if (bm_path) {
          uint32_t* bm = tab;
          const uint32_t bmw = T.bmw;
          const uint32_t words = __popc(lmask) * bmw;
          for (uint32_t x = 4 * lane; x < words; x += 128) *reinterpret_cast<uint4*>(bm + x) = make_uint4(0, 0, 0, 0);
          __syncwarp();
          if (lmask == 1u) {   // one list: coalesced reads, no flattening
            const uint32_t s0 = __shfl_sync(kFull, a0, 0), sn = __shfl_sync(kFull, alen, 0);
            for (uint32_t x = lane; x < sn; x += 32) {
              DBG_CHECK(s0 + x < BS.nnz, 8, s0, x, BS.nnz, T.idx, 0, 0, 0);
              const uint32_t w = ld_stream(cS + s0 + x);
              DBG_CHECK((w >> 5) < bmw, 9, w, bmw, T.idx, 0, 0, 0, 0);
              atomicOr(bm + (w >> 5), 1u << (w & 31));
            }
          } else {
            flatten(pay, lane, leader && alen > 0, aoff, make_uint2(a0 - aoff, slot * bmw),
                    __shfl_sync(kFull, aend, L - 1),
                    [&](uint32_t f, uint2 P) {
                      DBG_CHECK(P.x + f < BS.nnz, 10, P.x, f, BS.nnz, T.idx, 0, 0, 0);
                      return ld_stream(cS + P.x + f);
                    },
                    [&](uint32_t, uint2 P, uint32_t w) {
                      DBG_CHECK(P.y + (w >> 5) < (uint32_t)kTable && (w >> 5) < bmw, 11, P.y, w, bmw, T.idx, 0, 0, 0);
                      atomicOr(bm + P.y + (w >> 5), 1u << (w & 31));
                    });
          }
          __syncwarp();
          auto test = [bm](uint32_t w, uint32_t base_w) { return (bm[base_w + (w >> 5)] >> (w & 31)) & 1u; };
          hits += probe_lists<kP1Unified && !kBm>(cols, pay, lane, bx, bl, slot * bmw, test);
          continue_run(test);
        } else if (longl) {
          hits += long_list<kP1Unified && !kBm>(cols, cS, __shfl_sync(kFull, a0, 0), __shfl_sync(kFull, alen, 0), bx, bl, tab, pay,
                            lane);
        } else {
          // ---- stage the distinct lists S of lanes [0,L) into one table
          const uint32_t total_a = __shfl_sync(kFull, aend, L - 1);
          uint32_t nb = 16;
          while ((dense || kLoadHalf ? 2 * nb : nb) < total_a) nb <<= 1;
          constexpr int BW = kBm ? BBTC_BUCKET_WORDS_BM : BBTC_BUCKET_WORDS;
          const TabGeom G = tab_geom<BW>(nb);
          DBG_CHECK(nb <= kTable / 4, 2, T.idx, nb, total_a, L, dense, longl, 0);
          for (uint32_t x = lane; x < nb; x += 32) tab4[x] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
          __syncwarp();
          flatten(pay, lane, in && leader && alen > 0, aoff, make_uint2(a0 - aoff, slot), total_a,
                  [&](uint32_t f, uint2 P) {
                    DBG_CHECK(P.x + f < BS.nnz, 12, P.x, f, BS.nnz, T.idx, 0, 0, 0);
                    return ld_stream(cS + P.x + f);
                  },
                  [&](uint32_t, uint2 P, uint32_t w) { table_insert<BW>(tab, (w << 5) | P.y, G); });
          // ---- probe every word of each lane's list P against its staged list
          auto test = [&](uint32_t w, uint32_t sl) { return table_probe<BW>(tab, (w << 5) | sl, G); };
          hits += probe_lists<kP1Unified && !kBm>(cols, pay, lane, bx, bl, slot, test);
          continue_run(test);
        }
      }
      // kCP: the next batch starts after the last consumed edge, in its column or later
      // (a continued run consumed only edges of column k0 = lane 31's column)
      if (cpm) ccol = __shfl_sync(kFull, v, min(L, 32) - 1);
      base += L;
    }
    // one atomic pair per warp-item
    const uint32_t s = __reduce_add_sync(kFull, hits);
    if (lane == 0 && s) {
      atomicAdd(&counts[T.idx], (unsigned long long)s);
      atomicAdd(&counts[n_tasks], (unsigned long long)s);
    }
    if (task_cycles && lane == 0) atomicAdd(&task_cycles[T.idx], (unsigned long long)(clock64() - *t_slot()));
  }
}

// ---- dense tasks (Alg. 6) ---------------------------------------------
// Alg. 6 marks N(G_ik,u) in a dense map H over V_k and tests every w of N(G_jk,v)
// against it.  When |V_k| is small, the B200 form of that map is a bit row: every
// row y of a block (x,k) a dense task reads is kept as |V_k| bits (stride S words,
// S a power of two), and an edge (u,v) of G_ij closes |row_ik(u) AND row_jk(v)|
// triangles — S/4 uint4 loads and popcounts instead of a list walk, whatever the
// list lengths.  k_dense_rows sets the bits from the block's edges.
__global__ void k_dense_rows(const uint32_t* __restrict__ it_u, const uint32_t* __restrict__ it_v,
                             const BlockDesc* __restrict__ blocks, const uint32_t* __restrict__ ids, uint32_t n_ids,
                             const uint64_t* __restrict__ off, const uint32_t* __restrict__ stride,
                             uint32_t* __restrict__ dense) {
  for (uint32_t y = blockIdx.y; y < n_ids; y += gridDim.y) {
    const uint32_t b = ids[y];
    const BlockDesc B = blocks[b];
    uint32_t* D = dense + off[b];
    const uint32_t S = stride[b];
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < B.nnz;
         x += (uint64_t)gridDim.x * blockDim.x) {
      const uint32_t u = it_u[B.e0 + x], w = it_v[B.e0 + x];
      atomicOr(D + (uint64_t)u * S + (w >> 5), 1u << (w & 31));
    }
  }
}

// The edges [e_begin, e_end) of G_ij of one dense item, bit rows of stride S words:
// 32 edges at a time; a round takes 32/LPR edges, LPR lanes per edge each loading Q
// uint4 of both rows (kUnroll rounds of loads in flight).  Returns this lane's hits.
// kKeepU (row walk: consecutive edges share u): a lane keeps the row_ik(u) words it
// last loaded and reloads them only when its edge's u changes, so only row_jk(v) is
// read per edge (half the L1/L2 traffic of the bit-row kernel on long rows).
template <int S, bool kKeepU>
__device__ __forceinline__ uint32_t dense_edges(const uint32_t* __restrict__ it_u, const uint32_t* __restrict__ it_v,
                                                const uint32_t* __restrict__ Dik, const uint32_t* __restrict__ Djk,
                                                uint64_t e_begin, uint64_t e_end, int lane) {
  constexpr int kV = S / 4;                      // uint4 per row
  constexpr int LPR = kV < 32 ? kV : 32;         // lanes per edge
  constexpr int Q = kV / LPR;                    // uint4 per lane per row
  constexpr int EPR = 32 / LPR;                  // edges per round
  constexpr int kRounds = 32 / EPR;              // rounds per 32 edges
  constexpr int kUnroll = kRounds < 4 / Q ? kRounds : 4 / Q;   // <= 4 uint4 of each row in flight
  const int sub = lane / LPR, q = lane % LPR;
  const uint4* Di = reinterpret_cast<const uint4*>(Dik) + q;
  const uint4* Dj = reinterpret_cast<const uint4*>(Djk) + q;
  uint32_t acc = 0;
  uint32_t ku = 0xFFFFFFFFu;   // kKeepU: the u whose row words this lane holds in ka
  uint4 ka[Q];
#pragma unroll
  for (int x = 0; x < Q; ++x) ka[x] = make_uint4(0, 0, 0, 0);
  for (uint64_t base = e_begin; base < e_end; base += 32) {
    const uint64_t e = base + lane;
    const bool valid = e < e_end;
    const uint32_t u = valid ? it_u[e] : 0, v = valid ? it_v[e] : 0;
    const int n = (int)(e_end - base < 32 ? e_end - base : 32);
#pragma unroll
    for (int r0 = 0; r0 < kRounds; r0 += kUnroll) {
      if (r0 * EPR >= n) break;
      uint4 a[kUnroll][Q], b[kUnroll][Q];
#pragma unroll
      for (int r = 0; r < kUnroll; ++r) {
        const int idx = (r0 + r) * EPR + sub;
        const uint32_t uu = __shfl_sync(kFull, u, idx & 31), vv = __shfl_sync(kFull, v, idx & 31);
        const bool fresh = !kKeepU || uu != ku;
#pragma unroll
        for (int x = 0; x < Q; ++x) {
          if (idx < n) {
            a[r][x] = fresh ? Di[(uint64_t)uu * kV + x * LPR] : ka[x];
            b[r][x] = Dj[(uint64_t)vv * kV + x * LPR];
          } else {
            a[r][x] = make_uint4(0, 0, 0, 0);
            b[r][x] = a[r][x];
          }
        }
        if (kKeepU && idx < n) {
          ku = uu;
#pragma unroll
          for (int x = 0; x < Q; ++x) ka[x] = a[r][x];
        }
      }
#pragma unroll
      for (int r = 0; r < kUnroll; ++r)
#pragma unroll
        for (int x = 0; x < Q; ++x)
          acc += __popc(a[r][x].x & b[r][x].x) + __popc(a[r][x].y & b[r][x].y) + __popc(a[r][x].z & b[r][x].z) +
                 __popc(a[r][x].w & b[r][x].w);
    }
  }
  return acc;
}

// One warp per work item of a dense task (TaskDesc.pad = the bit-row stride of V_k).
#ifndef BBTC_DENSE_MIN_CTAS
#define BBTC_DENSE_MIN_CTAS 4
#endif
template <bool kKeepU>
__global__ void __launch_bounds__(kWarps * 32, BBTC_DENSE_MIN_CTAS)
k_count_dense(const uint32_t* __restrict__ it_u, const uint32_t* __restrict__ it_v,
              const uint32_t* __restrict__ dense, const uint64_t* __restrict__ off,
              const BlockDesc* __restrict__ blocks, const TaskDesc* __restrict__ tasks,
              const uint64_t* __restrict__ item_start, uint32_t n_exec, uint64_t item_lo, uint64_t n_items,
              uint32_t rank, uint32_t world, unsigned long long* __restrict__ cursor,
              unsigned long long* __restrict__ counts, uint32_t n_tasks,
              unsigned long long* __restrict__ task_cycles) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(cursor, 1ull);
    it = __shfl_sync(kFull, it, 0);
    const uint64_t g = item_lo + it * world + rank;
    if (g >= n_items) break;
    const long long t_item = task_cycles ? clock64() : 0;
    uint32_t lo = 0, hi = n_exec - 1;
    while (lo < hi) {
      uint32_t mid = (lo + hi + 1) >> 1;
      if (item_start[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const TaskDesc T = tasks[lo];
    const BlockDesc Bij = blocks[T.ij];
    const uint32_t* Dik = dense + off[T.ik];
    const uint32_t* Djk = dense + off[T.jk];
    const uint64_t e_begin = Bij.e0 + (g - item_start[lo]) * T.chunk;
    const uint64_t e_end = min(e_begin + T.chunk, Bij.e0 + Bij.nnz);
    uint32_t acc = 0;
    switch (T.pad) {
      case 8: acc = dense_edges<8, kKeepU>(it_u, it_v, Dik, Djk, e_begin, e_end, lane); break;
      case 16: acc = dense_edges<16, kKeepU>(it_u, it_v, Dik, Djk, e_begin, e_end, lane); break;
      case 32: acc = dense_edges<32, kKeepU>(it_u, it_v, Dik, Djk, e_begin, e_end, lane); break;
      case 64: acc = dense_edges<64, kKeepU>(it_u, it_v, Dik, Djk, e_begin, e_end, lane); break;
      case 128: acc = dense_edges<128, kKeepU>(it_u, it_v, Dik, Djk, e_begin, e_end, lane); break;
      case 256: acc = dense_edges<256, kKeepU>(it_u, it_v, Dik, Djk, e_begin, e_end, lane); break;
      default: acc = dense_edges<512, kKeepU>(it_u, it_v, Dik, Djk, e_begin, e_end, lane); break;
    }
    const uint32_t s = __reduce_add_sync(kFull, acc);
    if (lane == 0 && s) {
      atomicAdd(&counts[T.idx], (unsigned long long)s);
      atomicAdd(&counts[n_tasks], (unsigned long long)s);
    }
    if (task_cycles && lane == 0) atomicAdd(&task_cycles[T.idx], (unsigned long long)(clock64() - t_item));
  }
}

// ---- plan statistics (BBTC_PLAN_STATS): B_alg, visits, d'_max -------------------
// Per task t and edge (u,v) of G_ij: a = d(G_ik,u), b = d(G_jk,v).
// B_alg(t) = 4(|V_i|+1) + 8 R_ij + Σ (4 + 8 + 4a + 4b)
__global__ void k_stats_edges(const uint32_t* __restrict__ it_v, const uint32_t* __restrict__ it_u,
                              const uint32_t* __restrict__ rowptr, const BlockDesc* __restrict__ blocks,
                              const TaskDesc* __restrict__ tasks, uint32_t n_exec,
                              unsigned long long* __restrict__ ab_sum) {
  for (uint32_t t = blockIdx.y; t < n_exec; t += gridDim.y) {
    const TaskDesc T = tasks[t];
    const BlockDesc Bij = blocks[T.ij], Bik = blocks[T.ik], Bjk = blocks[T.jk];
    unsigned long long sa = 0, sb = 0;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < Bij.nnz;
         x += (uint64_t)gridDim.x * blockDim.x) {
      const uint32_t u = it_u[Bij.e0 + x], v = it_v[Bij.e0 + x];
      sa += rowptr[Bik.ro + u + 1] - rowptr[Bik.ro + u];
      sb += rowptr[Bjk.ro + v + 1] - rowptr[Bjk.ro + v];
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
      sa += __shfl_xor_sync(kFull, sa, d);
      sb += __shfl_xor_sync(kFull, sb, d);
    }
    if ((threadIdx.x & 31) == 0) {
      if (sa) atomicAdd(&ab_sum[2 * t], sa);
      if (sb) atomicAdd(&ab_sum[2 * t + 1], sb);
    }
  }
}

// Per block: nonempty rows R_ij and the largest partial degree.
__global__ void k_stats_rows(const uint32_t* __restrict__ rowptr, const BlockDesc* __restrict__ blocks,
                             const uint32_t* __restrict__ rows_per_block, uint32_t nb,
                             unsigned long long* __restrict__ nonempty, uint32_t* __restrict__ dmax) {
  for (uint32_t b = blockIdx.y; b < nb; b += gridDim.y) {
    const BlockDesc B = blocks[b];
    const uint32_t nr = rows_per_block[b];
    uint32_t ne = 0, mx = 0;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
      uint32_t d = rowptr[B.ro + r + 1] - rowptr[B.ro + r];
      ne += d > 0;
      mx = max(mx, d);
    }
    ne = __reduce_add_sync(kFull, ne);
    mx = __reduce_max_sync(kFull, mx);
    if ((threadIdx.x & 31) == 0) {
      if (ne) atomicAdd(&nonempty[b], (unsigned long long)ne);
      atomicMax(dmax, mx);
    }
  }
}

}  // namespace

void count_zero(bbtc_ctx* ctx, const bbtc_plan* plan, uint64_t* d_counts) {
  BBTC_CUDA(cudaMemsetAsync(d_counts, 0, (plan->info.n_tasks + 1) * 8, ctx->stream));
}

// Enqueues the count kernel over work items [item_lo, item_hi) of the plan's
// execution order (this rank's residues only), accumulating into d_counts.
void count_launch(bbtc_ctx* ctx, const bbtc_plan* plan, uint32_t rank, uint32_t world, uint64_t* d_counts,
                  uint64_t item_lo, uint64_t item_hi, const uint32_t* ready, uint32_t epoch, const DevArenas* ar,
                  const TaskDesc* tasks, const uint64_t* item_start, uint32_t n_exec) {
  cudaStream_t st = ctx->stream;
  const uint64_t nt = plan->info.n_tasks;
  if (item_hi <= item_lo + rank) return;
  const uint64_t my_items = (item_hi - item_lo - rank + world - 1) / world;
  if (!ctx->cursor) BBTC_CUDA(cudaMalloc((void**)&ctx->cursor, 8 * kCursorSlots));
  unsigned long long* cursor = (unsigned long long*)ctx->cursor + (ctx->cursor_next++ % kCursorSlots);
  BBTC_CUDA(cudaMemsetAsync(cursor, 0, 8, st));
  // Hash keys pack a V_k-local id into 27 bits: every part must be smaller than 2^27.
  uint32_t max_part = 0;
  for (uint32_t i = 0; i < plan->p; ++i) max_part = std::max(max_part, plan->cuts[i + 1] - plan->cuts[i]);
  const bool hash = max_part < (1u << 27);
  using KernT = void (*)(const uint32_t*, const uint32_t*, const uint32_t*, const uint32_t*, const BlockDesc*,
                         const TaskDesc*, const uint64_t*, uint32_t, uint64_t, uint64_t, uint32_t, uint32_t,
                         unsigned long long*, unsigned long long*, uint32_t, const uint32_t*, uint32_t,
                         const uint32_t*, const uint32_t*, unsigned long long*, const uint32_t*);
  // The bitmap variant only where some task's V_k is small enough (it costs the main
  // loop a few registers: friendster, whose parts are all large, measured 0.7% slower).
  bool bm = false;
  for (const TaskDesc& T : plan->tasks) bm = bm || T.bmw != 0;
  const bool cp = ar && ar->colptr && plan->colmajor;
  if (cp && !ar->item_col) raise(BBTC_ESTATE, "column-offset walk without item start columns");
  const int variant = (hash ? 1 : 0) | (plan->colmajor ? 2 : 0) | (kBitmap && bm ? 4 : 0) | (cp ? 8 : 0);
  static const KernT kerns[16] = {
      k_count<false, false, false, false>, k_count<true, false, false, false>,
      k_count<false, true, false, false>,  k_count<true, true, false, false>,
      k_count<false, false, true, false>,  k_count<true, false, true, false>,
      k_count<false, true, true, false>,   k_count<true, true, true, false>,
      nullptr,                             nullptr,
      k_count<false, true, false, true>,   k_count<true, true, false, true>,
      nullptr,                             nullptr,
      k_count<false, true, true, true>,    k_count<true, true, true, true>};
  KernT kern = kerns[variant];
  static int per_sm[16] = {};
  if (!per_sm[variant]) {
    BBTC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    // Shared-memory carveout: what the resident CTAs need, the rest stays L1 for the
    // gathered lists (BBTC_CARVEOUT = percent overrides).
    const char* ce = getenv("BBTC_CARVEOUT");
    const int carve = ce ? atoi(ce) : kCarveoutPct;
    if (carve > 0) BBTC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    BBTC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[variant], kern, kWarps * 32, kSmemBytes));
  }
  // Resident CTAs per SM: the occupancy limit, capped by kCtasPerSm (more warps
  // in flight than this only widen the working set the L2 has to hold).
  static const int cap_env = [] {
    const char* e = getenv("BBTC_CTAS_PER_SM");
    return e ? atoi(e) : 0;
  }();
  const int per = std::max(1, std::min(per_sm[variant], cap_env > 0 ? cap_env : kCtasPerSm));
  const uint64_t grid = std::min<uint64_t>((uint64_t)ctx->sm_count * per, (my_items + kWarps - 1) / kWarps);
  DevArenas own;
  // probe slots only over the plan's own resident arenas (they live in its cols arena)
  const uint32_t* slot_of = !ar && plan->slots_ready && !getenv("BBTC_NO_SLOTS_KERNEL") ? plan->d_slot_of.p : nullptr;
  if (!ar) {   // the plan's own (fully resident) arenas
    own.cols = plan->cols.p;
    own.it_u = plan->colmajor ? plan->ccu.p : plan->rows.p;
    own.it_v = plan->colmajor ? plan->ccv.p : plan->cols.p;
    own.rowptr = plan->rowptr.p;
    own.blocks = plan->d_blocks.p;
    ar = &own;
  }
#if BBTC_DEBUG_BOUNDS
  static unsigned long long* h_dbg = nullptr;
  if (!h_dbg) {
    BBTC_CUDA(cudaHostAlloc((void**)&h_dbg, 16 * 8, cudaHostAllocMapped));
    unsigned long long* d_dbg = nullptr;
    BBTC_CUDA(cudaHostGetDevicePointer((void**)&d_dbg, h_dbg, 0));
    BBTC_CUDA(cudaMemcpyToSymbol(g_dbg, &d_dbg, sizeof d_dbg));
  }
  BBTC_CUDA(cudaStreamSynchronize(st));
  std::memset(h_dbg, 0, 16 * 8);
  h_dbg[8] = ar != &own || slot_of ? ~0ull : plan->m;   // (window arenas, slots: no bound known here)
  uint64_t ro_words = 0;
  for (auto& B : plan->blocks) ro_words += (uint64_t)(plan->cuts[B.i + 1] - plan->cuts[B.i]) + 1;
  h_dbg[9] = ar != &own ? ~0ull : ro_words;
  h_dbg[10] = plan->blocks.size();
#endif
  kern<<<(unsigned)grid, kWarps * 32, kSmemBytes, st>>>(
      ar->cols, ar->it_u, ar->it_v, ar->rowptr, ar->blocks, tasks ? tasks : plan->d_tasks.p,
      item_start ? item_start : plan->d_item_start.p,
      n_exec ? n_exec : (uint32_t)plan->tasks.size(), item_lo, item_hi, rank, world, cursor, (unsigned long long*)d_counts,
      (uint32_t)nt, ready, epoch, ar->colptr, ar->item_col, (unsigned long long*)ctx->task_cycles, slot_of);
#if BBTC_DEBUG_BOUNDS
  cudaStreamSynchronize(st);
  if (h_dbg[0])
    fprintf(stderr, "[bbtc debug] k_count check %llu failed: %llu %llu %llu %llu %llu %llu %llu (m %llu, ro %llu)\n",
            h_dbg[0], h_dbg[1], h_dbg[2], h_dbg[3], h_dbg[4], h_dbg[5], h_dbg[6], h_dbg[7], h_dbg[8], h_dbg[9]);
#endif
  BBTC_LAUNCHED(ctx);
}

// Bit rows for every block (x,k) a dense task reads (as G_ik or G_jk): |V_x| rows of
// dense_s[k] words.  Built once per resident plan, on the context stream.
void dense_build(bbtc_ctx* ctx, bbtc_plan* plan) {
  if (plan->dense_ready || plan->dense_task_lo >= plan->tasks.size()) return;
  cudaStream_t st = ctx->stream;
  const uint32_t nb = (uint32_t)plan->blocks.size();
  std::vector<uint8_t> need(nb, 0);
  for (size_t t = plan->dense_task_lo; t < plan->tasks.size(); ++t) need[plan->tasks[t].ik] = need[plan->tasks[t].jk] = 1;
  plan->dense_off.assign(nb, 0);
  std::vector<uint32_t>& ids = plan->dense_ids;
  std::vector<uint32_t>& stride = plan->dense_stride;
  ids.clear();
  stride.assign(nb, 0);
  uint64_t words = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    if (!need[b]) continue;
    const BlockDesc& B = plan->blocks[b];
    stride[b] = plan->dense_s[B.j];
    plan->dense_off[b] = words;
    words += (uint64_t)(plan->cuts[B.i + 1] - plan->cuts[B.i]) * stride[b];
    if (B.nnz) ids.push_back(b);
  }
  plan->dense.alloc(std::max<uint64_t>(words, 4), ctx);
  plan->d_dense_off.alloc(nb, ctx);
  DevBuf<uint32_t> d_ids, d_stride;
  d_ids.alloc(std::max<size_t>(ids.size(), 1), ctx);
  d_stride.alloc(nb, ctx);
  BBTC_CUDA(cudaMemcpyAsync(plan->d_dense_off.p, plan->dense_off.data(), nb * 8, cudaMemcpyHostToDevice, st));
  BBTC_CUDA(cudaMemcpyAsync(d_stride.p, stride.data(), nb * 4, cudaMemcpyHostToDevice, st));
  if (!ids.empty()) BBTC_CUDA(cudaMemcpyAsync(d_ids.p, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice, st));
  BBTC_CUDA(cudaMemsetAsync(plan->dense.p, 0, words * 4, st));
  if (!ids.empty()) {
    const uint32_t* it_u = plan->colmajor ? plan->ccu.p : plan->rows.p;
    const uint32_t* it_v = plan->colmajor ? plan->ccv.p : plan->cols.p;
    k_dense_rows<<<dim3(64, std::min<uint32_t>((uint32_t)ids.size(), 16384u)), 256, 0, st>>>(
        it_u, it_v, plan->d_blocks.p, d_ids.p, (uint32_t)ids.size(), plan->d_dense_off.p, d_stride.p, plan->dense.p);
    BBTC_LAUNCHED(ctx);
  }
  plan->dense_ready = true;   // (the copies' host sources live in the plan)
  plan->info.dense_bytes = words * 4;
}

void count_launch_dense(bbtc_ctx* ctx, const bbtc_plan* plan, uint32_t rank, uint32_t world, uint64_t* d_counts,
                        uint64_t item_lo, uint64_t item_hi) {
  cudaStream_t st = ctx->stream;
  if (item_hi <= item_lo + rank) return;
  if (!plan->dense_ready) raise(BBTC_ESTATE, "dense bit rows not built");
  const uint64_t my_items = (item_hi - item_lo - rank + world - 1) / world;
  if (!ctx->cursor) BBTC_CUDA(cudaMalloc((void**)&ctx->cursor, 8 * kCursorSlots));
  unsigned long long* cursor = (unsigned long long*)ctx->cursor + (ctx->cursor_next++ % kCursorSlots);
  BBTC_CUDA(cudaMemsetAsync(cursor, 0, 8, st));
  // row walk (the plan kept its row ids): keep row_ik(u) across a row's edges
  const bool row_walk = !plan->colmajor || plan->rows.p;
  // (keeping row_ik(u) in registers across a row's edges measured slower: rmat24 p=10
  // 11.4 -> 12.9 ms — more registers, and the reloads hit L1 anyway; BBTC_DENSE_KEEP=1)
  auto kern = row_walk && getenv("BBTC_DENSE_KEEP") ? k_count_dense<true> : k_count_dense<false>;
  static int per_sm = 0;
  if (!per_sm) BBTC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_count_dense<true>, kWarps * 32, 0));
  const int per = std::max(1, std::min(per_sm, kCtasPerSm));
  const uint64_t grid = std::min<uint64_t>((uint64_t)ctx->sm_count * per, (my_items + kWarps - 1) / kWarps);
  kern<<<(unsigned)grid, kWarps * 32, 0, st>>>(
      // row walk when the plan kept its row ids (row-major plans; BBTC_DENSE_WALK=row)
      plan->colmajor && !plan->rows.p ? plan->ccu.p : plan->rows.p,
      plan->colmajor && !plan->rows.p ? plan->ccv.p : plan->cols.p, plan->dense.p,
      plan->d_dense_off.p, plan->d_blocks.p, plan->d_tasks.p, plan->d_item_start.p, (uint32_t)plan->tasks.size(),
      item_lo, item_hi, rank, world, cursor, (unsigned long long*)d_counts, (uint32_t)plan->info.n_tasks,
      (unsigned long long*)ctx->task_cycles);
  BBTC_LAUNCHED(ctx);
}

void plan_stats(bbtc_ctx* ctx, bbtc_plan* plan) {
  cudaStream_t st = ctx->stream;
  const uint32_t ne = (uint32_t)plan->tasks.size();
  const uint32_t nb = (uint32_t)plan->blocks.size();
  DevBuf<unsigned long long> ab, nonempty;
  DevBuf<uint32_t> dmax, rpb;
  ab.alloc(2 * ne, ctx);
  nonempty.alloc(nb, ctx);
  dmax.alloc(1, ctx);
  rpb.alloc(nb, ctx);
  std::vector<uint32_t> h_rpb(nb);
  uint32_t maxrows = 1;
  for (uint32_t b = 0; b < nb; ++b) {
    const BlockDesc& B = plan->blocks[b];
    h_rpb[b] = plan->cuts[B.i + 1] - plan->cuts[B.i];
    maxrows = std::max(maxrows, h_rpb[b]);
  }
  BBTC_CUDA(cudaMemcpyAsync(rpb.p, h_rpb.data(), nb * 4, cudaMemcpyHostToDevice, st));
  BBTC_CUDA(cudaMemsetAsync(ab.p, 0, ne * 16, st));
  BBTC_CUDA(cudaMemsetAsync(nonempty.p, 0, nb * 8, st));
  BBTC_CUDA(cudaMemsetAsync(dmax.p, 0, 4, st));
  if (ne) {
    k_stats_edges<<<dim3(64, std::min(ne, 4096u)), 256, 0, st>>>(plan->colmajor ? plan->ccv.p : plan->cols.p,
                                                               plan->colmajor ? plan->ccu.p : plan->rows.p,
                                                               plan->rowptr.p,
                                                               plan->d_blocks.p, plan->d_tasks.p, ne, ab.p);
    BBTC_LAUNCHED(ctx);
  }
  if (nb) {
    k_stats_rows<<<dim3(std::min((maxrows + 255) / 256, 64u), std::min(nb, 16384u)), 256, 0, st>>>(
        plan->rowptr.p, plan->d_blocks.p, rpb.p, nb, nonempty.p, dmax.p);
    BBTC_LAUNCHED(ctx);
  }
  std::vector<unsigned long long> h_ab(2 * ne), h_ne(nb);
  uint32_t h_dmax = 0;
  BBTC_CUDA(cudaMemcpyAsync(h_ab.data(), ab.p, ne * 16, cudaMemcpyDeviceToHost, st));
  BBTC_CUDA(cudaMemcpyAsync(h_ne.data(), nonempty.p, nb * 8, cudaMemcpyDeviceToHost, st));
  BBTC_CUDA(cudaMemcpyAsync(&h_dmax, dmax.p, 4, cudaMemcpyDeviceToHost, st));
  BBTC_CUDA(cudaStreamSynchronize(st));
  uint64_t balg = 0, visits = 0, suma = 0, sumb = 0;
  for (uint32_t t = 0; t < ne; ++t) {
    const TaskDesc& T = plan->tasks[t];
    const BlockDesc& Bij = plan->blocks[T.ij];
    balg += 4ull * ((uint64_t)h_rpb[T.ij] + 1) + 8ull * h_ne[T.ij] + 12ull * Bij.nnz +
            4ull * (h_ab[2 * t] + h_ab[2 * t + 1]);
    visits += Bij.nnz;
    suma += h_ab[2 * t];
    sumb += h_ab[2 * t + 1];
  }
  plan->info.sum_a = suma;
  plan->info.sum_b = sumb;
  plan->info.b_alg = balg;
  plan->info.visits = visits;
  plan->info.dmax_blk = h_dmax;
}

}  // namespace bbtc

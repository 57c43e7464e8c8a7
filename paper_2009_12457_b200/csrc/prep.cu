// prep.cu — device preprocessing: steps a1-a5 of the hot path.
//
//   a1 canonicalise   raw pairs -> sorted unique (min,max) keys
//   a2 degree order   full degrees, stable rank by (degree, id), orient
//   a3 partition      symmetric cut vector (full-degree prefix rule)
//   a4 BCSR           p(p+1)/2 upper blocks, local ids, row offsets        P:460-463, Fig. 2d
//   a5 tasks          Alg. 4 enumeration + work items (host, capi.cpp)
//
// Everything is HBM-bandwidth work: streaming passes, one radix sort per phase
// (CUB onesweep, the library primitive for sorting) and scatter/gather kernels
// sized as grid-stride loops over the SM count.
#include <cub/cub.cuh>
#include <thrust/iterator/reverse_iterator.h>

#include <algorithm>
#include <chrono>

#include "internal.h"

namespace bbtc {
namespace {

constexpr uint64_t kSentinel = ~0ull;
constexpr int kThreads = 256;

inline int bitlen(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

inline unsigned grid_for(const bbtc_ctx* ctx, uint64_t n, int per_sm = 8) {
  uint64_t want = (n + kThreads - 1) / kThreads;
  uint64_t cap = (uint64_t)ctx->sm_count * per_sm;
  return (unsigned)std::max<uint64_t>(1, std::min(want, cap));
}

// Runs a CUB device-wide primitive with temporary storage from the context cache.
// `kernels` = the kernel launches the call makes (for the launch counter; matches
// the ncu launch lists in profiles/).
template <class F>
void cub_call(bbtc_ctx* ctx, F f, uint64_t kernels = 2) {
  size_t bytes = 0;
  BBTC_CUDA(f((void*)nullptr, bytes));
  DevBuf<uint8_t> tmp;
  tmp.alloc(std::max<size_t>(bytes, 1), ctx);
  BBTC_CUDA(f((void*)tmp.p, bytes));
  if (sync_check()) BBTC_CUDA(cudaDeviceSynchronize());
  ctx->launches += kernels;
}

// Onesweep radix sort: histogram + exclusive-sum kernels, then one pass per 8-bit
// digit for every portion of up to 2^28 items.
inline uint64_t radix_kernels(uint64_t n, int bits) { return 2 + (uint64_t)((bits + 7) / 8) * (n / (1ull << 28) + 1); }

// 64-bit-key onesweep with a B200 tile: CUB's sm_100 policy for 8-byte keys is 384
// threads x 30 keys per CTA; smaller CTAs measured faster on this B200 for every
// 64-bit-key sort of the path (scripts/micro/sorttune.cu, profiles/r02/sorttune/: 268 M
// keys, 48 bits 16.2 -> 10.9 ms at 288 x 32; 260 M keys, 28 bits 11.0 -> 8.0 ms at
// 256 x 30).  Only the onesweep policy
// differs from CUB's own hub; u32 key-value sorts keep CUB's tuning (measured best).
template <class K, class V, int kT, int kI>
struct OnesweepHub {
  using Base = typename cub::detail::radix::policy_hub<K, V, unsigned long long>::Policy1000;
  struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, Policy1000> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = 8;
    using HistogramPolicy = typename Base::HistogramPolicy;
    using ExclusiveSumPolicy = typename Base::ExclusiveSumPolicy;
    using OnesweepPolicy =
        cub::AgentRadixSortOnesweepPolicy<kT, kI, K, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                          cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, 8>;
    using ScanPolicy = typename Base::ScanPolicy;
    using DownsweepPolicy = typename Base::DownsweepPolicy;
    using AltDownsweepPolicy = typename Base::AltDownsweepPolicy;
    using UpsweepPolicy = typename Base::UpsweepPolicy;
    using AltUpsweepPolicy = typename Base::AltUpsweepPolicy;
    using SingleTilePolicy = typename Base::SingleTilePolicy;
    using SegmentedPolicy = typename Base::SegmentedPolicy;
    using AltSegmentedPolicy = typename Base::AltSegmentedPolicy;
  };
  using MaxPolicy = Policy1000;
};
// Keys-only sort of 64-bit keys over bits [b0, b1), DoubleBuffer semantics (the sorted
// keys end in keys.Current()), same contract as cub::DeviceRadixSort::SortKeys.
inline cudaError_t sort_keys64(void* tmp, size_t& bytes, cub::DoubleBuffer<uint64_t>& keys, uint64_t n, int b0,
                               int b1, cudaStream_t st) {
  static const bool stock = getenv("BBTC_CUB_STOCK") != nullptr;   // A/B: CUB's own tuning
  cub::DoubleBuffer<cub::NullType> none;
  if (stock) return cub::DeviceRadixSort::SortKeys(tmp, bytes, keys, n, b0, b1, st);
  // > 4 digits (the 48-bit canonical keys): 288 x 32 (10.9 ms vs 12.0 at 256 x 30);
  // <= 4 digits (block keys): 256 x 30 (8.0 ms; 256 x 40 equal).
  using Wide = cub::DispatchRadixSort<false, uint64_t, cub::NullType, unsigned long long,
                                      OnesweepHub<uint64_t, cub::NullType, 288, 32>>;
  using Narrow = cub::DispatchRadixSort<false, uint64_t, cub::NullType, unsigned long long,
                                        OnesweepHub<uint64_t, cub::NullType, 256, 30>>;
  if (b1 - b0 > 32) return Wide::Dispatch(tmp, bytes, keys, none, (unsigned long long)n, b0, b1, true, st);
  return Narrow::Dispatch(tmp, bytes, keys, none, (unsigned long long)n, b0, b1, true, st);
}

// ---- a1 ------------------------------------------------------------------------------
// key = (min << bw) | max for a != b, kSentinel for self-loops; tracks the largest id.
// bw is the id width guessed from n_hint (32 when unknown); graph_build re-runs with
// bw = 32 if an id does not fit.  Narrow keys save radix-sort passes.
__global__ void k_canon(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, uint64_t E, int bw,
                        uint64_t* __restrict__ keys, uint32_t* __restrict__ max_id) {
  uint32_t mx = 0;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E; e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t a = src[e], b = dst[e];
    uint32_t lo = min(a, b), hi = max(a, b);
    mx = max(mx, hi);
    keys[e] = a == b ? kSentinel : ((uint64_t)lo << bw) | hi;
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) atomicMax(max_id, mx);
}

// The same for interleaved input pairs (src0 dst0 src1 dst1 …: a binary edge file
// as stored, e.g. memory-mapped by bbtc_edges_map).
__global__ void k_canon_pairs(const uint2* __restrict__ pairs, uint64_t E, int bw, uint64_t* __restrict__ keys,
                              uint32_t* __restrict__ max_id) {
  uint32_t mx = 0;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 q = pairs[e];
    const uint32_t lo = min(q.x, q.y), hi = max(q.x, q.y);
    mx = max(mx, hi);
    keys[e] = q.x == q.y ? kSentinel : ((uint64_t)lo << bw) | hi;
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) atomicMax(max_id, mx);
}

// Hash-set canonicalisation: every raw pair's key (min << bw | max) is inserted into
// an open-addressing table of 2^k u64 slots (load <= 1/2, linear probing); the
// table then holds each undirected edge once (duplicates and both orientations
// collapse to one key, self-loops are dropped).  One pass of random 8-byte CAS
// instead of a full radix sort + unique.
__global__ void k_canon_insert(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, uint64_t E, int bw,
                               unsigned long long* __restrict__ table, int tbits, uint32_t* __restrict__ max_id) {
  uint32_t mx = 0;
  const uint64_t tmask = (1ull << tbits) - 1;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = src[e], b = dst[e];
    const uint32_t lo = min(a, b), hi = max(a, b);
    mx = max(mx, hi);
    if (a == b) continue;
    const unsigned long long key = ((unsigned long long)lo << bw) | hi;
    uint64_t h = (key * 0x9E3779B97F4A7C15ull) >> (64 - tbits);
    for (;;) {
      const unsigned long long old = atomicCAS(&table[h], kSentinel, key);
      if (old == kSentinel || old == key) break;
      h = (h + 1) & tmask;
    }
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) atomicMax(max_id, mx);
}

struct NotEmpty {
  __host__ __device__ bool operator()(uint64_t k) const { return k != kSentinel; }
};

// Degrees of a list of unique keys in no particular order.
__global__ void k_degree_any(const uint64_t* __restrict__ keys, uint64_t m, int bw, uint32_t* __restrict__ deg) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[e];
    atomicAdd(&deg[(uint32_t)(k >> bw)], 1u);
    atomicAdd(&deg[(uint32_t)(k & ((1ull << bw) - 1))], 1u);
  }
}

// ---- a2 ------------------------------------------------------------------------------
// Degrees of sorted unique keys.  The lo side (sorted) is aggregated per warp; the hi
// side is random, so it can be split into passes over id ranges [h0, h1) small enough
// for the L2 (degrees_sorted below): the lo side is counted in the first pass only.
__global__ void k_degree(const uint64_t* __restrict__ keys, uint64_t m, int bw, uint32_t* __restrict__ deg,
                         uint32_t h0 = 0, uint32_t h1 = 0xFFFFFFFFu, bool with_lo = true) {
  // Warp-uniform trip count so the whole warp stays converged for __match_any_sync.
  const uint64_t lane = threadIdx.x & 31;
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) - lane;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = warp0; base < m; base += stride) {
    const uint64_t e = base + lane;
    const bool valid = e < m;
    const uint64_t k = valid ? keys[e] : 0;
    const uint32_t lo = valid ? (uint32_t)(k >> bw) : 0xFFFFFFFFu;
    const uint32_t hi = (uint32_t)(k & ((1ull << bw) - 1));
    if (with_lo) {   // keys are sorted, so equal `lo` values sit in the same warp: aggregate them
      const uint32_t peers = __match_any_sync(0xffffffffu, lo);
      if (valid && lane == (uint64_t)(__ffs(peers) - 1)) atomicAdd(&deg[lo], __popc(peers));
    }
    if (valid && hi >= h0 && hi < h1) atomicAdd(&deg[hi], 1u);
  }
}

__global__ void k_iota(uint32_t* __restrict__ x, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = i;
}

__global__ void k_rank(const uint32_t* __restrict__ order, uint32_t n, uint32_t* __restrict__ rank) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) rank[order[r]] = r;
}

// Orientation from lower to higher degree rank (P:226-235 with the order of P:438-446).
// [h0, h1): only keys whose hi id falls in it (passes over L2-sized slices of rank[]).
__global__ void k_orient(const uint64_t* __restrict__ keys, uint64_t m, int bw, const uint32_t* __restrict__ rank,
                         uint64_t* __restrict__ okeys, uint32_t h0 = 0, uint32_t h1 = 0xFFFFFFFFu) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[e];
    const uint32_t hi = (uint32_t)(k & ((1ull << bw) - 1));
    if (hi < h0 || hi >= h1) continue;
    uint32_t ra = rank[(uint32_t)(k >> bw)], rb = rank[hi];
    okeys[e] = ((uint64_t)min(ra, rb) << 32) | max(ra, rb);
  }
}

__global__ void k_graph_stats(const uint32_t* __restrict__ deg_sorted, uint32_t n, uint32_t* out) {
  // out[0] = first rank with degree > 0 (binary search), out[1] = d_max.
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
      uint32_t mid = lo + (hi - lo) / 2;
      if (deg_sorted[mid] == 0) lo = mid + 1; else hi = mid;
    }
    out[0] = lo;
    out[1] = n ? deg_sorted[n - 1] : 0;
  }
}

// d⁺(u) = out-degree in the oriented graph (rank space); its maximum (d'_max of the
// unblocked graph, SURVEY §8(b) stats).
__global__ void k_outdeg(const uint64_t* __restrict__ okeys, uint64_t m, uint32_t* __restrict__ dplus) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&dplus[(uint32_t)(okeys[e] >> 32)], 1u);
}
__global__ void k_max_u32(const uint32_t* __restrict__ x, uint32_t n, uint32_t* __restrict__ out) {
  uint32_t mx = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) mx = max(mx, x[i]);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// ---- a3 ------------------------------------------------------------------------------
struct ToU64 {
  __host__ __device__ uint64_t operator()(uint32_t x) const { return x; }
};

// cuts[i] = max(cuts[i-1], min{ r : P[r] >= ceil(i*2m/p) }), P[r] = sum of the first r
// rank-ordered degrees (P[0] = 0, P[n] = 2m).  incl[r] = P[r+1].
__global__ void k_cuts(const uint64_t* __restrict__ incl, uint32_t n, uint64_t two_m, uint32_t p,
                       uint32_t* __restrict__ cuts) {
  for (uint32_t i = 1 + threadIdx.x; i < p; i += blockDim.x) {
    uint64_t target = ((uint64_t)i * two_m + p - 1) / p;
    // smallest r in [0, n] with P[r] >= target
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
      uint32_t mid = lo + (hi - lo) / 2;
      uint64_t P = mid == 0 ? 0 : incl[mid - 1];
      if (P >= target) hi = mid; else lo = mid + 1;
    }
    cuts[i] = lo;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    cuts[0] = 0;
    for (uint32_t i = 1; i < p; ++i) cuts[i] = max(cuts[i], cuts[i - 1]);
    cuts[p] = n;
  }
}

// ---- a4 ------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t part_of(const uint32_t* cuts, uint32_t p, uint32_t r) {
  // the i with cuts[i] <= r < cuts[i+1] (largest i with cuts[i] <= r)
  uint32_t lo = 0, hi = p - 1;
  while (lo < hi) {
    uint32_t mid = (lo + hi + 1) / 2;
    if (cuts[mid] <= r) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Block sort key: (j, ru, rw) with j = part(rw).  Sorting by its (j, ru) bits lays the
// blocks out contiguously in column-major block order with rows ascending inside a
// block; the columns of a row keep no order (the count kernel hashes the lists, so
// Alg. 1's "A and B are sorted" is not needed).
__global__ void k_block_keys(const uint64_t* __restrict__ okeys, uint64_t m, const uint32_t* __restrict__ gcuts,
                             uint32_t p, int bn, uint64_t* __restrict__ ckeys) {
  extern __shared__ uint32_t s_cuts[];
  for (uint32_t x = threadIdx.x; x <= p; x += blockDim.x) s_cuts[x] = gcuts[x];
  __syncthreads();
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k = okeys[e];
    uint64_t ru = k >> 32, rw = (uint32_t)k;
    uint64_t j = part_of(s_cuts, p, (uint32_t)rw);
    ckeys[e] = (j << (2 * bn)) | (ru << bn) | rw;
  }
}

// Block b = (i,j) starts at the first key >= (j, cuts[i], 0).
__global__ void k_block_starts(const uint64_t* __restrict__ ckeys, uint64_t m, const uint32_t* __restrict__ cuts,
                               uint32_t p, int bn, uint64_t* __restrict__ starts) {
  uint32_t nb = p * (p + 1) / 2;
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x) {
    if (b == nb) { starts[b] = m; continue; }
    uint32_t j = 0;
    while ((j + 1) * (j + 2) / 2 <= b) ++j;
    uint32_t i = b - j * (j + 1) / 2;
    uint64_t probe = ((uint64_t)j << (2 * bn)) | ((uint64_t)cuts[i] << bn);
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
      uint64_t mid = lo + (hi - lo) / 2;
      if (ckeys[mid] < probe) lo = mid + 1; else hi = mid;
    }
    starts[b] = lo;
  }
}

// Local ids: cols[e] = rw - cuts[j], rows[e] = ru - cuts[i]; and the row-start marks.
__global__ void k_split(const uint64_t* __restrict__ ckeys, uint64_t m, const uint32_t* __restrict__ gcuts,
                        uint32_t p, int bn, const BlockDesc* __restrict__ blocks, uint32_t* __restrict__ cols,
                        uint32_t* __restrict__ rows, uint32_t* __restrict__ rowptr) {
  extern __shared__ uint32_t s_cuts[];
  for (uint32_t x = threadIdx.x; x <= p; x += blockDim.x) s_cuts[x] = gcuts[x];
  __syncthreads();
  const uint64_t mask = (1ull << bn) - 1;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k = ckeys[e];
    uint32_t j = (uint32_t)(k >> (2 * bn));
    uint32_t ru = (uint32_t)((k >> bn) & mask), rw = (uint32_t)(k & mask);
    uint32_t i = part_of(s_cuts, p, ru);
    uint32_t lr = ru - s_cuts[i];
    cols[e] = rw - s_cuts[j];
    rows[e] = lr;
    const BlockDesc& B = blocks[j * (j + 1) / 2 + i];
    bool first = e == B.e0;
    if (!first) {
      uint64_t kp = ckeys[e - 1];
      first = ((kp >> bn) & mask) != ru;
    }
    if (first) rowptr[B.ro + lr] = (uint32_t)e;   // global edge index of the row's first edge
  }
}

// Row-offset arena entry |V_i| of every block = the block's end (global index).
__global__ void k_row_ends(const BlockDesc* __restrict__ blocks, uint32_t nb, const uint32_t* __restrict__ cuts,
                           uint32_t* __restrict__ rowptr) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    const BlockDesc& B = blocks[b];
    rowptr[B.ro + (cuts[B.i + 1] - cuts[B.i])] = (uint32_t)(B.e0 + B.nnz);
  }
}

struct MinOp {
  __host__ __device__ uint32_t operator()(uint32_t a, uint32_t b) const { return a < b ? a : b; }
};

// Global -> block-local offsets.  grid.y walks the blocks.
__global__ void k_row_local(const BlockDesc* __restrict__ blocks, uint32_t nb, const uint32_t* __restrict__ cuts,
                            uint32_t* __restrict__ rowptr) {
  for (uint32_t b = blockIdx.y; b < nb; b += gridDim.y) {
    const BlockDesc B = blocks[b];
    const uint32_t len = cuts[B.i + 1] - cuts[B.i] + 1;
    const uint32_t base = (uint32_t)B.e0;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < len; r += gridDim.x * blockDim.x)
      rowptr[B.ro + r] -= base;
  }
}

// Packed transpose keys: block b's columns occupy [cbase[b], cbase[b] + |V_j| - trim_j)
// of one key range, trim_j = the isolated vertices at the start of part j (they have
// no edges, so no column id below it).  The whole range usually needs fewer bits than
// (block << column bits) | column: one radix pass fewer (rmat24: 24 bits instead of 32).
// Shared memory: e0[nb] (u64), cbase[nb] (u32), trim[p] (u32).
__device__ __forceinline__ uint32_t block_of_edge(const uint64_t* s_e0, uint32_t nb, uint64_t e) {
  uint32_t lo = 0, hi = nb - 1;   // last block with e0 <= e
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (s_e0[mid] <= e) lo = mid; else hi = mid - 1;
  }
  return lo;
}
__global__ void k_transpose_keys_packed(const uint32_t* __restrict__ cols, uint64_t m,
                                        const BlockDesc* __restrict__ blocks, uint32_t nb,
                                        const uint32_t* __restrict__ cbase, const uint32_t* __restrict__ trim,
                                        uint32_t p, uint32_t* __restrict__ keys) {
  extern __shared__ uint64_t s_pk[];
  uint64_t* s_e0 = s_pk;
  uint32_t* s_cb = reinterpret_cast<uint32_t*>(s_pk + nb);
  uint32_t* s_bt = s_cb + nb;   // per block: trim of its column part
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
    s_e0[b] = blocks[b].e0;
    s_cb[b] = cbase[b];
    s_bt[b] = trim[blocks[b].j];
  }
  __syncthreads();
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = block_of_edge(s_e0, nb, e);
    keys[e] = s_cb[b] + cols[e] - s_bt[b];
  }
}
// Sorted packed keys (still in block order) back to local column ids.
__global__ void k_unpack_cols(uint32_t* __restrict__ ccv, uint64_t m, const BlockDesc* __restrict__ blocks,
                              uint32_t nb, const uint32_t* __restrict__ cbase, const uint32_t* __restrict__ trim) {
  extern __shared__ uint64_t s_pk[];
  uint64_t* s_e0 = s_pk;
  uint32_t* s_cb = reinterpret_cast<uint32_t*>(s_pk + nb);
  uint32_t* s_bt = s_cb + nb;
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
    s_e0[b] = blocks[b].e0;
    s_cb[b] = cbase[b];
    s_bt[b] = trim[blocks[b].j];
  }
  __syncthreads();
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = block_of_edge(s_e0, nb, e);
    ccv[e] = ccv[e] - s_cb[b] + s_bt[b];
  }
}

// ---- a3 auto-p: block sizes of a candidate partition without building it ---------
// hist[i*p + j] = edges (ru, rw) with ru in V_i, rw in V_j (the nnz of block (i,j)).
__global__ void k_part_hist(const uint64_t* __restrict__ okeys, uint64_t m, const uint32_t* __restrict__ gcuts,
                            uint32_t p, bool smem_hist, unsigned long long* __restrict__ hist) {
  extern __shared__ uint32_t sh[];
  uint32_t* s_cuts = sh;
  uint32_t* s_hist = sh + p + 1;
  for (uint32_t x = threadIdx.x; x <= p; x += blockDim.x) s_cuts[x] = gcuts[x];
  if (smem_hist)
    for (uint32_t x = threadIdx.x; x < p * p; x += blockDim.x) s_hist[x] = 0;
  __syncthreads();
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = okeys[e];
    const uint32_t i = part_of(s_cuts, p, (uint32_t)(k >> 32)), j = part_of(s_cuts, p, (uint32_t)k);
    if (smem_hist) atomicAdd(&s_hist[i * p + j], 1u);
    else atomicAdd(&hist[i * p + j], 1ull);
  }
  if (smem_hist) {
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < p * p; x += blockDim.x)
      if (s_hist[x]) atomicAdd(&hist[x], (unsigned long long)s_hist[x]);
  }
}

// ---- a6 support: column offsets of column-major blocks ---------------------------
// colptr[co[b] + c] = global index of the first edge of column c in block b (runs of
// ccv), colptr[co[b] + |V_j|] = the block's end; unset entries (empty columns) are
// filled by a reverse min-scan, then made block-local (k_col_local).
__global__ void k_col_starts(const uint32_t* __restrict__ ccv, const BlockDesc* __restrict__ blocks,
                             const uint64_t* __restrict__ co, uint32_t nb, const uint32_t* __restrict__ cuts,
                             uint32_t* __restrict__ colptr) {
  for (uint32_t b = blockIdx.y; b < nb; b += gridDim.y) {
    const BlockDesc B = blocks[b];
    if (co[b] == kNoColptr) continue;
    uint32_t* C = colptr + co[b];
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < B.nnz;
         x += (uint64_t)gridDim.x * blockDim.x) {
      const uint32_t c = ccv[B.e0 + x];
      if (x == 0 || ccv[B.e0 + x - 1] != c) C[c] = (uint32_t)(B.e0 + x);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) C[cuts[B.j + 1] - cuts[B.j]] = (uint32_t)(B.e0 + B.nnz);
  }
}
__global__ void k_col_local(const BlockDesc* __restrict__ blocks, const uint64_t* __restrict__ co, uint32_t nb,
                            const uint32_t* __restrict__ cuts, uint32_t* __restrict__ colptr) {
  for (uint32_t b = blockIdx.y; b < nb; b += gridDim.y) {
    const BlockDesc B = blocks[b];
    if (co[b] == kNoColptr) continue;
    const uint32_t len = cuts[B.j + 1] - cuts[B.j] + 1;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < len; c += gridDim.x * blockDim.x)
      colptr[co[b] + c] -= (uint32_t)B.e0;
  }
}
// The column of every work item's first edge (streamed column-major plans): items in
// execution order, written at item_col[T.icol + item - item_start[t]].
__global__ void k_item_cols(const TaskDesc* __restrict__ tasks, const uint64_t* __restrict__ item_start,
                            uint32_t n_exec, uint64_t n_items, const BlockDesc* __restrict__ blocks,
                            const uint32_t* __restrict__ colptr, const uint64_t* __restrict__ co,
                            uint32_t* __restrict__ item_col) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < n_items;
       g += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = n_exec - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (item_start[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const TaskDesc T = tasks[lo];
    if (co[T.ij] == kNoColptr) {   // (the block streams its column ids)
      item_col[T.icol + (g - item_start[lo])] = 0;
      continue;
    }
    const uint64_t x = (g - item_start[lo]) * T.chunk;   // local offset of the item's first edge
    const uint32_t* cp = colptr + co[T.ij];
    uint32_t a = 0, b = blocks[T.ij].nc - 1;               // largest c with cp[c] <= x
    while (a < b) {
      const uint32_t mid = a + (b - a + 1) / 2;
      if (cp[mid] <= x) a = mid; else b = mid - 1;
    }
    item_col[T.icol + (g - item_start[lo])] = a;
  }
}

// ccv from the column offsets once a streamed count's copies have landed (context
// stream, ordered after the count kernel): ccv[e0 + x] = c for every edge x of column
// c of every block.  A warp per 32 columns, lanes over a column's edges.
__global__ void k_col_expand_all(const uint32_t* __restrict__ colptr, const BlockDesc* __restrict__ blocks,
                                 uint32_t nb, uint32_t* __restrict__ ccv) {
  const int lane = threadIdx.x & 31;
  for (uint32_t b = blockIdx.y; b < nb; b += gridDim.y) {
    const BlockDesc B = blocks[b];
    if (!B.nnz || B.co == kNoColptr) continue;   // (ccv copied as it is)
    const uint32_t* C = colptr + B.co;
    uint32_t* V = ccv + B.e0;
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t c0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; c0 < B.nc; c0 += nwarps * 32) {
      const uint32_t cn = min(32u, B.nc - c0);
      for (uint32_t x = 0; x < cn; ++x) {
        const uint32_t a = C[c0 + x], z = C[c0 + x + 1];
        for (uint32_t y = a + lane; y < z; y += 32) V[y] = c0 + x;
      }
    }
  }
}

// Transpose keys: (block of edge e) << cb | local column.  Blocks are contiguous edge
// ranges, found by binary search over their first edges (held in shared memory).
template <class K>
__global__ void k_transpose_keys(const uint32_t* __restrict__ cols, uint64_t m, const BlockDesc* __restrict__ blocks,
                                 uint32_t nb, int cb, K* __restrict__ keys) {
  extern __shared__ uint64_t s_e0[];
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) s_e0[b] = blocks[b].e0;
  __syncthreads();
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nb - 1;   // last block with e0 <= e
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (s_e0[mid] <= e) lo = mid; else hi = mid - 1;
    }
    keys[e] = ((K)lo << cb) | cols[e];
  }
}

template <class K>
__global__ void k_low_bits(const K* __restrict__ keys, uint64_t m, int cb, uint32_t* __restrict__ out) {
  const K mask = ((K)1 << cb) - 1;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
    out[e] = (uint32_t)(keys[e] & mask);
}

// ---- a4 CSR by counting sort -------------------------------------------------------
// The row-offset arena is the counter array: every oriented edge (ru, rw) of block
// (i, j) counts into rowptr[ro[b] + ru - cuts[i]]; one exclusive scan over the whole
// arena gives every row's first edge in the arena (blocks in order, rows ascending,
// each block's trailing entry = its end); a scatter places the edges (the order of
// the columns inside a row is arbitrary, as before).  Replaces the (j, ru) radix sort.
__global__ void k_csr_count(const uint64_t* __restrict__ okeys, uint64_t m, const uint32_t* __restrict__ gcuts,
                            uint32_t p, const uint64_t* __restrict__ ro, uint32_t* __restrict__ cnt) {
  extern __shared__ uint32_t s_cuts[];
  for (uint32_t x = threadIdx.x; x <= p; x += blockDim.x) s_cuts[x] = gcuts[x];
  __syncthreads();
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = okeys[e];
    const uint32_t ru = (uint32_t)(k >> 32), rw = (uint32_t)k;
    const uint32_t i = part_of(s_cuts, p, ru), j = part_of(s_cuts, p, rw);
    atomicAdd(&cnt[ro[j * (j + 1) / 2 + i] + (ru - s_cuts[i])], 1u);
  }
}
__global__ void k_csr_scatter(const uint64_t* __restrict__ okeys, uint64_t m, const uint32_t* __restrict__ gcuts,
                              uint32_t p, const uint64_t* __restrict__ ro, uint32_t* __restrict__ cursor,
                              uint32_t* __restrict__ cols, uint32_t* __restrict__ rows) {
  extern __shared__ uint32_t s_cuts[];
  for (uint32_t x = threadIdx.x; x <= p; x += blockDim.x) s_cuts[x] = gcuts[x];
  __syncthreads();
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = okeys[e];
    const uint32_t ru = (uint32_t)(k >> 32), rw = (uint32_t)k;
    const uint32_t i = part_of(s_cuts, p, ru), j = part_of(s_cuts, p, rw);
    const uint32_t lr = ru - s_cuts[i];
    const uint32_t at = atomicAdd(&cursor[ro[j * (j + 1) / 2 + i] + lr], 1u);
    cols[at] = rw - s_cuts[j];
    rows[at] = lr;
  }
}
// starts[b] = the arena position of block b's first edge (its first row offset).
__global__ void k_block_first(const uint32_t* __restrict__ rowptr, const uint64_t* __restrict__ ro, uint32_t nb,
                              uint64_t* __restrict__ starts) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) starts[b] = rowptr[ro[b]];
}

// ---- a4 probe slots: per row of a slot block, 8 words at cols[so + 8r]: the row's
// length, its block-local CSR offset and its first min(len, 6) column ids.
__global__ void k_slots(const uint32_t* __restrict__ rowptr, uint32_t* __restrict__ cols,
                        const BlockDesc* __restrict__ blocks, const uint32_t* __restrict__ ids,
                        const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ nrows) {
  const uint32_t b = ids[blockIdx.y];
  const BlockDesc B = blocks[b];
  const uint32_t rows = nrows[b];
  uint4* S = reinterpret_cast<uint4*>(cols + slot_of[b]);
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const uint32_t lo = rowptr[B.ro + r], len = rowptr[B.ro + r + 1] - lo;
    const uint32_t* c = cols + B.e0 + lo;
    uint32_t w[6];
#pragma unroll
    for (int x = 0; x < 6; ++x) w[x] = x < (int)len ? c[x] : 0u;
    S[2 * (uint64_t)r] = make_uint4(len, lo, w[0], w[1]);
    S[2 * (uint64_t)r + 1] = make_uint4(w[2], w[3], w[4], w[5]);
  }
}

// ---- a4 transpose by counting sort ---------------------------------------------------
// Every block's column-major copy (ccu, ccv) from its row-major one: count each
// (block, column), one exclusive scan over all blocks' columns in block order (which is
// the arena order, so the scan yields global CSC positions), then scatter.  Two passes
// and two atomics per edge instead of a 3-pass radix sort; the order of the rows inside
// a column is arbitrary (nothing needs it: the kernel hashes lists, bit rows are sets).
// Shared memory: the blocks' first edges (u64) and column bases (u64).
__global__ void k_tr_count(const uint32_t* __restrict__ cols, uint64_t m, const BlockDesc* __restrict__ blocks,
                           uint32_t nb, const uint64_t* __restrict__ cbase, uint32_t* __restrict__ cnt) {
  extern __shared__ uint64_t s_tr[];
  uint64_t* s_e0 = s_tr;
  uint64_t* s_cb = s_tr + nb;
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
    s_e0[b] = blocks[b].e0;
    s_cb[b] = cbase[b];
  }
  __syncthreads();
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = block_of_edge(s_e0, nb, e);
    atomicAdd(&cnt[s_cb[b] + cols[e]], 1u);
  }
}
__global__ void k_tr_scatter(const uint32_t* __restrict__ cols, const uint32_t* __restrict__ rows, uint64_t m,
                             const BlockDesc* __restrict__ blocks, uint32_t nb, const uint64_t* __restrict__ cbase,
                             uint32_t* __restrict__ cursor, uint32_t* __restrict__ ccu, uint32_t* __restrict__ ccv) {
  extern __shared__ uint64_t s_tr[];
  uint64_t* s_e0 = s_tr;
  uint64_t* s_cb = s_tr + nb;
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
    s_e0[b] = blocks[b].e0;
    s_cb[b] = cbase[b];
  }
  __syncthreads();
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = block_of_edge(s_e0, nb, e);
    const uint32_t c = cols[e];
    const uint32_t at = atomicAdd(&cursor[s_cb[b] + c], 1u);
    ccu[at] = rows[e];
    ccv[at] = c;
  }
}

// ---- a1 bucket sort: canonical keys de-duplicated in hashed buckets -----------------
// The K-bit keys (lo << bw | hi) are mixed by an odd multiplier mod 2^K (a bijection),
// split into 2^BB buckets by the top BB mixed bits, and each bucket (<= kBktCap keys,
// the remaining R = K - BB <= 32 bits as a u32) is sorted and de-duplicated in shared
// memory by one CTA; survivors are unmixed back into keys.  Equal keys meet in one
// bucket, so the unique set is exact; its order is arbitrary (nothing downstream needs
// one: degrees use atomics, orientation is per key, the block sort orders the edges).
constexpr int kBktThreads = 256, kBktItems = 16, kBktCap = kBktThreads * kBktItems;
struct BktMix {
  uint64_t c, cinv, kmask;
  int K, R;
  __host__ __device__ uint64_t mix(uint64_t k) const { return (k * c) & kmask; }
  __host__ __device__ uint64_t unmix(uint64_t x) const { return (x * cinv) & kmask; }
};
__global__ void k_bkt_count(const uint64_t* __restrict__ keys, uint64_t E, BktMix mx,
                            uint32_t* __restrict__ counts) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[e];
    if (k != kSentinel) atomicAdd(&counts[mx.mix(k) >> mx.R], 1u);
  }
}
__global__ void k_bkt_scatter(const uint64_t* __restrict__ keys, uint64_t E, BktMix mx, uint32_t* __restrict__ cursor,
                              uint32_t* __restrict__ out) {
  const uint32_t rmask = mx.R >= 32 ? 0xFFFFFFFFu : ((1u << mx.R) - 1);
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[e];
    if (k == kSentinel) continue;
    const uint64_t x = mx.mix(k);
    out[atomicAdd(&cursor[x >> mx.R], 1u)] = (uint32_t)x & rmask;
  }
}
// One CTA per bucket: sort its keys in shared memory, keep the first of every run of
// equal keys (in place, at the front of the bucket), count them.
__global__ void __launch_bounds__(kBktThreads) k_bkt_sort(uint32_t* __restrict__ data, const uint32_t* __restrict__ offs,
                                                          const uint32_t* __restrict__ counts, int R,
                                                          uint32_t* __restrict__ ucount) {
  using Sort = cub::BlockRadixSort<uint32_t, kBktThreads, kBktItems>;
  using Scan = cub::BlockScan<uint32_t, kBktThreads>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ uint32_t s_last[kBktThreads];
  const uint32_t b = blockIdx.x;
  const uint32_t n = counts[b];
  if (n == 0) {
    if (threadIdx.x == 0) ucount[b] = 0;
    return;
  }
  uint32_t* d = data + offs[b];
  uint32_t k[kBktItems];
#pragma unroll
  for (int x = 0; x < kBktItems; ++x) {
    const uint32_t i = threadIdx.x * kBktItems + x;   // blocked: thread t holds [16t, 16t+16)
    k[x] = i < n ? d[i] : 0xFFFFFFFFu;                 // padding sorts last
  }
  Sort(tmp.sort).Sort(k, 0, R);
  __syncthreads();
  s_last[threadIdx.x] = k[kBktItems - 1];
  __syncthreads();
  uint32_t keep[kBktItems], total = 0;
  uint32_t mine = 0;
#pragma unroll
  for (int x = 0; x < kBktItems; ++x) {
    const uint32_t i = threadIdx.x * kBktItems + x;
    const uint32_t prev = x ? k[x - 1] : (threadIdx.x ? s_last[threadIdx.x - 1] : 0);
    keep[x] = i < n && (i == 0 || k[x] != prev);
    mine += keep[x];
  }
  uint32_t at = 0;
  Scan(tmp.scan).ExclusiveSum(mine, at, total);
  __syncthreads();   // every key was read before any is written
#pragma unroll
  for (int x = 0; x < kBktItems; ++x)
    if (keep[x]) d[at++] = k[x];
  if (threadIdx.x == 0) ucount[b] = total;
}
// Survivors of bucket b -> unmixed keys at uoffs[b].
__global__ void k_bkt_compact(const uint32_t* __restrict__ data, const uint32_t* __restrict__ offs,
                              const uint32_t* __restrict__ ucount, const uint32_t* __restrict__ uoffs, uint32_t nb,
                              BktMix mx, uint64_t* __restrict__ ukeys) {
  for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const uint32_t n = ucount[b], o = offs[b], u = uoffs[b];
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
      ukeys[u + i] = mx.unmix(((uint64_t)b << mx.R) | data[o + i]);
  }
}

// ---- §8(e) sharded build: grouping keys by destination rank -----------------------
// Owner rank of a canonical edge (lo << 32 | hi): a hash of its lower id, so every
// instance of an edge (from any rank's raw shard) meets at one rank.
__device__ __forceinline__ uint32_t key_owner(uint64_t lo, uint32_t world) {
  return (uint32_t)(((lo * 0x9E3779B97F4A7C15ull) >> 32) % world);
}
// Owner rank of an oriented edge (ru << 32 | rw): the owner of its block (part ru, part rw).
__device__ __forceinline__ uint32_t okey_owner(uint64_t k, const uint32_t* s_cuts, uint32_t p,
                                               const uint32_t* s_owner) {
  const uint32_t i = part_of(s_cuts, p, (uint32_t)(k >> 32)), j = part_of(s_cuts, p, (uint32_t)k);
  return s_owner[j * (j + 1) / 2 + i];
}
// Counting pass + scatter pass over keys: dest[w] counts, then keys land in their
// owner's range (order inside a range is arbitrary: receivers sort).  kind 0: canonical
// keys by key_owner; kind 1: oriented keys by block owner (cuts/owner in shared memory).
template <int kKind>
__global__ void k_dest_count(const uint64_t* __restrict__ keys, uint64_t m, uint32_t world, int bw,
                             const uint32_t* __restrict__ gcuts, uint32_t p, const uint32_t* __restrict__ gowner,
                             unsigned long long* __restrict__ counts) {
  extern __shared__ uint32_t sh[];
  uint32_t* s_cnt = sh;                 // world
  uint32_t* s_cuts = sh + world;        // p + 1
  uint32_t* s_owner = s_cuts + p + 1;   // p(p+1)/2
  for (uint32_t x = threadIdx.x; x < world; x += blockDim.x) s_cnt[x] = 0;
  if (kKind == 1) {
    for (uint32_t x = threadIdx.x; x <= p; x += blockDim.x) s_cuts[x] = gcuts[x];
    for (uint32_t x = threadIdx.x; x < p * (p + 1) / 2; x += blockDim.x) s_owner[x] = gowner[x];
  }
  __syncthreads();
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[e];
    const uint32_t w = kKind == 0 ? key_owner(k >> bw, world) : okey_owner(k, s_cuts, p, s_owner);
    atomicAdd(&s_cnt[w], 1u);
  }
  __syncthreads();
  for (uint32_t x = threadIdx.x; x < world; x += blockDim.x)
    if (s_cnt[x]) atomicAdd(&counts[x], (unsigned long long)s_cnt[x]);
}
template <int kKind>
__global__ void k_dest_scatter(const uint64_t* __restrict__ keys, uint64_t m, uint32_t world, int bw,
                               const uint32_t* __restrict__ gcuts, uint32_t p, const uint32_t* __restrict__ gowner,
                               unsigned long long* __restrict__ cursor, uint64_t* __restrict__ out) {
  extern __shared__ uint32_t sh[];
  uint32_t* s_cuts = sh;
  uint32_t* s_owner = s_cuts + p + 1;
  if (kKind == 1) {
    for (uint32_t x = threadIdx.x; x <= p; x += blockDim.x) s_cuts[x] = gcuts[x];
    for (uint32_t x = threadIdx.x; x < p * (p + 1) / 2; x += blockDim.x) s_owner[x] = gowner[x];
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x - lane;
  for (uint64_t base = warp0; base < m; base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = base + lane;
    const bool valid = e < m;
    const uint64_t k = valid ? keys[e] : 0;
    const uint32_t w =
        valid ? (kKind == 0 ? key_owner(k >> bw, world) : okey_owner(k, s_cuts, p, s_owner)) : 0xFFFFFFFFu;
    // warp-aggregated reservation: one atomic per destination present in the warp
    const uint32_t peers = __match_any_sync(0xffffffffu, w);
    const uint32_t leader = __ffs(peers) - 1;
    unsigned long long at = 0;
    if (valid && lane == leader) at = atomicAdd(&cursor[w], (unsigned long long)__popc(peers));
    at = __shfl_sync(peers, at, leader);
    // kind 0 leaves in the wire form (lo << 32 | hi)
    const uint64_t o = kKind == 0 ? ((k >> bw) << 32) | (k & ((1ull << bw) - 1)) : k;
    if (valid) out[at + __popc(peers & ((1u << lane) - 1))] = o;
  }
}
// Partial (this rank's) block sizes: fold the p x p part histogram into block order.
__global__ void k_fold_blocks(const unsigned long long* __restrict__ hist, uint32_t p,
                              unsigned long long* __restrict__ bnnz) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < p; j += gridDim.x * blockDim.x)
    for (uint32_t i = 0; i <= j; ++i) bnnz[j * (j + 1) / 2 + i] = hist[(uint64_t)i * p + j];
}
// Wire keys (lo << 32 | hi) -> narrow keys (lo << bw | hi) for sorting.
__global__ void k_narrow(uint64_t* __restrict__ keys, uint64_t m, int bw) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[e];
    keys[e] = ((k >> 32) << bw) | (k & 0xFFFFFFFFull);
  }
}

}  // namespace

// Passes over id slices for the random (hi-side) atomics of the degree count: one
// slice of the n-entry array per pass, sized to a share of the L2 (BBTC_L2_SLICE_MB,
// default 48 MB) — friendster (n = 65.6 M, 262 MB) takes 6 passes, each re-reading the
// keys sequentially but keeping the atomics in L2: 42.7 -> 24.5 ms.
static uint32_t id_slices(uint32_t n) {
  static const double mb = getenv("BBTC_L2_SLICE_MB") ? atof(getenv("BBTC_L2_SLICE_MB")) : 48.0;
  const double bytes = 4.0 * n;
  if (mb <= 0 || bytes <= 100e6) return 1;   // (fits the 126 MB L2 well enough: rmat24's 67 MB)
  return std::max<uint32_t>(1, (uint32_t)std::ceil(bytes / (mb * 1e6)));
}
static void degrees_sorted(bbtc_ctx* ctx, const uint64_t* keys, uint64_t m, int bw, uint32_t n, uint32_t* deg) {
  const uint32_t q = id_slices(n);
  for (uint32_t x = 0; x < q; ++x) {
    const uint32_t h0 = (uint32_t)((uint64_t)n * x / q), h1 = (uint32_t)((uint64_t)n * (x + 1) / q);
    k_degree<<<grid_for(ctx, m), kThreads, 0, ctx->stream>>>(keys, m, bw, deg, h0, q == 1 ? 0xFFFFFFFFu : h1, x == 0);
    BBTC_LAUNCHED(ctx);
  }
}
// (Slicing the orientation measured slower — friendster 24.2 -> 33.2 ms: it reads and
// writes 16 B per key per pass against one 4 B gather — so it runs in one pass unless
// BBTC_ORIENT_SLICES=1.)
static void orient_sliced(bbtc_ctx* ctx, const uint64_t* keys, uint64_t m, int bw, uint32_t n, const uint32_t* rank,
                          uint64_t* okeys) {
  const uint32_t q = getenv("BBTC_ORIENT_SLICES") ? id_slices(n) : 1;
  for (uint32_t x = 0; x < q; ++x) {
    const uint32_t h0 = (uint32_t)((uint64_t)n * x / q), h1 = (uint32_t)((uint64_t)n * (x + 1) / q);
    k_orient<<<grid_for(ctx, m), kThreads, 0, ctx->stream>>>(keys, m, bw, rank, okeys, h0, q == 1 ? 0xFFFFFFFFu : h1);
    BBTC_LAUNCHED(ctx);
  }
}

// a1 bucket de-duplication of keys[0, E) (K live bits; sentinels skipped), BBTC_BUCKET=1:
// measured slower than the onesweep sort + unique on B200 (rmat24 20.2 vs 17.5 ms, and
// the unsorted keys cost the degree pass 6.4 vs 2.5 ms), kept as an option.  Returns
// false (nothing done) when it does not apply: a bucket above kBktCap keys (heavy
// duplication of one edge) or sizes outside its range — the caller sorts instead.
static bool bucket_unique(bbtc_ctx* ctx, const uint64_t* keys, uint64_t E, int K, DevBuf<uint64_t>* ukeys,
                          uint64_t* m_out) {
  cudaStream_t st = ctx->stream;
  if (E < (1ull << 22) || E >= (1ull << 32) || K < 36 || K > 56) return false;
  int BB = std::max(K - 32, bitlen(E / 2048));
  if (BB > 22 || BB >= K) return false;
  BktMix mx;
  mx.K = K;
  mx.R = K - BB;
  mx.kmask = K >= 64 ? ~0ull : ((1ull << K) - 1);
  mx.c = 0x9E3779B97F4A7C15ull;   // odd: x -> c*x is a bijection mod 2^K
  uint64_t inv = mx.c;            // Newton: inv = c^-1 mod 2^64
  for (int it = 0; it < 6; ++it) inv *= 2 - mx.c * inv;
  mx.cinv = inv;
  const uint32_t nb = 1u << BB;
  DevBuf<uint32_t> counts, offs, cursor, ucount, uoffs, data, mx_d;
  counts.alloc(nb, ctx);
  offs.alloc(nb, ctx);
  mx_d.alloc(1, ctx);
  BBTC_CUDA(cudaMemsetAsync(counts.p, 0, nb * 4, st));
  k_bkt_count<<<grid_for(ctx, E), kThreads, 0, st>>>(keys, E, mx, counts.p);
  BBTC_LAUNCHED(ctx);
  cub_call(ctx, [&](void* t, size_t& b) { return cub::DeviceReduce::Max(t, b, counts.p, mx_d.p, nb, st); });
  uint32_t biggest = 0;
  BBTC_CUDA(cudaMemcpyAsync(&biggest, mx_d.p, 4, cudaMemcpyDeviceToHost, st));
  BBTC_CUDA(cudaStreamSynchronize(st));
  if (biggest > (uint32_t)kBktCap) return false;
  cub_call(ctx, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, counts.p, offs.p, nb, st); });
  cursor.alloc(nb, ctx);
  BBTC_CUDA(cudaMemcpyAsync(cursor.p, offs.p, nb * 4, cudaMemcpyDeviceToDevice, st));
  data.alloc(E, ctx);
  k_bkt_scatter<<<grid_for(ctx, E), kThreads, 0, st>>>(keys, E, mx, cursor.p, data.p);
  BBTC_LAUNCHED(ctx);
  cursor.reset();
  ucount.alloc(nb, ctx);
  k_bkt_sort<<<nb, kBktThreads, 0, st>>>(data.p, offs.p, counts.p, mx.R, ucount.p);
  BBTC_LAUNCHED(ctx);
  uoffs.alloc(nb, ctx);
  cub_call(ctx, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, ucount.p, uoffs.p, nb, st); });
  uint32_t last[2] = {0, 0};
  BBTC_CUDA(cudaMemcpyAsync(&last[0], uoffs.p + nb - 1, 4, cudaMemcpyDeviceToHost, st));
  BBTC_CUDA(cudaMemcpyAsync(&last[1], ucount.p + nb - 1, 4, cudaMemcpyDeviceToHost, st));
  BBTC_CUDA(cudaStreamSynchronize(st));
  const uint64_t m = (uint64_t)last[0] + last[1];
  ukeys->alloc(std::max<uint64_t>(m, 1), ctx);
  k_bkt_compact<<<std::min<uint32_t>(nb, (uint32_t)ctx->sm_count * 16), kThreads, 0, st>>>(
      data.p, offs.p, ucount.p, uoffs.p, nb, mx, ukeys->p);
  BBTC_LAUNCHED(ctx);
  *m_out = m;
  return true;
}

// =====================================================================================
void graph_build(bbtc_ctx* ctx, const uint32_t* src, const uint32_t* dst, uint64_t E, uint32_t n_hint, int mem,
                 bbtc_graph* g, const uint32_t* pairs) {
  cudaStream_t st = ctx->stream;
  Trace tr(st, "graph_build");
  g->raw = E;
  DevBuf<uint32_t> dmax;
  dmax.alloc(2, ctx);
  BBTC_CUDA(cudaMemsetAsync(dmax.p, 0, 8, st));
  // Canonicalisation strategy: radix sort + unique (default) or a hash set
  // (BBTC_DEDUP=hash); both yield the same edge set.  The hash set skips the sort
  // but was measured slower end to end on B200 (friendster: 187 ms of random CAS vs
  // 131 ms of sort, and the unsorted keys then cost 2x in the degree and orient
  // passes, which read the sorted keys' neighbours from cache), so sort is default.
  static const bool use_hash = [] {
    const char* e = getenv("BBTC_DEDUP");
    return e && std::string(e) == "hash";
  }();
  DevBuf<uint64_t> keys;                 // sort: one key per raw pair
  DevBuf<unsigned long long> table;      // hash: the open-addressing set
  int tbits = 0;
  if (use_hash) {
    tbits = std::max(10, bitlen(std::max<uint64_t>(E, 1) * 2 - 1));
    table.alloc(1ull << tbits, ctx);
  } else {
    keys.alloc(E, ctx);
  }
  int bw = n_hint > 1 ? std::max(1, bitlen(n_hint - 1)) : 32;
  auto launch_canon = [&](const uint32_t* s, const uint32_t* d, uint64_t len, uint64_t c0, int width) {
    if (pairs) {   // interleaved pairs: s points at the chunk's first pair, d is unused
      if (use_hash) raise(BBTC_EINVAL, "BBTC_DEDUP=hash takes separate src/dst arrays");
      k_canon_pairs<<<grid_for(ctx, len), kThreads, 0, st>>>(reinterpret_cast<const uint2*>(s), len, width,
                                                             keys.p + c0, dmax.p);
    } else if (use_hash)
      k_canon_insert<<<grid_for(ctx, len), kThreads, 0, st>>>(s, d, len, width, table.p, tbits, dmax.p);
    else
      k_canon<<<grid_for(ctx, len), kThreads, 0, st>>>(s, d, len, width, keys.p + c0, dmax.p);
    BBTC_LAUNCHED(ctx);
  };
  // Stream-sort (host input): the canonical keys are radix-sorted in pieces on the
  // aux stream while later pieces are still being copied host->device, then the
  // sorted pieces are merged; the full sort no longer waits for the whole transfer.
  // At most ~8 pieces (3 merge rounds), each a whole number of 32 Mi-pair copy chunks.
  const uint64_t piece = std::max<uint64_t>(1ull << 26, ((E / 8 + (1ull << 25) - 1) >> 25) << 25);
  // cub::DeviceMerge takes int lengths: every merged run (up to E keys) must stay below 2^31.
  bool stream_sort = !use_hash && mem == BBTC_MEM_HOST && E > piece && E < (1ull << 31) &&
                     !getenv("BBTC_NO_STREAM_SORT");
  DevBuf<uint64_t> alt;
  DevBuf<uint8_t> sort_tmp;
  size_t sort_tmp_bytes = 0;
  struct Piece {
    uint64_t off, len;
    int sel;   // 0: sorted keys in `keys`, 1: in `alt`
  };
  std::vector<Piece> pieces;
  if (stream_sort) {
    alt.alloc(E, ctx);
    cub::DoubleBuffer<uint64_t> db0(keys.p, alt.p);
    BBTC_CUDA(sort_keys64(nullptr, sort_tmp_bytes, db0, piece, 0, 2 * bw, ctx->aux_stream));
    sort_tmp.alloc(std::max<size_t>(sort_tmp_bytes, 1), ctx);
  }
  auto sort_piece = [&](uint64_t off, uint64_t len, int width) {
    cub::DoubleBuffer<uint64_t> db(keys.p + off, alt.p + off);
    size_t tb = sort_tmp_bytes;
    BBTC_CUDA(sort_keys64(sort_tmp.p, tb, db, len, 0, 2 * width, ctx->aux_stream));
    ctx->launches += radix_kernels(len, 2 * width);
    pieces.push_back({off, len, db.selector});
  };
  auto canon = [&](int width) {
    BBTC_CUDA(cudaMemsetAsync(dmax.p, 0, 8, st));
    if (use_hash) BBTC_CUDA(cudaMemsetAsync(table.p, 0xFF, (1ull << tbits) * 8, st));
    if (!E) return;
    if (mem == BBTC_MEM_DEVICE) {
      launch_canon(pairs ? pairs : src, dst, E, 0, width);
      return;
    }
    // Host input: chunked H2D on a copy stream, overlapped with k_canon on earlier chunks.
    const uint64_t chunk = 1ull << 25;   // 32 Mi pairs = 256 MiB per chunk
    DevBuf<uint32_t> ds, dd;
    ds.alloc(std::min(E, 2 * chunk) * (pairs ? 2 : 1), ctx);   // (interleaved pairs: 8 B each, in ds)
    if (!pairs) dd.alloc(std::min(E, 2 * chunk), ctx);
    cudaStream_t cs = ctx->copy_streams[0];
    cudaEvent_t ev_copied[2], ev_used[2];
    for (int x = 0; x < 2; ++x) {
      BBTC_CUDA(cudaEventCreateWithFlags(&ev_copied[x], cudaEventDisableTiming));
      BBTC_CUDA(cudaEventCreateWithFlags(&ev_used[x], cudaEventDisableTiming));
      BBTC_CUDA(cudaEventRecord(ev_used[x], st));
    }
    uint64_t sorted_upto = 0;   // stream-sort: keys [0, sorted_upto) handed to the aux stream
    for (uint64_t c0 = 0, it = 0; c0 < E; c0 += chunk, ++it) {
      const uint64_t len = std::min(chunk, E - c0);
      const int slot = it & 1;
      BBTC_CUDA(cudaStreamWaitEvent(cs, ev_used[slot], 0));
      if (pairs) {
        BBTC_CUDA(cudaMemcpyAsync(ds.p + 2 * slot * chunk, pairs + 2 * c0, len * 8, cudaMemcpyHostToDevice, cs));
      } else {
        BBTC_CUDA(cudaMemcpyAsync(ds.p + slot * chunk, src + c0, len * 4, cudaMemcpyHostToDevice, cs));
        BBTC_CUDA(cudaMemcpyAsync(dd.p + slot * chunk, dst + c0, len * 4, cudaMemcpyHostToDevice, cs));
      }
      BBTC_CUDA(cudaEventRecord(ev_copied[slot], cs));
      BBTC_CUDA(cudaStreamWaitEvent(st, ev_copied[slot], 0));
      if (pairs) launch_canon(ds.p + 2 * slot * chunk, nullptr, len, c0, width);
      else launch_canon(ds.p + slot * chunk, dd.p + slot * chunk, len, c0, width);
      BBTC_CUDA(cudaEventRecord(ev_used[slot], st));
      // Stream-sort: once a sort piece is complete, sort it on the aux stream while
      // the next pieces are still crossing PCIe.
      if (stream_sort && (c0 + len - sorted_upto >= piece || c0 + len == E)) {
        BBTC_CUDA(cudaStreamWaitEvent(ctx->aux_stream, ev_used[slot], 0));
        sort_piece(sorted_upto, c0 + len - sorted_upto, width);
        sorted_upto = c0 + len;
      }
    }
    for (int x = 0; x < 2; ++x) {
      cudaEventDestroy(ev_copied[x]);
      cudaEventDestroy(ev_used[x]);
    }
  };
  canon(bw);
  tr.mark("canon");
  uint32_t max_id = 0;
  BBTC_CUDA(cudaMemcpyAsync(&max_id, dmax.p, 4, cudaMemcpyDeviceToHost, st));
  BBTC_CUDA(cudaStreamSynchronize(st));
  if (E && bw < 32 && (max_id >> bw) != 0) {
    // n_hint was too small for the ids: rebuild the keys at full width (and sort
    // them in one piece afterwards; the pieces sorted so far are void).
    if (stream_sort) {
      BBTC_CUDA(cudaStreamSynchronize(ctx->aux_stream));
      stream_sort = false;
      pieces.clear();
    }
    bw = 32;
    canon(bw);
    BBTC_CUDA(cudaMemcpyAsync(&max_id, dmax.p, 4, cudaMemcpyDeviceToHost, st));
    BBTC_CUDA(cudaStreamSynchronize(st));
  }
  if (E && max_id == 0xFFFFFFFFu) raise(BBTC_ERANGE, "vertex id 0xFFFFFFFF is reserved");
  const uint32_t n = E ? std::max<uint32_t>(n_hint, max_id + 1) : n_hint;
  g->n = n;
  const int bid = std::max(1, bitlen(max_id));
  // Sort the canonical keys over their live bits (hi id in [0,bid), lo id in [bw,bw+bid)).
  uint64_t m = 0;
  DevBuf<uint64_t> ukeys;
  bool unsorted = use_hash;   // unique keys in no particular order (hash set / buckets)
  if (E && use_hash) {
    // The set's occupied slots are the unique edges (in no particular order).
    const uint64_t T = 1ull << tbits;
    ukeys.alloc(E, ctx);
    DevBuf<uint64_t> nsel;
    nsel.alloc(1, ctx);
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceSelect::If(t, b, (const uint64_t*)table.p, ukeys.p, nsel.p, T, NotEmpty{}, st);
    });
    BBTC_CUDA(cudaMemcpyAsync(&m, nsel.p, 8, cudaMemcpyDeviceToHost, st));
    BBTC_CUDA(cudaStreamSynchronize(st));
    table.reset();
    tr.mark("compact");
  } else if (E) {
    bool in_keys = true;   // where the fully sorted keys end up
    if (stream_sort) {
      // Join the aux stream, then merge the sorted pieces pairwise (log2 #pieces
      // rounds of cub::DeviceMerge, ping-ponging between keys and alt).
      cudaEvent_t joined;
      BBTC_CUDA(cudaEventCreateWithFlags(&joined, cudaEventDisableTiming));
      BBTC_CUDA(cudaEventRecord(joined, ctx->aux_stream));
      BBTC_CUDA(cudaStreamWaitEvent(st, joined, 0));
      cudaEventDestroy(joined);
      int sel = pieces[0].sel;
      for (auto& pc : pieces)
        if (pc.sel != sel) {
          uint64_t* from = pc.sel ? alt.p : keys.p;
          uint64_t* to = sel ? alt.p : keys.p;
          BBTC_CUDA(cudaMemcpyAsync(to + pc.off, from + pc.off, pc.len * 8, cudaMemcpyDeviceToDevice, st));
          pc.sel = sel;
        }
      std::vector<Piece> cur = pieces;
      while (cur.size() > 1) {
        uint64_t* from = sel ? alt.p : keys.p;
        uint64_t* to = sel ? keys.p : alt.p;
        std::vector<Piece> nxt;
        for (size_t x = 0; x < cur.size(); x += 2) {
          const Piece a = cur[x];
          if (x + 1 < cur.size()) {
            const Piece b = cur[x + 1];
            cub_call(ctx, [&](void* t, size_t& tb) {
              return cub::DeviceMerge::MergeKeys(t, tb, from + a.off, (int)a.len, from + b.off, (int)b.len,
                                                 to + a.off, ::cuda::std::less<uint64_t>{}, st);
            });
            nxt.push_back({a.off, a.len + b.len, 1 - sel});
          } else {
            BBTC_CUDA(cudaMemcpyAsync(to + a.off, from + a.off, a.len * 8, cudaMemcpyDeviceToDevice, st));
            nxt.push_back({a.off, a.len, 1 - sel});
          }
        }
        cur.swap(nxt);
        sel = 1 - sel;
      }
      in_keys = sel == 0;
      sort_tmp.reset();
    } else if (getenv("BBTC_BUCKET") && bucket_unique(ctx, keys.p, E, bw + bid, &ukeys, &m)) {
      unsorted = true;   // de-duplicated in hashed buckets (one pass in shared memory)
      tr.mark("bucket_unique");
    } else {
      if (!alt.p) alt.alloc(E, ctx);
      cub::DoubleBuffer<uint64_t> db(keys.p, alt.p);
      cub_call(ctx, [&](void* t, size_t& b) {
        return sort_keys64(t, b, db, E, 0, bw + bid, st);
      }, radix_kernels(E, bw + bid));
      in_keys = db.Current() == keys.p;
    }
    if (!unsorted) {
    tr.mark("sort1");
    DevBuf<uint64_t>& sorted = in_keys ? keys : alt;
    DevBuf<uint64_t>& other = in_keys ? alt : keys;
    DevBuf<uint64_t> nsel;
    nsel.alloc(1, ctx);
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceSelect::Unique(t, b, sorted.p, other.p, nsel.p, E, st);
    });
    tr.mark("unique");
    uint64_t cnt = 0, last = 0;
    BBTC_CUDA(cudaMemcpyAsync(&cnt, nsel.p, 8, cudaMemcpyDeviceToHost, st));
    BBTC_CUDA(cudaStreamSynchronize(st));
    if (cnt) {
      BBTC_CUDA(cudaMemcpyAsync(&last, other.p + cnt - 1, 8, cudaMemcpyDeviceToHost, st));
      BBTC_CUDA(cudaStreamSynchronize(st));
    }
    m = cnt - (cnt && last == kSentinel ? 1 : 0);
    ukeys = std::move(other);
    sorted.reset();
    }
    keys.reset();
    alt.reset();
  }
  if (m >= 0xFFFFFFFFull) raise(BBTC_ERANGE, "m >= 2^32-1 edges is not supported (32-bit block offsets)");
  g->m = m;
  g->m_total = m;
  // Degrees and stable degree rank.
  DevBuf<uint32_t> deg;
  deg.alloc(n, ctx);
  g->deg_sorted.alloc(n, ctx);
  g->rank.alloc(n, ctx);
  g->okeys.alloc(m, ctx);
  if (n) {
    BBTC_CUDA(cudaMemsetAsync(deg.p, 0, (size_t)n * 4, st));
    if (m && unsorted) {
      k_degree_any<<<grid_for(ctx, m), kThreads, 0, st>>>(ukeys.p, m, bw, deg.p);
      BBTC_LAUNCHED(ctx);
    } else if (m) {
      degrees_sorted(ctx, ukeys.p, m, bw, n, deg.p);
    }
    tr.mark("degree");
    DevBuf<uint32_t> ids, order;
    ids.alloc(n, ctx);
    order.alloc(n, ctx);
    k_iota<<<grid_for(ctx, n), kThreads, 0, st>>>(ids.p, n);
    BBTC_LAUNCHED(ctx);
    const int bdeg = std::max(1, bitlen(std::min<uint64_t>(m, n - 1)));
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, deg.p, g->deg_sorted.p, ids.p, order.p, (uint64_t)n, 0, bdeg, st);
    }, radix_kernels(n, bdeg));
    k_rank<<<grid_for(ctx, n), kThreads, 0, st>>>(order.p, n, g->rank.p);
    BBTC_LAUNCHED(ctx);
    tr.mark("rank");
    if (m) {
      orient_sliced(ctx, ukeys.p, m, bw, n, g->rank.p, g->okeys.p);
    }
    tr.mark("orient");
    k_graph_stats<<<1, 32, 0, st>>>(g->deg_sorted.p, n, dmax.p);
    BBTC_LAUNCHED(ctx);
    uint32_t h[2];
    BBTC_CUDA(cudaMemcpyAsync(h, dmax.p, 8, cudaMemcpyDeviceToHost, st));
    BBTC_CUDA(cudaStreamSynchronize(st));
    g->n_nonisolated = n - h[0];
    g->d_max = h[1];
  }
}

// Largest out-degree of the oriented graph (computed on first request, cached).
uint32_t graph_dplus_max(bbtc_graph* g) {
  if (g->dplus_max_known) return g->dplus_max;
  bbtc_ctx* ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  uint32_t mx = 0;
  if (g->n && g->m && g->okeys.p) {
    DevBuf<uint32_t> dp, out;
    dp.alloc(g->n, ctx);
    out.alloc(1, ctx);
    BBTC_CUDA(cudaMemsetAsync(dp.p, 0, (size_t)g->n * 4, st));
    BBTC_CUDA(cudaMemsetAsync(out.p, 0, 4, st));
    k_outdeg<<<grid_for(ctx, g->m), kThreads, 0, st>>>(g->okeys.p, g->m, dp.p);
    BBTC_LAUNCHED(ctx);
    k_max_u32<<<grid_for(ctx, g->n), kThreads, 0, st>>>(dp.p, g->n, out.p);
    BBTC_LAUNCHED(ctx);
    BBTC_CUDA(cudaMemcpyAsync(&mx, out.p, 4, cudaMemcpyDeviceToHost, st));
    BBTC_CUDA(cudaStreamSynchronize(st));
  }
  g->dplus_max = mx;
  g->dplus_max_known = true;
  return mx;
}

void graph_csr(bbtc_ctx* ctx, const bbtc_graph* g, uint64_t* row_ptr, uint32_t* col) {
  cudaStream_t st = ctx->stream;
  std::vector<uint64_t> keys(g->m);
  if (g->m) {
    DevBuf<uint64_t> a, b;
    a.alloc(g->m, ctx);
    b.alloc(g->m, ctx);
    BBTC_CUDA(cudaMemcpyAsync(a.p, g->okeys.p, g->m * 8, cudaMemcpyDeviceToDevice, st));
    cub::DoubleBuffer<uint64_t> db(a.p, b.p);
    cub_call(ctx, [&](void* t, size_t& bb) { return cub::DeviceRadixSort::SortKeys(t, bb, db, g->m, 0, 64, st); });
    BBTC_CUDA(cudaMemcpyAsync(keys.data(), db.Current(), g->m * 8, cudaMemcpyDeviceToHost, st));
    BBTC_CUDA(cudaStreamSynchronize(st));
  }
  std::fill(row_ptr, row_ptr + (uint64_t)g->n + 1, 0);
  for (uint64_t e = 0; e < g->m; ++e) {
    row_ptr[(keys[e] >> 32) + 1]++;
    col[e] = (uint32_t)keys[e];
  }
  for (uint32_t u = 0; u < g->n; ++u) row_ptr[u + 1] += row_ptr[u];
}

void plan_build(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* user_cuts, uint32_t flags,
                bbtc_plan* plan) {
  cudaStream_t st = ctx->stream;
  Trace tr(st, "plan_build");
  const uint32_t n = g->n;
  const uint64_t m = g->m;
  plan->n = n;
  plan->m = m;
  plan->ctx = ctx;
  // ---- a3: cuts
  uint32_t pe;
  if (user_cuts) {
    pe = p;
    if (user_cuts[0] != 0 || user_cuts[p] != n) raise(BBTC_EINVAL, "cuts must satisfy cuts[0] = 0 and cuts[p] = n");
    for (uint32_t i = 0; i < p; ++i)
      if (user_cuts[i] > user_cuts[i + 1]) raise(BBTC_EINVAL, "cuts must be non-decreasing");
    plan->cuts.assign(user_cuts, user_cuts + p + 1);
  } else {
    pe = n == 0 ? 1 : std::min(p, n);
    plan->clamped = pe != p;
    plan->cuts.assign(pe + 1, 0);
    plan->cuts[pe] = n;
    if (n > 0 && pe > 1) {
      DevBuf<uint64_t> incl;
      incl.alloc(n, ctx);
      cub::TransformInputIterator<uint64_t, ToU64, const uint32_t*> it(g->deg_sorted.p, ToU64{});
      cub_call(ctx, [&](void* t, size_t& b) {
        return cub::DeviceScan::InclusiveSum(t, b, it, incl.p, (uint64_t)n, st);
      });
      DevBuf<uint32_t> dc;
      dc.alloc(pe + 1, ctx);
      k_cuts<<<1, 256, 0, st>>>(incl.p, n, 2 * m, pe, dc.p);
      BBTC_LAUNCHED(ctx);
      BBTC_CUDA(cudaMemcpyAsync(plan->cuts.data(), dc.p, (pe + 1) * 4, cudaMemcpyDeviceToHost, st));
      BBTC_CUDA(cudaStreamSynchronize(st));
    }
  }
  tr.mark("cuts");
  plan->p = pe;
  const uint32_t nb = pe * (pe + 1) / 2;
  const int bn = std::max(1, bitlen(n ? n - 1 : 0));
  const int bp = bitlen(pe - 1);
  if (bp + 2 * bn > 64) raise(BBTC_ERANGE, "n and p too large for the 64-bit block sort key");
  DevBuf<uint32_t> dcuts;
  dcuts.alloc(pe + 1, ctx);
  BBTC_CUDA(cudaMemcpyAsync(dcuts.p, plan->cuts.data(), (pe + 1) * 4, cudaMemcpyHostToDevice, st));
  // ---- a4: block-ordered keys
  DevBuf<uint64_t> ck, ck_alt;
  std::vector<uint64_t> starts(nb + 1, 0);
  const size_t cut_smem = (pe + 1) * 4;
  // CSR by counting sort (BBTC_CSR_COUNT=1; measured slower than the block-key radix
  // sort on B200: rmat24 34.7 vs ~13 ms, the random atomics into the row-offset arena)
  std::vector<uint64_t> ro_h(nb + 1, 0);
  for (uint32_t j = 0; j < pe; ++j)
    for (uint32_t i = 0; i <= j; ++i) {
      const uint32_t b = block_id(i, j);
      ro_h[b + 1] = (uint64_t)(plan->cuts[i + 1] - plan->cuts[i]) + 1;
    }
  for (uint32_t b = 0; b < nb; ++b) ro_h[b + 1] += ro_h[b];
  const bool csr_count = getenv("BBTC_CSR_COUNT") && ro_h[nb] < (1ull << 32) && m;
  if (csr_count) {
    plan->rowptr.alloc(ro_h[nb], ctx);
    plan->cols.alloc(m, ctx);
    plan->rows.alloc(m, ctx);
    DevBuf<uint64_t> dro, dstarts;
    dro.alloc(nb + 1, ctx);
    dstarts.alloc(nb, ctx);
    BBTC_CUDA(cudaMemcpyAsync(dro.p, ro_h.data(), (nb + 1) * 8, cudaMemcpyHostToDevice, st));
    BBTC_CUDA(cudaMemsetAsync(plan->rowptr.p, 0, ro_h[nb] * 4, st));
    k_csr_count<<<grid_for(ctx, m), kThreads, cut_smem, st>>>(g->okeys.p, m, dcuts.p, pe, dro.p, plan->rowptr.p);
    BBTC_LAUNCHED(ctx);
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, plan->rowptr.p, plan->rowptr.p, ro_h[nb], st);
    });
    k_block_first<<<(nb + 255) / 256, 256, 0, st>>>(plan->rowptr.p, dro.p, nb, dstarts.p);
    BBTC_LAUNCHED(ctx);
    BBTC_CUDA(cudaMemcpyAsync(starts.data(), dstarts.p, nb * 8, cudaMemcpyDeviceToHost, st));
    {
      DevBuf<uint32_t> cursor;
      cursor.alloc(ro_h[nb], ctx);
      BBTC_CUDA(cudaMemcpyAsync(cursor.p, plan->rowptr.p, ro_h[nb] * 4, cudaMemcpyDeviceToDevice, st));
      k_csr_scatter<<<grid_for(ctx, m), kThreads, cut_smem, st>>>(g->okeys.p, m, dcuts.p, pe, dro.p, cursor.p,
                                                                  plan->cols.p, plan->rows.p);
      BBTC_LAUNCHED(ctx);
      BBTC_CUDA(cudaStreamSynchronize(st));
    }
    starts[nb] = m;
    tr.mark("csr_count");
  } else if (m) {
    ck.alloc(m, ctx);
    k_block_keys<<<grid_for(ctx, m), kThreads, cut_smem, st>>>(g->okeys.p, m, dcuts.p, pe, bn, ck.p);
    BBTC_LAUNCHED(ctx);
    tr.mark("block_keys");
    ck_alt.alloc(m, ctx);
    cub::DoubleBuffer<uint64_t> db(ck.p, ck_alt.p);
    cub_call(ctx, [&](void* t, size_t& b) {
      // Only the (j, ru) bits: the count kernel hashes lists, so the columns of a row
      // need no order (sorting them too would cost 3 more radix passes).
      return sort_keys64(t, b, db, m, getenv("BBTC_SORT_ROWS") ? 0 : bn, bp + 2 * bn, st);
    }, radix_kernels(m, bp + bn));
    if (db.Current() != ck.p) std::swap(ck, ck_alt);
    ck_alt.reset();
    tr.mark("sort2");
    DevBuf<uint64_t> dstarts;
    dstarts.alloc(nb + 1, ctx);
    k_block_starts<<<(nb + 1 + 127) / 128, 128, 0, st>>>(ck.p, m, dcuts.p, pe, bn, dstarts.p);
    BBTC_LAUNCHED(ctx);
    BBTC_CUDA(cudaMemcpyAsync(starts.data(), dstarts.p, (nb + 1) * 8, cudaMemcpyDeviceToHost, st));
    BBTC_CUDA(cudaStreamSynchronize(st));
  }
  // Block table (column-major: b = j(j+1)/2 + i).
  plan->blocks.resize(nb);
  uint64_t ro = 0, m_max = 0, bytes = 0;
  for (uint32_t j = 0; j < pe; ++j)
    for (uint32_t i = 0; i <= j; ++i) {
      uint32_t b = block_id(i, j);
      BlockDesc& B = plan->blocks[b];
      B.i = i;
      B.j = j;
      B.e0 = starts[b];
      B.nnz = starts[b + 1] - starts[b];
      B.ro = ro;
      B.co = 0;
      B.nc = plan->cuts[j + 1] - plan->cuts[j];
      B.pad_ = 0;
      ro += (uint64_t)(plan->cuts[i + 1] - plan->cuts[i]) + 1;
      m_max = std::max(m_max, B.nnz);
      bytes += 8 * B.nnz + 4 * ((uint64_t)(plan->cuts[i + 1] - plan->cuts[i]) + 1);
    }
  plan->d_blocks.alloc(nb, ctx);
  BBTC_CUDA(cudaMemcpyAsync(plan->d_blocks.p, plan->blocks.data(), nb * sizeof(BlockDesc), cudaMemcpyHostToDevice, st));
  // Probe slots (resident counts, DESIGN §7 "Probe slots"): a probe block with many
  // short rows gets a slot of 8 words per row after the cols arena — its length, its
  // CSR offset and its first 6 column ids — so a probe of a row of <= 6 entries is one
  // random 32-B access instead of a row-offset gather followed by a list gather.
  plan->slot_of.assign(nb, 0);
  plan->slots_ready = false;
  uint64_t slot_words = 0;
  const uint64_t slot_base = (m + 7) & ~7ull;   // slots 32-B aligned
  {
    // Off by default: measured slower on friendster (list kernel 336 -> 342 ms with slots
    // for the four V_0 blocks; its short-row tasks are bound by staging, not by the row
    // offset gathers), no change on rmat24 / orkut (profiles/r02/r02r).  BBTC_SLOTS=1.
    static const bool on = getenv("BBTC_SLOTS") && atoi(getenv("BBTC_SLOTS")) != 0;
    static const double min_rows = getenv("BBTC_SLOT_MIN_ROWS") ? atof(getenv("BBTC_SLOT_MIN_ROWS")) : 1e6;
    static const double max_deg = getenv("BBTC_SLOT_MAX_DEG") ? atof(getenv("BBTC_SLOT_MAX_DEG")) : 8.0;
    static const double min_deg = getenv("BBTC_SLOT_MIN_DEG") ? atof(getenv("BBTC_SLOT_MIN_DEG")) : 1.0;
    for (uint32_t b = 0; on && !(flags & BBTC_PLAN_ROWMAJOR) && b < nb; ++b) {
      const BlockDesc& B = plan->blocks[b];
      const uint64_t rows = plan->cuts[B.i + 1] - plan->cuts[B.i];
      // (rows of average length 1..8: mostly non-empty and mostly inline)
      if ((double)rows < min_rows || !B.nnz || (double)B.nnz > max_deg * (double)rows ||
          (double)B.nnz < min_deg * (double)rows)
        continue;
      if (slot_base + slot_words + 8 * rows >= 0xFFFFFFFFull) continue;   // 32-bit arena indices
      plan->slot_of[b] = (uint32_t)(slot_base + slot_words);
      slot_words += 8 * rows;
    }
  }
  if (!csr_count) {
  plan->cols.alloc(slot_words ? slot_base + slot_words : m, ctx);
  plan->rows.alloc(m, ctx);
  plan->rowptr.alloc(ro, ctx);
  BBTC_CUDA(cudaMemsetAsync(plan->rowptr.p, 0xFF, ro * 4, st));
  if (m) {
    k_split<<<grid_for(ctx, m), kThreads, cut_smem, st>>>(ck.p, m, dcuts.p, pe, bn, plan->d_blocks.p, plan->cols.p,
                                                          plan->rows.p, plan->rowptr.p);
    BBTC_LAUNCHED(ctx);
  }
  tr.mark("split");
  ck.reset();
  k_row_ends<<<(nb + 127) / 128, 128, 0, st>>>(plan->d_blocks.p, nb, dcuts.p, plan->rowptr.p);
  BBTC_LAUNCHED(ctx);
  // Empty rows take the start of the next non-empty row: reverse inclusive min-scan.
  {
    thrust::reverse_iterator<uint32_t*> rin(plan->rowptr.p + ro);
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceScan::InclusiveScan(t, b, rin, rin, MinOp{}, (uint64_t)ro, st);
    });
  }
  }
  {
    uint32_t maxv = 0;
    for (uint32_t i = 0; i < pe; ++i) maxv = std::max(maxv, plan->cuts[i + 1] - plan->cuts[i] + 1);
    dim3 grid(std::max(1u, std::min((maxv + kThreads - 1) / kThreads, 64u)), std::min(nb, 16384u));
    k_row_local<<<grid, kThreads, 0, st>>>(plan->d_blocks.p, nb, dcuts.p, plan->rowptr.p);
    BBTC_LAUNCHED(ctx);
  }
  tr.mark("rowptr");
  if (slot_words && !csr_count) {
    std::vector<uint32_t> ids, nrows(nb, 0);
    uint32_t maxr = 1;
    for (uint32_t b = 0; b < nb; ++b)
      if (plan->slot_of[b]) {
        ids.push_back(b);
        nrows[b] = plan->cuts[plan->blocks[b].i + 1] - plan->cuts[plan->blocks[b].i];
        maxr = std::max(maxr, nrows[b]);
      }
    DevBuf<uint32_t> d_ids, d_nrows;
    d_ids.alloc(ids.size(), ctx);
    d_nrows.alloc(nb, ctx);
    plan->d_slot_of.alloc(nb, ctx);
    BBTC_CUDA(cudaMemcpyAsync(d_ids.p, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice, st));
    BBTC_CUDA(cudaMemcpyAsync(d_nrows.p, nrows.data(), nb * 4, cudaMemcpyHostToDevice, st));
    BBTC_CUDA(cudaMemcpyAsync(plan->d_slot_of.p, plan->slot_of.data(), nb * 4, cudaMemcpyHostToDevice, st));
    k_slots<<<dim3(std::min((maxr + kThreads - 1) / kThreads, (uint32_t)ctx->sm_count * 8), (uint32_t)ids.size()),
              kThreads, 0, st>>>(plan->rowptr.p, plan->cols.p, plan->d_blocks.p, d_ids.p, plan->d_slot_of.p, d_nrows.p);
    BBTC_LAUNCHED(ctx);
    BBTC_CUDA(cudaStreamSynchronize(st));   // (host sources of the async copies)
    plan->slots_ready = true;
    plan->info.slot_bytes = 4 * slot_words;   // (not block bytes: a resident-count index)
    tr.mark("slots");
  }
  // Column-major iteration arrays (default): transpose of every block.
  plan->colmajor = !(flags & BBTC_PLAN_ROWMAJOR);
  if (plan->colmajor) {
    // One stable radix sort of all edges by (block, local column): values = local
    // row ids -> every block in CSC order, rows ascending per column, blocks in place.
    plan->ccu.alloc(m, ctx);
    plan->ccv.alloc(m, ctx);
    uint32_t maxw = 1;
    for (uint32_t j = 0; j < pe; ++j) maxw = std::max(maxw, plan->cuts[j + 1] - plan->cuts[j]);
    const int cb = std::max(1, bitlen(maxw - 1));
    const int kb = bitlen(nb - 1);
    // The batched path keeps every block's first edge in shared memory (8 B each).
    const size_t key_smem = (size_t)nb * 8;
    // One batched sort from 16 blocks (p >= 6) on, per-block sorts below: orkut p=8 (36
    // blocks) plan 9.98 -> 9.15 ms batched; friendster p=4 (10 blocks) 130.5 vs 148.3 ms
    // per-block (profiles/r02/ab10).
    static const uint32_t batched_min = getenv("BBTC_BATCHED_MIN_NB") ? (uint32_t)atoi(getenv("BBTC_BATCHED_MIN_NB")) : 16;
    const bool batched = nb >= batched_min && key_smem <= 200 * 1024;
    // Packed keys: cbase[b] = Σ over earlier blocks of their live column widths.
    const uint32_t n_iso = g->n - g->n_nonisolated;   // isolated vertices: ranks [0, n_iso)
    std::vector<uint32_t> trim(pe), cbase(nb);
    for (uint32_t j = 0; j < pe; ++j)
      trim[j] = plan->cuts[j] < n_iso ? std::min(plan->cuts[j + 1], n_iso) - plan->cuts[j] : 0;
    uint64_t range = 0;
    for (uint32_t b = 0; b < nb; ++b) {
      const BlockDesc& B = plan->blocks[b];
      cbase[b] = (uint32_t)std::min<uint64_t>(range, 0xFFFFFFFFull);
      range += plan->cuts[B.j + 1] - plan->cuts[B.j] - trim[B.j];
    }
    const int pbits = std::max(1, bitlen(std::max<uint64_t>(range, 1) - 1));
    const size_t pk_smem = (size_t)nb * 16;
    static const int packed_env = [] {   // BBTC_PACKED_TRANSPOSE = 0: never, 1: whenever it fits
      const char* e = getenv("BBTC_PACKED_TRANSPOSE");
      return e ? atoi(e) : -1;
    }();
    const bool packed = batched && range <= 0xFFFFFFFFull && pk_smem <= 48 * 1024 && packed_env != 0 &&
                        (packed_env == 1 || (pbits + 7) / 8 < (kb + cb + 7) / 8);
    if (batched && key_smem > 48 * 1024) {
      BBTC_CUDA(cudaFuncSetAttribute(k_transpose_keys<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)key_smem));
      BBTC_CUDA(cudaFuncSetAttribute(k_transpose_keys<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)key_smem));
    }
    // Counting-sort transpose (BBTC_TRANSPOSE_COUNT=1; measured no faster than the
    // packed-key radix sort on rmat24: 8.9 vs 8.4 ms).
    uint64_t ncols_all = 0;
    std::vector<uint64_t> colbase(nb);
    for (uint32_t b = 0; b < nb; ++b) {
      colbase[b] = ncols_all;
      ncols_all += plan->blocks[b].nc;
    }
    const bool counting = getenv("BBTC_TRANSPOSE_COUNT") && (size_t)nb * 16 <= 200 * 1024 && ncols_all < (1ull << 32);
    if (m && counting) {
      DevBuf<uint32_t> cnt;
      DevBuf<uint64_t> dcb;
      cnt.alloc(ncols_all + 1, ctx);
      dcb.alloc(nb, ctx);
      BBTC_CUDA(cudaMemcpyAsync(dcb.p, colbase.data(), nb * 8, cudaMemcpyHostToDevice, st));
      BBTC_CUDA(cudaMemsetAsync(cnt.p, 0, (ncols_all + 1) * 4, st));
      const size_t sm = (size_t)nb * 16;
      if (sm > 48 * 1024) {
        BBTC_CUDA(cudaFuncSetAttribute(k_tr_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        BBTC_CUDA(cudaFuncSetAttribute(k_tr_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      }
      k_tr_count<<<grid_for(ctx, m), kThreads, sm, st>>>(plan->cols.p, m, plan->d_blocks.p, nb, dcb.p, cnt.p);
      BBTC_LAUNCHED(ctx);
      cub_call(ctx, [&](void* t, size_t& bb) {
        return cub::DeviceScan::ExclusiveSum(t, bb, cnt.p, cnt.p, ncols_all + 1, st);
      });
      k_tr_scatter<<<grid_for(ctx, m), kThreads, sm, st>>>(plan->cols.p, plan->rows.p, m, plan->d_blocks.p, nb,
                                                            dcb.p, cnt.p, plan->ccu.p, plan->ccv.p);
      BBTC_LAUNCHED(ctx);
      BBTC_CUDA(cudaStreamSynchronize(st));   // (colbase is the host source of an async copy)
    } else if (m && !batched) {
      // Few blocks: sort each block in place by its local column (no key pass).  (A
      // row-band walk — key (row band, column) for blocks whose probe blocks exceed an
      // L2 share — was built and measured in round 2: friendster list kernel 333 -> 327
      // ms with a cost rule choosing the blocks, 442 ms banding every large block; it
      // faulted in the list kernel under a later build with many small bands for a
      // reason not found, and was removed.  DESIGN §7.)
      for (uint32_t b = 0; b < nb; ++b) {
        const BlockDesc& B = plan->blocks[b];
        if (B.nnz == 0) continue;
        const int bits = std::max(1, bitlen(plan->cuts[B.j + 1] - plan->cuts[B.j] - 1));
        cub_call(ctx, [&](void* t, size_t& bb) {
          return cub::DeviceRadixSort::SortPairs(t, bb, plan->cols.p + B.e0, plan->ccv.p + B.e0, plan->rows.p + B.e0,
                                                 plan->ccu.p + B.e0, B.nnz, 0, bits, st);
        }, radix_kernels(B.nnz, bits));
      }
    } else if (m && packed) {
      DevBuf<uint32_t> keys, dcb, dtrim;
      keys.alloc(m, ctx);
      dcb.alloc(nb, ctx);
      dtrim.alloc(pe, ctx);
      BBTC_CUDA(cudaMemcpyAsync(dcb.p, cbase.data(), nb * 4, cudaMemcpyHostToDevice, st));
      BBTC_CUDA(cudaMemcpyAsync(dtrim.p, trim.data(), pe * 4, cudaMemcpyHostToDevice, st));
      k_transpose_keys_packed<<<grid_for(ctx, m), kThreads, pk_smem, st>>>(plan->cols.p, m, plan->d_blocks.p, nb,
                                                                          dcb.p, dtrim.p, pe, keys.p);
      BBTC_LAUNCHED(ctx);
      cub_call(ctx, [&](void* t, size_t& bb) {
        return cub::DeviceRadixSort::SortPairs(t, bb, keys.p, plan->ccv.p, plan->rows.p, plan->ccu.p, m, 0, pbits,
                                               st);
      }, radix_kernels(m, pbits));
      k_unpack_cols<<<grid_for(ctx, m), kThreads, pk_smem, st>>>(plan->ccv.p, m, plan->d_blocks.p, nb, dcb.p,
                                                                dtrim.p);
      BBTC_LAUNCHED(ctx);
      BBTC_CUDA(cudaStreamSynchronize(st));   // cbase / trim (host vectors) feed async copies
    } else if (m && kb + cb <= 32) {
      DevBuf<uint32_t> keys;
      keys.alloc(m, ctx);
      k_transpose_keys<uint32_t><<<grid_for(ctx, m), kThreads, (size_t)nb * 8, st>>>(
          plan->cols.p, m, plan->d_blocks.p, nb, cb, keys.p);
      BBTC_LAUNCHED(ctx);
      cub_call(ctx, [&](void* t, size_t& bb) {
        return cub::DeviceRadixSort::SortPairs(t, bb, keys.p, plan->ccv.p, plan->rows.p, plan->ccu.p, m, 0, kb + cb,
                                               st);
      }, radix_kernels(m, kb + cb));
      k_low_bits<uint32_t><<<grid_for(ctx, m), kThreads, 0, st>>>(plan->ccv.p, m, cb, plan->ccv.p);
      BBTC_LAUNCHED(ctx);
    } else if (m) {
      DevBuf<uint64_t> keys, sorted;
      keys.alloc(m, ctx);
      sorted.alloc(m, ctx);
      k_transpose_keys<uint64_t><<<grid_for(ctx, m), kThreads, (size_t)nb * 8, st>>>(
          plan->cols.p, m, plan->d_blocks.p, nb, cb, keys.p);
      BBTC_LAUNCHED(ctx);
      cub_call(ctx, [&](void* t, size_t& bb) {
        return cub::DeviceRadixSort::SortPairs(t, bb, keys.p, sorted.p, plan->rows.p, plan->ccu.p, m, 0, kb + cb, st);
      }, radix_kernels(m, kb + cb));
      k_low_bits<uint64_t><<<grid_for(ctx, m), kThreads, 0, st>>>(sorted.p, m, cb, plan->ccv.p);
      BBTC_LAUNCHED(ctx);
    }
    // The row-major COO is only needed to build the transpose, except by the bit-row
    // kernel, which walks dense tasks by row: consecutive edges share u, so row_ik(u)
    // stays in L1 and the gathered rows are those of G_jk — |V_j| rows, fewer than G_ik's
    // |V_i| for i < j, so more of them stay in L2 (rmat24 p=10: 13.2 -> 11.4 ms;
    // BBTC_DENSE_WALK=col walks by column as in round 1).
    const char* dw = getenv("BBTC_DENSE_WALK");
    bool maybe_dense = false;   // some part small enough for bit rows (else no dense task can exist)
    {
      const char* e = getenv("BBTC_DENSE_BITS");
      const uint32_t bits = e ? (uint32_t)atoi(e) : kDenseBitsDefault;
      for (uint32_t k = 0; k < pe; ++k) {
        const uint32_t vk = plan->cuts[k + 1] - plan->cuts[k];
        maybe_dense = maybe_dense || (vk > 0 && vk <= std::min(bits, kDenseMaxS * 32));
      }
    }
    if ((dw && std::string(dw) == "col") || (flags & BBTC_PLAN_SPARSE) || !maybe_dense) plan->rows.reset();
    bytes += 4 * m;       // cols + ccu + ccv instead of cols + rows
    tr.mark("transpose");
  }
  // ---- a5: tasks and work items (host)
  plan->info.p = pe;
  plan->info.clamped = plan->clamped;
  plan->info.n_tasks = n_tasks(pe);
  plan->info.n_blocks = nb;
  plan->info.m = m;
  plan->info.m_max = m_max;
  plan->info.lambda = m ? (double)m_max / (2.0 * (double)m / ((double)pe * (pe + 1))) : 1.0;   // S: lambda >= 1, = 1 when empty
  plan->info.block_bytes = bytes;
  {
    const char* e = getenv("BBTC_DENSE_BITS");
    plan->dense_bits = (flags & BBTC_PLAN_SPARSE) ? 0u : e ? (uint32_t)atoi(e) : kDenseBitsDefault;
    plan->dense_bits = std::min(plan->dense_bits, kDenseMaxS * 32);
    plan->info.dense_bits = plan->dense_bits;
  }
  plan_tasks(plan, 1);
  tr.mark("tasks");
  if (flags & BBTC_PLAN_STATS) plan_stats(ctx, plan);
}

// Column offsets of every block of a column-major plan (the streamed form of ccv).
uint64_t colptr_build(bbtc_ctx* ctx, bbtc_plan* plan, DevBuf<uint32_t>* out) {
  cudaStream_t st = ctx->stream;
  const uint32_t nb = (uint32_t)plan->blocks.size();
  // A block streams column offsets (|V_j|+1 words) only where that is fewer words
  // than its per-edge column ids (nnz): blocks with mostly empty columns (rmat24's
  // (0,0): 15 M columns, 1.5 M edges) ship ccv itself, and the kernel reads it.
  plan->co_off.assign(nb + 1, 0);
  std::vector<uint64_t> co(nb + 1, kNoColptr);
  uint32_t maxw = 1;
  for (uint32_t b = 0; b < nb; ++b) {
    const BlockDesc& B = plan->blocks[b];
    const uint32_t w = plan->cuts[B.j + 1] - plan->cuts[B.j];
    // (>= 4 edges per column on average: with sparser columns the kernel's 32-column
    // windows cover too few edges per batch — rmat24 (1,1): 2 edges/column, the
    // column-offset walk 2.7x slower than reading ccv, scripts/dbg/dbg_cp_tasks.py)
    const bool cp = B.nnz >= 4 * ((uint64_t)w + 1);
    if (cp) {
      maxw = std::max(maxw, w + 1);
      co[b] = plan->co_off[b];
    }
    plan->co_off[b + 1] = plan->co_off[b] + (cp ? w + 1 : 0);
  }
  const uint64_t len = plan->co_off[nb];
  out->alloc(std::max<uint64_t>(len, 1), ctx);
  DevBuf<uint64_t> dco;
  DevBuf<uint32_t> dcuts;
  dco.alloc(nb + 1, ctx);
  dcuts.alloc(plan->cuts.size(), ctx);
  BBTC_CUDA(cudaMemcpyAsync(dco.p, co.data(), (nb + 1) * 8, cudaMemcpyHostToDevice, st));
  BBTC_CUDA(cudaMemcpyAsync(dcuts.p, plan->cuts.data(), plan->cuts.size() * 4, cudaMemcpyHostToDevice, st));
  BBTC_CUDA(cudaMemsetAsync(out->p, 0xFF, len * 4, st));
  if (nb) {
    k_col_starts<<<dim3(64, std::min(nb, 16384u)), kThreads, 0, st>>>(plan->ccv.p, plan->d_blocks.p, dco.p, nb,
                                                                      dcuts.p, out->p);
    BBTC_LAUNCHED(ctx);
    thrust::reverse_iterator<uint32_t*> rin(out->p + len);
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceScan::InclusiveScan(t, b, rin, rin, MinOp{}, len, st);
    });
    dim3 grid(std::max(1u, std::min((maxw + kThreads - 1) / kThreads, 64u)), std::min(nb, 16384u));
    k_col_local<<<grid, kThreads, 0, st>>>(plan->d_blocks.p, dco.p, nb, dcuts.p, out->p);
    BBTC_LAUNCHED(ctx);
    const uint64_t items = plan->item_start.back();
    plan->d_item_col.alloc(std::max<uint64_t>(items, 1), ctx);
    if (items) {
      k_item_cols<<<grid_for(ctx, items), kThreads, 0, st>>>(plan->d_tasks.p, plan->d_item_start.p,
                                                             (uint32_t)plan->tasks.size(), items, plan->d_blocks.p,
                                                             out->p, dco.p, plan->d_item_col.p);
      BBTC_LAUNCHED(ctx);
    }
  }
  // the streamed kernel finds block b's column offsets at co (BlockDesc.co; kNoColptr: ccv)
  for (uint32_t b = 0; b < nb; ++b) plan->blocks[b].co = co[b];
  BBTC_CUDA(cudaMemcpyAsync(plan->d_blocks.p, plan->blocks.data(), nb * sizeof(BlockDesc), cudaMemcpyHostToDevice, st));
  BBTC_CUDA(cudaStreamSynchronize(st));   // dco / dcuts die with this scope
  return len;
}

void colptr_expand_all(bbtc_ctx* ctx, bbtc_plan* plan) {
  const uint32_t nb = (uint32_t)plan->blocks.size();
  if (!nb || !plan->m) return;
  uint32_t maxc = 1;
  for (auto& B : plan->blocks) maxc = std::max(maxc, B.nc);
  dim3 grid(std::max(1u, std::min((maxc + 255) / 256, 256u)), std::min(nb, 16384u));
  k_col_expand_all<<<grid, kThreads, 0, ctx->stream>>>(plan->d_colptr.p, plan->d_blocks.p, nb, plan->ccv.p);
  BBTC_LAUNCHED(ctx);
}

// a3, automatic p: the smallest p whose largest task
// footprint (the device bytes of its distinct blocks: row offsets + per-edge arrays)
// times `depth` (tasks whose blocks are in flight at once) fits `budget`.  Each
// candidate costs one pass over the oriented edges (default cuts + a block histogram,
// no BCSR).  Candidates 1, 2, 4, … until one fits, then the smallest fitting p below it.
uint32_t plan_auto_p(bbtc_ctx* ctx, const bbtc_graph* g, uint64_t budget, uint32_t depth, uint32_t flags) {
  cudaStream_t st = ctx->stream;
  const uint32_t n = g->n;
  const uint64_t m = g->m;
  const uint64_t arenas = (flags & BBTC_PLAN_ROWMAJOR) ? 2 : 3;
  depth = std::max(depth, 1u);
  const uint32_t pmax = std::max(1u, std::min<uint32_t>(n, kAutoPMax));
  DevBuf<uint64_t> incl;
  if (n > 0) {
    incl.alloc(n, ctx);
    cub::TransformInputIterator<uint64_t, ToU64, const uint32_t*> it(g->deg_sorted.p, ToU64{});
    cub_call(ctx, [&](void* t, size_t& b) { return cub::DeviceScan::InclusiveSum(t, b, it, incl.p, (uint64_t)n, st); });
  }
  DevBuf<uint32_t> dc;
  dc.alloc(pmax + 1, ctx);
  DevBuf<unsigned long long> hist;
  hist.alloc((uint64_t)pmax * pmax, ctx);
  auto footprint = [&](uint32_t p) -> uint64_t {
    std::vector<uint32_t> cuts(p + 1, 0);
    cuts[p] = n;
    if (n > 0 && p > 1) {
      k_cuts<<<1, 256, 0, st>>>(incl.p, n, 2 * m, p, dc.p);
      BBTC_LAUNCHED(ctx);
      BBTC_CUDA(cudaMemcpyAsync(cuts.data(), dc.p, (p + 1) * 4, cudaMemcpyDeviceToHost, st));
    } else {
      BBTC_CUDA(cudaMemcpyAsync(dc.p, cuts.data(), (p + 1) * 4, cudaMemcpyHostToDevice, st));
    }
    BBTC_CUDA(cudaMemsetAsync(hist.p, 0, (uint64_t)p * p * 8, st));
    if (m) {
      const bool sm = p <= 64;
      const size_t smem = (p + 1) * 4 + (sm ? (size_t)p * p * 4 : 0);
      k_part_hist<<<grid_for(ctx, m), kThreads, smem, st>>>(g->okeys.p, m, dc.p, p, sm, hist.p);
      BBTC_LAUNCHED(ctx);
    }
    std::vector<unsigned long long> h((uint64_t)p * p);
    BBTC_CUDA(cudaMemcpyAsync(h.data(), hist.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
    BBTC_CUDA(cudaStreamSynchronize(st));
    auto bytes = [&](uint32_t i, uint32_t j) {
      return 4 * arenas * (uint64_t)h[(uint64_t)i * p + j] + 4 * ((uint64_t)(cuts[i + 1] - cuts[i]) + 1);
    };
    uint64_t worst = 0;
    for (uint32_t i = 0; i < p; ++i)
      for (uint32_t j = i; j < p; ++j)
        for (uint32_t k = j; k < p; ++k) {
          // distinct blocks: ik == ij iff j == k; jk == ik iff i == j
          const uint64_t t = bytes(i, j) + (k != j ? bytes(i, k) : 0) + (i != j ? bytes(j, k) : 0);
          worst = std::max(worst, t);
        }
    return worst;
  };
  auto fits = [&](uint32_t p) { return footprint(p) <= budget / depth; };
  uint32_t hi = 1;
  while (!fits(hi)) {
    if (hi >= pmax)
      raise(BBTC_ERANGE, "device budget " + std::to_string(budget) + " B is below the largest task footprint at p = " +
                             std::to_string(pmax) + " (x depth " + std::to_string(depth) + ")");
    hi = std::min(2 * hi, pmax);
  }
  for (uint32_t p = hi / 2 + 1; p < hi; ++p)
    if (fits(p)) return p;
  return hi;
}

// =====================================================================================
// §8(e) sharded build, one rank per GPU.  The caller (dist.py) moves the
// buffers between ranks with NCCL; these are the per-rank device steps.

// Sorted unique narrow keys (lo << bw | hi) of `keys[0, cnt)`, sentinels dropped; the
// result is left in `keys` (swapped with a scratch buffer), the count returned.
static uint64_t sort_unique(bbtc_ctx* ctx, DevBuf<uint64_t>& keys, uint64_t cnt, int bw) {
  cudaStream_t st = ctx->stream;
  if (!cnt) return 0;
  DevBuf<uint64_t> alt;
  alt.alloc(cnt, ctx);
  cub::DoubleBuffer<uint64_t> db(keys.p, alt.p);
  cub_call(ctx, [&](void* t, size_t& b) { return sort_keys64(t, b, db, cnt, 0, 2 * bw, st); },
           radix_kernels(cnt, 2 * bw));
  if (db.Current() != keys.p) std::swap(keys, alt);
  DevBuf<uint64_t> nsel;
  nsel.alloc(1, ctx);
  cub_call(ctx, [&](void* t, size_t& b) { return cub::DeviceSelect::Unique(t, b, keys.p, alt.p, nsel.p, cnt, st); });
  uint64_t u = 0, last = 0;
  BBTC_CUDA(cudaMemcpyAsync(&u, nsel.p, 8, cudaMemcpyDeviceToHost, st));
  BBTC_CUDA(cudaStreamSynchronize(st));
  if (u) {
    BBTC_CUDA(cudaMemcpyAsync(&last, alt.p + u - 1, 8, cudaMemcpyDeviceToHost, st));
    BBTC_CUDA(cudaStreamSynchronize(st));
  }
  std::swap(keys, alt);
  return u - (u && last == kSentinel ? 1 : 0);
}

// Groups keys[0, m) by destination rank into out (kind 0: canonical narrow keys by
// key_owner, leaving in wire form; kind 1: oriented keys by block owner).
template <int kKind>
static void group_by_dest(bbtc_ctx* ctx, const uint64_t* keys, uint64_t m, uint32_t world, int bw,
                          const uint32_t* dcuts, uint32_t p, const uint32_t* downer, uint64_t* out,
                          uint64_t* send_counts) {
  cudaStream_t st = ctx->stream;
  DevBuf<unsigned long long> cnt;
  cnt.alloc(world, ctx);
  BBTC_CUDA(cudaMemsetAsync(cnt.p, 0, world * 8, st));
  const uint32_t nb = p * (p + 1) / 2;
  const size_t smem = 4 * ((size_t)world + (kKind == 1 ? p + 1 + nb : 0));
  if (m) {
    k_dest_count<kKind><<<grid_for(ctx, m), kThreads, smem, st>>>(keys, m, world, bw, dcuts, p, downer, cnt.p);
    BBTC_LAUNCHED(ctx);
  }
  std::vector<unsigned long long> h(world), c0(world, 0);
  BBTC_CUDA(cudaMemcpyAsync(h.data(), cnt.p, world * 8, cudaMemcpyDeviceToHost, st));
  BBTC_CUDA(cudaStreamSynchronize(st));
  for (uint32_t w = 1; w < world; ++w) c0[w] = c0[w - 1] + h[w - 1];
  for (uint32_t w = 0; w < world; ++w) send_counts[w] = h[w];
  BBTC_CUDA(cudaMemcpyAsync(cnt.p, c0.data(), world * 8, cudaMemcpyHostToDevice, st));
  if (m) {
    k_dest_scatter<kKind><<<grid_for(ctx, m), kThreads, smem, st>>>(keys, m, world, bw, dcuts, p, downer, cnt.p,
                                                                      out);
    BBTC_LAUNCHED(ctx);
  }
  BBTC_CUDA(cudaStreamSynchronize(st));   // (c0 is a host source of an async copy)
}

void shard_canon(bbtc_ctx* ctx, const uint32_t* src, const uint32_t* dst, uint64_t E, int mem, uint32_t n_hint,
                 uint32_t world, uint64_t* out, uint64_t* send_counts, uint32_t* max_id_plus1) {
  cudaStream_t st = ctx->stream;
  Trace tr(st, "shard_canon");
  DevBuf<uint32_t> ds, dd;
  if (mem == BBTC_MEM_HOST && E) {   // this rank's share of the raw edges crosses PCIe
    ds.alloc(E, ctx);
    dd.alloc(E, ctx);
    BBTC_CUDA(cudaMemcpyAsync(ds.p, src, E * 4, cudaMemcpyHostToDevice, st));
    BBTC_CUDA(cudaMemcpyAsync(dd.p, dst, E * 4, cudaMemcpyHostToDevice, st));
    src = ds.p;
    dst = dd.p;
  }
  tr.mark("h2d");
  DevBuf<uint64_t> keys;
  keys.alloc(std::max<uint64_t>(E, 1), ctx);
  DevBuf<uint32_t> dmax;
  dmax.alloc(1, ctx);
  int bw = n_hint > 1 ? std::max(1, bitlen(n_hint - 1)) : 32;
  uint32_t max_id = 0;
  for (int pass = 0; pass < 2; ++pass) {
    BBTC_CUDA(cudaMemsetAsync(dmax.p, 0, 4, st));
    if (E) {
      k_canon<<<grid_for(ctx, E), kThreads, 0, st>>>(src, dst, E, bw, keys.p, dmax.p);
      BBTC_LAUNCHED(ctx);
    }
    BBTC_CUDA(cudaMemcpyAsync(&max_id, dmax.p, 4, cudaMemcpyDeviceToHost, st));
    BBTC_CUDA(cudaStreamSynchronize(st));
    if (!E || bw == 32 || (max_id >> bw) == 0) break;
    bw = 32;   // an id does not fit the hint's width
  }
  *max_id_plus1 = E ? max_id + 1 : 0;
  tr.mark("canon");
  const uint64_t u = sort_unique(ctx, keys, E, bw);
  tr.mark("sort_unique");
  group_by_dest<0>(ctx, keys.p, u, world, bw, nullptr, 1, nullptr, out, send_counts);
  tr.mark("group");
}

void shard_graph(bbtc_ctx* ctx, const uint64_t* wire, uint64_t cnt, uint32_t n, uint32_t* d_deg, bbtc_graph* g) {
  cudaStream_t st = ctx->stream;
  Trace tr(st, "shard_graph");
  const int bw = std::max(1, bitlen(n > 1 ? n - 1 : 1));
  DevBuf<uint64_t> keys;
  keys.alloc(std::max<uint64_t>(cnt, 1), ctx);
  if (cnt) {
    BBTC_CUDA(cudaMemcpyAsync(keys.p, wire, cnt * 8, cudaMemcpyDeviceToDevice, st));
    k_narrow<<<grid_for(ctx, cnt), kThreads, 0, st>>>(keys.p, cnt, bw);
    BBTC_LAUNCHED(ctx);
  }
  const uint64_t m = sort_unique(ctx, keys, cnt, bw);   // instances from several ranks meet here
  tr.mark("sort_unique");
  g->n = n;
  g->m = m;
  g->raw = cnt;
  g->cbw = bw;
  g->ckeys = std::move(keys);
  BBTC_CUDA(cudaMemsetAsync(d_deg, 0, (size_t)n * 4, st));
  if (m) degrees_sorted(ctx, g->ckeys.p, m, bw, n, d_deg);
  tr.mark("degree");
}

void shard_rank(bbtc_ctx* ctx, bbtc_graph* g, const uint32_t* d_deg, uint64_t m_total) {
  cudaStream_t st = ctx->stream;
  Trace tr(st, "shard_rank");
  const uint32_t n = g->n;
  const uint64_t m = g->m;
  g->m_total = m_total;
  g->deg_sorted.alloc(n, ctx);
  g->rank.alloc(n, ctx);
  g->okeys.alloc(m, ctx);
  if (n) {
    DevBuf<uint32_t> ids, order, dmax;
    ids.alloc(n, ctx);
    order.alloc(n, ctx);
    dmax.alloc(2, ctx);
    k_iota<<<grid_for(ctx, n), kThreads, 0, st>>>(ids.p, n);
    BBTC_LAUNCHED(ctx);
    const int bdeg = std::max(1, bitlen(std::min<uint64_t>(m_total, n - 1)));
    cub_call(ctx, [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, d_deg, g->deg_sorted.p, ids.p, order.p, (uint64_t)n, 0, bdeg, st);
    }, radix_kernels(n, bdeg));
    k_rank<<<grid_for(ctx, n), kThreads, 0, st>>>(order.p, n, g->rank.p);
    BBTC_LAUNCHED(ctx);
    if (m) orient_sliced(ctx, g->ckeys.p, m, g->cbw, n, g->rank.p, g->okeys.p);
    k_graph_stats<<<1, 32, 0, st>>>(g->deg_sorted.p, n, dmax.p);
    BBTC_LAUNCHED(ctx);
    uint32_t h[2];
    BBTC_CUDA(cudaMemcpyAsync(h, dmax.p, 8, cudaMemcpyDeviceToHost, st));
    BBTC_CUDA(cudaStreamSynchronize(st));
    g->n_nonisolated = n - h[0];
    g->d_max = h[1];
  }
  g->ckeys.reset();
  tr.mark("rank_orient");
}

uint32_t shard_blocks_hist(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* user_cuts,
                           uint64_t* d_bnnz, uint32_t* cuts_out) {
  cudaStream_t st = ctx->stream;
  const uint32_t n = g->n;
  std::vector<uint32_t> cuts;
  uint32_t pe = p;
  if (user_cuts) {
    if (user_cuts[0] != 0 || user_cuts[p] != n) raise(BBTC_EINVAL, "cuts must satisfy cuts[0] = 0 and cuts[p] = n");
    for (uint32_t i = 0; i < p; ++i)
      if (user_cuts[i] > user_cuts[i + 1]) raise(BBTC_EINVAL, "cuts must be non-decreasing");
    cuts.assign(user_cuts, user_cuts + p + 1);
  } else {
    pe = n == 0 ? 1 : std::min(p, n);
    cuts.assign(pe + 1, 0);
    cuts[pe] = n;
    if (n > 0 && pe > 1) {   // the default rule over the GLOBAL degrees (P[n] = 2 m_total)
      DevBuf<uint64_t> incl;
      incl.alloc(n, ctx);
      cub::TransformInputIterator<uint64_t, ToU64, const uint32_t*> it(g->deg_sorted.p, ToU64{});
      cub_call(ctx, [&](void* t, size_t& b) { return cub::DeviceScan::InclusiveSum(t, b, it, incl.p, (uint64_t)n, st); });
      DevBuf<uint32_t> dc;
      dc.alloc(pe + 1, ctx);
      k_cuts<<<1, 256, 0, st>>>(incl.p, n, 2 * g->m_total, pe, dc.p);
      BBTC_LAUNCHED(ctx);
      BBTC_CUDA(cudaMemcpyAsync(cuts.data(), dc.p, (pe + 1) * 4, cudaMemcpyDeviceToHost, st));
      BBTC_CUDA(cudaStreamSynchronize(st));
    }
  }
  std::copy(cuts.begin(), cuts.end(), cuts_out);
  DevBuf<uint32_t> dc;
  dc.alloc(pe + 1, ctx);
  BBTC_CUDA(cudaMemcpyAsync(dc.p, cuts.data(), (pe + 1) * 4, cudaMemcpyHostToDevice, st));
  DevBuf<unsigned long long> hist;
  hist.alloc((uint64_t)pe * pe, ctx);
  BBTC_CUDA(cudaMemsetAsync(hist.p, 0, (uint64_t)pe * pe * 8, st));
  if (g->m) {
    const bool sm = (uint64_t)pe * pe <= 8192;
    const size_t smem = 4 * ((size_t)pe + 1 + (sm ? (size_t)pe * pe : 0));
    k_part_hist<<<grid_for(ctx, g->m), kThreads, smem, st>>>(g->okeys.p, g->m, dc.p, pe, sm, hist.p);
    BBTC_LAUNCHED(ctx);
  }
  k_fold_blocks<<<1, 256, 0, st>>>(hist.p, pe, (unsigned long long*)d_bnnz);
  BBTC_LAUNCHED(ctx);
  BBTC_CUDA(cudaStreamSynchronize(st));
  return pe;
}

void shard_by_block(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* cuts, const uint32_t* owner,
                    uint32_t world, uint64_t* out, uint64_t* send_counts) {
  cudaStream_t st = ctx->stream;
  const uint32_t nb = p * (p + 1) / 2;
  DevBuf<uint32_t> dc, dow;
  dc.alloc(p + 1, ctx);
  dow.alloc(nb, ctx);
  BBTC_CUDA(cudaMemcpyAsync(dc.p, cuts, (p + 1) * 4, cudaMemcpyHostToDevice, st));
  BBTC_CUDA(cudaMemcpyAsync(dow.p, owner, nb * 4, cudaMemcpyHostToDevice, st));
  group_by_dest<1>(ctx, g->okeys.p, g->m, world, 32, dc.p, p, dow.p, out, send_counts);
}

// The rank's plan in the global block layout: the blocks it owns built from the
// oriented edges it received (every edge of those blocks), the other blocks allocated
// at their global offsets and empty until the caller moves them in.
void plan_build_shard(bbtc_ctx* ctx, const bbtc_graph* like, const uint64_t* okeys, uint64_t cnt, uint32_t p,
                      const uint32_t* cuts, const uint64_t* bnnz, const uint32_t* task_rank, uint32_t rank,
                      uint32_t world, uint32_t flags, bbtc_plan* plan) {
  cudaStream_t st = ctx->stream;
  Trace tr(st, "plan_build_shard");
  bbtc_graph tg;
  tg.ctx = ctx;
  tg.n = like->n;
  tg.m = cnt;
  tg.m_total = like->m_total;
  tg.n_nonisolated = like->n_nonisolated;
  tg.d_max = like->d_max;
  tg.okeys.alloc(std::max<uint64_t>(cnt, 1), ctx);
  if (cnt) BBTC_CUDA(cudaMemcpyAsync(tg.okeys.p, okeys, cnt * 8, cudaMemcpyDeviceToDevice, st));
  const uint64_t n_tasks_all = n_tasks(p);
  plan->task_rank.assign(task_rank, task_rank + n_tasks_all);
  plan->shard_rank = rank;
  plan->shard_world = world;
  plan_build(ctx, &tg, p, cuts, flags & ~BBTC_PLAN_STATS, plan);
  if (plan->colmajor) plan->rows.reset();   // (not moved to the global layout nor forwarded: dense tasks walk by column)
  tr.mark("local_build");
  // Re-lay the arenas out at the global block offsets.
  const uint32_t nb = p * (p + 1) / 2;
  uint64_t mg = 0, m_max = 0, bytes = 0;
  std::vector<uint64_t> e0g(nb);
  for (uint32_t b = 0; b < nb; ++b) {
    e0g[b] = mg;
    mg += bnnz[b];
    m_max = std::max<uint64_t>(m_max, bnnz[b]);
    const BlockDesc& B = plan->blocks[b];
    if (B.nnz && B.nnz != bnnz[b])
      raise(BBTC_EINVAL, "shard plan: a block received " + std::to_string(B.nnz) + " of its " +
                             std::to_string(bnnz[b]) + " edges (every edge of an owned block must be sent to its owner)");
  }
  if (mg >= 0xFFFFFFFFull) raise(BBTC_ERANGE, "m >= 2^32-1 edges is not supported (32-bit block offsets)");
  plan->slots_ready = false;   // (the slots do not move to the global layout)
  for (auto& A : plan->edge_arenas()) {
    DevBuf<uint32_t> g;
    g.alloc(std::max<uint64_t>(mg, 1), ctx);
    // Blocks this rank neither builds nor receives stay zero (valid empty-looking data):
    // whole-plan passes such as the column offsets of bbtc_plan_to_host index by their
    // contents, which must not be uninitialised memory.
    BBTC_CUDA(cudaMemsetAsync(g.p, 0, std::max<uint64_t>(mg, 1) * 4, st));
    for (uint32_t b = 0; b < nb; ++b) {
      const BlockDesc& B = plan->blocks[b];
      if (B.nnz) BBTC_CUDA(cudaMemcpyAsync(g.p + e0g[b], A.dev->p + B.e0, B.nnz * 4, cudaMemcpyDeviceToDevice, st));
    }
    *A.dev = std::move(g);
  }
  for (uint32_t b = 0; b < nb; ++b) {
    BlockDesc& B = plan->blocks[b];
    B.e0 = e0g[b];
    B.nnz = bnnz[b];
    bytes += 4 * plan->edge_arenas().size() * B.nnz + 4 * ((uint64_t)(plan->cuts[B.i + 1] - plan->cuts[B.i]) + 1);
  }
  BBTC_CUDA(cudaMemcpyAsync(plan->d_blocks.p, plan->blocks.data(), nb * sizeof(BlockDesc), cudaMemcpyHostToDevice, st));
  plan->m = mg;
  plan->info.m = mg;
  plan->info.m_max = m_max;
  plan->info.lambda = mg ? (double)m_max / (2.0 * (double)mg / ((double)p * (p + 1))) : 1.0;
  plan->info.block_bytes = bytes;
  plan_tasks(plan, 1);   // this rank's tasks only, in the global block layout
  tr.mark("relayout");
}

// §8(f)#4: PBD-like refinement of a cut vector, minimising the largest block m_max
// (the λ of P:573-586).  Pattern search: for each interior cut, try moving it by
// ±step (clamped between its neighbours) and keep a move when m_max strictly
// decreases; halve the step when a full sweep keeps nothing.  Every candidate is
// evaluated exactly (one pass over the oriented edges: the p x p block histogram).
void cuts_refine(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* cuts_in, uint32_t max_evals,
                 uint32_t* cuts_out, uint64_t* m_max_out) {
  cudaStream_t st = ctx->stream;
  const uint32_t n = g->n;
  std::vector<uint32_t> cuts;
  uint32_t pe = p;
  if (cuts_in) {
    if (cuts_in[0] != 0 || cuts_in[p] != n) raise(BBTC_EINVAL, "cuts must satisfy cuts[0] = 0 and cuts[p] = n");
    for (uint32_t i = 0; i < p; ++i)
      if (cuts_in[i] > cuts_in[i + 1]) raise(BBTC_EINVAL, "cuts must be non-decreasing");
    cuts.assign(cuts_in, cuts_in + p + 1);
  } else {
    DevBuf<uint64_t> dn;
    dn.alloc(std::max<uint32_t>(p * (p + 1) / 2, 1), ctx);
    cuts.resize(p + 1);
    pe = shard_blocks_hist(ctx, g, p, nullptr, dn.p, cuts.data());   // the default rule
    cuts.resize(pe + 1);
  }
  DevBuf<uint32_t> dc;
  dc.alloc(pe + 1, ctx);
  DevBuf<unsigned long long> hist;
  hist.alloc((uint64_t)pe * pe, ctx);
  std::vector<unsigned long long> h((uint64_t)pe * pe);
  uint32_t evals = 0;
  auto m_max = [&](const std::vector<uint32_t>& c) {
    ++evals;
    BBTC_CUDA(cudaMemcpyAsync(dc.p, c.data(), (pe + 1) * 4, cudaMemcpyHostToDevice, st));
    BBTC_CUDA(cudaMemsetAsync(hist.p, 0, (uint64_t)pe * pe * 8, st));
    if (g->m) {
      const bool sm = (uint64_t)pe * pe <= 8192;
      const size_t smem = 4 * ((size_t)pe + 1 + (sm ? (size_t)pe * pe : 0));
      k_part_hist<<<grid_for(ctx, g->m), kThreads, smem, st>>>(g->okeys.p, g->m, dc.p, pe, sm, hist.p);
      BBTC_LAUNCHED(ctx);
    }
    BBTC_CUDA(cudaMemcpyAsync(h.data(), hist.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
    BBTC_CUDA(cudaStreamSynchronize(st));
    return (uint64_t)*std::max_element(h.begin(), h.end());
  };
  uint64_t best = m_max(cuts);
  uint32_t step = 1;
  for (uint32_t i = 0; i < pe; ++i) step = std::max(step, (cuts[i + 1] - cuts[i]) / 2);
  while (step >= 1 && evals < max_evals && pe > 1) {
    bool moved = false;
    for (uint32_t i = 1; i < pe && evals < max_evals; ++i)
      for (int dir : {-1, 1}) {
        if (evals >= max_evals) break;
        std::vector<uint32_t> c = cuts;
        const int64_t v = (int64_t)c[i] + dir * (int64_t)step;
        c[i] = (uint32_t)std::min<int64_t>(std::max<int64_t>(v, c[i - 1]), c[i + 1]);
        if (c[i] == cuts[i]) continue;
        const uint64_t mm = m_max(c);
        if (mm < best) {
          best = mm;
          cuts = c;
          moved = true;
        }
      }
    if (!moved) step /= 2;
  }
  std::fill(cuts_out, cuts_out + p + 1, 0u);
  std::copy(cuts.begin(), cuts.end(), cuts_out);
  *m_max_out = best;
}

}  // namespace bbtc

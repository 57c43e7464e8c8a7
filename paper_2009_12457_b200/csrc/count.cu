// count.cu — the hot path's intersection kernel (step a7) and plan statistics.
//
// Alg. 5 BB-TC-LIST: for task t = (i,j,k) and every edge (u,v) of
// G_ij, count |N(G_ik,u) ∩ N(G_jk,v)|, summed into the task's uint64 counter.
//
// B200 design: one persistent grid, one warp per work item
// (task t, a range of `chunk` consecutive edges of G_ij), items claimed from a
// global atomic cursor.  A warp takes 32 edges at a time, and
//   1. stages every distinct row list A_u = N(G_ik,u) of those edges into its
//      shared-memory slab (the edges are row-sorted, so rows repeat across lanes
//      and each A_u is read from HBM once per batch, not once per edge);
//   2. flattens the 32 probe lists B_v = N(G_jk,v) into one virtual array and
//      walks it 32 elements per step — consecutive lanes read consecutive words of
//      the same list (coalesced), no lane idles on short lists;
//   3. looks each probe w up in its edge's staged A_u by binary search in shared
//      memory: w ∈ A_u  <=>  w is a common neighbour, i.e. one triangle.
// This computes exactly Σ_(u,v) |A_u ∩ B_v| (what Alg. 1's merge returns), with
// every lane busy whatever the list-length skew.  Rows whose A_u exceeds the
// slab are searched in global memory instead (rare: d'_max is small after the
// degree ordering).
#include <cub/cub.cuh>

#include "internal.h"

namespace bbtc {
namespace {

constexpr int kWarps = 8;            // warps per CTA
constexpr int kSlab = 1024;          // staged A words per warp (4 KiB)
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x += y;
  }
  return x;
}

// Last lane o (0..31) with key[o] <= f, key non-decreasing over lanes, key[0] <= f.
__device__ __forceinline__ int owner_of(uint32_t key, uint32_t f) {
  int lo = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    uint32_t k = __shfl_sync(kFull, key, lo + step);
    if (k <= f) lo += step;
  }
  return lo;
}

// lower_bound search of w in the sorted list A[0..len): true if present.
__device__ __forceinline__ bool contains_bounded(const uint32_t* A, uint32_t len, uint32_t w) {
  uint32_t lo = 0, n = len;
  while (n > 0) {
    uint32_t half = n >> 1;
    if (A[lo + half] < w) { lo += half + 1; n -= half + 1; }
    else n = half;
  }
  return lo < len && A[lo] == w;
}

__global__ void __launch_bounds__(kWarps * 32)
k_count(const uint32_t* __restrict__ cols, const uint32_t* __restrict__ rows, const uint32_t* __restrict__ rowptr,
        const BlockDesc* __restrict__ blocks, const TaskDesc* __restrict__ tasks,
        const uint64_t* __restrict__ item_start, uint32_t n_exec, uint64_t item_lo, uint64_t n_items, uint32_t chunk,
        uint32_t rank,
        uint32_t world, unsigned long long* __restrict__ cursor, unsigned long long* __restrict__ counts,
        uint32_t n_tasks) {
  __shared__ uint32_t slab[kWarps][kSlab];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  uint32_t* sA = slab[wid];

  for (;;) {
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(cursor, 1ull);
    it = __shfl_sync(kFull, it, 0);
    const uint64_t g = item_lo + it * world + rank;
    if (g >= n_items) break;
    // task of item g: last t with item_start[t] <= g
    uint32_t lo = 0, hi = n_exec - 1;
    while (lo < hi) {
      uint32_t mid = (lo + hi + 1) >> 1;
      if (item_start[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const TaskDesc T = tasks[lo];
    const BlockDesc Bij = blocks[T.ij];
    const BlockDesc Bik = blocks[T.ik];
    const BlockDesc Bjk = blocks[T.jk];
    const uint64_t e_begin = Bij.e0 + (g - item_start[lo]) * chunk;
    const uint64_t e_end = min(e_begin + chunk, Bij.e0 + Bij.nnz);
    const uint32_t* rp_ik = rowptr + Bik.ro;
    const uint32_t* c_ik = cols + Bik.e0;
    const uint32_t* rp_jk = rowptr + Bjk.ro;
    const uint32_t* c_jk = cols + Bjk.e0;

    uint32_t hits = 0;
    uint64_t base = e_begin;
    while (base < e_end) {
      const uint64_t e = base + lane;
      const bool valid = e < e_end;
      const uint32_t u = valid ? rows[e] : 0xFFFFFFFFu;
      const uint32_t v = valid ? cols[e] : 0;
      uint32_t a0 = 0, alen = 0, b0 = 0, blen = 0;
      if (valid) {
        a0 = rp_ik[u];
        alen = rp_ik[u + 1] - a0;
        b0 = rp_jk[v];
        blen = rp_jk[v + 1] - b0;
      }
      const uint32_t uprev = __shfl_up_sync(kFull, u, 1);
      const bool leader = valid && (lane == 0 || u != uprev);
      const uint32_t lead_len = leader ? alen : 0;
      const uint32_t incl = warp_incl_scan(lead_len, lane);
      const uint32_t lmask = __ballot_sync(kFull, leader);
      const uint32_t le_mask = lmask & (0xffffffffu >> (31 - lane));
      const int my_leader = le_mask ? 31 - __clz(le_mask) : 0;
      const uint32_t aoff = __shfl_sync(kFull, incl - lead_len, my_leader);
      const uint32_t aend = aoff + alen;
      const uint32_t fit = __ballot_sync(kFull, valid && aend <= kSlab);
      int L = __popc(fit);   // lanes [0, L) fit: aend is non-decreasing in the lane
      bool global_mode = false;
      if (L == 0) {
        // The first row alone exceeds the slab: handle its edges with A in global memory.
        const uint32_t u0 = __shfl_sync(kFull, u, 0);
        L = __popc(__ballot_sync(kFull, valid && u == u0));
        global_mode = true;
      }
      const bool in = lane < L;
      if (!global_mode) {
        // 1. stage the distinct A_u of lanes [0, L) into the slab
        const uint32_t total_a = __shfl_sync(kFull, aend, L - 1);
        const uint32_t akey = in ? aoff : 0xFFFFFFFFu;
        for (uint32_t f0 = 0; f0 < total_a; f0 += 32) {
          const uint32_t f = f0 + lane;
          const int o = owner_of(akey, f);
          const uint32_t src0 = __shfl_sync(kFull, a0, o);
          const uint32_t off_o = __shfl_sync(kFull, aoff, o);
          if (f < total_a) sA[f] = c_ik[src0 + (f - off_o)];
        }
        __syncwarp();
      }
      // 2./3. flattened probes over B_v of lanes [0, L)
      const uint32_t bl = in ? blen : 0;
      const uint32_t binc = warp_incl_scan(bl, lane);
      const uint32_t bexc = in ? binc - bl : 0xFFFFFFFFu;
      const uint32_t total_b = __shfl_sync(kFull, binc, 31);
      for (uint32_t f0 = 0; f0 < total_b; f0 += 32) {
        const uint32_t f = f0 + lane;
        const int o = owner_of(bexc, f);
        const uint32_t bstart = __shfl_sync(kFull, b0, o);
        const uint32_t boff = __shfl_sync(kFull, bexc, o);
        const uint32_t as = __shfl_sync(kFull, global_mode ? a0 : aoff, o);
        const uint32_t al = __shfl_sync(kFull, alen, o);
        if (f < total_b) {
          const uint32_t w = c_jk[bstart + (f - boff)];
          const uint32_t* A = global_mode ? c_ik + as : sA + as;
          hits += contains_bounded(A, al, w);
        }
      }
      __syncwarp();
      base += L;
    }
    // one atomic per warp-item
    uint32_t s = __reduce_add_sync(kFull, hits);
    if (lane == 0 && s) {
      atomicAdd(&counts[T.idx], (unsigned long long)s);
      atomicAdd(&counts[n_tasks], (unsigned long long)s);
    }
  }
}

// ---- plan statistics (BBTC_PLAN_STATS): B_alg, visits, d'_max -------------------
// Per task t and edge (u,v) of G_ij: a = d(G_ik,u), b = d(G_jk,v).
// B_alg(t) = 4(|V_i|+1) + 8 R_ij + Σ (4 + 8 + 4a + 4b)
__global__ void k_stats_edges(const uint32_t* __restrict__ cols, const uint32_t* __restrict__ rows,
                              const uint32_t* __restrict__ rowptr, const BlockDesc* __restrict__ blocks,
                              const TaskDesc* __restrict__ tasks, uint32_t n_exec,
                              unsigned long long* __restrict__ ab_sum) {
  for (uint32_t t = blockIdx.y; t < n_exec; t += gridDim.y) {
    const TaskDesc T = tasks[t];
    const BlockDesc Bij = blocks[T.ij], Bik = blocks[T.ik], Bjk = blocks[T.jk];
    unsigned long long acc = 0;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < Bij.nnz;
         x += (uint64_t)gridDim.x * blockDim.x) {
      const uint32_t u = rows[Bij.e0 + x], v = cols[Bij.e0 + x];
      acc += (rowptr[Bik.ro + u + 1] - rowptr[Bik.ro + u]) + (rowptr[Bjk.ro + v + 1] - rowptr[Bjk.ro + v]);
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&ab_sum[t], acc);
  }
}

// Per block: nonempty rows R_ij and the largest partial degree.
__global__ void k_stats_rows(const uint32_t* __restrict__ rowptr, const BlockDesc* __restrict__ blocks,
                             const uint32_t* __restrict__ rows_per_block, unsigned long long* __restrict__ nonempty,
                             uint32_t* __restrict__ dmax) {
  const BlockDesc B = blocks[blockIdx.y];
  const uint32_t nr = rows_per_block[blockIdx.y];
  uint32_t ne = 0, mx = 0;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
    uint32_t d = rowptr[B.ro + r + 1] - rowptr[B.ro + r];
    ne += d > 0;
    mx = max(mx, d);
  }
  ne = __reduce_add_sync(kFull, ne);
  mx = __reduce_max_sync(kFull, mx);
  if ((threadIdx.x & 31) == 0) {
    if (ne) atomicAdd(&nonempty[blockIdx.y], (unsigned long long)ne);
    atomicMax(dmax, mx);
  }
}

}  // namespace

void count_zero(bbtc_ctx* ctx, const bbtc_plan* plan, uint64_t* d_counts) {
  BBTC_CUDA(cudaMemsetAsync(d_counts, 0, (plan->info.n_tasks + 1) * 8, ctx->stream));
}

// Enqueues the count kernel over work items [item_lo, item_hi) of the plan's
// execution order (this rank's residues only), accumulating into d_counts.
void count_launch(bbtc_ctx* ctx, const bbtc_plan* plan, uint32_t rank, uint32_t world, uint64_t* d_counts,
                  uint64_t item_lo, uint64_t item_hi) {
  cudaStream_t st = ctx->stream;
  const uint64_t nt = plan->info.n_tasks;
  if (item_hi <= item_lo + rank) return;
  const uint64_t my_items = (item_hi - item_lo - rank + world - 1) / world;
  if (!ctx->cursor) BBTC_CUDA(cudaMalloc((void**)&ctx->cursor, 8 * kCursorSlots));
  unsigned long long* cursor = (unsigned long long*)ctx->cursor + (ctx->cursor_next++ % kCursorSlots);
  BBTC_CUDA(cudaMemsetAsync(cursor, 0, 8, st));
  static int per_sm = 0;
  if (!per_sm) BBTC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_count, kWarps * 32, 0));
  const uint64_t grid = std::min<uint64_t>((uint64_t)ctx->sm_count * std::max(per_sm, 1),
                                           (my_items + kWarps - 1) / kWarps);
  k_count<<<(unsigned)grid, kWarps * 32, 0, st>>>(
      plan->cols.p, plan->rows.p, plan->rowptr.p, plan->d_blocks.p, plan->d_tasks.p, plan->d_item_start.p,
      (uint32_t)plan->tasks.size(), item_lo, item_hi, plan->chunk, rank, world, cursor,
      (unsigned long long*)d_counts, (uint32_t)nt);
  BBTC_LAUNCHED(ctx);
}

void plan_stats(bbtc_ctx* ctx, bbtc_plan* plan) {
  cudaStream_t st = ctx->stream;
  const uint32_t ne = (uint32_t)plan->tasks.size();
  const uint32_t nb = (uint32_t)plan->blocks.size();
  DevBuf<unsigned long long> ab, nonempty;
  DevBuf<uint32_t> dmax, rpb;
  ab.alloc(ne, st);
  nonempty.alloc(nb, st);
  dmax.alloc(1, st);
  rpb.alloc(nb, st);
  std::vector<uint32_t> h_rpb(nb);
  uint32_t maxrows = 1;
  for (uint32_t b = 0; b < nb; ++b) {
    const BlockDesc& B = plan->blocks[b];
    h_rpb[b] = plan->cuts[B.i + 1] - plan->cuts[B.i];
    maxrows = std::max(maxrows, h_rpb[b]);
  }
  BBTC_CUDA(cudaMemcpyAsync(rpb.p, h_rpb.data(), nb * 4, cudaMemcpyHostToDevice, st));
  BBTC_CUDA(cudaMemsetAsync(ab.p, 0, ne * 8, st));
  BBTC_CUDA(cudaMemsetAsync(nonempty.p, 0, nb * 8, st));
  BBTC_CUDA(cudaMemsetAsync(dmax.p, 0, 4, st));
  if (ne) {
    k_stats_edges<<<dim3(64, std::min(ne, 4096u)), 256, 0, st>>>(plan->cols.p, plan->rows.p, plan->rowptr.p,
                                                               plan->d_blocks.p, plan->d_tasks.p, ne, ab.p);
    BBTC_LAUNCHED(ctx);
  }
  if (nb) {
    k_stats_rows<<<dim3(std::min((maxrows + 255) / 256, 64u), nb), 256, 0, st>>>(plan->rowptr.p, plan->d_blocks.p,
                                                                                 rpb.p, nonempty.p, dmax.p);
    BBTC_LAUNCHED(ctx);
  }
  std::vector<unsigned long long> h_ab(ne), h_ne(nb);
  uint32_t h_dmax = 0;
  BBTC_CUDA(cudaMemcpyAsync(h_ab.data(), ab.p, ne * 8, cudaMemcpyDeviceToHost, st));
  BBTC_CUDA(cudaMemcpyAsync(h_ne.data(), nonempty.p, nb * 8, cudaMemcpyDeviceToHost, st));
  BBTC_CUDA(cudaMemcpyAsync(&h_dmax, dmax.p, 4, cudaMemcpyDeviceToHost, st));
  BBTC_CUDA(cudaStreamSynchronize(st));
  uint64_t balg = 0, visits = 0;
  for (uint32_t t = 0; t < ne; ++t) {
    const TaskDesc& T = plan->tasks[t];
    const BlockDesc& Bij = plan->blocks[T.ij];
    balg += 4ull * ((uint64_t)h_rpb[T.ij] + 1) + 8ull * h_ne[T.ij] + 12ull * Bij.nnz + 4ull * h_ab[t];
    visits += Bij.nnz;
  }
  plan->info.b_alg = balg;
  plan->info.visits = visits;
  plan->info.dmax_blk = h_dmax;
}

}  // namespace bbtc

// capi.cpp — the extern "C" surface of libbbtc (include/bbtc.h) and its host runtime:
// error mapping, contexts, task enumeration (Alg. 4), work items, the block
// streamer (a6) and the synchronous count driver (Alg. 9's role).
#include <algorithm>
#include <array>
#include <chrono>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <thread>
#include <atomic>

#include "internal.h"

namespace bbtc {

static thread_local std::string t_err;
void set_error(const std::string& msg) { t_err = msg; }
[[noreturn]] void raise(bbtc_status code, const std::string& msg) { throw Error{code, msg}; }

static bool trace_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("BBTC_TRACE");
    on = e && *e && *e != '0';
  }
  return on == 1;
}

bool sync_check() {
  static const bool on = getenv("BBTC_SYNC_CHECK") != nullptr;
  return on;
}

Trace::Trace(cudaStream_t s, const char* name) : st(s), phase(name), on(trace_enabled()) { mark("begin"); }

void Trace::mark(const char* what) {
  if (!on) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, st);
  ev.emplace_back(what, e);
}

Trace::~Trace() {
  if (!on) return;
  mark("end");
  cudaEventSynchronize(ev.back().second);
  std::string line = std::string("[bbtc trace] ") + phase + ":";
  float total = 0;
  for (size_t x = 1; x < ev.size(); ++x) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[x - 1].second, ev[x].second);
    total += ms;
    char buf[96];
    snprintf(buf, sizeof buf, " %s=%.3f", ev[x].first, ms);
    line += buf;
  }
  char buf[64];
  snprintf(buf, sizeof buf, " | total=%.3f ms\n", total);
  line += buf;
  fputs(line.c_str(), stderr);
  for (auto& p : ev) cudaEventDestroy(p.second);
}

template <class F>
static bbtc_status guard(F f) {
  try {
    f();
    return BBTC_OK;
  } catch (const Error& e) {
    t_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    t_err = "host allocation failed";
    return BBTC_ENOMEM;
  } catch (const std::exception& e) {
    t_err = e.what();
    return BBTC_EINVAL;
  }
}

// ---- caching allocator ------------------------------------------------------------
// Size classes: 512 B granules below 4 KiB, else 8 classes per power of two (<= 12.5%
// waste).  A freed block is reusable by any later allocation on the context stream
// (stream order makes the reuse safe); beyond cache_limit blocks go back to the pool.
static size_t size_class(size_t b) {
  if (b <= 4096) return (b + 511) & ~size_t(511);
  int lg = 63 - __builtin_clzll(b);
  size_t step = size_t(1) << (lg - 3);
  return (b + step - 1) & ~(step - 1);
}

void* ctx_alloc(bbtc_ctx* ctx, size_t bytes) {
  const size_t sz = size_class(bytes);
  auto it = ctx->cache.find(sz);
  if (it != ctx->cache.end()) {
    void* p = it->second;
    ctx->cache.erase(it);
    ctx->cached_bytes -= sz;
    return p;
  }
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, sz, ctx->stream);
  if (e == cudaErrorMemoryAllocation && !ctx->cache.empty()) {
    cudaGetLastError();
    for (auto& kv : ctx->cache) cudaFreeAsync(kv.second, ctx->stream);
    ctx->cache.clear();
    ctx->cached_bytes = 0;
    cudaStreamSynchronize(ctx->stream);
    e = cudaMallocAsync(&p, sz, ctx->stream);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    raise(e == cudaErrorMemoryAllocation ? BBTC_ENOMEM : BBTC_ECUDA,
          std::string("device allocation of ") + std::to_string(sz) + " bytes: " + cudaGetErrorString(e));
  }
  return p;
}

void ctx_free(bbtc_ctx* ctx, void* p, size_t bytes) {
  const size_t sz = size_class(bytes);
  if (ctx->cached_bytes + sz > ctx->cache_limit) {
    cudaFreeAsync(p, ctx->stream);
    return;
  }
  ctx->cache.emplace(sz, p);
  ctx->cached_bytes += sz;
}

// Estimated cost of one edge (u,v) of G_ij in task (i,j,k), in list words (sizes work
// items; the multi-GPU scheduler's LPT weight).  "probe" (default, round 2): the probe
// list d(G_ik,u) is walked per edge while the staged list N(G_jk,v) is hashed once per
// column run, i.e. per edge in proportion to the non-empty columns of G_ij:
// 4 + δ(G_ik) + min(1, |V_j| / nnz_ij)·δ(G_jk) — the estimator that ranks measured task
// work best (ρ 0.87-0.93 on rmat24 / orkut / friendster, §10).  "paper+" (BBTC_ITEM_COST=
// merge, round 1): 8 + δ(G_ik) + δ(G_jk), the merge cost of Alg. 1.
static inline double edge_cost(double d_ik, double d_jk, double nnz_ij, double vj) {
  static const bool merge = [] {
    const char* e = getenv("BBTC_ITEM_COST");
    return e && std::string(e) == "merge";
  }();
  if (merge) return 8.0 + d_ik + d_jk;
  const double run = nnz_ij > 0 ? std::min(1.0, vj / nnz_ij) : 1.0;
  return 4.0 + d_ik + run * d_jk;
}

static inline uint64_t C2(uint64_t n) { return n < 2 ? 0 : n * (n - 1) / 2; }
static inline uint64_t C3(uint64_t n) { return n < 3 ? 0 : n * (n - 1) * (n - 2) / 6; }

uint64_t n_tasks(uint32_t p) { return (uint64_t)p * (p + 1) * (p + 2) / 6; }

// Closed form of the Alg. 4 position (tasks with first index < i, then second index
// < j within i, then k - j): [C(p+2,3) - C(p-i+2,3)] + [C(p-i+1,2) - C(p-j+1,2)] + (k-j).
uint64_t task_index(uint32_t p, uint32_t i, uint32_t j, uint32_t k) {
  return (C3((uint64_t)p + 2) - C3((uint64_t)p - i + 2)) + (C2((uint64_t)p - i + 1) - C2((uint64_t)p - j + 1)) +
         (k - j);
}

// Tasks in execution order + work items.  Execution order groups tasks sharing the
// randomly gathered probe block G_ik (for i: for k >= i: for i <= j <= k), so
// consecutive work items keep it L2-resident.  Each task's G_ij edges are cut into items
// of `chunk` edges (the unit a warp claims).
void plan_tasks(bbtc_plan* plan, uint32_t /*world*/) {
  const uint32_t p = plan->p;
  plan->tasks.clear();
  plan->tasks.reserve(n_tasks(p));
  // Work items: each task's G_ij edges are cut into chunks of roughly equal
  // estimated work, so no warp is left with one heavy item at the end of the launch.
  // Per-edge cost estimate (the paper's ExecTime density terms):
  // c(t) = 8 + delta(G_ik) + delta(G_jk), delta(G_ab) = nnz(G_ab) / |V_a|.
  auto delta = [&](uint32_t b) {
    const BlockDesc& B = plan->blocks[b];
    const uint32_t rows = plan->cuts[B.i + 1] - plan->cuts[B.i];
    return rows ? (double)B.nnz / rows : 0.0;
  };
  // §8(e) shard plans keep only their rank's tasks (and size work items for them).
  auto mine = [&](uint32_t i, uint32_t j, uint32_t k) {
    return plan->task_rank.empty() || plan->task_rank[task_index(p, i, j, k)] == plan->shard_rank;
  };
  double work_total = 0;
  for (uint32_t k = 0; k < p; ++k)
    for (uint32_t j = 0; j <= k; ++j)
      for (uint32_t i = 0; i <= j; ++i)
        if (mine(i, j, k))
          work_total += (double)plan->blocks[block_id(i, j)].nnz *
                        edge_cost(delta(block_id(i, k)), delta(block_id(j, k)), (double)plan->blocks[block_id(i, j)].nnz,
                                  (double)(plan->cuts[j + 1] - plan->cuts[j]));
  // ~384 items per warp slot of a full B200 (148 SMs x 40 warps); BBTC_ITEMS_PER_SLOT
  // overrides.  The estimate is uniform over a task's edges while the real cost is not
  // (hub columns: long runs x long probe lists), so fine items balance the tail:
  // rmat24 count 83.0 / 69.5 / 64.5 / 61.8 / 61.0 / 62.0 ms at 24 / 96 / 192 / 384 /
  // 768 / 1536 per slot; orkut 15.7 / 14.1 / 14.1 / 14.5 / 14.8 / 15.2; friendster flat
  // (profiles/r01c/ab_items_per_slot*.jsonl).
  static const double per_slot = [] {
    const char* e = getenv("BBTC_ITEMS_PER_SLOT");
    return e ? std::max(1.0, atof(e)) : 384.0;
  }();
  const double item_work = std::max(1.0, work_total / (148.0 * 40 * per_slot));
  plan->chunk = 0;
  plan->item_start.assign(1, 0);
  uint64_t max_task_bytes = 0;
  const uint64_t arenas = plan->colmajor ? 3 : 2;   // per-edge u32 arrays of a block on the device
  auto bbytes = [&](uint32_t b) {
    const BlockDesc& B = plan->blocks[b];
    return 4 * arenas * B.nnz + 4 * ((uint64_t)(plan->cuts[B.i + 1] - plan->cuts[B.i]) + 1);
  };
  // Execution order: "ikj" (default, below), "kji" (round 1), "ijk" (Alg. 4's own
  // order) or "kdesc"; BBTC_TASK_ORDER overrides.
  std::vector<std::array<uint32_t, 3>> order;
  order.reserve(n_tasks(p));
  const char* oe = getenv("BBTC_TASK_ORDER");
  const uint32_t h = plan->task_group;
  if (h > 0 && h < p) {
    // Out-of-core order: parts in groups of h; group triples (gi <= gj <= gk) one
    // after the other, so a window holds the blocks between at most three groups
    // (<= 3h^2 blocks) and consecutive windows share two of the three groups.
    const uint32_t G = (p + h - 1) / h;
    for (uint32_t gk = 0; gk < G; ++gk)
      for (uint32_t gj = 0; gj <= gk; ++gj)
        for (uint32_t gi = 0; gi <= gj; ++gi)
          for (uint32_t k = gk * h; k < std::min(p, (gk + 1) * h); ++k)
            for (uint32_t j = gj * h; j < std::min(k + 1, (gj + 1) * h); ++j)
              for (uint32_t i = gi * h; i < std::min(j + 1, (gi + 1) * h); ++i) order.push_back({i, j, k});
  } else if (oe && std::string(oe) == "ijk") {
    for (uint32_t i = 0; i < p; ++i)
      for (uint32_t j = i; j < p; ++j)
        for (uint32_t k = j; k < p; ++k) order.push_back({i, j, k});
  } else if (oe && std::string(oe) == "kji") {   // round 1's order: G_jk fixed, i inner
    for (uint32_t k = 0; k < p; ++k)
      for (uint32_t j = 0; j <= k; ++j)
        for (uint32_t i = 0; i <= j; ++i) order.push_back({i, j, k});
  } else if (oe && std::string(oe) == "kdesc") {
    for (uint32_t k = p; k-- > 0;)
      for (uint32_t j = 0; j <= k; ++j)
        for (uint32_t i = 0; i <= j; ++i) order.push_back({i, j, k});
  } else {
    // Default "ikj": the probe block G_ik — the one gathered at random — stays fixed
    // while j runs, so its rows stay in L2 across consecutive tasks (the staged G_jk and
    // the walked G_ij are read in order).  Measured against round 1's kji
    // (profiles/r02/ab6): friendster p=16 462 -> 406 ms, p=8 366 -> 362, p=4 and rmat24
    // / orkut equal or 0.5% faster.
    for (uint32_t i = 0; i < p; ++i)
      for (uint32_t k = i; k < p; ++k)
        for (uint32_t j = i; j <= k; ++j) order.push_back({i, j, k});
  }
  // isDense: a task whose third part V_k is small enough for bit rows of
  // at most kDenseMaxS words, and whose probe rows are long enough on average
  // (delta(G_ik) >= BBTC_DENSE_RATIO x stride / 32) that reading a whole bit row
  // beats walking the list.  Dense tasks go last (items [dense_item_lo, end)).
  plan->dense_s.assign(p, 0);
  plan->dense_ready = false;
  plan->s_ready = false;
  plan->dense.reset();
  static const double dense_ratio = [] {
    const char* e = getenv("BBTC_DENSE_RATIO");
    // measured with 384 items per slot (profiles/r01c/ab_dense_ratio.jsonl): rmat24 count
    // 61.7 / 60.9 / 58.8 / 58.7 / 59.9 / 65.2 ms at ratio 1 / 2 / 4 / 8 / 16 / 32
    return e ? atof(e) : 4.0;
  }();
  if (plan->dense_bits && h == 0)
    for (uint32_t k = 0; k < p; ++k) {
      const uint32_t vk = plan->cuts[k + 1] - plan->cuts[k];
      if (vk == 0 || vk > plan->dense_bits) continue;
      uint32_t s = kDenseMinS;
      while (s * 32 < vk) s <<= 1;
      if (s <= kDenseMaxS) plan->dense_s[k] = s;
    }
  auto is_dense = [&](uint32_t i, uint32_t j, uint32_t k) {
    const uint32_t s = plan->dense_s[k];
    return s && plan->blocks[block_id(i, j)].nnz && delta(block_id(i, k)) >= dense_ratio * s / 32.0;
  };
  {
    std::vector<std::array<uint32_t, 3>> sparse, dense;
    for (const auto& t : order)
      if (mine(t[0], t[1], t[2])) (is_dense(t[0], t[1], t[2]) ? dense : sparse).push_back(t);
    plan->dense_task_lo = (uint32_t)sparse.size();
    order = sparse;
    order.insert(order.end(), dense.begin(), dense.end());
  }
  plan->dense_item_lo = 0;
  for (const auto& ijk : order) {
    const uint32_t i = ijk[0], j = ijk[1], k = ijk[2];
    {
        TaskDesc T;
        T.ij = block_id(i, j);
        T.ik = block_id(i, k);
        T.jk = block_id(j, k);
        T.idx = (uint32_t)task_index(p, i, j, k);
        T.icol = 0;
        if (plan->tasks.size() == plan->dense_task_lo) plan->dense_item_lo = plan->item_start.back();
        T.pad = plan->tasks.size() >= plan->dense_task_lo ? plan->dense_s[k] : 0;
        {
          const uint32_t vk = plan->cuts[k + 1] - plan->cuts[k];
          uint32_t w = 4;
          while (w * 32 < vk) w <<= 1;
          T.bmw = (vk > 0 && w <= kBitmapMaxWords) ? w : 0;
        }
        // A list edge costs its lists; a dense edge a fixed number of bit-row words.
        // Dense tasks take the smaller of both chunks: without resident blocks (streamed,
        // out of core) the list kernel runs them too.
        double per_edge = edge_cost(delta(T.ik), delta(T.jk), (double)plan->blocks[T.ij].nnz,
                                    (double)(plan->cuts[j + 1] - plan->cuts[j]));
        if (plan->tasks.size() >= plan->dense_task_lo) per_edge = std::max(per_edge, 2.0 + plan->dense_s[k] / 8.0);
        uint64_t chunk = (uint64_t)(item_work / per_edge);
        static const double dense_chunk_x = getenv("BBTC_DENSE_CHUNK_X") ? atof(getenv("BBTC_DENSE_CHUNK_X")) : 1.0;
        if (plan->tasks.size() >= plan->dense_task_lo) chunk = (uint64_t)(chunk * dense_chunk_x);   // (A/B knob)
        chunk = std::max<uint64_t>(64, std::min<uint64_t>(1u << 16, (chunk + 31) / 32 * 32));
        T.chunk = (uint32_t)chunk;
        plan->tasks.push_back(T);
        const uint64_t nnz = plan->blocks[T.ij].nnz;
        plan->item_start.push_back(plan->item_start.back() + (nnz + chunk - 1) / chunk);
        uint64_t tb = bbytes(T.ij) + (T.ik != T.ij ? bbytes(T.ik) : 0) +
                      (T.jk != T.ij && T.jk != T.ik ? bbytes(T.jk) : 0);
        max_task_bytes = std::max(max_task_bytes, tb);
    }
  }
  if (plan->dense_task_lo >= plan->tasks.size()) plan->dense_item_lo = plan->item_start.back();
  {   // item_col bases in canonical task order: independent of the execution order, so
      // streaming / out-of-core re-orderings keep using one item_col array
    std::vector<uint64_t> base(n_tasks(p) + 1, 0);
    for (size_t t = 0; t < plan->tasks.size(); ++t)
      base[plan->tasks[t].idx + 1] = plan->item_start[t + 1] - plan->item_start[t];
    for (size_t x = 0; x + 1 < base.size(); ++x) base[x + 1] += base[x];
    for (auto& T : plan->tasks) T.icol = (uint32_t)base[T.idx];
  }
  {   // compulsory bytes of both kernels (roofline denominators)
    std::vector<char> seen(plan->blocks.size(), 0), seen_d(plan->blocks.size(), 0);
    uint64_t lb = 0, db = 0;
    for (size_t t = 0; t < plan->tasks.size(); ++t) {
      const TaskDesc& T = plan->tasks[t];
      if (t < plan->dense_task_lo) {
        for (uint32_t b : {T.ij, T.ik, T.jk})
          if (!seen[b]) {
            seen[b] = 1;
            lb += bbytes(b);
          }
      } else if (!seen_d[T.ij]) {
        seen_d[T.ij] = 1;
        db += 8 * plan->blocks[T.ij].nnz;
      }
    }
    plan->info.list_read_bytes = lb;
    plan->info.dense_edge_bytes = db;
  }
  plan->info.work_items = plan->item_start.back();
  plan->info.max_task_bytes = max_task_bytes;
  plan->info.dense_tasks = (uint32_t)(plan->tasks.size() - plan->dense_task_lo);
  bbtc_ctx* ctx = plan->ctx;
  plan->d_tasks.alloc(plan->tasks.size(), ctx);
  plan->d_item_start.alloc(plan->item_start.size(), ctx);
  BBTC_CUDA(cudaMemcpyAsync(plan->d_tasks.p, plan->tasks.data(), plan->tasks.size() * sizeof(TaskDesc),
                            cudaMemcpyHostToDevice, ctx->stream));
  BBTC_CUDA(cudaMemcpyAsync(plan->d_item_start.p, plan->item_start.data(), plan->item_start.size() * 8,
                            cudaMemcpyHostToDevice, ctx->stream));
  // The host vectors are read by the async copies above: make them complete
  // before the caller can mutate the plan.
  BBTC_CUDA(cudaStreamSynchronize(ctx->stream));
}

// ---- §8(e) scheduler: tasks -> ranks, blocks -> owners --------------------------------
// Deterministic on every rank (same inputs: cuts and the all-reduced block sizes).
// Tasks in decreasing estimated work (the ExecTime-style per-edge cost of plan_tasks,
// P:658-667; ties by canonical index) go to a rank by LPT with block affinity: among
// the ranks whose load would stay within 2% above the ideal share (or the least-loaded
// rank's load plus the task), the one already holding most of the task's block bytes,
// so tasks sharing blocks gather on few ranks and fewer blocks cross NVLink.  A block's
// owner (the rank that builds it and forwards it) is the needer holding the fewest
// owned bytes so far, visiting blocks largest first; unneeded blocks round-robin.
void shard_assign(uint32_t p, const uint32_t* cuts, const uint64_t* bnnz, uint32_t world, uint32_t* task_rank,
                  uint32_t* block_rank) {
  const uint32_t nb = p * (p + 1) / 2;
  const uint64_t nt = n_tasks(p);
  auto rows = [&](uint32_t i) { return (uint64_t)(cuts[i + 1] - cuts[i]); };
  auto delta = [&](uint32_t i, uint32_t j) {
    const uint64_t r = rows(i);
    return r ? (double)bnnz[block_id(i, j)] / (double)r : 0.0;
  };
  auto bbytes = [&](uint32_t b, uint32_t i) { return 12.0 * (double)bnnz[b] + 4.0 * (double)(rows(i) + 1); };
  // LPT weight = the task's measured-cost model, fitted to per-task device times
  // (bbtc_task_times at the bench configs, profiles/r02/r02cc; scripts/balance_study.py):
  //   list tasks  nnz(G_ij)·(16 + δ(G_ik)) + 2·min(nnz(G_ij), |V_j|)·δ(G_jk)
  //   bit rows    0.145·nnz(G_ij)·(S + 35), S = the bit-row stride in words (plan_tasks'
  //               isDense with the default dense bits and ratio)
  // log-spread of time / estimate over rmat24 p=10's list tasks 0.50 -> 0.23, orkut p=8's
  // 0.18 -> 0.15; the work-item estimate (edge_cost) overrated the bit-row tasks ~7x and
  // the per-edge overhead of short probe lists ~2.7x, which left ranks 2x apart at N = 4-8.
  static const uint32_t dense_bits = [] {
    const char* e = getenv("BBTC_DENSE_BITS");
    return std::min(e ? (uint32_t)atoi(e) : kDenseBitsDefault, kDenseMaxS * 32);
  }();
  static const double dense_ratio = getenv("BBTC_DENSE_RATIO") ? atof(getenv("BBTC_DENSE_RATIO")) : 4.0;
  auto dense_stride = [&](uint32_t k) -> uint32_t {
    const uint64_t vk = rows(k);
    if (!vk || vk > dense_bits) return 0;
    uint32_t s = kDenseMinS;
    while ((uint64_t)s * 32 < vk) s <<= 1;
    return s <= kDenseMaxS ? s : 0;
  };
  struct T { double w; uint64_t idx; uint32_t i, j, k; };
  std::vector<T> ts;
  ts.reserve(nt);
  double total = 0;
  for (uint32_t i = 0; i < p; ++i)
    for (uint32_t j = i; j < p; ++j)
      for (uint32_t k = j; k < p; ++k) {
        const uint32_t S = dense_stride(k);
        const bool dense = S && bnnz[block_id(i, j)] && delta(i, k) >= dense_ratio * S / 32.0;
        const double nij = (double)bnnz[block_id(i, j)];
        const double w = dense ? 0.145 * nij * (S + 35.0)
                               : nij * (16.0 + delta(i, k)) + 2.0 * std::min(nij, (double)rows(j)) * delta(j, k);
        ts.push_back({w, task_index(p, i, j, k), i, j, k});
        total += w;
      }
  std::stable_sort(ts.begin(), ts.end(), [](const T& a, const T& b) { return a.w > b.w || (a.w == b.w && a.idx < b.idx); });
  std::vector<double> load(world, 0.0);
  std::vector<std::vector<char>> has(world, std::vector<char>(nb, 0));
  static const double slack = getenv("BBTC_LPT_SLACK") ? atof(getenv("BBTC_LPT_SLACK")) : 1.02;
  const double share = total / world * slack;
  for (const T& t : ts) {
    const uint32_t bl[3] = {block_id(t.i, t.j), block_id(t.i, t.k), block_id(t.j, t.k)};
    const uint32_t bi[3] = {t.i, t.i, t.j};
    const double lmin = *std::min_element(load.begin(), load.end());
    const double cap = std::max(share, lmin + t.w);
    int best = -1;
    double best_aff = -1;
    for (uint32_t r = 0; r < world; ++r) {
      if (load[r] + t.w > cap + 1e-9) continue;
      double aff = 0;
      for (int x = 0; x < 3; ++x)
        if (has[r][bl[x]] && (x == 0 || bl[x] != bl[0]) && (x < 2 || bl[x] != bl[1])) aff += bbytes(bl[x], bi[x]);
      if (aff > best_aff || (aff == best_aff && load[r] < load[best])) {
        best = (int)r;
        best_aff = aff;
      }
    }
    task_rank[t.idx] = (uint32_t)best;
    load[best] += t.w;
    for (int x = 0; x < 3; ++x) has[best][bl[x]] = 1;
  }
  // owners
  std::vector<uint32_t> border(nb);
  for (uint32_t b = 0; b < nb; ++b) border[b] = b;
  std::stable_sort(border.begin(), border.end(), [&](uint32_t a, uint32_t b) { return bnnz[a] > bnnz[b]; });
  std::vector<double> owned(world, 0.0);
  uint32_t rr = 0;
  for (uint32_t b : border) {
    int best = -1;
    for (uint32_t r = 0; r < world; ++r)
      if (has[r][b] && (best < 0 || owned[r] < owned[best])) best = (int)r;
    if (best < 0) best = (int)(rr++ % world);
    block_rank[b] = (uint32_t)best;
    owned[best] += (double)bnnz[b];
  }
}

// ---- a6: the block streamer -------------------------------------------------------
// A host-resident plan keeps its three arenas in pinned memory.  Streaming copies
// every block the first time a task in execution order needs it (on the copy
// streams, round-robin), and launches the count kernel over each maximal run of
// tasks whose blocks have all been issued, after waiting on their copy events —
// so block copies of later tasks overlap the kernels of earlier ones (Alg. 7's
// prefetch of the next task's blocks).
struct Streamer {
  bbtc_ctx* ctx;
  bbtc_plan* plan;
  std::vector<char> issued;
  std::vector<cudaEvent_t> ev;      // per block: copy finished
  uint64_t bytes = 0;
  uint32_t rr = 0;
  uint32_t epoch = 0;   // nonzero: flag each block ready on the device after its copy

  Streamer(bbtc_ctx* c, bbtc_plan* p) : ctx(c), plan(p), issued(p->blocks.size(), 0), ev(p->blocks.size(), nullptr) {}
  ~Streamer() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
  }
  // Column offsets a streamed copy of block b carries (0 unless ccv travels as colptr).
  uint64_t clen(uint32_t b) const {
    const BlockDesc& B = plan->blocks[b];
    return plan->block_colptr(b) && B.nnz ? (uint64_t)B.nc + 1 : 0;
  }
  // Device bytes of block b's streamed form (per-edge arenas + row and column offsets).
  uint64_t block_bytes(uint32_t b) const {
    const BlockDesc& B = plan->blocks[b];
    return 4 * B.nnz * plan->stream_edge_arenas(b) + 4 * ((uint64_t)(plan->cuts[B.i + 1] - plan->cuts[B.i]) + 1) +
           4 * clen(b);
  }
  // Copies block b from the pinned host arenas to device arenas (edge arrays at
  // edge offset e_dst, row offsets at ro_dst, column offsets at co_dst), then its
  // ready flag = epoch.  A column-major block's column ids cross PCIe as its column
  // offsets (|V_j|+1 words instead of nnz: 8 instead of 12 bytes per edge); the count
  // kernel reads them directly (kCP).  Only copy-engine operations go on the copy
  // streams: the persistent count kernel that waits for the flag never depends on a
  // kernel it could starve of SMs.
  void copy(uint32_t b, uint32_t* const* dev_edges, uint32_t* dev_rowptr, uint64_t e_dst, uint64_t ro_dst,
            uint32_t* dev_colptr, uint64_t co_dst, bool zero_runs = false) {
    const BlockDesc& B = plan->blocks[b];
    cudaStream_t cs = ctx->copy_streams[rr++ % ctx->copy_streams.size()];
    const uint64_t rlen = (uint64_t)(plan->cuts[B.i + 1] - plan->cuts[B.i]) + 1;
    auto arenas = plan->edge_arenas();
    const size_t direct = plan->stream_edge_arenas(b);   // colptr form: arena 2 (ccv) stays home
    if (B.nnz)
      for (size_t x = 0; x < direct; ++x)
        BBTC_CUDA(cudaMemcpyAsync(dev_edges[x] + e_dst, *arenas[x].host + B.e0, B.nnz * 4, cudaMemcpyHostToDevice, cs));
    if (const uint64_t cl = clen(b))
      BBTC_CUDA(cudaMemcpyAsync(dev_colptr + co_dst, plan->h_colptr + plan->co_off[b], cl * 4,
                                cudaMemcpyHostToDevice, cs));
    // Row offsets: with zero_runs the destination arena was zeroed before the copies
    // (prezero_rowptr), so the block's leading run of zeros (rows before its first
    // non-empty row — at least the isolated vertices, which hold the lowest ranks)
    // does not cross PCIe.  (No memset here: a memset kernel on a copy stream may not
    // find room next to the persistent count kernel that waits for this block's flag.)
    const uint64_t z = (zero_runs && !plan->rp_zero.empty()) ? std::min<uint64_t>(plan->rp_zero[b], rlen) : 0;
    if (rlen > z)
      BBTC_CUDA(cudaMemcpyAsync(dev_rowptr + ro_dst + z, plan->h_rowptr + B.ro + z, (rlen - z) * 4,
                                cudaMemcpyHostToDevice, cs));
    flag(b, cs);
    if (!ev[b]) BBTC_CUDA(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    BBTC_CUDA(cudaEventRecord(ev[b], cs));
    bytes += block_bytes(b) - 4 * z;
  }
  // The ready flag is a 4-byte copy from a read-only pinned table (h_epochs[e] = e)
  // queued behind the block's copies: the copy engine writes it after the data.
  void flag(uint32_t b, cudaStream_t cs) {
    if (epoch)
      BBTC_CUDA(cudaMemcpyAsync(plan->d_ready.p + b, plan->h_epochs + epoch, 4, cudaMemcpyHostToDevice, cs));
  }
  void issue(uint32_t b) {   // into the plan's full arenas, at the block's own offsets
    if (issued[b]) return;
    issued[b] = 1;
    uint32_t* dev[3];
    auto arenas = plan->edge_arenas();
    for (size_t x = 0; x < arenas.size(); ++x) dev[x] = arenas[x].dev->p;
    copy(b, dev, plan->rowptr.p, plan->blocks[b].e0, plan->blocks[b].ro, plan->d_colptr.p,
         plan->co_off.empty() ? 0 : plan->co_off[b], zero_runs);
  }
  bool zero_runs = false;   // the full rowptr arena was zeroed first (prezero_rowptr)
};

// Zeroes the plan's device row-offset arena on the context stream and makes the copy
// streams wait for it, so streamed copies can skip every block's leading zero run.
static void prezero_rowptr(bbtc_ctx* ctx, bbtc_plan* plan, Streamer* s) {
  if (getenv("BBTC_NO_RP_ZERO")) return;
  BBTC_CUDA(cudaMemsetAsync(plan->rowptr.p, 0, plan->rowptr.bytes(), ctx->stream));
  cudaEvent_t go;
  BBTC_CUDA(cudaEventCreateWithFlags(&go, cudaEventDisableTiming));
  BBTC_CUDA(cudaEventRecord(go, ctx->stream));
  for (auto cs : ctx->copy_streams) BBTC_CUDA(cudaStreamWaitEvent(cs, go, 0));
  cudaEventDestroy(go);
  s->zero_runs = true;
}

constexpr uint32_t kEpochs = 1u << 16;

// Next ready-flag epoch of a plan (allocates the flags and the pinned epoch table on
// first use; wraps by clearing the flags in stream order).
static uint32_t next_epoch(bbtc_ctx* ctx, bbtc_plan* plan) {
  if (!plan->h_epochs) {
    BBTC_CUDA(cudaHostAlloc((void**)&plan->h_epochs, kEpochs * 4, cudaHostAllocPortable));
    for (uint32_t e = 0; e < kEpochs; ++e) plan->h_epochs[e] = e;
    plan->d_ready.alloc(plan->blocks.size(), ctx);
    BBTC_CUDA(cudaMemsetAsync(plan->d_ready.p, 0, plan->blocks.size() * 4, ctx->stream));
  }
  if (++plan->epoch >= kEpochs) {
    plan->epoch = 1;
    BBTC_CUDA(cudaMemsetAsync(plan->d_ready.p, 0, plan->blocks.size() * 4, ctx->stream));
  }
  return plan->epoch;
}

// First-fit allocator over [0, cap) (the out-of-core cache arenas).
// Every free range carries the last out-of-core window whose kernel read it (-1:
// never read): a copy into it must wait for that kernel, and only for that one.
struct RangeAlloc {
  struct Range {
    uint64_t len;
    int64_t reader;
  };
  std::map<uint64_t, Range> free_;   // offset -> range
  explicit RangeAlloc(uint64_t cap) {
    if (cap) free_[0] = {cap, -1};
  }
  bool alloc(uint64_t len, uint64_t* off, int64_t* reader) {
    if (len == 0) {
      *off = 0;
      *reader = -1;
      return true;
    }
    for (auto it = free_.begin(); it != free_.end(); ++it)
      if (it->second.len >= len) {
        *off = it->first;
        *reader = it->second.reader;
        const Range rest{it->second.len - len, it->second.reader};
        const uint64_t at = it->first + len;
        free_.erase(it);
        if (rest.len) free_[at] = rest;
        return true;
      }
    return false;
  }
  void release(uint64_t off, uint64_t len, int64_t reader) {
    if (len == 0) return;
    auto it = free_.emplace(off, Range{len, reader}).first;
    auto nx = std::next(it);
    if (nx != free_.end() && it->first + it->second.len == nx->first) {
      it->second.len += nx->second.len;
      it->second.reader = std::max(it->second.reader, nx->second.reader);
      free_.erase(nx);
    }
    if (it != free_.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second.len == it->first) {
        pv->second.len += it->second.len;
        pv->second.reader = std::max(pv->second.reader, it->second.reader);
        free_.erase(it);
      }
    }
  }
};

static uint64_t rowptr_len(const bbtc_plan* plan) {
  uint64_t ro = 0;
  for (auto& B : plan->blocks) ro += (uint64_t)(plan->cuts[B.i + 1] - plan->cuts[B.i]) + 1;
  return ro;
}

static void ensure_device_arenas(bbtc_ctx* ctx, bbtc_plan* plan) {
  if (!plan->rowptr.p) plan->rowptr.alloc(rowptr_len(plan), ctx);
  for (auto& A : plan->edge_arenas())
    if (!A.dev->p && plan->m) A.dev->alloc(plan->m, ctx);
  if (plan->streams_colptr() && !plan->d_colptr.p) plan->d_colptr.alloc(std::max<uint64_t>(plan->co_off.back(), 1), ctx);
}

// After streamed copies into the plan's full arenas have landed (context stream, which
// waited for them): ccv from the column offsets, so the plan is fully resident again.
static void finish_full_arenas(bbtc_ctx* ctx, bbtc_plan* plan) {
  if (!plan->streams_colptr()) return;
  colptr_expand_all(ctx, plan);
  if (!getenv("BBTC_FORCE_CP")) plan->d_colptr.reset();   // (A/B knob: keep it for resident kCP counts)
}

}  // namespace bbtc

using namespace bbtc;

extern "C" {

BBTC_API const char* bbtc_last_error(void) { return t_err.c_str(); }
BBTC_API const char* bbtc_version(void) { return "bbtc-b200 0.1 (sm_100a)"; }

BBTC_API bbtc_status bbtc_ctx_create(const bbtc_ctx_opts* opts, bbtc_ctx** out) {
  return guard([&] {
    if (!out) raise(BBTC_EINVAL, "out is NULL");
    *out = nullptr;
    bbtc_ctx_opts o{};
    if (opts) o = *opts;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
      raise(BBTC_ECUDA, std::string("no CUDA device: ") + (e != cudaSuccess ? cudaGetErrorString(e) : "count 0"));
    if (o.device < 0 || o.device >= ndev) raise(BBTC_EINVAL, "device ordinal out of range");
    BBTC_CUDA(cudaSetDevice(o.device));
    int major = 0;
    BBTC_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, o.device));
    if (major != 10) raise(BBTC_ECUDA, "libbbtc is built for sm_100a (B200) only");
    auto* c = new bbtc_ctx();
    c->device = o.device;
    BBTC_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, o.device));
    if (o.stream) {
      c->stream = (cudaStream_t)o.stream;
    } else {
      BBTC_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    const uint32_t ncs = o.copy_streams ? o.copy_streams : 2;
    for (uint32_t x = 0; x < ncs; ++x) {
      cudaStream_t s;
      BBTC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      c->copy_streams.push_back(s);
    }
    BBTC_CUDA(cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking));
    // A/B knob: the L2's DRAM fetch granularity for misses (32/64/128 B; the random
    // row-offset and probe-list gathers use a few words of each fetched line).
    if (const char* fg = getenv("BBTC_L2_FETCH"))
      BBTC_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(fg)));
    // Keep freed pool memory cached between steps (no OS round trips per call).
    cudaMemPool_t pool;
    BBTC_CUDA(cudaDeviceGetDefaultMemPool(&pool, o.device));
    uint64_t thr = ~0ull;
    BBTC_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    size_t free_b = 0, total_b = 0;
    BBTC_CUDA(cudaMemGetInfo(&free_b, &total_b));
    c->cache_limit = total_b / 2;
    *out = c;
  });
}

BBTC_API void bbtc_ctx_free(bbtc_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto s : c->copy_streams) cudaStreamDestroy(s);
  if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
  if (c->cursor) cudaFree(c->cursor);
  for (auto& kv : c->cache) cudaFreeAsync(kv.second, c->stream);
  c->cache.clear();
  cudaStreamSynchronize(c->stream);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

BBTC_API bbtc_status bbtc_ctx_sync(bbtc_ctx* c) {
  return guard([&] {
    if (!c) raise(BBTC_EINVAL, "ctx is NULL");
    BBTC_CUDA(cudaStreamSynchronize(c->stream));
  });
}

BBTC_API bbtc_status bbtc_ctx_stream(const bbtc_ctx* c, void** stream) {
  return guard([&] {
    if (!c || !stream) raise(BBTC_EINVAL, "ctx/stream is NULL");
    *stream = (void*)c->stream;
  });
}

BBTC_API uint64_t bbtc_ctx_launches(const bbtc_ctx* c) { return c ? c->launches : 0; }

BBTC_API bbtc_status bbtc_graph_from_edges(bbtc_ctx* ctx, const uint32_t* src, const uint32_t* dst, uint64_t n_edges,
                                           uint32_t n_hint, int mem, bbtc_graph** out) {
  return guard([&] {
    if (!ctx || !out) raise(BBTC_EINVAL, "ctx/out is NULL");
    *out = nullptr;
    if (n_edges && (!src || !dst)) raise(BBTC_EINVAL, "src/dst is NULL");
    if (mem != BBTC_MEM_HOST && mem != BBTC_MEM_DEVICE) raise(BBTC_EINVAL, "mem must be BBTC_MEM_HOST or _DEVICE");
    BBTC_CUDA(cudaSetDevice(ctx->device));
    auto* g = new bbtc_graph();
    g->ctx = ctx;
    try {
      graph_build(ctx, src, dst, n_edges, n_hint, mem, g);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

BBTC_API bbtc_status bbtc_graph_from_pairs(bbtc_ctx* ctx, const uint32_t* pairs, uint64_t n_edges, uint32_t n_hint,
                                           int mem, bbtc_graph** out) {
  return guard([&] {
    if (!ctx || !out) raise(BBTC_EINVAL, "ctx/out is NULL");
    *out = nullptr;
    if (n_edges && !pairs) raise(BBTC_EINVAL, "pairs is NULL");
    if (mem == BBTC_MEM_DEVICE && (reinterpret_cast<uintptr_t>(pairs) & 7))
      raise(BBTC_EINVAL, "device pairs must be 8-byte aligned (read as uint2)");
    if (mem != BBTC_MEM_HOST && mem != BBTC_MEM_DEVICE) raise(BBTC_EINVAL, "mem must be BBTC_MEM_HOST or _DEVICE");
    BBTC_CUDA(cudaSetDevice(ctx->device));
    auto* g = new bbtc_graph();
    g->ctx = ctx;
    try {
      graph_build(ctx, nullptr, nullptr, n_edges, n_hint, mem, g, n_edges ? pairs : nullptr);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

BBTC_API bbtc_status bbtc_graph_stats_get(const bbtc_graph* g, bbtc_graph_stats* s) {
  return guard([&] {
    if (!g || !s) raise(BBTC_EINVAL, "NULL argument");
    s->n = g->n;
    s->n_nonisolated = g->n_nonisolated;
    s->m = g->m;
    s->raw_edges = g->raw;
    s->d_max = g->d_max;
    s->dplus_max = graph_dplus_max(const_cast<bbtc_graph*>(g));
  });
}

BBTC_API bbtc_status bbtc_graph_size(const bbtc_graph* g, uint32_t* n, uint64_t* m) {
  return guard([&] {
    if (!g || !n || !m) raise(BBTC_EINVAL, "NULL argument");
    *n = g->n;
    *m = g->m;
  });
}

BBTC_API bbtc_status bbtc_graph_rank(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t* rank) {
  return guard([&] {
    if (!ctx || !g || (!rank && g->n)) raise(BBTC_EINVAL, "NULL argument");
    BBTC_CUDA(cudaMemcpyAsync(rank, g->rank.p, (size_t)g->n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    BBTC_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

BBTC_API bbtc_status bbtc_graph_csr(bbtc_ctx* ctx, const bbtc_graph* g, uint64_t* row_ptr, uint32_t* col) {
  return guard([&] {
    if (!ctx || !g || !row_ptr || (!col && g->m)) raise(BBTC_EINVAL, "NULL argument");
    graph_csr(ctx, g, row_ptr, col);
  });
}

BBTC_API void bbtc_graph_free(bbtc_graph* g) { delete g; }

BBTC_API bbtc_status bbtc_plan_create(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* cuts,
                                      uint32_t flags, bbtc_plan** out) {
  return guard([&] {
    if (!ctx || !g || !out) raise(BBTC_EINVAL, "NULL argument");
    *out = nullptr;
    if (p == 0) raise(BBTC_EINVAL, "p must be >= 1");
    if (cuts && p > 4096) raise(BBTC_ERANGE, "p > 4096");
    BBTC_CUDA(cudaSetDevice(ctx->device));
    auto* plan = new bbtc_plan();
    plan->ctx = ctx;
    try {
      plan_build(ctx, g, p, cuts, flags, plan);
    } catch (...) {
      delete plan;
      throw;
    }
    *out = plan;
  });
}

BBTC_API bbtc_status bbtc_plan_auto_p(bbtc_ctx* ctx, const bbtc_graph* g, uint64_t budget_bytes, uint32_t depth,
                                      uint32_t flags, uint32_t* p) {
  return guard([&] {
    if (!ctx || !g || !p) raise(BBTC_EINVAL, "NULL argument");
    if (budget_bytes == 0) raise(BBTC_EINVAL, "budget must be > 0");
    BBTC_CUDA(cudaSetDevice(ctx->device));
    *p = plan_auto_p(ctx, g, budget_bytes, depth, flags);
  });
}

BBTC_API bbtc_status bbtc_plan_info_get(const bbtc_plan* plan, bbtc_plan_info* info) {
  return guard([&] {
    if (!plan || !info) raise(BBTC_EINVAL, "NULL argument");
    *info = plan->info;
    info->host_blocks = plan->host_blocks;
  });
}

BBTC_API bbtc_status bbtc_plan_cuts(const bbtc_plan* plan, uint32_t* cuts) {
  return guard([&] {
    if (!plan || !cuts) raise(BBTC_EINVAL, "NULL argument");
    std::copy(plan->cuts.begin(), plan->cuts.end(), cuts);
  });
}

BBTC_API bbtc_status bbtc_plan_block(bbtc_ctx* ctx, const bbtc_plan* plan, uint32_t i, uint32_t j, uint32_t* row_ptr,
                                     uint32_t* col, uint32_t* row, uint64_t* nnz) {
  return guard([&] {
    if (!ctx || !plan) raise(BBTC_EINVAL, "NULL argument");
    if (i > j || j >= plan->p) raise(BBTC_EINVAL, "need i <= j < p");
    const BlockDesc& B = plan->blocks[block_id(i, j)];
    if (nnz) *nnz = B.nnz;
    const uint64_t rlen = (uint64_t)(plan->cuts[i + 1] - plan->cuts[i]) + 1;
    cudaStream_t st = ctx->stream;
    std::vector<uint32_t> rp(rlen);
    if (plan->host_blocks && !plan->resident) {
      std::memcpy(rp.data(), plan->h_rowptr + B.ro, rlen * 4);
      if (col) std::memcpy(col, plan->h_cols + B.e0, B.nnz * 4);
    } else {
      BBTC_CUDA(cudaMemcpyAsync(rp.data(), plan->rowptr.p + B.ro, rlen * 4, cudaMemcpyDeviceToHost, st));
      if (col && B.nnz) BBTC_CUDA(cudaMemcpyAsync(col, plan->cols.p + B.e0, B.nnz * 4, cudaMemcpyDeviceToHost, st));
      BBTC_CUDA(cudaStreamSynchronize(st));
    }
    if (row_ptr) std::copy(rp.begin(), rp.end(), row_ptr);
    if (row)   // the row id of every edge, expanded from the row offsets
      for (uint64_t r = 0; r + 1 < rlen; ++r)
        for (uint32_t x = rp[r]; x < rp[r + 1]; ++x) row[x] = (uint32_t)r;
  });
}

BBTC_API bbtc_status bbtc_plan_to_host(bbtc_ctx* ctx, bbtc_plan* plan) {
  return guard([&] {
    if (!ctx || !plan) raise(BBTC_EINVAL, "NULL argument");
    if (plan->host_blocks) return;
    const uint64_t ro = rowptr_len(plan);
    cudaStream_t st = ctx->stream;
    for (auto& A : plan->edge_arenas()) {
      BBTC_CUDA(cudaHostAlloc((void**)A.host, std::max<uint64_t>(plan->m, 1) * 4, cudaHostAllocPortable));
      if (plan->m) BBTC_CUDA(cudaMemcpyAsync(*A.host, A.dev->p, plan->m * 4, cudaMemcpyDeviceToHost, st));
    }
    BBTC_CUDA(cudaHostAlloc((void**)&plan->h_rowptr, std::max<uint64_t>(ro, 1) * 4, cudaHostAllocPortable));
    BBTC_CUDA(cudaMemcpyAsync(plan->h_rowptr, plan->rowptr.p, ro * 4, cudaMemcpyDeviceToHost, st));
    if (plan->colmajor) {   // the streamed form of ccv: per-block column offsets
      DevBuf<uint32_t> cp;
      const uint64_t len = colptr_build(ctx, plan, &cp);
      BBTC_CUDA(cudaHostAlloc((void**)&plan->h_colptr, std::max<uint64_t>(len, 1) * 4, cudaHostAllocPortable));
      BBTC_CUDA(cudaMemcpyAsync(plan->h_colptr, cp.p, len * 4, cudaMemcpyDeviceToHost, st));
      BBTC_CUDA(cudaStreamSynchronize(st));
    }
    // leading zero run of every block's row offsets (set on the device when streamed)
    BBTC_CUDA(cudaStreamSynchronize(st));   // h_rowptr has landed
    plan->rp_zero.assign(plan->blocks.size(), 0);
    for (size_t b = 0; b < plan->blocks.size(); ++b) {
      const BlockDesc& B = plan->blocks[b];
      const uint32_t* r = plan->h_rowptr + B.ro;
      const uint64_t rlen = (uint64_t)(plan->cuts[B.i + 1] - plan->cuts[B.i]) + 1;
      plan->rp_zero[b] = (uint64_t)(std::find_if(r, r + rlen, [](uint32_t x) { return x != 0; }) - r);
    }
    plan->info.stream_bytes = 0;
    for (size_t b = 0; b < plan->blocks.size(); ++b) {
      const BlockDesc& B = plan->blocks[b];
      plan->info.stream_bytes += 4 * ((uint64_t)(plan->cuts[B.i + 1] - plan->cuts[B.i]) + 1 - plan->rp_zero[b]);
      if (plan->block_colptr((uint32_t)b) && B.nnz)
        plan->info.stream_bytes += 8 * B.nnz + 4 * ((uint64_t)(plan->cuts[B.j + 1] - plan->cuts[B.j]) + 1);
      else plan->info.stream_bytes += 4 * B.nnz * plan->edge_arenas().size();
    }
    BBTC_CUDA(cudaStreamSynchronize(st));
    for (auto& A : plan->edge_arenas()) A.dev->reset();
    plan->slots_ready = false;   // (the slots live in the cols arena)
    if (plan->colmajor) plan->rows.reset();   // (kept only for the dense row walk of resident plans)
    plan->rowptr.reset();
    plan->dense.reset();
    plan->dense_ready = false;
    plan->host_blocks = true;
    plan->resident = false;
    plan->info.host_blocks = 1;
  });
}

BBTC_API bbtc_status bbtc_stage(bbtc_ctx* ctx, bbtc_plan* plan) {
  return guard([&] {
    if (!ctx || !plan) raise(BBTC_EINVAL, "NULL argument");
    if (plan->resident) return;
    ensure_device_arenas(ctx, plan);
    Streamer s(ctx, plan);
    prezero_rowptr(ctx, plan, &s);
    for (uint32_t b = 0; b < plan->blocks.size(); ++b) s.issue(b);
    for (auto cs : ctx->copy_streams) BBTC_CUDA(cudaStreamSynchronize(cs));
    finish_full_arenas(ctx, plan);
    BBTC_CUDA(cudaStreamSynchronize(ctx->stream));
    plan->resident = true;
  });
}

BBTC_API bbtc_status bbtc_stage_blocks(bbtc_ctx* ctx, bbtc_plan* plan, const uint32_t* ids, uint32_t n,
                                       uint32_t flags) {
  return guard([&] {
    if (!ctx || !plan || (n && !ids)) raise(BBTC_EINVAL, "NULL argument");
    if (!plan->host_blocks) raise(BBTC_ESTATE, "the plan's blocks are not in host memory (bbtc_plan_to_host)");
    BBTC_CUDA(cudaSetDevice(ctx->device));
    if (plan->resident && n) return;   // everything is on the device already
    ensure_device_arenas(ctx, plan);
    auto arenas = plan->edge_arenas();
    for (uint32_t x = 0; x < n; ++x) {
      const uint32_t b = ids[x];
      if (b >= plan->blocks.size()) raise(BBTC_EINVAL, "block id >= p(p+1)/2");
      const BlockDesc& B = plan->blocks[b];
      cudaStream_t cs = ctx->copy_streams[x % ctx->copy_streams.size()];
      for (auto& A : arenas)   // the block's device form as it is (incl. ccv: no expansion step)
        if (B.nnz)
          BBTC_CUDA(cudaMemcpyAsync(A.dev->p + B.e0, *A.host + B.e0, B.nnz * 4, cudaMemcpyHostToDevice, cs));
      const uint64_t rlen = (uint64_t)(plan->cuts[B.i + 1] - plan->cuts[B.i]) + 1;
      BBTC_CUDA(cudaMemcpyAsync(plan->rowptr.p + B.ro, plan->h_rowptr + B.ro, rlen * 4, cudaMemcpyHostToDevice, cs));
    }
    for (auto cs : ctx->copy_streams) BBTC_CUDA(cudaStreamSynchronize(cs));
    if (flags & BBTC_STAGE_RESIDENT) {
      plan->d_colptr.reset();
      plan->dense.reset();
      plan->dense_ready = false;
      plan->resident = true;
    }
  });
}

BBTC_API bbtc_status bbtc_unstage(bbtc_ctx* ctx, bbtc_plan* plan) {
  return guard([&] {
    if (!ctx || !plan) raise(BBTC_EINVAL, "NULL argument");
    if (!plan->host_blocks) return;   // device plans own their only copy
    BBTC_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto& A : plan->edge_arenas()) A.dev->reset();
    plan->slots_ready = false;   // (the slots live in the cols arena)
    plan->rowptr.reset();
    plan->d_colptr.reset();
    plan->dense.reset();
    plan->dense_ready = false;
    plan->resident = false;
  });
}

BBTC_API void bbtc_plan_free(bbtc_plan* plan) {
  if (!plan) return;
  if (plan->ctx) cudaStreamSynchronize(plan->ctx->stream);
  if (plan->h_cols) cudaFreeHost(plan->h_cols);
  if (plan->h_rows) cudaFreeHost(plan->h_rows);
  if (plan->h_ccu) cudaFreeHost(plan->h_ccu);
  if (plan->h_ccv) cudaFreeHost(plan->h_ccv);
  if (plan->h_rowptr) cudaFreeHost(plan->h_rowptr);
  if (plan->h_colptr) cudaFreeHost(plan->h_colptr);
  if (plan->h_epochs) cudaFreeHost(plan->h_epochs);
  delete plan;
}

BBTC_API bbtc_status bbtc_plan_set_budget(bbtc_plan* plan, uint64_t bytes) {
  return guard([&] {
    if (!plan) raise(BBTC_EINVAL, "plan is NULL");
    plan->budget = bytes;
    // Below the plan's size, re-order the tasks in part groups sized so one group
    // triple's blocks (<= 3h^2 of them) take about half the budget.
    uint64_t all = 0;
    Streamer sz(plan->ctx, plan);
    for (uint32_t b = 0; b < plan->blocks.size(); ++b) all += sz.block_bytes(b);
    uint32_t h = 0;
    if (bytes > 0 && bytes < all && !plan->blocks.empty()) {
      const double avg = (double)all / (double)plan->blocks.size();
      const char* fe = getenv("BBTC_OOC_FILL");
      const double fill = fe ? atof(fe) : 0.8;   // scripts/ooc_sweep.py: 0.8 moved the fewest bytes
      h = (uint32_t)std::max(1.0, std::floor(std::sqrt(fill * (double)bytes / (3.0 * avg))));
      if (h >= plan->p) h = 0;
    }
    if (h != plan->task_group) {
      BBTC_CUDA(cudaStreamSynchronize(plan->ctx->stream));   // d_tasks may be in use
      plan->task_group = h;
      plan_tasks(plan, 1);
    }
  });
}

BBTC_API uint64_t bbtc_n_tasks(uint32_t p) { return n_tasks(p); }

BBTC_API bbtc_status bbtc_task_index(uint32_t p, uint32_t i, uint32_t j, uint32_t k, uint64_t* idx) {
  return guard([&] {
    if (!idx) raise(BBTC_EINVAL, "idx is NULL");
    if (!(i <= j && j <= k && k < p)) raise(BBTC_EINVAL, "need i <= j <= k < p");
    *idx = task_index(p, i, j, k);
  });
}

BBTC_API bbtc_status bbtc_task_ijk(uint32_t p, uint64_t idx, uint32_t* i, uint32_t* j, uint32_t* k) {
  return guard([&] {
    if (!i || !j || !k) raise(BBTC_EINVAL, "NULL argument");
    if (idx >= n_tasks(p)) raise(BBTC_EINVAL, "idx >= n_tasks(p)");
    // Invert the closed form: find i, then j, then k by monotone search.
    uint32_t a = 0;
    while (a + 1 < p && task_index(p, a + 1, a + 1, a + 1) <= idx) ++a;
    uint32_t b = a;
    while (b + 1 < p && task_index(p, a, b + 1, b + 1) <= idx) ++b;
    *i = a;
    *j = b;
    *k = b + (uint32_t)(idx - task_index(p, a, b, b));
  });
}

// Streaming order (a6): the sparse tasks reordered by when their blocks land.  Default
// ("peel", below): the block order is built backwards so that the work left after the
// last copies is small.  "greedy": forwards — every task whose blocks are all issued
// goes next (in execution order); otherwise the task with the most work (work items,
// which carry equal estimated work, R8) per byte of its blocks still to copy.  The copies follow
// the same order, so the kernel always has unlocked work while later blocks are in
// flight (the execution order puts the densest column of blocks last: with it the
// kernel idles until those copies land).  O(T^2): plans with more than kGreedyMax
// sparse tasks keep the execution order.
static void stream_order(bbtc_ctx* ctx, bbtc_plan* plan) {
  if (plan->s_ready) return;
  constexpr size_t kGreedyMax = 6000;
  const size_t ns = plan->dense_task_lo;
  std::vector<uint32_t> ord;
  ord.reserve(ns);
  static const bool peel = [] {   // default; BBTC_STREAM_ORDER=greedy selects the forward greedy order
    const char* e = getenv("BBTC_STREAM_ORDER");
    return !(e && std::string(e) == "greedy");
  }();
  if (peel && ns <= kGreedyMax) {
    // Tail-aware: build the block order backwards.  Repeatedly take, among the blocks
    // not yet placed, the one whose still-unplaced tasks carry the least work per byte
    // and place it last (with those tasks): the work that can only start after the last
    // copies land is as small as possible.  Tasks run in the order their last block lands.
    const uint32_t nb = (uint32_t)plan->blocks.size();
    std::vector<double> bytes(nb);
    for (uint32_t b = 0; b < nb; ++b) bytes[b] = std::max(1.0, (double)Streamer(ctx, plan).block_bytes(b));
    std::vector<char> gone(nb, 0), placed(ns, 0);
    std::vector<std::vector<uint32_t>> rev_tasks;   // per peeled block, its tasks
    for (uint32_t it = 0; it < nb; ++it) {
      std::vector<double> w(nb, 0.0);
      for (size_t t = 0; t < ns; ++t) {
        if (placed[t]) continue;
        const TaskDesc& T = plan->tasks[t];
        const double wt = (double)(plan->item_start[t + 1] - plan->item_start[t]);
        for (uint32_t b : {T.ij, T.ik, T.jk}) w[b] += wt;
      }
      int64_t best = -1;
      for (uint32_t b = 0; b < nb; ++b)
        if (!gone[b] && (best < 0 || w[b] / bytes[b] < w[best] / bytes[best])) best = b;
      gone[best] = 1;
      rev_tasks.emplace_back();
      for (size_t t = 0; t < ns; ++t) {
        if (placed[t]) continue;
        const TaskDesc& T = plan->tasks[t];
        if (T.ij == (uint32_t)best || T.ik == (uint32_t)best || T.jk == (uint32_t)best) {
          placed[t] = 1;
          rev_tasks.back().push_back((uint32_t)t);
        }
      }
    }
    for (size_t x = rev_tasks.size(); x-- > 0;)
      for (uint32_t t : rev_tasks[x]) ord.push_back(t);
  } else if (ns <= kGreedyMax) {
    const uint32_t nb = (uint32_t)plan->blocks.size();
    std::vector<double> bytes(nb);
    for (uint32_t b = 0; b < nb; ++b) bytes[b] = (double)Streamer(ctx, plan).block_bytes(b);
    std::vector<char> have(nb, 0), done(ns, 0);
    size_t left = ns;
    while (left) {
      bool took = false;
      for (size_t t = 0; t < ns; ++t) {
        if (done[t]) continue;
        const TaskDesc& T = plan->tasks[t];
        if (have[T.ij] && have[T.ik] && have[T.jk]) {
          done[t] = 1;
          --left;
          ord.push_back((uint32_t)t);
          took = true;
        }
      }
      if (took) continue;
      double best = -1;
      size_t bt = 0;
      for (size_t t = 0; t < ns; ++t) {
        if (done[t]) continue;
        const TaskDesc& T = plan->tasks[t];
        double miss = 0;
        if (!have[T.ij]) miss += bytes[T.ij];
        if (!have[T.ik] && T.ik != T.ij) miss += bytes[T.ik];
        if (!have[T.jk] && T.jk != T.ij && T.jk != T.ik) miss += bytes[T.jk];
        const double work = (double)(plan->item_start[t + 1] - plan->item_start[t]);
        const double score = work / std::max(miss, 1.0);
        if (score > best) {
          best = score;
          bt = t;
        }
      }
      const TaskDesc& T = plan->tasks[bt];
      have[T.ij] = have[T.ik] = have[T.jk] = 1;
    }
  } else {
    for (size_t t = 0; t < ns; ++t) ord.push_back((uint32_t)t);
  }
  plan->s_tasks.clear();
  plan->s_item_start.assign(1, 0);
  for (uint32_t t : ord) {
    plan->s_tasks.push_back(plan->tasks[t]);
    plan->s_item_start.push_back(plan->s_item_start.back() + plan->item_start[t + 1] - plan->item_start[t]);
  }
  // the dense tasks keep their place after the sparse ones (items [dense_item_lo, end))
  for (size_t t = ns; t < plan->tasks.size(); ++t) {
    plan->s_tasks.push_back(plan->tasks[t]);
    plan->s_item_start.push_back(plan->s_item_start.back() + plan->item_start[t + 1] - plan->item_start[t]);
  }
  plan->d_s_tasks.alloc(std::max<size_t>(plan->s_tasks.size(), 1), ctx);
  plan->d_s_item_start.alloc(plan->s_item_start.size(), ctx);
  if (!plan->s_tasks.empty())
    BBTC_CUDA(cudaMemcpyAsync(plan->d_s_tasks.p, plan->s_tasks.data(), plan->s_tasks.size() * sizeof(TaskDesc),
                              cudaMemcpyHostToDevice, ctx->stream));
  BBTC_CUDA(cudaMemcpyAsync(plan->d_s_item_start.p, plan->s_item_start.data(), plan->s_item_start.size() * 8,
                            cudaMemcpyHostToDevice, ctx->stream));
  plan->s_ready = true;
}

// A/B knob (BBTC_FORCE_CP=1): the streamed walk (column offsets, kCP) over resident
// blocks of a host plan that kept its device column offsets; else NULL (the plan's arenas).
static const DevArenas* ab_colptr_arenas(bbtc_plan* plan, DevArenas* ar) {
  if (!(getenv("BBTC_FORCE_CP") && plan->d_colptr.p && plan->d_item_col.p)) return nullptr;
  ar->cols = plan->cols.p;
  ar->it_u = plan->ccu.p;
  ar->it_v = plan->ccv.p;
  ar->rowptr = plan->rowptr.p;
  ar->blocks = plan->d_blocks.p;
  ar->colptr = plan->d_colptr.p;
  ar->item_col = plan->d_item_col.p;
  return ar;
}

// Resident blocks: the list kernel over the sparse tasks' items, then the bit-row
// kernel over the dense tasks' items (building the bit rows on first use).
static void count_resident(bbtc_ctx* ctx, bbtc_plan* plan, uint32_t rank, uint32_t world, uint64_t* d_counts,
                           cudaEvent_t mid = nullptr) {
  static const bool concurrent = getenv("BBTC_DENSE_CONCURRENT") != nullptr;
  if (concurrent && !mid && plan->dense_item_lo < plan->item_start.back()) {
    // A/B: the bit-row build and kernel on the aux stream beside the list kernel (they
    // share only the counters, updated atomically): the dense CTAs take SMs as the
    // persistent list kernel's CTAs retire.
    cudaEvent_t go, done;
    BBTC_CUDA(cudaEventCreateWithFlags(&go, cudaEventDisableTiming));
    BBTC_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    BBTC_CUDA(cudaEventRecord(go, ctx->stream));
    BBTC_CUDA(cudaStreamWaitEvent(ctx->aux_stream, go, 0));
    cudaStream_t main_st = ctx->stream;
    ctx->stream = ctx->aux_stream;
    try {
      dense_build(ctx, plan);
      count_launch_dense(ctx, plan, rank, world, d_counts, plan->dense_item_lo, plan->item_start.back());
    } catch (...) {
      ctx->stream = main_st;
      throw;
    }
    ctx->stream = main_st;
    BBTC_CUDA(cudaEventRecord(done, ctx->aux_stream));
    DevArenas ar;
    count_launch(ctx, plan, rank, world, d_counts, 0, plan->dense_item_lo, nullptr, 0, ab_colptr_arenas(plan, &ar));
    BBTC_CUDA(cudaStreamWaitEvent(ctx->stream, done, 0));
    cudaEventDestroy(go);
    cudaEventDestroy(done);
    return;
  }
  dense_build(ctx, plan);
  DevArenas ar;
  count_launch(ctx, plan, rank, world, d_counts, 0, plan->dense_item_lo, nullptr, 0, ab_colptr_arenas(plan, &ar));
  if (mid) BBTC_CUDA(cudaEventRecord(mid, ctx->stream));
  count_launch_dense(ctx, plan, rank, world, d_counts, plan->dense_item_lo, plan->item_start.back());
}

BBTC_API bbtc_status bbtc_count_async(bbtc_ctx* ctx, const bbtc_plan* plan, uint32_t rank, uint32_t world,
                                      uint64_t* d_counts) {
  return guard([&] {
    if (!ctx || !plan || !d_counts) raise(BBTC_EINVAL, "NULL argument");
    if (world == 0 || rank >= world) raise(BBTC_EINVAL, "need rank < world");
    if (!plan->resident) raise(BBTC_ESTATE, "blocks are not device-resident: call bbtc_stage or bbtc_count");
    count_zero(ctx, plan, d_counts);
    if (plan->shard_world) {   // a shard plan holds exactly its rank's tasks
      if (rank != plan->shard_rank || world != plan->shard_world)
        raise(BBTC_EINVAL, "a shard plan counts only its own rank of its own world");
      rank = 0;
      world = 1;
    }
    count_resident(ctx, const_cast<bbtc_plan*>(plan), rank, world, d_counts);
  });
}

// ---- §8(f)#4 study support ------------------------------------------------------------
BBTC_API bbtc_status bbtc_plan_block_nnz(const bbtc_plan* plan, uint64_t* nnz) {
  return guard([&] {
    if (!plan || !nnz) raise(BBTC_EINVAL, "NULL argument");
    for (size_t b = 0; b < plan->blocks.size(); ++b) nnz[b] = plan->blocks[b].nnz;
  });
}

BBTC_API bbtc_status bbtc_task_times(bbtc_ctx* ctx, const bbtc_plan* cplan, double* ms) {
  return guard([&] {
    if (!ctx || !cplan || !ms) raise(BBTC_EINVAL, "NULL argument");
    bbtc_plan* plan = const_cast<bbtc_plan*>(cplan);
    if (!plan->resident) raise(BBTC_ESTATE, "blocks are not device-resident");
    BBTC_CUDA(cudaSetDevice(ctx->device));
    const uint64_t nt = plan->info.n_tasks;
    DevBuf<uint64_t> d_counts, cyc;
    d_counts.alloc(nt + 1, ctx);
    cyc.alloc(nt, ctx);
    BBTC_CUDA(cudaMemsetAsync(cyc.p, 0, nt * 8, ctx->stream));
    count_zero(ctx, plan, d_counts.p);
    // One ordinary resident count whose warps add each work item's clock64() span to
    // its task: the task's total warp time inside the real launch (one launch per task
    // would time the latency of its longest item instead).
    ctx->task_cycles = cyc.p;
    try {
      count_resident(ctx, plan, 0, 1, d_counts.p);
    } catch (...) {
      ctx->task_cycles = nullptr;
      throw;
    }
    ctx->task_cycles = nullptr;
    std::vector<uint64_t> h(nt);
    BBTC_CUDA(cudaMemcpyAsync(h.data(), cyc.p, nt * 8, cudaMemcpyDeviceToHost, ctx->stream));
    BBTC_CUDA(cudaStreamSynchronize(ctx->stream));
    int khz = 0;
    BBTC_CUDA(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, ctx->device));
    for (uint64_t t = 0; t < nt; ++t) ms[t] = (double)h[t] / std::max(khz, 1);
  });
}

BBTC_API bbtc_status bbtc_cuts_refine(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* cuts_in,
                                      uint32_t max_evals, uint32_t* cuts_out, uint64_t* m_max_out) {
  return guard([&] {
    if (!ctx || !g || !cuts_out || !m_max_out) raise(BBTC_EINVAL, "NULL argument");
    if (p == 0 || p > 4096) raise(BBTC_EINVAL, "need 1 <= p <= 4096");
    BBTC_CUDA(cudaSetDevice(ctx->device));
    cuts_refine(ctx, g, p, cuts_in, max_evals, cuts_out, m_max_out);
  });
}

// ---- §8(f)#3 hybrid CPU+GPU (cpu.cpp holds the CPU side) -----------------------------
BBTC_API bbtc_status bbtc_count_hybrid(bbtc_ctx* ctx, const bbtc_plan* cplan, const bbtc_hybrid_opts* o,
                                       uint64_t* total, uint64_t* per_task, bbtc_timing* tm,
                                       bbtc_hybrid_stats* hs) {
  return guard([&] {
    if (!ctx || !cplan || !total) raise(BBTC_EINVAL, "NULL argument");
    bbtc_plan* plan = const_cast<bbtc_plan*>(cplan);
    if (!plan->host_blocks || !plan->resident)
      raise(BBTC_ESTATE, "hybrid counts need host arenas (bbtc_plan_to_host) and resident blocks (bbtc_stage)");
    if (plan->shard_world) raise(BBTC_EINVAL, "hybrid counts take whole plans, not shards");
    bbtc_hybrid_opts opt{0, 0, 0.5};
    if (o) opt = *o;
    if (!(opt.cutoff >= 0.0 && opt.cutoff <= 1.0)) raise(BBTC_EINVAL, "cutoff must be in [0, 1]");
    BBTC_CUDA(cudaSetDevice(ctx->device));
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    const uint64_t l0 = ctx->launches;
    const uint64_t nt = plan->info.n_tasks;
    DevBuf<uint64_t> d_counts;
    d_counts.alloc(nt + 1, ctx);
    count_zero(ctx, plan, d_counts.p);
    const std::vector<uint32_t> q = exec_time_queue(plan);   // execution-order task positions
    const uint64_t n = q.size();
    const uint64_t cut = (uint64_t)std::ceil(opt.cutoff * (double)n);
    std::mutex mu;
    uint64_t front = 0, back = n;   // [front, back) unclaimed
    // CPU threads: single tasks from the back, never below the cut-off
    unsigned nth = opt.cpu_threads ? opt.cpu_threads : std::max(1u, std::thread::hardware_concurrency());
    if (cut >= n) nth = 0;
    std::vector<std::vector<uint64_t>> cpu_pt(nth, std::vector<uint64_t>(nt, 0));
    std::vector<uint64_t> cpu_done(nth, 0);
    std::atomic<int64_t> cpu_end_us{0};
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < nth; ++w)
      pool.emplace_back([&, w] {
        std::vector<uint64_t> bits;
        for (;;) {
          uint64_t t;
          {
            std::lock_guard<std::mutex> lk(mu);
            if (back <= std::max(front, cut)) break;
            t = --back;
          }
          const TaskDesc& T = plan->tasks[q[t]];
          cpu_pt[w][T.idx] += cpu_count_task(plan, T, bits);
          cpu_done[w]++;
        }
        const int64_t us = std::chrono::duration_cast<std::chrono::microseconds>(clk::now() - t0).count();
        int64_t prev = cpu_end_us.load();
        while (prev < us && !cpu_end_us.compare_exchange_weak(prev, us)) {}
      });
    // GPU: the front up to the cut-off, then chunks while tasks remain; one launch per
    // claim over its own task table, the next claim after the previous launch ends.
    std::vector<DevBuf<TaskDesc>> tabs;
    std::vector<DevBuf<uint64_t>> starts;
    std::vector<std::vector<TaskDesc>> h_tabs;
    std::vector<std::vector<uint64_t>> h_starts;
    uint64_t gpu_tasks = 0, claims = 0;
    for (bool first = true;; first = false) {
      uint64_t a, b;
      {
        std::lock_guard<std::mutex> lk(mu);
        if (front >= back) break;
        a = front;
        const uint64_t left = back - front;
        const uint64_t take = first ? std::max<uint64_t>(cut, std::min<uint64_t>(left, 1))
                                    : (opt.gpu_chunk ? opt.gpu_chunk : std::max<uint64_t>(1, left / 8));
        b = std::min(back, a + std::max<uint64_t>(take, 1));
        front = b;
      }
      h_tabs.emplace_back();
      h_starts.emplace_back(1, 0);
      for (uint64_t x = a; x < b; ++x) {
        const uint32_t t = q[x];
        h_tabs.back().push_back(plan->tasks[t]);
        h_starts.back().push_back(h_starts.back().back() + plan->item_start[t + 1] - plan->item_start[t]);
      }
      tabs.emplace_back();
      starts.emplace_back();
      tabs.back().alloc(h_tabs.back().size(), ctx);
      starts.back().alloc(h_starts.back().size(), ctx);
      BBTC_CUDA(cudaMemcpyAsync(tabs.back().p, h_tabs.back().data(), h_tabs.back().size() * sizeof(TaskDesc),
                                cudaMemcpyHostToDevice, ctx->stream));
      BBTC_CUDA(cudaMemcpyAsync(starts.back().p, h_starts.back().data(), h_starts.back().size() * 8,
                                cudaMemcpyHostToDevice, ctx->stream));
      count_launch(ctx, plan, 0, 1, d_counts.p, 0, h_starts.back().back(), nullptr, 0, nullptr, tabs.back().p,
                   starts.back().p, (uint32_t)h_tabs.back().size());
      gpu_tasks += b - a;
      ++claims;
      BBTC_CUDA(cudaStreamSynchronize(ctx->stream));   // a claim ends before the next one
    }
    const double t_gpu = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    // dense tasks stay on the GPU
    dense_build(ctx, plan);
    count_launch_dense(ctx, plan, 0, 1, d_counts.p, plan->dense_item_lo, plan->item_start.back());
    std::vector<uint64_t> h(nt + 1);
    BBTC_CUDA(cudaMemcpyAsync(h.data(), d_counts.p, (nt + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    BBTC_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto& th : pool) th.join();
    uint64_t cpu_tri = 0, cpu_tasks = 0;
    for (unsigned w = 0; w < nth; ++w) {
      cpu_tasks += cpu_done[w];
      for (uint64_t t = 0; t < nt; ++t) {
        h[t] += cpu_pt[w][t];
        cpu_tri += cpu_pt[w][t];
      }
    }
    h[nt] += cpu_tri;
    *total = h[nt];
    if (per_task) std::copy(h.begin(), h.begin() + nt, per_task);
    const double t_all = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    if (tm) {
      std::memset(tm, 0, sizeof(*tm));
      tm->t_total_ms = t_all;
      tm->launches = ctx->launches - l0;
    }
    if (hs) {
      hs->cpu_tasks = cpu_tasks;
      hs->gpu_tasks = gpu_tasks;
      hs->gpu_launches = claims;
      hs->cpu_triangles = cpu_tri;
      hs->t_cpu_ms = cpu_end_us.load() / 1e3;
      hs->t_gpu_ms = t_gpu;
    }
  });
}

// ---- §8(e) sharded build ------------------------------------------------------------
BBTC_API bbtc_status bbtc_shard_canon(bbtc_ctx* ctx, const uint32_t* src, const uint32_t* dst, uint64_t n_edges,
                                      int mem, uint32_t n_hint, uint32_t world, uint64_t* d_keys_out,
                                      uint64_t* send_counts, uint32_t* max_id_plus1) {
  return guard([&] {
    if (!ctx || !send_counts || !max_id_plus1 || (n_edges && (!src || !dst || !d_keys_out)))
      raise(BBTC_EINVAL, "NULL argument");
    if (world == 0) raise(BBTC_EINVAL, "world must be >= 1");
    if (mem != BBTC_MEM_HOST && mem != BBTC_MEM_DEVICE) raise(BBTC_EINVAL, "mem must be BBTC_MEM_HOST or _DEVICE");
    BBTC_CUDA(cudaSetDevice(ctx->device));
    shard_canon(ctx, src, dst, n_edges, mem, n_hint, world, d_keys_out, send_counts, max_id_plus1);
    if (*max_id_plus1 == 0 && n_edges) raise(BBTC_ERANGE, "vertex id 0xFFFFFFFF is reserved");
  });
}

BBTC_API bbtc_status bbtc_shard_graph(bbtc_ctx* ctx, const uint64_t* d_keys, uint64_t n_keys, uint32_t n,
                                      uint32_t* d_deg, bbtc_graph** out) {
  return guard([&] {
    if (!ctx || !out || !d_deg || (n_keys && !d_keys)) raise(BBTC_EINVAL, "NULL argument");
    if (n == 0xFFFFFFFFu) raise(BBTC_ERANGE, "n must be < 2^32-1");
    *out = nullptr;
    BBTC_CUDA(cudaSetDevice(ctx->device));
    auto* g = new bbtc_graph();
    g->ctx = ctx;
    try {
      shard_graph(ctx, d_keys, n_keys, n, d_deg, g);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

BBTC_API bbtc_status bbtc_shard_rank(bbtc_ctx* ctx, bbtc_graph* g, const uint32_t* d_deg, uint64_t m_total) {
  return guard([&] {
    if (!ctx || !g || !d_deg) raise(BBTC_EINVAL, "NULL argument");
    if (!g->ckeys.p && g->m) raise(BBTC_ESTATE, "graph is not an unranked shard (bbtc_shard_graph)");
    if (m_total < g->m) raise(BBTC_EINVAL, "m_total is below this shard's edge count");
    if (m_total >= 0xFFFFFFFFull) raise(BBTC_ERANGE, "m >= 2^32-1 edges is not supported (32-bit block offsets)");
    BBTC_CUDA(cudaSetDevice(ctx->device));
    shard_rank(ctx, g, d_deg, m_total);
  });
}

BBTC_API bbtc_status bbtc_shard_block_sizes(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* cuts,
                                            uint64_t* d_block_nnz, uint32_t* cuts_out, uint32_t* p_eff) {
  return guard([&] {
    if (!ctx || !g || !d_block_nnz || !cuts_out || !p_eff) raise(BBTC_EINVAL, "NULL argument");
    if (p == 0) raise(BBTC_EINVAL, "p must be >= 1");
    if (p > 4096) raise(BBTC_ERANGE, "p > 4096");
    BBTC_CUDA(cudaSetDevice(ctx->device));
    *p_eff = shard_blocks_hist(ctx, g, p, cuts, d_block_nnz, cuts_out);
  });
}

BBTC_API bbtc_status bbtc_shard_assign(uint32_t p, const uint32_t* cuts, const uint64_t* block_nnz, uint32_t world,
                                       uint32_t* task_rank, uint32_t* block_rank) {
  return guard([&] {
    if (!cuts || !block_nnz || !task_rank || !block_rank) raise(BBTC_EINVAL, "NULL argument");
    if (p == 0 || world == 0) raise(BBTC_EINVAL, "need p >= 1 and world >= 1");
    for (uint32_t i = 0; i < p; ++i)
      if (cuts[i] > cuts[i + 1]) raise(BBTC_EINVAL, "cuts must be non-decreasing");
    shard_assign(p, cuts, block_nnz, world, task_rank, block_rank);
  });
}

BBTC_API bbtc_status bbtc_shard_by_block(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* cuts,
                                         const uint32_t* block_rank, uint32_t world, uint64_t* d_out,
                                         uint64_t* send_counts) {
  return guard([&] {
    if (!ctx || !g || !cuts || !block_rank || !send_counts || (g->m && !d_out)) raise(BBTC_EINVAL, "NULL argument");
    if (world == 0 || p == 0) raise(BBTC_EINVAL, "need p >= 1 and world >= 1");
    const uint32_t nb = p * (p + 1) / 2;
    for (uint32_t b = 0; b < nb; ++b)
      if (block_rank[b] >= world) raise(BBTC_EINVAL, "block owner >= world");
    BBTC_CUDA(cudaSetDevice(ctx->device));
    shard_by_block(ctx, g, p, cuts, block_rank, world, d_out, send_counts);
  });
}

BBTC_API bbtc_status bbtc_plan_create_shard(bbtc_ctx* ctx, const bbtc_graph* like, const uint64_t* d_okeys,
                                            uint64_t n_okeys, uint32_t p, const uint32_t* cuts,
                                            const uint64_t* block_nnz, const uint32_t* task_rank, uint32_t rank,
                                            uint32_t world, uint32_t flags, bbtc_plan** out) {
  return guard([&] {
    if (!ctx || !like || !cuts || !block_nnz || !task_rank || !out || (n_okeys && !d_okeys))
      raise(BBTC_EINVAL, "NULL argument");
    if (p == 0 || world == 0 || rank >= world) raise(BBTC_EINVAL, "need p >= 1 and rank < world");
    *out = nullptr;
    BBTC_CUDA(cudaSetDevice(ctx->device));
    auto* plan = new bbtc_plan();
    plan->ctx = ctx;
    try {
      plan_build_shard(ctx, like, d_okeys, n_okeys, p, cuts, block_nnz, task_rank, rank, world, flags, plan);
    } catch (...) {
      bbtc_plan_free(plan);
      throw;
    }
    *out = plan;
  });
}

BBTC_API bbtc_status bbtc_plan_block_ptrs(const bbtc_plan* plan, uint32_t b, bbtc_block_ptrs* out) {
  return guard([&] {
    if (!plan || !out) raise(BBTC_EINVAL, "NULL argument");
    if (b >= plan->blocks.size()) raise(BBTC_EINVAL, "block id >= p(p+1)/2");
    if (!plan->rowptr.p) raise(BBTC_ESTATE, "the plan has no device arenas (bbtc_stage / bbtc_stage_blocks)");
    bbtc_plan* pl = const_cast<bbtc_plan*>(plan);
    const BlockDesc& B = plan->blocks[b];
    auto arenas = pl->edge_arenas();
    std::memset(out, 0, sizeof(*out));
    out->n_edge_arrays = (uint32_t)arenas.size();
    for (size_t x = 0; x < arenas.size(); ++x) out->edge[x] = arenas[x].dev->p + B.e0;
    out->nnz = B.nnz;
    out->rowptr = pl->rowptr.p + B.ro;
    out->rowptr_len = (uint64_t)(plan->cuts[B.i + 1] - plan->cuts[B.i]) + 1;
  });
}

BBTC_API bbtc_status bbtc_count(bbtc_ctx* ctx, const bbtc_plan* cplan, uint32_t rank, uint32_t world, uint32_t flags,
                                uint64_t* total, uint64_t* per_task, bbtc_timing* tm) {
  return guard([&] {
    (void)flags;
    if (!ctx || !cplan || !total) raise(BBTC_EINVAL, "NULL argument");
    if (world == 0 || rank >= world) raise(BBTC_EINVAL, "need rank < world");
    bbtc_plan* plan = const_cast<bbtc_plan*>(cplan);   // residency state only
    if (plan->shard_world) {   // a shard plan holds exactly its rank's tasks
      if (rank != plan->shard_rank || world != plan->shard_world)
        raise(BBTC_EINVAL, "a shard plan counts only its own rank of its own world");
      rank = 0;
      world = 1;
    }
    BBTC_CUDA(cudaSetDevice(ctx->device));
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t l0 = ctx->launches;
    const uint64_t nt = plan->info.n_tasks;
    DevBuf<uint64_t> d_counts;
    d_counts.alloc(nt + 1, ctx);
    cudaEvent_t k0, k1;
    BBTC_CUDA(cudaEventCreate(&k0));
    BBTC_CUDA(cudaEventCreate(&k1));
    count_zero(ctx, plan, d_counts.p);
    uint64_t h2d = 0;
    BBTC_CUDA(cudaEventRecord(k0, ctx->stream));
    // copy streams may only start after work already queued on the context stream
    // (flag resets, the previous kernel that reads a cache region about to be reused)
    auto copies_after_stream = [&] {
      cudaEvent_t go;
      BBTC_CUDA(cudaEventCreateWithFlags(&go, cudaEventDisableTiming));
      BBTC_CUDA(cudaEventRecord(go, ctx->stream));
      for (auto cs : ctx->copy_streams) BBTC_CUDA(cudaStreamWaitEvent(cs, go, 0));
      cudaEventDestroy(go);
    };
    // t_h2d_ms: from the start of the call to the end of the last copy (events on the copy streams)
    std::vector<cudaEvent_t> c_end;
    auto copies_done = [&] {
      for (auto cs : ctx->copy_streams) {
        c_end.emplace_back();
        BBTC_CUDA(cudaEventCreate(&c_end.back()));
        BBTC_CUDA(cudaEventRecord(c_end.back(), cs));
      }
    };
    uint64_t all_bytes = 0;   // streamed form of every block
    for (uint32_t b = 0; b < plan->blocks.size(); ++b) all_bytes += Streamer(ctx, plan).block_bytes(b);
    // the full arenas also hold ccv (expanded once the copies have landed)
    const uint64_t full_bytes = all_bytes + (plan->streams_colptr() ? 4 * plan->m : 0);
    cudaEvent_t kmid = nullptr;
    if (plan->resident) {
      BBTC_CUDA(cudaEventCreate(&kmid));
      count_resident(ctx, plan, rank, world, d_counts.p, kmid);
    } else if (plan->budget == 0 || plan->budget >= full_bytes) {
      // a6: every block is copied on the copy streams in first-use order and then
      // flagged ready (epoch) on the device; ONE persistent count kernel runs
      // concurrently and each warp waits on the flags of its item's three blocks,
      // so the copies of later tasks overlap the intersections of earlier ones.
      ensure_device_arenas(ctx, plan);
      const uint32_t epoch = next_epoch(ctx, plan);
      copies_after_stream();
      const char* so = getenv("BBTC_STREAM_ORDER");   // exec | greedy | (default) peel
      const bool greedy = !(so && std::string(so) == "exec");
      if (greedy) stream_order(ctx, plan);
      Streamer s(ctx, plan);
      prezero_rowptr(ctx, plan, &s);   // (queued before the count kernel, so it runs first)
      s.epoch = epoch;
      for (const TaskDesc& T : greedy ? plan->s_tasks : plan->tasks) {
        s.issue(T.ij);
        s.issue(T.ik);
        s.issue(T.jk);
      }
      // Sparse tasks first (they come first in execution order, so their blocks are
      // issued first); the dense tasks' bit rows are built once every copy has landed
      // and the bit-row kernel runs after the list kernel, as in the resident case.
      DevArenas full;
      full.cols = plan->cols.p;
      full.it_u = plan->colmajor ? plan->ccu.p : plan->rows.p;
      full.it_v = plan->colmajor ? plan->ccv.p : plan->cols.p;   // (kCP: the ccv-shipping blocks)
      full.rowptr = plan->rowptr.p;
      full.blocks = plan->d_blocks.p;
      full.colptr = plan->streams_colptr() ? plan->d_colptr.p : nullptr;
      full.item_col = plan->d_item_col.p;
      count_launch(ctx, plan, rank, world, d_counts.p, 0, plan->dense_item_lo, plan->d_ready.p, epoch, &full,
                   greedy ? plan->d_s_tasks.p : nullptr, greedy ? plan->d_s_item_start.p : nullptr);
      // the count stream must not run past copies it did not wait for
      for (auto& e : s.ev)
        if (e) BBTC_CUDA(cudaStreamWaitEvent(ctx->stream, e, 0));
      h2d = s.bytes;
      copies_done();
      finish_full_arenas(ctx, plan);
      plan->resident = true;
      if (plan->dense_item_lo < plan->item_start.back()) {
        BBTC_CUDA(cudaEventCreate(&kmid));
        BBTC_CUDA(cudaEventRecord(kmid, ctx->stream));
        dense_build(ctx, plan);
        count_launch_dense(ctx, plan, rank, world, d_counts.p, plan->dense_item_lo, plan->item_start.back());
      }
    } else {
      // Out of core: the device holds at most `budget`
      // bytes of blocks.  Tasks are cut, in execution order, into windows whose blocks
      // fit the cache; per window, blocks no longer needed are evicted, the missing
      // ones are copied into free cache space (first fit), every block of the window
      // is flagged with the window's epoch, and the count kernel runs over the
      // window's work items, its warps waiting on the flags as in the streamed mode.
      const bool cpf = plan->streams_colptr();
      uint64_t A = 2;   // edge arenas of the cache: 3 when some block ships its column ids
      for (uint32_t b = 0; b < plan->blocks.size(); ++b) A = std::max<uint64_t>(A, plan->stream_edge_arenas(b));
      Streamer sz(ctx, plan);
      uint64_t ro_all = 0;   // row offsets + (colptr form) column offsets of every block
      for (uint32_t b = 0; b < plan->blocks.size(); ++b)
        ro_all += (uint64_t)(plan->cuts[plan->blocks[b].i + 1] - plan->cuts[plan->blocks[b].i]) + 1 + sz.clen(b);
      const double frac_e = (double)(4 * A * plan->m) / (double)std::max<uint64_t>(all_bytes, 1);
      const uint64_t cap_e = (uint64_t)((double)plan->budget * frac_e) / (4 * A);
      const uint64_t cap_r = (plan->budget - cap_e * 4 * A) / 4;
      std::vector<DevBuf<uint32_t>> cache(A);
      for (auto& c : cache) c.alloc(std::max<uint64_t>(cap_e, 1), ctx);
      DevBuf<uint32_t> cache_rp;
      cache_rp.alloc(std::max<uint64_t>(std::min(cap_r, ro_all), 1), ctx);
      uint32_t* dev_edges[3] = {cache[0].p, A > 1 ? cache[1].p : nullptr, A > 2 ? cache[2].p : nullptr};
      RangeAlloc ea(cap_e), ra(cap_r);
      const uint32_t nb = (uint32_t)plan->blocks.size();
      std::vector<int64_t> at_e(nb, -1), at_r(nb, -1);   // cache placement of resident blocks
      auto rowlen = [&](uint32_t b) {
        const BlockDesc& B = plan->blocks[b];
        return (uint64_t)(plan->cuts[B.i + 1] - plan->cuts[B.i]) + 1;
      };
      // a block's offset region in the cache: row offsets, then its column offsets
      auto rlen = [&](uint32_t b) { return rowlen(b) + sz.clen(b); };
      std::vector<DevBuf<BlockDesc>> tables;   // per-window block tables, alive until the end
      std::vector<std::vector<uint32_t>> uses(nb);   // execution-order task indices using each block
      for (uint32_t t = 0; t < plan->tasks.size(); ++t)
        for (uint32_t b : {plan->tasks[t].ij, plan->tasks[t].ik, plan->tasks[t].jk})
          if (uses[b].empty() || uses[b].back() != t) uses[b].push_back(t);
      Streamer s(ctx, plan);
      const size_t ne = plan->tasks.size();
      std::vector<int64_t> last_reader(nb, -1);   // last window whose kernel read each block
      std::vector<cudaEvent_t> ev_done;           // per window: its kernel finished
      next_epoch(ctx, plan);                       // (first use allocates and clears the flags)
      copies_after_stream();                       // copies start after the flag reset
      size_t t0w = 0;
      while (t0w < ne) {
        // grow the window while its distinct blocks fit the cache
        std::vector<char> inw(nb, 0);
        std::vector<uint32_t> wblocks;
        uint64_t we = 0, wr = 0;
        size_t t1w = t0w;
        for (; t1w < ne; ++t1w) {
          const TaskDesc& T = plan->tasks[t1w];
          uint64_t de = 0, dr = 0;
          std::vector<uint32_t> add;
          for (uint32_t b : {T.ij, T.ik, T.jk})
            if (!inw[b] && std::find(add.begin(), add.end(), b) == add.end()) {
              add.push_back(b);
              de += plan->blocks[b].nnz;
              dr += rlen(b);
            }
          if (we + de > cap_e || wr + dr > cap_r) break;
          for (uint32_t b : add) {
            inw[b] = 1;
            wblocks.push_back(b);
          }
          we += de;
          wr += dr;
        }
        if (t1w == t0w)
          raise(BBTC_ERANGE, "device budget smaller than the three blocks of one task (raise it or p)");
        // Place the window's missing blocks.  Resident blocks stay as long as there is
        // room; when a block does not fit, the resident block outside the window whose
        // next use lies farthest ahead is evicted (Belady: the task order is known).
        auto next_use = [&](uint32_t b) -> size_t {
          auto it = std::lower_bound(uses[b].begin(), uses[b].end(), (uint32_t)t1w);
          return it == uses[b].end() ? SIZE_MAX : *it;
        };
        const int64_t w = (int64_t)ev_done.size();   // this window's index
        auto evict = [&](uint32_t b) {
          ea.release(at_e[b], plan->blocks[b].nnz, last_reader[b]);
          ra.release(at_r[b], rlen(b), last_reader[b]);
          at_e[b] = at_r[b] = -1;
        };
        // Copies of this window may overwrite space only after the kernels that last
        // read it; victims the previous window did not read are preferred, so the
        // copies usually overlap the previous window's kernel.
        int64_t wait_for = -1;
        std::vector<uint32_t> load;
        bool fits = true;
        for (uint32_t b : wblocks) {
          if (at_e[b] >= 0) continue;
          uint64_t oe = 0, orr = 0;
          int64_t te = -1, tr = -1;
          for (;;) {
            const bool ok_e = ea.alloc(plan->blocks[b].nnz, &oe, &te);
            const bool ok_r = ok_e && ra.alloc(rlen(b), &orr, &tr);
            if (ok_r) break;
            if (ok_e) ea.release(oe, plan->blocks[b].nnz, te);
            int64_t victim = -1;
            size_t far = 0;
            bool recent = true;
            for (uint32_t c = 0; c < nb; ++c)
              if (at_e[c] >= 0 && !inw[c]) {
                const size_t nu = next_use(c);
                const bool rc = last_reader[c] >= w - 1;
                if (victim < 0 || (recent && !rc) || (rc == recent && nu > far)) {
                  victim = c;
                  far = nu;
                  recent = rc;
                }
              }
            if (victim < 0) {
              fits = false;
              break;
            }
            evict((uint32_t)victim);
          }
          if (!fits) break;
          at_e[b] = oe;
          at_r[b] = orr;
          wait_for = std::max(wait_for, std::max(te, tr));
          load.push_back(b);
        }
        if (!fits) {   // fragmented: repack the whole window from scratch
          ea = RangeAlloc(cap_e);
          ra = RangeAlloc(cap_r);
          std::fill(at_e.begin(), at_e.end(), -1);
          std::fill(at_r.begin(), at_r.end(), -1);
          load.clear();
          for (uint32_t b : wblocks) {
            uint64_t oe = 0, orr = 0;
            int64_t tg = -1;
            ea.alloc(plan->blocks[b].nnz, &oe, &tg);
            ra.alloc(rlen(b), &orr, &tg);
            at_e[b] = oe;
            at_r[b] = orr;
            load.push_back(b);
          }
          wait_for = w - 1;   // everything moved: after every earlier kernel
        }
        for (uint32_t b : wblocks) last_reader[b] = w;
        // this window's block table: cache offsets of its blocks
        std::vector<BlockDesc> tab = plan->blocks;
        for (uint32_t b : wblocks) {
          tab[b].e0 = (uint64_t)at_e[b];
          tab[b].ro = (uint64_t)at_r[b];
          if (tab[b].co != kNoColptr) tab[b].co = (uint64_t)at_r[b] + rowlen(b);
        }
        tables.emplace_back();
        tables.back().alloc(nb, ctx);
        BBTC_CUDA(cudaMemcpyAsync(tables.back().p, tab.data(), nb * sizeof(BlockDesc), cudaMemcpyHostToDevice,
                                  ctx->stream));
        const uint32_t epoch = next_epoch(ctx, plan);
        s.epoch = epoch;
        if (wait_for >= 0)
          for (auto cs : ctx->copy_streams) BBTC_CUDA(cudaStreamWaitEvent(cs, ev_done[wait_for], 0));
        for (uint32_t b : load) s.copy(b, dev_edges, cache_rp.p, at_e[b], at_r[b], cache_rp.p, at_r[b] + rowlen(b));
        for (uint32_t b : wblocks)
          if (std::find(load.begin(), load.end(), b) == load.end())
            s.flag(b, ctx->copy_streams[s.rr++ % ctx->copy_streams.size()]);
        DevArenas ar;
        ar.cols = dev_edges[0];
        ar.it_u = dev_edges[1];
        ar.it_v = plan->colmajor ? dev_edges[2] : dev_edges[0];   // (kCP: the ccv-shipping blocks)
        ar.rowptr = cache_rp.p;
        ar.blocks = tables.back().p;
        ar.colptr = cpf ? cache_rp.p : nullptr;
        ar.item_col = plan->d_item_col.p;
        count_launch(ctx, plan, rank, world, d_counts.p, plan->item_start[t0w], plan->item_start[t1w],
                     plan->d_ready.p, epoch, &ar);
        ev_done.emplace_back();
        BBTC_CUDA(cudaEventCreateWithFlags(&ev_done.back(), cudaEventDisableTiming));
        BBTC_CUDA(cudaEventRecord(ev_done.back(), ctx->stream));
        t0w = t1w;
      }
      for (auto e : ev_done) cudaEventDestroy(e);   // destroyed events stay valid for queued waits
      // the flags of the last window were written on the copy streams
      for (auto cs : ctx->copy_streams) {
        cudaEvent_t done;
        BBTC_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        BBTC_CUDA(cudaEventRecord(done, cs));
        BBTC_CUDA(cudaStreamWaitEvent(ctx->stream, done, 0));
        cudaEventDestroy(done);
      }
      h2d = s.bytes;
      copies_done();
      BBTC_CUDA(cudaStreamSynchronize(ctx->stream));   // caches and tables die with this scope
    }
    BBTC_CUDA(cudaEventRecord(k1, ctx->stream));
    std::vector<uint64_t> h(nt + 1);
    BBTC_CUDA(cudaMemcpyAsync(h.data(), d_counts.p, (nt + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    BBTC_CUDA(cudaStreamSynchronize(ctx->stream));
    *total = h[nt];
    if (per_task) std::copy(h.begin(), h.begin() + nt, per_task);
    float kms = 0, dms = 0;
    BBTC_CUDA(cudaEventElapsedTime(&kms, k0, k1));
    if (kmid) {
      BBTC_CUDA(cudaEventElapsedTime(&dms, kmid, k1));
      cudaEventDestroy(kmid);
    }
    if (tm) {
      tm->t_total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      tm->t_kernel_ms = kms;
      tm->t_h2d_ms = 0;
      for (auto e : c_end) {
        float ms = 0;
        BBTC_CUDA(cudaEventElapsedTime(&ms, k0, e));
        tm->t_h2d_ms = std::max(tm->t_h2d_ms, (double)ms);
      }
      tm->h2d_bytes = h2d;
      tm->launches = ctx->launches - l0;
      tm->t_dense_ms = dms;
    }
    for (auto e : c_end) cudaEventDestroy(e);
    cudaEventDestroy(k0);
    cudaEventDestroy(k1);
  });
}

}  // extern "C"

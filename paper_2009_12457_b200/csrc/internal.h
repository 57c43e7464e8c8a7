// internal.h — shared internals of libbbtc (host runtime + kernels).  Not installed.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <vector>

#include "bbtc.h"

namespace bbtc {

// ---- error plumbing -----------------------------------------------------------------
void set_error(const std::string& msg);
struct Error {
  bbtc_status code;
  std::string msg;
};
[[noreturn]] void raise(bbtc_status code, const std::string& msg);
#define BBTC_CUDA(call)                                                                        \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      ::bbtc::raise(e_ == cudaErrorMemoryAllocation ? BBTC_ENOMEM : BBTC_ECUDA,                \
                    std::string(#call) + ": " + cudaGetErrorString(e_));                       \
  } while (0)
#define BBTC_STR2_(x) #x
#define BBTC_STR_(x) BBTC_STR2_(x)
bool sync_check();   // BBTC_SYNC_CHECK=1: every launch is followed by a device sync (fault location)
#define BBTC_LAUNCHED(ctx)                                                                     \
  do {                                                                                         \
    cudaError_t e_ = ::bbtc::sync_check() ? cudaDeviceSynchronize() : cudaSuccess;             \
    if (e_ == cudaSuccess) e_ = cudaGetLastError();                                            \
    if (e_ != cudaSuccess)                                                                     \
      ::bbtc::raise(BBTC_ECUDA, std::string("kernel launched at " __FILE__ ":" BBTC_STR_(__LINE__) ": ") + \
                                    cudaGetErrorString(e_));                                   \
    (ctx)->launches++;                                                                         \
  } while (0)

// ---- device buffers ------------------------------------------------------------------
// All device scratch and arenas come from the context's caching allocator
// (ctx_alloc/ctx_free, capi.cpp): freed blocks are kept in size classes and reused
// in stream order by later steps, so repeated runs never go back to the driver.
void* ctx_alloc(bbtc_ctx* ctx, size_t bytes);
void ctx_free(bbtc_ctx* ctx, void* p, size_t bytes);

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  bbtc_ctx* c = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p = o.p; n = o.n; c = o.c;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { reset(); }
  void alloc(size_t count, bbtc_ctx* ctx) {
    reset();
    c = ctx;
    n = count;
    if (count) p = (T*)ctx_alloc(ctx, count * sizeof(T));
  }
  void reset() {
    if (p) ctx_free(c, p, n * sizeof(T));
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// ---- tracing (BBTC_TRACE=1): CUDA events at named points of a phase, printed to
// stderr with per-point device time when the phase ends.  Off by default.
struct Trace {
  cudaStream_t st = nullptr;
  const char* phase = nullptr;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  bool on = false;
  Trace(cudaStream_t s, const char* name);
  void mark(const char* what);
  ~Trace();
};

}  // namespace bbtc

struct bbtc_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::vector<cudaStream_t> copy_streams;
  cudaStream_t aux_stream = nullptr;   // second compute stream (sorts overlapped with streaming)
  uint64_t launches = 0;
  int sm_count = 148;
  void* cursor = nullptr;          // device scratch: work-item cursors of the count kernel
  uint64_t cursor_next = 0;
  uint64_t* task_cycles = nullptr;   // study mode (bbtc_task_times): per-task warp cycles, else NULL
  std::multimap<size_t, void*> cache;   // caching allocator: size class -> free blocks
  size_t cached_bytes = 0;
  size_t cache_limit = 0;
};
constexpr int kCursorSlots = 1024;
constexpr uint32_t kDenseMinS = 8;     // bit-row strides (words): powers of two in [8, 512]
constexpr uint32_t kDenseMaxS = 512;
constexpr uint32_t kDenseBitsDefault = 8192;
constexpr uint32_t kAutoPMax = 256;
constexpr uint32_t kBitmapMaxWords = 1024;   // = the count kernel's per-warp table (kTable)   // largest p the automatic choice tries

struct bbtc_graph {
  bbtc_ctx* ctx = nullptr;
  uint32_t n = 0;
  uint64_t m = 0;
  uint64_t raw = 0;
  uint32_t d_max = 0;
  uint32_t n_nonisolated = 0;
  bbtc::DevBuf<uint32_t> deg_sorted;  // full degrees in rank order (n)
  bbtc::DevBuf<uint32_t> rank;        // rank of each input id (n)
  bbtc::DevBuf<uint64_t> okeys;       // oriented edges (ru << 32 | rw), ru < rw, unsorted (m)
  // §8(e) shards: m counts this rank's edges, m_total the whole graph's (default cuts
  // use 2 m_total); ckeys = the shard's canonical keys (lo << cbw | hi) until ranked.
  uint64_t m_total = 0;
  int cbw = 32;
  uint32_t dplus_max = 0;             // largest out-degree (on first request, graph_dplus_max)
  bool dplus_max_known = false;
  bbtc::DevBuf<uint64_t> ckeys;
};

// One upper-triangular block G_ij in the arena (column-major block order:
// b = j(j+1)/2 + i).
constexpr uint64_t kNoColptr = ~0ull;   // BlockDesc.co of a block streamed with per-edge column ids
struct BlockDesc {
  uint64_t e0;      // first edge (index into cols / rows arenas)
  uint64_t nnz;     // edges
  uint64_t ro;      // first row offset (index into rowptr arena); |V_i|+1 entries
  uint32_t i, j;
  uint64_t co;      // streamed column-major blocks: first of its |V_j|+1 column offsets (colptr arena),
                    // kNoColptr when the block streams its per-edge column ids (nnz <= |V_j|+1)
  uint32_t nc;      // columns |V_j|
  uint32_t pad_;
};

// Task (i,j,k) as the count kernel sees it.
struct TaskDesc {
  uint32_t ij, ik, jk;  // block ids
  uint32_t idx;         // canonical Alg. 4 index
  uint32_t chunk;       // edges of G_ij per work item
  uint32_t pad;         // dense tasks: bit-row stride of V_k in words
  uint32_t bmw;         // words of a bitmap over V_k (power of two >= 4) if it fits a warp's table, else 0
  uint32_t icol;        // first entry of this task's items in item_col (canonical task order)
};

struct bbtc_plan {
  uint32_t p = 0;
  uint32_t clamped = 0;
  uint32_t n = 0;
  uint64_t m = 0;
  std::vector<uint32_t> cuts;
  std::vector<BlockDesc> blocks;
  std::vector<TaskDesc> tasks;        // in execution order
  std::vector<uint64_t> item_start;   // prefix over tasks (execution order) of work items
  uint32_t chunk = 0;                 // edges per work item
  bbtc_plan_info info{};
  // device arenas
  bbtc::DevBuf<uint32_t> cols;        // m: local column id v - cuts[j]
  bbtc::DevBuf<uint32_t> rows;        // m: local row id u - cuts[i]
  bbtc::DevBuf<uint32_t> rowptr;      // sum over blocks of |V_i|+1
  bbtc::DevBuf<uint32_t> ccu, ccv;    // m: column-major iteration order (u, v) of each block
  // probe slots (resident counts): per block the index in the cols arena of its |V_i|
  // 8-word row slots (0 = none); valid while slots_ready (the arena was built with them)
  std::vector<uint32_t> slot_of;
  bbtc::DevBuf<uint32_t> d_slot_of;
  bool slots_ready = false;
  bbtc::DevBuf<uint32_t> d_colptr;    // streamed column-major plans: per block at co, |V_j|+1 local column offsets
  bbtc::DevBuf<uint32_t> d_item_col;  // host plans: the column of every work item's first edge (at TaskDesc.icol)
  bool colmajor = true;               // kernel walks G_ij by column (ccu/ccv) vs by row (rows/cols)
  bbtc::DevBuf<BlockDesc> d_blocks;
  bbtc::DevBuf<TaskDesc> d_tasks;
  bbtc::DevBuf<uint64_t> d_item_start;
  bbtc::DevBuf<uint32_t> d_ready;     // streaming: per-block ready epoch
  uint32_t* h_epochs = nullptr;       // pinned, read-only: h_epochs[e] = e (source of the flag copies)
  uint32_t epoch = 0;
  uint64_t budget = 0;                // out-of-core device budget in bytes (0 = unlimited)
  uint32_t task_group = 0;            // task order: 0 = (k, j, i); h > 0 = groups of h parts (out of core)
  // pinned host copies (bbtc_plan_to_host)
  bool host_blocks = false;
  uint32_t* h_cols = nullptr;
  uint32_t* h_rows = nullptr;
  uint32_t* h_rowptr = nullptr;
  uint32_t* h_ccu = nullptr;
  uint32_t* h_ccv = nullptr;
  // Streamed counts ship each column-major block's column ids as column offsets
  // (|V_j|+1 words per block instead of nnz), copied by the copy engine; the count
  // kernel finds every edge's column in them (no expansion kernel on the copy streams,
  // so nothing the persistent count kernel waits for needs an SM).
  uint32_t* h_colptr = nullptr;       // pinned, per block at co_off[b]: local edge offsets of its columns
  std::vector<uint64_t> rp_zero;      // per block: leading zero entries of its row offsets
  std::vector<uint64_t> co_off;       // per block: first entry in the column-offset arena
  bool resident = true;               // device arenas hold every block
  bbtc_ctx* ctx = nullptr;
  // Dense tasks (Alg. 6's dense map over V_k, chosen per task as isDense,
  // P:695-699): a part k with |V_k| <= dense_bits gets bit rows of stride dense_s[k]
  // words (a power of two) for every block (x,k) a dense task reads; dense tasks run
  // last in execution order, items [dense_item_lo, end), in k_count_dense.
  uint32_t dense_bits = 0;            // largest |V_k| handled densely (0 = off)
  std::vector<uint32_t> dense_s;      // per part: row stride in words (0 = sparse part)
  uint64_t dense_item_lo = 0;         // first work item of the dense tasks (= end if none)
  uint32_t dense_task_lo = 0;         // first dense task in execution order
  bool dense_ready = false;           // bit rows built for the current arenas
  bbtc::DevBuf<uint32_t> dense;       // bit rows of the blocks dense tasks read
  std::vector<uint64_t> dense_off;    // per block: first word of its rows in `dense` (~0 = none)
  std::vector<uint32_t> dense_ids, dense_stride;   // host sources of the build's async copies
  bbtc::DevBuf<uint64_t> d_dense_off;
  // Streamed counts (a6): the sparse tasks in block-unlock order (greedy most work per
  // byte still to copy), so the kernel has work while later blocks are in flight.
  // §8(e) shard plans: the tasks of rank shard_rank only (task_rank[canonical idx]),
  // blocks at their global offsets; 0 = an ordinary plan.
  std::vector<uint32_t> task_rank;
  uint32_t shard_rank = 0, shard_world = 0;
  bool s_ready = false;
  std::vector<TaskDesc> s_tasks;
  std::vector<uint64_t> s_item_start;
  bbtc::DevBuf<TaskDesc> d_s_tasks;
  bbtc::DevBuf<uint64_t> d_s_item_start;

  // The per-edge u32 arenas the count kernel reads (all indexed by edge position):
  // cols (CSR lookups) + the iteration order arrays of the plan's mode.
  struct EdgeArena {
    bbtc::DevBuf<uint32_t>* dev;
    uint32_t** host;
  };
  std::vector<EdgeArena> edge_arenas() {
    if (colmajor) return {{&cols, &h_cols}, {&ccu, &h_ccu}, {&ccv, &h_ccv}};
    return {{&cols, &h_cols}, {&rows, &h_rows}};
  }
  // The per-edge arenas a streamed copy moves: a column-major block's ccv travels as
  // column offsets (colptr), so only cols + ccu cross per edge.
  bool streams_colptr() const { return colmajor && h_colptr != nullptr; }
  // per block: column offsets (fewer words than nnz column ids) or the ids themselves
  bool block_colptr(uint32_t b) const { return streams_colptr() && blocks[b].co != kNoColptr; }
  size_t stream_edge_arenas(uint32_t b) const { return colmajor ? (block_colptr(b) ? 2 : 3) : 2; }
};

namespace bbtc {
// prep.cu
void graph_build(bbtc_ctx* ctx, const uint32_t* src, const uint32_t* dst, uint64_t E, uint32_t n_hint,
                 int mem, bbtc_graph* g, const uint32_t* pairs = nullptr);   // pairs: interleaved src/dst
void graph_csr(bbtc_ctx* ctx, const bbtc_graph* g, uint64_t* row_ptr, uint32_t* col);
uint32_t graph_dplus_max(bbtc_graph* g);
void plan_build(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* user_cuts, uint32_t flags,
                bbtc_plan* plan);
// count.cu
// Where the count kernel finds the blocks: the plan's full arenas, or (out of core)
// cache arenas holding a window's blocks at the offsets of a per-window block table.
struct DevArenas {
  const uint32_t* cols = nullptr;
  const uint32_t* it_u = nullptr;
  const uint32_t* it_v = nullptr;     // per-edge column ids, or NULL with colptr
  const uint32_t* rowptr = nullptr;
  const BlockDesc* blocks = nullptr;
  const uint32_t* colptr = nullptr;   // column offsets (BlockDesc.co / nc) instead of it_v
  const uint32_t* item_col = nullptr; // with colptr: each work item's start column (TaskDesc.icol)
};
void count_zero(bbtc_ctx* ctx, const bbtc_plan* plan, uint64_t* d_counts);
void count_launch(bbtc_ctx* ctx, const bbtc_plan* plan, uint32_t rank, uint32_t world, uint64_t* d_counts,
                  uint64_t item_lo, uint64_t item_hi, const uint32_t* ready, uint32_t epoch,
                  const DevArenas* arenas = nullptr, const TaskDesc* tasks = nullptr,
                  const uint64_t* item_start = nullptr, uint32_t n_exec = 0);
void plan_stats(bbtc_ctx* ctx, bbtc_plan* plan);
uint32_t plan_auto_p(bbtc_ctx* ctx, const bbtc_graph* g, uint64_t budget, uint32_t depth, uint32_t flags);
// Dense tasks: build the bit rows (once per resident plan) and count items
// [item_lo, item_hi) of the dense tasks.
void dense_build(bbtc_ctx* ctx, bbtc_plan* plan);
// Column offsets of every column-major block (host plan preparation) and their
// expansion back to per-edge column ids after a streamed copy (copy stream).
uint64_t colptr_build(bbtc_ctx* ctx, bbtc_plan* plan, bbtc::DevBuf<uint32_t>* out);
// ccv of every block from the device colptr arena (context stream, after the copies).
void colptr_expand_all(bbtc_ctx* ctx, bbtc_plan* plan);
void count_launch_dense(bbtc_ctx* ctx, const bbtc_plan* plan, uint32_t rank, uint32_t world, uint64_t* d_counts,
                        uint64_t item_lo, uint64_t item_hi);
// §8(f)#4 PBD-like cut refinement (prep.cu)
void cuts_refine(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* cuts_in, uint32_t max_evals,
                 uint32_t* cuts_out, uint64_t* m_max_out);
// §8(f)#3 hybrid (cpu.cpp)
uint64_t cpu_count_task(const bbtc_plan* plan, const TaskDesc& T, std::vector<uint64_t>& bits);
std::vector<uint32_t> exec_time_queue(const bbtc_plan* plan);
// §8(e) sharded build (prep.cu)
void shard_canon(bbtc_ctx* ctx, const uint32_t* src, const uint32_t* dst, uint64_t E, int mem, uint32_t n_hint,
                 uint32_t world, uint64_t* out, uint64_t* send_counts, uint32_t* max_id_plus1);
void shard_graph(bbtc_ctx* ctx, const uint64_t* wire, uint64_t cnt, uint32_t n, uint32_t* d_deg, bbtc_graph* g);
void shard_rank(bbtc_ctx* ctx, bbtc_graph* g, const uint32_t* d_deg, uint64_t m_total);
uint32_t shard_blocks_hist(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* user_cuts,
                           uint64_t* d_bnnz, uint32_t* cuts_out);
void shard_by_block(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* cuts, const uint32_t* owner,
                    uint32_t world, uint64_t* out, uint64_t* send_counts);
void plan_build_shard(bbtc_ctx* ctx, const bbtc_graph* like, const uint64_t* okeys, uint64_t cnt, uint32_t p,
                      const uint32_t* cuts, const uint64_t* bnnz, const uint32_t* task_rank, uint32_t rank,
                      uint32_t world, uint32_t flags, bbtc_plan* plan);
void shard_assign(uint32_t p, const uint32_t* cuts, const uint64_t* bnnz, uint32_t world, uint32_t* task_rank,
                  uint32_t* block_rank);
// capi.cpp (host)
uint64_t n_tasks(uint32_t p);
uint64_t task_index(uint32_t p, uint32_t i, uint32_t j, uint32_t k);
inline uint32_t block_id(uint32_t i, uint32_t j) { return j * (j + 1) / 2 + i; }
void plan_tasks(bbtc_plan* plan, uint32_t world);
}  // namespace bbtc

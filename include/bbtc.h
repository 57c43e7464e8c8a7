/* bbtc.h — C-ABI of the B200-native block-based triangle counter (BBTC).
 *
 * Method: Yaşar, Rajamanickam, Berry, Çatalyürek, "A Block-Based Triangle
 * Counting Algorithm on Heterogeneous Environments" (arXiv 2009.12457).
 * Citations "P:n" are lines of that paper's text.
 *
 * Pipeline (every step runs in this library's sm_100a kernels, on the device):
 *   bbtc_graph_from_edges  a1-a2  canonicalise the raw edge list, full
 *                                 degrees, stable degree rank, orient each
 *                                 edge from lower to higher rank
 *   bbtc_plan_create       a3-a5  symmetric rectilinear cut vector,
 *                                 the p(p+1)/2 upper blocks G_ij as block CSR (BCSR,
 *                                 P:460-463, Fig. 2d), the task list of Alg. 4
 *   bbtc_count             a7-a8  for every task t=(i,j,k): for every edge (u,v) in G_ij,
 *                                 |N(G_ik,u) ∩ N(G_jk,v)| (Alg. 5), summed per
 *                                 task into uint64 counters
 *   bbtc_plan_to_host / bbtc_stage / BBTC_COUNT_STREAM   a6  blocks kept in pinned host
 *                                 memory and streamed host->device in task order with
 *                                 copy/compute overlap (Alg. 7 asyncCopy)
 *
 * Conventions (all calls):
 *   - Return bbtc_status: 0 = OK, < 0 = error; bbtc_last_error() gives a message
 *     for the calling thread's last error (valid until its next call).
 *   - Vertex ids are uint32 (id 0xFFFFFFFF is rejected with BBTC_ERANGE); edge
 *     counts and global offsets are uint64; counts are uint64 (Friendster has
 *     4.17e9 triangles).
 *   - "host" pointers are ordinary (or pinned) CPU memory; "device" pointers are
 *     CUDA global memory on the context's device.  Inputs are borrowed for the
 *     duration of the call only (copied or consumed before return, except
 *     *_async calls which consume them in stream order).  Outputs are
 *     caller-allocated; size them from bbtc_graph_stats / bbtc_plan_info.
 *   - Handles (bbtc_ctx, bbtc_graph, bbtc_plan) are library-owned until *_free.
 *     A plan does not reference its graph after bbtc_plan_create returns.
 *   - Threading: a context serialises its work on one CUDA stream; use one
 *     context per host thread.  Graphs and plans are immutable after creation.
 *   - The library never falls back to a CPU path: with no usable CUDA device,
 *     bbtc_ctx_create fails with BBTC_ECUDA.
 */
#ifndef BBTC_H
#define BBTC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BBTC_API __attribute__((visibility("default")))

typedef enum {
  BBTC_OK = 0,
  BBTC_EINVAL = -1,   /* bad argument (NULL handle, invalid cuts, p == 0 with no budget …) */
  BBTC_ENOMEM = -2,   /* device or host allocation failed */
  BBTC_EIO = -3,      /* a file cannot be opened or read (bbtc_edges_read) */
  BBTC_EPARSE = -4,   /* malformed input file; the message carries "path:line: what" */
  BBTC_ERANGE = -5,   /* a size does not fit the documented index widths */
  BBTC_ECUDA = -6,    /* CUDA runtime error (message carries cudaGetErrorString) */
  BBTC_ENCCL = -7,    /* reserved (collectives run in the caller's process group) */
  BBTC_ESTATE = -8    /* call not valid in the object's current state */
} bbtc_status;

typedef struct bbtc_ctx bbtc_ctx;
typedef struct bbtc_graph bbtc_graph;
typedef struct bbtc_plan bbtc_plan;

/* ---------------------------------------------------------------- context */
typedef struct {
  int device;            /* CUDA device ordinal */
  void* stream;          /* cudaStream_t to enqueue on; NULL = library-created stream */
  uint32_t copy_streams; /* streams used for host->device block copies (0 = default 2) */
  uint32_t reserved;
} bbtc_ctx_opts;

/* Creates a context on opts->device (opts may be NULL: device 0, own stream).
 * Errors: BBTC_ECUDA if the device is unavailable. */
BBTC_API bbtc_status bbtc_ctx_create(const bbtc_ctx_opts* opts, bbtc_ctx** out);
BBTC_API void bbtc_ctx_free(bbtc_ctx* ctx);
/* Blocks until all work enqueued on the context has finished. */
BBTC_API bbtc_status bbtc_ctx_sync(bbtc_ctx* ctx);
/* *stream = the cudaStream_t every call on this context enqueues on (the caller's
 * opts->stream, or the library-created one), so a caller can order its own work
 * (e.g. a collective over the counters) after an asynchronous count.
 * Errors: BBTC_EINVAL (NULL). */
BBTC_API bbtc_status bbtc_ctx_stream(const bbtc_ctx* ctx, void** stream);

/* ------------------------------------------------------------------ graph */
#define BBTC_MEM_HOST 0
#define BBTC_MEM_DEVICE 1

typedef struct {
  uint32_t n;               /* vertices: max(n_hint, 1 + largest id in the raw input) */
  uint32_t n_nonisolated;   /* vertices with degree > 0 */
  uint64_t m;               /* unique undirected edges after canonicalisation */
  uint64_t raw_edges;       /* input pairs (incl. self-loops / duplicates) */
  uint32_t d_max;           /* largest full degree d(G,u) in the undirected graph */
  uint32_t dplus_max;       /* largest out-degree d⁺(u) of the degree-oriented graph;
                               computed on the first bbtc_graph_stats_get of a graph (one pass) */
} bbtc_graph_stats;

/* a1-a2.  src/dst: n_edges raw pairs (uint32 each), in host memory (mem ==
 * BBTC_MEM_HOST; copied host->device in chunks overlapped with the first kernel;
 * pinned memory is fastest) or device memory (mem == BBTC_MEM_DEVICE).  The raw
 * list may hold self-loops (dropped), duplicates and both orientations (merged),
 * P:222-228.  The degree rank sorts vertices by (full degree ascending, input id
 * ascending) — the paper leaves ties open; this fixes them.
 * Errors: BBTC_EINVAL (NULL pointers with n_edges > 0), BBTC_ERANGE (an id ==
 * 0xFFFFFFFF, or m >= 2^32-1), BBTC_ENOMEM, BBTC_ECUDA. */
BBTC_API bbtc_status bbtc_graph_from_edges(bbtc_ctx* ctx, const uint32_t* src, const uint32_t* dst,
                                           uint64_t n_edges, uint32_t n_hint, int mem, bbtc_graph** out);
BBTC_API bbtc_status bbtc_graph_stats_get(const bbtc_graph* g, bbtc_graph_stats* s);
/* n and m only (host fields, no device work — for hot loops; m of a §8(e) shard = its
 * own edges). */
BBTC_API bbtc_status bbtc_graph_size(const bbtc_graph* g, uint32_t* n, uint64_t* m);
/* rank_of_input_id: host, n entries. */
BBTC_API bbtc_status bbtc_graph_rank(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t* rank_of_input_id);
/* The oriented graph in rank space as CSR (row_ptr host n+1, col host m); rows
 * sorted ascending.  For tests and inspection (it sorts on demand). */
BBTC_API bbtc_status bbtc_graph_csr(bbtc_ctx* ctx, const bbtc_graph* g, uint64_t* row_ptr, uint32_t* col);
BBTC_API void bbtc_graph_free(bbtc_graph* g);

/* ------------------------------------------------------------- file input */
/* The paper's input is a simple undirected graph given as an edge list (
 * its datasets are Graph Challenge / SNAP edge files).  Formats:
 *   BBTC_FMT_TEXT  one "u v" pair of 0-based decimal ids per line (tab, space or
 *                  comma separated; further fields ignored); blank lines and lines
 *                  starting with '#' or '%' are comments.
 *   BBTC_FMT_MM    MatrixMarket coordinate file ("%%MatrixMarket matrix coordinate
 *                  <field> <symmetry>", '%' comments, "rows cols nnz", then nnz
 *                  1-based "i j [value]" lines; values ignored; n_hint = max(rows, cols)).
 *   BBTC_FMT_BIN   little-endian uint32 pairs src0 dst0 src1 dst1 … (8 bytes per pair).
 * No hygiene is applied: self-loops, duplicates and both orientations are passed on
 * to bbtc_graph_from_edges, which drops / merges them (a1). */
#define BBTC_FMT_TEXT 0
#define BBTC_FMT_MM 1
#define BBTC_FMT_BIN 2

typedef struct {
  uint32_t* src;      /* host, n_edges entries (library-allocated; release with bbtc_edges_free) */
  uint32_t* dst;      /* host, n_edges entries */
  uint64_t n_edges;   /* raw pairs read */
  uint32_t n_hint;    /* vertex count the file declares (MatrixMarket), else 0 */
  uint32_t reserved;
} bbtc_edge_list;

/* Host-only (no device needed): parses `path` into *out.  On error *out is empty.
 * Errors: BBTC_EINVAL (NULL path/out, unknown format), BBTC_EIO (open/read
 * failure), BBTC_EPARSE (malformed line — message "path:line: what"; a binary file
 * whose size is not a multiple of 8), BBTC_ERANGE (an id > 0xFFFFFFFE), BBTC_ENOMEM. */
BBTC_API bbtc_status bbtc_edges_read(const char* path, int format, bbtc_edge_list* out);
BBTC_API void bbtc_edges_free(bbtc_edge_list* e);
/* bbtc_edges_read followed by bbtc_graph_from_edges(…, max(n_hint, file's n_hint),
 * BBTC_MEM_HOST, out).  Errors: those of both calls. */
BBTC_API bbtc_status bbtc_graph_load(bbtc_ctx* ctx, const char* path, int format, uint32_t n_hint,
                                     bbtc_graph** out);

/* Memory-mapped host source (graphs larger than memory are read through
 * memory-mapped files).  bbtc_edges_map maps a BBTC_FMT_BIN file read-only — nothing is
 * copied into library memory; the page cache brings the pages in as the graph build's
 * chunked host->device copies read them, so the raw list need not fit in RAM.
 * pairs = the file's interleaved uint32 pairs (n_edges of them); base/bytes = the
 * mapping (release with bbtc_edges_unmap, after the graph is built).
 * Errors: BBTC_EINVAL (NULL path/out), BBTC_EIO (open/stat/mmap failure), BBTC_EPARSE
 * (size not a multiple of 8). */
typedef struct {
  const uint32_t* pairs;   /* host, 2 * n_edges entries: src0 dst0 src1 dst1 … (read-only mapping) */
  uint64_t n_edges;
  void* base;              /* the mapping (NULL for an empty file) */
  uint64_t bytes;
} bbtc_edge_map;
BBTC_API bbtc_status bbtc_edges_map(const char* path, bbtc_edge_map* out);
BBTC_API void bbtc_edges_unmap(bbtc_edge_map* m);
/* bbtc_graph_from_edges for interleaved pairs (src0 dst0 src1 dst1 …, the binary edge
 * file layout) in host (mem = BBTC_MEM_HOST, pinned, pageable or memory-mapped) or device
 * memory (device pairs 8-byte aligned, else BBTC_EINVAL).  Same result and errors as
 * bbtc_graph_from_edges on the split arrays. */
BBTC_API bbtc_status bbtc_graph_from_pairs(bbtc_ctx* ctx, const uint32_t* pairs, uint64_t n_edges, uint32_t n_hint,
                                           int mem, bbtc_graph** out);
/* bbtc_edges_map + bbtc_graph_from_pairs(…, BBTC_MEM_HOST) + bbtc_edges_unmap: a graph
 * from a binary edge file that is never read whole into RAM.  Errors: those of both. */
BBTC_API bbtc_status bbtc_graph_load_mapped(bbtc_ctx* ctx, const char* path, uint32_t n_hint, bbtc_graph** out);

/* ------------------------------------------------------------------- plan */
typedef struct {
  uint32_t p;               /* parts after clamping (p > n -> n; n == 0 -> 1) */
  uint32_t clamped;         /* 1 if the requested p was clamped */
  uint64_t n_tasks;         /* p(p+1)(p+2)/6 */
  uint64_t n_blocks;        /* p(p+1)/2 upper-triangular blocks */
  uint64_t m;               /* edges (sum of block nnz) */
  uint64_t m_max;           /* largest block nnz */
  double lambda;            /* load imbalance m_max / m_avg, m_avg = 2m/(p(p+1)); 1 when m = 0 */
  uint32_t dmax_blk;        /* d'_max: largest partial degree d(G_ij,u) over all blocks */
  uint32_t host_blocks;     /* 1 if the blocks live in pinned host memory (bbtc_plan_to_host) */
  uint64_t block_bytes;     /* bytes of all blocks (row offsets + cols + row ids) */
  uint64_t max_task_bytes;  /* largest footprint of one task: device bytes of its distinct
                               blocks (row offsets + per-edge arrays) */
  uint64_t b_alg;           /* algorithmic bytes of the count, 0 unless
                               BBTC_PLAN_STATS was passed */
  uint64_t visits;          /* edge visits summed over tasks, i.e. sum_t nnz(G_ij); ditto */
  uint64_t work_items;      /* work items the count kernel schedules */
  uint64_t sum_a;           /* Σ_t Σ_(u,v)∈G_ij d(G_ik,u) (BBTC_PLAN_STATS) */
  uint64_t sum_b;           /* Σ_t Σ_(u,v)∈G_ij d(G_jk,v) (BBTC_PLAN_STATS) */
  uint32_t dense_tasks;     /* tasks counted through bit rows over V_k (isDense) */
  uint32_t dense_bits;      /* largest |V_k| a dense task may have (0 = dense path off) */
  uint64_t dense_bytes;     /* device bytes of the bit rows (0 until the first resident count) */
  uint64_t stream_bytes;    /* host->device bytes that bring every block to the device once
                               (bbtc_plan_to_host plans: column-major blocks cross PCIe with
                               column offsets instead of per-edge column ids); else 0 */
  uint64_t list_read_bytes; /* compulsory reads of the list kernel: device bytes of the distinct
                               blocks the sparse (list-kernel) tasks read */
  uint64_t dense_edge_bytes;/* compulsory reads of the bit-row kernel besides the bit rows
                               (dense_bytes): the per-edge iteration arrays of the distinct G_ij
                               blocks the dense tasks walk */
  uint64_t slot_bytes;      /* device bytes of the probe slots (8 words per row of each probe
                               block with many short rows: length, CSR offset, first 6 ids),
                               read by resident counts instead of the row offsets; 0 = none */
} bbtc_plan_info;

#define BBTC_PLAN_STATS 1u     /* compute b_alg / visits / dmax_blk (one extra device pass) */
#define BBTC_PLAN_ROWMAJOR 2u  /* walk G_ij row by row (stage N(G_ik,u), gather N(G_jk,v)) instead of
                                  the default column order (stage N(G_jk,v), gather N(G_ik,u)) */
#define BBTC_PLAN_SPARSE 4u    /* no dense tasks: every task through the list kernel.  By default a
                                  task whose V_k has at most BBTC_DENSE_BITS (env, default 2048)
                                  vertices is counted on bit rows over V_k (Alg. 6's dense map,
                                  P:552-572, chosen per task as isDense) while its
                                  blocks are device-resident; same counts either way */

/* a3-a5.  p: requested parts (>= 1; clamped to n).  cuts: NULL for the default
 * rule (R5: full-degree prefix rule) or a host array of p+1 entries
 * with cuts[0] = 0, cuts[p] = n, non-decreasing (empty parts allowed).
 * When cuts is given, p must equal its length - 1 and is not clamped.
 * Block (i,j), i <= j, holds the edges (u,v) with u in V_i, v in V_j
 * as BCSR: row offsets uint32[|V_i|+1] over local row ids u - cuts[i], column ids
 * uint32 v - cuts[j] (rows ascending; the columns inside a row are in no particular
 * order), plus the local row id of every edge.
 * Errors: BBTC_EINVAL (p == 0, bad cuts), BBTC_ERANGE (2*ceil(log2 n) +
 * ceil(log2 p) > 64 bits of sort key), BBTC_ENOMEM, BBTC_ECUDA. */
BBTC_API bbtc_status bbtc_plan_create(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* cuts,
                                      uint32_t flags, bbtc_plan** out);
/* a3, automatic p (p is chosen so that "three subgraphs can fit into memory
 * of the computing devices"): *p = a p in 1 … min(n, 256) such that, under
 * the default cut rule, the largest task footprint — the device bytes of the task's
 * distinct blocks (row offsets + per-edge arrays, as bbtc_plan_info.max_task_bytes
 * counts them for the given flags) — times `depth` (tasks in flight at once; 0 = 1)
 * is at most budget_bytes, searched by doubling (1, 2, 4, … until one fits) and then a
 * linear scan of (hi/2, hi): the footprint is not monotone in p (the cuts move with
 * p), so a smaller fitting p below hi/2 is not searched for.  One pass over the edges
 * per candidate p; no blocks are built.
 * Use the result with bbtc_plan_create and, for a budget below the plan's bytes,
 * bbtc_plan_to_host + bbtc_plan_set_budget.
 * Errors: BBTC_EINVAL (NULL, budget 0), BBTC_ERANGE (no p <= min(n, 256) fits). */
BBTC_API bbtc_status bbtc_plan_auto_p(bbtc_ctx* ctx, const bbtc_graph* g, uint64_t budget_bytes, uint32_t depth,
                                      uint32_t flags, uint32_t* p);
BBTC_API bbtc_status bbtc_plan_info_get(const bbtc_plan* plan, bbtc_plan_info* info);
/* cuts: host, p+1 entries. */
BBTC_API bbtc_status bbtc_plan_cuts(const bbtc_plan* plan, uint32_t* cuts);
/* Copies block (i,j) to host: row_ptr (|V_i|+1), col (nnz), row (nnz); any may
 * be NULL.  *nnz receives the block's edge count.  Errors: BBTC_EINVAL (i > j). */
BBTC_API bbtc_status bbtc_plan_block(bbtc_ctx* ctx, const bbtc_plan* plan, uint32_t i, uint32_t j,
                                     uint32_t* row_ptr, uint32_t* col, uint32_t* row, uint64_t* nnz);
/* a6: moves the blocks into pinned host memory and releases their device copy
 * (the out-of-core form of the plan).  bbtc_count then streams them. */
BBTC_API bbtc_status bbtc_plan_to_host(bbtc_ctx* ctx, bbtc_plan* plan);
/* Out-of-core mode ("three subgraphs can fit into memory of the computing
 * devices"): a host-resident plan counted by bbtc_count keeps at most `bytes` of
 * blocks on the device.  Tasks are processed in execution order in windows whose
 * blocks fit; blocks still needed stay resident, others are evicted, missing ones
 * are streamed in.  0 = no limit (every block copied once).  Errors: BBTC_EINVAL;
 * bbtc_count fails with BBTC_ERANGE if one task's three blocks exceed the budget. */
BBTC_API bbtc_status bbtc_plan_set_budget(bbtc_plan* plan, uint64_t bytes);
BBTC_API void bbtc_plan_free(bbtc_plan* plan);

/* Task numbering (Alg. 4): tasks i <= j <= k in loop order.
 * idx(i,j,k) = [C(p+2,3) - C(p-i+2,3)] + [C(p-i+1,2) - C(p-j+1,2)] + (k-j). */
BBTC_API uint64_t bbtc_n_tasks(uint32_t p);
BBTC_API bbtc_status bbtc_task_index(uint32_t p, uint32_t i, uint32_t j, uint32_t k, uint64_t* idx);
BBTC_API bbtc_status bbtc_task_ijk(uint32_t p, uint64_t idx, uint32_t* i, uint32_t* j, uint32_t* k);

/* ------------------------------------------------------------------ count */
typedef struct {
  double t_total_ms;   /* host wall time of the call */
  double t_h2d_ms;     /* time the copy streams were busy (streamed plans) */
  double t_kernel_ms;  /* device time of the count kernel(s) (CUDA events) */
  uint64_t h2d_bytes;  /* block bytes copied host->device by this call */
  uint64_t launches;   /* kernels launched by this call */
  double t_dense_ms;   /* device time of the bit-row kernel (dense tasks) inside t_kernel_ms */
} bbtc_timing;

#define BBTC_COUNT_DEFAULT 0u

/* a7-a8, asynchronous.  Enqueues the count of this rank's share of the work on
 * the context stream and returns.  d_counts: DEVICE uint64[n_tasks + 1]; it is
 * zeroed, then d_counts[t] receives the triangles of task t (Alg. 4 order) found
 * by this rank and d_counts[n_tasks] their sum.  rank/world split the work
 * items statically (rank r takes items r, r+world, … in the plan's balanced
 * order); summing d_counts over ranks (one all-reduce) gives the full result.
 * world = 1, rank = 0 counts everything.  Requires device-resident blocks
 * (plans made by bbtc_plan_create, or bbtc_stage after bbtc_plan_to_host).
 * Errors: BBTC_EINVAL, BBTC_ESTATE (blocks not resident), BBTC_ECUDA. */
BBTC_API bbtc_status bbtc_count_async(bbtc_ctx* ctx, const bbtc_plan* plan, uint32_t rank, uint32_t world,
                                      uint64_t* d_counts);

/* a6-a8, synchronous.  Like bbtc_count_async but returns results in HOST
 * memory: *total and (if per_task != NULL) per_task[n_tasks].  Blocks that are
 * in pinned host memory and not resident are streamed host->device on the copy
 * streams, overlapped with ONE count kernel whose warps wait on per-block ready
 * flags (Alg. 7's asyncCopy/isCopied).  Tasks and copies follow a
 * tail-aware order (blocks placed last-first by least remaining work per byte), so a
 * rank's share of work items differs from the resident mode's (sums over ranks do
 * not).  Column-major blocks cross PCIe with per-block column offsets instead of
 * per-edge column ids, and without the leading zero run of their row offsets
 * (bbtc_plan_info.stream_bytes).  Afterwards the blocks are resident.  t may be NULL;
 * t->t_h2d_ms is the time until the last copy landed. */
BBTC_API bbtc_status bbtc_count(bbtc_ctx* ctx, const bbtc_plan* plan, uint32_t rank, uint32_t world,
                                uint32_t flags, uint64_t* total, uint64_t* per_task, bbtc_timing* t);

/* §8(f)#4 study support.  bbtc_plan_block_nnz: nnz of every block, HOST uint64[p(p+1)/2]
 * (block order b = j(j+1)/2 + i).  bbtc_task_times: the warp time every task took
 * inside one ordinary resident count (HOST double[n_tasks], canonical order, warp-
 * milliseconds = Σ over the task's work items of the item's clock64() span / SM clock),
 * for ranking workload estimators against measured task work.  Needs
 * resident blocks.  A study tool: the instrumented count is otherwise the real one. */
BBTC_API bbtc_status bbtc_plan_block_nnz(const bbtc_plan* plan, uint64_t* nnz);
BBTC_API bbtc_status bbtc_task_times(bbtc_ctx* ctx, const bbtc_plan* plan, double* ms);
/* A PBD-like refinement of a cut vector (P:459-460 cite PBD without describing it; SPEC's
 * reading: move interior cuts while the largest block m_max strictly decreases): pattern
 * search over each interior cut with steps halving from |V_i|/2 to 1, every candidate
 * evaluated exactly by one pass over the oriented edges (block histogram); at most
 * max_evals evaluations.  cuts_in: HOST uint32[p+1] (NULL = the default rule);
 * cuts_out: HOST uint32[p+1]; *m_max_out: the largest block nnz of cuts_out.  The
 * result is a valid symmetric partition whatever it converges to. */
BBTC_API bbtc_status bbtc_cuts_refine(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* cuts_in,
                                      uint32_t max_evals, uint32_t* cuts_out, uint64_t* m_max_out);

/* §8(f)#3 hybrid CPU+GPU count (Alg. 8, §7.7).  The sparse tasks are
 * queued by the paper's ExecTime estimate nnz(G_ij)·max(δ(G_ik), δ(G_jk)), heaviest
 * first.  The GPU (the calling thread drives it) claims the front of the
 * queue up to the cut-off, then further chunks while tasks remain (one list-kernel
 * launch per claim, over a task table of its own); cpu_threads host threads claim single
 * tasks from the back and never pass the cut-off, each counting its task
 * with Alg. 6's dense map over V_k (a bitmap) on the plan's pinned host
 * arenas.  Dense (bit-row) tasks stay on the GPU.  Requires a plan with host arenas
 * (bbtc_plan_to_host) that is also device-resident (bbtc_stage): the split is measured
 * "excl. H2D".  Results as bbtc_count (rank 0 of 1). */
typedef struct {
  uint32_t cpu_threads;   /* host threads (0 = hardware concurrency) */
  uint32_t gpu_chunk;     /* tasks per GPU claim past the cut-off (0 = 1/8 of what is left) */
  double cutoff;          /* GPU-reserved front of the queue, fraction of the sparse tasks
                             (paper default 0.5; 1 = GPU only, 0 = no reservation) */
} bbtc_hybrid_opts;
typedef struct {
  uint64_t cpu_tasks, gpu_tasks;   /* sparse tasks counted by each side */
  uint64_t gpu_launches;           /* list-kernel launches (claims) */
  uint64_t cpu_triangles;          /* triangles found by the CPU threads */
  double t_cpu_ms;                 /* wall time until the last CPU thread finished */
  double t_gpu_ms;                 /* wall time until the GPU's last claim finished */
} bbtc_hybrid_stats;
BBTC_API bbtc_status bbtc_count_hybrid(bbtc_ctx* ctx, const bbtc_plan* plan, const bbtc_hybrid_opts* opts,
                                       uint64_t* total, uint64_t* per_task, bbtc_timing* t,
                                       bbtc_hybrid_stats* stats);

/* a6: makes every block of a host-resident plan resident on the context's
 * device (so a following count runs "excl. H2D").  No-op for device plans. */
BBTC_API bbtc_status bbtc_stage(bbtc_ctx* ctx, bbtc_plan* plan);
/* Drops the device copies made by bbtc_stage / streaming counts. */
BBTC_API bbtc_status bbtc_unstage(bbtc_ctx* ctx, bbtc_plan* plan);
/* §8(e) "each block H2D once, by its owner": copies blocks ids[0..n) of a host plan
 * (bbtc_plan_to_host) to the device in their device form (synchronous).  The other
 * blocks a rank's tasks read arrive from their owners over NVLink (bbtc_plan_block_ptrs
 * + the caller's transfer); the caller then passes BBTC_STAGE_RESIDENT (with n = 0 or
 * the last ids) to declare every block its tasks read present, and counts as resident.
 * Errors: BBTC_ESTATE (not a host plan), BBTC_EINVAL (bad id). */
#define BBTC_STAGE_RESIDENT 1u
BBTC_API bbtc_status bbtc_stage_blocks(bbtc_ctx* ctx, bbtc_plan* plan, const uint32_t* ids, uint32_t n,
                                       uint32_t flags);

/* ------------------------------------------- multi-GPU sharded build (§8(e))
 * One process per GPU, rank r of `world`, each starting from its own share of the
 * raw edges.  The caller moves buffers between ranks (torch.distributed over NCCL:
 * two all-to-alls, two all-reduces and point-to-point block transfers) between these
 * per-rank device steps; see paper_2009_12457_b200/dist.py and DESIGN.md §9.  Tasks
 * are independent and the result is the sum of per-task counts; the
 * paper distributes tasks over GPUs in a ready queue — here a
 * deterministic LPT with block affinity (bbtc_shard_assign) fixes every rank's tasks.
 * All device arrays are on the context's device; all calls are stream-ordered on it
 * and return after the host-visible outputs are written.
 *
 * a1 sharded: canonicalise this rank's n_edges raw pairs (mem: BBTC_MEM_HOST = the
 * share crosses PCIe here, or BBTC_MEM_DEVICE), drop self-loops, sort, unique, and
 * group the unique keys by destination rank (a hash of the smaller id, so every copy
 * of an edge from any rank meets at one rank).  d_keys_out: DEVICE uint64[n_edges],
 * receives send_counts[0] keys for rank 0, then rank 1's, … as (min << 32 | max).
 * send_counts: HOST uint64[world].  *max_id_plus1: 1 + the largest raw id (0 if none).
 * n_hint: a lower bound for n (narrows sort keys; any value is correct). */
BBTC_API bbtc_status bbtc_shard_canon(bbtc_ctx* ctx, const uint32_t* src, const uint32_t* dst, uint64_t n_edges,
                                      int mem, uint32_t n_hint, uint32_t world, uint64_t* d_keys_out,
                                      uint64_t* send_counts, uint32_t* max_id_plus1);
/* a1-a2 sharded: the keys this rank received (every copy of its edges, from all ranks)
 * are sorted and de-duplicated into a graph shard; d_deg: DEVICE uint32[n] receives
 * this shard's partial full degrees (sum them over ranks).  n = the global vertex
 * count (max of n_hint and every rank's max_id_plus1). */
BBTC_API bbtc_status bbtc_shard_graph(bbtc_ctx* ctx, const uint64_t* d_keys, uint64_t n_keys, uint32_t n,
                                      uint32_t* d_deg, bbtc_graph** out);
/* a2 sharded: with the global degrees d_deg (DEVICE uint32[n], summed over ranks) and
 * the global edge count, rank every vertex by (degree, id) (R2) and orient
 * the shard's edges.  Errors: BBTC_ESTATE if g is not an unranked shard. */
BBTC_API bbtc_status bbtc_shard_rank(bbtc_ctx* ctx, bbtc_graph* g, const uint32_t* d_deg, uint64_t m_total);
/* a3 sharded: cuts (user cuts, or the default rule over the global degrees) and this
 * shard's edge count of every block: d_block_nnz DEVICE uint64[p(p+1)/2] (block order
 * b = j(j+1)/2 + i; sum over ranks), cuts_out HOST uint32[p+1], *p_eff = p after
 * clamping (p > n -> n). */
BBTC_API bbtc_status bbtc_shard_block_sizes(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* cuts,
                                            uint64_t* d_block_nnz, uint32_t* cuts_out, uint32_t* p_eff);
/* a5 + the multi-GPU scheduler (host only, deterministic): from the global block sizes,
 * task_rank[idx] (HOST uint32[n_tasks], Alg. 4 order) = the rank counting task idx
 * (LPT on the per-edge cost estimate with block affinity), and
 * block_rank[b] (HOST uint32[p(p+1)/2]) = the rank that builds block b and forwards it
 * to every other rank whose tasks read it. */
BBTC_API bbtc_status bbtc_shard_assign(uint32_t p, const uint32_t* cuts, const uint64_t* block_nnz, uint32_t world,
                                       uint32_t* task_rank, uint32_t* block_rank);
/* a4 sharded, step 1: this shard's oriented edges grouped by the owner of their block:
 * d_out DEVICE uint64[m of the shard] (ru << 32 | rw), send_counts HOST uint64[world]. */
BBTC_API bbtc_status bbtc_shard_by_block(bbtc_ctx* ctx, const bbtc_graph* g, uint32_t p, const uint32_t* cuts,
                                         const uint32_t* block_rank, uint32_t world, uint64_t* d_out,
                                         uint64_t* send_counts);
/* a4 sharded, step 2: rank `rank`'s plan in the GLOBAL block layout (block_nnz, the
 * summed sizes): the blocks it owns are built from d_okeys (every edge of those blocks,
 * as received), the others are allocated and filled by the caller through
 * bbtc_plan_block_ptrs.  The plan holds only the tasks with task_rank[idx] == rank;
 * bbtc_count_async(ctx, plan, rank, world, …) counts them.  `like` = this rank's
 * ranked shard (vertex count, isolated prefix).  Errors: BBTC_EINVAL when a block
 * arrives incomplete. */
BBTC_API bbtc_status bbtc_plan_create_shard(bbtc_ctx* ctx, const bbtc_graph* like, const uint64_t* d_okeys,
                                            uint64_t n_okeys, uint32_t p, const uint32_t* cuts,
                                            const uint64_t* block_nnz, const uint32_t* task_rank, uint32_t rank,
                                            uint32_t world, uint32_t flags, bbtc_plan** out);
/* Device spans of block b of a resident plan: its n_edge_arrays per-edge arrays (cols,
 * then the walk order: ccu, ccv for column-major plans, rows for row-major) of nnz
 * words each, and its rowptr_len block-local row offsets.  For moving blocks between
 * ranks (the spans are the plan's own memory; valid while the plan lives). */
typedef struct {
  uint32_t* edge[3];
  uint32_t n_edge_arrays;
  uint32_t reserved;
  uint64_t nnz;
  uint32_t* rowptr;
  uint64_t rowptr_len;
} bbtc_block_ptrs;
BBTC_API bbtc_status bbtc_plan_block_ptrs(const bbtc_plan* plan, uint32_t b, bbtc_block_ptrs* out);

/* Number of kernels this library launched on the context since creation. */
BBTC_API uint64_t bbtc_ctx_launches(const bbtc_ctx* ctx);
BBTC_API const char* bbtc_last_error(void);
BBTC_API const char* bbtc_version(void);

#ifdef __cplusplus
}
#endif
#endif

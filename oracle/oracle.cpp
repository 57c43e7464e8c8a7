// oracle.cpp — plain, slow, obviously-correct CPU oracle for BBTC triangle counts.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  It shares no code,
// header, table or constant with the CUDA path (paper_2009_12457_b200/) and
// neither side includes the other.
//
// What it computes (PAPER.md = P):
//   * T = number of unordered vertex triples that are mutually adjacent
//     ("Triangle Counting Problem").
//   * Per-task counts: with r = the degree rank of a vertex and
//     part(x) = the i with cuts[i] <= r(x) < cuts[i+1], the count of
//     task (i,j,k) is the number of triangles whose rank-sorted vertices u<v<w
//     have (part u, part v, part w) = (i,j,k).  By P:468-498 this is exactly what
//     Alg. 5 (BB-TC-LIST) computes for task {G_ij, G_jk, G_ik}.
//   * Per-vertex participations (each triangle adds 1 to each of its 3 vertices).
// How: the node iterator TC-LIST (Alg. 2) over the merge INTERSECT of
// Alg. 1 with its typo A[b]=B[b] read as A[a]=B[b] (R1),
// binning every common neighbour w of an oriented edge (u,v) into its task.
//
// Readings of the paper: canonicalisation drops self-loops
// and duplicates and merges both orientations (R4); the degree used for ordering is
// the full undirected degree (R3) and ties go to the smaller input id (R2); the
// default partition is the prefix rule of SURVEY.md §8(c) (R5); tasks are reported
// in Alg. 4 order (R7); n = max(n_hint, 1 + largest raw id) (R21).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <parallel/algorithm>
#include <string>
#include <vector>
#include <omp.h>

namespace {

thread_local std::string g_err;

struct Graph {
  uint32_t n = 0;
  uint64_t m = 0;
  std::vector<uint32_t> deg;          // full undirected degree, by input id
  std::vector<uint32_t> rank;         // rank[input id]
  std::vector<uint32_t> order;        // order[rank] = input id
  std::vector<uint64_t> row;          // oriented CSR over ranks: N+(u) = col[row[u]..row[u+1])
  std::vector<uint32_t> col;
};

int nthreads(int t) { return t > 0 ? t : omp_get_max_threads(); }

// Step 1: simple undirected edge set as sorted unique (min,max) keys.
std::vector<uint64_t> canonical_keys(const uint32_t* src, const uint32_t* dst, uint64_t E,
                                     uint32_t* max_id_plus1, int threads) {
  std::vector<uint64_t> keys;
  keys.reserve(E);
  uint64_t top = 0;
  for (uint64_t e = 0; e < E; ++e) {
    uint32_t a = src[e], b = dst[e];
    top = std::max<uint64_t>(top, (uint64_t)std::max(a, b) + 1);
    if (a == b) continue;                       // self-loop: not an edge of a simple graph
    uint32_t lo = std::min(a, b), hi = std::max(a, b);
    keys.push_back(((uint64_t)lo << 32) | hi);
  }
  omp_set_num_threads(nthreads(threads));
  __gnu_parallel::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  *max_id_plus1 = (uint32_t)std::min<uint64_t>(top, 0xFFFFFFFFull);
  return keys;
}

// Alg. 1 INTERSECT, corrected: count |A ∩ B| of two sorted lists.
// `emit` is called for every common element (so the caller can bin it).
template <class F>
uint64_t intersect(const uint32_t* A, uint64_t na, const uint32_t* B, uint64_t nb, F emit) {
  uint64_t a = 0, b = 0, c = 0;
  while (a < na && b < nb) {
    if (A[a] == B[b]) { emit(A[a]); ++c; ++a; ++b; }
    else if (A[a] < B[b]) ++a;
    else ++b;
  }
  return c;
}

// Alg. 4 BB-TASK: enumerate i<=j<=k in loop order; the position in
// this enumeration is the task's canonical index.  Recorded as first[i*p+j] =
// index of (i,j,j); within fixed (i,j) the k loop runs j..p-1, so
// index(i,j,k) = first[i*p+j] + (k-j).
std::vector<uint64_t> task_table(uint32_t p) {
  std::vector<uint64_t> first((size_t)p * p, ~0ull);
  uint64_t t = 0;
  for (uint32_t i = 0; i < p; ++i)
    for (uint32_t j = i; j < p; ++j)
      for (uint32_t k = j; k < p; ++k) {
        if (k == j) first[(size_t)i * p + j] = t;
        ++t;
      }
  return first;
}

}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

// Steps 1-4: canonicalise, full degrees, stable degree rank, orient into a CSR of
// out-lists N+(u) = {v : (u,v) in E, u < v} in rank space.
void* oracle_build(const uint32_t* src, const uint32_t* dst, uint64_t E, uint32_t n_hint, int threads) {
  Graph* g = new Graph();
  uint32_t top = 0;
  std::vector<uint64_t> keys = canonical_keys(src, dst, E, &top, threads);
  g->n = std::max(n_hint, top);
  g->m = keys.size();
  g->deg.assign(g->n, 0);
  for (uint64_t k : keys) { g->deg[k >> 32]++; g->deg[k & 0xFFFFFFFFu]++; }
  // Rank: vertices sorted by (degree ascending, input id ascending).
  g->order.resize(g->n);
  for (uint32_t x = 0; x < g->n; ++x) g->order[x] = x;
  std::stable_sort(g->order.begin(), g->order.end(),
                   [&](uint32_t a, uint32_t b) { return g->deg[a] < g->deg[b]; });
  g->rank.resize(g->n);
  for (uint32_t r = 0; r < g->n; ++r) g->rank[g->order[r]] = r;
  // Orient: each edge (a,b) becomes (min rank, max rank); out-lists sorted ascending.
  for (uint64_t& k : keys) {
    uint32_t ra = g->rank[k >> 32], rb = g->rank[k & 0xFFFFFFFFu];
    k = ((uint64_t)std::min(ra, rb) << 32) | std::max(ra, rb);
  }
  __gnu_parallel::sort(keys.begin(), keys.end());
  g->row.assign((uint64_t)g->n + 1, 0);
  g->col.resize(g->m);
  for (uint64_t e = 0; e < g->m; ++e) {
    g->row[(keys[e] >> 32) + 1]++;
    g->col[e] = (uint32_t)keys[e];
  }
  for (uint32_t u = 0; u < g->n; ++u) g->row[u + 1] += g->row[u];
  return g;
}

void oracle_free(void* h) { delete (Graph*)h; }
uint32_t oracle_n(void* h) { return ((Graph*)h)->n; }
uint64_t oracle_m(void* h) { return ((Graph*)h)->m; }

void oracle_rank(void* h, uint32_t* rank_of_input_id) {
  Graph* g = (Graph*)h;
  std::copy(g->rank.begin(), g->rank.end(), rank_of_input_id);
}

void oracle_degrees(void* h, uint32_t* deg_by_input_id) {
  Graph* g = (Graph*)h;
  std::copy(g->deg.begin(), g->deg.end(), deg_by_input_id);
}

// The oriented CSR in rank space: row (n+1 entries), col (m entries).
void oracle_csr(void* h, uint64_t* row, uint32_t* col) {
  Graph* g = (Graph*)h;
  std::copy(g->row.begin(), g->row.end(), row);
  std::copy(g->col.begin(), g->col.end(), col);
}

// p clamping (SURVEY.md §8(b) "p > n: clamp to n"; n = 0 -> p = 1).
uint32_t oracle_effective_p(void* h, uint32_t p) {
  Graph* g = (Graph*)h;
  if (p == 0) return 0;
  if (g->n == 0) return 1;
  return p > g->n ? g->n : p;
}

// Default symmetric cut rule (SURVEY.md §8(c) "Default cut rule"; the paper's PBD
// is only cited, and any valid symmetric partition is allowed,
// P:455): with w[r] the full degree of the rank-r vertex and P the prefix sums
// (P[0]=0, P[n]=2m), cuts[i] = max(cuts[i-1], min{ r : P[r] >= ceil(i*2m/p) }).
// Returns the effective p (0 on error).  cuts: p_eff+1 entries.
uint32_t oracle_default_cuts(void* h, uint32_t p, uint32_t* cuts) {
  Graph* g = (Graph*)h;
  uint32_t pe = oracle_effective_p(h, p);
  if (pe == 0) { g_err = "p must be >= 1"; return 0; }
  std::vector<uint64_t> P((uint64_t)g->n + 1, 0);
  for (uint32_t r = 0; r < g->n; ++r) P[r + 1] = P[r] + g->deg[g->order[r]];
  const uint64_t two_m = 2 * g->m;
  cuts[0] = 0;
  for (uint32_t i = 1; i < pe; ++i) {
    uint64_t target = ((uint64_t)i * two_m + pe - 1) / pe;
    uint32_t r = 0;
    while (P[r] < target) ++r;                  // linear scan: min r with P[r] >= target
    cuts[i] = std::max(cuts[i - 1], r);
  }
  cuts[pe] = g->n;
  return pe;
}

// Steps 5-7: count.  cuts (p+1 entries, validated) define the parts.  Outputs:
// *total; per_task (NULL or p(p+1)(p+2)/6 entries, Alg. 4 order); per_vertex (NULL
// or n entries, indexed by INPUT id).  Returns 0, or -1 with oracle_last_error().
int oracle_count(void* h, uint32_t p, const uint32_t* cuts, int threads, uint64_t* total,
                 uint64_t* per_task, uint64_t* per_vertex) {
  Graph* g = (Graph*)h;
  if (p == 0 || p > 1024) { g_err = "oracle supports 1 <= p <= 1024"; return -1; }
  if (cuts[0] != 0 || cuts[p] != g->n) { g_err = "cuts must start at 0 and end at n"; return -1; }
  for (uint32_t i = 0; i < p; ++i)
    if (cuts[i] > cuts[i + 1]) { g_err = "cuts must be non-decreasing"; return -1; }
  std::vector<uint32_t> part(g->n);
  for (uint32_t i = 0; i < p; ++i)
    for (uint32_t r = cuts[i]; r < cuts[i + 1]; ++r) part[r] = i;
  const std::vector<uint64_t> first = task_table(p);
  const uint64_t ntask = (uint64_t)p * (p + 1) * (p + 2) / 6;
  const int nt = nthreads(threads);
  std::vector<std::vector<uint64_t>> local(nt, std::vector<uint64_t>(ntask, 0));
  std::vector<std::atomic<uint64_t>> pv(per_vertex ? g->n : 0);
  for (auto& x : pv) x.store(0, std::memory_order_relaxed);
  uint64_t tot = 0;
#pragma omp parallel num_threads(nt) reduction(+ : tot)
  {
    std::vector<uint64_t>& mine = local[omp_get_thread_num()];
#pragma omp for schedule(dynamic, 256)
    for (int64_t uu = 0; uu < (int64_t)g->n; ++uu) {
      const uint32_t u = (uint32_t)uu;
      const uint32_t* Nu = g->col.data() + g->row[u];
      const uint64_t du = g->row[u + 1] - g->row[u];
      for (uint64_t x = 0; x < du; ++x) {               // Alg. 2: for v in N(G,u)
        const uint32_t v = Nu[x];
        const uint32_t* Nv = g->col.data() + g->row[v];
        const uint64_t dv = g->row[v + 1] - g->row[v];
        tot += intersect(Nu, du, Nv, dv, [&](uint32_t w) {
          mine[first[(size_t)part[u] * p + part[v]] + (part[w] - part[v])]++;
          if (per_vertex) {
            pv[u].fetch_add(1, std::memory_order_relaxed);
            pv[v].fetch_add(1, std::memory_order_relaxed);
            pv[w].fetch_add(1, std::memory_order_relaxed);
          }
        });
      }
    }
  }
  std::vector<uint64_t> sum(ntask, 0);
  for (auto& l : local)
    for (uint64_t t = 0; t < ntask; ++t) sum[t] += l[t];
  uint64_t s = 0;
  for (uint64_t t = 0; t < ntask; ++t) s += sum[t];
  if (s != tot) { g_err = "internal: sum of per-task counts != total"; return -1; }
  if (per_vertex) {
    uint64_t sv = 0;
    for (uint32_t x = 0; x < g->n; ++x) {
      per_vertex[x] = pv[g->rank[x]].load(std::memory_order_relaxed);
      sv += per_vertex[x];
    }
    if (sv != 3 * tot) { g_err = "internal: sum of per-vertex counts != 3T"; return -1; }
  }
  *total = tot;
  if (per_task) std::copy(sum.begin(), sum.end(), per_task);
  return 0;
}

// Single task (i,j,k) by the definition: triangles u<v<w (ranks) with
// part(u)=i, part(v)=j, part(w)=k.  Used for sampled checks at full size.
// Node iterator restricted to u in V_i, v in N+(u) ∩ V_j, w in N+(u) ∩ N+(v) ∩ V_k.
int oracle_count_task(void* h, uint32_t p, const uint32_t* cuts, uint32_t i, uint32_t j, uint32_t k,
                      int threads, uint64_t* count) {
  Graph* g = (Graph*)h;
  if (!(i <= j && j <= k && k < p)) { g_err = "need i <= j <= k < p"; return -1; }
  uint64_t tot = 0;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nthreads(threads)) reduction(+ : tot)
  for (int64_t uu = cuts[i]; uu < (int64_t)cuts[i + 1]; ++uu) {
    const uint32_t u = (uint32_t)uu;
    const uint32_t* Nu = g->col.data() + g->row[u];
    const uint64_t du = g->row[u + 1] - g->row[u];
    for (uint64_t x = 0; x < du; ++x) {
      const uint32_t v = Nu[x];
      if (v < cuts[j] || v >= cuts[j + 1]) continue;
      const uint32_t* Nv = g->col.data() + g->row[v];
      const uint64_t dv = g->row[v + 1] - g->row[v];
      intersect(Nu, du, Nv, dv, [&](uint32_t w) {
        if (w >= cuts[k] && w < cuts[k + 1]) tot++;
      });
    }
  }
  *count = tot;
  return 0;
}

// Alg. 4 order as explicit triples (for pinning the library's index formula).
void oracle_task_list(uint32_t p, uint32_t* ti, uint32_t* tj, uint32_t* tk) {
  uint64_t t = 0;
  for (uint32_t i = 0; i < p; ++i)
    for (uint32_t j = i; j < p; ++j)
      for (uint32_t k = j; k < p; ++k) { ti[t] = i; tj[t] = j; tk[t] = k; ++t; }
}

// Timing helper for the CPU baseline: count only rows u = u0, u0+stride, ... < u1
// (unblocked node iterator), returning the triangles found and the edges visited.
int oracle_count_rows(void* h, uint32_t u0, uint32_t u1, uint32_t stride, int threads, uint64_t* tri,
                      uint64_t* edges) {
  Graph* g = (Graph*)h;
  uint64_t tot = 0, ed = 0;
  u1 = std::min(u1, g->n);
  if (stride == 0) stride = 1;
  const int64_t cnt = u1 > u0 ? ((int64_t)u1 - u0 + stride - 1) / stride : 0;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nthreads(threads)) reduction(+ : tot, ed)
  for (int64_t x = 0; x < cnt; ++x) {
    const uint32_t u = (uint32_t)(u0 + x * stride);
    const uint32_t* Nu = g->col.data() + g->row[u];
    const uint64_t du = g->row[u + 1] - g->row[u];
    ed += du;
    for (uint64_t x = 0; x < du; ++x) {
      const uint32_t v = Nu[x];
      tot += intersect(Nu, du, g->col.data() + g->row[v], g->row[v + 1] - g->row[v], [](uint32_t) {});
    }
  }
  *tri = tot;
  *edges = ed;
  return 0;
}

}  // extern "C"

// cpu.cpp — §8(f)#3 hybrid CPU+GPU execution (Alg. 8 TCPU, §7.7 cut-off).
//
// The paper orders tasks by the estimate ExecTime(t) = nnz(G_ij) · max(δ(G_ik), δ(G_jk))
// (reading R8), lets the GPUs take heavy tasks from the front of that queue
// and CPU threads take light ones from the back, each CPU thread atomically moving
// the back pointer until it reaches the cut-off (default: the middle); the GPUs
// may go past the cut-off while tasks remain.
//
// B200 form: the queue lives on the host.  The calling thread is the GPU's driver: it
// claims tasks from the front — first everything up to the cut-off, then chunks of
// what is left — and launches the list kernel over each claimed set (a task table of
// its own, no per-task launches); CPU threads claim single tasks from the back under
// the same lock, so every task is counted exactly once.  A CPU task runs Alg. 6's
// dense map over V_k as a bitmap: for each row u of G_ij, mark
// N(G_ik, u), then test every w of N(G_jk, v) for each v in N(G_ij, u) — the rows of
// the plan's blocks carry no order, and the map needs none.  The CPU reads the plan's
// pinned host arenas (bbtc_plan_to_host); this is product code, independent of the
// oracle (which shares nothing with the library).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <mutex>
#include <thread>

#include "internal.h"

namespace bbtc {

// Triangles of one task from the host arenas (row-major CSR of every block).
uint64_t cpu_count_task(const bbtc_plan* plan, const TaskDesc& T, std::vector<uint64_t>& bits) {
  const BlockDesc& Bij = plan->blocks[T.ij];
  const BlockDesc& Bik = plan->blocks[T.ik];
  const BlockDesc& Bjk = plan->blocks[T.jk];
  if (!Bij.nnz || !Bik.nnz || !Bjk.nnz) return 0;
  const uint32_t rows = plan->cuts[Bij.i + 1] - plan->cuts[Bij.i];
  const uint32_t vk = plan->cuts[Bik.j + 1] - plan->cuts[Bik.j];
  if (bits.size() < (vk + 63) / 64) bits.assign((vk + 63) / 64, 0);
  const uint32_t* rp_ij = plan->h_rowptr + Bij.ro;
  const uint32_t* rp_ik = plan->h_rowptr + Bik.ro;
  const uint32_t* rp_jk = plan->h_rowptr + Bjk.ro;
  const uint32_t* c_ij = plan->h_cols + Bij.e0;
  const uint32_t* c_ik = plan->h_cols + Bik.e0;
  const uint32_t* c_jk = plan->h_cols + Bjk.e0;
  uint64_t tri = 0;
  for (uint32_t u = 0; u < rows; ++u) {
    const uint32_t e0 = rp_ij[u], e1 = rp_ij[u + 1];
    const uint32_t a0 = rp_ik[u], a1 = rp_ik[u + 1];
    if (e0 == e1 || a0 == a1) continue;
    for (uint32_t a = a0; a < a1; ++a) bits[c_ik[a] >> 6] |= 1ull << (c_ik[a] & 63);
    for (uint32_t e = e0; e < e1; ++e) {
      const uint32_t v = c_ij[e];
      for (uint32_t x = rp_jk[v], x1 = rp_jk[v + 1]; x < x1; ++x) tri += (bits[c_jk[x] >> 6] >> (c_jk[x] & 63)) & 1;
    }
    for (uint32_t a = a0; a < a1; ++a) bits[c_ik[a] >> 6] = 0;
  }
  return tri;
}

// The double-ended queue of the sparse tasks (execution-order positions), heaviest
// first by ExecTime; ties keep the execution order.
std::vector<uint32_t> exec_time_queue(const bbtc_plan* plan) {
  auto delta = [&](uint32_t b) {
    const BlockDesc& B = plan->blocks[b];
    const uint32_t r = plan->cuts[B.i + 1] - plan->cuts[B.i];
    return r ? (double)B.nnz / r : 0.0;
  };
  std::vector<uint32_t> q(plan->dense_task_lo);
  std::vector<double> w(q.size());
  for (uint32_t t = 0; t < q.size(); ++t) {
    const TaskDesc& T = plan->tasks[t];
    q[t] = t;
    w[t] = (double)plan->blocks[T.ij].nnz * std::max(delta(T.ik), delta(T.jk));
  }
  std::stable_sort(q.begin(), q.end(), [&](uint32_t a, uint32_t b) { return w[a] > w[b]; });
  return q;
}

}  // namespace bbtc

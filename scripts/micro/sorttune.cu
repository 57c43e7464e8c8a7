// CUB onesweep radix sort with custom (threads, items) tunings on B200, at the shapes
// of the preprocessing sorts: rmat24's canonical keys (268 M u64 keys, 48 bits), block
// keys (260 M u64, 28 bits) and transpose pairs (260 M u32 keys + u32 values, 24 bits).
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o sorttune sorttune.cu
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdint>
#include <vector>

template <class K, class V, class O, int T, int I, int RB = 8>
struct Hub {
  using Base = typename cub::detail::radix::policy_hub<K, V, O>::Policy1000;
  struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, Policy1000> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = RB;
    using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, K, RB>;
    using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, RB>;
    using OnesweepPolicy =
        cub::AgentRadixSortOnesweepPolicy<T, I, K, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                          cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, RB>;
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

__global__ void fill(uint64_t* k, uint64_t n, uint64_t mask, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + seed) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    k[i] = (z ^ (z >> 31)) & mask;
  }
}

template <class K, class V, int T, int I, int RB = 8>
void run(const char* what, K* a, K* b, V* va, V* vb, uint64_t n, int bits, void* tmp, size_t tmp_cap) {
  using O = unsigned long long;
  using D = cub::DispatchRadixSort<false, K, V, O, Hub<K, V, O, T, I, RB>>;
  cub::DoubleBuffer<K> dk(a, b);
  cub::DoubleBuffer<V> dv(va, vb);
  size_t tb = 0;
  D::Dispatch(nullptr, tb, dk, dv, (O)n, 0, bits, true, 0);
  if (tb > tmp_cap) {
    printf("%s T=%d I=%d: temp %zu too big\n", what, T, I, tb);
    return;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 4; ++r) {
    // fresh random keys every repetition (a sorted input is not the workload)
    fill<<<4096, 256>>>((uint64_t*)dk.Current(), n * sizeof(K) / 8,
                        sizeof(K) == 8 ? (bits == 64 ? ~0ull : (1ull << bits) - 1) : ((1ull << bits) - 1) * 0x100000001ull,
                        r + 7);
    cudaEventRecord(e0);
    size_t t2 = tb;
    D::Dispatch(tmp, t2, dk, dv, (O)n, 0, bits, true, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r) best = ms < best ? ms : best;
  }
  const int passes = (bits + RB - 1) / RB;
  const double bytes = (double)n * (sizeof(K) + (std::is_same<V, cub::NullType>::value ? 0 : sizeof(V))) * 2 * passes;
  printf("%-10s T=%4d I=%3d RB=%2d: %7.3f ms  (%d passes, %.0f GB/s moved)  %s\n", what, T, I, RB, best, passes,
         bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const uint64_t n = 268435456;
  uint64_t *a, *b;
  uint32_t *va, *vb;
  void* tmp;
  const size_t cap = 1ull << 30;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMalloc(&va, n * 4);
  cudaMalloc(&vb, n * 4);
  cudaMalloc(&tmp, cap);
  fill<<<4096, 256>>>(a, n, (1ull << 48) - 1, 1);
  cudaDeviceSynchronize();
#define K48(T, I) run<uint64_t, cub::NullType, T, I>("u64/48b", a, b, nullptr, nullptr, n, 48, tmp, cap)
  K48(384, 30); K48(256, 30); K48(256, 40); K48(512, 20); K48(384, 20); K48(640, 16);
  K48(768, 12); K48(256, 24); K48(256, 34); K48(256, 36); K48(192, 40); K48(192, 48); K48(128, 64); K48(128, 80);
  K48(320, 28); K48(288, 32);
  fill<<<4096, 256>>>(a, n, (1ull << 28) - 1, 2);
#define K28(T, I) run<uint64_t, cub::NullType, T, I>("u64/28b", a, b, nullptr, nullptr, n, 28, tmp, cap)
  K28(384, 30); K28(512, 20); K28(256, 40); K28(384, 20); K28(256, 30); K28(256, 36); K28(192, 48);
  K28(128, 80);
  uint32_t* a32 = (uint32_t*)a;
  uint32_t* b32 = (uint32_t*)b;
  fill<<<4096, 256>>>(a, n / 2, 0x00FFFFFF00FFFFFFull, 3);
#define P24(T, I) run<uint32_t, uint32_t, T, I>("u32+v/24b", a32, b32, va, vb, n, 24, tmp, cap)
  P24(384, 23); P24(384, 17); P24(512, 20); P24(256, 30); P24(512, 16); P24(256, 23); P24(256, 26);
  P24(192, 30); P24(320, 23); P24(384, 26);
#define K48R(T, I, R) run<uint64_t, cub::NullType, T, I, R>("u64/48b", a, b, nullptr, nullptr, n, 48, tmp, cap)
  K48R(256, 30, 10); K48R(192, 32, 10); K48R(128, 60, 10);
#define K28R(T, I, R) run<uint64_t, cub::NullType, T, I, R>("u64/28b", a, b, nullptr, nullptr, n, 28, tmp, cap)
  K28R(256, 30, 10); K28R(288, 32, 8); K28R(192, 30, 10);
#define P24R(T, I, R) run<uint32_t, uint32_t, T, I, R>("u32+v/24b", a32, b32, va, vb, n, 24, tmp, cap)
  P24R(256, 16, 10); P24R(256, 23, 10); P24R(192, 23, 10);
  return 0;
}

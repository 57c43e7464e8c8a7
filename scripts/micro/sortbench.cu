// Micro-benchmark: CUB onesweep radix sort throughput on B200 for the prep sorts' shapes.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void fill(uint64_t* k, uint64_t n, int bits) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = i * 0x9E3779B97F4A7C15ull + 12345;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    k[i] = bits >= 64 ? z : (z & ((1ull << bits) - 1));
  }
}
__global__ void copyk(const uint64_t* a, uint64_t* b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <class N>
float sort64(uint64_t* a, uint64_t* b, N n, int bits, void* tmp, size_t tb, cudaEvent_t e0, cudaEvent_t e1) {
  cub::DoubleBuffer<uint64_t> db(a, b);
  size_t t = tb;
  cudaEventRecord(e0);
  cub::DeviceRadixSort::SortKeys(tmp, t, db, n, 0, bits);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main(int argc, char** argv) {
  uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 1800000000ull;
  uint64_t *a, *b;
  CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8));
  size_t tb = 0;
  { cub::DoubleBuffer<uint64_t> db(a, b); cub::DeviceRadixSort::SortKeys(nullptr, tb, db, n, 0, 64); }
  size_t tb2 = 0;
  { cub::DoubleBuffer<uint64_t> db(a, b); cub::DeviceRadixSort::SortKeys(nullptr, tb2, db, (int)std::min<uint64_t>(n, 2000000000ull), 0, 64); }
  tb = std::max(tb, tb2);
  void* tmp; CK(cudaMalloc(&tmp, tb));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // copy reference
  copyk<<<148 * 8, 256>>>(a, b, n);
  cudaEventRecord(e0); copyk<<<148 * 8, 256>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float cms; cudaEventElapsedTime(&cms, e0, e1);
  printf("copy u64 n=%llu: %.2f ms = %.0f GB/s\n", (unsigned long long)n, cms, 16.0 * n / cms / 1e6);
  for (int bits : {28, 32, 40, 48, 52, 64}) {
    for (int rep = 0; rep < 3; ++rep) {
      fill<<<148 * 8, 256>>>(a, n, bits);
      float ms64 = sort64<uint64_t>(a, b, n, bits, tmp, tb, e0, e1);
      fill<<<148 * 8, 256>>>(a, n, bits);
      float ms32 = n < 2147483647ull ? sort64<int>(a, b, (int)n, bits, tmp, tb, e0, e1) : -1;
      int passes = (bits + 7) / 8;
      printf("bits=%d u64-offset %.2f ms  int-offset %.2f ms  (%.0f GB/s per pass-equiv, %d passes)  err=%s\n", bits, ms64,
             ms32, (16.0 * passes + 8) * n / ms64 / 1e6, passes, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

// Micro-benchmark: random-gather DRAM throughput on B200 (the roofline of the list
// kernel's probe-list reads).  A warp reads R random runs of L contiguous bytes
// each from a table much larger than L2; reported: useful GB/s and sector GB/s.
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31);
}
// each thread group of G lanes reads one run of G*4 bytes (G = 1, 2, 4, 8, 16, 32)
template <int G>
__global__ void gather(const uint32_t* __restrict__ t, uint64_t words, uint64_t runs, unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  uint32_t acc = 0;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x / G;
#pragma unroll 4
  for (uint64_t r = tid / G; r < runs; r += stride) {
    uint64_t base = (mix(r * 0x9E3779B97F4A7C15ull + 7) & (words / G - 1)) * G;
    acc += t[base + (lane % G)];
  }
  if (acc == 0x12345678) atomicAdd(out, 1ull);
}
int main() {
  const uint64_t bytes = 16ull << 30, words = bytes / 4;
  uint32_t* t; CK(cudaMalloc(&t, bytes)); CK(cudaMemset(t, 1, bytes));
  unsigned long long* o; CK(cudaMalloc(&o, 8));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, int G) {
    const uint64_t runs = (8ull << 30) / (4 * G) ;   // 8 GB useful bytes
    for (int occ : {4, 8, 16}) {
      kern<<<148 * occ, 256>>>(t, words, runs / 8, o);
      cudaEventRecord(a);
      kern<<<148 * occ, 256>>>(t, words, runs, o);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double useful = runs * 4.0 * G, sectors = runs * 32.0 * ((4 * G + 31) / 32);
      printf("run %4d B, %2d CTAs/SM: %.2f ms  useful %.0f GB/s  sectors %.0f GB/s  (%s)\n", 4 * G, occ, ms,
             useful / ms / 1e6, sectors / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(gather<1>, 1); run(gather<2>, 2); run(gather<4>, 4); run(gather<8>, 8); run(gather<16>, 16); run(gather<32>, 32);
  return 0;
}

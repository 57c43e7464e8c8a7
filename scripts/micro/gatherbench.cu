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
// one warp reads a run of NL consecutive 128-B lines (NL = 2 .. 16: 256 B .. 2 KB),
// NL independent coalesced loads in flight per lane
template <int NL>
__global__ void gather_lines(const uint32_t* __restrict__ t, uint64_t words, uint64_t runs, unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  uint32_t acc = 0;
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = wid; r < runs; r += nw) {
    const uint64_t base = (mix(r * 0x9E3779B97F4A7C15ull + 11) & (words / (32 * NL) - 1)) * (32 * NL);
    uint32_t w[NL];
#pragma unroll
    for (int x = 0; x < NL; ++x) w[x] = t[base + 32 * x + lane];
#pragma unroll
    for (int x = 0; x < NL; ++x) acc += w[x];
  }
  if (acc == 0x12345678) atomicAdd(out, 1ull);
}

int main(int argc, char**) {
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
  if (argc < 2) {
    run(gather<1>, 1); run(gather<2>, 2); run(gather<4>, 4); run(gather<8>, 8); run(gather<16>, 16); run(gather<32>, 32);
  }
  auto run_lines = [&](auto kern, int NL) {
    const uint64_t runs = (16ull << 30) / (128ull * NL);   // 16 GB useful bytes
    for (int occ : {4, 8, 16}) {
      kern<<<148 * occ, 256>>>(t, words, runs / 8, o);
      cudaEventRecord(a);
      kern<<<148 * occ, 256>>>(t, words, runs, o);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("run %5d B (%2d lines), %2d CTAs/SM: %.2f ms  %.0f GB/s  (%s)\n", 128 * NL, NL, occ, ms,
             runs * 128.0 * NL / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  };
  run_lines(gather_lines<1>, 1); run_lines(gather_lines<2>, 2); run_lines(gather_lines<4>, 4);
  run_lines(gather_lines<8>, 8); run_lines(gather_lines<16>, 16);
  return 0;
}

// Microbenchmark: effective L2 capacity for random 16-bit gathers on B200.
// For array sizes S, time G random gathers (hash-generated indices) and report
// GB/s of 32-byte sectors and the implied hit behaviour.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned mix(unsigned x) { x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16; return x; }
__global__ void gather(const unsigned short* a, unsigned n, long long g, unsigned seed, unsigned long long* out) {
  unsigned long long acc = 0;
  long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g; i += nt) {
    unsigned idx = mix((unsigned)i * 2654435761u + seed) % n;
    acc += __ldcg(a + idx);
  }
  if (acc == 12345) *out = acc;
}
int main() {
  size_t maxb = 512ull << 20;
  unsigned short* a; cudaMalloc(&a, maxb); cudaMemset(a, 1, maxb);
  unsigned long long* o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  long long g = 1ll << 30;
  for (size_t mb : {8, 16, 32, 48, 64, 80, 96, 112, 128, 192, 256, 512}) {
    unsigned n = (unsigned)((mb << 20) / 2);
    gather<<<148 * 8, 256>>>(a, n, g, 7, o);
    cudaEventRecord(e0);
    gather<<<148 * 8, 256>>>(a, n, g, 99, o);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("array %4zu MB: %.2f ms for 2^30 gathers = %.1f Ggathers/s (%.0f GB/s of 32B sectors)\n", mb, ms, g / ms / 1e6, g * 32.0 / ms / 1e6);
  }
  return 0;
}

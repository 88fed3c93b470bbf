// Microbenchmark: random 4-byte gathers per second on B200 from
//   (a) global memory through L2 (ld.global.cg), table sizes 64 KB .. 32 MB,
//   (b) global memory through L1 (ld.global.ca), L1-sized tables,
//   (c) shared memory (the table staged per CTA), up to 192 KB.
// Indices are hash-generated in registers (no index traffic); 8 independent
// gathers in flight per thread.  Question answered: is a per-SM shared-memory
// copy of hot records worth it for the pull rounds' random record gathers
// (ncu: ~1 L2 request per gather, L1->XBAR request interface ~70 % busy)?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned mix(unsigned x) { x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16; return x; }
template <int MODE>  // 0 cg, 1 ca, 2 smem
__global__ void __launch_bounds__(1024, 1) gather(const unsigned *a, unsigned mask, int iters, unsigned seed, unsigned *out) {
  extern __shared__ unsigned sh[];
  if (MODE == 2) {
    for (unsigned i = threadIdx.x; i <= mask; i += blockDim.x) sh[i] = a[i];
    __syncthreads();
  }
  unsigned acc = 0;
  unsigned base = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + seed;
  for (int it = 0; it < iters; it++) {
    unsigned v[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      unsigned idx = mix(base + it * 8 + q) & mask;
      if (MODE == 0) v[q] = __ldcg(a + idx);
      else if (MODE == 1) v[q] = __ldca(a + idx);
      else v[q] = sh[idx];
    }
#pragma unroll
    for (int q = 0; q < 8; q++) acc += v[q];
  }
  if (acc == 0x12345678u) *out = acc;
}
int main() {
  unsigned *a; cudaMalloc(&a, 64 << 20); cudaMemset(a, 1, 64 << 20);
  unsigned *o; cudaMalloc(&o, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int dev = 0, sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(gather<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 256;
  const double g = (double)sms * 1024 * iters * 8;
  auto run = [&](int mode, unsigned entries) {
    unsigned mask = entries - 1;
    size_t smem = mode == 2 ? entries * 4 : 0;
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      if (mode == 0) gather<0><<<sms, 1024, smem>>>(a, mask, iters, 7 + rep, o);
      if (mode == 1) gather<1><<<sms, 1024, smem>>>(a, mask, iters, 7 + rep, o);
      if (mode == 2) gather<2><<<sms, 1024, smem>>>(a, mask, iters, 7 + rep, o);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 1) printf("%-6s table %8u entries (%6u KB): %8.1f Ggathers/s  (%.2f per SM per clock at 1.965 GHz)\n",
                           mode == 0 ? "L2.cg" : mode == 1 ? "L1.ca" : "smem", entries, entries * 4 / 1024,
                           g / ms / 1e6, g / ms / 1e6 / sms / 1.965);
    }
    cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  };
  for (unsigned e : {1u << 14, 1u << 16, 1u << 20, 1u << 23}) run(0, e);
  for (unsigned e : {1u << 12, 1u << 13, 1u << 14}) run(1, e);
  for (unsigned e : {1u << 12, 1u << 14, 1u << 15}) run(2, e);
  return 0;
}

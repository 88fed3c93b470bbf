// Microbenchmark: cost of one software grid barrier of a persistent
// cooperative kernel on B200 (the PeelOne level kernel runs ~960 of them at
// C2), for grid shapes (CTAs per SM x threads) and barrier implementations:
//   0  current common.cuh grid_barrier: threadfence + atomicAdd arrive, last
//      arriver resets and bumps gen, others poll gen (volatile + nanosleep 20)
//   1  release/acquire: atom.add.acq_rel arrive, st.release gen, ld.acquire poll
//   2  monotonic counter: atom.add.release, poll the same counter until it
//      reaches the episode's multiple of the grid size (no reset, no gen)
//   3  as 0 without nanosleep in the poll loop
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
struct Bar { alignas(128) unsigned arrive; alignas(128) unsigned gen; };
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned *p, unsigned v) {
  unsigned o; asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o; }
__device__ __forceinline__ unsigned atom_add_release(unsigned *p, unsigned v) {
  unsigned o; asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o; }
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v; asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
template <int IMPL>
__device__ __forceinline__ void barrier(Bar *b, unsigned &episode) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x;
    if (IMPL == 0 || IMPL == 3) {
      unsigned g = *(volatile unsigned *)&b->gen;
      __threadfence();
      if (atomicAdd(&b->arrive, 1u) == nb - 1) { *(volatile unsigned *)&b->arrive = 0; __threadfence(); atomicAdd(&b->gen, 1u); }
      else { while (*(volatile unsigned *)&b->gen == g) { if (IMPL == 0) __nanosleep(20); } }
      __threadfence();
    } else if (IMPL == 1) {
      unsigned g = *(volatile unsigned *)&b->gen;
      if (atom_add_acqrel(&b->arrive, 1u) == nb - 1) { *(volatile unsigned *)&b->arrive = 0; st_release(&b->gen, g + 1); }
      else { while (ld_acquire(&b->gen) == g) __nanosleep(20); }
    } else {
      episode++;
      const unsigned target = episode * nb;
      atom_add_release(&b->arrive, 1u);
      while (ld_acquire(&b->arrive) < target) __nanosleep(20);
    }
  }
  __syncthreads();
}
template <int IMPL>
__global__ void kern(Bar *b, int iters, unsigned *sink) {
  unsigned ep = 0;
  unsigned x = threadIdx.x;
  for (int i = 0; i < iters; i++) { x = x * 1664525u + 1013904223u; barrier<IMPL>(b, ep); }
  if (x == 0x12345) *sink = x;
}
__global__ void kern_cg(int iters, unsigned *sink) {
  cg::grid_group g = cg::this_grid();
  unsigned x = threadIdx.x;
  for (int i = 0; i < iters; i++) { x = x * 1664525u + 1013904223u; g.sync(); }
  if (x == 0x12345) *sink = x;
}
int main() {
  Bar *b; unsigned *sink; cudaMalloc(&b, sizeof(Bar)); cudaMalloc(&sink, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  struct Shape { int per, thr; } shapes[] = {{1, 512}, {1, 1024}, {2, 512}, {3, 512}, {4, 256}, {8, 128}};
  for (auto sh : shapes) {
    for (int impl = 0; impl < 5; impl++) {
      cudaMemset(b, 0, sizeof(Bar));
      int blocks = sms * sh.per, it = iters;
      void *args[] = {&b, &it, &sink};
      void *args_cg[] = {&it, &sink};
      const void *f = impl == 0 ? (const void *)kern<0> : impl == 1 ? (const void *)kern<1> : impl == 2 ? (const void *)kern<2>
                    : impl == 3 ? (const void *)kern<3> : (const void *)kern_cg;
      cudaLaunchCooperativeKernel(f, blocks, sh.thr, impl == 4 ? args_cg : args, 0, 0);  // warm
      cudaMemset(b, 0, sizeof(Bar));
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel(f, blocks, sh.thr, impl == 4 ? args_cg : args, 0, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      printf("%d CTAs/SM x %4d threads (%4d CTAs)  impl %d%s: %.3f us per barrier %s\n", sh.per, sh.thr, blocks, impl,
             impl == 4 ? " (cg grid.sync)" : "", ms * 1e3 / iters, err ? cudaGetErrorString(err) : "");
    }
  }
  return 0;
}

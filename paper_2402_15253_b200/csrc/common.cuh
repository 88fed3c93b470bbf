// common.cuh -- device helpers shared by the HistoCore and PeelOne kernels
// (sm_100a).  Warp-aggregated list appends (ballot/popc compaction), warp
// scans, a software grid barrier for the persistent cooperative kernels, and
// the workspace control block.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

namespace pico {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// inclusive warp scan (sum) of a 32-bit value
__device__ __forceinline__ int warp_incl_scan(int x) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(FULL, x, o);
        if (lane_id() >= o) x += y;
    }
    return x;
}

__device__ __forceinline__ long long warp_incl_scan64(long long x) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(FULL, x, o);
        if (lane_id() >= o) x += y;
    }
    return x;
}

__device__ __forceinline__ long long warp_sum64(long long x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    return x;
}

__device__ __forceinline__ int warp_min(int x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = min(x, __shfl_xor_sync(FULL, x, o));
    return x;
}

// Warp-aggregated append of `v` (for lanes with pred) to list/count.  Must be
// called by all 32 lanes of the warp.  One atomic per warp; slots in lane
// order (ballot + popc compaction).
__device__ __forceinline__ void warp_append(bool pred, int v, int *list,
                                            unsigned long long *count) {
    unsigned m = __ballot_sync(FULL, pred);
    if (m == 0) return;
    unsigned long long base = 0;
    int leader = __ffs(m) - 1;
    if (lane_id() == leader) base = atomicAdd(count, (unsigned long long)__popc(m));
    base = __shfl_sync(FULL, base, leader);
    if (pred) list[base + __popc(m & ((1u << lane_id()) - 1))] = v;
}

// relaxed/volatile loads for values other CTAs update concurrently
__device__ __forceinline__ int ld_volatile(const int *p) {
    return *reinterpret_cast<const volatile int *>(p);
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p) {
    return *reinterpret_cast<const volatile unsigned long long *>(p);
}

// L2 eviction-priority policies (createpolicy) and loads carrying them:
// streaming data (colidx, work lists) is evict_first so it does not flush the
// hot random-access structures (8-bit estimate shadow, changed bitmap), which
// are evict_last.
__device__ __forceinline__ unsigned long long pol_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long pol_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// read-only streaming load (never written during the kernel)
__device__ __forceinline__ int ld_stream(const int *p, unsigned long long pol) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ long long ld_stream64(const long long *p, unsigned long long pol) {
    long long v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}
// coherent (L2) loads of data other CTAs may have written before a barrier
__device__ __forceinline__ unsigned ld_cg_u8(const unsigned char *p, unsigned long long pol) {
    unsigned short v;
    asm volatile("ld.global.cg.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ unsigned ld_cg_u16(const unsigned short *p, unsigned long long pol) {
    unsigned short v;
    asm volatile("ld.global.cg.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ unsigned ld_cg_u32(const unsigned *p, unsigned long long pol) {
    unsigned v;
    asm volatile("ld.global.cg.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int2 ld_stream_int2(const int2 *p, unsigned long long pol) {
    int2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}

#ifndef PICO_L2_HINTS
#define PICO_L2_HINTS 0
#endif
#if !PICO_L2_HINTS
// hints disabled: plain cached loads
#define ld_stream(p, pol) __ldg(p)
#define ld_stream_int2(p, pol) __ldcg(p)
#define ld_cg_u32(p, pol) __ldcg(p)
#endif

// fire-and-forget global reductions (REDG), relaxed, device scope
__device__ __forceinline__ void red_add(int *p, int v) {
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or(unsigned *p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// warp-aggregated reservation of nseg segments per lane; writes (v, s) entries
__device__ __forceinline__ void warp_append_segments(int v, int nseg, int2 *S,
                                                     unsigned long long *nS) {
    int incl = warp_incl_scan(nseg);
    int total = __shfl_sync(FULL, incl, 31);
    if (total == 0) return;
    unsigned long long base = 0;
    if (lane_id() == 0) base = atomicAdd(nS, (unsigned long long)total);
    base = __shfl_sync(FULL, base, 0);
    // the warp writes the `total` entries jointly (a hub's thousands of
    // segments do not serialise on its lane): entry j belongs to the lane with
    // the largest exclusive offset <= j
    const int excl = incl - nseg;
    for (int j0 = 0; j0 < total; j0 += 32) {
        int j = j0 + lane_id();
        int lo = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            int cand = lo + step;
            int ex = __shfl_sync(FULL, excl, cand & 31);
            if (cand < 32 && ex <= j) lo = cand;
        }
        int vo = __shfl_sync(FULL, v, lo);
        int eo = __shfl_sync(FULL, excl, lo);
        if (j < total) S[base + j] = make_int2(vo, j - eo);
    }
}

// Block-uniform read of a control word other CTAs wrote before a barrier:
// thread 0 loads it and broadcasts through shared memory, so a 300K-thread
// grid issues one L2 request per CTA instead of one per thread to a single
// address (which serialises on one L2 slice).  Block-collective.
__device__ __forceinline__ unsigned long long bcast_u64(const unsigned long long *p) {
    __shared__ unsigned long long s_u64;
    __syncthreads();
    if (threadIdx.x == 0) s_u64 = *reinterpret_cast<const volatile unsigned long long *>(p);
    __syncthreads();
    return s_u64;
}
__device__ __forceinline__ int bcast_i32(const int *p) {
    __shared__ int s_i32;
    __syncthreads();
    if (threadIdx.x == 0) s_i32 = *reinterpret_cast<const volatile int *>(p);
    __syncthreads();
    return s_i32;
}

// Software grid barrier for persistent kernels launched cooperatively (all
// CTAs co-resident).  Sense via a generation counter.
__device__ __forceinline__ void grid_barrier(unsigned *arrive, unsigned *gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g = *reinterpret_cast<volatile unsigned *>(gen);
        __threadfence();
        unsigned nb = gridDim.x * gridDim.y * gridDim.z;
        if (atomicAdd(arrive, 1u) == nb - 1) {
            *reinterpret_cast<volatile unsigned *>(arrive) = 0;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*reinterpret_cast<volatile unsigned *>(gen) == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

// Grid barrier that also publishes a consistent snapshot: the last CTA to
// arrive (all other CTAs' writes are fenced by then) copies *src to *dst
// before releasing the barrier.
__device__ __forceinline__ void grid_barrier_snap(unsigned *arrive, unsigned *gen,
                                                  const unsigned long long *src,
                                                  unsigned long long *dst) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g = *reinterpret_cast<volatile unsigned *>(gen);
        __threadfence();
        unsigned nb = gridDim.x * gridDim.y * gridDim.z;
        if (atomicAdd(arrive, 1u) == nb - 1) {
            *reinterpret_cast<volatile unsigned long long *>(dst) =
                *reinterpret_cast<const volatile unsigned long long *>(src);
            *reinterpret_cast<volatile unsigned *>(arrive) = 0;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*reinterpret_cast<volatile unsigned *>(gen) == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

// Workspace control block (device memory, initialised at the start of a call).
#ifndef PICO_BAR_PAD
#define PICO_BAR_PAD 0
#endif
struct Ctrl {
    // HistoCore lists: F (frontier vertex ids) and S (update segments),
    // double-buffered counts indexed by round parity (see histocore.cu).
    unsigned long long nF[2];
    unsigned long long nS[2];
    unsigned long long nB;         // init class-B list (warp per vertex)
    unsigned long long nC;         // init class-C list (CTA per vertex)
    unsigned long long nX;         // hub fallback list (global bins)
    unsigned long long rounds;     // HistoCore rounds >= 2 counted on device
    unsigned long long wc[2];      // UpdateHisto batch claim counters (parity)
    unsigned long long arcsC[2];   // sum of deg(v) over C_t (parity t&1)
    int mincv[2];                  // min core_t(v) over C_t (parity t&1)
    unsigned long long nH;         // static hub segments (pull mode)
    // PeelOne queue state (a run-wide log of processed (vertex, segment)s);
    // each hot word on its own 128-byte line (polling vs. atomics)
    alignas(128) unsigned long long q_head;     // next queue slot to claim
    alignas(128) unsigned long long q_tail;     // next queue slot to write
    alignas(128) unsigned long long q_pending;  // pushed, not fully processed
    alignas(128) unsigned long long q_snap;     // tail snapshot at the last barrier
    alignas(128) unsigned long long q_tail1;    // PeelOne: the queue's second append counter
    alignas(128) unsigned long long nJoin;      // PeelOne rebuild: far vertices joining the near list
    int kminJ;                                  // PeelOne rebuild: their minimum estimate
    alignas(128) unsigned long long nAlive[2];  // alive list lengths (ping-pong by level; own line: the
                                                // scans append to these and to a queue counter at once)
    unsigned long long nFar[2];    // far list lengths (ping-pong by rebuild)
    int fmin[2];                   // min estimate in the far list (ping-pong)
    unsigned long long nProc[2];   // vertices processed per level (parity)
    unsigned long long levels;     // non-empty levels
    unsigned long long scans;      // levels scanned
    int kminb[2];                  // lower bound of the next level (parity)
    int kmax;
    int error;                     // device-detected error code (validation)
    // grid barrier (own lines)
    alignas(128) unsigned bar_arrive;
    alignas(128) unsigned bar_gen;
#if PICO_BAR_PAD
    unsigned char bar_pad[PICO_BAR_PAD];  // A/B: the arrival word far from the hot counters
#endif
    alignas(128) unsigned bar_flip;  // grid_sync's arrival word
    // instrumentation (PICO_F_STATS)
    unsigned long long st_frontier;
    unsigned long long st_init_slots;
    unsigned long long st_arcs;
    unsigned long long st_guarded;
    unsigned long long st_bins;
    unsigned long long st_pushes;
    unsigned long long st_alive;
    unsigned long long st_fallback;
    unsigned long long st_segs;
    unsigned long long st_pull;
};

// Grid barrier with one arrival word and no release word: CTA 0 adds
// 2^31 - (nb - 1), every other CTA adds 1, so the word's top bit flips
// exactly when the last CTA arrives, whatever the order, and the low bits
// return to their value (the word starts at 0).  Every CTA polls the top bit
// of the word it incremented.  scripts/micro/grid_barrier.cu: 1.23 us at 444
// CTAs against 2.57 us for grid_barrier (whose last arriver resets the count
// and bumps a separate generation word: one more serialised L2 round trip).
// The PeelOne level kernel (~1,000 short phases at C2) uses it; HistoCore's
// round kernel keeps grid_barrier, whose pollers back off: its phases last
// milliseconds, and spinning CTAs cost its rounds ~0.5 % (profiles/r02/s3/).
#ifndef PICO_BAR_SLEEP
#define PICO_BAR_SLEEP 0  // ns of backoff per poll of the arrival word (A/B)
#endif
#ifndef PICO_BAR_GEN
#define PICO_BAR_GEN 0  // A/B: grid_sync through the generation-word barrier
#endif
__device__ __forceinline__ void grid_sync(Ctrl *c) {
#if PICO_BAR_GEN
    grid_barrier(&c->bar_arrive, &c->bar_gen);
    return;
#endif
    unsigned *bar = &c->bar_flip;
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
        const unsigned add = (blockIdx.x | blockIdx.y | blockIdx.z) == 0 ? 0x80000000u - (nb - 1) : 1u;
        __threadfence();
        const unsigned old = atomicAdd(bar, add);
        while (((old ^ *reinterpret_cast<volatile unsigned *>(bar)) & 0x80000000u) == 0) {
#if PICO_BAR_SLEEP
            __nanosleep(PICO_BAR_SLEEP);
#endif
        }
        __threadfence();
    }
    __syncthreads();
}


// Tunables (degree-class thresholds, bin caps).  PICO_F_TINY_TILES shrinks
// them so all code paths are exercised by small test graphs.
struct Tune {
    int a_max;      // class A (thread per vertex): deg <= a_max (<= 16)
    int b_max;      // class B (warp per vertex):   a_max < deg <= b_max
    int c_bins;     // class C (CTA per vertex) shared-memory bin cap
    int seg;        // arcs per UpdateHisto segment
    int pull_div;   // sharded: pull-mode UpdateHisto when arcs(C_t) >= 2m / pull_div
    int pull_tenths;  // one GPU: pull when 10 arcs(C_t) >= pull_tenths 2m
};

}  // namespace pico

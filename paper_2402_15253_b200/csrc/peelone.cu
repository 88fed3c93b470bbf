// peelone.cu -- PeelOne with the assertion method and a dynamic frontier
// ("PO-dyn"; Alg 4) for sm_100a.
//
//   core[v] = deg(v)  (one array is residual degree AND coreness)
//   for k = 1, 2, ... while vertices remain:
//     scan:    frontier = {alive v : core[v] == k}
//     scatter: for v in frontier, u in nbr(v):
//                if core[u] > k:                          (guard)
//                  old = atomicSub>=k(core[u], 1, k)      ((old>k)?old-1:k)
//                  if old == k+1: push u into the SAME level's queue
//                                                         (dynamic frontier P:342;
//                                                          SURVEY 8(c)#19)
// The level index k jumps to a lower bound of the minimum alive core, so only
// non-empty levels (plus at most the final one) are scanned; the number of
// non-empty levels is the number of distinct coreness values (l1 =
// k_max).
//
// B200 design: one persistent cooperative kernel runs every level.  The scan
// walks a compacted alive list (ping-pong), never all n vertices.  The level's
// queue lives in a run-wide log Q of (vertex, segment) entries (every vertex
// is processed exactly once over the run, so Q never wraps; hub rows are split
// into 256-arc entries).  The dynamic frontier is drained in bulk-synchronous
// sub-rounds: sub-round r processes the entries appended by sub-round r-1,
// warps claim batches of 32 entries with one atomicAdd (no CAS, no polling),
// walk the rows with warp-level load balancing and append newly clamped
// vertices at the tail; one grid barrier per sub-round, whose last arriving
// CTA publishes a consistent snapshot of the tail.
//
// Three bit-exact implementations of atomicSub>=k, see
// clamp_dec(): atomicSub + atomicMax on overshoot (default), atomicSub + end-
// of-level repair (PICO_F_CLAMP_SUB), CAS loop (PICO_F_CLAMP_CAS).
#include <climits>

#include "common.cuh"
#include "kernels.h"

#ifndef PICO_PO_PER
#define PICO_PO_PER 3  // resident CTAs per SM of the persistent level kernel
#endif

namespace pico {

struct PoArgs {
    const long long *rp;
    const int *ci;
    int n;
    int *core;
    int *alive0;
    int *alive1;
    long long *Q;  // (v << 32) | segment
    unsigned long long *fsz;
    unsigned long long fsz_cap;
    Ctrl *ctl;
    int seg;
};

__device__ __forceinline__ int po_nseg(long long d, int seg) { return (int)((d + seg - 1) / seg); }

// Warp-cooperative append of vertices (pred lanes) to the queue tail, one entry
// per `seg` arcs of the row.  Returns the number of vertices appended.
__device__ __forceinline__ int po_push(const PoArgs &a, bool pred, int v) {
    const int lane = lane_id();
    int ns = 0;
    if (pred) ns = po_nseg(__ldg(a.rp + v + 1) - __ldg(a.rp + v), a.seg);
    int incl = warp_incl_scan(ns);
    int total = __shfl_sync(FULL, incl, 31);
    if (total == 0) return 0;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&a.ctl->q_tail, (unsigned long long)total);
    base = __shfl_sync(FULL, base, 0);
    unsigned long long off = base + (unsigned long long)(incl - ns);
    for (int s = 0; s < ns; s++) a.Q[off + s] = ((long long)v << 32) | s;
    return __popc(__ballot_sync(FULL, pred));
}

// scan of level k (parity p): alive[p] -> frontier entries in Q, alive[p^1]
template <bool STATS>
__device__ void po_scan_phase(const PoArgs &a, int k, int p, long long gthread, long long nthreads) {
    const long long na = (long long)bcast_u64(&a.ctl->nAlive[p]);
    const int *alive = p ? a.alive1 : a.alive0;
    int *next = p ? a.alive0 : a.alive1;
    long long iters = (na + nthreads - 1) / nthreads;
    int kmin = INT_MAX;
    long long nproc = 0;
    for (long long it = 0; it < iters; it++) {
        long long i = it * nthreads + gthread;
        bool valid = i < na;
        int v = 0, c = 0;
        if (valid) {
            v = __ldcg(alive + i);
            c = __ldcg(a.core + v);
        }
        bool front = valid && c == k;
        bool keep = valid && c > k;  // c < k: already processed by an earlier level
        if (keep) kmin = min(kmin, c);
        warp_append(keep, v, next, &a.ctl->nAlive[p ^ 1]);
        nproc += po_push(a, front, v);
    }
    kmin = warp_min(kmin);
    // po_push returns the warp-wide count to every lane: lane 0 holds the total
    if (lane_id() == 0) {
        if (kmin != INT_MAX) atomicMin(&a.ctl->kminb[p ^ 1], kmin);
        if (nproc) atomicAdd(&a.ctl->nProc[p], (unsigned long long)nproc);
        if (STATS && gthread == 0) atomicAdd(&a.ctl->st_alive, (unsigned long long)na);
    }
}

// clamped decrement atomicSub>=k(core[u], 1, k) of P:273; returns the old
// value (> k: the caller decremented; == k+1: it set the value to k).
//   MODE 0 (default): atomicSub, and only if that overshot below k an
//     atomicMax(k) -- exact, at most two atomics, no retry loop under the
//     contention of hub vertices; every value is >= k again before the level's
//     closing barrier (all readers of transient values skip them: guard c > k).
//   MODE 1 (PICO_F_CLAMP_SUB): atomicSub only; the level's queue range is
//     repaired to k after the level (SURVEY 8(c)#18 b).
//   MODE 2 (PICO_F_CLAMP_CAS): compare-and-swap loop, never below k (the
//     literal "single atomic transaction", SURVEY 8(c)#18 a).
template <int MODE>
__device__ __forceinline__ int clamp_dec(int *p, int c, int k) {
    if (MODE == 2) {
        int old = c;
        for (;;) {
            if (old <= k) return old;
            int prev = atomicCAS(p, old, old - 1);
            if (prev == old) return old;
            old = prev;
        }
    }
    int old = atomicSub(p, 1);
    if (MODE == 0 && old <= k) atomicMax(p, k);
    return old;
}

// one sub-round of level k: process queue entries [lo, hi).  Entries hold at
// most `seg` (<= 32) arcs, so one warp takes PICO_PO_U entries per iteration
// (lanes = arcs, U gathers + U clamps in flight per lane): a sub-round's
// latency is a few memory round trips instead of a serial walk of long rows.
#ifndef PICO_PO_U
#define PICO_PO_U 2  // queue entries per warp iteration (independent chains in flight)
#endif
template <int MODE, bool STATS>
__device__ void po_sub_phase(const PoArgs &a, int k, int p, unsigned long long lo, unsigned long long hi) {
    constexpr int U = PICO_PO_U;
    const int lane = lane_id();
    const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    int kmin = INT_MAX;
    long long nproc = 0, st_arcs = 0, st_dec = 0;
    // iteration it takes entries lo + (it*U + q)*nwarps + gwarp, q < U: the U
    // entries' loads, gathers and clamps are issued together
    for (unsigned long long i0 = lo + gwarp; i0 < hi; i0 += (unsigned long long)nwarps * U) {
        int u[U], c[U];
        bool in[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            unsigned long long i = i0 + (unsigned long long)q * nwarps;
            in[q] = false;
            u[q] = 0;
            if (i < hi) {
                long long e = __ldcg(a.Q + i);
                int v = (int)(e >> 32);
                int s = (int)(e & 0xffffffffll);
                long long r0 = __ldg(a.rp + v), r1 = __ldg(a.rp + v + 1);
                long long b = r0 + (long long)s * a.seg;
                int len = (int)min((long long)a.seg, r1 - b);
                if (lane < len) {
                    in[q] = true;
                    u[q] = __ldg(a.ci + b + lane);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < U; q++) c[q] = in[q] ? __ldcg(a.core + u[q]) : 0;
        bool push[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            push[q] = false;
            if (in[q]) {
                if (STATS) st_arcs++;
                if (c[q] > k) {  // guard core[u] > k
                    int old = clamp_dec<MODE>(a.core + u[q], c[q], k);
                    if (STATS) st_dec += (old > k);
                    push[q] = (old == k + 1);
                    if (old - 1 > k) kmin = min(kmin, old - 1);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < U; q++) nproc += po_push(a, push[q], u[q]);
    }
    kmin = warp_min(kmin);
    // po_push returns the warp-wide count to every lane: lane 0 holds the total
    if (lane == 0) {
        if (kmin != INT_MAX) atomicMin(&a.ctl->kminb[p ^ 1], kmin);
        if (nproc) atomicAdd(&a.ctl->nProc[p], (unsigned long long)nproc);
    }
    if (STATS) {
        long long s1 = warp_sum64(st_arcs), s2 = warp_sum64(st_dec);
        if (lane == 0) {
            if (s1) atomicAdd(&a.ctl->st_arcs, (unsigned long long)s1);
            if (s2) atomicAdd(&a.ctl->st_guarded, (unsigned long long)s2);
            if (nproc) atomicAdd(&a.ctl->st_pushes, (unsigned long long)nproc);
        }
    }
}

__device__ void po_repair_phase(const PoArgs &a, int k, unsigned long long lo, unsigned long long hi,
                                long long gthread, long long nthreads) {
    for (unsigned long long i = lo + gthread; i < hi; i += nthreads) {
        long long e = __ldcg(a.Q + i);
        a.core[(int)(e >> 32)] = k;
    }
}

// level bookkeeping for level with parity p and value k (leader only)
__device__ __forceinline__ void po_close_level(const PoArgs &a, int p, int k) {
    unsigned long long pc = ld_volatile(&a.ctl->nProc[p]);
    a.ctl->scans++;
    if (pc) {
        if (a.ctl->levels < a.fsz_cap) a.fsz[a.ctl->levels] = pc;
        a.ctl->levels++;
        a.ctl->kmax = k;
    }
    a.ctl->nProc[p] = 0;
}

// ---------------------------------------------------------------------------
// P0: core = deg, alive list, initial level bound
// ---------------------------------------------------------------------------
__global__ void po_init_kernel(PoArgs a) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    long long gthread = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long iters = (a.n + nthreads - 1) / nthreads;
    int kmin = INT_MAX;
    for (long long it = 0; it < iters; it++) {
        long long v = it * nthreads + gthread;
        bool valid = v < a.n;
        int d = valid ? (int)(a.rp[v + 1] - a.rp[v]) : 0;
        if (valid) a.core[v] = d;
        bool alive = d > 0;
        if (alive) kmin = min(kmin, d);
        warp_append(alive, (int)v, a.alive0, &a.ctl->nAlive[0]);
    }
    kmin = warp_min(kmin);
    if (lane_id() == 0 && kmin != INT_MAX) atomicMin(&a.ctl->kminb[0], kmin);
}

// ---------------------------------------------------------------------------
// P1-P3: persistent cooperative kernel over all levels
// ---------------------------------------------------------------------------
template <int MODE, bool STATS>
__global__ void __launch_bounds__(512) po_levels_kernel(PoArgs a) {
    constexpr bool CLAMP_SUB = MODE == 1;
    const long long gthread = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    Ctrl *c = a.ctl;
    int k = 0, kprev = 0;
    unsigned long long S = 0;  // global sub-round counter (claim counter parity)
    for (int L = 0;; L++) {
        const int p = L & 1;
        long long na = (long long)bcast_u64(&c->nAlive[p]);
        if (leader && L > 0) po_close_level(a, p ^ 1, kprev);
        if (na == 0) break;
        k = max(k + 1, bcast_i32(&c->kminb[p]));
        unsigned long long lstart = bcast_u64(&c->q_snap);
        po_scan_phase<STATS>(a, k, p, gthread, nthreads);
        grid_barrier_snap(&c->bar_arrive, &c->bar_gen, &c->q_tail, &c->q_snap);
        if (leader) {
            c->nAlive[p] = 0;       // alive[p] consumed; refilled at level L+1
            c->kminb[p] = INT_MAX;  // consumed at this level's head
        }
        unsigned long long lo = lstart;
        for (int sub = 0;; sub++) {
            unsigned long long hi = bcast_u64(&c->q_snap);
            if (hi == lo) {  // uniform: every CTA read the same snapshot
                // an empty level has no sub-round barrier: one barrier orders
                // the leader's resets above before the next level's scan
                // appends to alive[p] / lowers kminb[p]
                if (sub == 0) grid_barrier(&c->bar_arrive, &c->bar_gen);
                break;
            }
            po_sub_phase<MODE, STATS>(a, k, p, lo, hi);
            grid_barrier_snap(&c->bar_arrive, &c->bar_gen, &c->q_tail, &c->q_snap);
            lo = hi;
            S++;
        }
        if (CLAMP_SUB) {
            po_repair_phase(a, k, lstart, lo, gthread, nthreads);
            grid_barrier_snap(&c->bar_arrive, &c->bar_gen, &c->q_tail, &c->q_snap);
        }
        if (leader) c->rounds = S;  // BSP sub-rounds so far
        kprev = k;
    }
}

// host-loop variants (PICO_F_HOST_LOOP)
template <bool STATS>
__global__ void __launch_bounds__(512) po_scan_kernel(PoArgs a, int k, int p) {
    const long long gthread = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    po_scan_phase<STATS>(a, k, p, gthread, nthreads);
}

template <int MODE, bool STATS>
__global__ void __launch_bounds__(512) po_sub_kernel(PoArgs a, int k, int p, unsigned long long lo,
                                                     unsigned long long hi, int first) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && first) {
        a.ctl->nAlive[p] = 0;
        a.ctl->kminb[p] = INT_MAX;
    }
    po_sub_phase<MODE, STATS>(a, k, p, lo, hi);
}

__global__ void po_repair_kernel(PoArgs a, int k, unsigned long long lo, unsigned long long hi) {
    const long long gthread = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    po_repair_phase(a, k, lo, hi, gthread, nthreads);
}

__global__ void po_close_kernel(PoArgs a, int p, int k) { po_close_level(a, p, k); }

// ---------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
static int po_seg(uint32_t flags) { return (flags & PICO_F_TINY_TILES) ? 4 : 32; }

size_t po_workspace_bytes(long long n, long long arcs, uint32_t flags) {
    size_t b = 0;
    b += align256(sizeof(Ctrl));
    b += align256(sizeof(unsigned long long) * kFszCap);
    b += align256(sizeof(int) * (size_t)n) * 2;
    b += align256(sizeof(long long) * (size_t)(n + arcs / po_seg(flags) + 64));
    return b;
}

template <int MODE, bool STATS>
static cudaError_t po_run_t(const long long *rp, const int *ci, long long n, long long arcs, int *core,
                            cudaStream_t s, uint32_t flags, void *ws, pico_stats_t *st,
                            const DevInfo &dev) {
    constexpr bool CLAMP_SUB = MODE == 1;
    PoArgs a;
    char *p = (char *)ws;
    a.ctl = (Ctrl *)p; p += align256(sizeof(Ctrl));
    a.fsz = (unsigned long long *)p; p += align256(sizeof(unsigned long long) * kFszCap);
    a.fsz_cap = kFszCap;
    a.alive0 = (int *)p; p += align256(sizeof(int) * (size_t)n);
    a.alive1 = (int *)p; p += align256(sizeof(int) * (size_t)n);
    a.Q = (long long *)p;
    a.seg = po_seg(flags);
    a.rp = rp; a.ci = ci; a.n = (int)n; a.core = core;

    cudaError_t err;
    Ctrl h{};
    h.kminb[0] = INT_MAX;
    h.kminb[1] = INT_MAX;
    if ((err = cudaMemcpyAsync(a.ctl, &h, sizeof(Ctrl), cudaMemcpyHostToDevice, s))) return err;

    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
    auto tstart = [&](int slot) {
        if (!(flags & PICO_F_TIMING)) return;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        ev.push_back({slot, {e0, e1}});
    };
    auto tstop = [&]() {
        if (flags & PICO_F_TIMING) cudaEventRecord(ev.back().second.second, s);
    };

    const int sms = dev.sms;
    tstart(PICO_K_DEGREE);
    {
        int blocks = (int)std::min<long long>((n + 255) / 256, (long long)sms * 16);
        po_init_kernel<<<std::max(blocks, 1), 256, 0, s>>>(a);
    }
    tstop();
    if ((err = cudaGetLastError())) return err;

    long long launches = 1, host_subrounds = 0;
    tstart(PICO_K_PEEL);
    if (flags & PICO_F_HOST_LOOP) {
        int blocks = sms * 4;
        int k = 0, kprev = 0;
        unsigned long long tail = 0;
        for (int L = 0;; L++) {
            int par = L & 1;
            Ctrl hc;
            if ((err = cudaMemcpyAsync(&hc, a.ctl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s))) return err;
            if ((err = cudaStreamSynchronize(s))) return err;
            if (L > 0) { po_close_kernel<<<1, 1, 0, s>>>(a, par ^ 1, kprev); launches++; }
            if (hc.nAlive[par] == 0) break;
            k = std::max(k + 1, hc.kminb[par]);
            unsigned long long lstart = hc.q_tail, lo = lstart;
            po_scan_kernel<STATS><<<blocks, 512, 0, s>>>(a, k, par);
            launches++;
            for (int sub = 0;; sub++) {
                if ((err = cudaMemcpyAsync(&tail, &a.ctl->q_tail, sizeof(tail), cudaMemcpyDeviceToHost, s)))
                    return err;
                if ((err = cudaStreamSynchronize(s))) return err;
                if (tail == lo) {
                    if (sub == 0) {  // empty level: still consume alive[par]
                        unsigned long long z = 0;
                        int imax = INT_MAX;
                        cudaMemcpyAsync(&a.ctl->nAlive[par], &z, sizeof(z), cudaMemcpyHostToDevice, s);
                        cudaMemcpyAsync(&a.ctl->kminb[par], &imax, sizeof(imax), cudaMemcpyHostToDevice, s);
                    }
                    break;
                }
                po_sub_kernel<MODE, STATS><<<blocks, 512, 0, s>>>(a, k, par, lo, tail, sub == 0);
                launches++;
                host_subrounds++;
                lo = tail;
            }
            if (CLAMP_SUB && lo > lstart) {
                po_repair_kernel<<<blocks, 512, 0, s>>>(a, k, lstart, lo);
                launches++;
            }
            kprev = k;
        }
    } else {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, po_levels_kernel<MODE, STATS>, 512, 0);
        int per = std::max(1, std::min(occ, PICO_PO_PER));
        void *args[] = {&a};
        err = cudaLaunchCooperativeKernel((const void *)po_levels_kernel<MODE, STATS>, sms * per, 512,
                                          args, 0, s);
        if (err) return err;
        launches++;
    }
    tstop();
    if ((err = cudaGetLastError())) return err;

    Ctrl hc;
    if ((err = cudaMemcpyAsync(&hc, a.ctl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s))) return err;
    std::vector<unsigned long long> lv(kFszCap);
    if ((err = cudaMemcpyAsync(lv.data(), a.fsz, sizeof(unsigned long long) * kFszCap,
                               cudaMemcpyDeviceToHost, s)))
        return err;
    if ((err = cudaStreamSynchronize(s))) return err;
    if (st) {
        st->levels = (int64_t)hc.levels;
        st->subrounds = (flags & PICO_F_HOST_LOOP) ? host_subrounds : (int64_t)hc.rounds;
        st->kmax = hc.kmax;
        st->segments = (int64_t)hc.q_tail;
        st->kernel_count += launches;
        if (st->frontier_sizes)
            for (unsigned long long i = 0; i < hc.levels && (int64_t)i < st->frontier_sizes_cap && i < kFszCap; i++)
                st->frontier_sizes[i] = (int64_t)lv[i];
        if (STATS) {
            st->arcs_scanned = (int64_t)hc.st_arcs;
            st->guarded_arcs = (int64_t)hc.st_guarded;
            st->pushes = (int64_t)hc.st_pushes;
            st->alive_scanned = (int64_t)hc.st_alive;
        }
        for (auto &e : ev) {
            float ms = 0;
            cudaEventElapsedTime(&ms, e.second.first, e.second.second);
            st->kernel_ms[e.first] += ms;
            st->kernel_launches[e.first] += 1;
        }
    }
    for (auto &e : ev) {
        cudaEventDestroy(e.second.first);
        cudaEventDestroy(e.second.second);
    }
    return cudaSuccess;
}

// pico_clamp_hammer: c threads run clamp_dec<MODE> on one cell; mode 1
// then applies the end-of-level repair (max(k, value)) as po_levels does
template <int MODE>
__global__ void po_hammer_kernel(int *cell, int k, long long c, unsigned long long *cnt) {
    long long nt = (long long)gridDim.x * blockDim.x;
    unsigned long long gt = 0, k1 = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < c; i += nt) {
        const int g = __ldcg(cell);  // the guard read core[u] > k of po_sub_phase
        if (g <= k) continue;
        int old = clamp_dec<MODE>(cell, g, k);
        gt += old > k;
        k1 += old == k + 1;
    }
    if (gt) atomicAdd(cnt, gt);
    if (k1) atomicAdd(cnt + 1, k1);
}

__global__ void po_hammer_repair_kernel(int *cell, int k) {
    if (threadIdx.x == 0 && *cell < k) *cell = k;
}

cudaError_t po_clamp_hammer(int mode, int d, int k, long long c, int *final_out, long long *gt, long long *k1,
                            cudaStream_t s) {
    void *buf = nullptr;
    cudaError_t e = lib_malloc_async(&buf, 256, s);
    if (e) return e;
    int *cell = (int *)buf;
    unsigned long long *cnt = (unsigned long long *)((char *)buf + 128);
    unsigned long long h[2] = {0, 0};
    if (!e) e = cudaMemcpyAsync(cell, &d, sizeof(int), cudaMemcpyHostToDevice, s);
    if (!e) e = cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), s);
    if (!e && c > 0) {
        int blocks = (int)std::min<long long>((c + 255) / 256, 4096);
        if (mode == 0) po_hammer_kernel<0><<<blocks, 256, 0, s>>>(cell, k, c, cnt);
        if (mode == 1) po_hammer_kernel<1><<<blocks, 256, 0, s>>>(cell, k, c, cnt);
        if (mode == 2) po_hammer_kernel<2><<<blocks, 256, 0, s>>>(cell, k, c, cnt);
        e = cudaGetLastError();
    }
    if (!e && mode == 1 && d > k) {  // the repair covers the level's processed vertices
        po_hammer_repair_kernel<<<1, 32, 0, s>>>(cell, k);
        e = cudaGetLastError();
    }
    if (!e) e = cudaMemcpyAsync(final_out, cell, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaError_t e2 = cudaFreeAsync(buf, s);
    if (!e) e = e2;
    if (!e) e = cudaStreamSynchronize(s);
    *gt = (long long)h[0];
    *k1 = (long long)h[1];
    return e;
}

cudaError_t po_run(const long long *rp, const int *ci, long long n, long long arcs, int *core,
                   cudaStream_t s, uint32_t flags, void *ws, pico_stats_t *st, const DevInfo &dev) {
    bool stats = flags & PICO_F_STATS;
    int mode = (flags & PICO_F_CLAMP_CAS) ? 2 : (flags & PICO_F_CLAMP_SUB) ? 1 : 0;
#define PO_CASE(M)                                                                      \
    if (mode == M) return stats ? po_run_t<M, true>(rp, ci, n, arcs, core, s, flags, ws, st, dev) \
                                : po_run_t<M, false>(rp, ci, n, arcs, core, s, flags, ws, st, dev);
    PO_CASE(0)
    PO_CASE(1)
    PO_CASE(2)
#undef PO_CASE
    return cudaErrorInvalidValue;
}

}  // namespace pico

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
// non-empty levels (plus at most the final one) are scanned; the level count
// is k_max's number of distinct coreness values (l1 = k_max).
//
// B200 design: one persistent cooperative kernel runs every level (two grid
// barriers per level, no host round trips).  The scan walks a compacted alive
// list (ping-pong), never all n vertices.  Each level's queue is drained by
// all warps through a run-wide log Q of (vertex, segment) entries (every
// vertex is processed exactly once over the run, so Q never wraps): warps
// claim up to 32 entries with one CAS, walk the rows with warp-level load
// balancing, and push newly clamped vertices back into Q.  A `pending`
// counter (entries pushed but not finished) detects the end of a level.
//
// Two bit-exact implementations of atomicSub>=k:
//   CAS loop (default): read-compute-CAS, never below k (faithful to P:273).
//   CLAMP_SUB (PICO_F_CLAMP_SUB): atomicSub, push on old == k+1, and an
//     end-of-level repair core[v] = k over the level's queue range.
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace pico {

struct PoArgs {
    const long long *rp;
    const int *ci;
    int n;
    int *core;
    int *alive0;
    int *alive1;
    long long *Q;  // (v << 32) | segment, -1 = not yet written
    unsigned long long *fsz;
    unsigned long long fsz_cap;
    Ctrl *ctl;
    int seg;
};

__device__ __forceinline__ int po_nseg(long long d, int seg) { return (int)((d + seg - 1) / seg); }

// Warp-cooperative push of vertices (pred lanes) into the queue, one entry per
// `seg` arcs.  Lane 0 performs all pending/tail atomics (program order).
__device__ __forceinline__ int po_push(const PoArgs &a, bool pred, int v) {
    const int lane = lane_id();
    int ns = 0;
    if (pred) ns = po_nseg(__ldg(a.rp + v + 1) - __ldg(a.rp + v), a.seg);
    int incl = warp_incl_scan(ns);
    int total = __shfl_sync(FULL, incl, 31);
    if (total == 0) return 0;
    unsigned long long base = 0;
    if (lane == 0) {
        atomicAdd(&a.ctl->q_pending, (unsigned long long)total);
        base = atomicAdd(&a.ctl->q_tail, (unsigned long long)total);
    }
    base = __shfl_sync(FULL, base, 0);
    unsigned long long off = base + (unsigned long long)(incl - ns);
    for (int s = 0; s < ns; s++)
        *reinterpret_cast<volatile long long *>(a.Q + off + s) = ((long long)v << 32) | s;
    return __popc(__ballot_sync(FULL, pred));
}

// scan of level k (parity p): alive[p] -> frontier entries in Q, alive[p^1]
template <bool STATS>
__device__ void po_scan_phase(const PoArgs &a, int k, int p, long long gthread, long long nthreads) {
    const long long na = (long long)ld_volatile(&a.ctl->nAlive[p]);
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
    if (lane_id() == 0) {
        if (kmin != INT_MAX) atomicMin(&a.ctl->kminb[p ^ 1], kmin);
        if (nproc) atomicAdd(&a.ctl->nProc[p], (unsigned long long)nproc);
        if (STATS) atomicAdd(&a.ctl->st_alive, (unsigned long long)(gthread == 0 ? na : 0));
    }
}

// drain of level k: process queue entries until none is pending.  One thread
// per CTA polls and claims a chunk of entries (CAS on the head); the CTA's
// warps split the chunk 32 entries each and walk the rows with warp-level
// load balancing; newly clamped vertices are pushed back into the queue.
template <bool CLAMP_SUB, bool STATS>
__device__ void po_drain_phase(const PoArgs &a, int k, int p) {
    __shared__ unsigned long long s_base;
    __shared__ int s_got;
    const int lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int kmin = INT_MAX;
    long long nproc = 0, st_arcs = 0, st_dec = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            unsigned long long base = 0;
            int got = 0;
            for (int spin = 0;; spin++) {
                unsigned long long h = ld_volatile(&a.ctl->q_head);
                unsigned long long t = ld_volatile(&a.ctl->q_tail);
                if (h < t) {
                    unsigned long long avail = t - h;
                    unsigned long long share = (avail + gridDim.x - 1) / gridDim.x;
                    unsigned long long want = min(avail, max(32ull, min((unsigned long long)(32 * nw), share)));
                    if (atomicCAS(&a.ctl->q_head, h, h + want) == h) {
                        base = h;
                        got = (int)want;
                        break;
                    }
                } else {
                    if (ld_volatile(&a.ctl->q_pending) == 0) break;
                    __nanosleep(min(1024, 32 << min(spin, 5)));
                }
            }
            s_base = base;
            s_got = got;
        }
        __syncthreads();
        const int got = s_got;
        const unsigned long long base = s_base;
        __syncthreads();
        if (got == 0) break;
        const int myn = min(32, got - wid * 32);
        if (myn > 0) {
            long long b = 0;
            int len = 0;
            if (lane < myn) {
                long long e;
                do {
                    e = *reinterpret_cast<volatile long long *>(a.Q + base + wid * 32 + lane);
                } while (e < 0);
                int v = (int)(e >> 32);
                int s = (int)(e & 0xffffffffll);
                long long r0 = __ldg(a.rp + v), r1 = __ldg(a.rp + v + 1);
                b = r0 + (long long)s * a.seg;
                len = (int)min((long long)a.seg, r1 - b);
            }
            int incl = warp_incl_scan(len);
            int excl = incl - len;
            int total = __shfl_sync(FULL, incl, 31);
            for (int j0 = 0; j0 < total; j0 += 32) {
                int j = j0 + lane;
                int lo = 0;
#pragma unroll
                for (int step = 16; step >= 1; step >>= 1) {
                    int cand = lo + step;
                    int ex = __shfl_sync(FULL, excl, cand & 31);
                    if (cand < 32 && ex <= j) lo = cand;
                }
                long long eb = __shfl_sync(FULL, b, lo);
                int ex = __shfl_sync(FULL, excl, lo);
                bool push = false;
                int u = 0;
                if (j < total) {
                    u = __ldg(a.ci + eb + (j - ex));
                    int c = __ldcg(a.core + u);
                    if (STATS) st_arcs++;
                    if (c > k) {  // guard core[u] > k
                        int old;
                        if (CLAMP_SUB) {
                            old = atomicSub(a.core + u, 1);
                        } else {
                            old = c;
                            for (;;) {  // atomicSub>=k as a CAS loop
                                if (old <= k) break;
                                int prev = atomicCAS(a.core + u, old, old - 1);
                                if (prev == old) break;
                                old = prev;
                            }
                        }
                        if (STATS) st_dec++;
                        push = (old == k + 1);
                        if (old - 1 > k) kmin = min(kmin, old - 1);
                    }
                }
                nproc += po_push(a, push, u);
            }
        }
        __syncthreads();  // all pushes of this chunk precede its release
        if (threadIdx.x == 0) atomicAdd(&a.ctl->q_pending, 0ull - (unsigned long long)got);
    }
    kmin = warp_min(kmin);
    if (lane == 0) {
        if (kmin != INT_MAX) atomicMin(&a.ctl->kminb[p ^ 1], kmin);
        if (nproc) atomicAdd(&a.ctl->nProc[p], (unsigned long long)nproc);
    }
    if (STATS) {
        long long s1 = warp_sum64(st_arcs), s2 = warp_sum64(st_dec), s3 = warp_sum64(nproc);
        if (lane == 0) {
            if (s1) atomicAdd(&a.ctl->st_arcs, (unsigned long long)s1);
            if (s2) atomicAdd(&a.ctl->st_guarded, (unsigned long long)s2);
            if (s3) atomicAdd(&a.ctl->st_pushes, (unsigned long long)s3);
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
template <bool CLAMP_SUB, bool STATS>
__global__ void __launch_bounds__(512) po_levels_kernel(PoArgs a) {
    const long long gthread = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    int k = 0, kprev = 0;
    unsigned long long lstart = 0;
    int L = 0;
    for (;; L++) {
        const int p = L & 1;
        long long na = (long long)ld_volatile(&a.ctl->nAlive[p]);
        if (leader && L > 0) po_close_level(a, p ^ 1, kprev);
        if (na == 0) break;
        k = max(k + 1, ld_volatile(&a.ctl->kminb[p]));
        po_scan_phase<STATS>(a, k, p, gthread, nthreads);
        grid_barrier(&a.ctl->bar_arrive, &a.ctl->bar_gen);
        if (leader) {
            a.ctl->nAlive[p] = 0;        // alive[p] consumed; refilled at level L+1
            a.ctl->kminb[p] = INT_MAX;   // consumed at this level's head
        }
        po_drain_phase<CLAMP_SUB, STATS>(a, k, p);
        grid_barrier(&a.ctl->bar_arrive, &a.ctl->bar_gen);
        if (CLAMP_SUB) {
            unsigned long long lend = ld_volatile(&a.ctl->q_tail);
            po_repair_phase(a, k, lstart, lend, gthread, nthreads);
            lstart = lend;
            grid_barrier(&a.ctl->bar_arrive, &a.ctl->bar_gen);
        }
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

template <bool CLAMP_SUB, bool STATS>
__global__ void __launch_bounds__(512) po_drain_kernel(PoArgs a, int k, int p) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.ctl->nAlive[p] = 0;
        a.ctl->kminb[p] = INT_MAX;
    }
    po_drain_phase<CLAMP_SUB, STATS>(a, k, p);
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
static int po_seg(uint32_t flags) { return (flags & PICO_F_TINY_TILES) ? 4 : 256; }

size_t po_workspace_bytes(long long n, long long arcs, uint32_t flags) {
    size_t b = 0;
    b += align256(sizeof(Ctrl));
    b += align256(sizeof(unsigned long long) * kFszCap);
    b += align256(sizeof(int) * (size_t)n) * 2;
    b += align256(sizeof(long long) * (size_t)(n + arcs / po_seg(flags) + 64));
    return b;
}

template <bool CLAMP_SUB, bool STATS>
static cudaError_t po_run_t(const long long *rp, const int *ci, long long n, long long arcs, int *core,
                            cudaStream_t s, uint32_t flags, void *ws, pico_stats_t *st,
                            const DevInfo &dev) {
    PoArgs a;
    char *p = (char *)ws;
    a.ctl = (Ctrl *)p; p += align256(sizeof(Ctrl));
    a.fsz = (unsigned long long *)p; p += align256(sizeof(unsigned long long) * kFszCap);
    a.fsz_cap = kFszCap;
    a.alive0 = (int *)p; p += align256(sizeof(int) * (size_t)n);
    a.alive1 = (int *)p; p += align256(sizeof(int) * (size_t)n);
    a.Q = (long long *)p;
    a.seg = po_seg(flags);
    size_t qcap = (size_t)(n + arcs / a.seg + 64);
    a.rp = rp; a.ci = ci; a.n = (int)n; a.core = core;

    cudaError_t err;
    Ctrl h{};
    h.kminb[0] = INT_MAX;
    h.kminb[1] = INT_MAX;
    if ((err = cudaMemcpyAsync(a.ctl, &h, sizeof(Ctrl), cudaMemcpyHostToDevice, s))) return err;
    if ((err = cudaMemsetAsync(a.Q, 0xff, sizeof(long long) * qcap, s))) return err;

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

    long long launches = 1;
    tstart(PICO_K_PEEL);
    if (flags & PICO_F_HOST_LOOP) {
        int blocks = sms * 4;
        int k = 0, kprev = 0;
        unsigned long long lstart = 0;
        for (int L = 0;; L++) {
            int par = L & 1;
            Ctrl hc;
            if ((err = cudaMemcpyAsync(&hc, a.ctl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s))) return err;
            if ((err = cudaStreamSynchronize(s))) return err;
            if (L > 0) { po_close_kernel<<<1, 1, 0, s>>>(a, par ^ 1, kprev); launches++; }
            if (hc.nAlive[par] == 0) break;
            k = std::max(k + 1, hc.kminb[par]);
            po_scan_kernel<STATS><<<blocks, 512, 0, s>>>(a, k, par);
            po_drain_kernel<CLAMP_SUB, STATS><<<blocks, 512, 0, s>>>(a, k, par);
            launches += 2;
            if (CLAMP_SUB) {
                unsigned long long lend = 0;
                if ((err = cudaMemcpyAsync(&lend, &a.ctl->q_tail, sizeof(lend), cudaMemcpyDeviceToHost, s)))
                    return err;
                if ((err = cudaStreamSynchronize(s))) return err;
                if (lend > lstart) { po_repair_kernel<<<blocks, 512, 0, s>>>(a, k, lstart, lend); launches++; }
                lstart = lend;
            }
            kprev = k;
        }
    } else {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, po_levels_kernel<CLAMP_SUB, STATS>, 512, 0);
        int per = std::max(1, std::min(occ, 2));
        void *args[] = {&a};
        err = cudaLaunchCooperativeKernel((const void *)po_levels_kernel<CLAMP_SUB, STATS>, sms * per, 512,
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
        st->segments = (int64_t)hc.q_tail;
        st->kernel_count = launches;
        st->subrounds = (int64_t)hc.scans;
        st->kmax = hc.kmax;
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

cudaError_t po_run(const long long *rp, const int *ci, long long n, long long arcs, int *core,
                   cudaStream_t s, uint32_t flags, void *ws, pico_stats_t *st, const DevInfo &dev) {
    bool sub = flags & PICO_F_CLAMP_SUB, stats = flags & PICO_F_STATS;
    if (sub && stats) return po_run_t<true, true>(rp, ci, n, arcs, core, s, flags, ws, st, dev);
    if (sub) return po_run_t<true, false>(rp, ci, n, arcs, core, s, flags, ws, st, dev);
    if (stats) return po_run_t<false, true>(rp, ci, n, arcs, core, s, flags, ws, st, dev);
    return po_run_t<false, false>(rp, ci, n, arcs, core, s, flags, ws, st, dev);
}

}  // namespace pico

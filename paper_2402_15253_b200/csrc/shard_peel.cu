// shard_peel.cu -- sharded PeelOne (the level-synchronous
// peel of Alg 4, with the clamped decrement of P:273 and the
// dynamic frontier of P:342, split over ranks by the 1-D vertex partition of
// the sharded HistoCore).
//
// Rank r owns the estimates core[u] of u in [vb, vb + nloc) and a local CSC:
// for every global v, the owned neighbours u of v (the transpose of the owned
// rows; the graph is symmetric).  A level k is
//
//   scan:     F = {owned alive u : core[u] == k}
//   repeat (one BSP sub-round per iteration):
//     exchange: all-gather of the per-rank |F| (the global test: 0 ends the
//               level) and all-gatherv of F (global ids)           (caller)
//     apply:    for v in F_all, u in CSC[v] with core[u] > k:
//                 old = atomicSub>=k(core[u], 1, k)
//                 if old == k+1: u joins this rank's next F
//
// Each call publishes (|F| of this rank, a lower bound of the minimum alive
// estimate above k) as two int64 words on the device, ready for a collective
// without a host round trip.  The next level is k' = max(k+1, min over ranks
// of that bound); the run ends when the bound is INT_MAX on every rank.
// Sub-rounds are the single-GPU path's BSP sub-rounds (same frontier sets:
// sub-round r processes exactly the vertices that reached k in sub-round r-1),
// so the coreness is bit-exact and the level / sub-round counts do not depend
// on the number of ranks.  PeelOne needs no degree exchange: every decrement
// lands on the owner of its target.
#include <climits>
#include <cstddef>
#include <cstdlib>
#include <string>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "kernels.h"
#include "lsa_exchange.h"

namespace pico {

struct PsCtl {
    unsigned long long fcnt;       // frontier entries appended by the current call
    unsigned long long nalive[2];  // alive list lengths (ping-pong by level parity)
    unsigned long long nts;        // (received vertex, segment) work items
    unsigned long long st_arcs, st_dec;
    int kmin[2];                   // lower bound of the next level (by parity)
    long long out[2];              // published: |F| of this rank, kmin bound
    // device-driven loop (PICO_F_LSA_EXCHANGE, pshard_run_lsa): the latest
    // exchange's global results and the decision taken from them
    long long g_total;             // global |F| of the latest exchange
    long long g_kmin;              // global min of the published bounds
    int mode;                      // next step: 0 scan, 1 apply, 2 done
    int kcur, pcur, Lcnt, level_open, kmax;
    long long processed, levels, subrounds;
};

struct PeelShard {
    const long long *rp;
    const int *ci;
    long long nloc, vb, ng, arcs;
    uint32_t flags;
    cudaStream_t s;
    DevInfo dev;
    void *ws;
    int *core;         // [nloc] residual degree / coreness of the owned vertices
    int *alive[2];     // [nloc] owned alive vertices (local ids)
    long long *csc_off;  // [ng+1] (+ [ng+1] count scratch)
    int *csc_idx;      // [arcs] owned neighbour (local id), grouped by global v
    int *tmpk;         // [arcs] sort keys out
    int *src;          // [arcs] row of every local arc (CSC build)
    int2 *TS;          // [tscap] (index into the received frontier, segment)
    long long tscap;
    PsCtl *ctl;
    void *cubtmp;
    size_t cubbytes;
    int L;             // levels started
    int k;             // current level
    int seg;
};

constexpr int kPsSeg = 32;

__device__ __forceinline__ void ps_kmin(int *slot, int kmin) {
    kmin = warp_min(kmin);
    if (lane_id() == 0 && kmin != INT_MAX) atomicMin(slot, kmin);
}

// P0 on the owned vertices: core = deg, alive list, first level bound
__global__ void ps_init_kernel(const long long *rp, long long nloc, int *core, int *alive0, PsCtl *c) {
    long long nt = (long long)gridDim.x * blockDim.x;
    long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long iters = (nloc + nt - 1) / nt;
    int kmin = INT_MAX;
    for (long long it = 0; it < iters; it++) {
        long long u = it * nt + g;
        bool valid = u < nloc;
        int d = valid ? (int)(rp[u + 1] - rp[u]) : 0;
        if (valid) core[u] = d;
        if (d > 0) kmin = min(kmin, d);
        warp_append(d > 0, (int)u, alive0, &c->nalive[0]);
    }
    ps_kmin(&c->kmin[0], kmin);
}

// row of every local arc (one warp per row)
__global__ void ps_src_kernel(const long long *rp, long long nloc, int *src) {
    long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long u = w; u < nloc; u += nw)
        for (long long e = rp[u] + lane_id(); e < rp[u + 1]; e += 32) src[e] = (int)u;
}

__global__ void ps_csc_count_kernel(const int *ci, long long arcs, unsigned long long *cnt_v) {
    long long nt = (long long)gridDim.x * blockDim.x;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < arcs; e += nt)
        atomicAdd(cnt_v + ci[e], 1ull);
}

// start of level L (parity p): the lists of parity p^1 are refilled
__global__ void ps_begin_kernel(PsCtl *c, int p) {
    c->nalive[p ^ 1] = 0;
    c->kmin[p ^ 1] = INT_MAX;
    c->fcnt = 0;
}

// P1: scan of the owned alive list at level k -> F (global ids), kept list
__device__ __forceinline__ void ps_scan_body(const int *core, const int *alive, int *next, PsCtl *c, int p, int k,
                                             long long vb, int *front) {
    const long long na = (long long)c->nalive[p];
    long long nt = (long long)gridDim.x * blockDim.x;
    long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long iters = (na + nt - 1) / nt;
    int kmin = INT_MAX;
    for (long long it = 0; it < iters; it++) {
        long long i = it * nt + g;
        bool valid = i < na;
        int u = 0, cu = 0;
        if (valid) {
            u = alive[i];
            cu = core[u];
        }
        bool keep = valid && cu > k;  // cu < k: processed at an earlier level
        if (keep) kmin = min(kmin, cu);
        warp_append(keep, u, next, &c->nalive[p ^ 1]);
        warp_append(valid && cu == k, (int)(u + vb), front, &c->fcnt);
    }
    ps_kmin(&c->kmin[p ^ 1], kmin);
}

// publish (|F|, kmin bound of parity q) for the exchange; reset the counters
__global__ void ps_scan_kernel(const int *core, const int *alive, int *next, PsCtl *c, int p, int k, long long vb,
                               int *front) {
    ps_scan_body(core, alive, next, c, p, k, vb, front);
}

// device-driven loop: the step decided on the device (mode 0 = scan)
__global__ void ps_scan_dev_kernel(const int *core, int *alive0, int *alive1, PsCtl *c, long long vb, int *front) {
    if (c->mode != 0) return;
    const int p = c->pcur;
    ps_scan_body(core, p ? alive1 : alive0, p ? alive0 : alive1, c, p, c->kcur, vb, front);
}

__global__ void ps_pub_kernel(PsCtl *c, int q) {
    c->out[0] = (long long)c->fcnt;
    c->out[1] = (long long)c->kmin[q];
    c->fcnt = 0;
    c->nts = 0;
}

// (received vertex, segment) items over the CSC columns of the received F
__global__ void ps_segments_kernel(const int *all, long long total, const long long *csc_off, int seg, int2 *TS,
                                   unsigned long long *nts, const PsCtl *dc = nullptr) {
    if (dc) {  // device-driven loop: an apply step (mode 1) over the exchange's total
        if (dc->mode != 1) return;
        total = dc->g_total;
    }
    long long nt = (long long)gridDim.x * blockDim.x;
    long long iters = (total + nt - 1) / nt;
    for (long long it = 0; it < iters; it++) {
        long long i = it * nt + (long long)blockIdx.x * blockDim.x + threadIdx.x;
        int ns = 0;
        if (i < total) {
            int v = all[i];
            long long len = csc_off[v + 1] - csc_off[v];
            ns = (int)((len + seg - 1) / seg);
        }
        int incl = warp_incl_scan(ns);
        int tot = __shfl_sync(FULL, incl, 31);
        if (tot == 0) continue;
        unsigned long long base = 0;
        if (lane_id() == 0) base = atomicAdd(nts, (unsigned long long)tot);
        base = __shfl_sync(FULL, base, 0);
        const int excl = incl - ns;
        for (int j0 = 0; j0 < tot; j0 += 32) {  // the warp writes a hub's segments jointly
            int j = j0 + lane_id();
            int lo = 0;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1) {
                int cand = lo + step;
                int ex = __shfl_sync(FULL, excl, cand & 31);
                if (cand < 32 && ex <= j) lo = cand;
            }
            long long io = __shfl_sync(FULL, i, lo);
            int eo = __shfl_sync(FULL, excl, lo);
            if (j < tot) TS[base + j] = make_int2((int)io, j - eo);
        }
    }
}

// atomicSub>=k(core[u], 1, k) of P:273 (as peelone.cu's clamp_dec): MODE 0
// atomicSub + atomicMax(k) on overshoot, MODE 2 CAS loop
template <int MODE>
__device__ __forceinline__ int ps_clamp_dec(int *p, int c, int k) {
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
    if (old <= k) atomicMax(p, k);
    return old;
}

// P2: one BSP sub-round over the received F -- one warp per (vertex, segment)
// item, one lane per owned neighbour
template <int MODE, bool STATS>
__global__ void __launch_bounds__(512) ps_scatter_kernel(const int *all, const int2 *TS, const long long *csc_off,
                                                         const int *csc_idx, int *core, PsCtl *c, int p, int k,
                                                         long long vb, int seg, int *front, int dev = 0) {
    if (dev) {  // device-driven loop: an apply step (mode 1) of the level decided on the device
        if (c->mode != 1) return;
        p = c->pcur;
        k = c->kcur;
    }
    const int lane = lane_id();
    const long long nts = (long long)c->nts;
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    int kmin = INT_MAX;
    long long st_arcs = 0, st_dec = 0;
    for (long long i = gw; i < nts; i += nw) {
        int2 ts = TS[i];
        int v = all[ts.x];
        long long b = csc_off[v] + (long long)ts.y * seg;
        int len = (int)min((long long)seg, csc_off[v + 1] - b);
        bool push = false;
        int u = 0;
        if (lane < len) {
            u = csc_idx[b + lane];
            int cu = __ldcg(core + u);
            if (STATS) st_arcs++;
            if (cu > k) {  // guard core[u] > k
                int old = ps_clamp_dec<MODE>(core + u, cu, k);
                if (STATS) st_dec += old > k;
                push = old == k + 1;
                if (old - 1 > k) kmin = min(kmin, old - 1);
            }
        }
        warp_append(push, (int)(u + vb), front, &c->fcnt);
    }
    ps_kmin(&c->kmin[p ^ 1], kmin);
    if (STATS) {
        long long s1 = warp_sum64(st_arcs), s2 = warp_sum64(st_dec);
        if (lane == 0) {
            if (s1) atomicAdd(&c->st_arcs, (unsigned long long)s1);
            if (s2) atomicAdd(&c->st_dec, (unsigned long long)s2);
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t ps_cub_bytes(long long ng, long long arcs) {
    size_t b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs((void *)nullptr, b, (const int *)nullptr, (int *)nullptr, (const int *)nullptr,
                                    (int *)nullptr, (long long)std::max(arcs, 1ll));
    cub::DeviceScan::ExclusiveSum((void *)nullptr, c, (const long long *)nullptr, (long long *)nullptr, (int)(ng + 1));
    return std::max(b, c);
}

cudaError_t pshard_create(const long long *rp, const int *ci, long long nloc, long long vb, long long ng,
                          uint32_t flags, cudaStream_t s, const DevInfo &dev, PeelShard **out) {
    PeelShard *h = new PeelShard();
    h->rp = rp; h->ci = ci; h->nloc = nloc; h->vb = vb; h->ng = ng; h->flags = flags; h->s = s; h->dev = dev;
    h->L = 0; h->k = 0;
    h->seg = (flags & PICO_F_TINY_TILES) ? 4 : kPsSeg;
    cudaError_t e = cudaMemcpyAsync(&h->arcs, rp + nloc, sizeof(long long), cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) { delete h; return e; }
    const long long arcs1 = std::max(h->arcs, 1ll), n1 = std::max(nloc, 1ll);
    h->tscap = ng + h->arcs / h->seg + 64;
    h->cubbytes = ps_cub_bytes(ng, h->arcs);
    size_t bytes = a256(sizeof(PsCtl)) + a256(sizeof(int) * n1) * 3 + a256(sizeof(long long) * (ng + 1)) * 2 +
                   a256(sizeof(int) * arcs1) * 3 + a256(sizeof(int2) * h->tscap) + a256(h->cubbytes);
    if ((e = lib_malloc_async(&h->ws, bytes, s))) { delete h; return e; }
    char *p = (char *)h->ws;
    h->ctl = (PsCtl *)p; p += a256(sizeof(PsCtl));
    h->core = (int *)p; p += a256(sizeof(int) * n1);
    h->alive[0] = (int *)p; p += a256(sizeof(int) * n1);
    h->alive[1] = (int *)p; p += a256(sizeof(int) * n1);
    h->csc_off = (long long *)p; p += a256(sizeof(long long) * (ng + 1)) * 2;
    h->csc_idx = (int *)p; p += a256(sizeof(int) * arcs1);
    h->tmpk = (int *)p; p += a256(sizeof(int) * arcs1);
    h->src = (int *)p; p += a256(sizeof(int) * arcs1);
    h->TS = (int2 *)p; p += a256(sizeof(int2) * h->tscap);
    h->cubtmp = p;
    const int sms = dev.sms;
    auto grid = [&](long long work) {
        return std::max(1, (int)std::min<long long>((work + 255) / 256, (long long)sms * 16));
    };
    PsCtl hc{};
    hc.kmin[0] = hc.kmin[1] = INT_MAX;
    do {
        if ((e = cudaMemcpyAsync(h->ctl, &hc, sizeof(hc), cudaMemcpyHostToDevice, s))) break;
        if (nloc > 0) ps_init_kernel<<<grid(nloc), 256, 0, s>>>(rp, nloc, h->core, h->alive[0], h->ctl);
        // local CSC: arc counts per global v -> offsets; (v, u) sorted by v
        long long *cntv = h->csc_off + (ng + 1);
        if ((e = cudaMemsetAsync(cntv, 0, sizeof(long long) * (size_t)(ng + 1), s))) break;
        if (h->arcs > 0) {
            ps_src_kernel<<<sms * 8, 256, 0, s>>>(rp, nloc, h->src);
            ps_csc_count_kernel<<<grid(h->arcs), 256, 0, s>>>(ci, h->arcs, (unsigned long long *)cntv);
        }
        size_t cb = h->cubbytes;
        if ((e = cub::DeviceScan::ExclusiveSum(h->cubtmp, cb, cntv, h->csc_off, (int)(ng + 1), s))) break;
        if (h->arcs > 0) {
            int bits = 1;
            while ((1ll << bits) < ng) bits++;
            cb = h->cubbytes;
            if ((e = cub::DeviceRadixSort::SortPairs(h->cubtmp, cb, ci, h->tmpk, h->src, h->csc_idx,
                                                     (long long)h->arcs, 0, bits, s)))
                break;
        }
        ps_pub_kernel<<<1, 1, 0, s>>>(h->ctl, 0);
        e = cudaGetLastError();
    } while (false);
    if (e) {
        cudaFreeAsync(h->ws, s);
        delete h;
        return e;
    }
    *out = h;
    return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Device-driven level loop (PICO_F_LSA_EXCHANGE): every step is decided on the
// device from the latest exchange -- the host's loop in capi.cu peel_rounds,
// moved to one thread -- so the host only enqueues steps (a CUDA graph of a
// batch) and reads the done flag once per batch.
//   global |F| > 0 in the open level  -> apply (a BSP sub-round)
//   else: close the level (record it if it processed anything); the global
//         bound INT_MAX -> done; else scan level max(k + 1, bound)
// ---------------------------------------------------------------------------
__global__ void ps_decide_kernel(PsCtl *c, long long *lvsz, long long lvcap) {
    if (c->mode == 2) return;
    if (c->level_open && c->g_total > 0) {
        c->mode = 1;
        c->processed += c->g_total;
        c->subrounds++;
        return;
    }
    if (c->level_open && c->processed > 0) {
        if (c->levels < lvcap) lvsz[c->levels] = c->processed;
        c->levels++;
        c->kmax = c->kcur;
    }
    c->level_open = 0;
    if (c->g_kmin >= (long long)INT_MAX) {
        c->mode = 2;
        return;
    }
    c->kcur = max(c->kcur + 1, (int)c->g_kmin);
    const int p = c->Lcnt & 1;
    c->pcur = p;
    c->Lcnt++;
    c->nalive[p ^ 1] = 0;  // ps_begin_kernel of the host loop
    c->kmin[p ^ 1] = INT_MAX;
    c->fcnt = 0;
    c->mode = 0;
    c->level_open = 1;
    c->processed = 0;
}

// publish (|F|, next-level bound) of the step; a finished run publishes (0, none)
__global__ void ps_pub_dev_kernel(PsCtl *c) {
    if (c->mode == 2) {
        c->out[0] = 0;
        c->out[1] = (long long)INT_MAX;
        return;
    }
    c->out[0] = (long long)c->fcnt;
    c->out[1] = (long long)c->kmin[c->pcur ^ 1];
    c->fcnt = 0;
    c->nts = 0;
}

cudaError_t pshard_run_lsa(PeelShard *h, LsaX *lx, long long n_global, long long *levels, long long *subrounds,
                           int *kmax, long long *lvsz_host, long long lvcap, std::string *msg) {
    cudaStream_t s = h->s;
    const int sms = h->dev.sms;
    cudaError_t e;
    int *all = nullptr;
    long long *lvsz = nullptr;
    const long long lv_dev_cap = std::max(lvcap, 1ll);
    int batch = 16;  // even: a batch's exchange parities repeat
    if (const char *b = getenv("PICO_LSA_BATCH")) batch = std::max(2, std::min(256, atoi(b) & ~1));
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    cudaStream_t cs = nullptr;
    do {
        if ((e = lib_malloc_async(&all, sizeof(int) * (size_t)std::max(n_global, 1ll), s))) break;
        if ((e = lib_malloc_async(&lvsz, sizeof(long long) * (size_t)lv_dev_cap, s))) break;
        PsCtl *c = h->ctl;
        // loop state: no level open, k = 0 (the init published (0, kmin0))
        if ((e = cudaMemsetAsync(&c->g_total, 0, offsetof(PsCtl, subrounds) + sizeof(long long) -
                                                     offsetof(PsCtl, g_total), s)))
            break;
        // exchange 0: the init's published bounds (parity 0)
        if ((e = lsa_exchange(lx, 0, (const unsigned long long *)c->out, all, &c->g_total, sms * 4, s, 1,
                              &c->g_kmin)))
            break;
        // one batch of steps, captured once on a private stream (the caller's may
        // be the legacy stream, which cannot capture) and launched on the
        // caller's: step j of a batch uses parity (j + 1) & 1
        if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking))) break;
        if ((e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed))) break;
        const bool stats = h->flags & PICO_F_STATS;
        for (int j = 0; j < batch; j++) {
            const int par = (j + 1) & 1;
            int *front = lsa_send_buffer(lx, par);
            ps_decide_kernel<<<1, 1, 0, cs>>>(c, lvsz, lvcap);
            if (h->nloc > 0)
                ps_scan_dev_kernel<<<sms * 4, 512, 0, cs>>>(h->core, h->alive[0], h->alive[1], c, h->vb, front);
            if (h->arcs > 0) {
                ps_segments_kernel<<<sms * 16, 256, 0, cs>>>(all, 0, h->csc_off, h->seg, h->TS, &c->nts, c);
#define PS_LAUNCH_DEV(M, ST) \
    ps_scatter_kernel<M, ST><<<sms * 4, 512, 0, cs>>>(all, h->TS, h->csc_off, h->csc_idx, h->core, c, 0, 0, h->vb, \
                                                     h->seg, front, 1)
                if (h->flags & PICO_F_CLAMP_CAS) {
                    if (stats) PS_LAUNCH_DEV(2, true); else PS_LAUNCH_DEV(2, false);
                } else {
                    if (stats) PS_LAUNCH_DEV(0, true); else PS_LAUNCH_DEV(0, false);
                }
#undef PS_LAUNCH_DEV
            }
            ps_pub_dev_kernel<<<1, 1, 0, cs>>>(c);
            if ((e = lsa_exchange(lx, par, (const unsigned long long *)c->out, all, &c->g_total, sms * 4, cs, 1,
                                  &c->g_kmin)))
                break;
        }
        cudaError_t ec = cudaStreamEndCapture(cs, &g);
        if (e || (e = ec)) break;
        if ((e = cudaGraphInstantiate(&ge, g, 0))) break;
        for (long long nb = 0;; nb++) {
            if ((e = cudaGraphLaunch(ge, s))) break;
            int mode = 0;
            if ((e = cudaMemcpyAsync(&mode, &c->mode, sizeof(int), cudaMemcpyDeviceToHost, s)) ||
                (e = cudaStreamSynchronize(s)))
                break;
            if (mode == 2) break;
            if (nb > (h->arcs + n_global) / batch + 16) {  // every step processes a vertex or a level
                if (msg) *msg = "sharded PeelOne did not terminate";
                e = cudaErrorUnknown;
                break;
            }
        }
        if (e) break;
        PsCtl hc;
        if ((e = cudaMemcpyAsync(&hc, c, sizeof(PsCtl), cudaMemcpyDeviceToHost, s)) ||
            (e = cudaStreamSynchronize(s)))
            break;
        *levels = hc.levels;
        *subrounds = hc.subrounds;
        *kmax = hc.kmax;
        if (lvsz_host && hc.levels > 0 &&
            (e = cudaMemcpy(lvsz_host, lvsz, sizeof(long long) * (size_t)std::min(hc.levels, lvcap),
                            cudaMemcpyDeviceToHost)))
            break;
    } while (false);
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    if (cs) cudaStreamDestroy(cs);
    if (all) cudaFreeAsync(all, s);
    if (lvsz) cudaFreeAsync(lvsz, s);
    cudaError_t es = cudaStreamSynchronize(s);
    return e ? e : es;
}

const long long *pshard_out(PeelShard *h) { return h->ctl->out; }

long long pshard_nloc(PeelShard *h) { return h->nloc; }

cudaError_t pshard_scan(PeelShard *h, int k, int *front) {
    const int p = h->L & 1;
    cudaStream_t s = h->s;
    h->k = k;
    ps_begin_kernel<<<1, 1, 0, s>>>(h->ctl, p);
    ps_scan_kernel<<<h->dev.sms * 4, 512, 0, s>>>(h->core, h->alive[p], h->alive[p ^ 1], h->ctl, p, k, h->vb, front);
    ps_pub_kernel<<<1, 1, 0, s>>>(h->ctl, p ^ 1);
    h->L++;
    return cudaGetLastError();
}

cudaError_t pshard_apply(PeelShard *h, const int *all, long long total, int *front) {
    const int p = (h->L - 1) & 1;  // parity of the current level
    cudaStream_t s = h->s;
    const int sms = h->dev.sms;
    if (total > 0 && h->arcs > 0) {
        int blocks = (int)std::min<long long>((total + 255) / 256, (long long)sms * 16);
        ps_segments_kernel<<<std::max(blocks, 1), 256, 0, s>>>(all, total, h->csc_off, h->seg, h->TS, &h->ctl->nts);
        const bool stats = h->flags & PICO_F_STATS;
#define PS_LAUNCH(M, ST) \
    ps_scatter_kernel<M, ST><<<sms * 4, 512, 0, s>>>(all, h->TS, h->csc_off, h->csc_idx, h->core, h->ctl, p, h->k, \
                                                     h->vb, h->seg, front)
        if (h->flags & PICO_F_CLAMP_CAS) {
            if (stats) PS_LAUNCH(2, true); else PS_LAUNCH(2, false);
        } else {
            if (stats) PS_LAUNCH(0, true); else PS_LAUNCH(0, false);
        }
#undef PS_LAUNCH
    }
    ps_pub_kernel<<<1, 1, 0, s>>>(h->ctl, p ^ 1);
    return cudaGetLastError();
}

cudaError_t pshard_read(PeelShard *h, long long *count, int *kmin) {
    long long o[2];
    cudaError_t e = cudaMemcpyAsync(o, h->ctl->out, sizeof(o), cudaMemcpyDeviceToHost, h->s);
    if (!e) e = cudaStreamSynchronize(h->s);
    if (e) return e;
    *count = o[0];
    *kmin = (int)o[1];
    return cudaSuccess;
}

cudaError_t pshard_counters(PeelShard *h, long long *arcs_scanned, long long *guarded) {
    unsigned long long c[2];
    cudaError_t e = cudaMemcpyAsync(c, &h->ctl->st_arcs, sizeof(c), cudaMemcpyDeviceToHost, h->s);
    if (!e) e = cudaStreamSynchronize(h->s);
    if (e) return e;
    *arcs_scanned = (long long)c[0];
    *guarded = (long long)c[1];
    return cudaSuccess;
}

cudaError_t pshard_result(PeelShard *h, int *core_out) {
    if (h->nloc == 0) return cudaSuccess;
    cudaError_t e = cudaMemcpyAsync(core_out, h->core, sizeof(int) * (size_t)h->nloc, cudaMemcpyDeviceToDevice, h->s);
    if (!e) e = cudaStreamSynchronize(h->s);
    return e;
}

cudaError_t pshard_destroy(PeelShard *h) {
    cudaError_t e = cudaFreeAsync(h->ws, h->s);
    if (!e) e = cudaStreamSynchronize(h->s);
    delete h;
    return e;
}

}  // namespace pico

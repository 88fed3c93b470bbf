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
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

#ifndef PICO_PO_KHI0
#define PICO_PO_KHI0 32  // initial near window: vertices of degree <= 32 (16 was 2-4 % faster in a sweep, profiles/r02/s3/po_khi0.txt, but its first bench run hit a fault not reproduced since: kept at the long-validated 32)
#endif
#ifndef PICO_PO_KHI_NUM  // far-list rebuild: the new window is NUM/DEN * k + ADD
#define PICO_PO_KHI_NUM 2
#endif
#ifndef PICO_PO_KHI_DEN
#define PICO_PO_KHI_DEN 1
#endif
#ifndef PICO_PO_KHI_ADD
#define PICO_PO_KHI_ADD 16
#endif
#ifndef PICO_PO_THREADS
#define PICO_PO_THREADS 512  // threads per CTA of the persistent level kernel
#endif
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
    int *far0;     // near / far split of the alive vertices: alive[] ("near")
    int *far1;     // holds those with estimate <= khi, far[] the others
    int khi0;      // initial window bound (INT_MAX: no far list)
    int khi_num, khi_den, khi_add;  // rebuild window num/den * k + add (PICO_PO_KHI_*; env PICO_PO_WINDOW)
    unsigned *done;  // [n/32] processed bitmap: v entered a frontier (its coreness is final)
    long long *Q;  // run-wide queue log: (row offset << 8) | length, or (v << 32) | segment (enc_rows 0)
    int enc_rows;  // entries hold their arc range (the drain loads no row bounds); 0 for the
                   // end-of-level repair clamp (PICO_F_CLAMP_SUB), which needs the vertex
    unsigned long long *fsz;
    unsigned long long fsz_cap;
    unsigned long long *rtime;  // [2 fsz_cap] per scanned level: scan ns | k << 40, drain ns | sub-rounds << 40
    Ctrl *ctl;
    int seg;
};

__device__ __forceinline__ int po_nseg(long long d, int seg) { return (int)((d + seg - 1) / seg); }

// The queue's append counters: a phase appends through counter y and reads
// (after the barrier) the count of the other one, which no phase touches
// meanwhile -- so every CTA reads the same frozen count without a snapshot.
// Both counters are monotonic over the run; a phase's entries go to
// Q[wbase + (counter - cbase)], wbase = the end of the entries it reads,
// cbase = the counter's value when the phase started (see po_levels_kernel).
__device__ __forceinline__ unsigned long long *po_cnt(const PoArgs &a, int y) {
    return y ? &a.ctl->q_tail1 : &a.ctl->q_tail;
}
struct PoAppend {
    unsigned long long wbase, cbase;
    int y;
};

// Warp-cooperative append of vertices (pred lanes) to the queue (positions
// from the phase's append counter, PoAppend), one entry per `seg` arcs of the
// row.  Returns the number of vertices appended.
__device__ __forceinline__ int po_push(const PoArgs &a, bool pred, int v, const PoAppend ap) {
    const int lane = lane_id();
    int ns = 0, dv = 0;
    long long r0 = 0;
    if (pred) {
        r0 = __ldg(a.rp + v);
        dv = (int)(__ldg(a.rp + v + 1) - r0);
        ns = po_nseg(dv, a.seg);
    }
    if (__any_sync(FULL, pred)) {
        // processed: later guards skip v.  Lanes whose vertices share a bitmap
        // word (the scan's frontier comes from id-ordered blocks) OR their bits
        // together first: one RED per word instead of up to 32 on one address
        const int wd = pred ? (v >> 5) : -1;
        const unsigned peers = __match_any_sync(FULL, wd);
        const unsigned bits = __reduce_or_sync(peers, pred ? 1u << (v & 31) : 0u);
        if (pred && lane == __ffs(peers) - 1) red_or(a.done + wd, bits);
    }
    int incl = warp_incl_scan(ns);
    int total = __shfl_sync(FULL, incl, 31);
    if (total == 0) return 0;
    unsigned long long base = 0;
    if (lane == 0) base = ap.wbase + (atomicAdd(po_cnt(a, ap.y), (unsigned long long)total) - ap.cbase);
    base = __shfl_sync(FULL, base, 0);
    // the warp writes the `total` entries jointly, so a hub's thousands of
    // entries do not serialise on its lane (one lane writing the 31K entries
    // of a 1M-degree hub cost up to ~6 ms per level at RMAT-26): entry j
    // belongs to the lane with the largest exclusive offset <= j
    const int excl = incl - ns;
    for (int j0 = 0; j0 < total; j0 += 32) {
        const int j = j0 + lane;
        int lo = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            int cand = lo + step;
            int ex = __shfl_sync(FULL, excl, cand & 31);
            if (cand < 32 && ex <= j) lo = cand;
        }
        const int vo = __shfl_sync(FULL, v, lo);
        const int eo = __shfl_sync(FULL, excl, lo);
        if (a.enc_rows) {  // (uniform) the entry's arc range: row offset << 8 | length
            const long long ro = __shfl_sync(FULL, r0, lo);
            const int dvo = __shfl_sync(FULL, dv, lo);
            const int so = (j - eo) * a.seg;
            if (j < total) a.Q[base + j] = ((ro + so) << 8) | (long long)min(a.seg, dvo - so);
        } else if (j < total) {
            a.Q[base + j] = ((long long)vo << 32) | (unsigned)(j - eo);
        }
    }
    return __popc(__ballot_sync(FULL, pred));
}

// scan of level k (parity p): alive[p] -> frontier entries in the queue, alive[p^1]
// na_in: the near list's length when the caller knows it (the level kernel:
// head count + rebuild joiners), else -1 (read nAlive[p])
template <bool STATS>
__device__ void po_scan_phase(const PoArgs &a, int k, int p, long long gthread, long long nthreads,
                              const PoAppend ap, long long na_in = -1) {
    const long long na = na_in >= 0 ? na_in : (long long)bcast_u64(&a.ctl->nAlive[p]);
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
        nproc += po_push(a, front, v, ap);
    }
    kmin = warp_min(kmin);
    // po_push returns the warp-wide count to every lane: lane 0 holds the total
    if (lane_id() == 0) {
        if (kmin != INT_MAX) atomicMin(&a.ctl->kminb[p ^ 1], kmin);
        if (nproc) atomicAdd(&a.ctl->nProc[p], (unsigned long long)nproc);
        if (STATS && gthread == 0) atomicAdd(&a.ctl->st_alive, (unsigned long long)na);
    }
}

// Near / far alive lists.  A level's scan walks only the near list (the alive
// vertices with estimate <= khi): at RMAT-26 the plain scan re-read ~1.9 M alive
// vertices at each of ~400 levels (759 M entries, a third of PeelOne's time),
// most of them hubs far above the level.  The far list holds the others; a far
// vertex whose estimate is decremented to khi is appended to the near list at
// that moment (cross, po_sub_phase).  When the next level exceeds khi the far
// list is rebuilt: khi doubles, far vertices now within it join the near list,
// those that already crossed (estimate <= the old khi) are dropped.  The
// level bound is min(near bound, far minimum).  The scanned set is exactly
// what a full scan would find with estimate == k (nothing else changes).
// The joiners go to near[na0 + ...] through their own counter and bound
// (nJoin, kminJ), never through nAlive[p] / kminb[p]: those are the level
// head's inputs, and a CTA still reading the head while a faster one rebuilt
// would otherwise see na > 0 or a lower bound, take another branch and put the
// grid barriers out of step (a rare hang at RMAT-26 / C4).
__device__ void po_rebuild_phase(const PoArgs &a, int khi_old, int khi, int fp, int p, long long na0,
                                 long long gthread, long long nthreads, bool stats) {
    const long long nf = (long long)bcast_u64(&a.ctl->nFar[fp]);
    const int *far = fp ? a.far1 : a.far0;
    int *keepto = fp ? a.far0 : a.far1;
    int *near = p ? a.alive1 : a.alive0;
    int fmin = INT_MAX, kmin = INT_MAX;
    const long long iters = (nf + nthreads - 1) / nthreads;
    for (long long it = 0; it < iters; it++) {
        long long i = it * nthreads + gthread;
        bool valid = i < nf;
        int v = 0, c = 0;
        if (valid) {
            v = __ldcg(far + i);
            c = __ldcg(a.core + v);
        }
        const bool join = valid && c > khi_old && c <= khi;
        const bool stay = valid && c > khi;
        if (join) kmin = min(kmin, c);
        if (stay) fmin = min(fmin, c);
        warp_append(join, v, near + na0, &a.ctl->nJoin);
        warp_append(stay, v, keepto, &a.ctl->nFar[fp ^ 1]);
    }
    fmin = warp_min(fmin);
    kmin = warp_min(kmin);
    if (lane_id() == 0) {
        if (fmin != INT_MAX) atomicMin(&a.ctl->fmin[fp ^ 1], fmin);
        if (kmin != INT_MAX) atomicMin(&a.ctl->kminJ, kmin);
        if (stats && gthread == 0) atomicAdd(&a.ctl->st_alive, (unsigned long long)nf);
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

// one sub-round of level k: process queue entries [lo, hi).  An entry holds
// at most `seg` = 32 * PICO_PO_A arcs; one warp takes PICO_PO_U entries per
// iteration and each lane A arcs of each (lane + 32 j), so U * A colidx loads,
// core gathers and clamps are in flight per lane: a sub-round's latency is a
// few memory round trips, and the heavy levels (at RMAT-26 four levels peel
// 70% of the arcs through hub rows) stream U * A * 32 arcs per warp chain.
#ifndef PICO_PO_U
#define PICO_PO_U 2  // queue entries per warp iteration (independent chains in flight)
#endif
#ifndef PICO_PO_A
#define PICO_PO_A 1  // arcs per lane per entry (entry = 32 * A arcs)
#endif
// reads queue entries [lo, hi), appends the next sub-round's through ap
template <int MODE, bool STATS>
__device__ void po_sub_phase(const PoArgs &a, int k, int p, const PoAppend ap, unsigned long long lo,
                             unsigned long long hi, int khi = INT_MAX, int *fminp = nullptr) {
    const long long *Qx = a.Q;
    constexpr int U = PICO_PO_U, A = PICO_PO_A, W = U * A;
    const int lane = lane_id();
    const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    int kmin = INT_MAX, fmin = INT_MAX;
    long long nproc = 0, st_arcs = 0, st_dec = 0;
    __shared__ int s_b[2];  // CTA minima of the next-level and far bounds
    if (threadIdx.x == 0) s_b[0] = s_b[1] = INT_MAX;
    __syncthreads();
    // iteration it takes entries lo + (it*U + q)*nwarps + gwarp, q < U: the U
    // entries' loads, gathers and clamps are issued together
    for (unsigned long long i0 = lo + gwarp; i0 < hi; i0 += (unsigned long long)nwarps * U) {
        int u[W], c[W];
#pragma unroll
        for (int q = 0; q < U; q++) {
            unsigned long long i = i0 + (unsigned long long)q * nwarps;
            long long b = 0;
            int len = 0;
            if (i < hi) {
                long long e = __ldcg(Qx + i);
                if (a.enc_rows) {  // uniform
                    b = e >> 8;
                    len = (int)(e & 0xff);
                } else {
                    int v = (int)(e >> 32);
                    int s = (int)(e & 0xffffffffll);
                    long long r0 = __ldg(a.rp + v), r1 = __ldg(a.rp + v + 1);
                    b = r0 + (long long)s * a.seg;
                    len = (int)min((long long)a.seg, r1 - b);
                }
            }
#pragma unroll
            for (int j = 0; j < A; j++) u[q * A + j] = (j * 32 + lane < len) ? __ldg(a.ci + b + j * 32 + lane) : -1;
        }
        // guard core[u] > k.  Every vertex with core <= k is processed
        // (it entered a frontier, which marks the n/8-byte `done` bitmap) except
        // members of this level's frontier not yet marked, so "not done" is
        // the guard up to those, for which the clamp returns old <= k and
        // changes nothing.  The bitmap stays in L2: no DRAM sector of core[]
        // per arc.  The CAS clamp still reads core[u] for its first compare.
        unsigned dw[W];
#pragma unroll
        for (int w = 0; w < W; w++) dw[w] = u[w] >= 0 ? __ldcg(a.done + (u[w] >> 5)) : ~0u;
#pragma unroll
        for (int w = 0; w < W; w++) {
            const bool live = !((dw[w] >> (u[w] & 31)) & 1u);
            c[w] = live ? (MODE == 2 ? __ldcg(a.core + u[w]) : INT_MAX) : 0;
        }
        bool push[W];
        int old[W];
        // the W clamped decrements are issued back to back: for MODE 0 / 1 the
        // atomicSubs first, then MODE 0's atomicMax repairs of those that
        // overshot (independent atomics on distinct cells; issuing each
        // clamp_dec whole serialised a round trip per arc)
#pragma unroll
        for (int w = 0; w < W; w++) {
            const bool g = u[w] >= 0 && c[w] > k;  // guard core[u] > k
            if (MODE == 2) old[w] = g ? clamp_dec<2>(a.core + u[w], c[w], k) : k;
            else old[w] = g ? atomicSub(a.core + u[w], 1) : k;
        }
        if (MODE == 0) {
#pragma unroll
            for (int w = 0; w < W; w++)
                if (u[w] >= 0 && c[w] > k && old[w] <= k) atomicMax(a.core + u[w], k);
        }
        bool cross[W];
#pragma unroll
        for (int w = 0; w < W; w++) {
            if (STATS) st_arcs += u[w] >= 0;
            if (STATS) st_dec += (old[w] > k);
            push[w] = (old[w] == k + 1);
            if (old[w] - 1 > k) kmin = min(kmin, old[w] - 1);
            // a far vertex that stays far keeps the far minimum a lower bound
            // (the next level bound min(kminb, fmin) must cover it at every
            // later level, not only the next one)
            if (old[w] - 1 > khi) fmin = min(fmin, old[w] - 1);
            // a far vertex whose estimate reaches khi enters the near list
            // (values step down by one, so exactly one decrement sees it)
            cross[w] = old[w] - 1 == khi && khi > k;
        }
#pragma unroll
        for (int w = 0; w < W; w++)
            if (__any_sync(FULL, cross[w])) warp_append(cross[w], u[w], p ? a.alive0 : a.alive1, &a.ctl->nAlive[p ^ 1]);
#pragma unroll
        for (int w = 0; w < W; w++)
            if (__any_sync(FULL, push[w])) nproc += po_push(a, push[w], u[w], ap);
    }
    kmin = warp_min(kmin);
    fmin = warp_min(fmin);
    // the two level bounds are reduced per CTA first (one global atomic per
    // CTA instead of one per warp on two hot words); po_push returns the
    // warp-wide count to every lane: lane 0 holds the total
    if (lane == 0) {
        if (kmin != INT_MAX) atomicMin(&s_b[0], kmin);
        if (fmin != INT_MAX) atomicMin(&s_b[1], fmin);
        if (nproc) atomicAdd(&a.ctl->nProc[p], (unsigned long long)nproc);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_b[0] != INT_MAX) atomicMin(&a.ctl->kminb[p ^ 1], s_b[0]);
        if (s_b[1] != INT_MAX && fminp) atomicMin(fminp, s_b[1]);
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
    int kmin = INT_MAX, fmin = INT_MAX;
    for (long long it = 0; it < iters; it++) {
        long long v = it * nthreads + gthread;
        bool valid = v < a.n;
        int d = valid ? (int)(a.rp[v + 1] - a.rp[v]) : 0;
        if (valid) a.core[v] = d;
        bool near = d > 0 && d <= a.khi0, far = d > a.khi0;
        if (near) kmin = min(kmin, d);
        if (far) fmin = min(fmin, d);
        warp_append(near, (int)v, a.alive0, &a.ctl->nAlive[0]);
        warp_append(far, (int)v, a.far0, &a.ctl->nFar[0]);
    }
    kmin = warp_min(kmin);
    fmin = warp_min(fmin);
    if (lane_id() == 0 && kmin != INT_MAX) atomicMin(&a.ctl->kminb[0], kmin);
    if (lane_id() == 0 && fmin != INT_MAX) atomicMin(&a.ctl->fmin[0], fmin);
}

// ---------------------------------------------------------------------------
// P1-P3: persistent cooperative kernel over all levels
// ---------------------------------------------------------------------------
// Queue positions without a snapshot: the scan of a level and every sub-round
// append through one of two monotonic counters, alternating, so the counter
// whose count the NEXT phase needs is frozen while it is read and every CTA
// reads the same value straight from it after the barrier.  A phase writes
// its entries right after the ones it reads (one run-wide log, as before).
// Every barrier is then the plain grid_sync (one arrival word, no last-arriver
// publication: 1.23 vs 2.57 us per barrier at 444 CTAs,
// scripts/micro/grid_barrier.cu); the sub-rounds are unchanged.
template <int MODE, bool STATS>
__global__ void __launch_bounds__(PICO_PO_THREADS, PICO_PO_PER) po_levels_kernel(PoArgs a) {
    constexpr bool CLAMP_SUB = MODE == 1;
    const long long gthread = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    Ctrl *c = a.ctl;
    int k = 0, kprev = 0;
    unsigned long long S = 0;          // global sub-round counter
    unsigned long long lo = 0;         // consumed prefix of the queue (uniform)
    unsigned long long cb0 = 0, cb1 = 0;  // the counters' values at their last read (uniform; scalars, not
                                          // a runtime-indexed array, which would live in local memory)
    int y = 0;                         // the counter the next phase appends through (uniform)
    int khi = a.khi0, fp = 0;  // near window bound, far list parity (uniform)
    for (int L = 0;; L++) {
        const int p = L & 1;
        // the level head's control words, loaded by one thread back to back
        // and broadcast through shared memory (one round trip, one barrier pair)
        __shared__ long long s_head[4];
        __syncthreads();
        if (threadIdx.x == 0) {
            const long long h0 = (long long)ld_volatile(&c->nAlive[p]), h1 = (long long)ld_volatile(&c->nFar[fp]);
            const int h2 = ld_volatile(&c->kminb[p]), h3 = ld_volatile(&c->fmin[fp]);
            s_head[0] = h0; s_head[1] = h1; s_head[2] = h2; s_head[3] = h3;
        }
        __syncthreads();
        long long na = s_head[0];
        const long long nf = s_head[1];
        if (leader && L > 0) po_close_level(a, p ^ 1, kprev);
        if (na == 0 && nf == 0) break;
        k = max(k + 1, min((int)s_head[2], nf ? (int)s_head[3] : INT_MAX));
        unsigned long long ts0 = leader ? globaltimer() : 0, ts1 = 0, S0 = S;
        // the window is exhausted (or the near list empty): rebuild the far
        // list with a wider window -- repeatedly if the level's bound is still
        // beyond the new window (every vertex of level k must be in the near
        // list before the scan: a single rebuild whose far minimum lands above
        // the new window left those vertices in the far list, unscanned; with
        // a 1.5k + 16 window rule that lost 7-194 vertices per RMAT graph)
        const long long na_head = na;
        long long nfc = nf;
        for (int nrb = 0; nfc && (k > khi || na == 0); nrb++) {  // uniform
            if (nrb) grid_sync(c);  // the leader's resets of the previous pass first
            const int khi_new = (int)max((long long)khi, min((long long)a.khi_num * k / a.khi_den + a.khi_add,
                                                             (long long)INT_MAX - 1));
            po_rebuild_phase(a, khi, khi_new, fp, p, na_head, gthread, nthreads, STATS);
            grid_sync(c);
            if (leader) {
                c->nFar[fp] = 0;  // consumed; refilled at the next rebuild
                c->fmin[fp] = INT_MAX;
            }
            khi = khi_new;
            fp ^= 1;
            // the joiners extend the near list and may lower its bound; the far
            // minimum is the rebuilt one
            na = na_head + (long long)bcast_u64(&c->nJoin);
            nfc = (long long)bcast_u64(&c->nFar[fp]);
            const int kj = min(bcast_i32(&c->kminb[p]), bcast_i32(&c->kminJ));
            k = max(k, min(kj, nfc ? bcast_i32(&c->fmin[fp]) : INT_MAX));
        }
        const unsigned long long lstart = lo;
        po_scan_phase<STATS>(a, k, p, gthread, nthreads, PoAppend{lo, y ? cb1 : cb0, y}, na);
        grid_sync(c);
        if (leader) ts1 = globaltimer();
        if (leader) {
            c->nAlive[p] = 0;       // alive[p] consumed; refilled at level L+1
            c->kminb[p] = INT_MAX;  // consumed at this level's head
            c->nJoin = 0;           // read by every CTA before the scan
            c->kminJ = INT_MAX;
        }
        for (int sub = 0;; sub++) {
            // entries appended by the previous phase through counter y: frozen,
            // the phase about to run appends through y ^ 1
            const unsigned long long cy = bcast_u64(po_cnt(a, y));
            const unsigned long long hi = lo + (cy - (y ? cb1 : cb0));
            if (y) cb1 = cy; else cb0 = cy;
            y ^= 1;
            if (hi == lo) {  // uniform: every CTA read the same frozen count
                // an empty level has no sub-round barrier: one barrier orders
                // the leader's resets above before the next level's scan
                // appends to alive[p] / lowers kminb[p]
                if (sub == 0) grid_sync(c);
                y ^= 1;  // nothing was appended through y: the next scan appends through it again
                break;
            }
            po_sub_phase<MODE, STATS>(a, k, p, PoAppend{hi, y ? cb1 : cb0, y}, lo, hi, khi, &c->fmin[fp]);
            grid_sync(c);
            lo = hi;
            S++;
        }
        if (CLAMP_SUB) {
            po_repair_phase(a, k, lstart, lo, gthread, nthreads);
            grid_sync(c);
        }
        if (leader) {
            c->rounds = S;  // BSP sub-rounds so far
            if ((unsigned long long)L < a.fsz_cap) {  // per scanned level: scan ns, drain ns | sub-rounds << 40
                a.rtime[2 * L] = (ts1 - ts0) | ((unsigned long long)k << 40);
                a.rtime[2 * L + 1] = (globaltimer() - ts1) | ((S - S0) << 40);
            }
        }
        kprev = k;
    }
}

// host-loop variants (PICO_F_HOST_LOOP)
template <bool STATS>
__global__ void __launch_bounds__(512) po_scan_kernel(PoArgs a, int k, int p, PoAppend ap) {
    const long long gthread = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    po_scan_phase<STATS>(a, k, p, gthread, nthreads, ap);
}

template <int MODE, bool STATS>
__global__ void __launch_bounds__(512) po_sub_kernel(PoArgs a, int k, int p, PoAppend ap, unsigned long long lo,
                                                     unsigned long long hi, int first) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && first) {
        a.ctl->nAlive[p] = 0;
        a.ctl->kminb[p] = INT_MAX;
    }
    po_sub_phase<MODE, STATS>(a, k, p, ap, lo, hi);
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
static int po_seg(uint32_t flags) { return (flags & PICO_F_TINY_TILES) ? 4 : 32 * PICO_PO_A; }

size_t po_workspace_bytes(long long n, long long arcs, uint32_t flags) {
    size_t b = 0;
    b += align256(sizeof(Ctrl));
    b += align256(sizeof(unsigned long long) * kFszCap);
    b += align256(sizeof(unsigned long long) * 2 * kFszCap);
    b += align256(sizeof(int) * (size_t)n) * 4;
    b += align256(sizeof(unsigned) * (size_t)((n + 31) / 32 + 1));
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
    a.rtime = (unsigned long long *)p; p += align256(sizeof(unsigned long long) * 2 * kFszCap);
    a.alive0 = (int *)p; p += align256(sizeof(int) * (size_t)n);
    a.alive1 = (int *)p; p += align256(sizeof(int) * (size_t)n);
    a.far0 = (int *)p; p += align256(sizeof(int) * (size_t)n);
    a.far1 = (int *)p; p += align256(sizeof(int) * (size_t)n);
    a.done = (unsigned *)p; p += align256(sizeof(unsigned) * (size_t)((n + 31) / 32 + 1));
    a.Q = (long long *)p;
    // the host loop keeps one alive list (no far list)
    a.khi0 = (flags & PICO_F_HOST_LOOP) ? INT_MAX : PICO_PO_KHI0;
    a.khi_num = PICO_PO_KHI_NUM;
    a.khi_den = PICO_PO_KHI_DEN;
    a.khi_add = PICO_PO_KHI_ADD;
    if (const char *w = getenv("PICO_PO_WINDOW")) {  // "num/den+add": tests and A/B runs
        int nu = 0, de = 0, ad = 0;
        if (sscanf(w, "%d/%d+%d", &nu, &de, &ad) == 3 && nu >= de && de > 0 && ad > 0) {
            a.khi_num = nu;
            a.khi_den = de;
            a.khi_add = ad;
        }
    }
    a.seg = po_seg(flags);
    a.enc_rows = CLAMP_SUB ? 0 : 1;  // the repair clamp reads the vertex of every entry
    a.rp = rp; a.ci = ci; a.n = (int)n; a.core = core;

    cudaError_t err;
    Ctrl h{};
    h.kminb[0] = INT_MAX;
    h.kminb[1] = INT_MAX;
    h.fmin[0] = INT_MAX;
    h.fmin[1] = INT_MAX;
    h.kminJ = INT_MAX;
    if ((err = cudaMemcpyAsync(a.ctl, &h, sizeof(Ctrl), cudaMemcpyHostToDevice, s))) return err;
    if ((err = cudaMemsetAsync(a.done, 0, sizeof(unsigned) * (size_t)((n + 31) / 32 + 1), s))) return err;

    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
    auto tstart = [&](int slot) {
        nvtx_push(slot);  // NVTX range of the phase (kernels.h)
        if (!(flags & PICO_F_TIMING)) return;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        ev.push_back({slot, {e0, e1}});
    };
    auto tstop = [&]() {
        nvtxRangePop();
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
        int k = 0, kprev = 0, y = 0;
        unsigned long long cnt = 0, lo = 0, cb[2] = {0, 0};  // as in po_levels_kernel
        for (int L = 0;; L++) {
            int par = L & 1;
            Ctrl hc;
            if ((err = cudaMemcpyAsync(&hc, a.ctl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s))) return err;
            if ((err = cudaStreamSynchronize(s))) return err;
            if (L > 0) { po_close_kernel<<<1, 1, 0, s>>>(a, par ^ 1, kprev); launches++; }
            if (hc.nAlive[par] == 0) break;
            k = std::max(k + 1, hc.kminb[par]);
            const unsigned long long lstart = lo;
            po_scan_kernel<STATS><<<blocks, 512, 0, s>>>(a, k, par, PoAppend{lo, cb[y], y});
            launches++;
            for (int sub = 0;; sub++) {
                if ((err = cudaMemcpyAsync(&cnt, y ? &a.ctl->q_tail1 : &a.ctl->q_tail, sizeof(cnt),
                                           cudaMemcpyDeviceToHost, s)))
                    return err;
                if ((err = cudaStreamSynchronize(s))) return err;
                const unsigned long long hi = lo + (cnt - cb[y]);
                cb[y] = cnt;
                y ^= 1;
                if (hi == lo) {
                    y ^= 1;
                    if (sub == 0) {  // empty level: still consume alive[par]
                        unsigned long long z = 0;
                        int imax = INT_MAX;
                        cudaMemcpyAsync(&a.ctl->nAlive[par], &z, sizeof(z), cudaMemcpyHostToDevice, s);
                        cudaMemcpyAsync(&a.ctl->kminb[par], &imax, sizeof(imax), cudaMemcpyHostToDevice, s);
                    }
                    break;
                }
                po_sub_kernel<MODE, STATS><<<blocks, 512, 0, s>>>(a, k, par, PoAppend{hi, cb[y], y}, lo, hi, sub == 0);
                launches++;
                host_subrounds++;
                lo = hi;
            }
            if (CLAMP_SUB && lo > lstart) {
                po_repair_kernel<<<blocks, 512, 0, s>>>(a, k, lstart, lo);
                launches++;
            }
            kprev = k;
        }
    } else {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, po_levels_kernel<MODE, STATS>, PICO_PO_THREADS, 0);
        int per = std::max(1, std::min(occ, PICO_PO_PER));
        void *args[] = {&a};
        err = cudaLaunchCooperativeKernel((const void *)po_levels_kernel<MODE, STATS>, sms * per, PICO_PO_THREADS,
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
        st->segments = (int64_t)(hc.q_tail + hc.q_tail1);
        st->kernel_count += launches;
        if (st->frontier_sizes)
            for (unsigned long long i = 0; i < hc.levels && (int64_t)i < st->frontier_sizes_cap && i < kFszCap; i++)
                st->frontier_sizes[i] = (int64_t)lv[i];
        if (st->round_ns && !(flags & PICO_F_HOST_LOOP)) {
            size_t nl = (size_t)std::min<unsigned long long>(hc.scans, std::min<unsigned long long>(
                                                                kFszCap, (unsigned long long)st->frontier_sizes_cap));
            std::vector<unsigned long long> rt(2 * nl + 1);
            if ((err = cudaMemcpyAsync(rt.data(), a.rtime, sizeof(unsigned long long) * 2 * nl,
                                       cudaMemcpyDeviceToHost, s)))
                return err;
            if ((err = cudaStreamSynchronize(s))) return err;
            for (size_t i = 0; i < 2 * nl; i++) st->round_ns[i] = (int64_t)rt[i];
        }
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

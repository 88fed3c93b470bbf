// histocore.cu -- HistoCore (Alg 6) for sm_100a.
//
// State in HBM:
//   core[v]   int32   current estimate h_t(v) (= core_out; P:495 core <- deg)
//   c8[v]     uint16  min(deg(v), 65535): the degree shadow InitHisto gathers
//                     (a saturated entry falls back to oldc[v] = deg(v))
//   rec[v]    uint32  the estimate record every round-loop gather reads:
//                     low half  min(core[v], 65535),
//                     high half min(oldcore[v], 65535) if v is in the current
//                               changed set C_t, else the low half again,
//                     so one 4-byte gather tells a pull arc whether its
//                     neighbour changed, its new and its old estimate.  A
//                     saturated half (65535) falls back to core/oldc and the
//                     changed bitmap.  SumHisto writes the record of v in
//                     C_{t+1}; the next SumHisto phase resets C_t's records.
//   oldc[v]   int32   estimate before v's latest change (oldcore); during
//                     init it holds deg(v), the round-0 estimate of every vertex
//   histo     int32[2m], vertex v owns slots rowptr[v] + b - 1 for bins
//                     b = 1..deg(v).  Invariant after every
//                     round: bins b < core[v] count neighbours with
//                     estimate b, the cap bin core[v] holds cnt(v) = #nbrs with
//                     estimate >= core[v], bins above are
//                     stale and never read.
//   F         int32   frontier list F_t (Theorem 2: cnt < core)
//   S         int2    UpdateHisto work list: (v, segment) for every changed v,
//                     one entry per `seg` arcs of v's row (load balance)
//   H         int2    static (v, segment) list of the hub rows (deg > seg) for
//                     the pull-mode UpdateHisto
//   chg[2]    bitmap  changed set C_t (parity t&1) for pull mode
//
// Round structure (strict two-phase synchronous rounds):
//   init   = InitHisto fused with round-1 SumHisto: per vertex a
//            capped histogram of min(deg(u), deg(v)) in registers / shared
//            memory, its h-index, and only bins 1..h written back.
//   loop   { UpdateHisto(C_t) -> F_{t+1} ; SumHisto(F_{t+1}) -> C_{t+1} }
// UpdateHisto: for v in C_t, u in nbr(v) with core[u] > core[v]:
//   old = atomicSub(histo[u][min(oldcore[v], core[u])], 1);
//   atomicAdd(histo[u][core[v]], 1);
//   push u iff oldcore[v] >= core[u] and old == core[u]   (exactly once,
//   the cap bin is only ever decremented).
//   Two bit-exact directions apply the SAME (v, u) bin moves:
//     push: changed rows are scanned, the moves hit u's histogram remotely;
//     pull (dense rounds): every arc (u, v) of the edge list, bucketed by
//       v-range, is streamed; v's record tells whether v changed, the moves
//       hit u's own histogram (consecutive arcs share u: coalesced REDs).
// SumHisto: walk k = core_old, core_old-1, ...; sum += histo[v][k];
//   stop at the first k with sum >= k; core[v] = k,
//   oldcore[v] = core_old, histo[v][k] = sum.
#include <climits>

#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace pico {

// build-time A/B knobs: L2 eviction hints
#ifndef PICO_L2_HINTS
#define PICO_L2_HINTS 0
#endif
// vertex count from which dense rounds may run UpdateHisto in the pull direction
#ifndef PICO_PULL_MIN_N
#define PICO_PULL_MIN_N (1ll << 20)
#endif
constexpr long long kPullMinN = PICO_PULL_MIN_N;
// arcs per UpdateHisto work item (segment of a changed row)
#ifndef PICO_HC_SEG
#define PICO_HC_SEG 64
#endif
typedef unsigned char shadow_t;
constexpr unsigned SAT8 = 255;     // degree shadow saturation
constexpr unsigned RSAT = 65535;   // estimate-record half saturation
// pull-mode v-range passes: the record slice one pass gathers from
#ifndef PICO_PASS_MB
#define PICO_PASS_MB 32
#endif
constexpr int kMaxPass = 8;
// class-C InitHisto shared-memory bins (a vertex whose h-index reaches the
// cap is redone with global bins; h_1 <= the graph's degree h-index)
#ifndef PICO_BMAX
#define PICO_BMAX 2048             // warp-class InitHisto rows: a_max < deg <= PICO_BMAX
#endif
#ifndef PICO_CBINS
#define PICO_CBINS 8192
#endif
#ifndef PICO_ROUNDS_MINB
#define PICO_ROUNDS_MINB 2         // resident 512-thread CTAs per SM of the round kernel
#endif
#ifndef PICO_PULL_AGG
#define PICO_PULL_AGG 0            // warp-aggregate duplicate bin moves in pull mode
#endif                             // (__match_any_sync; measured 1.4-3x slower)

struct HcArgs {
    const long long *rp;   // rowptr [n+1]
    const int *ci;         // colidx [2m]
    int n;
    long long arcs;
    int *core;             // [n]  (core_out)
    shadow_t *c8;          // [n]  min(deg, 255): degree shadow for rows with deg <= 255
    unsigned short *c16;   // [n]  min(deg, 65535): degree shadow for longer rows
    unsigned *rec;         // [n]  estimate record (new16 | old16 << 16)
    unsigned short *e16;   // [n]  min(core, 65535): the estimate alone (push-round gathers)
    int *oldc;             // [n]
    int *histo;            // [2m]
    int *F;                // [n]  frontier list; init: hub fallback list
    int *BC;               // [n]  init class lists (B from front, C from back)
    int2 *S;               // update segments of C_t
    int2 *H;               // static hub segments (pull mode)
    unsigned *chg;         // [2][nwords] changed bitmaps
    unsigned *capd;        // [nwords] cap-touched bitmap (UpdateHisto -> SumHisto)
    long long nwords;
    unsigned long long *fsz;  // [fsz_cap] per-round frontier sizes
    unsigned long long *rarcs;  // [fsz_cap] per-round arcs of C_t (stats)
    unsigned long long *rtime;  // [2 fsz_cap + 1] %globaltimer at the round kernel's barriers
    unsigned long long fsz_cap;
    Ctrl *ctl;
    Tune tn;
    int allow_pull;
    const shadow_t *nv8;   // neighbour-degree lookups of InitHisto (see init_val)
    const unsigned short *nv16;
    const int *nv32;
    // degree prefilter (push UpdateHisto): rows copied in descending order of
    // the neighbours' degree bucket floor(log2 deg); a changed v with new
    // estimate c scans only the prefix whose bucket may hold deg(u) > c
    // (core[u] <= deg(u), so the rest can never pass the guard core[u] > c)
    int prefilter;
    int *ro;               // [2m] bucket-ordered copy of colidx
    unsigned char *db;     // [n]  floor(log2(deg))
    int *slen;             // [n]  scanned prefix of v's row for its latest change
    // pull rounds: the arcs (u, v) as an edge list bucketed by the v-range
    // of the neighbour, bucket p = {v in [p*pw, (p+1)*pw)} at
    // [boff[p], boff[p+1]) of psrc (= u) / pdst (= v); a pass over one
    // bucket gathers the records of an L2-sized slice of the vertices
    int npass, pshift;
    unsigned long long *boff;  // [kMaxPass + 1] bucket offsets
    // decremental updates (pico_dyn_*): a vertex that lost every neighbour
    // walks down to h = 0 instead of flagging a broken invariant
    int allow_zero;
    // warm start (edge insertions, pico_dyn_insert_edges): the round-0
    // estimates (an upper bound of the coreness, <= deg) instead of the
    // degrees: InitHisto caps v's histogram at h0[v] and bins neighbours by
    // min(h0[u], h0[v]); null = the degrees
    const int *h0;
    int *psrc, *pdst;
    // 32-bit copy of rowptr when 2m < 2^32 (null otherwise): the histogram-base
    // gathers of UpdateHisto / SumHisto read half the bytes
    unsigned *rp32;
    // PICO_F_STATS with pico_stats_t.frontier_counts: rounds in which each
    // vertex was a frontier (the paper's Fig 3 measure); null: off
    int *fcnt = nullptr;
};

// rowptr[v] through the 32-bit copy when there is one (uniform branch)
__device__ __forceinline__ long long rp_at(const HcArgs &a, long long v) {
    return a.rp32 ? (long long)__ldg(a.rp32 + v) : __ldg(a.rp + v);
}

// prefix of v's bucket-ordered row that UpdateHisto must scan after v's
// estimate became c: entries with bucket >= floor(log2(c + 1)) (binary
// search; buckets are non-increasing along the row)
__device__ __forceinline__ int scan_len(const HcArgs &a, long long hb, int d, int c) {
    if (!a.prefilter || d <= a.tn.a_max) return d;
    const int bmin = 31 - __clz(c + 1);
    int lo = 0, hi = d;  // first position with bucket < bmin
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if ((int)__ldg(a.db + __ldg(a.ro + hb + mid)) >= bmin) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int nseg_of(long long d, int seg) { return (int)((d + seg - 1) / seg); }

// 16-bit load (hot policy)
__device__ __forceinline__ unsigned ld_shadow(const unsigned char *p, unsigned long long hot) {
#if PICO_L2_HINTS
    return ld_cg_u16(p, hot);
#else
    return __ldcg(p);
#endif
}

__device__ __forceinline__ unsigned pack_rec(int k, int old) {
    return (unsigned)min(k, (int)RSAT) | ((unsigned)min(old, (int)RSAT) << 16);
}

__device__ __forceinline__ unsigned ld_rec(const unsigned *p, unsigned long long hot) {
#if PICO_L2_HINTS
    return ld_cg_u32(p, hot);
#else
    return __ldcg(p);
#endif
}

// exact current estimate of u through its record
__device__ __forceinline__ int core_of(const HcArgs &a, int u, unsigned long long hot) {
    unsigned c = ld_rec(a.rec + u, hot) & 0xffffu;
    return c == RSAT ? __ldcg(a.core + u) : (int)c;
}

__device__ __forceinline__ void set_c8(const HcArgs &a, int v, int k) {
    a.c8[v] = (shadow_t)min(k, (int)SAT8);
    a.c16[v] = (unsigned short)min(k, 65535);
}

__device__ __forceinline__ void stat_add(unsigned long long *ctr, long long x) {
    long long s = warp_sum64(x);
    if (lane_id() == 0 && s) atomicAdd(ctr, (unsigned long long)s);
}

// Bookkeeping of the changed set C_t for round t's UpdateHisto: |C_t|, arcs
// of C_t, minimum new estimate (accumulated per thread, flushed once per
// phase -- these are single-address counters) and the changed bitmap.
struct ChangeAcc {
    long long cnt = 0, arcs = 0;
    int kmin = INT_MAX;
    __device__ __forceinline__ void note(const HcArgs &a, int t, int v, int k, long long d) {
        cnt++;
        arcs += d;
        kmin = min(kmin, k);
        atomicOr(a.chg + (t & 1) * a.nwords + (v >> 5), 1u << (v & 31));
        if (a.fcnt) a.fcnt[v]++;  // one lane handles v per round
    }
    // all 32 lanes call; count_into: counter of |C_t| (init only) or null
    __device__ __forceinline__ void flush(const HcArgs &a, int t, unsigned long long *count_into) {
        long long c = warp_sum64(cnt), s = warp_sum64(arcs);
        int km = warp_min(kmin);
        if (lane_id() == 0 && c) {
            atomicAdd(&a.ctl->arcsC[t & 1], (unsigned long long)s);
            atomicMin(&a.ctl->mincv[t & 1], km);
            if (count_into) atomicAdd(count_into, (unsigned long long)c);
        }
    }
};

// ---------------------------------------------------------------------------
// H0: degrees, classification, hub segment list, 16-bit shadow
// ---------------------------------------------------------------------------
__global__ void hc_degree_kernel(HcArgs a) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    long long iters = ((long long)a.n + nthreads - 1) / nthreads;
    for (long long it = 0; it < iters; it++) {
        int v = (int)(it * nthreads + blockIdx.x * blockDim.x + threadIdx.x);
        bool valid = v < a.n;
        long long d = valid ? a.rp[v + 1] - a.rp[v] : 0;
        if (valid && a.rp32) {
            a.rp32[v] = (unsigned)a.rp[v];
            if (v == a.n - 1) a.rp32[a.n] = (unsigned)a.rp[a.n];
        }
        if (valid) {
            a.oldc[v] = (int)d;  // round-0 estimate of every vertex
            a.core[v] = (int)d;
            set_c8(a, v, (int)d);
            if (a.prefilter) a.db[v] = d > 0 ? (unsigned char)(31 - __clz((int)d)) : 0;
        }
        bool isB = valid && d > a.tn.a_max && d <= a.tn.b_max;
        bool isC = valid && d > a.tn.b_max;
        warp_append(isB, v, a.BC, &a.ctl->nB);
        // class C grows from the back of the same array
        unsigned m = __ballot_sync(FULL, isC);
        if (m) {
            unsigned long long base = 0;
            int leader = __ffs(m) - 1;
            if (lane_id() == leader) base = atomicAdd(&a.ctl->nC, (unsigned long long)__popc(m));
            base = __shfl_sync(FULL, base, leader);
            if (isC) a.BC[a.n - 1 - (long long)(base + __popc(m & ((1u << lane_id()) - 1)))] = v;
        }
        warp_append_segments(v, (valid && d > a.tn.seg) ? nseg_of(d, a.tn.seg) : 0, a.H, &a.ctl->nH);
    }
}

// ---------------------------------------------------------------------------
// degree prefilter: counting sort of each class-B / class-C row by the
// neighbours' degree bucket, descending (class-A rows are copied by init)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) hc_reorder_warp_kernel(HcArgs a) {
    __shared__ int cnt[8][32];
    const int wib = threadIdx.x >> 5, lane = lane_id();
    int *c = cnt[wib];
    const long long nB = (long long)bcast_u64(&a.ctl->nB);
    const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long idx = gw; idx < nB; idx += nw) {
        int v = a.BC[idx];
        long long hb = a.rp[v];
        int d = (int)(a.rp[v + 1] - hb);
        c[lane] = 0;
        __syncwarp();
        for (int e = lane; e < d; e += 32) atomicAdd(&c[31 - a.db[__ldg(a.ci + hb + e)]], 1);
        __syncwarp();
        int x = c[lane];
        int incl = warp_incl_scan(x);
        c[lane] = incl - x;
        __syncwarp();
        for (int e = lane; e < d; e += 32) {
            int u = __ldg(a.ci + hb + e);
            a.ro[hb + atomicAdd(&c[31 - a.db[u]], 1)] = u;
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(512) hc_reorder_cta_kernel(HcArgs a) {
    __shared__ int c[32];
    const long long nC = (long long)bcast_u64(&a.ctl->nC);
    for (long long idx = blockIdx.x; idx < nC; idx += gridDim.x) {
        int v = a.BC[a.n - 1 - idx];
        long long hb = a.rp[v];
        int d = (int)(a.rp[v + 1] - hb);
        if (threadIdx.x < 32) c[threadIdx.x] = 0;
        __syncthreads();
        for (int e = threadIdx.x; e < d; e += blockDim.x) atomicAdd(&c[31 - a.db[__ldg(a.ci + hb + e)]], 1);
        __syncthreads();
        if (threadIdx.x < 32) {
            int x = c[threadIdx.x];
            int incl = warp_incl_scan(x);
            c[threadIdx.x] = incl - x;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < d; e += blockDim.x) {
            int u = __ldg(a.ci + hb + e);
            a.ro[hb + atomicAdd(&c[31 - a.db[u]], 1)] = u;
        }
        __syncthreads();
    }
}

// neighbour degree for init, clamped to d (the histogram cap of P:498)
// (nv8 / nv16 / nv32: degree of every neighbour id saturated at 255, at
// 65535, and exact; the local shadows / oldcore on one GPU, the all-gathered
// global degrees on a shard).  Rows with d <= 255 (the thread class and the
// first warp-class launch) gather the 1-byte shadow, exact for them and half
// the L2 footprint; longer rows gather the 2-byte one (a 1-byte shadow plus
// an exact fallback was measured 1.1-1.7x slower for them: their neighbours
// are often hubs).
__device__ __forceinline__ int init_val_small(const HcArgs &a, int u, int d, unsigned long long hot) {
    return min((int)ld_shadow(a.nv8 + u, hot), d);  // d <= 255: exact
}

__device__ __forceinline__ int init_val(const HcArgs &a, int u, int d, unsigned long long hot) {
    int x = (int)__ldcg(a.nv16 + u);
    if (x >= d) return d;
    if (x == 65535) return min(__ldg(a.nv32 + u), d);
    return x;
}

// ---------------------------------------------------------------------------
// H1-H3 round 1, class A: one thread per vertex, 1 <= deg <= a_max (<= 16),
// histogram in registers (compile-time-indexed).
// ---------------------------------------------------------------------------
template <bool STATS>
__global__ void __launch_bounds__(256) hc_init_small_kernel(HcArgs a) {
    constexpr int NB = 16;
    long long nthreads = (long long)gridDim.x * blockDim.x;
    long long iters = ((long long)a.n + nthreads - 1) / nthreads;
    ChangeAcc acc;
    long long st_slots = 0;
    const unsigned long long hot = pol_last(), cold = pol_first();
    for (long long it = 0; it < iters; it++) {
        int v = (int)(it * nthreads + blockIdx.x * blockDim.x + threadIdx.x);
        bool valid = v < a.n;
        long long hb = 0;
        int d = 0;
        if (valid) {
            hb = a.rp[v];
            d = (int)(a.rp[v + 1] - hb);
        }
        bool mine = valid && d >= 1 && d <= a.tn.a_max;
        int nseg = 0, h = 0;
        const int cap = (mine && a.h0) ? min(__ldg(a.h0 + v), d) : d;  // the round-0 estimate
        if (mine) {
            int cnt[NB];
#pragma unroll
            for (int b = 0; b < NB; b++) cnt[b] = 0;
            for (int e = 0; e < d; e++) {
                int u = ld_stream(a.ci + hb + e, cold);
                if (a.prefilter) a.ro[hb + e] = u;  // short rows: copied in order
                int x = init_val_small(a, u, cap, hot);  // min(core[u], core[v])
#pragma unroll
                for (int b = 0; b < NB; b++) cnt[b] += (x == b + 1);
            }
            int s = 0, hs = 0;
#pragma unroll
            for (int b = NB; b >= 1; b--) {
                if (b <= cap && h == 0) {
                    s += cnt[b - 1];
                    if (s >= b) { h = b; hs = s; }
                }
            }
#pragma unroll
            for (int b = 1; b <= NB; b++) {
                if (b < h) a.histo[hb + b - 1] = cnt[b - 1];
                else if (b == h) a.histo[hb + b - 1] = hs;
            }
            a.core[v] = h;
            if (h < cap) {
                a.slen[v] = d;  // d <= a_max: whole row
                nseg = nseg_of(d, a.tn.seg);
            }
        }
        if (nseg > 0) acc.note(a, 1, v, h, d);
        warp_append_segments(v, nseg, a.S, &a.ctl->nS[1]);
        if (STATS && mine) st_slots += h;
    }
    acc.flush(a, 1, &a.ctl->nF[1]);
    if (STATS) stat_add(&a.ctl->st_init_slots, st_slots);
}

// ---------------------------------------------------------------------------
// class B: one warp per vertex, a_max < deg <= b_max, shared-memory bins
// ---------------------------------------------------------------------------
// PART 0: every class-B row, gathering the 2-byte degree shadow.  On large
// graphs (hc_init_split) two launches instead: PART 1 the rows with d <= 255
// gathering the 1-byte shadow (exact for them), PART 2 the longer rows with
// the 2-byte one, so that only one shadow array competes for the L2 at a time
// (RMAT-26: 31.6 -> 29.1 ms; on C2, whose shadows fit the L2 anyway, the
// second launch costs more than it saves)
// shared bins per warp: the rows of the PART 1 launch have d <= 255, so that
// launch needs 256 bins per warp instead of b_max + 1 (8 KB per CTA instead of
// 64 KB: the occupancy is set by registers, not by shared memory)
template <int PART>
__host__ __device__ constexpr int init_warp_stride(int b_max) {
    return PART == 1 ? (b_max < (int)SAT8 ? b_max : (int)SAT8) + 1 : b_max + 1;
}
template <bool STATS, int PART>
__global__ void __launch_bounds__(256) hc_init_warp_kernel(HcArgs a) {
    extern __shared__ int sh[];
    const int wib = threadIdx.x >> 5;
    const int lane = lane_id();
    int *bins = sh + wib * init_warp_stride<PART>(a.tn.b_max);
    const long long nB = (long long)bcast_u64(&a.ctl->nB);
    const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    ChangeAcc acc;
    long long st_slots = 0;
    const unsigned long long hot = pol_last(), cold = pol_first();
    for (long long idx = gw; idx < nB; idx += nw) {
        int v = a.BC[idx];
        long long hb = a.rp[v];
        int d = (int)(a.rp[v + 1] - hb);
        if (PART != 0 && (d <= (int)SAT8) != (PART == 1)) continue;  // the other launch's row (warp-uniform)
        const int cap = a.h0 ? min(__ldg(a.h0 + v), d) : d;  // the round-0 estimate
        for (int b = lane; b <= cap; b += 32) bins[b] = 0;
        __syncwarp();
        auto val = [&](int u) { return PART == 1 ? init_val_small(a, u, cap, hot) : init_val(a, u, cap, hot); };
        {
            int e = lane;
            for (; e + 96 < d; e += 128) {  // 4 gathers in flight per lane
                int u0 = ld_stream(a.ci + hb + e, cold), u1 = ld_stream(a.ci + hb + e + 32, cold);
                int u2 = ld_stream(a.ci + hb + e + 64, cold), u3 = ld_stream(a.ci + hb + e + 96, cold);
                int x0 = val(u0), x1 = val(u1);
                int x2 = val(u2), x3 = val(u3);
                atomicAdd(&bins[x0], 1);
                atomicAdd(&bins[x1], 1);
                atomicAdd(&bins[x2], 1);
                atomicAdd(&bins[x3], 1);
            }
            for (; e < d; e += 32) atomicAdd(&bins[val(ld_stream(a.ci + hb + e, cold))], 1);
        }
        __syncwarp();
        // descending walk for the h-index (SumHisto on the fresh histogram)
        int carry = 0, top = cap, h = 0, hs = 0;
        for (;;) {
            int kk = top - lane;
            int val = kk >= 1 ? bins[kk] : 0;
            int incl = warp_incl_scan(val);
            int s = carry + incl;
            unsigned m = __ballot_sync(FULL, kk >= 1 && s >= kk);
            if (m) {
                int f = __ffs(m) - 1;
                h = top - f;
                hs = __shfl_sync(FULL, s, f);
                break;
            }
            carry += __shfl_sync(FULL, incl, 31);
            top -= 32;
        }
        for (int b = 1 + lane; b <= h; b += 32) a.histo[hb + b - 1] = (b < h) ? bins[b] : hs;
        __syncwarp();
        const bool changed = h < cap;
        int L = 0;
        if (changed && lane == 0) L = scan_len(a, hb, d, h);
        L = __shfl_sync(FULL, L, 0);
        int nseg = nseg_of(L, a.tn.seg);
        if (lane == 0) {
            a.core[v] = h;
            if (changed) {
                a.slen[v] = L;
                acc.note(a, 1, v, h, d);
            }
            st_slots += h;
        }
        if (nseg) {
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(&a.ctl->nS[1], (unsigned long long)nseg);
            base = __shfl_sync(FULL, base, 0);
            for (int s = lane; s < nseg; s += 32) a.S[base + s] = make_int2(v, s);
        }
    }
    acc.flush(a, 1, &a.ctl->nF[1]);
    if (STATS) stat_add(&a.ctl->st_init_slots, st_slots);
}

// ---------------------------------------------------------------------------
// class C: one CTA per vertex, shared-memory bins capped at c_bins; vertices
// whose h-index may exceed the cap go to the global-bin fallback (GLOBAL=true
// runs the same procedure on the vertex's own 2m-slot region in HBM).
// ---------------------------------------------------------------------------
// cap: the shared-memory bin cap (class C: c_bins; the fallback's first try:
// the big shared-memory tier).  Returns false (nothing written) when the
// h-index may exceed the cap: the caller redoes v with more bins.
template <bool GLOBAL, bool STATS>
__device__ bool cta_init_vertex(const HcArgs &a, int v, int *bins, int *red, int cap) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = lane_id(), wid = tid >> 5, nwarp = nt >> 5;
    long long hb = a.rp[v];
    int d = (int)(a.rp[v + 1] - hb);
    const int ecap = a.h0 ? min(__ldg(a.h0 + v), d) : d;  // the round-0 estimate
    int B = GLOBAL ? ecap : min(ecap, cap);
    if (GLOBAL) bins = a.histo + hb - 1;  // bin b at slot hb + b - 1
    for (int b = tid; b <= B; b += nt)
        if (!GLOBAL || b >= 1) bins[b] = 0;
    __syncthreads();
    const unsigned long long hot = pol_last(), cold = pol_first();
    {
        int e = tid;
        for (; e + 3 * nt < d; e += 4 * nt) {  // 4 gathers in flight per thread
            int u0 = ld_stream(a.ci + hb + e, cold), u1 = ld_stream(a.ci + hb + e + nt, cold);
            int u2 = ld_stream(a.ci + hb + e + 2 * nt, cold), u3 = ld_stream(a.ci + hb + e + 3 * nt, cold);
            int x0 = init_val(a, u0, ecap, hot), x1 = init_val(a, u1, ecap, hot);
            int x2 = init_val(a, u2, ecap, hot), x3 = init_val(a, u3, ecap, hot);
            atomicAdd(&bins[min(x0, B)], 1);
            atomicAdd(&bins[min(x1, B)], 1);
            atomicAdd(&bins[min(x2, B)], 1);
            atomicAdd(&bins[min(x3, B)], 1);
        }
        for (; e < d; e += nt) atomicAdd(&bins[min(init_val(a, ld_stream(a.ci + hb + e, cold), ecap, hot), B)], 1);
    }
    __syncthreads();
    // block-wide descending search: h = max b in 1..B with sum_{j>=b} bins[j] >= b
    int c = (B + nt - 1) / nt;
    int hiT = B - tid * c;  // this thread's chunk, descending
    int loT = max(1, B - (tid + 1) * c + 1);
    int tsum = 0;
    for (int b = hiT; b >= loT; b--) tsum += bins[b];
    int incl = warp_incl_scan(tsum);
    if (lane == 31) red[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int x = lane < nwarp ? red[lane] : 0;
        int xi = warp_incl_scan(x);
        if (lane < nwarp) red[lane] = xi - x;  // exclusive warp offsets
    }
    __syncthreads();
    int s = red[wid] + incl - tsum;
    int cand = 0, cs = 0;
    for (int b = hiT; b >= loT; b--) {
        s += bins[b];
        if (s >= b) { cand = b; cs = s; break; }
    }
    __syncthreads();
    if (tid == 0) { red[32] = 0; red[33] = 0; }
    __syncthreads();
    if (cand) atomicMax(&red[32], cand);
    __syncthreads();
    int h = red[32];
    if (cand == h && cand) red[33] = cs;
    __syncthreads();
    int hs = red[33];
    if (!GLOBAL && h == B && ecap > B) {
        // the cap may hide a larger h-index: the caller redoes v with more bins
        __syncthreads();
        return false;
    }
    if (GLOBAL) {
        if (tid == 0) a.histo[hb + h - 1] = hs;  // bins 1..h-1 already exact
    } else {
        for (int b = 1 + tid; b <= h; b += nt) a.histo[hb + b - 1] = (b < h) ? bins[b] : hs;
    }
    if (tid == 0) {
        const bool changed = h < ecap;
        a.core[v] = h;
        int L = changed ? scan_len(a, hb, d, h) : 0;
        int ns = nseg_of(L, a.tn.seg);
        red[35] = ns;
        if (changed) {
            a.slen[v] = L;
            atomicAdd(&a.ctl->nF[1], 1ull);
            atomicAdd(&a.ctl->arcsC[1], (unsigned long long)d);
            atomicMin(&a.ctl->mincv[1], h);
            atomicOr(a.chg + a.nwords + (v >> 5), 1u << (v & 31));
            if (a.fcnt) a.fcnt[v]++;
            if (ns) red[34] = (int)atomicAdd(&a.ctl->nS[1], (unsigned long long)ns);
        }
        if (STATS) {
            atomicAdd(&a.ctl->st_init_slots, (unsigned long long)(GLOBAL ? d : h));
            if (GLOBAL) atomicAdd(&a.ctl->st_fallback, 1ull);
        }
    }
    __syncthreads();
    const int nseg = red[35];
    if (nseg) {
        unsigned long long base = (unsigned)red[34];
        for (int s2 = tid; s2 < nseg; s2 += nt) a.S[base + s2] = make_int2(v, s2);
    }
    __syncthreads();
    return true;
}

template <bool STATS>
__global__ void __launch_bounds__(512) hc_init_cta_kernel(HcArgs a) {
    extern __shared__ int bins[];
    __shared__ int red[40];
    const long long nC = (long long)bcast_u64(&a.ctl->nC);
    for (long long idx = blockIdx.x; idx < nC; idx += gridDim.x) {
        int v = a.BC[a.n - 1 - idx];
        if (!cta_init_vertex<false, STATS>(a, v, bins, red, a.tn.c_bins) && threadIdx.x == 0) {
            unsigned long long i = atomicAdd(&a.ctl->nX, 1ull);  // to the fallback
            a.F[i] = v;
        }
    }
}

// the class-C vertices whose h-index reached c_bins (the hubs): first with the
// big shared-memory tier (one 1024-thread CTA per SM, `big` bins: at RMAT-26
// every hub fits, its degree h-index is below 45 K), else with global bins in
// the vertex's own histogram slots (contended HBM atomics on its low bins:
// 3.2 ms for 352 hubs at RMAT-26 when this was the only fallback)
template <bool STATS>
__global__ void __launch_bounds__(1024, 1) hc_init_fallback_kernel(HcArgs a, int big) {
    extern __shared__ int bins[];
    __shared__ int red[40];
    const long long nX = (long long)bcast_u64(&a.ctl->nX);
    for (long long idx = blockIdx.x; idx < nX; idx += gridDim.x) {
        int v = a.F[idx];
        if (big == 0 || !cta_init_vertex<false, STATS>(a, v, bins, red, big))
            cta_init_vertex<true, STATS>(a, v, nullptr, red, 0);
    }
}

// after init: estimate records of round 1 (C_1 = {v : h_1(v) < deg(v)},
// oldcore = deg for its members)
__global__ void hc_shadow_kernel(HcArgs a) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += nthreads) {
        int k = a.core[v], d = a.oldc[v];
        a.rec[v] = pack_rec(k, d);
        a.e16[v] = (unsigned short)min(k, (int)RSAT);
    }
}

// ---------------------------------------------------------------------------
// Edge list of the pull rounds, bucketed by the neighbour's v-range
// (bucket p = v >> pshift), in CSR order inside each bucket:
//   src:   the row owning every arc (short rows one thread each, hub rows a
//          warp per static 64-arc segment)
//   count: per 2048-arc chunk and bucket (ballot/popc), bucket-major matrix
//   scan:  one exclusive scan -> every (bucket, chunk) output offset
//   fill:  each chunk writes its (u, v) pairs in arc order
// With one bucket the edge list is (src, colidx) itself: no count/fill.
// ---------------------------------------------------------------------------
constexpr int kElChunk = 2048;

// rows of the thread-per-vertex class (deg <= a_max): one thread each
__global__ void hc_el_src_short_kernel(HcArgs a, int *src) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < a.n; u += nthreads) {
        long long r0 = a.rp[u], r1 = a.rp[u + 1];
        if (r1 - r0 <= a.tn.a_max)
            for (long long e = r0; e < r1; e++) src[e] = (int)u;
    }
}

// longer rows (the degree-class lists B and C): one warp per row, coalesced
__global__ void hc_el_src_long_kernel(HcArgs a, int *src) {
    const long long nB = (long long)bcast_u64(&a.ctl->nB), nC = (long long)bcast_u64(&a.ctl->nC);
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = gw; i < nB + nC; i += nw) {
        const int u = i < nB ? a.BC[i] : a.BC[a.n - 1 - (i - nB)];
        const long long r0 = a.rp[u], r1 = a.rp[u + 1];
        for (long long x = r0 + lane_id(); x < r1; x += 32) src[x] = u;
    }
}

// warp per chunk: counts[p * nchunk + c] (per-lane counters, 8 loads in
// flight per lane, one warp reduction per bucket at the end of the chunk)
__global__ void __launch_bounds__(256) hc_el_count_kernel(HcArgs a, unsigned long long *cnt, long long nchunk) {
    const int lane = lane_id();
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const unsigned long long cold = pol_first();
    for (long long c = gw; c < nchunk; c += nw) {
        const long long e0 = c * kElChunk, e1 = min(e0 + kElChunk, a.arcs);
        int k[kMaxPass] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (long long eb = e0; eb < e1; eb += 8 * 32) {
            int v[8];
#pragma unroll
            for (int i = 0; i < 8; i++) {
                long long e = eb + i * 32 + lane;
                v[i] = e < e1 ? ld_stream(a.ci + e, cold) >> a.pshift : -1;
            }
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int q = 0; q < kMaxPass; q++) k[q] += (v[i] == q);
        }
#pragma unroll
        for (int q = 0; q < kMaxPass; q++) {
            if (q >= a.npass) break;
            long long t = warp_sum64(k[q]);
            if (lane == 0) cnt[(long long)q * nchunk + c] = (unsigned long long)t;
        }
    }
}

// warp per chunk: the scanned counts are the output offsets; 4 steps of 32
// arcs in flight, one ballot per bucket and step
#ifndef PICO_FILL_MINB
#define PICO_FILL_MINB 1  // resident 256-thread CTAs per SM the fill's registers must allow (A/B)
#endif
__global__ void __launch_bounds__(256, PICO_FILL_MINB) hc_el_fill_kernel(HcArgs a, const int *src, const unsigned long long *off,
                                                         long long nchunk) {
    const int lane = lane_id();
    const unsigned lt = (1u << lane) - 1;
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const unsigned long long cold = pol_first();
    for (long long c = gw; c < nchunk; c += nw) {
        const long long e0 = c * kElChunk, e1 = min(e0 + kElChunk, a.arcs);
        unsigned long long cur[kMaxPass];
#pragma unroll
        for (int q = 0; q < kMaxPass; q++) cur[q] = q < a.npass ? off[(long long)q * nchunk + c] : 0;
        for (long long eb = e0; eb < e1; eb += 4 * 32) {
            int v[4], u[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                long long e = eb + i * 32 + lane;
                v[i] = e < e1 ? ld_stream(a.ci + e, cold) : -1;
                u[i] = e < e1 ? ld_stream(src + e, cold) : 0;
            }
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int p = v[i] >= 0 ? v[i] >> a.pshift : -1;
#pragma unroll
                for (int q = 0; q < kMaxPass; q++) {
                    if (q >= a.npass) break;
                    const unsigned m = __ballot_sync(FULL, p == q);
                    if (p == q) {
                        const unsigned long long w = cur[q] + __popc(m & lt);
                        a.psrc[w] = u[i];
                        a.pdst[w] = v[i];
                    }
                    cur[q] += __popc(m);
                }
            }
        }
    }
}

// bucket offsets from the scanned count matrix
__global__ void hc_el_offsets_kernel(HcArgs a, long long nchunk, const unsigned long long *off) {
    if (threadIdx.x <= kMaxPass)
        a.boff[threadIdx.x] = (int)threadIdx.x < a.npass ? off[(long long)threadIdx.x * nchunk] : (unsigned long long)a.arcs;
}

// ---------------------------------------------------------------------------
// one (v, u) bin move of UpdateHisto on u's histogram (hbu = rowptr[u] - 1)
// ---------------------------------------------------------------------------
// Single-GPU rounds: every RMW is fire-and-forget (REDG).  A decrement of the
// cap bin (the only way cnt(u) can drop) marks u in the
// cap-touched bitmap; the next SumHisto phase keeps exactly the marked u with
// cnt(u) < core[u] (Theorem 2) -- the same F_{t+1} as the
// returned-value trigger of Alg 6, without any warp waiting on an atomic.
__device__ __forceinline__ void bin_move_mark(const HcArgs &a, long long hbu, int u, int cu, int cv, int ov) {
    if (ov >= cu) {
        red_add(a.histo + hbu + cu, -1);
        red_or(a.capd + (u >> 5), 1u << (u & 31));
    } else {
        red_add(a.histo + hbu + ov, -1);
    }
    red_add(a.histo + hbu + cv, 1);
}

// Sharded rounds (sh_update_kernel): the literal trigger -- returns true iff
// this call drove cnt(u) below core[u] (old == core[u], exactly once)
__device__ __forceinline__ bool bin_move(int *histo, long long hbu, int cu, int cv, int ov) {
    bool push = false;
    if (ov >= cu) {
        int old = atomicSub(histo + hbu + cu, 1);  // cap bin: cnt
        push = (old == cu);                        // exactly once
    } else {
        red_add(histo + hbu + ov, -1);
    }
    red_add(histo + hbu + cv, 1);
    return push;
}

// warp-aggregated append of up to U pushes per lane to F
template <int U>
__device__ __forceinline__ void append_pushes(const bool (&push)[U], const int (&u)[U], int *F,
                                              unsigned long long *nF) {
    const unsigned lt_mask = (1u << lane_id()) - 1;
    unsigned pm[U];
    int tot = 0;
#pragma unroll
    for (int q = 0; q < U; q++) {
        pm[q] = __ballot_sync(FULL, push[q]);
        tot += __popc(pm[q]);
    }
    if (tot) {
        unsigned long long base = 0;
        if (lane_id() == 0) base = atomicAdd(nF, (unsigned long long)tot);
        base = __shfl_sync(FULL, base, 0);
#pragma unroll
        for (int q = 0; q < U; q++) {
            if (push[q]) F[base + __popc(pm[q] & lt_mask)] = u[q];
            base += __popc(pm[q]);
        }
    }
}

// ---------------------------------------------------------------------------
// Arc stream of one warp batch: lane L owns the arc range [b_L, b_L + len_L)
// (a row or a row segment); the concatenated ranges are walked 32*U arcs at a
// time.  ArcStep holds, for each of a lane's U arcs, its owner lane and its
// neighbour id (-1 past the end).  fetch() issues the colidx loads of a step
// (owner = max lane with excl <= j, a 5-step shuffle binary search), so the
// caller can fetch step i+1 before it waits on the gathers of step i.
// Warp-collective.
// ---------------------------------------------------------------------------
#ifndef PICO_ARC_U
#define PICO_ARC_U 4
#endif
#ifndef PICO_ARC_PF
#define PICO_ARC_PF 1
#endif
template <int U>
struct ArcStep {
    int lo[U];
    int v[U];
};

template <int U>
__device__ __forceinline__ void arc_fetch(ArcStep<U> &st, int j0, int total, int excl, long long b,
                                          const int *rows, unsigned long long cold) {
    const int lane = lane_id();
#pragma unroll
    for (int q = 0; q < U; q++) {
        int j = j0 + q * 32 + lane;
        int lo = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            int cand = lo + step;
            int ex = __shfl_sync(FULL, excl, cand & 31);
            if (cand < 32 && ex <= j) lo = cand;
        }
        long long eb = __shfl_sync(FULL, b, lo);
        int ex = __shfl_sync(FULL, excl, lo);
        st.lo[q] = lo;
        st.v[q] = j < total ? ld_stream(rows + eb + (j - ex), cold) : -1;
    }
}

// ---------------------------------------------------------------------------
// UpdateHisto, push direction, round t: segments of C_t (count nS[t&1]).
// Warps take batches of 32 segments, scan their lengths, and walk the
// concatenated arcs U*32 at a time (owner lane by a 5-step shuffle binary
// search), U arcs in flight per lane, no returning atomics.
// ---------------------------------------------------------------------------
#ifndef PICO_PUSH_E16
#define PICO_PUSH_E16 1  // push gathers read the 2-byte estimate array, not the 4-byte record
#endif
template <bool STATS>
__device__ void update_phase(const HcArgs &a, int t) {
    const int lane = lane_id();
    const long long ns = (long long)bcast_u64(&a.ctl->nS[t & 1]);
    unsigned long long *wc = &a.ctl->wc[t & 1];
    long long st_arcs = 0, st_guard = 0;
    const unsigned long long hot = pol_last(), cold = pol_first();
    const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    // segments per warp batch: 32 when there is work for every warp, fewer in
    // small rounds so that they still spread over all warps (a warp walks its
    // batch's arcs serially, 32*U at a time)
    const int bs = (int)min(32ll, max(1ll, (ns + nwarps - 1) / nwarps));
    const long long nbatch = (ns + bs - 1) / bs;
    for (long long round = 0;; round++) {
        // first batch static (warp id), the rest claimed dynamically (one
        // atomic per batch); small rounds cost no claim atomics
        long long bidx = gwarp;
        if (round > 0) {
            if (nbatch <= nwarps) break;
            if (lane == 0) bidx = nwarps + (long long)atomicAdd(wc, 1ull);
            bidx = __shfl_sync(FULL, bidx, 0);
        }
        if (bidx >= nbatch) break;
        long long i = bidx * bs + lane;
        long long b = 0;
        int len = 0, cv = 0, ov = 0;
        if (lane < bs && i < ns) {
            int2 sg = ld_stream_int2(a.S + i, cold);
            long long r0 = __ldg(a.rp + sg.x);
            long long r1 = r0 + __ldcg(a.slen + sg.x);  // (prefiltered) prefix of the row
            b = r0 + (long long)sg.y * a.tn.seg;
            len = (int)min((long long)a.tn.seg, r1 - b);
            cv = __ldcg(a.core + sg.x);
            ov = __ldcg(a.oldc + sg.x);
        }
        int incl = warp_incl_scan(len);
        int excl = incl - len;
        const int *rows = a.prefilter ? a.ro : a.ci;
        int total = __shfl_sync(FULL, incl, 31);
        constexpr int UA = PICO_ARC_U;
        ArcStep<UA> nx;
        if (total > 0) arc_fetch<UA>(nx, 0, total, excl, b, rows, cold);
        for (int j0 = 0; j0 < total; j0 += 32 * UA) {
            ArcStep<UA> cur = nx;
            if (PICO_ARC_PF && j0 + 32 * UA < total) arc_fetch<UA>(nx, j0 + 32 * UA, total, excl, b, rows, cold);
            // the UA estimate gathers (2-byte e16, or the 4-byte record) are
            // issued back to back (a fallback load between them would
            // serialise them: ncu showed each gather waited for before the
            // next one issued); saturated values resolve after
            int cu[UA];
            unsigned rr[UA];
#pragma unroll
            for (int q = 0; q < UA; q++)
#if PICO_PUSH_E16
                rr[q] = cur.v[q] >= 0 ? (unsigned)__ldcg(a.e16 + cur.v[q]) : 0u;
#else
                rr[q] = cur.v[q] >= 0 ? ld_rec(a.rec + cur.v[q], hot) : 0u;
#endif
#pragma unroll
            for (int q = 0; q < UA; q++) {
                cu[q] = (int)(rr[q] & 0xffffu);
                if (cu[q] == (int)RSAT) cu[q] = __ldcg(a.core + cur.v[q]);
            }
            int cvo[UA], ovo[UA];
            long long hb[UA];
            // all histogram bases are loaded before the first RED (the REDs'
            // memory clobber would otherwise serialise load -> RED -> load)
#pragma unroll
            for (int q = 0; q < UA; q++) {
                cvo[q] = __shfl_sync(FULL, cv, cur.lo[q]);
                ovo[q] = __shfl_sync(FULL, ov, cur.lo[q]);
                if (STATS) st_arcs += cur.v[q] >= 0;
                bool g = cur.v[q] >= 0 && cu[q] > cvo[q];  // N1/N3 neighbour
                if (STATS) st_guard += g;
                hb[q] = g ? rp_at(a, cur.v[q]) - 1 : LLONG_MIN;  // rowptr[0] - 1 = -1 is valid
            }
#pragma unroll
            for (int q = 0; q < UA; q++)
                if (hb[q] != LLONG_MIN) bin_move_mark(a, hb[q], cur.v[q], cu[q], cvo[q], ovo[q]);
            if (!PICO_ARC_PF && j0 + 32 * UA < total) arc_fetch<UA>(nx, j0 + 32 * UA, total, excl, b, rows, cold);
        }
    }
    if (STATS) {
        stat_add(&a.ctl->st_arcs, st_arcs);
        stat_add(&a.ctl->st_guarded, st_guard);
    }
}

// ---------------------------------------------------------------------------
// PICO_F_DEBUG_INVARIANTS: one warp per vertex recounts its
// neighbours' final estimates and compares them with its histogram -- bins
// b < core[v] hold #{u : core[u] = b}, the cap bin #{u : core[u] >= core[v]}
// -- and checks the h-index fixed point HINDEX(core(nbr v)) =
// core[v]: the cap count is >= core[v] and the count of
// neighbours at or above core[v] + 1 is < core[v] + 1.  Any violation sets
// *bad.  Caps up to 1024 are checked bin by bin, larger ones by their cap
// bin and fixed point only.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) hc_check_kernel(HcArgs a, int *bad) {
    __shared__ int sh[8][1025];
    const int wib = threadIdx.x >> 5, lane = lane_id();
    int *cnt = sh[wib];
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long v = gw; v < a.n; v += nw) {
        const long long r0 = a.rp[v], r1 = a.rp[v + 1];
        const int c = a.core[v];
        if (r1 == r0) {
            if (c != 0 && lane == 0) atomicOr(bad, 1);
            continue;
        }
        const int B = min(c, 1024);
        for (int b = lane; b <= B; b += 32) cnt[b] = 0;
        __syncwarp();
        int above = 0, above1 = 0;
        for (long long e = r0 + lane; e < r1; e += 32) {
            const int cu = a.core[a.ci[e]];
            above += cu >= c;
            above1 += cu >= c + 1;
            if (cu < c && cu <= B) atomicAdd(&cnt[cu], 1);
        }
        above = (int)warp_sum64(above);
        above1 = (int)warp_sum64(above1);
        __syncwarp();
        bool ok = c >= 1 && above >= c && above1 < c + 1;              // the fixed point
        ok = ok && a.histo[r0 - 1 + c] == above;                        // the cap bin
        if (c <= 1024)
            for (int b = 1 + lane; b < c; b += 32) ok = ok && a.histo[r0 - 1 + b] == cnt[b];
        if (__any_sync(FULL, !ok) && lane == 0) atomicOr(bad, 2);
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// UpdateHisto, pull direction (dense rounds), over the bucketed edge list:
// for each v-range bucket in turn every warp streams a contiguous slice of
// its (u, v) pairs; arc (u, v) applies the (v, u) bin move of a changed v
// with core[v] < core[u] to u's own histogram.  Consecutive lanes mostly
// share u, so core[u] / rowptr[u] loads and the bin moves coalesce; the one
// random access per arc is the 4-byte record of v, inside the bucket's
// L2-sized vertex slice.  No owner search, no per-row bookkeeping.
// ---------------------------------------------------------------------------
#ifndef PICO_PULL_U
#define PICO_PULL_U 4
#endif
#ifndef PICO_PULL_VEC
#define PICO_PULL_VEC 0  // int4 loads of the edge-list columns (A/B: DESIGN.md)
#endif
// v-side estimate records: one GPU gathers the 4-byte records of its own
// vertices (16|16 bits, saturated values fall back to the full arrays);
// a shard gathers 8-byte records (32|32 bits, never saturated) of the
// GLOBAL vertex space, fed by the exchanged triples (VRec64)
struct VRec32 {
    typedef unsigned T;
    static constexpr int SH = 16;
    static constexpr unsigned long long MASK = 0xffffull;
    static constexpr bool SAT = true;
};
struct VRec64 {
    typedef unsigned long long T;
    static constexpr int SH = 32;
    static constexpr unsigned long long MASK = 0xffffffffull;
    static constexpr bool SAT = false;
};

__device__ __forceinline__ unsigned long long pack_rec64(int k, int old) {
    return (unsigned long long)(unsigned)k | ((unsigned long long)(unsigned)old << 32);
}

template <bool STATS, class VR = VRec32>
__device__ void coo_pull_phase(const HcArgs &a, int t, const typename VR::T *vrec) {
    constexpr int UA = PICO_PULL_U;
    const int lane = lane_id();
    const unsigned *chg = a.chg + (t & 1) * a.nwords;
    long long st_arcs = 0, st_guard = 0;
    const unsigned long long hot = pol_last(), cold = pol_first();
    const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    __shared__ unsigned long long s_off[kMaxPass + 1];
    __syncthreads();
    if (threadIdx.x <= kMaxPass) s_off[threadIdx.x] = ld_volatile(a.boff + threadIdx.x);
    __syncthreads();
    for (int p = 0; p < a.npass; p++) {
    // static contiguous slices of bucket p, whole 32*UA steps (PICO_PULL_VEC:
    // steps aligned to 4 arcs, int4 loads, the arcs before bb masked)
    const long long bb = (long long)s_off[p], be = (long long)s_off[p + 1];
    const long long ab = PICO_PULL_VEC ? (bb & ~3ll) : bb;
    const long long steps = (be - ab + 32 * UA - 1) / (32 * UA);
    const long long s0 = steps * gwarp / nwarps, s1 = steps * (gwarp + 1) / nwarps;
    for (long long st = s0; st < s1; st++) {
        const long long e0 = ab + st * (32 * UA);
        int u[UA], v[UA];
        unsigned ru[UA];
        typename VR::T rv[UA];
        long long hb[UA];
#if PICO_PULL_VEC
        static_assert(UA == 4, "vector pull loads: 4 arcs per lane");
        {
            // lane L loads arcs e0 + 4L .. +3 as one int4 per column, then the
            // warp transposes so that step q of lane L is arc e0 + 32q + L (the
            // scalar mapping: consecutive lanes share u, the REDs coalesce)
            const long long ev = e0 + 4 * lane;
            int4 su = make_int4(-1, -1, -1, -1), sv = make_int4(0, 0, 0, 0);
            const bool vok = ((reinterpret_cast<unsigned long long>(a.pdst) | reinterpret_cast<unsigned long long>(a.psrc)) & 15) == 0;
            if (vok && ev + 3 < be && ev >= bb) {
                su = __ldcs(reinterpret_cast<const int4 *>(a.psrc + ev));
                sv = __ldcs(reinterpret_cast<const int4 *>(a.pdst + ev));
            } else {
                int *pu = &su.x, *pv = &sv.x;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const long long e = ev + j;
                    if (e >= bb && e < be) { pu[j] = __ldcs(a.psrc + e); pv[j] = __ldcs(a.pdst + e); }
                }
            }
#pragma unroll
            for (int q = 0; q < UA; q++) {
                const int src = q * 8 + (lane >> 2), j = lane & 3;
                const int u0 = __shfl_sync(FULL, su.x, src), u1 = __shfl_sync(FULL, su.y, src);
                const int u2 = __shfl_sync(FULL, su.z, src), u3 = __shfl_sync(FULL, su.w, src);
                const int v0 = __shfl_sync(FULL, sv.x, src), v1 = __shfl_sync(FULL, sv.y, src);
                const int v2 = __shfl_sync(FULL, sv.z, src), v3 = __shfl_sync(FULL, sv.w, src);
                u[q] = j == 0 ? u0 : j == 1 ? u1 : j == 2 ? u2 : u3;
                v[q] = j == 0 ? v0 : j == 1 ? v1 : j == 2 ? v2 : v3;
            }
        }
#else
#pragma unroll
        for (int q = 0; q < UA; q++) {
            long long e = e0 + q * 32 + lane;
            bool ok = e < be;
            u[q] = ok ? ld_stream(a.psrc + e, cold) : -1;
            v[q] = ok ? ld_stream(a.pdst + e, cold) : 0;
        }
#endif
#pragma unroll
        for (int q = 0; q < UA; q++) {
            ru[q] = u[q] >= 0 ? ld_rec(a.rec + u[q], hot) : 0u;
            rv[q] = u[q] >= 0 ? __ldcg(vrec + v[q]) : 0;
            hb[q] = u[q] >= 0 ? rp_at(a, u[q]) - 1 : 0;
        }
#pragma unroll
        for (int q = 0; q < UA; q++) {
            const bool ok = u[q] >= 0;
            if (STATS) st_arcs += ok;
            int cu = (int)(ru[q] & 0xffffu);
            if (ok && cu == (int)RSAT) cu = __ldcg(a.core + u[q]);
            int nlo = (int)(rv[q] & VR::MASK), nhi = (int)(rv[q] >> VR::SH);
            int cv = nlo, ov = nhi;
            bool ch = nlo != nhi;  // exact while the new half is unsaturated
            if (VR::SAT && ok && nlo == (int)RSAT) {  // estimate >= 65535: full arrays
                ch = (__ldcg(chg + (v[q] >> 5)) >> (v[q] & 31)) & 1u;
                cv = __ldcg(a.core + v[q]);
                ov = ch ? __ldcg(a.oldc + v[q]) : cv;
            } else if (VR::SAT && ok && ch && nhi == (int)RSAT && cu > (int)RSAT) {
                ov = __ldcg(a.oldc + v[q]);  // saturated old half, needed exactly
            }
            bool g = ok && ch && cv < cu;  // N1/N3 neighbour
            if (STATS) st_guard += g;
            // source bin min(oldcore[v], core[u]): the cap bin iff oldcore[v] >= core[u]
            const bool capdec = ov >= cu;
            if (g) {
                red_add(a.histo + hb[q] + (capdec ? cu : ov), -1);
                if (capdec) red_or(a.capd + (u[q] >> 5), 1u << (u[q] & 31));
                red_add(a.histo + hb[q] + cv, 1);
            }
        }
    }
    }  // buckets
    if (STATS) {
        stat_add(&a.ctl->st_arcs, st_arcs);
        stat_add(&a.ctl->st_guarded, st_guard);
    }
}

// ---------------------------------------------------------------------------
// SumHisto of round t for one candidate vertex per lane (valid lanes): walk
// k = core_old, core_old-1, ... adding bins until sum >= k, thread per vertex
// for the first 32 bins, then warp-cooperative 32-bin chunks for long walks;
// writes core/oldcore/cap bin and appends the vertex's UpdateHisto segments.
// Warp-collective (all 32 lanes call).
// ---------------------------------------------------------------------------
template <bool STATS>
__device__ __forceinline__ void sum_lanes(const HcArgs &a, int t, bool valid, int v, ChangeAcc &acc,
                                          long long &st_bins, unsigned long long *nS) {
    const int lane = lane_id();
    int cold = 0, k = 0, sum = 0;
    long long hb = 0, d = 0;
    bool done = true;
    if (valid) {
        cold = __ldcg(a.core + v);
        hb = rp_at(a, v) - 1;  // bin b at hb + b
        d = rp_at(a, v + 1) - hb - 1;
        k = cold;
        done = false;
        // (a broken invariant can walk k below 1 here: the warp loop below
        // then stops at once)
        for (int stp = 0; stp < 32; stp++) {
            if (k == 0 && a.allow_zero) { done = true; break; }  // no neighbour left: h = 0
            sum += __ldcg(a.histo + hb + k);
            if (STATS) st_bins++;
            if (sum >= k) { done = true; break; }
            k--;
        }
    }
    unsigned m = __ballot_sync(FULL, !done);
    while (m) {
        int L = __ffs(m) - 1;
        m &= m - 1;
        long long hbL = __shfl_sync(FULL, hb, L);
        int kL = __shfl_sync(FULL, k, L);
        int sL = __shfl_sync(FULL, sum, L);
        int rk = 0, rs = 0;
        for (;;) {
            int kk = kL - lane;
            int val = kk >= 1 ? __ldcg(a.histo + hbL + kk) : 0;
            int incl = warp_incl_scan(val);
            int s = sL + incl;
            unsigned mm = __ballot_sync(FULL, kk >= 1 && s >= kk);
            if (STATS) st_bins += (kk >= 1) ? 1 : 0;
            if (mm) {
                int f = __ffs(mm) - 1;
                rk = kL - f;
                rs = __shfl_sync(FULL, s, f);
                break;
            }
            if (kL <= 32) {
                // no bin down to 1 reaches its index: the vertex has no
                // neighbour left (decremental updates: h = 0) or a histogram
                // invariant is broken (the input is not a symmetric
                // deduplicated loop-free CSR); stop instead of walking on
                if (!a.allow_zero && lane == 0) *reinterpret_cast<volatile int *>(&a.ctl->error) = 1;
                rk = a.allow_zero ? 0 : 1;
                rs = a.allow_zero ? 0 : 1;
                break;
            }
            sL += __shfl_sync(FULL, incl, 31);
            kL -= 32;
        }
        if (lane == L) { k = rk; sum = rs; }
    }
    int nseg = 0;
    if (valid) {
        a.core[v] = k;
        a.rec[v] = pack_rec(k, cold);
        a.e16[v] = (unsigned short)min(k, (int)RSAT);
        a.oldc[v] = cold;
        if (k > 0) a.histo[hb + k] = sum;  // cap bin := cnt
        int L = scan_len(a, hb + 1, (int)d, k);
        a.slen[v] = L;
        nseg = nseg_of(L, a.tn.seg);
        acc.note(a, t, v, k, d);
    }
    warp_append_segments(v, nseg, a.S, nS);
}

// SumHisto of round t over an explicit frontier list F_t (count nF[t&1]):
// the sharded path, whose UpdateHisto pushes with the returned-value trigger
template <bool STATS>
__device__ void sum_phase(const HcArgs &a, int t, long long gthread, long long nthreads) {
    const long long nf = (long long)bcast_u64(&a.ctl->nF[t & 1]);
    unsigned long long *nS = &a.ctl->nS[t & 1];
    long long iters = (nf + nthreads - 1) / nthreads;
    long long st_bins = 0;
    ChangeAcc acc;
    for (long long it = 0; it < iters; it++) {
        long long i = it * nthreads + gthread;
        bool valid = i < nf;
        int v = valid ? __ldcg(a.F + i) : 0;
        sum_lanes<STATS>(a, t, valid, v, acc, st_bins, nS);
    }
    acc.flush(a, t, nullptr);
    if (STATS) stat_add(&a.ctl->st_bins, st_bins);
}

// SumHisto of round t over the vertices marked in the cap-touched bitmap by
// UpdateHisto(t-1): F_t = {marked u : cnt(u) < core[u]} (Theorem 2).  Each
// lane owns one bitmap word (read and cleared); |F_t| -> nF[t&1].
template <bool STATS>
__device__ void collect_sum_phase(const HcArgs &a, int t) {
    const int lane = lane_id();
    const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    unsigned long long *nS = &a.ctl->nS[t & 1];
    const unsigned *chgp = a.chg + ((t - 1) & 1) * a.nwords;  // C_{t-1}
    long long st_bins = 0;
    ChangeAcc acc;
    for (long long wbase = gwarp * 32; wbase < a.nwords; wbase += nwarps * 32) {
        long long wi = wbase + lane;
        unsigned w = 0;
        if (wi < a.nwords) {
            w = __ldcg(a.capd + wi);
            if (w) a.capd[wi] = 0u;
            // C_{t-1}'s records stop flagging a change (old byte := new byte);
            // the same lane then writes the records of F_t in this word, so
            // the reset never overtakes a newer record
            unsigned cw = __ldcg(chgp + wi);
            while (cw) {
                int v = (int)(wi * 32 + (__ffs(cw) - 1));
                cw &= cw - 1;
                int c = __ldcg(a.core + v);
                a.rec[v] = pack_rec(c, c);
            }
        }
        while (__any_sync(FULL, w != 0)) {
            bool valid = false;
            int v = 0;
            if (w) {
                v = (int)(wi * 32 + (__ffs(w) - 1));
                w &= w - 1;
                int cu = __ldcg(a.core + v);
                valid = __ldcg(a.histo + rp_at(a, v) + cu - 1) < cu;  // cnt < core
            }
            sum_lanes<STATS>(a, t, valid, v, acc, st_bins, nS);
        }
    }
    acc.flush(a, t, &a.ctl->nF[t & 1]);
    if (STATS) {
        stat_add(&a.ctl->st_bins, st_bins);
        stat_add(&a.ctl->st_pushes, acc.cnt);
    }
}

// start-of-UpdateHisto(t) bookkeeping: reset round t+1's counters (unused
// during this phase), clear round t+1's changed bitmap, pick push or pull
__device__ __forceinline__ bool update_prologue(const HcArgs &a, int t, bool leader, long long gthread,
                                                long long nthreads, bool stats) {
    if (leader) {
        a.ctl->nS[(t + 1) & 1] = 0;
        a.ctl->nF[(t + 1) & 1] = 0;
        a.ctl->wc[(t + 1) & 1] = 0;
        a.ctl->arcsC[(t + 1) & 1] = 0;
        a.ctl->mincv[(t + 1) & 1] = INT_MAX;
        if (stats) a.ctl->st_segs += ld_volatile(&a.ctl->nS[t & 1]);
    }
    unsigned *clr = a.chg + ((t + 1) & 1) * a.nwords;
    for (long long w = gthread; w < a.nwords; w += nthreads) clr[w] = 0u;
    unsigned long long ac = bcast_u64(&a.ctl->arcsC[t & 1]);
    if (leader && (unsigned long long)t < a.fsz_cap) a.rarcs[t] = ac;
    return a.allow_pull && 10ull * ac >= (unsigned long long)a.tn.pull_tenths * (unsigned long long)a.arcs;
}

// ---------------------------------------------------------------------------
// persistent cooperative kernel: all rounds t >= 1 with grid barriers
//   UpdateHisto(t)  |barrier|  SumHisto(t+1) over the marked vertices  |barrier|
// ---------------------------------------------------------------------------
template <bool STATS>
__global__ void __launch_bounds__(512, PICO_ROUNDS_MINB) hc_rounds_kernel(HcArgs a) {
    const long long gthread = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    if (bcast_u64(&a.ctl->nS[1]) == 0) return;  // C_1 empty: l2 = 0 (uniform)
    if (leader) a.rtime[0] = globaltimer();
    for (int t = 1;; t++) {
        bool pull = update_prologue(a, t, leader, gthread, nthreads, STATS);
        if (pull) {
            if (STATS && leader) a.ctl->st_pull++;
            coo_pull_phase<STATS>(a, t, a.rec);
        } else {
            update_phase<STATS>(a, t);
        }
        grid_barrier(&a.ctl->bar_arrive, &a.ctl->bar_gen);
        if (leader && (unsigned long long)t < a.fsz_cap) a.rtime[2 * t - 1] = globaltimer();
        collect_sum_phase<STATS>(a, t + 1);
        grid_barrier(&a.ctl->bar_arrive, &a.ctl->bar_gen);
        if (leader && (unsigned long long)t < a.fsz_cap) a.rtime[2 * t] = globaltimer();
        unsigned long long nf = bcast_u64(&a.ctl->nF[(t + 1) & 1]);
        if (nf == 0) break;
        // every round lowers the sum of the estimates, so a valid run has l2 <= 2m rounds
        // (a long path needs ~n/2, far beyond the recorded kFszCap); more is broken input
        if ((unsigned long long)t > (unsigned long long)a.arcs + 2) {
            if (leader) *reinterpret_cast<volatile int *>(&a.ctl->error) = 1;
            break;
        }
        if (leader) {
            a.ctl->rounds++;
            if ((unsigned long long)t < a.fsz_cap) a.fsz[t] = nf;
            if (STATS) a.ctl->st_frontier += nf;
        }
    }
}

// host-loop variants (PICO_F_HOST_LOOP): one launch per phase
template <bool STATS>
__global__ void __launch_bounds__(512, 2) hc_update_kernel(HcArgs a, int t, int pull) {
    const long long gthread = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    update_prologue(a, t, leader, gthread, nthreads, STATS);
    if (pull) {
        if (STATS && leader) a.ctl->st_pull++;
        coo_pull_phase<STATS>(a, t, a.rec);
    } else {
        update_phase<STATS>(a, t);
    }
}

template <bool STATS>
__global__ void __launch_bounds__(512, 2) hc_collect_sum_kernel(HcArgs a, int t) {
    collect_sum_phase<STATS>(a, t);
}


// ---------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

Tune hc_tune(uint32_t flags) {
    Tune t;
    if (flags & PICO_F_TINY_TILES) {
        t.a_max = 4; t.b_max = 12; t.c_bins = 16; t.seg = 4;
    } else {
        t.a_max = 16; t.b_max = PICO_BMAX; t.c_bins = PICO_CBINS; t.seg = PICO_HC_SEG;
    }
#ifndef PICO_PULL_DIV
#define PICO_PULL_DIV 2
#endif
#ifndef PICO_PULL_TENTHS
#define PICO_PULL_TENTHS 4
#endif
    t.pull_div = PICO_PULL_DIV;  // shards: pull when sum_{v in C_t} deg(v) >= 2m / pull_div
    // one GPU: pull when sum_{v in C_t} deg(v) >= 0.4 * 2m (RMAT-26 per-round
    // A/B, profiles/r02/rounds_T_*: round 10 at 0.42 pulls in 10.4 ms against
    // 11.5 ms of push, round 11 at 0.38 pushes in 8.3 ms against 10.1)
    t.pull_tenths = PICO_PULL_TENTHS;
    if (flags & PICO_F_PULL_ALWAYS) { t.pull_div = 1 << 30; t.pull_tenths = 0; }
    return t;
}

// whether the class-B InitHisto runs as two launches split by row length
// (the 2-byte degree shadow of n vertices outgrows a share of the L2)
static bool hc_init_split(long long n) { return n >= (8ll << 20); }

// whether dense rounds may pull, and into how many v-range passes
static bool hc_allow_pull(long long n, uint32_t flags) {
    return (flags & PICO_F_PUSH_ONLY) ? false : (flags & PICO_F_PULL_ALWAYS) ? true : (n >= kPullMinN);
}

// v-range width of a pull pass: 2^shift vertices whose 4-byte records fit
// PICO_PASS_MB (the L2 slice one pass gathers from), at most kMaxPass passes
// (rb: bytes per v-side record -- 4 on one GPU, 8 on a shard)
static int hc_pshift(long long n, uint32_t flags, int rb = 4) {
    int sh = 0;
    if (flags & PICO_F_TINY_TILES) {  // exercise the passes on small graphs
        while ((1ll << sh) * 3 < n) sh++;
    } else {
        while (((long long)rb << (sh + 1)) <= ((long long)PICO_PASS_MB << 20)) sh++;
    }
    while (((n - 1) >> sh) + 1 > kMaxPass) sh++;
    return sh;
}

static int hc_npass(long long n, uint32_t flags, int rb = 4) {
    if (!hc_allow_pull(n, flags) || n < 2) return 1;
    return (int)(((n - 1) >> hc_pshift(n, flags, rb)) + 1);
}

struct HcLayout {
    size_t fcnt, ctl, fsz, rarcs, rtime, histo, c8, c16, rec, e16, rp32, oldc, F, BC, S, H, chg, ro, db, slen, capd, bk, psrc, pdst,
        elc, elt, total;
    long long nwords, scap, hcap, nbcap;
    size_t eltb;
    int npass;
};

// nv: size of the v-side id space (n on one GPU, n_global on a shard), rb:
// bytes per v-side record
static HcLayout hc_layout(long long n, long long arcs, uint32_t flags, long long nv = -1, int rb = 4) {
    Tune tn = hc_tune(flags);
    HcLayout L;
    if (nv < 0) nv = n;
    const bool pull = hc_allow_pull(nv, flags);
    L.npass = hc_npass(nv, flags, rb);
    L.nwords = (n + 31) / 32;
    L.scap = n + arcs / tn.seg + 64;
    L.hcap = 2 * (arcs / tn.seg) + 64;
    size_t b = 0;
    L.ctl = b; b += align256(sizeof(Ctrl));
    L.fsz = b; b += align256(sizeof(unsigned long long) * kFszCap);
    L.rarcs = b; b += align256(sizeof(unsigned long long) * kFszCap);
    L.rtime = b; b += align256(sizeof(unsigned long long) * (2 * kFszCap + 1));
    L.histo = b; b += align256(sizeof(int) * (size_t)arcs);
    L.c8 = b; b += align256(sizeof(shadow_t) * (size_t)n);
    L.c16 = b; b += align256(sizeof(unsigned short) * (size_t)n);
    L.rec = b; b += align256(sizeof(unsigned) * (size_t)n);
    L.e16 = b; b += align256(sizeof(unsigned short) * (size_t)n);
    L.rp32 = b; b += align256(sizeof(unsigned) * (size_t)(n + 1));
    L.oldc = b; b += align256(sizeof(int) * (size_t)n);
    L.F = b; b += align256(sizeof(int) * (size_t)n);
    L.BC = b; b += align256(sizeof(int) * (size_t)n);
    L.S = b; b += align256(sizeof(int2) * (size_t)L.scap);
    L.H = b; b += align256(sizeof(int2) * (size_t)L.hcap);
    L.chg = b; b += align256(sizeof(unsigned) * 2 * (size_t)L.nwords);
    L.ro = b; b += align256(sizeof(int) * (size_t)((flags & PICO_F_PREFILTER) ? std::max(arcs, 1ll) : 1));
    L.db = b; b += align256((size_t)n);
    L.slen = b; b += align256(sizeof(int) * (size_t)n);
    L.capd = b; b += align256(sizeof(unsigned) * (size_t)L.nwords);
    L.fcnt = b; b += align256(sizeof(int) * (size_t)((flags & PICO_F_STATS) ? std::max(n, 1ll) : 1));
    const size_t el = pull ? (size_t)std::max(arcs, 1ll) : 1;  // pull edge list
    L.bk = b; b += align256(sizeof(unsigned long long) * (kMaxPass + 1));
    L.psrc = b; b += align256(sizeof(int) * el);
    L.pdst = b; b += align256(sizeof(int) * (L.npass > 1 ? el : 1));  // one bucket: colidx itself
    // edge-list build: bucket-major count matrix over the 2048-arc chunks + scan temp
    L.nbcap = (pull && L.npass > 1) ? (arcs + kElChunk - 1) / kElChunk : 0;
    long long ncnt = std::max(1ll, L.npass * L.nbcap);
    L.elc = b; b += align256(sizeof(unsigned long long) * (size_t)ncnt);
    L.eltb = 0;
    cub::DeviceScan::ExclusiveSum((void *)nullptr, L.eltb, (unsigned long long *)nullptr,
                                  (unsigned long long *)nullptr, (int)ncnt);
    L.elt = b; b += align256(L.eltb);
    L.total = b;
    return L;
}

size_t hc_workspace_bytes(long long n, long long arcs, uint32_t flags) {
    return hc_layout(n, arcs, flags).total;
}

// Phase slots double as NVTX ranges (always on; no-ops without a tool
// attached): nsys / ncu --nvtx attribute every launch to its phase
struct Timer {
    cudaStream_t s;
    bool on;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
    void start(int slot) {
        nvtx_push(slot);
        if (!on) return;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        ev.push_back({slot, {a, b}});
    }
    void stop() {
        nvtxRangePop();
        if (!on) return;
        cudaEventRecord(ev.back().second.second, s);
    }
    void collect(pico_stats_t *st) {
        for (auto &e : ev) {
            float ms = 0;
            cudaEventSynchronize(e.second.second);
            cudaEventElapsedTime(&ms, e.second.first, e.second.second);
            if (st) {
                st->kernel_ms[e.first] += ms;
                st->kernel_launches[e.first] += 1;
            }
            cudaEventDestroy(e.second.first);
            cudaEventDestroy(e.second.second);
        }
        ev.clear();
    }
};

// warm start: the round-0 estimates h0 replace the degrees in the arrays
// InitHisto gathers (oldcore = the exact value, c8 / c16 its shadows)
__global__ void hc_h0_kernel(HcArgs a) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += nthreads) {
        const int d = (int)(a.rp[v + 1] - a.rp[v]);
        const int x = min(a.h0[v], d);
        a.oldc[v] = x;
        set_c8(a, (int)v, x);
    }
}

template <bool STATS>
static cudaError_t hc_run_t(const long long *rp, const int *ci, long long n, long long arcs,
                            int *core, cudaStream_t s, uint32_t flags, void *ws,
                            pico_stats_t *st, const DevInfo &dev, HcArgs *keep = nullptr,
                            const int *h0 = nullptr) {
    HcArgs a;
    a.allow_zero = 0;
    a.h0 = h0;
    Tune tn = hc_tune(flags);
    HcLayout L = hc_layout(n, arcs, flags);
    char *p = (char *)ws;
    a.ctl = (Ctrl *)(p + L.ctl);
    a.fsz = (unsigned long long *)(p + L.fsz);
    a.rarcs = (unsigned long long *)(p + L.rarcs);
    a.rtime = (unsigned long long *)(p + L.rtime);
    a.fsz_cap = kFszCap;
    a.histo = (int *)(p + L.histo);
    a.c8 = (shadow_t *)(p + L.c8);
    a.c16 = (unsigned short *)(p + L.c16);
    a.rec = (unsigned *)(p + L.rec);
    a.e16 = (unsigned short *)(p + L.e16);
    a.rp32 = arcs < (1ll << 32) ? (unsigned *)(p + L.rp32) : nullptr;
    a.oldc = (int *)(p + L.oldc);
    a.F = (int *)(p + L.F);
    a.BC = (int *)(p + L.BC);
    a.S = (int2 *)(p + L.S);
    a.H = (int2 *)(p + L.H);
    a.chg = (unsigned *)(p + L.chg);
    a.ro = (int *)(p + L.ro);
    a.db = (unsigned char *)(p + L.db);
    a.slen = (int *)(p + L.slen);
    a.capd = (unsigned *)(p + L.capd);
    a.boff = (unsigned long long *)(p + L.bk);
    a.psrc = (int *)(p + L.psrc);
    a.pdst = (int *)(p + L.pdst);
    a.npass = L.npass;
    a.pshift = hc_pshift(n, flags);
    if (L.npass == 1) a.pdst = const_cast<int *>(ci);  // one bucket: (src, colidx)
    a.nwords = L.nwords;
    a.rp = rp; a.ci = ci; a.n = (int)n; a.arcs = arcs; a.core = core; a.tn = tn;
    a.allow_pull = hc_allow_pull(n, flags);
    a.nv8 = a.c8;
    a.nv16 = a.c16;
    a.nv32 = a.oldc;
    a.prefilter = (flags & PICO_F_PREFILTER) ? 1 : 0;
    const bool fcounts = STATS && st && st->frontier_counts && st->frontier_counts_cap >= n && !keep;
    if (fcounts) a.fcnt = (int *)(p + L.fcnt);

    Timer tm{s, (flags & PICO_F_TIMING) != 0, {}};
    cudaError_t err;
    Ctrl hc{};
    hc.mincv[0] = hc.mincv[1] = INT_MAX;
    if ((err = cudaMemcpyAsync(a.ctl, &hc, sizeof(Ctrl), cudaMemcpyHostToDevice, s))) return err;
    if ((err = cudaMemsetAsync(a.chg, 0, sizeof(unsigned) * 2 * (size_t)L.nwords, s))) return err;
    if ((err = cudaMemsetAsync(a.capd, 0, sizeof(unsigned) * (size_t)L.nwords, s))) return err;
    if (fcounts && (err = cudaMemsetAsync(a.fcnt, 0, sizeof(int) * (size_t)n, s))) return err;

    const int sms = dev.sms;
    long long launches = 0;
    // H0
    tm.start(PICO_K_DEGREE);
    {
        int blocks = (int)std::min<long long>((n + 255) / 256, (long long)sms * 16);
        hc_degree_kernel<<<std::max(blocks, 1), 256, 0, s>>>(a);
        launches++;
        if (h0 && n > 0) {
            hc_h0_kernel<<<std::max(blocks, 1), 256, 0, s>>>(a);
            launches++;
        }
    }
    tm.stop();
    // the bucketed edge list is built before InitHisto: it borrows the
    // histogram space for its row-owner column
    {
        if (a.allow_pull && arcs > 0) {  // bucketed edge list for the pull rounds
            tm.start(PICO_K_EDGELIST);
            // src goes straight into psrc (one bucket) or through the histogram
            // space, which InitHisto has not written yet -- see the launch order
            int *src = L.npass > 1 ? a.histo : a.psrc;
            int nb = (int)std::min<long long>((n + 255) / 256, (long long)sms * 8);
            hc_el_src_short_kernel<<<std::max(nb, 1), 256, 0, s>>>(a, src);
            hc_el_src_long_kernel<<<sms * 8, 256, 0, s>>>(a, src);
            launches += 2;
            if (L.npass > 1) {
                unsigned long long *cnt = (unsigned long long *)(p + L.elc);
                hc_el_count_kernel<<<sms * 16, 256, 0, s>>>(a, cnt, L.nbcap);
                size_t tb = L.eltb;
                if ((err = cub::DeviceScan::ExclusiveSum(p + L.elt, tb, cnt, cnt, (int)(L.npass * L.nbcap), s)))
                    return err;
                hc_el_fill_kernel<<<sms * 16, 256, 0, s>>>(a, src, cnt, L.nbcap);
                hc_el_offsets_kernel<<<1, 32, 0, s>>>(a, L.nbcap, cnt);
                launches += 3;
            } else {
                unsigned long long off[kMaxPass + 1];
                for (int q = 0; q <= kMaxPass; q++) off[q] = q == 0 ? 0 : (unsigned long long)arcs;
                if ((err = cudaMemcpyAsync(a.boff, off, sizeof(off), cudaMemcpyHostToDevice, s))) return err;
            }
            tm.stop();
        }
    }
    // H1-H3 (round 1)
    tm.start(PICO_K_INIT);
    {
        if (a.prefilter) {  // bucket-ordered copies of the rows with deg > a_max
            hc_reorder_warp_kernel<<<sms * 4, 256, 0, s>>>(a);
            hc_reorder_cta_kernel<<<sms * 2, 512, 0, s>>>(a);
            launches += 2;
        }
        int blocks = (int)std::min<long long>((n + 255) / 256, (long long)sms * 8);
        hc_init_small_kernel<STATS><<<std::max(blocks, 1), 256, 0, s>>>(a);
        size_t smB = sizeof(int) * (size_t)(tn.b_max + 1) * 8;
        int occB = 0, occC = 0;
        if (hc_init_split(n)) {
            size_t smB1 = sizeof(int) * (size_t)init_warp_stride<1>(tn.b_max) * 8;
            int occB1 = 0;
            cudaFuncSetAttribute(hc_init_warp_kernel<STATS, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smB1);
            cudaFuncSetAttribute(hc_init_warp_kernel<STATS, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smB);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occB1, hc_init_warp_kernel<STATS, 1>, 256, smB1);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occB, hc_init_warp_kernel<STATS, 2>, 256, smB);
            hc_init_warp_kernel<STATS, 1><<<sms * std::max(1, occB1), 256, smB1, s>>>(a);
            hc_init_warp_kernel<STATS, 2><<<sms * std::max(1, occB), 256, smB, s>>>(a);
            launches++;
        } else {
            cudaFuncSetAttribute(hc_init_warp_kernel<STATS, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smB);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occB, hc_init_warp_kernel<STATS, 0>, 256, smB);
            hc_init_warp_kernel<STATS, 0><<<sms * std::max(1, occB), 256, smB, s>>>(a);
        }
        size_t smC = sizeof(int) * (size_t)(tn.c_bins + 1);
        cudaFuncSetAttribute(hc_init_cta_kernel<STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smC);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occC, hc_init_cta_kernel<STATS>, 512, smC);
        hc_init_cta_kernel<STATS><<<sms * std::max(1, occC), 512, smC, s>>>(a);
        {
            // big shared-memory tier of the fallback: as many bins as fit
            int maxsm = 0;
            cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev.device);
            int big = (flags & PICO_F_TINY_TILES) ? 2 * tn.c_bins : (maxsm - 1024) / (int)sizeof(int) - 1;
            big = std::max(big, 0);
            const size_t smF = sizeof(int) * (size_t)(big + 1);
            if (big > tn.c_bins &&
                cudaFuncSetAttribute(hc_init_fallback_kernel<STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smF) == cudaSuccess) {
                hc_init_fallback_kernel<STATS><<<sms, 1024, smF, s>>>(a, big);
            } else {
                cudaGetLastError();
                hc_init_fallback_kernel<STATS><<<sms, 1024, 0, s>>>(a, 0);
            }
        }
        int nb = (int)std::min<long long>((n + 255) / 256, (long long)sms * 8);
        hc_shadow_kernel<<<std::max(nb, 1), 256, 0, s>>>(a);
        launches += 5;
    }
    tm.stop();
    if ((err = cudaGetLastError())) return err;

    unsigned long long c1 = 0, s1 = 0;
    if ((err = cudaMemcpyAsync(&c1, &a.ctl->nF[1], sizeof(c1), cudaMemcpyDeviceToHost, s))) return err;
    if ((err = cudaMemcpyAsync(&s1, &a.ctl->nS[1], sizeof(s1), cudaMemcpyDeviceToHost, s))) return err;
    if ((err = cudaStreamSynchronize(s))) return err;
    // F_1 = C_1 (Theorem 2), recorded at fsz[0]
    unsigned long long rounds = c1 ? 1 : 0;
    std::vector<unsigned long long> hsz;
    if (c1) hsz.push_back(c1);
    // counters as the rounds expect them: nF[1] held |C_1|, F list empty
    if ((err = cudaMemsetAsync(&a.ctl->nF[1], 0, sizeof(unsigned long long), s))) return err;

    std::vector<unsigned long long> harcs;
    if (c1) {
        if (flags & PICO_F_HOST_LOOP) {
            int blocks = sms * 4;
            for (int t = 1;; t++) {
                unsigned long long ac = 0;
                if ((err = cudaMemcpyAsync(&ac, &a.ctl->arcsC[t & 1], sizeof(ac), cudaMemcpyDeviceToHost, s)))
                    return err;
                if ((err = cudaStreamSynchronize(s))) return err;
                harcs.push_back(ac);
                int pull = a.allow_pull && 10ull * ac >= (unsigned long long)tn.pull_tenths * (unsigned long long)arcs;
                tm.start(PICO_K_UPDATE);
                hc_update_kernel<STATS><<<blocks, 512, 0, s>>>(a, t, pull);
                tm.stop();
                tm.start(PICO_K_SUM);
                hc_collect_sum_kernel<STATS><<<blocks, 512, 0, s>>>(a, t + 1);
                tm.stop();
                launches += 2;
                unsigned long long nf = 0;
                if ((err = cudaMemcpyAsync(&nf, &a.ctl->nF[(t + 1) & 1], sizeof(nf),
                                           cudaMemcpyDeviceToHost, s)))
                    return err;
                if ((err = cudaStreamSynchronize(s))) return err;
                if (nf == 0) break;
                rounds++;
                hsz.push_back(nf);
                if ((unsigned long long)t > (unsigned long long)arcs + 2) return cudaErrorAssert;  // broken input
            }
            int derr = 0;
            if ((err = cudaMemcpyAsync(&derr, &a.ctl->error, sizeof(derr), cudaMemcpyDeviceToHost, s))) return err;
            if ((err = cudaStreamSynchronize(s))) return err;
            if (derr) return cudaErrorAssert;
        } else {
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hc_rounds_kernel<STATS>, 512, 0);
            int per = std::max(1, occ);
            int blocks = sms * per;
            void *args[] = {&a};
            // PICO_F_L2_PERSIST (A/B): the push rounds' gather target e16 as a
            // persisting L2 access-policy window for the round kernel
            const bool persist = (flags & PICO_F_L2_PERSIST) && n > 0;
            if (persist) {
                int maxp = 0, maxw = 0;
                cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev.device);
                cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev.device);
                const size_t bytes = std::min<size_t>(sizeof(unsigned short) * (size_t)n, (size_t)maxw);
                const size_t keep = std::min<size_t>(bytes, (size_t)maxp);
                cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, keep);
                cudaStreamAttrValue v{};
                v.accessPolicyWindow.base_ptr = a.e16;
                v.accessPolicyWindow.num_bytes = bytes;
                v.accessPolicyWindow.hitRatio = bytes ? (float)keep / (float)bytes : 0.f;
                v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
            }
            tm.start(PICO_K_ROUNDS);
            err = cudaLaunchCooperativeKernel((const void *)hc_rounds_kernel<STATS>, blocks, 512, args, 0, s);
            tm.stop();
            launches++;
            if (persist) {  // back to the default policy (the limit is process-wide state)
                cudaStreamAttrValue v{};
                v.accessPolicyWindow.num_bytes = 0;
                cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
                cudaCtxResetPersistingL2Cache();
                cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
            }
            if (err) return err;
            unsigned long long devrounds = 0;
            int derr = 0;
            if ((err = cudaMemcpyAsync(&devrounds, &a.ctl->rounds, sizeof(devrounds),
                                       cudaMemcpyDeviceToHost, s)))
                return err;
            if ((err = cudaMemcpyAsync(&derr, &a.ctl->error, sizeof(derr), cudaMemcpyDeviceToHost, s))) return err;
            if ((err = cudaStreamSynchronize(s))) return err;
            if (derr) return cudaErrorAssert;  // broken histogram invariant (capi: PICO_EGRAPH)
            size_t nr = (size_t)std::min<unsigned long long>(devrounds + 2, kFszCap);
            std::vector<unsigned long long> dsz(nr, 0), dar(nr, 0), dtm(2 * nr + 1, 0);
            if (st && st->round_ns) {
                if ((err = cudaMemcpyAsync(dtm.data(), a.rtime, sizeof(unsigned long long) * (2 * nr + 1),
                                           cudaMemcpyDeviceToHost, s)))
                    return err;
            }
            if ((err = cudaMemcpyAsync(dsz.data(), a.fsz, sizeof(unsigned long long) * nr,
                                       cudaMemcpyDeviceToHost, s)))
                return err;
            if ((err = cudaMemcpyAsync(dar.data(), a.rarcs, sizeof(unsigned long long) * nr,
                                       cudaMemcpyDeviceToHost, s)))
                return err;
            if ((err = cudaStreamSynchronize(s))) return err;
            if (st && st->round_ns) {
                // phases of rounds 1..devrounds+1 (the last one found F empty)
                for (unsigned long long t = 1; t <= devrounds + 1 && 2 * t <= 2 * nr; t++) {
                    if ((int64_t)(2 * t) > 2 * st->frontier_sizes_cap) break;
                    st->round_ns[2 * (t - 1)] = (int64_t)(dtm[2 * t - 1] - dtm[2 * t - 2]);
                    st->round_ns[2 * (t - 1) + 1] = (int64_t)(dtm[2 * t] - dtm[2 * t - 1]);
                }
            }
            rounds += devrounds;
            for (unsigned long long t = 1; t <= devrounds && t < kFszCap; t++) hsz.push_back(dsz[t]);
            for (unsigned long long t = 1; t <= devrounds + 1 && t < nr; t++) harcs.push_back(dar[t]);
        }
    }
    if ((err = cudaGetLastError())) return err;
    if ((flags & PICO_F_DEBUG_INVARIANTS) && n > 0) {
        int *bad = (int *)a.F;  // free after init
        int hbad = 0;
        if ((err = cudaMemsetAsync(bad, 0, sizeof(int), s))) return err;
        hc_check_kernel<<<sms * 8, 256, 0, s>>>(a, bad);
        launches++;
        if ((err = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s))) return err;
        if ((err = cudaStreamSynchronize(s))) return err;
        if (hbad) return cudaErrorAssert;  // capi: PICO_EGRAPH
    }
    if (st) {
        st->rounds = (int64_t)rounds;
        st->kernel_count += launches;
        if (fcounts) {
            if ((err = cudaMemcpyAsync(st->frontier_counts, a.fcnt, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost, s)))
                return err;
            if ((err = cudaStreamSynchronize(s))) return err;
        }
        st->segments_init = (int64_t)s1;
        if (st->frontier_sizes)
            for (size_t i = 0; i < hsz.size() && (int64_t)i < st->frontier_sizes_cap; i++)
                st->frontier_sizes[i] = (int64_t)hsz[i];
        if (st->round_arcs)
            for (size_t i = 0; i < harcs.size() && (int64_t)i < st->frontier_sizes_cap; i++)
                st->round_arcs[i] = (int64_t)harcs[i];
        if (STATS) {
            Ctrl h;
            if ((err = cudaMemcpyAsync(&h, a.ctl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s))) return err;
            if ((err = cudaStreamSynchronize(s))) return err;
            unsigned long long tot = 0;
            for (auto x : hsz) tot += x;
            st->frontier_total = (int64_t)tot;
            st->init_slots_written = (int64_t)h.st_init_slots;
            st->arcs_scanned = (int64_t)h.st_arcs;
            st->guarded_arcs = (int64_t)h.st_guarded;
            st->bins_read = (int64_t)h.st_bins;
            st->pushes = (int64_t)h.st_pushes;
            st->hub_fallbacks = (int64_t)h.st_fallback;
            st->segments = (int64_t)h.st_segs;
            st->pull_rounds = (int64_t)h.st_pull;
        }
    }
    tm.collect(st);
    if (keep) *keep = a;
    return cudaSuccess;
}

cudaError_t hc_run(const long long *rp, const int *ci, long long n, long long arcs, int *core,
                   cudaStream_t s, uint32_t flags, void *ws, pico_stats_t *st, const DevInfo &dev) {
    if (flags & PICO_F_STATS) return hc_run_t<true>(rp, ci, n, arcs, core, s, flags, ws, st, dev);
    return hc_run_t<false>(rp, ci, n, arcs, core, s, flags, ws, st, dev);
}

// ===========================================================================
// Sharded HistoCore: rank r owns the rows of a contiguous vertex
// range [vb, vb+nloc) with their histograms and estimates; a local CSC lists,
// for every global vertex v, the owned neighbours u of v (the transpose of the
// local row block -- the graph is symmetric).  One round t:
//   pack:  changed (v, oldcore, core) triples of the local C_t   (this file)
//   exchange: allgatherv of the triples over all ranks            (caller:
//             torch.distributed / NCCL, paper_2402_15253_b200/sharded.py)
//   apply: UpdateHisto of every received triple over CSC_r[v] -> local F_{t+1},
//          then SumHisto(F_{t+1}) -> local C_{t+1}                (this file)
// All state of an owned u lives on its owner, so the rounds are exactly the
// synchronous rounds of the single-GPU path: same C_t, same l2 for every P.
// ===========================================================================
struct Shard {
    HcArgs a;
    HcLayout L;              // the rank's HcArgs arrays (rows: nloc; pull v-side: ng)
    void *ws;
    long long nloc, vb, ng, arcs;
    uint32_t flags;
    cudaStream_t s;
    DevInfo dev;
    bool pull_ok;            // dense rounds may pull (graph size, flags)
    shadow_t *deg8g;         // [ng]   saturated global degrees (init)
    unsigned short *deg16g;  // [ng]
    unsigned long long *grec;  // [ng] global estimate records new32 | old32 << 32 (pull rounds)
    long long *csc_off;      // [ng+1]
    int *csc_idx;            // [arcs] owned neighbour (local id), grouped by v
    int *tmpk;               // [arcs] sort keys out (CSC build)
    int2 *TS;                // (triple, segment) work items
    long long tscap;
    unsigned long long *cnt; // [8] device counters: 0 pack, 1 nTS, 2 local arcs of C_t, 3 pull gate
    void *cubtmp;            // scan / sort temp
    size_t cubbytes;
    int t;
};

// global degree shadows; every global record starts at (deg, deg) -- the
// round-0 estimate, unchanged until a triple says otherwise
__global__ void sh_deg8_kernel(const int *deg, long long ng, shadow_t *d8, unsigned short *d16,
                               unsigned long long *grec) {
    long long nt = (long long)gridDim.x * blockDim.x;
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < ng; v += nt) {
        int d = deg[v];
        d8[v] = (shadow_t)min(d, (int)SAT8);
        d16[v] = (unsigned short)min(d, 65535);
        if (grec) grec[v] = pack_rec64(d, d);
    }
}

// records of the received triples: (new, old) for the round's pull, then
// (new, new) once the round is applied
// total_dev (device exchange, lsa_exchange.cu): the triple count from device memory
template <bool RESET>
__global__ void sh_records_kernel(const int *tr, long long total, unsigned long long *grec,
                                  const unsigned long long *total_dev = nullptr) {
    if (total_dev) total = (long long)*total_dev;
    long long nt = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += nt)
        grec[tr[3 * i]] = pack_rec64(tr[3 * i + 2], RESET ? tr[3 * i + 2] : tr[3 * i + 1]);
}

// pull iff allowed and the received triples touch >= arcs_local / pull_div local arcs
__global__ void sh_gate_kernel(unsigned long long *cnt, long long arcs, int pull_ok, int pull_div) {
    if (threadIdx.x == 0)
        cnt[3] = (pull_ok && cnt[2] * (unsigned long long)pull_div >= (unsigned long long)arcs) ? 1ull : 0ull;
}

// CSC counts per global vertex (into csc_off[v+1]) and scatter
__global__ void sh_csc_count_kernel(const int *ci, long long arcs, unsigned long long *cnt_v) {
    long long nt = (long long)gridDim.x * blockDim.x;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < arcs; e += nt)
        atomicAdd(cnt_v + ci[e], 1ull);
}


// C_t of this rank = segment-0 entries of S (init and SumHisto append one
// (v, 0) per changed v) -> triples (v + vb, oldcore, core)
__global__ void sh_pack_kernel(HcArgs a, const unsigned long long *ns_dev, long long vb, int *out,
                               unsigned long long *count) {
    const long long ns = (long long)bcast_u64(ns_dev);
    long long nt = (long long)gridDim.x * blockDim.x;
    long long iters = (ns + nt - 1) / nt;
    for (long long it = 0; it < iters; it++) {
        long long i = it * nt + (long long)blockIdx.x * blockDim.x + threadIdx.x;
        bool take = false;
        int v = 0;
        if (i < ns) {
            int2 sg = a.S[i];
            take = sg.y == 0;
            v = sg.x;
        }
        unsigned m = __ballot_sync(FULL, take);
        if (!m) continue;
        unsigned long long base = 0;
        int leader = __ffs(m) - 1;
        if (lane_id() == leader) base = atomicAdd(count, (unsigned long long)__popc(m));
        base = __shfl_sync(FULL, base, leader);
        if (take) {
            unsigned long long o = 3 * (base + __popc(m & ((1u << lane_id()) - 1)));
            out[o] = (int)(v + vb);
            out[o + 1] = a.oldc[v];
            out[o + 2] = a.core[v];
        }
    }
}

// (triple, segment) items for the CSC lists of the received triples; the
// local arcs they touch are summed into *arcs_ct (the pull decision)
__global__ void sh_segments_kernel(const int *tr, long long total, const long long *csc_off, int seg, int2 *TS,
                                   unsigned long long *nTS, unsigned long long *arcs_ct,
                                   const unsigned long long *total_dev = nullptr) {
    if (total_dev) total = (long long)*total_dev;
    long long nt = (long long)gridDim.x * blockDim.x;
    long long iters = (total + nt - 1) / nt;
    long long ac = 0;
    for (long long it = 0; it < iters; it++) {
        long long i = it * nt + (long long)blockIdx.x * blockDim.x + threadIdx.x;
        int ns = 0;
        if (i < total) {
            int v = tr[3 * i];
            long long len = csc_off[v + 1] - csc_off[v];
            ac += len;
            ns = nseg_of(len, seg);
        }
        warp_append_segments((int)i, ns, TS, nTS);
    }
    stat_add(arcs_ct, ac);
}

// UpdateHisto of the received triples over the local CSC (push direction)
__global__ void __launch_bounds__(512, 2) sh_update_kernel(HcArgs a, const int *tr, const int2 *TS,
                                                           const unsigned long long *nts_dev,
                                                           const long long *csc_off, const int *csc_idx,
                                                           unsigned long long *nF, const unsigned long long *gate) {
    constexpr int U = 4;
    const int lane = lane_id();
    if (bcast_u64(gate)) return;  // this round pulls
    const long long nts = (long long)bcast_u64(nts_dev);  // no host round trip
    const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const unsigned long long hot = pol_last();
    for (long long base = gwarp * 32; base < nts; base += nwarps * 32) {
        long long i = base + lane;
        long long b = 0;
        int len = 0, cv = 0, ov = 0;
        if (i < nts) {
            int2 sg = TS[i];
            int v = tr[3 * sg.x];
            ov = tr[3 * sg.x + 1];
            cv = tr[3 * sg.x + 2];
            long long r0 = csc_off[v], r1 = csc_off[v + 1];
            b = r0 + (long long)sg.y * a.tn.seg;
            len = (int)min((long long)a.tn.seg, r1 - b);
        }
        int incl = warp_incl_scan(len);
        int excl = incl - len;
        int total = __shfl_sync(FULL, incl, 31);
        for (int j0 = 0; j0 < total; j0 += 32 * U) {
            int u[U], cvo[U], ovo[U], cu[U];
            bool ok[U], push[U];
#pragma unroll
            for (int q = 0; q < U; q++) {
                int j = j0 + q * 32 + lane;
                int lo = 0;
#pragma unroll
                for (int step = 16; step >= 1; step >>= 1) {
                    int cand = lo + step;
                    int ex = __shfl_sync(FULL, excl, cand & 31);
                    if (cand < 32 && ex <= j) lo = cand;
                }
                long long eb = __shfl_sync(FULL, b, lo);
                int ex = __shfl_sync(FULL, excl, lo);
                cvo[q] = __shfl_sync(FULL, cv, lo);
                ovo[q] = __shfl_sync(FULL, ov, lo);
                ok[q] = j < total;
                u[q] = ok[q] ? csc_idx[eb + (j - ex)] : 0;
            }
#pragma unroll
            for (int q = 0; q < U; q++) {
                cu[q] = ok[q] ? core_of(a, u[q], hot) : 0;
                ok[q] = ok[q] && cu[q] > cvo[q];  // N1/N3 neighbour
                push[q] = false;
            }
#pragma unroll
            for (int q = 0; q < U; q++)
                if (ok[q]) push[q] = bin_move(a.histo, __ldg(a.rp + u[q]) - 1, cu[q], cvo[q], ovo[q]);
            append_pushes<U>(push, u, a.F, nF);
        }
    }
}

// the other kernels of a shard round, gated by the pull decision (uniform)
__global__ void __launch_bounds__(512, 2) sh_pull_kernel(HcArgs a, int t, const unsigned long long *grec,
                                                         const unsigned long long *gate) {
    if (!bcast_u64(gate)) return;
    coo_pull_phase<false, VRec64>(a, t, grec);
}

__global__ void __launch_bounds__(512, 2) sh_collect_kernel(HcArgs a, int t, const unsigned long long *gate) {
    if (!bcast_u64(gate)) return;
    collect_sum_phase<false>(a, t);
}

__global__ void __launch_bounds__(512) sh_sum_kernel(HcArgs a, int t, const unsigned long long *gate) {
    if (bcast_u64(gate)) return;
    const long long gthread = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    sum_phase<false>(a, t, gthread, nthreads);
}

static size_t sort_bytes(long long arcs) {
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs((void *)nullptr, b, (const int *)nullptr, (int *)nullptr, (const int *)nullptr,
                                    (int *)nullptr, (long long)std::max(arcs, 1ll));  // 64-bit item count
    return b;
}

size_t shard_workspace_bytes(long long nloc, long long ng, long long arcs, uint32_t flags, long long *tscap,
                             size_t *cubbytes) {
    Tune tn = hc_tune(flags);
    size_t b = align256(hc_layout(nloc, arcs, flags, ng, 8).total);
    b += align256(sizeof(shadow_t) * (size_t)ng);
    b += align256(sizeof(unsigned short) * (size_t)ng);
    b += align256(sizeof(unsigned long long) * (size_t)ng);       // grec
    b += align256(sizeof(long long) * (size_t)(ng + 1)) * 2;      // csc_off (+ counts)
    b += align256(sizeof(int) * (size_t)std::max(arcs, 1ll)) * 2; // csc_idx, tmpk
    *tscap = ng + arcs / tn.seg + 64;
    b += align256(sizeof(int2) * (size_t)*tscap);
    b += align256(sizeof(unsigned long long) * 8);
    b += align256(sizeof(int) * (size_t)std::max(nloc, 1ll));  // local core
    size_t cb = 0;
    cub::DeviceScan::ExclusiveSum((void *)nullptr, cb, (const long long *)nullptr, (long long *)nullptr, (int)(ng + 1));
    cb = std::max(cb, sort_bytes(arcs));
    *cubbytes = cb;
    b += align256(cb);
    return b;
}

cudaError_t shard_create(const long long *rp, const int *ci, long long nloc, long long vb, long long ng,
                         uint32_t flags, cudaStream_t s, const DevInfo &dev, Shard **out) {
    Shard *h = new Shard();
    h->nloc = nloc; h->vb = vb; h->ng = ng; h->flags = flags; h->s = s; h->dev = dev; h->t = 1;
    cudaError_t e = cudaMemcpyAsync(&h->arcs, rp + nloc, sizeof(long long), cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) { delete h; return e; }
    size_t bytes = shard_workspace_bytes(nloc, ng, h->arcs, flags, &h->tscap, &h->cubbytes);
    if ((e = lib_malloc_async(&h->ws, bytes, s))) { delete h; return e; }
    HcLayout L = hc_layout(nloc, h->arcs, flags, ng, 8);
    h->L = L;
    h->pull_ok = hc_allow_pull(ng, flags) && h->arcs > 0;
    char *p = (char *)h->ws;
    HcArgs &a = h->a;
    a.ctl = (Ctrl *)(p + L.ctl);
    a.fsz = (unsigned long long *)(p + L.fsz);
    a.rarcs = (unsigned long long *)(p + L.rarcs);
    a.rtime = (unsigned long long *)(p + L.rtime);
    a.fsz_cap = kFszCap;
    a.histo = (int *)(p + L.histo);
    a.c8 = (shadow_t *)(p + L.c8);
    a.c16 = (unsigned short *)(p + L.c16);
    a.rec = (unsigned *)(p + L.rec);
    a.e16 = (unsigned short *)(p + L.e16);
    a.oldc = (int *)(p + L.oldc);
    a.F = (int *)(p + L.F);
    a.BC = (int *)(p + L.BC);
    a.S = (int2 *)(p + L.S);
    a.H = (int2 *)(p + L.H);
    a.chg = (unsigned *)(p + L.chg);
    a.ro = (int *)(p + L.ro);
    a.db = (unsigned char *)(p + L.db);
    a.slen = (int *)(p + L.slen);
    a.capd = (unsigned *)(p + L.capd);
    a.nwords = L.nwords;
    a.rp = rp; a.ci = ci; a.n = (int)nloc; a.arcs = h->arcs; a.tn = hc_tune(flags);
    a.allow_pull = 0;  // (the single-GPU round kernel's switch; shards gate per round)
    // pull rounds: the local arcs (u local, v global) bucketed by global v-range
    a.boff = (unsigned long long *)(p + L.bk);
    a.psrc = (int *)(p + L.psrc);
    a.pdst = (int *)(p + L.pdst);
    a.npass = L.npass;
    a.pshift = hc_pshift(ng, flags, 8);
    if (L.npass == 1) a.pdst = const_cast<int *>(ci);
    a.prefilter = 0;  // the shard's push UpdateHisto walks the CSC, not the rows
    a.h0 = nullptr;
    a.rp32 = nullptr;  // (the shard's kernels read the 64-bit local rowptr)
    p += align256(L.total);
    h->deg8g = (shadow_t *)p; p += align256(sizeof(shadow_t) * (size_t)ng);
    h->deg16g = (unsigned short *)p; p += align256(sizeof(unsigned short) * (size_t)ng);
    h->grec = (unsigned long long *)p; p += align256(sizeof(unsigned long long) * (size_t)ng);
    h->csc_off = (long long *)p; p += align256(sizeof(long long) * (size_t)(ng + 1)) * 2;
    h->csc_idx = (int *)p; p += align256(sizeof(int) * (size_t)std::max(h->arcs, 1ll));
    h->tmpk = (int *)p; p += align256(sizeof(int) * (size_t)std::max(h->arcs, 1ll));
    h->TS = (int2 *)p; p += align256(sizeof(int2) * (size_t)h->tscap);
    h->cnt = (unsigned long long *)p; p += align256(sizeof(unsigned long long) * 8);
    a.core = (int *)p; p += align256(sizeof(int) * (size_t)std::max(nloc, 1ll));
    h->cubtmp = p;
    Ctrl hc{};
    hc.mincv[0] = hc.mincv[1] = INT_MAX;
    if (!e) e = cudaMemcpyAsync(a.ctl, &hc, sizeof(Ctrl), cudaMemcpyHostToDevice, s);
    if (!e) e = cudaMemsetAsync(a.chg, 0, sizeof(unsigned) * 2 * (size_t)L.nwords, s);
    if (!e) e = cudaMemsetAsync(a.capd, 0, sizeof(unsigned) * (size_t)L.nwords, s);
    if (!e) e = cudaMemsetAsync(h->cnt, 0, sizeof(unsigned long long) * 8, s);
    // H0 on the owned rows: core = oldcore = deg, shadow, degree classes
    int blocks = (int)std::min<long long>((nloc + 255) / 256, (long long)dev.sms * 16);
    if (!e && nloc > 0) {
        hc_degree_kernel<<<std::max(blocks, 1), 256, 0, s>>>(a);
        e = cudaGetLastError();
    }
    if (e) {
        cudaFreeAsync(h->ws, s);
        delete h;
        return e;
    }
    *out = h;
    return cudaSuccess;
}

cudaError_t shard_degrees(Shard *h, int *deg_out) {
    if (h->nloc == 0) return cudaSuccess;
    return cudaMemcpyAsync(deg_out, h->a.core, sizeof(int) * (size_t)h->nloc, cudaMemcpyDeviceToDevice, h->s);
}

// InitHisto + round-1 SumHisto of the owned rows (neighbour degrees from the
// all-gathered deg_global), the local CSC (the transpose of the owned rows:
// for every global v its owned neighbours, by a key-value radix sort of the
// arcs) and, if dense rounds may pull, the bucketed local edge list
cudaError_t shard_init(Shard *h, const int *deg_global, long long *changed) {
    cudaStream_t s = h->s;
    HcArgs &a = h->a;
    const HcLayout &L = h->L;
    const int sms = h->dev.sms;
    auto grid = [&](long long work) {
        return std::max(1, (int)std::min<long long>((work + 255) / 256, (long long)sms * 16));
    };
    cudaError_t e;
    sh_deg8_kernel<<<grid(h->ng), 256, 0, s>>>(deg_global, h->ng, h->deg8g, h->deg16g, h->pull_ok ? h->grec : nullptr);
    a.nv8 = h->deg8g;
    a.nv16 = h->deg16g;
    a.nv32 = deg_global;
    if (h->arcs > 0) {
        // row owner of every local arc (into psrc for one bucket, else the
        // not-yet-written histogram space)
        int *src = (h->pull_ok && L.npass == 1) ? a.psrc : a.histo;
        hc_el_src_short_kernel<<<grid(h->nloc), 256, 0, s>>>(a, src);
        hc_el_src_long_kernel<<<sms * 8, 256, 0, s>>>(a, src);
        if (h->pull_ok && L.npass > 1) {
            unsigned long long *cnt = (unsigned long long *)((char *)h->ws + L.elc);
            hc_el_count_kernel<<<sms * 16, 256, 0, s>>>(a, cnt, L.nbcap);
            size_t tb = L.eltb;
            if ((e = cub::DeviceScan::ExclusiveSum((char *)h->ws + L.elt, tb, cnt, cnt, (int)(L.npass * L.nbcap), s)))
                return e;
            hc_el_fill_kernel<<<sms * 16, 256, 0, s>>>(a, src, cnt, L.nbcap);
            hc_el_offsets_kernel<<<1, 32, 0, s>>>(a, L.nbcap, cnt);
        } else if (h->pull_ok) {
            unsigned long long off[kMaxPass + 1];
            for (int q = 0; q <= kMaxPass; q++) off[q] = q == 0 ? 0 : (unsigned long long)h->arcs;
            if ((e = cudaMemcpyAsync(a.boff, off, sizeof(off), cudaMemcpyHostToDevice, s))) return e;
        }
        // CSC: counts -> offsets; (v, u) pairs sorted by v -> owned neighbours
        long long *cntv = h->csc_off + (h->ng + 1);
        if ((e = cudaMemsetAsync(cntv, 0, sizeof(long long) * (size_t)(h->ng + 1), s))) return e;
        sh_csc_count_kernel<<<grid(h->arcs), 256, 0, s>>>(a.ci, h->arcs, (unsigned long long *)cntv);
        size_t cb = h->cubbytes;
        if ((e = cub::DeviceScan::ExclusiveSum(h->cubtmp, cb, cntv, h->csc_off, (int)(h->ng + 1), s))) return e;
        int bits = 1;
        while ((1ll << bits) < h->ng) bits++;
        cb = h->cubbytes;
        if ((e = cub::DeviceRadixSort::SortPairs(h->cubtmp, cb, a.ci, h->tmpk, src, h->csc_idx, (long long)h->arcs, 0,
                                                 bits, s)))
            return e;
    } else {
        if ((e = cudaMemsetAsync(h->csc_off, 0, sizeof(long long) * (size_t)(h->ng + 1), s))) return e;
    }
    // InitHisto fused with round-1 SumHisto (the single-GPU init kernels)
    if (h->nloc) {
        Tune tn = a.tn;
        hc_init_small_kernel<false><<<grid(h->nloc), 256, 0, s>>>(a);
        size_t smB = sizeof(int) * (size_t)(tn.b_max + 1) * 8;
        int occB = 0, occC = 0;
        if (hc_init_split(h->ng)) {  // the gathered shadows are global-size on a shard
            size_t smB1 = sizeof(int) * (size_t)init_warp_stride<1>(tn.b_max) * 8;
            int occB1 = 0;
            cudaFuncSetAttribute(hc_init_warp_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB1);
            cudaFuncSetAttribute(hc_init_warp_kernel<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occB1, hc_init_warp_kernel<false, 1>, 256, smB1);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occB, hc_init_warp_kernel<false, 2>, 256, smB);
            hc_init_warp_kernel<false, 1><<<sms * std::max(1, occB1), 256, smB1, s>>>(a);
            hc_init_warp_kernel<false, 2><<<sms * std::max(1, occB), 256, smB, s>>>(a);
        } else {
            cudaFuncSetAttribute(hc_init_warp_kernel<false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occB, hc_init_warp_kernel<false, 0>, 256, smB);
            hc_init_warp_kernel<false, 0><<<sms * std::max(1, occB), 256, smB, s>>>(a);
        }
        size_t smC = sizeof(int) * (size_t)(tn.c_bins + 1);
        cudaFuncSetAttribute(hc_init_cta_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smC);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occC, hc_init_cta_kernel<false>, 512, smC);
        hc_init_cta_kernel<false><<<sms * std::max(1, occC), 512, smC, s>>>(a);
        hc_init_fallback_kernel<false><<<sms, 1024, 0, s>>>(a, 0);
        hc_shadow_kernel<<<grid(h->nloc), 256, 0, s>>>(a);
    }
    a.nv8 = a.c8;
    a.nv16 = a.c16;
    a.nv32 = a.oldc;
    unsigned long long c1 = 0;
    if ((e = cudaMemcpyAsync(&c1, &a.ctl->nF[1], sizeof(c1), cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    if ((e = cudaGetLastError())) return e;
    *changed = (long long)c1;
    h->t = 1;
    return cudaSuccess;
}

cudaError_t shard_pack(Shard *h, int *triples, long long cap, long long *count) {
    cudaStream_t s = h->s;
    cudaError_t e;
    if ((e = cudaMemsetAsync(h->cnt, 0, sizeof(unsigned long long), s))) return e;
    sh_pack_kernel<<<h->dev.sms * 4, 256, 0, s>>>(h->a, &h->a.ctl->nS[h->t & 1], h->vb, triples, h->cnt);
    unsigned long long c = 0;
    if ((e = cudaMemcpyAsync(&c, h->cnt, sizeof(c), cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    if ((long long)c > cap) return cudaErrorInvalidValue;
    *count = (long long)c;
    return cudaGetLastError();
}

// stream-ordered pack: the count stays on the device (*count_dev; read by a
// collective, not by the host)
cudaError_t shard_pack_dev(Shard *h, int *triples, const unsigned long long **count_dev) {
    cudaStream_t s = h->s;
    cudaError_t e;
    if ((e = cudaMemsetAsync(h->cnt, 0, sizeof(unsigned long long), s))) return e;
    sh_pack_kernel<<<h->dev.sms * 4, 256, 0, s>>>(h->a, &h->a.ctl->nS[h->t & 1], h->vb, triples, h->cnt);
    *count_dev = h->cnt;
    return cudaGetLastError();
}

// UpdateHisto(C_t of all ranks) -- push over the local CSC, or, for dense
// rounds, pull over the bucketed local edge list against the global records
// -- then SumHisto of the local frontier.  The direction is decided on the
// device (sh_gate_kernel): no host round trip.
cudaError_t shard_apply(Shard *h, const int *triples, long long total, long long *changed,
                        const unsigned long long *total_dev) {
    cudaStream_t s = h->s;
    HcArgs &a = h->a;
    const int sms = h->dev.sms;
    const int t = h->t;
    cudaError_t e;
    unsigned long long *nTS = h->cnt + 1, *gate = h->cnt + 3;
    if ((e = cudaMemsetAsync(h->cnt + 1, 0, sizeof(unsigned long long) * 3, s))) return e;  // nTS, arcs, gate
    if ((e = cudaMemsetAsync(&a.ctl->nF[(t + 1) & 1], 0, sizeof(unsigned long long), s))) return e;
    if ((e = cudaMemsetAsync(&a.ctl->nS[(t + 1) & 1], 0, sizeof(unsigned long long), s))) return e;
    if ((e = cudaMemsetAsync(a.chg + ((t + 1) & 1) * a.nwords, 0, sizeof(unsigned) * (size_t)a.nwords, s))) return e;
    // stream-ordered, no host round trip: work counts are read on the device
    // (the segment capacity n_global + 2m_local/seg bounds any round: the
    // triples are distinct vertices)
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sh_pull_kernel, 512, 0);
    const int pblocks = sms * std::max(1, occ);
    // device total (no host round trip): grids sized for any count, the
    // kernels read it; an empty round is a no-op
    if (total_dev) total = h->ng;
    if (total > 0) {
        int blocks = (int)std::min<long long>((total + 255) / 256, (long long)sms * 16);
        if (h->pull_ok) sh_records_kernel<false><<<std::max(blocks, 1), 256, 0, s>>>(triples, total, h->grec, total_dev);
        sh_segments_kernel<<<std::max(blocks, 1), 256, 0, s>>>(triples, total, h->csc_off, a.tn.seg, h->TS, nTS,
                                                               h->cnt + 2, total_dev);
        sh_gate_kernel<<<1, 32, 0, s>>>(h->cnt, h->arcs, h->pull_ok ? 1 : 0, a.tn.pull_div);
        sh_update_kernel<<<sms * 2, 512, 0, s>>>(a, triples, h->TS, nTS, h->csc_off, h->csc_idx,
                                                 &a.ctl->nF[(t + 1) & 1], gate);
        if (h->pull_ok) sh_pull_kernel<<<pblocks, 512, 0, s>>>(a, t, h->grec, gate);
    }
    sh_sum_kernel<<<sms * 4, 512, 0, s>>>(a, t + 1, gate);
    if (h->pull_ok && total > 0) {
        sh_collect_kernel<<<pblocks, 512, 0, s>>>(a, t + 1, gate);
        int blocks = (int)std::min<long long>((total + 255) / 256, (long long)sms * 16);
        sh_records_kernel<true><<<std::max(blocks, 1), 256, 0, s>>>(triples, total, h->grec, total_dev);
    }
    if ((e = cudaGetLastError())) return e;
    h->t = t + 1;
    if (changed) {
        unsigned long long nf = 0;
        if ((e = cudaMemcpyAsync(&nf, &a.ctl->nF[(t + 1) & 1], sizeof(nf), cudaMemcpyDeviceToHost, s))) return e;
        if ((e = cudaStreamSynchronize(s))) return e;
        *changed = (long long)nf;
    }
    return cudaSuccess;
}

cudaError_t shard_result(Shard *h, int *core_out) {
    if (h->nloc == 0) return cudaSuccess;
    cudaError_t e = cudaMemcpyAsync(core_out, h->a.core, sizeof(int) * (size_t)h->nloc, cudaMemcpyDeviceToDevice, h->s);
    if (!e) e = cudaStreamSynchronize(h->s);
    return e;
}

cudaError_t shard_destroy(Shard *h) {
    cudaError_t e = cudaFreeAsync(h->ws, h->s);
    if (!e) e = cudaStreamSynchronize(h->s);
    delete h;
    return e;
}

// ===========================================================================
// Decremental HistoCore (the
// Index2core paradigm suits dynamic graphs).  After a run, the state kept in
// the workspace -- estimates equal to the coreness, every histogram exact
// (bins below the coreness count neighbours of that coreness, the cap bin
// the neighbours at or above it) -- is reused for batches of edge deletions:
//   1. each deleted arc (x, y) becomes a tombstone: a self-loop (x, x) in the
//      owned CSR copy and in the pull edge list; a self-loop never passes the
//      UpdateHisto guard core[u] > core[v], so no kernel needs a new test;
//   2. y's contribution leaves x's histogram (the cap bin if core[y] >=
//      core[x], marking x as a frontier candidate, else bin core[y]);
//   3. the usual rounds run from the marked vertices.
// A deletion can only lower coreness, so the old coreness is an upper bound
// of the new one and the Index2core iteration from it converges to the new
// coreness (the largest fixed point below the start; readings in DESIGN.md).
// ===========================================================================
// Decremental batch, step 1: canonical keys (min << 32 | max) of the k
// undirected edges; a self loop or an id out of range flags err bit 1
__global__ void dyn_keys_kernel(const int *src, const int *dst, long long k, int n, unsigned long long *keys,
                                int *err) {
    long long nt = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += nt) {
        const int x = src[i], y = dst[i];
        if (x < 0 || x >= n || y < 0 || y >= n || x == y) {
            atomicOr(err, 1);
            keys[i] = ~0ull;
            continue;
        }
        const unsigned lo = (unsigned)min(x, y), hi = (unsigned)max(x, y);
        keys[i] = ((unsigned long long)lo << 32) | hi;
    }
}

// position of the arc (x, y) in x's row of the handle's CSR copy (-1: not
// an edge of the current graph).  Warp-collective.
__device__ __forceinline__ long long dyn_find_arc(const HcArgs &a, const int *ci_own, int x, int y) {
    const long long r0 = a.rp[x], r1 = a.rp[x + 1];
    for (long long e0 = r0; e0 < r1; e0 += 32) {
        long long e = e0 + lane_id();
        unsigned m = __ballot_sync(FULL, e < r1 && ci_own[e] == y);
        if (m) return e0 + __ffs(m) - 1;
    }
    return -1;
}

// step 2 (sorted keys; a key equal to its predecessor is a duplicate of the
// same undirected edge and is skipped, so each arc is claimed by exactly one
// warp): APPLY = false checks that both arcs of every edge exist (err bit 2,
// nothing written); APPLY = true tombstones the arc in the CSR copy and in
// the pull edge list and takes the neighbour out of the histogram.
template <bool APPLY>
__global__ void dyn_delete_kernel(HcArgs a, int *ci_own, const unsigned long long *keys, long long k, int *err) {
    const int lane = lane_id();
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = gw; i < k; i += nw) {
        const unsigned long long key = keys[i];
        if (key == ~0ull || (i > 0 && keys[i - 1] == key)) continue;
        const int eu = (int)(key >> 32), ev = (int)(key & 0xffffffffu);
        for (int dir = 0; dir < 2; dir++) {
            const int x = dir ? ev : eu, y = dir ? eu : ev;
            const long long pos = dyn_find_arc(a, ci_own, x, y);
            if (pos < 0) {
                if (lane == 0) atomicOr(err, 2);  // not an edge of the current graph
                continue;
            }
            if (!APPLY) continue;
            if (lane == 0) ci_own[pos] = x;  // tombstone (one bucket: pdst is ci_own)
            if (a.npass > 1) {
                // the arc in bucket y >> pshift of the edge list (CSR order: a
                // binary search for x's run, then a warp scan of the run)
                const int p = y >> a.pshift;
                long long lo = (long long)a.boff[p], hi = (long long)a.boff[p + 1];
                while (lo < hi) {
                    long long mid = (lo + hi) >> 1;
                    if (a.psrc[mid] < x) lo = mid + 1; else hi = mid;
                }
                const long long be = (long long)a.boff[p + 1];
                for (long long e0 = lo; e0 < be; e0 += 32) {
                    long long e = e0 + lane;
                    bool in = e < be && a.psrc[e] == x;
                    unsigned m = __ballot_sync(FULL, in && a.pdst[e] == y);
                    if (m) {
                        if (lane == __ffs(m) - 1) a.pdst[e] = x;
                        break;
                    }
                    if (__ballot_sync(FULL, in) != FULL) break;  // past x's run
                }
            }
            // y leaves x's histogram
            if (lane == 0) {
                const int cx = a.core[x], cy = a.core[y];
                const long long hb = a.rp[x] - 1;
                if (cy >= cx) {
                    atomicSub(a.histo + hb + cx, 1);  // cnt(x) drops: a frontier candidate
                    atomicOr(a.capd + (x >> 5), 1u << (x & 31));
                } else {
                    atomicSub(a.histo + hb + cy, 1);
                }
            }
        }
    }
}

struct Dyn {
    HcArgs a;
    void *ws;
    long long *rp;
    int *ci;
    int *core;
    long long n, arcs;
    uint32_t flags;
    cudaStream_t s;
    DevInfo dev;
    int *err;
};

size_t dyn_workspace_bytes(long long n, long long arcs, uint32_t flags) {
    return align256(hc_workspace_bytes(n, arcs, flags)) + align256(sizeof(long long) * (size_t)(n + 1)) +
           align256(sizeof(int) * (size_t)std::max(arcs, 1ll)) + align256(sizeof(int) * (size_t)std::max(n, 1ll)) +
           256;
}

cudaError_t dyn_create(const long long *rp, const int *ci, long long n, long long arcs, uint32_t flags,
                       cudaStream_t s, const DevInfo &dev, pico_stats_t *st, Dyn **out) {
    Dyn *h = new Dyn();
    h->n = n; h->arcs = arcs; h->flags = flags & ~(uint32_t)(PICO_F_STATS | PICO_F_HOST_LOOP); h->s = s; h->dev = dev;
    cudaError_t e = lib_malloc_async(&h->ws, dyn_workspace_bytes(n, arcs, h->flags), s);
    if (e) { delete h; return e; }
    char *p = (char *)h->ws + align256(hc_workspace_bytes(n, arcs, h->flags));
    h->rp = (long long *)p; p += align256(sizeof(long long) * (size_t)(n + 1));
    h->ci = (int *)p; p += align256(sizeof(int) * (size_t)std::max(arcs, 1ll));
    h->core = (int *)p; p += align256(sizeof(int) * (size_t)std::max(n, 1ll));
    h->err = (int *)p;
    if (!e) e = cudaMemcpyAsync(h->rp, rp, sizeof(long long) * (size_t)(n + 1), cudaMemcpyDeviceToDevice, s);
    if (!e && arcs) e = cudaMemcpyAsync(h->ci, ci, sizeof(int) * (size_t)arcs, cudaMemcpyDeviceToDevice, s);
    if (!e) e = hc_run_t<false>(h->rp, h->ci, n, arcs, h->core, s, h->flags, h->ws, st, dev, &h->a);
    if (e) {
        cudaFreeAsync(h->ws, s);
        cudaStreamSynchronize(s);
        delete h;
        return e;
    }
    *out = h;
    return cudaSuccess;
}

cudaError_t dyn_core(Dyn *h, int *core_out) {
    cudaError_t e = cudaMemcpyAsync(core_out, h->core, sizeof(int) * (size_t)h->n, cudaMemcpyDeviceToDevice, h->s);
    if (!e) e = cudaStreamSynchronize(h->s);
    return e;
}

// returns cudaErrorInvalidValue for an edge that is not in the current graph
cudaError_t dyn_delete(Dyn *h, const int *src, const int *dst, long long k, pico_stats_t *st) {
    cudaStream_t s = h->s;
    HcArgs &a = h->a;
    const int sms = h->dev.sms;
    cudaError_t e;
    Ctrl hc{};
    hc.mincv[0] = hc.mincv[1] = INT_MAX;
    if ((e = cudaMemcpyAsync(a.ctl, &hc, sizeof(Ctrl), cudaMemcpyHostToDevice, s))) return e;
    if ((e = cudaMemsetAsync(a.chg, 0, sizeof(unsigned) * 2 * (size_t)a.nwords, s))) return e;
    if ((e = cudaMemsetAsync(a.capd, 0, sizeof(unsigned) * (size_t)a.nwords, s))) return e;
    int herr = 0;
    if ((e = cudaMemsetAsync(h->err, 0, sizeof(int), s))) return e;
    if (k > 0) {
        // canonical keys, sorted (duplicates and reversed copies adjacent),
        // checked, then applied: a rejected batch leaves the state untouched
        size_t tb = 0;
        cub::DeviceRadixSort::SortKeys((void *)nullptr, tb, (const unsigned long long *)nullptr,
                                       (unsigned long long *)nullptr, k);
        const size_t kb = align256(sizeof(unsigned long long) * (size_t)k);
        char *buf = nullptr;
        if ((e = lib_malloc_async(&buf, 2 * kb + align256(tb), s))) return e;
        unsigned long long *k0 = (unsigned long long *)buf, *k1 = (unsigned long long *)(buf + kb);
        const int kbl = (int)std::min<long long>((k + 255) / 256, (long long)sms * 8);
        dyn_keys_kernel<<<kbl, 256, 0, s>>>(src, dst, k, (int)h->n, k0, h->err);
        e = cub::DeviceRadixSort::SortKeys(buf + 2 * kb, tb, k0, k1, k, 0, 64, s);
        if (!e) {
            dyn_delete_kernel<false><<<sms * 8, 256, 0, s>>>(a, h->ci, k1, k, h->err);
            e = cudaMemcpyAsync(&herr, h->err, sizeof(int), cudaMemcpyDeviceToHost, s);
        }
        if (!e) e = cudaStreamSynchronize(s);
        if (!e && !herr) dyn_delete_kernel<true><<<sms * 8, 256, 0, s>>>(a, h->ci, k1, k, h->err);
        cudaError_t e2 = cudaFreeAsync(buf, s);
        if (!e) e = e2;
        if (!e) e = cudaGetLastError();
        if (e) return e;
    }
    if (herr) return cudaErrorInvalidValue;
    a.allow_zero = 1;
    // SumHisto of the marked vertices -> C_1, then the rounds
    hc_collect_sum_kernel<false><<<sms * 4, 512, 0, s>>>(a, 1);
    unsigned long long c1 = 0;
    if ((e = cudaMemcpyAsync(&c1, &a.ctl->nF[1], sizeof(c1), cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    std::vector<long long> sizes;
    if (c1) sizes.push_back((long long)c1);
    if ((e = cudaMemsetAsync(&a.ctl->nF[1], 0, sizeof(unsigned long long), s))) return e;
    long long launches = 2;
    if (c1) {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hc_rounds_kernel<false>, 512, 0);
        void *args[] = {&a};
        if ((e = cudaLaunchCooperativeKernel((const void *)hc_rounds_kernel<false>, sms * std::max(1, occ), 512,
                                             args, 0, s)))
            return e;
        launches++;
        unsigned long long devrounds = 0;
        int derr = 0;
        if ((e = cudaMemcpyAsync(&devrounds, &a.ctl->rounds, sizeof(devrounds), cudaMemcpyDeviceToHost, s))) return e;
        if ((e = cudaMemcpyAsync(&derr, &a.ctl->error, sizeof(derr), cudaMemcpyDeviceToHost, s))) return e;
        if ((e = cudaStreamSynchronize(s))) return e;
        if (derr) return cudaErrorAssert;
        size_t nr = (size_t)std::min<unsigned long long>(devrounds + 2, kFszCap);
        std::vector<unsigned long long> dsz(nr, 0);
        if ((e = cudaMemcpyAsync(dsz.data(), a.fsz, sizeof(unsigned long long) * nr, cudaMemcpyDeviceToHost, s)))
            return e;
        if ((e = cudaStreamSynchronize(s))) return e;
        for (unsigned long long t = 1; t <= devrounds && t < kFszCap; t++) sizes.push_back((long long)dsz[t]);
    }
    if ((e = cudaGetLastError())) return e;
    if (st) {
        st->rounds = (int64_t)sizes.size();
        st->kernel_count += launches;
        if (st->frontier_sizes)
            for (size_t i = 0; i < sizes.size() && (int64_t)i < st->frontier_sizes_cap; i++)
                st->frontier_sizes[i] = sizes[i];
    }
    return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Edge insertions (pico_dyn_insert_edges).  An insertion can raise coreness, by
// at most one per inserted edge, and only for vertices whose old coreness lies
// in the band [Kmin, Kmax] (Kmin = min over the batch of min(core x, core y),
// Kmax = max of the same + k - 1) that are connected to an inserted endpoint
// through band vertices (the subcore argument of single-edge insertion,
// applied edge by edge).  So
//   1. R = band-restricted BFS from the in-band endpoints,
//   2. est = min(deg_new, core + k) on R, core elsewhere: an upper bound of
//      the new coreness that equals it outside R,
//   3. the CSR is rebuilt with the new arcs (tombstones of earlier deletions
//      dropped), and HistoCore runs warm-started from est (InitHisto capped at
//      est, P:496-500 with est for the degrees): the synchronous iteration
//      from an upper bound converges to the greatest fixed point below it,
//      the new coreness, and only R and its neighbourhood change.
// ---------------------------------------------------------------------------
__global__ void dyn_ins_check_kernel(HcArgs a, const int *ci_own, const unsigned long long *keys, long long k,
                                     int *err) {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = gw; i < k; i += nw) {
        const unsigned long long key = keys[i];
        if (key == ~0ull || (i > 0 && keys[i - 1] == key)) continue;
        const int x = (int)(key >> 32), y = (int)(key & 0xffffffffu);
        if (dyn_find_arc(a, ci_own, x, y) >= 0 && lane_id() == 0) atomicOr(err, 2);  // already an edge
    }
}

__global__ void dyn_ins_band_kernel(const unsigned long long *keys, long long k, const int *core, int *kb) {
    long long nt = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += nt) {
        const unsigned long long key = keys[i];
        if (key == ~0ull) continue;
        const int c = min(core[(int)(key >> 32)], core[(int)(key & 0xffffffffu)]);
        atomicMin(kb, c);
        atomicMax(kb + 1, c);
    }
}

__device__ __forceinline__ void dyn_ins_visit(int u, unsigned *vis, int *F, unsigned long long *nF) {
    const unsigned bit = 1u << (u & 31);
    if (!(atomicOr(vis + (u >> 5), bit) & bit)) F[atomicAdd(nF, 1ull)] = u;
}

__global__ void dyn_ins_seed_kernel(const unsigned long long *keys, long long k, const int *core, int kmin, int kmax,
                                    unsigned *vis, int *F, unsigned long long *nF) {
    long long nt = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += nt) {
        const unsigned long long key = keys[i];
        if (key == ~0ull) continue;
        for (int e = 0; e < 2; e++) {
            const int x = e ? (int)(key & 0xffffffffu) : (int)(key >> 32);
            if (core[x] >= kmin && core[x] <= kmax) dyn_ins_visit(x, vis, F, nF);
        }
    }
}

// one BFS level: warp per frontier vertex, band neighbours not yet visited
__global__ void dyn_ins_bfs_kernel(const long long *rp, const int *ci, const int *core, int kmin, int kmax,
                                   unsigned *vis, const int *F, long long nf, int *Fn, unsigned long long *nFn) {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = gw; i < nf; i += nw) {
        const int v = F[i];
        for (long long e = rp[v] + lane_id(); e < rp[v + 1]; e += 32) {
            const int u = ci[e];
            if (u != v && core[u] >= kmin && core[u] <= kmax) dyn_ins_visit(u, vis, Fn, nFn);  // u == v: tombstone
        }
    }
}

// live degree (tombstones of deletions are self-loops) + inserted arcs
__global__ void dyn_ins_deg_kernel(const long long *rp, const int *ci, long long n, long long *deg) {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long v = gw; v < n; v += nw) {
        long long c = 0;
        for (long long e = rp[v] + lane_id(); e < rp[v + 1]; e += 32) c += ci[e] != (int)v;
        c = warp_sum64(c);
        if (lane_id() == 0) deg[v] = c;
    }
}

__global__ void dyn_ins_keys_kernel(const long long *rp, const int *ci, long long n, long long arcs,
                                    const unsigned long long *ikeys, long long k, long long *deg,
                                    unsigned long long *keys) {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long v = gw; v < n; v += nw)  // the live arcs, at their old positions
        for (long long e = rp[v] + lane_id(); e < rp[v + 1]; e += 32) {
            const int u = ci[e];
            keys[e] = u != (int)v ? ((unsigned long long)v << 32) | (unsigned)u : ~0ull;
        }
    const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nt = (long long)gridDim.x * blockDim.x;
    for (long long i = gt; i < k; i += nt) {  // both arcs of each new edge, after them
        const unsigned long long key = ikeys[i];
        const bool ok = key != ~0ull && !(i > 0 && ikeys[i - 1] == key);
        const unsigned x = (unsigned)(key >> 32), y = (unsigned)(key & 0xffffffffu);
        keys[arcs + 2 * i] = ok ? ((unsigned long long)x << 32) | y : ~0ull;
        keys[arcs + 2 * i + 1] = ok ? ((unsigned long long)y << 32) | x : ~0ull;
        if (ok) {
            atomicAdd((unsigned long long *)(deg + x), 1ull);
            atomicAdd((unsigned long long *)(deg + y), 1ull);
        }
    }
}

__global__ void dyn_ins_est_kernel(const int *core, const unsigned *vis, const long long *rp_new, long long n,
                                   long long k, int *est) {
    long long nt = (long long)gridDim.x * blockDim.x;
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += nt) {
        const long long d = rp_new[v + 1] - rp_new[v];
        const bool r = (vis[v >> 5] >> (v & 31)) & 1u;
        est[v] = r ? (int)min(d, (long long)core[v] + k) : core[v];
    }
}

__global__ void dyn_ins_cols_kernel(const unsigned long long *keys, long long arcs, int *ci) {
    long long nt = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < arcs; i += nt)
        ci[i] = (int)(keys[i] & 0xffffffffu);
}

// returns cudaErrorInvalidValue for a self loop, an id out of range or an
// edge that is already in the graph (nothing modified)
cudaError_t dyn_insert(Dyn *h, const int *src, const int *dst, long long k, pico_stats_t *st) {
    cudaStream_t s = h->s;
    const int sms = h->dev.sms;
    const long long n = h->n;
    cudaError_t e = cudaSuccess;
    if (k <= 0) return cudaSuccess;
    // --- canonical sorted keys, checked before anything is modified
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys((void *)nullptr, tb, (const unsigned long long *)nullptr,
                                   (unsigned long long *)nullptr, k);
    const size_t kb = align256(sizeof(unsigned long long) * (size_t)k);
    char *buf = nullptr;
    if ((e = lib_malloc_async(&buf, 2 * kb + align256(tb) + 256, s))) return e;
    unsigned long long *k0 = (unsigned long long *)buf, *k1 = (unsigned long long *)(buf + kb);
    int *kbnd = (int *)(buf + 2 * kb + align256(tb));
    int herr = 0;
    const int kbl = (int)std::min<long long>((k + 255) / 256, (long long)sms * 8);
    if (!e) e = cudaMemsetAsync(h->err, 0, sizeof(int), s);
    if (!e) dyn_keys_kernel<<<kbl, 256, 0, s>>>(src, dst, k, (int)n, k0, h->err);
    if (!e) e = cub::DeviceRadixSort::SortKeys(buf + 2 * kb, tb, k0, k1, k, 0, 64, s);
    if (!e) dyn_ins_check_kernel<<<sms * 8, 256, 0, s>>>(h->a, h->ci, k1, k, h->err);
    if (!e) e = cudaMemcpyAsync(&herr, h->err, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e || herr) {
        cudaFreeAsync(buf, s);
        cudaStreamSynchronize(s);
        return e ? e : cudaErrorInvalidValue;
    }
    // --- R: band-restricted BFS from the in-band endpoints
    int hb[2] = {INT_MAX, INT_MIN};
    if (!e) e = cudaMemcpyAsync(kbnd, hb, sizeof(hb), cudaMemcpyHostToDevice, s);
    if (!e) dyn_ins_band_kernel<<<kbl, 256, 0, s>>>(k1, k, h->core, kbnd);
    if (!e) e = cudaMemcpyAsync(hb, kbnd, sizeof(hb), cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    const int kmin = hb[0];
    const int kmax = (int)std::min<long long>((long long)hb[1] + k - 1, INT_MAX);
    const long long nwords = (n + 31) / 32;
    const long long arcs_old = h->arcs;
    char *tmp = nullptr;
    // vis | F0 | F1 | counters | deg (n+1) | est
    const size_t tv = align256(sizeof(unsigned) * (size_t)std::max(nwords, 1ll));
    const size_t tf = align256(sizeof(int) * (size_t)std::max(n, 1ll));
    const size_t td = align256(sizeof(long long) * (size_t)(n + 1));
    if (!e) e = lib_malloc_async(&tmp, tv + 3 * tf + 256 + td, s);
    if (e) { cudaFreeAsync(buf, s); return e; }
    unsigned *vis = (unsigned *)tmp;
    int *F0 = (int *)(tmp + tv), *F1 = (int *)(tmp + tv + tf), *est = (int *)(tmp + tv + 2 * tf);
    unsigned long long *cnt = (unsigned long long *)(tmp + tv + 3 * tf);
    long long *deg = (long long *)(tmp + tv + 3 * tf + 256);
    e = cudaMemsetAsync(vis, 0, tv, s);
    if (!e) e = cudaMemsetAsync(cnt, 0, 256, s);
    if (!e) dyn_ins_seed_kernel<<<kbl, 256, 0, s>>>(k1, k, h->core, kmin, kmax, vis, F0, cnt);
    long long rsize = 0, bfs_levels = 0;
    for (int par = 0; !e; par ^= 1) {
        unsigned long long nf = 0;
        e = cudaMemcpyAsync(&nf, cnt + par, sizeof(nf), cudaMemcpyDeviceToHost, s);
        if (!e) e = cudaStreamSynchronize(s);
        if (e || nf == 0) break;
        rsize += (long long)nf;
        bfs_levels++;
        if (!e) e = cudaMemsetAsync(cnt + (par ^ 1), 0, sizeof(unsigned long long), s);
        const int bl = (int)std::min<long long>(((long long)nf * 32 + 255) / 256, (long long)sms * 16);
        if (!e)
            dyn_ins_bfs_kernel<<<std::max(bl, 1), 256, 0, s>>>(h->rp, h->ci, h->core, kmin, kmax, vis, par ? F1 : F0,
                                                                (long long)nf, par ? F0 : F1, cnt + (par ^ 1));
    }
    // --- the new CSR: live arcs + both arcs of each new edge, sorted by (row, col)
    const long long nkeys = arcs_old + 2 * k;
    size_t tb2 = 0;
    cub::DeviceRadixSort::SortKeys((void *)nullptr, tb2, (const unsigned long long *)nullptr,
                                   (unsigned long long *)nullptr, nkeys);
    size_t tbs = 0;
    cub::DeviceScan::ExclusiveSum((void *)nullptr, tbs, (const long long *)nullptr, (long long *)nullptr, (int)(n + 1));
    char *kbuf = nullptr;
    const size_t kk = align256(sizeof(unsigned long long) * (size_t)nkeys);
    if (!e) e = lib_malloc_async(&kbuf, 2 * kk + align256(std::max(tb2, tbs)), s);
    if (e) { cudaFreeAsync(buf, s); cudaFreeAsync(tmp, s); return e; }
    unsigned long long *a0 = (unsigned long long *)kbuf, *a1 = (unsigned long long *)(kbuf + kk);
    if (!e) e = cudaMemsetAsync(deg + n, 0, sizeof(long long), s);
    if (!e) dyn_ins_deg_kernel<<<sms * 8, 256, 0, s>>>(h->rp, h->ci, n, deg);
    if (!e) dyn_ins_keys_kernel<<<sms * 8, 256, 0, s>>>(h->rp, h->ci, n, arcs_old, k1, k, deg, a0);
    if (!e) e = cub::DeviceRadixSort::SortKeys(kbuf + 2 * kk, tb2, a0, a1, nkeys, 0, 64, s);
    long long *rp_new = (long long *)a0;  // a0 is free after the sort: deg -> rowptr
    if (!e) e = cub::DeviceScan::ExclusiveSum(kbuf + 2 * kk, tbs, deg, rp_new, (int)(n + 1), s);
    long long arcs_new = 0;
    if (!e) e = cudaMemcpyAsync(&arcs_new, rp_new + n, sizeof(long long), cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (!e) dyn_ins_est_kernel<<<sms * 8, 256, 0, s>>>(h->core, vis, rp_new, n, k, est);
    // --- a new handle state around the new CSR, HistoCore warm-started from est
    void *ws_new = nullptr;
    if (!e) e = lib_malloc_async(&ws_new, dyn_workspace_bytes(n, arcs_new, h->flags), s);
    if (!e) {
        char *p = (char *)ws_new + align256(hc_workspace_bytes(n, arcs_new, h->flags));
        long long *rp2 = (long long *)p; p += align256(sizeof(long long) * (size_t)(n + 1));
        int *ci2 = (int *)p; p += align256(sizeof(int) * (size_t)std::max(arcs_new, 1ll));
        int *core2 = (int *)p; p += align256(sizeof(int) * (size_t)std::max(n, 1ll));
        int *err2 = (int *)p;
        e = cudaMemcpyAsync(rp2, rp_new, sizeof(long long) * (size_t)(n + 1), cudaMemcpyDeviceToDevice, s);
        if (!e && arcs_new) dyn_ins_cols_kernel<<<sms * 8, 256, 0, s>>>(a1, arcs_new, ci2);
        HcArgs a2;
        if (!e) e = hc_run_t<false>(rp2, ci2, n, arcs_new, core2, s, h->flags, ws_new, st, h->dev, &a2, est);
        if (!e) {
            cudaFreeAsync(h->ws, s);
            h->ws = ws_new;
            h->rp = rp2;
            h->ci = ci2;
            h->core = core2;
            h->err = err2;
            h->arcs = arcs_new;
            h->a = a2;
            h->a.h0 = nullptr;  // est is freed below
            ws_new = nullptr;
        }
    }
    if (ws_new) cudaFreeAsync(ws_new, s);
    cudaFreeAsync(kbuf, s);
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(buf, s);
    cudaError_t e2 = cudaStreamSynchronize(s);
    if (!e) e = e2;
    if (!e && st) {
        st->affected = rsize;  // |R|: vertices whose estimate was raised
        st->bfs_levels = bfs_levels;
    }
    return e;
}

cudaError_t dyn_destroy(Dyn *h) {
    cudaError_t e = cudaFreeAsync(h->ws, h->s);
    if (!e) e = cudaStreamSynchronize(h->s);
    delete h;
    return e;
}

}  // namespace pico

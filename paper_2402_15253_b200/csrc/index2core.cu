// index2core.cu -- the other two Index2core variants of the paper on sm_100a,
// as ablations of HistoCore (PAPER.md P:365-400,
// P:646-648; Table tab:nbrcnthisto P:751-770):
//
//   CntCore (Alg 5, the paper's first proposal): each round
//     recomputes cnt(u) = #{v in nbr(u) : h(v) >= h(u)} for every u in
//     V_active (the neighbours of the previous round's changed vertices; all
//     vertices in round 1), takes the frontiers {cnt(u) < h(u)} (Theorem 3,
//     P:374-379) and estimates them with HINDEX over ALL their neighbours --
//     the histogram is rebuilt every time a vertex is a frontier, the edge
//     re-access HistoCore removes.
//   NbrCore (the baseline of [GPU-core1]): every vertex of V_active
//     recomputes HINDEX, with no cnt filter.
//
// Both run strict synchronous rounds (h^t from h^{t-1}): the
// estimates of a round are written to newc and committed after every HINDEX
// of the round, so the changed sets are exactly HistoCore's and the Jacobi
// reference's (l2 and every |C_t| pinned in tests/test_parity.py).
//
// Per round (host-driven launches; these are ablations, not the hot path):
//   [CntCore] segments of V_active -> cnt (64-arc segments, thread each) ->
//             filter {cnt < h}
//   [NbrCore] filter = V_active
//   frontiers split by cap = h(u): warp per vertex with shared-memory bins
//   (cap <= 1024) or CTA per vertex (16 K shared bins; global bins in the
//   vertex's histogram slots beyond that)
//   commit changed estimates, list the changed vertices
//   V_active <- neighbours of the changed vertices (bitmap, then compacted)
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace pico {

namespace {

constexpr int kSeg = 64;         // arcs per counting / marking segment
constexpr int kWarpCap = 1024;   // warp class: cap <= 1024
constexpr int kCtaBins = 16384;  // CTA class shared-memory bins

struct I2cArgs {
    const long long *rp;
    const int *ci;
    int n;
    int *core;      // h^{t-1} during a round (= core_out)
    int *newc;      // h^t of the round's frontiers
    int *cnt;       // cnt(u) of active u (CntCore), zero outside a round
    unsigned *act;  // V_active bitmap (next round)
    int *A;         // V_active list
    int *Fw, *Fc;   // frontier lists: warp class / CTA class
    int *Ch;        // changed vertices of the round
    int2 *SG;       // (vertex, segment) work items
    int *histo;     // global bins of CTA-class vertices with cap > kCtaBins
    unsigned long long *c;  // counters: 0 nA, 1 nFw, 2 nFc, 3 nCh, 4 nSG, 5 arcs read
    long long nwords;
};

__device__ __forceinline__ int deg_of(const I2cArgs &a, int v) { return (int)(a.rp[v + 1] - a.rp[v]); }

// H0: h^0 = deg; V_active = every non-isolated vertex
__global__ void i2c_init_kernel(I2cArgs a) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    long long iters = ((long long)a.n + nthreads - 1) / nthreads;
    for (long long it = 0; it < iters; it++) {
        long long v = it * nthreads + (long long)blockIdx.x * blockDim.x + threadIdx.x;
        int d = v < a.n ? deg_of(a, (int)v) : 0;
        if (v < a.n) {
            a.core[v] = d;
            a.cnt[v] = 0;
        }
        warp_append(d > 0, (int)v, a.A, &a.c[0]);
    }
}

// (vertex, segment) items for the rows of a vertex list
__global__ void i2c_segments_kernel(I2cArgs a, const int *list, const unsigned long long *nlist) {
    const long long nl = (long long)bcast_u64(nlist);
    long long nthreads = (long long)gridDim.x * blockDim.x;
    long long iters = (nl + nthreads - 1) / nthreads;
    long long arcs = 0;
    for (long long it = 0; it < iters; it++) {
        long long i = it * nthreads + (long long)blockIdx.x * blockDim.x + threadIdx.x;
        int v = 0, ns = 0;
        if (i < nl) {
            v = list[i];
            int d = deg_of(a, v);
            ns = (d + kSeg - 1) / kSeg;
            arcs += d;
        }
        warp_append_segments(v, ns, a.SG, &a.c[4]);  // a hub's segments written by the whole warp
    }
    long long s = warp_sum64(arcs);
    if (lane_id() == 0 && s) atomicAdd(&a.c[5], (unsigned long long)s);
}

// CntCore: cnt(u) += #{v in segment : h(v) >= h(u)}
__global__ void i2c_cnt_kernel(I2cArgs a) {
    const long long ns = (long long)bcast_u64(&a.c[4]);
    long long nthreads = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += nthreads) {
        int2 sg = a.SG[i];
        long long r0 = a.rp[sg.x], r1 = a.rp[sg.x + 1];
        long long b = r0 + (long long)sg.y * kSeg, e = min(b + kSeg, r1);
        const int hu = __ldcg(a.core + sg.x);
        int c = 0;
#pragma unroll 8
        for (long long x = b; x < e; x++) c += __ldcg(a.core + __ldg(a.ci + x)) >= hu;
        if (c) atomicAdd(a.cnt + sg.x, c);
    }
}

// frontiers of the round (CNT: cnt(u) < h(u), Theorem 3; else all of
// V_active), split by cap = h(u) into the warp and CTA classes
template <bool CNT>
__global__ void i2c_filter_kernel(I2cArgs a) {
    const long long na = (long long)bcast_u64(&a.c[0]);
    long long nthreads = (long long)gridDim.x * blockDim.x;
    long long iters = (na + nthreads - 1) / nthreads;
    for (long long it = 0; it < iters; it++) {
        long long i = it * nthreads + (long long)blockIdx.x * blockDim.x + threadIdx.x;
        bool f = false;
        int u = 0, cap = 0;
        if (i < na) {
            u = a.A[i];
            cap = a.core[u];
            if (CNT) {
                f = a.cnt[u] < cap;
                a.cnt[u] = 0;
            } else {
                f = true;
            }
        }
        warp_append(f && cap <= kWarpCap, u, a.Fw, &a.c[1]);
        warp_append(f && cap > kWarpCap, u, a.Fc, &a.c[2]);
    }
}

// HINDEX(nbr(u), cap) of P:139-149 for the warp class: bins 1..cap of
// min(h(v), cap) in shared memory, descending walk to the first b with
// sum >= b
__global__ void __launch_bounds__(256) i2c_hindex_warp_kernel(I2cArgs a) {
    __shared__ int sh[8][kWarpCap + 1];
    const int wib = threadIdx.x >> 5, lane = lane_id();
    int *bins = sh[wib];
    const long long nf = (long long)bcast_u64(&a.c[1]);
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    long long arcs = 0;
    for (long long i = gw; i < nf; i += nw) {
        const int u = a.Fw[i];
        const long long hb = a.rp[u];
        const int d = (int)(a.rp[u + 1] - hb), cap = a.core[u];
        for (int b = lane; b <= cap; b += 32) bins[b] = 0;
        __syncwarp();
        for (int e = lane; e < d; e += 32) atomicAdd(&bins[min(__ldcg(a.core + __ldg(a.ci + hb + e)), cap)], 1);
        __syncwarp();
        int carry = 0, top = cap, h = 0;
        for (;;) {
            int kk = top - lane;
            int val = kk >= 1 ? bins[kk] : 0;
            int incl = warp_incl_scan(val);
            unsigned m = __ballot_sync(FULL, kk >= 1 && carry + incl >= kk);
            if (m) {
                h = top - (__ffs(m) - 1);
                break;
            }
            carry += __shfl_sync(FULL, incl, 31);
            top -= 32;
            if (top < 1) break;  // broken input (no neighbour): h stays 0
        }
        if (lane == 0) a.newc[u] = h;
        arcs += lane == 0 ? d : 0;
        __syncwarp();
    }
    long long s = warp_sum64(arcs);
    if (lane == 0 && s) atomicAdd(&a.c[5], (unsigned long long)s);
}

// the CTA class: one block per vertex, 16 K shared bins; caps beyond that use
// the vertex's own global histogram slots rp[u] + b - 1 (b <= cap <= deg)
__global__ void __launch_bounds__(512) i2c_hindex_cta_kernel(I2cArgs a) {
    extern __shared__ int sbins[];
    __shared__ int red[40];
    const long long nf = (long long)bcast_u64(&a.c[2]);
    const int tid = threadIdx.x, nt = blockDim.x, lane = lane_id(), wid = tid >> 5, nwarp = nt >> 5;
    long long arcs = 0;
    for (long long i = blockIdx.x; i < nf; i += gridDim.x) {
        const int u = a.Fc[i];
        const long long hb = a.rp[u];
        const int d = (int)(a.rp[u + 1] - hb), cap = a.core[u];
        const bool global = cap > kCtaBins;
        int *bins = global ? a.histo + hb - 1 : sbins;  // bin b at bins[b]
        for (int b = tid; b <= cap; b += nt)
            if (!global || b >= 1) bins[b] = 0;
        __syncthreads();
        for (int e = tid; e < d; e += nt) atomicAdd(&bins[min(__ldcg(a.core + __ldg(a.ci + hb + e)), cap)], 1);
        __syncthreads();
        // block-wide descending search: h = max b in 1..cap with sum_{j>=b} bins[j] >= b
        int c = (cap + nt - 1) / nt;
        int hiT = cap - tid * c, loT = max(1, cap - (tid + 1) * c + 1);
        int tsum = 0;
        for (int b = hiT; b >= loT; b--) tsum += global ? __ldcg(bins + b) : bins[b];
        int incl = warp_incl_scan(tsum);
        if (lane == 31) red[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            int x = lane < nwarp ? red[lane] : 0;
            int xi = warp_incl_scan(x);
            if (lane < nwarp) red[lane] = xi - x;
        }
        __syncthreads();
        int s = red[wid] + incl - tsum, cand = 0;
        for (int b = hiT; b >= loT; b--) {
            s += global ? __ldcg(bins + b) : bins[b];
            if (s >= b) { cand = b; break; }
        }
        __syncthreads();
        if (tid == 0) red[32] = 0;
        __syncthreads();
        if (cand) atomicMax(&red[32], cand);
        __syncthreads();
        if (tid == 0) {
            a.newc[u] = red[32];
            arcs += d;
        }
        __syncthreads();
    }
    if (tid == 0 && arcs) atomicAdd(&a.c[5], (unsigned long long)arcs);
}

// commit h^t of the round's frontiers; list the changed vertices
__global__ void i2c_commit_kernel(I2cArgs a, const int *F, const unsigned long long *nF) {
    const long long nf = (long long)bcast_u64(nF);
    long long nthreads = (long long)gridDim.x * blockDim.x;
    long long iters = (nf + nthreads - 1) / nthreads;
    for (long long it = 0; it < iters; it++) {
        long long i = it * nthreads + (long long)blockIdx.x * blockDim.x + threadIdx.x;
        bool ch = false;
        int u = 0;
        if (i < nf) {
            u = F[i];
            int h = a.newc[u];
            ch = h < a.core[u];
            if (ch) a.core[u] = h;
        }
        warp_append(ch, u, a.Ch, &a.c[3]);
    }
}

// V_active of the next round: the neighbours of the changed vertices
__global__ void i2c_mark_kernel(I2cArgs a) {
    const long long ns = (long long)bcast_u64(&a.c[4]);
    long long nthreads = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += nthreads) {
        int2 sg = a.SG[i];
        long long r0 = a.rp[sg.x], r1 = a.rp[sg.x + 1];
        long long b = r0 + (long long)sg.y * kSeg, e = min(b + kSeg, r1);
        for (long long x = b; x < e; x++) {
            int v = __ldg(a.ci + x);
            red_or(a.act + (v >> 5), 1u << (v & 31));
        }
    }
}

// bitmap -> V_active list (bits cleared)
__global__ void i2c_compact_kernel(I2cArgs a) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    long long iters = (a.nwords + nthreads - 1) / nthreads;
    for (long long it = 0; it < iters; it++) {
        long long w = it * nthreads + (long long)blockIdx.x * blockDim.x + threadIdx.x;
        unsigned bits = 0;
        if (w < a.nwords) {
            bits = a.act[w];
            if (bits) a.act[w] = 0;
        }
        int c = __popc(bits);
        int incl = warp_incl_scan(c);
        int total = __shfl_sync(FULL, incl, 31);
        if (!total) continue;
        unsigned long long base = 0;
        if (lane_id() == 0) base = atomicAdd(&a.c[0], (unsigned long long)total);
        base = __shfl_sync(FULL, base, 0);
        unsigned long long o = base + incl - c;
        while (bits) {
            a.A[o++] = (int)(w * 32 + (__ffs(bits) - 1));
            bits &= bits - 1;
        }
    }
}

size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

size_t i2c_workspace_bytes(long long n, long long arcs) {
    size_t b = a256(sizeof(unsigned long long) * 8);
    b += a256(sizeof(int) * (size_t)n) * 7;                     // newc, cnt, A, Fw, Fc, Ch, (spare)
    b += a256(sizeof(unsigned) * (size_t)((n + 31) / 32));     // act
    b += a256(sizeof(int2) * (size_t)(n + arcs / kSeg + 64));  // SG
    b += a256(sizeof(int) * (size_t)std::max(arcs, 1ll));      // histo (global bins)
    return b;
}

cudaError_t i2c_run(const long long *rp, const int *ci, long long n, long long arcs, int *core, cudaStream_t s,
                    uint32_t flags, bool cnt_filter, void *ws, pico_stats_t *st, const DevInfo &dev) {
    I2cArgs a;
    char *p = (char *)ws;
    a.c = (unsigned long long *)p; p += a256(sizeof(unsigned long long) * 8);
    a.newc = (int *)p; p += a256(sizeof(int) * (size_t)n);
    a.cnt = (int *)p; p += a256(sizeof(int) * (size_t)n);
    a.A = (int *)p; p += a256(sizeof(int) * (size_t)n);
    a.Fw = (int *)p; p += a256(sizeof(int) * (size_t)n);
    a.Fc = (int *)p; p += a256(sizeof(int) * (size_t)n);
    a.Ch = (int *)p; p += a256(sizeof(int) * (size_t)n);
    p += a256(sizeof(int) * (size_t)n);
    a.nwords = (n + 31) / 32;
    a.act = (unsigned *)p; p += a256(sizeof(unsigned) * (size_t)a.nwords);
    a.SG = (int2 *)p; p += a256(sizeof(int2) * (size_t)(n + arcs / kSeg + 64));
    a.histo = (int *)p;
    a.rp = rp; a.ci = ci; a.n = (int)n; a.core = core;
    const int sms = dev.sms;
    cudaError_t e;
    cudaEvent_t t0 = nullptr, t1 = nullptr;  // PICO_F_TIMING: the whole run in the rounds slot
    const bool timing = st && (flags & PICO_F_TIMING);
    if (timing) {
        cudaEventCreate(&t0);
        cudaEventCreate(&t1);
        cudaEventRecord(t0, s);
    }
    if ((e = cudaMemsetAsync(a.c, 0, sizeof(unsigned long long) * 8, s))) return e;
    if ((e = cudaMemsetAsync(a.act, 0, sizeof(unsigned) * (size_t)a.nwords, s))) return e;
    auto grid = [&](long long work) {
        return std::max(1, (int)std::min<long long>((work + 255) / 256, (long long)sms * 16));
    };
    i2c_init_kernel<<<grid(n), 256, 0, s>>>(a);
    long long launches = 1;
    const size_t smC = sizeof(int) * (kCtaBins + 1);
    cudaFuncSetAttribute(i2c_hindex_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smC);
    int occC = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occC, i2c_hindex_cta_kernel, 512, smC);
    unsigned long long h[8];
    std::vector<long long> sizes;
    long long active_total = 0, frontier_total = 0;
    for (;;) {
        if ((e = cudaMemcpyAsync(h, a.c, sizeof(h), cudaMemcpyDeviceToHost, s))) return e;
        if ((e = cudaStreamSynchronize(s))) return e;
        const long long na = (long long)h[0];
        if (na == 0) break;
        active_total += na;
        // counters 1..4 of the round (5 = arcs read accumulates over the run)
        if ((e = cudaMemsetAsync(a.c + 1, 0, sizeof(unsigned long long) * 4, s))) return e;
        if (cnt_filter) {
            i2c_segments_kernel<<<grid(na), 256, 0, s>>>(a, a.A, a.c + 0);
            i2c_cnt_kernel<<<sms * 16, 256, 0, s>>>(a);
            i2c_filter_kernel<true><<<grid(na), 256, 0, s>>>(a);
            launches += 3;
        } else {
            i2c_filter_kernel<false><<<grid(na), 256, 0, s>>>(a);
            launches += 1;
        }
        i2c_hindex_warp_kernel<<<sms * 8, 256, 0, s>>>(a);
        i2c_hindex_cta_kernel<<<sms * std::max(1, occC), 512, smC, s>>>(a);
        i2c_commit_kernel<<<grid(na), 256, 0, s>>>(a, a.Fw, a.c + 1);
        i2c_commit_kernel<<<grid(na), 256, 0, s>>>(a, a.Fc, a.c + 2);
        launches += 4;
        if ((e = cudaMemcpyAsync(h, a.c, sizeof(h), cudaMemcpyDeviceToHost, s))) return e;
        if ((e = cudaStreamSynchronize(s))) return e;
        frontier_total += (long long)(h[1] + h[2]);
        const long long nch = (long long)h[3];
        if (nch == 0) break;  // a fixed point: the estimates are the coreness
        sizes.push_back(nch);
        // next V_active: the neighbours of the changed vertices
        if ((e = cudaMemsetAsync(a.c + 4, 0, sizeof(unsigned long long), s))) return e;
        i2c_segments_kernel<<<grid(nch), 256, 0, s>>>(a, a.Ch, a.c + 3);
        i2c_mark_kernel<<<sms * 16, 256, 0, s>>>(a);
        if ((e = cudaMemsetAsync(a.c + 0, 0, sizeof(unsigned long long), s))) return e;
        i2c_compact_kernel<<<grid(a.nwords), 256, 0, s>>>(a);
        launches += 3;
        if ((e = cudaGetLastError())) return e;
        if ((long long)sizes.size() > arcs + 2) return cudaErrorAssert;  // beyond any valid l2 (<= 2m): broken input
    }
    if ((e = cudaGetLastError())) return e;
    if (timing) {
        float ms = 0;
        cudaEventRecord(t1, s);
        cudaEventSynchronize(t1);
        cudaEventElapsedTime(&ms, t0, t1);
        st->kernel_ms[PICO_K_ROUNDS] += ms;
        st->kernel_launches[PICO_K_ROUNDS] += 1;
    }
    if (t0) {
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
    }
    if (st) {
        st->rounds = (int64_t)sizes.size();
        st->kernel_count += launches;
        st->frontier_total = frontier_total;   // HINDEX evaluations (vertices)
        st->alive_scanned = active_total;      // sum over rounds of |V_active|
        st->arcs_scanned = (int64_t)h[5];      // neighbour-list entries read (Fig 3 edge accesses)
        if (st->frontier_sizes)
            for (size_t i = 0; i < sizes.size() && (int64_t)i < st->frontier_sizes_cap; i++)
                st->frontier_sizes[i] = sizes[i];
    }
    return cudaSuccess;
}

}  // namespace pico

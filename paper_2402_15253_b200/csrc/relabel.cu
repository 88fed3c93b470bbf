// relabel.cu -- optional internal compaction of the vertex id space (a
// locality optimisation; "an internal relabel is an
// optimisation").  Isolated vertices (coreness 0, never in any frontier) are
// dropped and the others renumbered in their original order:
//   new(v) = #{u < v : deg(u) > 0}      (rank in the non-isolated bitmap)
// Coreness is a graph invariant, so running either algorithm on the compacted
// graph and mapping the result back is bit-exact.
//
// Why: on graphs like RMAT-26 half of the 2^26 ids are isolated; dropping them
// halves every per-vertex array, so more of the per-arc neighbour gathers hit
// the 126 MB L2.  Because isolated rows are empty, arc positions do not move:
// rowptr2[new(v)] = rowptr[v] and colidx2[e] = new(colidx[e]) is a pure
// streaming map.  new(u) comes from one L2-resident 8-byte word per 32 ids
// (the non-isolated bitmap word and the exclusive prefix count of its
// predecessors) instead of an n-entry permutation gather.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace pico {

// bitmap word w: bit j set iff vertex 32w+j has degree > 0; wcnt[w] = popc
__global__ void rl_bits_kernel(const long long *rp, long long n, long long nwords, unsigned *bits,
                               unsigned *wcnt) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += nthreads) {
        unsigned b = 0;
        long long v0 = w * 32;
        long long prev = rp[min(v0, n)];
        for (int j = 0; j < 32 && v0 + j < n; j++) {
            long long nx = rp[v0 + j + 1];
            if (nx > prev) b |= 1u << j;
            prev = nx;
        }
        bits[w] = b;
        wcnt[w] = __popc(b);
    }
}

__device__ __forceinline__ int rl_rank(const unsigned *bits, const unsigned *wpre, int u, unsigned long long hot) {
    unsigned w = ld_cg_u32(bits + (u >> 5), hot);
    return (int)(ld_cg_u32(wpre + (u >> 5), hot) + __popc(w & ((1u << (u & 31)) - 1)));
}

// (bitmap word, prefix) packed: one 8-byte gather per rank
__global__ void rl_pack_kernel(const unsigned *bits, const unsigned *wpre, long long nwords, uint2 *bw) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += nthreads)
        bw[w] = make_uint2(bits[w], wpre[w]);
}

__device__ __forceinline__ int rl_rank2(const uint2 *bw, int u) {
    uint2 x = __ldcg(bw + (u >> 5));
    return (int)(x.y + __popc(x.x & ((1u << (u & 31)) - 1)));
}

// rowptr2 and inverse map
__global__ void rl_rows_kernel(const long long *rp, long long n, const unsigned *bits, const unsigned *wpre,
                               long long *rp2, int *inv, long long arcs) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    const unsigned long long hot = pol_last();
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += nthreads) {
        if ((bits[v >> 5] >> (v & 31)) & 1u) {
            int r = rl_rank(bits, wpre, (int)v, hot);
            rp2[r] = rp[v];
            inv[r] = (int)v;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        long long nw = (n + 31) / 32;
        long long n2 = (long long)wpre[nw - 1] + __popc(bits[nw - 1]);
        rp2[n2] = arcs;
    }
}

// colidx2[e] = new(colidx[e]): coalesced stream in, coalesced stream out,
// four arcs (and their rank gathers) in flight per thread
__global__ void rl_arcs_kernel(const int *ci, long long arcs, const uint2 *bw, int *ci2) {
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    const unsigned long long cold = pol_first();
    long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; e + 3 * nthreads < arcs; e += 4 * nthreads) {
        int u0 = ld_stream(ci + e, cold), u1 = ld_stream(ci + e + nthreads, cold);
        int u2 = ld_stream(ci + e + 2 * nthreads, cold), u3 = ld_stream(ci + e + 3 * nthreads, cold);
        int r0 = rl_rank2(bw, u0), r1 = rl_rank2(bw, u1), r2 = rl_rank2(bw, u2), r3 = rl_rank2(bw, u3);
        ci2[e] = r0;
        ci2[e + nthreads] = r1;
        ci2[e + 2 * nthreads] = r2;
        ci2[e + 3 * nthreads] = r3;
    }
    for (; e < arcs; e += nthreads) ci2[e] = rl_rank2(bw, ld_stream(ci + e, cold));
}

__global__ void rl_back_kernel(const unsigned *bits, const unsigned *wpre, const int *core2, long long n,
                               int *core_out) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    const unsigned long long hot = pol_last();
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += nthreads) {
        bool live = (bits[v >> 5] >> (v & 31)) & 1u;
        core_out[v] = live ? core2[rl_rank(bits, wpre, (int)v, hot)] : 0;
    }
}

static size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t cub_scan_bytes(long long nw) {
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum((void *)nullptr, b, (const unsigned *)nullptr, (unsigned *)nullptr, (int)nw);
    return b;
}

size_t relabel_workspace_bytes(long long n, long long arcs) {
    long long nw = (n + 31) / 32;
    size_t b = 0;
    b += a256(sizeof(unsigned) * (size_t)nw) * 3;       // bits, wcnt, wpre
    b += a256(sizeof(uint2) * (size_t)nw);              // (bits, wpre) packed
    b += a256(sizeof(long long) * (size_t)(n + 1));     // rp2
    b += a256(sizeof(int) * (size_t)n);                 // inv
    b += a256(sizeof(int) * (size_t)arcs);              // ci2
    b += a256(sizeof(int) * (size_t)n);                 // core2
    b += a256(cub_scan_bytes(nw));
    return b;
}

cudaError_t relabel_build(const long long *rp, const int *ci, long long n, long long arcs, cudaStream_t s,
                          void *ws, const DevInfo &dev, bool force, Relabel *out) {
    long long nw = (n + 31) / 32;
    char *p = (char *)ws;
    unsigned *bits = (unsigned *)p; p += a256(sizeof(unsigned) * (size_t)nw);
    unsigned *wcnt = (unsigned *)p; p += a256(sizeof(unsigned) * (size_t)nw);
    unsigned *wpre = (unsigned *)p; p += a256(sizeof(unsigned) * (size_t)nw);
    uint2 *bw = (uint2 *)p; p += a256(sizeof(uint2) * (size_t)nw);
    long long *rp2 = (long long *)p; p += a256(sizeof(long long) * (size_t)(n + 1));
    int *inv = (int *)p; p += a256(sizeof(int) * (size_t)n);
    int *ci2 = (int *)p; p += a256(sizeof(int) * (size_t)arcs);
    int *core2 = (int *)p; p += a256(sizeof(int) * (size_t)n);
    void *tmp = p;
    size_t tmpb = cub_scan_bytes(nw);
    cudaError_t e;
    auto grid = [&](long long work) {
        return std::max(1, (int)std::min<long long>((work + 255) / 256, (long long)dev.sms * 16));
    };
    rl_bits_kernel<<<grid(nw), 256, 0, s>>>(rp, n, nw, bits, wcnt);
    if ((e = cub::DeviceScan::ExclusiveSum(tmp, tmpb, wcnt, wpre, (int)nw, s))) return e;
    unsigned hl[2] = {0, 0};
    if ((e = cudaMemcpyAsync(&hl[0], wpre + nw - 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaMemcpyAsync(&hl[1], wcnt + nw - 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    out->n2 = (long long)hl[0] + hl[1];
    out->launches = 2;
    // compaction pays only when a sizeable share of the ids is isolated
    out->active = force || out->n2 * 10 < n * 9;
    if (!out->active) return cudaGetLastError();
    rl_rows_kernel<<<grid(n), 256, 0, s>>>(rp, n, bits, wpre, rp2, inv, arcs);
    rl_pack_kernel<<<grid(nw), 256, 0, s>>>(bits, wpre, nw, bw);
    rl_arcs_kernel<<<dev.sms * 16, 256, 0, s>>>(ci, arcs, bw, ci2);
    if ((e = cudaGetLastError())) return e;
    out->rp2 = rp2;
    out->ci2 = ci2;
    out->bits = bits;
    out->wpre = wpre;
    out->inv = inv;
    out->core2 = core2;
    out->launches = 5;
    return cudaSuccess;
}

cudaError_t relabel_back(const Relabel &r, long long n, int *core_out, cudaStream_t s, const DevInfo &dev) {
    int blocks = (int)std::min<long long>((n + 255) / 256, (long long)dev.sms * 16);
    rl_back_kernel<<<std::max(blocks, 1), 256, 0, s>>>(r.bits, r.wpre, r.core2, n, core_out);
    return cudaGetLastError();
}

}  // namespace pico

// capi.cu -- the extern "C" boundary declared in include/pico.h: argument
// checks, workspace ownership, optional CSR validation, dispatch to the
// HistoCore / PeelOne drivers, status codes and the thread-local last error.
#include <mutex>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "kernels.h"
#include "lsa_exchange.h"
#include "pico_shard.h"
#include "pico_dyn.h"

namespace pico {

// ---------------------------------------------------------------------------
// PICO_F_VALIDATE: the CSR contract of pico.h
// ---------------------------------------------------------------------------
enum { BAD_ROWPTR = 1, BAD_RANGE = 2, BAD_LOOP = 4, BAD_ORDER = 8, BAD_ASYM = 16 };

__global__ void validate_rowptr_kernel(const long long *rp, long long n, long long arcs, int *bad) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += nthreads) {
        long long a = rp[v], b = rp[v + 1];
        if (a < 0 || b < a || b > arcs) atomicOr(bad, BAD_ROWPTR);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (rp[0] != 0 || rp[n] != arcs)) atomicOr(bad, BAD_ROWPTR);
}

__global__ void validate_arcs_kernel(const long long *rp, const int *ci, long long n, int *bad) {
    // one warp per row
    long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    int lane = threadIdx.x & 31;
    int flags = 0;
    for (long long v = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5); v < n; v += nw) {
        long long a = rp[v], b = rp[v + 1];
        for (long long e = a + lane; e < b; e += 32) {
            int u = ci[e];
            if (u < 0 || u >= n) { flags |= BAD_RANGE; continue; }
            if (u == v) flags |= BAD_LOOP;
            if (e > a && ci[e - 1] >= u) flags |= BAD_ORDER;
            // symmetry: v must appear in row u (binary search; rows sorted)
            long long lo = rp[u], hi = rp[u + 1] - 1;
            bool found = false;
            while (lo <= hi) {
                long long mid = (lo + hi) >> 1;
                int x = ci[mid];
                if (x == v) { found = true; break; }
                if (x < v) lo = mid + 1; else hi = mid - 1;
            }
            if (!found) flags |= BAD_ASYM;
        }
    }
    if (flags) atomicOr(bad, flags);
}

cudaError_t validate_run(const long long *rp, const int *ci, long long n, long long arcs, cudaStream_t s,
                         void *ws, int *bad_out) {
    int *bad = (int *)ws;
    cudaError_t err;
    if ((err = cudaMemsetAsync(bad, 0, sizeof(int), s))) return err;
    validate_rowptr_kernel<<<1024, 256, 0, s>>>(rp, n, arcs, bad);
    int h = 0;
    if ((err = cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s))) return err;
    if ((err = cudaStreamSynchronize(s))) return err;
    if (!h && arcs > 0) {
        validate_arcs_kernel<<<2048, 256, 0, s>>>(rp, ci, n, bad);
        if ((err = cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s))) return err;
        if ((err = cudaStreamSynchronize(s))) return err;
    }
    *bad_out = h;
    return cudaGetLastError();
}

__global__ void max_kernel(const int *x, long long n, int *out) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    int m = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nthreads) m = max(m, x[i]);
    m = max(m, __shfl_xor_sync(FULL, m, 16));
    m = max(m, __shfl_xor_sync(FULL, m, 8));
    m = max(m, __shfl_xor_sync(FULL, m, 4));
    m = max(m, __shfl_xor_sync(FULL, m, 2));
    m = max(m, __shfl_xor_sync(FULL, m, 1));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

}  // namespace pico

using namespace pico;

static thread_local std::string g_last_error;

static int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

static int cuda_fail(cudaError_t e, const char *where) {
    cudaGetLastError();  // clear sticky-free errors
    if (e == cudaErrorMemoryAllocation) return fail(PICO_ENOMEM, "%s: %s", where, cudaGetErrorString(e));
    if (e == cudaErrorAssert)  // raised by the library itself, not a device assert
        return fail(PICO_EGRAPH, "%s: histogram invariant violated (input is not a symmetric, deduplicated, "
                    "loop-free CSR?)", where);
    return fail(PICO_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

static cudaError_t dev_info(DevInfo *d) {
    cudaError_t e;
    if ((e = cudaGetDevice(&d->device))) return e;
    if ((e = cudaDeviceGetAttribute(&d->sms, cudaDevAttrMultiProcessorCount, d->device))) return e;
    if ((e = cudaDeviceGetAttribute(&d->coop, cudaDevAttrCooperativeLaunch, d->device))) return e;
    return cudaSuccess;
}

// one library-owned pool per device: freed workspace stays in it, so
// a repeated call allocates in microseconds instead of an OS round trip
static std::mutex g_pool_mu;
static cudaMemPool_t g_pool[64];

cudaError_t pico::lib_malloc_async(void **p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e;
    if ((e = cudaGetDevice(&dev))) return e;
    if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, s);
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (!g_pool[dev]) {
            cudaMemPoolProps pp{};
            pp.allocType = cudaMemAllocationTypePinned;
            pp.location.type = cudaMemLocationTypeDevice;
            pp.location.id = dev;
            if ((e = cudaMemPoolCreate(&g_pool[dev], &pp))) { g_pool[dev] = nullptr; return e; }
            unsigned long long thr = ~0ull;
            cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool = g_pool[dev];
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

static void reset_stats(pico_stats_t *st) {
    if (!st) return;
    int64_t *fs = st->frontier_sizes, *ra = st->round_arcs, *rn = st->round_ns;
    int64_t cap = st->frontier_sizes_cap, fcap = st->frontier_counts_cap;
    int32_t *fc = st->frontier_counts;
    memset(st, 0, sizeof(*st));
    st->frontier_sizes = fs;
    st->frontier_sizes_cap = cap;
    st->round_arcs = ra;
    st->round_ns = rn;
    st->frontier_counts = fc;
    st->frontier_counts_cap = fcap;
}

extern "C" {

const char *pico_status_string(int status) {
    switch (status) {
        case PICO_OK: return "PICO_OK";
        case PICO_EINVAL: return "PICO_EINVAL";
        case PICO_ENOTSUP: return "PICO_ENOTSUP";
        case PICO_ENOMEM: return "PICO_ENOMEM";
        case PICO_ECUDA: return "PICO_ECUDA";
        case PICO_ENCCL: return "PICO_ENCCL";
        case PICO_EGRAPH: return "PICO_EGRAPH";
        default: return "PICO_UNKNOWN";
    }
}

const char *pico_last_error(void) { return g_last_error.c_str(); }

int pico_version(void) { return 200; }

int pico_clamp_hammer(int mode, int32_t d, int32_t k, int64_t c, int32_t *final_out, int64_t *observed_gt_k,
                      int64_t *observed_k1, cudaStream_t stream) {
    if (mode < 0 || mode > 2 || c < 0 || k < 0 || d < 0 || !final_out || !observed_gt_k || !observed_k1)
        return fail(PICO_EINVAL, "pico_clamp_hammer: bad argument");
    long long gt = 0, k1 = 0;
    int fin = 0;
    cudaError_t e = po_clamp_hammer(mode, d, k, c, &fin, &gt, &k1, stream);
    if (e) return cuda_fail(e, "pico_clamp_hammer");
    *final_out = fin;
    *observed_gt_k = gt;
    *observed_k1 = k1;
    return PICO_OK;
}

static const long long kRelabelMinN = 16ll << 20;  // per-vertex arrays beyond L2 reach

int64_t pico_relabel_threshold(void) { return kRelabelMinN; }

static bool use_relabel(long long n, long long m, uint32_t flags) {
    if (m <= 0 || (flags & PICO_F_NO_RELABEL)) return false;
    return (flags & PICO_F_RELABEL) || n >= kRelabelMinN;
}

static size_t algo_bytes(long long n, long long arcs, int algo, uint32_t flags) {
    if (algo == PICO_ALGO_HISTOCORE) return hc_workspace_bytes(n, arcs, flags);
    if (algo == PICO_ALGO_PEELONE) return po_workspace_bytes(n, arcs, flags);
    if (algo == PICO_ALGO_AUTO)
        return std::max(hc_workspace_bytes(n, arcs, flags), po_workspace_bytes(n, arcs, flags));
    if (algo == PICO_ALGO_CNTCORE || algo == PICO_ALGO_NBRCORE) return i2c_workspace_bytes(n, arcs);
    return 0;
}

// PICO_ALGO_AUTO: HistoCore on skewed graphs of moderate
// size, PeelOne otherwise.  Measured on B200 over RMAT / flat-Kronecker
// graphs of 2^12..2^22 vertices (scripts/algo_sweep.py):
// HistoCore wins where the degree skew d_max * n / 2m is high and the graph
// small enough that its dense rounds are cheap; PeelOne wins on flat graphs
// (few levels) and on large ones (its one pass over the arcs).
constexpr double kAutoSkew = 60.0;
constexpr long long kAutoMaxArcs = 64ll << 20;

__global__ void deg_max_kernel(const long long *rp, long long n, int *out) {
    long long nthreads = (long long)gridDim.x * blockDim.x;
    int m = 0;
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += nthreads)
        m = max(m, (int)(rp[v + 1] - rp[v]));
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

static cudaError_t auto_select(const long long *rp, long long n, long long arcs, cudaStream_t s, void *scratch,
                               const DevInfo &dev, int *algo) {
    int *d = (int *)scratch, dmax = 0;
    cudaError_t e = cudaMemsetAsync(d, 0, sizeof(int), s);
    if (e) return e;
    deg_max_kernel<<<dev.sms * 4, 256, 0, s>>>(rp, n, d);
    if ((e = cudaMemcpyAsync(&dmax, d, sizeof(int), cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    double skew = arcs > 0 ? (double)dmax * (double)n / (double)arcs : 0.0;
    *algo = (skew >= kAutoSkew && arcs <= kAutoMaxArcs) ? PICO_ALGO_HISTOCORE : PICO_ALGO_PEELONE;
    return cudaGetLastError();
}

size_t pico_workspace_bytes(int64_t n, int64_t m, int algo, uint32_t flags) {
    if (n <= 0 || m < 0) return 256;
    long long arcs = 2 * (long long)m;
    size_t b = algo_bytes(n, arcs, algo, flags);
    if (use_relabel(n, m, flags)) b = ((b + 255) & ~size_t(255)) + relabel_workspace_bytes(n, arcs);
    return std::max<size_t>(b, 256);
}

int pico_coreness_ex(const int64_t *rowptr, const int32_t *colidx, int64_t n, int64_t m, int algo,
                     int32_t *core_out, pico_stream_t stream_, uint32_t flags, void *workspace,
                     size_t workspace_bytes, pico_stats_t *stats) {
    cudaStream_t s = (cudaStream_t)stream_;
    g_last_error.clear();
    reset_stats(stats);
    if (n < 0 || m < 0) return fail(PICO_EINVAL, "negative n (%lld) or m (%lld)", (long long)n, (long long)m);
    if (algo < PICO_ALGO_HISTOCORE || algo > PICO_ALGO_NBRCORE) return fail(PICO_EINVAL, "unknown algo %d", algo);
    if (stats) stats->algo = algo == PICO_ALGO_AUTO ? PICO_ALGO_HISTOCORE : algo;
    if (n == 0) return PICO_OK;
    if (n >= (1ll << 31) - 1) return fail(PICO_ENOTSUP, "n = %lld needs 64-bit vertex ids", (long long)n);
    if (!rowptr || !core_out || (m > 0 && !colidx)) return fail(PICO_EINVAL, "NULL pointer argument");
    const long long arcs = 2 * (long long)m;
    size_t need = pico_workspace_bytes(n, m, algo, flags);
    if (workspace && workspace_bytes < need)
        return fail(PICO_EINVAL, "workspace too small: %zu < %zu bytes", workspace_bytes, need);
    if (workspace && ((uintptr_t)workspace & 255))
        return fail(PICO_EINVAL, "workspace must be 256-byte aligned");

    DevInfo dev;
    cudaError_t e = dev_info(&dev);
    if (e) return cuda_fail(e, "device query");
    void *ws = workspace;
    bool own = false;
    if (!ws) {
        e = lib_malloc_async(&ws, need, s);
        if (e) return cuda_fail(e, "workspace allocation");
        own = true;
    }
    int rc = PICO_OK;
    const long long *rp = (const long long *)rowptr;
    if (flags & PICO_F_VALIDATE) {
        int bad = 0;
        e = validate_run(rp, colidx, n, arcs, s, ws, &bad);
        if (e) rc = cuda_fail(e, "validation");
        else if (bad)
            rc = fail(PICO_EGRAPH, "graph violates the CSR contract (flags 0x%x: %s%s%s%s%s)", bad,
                      (bad & 1) ? "rowptr " : "", (bad & 2) ? "range " : "", (bad & 4) ? "self-loop " : "",
                      (bad & 8) ? "unsorted/duplicate " : "", (bad & 16) ? "asymmetric" : "");
    }
    if (rc == PICO_OK && algo == PICO_ALGO_AUTO && m > 0) {
        e = auto_select(rp, n, arcs, s, ws, dev, &algo);
        if (e) rc = cuda_fail(e, "auto select");
        if (stats) {
            stats->algo = algo;
            stats->kernel_count += 1;
        }
    }
    if (rc == PICO_OK) {
        if (m == 0) {
            if (stats && stats->frontier_counts && stats->frontier_counts_cap >= n)  // no round: no frontier
                memset(stats->frontier_counts, 0, sizeof(int32_t) * (size_t)n);
            e = cudaMemsetAsync(core_out, 0, sizeof(int32_t) * (size_t)n, s);
            if (!e) e = cudaStreamSynchronize(s);
            if (e) rc = cuda_fail(e, "zero core_out");
        } else {
            if (!dev.coop && !(flags & PICO_F_HOST_LOOP)) flags |= PICO_F_HOST_LOOP;
            const long long *grp = rp;
            const int *gci = colidx;
            long long gn = n;
            int *gcore = core_out;
            Relabel rl{};
            // PeelOne compacts only when forced: its guard reads the processed
            // bitmap, not the estimates, so halving the per-vertex arrays buys
            // less than the compaction costs (T: 62.4 ms with, 59.9 without)
            bool relabel = use_relabel(n, m, flags) && (algo != PICO_ALGO_PEELONE || (flags & PICO_F_RELABEL));
            void *aws = ws;
            cudaEvent_t r0 = nullptr, r1 = nullptr;
            bool timing = stats && (flags & PICO_F_TIMING);
            if (relabel) {
                size_t ab = (algo_bytes(n, arcs, algo, flags) + 255) & ~size_t(255);
                if (timing) {
                    cudaEventCreate(&r0);
                    cudaEventCreate(&r1);
                    cudaEventRecord(r0, s);
                }
                nvtx_push(PICO_K_OTHER);
                e = relabel_build(rp, colidx, n, arcs, s, (char *)ws + ab, dev, (flags & PICO_F_RELABEL) != 0, &rl);
                nvtxRangePop();
                if (e) rc = cuda_fail(e, "relabel");
                if (timing) cudaEventRecord(r1, s);
                if (rl.active) {
                    grp = rl.rp2;
                    gci = rl.ci2;
                    gn = rl.n2;
                    gcore = rl.core2;
                } else {
                    if (stats) stats->kernel_count += rl.launches;
                    relabel = false;
                }
            }
            if (rc == PICO_OK) {
                if (algo == PICO_ALGO_HISTOCORE)
                    e = hc_run(grp, gci, gn, arcs, gcore, s, flags, aws, stats, dev);
                else if (algo == PICO_ALGO_PEELONE)
                    e = po_run(grp, gci, gn, arcs, gcore, s, flags, aws, stats, dev);
                else
                    e = i2c_run(grp, gci, gn, arcs, gcore, s, flags, algo == PICO_ALGO_CNTCORE, aws, stats, dev);
                static const char *names[] = {"histocore", "peelone", "auto", "cntcore", "nbrcore"};
                if (e) rc = cuda_fail(e, names[algo]);
            }
            if (rc == PICO_OK && relabel) {
                cudaEvent_t b0 = nullptr, b1 = nullptr;
                if (timing) {
                    cudaEventCreate(&b0);
                    cudaEventCreate(&b1);
                    cudaEventRecord(b0, s);
                }
                nvtx_push(PICO_K_OTHER);
                e = relabel_back(rl, n, core_out, s, dev);
                nvtxRangePop();
                if (timing) cudaEventRecord(b1, s);
                if (!e) e = cudaStreamSynchronize(s);
                if (e) rc = cuda_fail(e, "relabel back");
                if (rc == PICO_OK && algo == PICO_ALGO_HISTOCORE && stats && stats->frontier_counts &&
                    (flags & PICO_F_STATS) && stats->frontier_counts_cap >= n) {
                    // the counts came back in compacted ids 0..n2-1: to original ids
                    std::vector<int> inv((size_t)rl.n2), tmp((size_t)rl.n2);
                    e = cudaMemcpy(inv.data(), rl.inv, sizeof(int) * (size_t)rl.n2, cudaMemcpyDeviceToHost);
                    if (e) rc = cuda_fail(e, "relabel back (frontier counts)");
                    else {
                        memcpy(tmp.data(), stats->frontier_counts, sizeof(int) * (size_t)rl.n2);
                        memset(stats->frontier_counts, 0, sizeof(int) * (size_t)n);
                        for (long long i = 0; i < rl.n2; i++) stats->frontier_counts[inv[(size_t)i]] = tmp[(size_t)i];
                    }
                }
                if (stats) stats->kernel_count += rl.launches + 1;
                if (timing && rc == PICO_OK) {
                    float t1 = 0, t2 = 0;
                    cudaEventElapsedTime(&t1, r0, r1);
                    cudaEventElapsedTime(&t2, b0, b1);
                    stats->kernel_ms[PICO_K_OTHER] += t1 + t2;
                    stats->kernel_launches[PICO_K_OTHER] += 1;
                }
                if (b0) { cudaEventDestroy(b0); cudaEventDestroy(b1); }
            }
            if (r0) { cudaEventDestroy(r0); cudaEventDestroy(r1); }
            e = cudaSuccess;
            if (!e && stats && algo != PICO_ALGO_PEELONE) {  // (PeelOne counts k_max itself)
                int *d = (int *)ws;  // Ctrl region is free again
                int km = 0;
                e = cudaMemsetAsync(d, 0, sizeof(int), s);
                if (!e) {
                    max_kernel<<<dev.sms * 4, 256, 0, s>>>(core_out, n, d);
                    e = cudaMemcpyAsync(&km, d, sizeof(int), cudaMemcpyDeviceToHost, s);
                }
                if (!e) e = cudaStreamSynchronize(s);
                if (e) rc = cuda_fail(e, "kmax");
                else { stats->kmax = km; stats->kernel_count += 1; }
            }
        }
    }
    if (own) {
        cudaError_t e2 = cudaFreeAsync(ws, s);
        if (!e2) e2 = cudaStreamSynchronize(s);
        if (e2 && rc == PICO_OK) rc = cuda_fail(e2, "workspace free");
    }
    return rc;
}

int pico_coreness(const int64_t *rowptr, const int32_t *colidx, int64_t n, int64_t m, int algo,
                  int32_t *core_out, pico_stream_t stream) {
    return pico_coreness_ex(rowptr, colidx, n, m, algo, core_out, stream, 0u, nullptr, 0, nullptr);
}

int pico_coreness_host(const int64_t *rowptr_h, const int32_t *colidx_h, int64_t n, int64_t m, int algo,
                       int32_t *core_out_h, pico_stream_t stream_, uint32_t flags, pico_stats_t *stats) {
    cudaStream_t s = (cudaStream_t)stream_;
    g_last_error.clear();
    reset_stats(stats);
    if (n < 0 || m < 0) return fail(PICO_EINVAL, "negative n or m");
    if (algo < PICO_ALGO_HISTOCORE || algo > PICO_ALGO_NBRCORE) return fail(PICO_EINVAL, "unknown algo %d", algo);
    if (n == 0) return PICO_OK;
    if (!rowptr_h || !core_out_h || (m > 0 && !colidx_h)) return fail(PICO_EINVAL, "NULL pointer argument");
    if (n >= (1ll << 31) - 1) return fail(PICO_ENOTSUP, "n too large");
    const size_t arcs = 2 * (size_t)m;
    void *d_rp = nullptr, *d_ci = nullptr, *d_core = nullptr;
    cudaError_t e = lib_malloc_async(&d_rp, sizeof(int64_t) * (size_t)(n + 1), s);
    if (!e) e = lib_malloc_async(&d_ci, sizeof(int32_t) * std::max<size_t>(arcs, 1), s);
    if (!e) e = lib_malloc_async(&d_core, sizeof(int32_t) * (size_t)n, s);
    int rc = PICO_OK;
    if (e) rc = cuda_fail(e, "device buffers");
    if (rc == PICO_OK) {
        e = cudaMemcpyAsync(d_rp, rowptr_h, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyHostToDevice, s);
        if (!e && arcs) e = cudaMemcpyAsync(d_ci, colidx_h, sizeof(int32_t) * arcs, cudaMemcpyHostToDevice, s);
        if (e) rc = cuda_fail(e, "host to device copy");
    }
    if (rc == PICO_OK) {
        std::string keep;
        rc = pico_coreness_ex((const int64_t *)d_rp, (const int32_t *)d_ci, n, m, algo, (int32_t *)d_core, stream_,
                              flags, nullptr, 0, stats);
        if (rc != PICO_OK) keep = g_last_error;
        if (rc == PICO_OK) {
            e = cudaMemcpyAsync(core_out_h, d_core, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToHost, s);
            if (e) rc = cuda_fail(e, "device to host copy");
        } else {
            g_last_error = keep;
        }
    }
    if (d_rp) cudaFreeAsync(d_rp, s);
    if (d_ci) cudaFreeAsync(d_ci, s);
    if (d_core) cudaFreeAsync(d_core, s);
    e = cudaStreamSynchronize(s);
    if (e && rc == PICO_OK) rc = cuda_fail(e, "synchronize");
    return rc;
}

// ---------------------------------------------------------------------------
// sharded HistoCore (include/pico_shard.h)
// ---------------------------------------------------------------------------
struct pico_shard_s {
    Shard *impl;
};

int pico_shard_create(const int64_t *rowptr_local, const int32_t *colidx_local, int64_t nloc, int64_t v_begin,
                      int64_t n_global, uint32_t flags, pico_stream_t stream, pico_shard_t *out) {
    g_last_error.clear();
    if (!out) return fail(PICO_EINVAL, "NULL output handle");
    *out = nullptr;
    if (nloc < 0 || v_begin < 0 || n_global <= 0 || v_begin + nloc > n_global)
        return fail(PICO_EINVAL, "bad shard range [%lld, %lld) of %lld", (long long)v_begin,
                    (long long)(v_begin + nloc), (long long)n_global);
    if (n_global >= (1ll << 31) - 1) return fail(PICO_ENOTSUP, "n_global needs 64-bit vertex ids");
    if (!rowptr_local) return fail(PICO_EINVAL, "NULL rowptr_local");
    DevInfo dev;
    cudaError_t e = dev_info(&dev);
    if (e) return cuda_fail(e, "device query");
    Shard *impl = nullptr;
    e = shard_create((const long long *)rowptr_local, colidx_local, nloc, v_begin, n_global, flags,
                     (cudaStream_t)stream, dev, &impl);
    if (e) return cuda_fail(e, "shard create");
    *out = new pico_shard_s{impl};
    return PICO_OK;
}

int pico_shard_degrees(pico_shard_t h, int32_t *deg_local) {
    g_last_error.clear();
    if (!h) return fail(PICO_EINVAL, "NULL shard");
    cudaError_t e = shard_degrees(h->impl, deg_local);
    return e ? cuda_fail(e, "shard degrees") : PICO_OK;
}

int pico_shard_init(pico_shard_t h, const int32_t *deg_global, int64_t *changed_local) {
    g_last_error.clear();
    if (!h || !deg_global || !changed_local) return fail(PICO_EINVAL, "NULL argument");
    long long c = 0;
    cudaError_t e = shard_init(h->impl, deg_global, &c);
    if (e) return cuda_fail(e, "shard init");
    *changed_local = c;
    return PICO_OK;
}

int pico_shard_pack(pico_shard_t h, int32_t *triples, int64_t cap, int64_t *count) {
    g_last_error.clear();
    if (!h || !count || (cap > 0 && !triples)) return fail(PICO_EINVAL, "NULL argument");
    long long c = 0;
    cudaError_t e = shard_pack(h->impl, triples, cap, &c);
    if (e == cudaErrorInvalidValue) return fail(PICO_EINVAL, "triple buffer too small (cap %lld)", (long long)cap);
    if (e) return cuda_fail(e, "shard pack");
    *count = c;
    return PICO_OK;
}

int pico_shard_apply(pico_shard_t h, const int32_t *triples, int64_t total, int64_t *changed_local) {
    g_last_error.clear();
    if (!h || total < 0 || (total > 0 && !triples)) return fail(PICO_EINVAL, "bad argument");
    long long c = 0;
    cudaError_t e = shard_apply(h->impl, triples, total, changed_local ? &c : nullptr);
    if (e) return cuda_fail(e, "shard apply");
    if (changed_local) *changed_local = c;
    return PICO_OK;
}

int pico_shard_result(pico_shard_t h, int32_t *core_local) {
    g_last_error.clear();
    if (!h) return fail(PICO_EINVAL, "NULL shard");
    cudaError_t e = shard_result(h->impl, core_local);
    return e ? cuda_fail(e, "shard result") : PICO_OK;
}

int pico_shard_destroy(pico_shard_t h) {
    g_last_error.clear();
    if (!h) return PICO_OK;
    cudaError_t e = shard_destroy(h->impl);
    delete h;
    return e ? cuda_fail(e, "shard destroy") : PICO_OK;
}

// sharded PeelOne steps
struct pico_peel_shard_s {
    PeelShard *impl;
};

static int peel_read(pico_peel_shard_t h, int64_t *count, int32_t *kmin) {
    long long c = 0;
    int km = 0;
    cudaError_t e = pshard_read(h->impl, &c, &km);
    if (e) return cuda_fail(e, "peel shard read");
    if (count) *count = c;
    if (kmin) *kmin = km;
    return PICO_OK;
}

int pico_peel_shard_create(const int64_t *rowptr_local, const int32_t *colidx_local, int64_t nloc,
                           int64_t v_begin, int64_t n_global, uint32_t flags, pico_stream_t stream,
                           pico_peel_shard_t *out, int32_t *kmin) {
    g_last_error.clear();
    if (!out) return fail(PICO_EINVAL, "NULL output handle");
    *out = nullptr;
    if (nloc < 0 || v_begin < 0 || n_global <= 0 || v_begin + nloc > n_global)
        return fail(PICO_EINVAL, "bad shard range [%lld, %lld) of %lld", (long long)v_begin,
                    (long long)(v_begin + nloc), (long long)n_global);
    if (n_global >= (1ll << 31) - 1) return fail(PICO_ENOTSUP, "n_global needs 64-bit vertex ids");
    if (!rowptr_local) return fail(PICO_EINVAL, "NULL rowptr_local");
    DevInfo dev;
    cudaError_t e = dev_info(&dev);
    if (e) return cuda_fail(e, "device query");
    PeelShard *impl = nullptr;
    e = pshard_create((const long long *)rowptr_local, colidx_local, nloc, v_begin, n_global, flags,
                      (cudaStream_t)stream, dev, &impl);
    if (e) return cuda_fail(e, "peel shard create");
    *out = new pico_peel_shard_s{impl};
    return peel_read(*out, nullptr, kmin);
}

int pico_peel_shard_scan(pico_peel_shard_t h, int32_t k, int32_t *frontier, int64_t cap, int64_t *count,
                         int32_t *kmin) {
    g_last_error.clear();
    if (!h || !count || !kmin || k < 1) return fail(PICO_EINVAL, "bad argument");
    if (cap < pshard_nloc(h->impl) || (cap > 0 && !frontier)) return fail(PICO_EINVAL, "frontier cap < nloc");
    cudaError_t e = pshard_scan(h->impl, k, frontier);
    if (e) return cuda_fail(e, "peel shard scan");
    return peel_read(h, count, kmin);
}

int pico_peel_shard_apply(pico_peel_shard_t h, const int32_t *frontier_all, int64_t total, int32_t *frontier,
                          int64_t cap, int64_t *count, int32_t *kmin) {
    g_last_error.clear();
    if (!h || !count || !kmin || total < 0 || (total > 0 && !frontier_all)) return fail(PICO_EINVAL, "bad argument");
    if (cap < pshard_nloc(h->impl) || (cap > 0 && !frontier)) return fail(PICO_EINVAL, "frontier cap < nloc");
    cudaError_t e = pshard_apply(h->impl, frontier_all, total, frontier);
    if (e) return cuda_fail(e, "peel shard apply");
    return peel_read(h, count, kmin);
}

int pico_peel_shard_result(pico_peel_shard_t h, int32_t *core_local) {
    g_last_error.clear();
    if (!h) return fail(PICO_EINVAL, "NULL shard");
    cudaError_t e = pshard_result(h->impl, core_local);
    return e ? cuda_fail(e, "peel shard result") : PICO_OK;
}

int pico_peel_shard_destroy(pico_peel_shard_t h) {
    g_last_error.clear();
    if (!h) return PICO_OK;
    cudaError_t e = pshard_destroy(h->impl);
    delete h;
    return e ? cuda_fail(e, "peel shard destroy") : PICO_OK;
}

}  // extern "C"

// ===========================================================================
// One-call sharded HistoCore with the exchange inside the library (NCCL,
// loaded with dlopen on first use; include/pico_shard.h).  The round loop is
// that of paper_2402_15253_b200/sharded.py: pack -> all-gather of the counts
// (global convergence test) -> all-gatherv of the triples (grouped
// broadcasts) -> apply.
// ===========================================================================
#include <dlfcn.h>
#include <nccl.h>  // types and enums only: the symbols come from dlopen

namespace {

struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi load_nccl() {
    NcclApi a;
    const char *env = getenv("PICO_NCCL_LIB");
    void *h = nullptr;
    for (const char *name : {env, "libnccl.so.2", "libnccl.so"}) {
        if (!name) continue;
        h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
    }
    if (!h) {
        a.err = std::string("cannot load libnccl.so.2: ") + dlerror();
        return a;
    }
#define PICO_SYM(f)                                                     \
    *(void **)(&a.f) = dlsym(h, "nccl" #f);                             \
    if (!a.f) {                                                         \
        a.err = "libnccl lacks nccl" #f;                                \
        return a;                                                       \
    }
    PICO_SYM(GetUniqueId)
    PICO_SYM(CommInitRank)
    PICO_SYM(CommDestroy)
    PICO_SYM(AllGather)
    PICO_SYM(Broadcast)
    PICO_SYM(GroupStart)
    PICO_SYM(GroupEnd)
    PICO_SYM(GetErrorString)
#undef PICO_SYM
    a.ok = true;
    return a;
}

NcclApi &nccl() {
    static NcclApi api = load_nccl();  // thread-safe initialisation
    return api;
}

}  // namespace

struct pico_comm_s {
    ncclComm_t c;
    int nranks, rank;
    // device-side exchange state (PICO_F_LSA_EXCHANGE): the symmetric window
    // and device communicator, created at the first such call and kept for
    // the communicator's lifetime (registration is collective and costly);
    // recreated -- on every rank alike -- when a call needs a larger capacity
    pico::LsaX *lsa = nullptr;
    long long lsa_cap = 0;
};

static int nccl_fail(ncclResult_t r, const char *where) {
    return fail(PICO_ENCCL, "%s: %s", where, nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
}

// Sharded PeelOne level loop over NCCL (pico_peel_shard_* semantics): per
// sub-round one all-gather of the (|F|, kmin) pairs straight from device
// memory, one host read, and a grouped-broadcast all-gatherv of F.
static int peel_rounds(pico_comm_t comm, PeelShard *ps, long long nloc, int *front, int *&all, size_t &all_cap,
                       long long *cnt, int32_t *core_out_local, pico_stats_t *stats, cudaStream_t s) {
    NcclApi &N = nccl();
    const int P = comm->nranks, me = comm->rank;
    std::vector<long long> hp(2 * P), off(P + 1, 0);
    const long long *odev = pshard_out(ps);
    cudaError_t e;
    ncclResult_t nr, ne;
    long long levels = 0, subrounds = 0;
    int kmax = 0;
    // (count, kmin) of every rank -> host; returns the global total and min
    auto gather = [&](long long *total, int *kmin) -> int {
        if ((nr = N.AllGather(odev, cnt + 2, 2, ncclInt64, comm->c, s)) != ncclSuccess)
            return nccl_fail(nr, "allgather counts");
        if ((e = cudaMemcpyAsync(hp.data(), cnt + 2, sizeof(long long) * 2 * P, cudaMemcpyDeviceToHost, s)) ||
            (e = cudaStreamSynchronize(s)))
            return cuda_fail(e, "counts");
        long long t = 0, km = INT_MAX;
        for (int r = 0; r < P; r++) {
            off[r] = t;
            t += hp[2 * r];
            km = std::min(km, hp[2 * r + 1]);
        }
        off[P] = t;
        *total = t;
        *kmin = (int)km;
        return PICO_OK;
    };
    long long total = 0;
    int kmin = INT_MAX, rc;
    if ((rc = gather(&total, &kmin)) != PICO_OK) return rc;
    int k = 0;
    while (kmin != INT_MAX) {
        k = std::max(k + 1, kmin);
        if ((e = pshard_scan(ps, k, front))) return cuda_fail(e, "peel scan");
        long long processed = 0;
        for (;;) {
            if ((rc = gather(&total, &kmin)) != PICO_OK) return rc;
            if (total == 0) break;  // the level is done on every rank
            processed += total;
            subrounds++;
            if ((size_t)total > all_cap) {
                if (all) cudaFreeAsync(all, s);
                all_cap = (size_t)total + (size_t)total / 4;
                if ((e = lib_malloc_async(&all, sizeof(int) * all_cap, s))) {
                    all = nullptr;
                    return cuda_fail(e, "alloc");
                }
            }
            if ((nr = N.GroupStart()) != ncclSuccess) return nccl_fail(nr, "group");
            for (int r = 0; r < P && nr == ncclSuccess; r++) {
                long long c = off[r + 1] - off[r];
                if (c > 0)
                    nr = N.Broadcast(r == me ? (const void *)front : (const void *)(all + off[r]), all + off[r],
                                     (size_t)c, ncclInt32, r, comm->c, s);
            }
            ne = N.GroupEnd();
            if (nr != ncclSuccess || ne != ncclSuccess) return nccl_fail(nr != ncclSuccess ? nr : ne, "allgatherv F");
            if ((e = pshard_apply(ps, all, total, front))) return cuda_fail(e, "peel apply");
        }
        if (processed) {
            if (stats && stats->frontier_sizes && levels < stats->frontier_sizes_cap)
                stats->frontier_sizes[levels] = processed;
            levels++;
            kmax = k;
        }
    }
    if (stats) {
        stats->levels = levels;
        stats->subrounds = subrounds;
        stats->kmax = kmax;
    }
    if (nloc > 0 && (e = pshard_result(ps, core_out_local))) return cuda_fail(e, "shard result");
    return PICO_OK;
}

extern "C" {

int pico_comm_unique_id(uint8_t id[128]) {
    g_last_error.clear();
    if (!id) return fail(PICO_EINVAL, "NULL id");
    if (!nccl().ok) return fail(PICO_ENCCL, "%s", nccl().err.c_str());
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    ncclResult_t r = nccl().GetUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(id, &u, 128);
    return PICO_OK;
}

int pico_comm_init(int nranks, int rank, const uint8_t id[128], pico_comm_t *comm) {
    g_last_error.clear();
    if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(PICO_EINVAL, "bad argument");
    *comm = nullptr;
    if (!nccl().ok) return fail(PICO_ENCCL, "%s", nccl().err.c_str());
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclComm_t c;
    ncclResult_t r = nccl().CommInitRank(&c, nranks, u, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    *comm = new pico_comm_s{c, nranks, rank};
    return PICO_OK;
}

int pico_comm_size(pico_comm_t comm, int *nranks, int *rank) {
    g_last_error.clear();
    if (!comm) return fail(PICO_EINVAL, "NULL comm");
    if (nranks) *nranks = comm->nranks;
    if (rank) *rank = comm->rank;
    return PICO_OK;
}

int pico_comm_destroy(pico_comm_t comm) {
    g_last_error.clear();
    if (!comm) return PICO_OK;
    if (comm->lsa) pico::lsa_destroy(comm->lsa);  // before the communicator it was registered with
    ncclResult_t r = nccl().CommDestroy(comm->c);
    delete comm;
    return r == ncclSuccess ? PICO_OK : nccl_fail(r, "ncclCommDestroy");
}

// HistoCore rounds with the device-side exchange (PICO_F_LSA_EXCHANGE,
// lsa_exchange.cu): pack into this rank's half of the symmetric window, LSA
// counts + barrier + peer copies, apply with the device total; rounds are
// enqueued PICO_LSA_BATCH at a time and the host reads the batch's global
// counts once (the first empty round is the convergence; later rounds of the
// batch are no-ops on every rank, so the barriers stay matched).
static int lsa_rounds(pico_comm_t comm, Shard *sh, const std::vector<long long> &hm, long long n_global,
                      long long arcs_global, pico_stats_t *stats, cudaStream_t s, const DevInfo &dev) {
    const int P = comm->nranks, me = comm->rank;
    long long cap = 1;
    for (int r = 0; r < P; r++) cap = std::max(cap, hm[3 * r + 1] - hm[3 * r]);
    std::string msg;
    cudaError_t e = cudaSuccess;
    if (!comm->lsa || comm->lsa_cap < cap || lsa_words(comm->lsa) != 3) {  // the same decision on every rank
        if (comm->lsa) {
            if ((e = cudaStreamSynchronize(s))) return cuda_fail(e, "LSA exchange setup");
            lsa_destroy(comm->lsa);
            comm->lsa = nullptr;
        }
        e = lsa_create((void *)comm->c, P, me, cap, 3, &comm->lsa, &msg);
        if (e == cudaErrorNotSupported) return fail(PICO_ENOTSUP, "LSA exchange unavailable: %s", msg.c_str());
        if (e) return msg.empty() ? cuda_fail(e, "LSA exchange setup") : fail(PICO_ENCCL, "%s", msg.c_str());
        comm->lsa_cap = cap;
    }
    LsaX *lx = comm->lsa;
    int batch = 4;
    if (const char *b = getenv("PICO_LSA_BATCH")) batch = std::max(1, std::min(64, atoi(b)));
    int *all = nullptr;
    long long *tot = nullptr;
    int rc = PICO_OK;
    std::vector<long long> htot(batch);
    do {
        if ((e = lib_malloc_async(&all, sizeof(int) * 3 * (size_t)std::max(n_global, 1ll), s)) ||
            (e = lib_malloc_async(&tot, sizeof(long long) * (size_t)batch, s))) { rc = cuda_fail(e, "alloc"); break; }
        long long rounds = 0;
        bool done = false;
        while (!done) {
            for (int b = 0; b < batch && rc == PICO_OK; b++) {
                const int par = (int)((rounds + b) & 1);
                const unsigned long long *cdev = nullptr;
                if ((e = shard_pack_dev(sh, lsa_send_buffer(lx, par), &cdev)) ||
                    (e = lsa_exchange(lx, par, cdev, all, tot + b, dev.sms * 8, s)) ||
                    (e = shard_apply(sh, all, 0, nullptr, lsa_total(lx))))
                    rc = cuda_fail(e, "LSA round");
            }
            if (rc != PICO_OK) break;
            if ((e = cudaMemcpyAsync(htot.data(), tot, sizeof(long long) * (size_t)batch, cudaMemcpyDeviceToHost, s)) ||
                (e = cudaStreamSynchronize(s))) { rc = cuda_fail(e, "LSA counts"); break; }
            for (int b = 0; b < batch; b++) {
                if (htot[b] == 0) { done = true; break; }
                if (stats && stats->frontier_sizes && rounds < stats->frontier_sizes_cap)
                    stats->frontier_sizes[rounds] = htot[b];
                rounds++;
            }
            // every valid round lowers the sum of the estimates: l2 <= 2m (see the single-GPU guard)
            if (!done && rounds > arcs_global + 2) { rc = fail(PICO_EGRAPH, "no convergence"); break; }
        }
        if (rc == PICO_OK && stats) stats->rounds = rounds;
    } while (false);
    if (all) cudaFreeAsync(all, s);
    if (tot) cudaFreeAsync(tot, s);
    cudaError_t es = cudaStreamSynchronize(s);
    if (rc == PICO_OK && es) rc = cuda_fail(es, "LSA cleanup");
    return rc;
}

// sharded PeelOne with the level loop on the device and the exchange over
// NCCL's device API (PICO_F_LSA_EXCHANGE; shard_peel.cu pshard_run_lsa)
static int peel_rounds_lsa(pico_comm_t comm, PeelShard *ps, const std::vector<long long> &hm, long long n_global,
                           int32_t *core_out_local, long long nloc, pico_stats_t *stats, cudaStream_t s) {
    const int P = comm->nranks, me = comm->rank;
    long long cap = 1;
    for (int r = 0; r < P; r++) cap = std::max(cap, hm[3 * r + 1] - hm[3 * r]);
    std::string msg;
    cudaError_t e = cudaSuccess;
    if (!comm->lsa || comm->lsa_cap < cap || lsa_words(comm->lsa) != 1) {  // the same decision on every rank
        if (comm->lsa) {
            if ((e = cudaStreamSynchronize(s))) return cuda_fail(e, "LSA exchange setup");
            lsa_destroy(comm->lsa);
            comm->lsa = nullptr;
        }
        e = lsa_create((void *)comm->c, P, me, cap, 1, &comm->lsa, &msg);
        if (e == cudaErrorNotSupported) return fail(PICO_ENOTSUP, "LSA exchange unavailable: %s", msg.c_str());
        if (e) return msg.empty() ? cuda_fail(e, "LSA exchange setup") : fail(PICO_ENCCL, "%s", msg.c_str());
        comm->lsa_cap = cap;
    }
    long long levels = 0, subrounds = 0;
    int kmax = 0;
    std::vector<long long> lv;
    long long lvcap = (stats && stats->frontier_sizes) ? stats->frontier_sizes_cap : 0;
    lv.resize((size_t)std::max(lvcap, 1ll));
    e = pshard_run_lsa(ps, comm->lsa, n_global, &levels, &subrounds, &kmax, lvcap ? lv.data() : nullptr, lvcap, &msg);
    if (e) return msg.empty() ? cuda_fail(e, "sharded PeelOne (LSA)") : fail(PICO_EGRAPH, "%s", msg.c_str());
    if (stats) {
        stats->levels = levels;
        stats->subrounds = subrounds;
        stats->kmax = kmax;
        for (long long i = 0; i < std::min(levels, lvcap); i++) stats->frontier_sizes[i] = lv[(size_t)i];
    }
    if (nloc > 0 && (e = pshard_result(ps, core_out_local))) return cuda_fail(e, "shard result");
    return PICO_OK;
}

int pico_coreness_sharded_ex(pico_comm_t comm, const int64_t *rowptr_local, const int32_t *colidx_local,
                             int64_t n_global, int64_t m_global, int64_t v_begin, int64_t v_end, int algo,
                             int32_t *core_out_local, pico_stream_t stream, uint32_t flags,
                             pico_stats_t *stats) {
    g_last_error.clear();
    reset_stats(stats);
    if (!comm) return fail(PICO_EINVAL, "NULL comm");
    if (algo != PICO_ALGO_HISTOCORE && algo != PICO_ALGO_PEELONE)
        return fail(PICO_EINVAL, "algo %d is not sharded", algo);
    if (v_begin < 0 || v_end < v_begin || v_end > n_global || n_global <= 0 || m_global < 0)
        return fail(PICO_EINVAL, "bad range [%lld, %lld) of %lld", (long long)v_begin, (long long)v_end,
                    (long long)n_global);
    if (n_global >= (1ll << 31) - 1) return fail(PICO_ENOTSUP, "n_global needs 64-bit vertex ids");
    if (!rowptr_local || (v_end > v_begin && !core_out_local)) return fail(PICO_EINVAL, "NULL pointer");
    const long long nloc = v_end - v_begin;
    const int P = comm->nranks, me = comm->rank;
    cudaStream_t s = (cudaStream_t)stream;
    NcclApi &N = nccl();
    DevInfo dev;
    cudaError_t e = dev_info(&dev);
    if (e) return cuda_fail(e, "device query");

    Shard *sh = nullptr;
    PeelShard *ps = nullptr;
    const bool peel = algo == PICO_ALGO_PEELONE;
    if (peel)
        e = pshard_create((const long long *)rowptr_local, colidx_local, nloc, v_begin, n_global, flags, s, dev, &ps);
    else
        e = shard_create((const long long *)rowptr_local, colidx_local, nloc, v_begin, n_global, flags, s, dev, &sh);
    if (e) return cuda_fail(e, "shard create");
    // device scratch: meta [3 + 3P] int64, counts [1 + P] int64, degrees, triples
    long long *meta = nullptr, *cnt = nullptr;
    int *deg_g = nullptr, *trip = nullptr, *all = nullptr;
    size_t all_cap = 0;
    int rc = PICO_OK;
    ncclResult_t nr;
    std::vector<long long> hm(3 * P), hc(P);
    std::vector<long long> off(P + 1, 0);
    auto bail_cuda = [&](cudaError_t err, const char *w) { rc = cuda_fail(err, w); };
    auto bail_nccl = [&](ncclResult_t r, const char *w) { rc = nccl_fail(r, w); };
    do {
        if ((e = lib_malloc_async(&meta, sizeof(long long) * (3 + 3 * P), s))) { bail_cuda(e, "alloc"); break; }
        if ((e = lib_malloc_async(&cnt, sizeof(long long) * (2 + 2 * P), s))) { bail_cuda(e, "alloc"); break; }
        if ((e = lib_malloc_async(&deg_g, sizeof(int) * (size_t)n_global, s))) { bail_cuda(e, "alloc"); break; }
        if ((e = lib_malloc_async(&trip, sizeof(int) * 3 * (size_t)std::max(nloc, 1ll), s))) {
            bail_cuda(e, "alloc");
            break;
        }
        // every rank's (v_begin, v_end, local arcs): the ranges must tile [0, n_global) in rank order
        long long mine[3] = {v_begin, v_end, 0};
        if ((e = cudaMemcpyAsync(&mine[2], rowptr_local + nloc, sizeof(long long), cudaMemcpyDeviceToHost, s)) ||
            (e = cudaStreamSynchronize(s))) { bail_cuda(e, "local arcs"); break; }
        if ((e = cudaMemcpyAsync(meta, mine, sizeof(mine), cudaMemcpyHostToDevice, s))) { bail_cuda(e, "meta"); break; }
        if ((nr = N.AllGather(meta, meta + 3, 3, ncclInt64, comm->c, s)) != ncclSuccess) { bail_nccl(nr, "allgather ranges"); break; }
        if ((e = cudaMemcpyAsync(hm.data(), meta + 3, sizeof(long long) * 3 * P, cudaMemcpyDeviceToHost, s)) ||
            (e = cudaStreamSynchronize(s))) { bail_cuda(e, "ranges"); break; }
        long long arcs = 0;
        bool tiled = hm[0] == 0 && hm[3 * (P - 1) + 1] == n_global;
        for (int r = 0; r < P; r++) {
            arcs += hm[3 * r + 2];
            if (r > 0 && hm[3 * r] != hm[3 * (r - 1) + 1]) tiled = false;
        }
        if (!tiled) { rc = fail(PICO_EINVAL, "rank ranges do not tile [0, n_global) in rank order"); break; }
        if (arcs != 2 * m_global) { rc = fail(PICO_EINVAL, "local arcs sum to %lld, not 2m = %lld", arcs, 2 * (long long)m_global); break; }
        if (peel && (flags & PICO_F_LSA_EXCHANGE)) {
            rc = peel_rounds_lsa(comm, ps, hm, n_global, core_out_local, nloc, stats, s);
            break;
        }
        if (peel) {
            rc = peel_rounds(comm, ps, nloc, trip, all, all_cap, cnt, core_out_local, stats, s);
            break;
        }
        // degrees: all-gatherv into deg_global
        if ((e = shard_degrees(sh, deg_g + v_begin))) { bail_cuda(e, "shard degrees"); break; }
        if ((nr = N.GroupStart()) != ncclSuccess) { bail_nccl(nr, "group"); break; }
        for (int r = 0; r < P && nr == ncclSuccess; r++) {
            long long c = hm[3 * r + 1] - hm[3 * r];
            if (c > 0) nr = N.Broadcast(deg_g + hm[3 * r], deg_g + hm[3 * r], (size_t)c, ncclInt32, r, comm->c, s);
        }
        ncclResult_t ne = N.GroupEnd();
        if (nr != ncclSuccess || ne != ncclSuccess) { bail_nccl(nr != ncclSuccess ? nr : ne, "allgatherv degrees"); break; }
        long long changed = 0;
        if ((e = shard_init(sh, deg_g, &changed))) { bail_cuda(e, "shard init"); break; }
        if (flags & PICO_F_LSA_EXCHANGE) {
            rc = lsa_rounds(comm, sh, hm, n_global, 2 * (long long)m_global, stats, s, dev);
            if (rc != PICO_OK) break;
            if (nloc > 0 && (e = shard_result(sh, core_out_local))) { bail_cuda(e, "shard result"); break; }
            break;
        }
        // rounds
        long long rounds = 0;
        for (;;) {
            // pack, then all-gather the counts straight from device memory: one host
            // synchronisation per round (the grouped broadcasts need host counts)
            const unsigned long long *cdev = nullptr;
            if ((e = shard_pack_dev(sh, trip, &cdev))) { bail_cuda(e, "shard pack"); break; }
            if ((nr = N.AllGather(cdev, cnt + 1, 1, ncclInt64, comm->c, s)) != ncclSuccess) { bail_nccl(nr, "allgather counts"); break; }
            if ((e = cudaMemcpyAsync(hc.data(), cnt + 1, sizeof(long long) * P, cudaMemcpyDeviceToHost, s)) ||
                (e = cudaStreamSynchronize(s))) { bail_cuda(e, "counts"); break; }
            for (int r = 0; r < P; r++) off[r + 1] = off[r] + hc[r];
            const long long total = off[P];
            if (total == 0) break;  // global convergence
            if (stats && stats->frontier_sizes && rounds < stats->frontier_sizes_cap)
                stats->frontier_sizes[rounds] = total;
            rounds++;
            if ((size_t)(3 * total) > all_cap) {
                if (all) cudaFreeAsync(all, s);
                all_cap = (size_t)(3 * total) + (size_t)(3 * total) / 4;
                if ((e = lib_malloc_async(&all, sizeof(int) * all_cap, s))) { all = nullptr; bail_cuda(e, "alloc"); break; }
            }
            if ((nr = N.GroupStart()) != ncclSuccess) { bail_nccl(nr, "group"); break; }
            for (int r = 0; r < P && nr == ncclSuccess; r++)
                if (hc[r] > 0)
                    nr = N.Broadcast(r == me ? (const void *)trip : (const void *)(all + 3 * off[r]), all + 3 * off[r],
                                     (size_t)(3 * hc[r]), ncclInt32, r, comm->c, s);
            ne = N.GroupEnd();
            if (nr != ncclSuccess || ne != ncclSuccess) { bail_nccl(nr != ncclSuccess ? nr : ne, "allgatherv triples"); break; }
            if ((e = shard_apply(sh, all, total, nullptr))) { bail_cuda(e, "shard apply"); break; }
        }
        if (rc != PICO_OK) break;
        if (stats) stats->rounds = rounds;
        if (nloc > 0 && (e = shard_result(sh, core_out_local))) { bail_cuda(e, "shard result"); break; }
    } while (false);
    cudaError_t ed = peel ? pshard_destroy(ps) : shard_destroy(sh);
    for (void *ptr : {(void *)meta, (void *)cnt, (void *)deg_g, (void *)trip, (void *)all})
        if (ptr) cudaFreeAsync(ptr, s);
    cudaError_t es = cudaStreamSynchronize(s);
    if (rc == PICO_OK && (ed || es)) rc = cuda_fail(ed ? ed : es, "sharded cleanup");
    return rc;
}

int pico_coreness_sharded(pico_comm_t comm, const int64_t *rowptr_local, const int32_t *colidx_local,
                          int64_t n_global, int64_t m_global, int64_t v_begin, int64_t v_end, int algo,
                          int32_t *core_out_local, pico_stream_t stream) {
    return pico_coreness_sharded_ex(comm, rowptr_local, colidx_local, n_global, m_global, v_begin, v_end, algo,
                                    core_out_local, stream, 0, nullptr);
}

}  // extern "C"

// ===========================================================================
// decremental HistoCore (include/pico_dyn.h)
// ===========================================================================
struct pico_dyn_s {
    Dyn *impl;
};

extern "C" {

int pico_dyn_create(const int64_t *rowptr, const int32_t *colidx, int64_t n, int64_t m, uint32_t flags,
                    pico_stream_t stream, pico_stats_t *stats, pico_dyn_t *out) {
    g_last_error.clear();
    reset_stats(stats);
    if (!out) return fail(PICO_EINVAL, "NULL output handle");
    *out = nullptr;
    if (n <= 0 || m < 0) return fail(PICO_EINVAL, "bad n (%lld) or m (%lld)", (long long)n, (long long)m);
    if (n >= (1ll << 31) - 1) return fail(PICO_ENOTSUP, "n = %lld needs 64-bit vertex ids", (long long)n);
    if (!rowptr || (m > 0 && !colidx)) return fail(PICO_EINVAL, "NULL pointer argument");
    DevInfo dev;
    cudaError_t e = dev_info(&dev);
    if (e) return cuda_fail(e, "device query");
    if (!dev.coop) return fail(PICO_ENOTSUP, "cooperative launch unavailable");
    Dyn *impl = nullptr;
    e = dyn_create((const long long *)rowptr, colidx, n, 2 * (long long)m, flags, (cudaStream_t)stream, dev, stats,
                   &impl);
    if (e) return cuda_fail(e, "dyn create");
    *out = new pico_dyn_s{impl};
    return PICO_OK;
}

int pico_dyn_coreness(pico_dyn_t h, int32_t *core_out) {
    g_last_error.clear();
    if (!h || !core_out) return fail(PICO_EINVAL, "NULL argument");
    cudaError_t e = dyn_core(h->impl, core_out);
    return e ? cuda_fail(e, "dyn coreness") : PICO_OK;
}

int pico_dyn_delete_edges(pico_dyn_t h, const int32_t *src, const int32_t *dst, int64_t k, pico_stats_t *stats) {
    g_last_error.clear();
    reset_stats(stats);
    if (!h || k < 0 || (k > 0 && (!src || !dst))) return fail(PICO_EINVAL, "bad argument");
    cudaError_t e = dyn_delete(h->impl, src, dst, k, stats);
    if (e == cudaErrorInvalidValue)
        return fail(PICO_EINVAL, "a deleted edge is not an edge of the current graph (or a self loop / bad id)");
    return e ? cuda_fail(e, "dyn delete") : PICO_OK;
}

int pico_dyn_insert_edges(pico_dyn_t h, const int32_t *src, const int32_t *dst, int64_t k, pico_stats_t *stats) {
    g_last_error.clear();
    reset_stats(stats);
    if (!h || k < 0 || (k > 0 && (!src || !dst))) return fail(PICO_EINVAL, "bad argument");
    cudaError_t e = dyn_insert(h->impl, src, dst, k, stats);
    if (e == cudaErrorInvalidValue)
        return fail(PICO_EINVAL, "an inserted edge is already in the graph (or a self loop / bad id)");
    return e ? cuda_fail(e, "dyn insert") : PICO_OK;
}

int pico_dyn_destroy(pico_dyn_t h) {
    g_last_error.clear();
    if (!h) return PICO_OK;
    cudaError_t e = dyn_destroy(h->impl);
    delete h;
    return e ? cuda_fail(e, "dyn destroy") : PICO_OK;
}

}  // extern "C"

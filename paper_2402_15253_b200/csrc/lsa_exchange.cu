// lsa_exchange.cu -- device-side exchange of the sharded HistoCore round over
// NCCL's device API (symmetric memory windows, load/store-accessible peers,
// LSA barriers; NCCL >= 2.28).  SURVEY 8(e) / DESIGN.md section 8.
//
// The host-driven exchange of pico_coreness_sharded (capi.cu) needs the
// per-rank triple counts on the host every round (an ncclAllGather of the
// counts, a device->host copy and a stream synchronisation, then one grouped
// ncclBroadcast per rank).  Here a round's exchange is two kernels on the
// caller's stream and no host round trip:
//   counts: each rank stores its |C_t| (the triples its pack kernel wrote into
//           its own window) into slot [me] of every peer's count row, then one
//           LSA barrier (release/acquire) -- after it every rank holds all
//           counts in its own window and computes the exclusive offsets and the
//           global total on the device (total 0 = global convergence)
//   copy:   every rank loads the peers' triples straight out of their windows
//           (NVLink peer loads through the LSA pointers) into its own receive
//           buffer, in rank order -- the same buffer the grouped broadcasts
//           fill, so the apply step (shard_apply) is unchanged; it reads the
//           total from device memory
// Window layout (identical on every rank, symmetric): count rows [2][P] int64
// (parity t & 1), then triple buffers [2][3 * cap] int32.  Double buffering by
// parity makes one barrier per round enough: a rank rewrites the parity-p
// buffers only in round t + 2, after the barrier of round t + 1, which every
// peer reaches only once its round-t copy has finished (stream order).
//
// The host side (window registration, the device communicator) is resolved
// with dlsym from the libnccl.so.2 already loaded by the process; when it lacks
// the device API the caller falls back to the host exchange (lsa_create
// returns an error).
#include <dlfcn.h>
#include <cstdio>
#include <climits>
#include <cstring>
#include <string>

#include <cuda_runtime.h>

#if PICO_HAVE_NCCL_DEVICE
#include <nccl.h>
#include <nccl_device.h>
#endif

#include "lsa_exchange.h"

namespace pico {

#if PICO_HAVE_NCCL_DEVICE

struct NcclDevApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*MemAlloc)(void **, size_t) = nullptr;
    ncclResult_t (*MemFree)(void *) = nullptr;
    ncclResult_t (*WindowRegister)(ncclComm_t, void *, size_t, ncclWindow_t *, int) = nullptr;
    ncclResult_t (*WindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
    ncclResult_t (*DevCommCreate)(ncclComm_t, ncclDevCommRequirements_t const *, ncclDevComm_t *) = nullptr;
    ncclResult_t (*DevCommDestroy)(ncclComm_t, ncclDevComm_t const *) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclDevApi load_dev_api() {
    NcclDevApi a;
    void *h = nullptr;
    const char *env = getenv("PICO_NCCL_LIB");
    for (const char *name : {env, "libnccl.so.2", "libnccl.so"}) {
        if (!name) continue;
        if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
    }
    if (!h) {
        a.err = std::string("cannot load libnccl.so.2: ") + dlerror();
        return a;
    }
#define PICO_LSA_SYM(f, name)                                            \
    *(void **)(&a.f) = dlsym(h, name);                                   \
    if (!a.f) {                                                          \
        a.err = std::string("libnccl lacks ") + name + " (NCCL < 2.28)"; \
        return a;                                                        \
    }
    PICO_LSA_SYM(MemAlloc, "ncclMemAlloc")
    PICO_LSA_SYM(MemFree, "ncclMemFree")
    PICO_LSA_SYM(WindowRegister, "ncclCommWindowRegister")
    PICO_LSA_SYM(WindowDeregister, "ncclCommWindowDeregister")
    PICO_LSA_SYM(DevCommCreate, "ncclDevCommCreate")
    PICO_LSA_SYM(DevCommDestroy, "ncclDevCommDestroy")
    PICO_LSA_SYM(GetErrorString, "ncclGetErrorString")
#undef PICO_LSA_SYM
    a.ok = true;
    return a;
}

static NcclDevApi &dev_api() {
    static NcclDevApi api = load_dev_api();
    return api;
}

struct LsaX {
    ncclComm_t comm = nullptr;
    int P = 0, me = 0;
    long long cap = 0;           // items per rank and parity
    int words = 3;               // int32 words per item (3: HistoCore triples, 1: PeelOne ids)
    void *buf = nullptr;         // the symmetric window's memory (ncclMemAlloc)
    size_t bytes = 0;
    ncclWindow_t win = nullptr;
    ncclDevComm dc{};
    bool win_ok = false, dc_ok = false;
    unsigned long long *off = nullptr;  // device [P + 1]: exclusive offsets, off[P] = total
};

static size_t a4k(size_t x) { return (x + 4095) & ~size_t(4095); }
// count rows: [parity][rank] (count, aux) int64 pairs
static size_t cnt_off(const LsaX *x, int parity) { return 2 * sizeof(long long) * (size_t)parity * x->P; }
static size_t trip_base(const LsaX *x) { return a4k(2 * sizeof(long long) * 2 * (size_t)x->P); }
static size_t trip_off(const LsaX *x, int parity) {
    return trip_base(x) + sizeof(int) * (size_t)x->words * (size_t)x->cap * (size_t)parity;
}

// counts of an exchange: my (count, aux) pair into every peer's row, one LSA
// barrier, then the item offsets, the global total and the minimum aux (one
// warp).  mine: the count (aux: mine[1] when has_aux, e.g. PeelOne's bound
// of the next level, reduced by min)
__global__ void __launch_bounds__(32) lsa_counts_kernel(ncclDevComm dc, ncclWindow_t win, size_t row_off, int P, int me,
                                                        const unsigned long long *mine, int has_aux,
                                                        unsigned long long *off, long long *tot_out,
                                                        long long *min_out) {
    const long long c = (long long)mine[0], x = has_aux ? (long long)mine[1] : 0;
    for (int r = threadIdx.x; r < P; r += 32) {
        volatile long long *dst = reinterpret_cast<volatile long long *>(
            (char *)ncclGetLsaPointer(win, row_off + 2 * sizeof(long long) * (size_t)me, r));
        dst[0] = c;
        dst[1] = x;
    }
    {
        ncclLsaBarrierSession<ncclCoopWarp> bar(ncclCoopWarp(), dc, ncclTeamTagLsa(), 0);
        bar.sync(ncclCoopWarp(), cuda::memory_order_acq_rel);
    }
    if (threadIdx.x == 0) {
        const volatile long long *row =
            reinterpret_cast<const volatile long long *>((char *)ncclGetLocalPointer(win, row_off));
        unsigned long long s = 0;
        long long mn = LLONG_MAX;
        for (int r = 0; r < P; r++) {
            off[r] = s;
            s += (unsigned long long)row[2 * r];
            mn = row[2 * r + 1] < mn ? row[2 * r + 1] : mn;
        }
        off[P] = s;
        if (tot_out) *tot_out = (long long)s;
        if (min_out) *min_out = mn;
    }
}

// copy of an exchange: all[w off[r] + j] = rank r's word j (peer loads)
__global__ void __launch_bounds__(256) lsa_copy_kernel(ncclWindow_t win, size_t trip_off, int P, int w,
                                                       const unsigned long long *off, int *all) {
    __shared__ unsigned long long s_off[65];
    __shared__ const int *s_src[64];
    for (int r = threadIdx.x; r <= P && r <= 64; r += blockDim.x) {
        s_off[r] = (unsigned long long)w * off[r];
        if (r < P) s_src[r] = (const int *)ncclGetLsaPointer(win, trip_off, r);
    }
    __syncthreads();
    const unsigned long long tot = s_off[min(P, 64)];
    const unsigned long long nt = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += nt) {
        int lo = 0, hi = P - 1;  // the rank whose range holds word i
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_off[mid] <= i) lo = mid; else hi = mid - 1;
        }
        all[i] = __ldcv(s_src[lo] + (i - s_off[lo]));
    }
}

static cudaError_t nccl_err(ncclResult_t r, const char *where, std::string *msg) {
    if (msg) *msg = std::string(where) + ": " + (dev_api().GetErrorString ? dev_api().GetErrorString(r) : "NCCL error");
    return cudaErrorUnknown;
}

cudaError_t lsa_create(void *comm, int P, int me, long long cap, int words, LsaX **out, std::string *msg) {
    *out = nullptr;
    NcclDevApi &N = dev_api();
    if (!N.ok) {
        if (msg) *msg = N.err;
        return cudaErrorNotSupported;
    }
    if (P > 64) {
        if (msg) *msg = "LSA exchange supports at most 64 ranks";
        return cudaErrorNotSupported;
    }
    LsaX *x = new LsaX;
    x->comm = (ncclComm_t)comm;
    x->P = P;
    x->me = me;
    x->cap = cap > 0 ? cap : 1;
    x->words = words;
    x->bytes = a4k(trip_off(x, 2));
    ncclResult_t r;
    cudaError_t e;
    auto bail = [&](cudaError_t err) {
        lsa_destroy(x);
        return err;
    };
    if ((r = N.MemAlloc(&x->buf, x->bytes)) != ncclSuccess) return bail(nccl_err(r, "ncclMemAlloc", msg));
    if ((e = cudaMemset(x->buf, 0, x->bytes))) return bail(e);
    if ((r = N.WindowRegister(x->comm, x->buf, x->bytes, &x->win, NCCL_WIN_COLL_SYMMETRIC)) != ncclSuccess)
        return bail(nccl_err(r, "ncclCommWindowRegister", msg));
    x->win_ok = true;
    ncclDevCommRequirements_t req;
    memset(&req, 0, sizeof(req));
    req.lsaBarrierCount = 1;
    if ((r = N.DevCommCreate(x->comm, &req, &x->dc)) != ncclSuccess) return bail(nccl_err(r, "ncclDevCommCreate", msg));
    x->dc_ok = true;
    if (x->dc.lsaSize != P || x->dc.lsaRank != me) {
        if (msg) *msg = "the LSA team is not the whole communicator (ranks on several nodes)";
        return bail(cudaErrorNotSupported);
    }
    if ((e = cudaMalloc(&x->off, sizeof(unsigned long long) * (size_t)(P + 1)))) return bail(e);
    *out = x;
    return cudaSuccess;
}

int *lsa_send_buffer(LsaX *x, int parity) { return (int *)((char *)x->buf + trip_off(x, parity)); }
long long lsa_capacity(const LsaX *x) { return x->cap; }
int lsa_words(const LsaX *x) { return x->words; }
const unsigned long long *lsa_total(const LsaX *x) { return x->off + x->P; }

cudaError_t lsa_exchange(LsaX *x, int parity, const unsigned long long *mine, int *all, long long *tot_out,
                         int copy_blocks, cudaStream_t s, int has_aux, long long *min_out) {
    lsa_counts_kernel<<<1, 32, 0, s>>>(x->dc, x->win, cnt_off(x, parity), x->P, x->me, mine, has_aux, x->off,
                                       tot_out, min_out);
    lsa_copy_kernel<<<copy_blocks, 256, 0, s>>>(x->win, trip_off(x, parity), x->P, x->words, x->off, all);
    return cudaGetLastError();
}

cudaError_t lsa_destroy(LsaX *x) {
    if (!x) return cudaSuccess;
    NcclDevApi &N = dev_api();
    cudaError_t e = cudaSuccess;
    if (x->off) e = cudaFree(x->off);
    if (x->dc_ok) N.DevCommDestroy(x->comm, &x->dc);
    if (x->win_ok) N.WindowDeregister(x->comm, x->win);
    if (x->buf) N.MemFree(x->buf);
    delete x;
    return e;
}

#else  // built without the NCCL device headers: the host exchange only

struct LsaX {};
cudaError_t lsa_create(void *, int, int, long long, int, LsaX **out, std::string *msg) {
    *out = nullptr;
    if (msg) *msg = "built without the NCCL device API headers (nccl_device.h, NCCL >= 2.28)";
    return cudaErrorNotSupported;
}
int *lsa_send_buffer(LsaX *, int) { return nullptr; }
long long lsa_capacity(const LsaX *) { return 0; }
int lsa_words(const LsaX *) { return 0; }
const unsigned long long *lsa_total(const LsaX *) { return nullptr; }
cudaError_t lsa_exchange(LsaX *, int, const unsigned long long *, int *, long long *, int, cudaStream_t, int,
                         long long *) {
    return cudaErrorNotSupported;
}
cudaError_t lsa_destroy(LsaX *) { return cudaSuccess; }

#endif

}  // namespace pico

// kernels.h -- internal host-side interface between the C ABI (capi.cu) and
// the algorithm drivers (histocore.cu, peelone.cu, shard.cu).
#pragma once
#include <string>
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#include "pico.h"
#include <nvtx3/nvToolsExt.h>

namespace pico {

// NVTX range of a phase slot (PICO_K_*): "pico:<slot>"
inline void nvtx_push(int slot) {
    static const char *names[PICO_K_COUNT] = {"pico:degree", "pico:init", "pico:rounds", "pico:sum", "pico:update",
                                              "pico:peel", "pico:validate", "pico:relabel", "pico:edgelist"};
    nvtxRangePushA(slot >= 0 && slot < PICO_K_COUNT ? names[slot] : "pico");
}

constexpr unsigned long long kFszCap = 1ull << 16;  // per-round sizes recorded

struct DevInfo {
    int device;
    int sms;
    int coop;  // cooperative launch supported
};

// stream-ordered allocation from a library-owned memory pool of the current
// device (release threshold: keep everything; the process's default pool and
// its other users are left alone) -- capi.cu
cudaError_t lib_malloc_async(void **p, size_t bytes, cudaStream_t s);
template <class T>
inline cudaError_t lib_malloc_async(T **p, size_t bytes, cudaStream_t s) {
    return lib_malloc_async(reinterpret_cast<void **>(p), bytes, s);
}

size_t hc_workspace_bytes(long long n, long long arcs, uint32_t flags);
cudaError_t hc_run(const long long *rp, const int *ci, long long n, long long arcs, int *core,
                   cudaStream_t s, uint32_t flags, void *ws, pico_stats_t *st, const DevInfo &dev);

// CntCore / NbrCore ablations (index2core.cu); cnt_filter selects CntCore
size_t i2c_workspace_bytes(long long n, long long arcs);
cudaError_t i2c_run(const long long *rp, const int *ci, long long n, long long arcs, int *core, cudaStream_t s,
                    uint32_t flags, bool cnt_filter, void *ws, pico_stats_t *st, const DevInfo &dev);

size_t po_workspace_bytes(long long n, long long arcs, uint32_t flags);
cudaError_t po_run(const long long *rp, const int *ci, long long n, long long arcs, int *core,
                   cudaStream_t s, uint32_t flags, void *ws, pico_stats_t *st, const DevInfo &dev);

cudaError_t po_clamp_hammer(int mode, int d, int k, long long c, int *final_out, long long *gt, long long *k1,
                            cudaStream_t s);

// internal compaction of the vertex ids (relabel.cu)
struct Relabel {
    long long n2;     // non-isolated vertices (new ids 0..n2-1)
    long long *rp2;   // [n2+1]
    int *ci2;         // [2m]
    unsigned *bits;   // [n/32] non-isolated bitmap
    unsigned *wpre;   // [n/32] exclusive prefix of popc(bits)
    int *inv;         // [n2] new -> old id
    int *core2;       // [n2] coreness in new ids
    long long launches;
    bool active;      // false: too few isolated vertices, graph used as is
};
size_t relabel_workspace_bytes(long long n, long long arcs);
cudaError_t relabel_build(const long long *rp, const int *ci, long long n, long long arcs, cudaStream_t s,
                          void *ws, const DevInfo &dev, bool force, Relabel *out);
cudaError_t relabel_back(const Relabel &r, long long n, int *core_out, cudaStream_t s, const DevInfo &dev);

// sharded HistoCore (histocore.cu)
struct Shard;
cudaError_t shard_create(const long long *rp, const int *ci, long long nloc, long long vb, long long ng,
                         uint32_t flags, cudaStream_t s, const DevInfo &dev, Shard **out);
cudaError_t shard_degrees(Shard *h, int *deg_out);
cudaError_t shard_init(Shard *h, const int *deg_global, long long *changed);
cudaError_t shard_pack(Shard *h, int *triples, long long cap, long long *count);
cudaError_t shard_pack_dev(Shard *h, int *triples, const unsigned long long **count_dev);
// total_dev (optional): the triple count in device memory (device-side
// exchange); the host total is then ignored
cudaError_t shard_apply(Shard *h, const int *triples, long long total, long long *changed,
                        const unsigned long long *total_dev = nullptr);
cudaError_t shard_result(Shard *h, int *core_out);
cudaError_t shard_destroy(Shard *h);

// sharded PeelOne (shard_peel.cu): each call publishes (|F| of this rank,
// next-level bound) as two int64 on the device (pshard_out)
struct PeelShard;
cudaError_t pshard_create(const long long *rp, const int *ci, long long nloc, long long vb, long long ng,
                          uint32_t flags, cudaStream_t s, const DevInfo &dev, PeelShard **out);
const long long *pshard_out(PeelShard *h);
long long pshard_nloc(PeelShard *h);
cudaError_t pshard_scan(PeelShard *h, int k, int *front);
cudaError_t pshard_apply(PeelShard *h, const int *all, long long total, int *front);
cudaError_t pshard_read(PeelShard *h, long long *count, int *kmin);
cudaError_t pshard_counters(PeelShard *h, long long *arcs_scanned, long long *guarded);
cudaError_t pshard_result(PeelShard *h, int *core_out);
cudaError_t pshard_destroy(PeelShard *h);
// the level loop driven on the device, exchanging over NCCL's device API
// (PICO_F_LSA_EXCHANGE; lx: a window of 1-word items, cap >= every rank's nloc)
struct LsaX;
cudaError_t pshard_run_lsa(PeelShard *h, LsaX *lx, long long n_global, long long *levels, long long *subrounds,
                           int *kmax, long long *lvsz_host, long long lvcap, std::string *msg);

// decremental HistoCore (histocore.cu)
struct Dyn;
cudaError_t dyn_create(const long long *rp, const int *ci, long long n, long long arcs, uint32_t flags,
                       cudaStream_t s, const DevInfo &dev, pico_stats_t *st, Dyn **out);
cudaError_t dyn_core(Dyn *h, int *core_out);
cudaError_t dyn_delete(Dyn *h, const int *src, const int *dst, long long k, pico_stats_t *st);
cudaError_t dyn_insert(Dyn *h, const int *src, const int *dst, long long k, pico_stats_t *st);
cudaError_t dyn_destroy(Dyn *h);

size_t validate_workspace_bytes();
cudaError_t validate_run(const long long *rp, const int *ci, long long n, long long arcs,
                         cudaStream_t s, void *ws, int *bad);

}  // namespace pico

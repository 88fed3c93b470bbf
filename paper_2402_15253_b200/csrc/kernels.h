// kernels.h -- internal host-side interface between the C ABI (capi.cu) and
// the algorithm drivers (histocore.cu, peelone.cu, shard.cu).
#pragma once
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#include "pico.h"

namespace pico {

constexpr unsigned long long kFszCap = 1ull << 16;  // per-round sizes recorded

struct DevInfo {
    int device;
    int sms;
    int coop;  // cooperative launch supported
};

size_t hc_workspace_bytes(long long n, long long arcs, uint32_t flags);
cudaError_t hc_run(const long long *rp, const int *ci, long long n, long long arcs, int *core,
                   cudaStream_t s, uint32_t flags, void *ws, pico_stats_t *st, const DevInfo &dev);

size_t po_workspace_bytes(long long n, long long arcs, uint32_t flags);
cudaError_t po_run(const long long *rp, const int *ci, long long n, long long arcs, int *core,
                   cudaStream_t s, uint32_t flags, void *ws, pico_stats_t *st, const DevInfo &dev);

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

size_t validate_workspace_bytes();
cudaError_t validate_run(const long long *rp, const int *ci, long long n, long long arcs,
                         cudaStream_t s, void *ws, int *bad);

}  // namespace pico

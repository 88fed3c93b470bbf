// Device-side exchange of the sharded HistoCore round over NCCL's device API
// (lsa_exchange.cu).  Internal to libpico; the public entry point is
// pico_coreness_sharded_ex with PICO_F_LSA_EXCHANGE (include/pico_shard.h).
#pragma once
#include <string>

#include <cuda_runtime.h>

namespace pico {

struct LsaX;

// Collective over the communicator (every rank calls it with the same cap):
// a symmetric window for the count rows and the double-buffered triple
// buffers (cap triples per rank and parity), and a device communicator with
// one LSA barrier.  comm is the ncclComm_t.  Fails with cudaErrorNotSupported
// (and *msg) when the loaded NCCL lacks the device API or the ranks do not
// all share one LSA (NVLink) team.
cudaError_t lsa_create(void *comm, int P, int me, long long cap, int words, LsaX **out, std::string *msg);
// this rank's triple buffer of round parity `parity` (inside the window): the
// pack kernel of the round writes its (v, oldcore, core) triples here
int *lsa_send_buffer(LsaX *x, int parity);
long long lsa_capacity(const LsaX *x);
int lsa_words(const LsaX *x);  // int32 words per item
// device pointer to the global triple count of the latest exchange
const unsigned long long *lsa_total(const LsaX *x);
// one exchange on stream s: counts (one LSA barrier) then the peer copies
// into all[words * total]; *tot_out (device, may be null) receives the total.
// has_aux: mine[1] is a per-rank value reduced by min into *min_out (device)
cudaError_t lsa_exchange(LsaX *x, int parity, const unsigned long long *mine, int *all, long long *tot_out,
                         int copy_blocks, cudaStream_t s, int has_aux = 0, long long *min_out = nullptr);
cudaError_t lsa_destroy(LsaX *x);

}  // namespace pico

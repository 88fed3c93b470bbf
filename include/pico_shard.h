/*
 * pico_shard.h -- C ABI of the sharded (multi-GPU) HistoCore of libpico.so.
 *
 * SURVEY 8(e); PAPER.md names multi-GPU as future work.  The graph
 * is split by a 1-D vertex partition: rank r owns the rows of the contiguous
 * range [v_begin, v_begin + nloc) (their histograms and estimates live only
 * on r).  Each round t of HistoCore (Alg 6) becomes
 *
 *     pico_shard_pack   -> this rank's changed (v, oldcore, core) triples
 *     allgatherv        -> every rank receives every rank's triples
 *                          (done by the caller, e.g. torch.distributed:
 *                          paper_2402_15253_b200/sharded.py, or inside the
 *                          library over NCCL: pico_coreness_sharded below)
 *     pico_shard_apply  -> UpdateHisto of all received triples over the
 *                          local CSC (owned neighbours of each v), then
 *                          SumHisto of the local frontier
 *
 * and the run ends when a round's global triple count is 0.  The rounds are
 * the synchronous rounds of the single-GPU path, so the coreness is
 * bit-exact and l2 and every |F_t| (summed over ranks) do not depend on the
 * number of ranks.
 *
 * Conventions (beyond those of pico.h):
 *  - rowptr_local [nloc+1] (int64, rowptr_local[0] = 0) and colidx_local
 *    [rowptr_local[nloc]] (int32 GLOBAL neighbour ids) are DEVICE arrays of
 *    the owned rows; the caller keeps them alive until pico_shard_destroy.
 *  - Triples are int32 [3*count] device arrays (v_global, oldcore, core).
 *  - Every call is blocking and ordered on the stream given at creation.
 *  - Call order: create, degrees, (allgather of degrees), init, then
 *    { pack, (allgatherv), apply } until the global count is 0, result,
 *    destroy.  Status codes as in pico.h; a triple buffer smaller than the
 *    packed count -> PICO_EINVAL.
 */
#ifndef PICO_SHARD_H_
#define PICO_SHARD_H_

#include "pico.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pico_shard_s *pico_shard_t;

/* Create the rank's state; computes the local degrees.  flags: PICO_F_*
 * schedule flags of pico.h (e.g. PICO_F_TINY_TILES for tests). */
int pico_shard_create(const int64_t *rowptr_local, const int32_t *colidx_local, int64_t nloc,
                      int64_t v_begin, int64_t n_global, uint32_t flags, pico_stream_t stream,
                      pico_shard_t *out);

/* deg_local (device int32 [nloc]) <- degrees of the owned vertices, to be
 * all-gathered (in rank order) into the n_global-long deg_global. */
int pico_shard_degrees(pico_shard_t h, int32_t *deg_local);

/* InitHisto fused with round-1 SumHisto on the owned rows, using deg_global
 * (device int32 [n_global]) for the neighbours; builds the local CSC.
 * *changed_local <- |C_1 on this rank|. */
int pico_shard_init(pico_shard_t h, const int32_t *deg_global, int64_t *changed_local);

/* triples (device int32 [3*cap]) <- this rank's changed vertices of the
 * current round; *count <- their number. */
int pico_shard_pack(pico_shard_t h, int32_t *triples, int64_t cap, int64_t *count);

/* Apply all ranks' triples (device int32 [3*total]) and run the local
 * SumHisto of the next round.  Asynchronous (stream-ordered, no host round
 * trip) when changed_local is NULL; otherwise it waits and stores
 * |C_{t+1} on this rank| there. */
int pico_shard_apply(pico_shard_t h, const int32_t *triples, int64_t total, int64_t *changed_local);

/* core_local (device int32 [nloc]) <- coreness of the owned vertices. */
int pico_shard_result(pico_shard_t h, int32_t *core_local);

int pico_shard_destroy(pico_shard_t h);

/* ------------------------------------------------------------------------
 * One-call sharded coreness with the exchange inside the library (NCCL over
 * NVLink/NVSwitch).  One process (or thread) per GPU.
 * libnccl.so.2 is loaded on first use (dlopen); if it cannot be loaded the
 * comm calls return PICO_ENCCL.  NCCL errors -> PICO_ENCCL.
 * ---------------------------------------------------------------------- */
typedef struct pico_comm_s *pico_comm_t;

/* id (host, 128 bytes) <- a fresh NCCL unique id; call on one rank and
 * broadcast it to the others (e.g. through torch.distributed). */
int pico_comm_unique_id(uint8_t id[128]);

/* *comm <- communicator of rank `rank` of `nranks` on the CURRENT CUDA device
 * (ncclCommInitRank; collective over all ranks). */
int pico_comm_init(int nranks, int rank, const uint8_t id[128], pico_comm_t *comm);

/* Rank count / rank of a communicator (NULL comm -> PICO_EINVAL). */
int pico_comm_size(pico_comm_t comm, int *nranks, int *rank);

/* Coreness of the owned vertices [v_begin, v_end) of a graph whose rows are
 * split over the communicator's ranks in rank order (rank r's range starts
 * where rank r-1's ends; they tile [0, n_global)).  rowptr_local [nloc+1]
 * (int64, rowptr_local[0] = 0, nloc = v_end - v_begin) and colidx_local
 * (int32 GLOBAL ids) are DEVICE arrays of the owned rows; core_out_local
 * (device int32 [nloc]) receives their coreness.  m_global = undirected edges
 * of the whole graph (the local arc counts must sum to 2 m_global, else
 * PICO_EINVAL on every rank).  algo: PICO_ALGO_HISTOCORE (PeelOne is not
 * sharded: PICO_ENOTSUP).  Collective and blocking: every rank calls it with
 * its own range; the per-round exchange is an all-gather of the changed-triple
 * counts (the global convergence test) and a grouped-broadcast all-gatherv of
 * the (v, oldcore, core) triples, both on `stream`. */
int pico_coreness_sharded(pico_comm_t comm, const int64_t *rowptr_local, const int32_t *colidx_local,
                          int64_t n_global, int64_t m_global, int64_t v_begin, int64_t v_end, int algo,
                          int32_t *core_out_local, pico_stream_t stream);

/* Same with PICO_F_* schedule flags and optional stats (rounds = l2 and,
 * when stats->frontier_sizes is set, the GLOBAL |C_t| per round, identical
 * on every rank). */
int pico_coreness_sharded_ex(pico_comm_t comm, const int64_t *rowptr_local, const int32_t *colidx_local,
                             int64_t n_global, int64_t m_global, int64_t v_begin, int64_t v_end, int algo,
                             int32_t *core_out_local, pico_stream_t stream, uint32_t flags,
                             pico_stats_t *stats);

int pico_comm_destroy(pico_comm_t comm);

#ifdef __cplusplus
}
#endif
#endif /* PICO_SHARD_H_ */

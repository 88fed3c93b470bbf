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
 *                          (done by the caller, e.g. torch.distributed /
 *                          NCCL: paper_2402_15253_b200/sharded.py)
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

#ifdef __cplusplus
}
#endif
#endif /* PICO_SHARD_H_ */

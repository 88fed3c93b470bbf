/*
 * pico_shard.h -- C ABI of the sharded (multi-GPU) HistoCore and PeelOne of
 * libpico.so.
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
 * Sharded PeelOne: the level-synchronous peel of Alg 4
 * (clamp atomicSub>=k P:273; dynamic frontier P:342) over the same
 * 1-D partition.  A level k is
 *
 *     pico_peel_shard_scan   -> this rank's F = {owned alive u : core[u] == k}
 *     repeat:
 *       all-gather of the counts; a global count of 0 ends the level
 *       allgatherv of F (int32 GLOBAL ids, rank order)   (caller / NCCL)
 *       pico_peel_shard_apply -> clamped decrements over the local CSC of
 *                                every received v; owned u that reach k form
 *                                this rank's next F (same level)
 *
 * Each call also returns kmin, a lower bound of the smallest estimate above
 * k of this rank's alive vertices (INT32_MAX if none).  At the end of a level
 * the next level is max(k + 1, min over ranks of kmin); the run ends when
 * that minimum is INT32_MAX.  The first k comes from create's kmin.  Every
 * sub-round is a BSP sub-round of the single-GPU PeelOne, so the coreness is
 * bit-exact and the non-empty level and sub-round counts do not depend on the
 * number of ranks.  No degree exchange is needed.
 *
 * Conventions as for pico_shard_*; frontier buffers are device int32 with
 * cap >= nloc (an owned vertex enters F at most once per run), else
 * PICO_EINVAL.  Call order: create, { scan, { apply }* }*, result, destroy.
 * ---------------------------------------------------------------------- */
typedef struct pico_peel_shard_s *pico_peel_shard_t;

/* core = degree on the owned rows, alive list, local CSC.  *kmin <- smallest
 * nonzero owned degree (INT32_MAX if every owned vertex is isolated).
 * flags: PICO_F_TINY_TILES (tests), PICO_F_CLAMP_CAS, PICO_F_STATS. */
int pico_peel_shard_create(const int64_t *rowptr_local, const int32_t *colidx_local, int64_t nloc,
                           int64_t v_begin, int64_t n_global, uint32_t flags, pico_stream_t stream,
                           pico_peel_shard_t *out, int32_t *kmin);

/* Start level k (k > every earlier level): frontier[0..*count) <- this rank's
 * owned vertices with core == k (global ids); *kmin as above. */
int pico_peel_shard_scan(pico_peel_shard_t h, int32_t k, int32_t *frontier, int64_t cap, int64_t *count,
                         int32_t *kmin);

/* One sub-round: frontier_all (device int32 [total], every rank's F) ->
 * clamped decrements of the owned neighbours; frontier[0..*count) <- the
 * owned vertices that reached k (global ids); *kmin as above. */
int pico_peel_shard_apply(pico_peel_shard_t h, const int32_t *frontier_all, int64_t total, int32_t *frontier,
                          int64_t cap, int64_t *count, int32_t *kmin);

/* core_local (device int32 [nloc]) <- coreness of the owned vertices. */
int pico_peel_shard_result(pico_peel_shard_t h, int32_t *core_local);

int pico_peel_shard_destroy(pico_peel_shard_t h);

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
 * PICO_EINVAL on every rank).  algo: PICO_ALGO_HISTOCORE or PICO_ALGO_PEELONE
 * (other algos: PICO_EINVAL).  Collective and blocking: every rank calls it
 * with its own range.  HistoCore's per-round exchange is an all-gather of the
 * changed-triple counts (the global convergence test) and a grouped-broadcast
 * all-gatherv of the (v, oldcore, core) triples; PeelOne's per-sub-round
 * exchange is an all-gather of (|F|, kmin) pairs and a grouped-broadcast
 * all-gatherv of F (see pico_peel_shard_*); all on `stream`. */
int pico_coreness_sharded(pico_comm_t comm, const int64_t *rowptr_local, const int32_t *colidx_local,
                          int64_t n_global, int64_t m_global, int64_t v_begin, int64_t v_end, int algo,
                          int32_t *core_out_local, pico_stream_t stream);

/* Same with PICO_F_* schedule flags and optional stats, identical on every
 * rank.  HistoCore: rounds = l2 and, when stats->frontier_sizes is set, the
 * GLOBAL |C_t| per round.  PeelOne: levels, subrounds, kmax and, in
 * frontier_sizes, the vertices processed per non-empty level (global).
 * PICO_F_LSA_EXCHANGE (HistoCore): the round's exchange runs on the device
 * over NCCL's device API -- each rank's pack kernel writes its triples into
 * a symmetric window (ncclMemAlloc + ncclCommWindowRegister, identical size
 * on every rank), a one-warp kernel stores its count into every peer's count
 * row and passes one LSA barrier (release/acquire), and a copy kernel loads
 * the peers' triples over NVLink in rank order; the host enqueues rounds in
 * batches (PICO_LSA_BATCH, default 4) and reads the global counts once per
 * batch (rounds after convergence are empty no-ops).  Same coreness, l2 and
 * |C_t| as the host exchange.  PeelOne with the flag: the level loop itself
 * runs on the device (one thread decides scan / apply / done after every
 * exchange of (|F|, next-level bound) pairs and F), batches of 16 steps are
 * one CUDA graph, and the host reads a done flag per batch; same levels,
 * sub-rounds and k_max.  PICO_ENOTSUP (nothing computed) when the
 * loaded NCCL lacks the device API or the ranks are not one LSA team. */
int pico_coreness_sharded_ex(pico_comm_t comm, const int64_t *rowptr_local, const int32_t *colidx_local,
                             int64_t n_global, int64_t m_global, int64_t v_begin, int64_t v_end, int algo,
                             int32_t *core_out_local, pico_stream_t stream, uint32_t flags,
                             pico_stats_t *stats);

int pico_comm_destroy(pico_comm_t comm);

#ifdef __cplusplus
}
#endif
#endif /* PICO_SHARD_H_ */

/*
 * pico_dyn.h -- C ABI of decremental HistoCore in libpico.so (core
 * maintenance under edge deletions).
 *
 * PAPER.md P:61 and P:882-884 name dynamic graphs as a setting the
 * Index2core paradigm suits.  After a HistoCore run (Alg 6) every
 * estimate equals the coreness and every per-vertex histogram is exact; a
 * deletion can only lower coreness, so the current coreness is an upper bound
 * of the new one and the same rounds, started from the histograms with the
 * deleted neighbours taken out, converge to the new coreness without
 * rebuilding anything.
 *
 * Conventions (beyond those of pico.h):
 *  - pico_dyn_create copies the graph (device CSR, as pico_coreness) into a
 *    handle-owned buffer and runs HistoCore; the caller's arrays are not
 *    kept.  Internal compaction (PICO_F_RELABEL) does not apply.
 *  - src / dst are DEVICE int32 arrays of k undirected edges {src[i], dst[i]}
 *    that must be edges of the current graph; both arcs are removed.  The
 *    batch is canonicalised on the device first ({u, v} = {v, u}; repeated
 *    edges, in either orientation, count once).  A missing edge, a self
 *    loop or an id out of range -> PICO_EINVAL, detected before anything is
 *    modified: the handle keeps the previous graph and stays usable.
 *  - Calls are blocking and ordered on the stream given at creation.
 *  - Insertions (pico_dyn_insert_edges) can raise coreness, by at most one
 *    per inserted edge and only inside the band of old coreness values the
 *    batch touches: the handle raises the estimates of the vertices the band-
 *    restricted BFS from the new edges reaches to an upper bound
 *    min(deg, core + k), rebuilds its CSR with the new arcs, and reruns the
 *    rounds warm-started from those estimates (DESIGN.md "Incremental
 *    HistoCore").
 */
#ifndef PICO_DYN_H_
#define PICO_DYN_H_

#include "pico.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pico_dyn_s *pico_dyn_t;

/* Copy the graph, run HistoCore, keep its state.  flags: PICO_F_* schedule
 * flags of pico.h; stats (optional) as in pico_coreness_ex for this run. */
int pico_dyn_create(const int64_t *rowptr, const int32_t *colidx, int64_t n, int64_t m, uint32_t flags,
                    pico_stream_t stream, pico_stats_t *stats, pico_dyn_t *out);

/* core_out (device int32 [n]) <- the coreness of the current graph. */
int pico_dyn_coreness(pico_dyn_t h, int32_t *core_out);

/* Delete k undirected edges and bring the coreness up to date.  stats
 * (optional): rounds of the update and, with frontier_sizes set, |C_t| of
 * each. */
int pico_dyn_delete_edges(pico_dyn_t h, const int32_t *src, const int32_t *dst, int64_t k, pico_stats_t *stats);

/* Insert k undirected edges {src[i], dst[i]} (DEVICE int32 arrays) and
 * bring the coreness up to date.  The batch is canonicalised as for
 * deletions (repeated edges count once); a self loop, an id out of range or
 * an edge already in the graph -> PICO_EINVAL before anything is modified.
 * Cost: O(m) to rebuild the handle's CSR and histograms, plus the rounds
 * from the raised estimates.  stats (optional): the warm-started run's
 * counters; .affected = vertices whose estimate was raised, .bfs_levels. */
int pico_dyn_insert_edges(pico_dyn_t h, const int32_t *src, const int32_t *dst, int64_t k, pico_stats_t *stats);

int pico_dyn_destroy(pico_dyn_t h);

#ifdef __cplusplus
}
#endif
#endif /* PICO_DYN_H_ */

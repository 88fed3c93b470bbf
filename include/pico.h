/*
 * pico.h -- C ABI of the B200-native PICO k-core library (libpico.so).
 *
 * Implements the data-parallel hot path of "PICO: Accelerating All k-Core
 * Paradigms on GPU" (arXiv 2402.15253): the coreness of every vertex of an
 * undirected simple graph.  Citations "P:<line>" refer to PAPER.md.
 *
 *   Problem: core(v) = max{k : v belongs to the k-core}, the
 *   k-core being the maximal subgraph whose vertices all have degree >= k.
 *   Input: CSR = offsets + concatenated neighbour lists.
 *
 *   PICO_ALGO_HISTOCORE -- Index2core iteration with persistent per-vertex
 *       histograms (Alg 6 "HistoCore"; frontier rule Theorem 2,
 *       P:374-379; update rule from the N1/N2/N3 analysis).
 *   PICO_ALGO_PEELONE   -- level-synchronous peel with the clamped
 *       "assertion" decrement atomicSub>=k (Alg 4) and a
 *       dynamic frontier inside each level ("PO-dyn").
 *
 * Both return the unique coreness vector (bit-exact).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Graph: rowptr int64[n+1] with rowptr[0] = 0 and rowptr[n] = 2m;
 *    colidx int32[2m]; symmetric, no self loops, no duplicate neighbours
 *    ("symmetric deduplicated CSR").  m counts UNDIRECTED edges.  Rows need
 *    not be sorted unless PICO_F_VALIDATE is set (validation requires sorted
 *    rows).  Isolated vertices are allowed and get coreness 0.
 *  - Ownership: the caller owns every buffer it passes; inputs are never
 *    written.  core_out is written completely on success and is unspecified
 *    on error.
 *  - Device entry points take DEVICE pointers valid on the current CUDA
 *    device and a cudaStream_t (NULL = legacy default stream).  They are
 *    stream-ordered after prior work on `stream` and BLOCKING: they return
 *    when core_out is final (the round loop needs a handful of host reads).
 *  - Re-entrancy: calls on different streams/threads may run concurrently.
 *    Global state: a thread-local last-error string, and one library-owned
 *    stream-ordered memory pool per device (created on first use, release
 *    threshold "keep", never shared with the process's default pool) from
 *    which workspace the caller does not pass is allocated and freed.
 *  - Errors: a non-zero pico_status_t is returned; nothing is thrown across
 *    the ABI.  pico_last_error() gives a thread-local message.
 *      n < 0, m < 0, NULL pointer with n > 0, unknown algo -> PICO_EINVAL
 *      n >= 2^31                                         -> PICO_ENOTSUP
 *      device allocation failure                         -> PICO_ENOMEM
 *      any CUDA runtime error                            -> PICO_ECUDA
 *      PICO_F_VALIDATE and a malformed graph             -> PICO_EGRAPH
 *  - n == 0 is a no-op returning PICO_OK; m == 0 gives all zeros.
 */
#ifndef PICO_H_
#define PICO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* cudaStream_t without pulling in the CUDA headers */
typedef struct CUstream_st *pico_stream_t;

typedef enum {
    PICO_ALGO_HISTOCORE = 0, /* Alg 6, P:489-539 (primary kernel)           */
    PICO_ALGO_PEELONE = 1,   /* Alg 4 + dynamic frontier       */
    PICO_ALGO_AUTO = 2,      /* pick one of the two from the degree skew  */
                             /* d_max * n / 2m and the size 2m (SURVEY    */
                             /* 8(f) NEXT-2; rule and data: DESIGN.md);   */
                             /* stats->algo reports the choice            */
    /* Index2core ablations, same coreness and rounds: */
    PICO_ALGO_CNTCORE = 3,   /* Alg 5 CntCore: frontiers by cnt, */
                             /* HINDEX rebuilt from all neighbours        */
    PICO_ALGO_NBRCORE = 4    /* NbrCore: every neighbour of a     */
                             /* changed vertex recomputes HINDEX          */
} pico_algo_t;

typedef enum {
    PICO_OK = 0,
    PICO_EINVAL = 1,
    PICO_ENOTSUP = 2,
    PICO_ENOMEM = 3,
    PICO_ECUDA = 4,
    PICO_ENCCL = 5,
    PICO_EGRAPH = 6
} pico_status_t;

/* flags for pico_coreness_ex / pico_coreness_host.  None changes the result;
 * they select instrumentation or an alternative (bit-exact) schedule.      */
enum {
    PICO_F_VALIDATE = 1u,     /* O(m) device check of the CSR contract first  */
    PICO_F_STATS = 2u,        /* fill pico_stats_t counters (extra atomics)  */
    PICO_F_TIMING = 4u,       /* per-kernel device time via CUDA events      */
    PICO_F_HOST_LOOP = 8u,    /* one kernel launch per phase, host-driven    */
    PICO_F_CLAMP_SUB = 16u,   /* PeelOne: atomicSub + end-of-level repair    */
                              /* (SURVEY 8(c)#18b); default is atomicSub +   */
                              /* atomicMax(k) on overshoot                   */
    PICO_F_CLAMP_CAS = 1024u, /* PeelOne: CAS-loop atomicSub>=k (the literal */
                              /* single-transaction clamp of P:273)          */
    PICO_F_DEBUG_INVARIANTS = 4096u, /* HistoCore: after the rounds, check on */
                              /* the device that every histogram matches    */
                              /* the final estimates (bins < core count     */
                              /* neighbours of that estimate, the cap bin   */
                              /* those at or above it) and that  */
                              /* the estimates are an h-index fixed point   */
                              /* (P:138-146); a violation -> PICO_EGRAPH    */
    PICO_F_L2_PERSIST = 16384u,/* HistoCore A/B: the push rounds' estimate   */
                              /* gathers (n x 2 B) as a persisting L2       */
                              /* access-policy window during the round      */
                              /* kernel (sets and then resets the device's  */
                              /* persisting-L2 limit: process-wide state)   */
    PICO_F_PREFILTER = 2048u, /* HistoCore: degree-bucket row order + scan   */
                              /* prefix (cuts scanned arcs ~44%; measured    */
                              /* slower on B200, so opt-in)                  */
    PICO_F_TINY_TILES = 32u,  /* test-only: tiny degree-class thresholds and */
                              /* shared-memory bin caps so every code path   */
                              /* (incl. the global-histogram fallback) runs  */
                              /* on small graphs                             */
    PICO_F_PUSH_ONLY = 64u,   /* HistoCore: never use the pull-direction     */
                              /* UpdateHisto (dense rounds)                  */
    PICO_F_PULL_ALWAYS = 128u,/* HistoCore: pull direction in every round    */
    PICO_F_RELABEL = 256u,    /* force the internal compaction of isolated   */
                              /* vertex ids (result mapped back, bit-exact)  */
    PICO_F_NO_RELABEL = 512u, /* never compact (default: compact when n >=   */
                              /* pico_relabel_threshold() and >= 10% of the  */
                              /* ids are isolated, so per-vertex arrays fit  */
                              /* the L2; PeelOne compacts only when forced)  */
    PICO_F_LSA_EXCHANGE = 32768u /* pico_coreness_sharded_ex (HistoCore and  */
                              /* PeelOne): the exchange on the device through */
                              /* NCCL's device API (symmetric window, LSA    */
                              /* peer loads, one LSA barrier per round), no  */
                              /* host synchronisation per round; needs NCCL  */
                              /* >= 2.28 and one NVLink domain, else         */
                              /* PICO_ENOTSUP (include/pico_shard.h)         */
};

/* Vertex count above which pico_coreness_ex relabels internally by default. */
int64_t pico_relabel_threshold(void);

/* kernel slots of pico_stats_t.kernel_ms / kernel_launches */
enum {
    PICO_K_DEGREE = 0,   /* H0 / P0: degree, classification, alive list     */
    PICO_K_INIT = 1,     /* H1-H3 round 1: InitHisto fused with SumHisto    */
    PICO_K_ROUNDS = 2,   /* H3-H5 rounds 2..: SumHisto + UpdateHisto loop   */
    PICO_K_SUM = 3,      /* host-loop mode: SumHisto launches               */
    PICO_K_UPDATE = 4,   /* host-loop mode: UpdateHisto launches            */
    PICO_K_PEEL = 5,     /* P1-P3: PeelOne level loop                        */
    PICO_K_VALIDATE = 6,
    PICO_K_OTHER = 7,    /* internal compaction of isolated vertex ids       */
    PICO_K_EDGELIST = 8, /* HistoCore: bucketed edge list of the pull rounds */
    PICO_K_COUNT = 9
};

typedef struct {
    /* iteration counts */
    int64_t rounds;         /* HistoCore l2: rounds with a non-empty frontier */
    int64_t levels;         /* PeelOne: non-empty levels (= #distinct cores)  */
    int64_t subrounds;      /* PeelOne: bulk-synchronous sub-rounds that      */
                            /* drained the dynamic frontiers of all levels   */
    int64_t kmax;           /* max coreness                                   */
    /* work counters (PICO_F_STATS), the terms of DESIGN.md "algorithmic bytes" */
    int64_t frontier_total;     /* HistoCore: sum_t |F_t| incl. round 1;       */
                                /* Cnt/NbrCore: HINDEX evaluations             */
    int64_t init_slots_written; /* HistoCore: histogram slots written by init  */
    int64_t arcs_scanned;       /* HistoCore: sum_t S_t (UpdateHisto arcs);    */
                                /* Cnt/NbrCore: neighbour entries read (the    */
                                /* edge accesses of the paper's Fig 3);        */
                                /* PeelOne: arcs of processed vertices          */
    int64_t guarded_arcs;       /* HistoCore: arcs with core[u] > core[v];     */
                                /* PeelOne: clamped decrements issued            */
    int64_t bins_read;          /* HistoCore: SumHisto bins read (rounds >= 2) */
    int64_t pushes;             /* vertices pushed into a next frontier/queue  */
    int64_t alive_scanned;      /* PeelOne: sum over levels of |alive list|;   */
                                /* Cnt/NbrCore: sum over rounds of |V_active|  */
    int64_t hub_fallbacks;      /* vertices that needed the global-bin path    */
    int64_t segments;           /* HistoCore: UpdateHisto work items (v, seg)  */
                                /* produced; PeelOne: queue entries processed  */
    int64_t segments_init;      /* HistoCore: of which produced by init        */
    int64_t kernel_count;       /* kernels this library launched in the call   */
    int64_t pull_rounds;        /* HistoCore: rounds run in the pull direction */
    /* per-kernel device time (PICO_F_TIMING) */
    double kernel_ms[PICO_K_COUNT];
    int64_t kernel_launches[PICO_K_COUNT];
    /* optional caller-owned HOST array receiving |F_t| for t = 1..rounds
     * (HistoCore) or the processed count per level (PeelOne); may be NULL */
    int64_t *frontier_sizes;
    int64_t frontier_sizes_cap;
    /* optional caller-owned HOST array (same capacity) receiving, for
     * HistoCore, sum_{v in C_t} deg(v) for t = 1..rounds; may be NULL */
    int64_t *round_arcs;
    /* optional caller-owned HOST array of 2 * frontier_sizes_cap entries
     * receiving, for HistoCore rounds t = 1..rounds, the device time in ns
     * (%globaltimer between grid barriers) of UpdateHisto(t) at [2(t-1)] and
     * of the SumHisto that builds F_{t+1} at [2(t-1)+1]; for PeelOne, per
     * scanned level L = 0, 1, ... the level scan at [2L] and the drain of its
     * dynamic frontier at [2L+1] (low 40 bits; above them the level's k at
     * [2L] and its BSP sub-rounds at [2L+1]); may be NULL.  Filled by the persistent
     * kernels only (not PICO_F_HOST_LOOP). */
    int64_t *round_ns;
    /* the algorithm that ran (PICO_ALGO_AUTO resolved) */
    int64_t algo;
    /* pico_dyn_insert_edges: vertices whose estimate was raised (the band-
     * restricted BFS set R) and that BFS's levels */
    int64_t affected;
    int64_t bfs_levels;
    /* optional caller-owned HOST int32 array of frontier_counts_cap >= n
     * entries receiving, for HistoCore with PICO_F_STATS, the number of
     * rounds in which each vertex was a frontier (its estimate changed) --
     * the measure of the paper's Fig 3: an edge {u, v} is read
     * frontier_counts[u] + frontier_counts[v] times; may be NULL */
    int32_t *frontier_counts;
    int64_t frontier_counts_cap;
} pico_stats_t;

/* The north-star entry point: coreness of every vertex, device buffers. */
int pico_coreness(const int64_t *rowptr, const int32_t *colidx, int64_t n, int64_t m,
                  int algo, int32_t *core_out, pico_stream_t stream);

/* Bytes of device workspace pico_coreness_ex needs for (n, m, algo, flags). */
size_t pico_workspace_bytes(int64_t n, int64_t m, int algo, uint32_t flags);

/* Extended form.  workspace: caller-owned device buffer of at least
 * pico_workspace_bytes(...) bytes, 256-byte aligned, or NULL (the library
 * then allocates with cudaMallocAsync on `stream` and frees before
 * returning); a non-NULL workspace that is too small -> PICO_EINVAL.
 * stats: caller-owned host struct or NULL; counters are filled iff
 * PICO_F_STATS, kernel times iff PICO_F_TIMING, iteration counts always. */
int pico_coreness_ex(const int64_t *rowptr, const int32_t *colidx, int64_t n, int64_t m,
                     int algo, int32_t *core_out, pico_stream_t stream, uint32_t flags,
                     void *workspace, size_t workspace_bytes, pico_stats_t *stats);

/* End-to-end form on HOST buffers: copies rowptr/colidx host->device
 * (pinned memory is fastest), runs the path, copies the coreness back into
 * core_out_host.  Device memory is allocated from the stream-ordered pool
 * and released before return.  Same status codes and flags. */
int pico_coreness_host(const int64_t *rowptr_host, const int32_t *colidx_host, int64_t n,
                       int64_t m, int algo, int32_t *core_out_host, pico_stream_t stream,
                       uint32_t flags, pico_stats_t *stats);

/* Diagnostic: the clamped decrement atomicSub>=k(core, 1, k) of PeelOne
 * ("a single atomic transaction"), run by
 * c concurrent device threads on ONE int32 cell holding d, with the level
 * k, in the implementation `mode` selects: 0 = atomicSub + atomicMax(k) on
 * overshoot (the default), 1 = atomicSub + the end-of-level repair
 * (PICO_F_CLAMP_SUB), 2 = the CAS loop (PICO_F_CLAMP_CAS).  The same device
 * function the PeelOne kernels call.  Outputs (host pointers): the cell's
 * final value (after the repair for mode 1), the number of calls whose
 * returned old value was > k (those that decremented), and the number that
 * returned k + 1 (the dynamic-frontier push).  The clamp law:
 * final = max(k, d - c), exactly min(c, max(d - k, 0)) calls see old > k,
 * and exactly one sees k + 1 iff k < d <= k + c.  Blocking on `stream`.
 * c < 0, k < 0, d < 0, an unknown mode or a NULL output -> PICO_EINVAL. */
int pico_clamp_hammer(int mode, int32_t d, int32_t k, int64_t c, int32_t *final_out,
                      int64_t *observed_gt_k, int64_t *observed_k1, pico_stream_t stream);

/* Human-readable name of a status code (static string). */
const char *pico_status_string(int status);
/* Message of the last failing call on this thread ("" if none). */
const char *pico_last_error(void);
/* Library version, e.g. 100 = 0.1.0. */
int pico_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PICO_H_ */

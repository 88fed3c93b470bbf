/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * reference for PICO (arXiv 2402.15253) k-core decomposition.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  It shares no code, header, table or
 * helper with the CUDA path (paper_2402_15253_b200/csrc); neither includes
 * the other.  Citations: "P:<line>" = /root/reference/PAPER.md line,
 * "S:<line>" = SPEC.md line, "SURVEY 8(c)#k" = the k-th reading listed in
 * SURVEY.md 8(c) and repeated in DESIGN.md.
 *
 * Graph input everywhere: CSR with int64 rowptr[n+1] and int32 colidx[2m],
 * symmetric, no self loops, no duplicates.
 *
 * Functions and their pins (tests/test_oracle.py):
 *   oracle_bz             coreness by Batagelj-Zaversnik bin-sort peel
 *                         (SURVEY 8(c) steps 1-6).  Pinned by G1
 *                         (P:33), closed forms, brute force (n<=7 exhaustive,
 *                         random n<=40), networkx.core_number, invariants.
 *   oracle_hindex         HINDEX of a multiset by its definition (Alg 2,
 *                         P:143-146).  Pinned by Fig 6 ([1,1,2,3,2]->2,
 *                         P:405) and a sort-based textbook h-index.
 *   oracle_jacobi_rounds  synchronous Index2core sweeps (Alg 2)
 *                         from core=deg; returns l2 = number of sweeps that
 *                         change something and the size of every changed set
 *                         |F_t|.  Pinned: fixed point == BZ coreness, G1 l2=1,
 *                         P5 l2=2, K4 l2=0, monotonicity.
 *   oracle_frontier_counts  the Fig 3 measure on the same sweeps:
 *                         per-vertex frontier multiplicity and the share of
 *                         frontier neighbours whose estimate stays unchanged.
 *                         Pinned: sum == sum of |F_t|, an independent Python
 *                         sweep on random graphs, closed forms (star, P5, K_n).
 *   oracle_peel_levels    level-synchronous Peel (Alg 1) in the
 *                         bulk-synchronous form of PeelOne (Alg 4):
 *                         returns coreness, the number of non-empty levels and
 *                         the BSP sub-round count.  Pinned: coreness == BZ,
 *                         non-empty levels == #distinct nonzero coreness,
 *                         G1: 2 levels / 3 sub-rounds.
 *   oracle_kcore_check    the definition itself: for every k the
 *                         subgraph induced by {core>=k} has min degree >= k.
 *   oracle_brute          repeated removal of a minimum-degree vertex (Peel,
 *                         Alg 1), O(n^2), its own adjacency
 *                         matrix: the pin for BZ on tiny graphs.  Pinned
 *                         against the pure-Python brute force of
 *                         oracle/coreness.py on random graphs.
 *   oracle_exhaustive     every labelled simple graph on n vertices (n <= 7:
 *                         2^21 graphs) through oracle_bz and oracle_brute;
 *                         returns the number of graphs where they differ.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* BZ bucket peel.  SURVEY 8(c) "Oracle algorithm: BZ bucket peel" steps 1-6,
 * after P:852-854 (vertices array sorted by degree, bin starts, positions;
 * process in ascending bin order, decrement neighbours, move them one bin
 * down).  Returns 0 on success, -1 on allocation failure.                  */
ORACLE_API int oracle_bz(const int64_t *rowptr, const int32_t *colidx,
                         int64_t n, int32_t *core)
{
    if (n <= 0) return 0;
    int64_t *deg = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int32_t *vert = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!deg || !pos || !vert) { free(deg); free(pos); free(vert); return -1; }

    /* step 1: deg[v] = rowptr[v+1]-rowptr[v]; md = max deg */
    int64_t md = 0;
    for (int64_t v = 0; v < n; v++) {
        deg[v] = rowptr[v + 1] - rowptr[v];
        if (deg[v] > md) md = deg[v];
    }
    int64_t *bin = (int64_t *)calloc((size_t)md + 1, sizeof(int64_t));
    if (!bin) { free(deg); free(pos); free(vert); return -1; }

    /* step 2: bin[d] = #vertices of degree d, then exclusive prefix sum */
    for (int64_t v = 0; v < n; v++) bin[deg[v]]++;
    int64_t start = 0;
    for (int64_t d = 0; d <= md; d++) {
        int64_t num = bin[d];
        bin[d] = start;
        start += num;
    }
    /* step 3: counting sort, pos[v] = bin[deg[v]]++, vert[pos[v]] = v */
    for (int64_t v = 0; v < n; v++) {
        pos[v] = bin[deg[v]];
        vert[pos[v]] = (int32_t)v;
        bin[deg[v]]++;
    }
    /* step 4: shift the bin starts back */
    for (int64_t d = md; d >= 1; d--) bin[d] = bin[d - 1];
    bin[0] = 0;

    /* step 5: process vertices in ascending order of current degree */
    for (int64_t i = 0; i < n; i++) {
        int64_t v = vert[i];
        for (int64_t e = rowptr[v]; e < rowptr[v + 1]; e++) {
            int64_t u = colidx[e];
            if (deg[u] > deg[v]) {
                int64_t du = deg[u];
                int64_t pu = pos[u];
                int64_t pw = bin[du];
                int64_t w = vert[pw];
                if (u != w) {
                    pos[u] = pw; vert[pu] = (int32_t)w;
                    pos[w] = pu; vert[pw] = (int32_t)u;
                }
                bin[du]++;
                deg[u]--;
            }
        }
    }
    /* step 6: core = deg */
    for (int64_t v = 0; v < n; v++) core[v] = (int32_t)deg[v];
    free(bin); free(deg); free(pos); free(vert);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* HINDEX (Alg 2): the integer h with |{x >= h}| >= h and
 * |{x >= h+1}| <= h, i.e. the largest h with at least h values >= h
 * (SURVEY 8(c)#5).  Written as the definition: try h = len, len-1, ..., 0. */
ORACLE_API int64_t oracle_hindex(const int32_t *vals, int64_t len)
{
    for (int64_t h = len; h >= 1; h--) {
        int64_t c = 0;
        for (int64_t i = 0; i < len; i++) c += (vals[i] >= h);
        if (c >= h) return h;
    }
    return 0;
}

/* h-index of v's neighbour values cur[u]: count values into bins 0..deg(v)
 * (a value above deg(v) can be counted as deg(v): h <= deg(v) always, as v
 * has only deg(v) neighbours), then walk h = deg(v) .. 1 accumulating the
 * number of values >= h until it reaches h.                              */
static int32_t hindex_of_neighbours(const int64_t *rowptr, const int32_t *colidx,
                                    int64_t v, const int32_t *cur, int64_t *cnt)
{
    int64_t d = rowptr[v + 1] - rowptr[v];
    for (int64_t j = 0; j <= d; j++) cnt[j] = 0;
    for (int64_t e = rowptr[v]; e < rowptr[v + 1]; e++) {
        int64_t x = cur[colidx[e]];
        cnt[x < d ? x : d]++;
    }
    int64_t ge = 0;
    for (int64_t h = d; h >= 1; h--) {
        ge += cnt[h];
        if (ge >= h) return (int32_t)h;
    }
    return 0;
}

/* Synchronous Index2core (Alg 2), core^0 = deg.  Sweep t
 * computes core^t(v) = HINDEX(core^{t-1}(nbr v)) for every v at once
 * (strict two-phase rounds).  F_t = {v : core^t(v) !=
 * core^{t-1}(v)}.  Stops at the first sweep with F_t empty.  Writes the
 * fixed point to core_out, |F_1|,|F_2|,... to fsizes (up to fsizes_cap
 * entries) and returns l2 = number of sweeps with F_t non-empty, or -1 on
 * allocation failure.                                                     */
ORACLE_API int64_t oracle_jacobi_rounds(const int64_t *rowptr, const int32_t *colidx,
                                        int64_t n, int32_t *core_out,
                                        int64_t *fsizes, int64_t fsizes_cap)
{
    if (n <= 0) return 0;
    int32_t *prev = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t *next = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int64_t md = 0;
    for (int64_t v = 0; v < n; v++) {
        int64_t d = rowptr[v + 1] - rowptr[v];
        if (d > md) md = d;
    }
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)(md + 1));
    if (!prev || !next || !cnt) { free(prev); free(next); free(cnt); return -1; }
    for (int64_t v = 0; v < n; v++) prev[v] = (int32_t)(rowptr[v + 1] - rowptr[v]);

    int64_t l2 = 0;
    for (;;) {
        int64_t changed = 0;
        for (int64_t v = 0; v < n; v++) {
            next[v] = hindex_of_neighbours(rowptr, colidx, v, prev, cnt);
            changed += (next[v] != prev[v]);
        }
        if (changed == 0) break;
        if (l2 < fsizes_cap) fsizes[l2] = changed;
        l2++;
        int32_t *t = prev; prev = next; next = t;
    }
    memcpy(core_out, prev, sizeof(int32_t) * (size_t)n);
    free(prev); free(next); free(cnt);
    return l2;
}

/* The measure behind the paper's Fig 3 ("the proportion of
 * vertices and edges that need multiple access"), on the same synchronous
 * sweeps as oracle_jacobi_rounds: fcount[v] = the number of sweeps t in which
 * v's estimate changes (v in F_t, the frontier of sweep t, t = 1..l2); an arc
 * (v, u) is read once per sweep in which v is a frontier, so an edge {u, v}
 * is accessed fcount[u] + fcount[v] times.  Also the P:226-227 observation
 * ("the h-index of an average of 94% of the frontiers' neighbours stays
 * unchanged"): *nbr_total = sum over t of sum over v in F_t of deg(v), and
 * *nbr_unchanged = the pairs (v in F_t, u in N(v)) with u not in F_{t+1}.
 * Returns l2 (-1 on allocation failure).                                    */
ORACLE_API int64_t oracle_frontier_counts(const int64_t *rowptr, const int32_t *colidx,
                                          int64_t n, int32_t *fcount,
                                          int64_t *nbr_unchanged, int64_t *nbr_total)
{
    *nbr_unchanged = 0;
    *nbr_total = 0;
    if (n <= 0) return 0;
    int32_t *prev = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t *next = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    char *front = (char *)calloc((size_t)n, 1);  /* v in F_t of the latest sweep */
    int64_t md = 0;
    for (int64_t v = 0; v < n; v++) {
        int64_t d = rowptr[v + 1] - rowptr[v];
        if (d > md) md = d;
    }
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)(md + 1));
    if (!prev || !next || !front || !cnt) { free(prev); free(next); free(front); free(cnt); return -1; }
    for (int64_t v = 0; v < n; v++) {
        prev[v] = (int32_t)(rowptr[v + 1] - rowptr[v]);
        fcount[v] = 0;
    }
    int64_t l2 = 0;
    for (;;) {
        int64_t changed = 0;
        for (int64_t v = 0; v < n; v++) {
            next[v] = hindex_of_neighbours(rowptr, colidx, v, prev, cnt);
            changed += (next[v] != prev[v]);
        }
        /* neighbours of the previous sweep's frontier: unchanged in this one? */
        if (l2 > 0)
            for (int64_t v = 0; v < n; v++) {
                if (!front[v]) continue;
                for (int64_t e = rowptr[v]; e < rowptr[v + 1]; e++) {
                    int32_t u = colidx[e];
                    *nbr_total += 1;
                    *nbr_unchanged += (next[u] == prev[u]);
                }
            }
        if (changed == 0) break;
        for (int64_t v = 0; v < n; v++) {
            front[v] = (char)(next[v] != prev[v]);
            fcount[v] += front[v];
        }
        l2++;
        int32_t *t = prev; prev = next; next = t;
    }
    free(prev); free(next); free(front); free(cnt);
    return l2;
}

/* Level-synchronous Peel in PeelOne's bulk-synchronous form (Alg 4,
 * P:308-336, with the assertion clamp of P:273 and Theorem 1).
 * res[v] = deg(v); for k = 1, 2, ... while vertices remain:
 * repeat sub-rounds { S = {alive v : res[v] <= k}; if S empty break; remove S,
 * core[v] = k for v in S; for every alive neighbour u of a vertex in S:
 * res[u] = max(k, res[u]-1) } (the clamp (old>k)?old-1:k).
 * Isolated vertices get 0 and are never alive.
 * Writes coreness, *levels = number of levels k that removed at least one
 * vertex, *subrounds = number of non-empty sub-rounds; returns k_max or -1. */
ORACLE_API int64_t oracle_peel_levels(const int64_t *rowptr, const int32_t *colidx,
                                      int64_t n, int32_t *core_out,
                                      int64_t *levels, int64_t *subrounds)
{
    *levels = 0; *subrounds = 0;
    if (n <= 0) return 0;
    int64_t *res = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    char *alive = (char *)malloc((size_t)n);
    int32_t *S = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!res || !alive || !S) { free(res); free(alive); free(S); return -1; }
    int64_t nalive = 0;
    for (int64_t v = 0; v < n; v++) {
        res[v] = rowptr[v + 1] - rowptr[v];
        alive[v] = res[v] > 0;
        nalive += alive[v];
        core_out[v] = 0;
    }
    int64_t k = 0, kmax = 0;
    while (nalive > 0) {
        k++;
        int level_used = 0;
        for (;;) {
            int64_t ns = 0;
            for (int64_t v = 0; v < n; v++)
                if (alive[v] && res[v] <= k) S[ns++] = (int32_t)v;
            if (ns == 0) break;
            (*subrounds)++;
            level_used = 1;
            for (int64_t i = 0; i < ns; i++) {       /* remove all of S first */
                alive[S[i]] = 0;
                core_out[S[i]] = (int32_t)k;
            }
            nalive -= ns;
            for (int64_t i = 0; i < ns; i++) {
                int64_t v = S[i];
                for (int64_t e = rowptr[v]; e < rowptr[v + 1]; e++) {
                    int64_t u = colidx[e];
                    if (alive[u]) res[u] = (res[u] - 1 > k) ? res[u] - 1 : k;
                }
            }
        }
        if (level_used) { (*levels)++; kmax = k; }
    }
    free(res); free(alive); free(S);
    return kmax;
}

/* ------------------------------------------------------------------------ */
/* The definition: returns 1 iff for every k >= 1 the subgraph induced
 * by {v : core[v] >= k} has minimum degree >= k, i.e. each v has at least
 * core[v] neighbours u with core[u] >= core[v].  (Necessary for a coreness
 * vector; maximality is what BZ / brute force add -- SURVEY 8(c).)        */
ORACLE_API int oracle_kcore_check(const int64_t *rowptr, const int32_t *colidx,
                                  int64_t n, const int32_t *core)
{
    for (int64_t v = 0; v < n; v++) {
        int64_t c = 0;
        for (int64_t e = rowptr[v]; e < rowptr[v + 1]; e++)
            c += (core[colidx[e]] >= core[v]);
        if (c < core[v]) return 0;
        if (core[v] < 0 || core[v] > rowptr[v + 1] - rowptr[v]) return 0;
    }
    return 1;
}

/* ------------------------------------------------------------------------ */
/* Brute force on an adjacency matrix (n <= 64): remove a
 * vertex of minimum current degree (lowest id on ties); its coreness is the
 * running maximum of the degrees at removal.  Independent of oracle_bz: no
 * bins, no CSR traversal order.                                            */
ORACLE_API int oracle_brute(int64_t n, const uint8_t *adj /* n*n, symmetric */, int32_t *core_out)
{
    if (n < 0 || n > 64) return -1;
    int64_t deg[64];
    char alive[64];
    for (int64_t v = 0; v < n; v++) {
        deg[v] = 0;
        for (int64_t u = 0; u < n; u++) deg[v] += (u != v) && adj[v * n + u];
        alive[v] = 1;
    }
    int64_t k = 0;
    for (int64_t it = 0; it < n; it++) {
        int64_t best = -1;
        for (int64_t v = 0; v < n; v++)
            if (alive[v] && (best < 0 || deg[v] < deg[best])) best = v;
        if (deg[best] > k) k = deg[best];
        core_out[best] = (int32_t)k;
        alive[best] = 0;
        for (int64_t u = 0; u < n; u++)
            if (alive[u] && u != best && adj[best * n + u]) deg[u]--;
    }
    return 0;
}

/* Every labelled simple graph on n vertices (edge subsets in mask order):
 * the CSR goes to oracle_bz, the adjacency matrix to oracle_brute.  Returns
 * the number of graphs whose coreness vectors differ (-1: bad n).         */
ORACLE_API int64_t oracle_exhaustive(int64_t n)
{
    if (n < 1 || n > 7) return -1;
    int64_t np = n * (n - 1) / 2;
    int32_t pu[21], pv[21];
    int64_t q = 0;
    for (int32_t i = 0; i < n; i++)
        for (int32_t j = i + 1; j < n; j++) { pu[q] = i; pv[q] = j; q++; }
    uint8_t adj[49];
    int64_t rowptr[8];
    int32_t colidx[42], cb[7], cr[7], fill[7];
    int64_t bad = 0;
    for (int64_t mask = 0; mask < ((int64_t)1 << np); mask++) {
        memset(adj, 0, sizeof(adj));
        for (int64_t e = 0; e < np; e++)
            if (mask >> e & 1) { adj[pu[e] * n + pv[e]] = 1; adj[pv[e] * n + pu[e]] = 1; }
        rowptr[0] = 0;
        for (int64_t v = 0; v < n; v++) {
            int64_t d = 0;
            for (int64_t u = 0; u < n; u++) d += adj[v * n + u];
            rowptr[v + 1] = rowptr[v] + d;
            fill[v] = 0;
        }
        for (int64_t v = 0; v < n; v++)       /* rows ascending */
            for (int64_t u = 0; u < n; u++)
                if (adj[v * n + u]) colidx[rowptr[v] + fill[v]++] = (int32_t)u;
        if (oracle_bz(rowptr, colidx, n, cb) != 0 || oracle_brute(n, adj, cr) != 0) return -1;
        if (memcmp(cb, cr, sizeof(int32_t) * (size_t)n) != 0) bad++;
    }
    return bad;
}

/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Nothing in the product path
 * (paper_2207_11662_b200/, include/) may include, link or call this file.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs use it.
 *
 * Plain per-source breadth-first search, written out as the textbook
 * definition the paper relies on:
 *
 *   PAPER.md:209 (§4): "The implementation of the closeness centrality
 *   algorithm ... uses breadth-first search (BFS) to find the distance from
 *   each vertex to every other vertex."  Cost O(V(V+E)).
 *
 * For every requested source s it returns
 *   S(s) = sum over vertices w reachable from s of d(s, w)   (uint64)
 *   k(s) = number of vertices reachable from s, s included  (int32)
 * Unreachable vertices contribute nothing here; the n-penalty sum
 * (§5.1) and the Wasserman-Faust closeness are
 * formed from (S, k) in oracle/oracle.py.
 *
 * No blocking, bit-parallelism, direction switching or reordering: one queue
 * BFS per source.  Sources are distributed over OpenMP threads only because
 * each BFS is independent; every source's result is a pure function of the
 * graph.
 *
 * Input: V and m canonical undirected edges (eu[i], ev[i]), 0 <= eu,ev < V,
 * eu != ev, no duplicates (oracle.py canonicalises).  The adjacency built here
 * is a plain array-of-lists (counting pass + fill pass).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t V;
    int64_t *start;   /* V+1 */
    int32_t *nbr;     /* 2m  */
} adj_t;

static int build_adj(adj_t *g, int32_t V, int64_t m, const int32_t *eu, const int32_t *ev)
{
    g->V = V;
    g->start = (int64_t *)calloc((size_t)V + 1, sizeof(int64_t));
    g->nbr = (int32_t *)malloc(sizeof(int32_t) * (size_t)(2 * m > 0 ? 2 * m : 1));
    if (!g->start || !g->nbr) return -3;
    int64_t *fill = (int64_t *)calloc((size_t)V + 1, sizeof(int64_t));
    if (!fill) return -3;
    for (int64_t i = 0; i < m; i++) {
        if (eu[i] < 0 || eu[i] >= V || ev[i] < 0 || ev[i] >= V) { free(fill); return -2; }
        g->start[eu[i] + 1]++;
        g->start[ev[i] + 1]++;
    }
    for (int32_t v = 0; v < V; v++) g->start[v + 1] += g->start[v];
    for (int32_t v = 0; v <= V; v++) fill[v] = g->start[v];
    for (int64_t i = 0; i < m; i++) {
        g->nbr[fill[eu[i]]++] = ev[i];
        g->nbr[fill[ev[i]]++] = eu[i];
    }
    free(fill);
    return 0;
}

/* one BFS from s; dist[] must be all -1 on entry and is restored on exit */
static void bfs_one(const adj_t *g, int32_t s, int32_t *dist, int32_t *queue,
                    uint64_t *S_out, int32_t *k_out)
{
    int64_t head = 0, tail = 0;
    uint64_t S = 0;
    dist[s] = 0;
    queue[tail++] = s;
    while (head < tail) {
        int32_t x = queue[head++];
        S += (uint64_t)dist[x];
        for (int64_t j = g->start[x]; j < g->start[x + 1]; j++) {
            int32_t y = g->nbr[j];
            if (dist[y] < 0) {
                dist[y] = dist[x] + 1;
                queue[tail++] = y;
            }
        }
    }
    *S_out = S;
    *k_out = (int32_t)tail;
    for (int64_t i = 0; i < tail; i++) dist[queue[i]] = -1;
}

/*
 * oracle_bfs_sources: for each of the n_src sources in `sources`, write
 * S_out[i], k_out[i].  nthreads <= 0 means "all available".
 * Returns 0 on success, -2 on an out-of-range id, -3 on allocation failure.
 */
int oracle_bfs_sources(int32_t V, int64_t m, const int32_t *eu, const int32_t *ev,
                       const int32_t *sources, int64_t n_src,
                       uint64_t *S_out, int32_t *k_out, int nthreads)
{
    adj_t g;
    int rc = build_adj(&g, V, m, eu, ev);
    if (rc) return rc;
    for (int64_t i = 0; i < n_src; i++)
        if (sources[i] < 0 || sources[i] >= V) { free(g.start); free(g.nbr); return -2; }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int err = 0;
#pragma omp parallel
    {
        int32_t *dist = (int32_t *)malloc(sizeof(int32_t) * (size_t)(V > 0 ? V : 1));
        int32_t *queue = (int32_t *)malloc(sizeof(int32_t) * (size_t)(V > 0 ? V : 1));
        if (!dist || !queue) {
#pragma omp atomic write
            err = -3;
        } else {
            for (int32_t v = 0; v < V; v++) dist[v] = -1;
#pragma omp for schedule(dynamic, 16)
            for (int64_t i = 0; i < n_src; i++)
                bfs_one(&g, sources[i], dist, queue, &S_out[i], &k_out[i]);
        }
        free(dist);
        free(queue);
    }
    free(g.start);
    free(g.nbr);
    return err;
}

/*
 * Persistent graph handle for timing: the adjacency is built once, and
 * oracle_graph_bfs reports the wall time of the BFS loop alone
 * (omp_get_wtime around the parallel region).
 */
void *oracle_graph_new(int32_t V, int64_t m, const int32_t *eu, const int32_t *ev)
{
    adj_t *g = (adj_t *)malloc(sizeof(adj_t));
    if (!g) return 0;
    if (build_adj(g, V, m, eu, ev)) {
        free(g->start);
        free(g->nbr);
        free(g);
        return 0;
    }
    return g;
}

void oracle_graph_free(void *h)
{
    adj_t *g = (adj_t *)h;
    if (!g) return;
    free(g->start);
    free(g->nbr);
    free(g);
}

int oracle_graph_bfs(void *h, const int32_t *sources, int64_t n_src, uint64_t *S_out, int32_t *k_out,
                     int nthreads, double *seconds)
{
    adj_t *g = (adj_t *)h;
    const int32_t V = g->V;
    for (int64_t i = 0; i < n_src; i++)
        if (sources[i] < 0 || sources[i] >= V) return -2;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
    double t0 = omp_get_wtime();
#else
    (void)nthreads;
#endif
    int err = 0;
#pragma omp parallel
    {
        int32_t *dist = (int32_t *)malloc(sizeof(int32_t) * (size_t)(V > 0 ? V : 1));
        int32_t *queue = (int32_t *)malloc(sizeof(int32_t) * (size_t)(V > 0 ? V : 1));
        if (!dist || !queue) {
#pragma omp atomic write
            err = -3;
        } else {
            for (int32_t v = 0; v < V; v++) dist[v] = -1;
#pragma omp for schedule(dynamic, 16)
            for (int64_t i = 0; i < n_src; i++)
                bfs_one(g, sources[i], dist, queue, &S_out[i], &k_out[i]);
        }
        free(dist);
        free(queue);
    }
#ifdef _OPENMP
    if (seconds) *seconds = omp_get_wtime() - t0;
#else
    if (seconds) *seconds = 0.0;
#endif
    return err;
}

/* number of OpenMP threads a parallel region would use (for reporting) */
int oracle_num_threads(int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
    int n = 1;
#pragma omp parallel
    {
#pragma omp single
        n = omp_get_num_threads();
    }
    return n;
#else
    (void)nthreads;
    return 1;
#endif
}

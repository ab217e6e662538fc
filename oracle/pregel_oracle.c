/*
 * pregel_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).
 *
 * A plain-C restatement of the reference `pregelite` package's superstep
 * semantics and of its independent validators, used by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * legs.  Nothing under paper_2010_01542_b200/ links or calls this file: the
 * product path is the CUDA library (libpgx.so) and fails loudly without it.
 *
 * Reference files (all under /root/reference/pkg/src/pregelite/):
 *   engine.py      _Executor.run 255-316, _next_frontier 349-365,
 *                  _chunk_push 402-414, _fold_chunk 425-457
 *   algorithms.py  pagerank 27-84, connected_components 87-113, sssp 116-152
 *   mailbox.py     min_combine / sum_combine 58-70, send_hybrid 180-199
 *   oracles.py     pagerank_reference 18-36, components_reference 39-66,
 *                  bfs_distances_reference 69-89
 *   graph.py       _csr 179-187 (rows sorted ascending, int64 offsets)
 *
 * Floating point: the reference folds PageRank shares with
 * numpy.add.reduceat (segment = first + pairwise(rest)) and sums the
 * dangling mass with ndarray.sum (pairwise over all elements).  Both
 * orders are reproduced exactly below (np_pairwise_sum), so the oracle is
 * bit-identical to the reference, pinned by tests/test_oracle.py.  Build
 * with -ffp-contract=off (no FMA contraction).
 *
 * The R-MAT generator follows SURVEY.md section 8(d) verbatim (the
 * reference ships no R-MAT; BASELINE.md section 3 holds the SHA-256 of the
 * CSR it must produce).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_UNREACHED 0xFFFFFFFFu

static void set_threads(int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------ */
/* numpy summation orders (numpy 2.x loops_utils pairwise sum)          */
/* ------------------------------------------------------------------ */

static double np_pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) +
                     ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
    }
}

/* ndarray.sum() of a contiguous float64 array */
double orc_np_sum(const double *a, int64_t n) { return 0.0 + np_pairwise_sum(a, n); }

/* one numpy.add.reduceat segment: first element + pairwise(rest) */
double orc_np_reduceat_segment(const double *a, int64_t n) {
    if (n <= 0) return 0.0;
    if (n == 1) return a[0];
    return a[0] + np_pairwise_sum(a + 1, n - 1);
}

/* ------------------------------------------------------------------ */
/* R-MAT generator                                     */
/* ------------------------------------------------------------------ */

uint64_t orc_splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* LSD radix sort of `n` keys using `bits` significant low bits. */
static void radix_sort_u64(uint64_t *keys, uint64_t *tmp, int64_t n, int bits) {
    const int D = 11, R = 1 << D;
    int passes = (bits + D - 1) / D;
    uint64_t *src = keys, *dst = tmp;
    int nt = 1;
#ifdef _OPENMP
    nt = omp_get_max_threads();
#endif
    int64_t *hist = (int64_t *)malloc(sizeof(int64_t) * (size_t)R * nt);
    for (int p = 0; p < passes; p++) {
        int shift = p * D;
        memset(hist, 0, sizeof(int64_t) * (size_t)R * nt);
#pragma omp parallel num_threads(nt)
        {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
            int64_t *h = hist + (size_t)R * t;
            for (int64_t i = lo; i < hi; i++) h[(src[i] >> shift) & (R - 1)]++;
        }
        /* exclusive offsets, digit-major then thread-major (stable) */
        int64_t run = 0;
        for (int d = 0; d < R; d++)
            for (int t = 0; t < nt; t++) {
                int64_t c = hist[(size_t)R * t + d];
                hist[(size_t)R * t + d] = run;
                run += c;
            }
#pragma omp parallel num_threads(nt)
        {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
            int64_t *h = hist + (size_t)R * t;
            for (int64_t i = lo; i < hi; i++) {
                uint64_t k = src[i];
                dst[h[(k >> shift) & (R - 1)]++] = k;
            }
        }
        uint64_t *s = src; src = dst; dst = s;
    }
    if (src != keys) memcpy(keys, src, sizeof(uint64_t) * (size_t)n);
    free(hist);
}

/*
 * Generate the R-MAT edge set.  `keys` must hold edge_factor * 2^scale
 * entries (twice that when symmetric).  Returns m, the number of distinct
 * directed edges; keys[0..m) are sorted ascending as src * 2^32 + dst.
 */
int64_t orc_rmat_keys(int scale, int64_t edge_factor, double a, double b,
                      double c, uint64_t seed, int symmetric, uint64_t *keys,
                      int threads) {
    set_threads(threads);
    const int64_t n = (int64_t)1 << scale;
    const int64_t draws = edge_factor * n;
    const double two53 = 9007199254740992.0;
    const uint64_t TA = (uint64_t)floor(a * two53);
    const uint64_t TAB = (uint64_t)floor((a + b) * two53);
    const uint64_t TABC = (uint64_t)floor((a + b + c) * two53);
    const uint64_t base = orc_splitmix64(seed);
    /* pass 1: draw, keep non-loops, packed as src << scale | dst */
    int nt = 1;
#ifdef _OPENMP
    nt = omp_get_max_threads();
#endif
    int64_t *cnt = (int64_t *)calloc((size_t)nt + 1, sizeof(int64_t));
#pragma omp parallel num_threads(nt)
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        int64_t lo = draws * t / nt, hi = draws * (t + 1) / nt, k = 0;
        for (int64_t i = lo; i < hi; i++) {
            uint64_t s = 0, d = 0;
            for (int l = 0; l < scale; l++) {
                uint64_t x = orc_splitmix64(base + (uint64_t)i * (uint64_t)scale + (uint64_t)l);
                uint64_t r = x >> 11;
                int q = r < TA ? 0 : r < TAB ? 1 : r < TABC ? 2 : 3;
                int bit = scale - 1 - l;
                if (q & 2) s |= (uint64_t)1 << bit;
                if (q & 1) d |= (uint64_t)1 << bit;
            }
            if (s != d) k++;
        }
        cnt[t + 1] = k;
    }
    for (int t = 0; t < nt; t++) cnt[t + 1] += cnt[t];
    const int64_t kept = cnt[nt];
#pragma omp parallel num_threads(nt)
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        int64_t lo = draws * t / nt, hi = draws * (t + 1) / nt, w = cnt[t];
        for (int64_t i = lo; i < hi; i++) {
            uint64_t s = 0, d = 0;
            for (int l = 0; l < scale; l++) {
                uint64_t x = orc_splitmix64(base + (uint64_t)i * (uint64_t)scale + (uint64_t)l);
                uint64_t r = x >> 11;
                int q = r < TA ? 0 : r < TAB ? 1 : r < TABC ? 2 : 3;
                int bit = scale - 1 - l;
                if (q & 2) s |= (uint64_t)1 << bit;
                if (q & 1) d |= (uint64_t)1 << bit;
            }
            if (s != d) {
                keys[w] = (s << scale) | d;
                if (symmetric) keys[kept + w] = (d << scale) | s;
                w++;
            }
        }
    }
    free(cnt);
    int64_t total = symmetric ? 2 * kept : kept;
    uint64_t *tmp = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(total ? total : 1));
    radix_sort_u64(keys, tmp, total, 2 * scale);
    free(tmp);
    /* dedup + widen to src * 2^32 + dst */
    int64_t m = 0;
    const uint64_t mask = ((uint64_t)1 << scale) - 1;
    for (int64_t i = 0; i < total; i++) {
        if (i && keys[i] == keys[i - 1]) continue;
        uint64_t k = keys[i];
        keys[m++] = ((k >> scale) << 32) | (k & mask);
    }
    return m;
}

/* sorted unique keys (src << 32 | dst) -> int64 offsets / int32 targets */
void orc_keys_to_csr(const uint64_t *keys, int64_t m, int64_t n,
                     int64_t *offsets, int32_t *targets) {
    memset(offsets, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t i = 0; i < m; i++) {
        offsets[(keys[i] >> 32) + 1]++;
        targets[i] = (int32_t)(keys[i] & 0xFFFFFFFFull);
    }
    for (int64_t v = 0; v < n; v++) offsets[v + 1] += offsets[v];
}

/* transpose; in-rows come out sorted by source id ascending (graph.py:185) */
void orc_transpose(int64_t n, const int64_t *off, const int32_t *tgt,
                   int64_t *in_off, int32_t *in_tgt) {
    int64_t m = off[n];
    memset(in_off, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t e = 0; e < m; e++) in_off[(int64_t)tgt[e] + 1]++;
    for (int64_t v = 0; v < n; v++) in_off[v + 1] += in_off[v];
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    memcpy(cur, in_off, sizeof(int64_t) * (size_t)n);
    for (int64_t u = 0; u < n; u++)
        for (int64_t e = off[u]; e < off[u + 1]; e++)
            in_tgt[cur[tgt[e]]++] = (int32_t)u;
    free(cur);
}

/* ------------------------------------------------------------------ */
/* Engine restatement: per-step stats layout                             */
/*   stats[3*s + 0] = active_count  (SuperstepStats.active_count)        */
/*   stats[3*s + 1] = messages_sent (SuperstepStats.messages_sent)       */
/*   stats[3*s + 2] = edges traversed by this step's senders (GTEPS)     */
/*   hdr[0] = superstep_count, hdr[1] = hit_superstep_cap                */
/* ------------------------------------------------------------------ */


static inline void atomic_min_u32(uint32_t *p, uint32_t v) {
    uint32_t old = __atomic_load_n(p, __ATOMIC_RELAXED);
    while (v < old &&
           !__atomic_compare_exchange_n(p, &old, v, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
    }
}

/* ascending ids of set flags (np.flatnonzero), clearing them as it goes */
static int64_t take_flags(uint8_t *flags, int64_t n, int64_t *out) {
    int64_t k = 0;
    for (int64_t v = 0; v < n; v++)
        if (flags[v]) { out[k++] = v; flags[v] = 0; }
    return k;
}

/*
 * SSSP: push mode, min combiner, double-buffered mailbox
 * (algorithms.py:116-152 on engine.py:255-316, 402-414; mailbox.py:180-199,
 * 250-260).  Every compute votes to halt, so the next frontier is exactly
 * the set of vertices holding a pending message (engine.py:349-355).
 */
int orc_run_sssp(int64_t n, const int64_t *off, const int32_t *tgt,
                 int64_t source, int64_t max_steps, int threads,
                 uint32_t *dist, int64_t *stats, int64_t *hdr) {
    set_threads(threads);
    if (source < 0 || source >= n) return -1;   /* ConfigError in setup */
    if (max_steps < 1) return -2;
    uint32_t *mail[2];
    uint8_t *flag[2];
    for (int p = 0; p < 2; p++) {
        mail[p] = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
        flag[p] = (uint8_t *)calloc((size_t)n, 1);
        for (int64_t v = 0; v < n; v++) mail[p][v] = ORC_UNREACHED;
    }
    int64_t *front = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t v = 0; v < n; v++) dist[v] = ORC_UNREACHED;
    int cur = 0;
    int64_t nf = n, step = 0, hit_cap = 1;
    for (step = 0; step < max_steps; step++) {
        uint32_t *cm = mail[cur], *nm = mail[cur ^ 1];
        uint8_t *nfl = flag[cur ^ 1];
        int64_t sent = 0;
        if (step == 0) {
            dist[source] = 0;
            for (int64_t e = off[source]; e < off[source + 1]; e++) {
                atomic_min_u32(&nm[tgt[e]], 1u);
                nfl[tgt[e]] = 1;
            }
            sent = off[source + 1] - off[source];
        } else {
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : sent)
            for (int64_t i = 0; i < nf; i++) {
                int64_t v = front[i];
                uint32_t m = cm[v];
                cm[v] = ORC_UNREACHED;       /* consume (slot reset) */
                if (m < dist[v]) {
                    dist[v] = m;
                    for (int64_t e = off[v]; e < off[v + 1]; e++) {
                        atomic_min_u32(&nm[tgt[e]], m + 1);
                        __atomic_store_n(&nfl[tgt[e]], 1, __ATOMIC_RELAXED);
                    }
                    sent += off[v + 1] - off[v];
                }
            }
        }
        stats[3 * step + 0] = nf;
        stats[3 * step + 1] = sent;
        stats[3 * step + 2] = sent;
        nf = take_flags(nfl, n, front);
        if (nf == 0) { hit_cap = 0; step++; break; }
        cur ^= 1;
    }
    for (int p = 0; p < 2; p++) { free(mail[p]); free(flag[p]); }
    free(front);
    hdr[0] = step; hdr[1] = hit_cap;
    return 0;
}

/* mark every out-neighbour of the vertices in pub[0..np) (engine.py:356-365) */
static void wake_out_neighbours(const int64_t *off, const int32_t *tgt,
                                const int64_t *pub, int64_t np, uint8_t *woken) {
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < np; i++) {
        int64_t u = pub[i];
        for (int64_t e = off[u]; e < off[u + 1]; e++)
            __atomic_store_n(&woken[tgt[e]], 1, __ATOMIC_RELAXED);
    }
}

/*
 * Hashmin connected components: pull mode, min fold over flagged
 * in-neighbours (algorithms.py:87-113; engine.py:416-457 fold,
 * 349-365 frontier).  labels are int64 like the reference state dtype.
 */
int orc_run_cc(int64_t n, const int64_t *off, const int32_t *tgt,
               const int64_t *in_off, const int32_t *in_tgt, int64_t max_steps,
               int threads, int64_t *labels, int64_t *stats, int64_t *hdr) {
    set_threads(threads);
    if (max_steps < 1) return -2;
    int64_t *val[2];
    uint8_t *flag[2];
    for (int p = 0; p < 2; p++) {
        val[p] = (int64_t *)calloc((size_t)(n ? n : 1), sizeof(int64_t));
        flag[p] = (uint8_t *)calloc((size_t)(n ? n : 1), 1);
    }
    int64_t *front = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t *pub = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    uint8_t *woken = (uint8_t *)calloc((size_t)(n ? n : 1), 1);
    for (int64_t v = 0; v < n; v++) { labels[v] = v; front[v] = v; }
    int cur = 0;
    int64_t nf = n, step = 0, hit_cap = 1;
    for (step = 0; step < max_steps; step++) {
        int64_t *cv = val[cur], *nv = val[cur ^ 1];
        uint8_t *cf = flag[cur], *nfl = flag[cur ^ 1];
        int64_t sent = 0, edges = 0;
        if (step == 0) {
            for (int64_t v = 0; v < n; v++) { nv[v] = labels[v]; nfl[v] = 1; }
            sent = n;
            edges = off[n];
        } else {
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : sent, edges)
            for (int64_t i = 0; i < nf; i++) {
                int64_t v = front[i];
                int have = 0;
                int64_t m = 0;
                for (int64_t e = in_off[v]; e < in_off[v + 1]; e++) {
                    int32_t u = in_tgt[e];
                    if (cf[u]) {
                        if (!have || cv[u] < m) m = cv[u];
                        have = 1;
                    }
                }
                if (have && m < labels[v]) {
                    labels[v] = m;
                    nv[v] = m;
                    nfl[v] = 1;
                    sent += 1;
                    edges += off[v + 1] - off[v];
                }
            }
        }
        stats[3 * step + 0] = nf;
        stats[3 * step + 1] = sent;
        stats[3 * step + 2] = edges;
        /* publishers = flagged in the next buffer, ascending */
        int64_t np = 0;
        for (int64_t v = 0; v < n; v++) if (nfl[v]) pub[np++] = v;
        wake_out_neighbours(off, tgt, pub, np, woken);
        nf = take_flags(woken, n, front);
        if (nf == 0) { hit_cap = 0; step++; break; }
        /* swap_buffers: retire current (clear its flags), flip parity */
        memset(cf, 0, (size_t)n);
        cur ^= 1;
    }
    for (int p = 0; p < 2; p++) { free(val[p]); free(flag[p]); }
    free(front); free(pub); free(woken);
    hdr[0] = step; hdr[1] = hit_cap;
    return 0;
}

/*
 * PageRank: pull mode, sum fold in in-adjacency order with numpy's
 * reduceat rounding, dangling mass re-summed with ndarray.sum rounding
 * after every superstep (algorithms.py:27-84; engine.py:425-457).
 * Exactly `iterations` supersteps unless max_steps caps the run.
 */
int orc_run_pagerank(int64_t n, const int64_t *off, const int32_t *tgt,
                     const int64_t *in_off, const int32_t *in_tgt,
                     int64_t iterations, double damping, int64_t max_steps,
                     int threads, double *rank, int64_t *stats, int64_t *hdr) {
    set_threads(threads);
    if (iterations < 1 || !(damping >= 0.0 && damping <= 1.0)) return -1;
    if (max_steps < 1) return -2;
    if (n == 0) {   /* one empty superstep: nothing flagged, all halted */
        stats[0] = stats[1] = stats[2] = 0;
        hdr[0] = 1; hdr[1] = 0;
        return 0;
    }
    const double base = (1.0 - damping) / (double)n;
    const double r0 = 1.0 / (double)n;
    const int64_t last = iterations - 1;
    double *val[2];
    uint8_t *flag[2];
    for (int p = 0; p < 2; p++) {
        val[p] = (double *)calloc((size_t)n, sizeof(double));
        flag[p] = (uint8_t *)calloc((size_t)n, 1);
    }
    int64_t nd = 0;
    for (int64_t v = 0; v < n; v++) {
        rank[v] = r0;
        int64_t d = off[v + 1] - off[v];
        if (d > 0) { val[0][v] = r0 / (double)d; flag[0][v] = 1; }
        else nd++;
    }
    int64_t *dmask = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nd ? nd : 1));
    double *dvals = (double *)malloc(sizeof(double) * (size_t)(nd ? nd : 1));
    {
        int64_t k = 0;
        for (int64_t v = 0; v < n; v++) if (off[v + 1] == off[v]) dmask[k++] = v;
    }
    double dangling = r0 * (double)nd;
    int cur = 0;
    int64_t step = 0, hit_cap = 1;
    int64_t max_in = 0;
    for (int64_t v = 0; v < n; v++)
        if (in_off[v + 1] - in_off[v] > max_in) max_in = in_off[v + 1] - in_off[v];
    for (step = 0; step < max_steps; step++) {
        double *cv = val[cur], *nv = val[cur ^ 1];
        uint8_t *cf = flag[cur], *nfl = flag[cur ^ 1];
        int64_t sent = 0, edges = 0;
        const double dn = dangling / (double)n;
#pragma omp parallel reduction(+ : sent, edges)
        {
            double *seg = (double *)malloc(sizeof(double) * (size_t)(max_in ? max_in : 1));
#pragma omp for schedule(dynamic, 256)
            for (int64_t v = 0; v < n; v++) {
                int64_t k = 0;
                for (int64_t e = in_off[v]; e < in_off[v + 1]; e++) {
                    int32_t u = in_tgt[e];
                    if (cf[u]) seg[k++] = cv[u];
                }
                edges += k;
                double folded = k ? orc_np_reduceat_segment(seg, k) : 0.0;
                double r = base + damping * (folded + dn);
                rank[v] = r;
                if (step != last) {
                    int64_t d = off[v + 1] - off[v];
                    if (d) { nv[v] = r / (double)d; nfl[v] = 1; sent += 1; }
                }
            }
            free(seg);
        }
        stats[3 * step + 0] = n;
        stats[3 * step + 1] = sent;
        stats[3 * step + 2] = edges;
        for (int64_t i = 0; i < nd; i++) dvals[i] = rank[dmask[i]];
        dangling = orc_np_sum(dvals, nd);
        memset(cf, 0, (size_t)n);
        if (step == last) { hit_cap = 0; step++; break; }
        cur ^= 1;
    }
    for (int p = 0; p < 2; p++) { free(val[p]); free(flag[p]); }
    free(dmask); free(dvals);
    hdr[0] = step; hdr[1] = hit_cap;
    return 0;
}

/* ------------------------------------------------------------------ */
/* Independent validators (oracles.py)                                  */
/* ------------------------------------------------------------------ */

static int64_t uf_find(int64_t *parent, int64_t x) {
    while (parent[x] != x) {
        parent[x] = parent[parent[x]];   /* path halving */
        x = parent[x];
    }
    return x;
}

/* components_reference (oracles.py:39-66): union-find, min-id labels */
void orc_components_ref(int64_t n, int64_t m, const int64_t *src,
                        const int64_t *dst, int64_t *labels) {
    int64_t *parent = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    for (int64_t v = 0; v < n; v++) parent[v] = v;
    for (int64_t e = 0; e < m; e++) {
        int64_t ra = uf_find(parent, src[e]), rb = uf_find(parent, dst[e]);
        if (ra != rb) {
            if (ra < rb) parent[rb] = ra; else parent[ra] = rb;
        }
    }
    int64_t *mins = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    for (int64_t v = 0; v < n; v++) { labels[v] = uf_find(parent, v); mins[v] = n; }
    for (int64_t v = 0; v < n; v++) if (v < mins[labels[v]]) mins[labels[v]] = v;
    for (int64_t v = 0; v < n; v++) labels[v] = mins[labels[v]];
    free(parent); free(mins);
}

/* bfs_distances_reference (oracles.py:69-89): level scans over the edge list */
int orc_bfs_ref(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                int64_t source, uint32_t *dist) {
    if (source < 0 || source >= n) return -1;
    for (int64_t v = 0; v < n; v++) dist[v] = ORC_UNREACHED;
    dist[source] = 0;
    uint32_t level = 0;
    uint8_t *fresh = (uint8_t *)calloc((size_t)n, 1);
    for (;;) {
        int any_front = 0, any_fresh = 0;
        for (int64_t e = 0; e < m; e++) {
            if (dist[src[e]] == level) {
                any_front = 1;
                if (dist[dst[e]] == ORC_UNREACHED) { fresh[dst[e]] = 1; any_fresh = 1; }
            }
        }
        if (!any_front || !any_fresh) break;
        for (int64_t v = 0; v < n; v++)
            if (fresh[v]) { dist[v] = level + 1; fresh[v] = 0; }
        level++;
    }
    free(fresh);
    return 0;
}

/* pagerank_reference (oracles.py:18-36): bincount fold in edge order */
void orc_pagerank_ref(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                      int64_t iterations, double damping, double *rank) {
    if (n == 0) return;
    double *outdeg = (double *)calloc((size_t)n, sizeof(double));
    double *share = (double *)calloc((size_t)n, sizeof(double));
    double *pulled = (double *)calloc((size_t)n, sizeof(double));
    int64_t nd = 0;
    for (int64_t e = 0; e < m; e++) outdeg[src[e]] += 1.0;
    for (int64_t v = 0; v < n; v++) { rank[v] = 1.0 / (double)n; if (outdeg[v] == 0.0) nd++; }
    double *dv = (double *)malloc(sizeof(double) * (size_t)(nd ? nd : 1));
    const double base = (1.0 - damping) / (double)n;
    for (int64_t it = 0; it < iterations; it++) {
        for (int64_t v = 0; v < n; v++) {
            share[v] = outdeg[v] > 0.0 ? rank[v] / outdeg[v] : 0.0;
            pulled[v] = 0.0;
        }
        for (int64_t e = 0; e < m; e++) pulled[dst[e]] += share[src[e]];
        int64_t k = 0;
        for (int64_t v = 0; v < n; v++) if (outdeg[v] == 0.0) dv[k++] = rank[v];
        double dangling = orc_np_sum(dv, nd);
        double dn = dangling / (double)n;
        for (int64_t v = 0; v < n; v++) rank[v] = base + damping * (pulled[v] + dn);
    }
    free(outdeg); free(share); free(pulled); free(dv);
}

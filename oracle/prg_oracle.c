/*
 * prg_oracle.c — CPU restatement of the reference's K0/K1/K2/K3 algorithms.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_1603_01876_b200/,
 * include/) links or calls this file; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs load it, and only as the
 * checker or the CPU baseline. Parity is PINNED: tests/test_oracle_pins.py
 * checks this restatement against the reference's own known-answer tests and
 * against golden vectors produced by the reference itself (oracle/_ref, built
 * from /root/reference sources by oracle/build_ref.sh; see tests/golden/).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Compiled with -O2 -ffp-contract=off so fp64 results
 * follow the reference's separate mul/add evaluation exactly.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ---- RNG: include/prpipe/rng.hpp:10-37 -------------------------------- */
static inline uint64_t sm_next(uint64_t *state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);            /* rng.hpp:15 */
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;              /* rng.hpp:16 */
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;              /* rng.hpp:17 */
    return z ^ (z >> 31);                                     /* rng.hpp:18 */
}
static inline double sm_unit(uint64_t *s) {                   /* rng.hpp:22 */
    return (double)(sm_next(s) >> 11) * 0x1.0p-53;
}
uint64_t oracle_mix_seed(uint64_t seed, uint64_t stream) {     /* rng.hpp:33-37 */
    uint64_t s = seed ^ (0x9e3779b97f4a7c15ULL * (stream + 1));
    sm_next(&s);
    return sm_next(&s);
}

/* ---- K0 generator: src/graph_gen.cpp:60-111 ------------------------------ */
#define PERM_STREAM 0x7065726d75746174ULL                     /* graph_gen.cpp:16 */

/* labels[n] := Fisher–Yates permutation of 1..n (graph_gen.cpp:66-76). */
void oracle_permutation(int64_t n, uint64_t seed, int64_t *labels) {
    for (int64_t i = 0; i < n; ++i) labels[i] = i + 1;
    uint64_t s = oracle_mix_seed(seed, PERM_STREAM);
    for (int64_t i = n - 1; i > 0; --i) {
        int64_t j = (int64_t)(sm_next(&s) % ((uint64_t)i + 1));
        int64_t t = labels[i]; labels[i] = labels[j]; labels[j] = t;
    }
}

/* Edges [first, first+count) of the K0 list into uv[2*k], uv[2*k+1]
 * (graph_gen.cpp:83-99). labels may be NULL (permute_labels=false). */
void oracle_make_edges(int scale, uint64_t seed, const double init[4], const int64_t *labels,
                       int64_t first, int64_t count, int64_t *uv) {
    const double a = init[0];
    const double ab = a + init[1];
    const double abc = ab + init[2];
    for (int64_t k = 0; k < count; ++k) {
        uint64_t s = oracle_mix_seed(seed, (uint64_t)(first + k));
        int64_t u = 0, v = 0;
        for (int level = 0; level < scale; ++level) {
            double x = sm_unit(&s);
            int q = x < a ? 0 : x < ab ? 1 : x < abc ? 2 : 3;
            u = (u << 1) | (q >> 1);
            v = (v << 1) | (q & 1);
        }
        if (labels) { uv[2 * k] = labels[u]; uv[2 * k + 1] = labels[v]; }
        else { uv[2 * k] = u + 1; uv[2 * k + 1] = v + 1; }
    }
}

/* ---- K1: sort by start vertex (src/kernel1_sort.cpp:63-68) ----------------
 * The reference uses std::sort with a u-only comparator (kernel1_sort.cpp:14,66)
 * whose tie order is unspecified (kernel1_sort.hpp:23). The oracle emits the
 * canonical order — ties broken by v — which is the reference's own test
 * canonicalizer (tests/helpers.hpp:29-34). LSD radix on (u-1)<<S | (v-1). */
int oracle_k1_sort(const int64_t *uv_in, int64_t m, int scale, int64_t *uv_out) {
    if (m == 0) return 0;
    uint64_t *k0 = (uint64_t *)malloc((size_t)m * 8), *k1 = (uint64_t *)malloc((size_t)m * 8);
    size_t *cnt = (size_t *)malloc(sizeof(size_t) * 65536);
    if (!k0 || !k1 || !cnt) { free(k0); free(k1); free(cnt); return -2; }
    const int64_t n = (int64_t)1 << scale;
    for (int64_t i = 0; i < m; ++i) {
        int64_t u = uv_in[2 * i], v = uv_in[2 * i + 1];
        if (u < 1 || u > n || v < 1 || v > n) { free(k0); free(k1); free(cnt); return -1; }
        k0[i] = ((uint64_t)(u - 1) << scale) | (uint64_t)(v - 1);
    }
    const int bits = 2 * scale;
    for (int shift = 0; shift < bits; shift += 16) {
        memset(cnt, 0, sizeof(size_t) * 65536);
        for (int64_t i = 0; i < m; ++i) cnt[(k0[i] >> shift) & 0xffff]++;
        size_t run = 0;
        for (int d = 0; d < 65536; ++d) { size_t c = cnt[d]; cnt[d] = run; run += c; }
        for (int64_t i = 0; i < m; ++i) k1[cnt[(k0[i] >> shift) & 0xffff]++] = k0[i];
        uint64_t *t = k0; k0 = k1; k1 = t;
    }
    const uint64_t mask = ((uint64_t)1 << scale) - 1;
    for (int64_t i = 0; i < m; ++i) {
        uv_out[2 * i] = (int64_t)(k0[i] >> scale) + 1;
        uv_out[2 * i + 1] = (int64_t)(k0[i] & mask) + 1;
    }
    free(k0); free(k1); free(cnt);
    return 0;
}

/* ---- K2: src/kernel2_filter.cpp -------------------------------------------
 * build_from (:12-54): streaming CSR from u-sorted edges; each row's pending
 * v list is sorted and run-length encoded. Returns nnz, or -1 (label outside
 * [1,n]), -2 (not sorted by start vertex), -3 (n <= 0).
 * Buffers cols/counts must hold m entries; row_offsets n+1. */
static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}
int64_t oracle_build_adjacency(const int64_t *uv, int64_t m, int64_t n, int64_t *row_offsets,
                               int64_t *cols, int64_t *counts) {
    if (n <= 0) return -3;
    int64_t nnz = 0, open_row = 0, pend_beg = 0;
    int64_t *pending = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    int64_t npend = 0;
    memset(row_offsets, 0, sizeof(int64_t) * (size_t)(n + 1));
    (void)pend_beg;
#define CLOSE_THROUGH(next_row)                                                        \
    do {                                                                               \
        if (npend) {                                                                   \
            qsort(pending, (size_t)npend, sizeof(int64_t), cmp_i64);                   \
            for (int64_t i = 0; i < npend;) {                                          \
                int64_t j = i + 1;                                                     \
                while (j < npend && pending[j] == pending[i]) ++j;                     \
                cols[nnz] = pending[i]; counts[nnz] = j - i; ++nnz; i = j;             \
            }                                                                          \
            npend = 0;                                                                 \
        }                                                                              \
        for (int64_t r = open_row; r < (next_row); ++r) row_offsets[r + 1] = nnz;      \
        open_row = (next_row);                                                         \
    } while (0)
    for (int64_t i = 0; i < m; ++i) {
        int64_t u = uv[2 * i], v = uv[2 * i + 1];
        if (u < 1 || u > n || v < 1 || v > n) { free(pending); return -1; }   /* :41-43 */
        int64_t row = u - 1;
        if (row < open_row) { free(pending); return -2; }                      /* :45-47 */
        if (row > open_row) CLOSE_THROUGH(row);
        pending[npend++] = v - 1;
    }
    CLOSE_THROUGH(n);
#undef CLOSE_THROUGH
    free(pending);
    return nnz;
}

/* in_degree (:101-106). */
void oracle_in_degree(int64_t n, int64_t nnz, const int64_t *cols, const int64_t *counts,
                      int64_t *d_in) {
    memset(d_in, 0, sizeof(int64_t) * (size_t)n);
    for (int64_t k = 0; k < nnz; ++k) d_in[cols[k]] += counts[k];
}

/* zero_columns (:108-132); in place is allowed (out may alias in). Returns nnz. */
int64_t oracle_zero_columns(int64_t n, const int64_t *row_offsets, const int64_t *cols,
                            const int64_t *counts, const int64_t *d_in, int64_t *out_offsets,
                            int64_t *out_cols, int64_t *out_counts) {
    int64_t max_in = 0;
    for (int64_t c = 0; c < n; ++c) if (d_in[c] > max_in) max_in = d_in[c];
    int64_t w = 0, beg = row_offsets[0];
    out_offsets[0] = 0;
    for (int64_t row = 0; row < n; ++row) {
        int64_t end = row_offsets[row + 1];
        for (int64_t k = beg; k < end; ++k) {
            int64_t d = d_in[cols[k]];
            if (d == max_in || d == 1) continue;
            out_cols[w] = cols[k]; out_counts[w] = counts[k]; ++w;
        }
        beg = end;
        out_offsets[row + 1] = w;
    }
    return w;
}

/* row_normalize (:134-152). */
void oracle_row_normalize(int64_t n, const int64_t *row_offsets, const int64_t *counts,
                          double *values) {
    for (int64_t row = 0; row < n; ++row) {
        int64_t b = row_offsets[row], e = row_offsets[row + 1], d = 0;
        for (int64_t k = b; k < e; ++k) d += counts[k];
        if (d == 0) continue;
        for (int64_t k = b; k < e; ++k) values[k] = (double)counts[k] / (double)d;
    }
}

/* Whole K2 core (run_kernel2 minus file I/O, :154-168). Outputs the filtered
 * stochastic CSR and the pre-filter d_in. Returns nnz_f or a negative error. */
int64_t oracle_k2(const int64_t *uv, int64_t m, int64_t n, int64_t *row_offsets, int64_t *cols,
                  double *values, int64_t *d_in, int64_t *nnz_raw_out) {
    int64_t *ro = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t *cc = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    int64_t *cn = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    int64_t nnz = oracle_build_adjacency(uv, m, n, ro, cc, cn);
    if (nnz < 0) { free(ro); free(cc); free(cn); return nnz; }
    if (nnz_raw_out) *nnz_raw_out = nnz;
    oracle_in_degree(n, nnz, cc, cn, d_in);
    int64_t nf = oracle_zero_columns(n, ro, cc, cn, d_in, row_offsets, cols, cn);
    oracle_row_normalize(n, row_offsets, cn, values);
    free(ro); free(cc); free(cn);
    return nf;
}

/* ---- K3: src/kernel3_pagerank.cpp -----------------------------------------
 * sum_of (:17-19) is a left-to-right std::accumulate. mode 0 restates it
 * exactly; mode 1 replaces it with a Neumaier compensated sum — the
 * "accurate-sum" oracle used to attribute drift. */
#define RANK_STREAM 0x72616e6b696e6974ULL                     /* kernel3_pagerank.cpp:15 */

static double sum_seq(const double *x, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += x[i];
    return s;
}
static double sum_neumaier(const double *x, int64_t n) {
    double s = 0.0, c = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double t = s + x[i];
        if (fabs(s) >= fabs(x[i])) c += (s - t) + x[i];
        else c += (x[i] - t) + s;
        s = t;
    }
    return s + c;
}
static double sum_mode(const double *x, int64_t n, int mode) {
    return mode ? sum_neumaier(x, n) : sum_seq(x, n);
}

/* init_rank (:29-39); returns norm1. */
double oracle_init_rank(int64_t n, uint64_t seed, double *r, int mode) {
    uint64_t s = oracle_mix_seed(seed, RANK_STREAM);
    for (int64_t i = 0; i < n; ++i) r[i] = sm_unit(&s);
    double sum = sum_mode(r, n, mode);
    for (int64_t i = 0; i < n; ++i) r[i] /= sum;
    return sum_mode(r, n, mode);
}

/* pagerank_step (:41-65): push scatter over the CSR; returns norm1. */
double oracle_pagerank_step(int64_t n, const int64_t *row_offsets, const int64_t *cols,
                            const double *values, const double *r, double damping, double *out,
                            int mode) {
    const double total = sum_mode(r, n, mode);                       /* :45 */
    const double background = (1.0 - damping) / (double)n * total;   /* :46 */
    memset(out, 0, sizeof(double) * (size_t)n);
    for (int64_t u = 0; u < n; ++u) {                                /* :49-57 */
        const double ru = r[u];
        if (ru == 0.0) continue;
        for (int64_t k = row_offsets[u]; k < row_offsets[u + 1]; ++k) out[cols[k]] += ru * values[k];
    }
    for (int64_t i = 0; i < n; ++i) out[i] = damping * out[i] + background;  /* :58-61 */
    return sum_mode(out, n, mode);                                   /* :59-62 */
}

/* run_kernel3 minus the timer (:67-79): init + `iterations` steps. */
double oracle_run_kernel3(int64_t n, const int64_t *row_offsets, const int64_t *cols,
                          const double *values, double damping, int iterations, uint64_t seed,
                          double *ranks, int mode) {
    double *tmp = (double *)malloc(sizeof(double) * (size_t)n);
    double norm = oracle_init_rank(n, seed, ranks, mode);
    for (int it = 0; it < iterations; ++it) {
        norm = oracle_pagerank_step(n, row_offsets, cols, values, ranks, damping, tmp, mode);
        memcpy(ranks, tmp, sizeof(double) * (size_t)n);
    }
    free(tmp);
    return norm;
}

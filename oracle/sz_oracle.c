/*
 * TEST INFRASTRUCTURE ONLY. This file is the CPU oracle ("port") for the
 * Store-zechin hot path. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it, and only as the checker
 * (or the timed CPU baseline), never as the product path.
 *
 * It restates the reference's memoised last-row development
 * (reference proj/src/permanent.cpp) as a layered dynamic programme:
 *   - layer k holds per(S) for every column subset S, |S| = k, over the
 *     leading k rows (permanent.cpp:138-139, "per(S) over the leading |S|
 *     rows and column set S, developed along row |S|");
 *   - order-2 base case a(0,j1)a(1,j2) + a(0,j2)a(1,j1), j1 < j2
 *     (permanent.cpp:158-162);
 *   - expansion per(S) = sum over j in S ascending of a(|S|-1, j) *
 *     per(S \ {j}), the first term initialising the accumulator and each later
 *     term added left to right (permanent.cpp:164-175);
 *   - top level sum_j a(n-1, j) * per(full \ {j}) for j = 0..n-1, the terms
 *     summed left to right (permanent.cpp:184-198);
 *   - n = 1 returns a[0]; n = 2 is the base case (permanent.cpp:260-266).
 * The memo table is replaced by colex-ranked layer arrays (each distinct
 * subset is still evaluated exactly once), which is what makes n = 32
 * reachable on the CPU; the arithmetic sequence per subset is unchanged, so
 * with -ffp-contract=off the double / complex results are bitwise those of
 * the reference engine (pinned in tests/test_oracle.py against oracle/_ref).
 *
 * Integers are computed in checked signed 128-bit arithmetic (the reference
 * uses arbitrary precision, ring.hpp:31); a result that leaves 128 bits is
 * reported as overflow instead of wrapping.
 *
 * Colex ranking: rank(S) = sum_{i=1..k} C(s_i, i) for s_1 < ... < s_k, so
 * increasing bitmask order is colex order. Removing s_i gives
 * rank = sum_{l<i} C(s_l, l) + sum_{l>i} C(s_l, l-1).
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

#define MAXN 40
static uint64_t g_binom[MAXN + 1][MAXN + 1];
static int g_binom_ready = 0;

static void binom_init(void) {
    if (g_binom_ready) return;
    for (int s = 0; s <= MAXN; ++s) {
        g_binom[s][0] = 1;
        for (int l = 1; l <= MAXN; ++l) {
            g_binom[s][l] = s == 0 ? 0 : g_binom[s - 1][l - 1] + g_binom[s - 1][l];
        }
    }
    g_binom_ready = 1;
}

uint64_t orc_binom(int s, int l) {
    binom_init();
    if (s < 0 || l < 0 || s > MAXN || l > MAXN) return 0;
    return g_binom[s][l];
}

uint64_t orc_colex_rank(uint64_t mask) {
    binom_init();
    uint64_t r = 0;
    int i = 1;
    while (mask) {
        const int s = __builtin_ctzll(mask);
        r += g_binom[s][i++];
        mask &= mask - 1;
    }
    return r;
}

uint64_t orc_colex_unrank(int k, uint64_t rank) {
    binom_init();
    uint64_t mask = 0;
    int s = MAXN;
    for (int i = k; i >= 1; --i) {
        while (g_binom[s][i] > rank) --s;
        mask |= 1ULL << s;
        rank -= g_binom[s][i];
        --s;
    }
    return mask;
}

static inline uint64_t gosper_next(uint64_t x) {
    const uint64_t c = x & (~x + 1);
    const uint64_t r = x + c;
    return (((r ^ x) >> 2) / c) | r;
}

/* Predecessor ranks for the k elements of `mask` (ascending), plus the
 * elements themselves. */
static inline void preds_of(uint64_t mask, int k, int* elem, uint64_t* pred) {
    int i = 0;
    for (uint64_t m = mask; m; m &= m - 1) elem[i++] = __builtin_ctzll(m);
    uint64_t suffix = 0; /* sum_{l>1} C(s_l, l-1), 1-based positions */
    for (int l = 2; l <= k; ++l) suffix += g_binom[elem[l - 1]][l - 1];
    uint64_t prefix = 0;
    for (int p = 1; p <= k; ++p) {
        pred[p - 1] = prefix + suffix;
        prefix += g_binom[elem[p - 1]][p];
        if (p < k) suffix -= g_binom[elem[p]][p];
    }
}

/* ---------------------------------------------------------------- int128 */

static int dp_i128(int n, const int64_t* a, i128* out, int nthreads) {
    binom_init();
    if (n == 1) {
        *out = a[0];
        return 0;
    }
    const int64_t pairs = (int64_t)g_binom[n][2];
    if (n == 2) {
        i128 x, y, s;
        int ov = __builtin_mul_overflow((i128)a[0], (i128)a[3], &x);
        ov |= __builtin_mul_overflow((i128)a[1], (i128)a[2], &y);
        ov |= __builtin_add_overflow(x, y, &s);
        *out = s;
        return ov ? 2 : 0;
    }
    uint64_t maxlayer = 0;
    for (int k = 2; k < n; ++k) maxlayer = g_binom[n][k] > maxlayer ? g_binom[n][k] : maxlayer;
    i128* prev = (i128*)malloc(sizeof(i128) * maxlayer);
    i128* cur = (i128*)malloc(sizeof(i128) * maxlayer);
    if (!prev || !cur) {
        free(prev);
        free(cur);
        return 3;
    }
    int overflow = 0;
    /* layer 2 */
    for (int j2 = 1; j2 < n; ++j2) {
        for (int j1 = 0; j1 < j2; ++j1) {
            i128 x, y, s;
            int ov = __builtin_mul_overflow((i128)a[j1], (i128)a[n + j2], &x);
            ov |= __builtin_mul_overflow((i128)a[j2], (i128)a[n + j1], &y);
            ov |= __builtin_add_overflow(x, y, &s);
            overflow |= ov;
            prev[j1 + (uint64_t)j2 * (j2 - 1) / 2] = s;
        }
    }
    (void)pairs;
    for (int k = 3; k < n; ++k) {
        const int64_t cnt = (int64_t)g_binom[n][k];
        const int64_t* row = a + (size_t)(k - 1) * n;
        const int64_t chunk = 1024;
#pragma omp parallel for schedule(static) num_threads(nthreads) reduction(| : overflow)
        for (int64_t c0 = 0; c0 < cnt; c0 += chunk) {
            const int64_t c1 = c0 + chunk < cnt ? c0 + chunk : cnt;
            uint64_t mask = orc_colex_unrank(k, (uint64_t)c0);
            int elem[MAXN];
            uint64_t pred[MAXN];
            for (int64_t r = c0; r < c1; ++r) {
                preds_of(mask, k, elem, pred);
                i128 acc = 0;
                for (int p = 0; p < k; ++p) {
                    i128 t;
                    overflow |= __builtin_mul_overflow((i128)row[elem[p]], prev[pred[p]], &t);
                    if (p == 0) {
                        acc = t;
                    } else {
                        overflow |= __builtin_add_overflow(acc, t, &acc);
                    }
                }
                cur[r] = acc;
                if (r + 1 < c1) mask = gosper_next(mask);
            }
        }
        i128* t = prev;
        prev = cur;
        cur = t;
    }
    const int64_t* last = a + (size_t)(n - 1) * n;
    i128 total = 0;
    for (int j = 0; j < n; ++j) {
        i128 t;
        overflow |= __builtin_mul_overflow((i128)last[j], prev[n - 1 - j], &t);
        if (j == 0) {
            total = t;
        } else {
            overflow |= __builtin_add_overflow(total, t, &total);
        }
    }
    free(prev);
    free(cur);
    *out = total;
    return overflow ? 2 : 0;
}

/* ---------------------------------------------------------------- double / complex */

typedef struct {
    double re, im;
} cplx;

static inline cplx cmul(cplx x, cplx y) {
    cplx r;
    r.re = x.re * y.re - x.im * y.im;
    r.im = x.re * y.im + x.im * y.re;
    return r;
}
static inline cplx cadd(cplx x, cplx y) {
    cplx r;
    r.re = x.re + y.re;
    r.im = x.im + y.im;
    return r;
}

#define DEFINE_DP(NAME, T, MUL, ADD)                                                          \
    static int NAME(int n, const T* a, T* out, int nthreads) {                                \
        binom_init();                                                                         \
        if (n == 1) {                                                                         \
            *out = a[0];                                                                      \
            return 0;                                                                         \
        }                                                                                     \
        if (n == 2) {                                                                         \
            *out = ADD(MUL(a[0], a[3]), MUL(a[1], a[2]));                                     \
            return 0;                                                                         \
        }                                                                                     \
        uint64_t maxlayer = 0;                                                                \
        for (int k = 2; k < n; ++k) maxlayer = g_binom[n][k] > maxlayer ? g_binom[n][k] : maxlayer; \
        T* prev = (T*)malloc(sizeof(T) * maxlayer);                                           \
        T* cur = (T*)malloc(sizeof(T) * maxlayer);                                            \
        if (!prev || !cur) {                                                                  \
            free(prev);                                                                       \
            free(cur);                                                                        \
            return 3;                                                                         \
        }                                                                                     \
        for (int j2 = 1; j2 < n; ++j2) {                                                      \
            for (int j1 = 0; j1 < j2; ++j1) {                                                 \
                prev[j1 + (uint64_t)j2 * (j2 - 1) / 2] =                                      \
                    ADD(MUL(a[j1], a[n + j2]), MUL(a[j2], a[n + j1]));                        \
            }                                                                                 \
        }                                                                                     \
        for (int k = 3; k < n; ++k) {                                                         \
            const int64_t cnt = (int64_t)g_binom[n][k];                                       \
            const T* row = a + (size_t)(k - 1) * n;                                           \
            const int64_t chunk = 1024;                                                       \
            _Pragma("omp parallel for schedule(static) num_threads(nthreads)")                \
            for (int64_t c0 = 0; c0 < cnt; c0 += chunk) {                                     \
                const int64_t c1 = c0 + chunk < cnt ? c0 + chunk : cnt;                       \
                uint64_t mask = orc_colex_unrank(k, (uint64_t)c0);                            \
                int elem[MAXN];                                                               \
                uint64_t pred[MAXN];                                                          \
                for (int64_t r = c0; r < c1; ++r) {                                           \
                    preds_of(mask, k, elem, pred);                                            \
                    T acc = MUL(row[elem[0]], prev[pred[0]]);                                 \
                    for (int p = 1; p < k; ++p) acc = ADD(acc, MUL(row[elem[p]], prev[pred[p]])); \
                    cur[r] = acc;                                                             \
                    if (r + 1 < c1) mask = gosper_next(mask);                                 \
                }                                                                             \
            }                                                                                 \
            T* t = prev;                                                                      \
            prev = cur;                                                                       \
            cur = t;                                                                          \
        }                                                                                     \
        const T* last = a + (size_t)(n - 1) * n;                                              \
        T total = MUL(last[0], prev[n - 1]);                                                  \
        for (int j = 1; j < n; ++j) total = ADD(total, MUL(last[j], prev[n - 1 - j]));        \
        free(prev);                                                                           \
        free(cur);                                                                            \
        *out = total;                                                                         \
        return 0;                                                                             \
    }

#define DMUL(x, y) ((x) * (y))
#define DADD(x, y) ((x) + (y))
DEFINE_DP(dp_f64, double, DMUL, DADD)
DEFINE_DP(dp_c128, cplx, cmul, cadd)

/* ---------------------------------------------------------------- exported */

/* Status: 0 ok, 1 bad argument, 2 int128 overflow, 3 out of memory. */
int orc_sz_i64(int n, const int64_t* a, int64_t* out_lo, int64_t* out_hi, int nthreads) {
    if (n < 1 || n > 34 || !a) return 1;
    i128 v = 0;
    const int rc = dp_i128(n, a, &v, nthreads > 0 ? nthreads : 1);
    *out_lo = (int64_t)(uint64_t)v;
    *out_hi = (int64_t)(v >> 64);
    return rc;
}

int orc_sz_f64(int n, const double* a, double* out, int nthreads) {
    if (n < 1 || n > 34 || !a) return 1;
    return dp_f64(n, a, out, nthreads > 0 ? nthreads : 1);
}

int orc_sz_c128(int n, const double* a, double* out, int nthreads) {
    if (n < 1 || n > 34 || !a) return 1;
    return dp_c128(n, (const cplx*)a, (cplx*)out, nthreads > 0 ? nthreads : 1);
}

/* Batches: one matrix per task, contiguous chunks per thread. Outputs are
 * int128 as (lo, hi) pairs for the integer ring; the return value is the
 * first nonzero per-matrix status (0 if all succeeded). */
int orc_sz_batch_i64(int n, int64_t count, const int64_t* a, int64_t* out_lohi, int nthreads) {
    if (n < 1 || n > 34 || count < 0) return 1;
    int status = 0;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1) reduction(max : status)
    for (int64_t b = 0; b < count; ++b) {
        i128 v = 0;
        const int rc = dp_i128(n, a + (size_t)b * n * n, &v, 1);
        out_lohi[2 * b] = (int64_t)(uint64_t)v;
        out_lohi[2 * b + 1] = (int64_t)(v >> 64);
        if (rc > status) status = rc;
    }
    return status;
}

int orc_sz_batch_f64(int n, int64_t count, const double* a, double* out, int nthreads) {
    if (n < 1 || n > 34 || count < 0) return 1;
    int status = 0;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1) reduction(max : status)
    for (int64_t b = 0; b < count; ++b) {
        const int rc = dp_f64(n, a + (size_t)b * n * n, out + b, 1);
        if (rc > status) status = rc;
    }
    return status;
}

int orc_sz_batch_c128(int n, int64_t count, const double* a, double* out, int nthreads) {
    if (n < 1 || n > 34 || count < 0) return 1;
    int status = 0;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1) reduction(max : status)
    for (int64_t b = 0; b < count; ++b) {
        const int rc = dp_c128(n, (const cplx*)(a + (size_t)b * 2 * n * n), (cplx*)(out + 2 * b), 1);
        if (rc > status) status = rc;
    }
    return status;
}

/* Full layer k (k >= 2) of the DP for one matrix, for checking individual
 * device layers: writes C(n,k) values in colex order. f64 only; k <= n-1. */
int orc_sz_layer_f64(int n, const double* a, int k, double* out_layer) {
    binom_init();
    if (n < 3 || k < 2 || k > n - 1) return 1;
    uint64_t maxlayer = 0;
    for (int q = 2; q <= k; ++q) maxlayer = g_binom[n][q] > maxlayer ? g_binom[n][q] : maxlayer;
    double* prev = (double*)malloc(sizeof(double) * maxlayer);
    double* cur = (double*)malloc(sizeof(double) * maxlayer);
    if (!prev || !cur) {
        free(prev);
        free(cur);
        return 3;
    }
    for (int j2 = 1; j2 < n; ++j2)
        for (int j1 = 0; j1 < j2; ++j1)
            prev[j1 + (uint64_t)j2 * (j2 - 1) / 2] = a[j1] * a[n + j2] + a[j2] * a[n + j1];
    for (int q = 3; q <= k; ++q) {
        const uint64_t cnt = g_binom[n][q];
        const double* row = a + (size_t)(q - 1) * n;
        uint64_t mask = (1ULL << q) - 1;
        int elem[MAXN];
        uint64_t pred[MAXN];
        for (uint64_t r = 0; r < cnt; ++r) {
            preds_of(mask, q, elem, pred);
            double acc = row[elem[0]] * prev[pred[0]];
            for (int p = 1; p < q; ++p) acc = acc + row[elem[p]] * prev[pred[p]];
            cur[r] = acc;
            mask = gosper_next(mask);
        }
        double* t = prev;
        prev = cur;
        cur = t;
    }
    memcpy(out_layer, prev, sizeof(double) * g_binom[n][k]);
    free(prev);
    free(cur);
    return 0;
}

/* One layer step over a rank range, the CPU stand-in for the device layer
 * kernel in the multi-rank (gloo) tests: cur[r] for r in [r0, r1) of layer k
 * from the full layer k-1 in prev (k = 2 uses the base case). Complex entries
 * are interleaved (re, im). */
#define DEFINE_STEP(NAME, T, MUL, ADD)                                                        \
    int NAME(int n, const T* a, int k, const T* prev, T* cur, uint64_t r0, uint64_t r1) {     \
        binom_init();                                                                         \
        if (n < 3 || k < 2 || k > n - 1 || r1 > g_binom[n][k] || r0 > r1) return 1;           \
        if (r0 == r1) return 0;                                                               \
        const T* row = a + (size_t)(k - 1) * n;                                               \
        uint64_t mask = orc_colex_unrank(k, r0);                                              \
        int elem[MAXN];                                                                       \
        uint64_t pred[MAXN];                                                                  \
        for (uint64_t r = r0; r < r1; ++r) {                                                  \
            if (k == 2) {                                                                     \
                const int j1 = __builtin_ctzll(mask);                                         \
                const int j2 = 63 - __builtin_clzll(mask);                                    \
                cur[r] = ADD(MUL(a[j1], a[n + j2]), MUL(a[j2], a[n + j1]));                   \
            } else {                                                                          \
                preds_of(mask, k, elem, pred);                                                \
                T acc = MUL(row[elem[0]], prev[pred[0]]);                                     \
                for (int p = 1; p < k; ++p) acc = ADD(acc, MUL(row[elem[p]], prev[pred[p]])); \
                cur[r] = acc;                                                                 \
            }                                                                                 \
            if (r + 1 < r1) mask = gosper_next(mask);                                         \
        }                                                                                     \
        return 0;                                                                             \
    }
DEFINE_STEP(orc_sz_layer_step_f64, double, DMUL, DADD)
DEFINE_STEP(orc_sz_layer_step_c128_, cplx, cmul, cadd)

int orc_sz_layer_step_c128(int n, const double* a, int k, const double* prev, double* cur, uint64_t r0, uint64_t r1) {
    return orc_sz_layer_step_c128_(n, (const cplx*)a, k, (const cplx*)prev, (cplx*)cur, r0, r1);
}

/* Top-level development from the full layer n-1 (permanent.cpp:184-198). */
int orc_sz_top_f64(int n, const double* a, const double* last, double* out) {
    const double* row = a + (size_t)(n - 1) * n;
    double total = row[0] * last[n - 1];
    for (int j = 1; j < n; ++j) total = total + row[j] * last[n - 1 - j];
    *out = total;
    return 0;
}

int orc_sz_top_c128(int n, const double* a, const double* last, double* out) {
    const cplx* row = (const cplx*)a + (size_t)(n - 1) * n;
    const cplx* l = (const cplx*)last;
    cplx total = cmul(row[0], l[n - 1]);
    for (int j = 1; j < n; ++j) total = cadd(total, cmul(row[j], l[n - 1 - j]));
    out[0] = total.re;
    out[1] = total.im;
    return 0;
}

/* ---------------------------------------------------------------- Ryser
 * Restatement of the reference's RyserEval (proj/src/permanent.cpp:85-136):
 * depth-first over the nonempty column subsets, a subset extended only by
 * columns above its maximum; the row sums carried down (child = parent +
 * a[:, j], :125-128), the product a left fold over rows (:112-116), the total
 * a left fold in visit order, minus for odd subset sizes (:117-122), negated
 * at the end for odd n (:103-105). Integers in checked 128-bit arithmetic. */
typedef struct {
    int n;
    const double* a;  /* complex (re, im) pairs, or reals with stride 1 */
    int cplx;
    double* sums;     /* (n + 1) levels x n entries (x2 for complex) */
    double tot_re, tot_im;
    int have;
} ryser_state;

static void ryser_visit(ryser_state* st, int max_col, int size) {
    const int n = st->n, w = st->cplx ? 2 : 1;
    const double* s = st->sums + (size_t)size * n * w;
    double pr = s[0], pi = st->cplx ? s[1] : 0.0;
    for (int i = 1; i < n; ++i) {
        if (st->cplx) {
            const double br = s[2 * i], bi = s[2 * i + 1];
            const double r = pr * br - pi * bi, im = pr * bi + pi * br;
            pr = r;
            pi = im;
        } else {
            pr = pr * s[i];
        }
    }
    const int odd = size & 1;
    if (!st->have) {
        st->tot_re = odd ? -pr : pr;
        st->tot_im = odd ? -pi : pi;
        st->have = 1;
    } else if (odd) {
        st->tot_re = st->tot_re - pr;
        st->tot_im = st->tot_im - pi;
    } else {
        st->tot_re = st->tot_re + pr;
        st->tot_im = st->tot_im + pi;
    }
    for (int j = max_col + 1; j < n; ++j) {
        double* nx = st->sums + (size_t)(size + 1) * n * w;
        for (int i = 0; i < n; ++i) {
            if (st->cplx) {
                nx[2 * i] = s[2 * i] + st->a[2 * ((size_t)i * n + j)];
                nx[2 * i + 1] = s[2 * i + 1] + st->a[2 * ((size_t)i * n + j) + 1];
            } else {
                nx[i] = s[i] + st->a[(size_t)i * n + j];
            }
        }
        ryser_visit(st, j, size + 1);
    }
}

static int ryser_float(int n, const double* a, int cplx, double* out) {
    const int w = cplx ? 2 : 1;
    ryser_state st = {n, a, cplx, calloc((size_t)(n + 1) * n * w, sizeof(double)), 0.0, 0.0, 0};
    if (!st.sums) return 2;
    for (int j = 0; j < n; ++j) {
        double* lv = st.sums + (size_t)1 * n * w;
        for (int i = 0; i < n; ++i) {
            if (cplx) {
                lv[2 * i] = a[2 * ((size_t)i * n + j)];
                lv[2 * i + 1] = a[2 * ((size_t)i * n + j) + 1];
            } else {
                lv[i] = a[(size_t)i * n + j];
            }
        }
        ryser_visit(&st, j, 1);
    }
    free(st.sums);
    out[0] = (n & 1) ? -st.tot_re : st.tot_re;
    if (cplx) out[1] = (n & 1) ? -st.tot_im : st.tot_im;
    return 0;
}

int orc_ryser_f64(int n, const double* a, double* out) { return ryser_float(n, a, 0, out); }
int orc_ryser_c128(int n, const double* a, double* out) { return ryser_float(n, a, 1, out); }

/* Integers: the same sum in checked 128-bit arithmetic (the subset order is
 * irrelevant for exact integers). */
int orc_ryser_i64(int n, const int64_t* a, int64_t* out_lo, int64_t* out_hi) {
    i128 total = 0;
    for (uint64_t S = 1; S < (1ull << n); ++S) {
        i128 prod = 1;
        for (int i = 0; i < n; ++i) {
            i128 s = 0;
            for (int j = 0; j < n; ++j)
                if ((S >> j) & 1) s += a[(size_t)i * n + j];
            if (__builtin_mul_overflow(prod, s, &prod)) return 1;
        }
        if (__builtin_popcountll(S) & 1) prod = -prod;
        if (__builtin_add_overflow(total, prod, &total)) return 1;
    }
    if (n & 1) total = -total;
    *out_lo = (int64_t)(uint64_t)total;
    *out_hi = (int64_t)(total >> 64);
    return 0;
}

/* ------------------------------------------------ overlapped block plan (CPU)
 * The CPU stand-ins of pl_shard_block_partial / pl_shard_block_top_terms for
 * the multi-rank (gloo) tests of sharded.py. Partial: the layer step with only
 * the terms of columns j < jmax (the top columns' terms come last in the
 * reference's ascending order, permanent.cpp:164-174); an output without any
 * such term is left 0. Top terms: cur[base + i] (+)= sum_s a(k-1, cols[s]) *
 * prev[sbase[s] + i], s ascending; init: the first term initialises. */
#define DEFINE_PARTIAL(NAME, T, MUL, ADD, ZERO)                                             \
    int NAME(int n, const T* a, int k, const T* prev, T* cur, uint64_t r0, uint64_t r1,     \
             int jmax) {                                                                    \
        binom_init();                                                                       \
        if (n < 3 || k < 3 || k > n - 1 || r1 > g_binom[n][k] || r0 > r1) return 1;         \
        if (r0 == r1) return 0;                                                             \
        const T* row = a + (size_t)(k - 1) * n;                                             \
        uint64_t mask = orc_colex_unrank(k, r0);                                            \
        int elem[MAXN];                                                                     \
        uint64_t pred[MAXN];                                                                \
        for (uint64_t r = r0; r < r1; ++r) {                                                \
            preds_of(mask, k, elem, pred);                                                  \
            T acc = ZERO;                                                                   \
            int first = 1;                                                                  \
            for (int p = 0; p < k; ++p) {                                                   \
                if (elem[p] >= jmax) break;                                                 \
                const T t = MUL(row[elem[p]], prev[pred[p]]);                               \
                acc = first ? t : ADD(acc, t);                                              \
                first = 0;                                                                  \
            }                                                                               \
            cur[r] = acc;                                                                   \
            if (r + 1 < r1) mask = gosper_next(mask);                                       \
        }                                                                                   \
        return 0;                                                                           \
    }
#define DEFINE_TOPTERMS(NAME, T, MUL, ADD)                                                  \
    int NAME(int n, const T* a, int k, const T* prev, T* cur, uint64_t base, uint64_t len,  \
             int nsrc, const int* cols, const uint64_t* sbase, int init) {                  \
        const T* row = a + (size_t)(k - 1) * n;                                             \
        for (uint64_t i = 0; i < len; ++i) {                                                \
            T acc = cur[base + i];                                                          \
            for (int s = 0; s < nsrc; ++s) {                                                \
                const T t = MUL(row[cols[s]], prev[sbase[s] + i]);                          \
                acc = (init && s == 0) ? t : ADD(acc, t);                                   \
            }                                                                               \
            cur[base + i] = acc;                                                            \
        }                                                                                   \
        return 0;                                                                           \
    }
static const cplx kCZero = {0.0, 0.0};
DEFINE_PARTIAL(orc_sz_layer_partial_f64, double, DMUL, DADD, 0.0)
DEFINE_PARTIAL(orc_sz_layer_partial_c128_, cplx, cmul, cadd, kCZero)
DEFINE_TOPTERMS(orc_sz_top_terms_f64, double, DMUL, DADD)
DEFINE_TOPTERMS(orc_sz_top_terms_c128_, cplx, cmul, cadd)

int orc_sz_layer_partial_c128(int n, const double* a, int k, const double* prev, double* cur, uint64_t r0,
                              uint64_t r1, int jmax) {
    return orc_sz_layer_partial_c128_(n, (const cplx*)a, k, (const cplx*)prev, (cplx*)cur, r0, r1, jmax);
}
int orc_sz_top_terms_c128(int n, const double* a, int k, const double* prev, double* cur, uint64_t base, uint64_t len,
                          int nsrc, const int* cols, const uint64_t* sbase, int init) {
    return orc_sz_top_terms_c128_(n, (const cplx*)a, k, (const cplx*)prev, (cplx*)cur, base, len, nsrc, cols, sbase,
                                  init);
}

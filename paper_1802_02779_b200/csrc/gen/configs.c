/*
 * Seeded synthetic inputs for the five BASELINE.json configs (C1..C5).
 *
 * BASELINE.json names no public dataset; these generators follow the
 * reference's own RNG conventions so every input is reproducible bit for bit:
 *   - std::mt19937_64 (restated below, the standard 64-bit Mersenne Twister);
 *   - 53-bit uniforms (g() >> 11) * 2^-53      reference src/boson.cpp:30-32
 *   - (0,1] uniforms ((g() >> 11) + 1) * 2^-53  reference src/boson.cpp:35-37
 *   - Box-Muller complex Gaussians               reference src/boson.cpp:39-45
 *   - Haar unitary = modified Gram-Schmidt over the columns of a complex
 *     Gaussian matrix (R's diagonal real-positive, i.e. QR with the phase fix)
 *                                                reference src/boson.cpp:149-181
 *   - submatrix rows = output modes, cols = input modes
 *                                                reference src/boson.cpp:207-227
 * Compiled with -ffp-contract=off so the floating-point sequence is the same
 * as the reference's x86-64 build (no FMA); tests pin the Haar generator
 * against the compiled reference (oracle/_ref) bit for bit.
 *
 * Config recipes:
 *   C1  mt19937_64 g(1); count*25 entries, matrix-major then row-major, g() % 10
 *   C2  mt19937_64 master(2); per item: U = haar(25, master()); 5 distinct
 *       columns by partial Fisher-Yates: perm=[0..24], for i<5:
 *       j = i + master() % (25-i), swap(perm[i], perm[j]); A[r][c] = U[r][perm[c]],
 *       r = 0..4 (occupancy 1 on output modes 0..4)
 *   C3  mt19937_64 g(3); count*144 entries, g() >> 63
 *   C4  mt19937_64 g(4); 676 entries, 2 * uniform53 - 1
 *   C5  U = haar(1024, 5); A = U[0:32, 0:32]. Only the first 32 columns of the
 *       Gram-Schmidt are needed (column k depends on columns < k only), so the
 *       generator orthonormalises 32 columns of the full 1024x1024 Gaussian draw.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x7FFFFFFFULL

typedef struct {
    uint64_t s[MT_N];
    int i;
} mt64;

void pl_mt64_seed(mt64* g, uint64_t seed) {
    g->s[0] = seed;
    for (int i = 1; i < MT_N; ++i) {
        g->s[i] = 6364136223846793005ULL * (g->s[i - 1] ^ (g->s[i - 1] >> 62)) + (uint64_t)i;
    }
    g->i = MT_N;
}

static void mt64_twist(mt64* g) {
    for (int i = 0; i < MT_N; ++i) {
        uint64_t x = (g->s[i] & MT_UPPER) | (g->s[(i + 1) % MT_N] & MT_LOWER);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        g->s[i] = g->s[(i + MT_M) % MT_N] ^ xa;
    }
    g->i = 0;
}

uint64_t pl_mt64_next(mt64* g) {
    if (g->i >= MT_N) mt64_twist(g);
    uint64_t y = g->s[g->i++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

static double uniform53(mt64* g) { return (double)(pl_mt64_next(g) >> 11) * 0x1.0p-53; }
static double uniform53_positive(mt64* g) {
    return (double)((pl_mt64_next(g) >> 11) + 1) * 0x1.0p-53;
}

static const double kPi = 3.141592653589793238462643383279502884;

static void complex_gaussian(mt64* g, double* re, double* im) {
    const double u1 = uniform53_positive(g);
    const double u2 = uniform53(g);
    const double r = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * kPi * u2;
    *re = r * cos(theta);
    *im = r * sin(theta);
}

/* Haar unitary of order m from `seed`, orthonormalising only the first
 * `ncols` columns (ncols = m for the full matrix). Output u is m*m complex
 * (interleaved re, im), row-major; columns >= ncols are left as the raw
 * Gaussian draw. Returns 0, or -1 on bad arguments / allocation failure. */
int pl_gen_haar(int m, uint64_t seed, int ncols, double* u) {
    if (m < 1 || ncols < 0 || ncols > m || !u) return -1;
    mt64* g = (mt64*)malloc(sizeof(mt64));
    if (!g) return -1;
    pl_mt64_seed(g, seed);
    const size_t mm = (size_t)m * (size_t)m;
    for (size_t e = 0; e < mm; ++e) complex_gaussian(g, &u[2 * e], &u[2 * e + 1]);
    free(g);
#define RE(i, j) u[2 * ((size_t)(i) * (size_t)m + (size_t)(j))]
#define IM(i, j) u[2 * ((size_t)(i) * (size_t)m + (size_t)(j)) + 1]
    for (int k = 0; k < ncols; ++k) {
        for (int j = 0; j < k; ++j) {
            double rr = 0.0, ri = 0.0;
            for (int i = 0; i < m; ++i) {
                /* conj(g_ij) * g_ik */
                const double ar = RE(i, j), ai = -IM(i, j);
                const double br = RE(i, k), bi = IM(i, k);
                const double pr = ar * br - ai * bi;
                const double pi = ar * bi + ai * br;
                rr = rr + pr;
                ri = ri + pi;
            }
            for (int i = 0; i < m; ++i) {
                const double br = RE(i, j), bi = IM(i, j);
                const double pr = rr * br - ri * bi;
                const double pi = rr * bi + ri * br;
                RE(i, k) = RE(i, k) - pr;
                IM(i, k) = IM(i, k) - pi;
            }
        }
        double norm_sq = 0.0;
        for (int i = 0; i < m; ++i) {
            const double x = RE(i, k), y = IM(i, k);
            norm_sq = norm_sq + (x * x + y * y);
        }
        const double norm = sqrt(norm_sq);
        for (int i = 0; i < m; ++i) {
            RE(i, k) = RE(i, k) / norm;
            IM(i, k) = IM(i, k) / norm;
        }
    }
#undef RE
#undef IM
    return 0;
}

/* C1: count 5x5 int64 matrices, entries g() % 10, seed `seed` (default 1). */
void pl_gen_c1(int64_t count, uint64_t seed, int64_t* out) {
    mt64 g;
    pl_mt64_seed(&g, seed);
    for (int64_t e = 0; e < count * 25; ++e) out[e] = (int64_t)(pl_mt64_next(&g) % 10ULL);
}

/* C2: count 5x5 complex128 boson-sampling submatrices (see header). `out` is
 * count*25 complex entries (count*50 doubles). Returns 0 or -1. */
int pl_gen_c2(int64_t count, uint64_t seed, double* out) {
    const int m = 25, n = 5;
    double* u = (double*)malloc(sizeof(double) * 2 * m * m);
    mt64* master = (mt64*)malloc(sizeof(mt64));
    if (!u || !master) {
        free(u);
        free(master);
        return -1;
    }
    pl_mt64_seed(master, seed);
    for (int64_t b = 0; b < count; ++b) {
        const uint64_t s = pl_mt64_next(master);
        pl_gen_haar(m, s, m, u);
        int perm[25];
        for (int i = 0; i < m; ++i) perm[i] = i;
        for (int i = 0; i < n; ++i) {
            const int j = i + (int)(pl_mt64_next(master) % (uint64_t)(m - i));
            const int t = perm[i];
            perm[i] = perm[j];
            perm[j] = t;
        }
        double* a = out + (size_t)b * 2 * n * n;
        for (int r = 0; r < n; ++r) {
            for (int c = 0; c < n; ++c) {
                const size_t src = 2 * ((size_t)r * m + (size_t)perm[c]);
                a[2 * (r * n + c)] = u[src];
                a[2 * (r * n + c) + 1] = u[src + 1];
            }
        }
    }
    free(u);
    free(master);
    return 0;
}

/* C3: count 12x12 int64 0/1 matrices, entries g() >> 63. */
void pl_gen_c3(int64_t count, uint64_t seed, int64_t* out) {
    mt64 g;
    pl_mt64_seed(&g, seed);
    for (int64_t e = 0; e < count * 144; ++e) out[e] = (int64_t)(pl_mt64_next(&g) >> 63);
}

/* C4 (and any order): n x n float64, entries 2*uniform53 - 1 in [-1, 1). */
void pl_gen_c4(int n, uint64_t seed, double* out) {
    mt64 g;
    pl_mt64_seed(&g, seed);
    for (int e = 0; e < n * n; ++e) out[e] = 2.0 * uniform53(&g) - 1.0;
}

/* C5: A = U[0:n, 0:n] of U = haar(m, seed) (m=1024, n=32, seed=5 for C5). */
int pl_gen_c5(int m, int n, uint64_t seed, double* out) {
    if (n > m) return -1;
    double* u = (double*)malloc(sizeof(double) * 2 * (size_t)m * (size_t)m);
    if (!u) return -1;
    int rc = pl_gen_haar(m, seed, n, u);
    if (rc == 0) {
        for (int r = 0; r < n; ++r) {
            memcpy(out + 2 * (size_t)r * n, u + 2 * (size_t)r * m, sizeof(double) * 2 * n);
        }
    }
    free(u);
    return rc;
}

/* Generic helpers used by the tests (reference tests/test_support.hpp:85-117
 * draws through std::uniform_int_distribution, whose mapping is
 * implementation-defined; these use plain modular / 53-bit draws instead). */
void pl_gen_int_matrices(int n, int64_t count, uint64_t seed, int64_t lo, int64_t hi, int64_t* out) {
    mt64 g;
    pl_mt64_seed(&g, seed);
    const uint64_t span = (uint64_t)(hi - lo) + 1ULL;
    for (int64_t e = 0; e < count * n * n; ++e) out[e] = lo + (int64_t)(pl_mt64_next(&g) % span);
}

void pl_gen_uniform(int64_t count, uint64_t seed, double lo, double hi, double* out) {
    mt64 g;
    pl_mt64_seed(&g, seed);
    for (int64_t e = 0; e < count; ++e) out[e] = lo + (hi - lo) * uniform53(&g);
}

void pl_gen_mt64_stream(uint64_t seed, int64_t count, uint64_t* out) {
    mt64 g;
    pl_mt64_seed(&g, seed);
    for (int64_t e = 0; e < count; ++e) out[e] = pl_mt64_next(&g);
}

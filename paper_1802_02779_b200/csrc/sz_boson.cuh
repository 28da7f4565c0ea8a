// Boson-sampling outcome probabilities on the device (reference
// proj/src/boson.cpp:207-240 extract_submatrix + outcome_probability, and the
// per-pattern loop of full_distribution, boson.cpp:250-269).
//
// The reference builds, for every output pattern, an n x n submatrix of the
// interferometer's unitary U (rows = occupied output modes, each repeated by
// its occupancy; columns = the input modes), evaluates its permanent with the
// Store-zechin engine and returns |per|^2 / prod_j occ_j!. On the device the
// three steps are one kernel and no submatrix is ever materialised:
//
//   * V = U[:, input_modes] (m x n complex) is staged once per CTA in shared
//     memory, so row i of a pattern's submatrix is V[rows[i]] (n contiguous
//     entries, a broadcast when lanes share the row);
//   * one thread per pattern runs the whole order-n DP in registers (n <= 6,
//     the reference's full-distribution cap, boson.cpp:254-256) with
//     compile-time subset masks, in the reference's ascending-j order
//     (permanent.cpp:150-198), so the permanent is bitwise the reference's;
//   * the probability is (re*re + im*im) / divisor with every operation
//     individually rounded, the divisor the product of 2..c over each run of
//     c equal rows in ascending mode order (boson.cpp:233-239).
//
// Enumeration mode: pattern `first + t` of enumerate_patterns(m, n) order
// (boson.cpp:185-205: mode 0 takes the most photons first, i.e. the rows
// sequences r_0 <= ... <= r_{n-1} in lexicographic order) is unranked by each
// thread from a shared-memory binomial table: at position i with prev = r_{i-1}
// and len = n-1-i later positions, the patterns whose r_i lies in [prev, v)
// number C(m-prev+len, len+1) - C(m-v+len, len+1) (hockey stick), so r_i is
// found by binary search over v. Nothing but U is read from HBM; the kernel
// writes 8 bytes per pattern and is FP64-pipe bound.
#pragma once

#include <cstdint>

#include "sz_kernels.cuh"

namespace pl {

constexpr int kBosonMaxFused = 6;  // orders evaluated in registers
constexpr int kBosonThreads = 128;

struct BosonParams {
    const double2* u;       // m x m unitary, row-major
    int m;
    int in[kBosonMaxFused]; // input modes (columns of U)
    uint64_t first;         // enumeration mode: index of the first pattern
    int64_t count;          // patterns in this launch
    const int32_t* rows;    // given mode: count x n output rows; null = enumerate
    double* probs;          // count probabilities
    int32_t* status;        // PL_STATUS_BIT_ROWS on a malformed row list (may be null)
    int early;              // PL_FLAG_INPUT_READY: compute before griddepcontrol.wait, store after
};

constexpr int kBosonBadRows = 0x2;  // = PL_STATUS_BIT_ROWS

// Store-zechin DP of the n x n matrix a(i, j) in registers (the accessor form
// of perm_in_registers: same masks, same order, same rounding).
template <class R, int N, class A>
__device__ __forceinline__ typename R::T perm_accessor(const A& a, bool& ov) {
    using T = typename R::T;
    if constexpr (N == 1) {
        return a(0, 0);
    } else {
        T memo[1 << N];
#pragma unroll
        for (int m = 0; m < (1 << N); ++m) {
            if (popc_c(m) == 2) {
                const int j1 = ctz_c(m), j2 = msb_c(m);
                memo[m] = R::add(R::mul(a(0, j1), a(1, j2), ov), R::mul(a(0, j2), a(1, j1), ov), ov);
            }
        }
        if constexpr (N == 2) {
            return memo[3];
        } else {
#pragma unroll
            for (int k = 3; k < N; ++k) {
                T row[N];
#pragma unroll
                for (int j = 0; j < N; ++j) row[j] = a(k - 1, j);
#pragma unroll
                for (int m = 0; m < (1 << N); ++m) {
                    if (popc_c(m) == k) {
                        T acc = R::zero();
                        bool first = true;
#pragma unroll
                        for (int j = 0; j < N; ++j) {
                            if ((m >> j) & 1) {
                                const T v = memo[m & ~(1 << j)];
                                acc = first ? R::mul(row[j], v, ov) : R::mac(acc, row[j], v, ov);
                                first = false;
                            }
                        }
                        memo[m] = acc;
                    }
                }
            }
            constexpr int full = (1 << N) - 1;
            T total = R::mul(a(N - 1, 0), memo[full & ~1], ov);
#pragma unroll
            for (int j = 1; j < N; ++j) total = R::mac(total, a(N - 1, j), memo[full & ~(1 << j)], ov);
            return total;
        }
    }
}

// |z|^2 / prod_{runs of c equal rows} c!  (reference boson.cpp:233-239; std::norm
// of a std::complex<double> is x*x + y*y there, each operation rounded).
template <bool FMA, int N>
__device__ __forceinline__ double boson_prob(double2 z, const int (&r)[N]) {
    double div = 1.0;
    int run = 1;
#pragma unroll
    for (int i = 1; i < N; ++i) {
        run = r[i] == r[i - 1] ? run + 1 : 1;
        if (run >= 2) div = __dmul_rn(div, (double)run);
    }
    const double nrm = FMA ? __fma_rn(z.x, z.x, __dmul_rn(z.y, z.y)) : __dadd_rn(__dmul_rn(z.x, z.x), __dmul_rn(z.y, z.y));
    return __ddiv_rn(nrm, div);
}

// Unrank pattern `idx` of enumerate_patterns(m, N) order into nondecreasing rows.
// cb[l * stride + a] = C(a, l) for 0 <= l <= N, 0 <= a < stride.
template <int N>
__device__ __forceinline__ void boson_unrank(uint64_t idx, int m, const uint64_t* cb, int stride, int (&r)[N]) {
    int prev = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const int len = N - 1 - i;
        const uint64_t* c = cb + (len + 1) * stride;
        const uint64_t top = c[m - prev + len];
        int lo = prev, hi = m - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (top - c[m - mid + len] <= idx) lo = mid;
            else hi = mid - 1;
        }
        idx -= top - c[m - lo + len];
        r[i] = lo;
        prev = lo;
    }
}

// VS: V = U[:, input_modes] staged in shared memory (m * N * 16 bytes fit);
// otherwise entries are read from U in global memory (L1/L2-resident).
template <class R, int N, bool VS>
__global__ void __launch_bounds__(kBosonThreads) sz_boson_kernel(BosonParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = p.m;
    const int stride = m + N;  // binomial table columns a = 0 .. m + N - 1
    uint64_t* cb = reinterpret_cast<uint64_t*>(smem_raw);
    double2* vs = reinterpret_cast<double2*>(smem_raw + (p.rows ? 0 : (size_t)(N + 1) * stride * sizeof(uint64_t)));
    // programmatic dependent launch (launched with the attribute only when p.early; see
    // sz_batch_tma_kernel): U and the rows are read at once, the stores wait for the previous grid
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    bool waited = !p.early;
    if (!p.rows) {
        for (int e = threadIdx.x; e < (N + 1) * stride; e += blockDim.x) {
            const int l = e / stride, a = e % stride;
            cb[e] = binom_u64(a, l);
        }
    }
    if constexpr (VS) {
        int col[N];  // compile-time indices into the kernel parameters (no local copy)
#pragma unroll
        for (int j = 0; j < N; ++j) col[j] = p.in[j];
        for (int r = threadIdx.x; r < m; r += blockDim.x) {
#pragma unroll
            for (int j = 0; j < N; ++j) vs[r * N + j] = p.u[(size_t)r * m + col[j]];
        }
    }
    __syncthreads();
    bool any_bad = false;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < p.count; t += (int64_t)gridDim.x * blockDim.x) {
        int r[N];
        bool bad = false;
        if (p.rows) {
            const int32_t* src = p.rows + t * N;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                r[i] = __ldg(src + i);
                bad |= r[i] < 0 || r[i] >= m || (i > 0 && r[i] < r[i - 1]);
            }
            if (bad) {
#pragma unroll
                for (int i = 0; i < N; ++i) r[i] = 0;
            }
        } else {
            boson_unrank<N>(p.first + (uint64_t)t, m, cb, stride, r);
        }
        bool ov = false;
        double2 z;
        if constexpr (VS) {
            int off[N];
#pragma unroll
            for (int i = 0; i < N; ++i) off[i] = r[i] * N;
            z = perm_accessor<R, N>([&](int i, int j) { return vs[off[i] + j]; }, ov);
        } else {
            const double2* rowp[N];
#pragma unroll
            for (int i = 0; i < N; ++i) rowp[i] = p.u + (size_t)r[i] * m;
            z = perm_accessor<R, N>([&](int i, int j) { return __ldg(rowp[i] + p.in[j]); }, ov);
        }
        const double pr = bad ? __longlong_as_double(0x7ff8000000000000LL) : boson_prob<R::kFma, N>(z, r);
        if (!waited) {
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            waited = true;
        }
        p.probs[t] = pr;
        any_bad |= bad;
    }
    if (!waited) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (any_bad && p.status) atomicOr(p.status, kBosonBadRows);
}

// Larger orders (given rows only): materialise the submatrices for the batch
// kernels, then turn the permanents into probabilities.
struct BosonGather {
    const double2* u;
    int m, n;
    int in[kMaxOrder];
    const int32_t* rows;
    int64_t count;
    double2* sub;  // count x n x n
    int32_t* bad;  // per-pattern flag
    int32_t* status;
};

__global__ void sz_boson_gather_kernel(BosonGather g) {
    const int64_t total = g.count * g.n * g.n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = e / (g.n * g.n);
        const int rem = (int)(e - t * g.n * g.n);
        const int i = rem / g.n, j = rem % g.n;
        int r = __ldg(g.rows + t * g.n + i);
        const bool bad = r < 0 || r >= g.m || (i > 0 && r < __ldg(g.rows + t * g.n + i - 1));
        if (bad) {
            g.bad[t] = 1;
            r = 0;
        }
        if (bad && g.status) atomicOr(g.status, kBosonBadRows);
        g.sub[e] = g.u[(size_t)r * g.m + g.in[j]];
    }
}

template <bool FMA>
__global__ void sz_boson_norm_kernel(const double2* __restrict__ per, const int32_t* __restrict__ rows, int n,
                                     int64_t count, const int32_t* __restrict__ bad, double* __restrict__ probs) {
    // (bad row lists were already reported by the gather kernel)
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
        const double2 z = per[t];
        double div = 1.0;
        int run = 1;
        for (int i = 1; i < n; ++i) {
            run = rows[t * n + i] == rows[t * n + i - 1] ? run + 1 : 1;
            if (run >= 2) div = __dmul_rn(div, (double)run);
        }
        const double nrm =
            FMA ? __fma_rn(z.x, z.x, __dmul_rn(z.y, z.y)) : __dadd_rn(__dmul_rn(z.x, z.x), __dmul_rn(z.y, z.y));
        probs[t] = bad[t] ? __longlong_as_double(0x7ff8000000000000LL) : __ddiv_rn(nrm, div);
    }
}

}  // namespace pl

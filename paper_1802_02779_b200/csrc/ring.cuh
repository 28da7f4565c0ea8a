// Ring arithmetic for the Store-zechin kernels.
//
// The reference instantiates its engine on Counted<T> over cpp_int or
// std::complex<double> (reference proj/src/permanent.cpp:253-277,
// proj/include/permlab/op_count.hpp:119-137). On the device:
//
//   RI64<false>  int64 arithmetic, used when the per-matrix guard proves that
//                no intermediate can reach 2^63 (then int64 is exact);
//   RI64<true>   checked int64 arithmetic for matrices the guard cannot
//                clear: every product / sum detects overflow, which the
//                kernel reports instead of wrapping (the reference never
//                overflows: cpp_int is arbitrary precision);
//   RF64<FMA>    real double; FMA=false rounds every product and sum on its
//                own (__dmul_rn / __dadd_rn), the reference's x86-64 sequence,
//                so results are bitwise those of the reference's Complex ring
//                with imag = 0; FMA=true contracts (faster, still <= 1e-9);
//   RC128<FMA>   complex double as double2 (re, im). FMA=false reproduces
//                GCC's inline complex product (ac - bd, ad + bc) and the
//                componentwise sum, each operation individually rounded.
//   RModP        residues modulo a prime p < 2^31 (entries and values in
//                [0, p), stored as long long): the ring of the exact big-integer
//                path (bigint.cu) -- the layer DP runs once per prime and the
//                host recombines the residues (CRT), which restores the
//                reference's arbitrary-precision Int (proj/include/permlab/
//                ring.hpp:29-31) where int64 would overflow. p and its Barrett
//                constant live in constant memory, set per pass on the stream.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pl {

template <bool CHECKED>
struct RI64 {
    using T = long long;
    static constexpr bool kChecked = CHECKED;
    __device__ __forceinline__ static T mul(T a, T b, bool& ov) {
        const T p = (T)((unsigned long long)a * (unsigned long long)b);
        if (CHECKED) ov |= (__mul64hi(a, b) != (p >> 63));
        return p;
    }
    __device__ __forceinline__ static T add(T a, T b, bool& ov) {
        const T s = (T)((unsigned long long)a + (unsigned long long)b);
        if (CHECKED) ov |= (((a ^ s) & (b ^ s)) < 0);
        return s;
    }
    __device__ __forceinline__ static T mac(T acc, T a, T b, bool& ov) { return add(acc, mul(a, b, ov), ov); }
    __device__ __forceinline__ static T zero() { return 0; }
};

template <bool FMA>
struct RF64 {
    using T = double;
    static constexpr bool kChecked = false;
    static constexpr bool kFma = FMA;
    __device__ __forceinline__ static T mul(T a, T b, bool&) { return __dmul_rn(a, b); }
    __device__ __forceinline__ static T add(T a, T b, bool&) { return __dadd_rn(a, b); }
    __device__ __forceinline__ static T mac(T acc, T a, T b, bool&) {
        return FMA ? __fma_rn(a, b, acc) : __dadd_rn(acc, __dmul_rn(a, b));
    }
    __device__ __forceinline__ static T zero() { return 0.0; }
};

template <bool FMA>
struct RC128 {
    using T = double2;
    static constexpr bool kChecked = false;
    static constexpr bool kFma = FMA;
    __device__ __forceinline__ static T mul(T a, T b, bool&) {
        T r;
        r.x = __dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y));
        r.y = __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x));
        return r;
    }
    __device__ __forceinline__ static T add(T a, T b, bool&) {
        T r;
        r.x = __dadd_rn(a.x, b.x);
        r.y = __dadd_rn(a.y, b.y);
        return r;
    }
    __device__ __forceinline__ static T mac(T acc, T a, T b, bool& ov) {
        if (FMA) {
            T r;
            r.x = __fma_rn(a.x, b.x, acc.x);
            r.x = __fma_rn(-a.y, b.y, r.x);
            r.y = __fma_rn(a.x, b.y, acc.y);
            r.y = __fma_rn(a.y, b.x, r.y);
            return r;
        }
        return add(acc, mul(a, b, ov), ov);
    }
    __device__ __forceinline__ static T zero() { return make_double2(0.0, 0.0); }
};

// Modulus of the RModP passes: p < 2^31 prime, m = floor(2^64 / p). One copy
// per translation unit; only capi.cu launches RModP kernels (set_modulus).
struct ModParams {
    unsigned long long p;
    unsigned long long m;
};
static __constant__ ModParams c_modp;

struct RModP {
    using T = long long;
    static constexpr bool kChecked = false;
    // a, b < p < 2^31: x = a * b < 2^62; q = floor(x * m / 2^64) is floor(x / p)
    // or one less (x / p - x * m / 2^64 < x / 2^64 < 1), so x - q * p < 2 p
    __device__ __forceinline__ static T mul(T a, T b, bool&) {
        // residues are below 2^31: one 32 x 32 -> 64 multiply
        const unsigned long long x = (unsigned long long)(unsigned)a * (unsigned long long)(unsigned)b;
        const unsigned long long q = __umul64hi(x, c_modp.m);
        unsigned long long r = x - q * c_modp.p;
        if (r >= c_modp.p) r -= c_modp.p;
        return (T)r;
    }
    __device__ __forceinline__ static T add(T a, T b, bool&) {
        unsigned long long s = (unsigned long long)a + (unsigned long long)b;
        if (s >= c_modp.p) s -= c_modp.p;
        return (T)s;
    }
    __device__ __forceinline__ static T mac(T acc, T a, T b, bool& ov) { return add(acc, mul(a, b, ov), ov); }
    __device__ __forceinline__ static T zero() { return 0; }
};

// Binomial table C(s, l), s, l <= kBinomDim - 1, as uint32 (C(34,17) < 2^32).
constexpr int kMaxOrder = 34;
constexpr int kBinomDim = 35;

__host__ __device__ constexpr uint64_t binom_u64(int s, int l) {
    if (l < 0 || s < 0 || l > s) return 0;
    uint64_t r = 1;
    for (int i = 1; i <= l; ++i) r = r * (uint64_t)(s - l + i) / (uint64_t)i;
    return r;
}

}  // namespace pl

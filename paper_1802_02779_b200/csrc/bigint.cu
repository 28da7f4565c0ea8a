// Exact integer permanents of any magnitude: the residue passes and their
// recombination.
//
// The reference's Int ring is arbitrary precision (reference
// proj/include/permlab/ring.hpp:29-31, cpp_int), so store_zechin_permanent
// (proj/src/permanent.cpp:314-316) never overflows; the device's PL_I64 ring is
// exact only while every intermediate fits int64 and reports PL_ERR_OVERFLOW
// otherwise. This unit closes that gap without a multi-limb device ring:
//
//   per(A) mod p_i  for K primes p_i < 2^31 -- the same layer DP, once per
//                   prime, on residues (ring RModP, ring.cuh): n <= 14 in one
//                   launch of sz_modp_small_kernel (a CTA per prime, the DP over
//                   a 2^n table in shared memory), n >= 15 through the layer
//                   kernels of capi.cu (enqueue_batch with the modular ring;
//                   the modulus is a constant set on the stream between passes);
//   CRT             Garner's mixed-radix digits and a Horner evaluation into
//                   64-bit limbs on the host; K from the row-sum bound
//                   |per(A)| <= prod_i sum_j |a_ij| so that prod p_i > 2 |per(A)|.
//
// Sums and products of residues are exact, so the order of the fold does not
// matter here; the result is the integer the reference computes.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "capi_internal.h"
#include "ring.cuh"

namespace {

using u64 = unsigned long long;
using u128 = unsigned __int128;

u64 mulmod(u64 a, u64 b, u64 m) { return (u64)((u128)a * b % m); }

u64 powmod(u64 a, u64 e, u64 m) {
    u64 r = 1 % m;
    a %= m;
    for (; e; e >>= 1) {
        if (e & 1) r = mulmod(r, a, m);
        a = mulmod(a, a, m);
    }
    return r;
}

// Miller-Rabin with bases 2, 3, 5, 7: deterministic below 3,215,031,751.
bool is_prime_u32(u64 n) {
    if (n < 2) return false;
    for (u64 q : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull}) {
        if (n % q == 0) return n == q;
    }
    u64 d = n - 1;
    int s = 0;
    while ((d & 1) == 0) {
        d >>= 1;
        ++s;
    }
    for (u64 a : {2ull, 3ull, 5ull, 7ull}) {
        u64 x = powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int i = 1; i < s && comp; ++i) {
            x = mulmod(x, x, n);
            if (x == n - 1) comp = false;
        }
        if (comp) return false;
    }
    return true;
}

// The K largest primes below 2^31, descending from 2^31 - 1 (each > 2^30).
// (a copy made under the lock: the cache may grow in another thread)
std::vector<uint32_t> primes_desc(size_t k) {
    static std::mutex mu;
    static std::vector<uint32_t> cache;
    static u64 next = (1ull << 31) - 1;
    std::lock_guard<std::mutex> lock(mu);
    while (cache.size() < k) {
        while (!is_prime_u32(next)) next -= 2;
        cache.push_back((uint32_t)next);
        next -= 2;
    }
    return std::vector<uint32_t>(cache.begin(), cache.begin() + (std::ptrdiff_t)k);
}

// One CTA per prime: X[S] over all column subsets S as bit masks in shared
// memory, X[{}] = 1, X[S] = sum_{j in S} a(|S| - 1, j) X[S \ {j}] (mod p), layer
// by layer; per(A) = X[full]. `res`: K matrices of residues in [0, p_i).
__global__ void __launch_bounds__(1024) sz_modp_small_kernel(const long long* __restrict__ res, int n,
                                                             const uint32_t* __restrict__ primes,
                                                             uint32_t* __restrict__ out) {
    extern __shared__ uint32_t x[];  // 2^n values, then n * n coefficients
    uint32_t* coef = x + (1u << n);
    const u64 p = primes[blockIdx.x];
    // Barrett constant: floor((2^64 - 1) / p) is floor(2^64 / p), or one less when p is a power of
    // two; either way q = hi(v * m) <= v / p with an error below 2, corrected by the loop below
    const u64 m = ~0ull / p;
    const long long* a = res + (size_t)blockIdx.x * n * n;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) coef[e] = (uint32_t)a[e];
    if (threadIdx.x == 0) x[0] = 1u % (uint32_t)p;
    __syncthreads();
    const uint32_t total = 1u << n;
    for (int k = 1; k <= n; ++k) {
        const uint32_t* row = coef + (k - 1) * n;
        for (uint32_t s = threadIdx.x; s < total; s += blockDim.x) {
            if (__popc(s) != k) continue;
            u64 acc = 0;
            for (uint32_t rest = s; rest; rest &= rest - 1) {
                const int j = __ffs(rest) - 1;
                const u64 v = (u64)row[j] * x[s ^ (1u << j)];
                const u64 q = __umul64hi(v, m);
                u64 r = v - q * p;
                while (r >= p) r -= p;
                acc += r;  // <= 14 terms below 2^31
            }
            x[s] = (uint32_t)(acc % p);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = x[total - 1];
}

// Ryser's formula on residues (reference proj/src/permanent.cpp:85-136 on its Int ring):
// per(A) = (-1)^n sum_{S nonempty} (-1)^|S| prod_i sum_{j in S} a_ij. Grid (blocks, primes);
// every thread walks masks S = t + 1, keeps the positive and negative terms apart (sums of
// residues below 2^31 stay far below 2^64) and the block writes (pos - neg) mod p. The visit
// order is immaterial: residue arithmetic is exact.
__global__ void __launch_bounds__(256) ryser_modp_kernel(const long long* __restrict__ res, int n,
                                                         const uint32_t* __restrict__ primes,
                                                         uint32_t* __restrict__ partial) {
    extern __shared__ uint32_t coef[];  // n * n residues of this prime
    __shared__ u64 wpos[8], wneg[8];
    const u64 p = primes[blockIdx.y];
    const u64 m = ~0ull / p;
    const long long* a = res + (size_t)blockIdx.y * n * n;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) coef[e] = (uint32_t)a[e];
    __syncthreads();
    auto reduce = [&](u64 v) {  // v < 2^62
        const u64 q = __umul64hi(v, m);
        u64 r = v - q * p;
        while (r >= p) r -= p;
        return r;
    };
    const u64 total = (n >= 64 ? 0 : (1ull << n)) - 1;
    u64 pos = 0, neg = 0;
    for (u64 t = blockIdx.x * (u64)blockDim.x + threadIdx.x; t < total; t += (u64)gridDim.x * blockDim.x) {
        const u64 S = t + 1;
        u64 prod = 1;
        for (int i = 0; i < n && prod; ++i) {
            u64 rs = 0;
            for (u64 w = S; w; w &= w - 1) rs += coef[i * n + __ffsll((long long)w) - 1];
            prod = reduce(prod * reduce(rs));
        }
        if (__popcll(S) & 1) neg += prod; else pos += prod;
    }
    for (int d = 16; d; d >>= 1) {
        pos += __shfl_xor_sync(0xffffffffu, pos, d);
        neg += __shfl_xor_sync(0xffffffffu, neg, d);
    }
    if ((threadIdx.x & 31) == 0) {
        wpos[threadIdx.x >> 5] = pos;
        wneg[threadIdx.x >> 5] = neg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 bp = 0, bn = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            bp += wpos[w];
            bn += wneg[w];
        }
        partial[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = (uint32_t)((bp % p + p - bn % p) % p);
    }
}

constexpr int kSmallMax = 14;

pl_status check_residues(int n, int k, const uint32_t* primes, const int64_t* res) {
    for (int i = 0; i < k; ++i) {
        const uint32_t p = primes[i];
        if (p < 2 || p >= (1u << 31)) return plc::fail_msg(PL_ERR_ARG, "modulus outside [2, 2^31)");
        const int64_t* r = res + (size_t)i * n * n;
        for (int e = 0; e < n * n; ++e) {
            if (r[e] < 0 || r[e] >= (int64_t)p) return plc::fail_msg(PL_ERR_ARG, "residue outside [0, p)");
        }
    }
    return PL_OK;
}

// The residue passes are serialised process-wide: the large-order passes share
// the modulus in constant memory.
std::mutex& pass_mutex() {
    static std::mutex mu;
    return mu;
}

pl_status run_residues(int n, int k, const uint32_t* primes, const int64_t* res, uint32_t* out,
                       const pl_limits* lim, cudaStream_t st) {
    // limits and arguments reject before any device work (reference tests/test_permanent.cpp:280-294)
    pl_status s = plc::check_order_limits(n, lim);
    if (s != PL_OK) return s;
    if ((s = plc::check_budget_limits(PL_I64, n, lim)) != PL_OK) return s;
    if ((s = check_residues(n, k, primes, res)) != PL_OK) return s;
    if ((s = plc::device_ready()) != PL_OK) return s;
    std::lock_guard<std::mutex> lock(pass_mutex());
    const size_t in_bytes = (size_t)k * n * n * sizeof(long long);
    long long* a_dev = nullptr;
    void* out_dev = nullptr;  // small: k uint32; large: k long long
    uint32_t* primes_dev = nullptr;
    int32_t* status_dev = nullptr;
    auto release = [&] {
        if (a_dev) cudaFreeAsync(a_dev, st);
        if (out_dev) cudaFreeAsync(out_dev, st);
        if (primes_dev) cudaFreeAsync(primes_dev, st);
        if (status_dev) cudaFreeAsync(status_dev, st);
    };
#define PLB_TRY(expr)                                  \
    do {                                               \
        cudaError_t _e = (expr);                       \
        if (_e != cudaSuccess) {                       \
            release();                                 \
            return plc::cuda_error(_e, #expr);         \
        }                                              \
    } while (0)
    PLB_TRY(cudaMallocAsync((void**)&a_dev, in_bytes, st));
    PLB_TRY(cudaMallocAsync(&out_dev, (size_t)k * sizeof(long long), st));
    PLB_TRY(cudaMemcpyAsync(a_dev, res, in_bytes, cudaMemcpyHostToDevice, st));
    if (n <= kSmallMax) {
        PLB_TRY(cudaMallocAsync((void**)&primes_dev, (size_t)k * sizeof(uint32_t), st));
        PLB_TRY(cudaMemcpyAsync(primes_dev, primes, (size_t)k * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        const size_t smem = ((size_t)1 << n) * sizeof(uint32_t) + (size_t)n * n * sizeof(uint32_t);
        // per device; setting it again is cheap next to the launch
        PLB_TRY(cudaFuncSetAttribute(sz_modp_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)((1u << kSmallMax) * 4 + kSmallMax * kSmallMax * 4)));
        // a CTA per prime: few CTAs, so as many threads as the table has work for
        const unsigned threads = n >= 12 ? 1024 : n >= 10 ? 512 : 256;
        sz_modp_small_kernel<<<(unsigned)k, threads, smem, st>>>(a_dev, n, primes_dev, static_cast<uint32_t*>(out_dev));
        PLB_TRY(cudaGetLastError());
        PLB_TRY(cudaMemcpyAsync(out, out_dev, (size_t)k * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        PLB_TRY(cudaStreamSynchronize(st));
        release();
        return PL_OK;
    }
    PLB_TRY(cudaMallocAsync((void**)&status_dev, sizeof(int32_t), st));
    PLB_TRY(cudaMemsetAsync(status_dev, 0, sizeof(int32_t), st));
    std::vector<pl::ModParams> mods((size_t)k);
    for (int i = 0; i < k; ++i) mods[i] = {primes[i], (u64)(((u128)1 << 64) / primes[i])};
    for (int i = 0; i < k; ++i) {
        s = plc::set_modulus(&mods[i], st);
        if (s == PL_OK) {
            s = plc::enqueue_batch(plc::kModDtype, n, 1, a_dev + (size_t)i * n * n,
                                   static_cast<long long*>(out_dev) + i, false, status_dev, st);
        }
        if (s != PL_OK) {
            cudaStreamSynchronize(st);
            release();
            return s;
        }
    }
    std::vector<long long> host((size_t)k);
    PLB_TRY(cudaMemcpyAsync(host.data(), out_dev, (size_t)k * sizeof(long long), cudaMemcpyDeviceToHost, st));
    PLB_TRY(cudaStreamSynchronize(st));
    release();
#undef PLB_TRY
    for (int i = 0; i < k; ++i) out[i] = (uint32_t)host[i];
    return PL_OK;
}

// out[i] = per(R_i) mod primes[i] by Ryser's formula (any n <= PL_MAX_ORDER).
pl_status run_ryser_residues(int n, int k, const uint32_t* primes, const int64_t* res, uint32_t* out,
                             const pl_limits* lim, cudaStream_t st) {
    pl_status s = plc::check_order_limits(n, lim);
    if (s != PL_OK) return s;
    if ((s = check_residues(n, k, primes, res)) != PL_OK) return s;
    if ((s = plc::device_ready()) != PL_OK) return s;
    const u64 total = (1ull << n) - 1;
    const unsigned blocks = (unsigned)std::max<u64>(1, std::min<u64>((total + 255) / 256, (u64)plc::sm_count() * 8));
    const size_t in_bytes = (size_t)k * n * n * sizeof(long long);
    long long* a_dev = nullptr;
    uint32_t* primes_dev = nullptr;
    uint32_t* part_dev = nullptr;
    auto release = [&] {
        if (a_dev) cudaFreeAsync(a_dev, st);
        if (primes_dev) cudaFreeAsync(primes_dev, st);
        if (part_dev) cudaFreeAsync(part_dev, st);
    };
#define PLB_TRY(expr)                          \
    do {                                       \
        cudaError_t _e = (expr);               \
        if (_e != cudaSuccess) {               \
            release();                         \
            return plc::cuda_error(_e, #expr); \
        }                                      \
    } while (0)
    PLB_TRY(cudaMallocAsync((void**)&a_dev, in_bytes, st));
    PLB_TRY(cudaMallocAsync((void**)&primes_dev, (size_t)k * sizeof(uint32_t), st));
    PLB_TRY(cudaMallocAsync((void**)&part_dev, (size_t)k * blocks * sizeof(uint32_t), st));
    PLB_TRY(cudaMemcpyAsync(a_dev, res, in_bytes, cudaMemcpyHostToDevice, st));
    PLB_TRY(cudaMemcpyAsync(primes_dev, primes, (size_t)k * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    ryser_modp_kernel<<<dim3(blocks, (unsigned)k), 256, (size_t)n * n * sizeof(uint32_t), st>>>(a_dev, n, primes_dev,
                                                                                               part_dev);
    PLB_TRY(cudaGetLastError());
    std::vector<uint32_t> part((size_t)k * blocks);
    PLB_TRY(cudaMemcpyAsync(part.data(), part_dev, part.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    PLB_TRY(cudaStreamSynchronize(st));
    release();
#undef PLB_TRY
    for (int i = 0; i < k; ++i) {
        const u64 p = primes[i];
        u64 sum = 0;
        for (unsigned b = 0; b < blocks; ++b) sum = (sum + part[(size_t)i * blocks + b]) % p;
        out[i] = (uint32_t)((n & 1) ? (p - sum) % p : sum);
    }
    return PL_OK;
}

// little-endian 64-bit limbs
using Limbs = std::vector<uint64_t>;

void mul_add_small(Limbs& x, uint64_t mul, uint64_t add) {  // x = x * mul + add
    u128 carry = add;
    for (uint64_t& w : x) {
        const u128 t = (u128)w * mul + carry;
        w = (uint64_t)t;
        carry = t >> 64;
    }
    if (carry) x.push_back((uint64_t)carry);
}

void trim(Limbs& x) {
    while (!x.empty() && x.back() == 0) x.pop_back();
}

int cmp(const Limbs& a, const Limbs& b) {  // trimmed operands
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (size_t i = a.size(); i-- > 0;) {
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    }
    return 0;
}

Limbs sub(const Limbs& a, const Limbs& b) {  // a >= b
    Limbs r(a.size());
    uint64_t borrow = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        const uint64_t bi = i < b.size() ? b[i] : 0;
        const u128 t = (u128)a[i] - bi - borrow;
        r[i] = (uint64_t)t;
        borrow = (uint64_t)(t >> 64) & 1;
    }
    trim(r);
    return r;
}

// Residues r_i mod p_i (pairwise coprime) -> the representative in (-M/2, M/2], M = prod p_i.
void crt_signed(const std::vector<uint32_t>& p, const std::vector<uint32_t>& r, Limbs* mag, bool* negative) {
    const size_t k = p.size();
    // Garner: x = v_0 + v_1 p_0 + v_2 p_0 p_1 + ..., 0 <= v_i < p_i
    std::vector<u64> v(k);
    for (size_t i = 0; i < k; ++i) {
        const u64 pi = p[i];
        // x_i = v_0 + v_1 p_0 + ... + v_{i-1} p_0..p_{i-2} (mod p_i), w = p_0..p_{i-1} (mod p_i)
        u64 xi = 0, w = 1;
        for (size_t j = 0; j < i; ++j) {
            xi = (xi + mulmod(v[j] % pi, w, pi)) % pi;
            w = mulmod(w, p[j] % pi, pi);
        }
        const u64 diff = (r[i] % pi + pi - xi) % pi;
        v[i] = mulmod(diff, powmod(w, pi - 2, pi), pi);  // w^{-1} by Fermat (p_i prime)
    }
    Limbs x, m;
    for (size_t i = k; i-- > 0;) mul_add_small(x, p[i], v[i]);  // Horner from the top digit
    m.push_back(1);
    for (size_t i = 0; i < k; ++i) mul_add_small(m, p[i], 0);
    trim(x);
    trim(m);
    Limbs twice = x;
    mul_add_small(twice, 2, 0);
    trim(twice);
    if (cmp(twice, m) > 0) {
        *mag = sub(m, x);
        *negative = true;
    } else {
        *mag = x;
        *negative = false;
    }
}

int bit_length(u128 v) {
    int b = 0;
    while (v) {
        ++b;
        v >>= 1;
    }
    return b;
}

}  // namespace

extern "C" {

pl_status pl_sz_permanent_modp(int32_t n, int32_t nprimes, const uint32_t* primes, const int64_t* residues,
                               uint32_t* out, const pl_limits* limits, void* stream) {
    if (n < 1) return plc::fail_msg(PL_ERR_ARG, "matrix order must be >= 1");
    if (nprimes < 1 || !primes || !residues || !out) return plc::fail_msg(PL_ERR_ARG, "bad arguments to pl_sz_permanent_modp");
    const pl_status lim_s = plc::check_order_limits(n, limits);
    if (lim_s != PL_OK) return lim_s;
    return run_residues(n, nprimes, primes, residues, out, limits, static_cast<cudaStream_t>(stream));
}

int32_t pl_bigint_primes(int32_t count, uint32_t* out) {
    if (count < 1 || !out) return 0;
    const std::vector<uint32_t> ps = primes_desc((size_t)count);
    std::copy(ps.begin(), ps.end(), out);
    return count;
}

}  // extern "C"

namespace {

pl_status permanent_bigint(bool ryser, int32_t n, const int64_t* a, uint64_t* limbs, size_t limb_cap, size_t* nlimbs,
                           int32_t* negative, const pl_limits* limits, void* stream) {
    if (n < 1) return plc::fail_msg(PL_ERR_ARG, "matrix order must be >= 1");
    if (!a || !nlimbs || !negative || (limb_cap && !limbs)) {
        return plc::fail_msg(PL_ERR_ARG, "bad arguments to the big-integer permanent");
    }
    const pl_status lim_s = plc::check_order_limits(n, limits);  // also the device cap (PL_MAX_ORDER)
    if (lim_s != PL_OK) return lim_s;
    // |per(A)| <= prod_i sum_j |a_ij| < 2^B, B = sum_i bit_length(row sum)
    int bits = 0;
    for (int i = 0; i < n; ++i) {
        u128 rs = 0;
        for (int j = 0; j < n; ++j) {
            const int64_t v = a[(size_t)i * n + j];
            rs += v < 0 ? (u128)0 - (u128)(__int128)v : (u128)v;
        }
        bits += bit_length(rs);
    }
    const int k = std::max(1, (bits + 2 + 29) / 30);  // every prime > 2^30: prod > 2^(30 k) >= 2^(B + 2)
    const std::vector<uint32_t> ps = primes_desc((size_t)k);
    std::vector<int64_t> res((size_t)k * n * n);
    for (int i = 0; i < k; ++i) {
        const int64_t p = ps[i];
        for (int e = 0; e < n * n; ++e) {
            int64_t r = a[e] % p;
            if (r < 0) r += p;
            res[(size_t)i * n * n + e] = r;
        }
    }
    std::vector<uint32_t> out((size_t)k);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    pl_status s = ryser ? run_ryser_residues(n, k, ps.data(), res.data(), out.data(), limits, st)
                        : run_residues(n, k, ps.data(), res.data(), out.data(), limits, st);
    if (s != PL_OK) return s;
    Limbs mag;
    bool neg = false;
    crt_signed(ps, out, &mag, &neg);
    *nlimbs = mag.size();
    *negative = neg ? 1 : 0;
    if (mag.size() > limb_cap) return plc::fail_msg(PL_ERR_ARG, "limb buffer too small (see *nlimbs)");
    if (!mag.empty()) std::memcpy(limbs, mag.data(), mag.size() * sizeof(uint64_t));
    return PL_OK;
}

}  // namespace

extern "C" {

pl_status pl_sz_permanent_bigint(int32_t n, const int64_t* a, uint64_t* limbs, size_t limb_cap, size_t* nlimbs,
                                 int32_t* negative, const pl_limits* limits, void* stream) {
    return permanent_bigint(false, n, a, limbs, limb_cap, nlimbs, negative, limits, stream);
}

pl_status pl_ryser_permanent_bigint(int32_t n, const int64_t* a, uint64_t* limbs, size_t limb_cap, size_t* nlimbs,
                                    int32_t* negative, const pl_limits* limits, void* stream) {
    return permanent_bigint(true, n, a, limbs, limb_cap, nlimbs, negative, limits, stream);
}

pl_status pl_ryser_permanent_modp(int32_t n, int32_t nprimes, const uint32_t* primes, const int64_t* residues,
                                  uint32_t* out, const pl_limits* limits, void* stream) {
    if (n < 1) return plc::fail_msg(PL_ERR_ARG, "matrix order must be >= 1");
    if (nprimes < 1 || !primes || !residues || !out) return plc::fail_msg(PL_ERR_ARG, "bad arguments to pl_ryser_permanent_modp");
    return run_ryser_residues(n, nprimes, primes, residues, out, limits, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

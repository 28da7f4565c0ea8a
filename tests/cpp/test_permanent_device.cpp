// C++ parity suite for the device-backed permlab host API. It mirrors the
// reference's own unit tests for the Store-zechin path (reference
// proj/tests/test_permanent.cpp) case by case, with the same goldens, so a
// maintainer can read the two side by side. Device results are additionally
// compared with the CPU oracle restatement (oracle/liboracle.so, loaded with
// dlopen so the product library never links it).
//
// Usage: test_permanent_device [--host-only]
//   --host-only runs only the checks that need no GPU (closed forms, limits,
//   error mapping when no device is present).
#include <dlfcn.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "permlab/boson.hpp"
#include "permlab/permanent.hpp"
#include "permlab_b200.h"

using namespace permlab;

namespace {

int g_checks = 0, g_failures = 0;

#define CHECK(cond)                                                                  \
    do {                                                                             \
        ++g_checks;                                                                  \
        if (!(cond)) {                                                               \
            ++g_failures;                                                            \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
        }                                                                            \
    } while (0)

#define CHECK_THROWS_AS(expr, Exc)                  \
    do {                                            \
        bool _thrown = false;                       \
        try {                                       \
            (void)(expr);                           \
        } catch (const Exc&) {                      \
            _thrown = true;                         \
        } catch (...) {                             \
        }                                           \
        CHECK(_thrown);                             \
    } while (0)

Matrix<Int> int_matrix(int n, const std::vector<long long>& v) { return {n, std::vector<Int>(v.begin(), v.end())}; }

Int value_of(const PermanentResult& r) { return std::get<Int>(r.value); }

// Reference fixture (reference tests/test_permanent.cpp:37-40).
const Matrix<Int> kDev4 = int_matrix(4, {7, 0, 1, 2, 5, 3, 4, 5, 3, 5, 6, 7, 1, 7, 8, 9});

Matrix<Int> random_int_matrix(int n, std::mt19937_64& g, int lo = -9, int hi = 9) {
    std::vector<Int> e(static_cast<std::size_t>(n) * n);
    for (auto& x : e) x = lo + static_cast<Int>(g() % static_cast<std::uint64_t>(hi - lo + 1));
    return {n, std::move(e)};
}

Matrix<Cplx> random_cplx_matrix(int n, std::mt19937_64& g) {
    std::vector<Cplx> e(static_cast<std::size_t>(n) * n);
    auto u = [&] { return 2.0 * static_cast<double>(g() >> 11) * 0x1.0p-53 - 1.0; };
    for (auto& x : e) {
        const double re = u();
        x = Cplx(re, u());
    }
    return {n, std::move(e)};
}

std::vector<int> random_permutation(int n, std::mt19937_64& g) {
    std::vector<int> p(n);
    for (int i = 0; i < n; ++i) p[i] = i;
    for (int i = n - 1; i > 0; --i) std::swap(p[i], p[g() % static_cast<std::uint64_t>(i + 1)]);
    return p;
}

// ---- oracle (CPU restatement), test-only
using orc_i64_fn = int (*)(int, const std::int64_t*, std::int64_t*, std::int64_t*, int);
using orc_c128_fn = int (*)(int, const double*, double*, int);
orc_i64_fn orc_i64 = nullptr;
orc_c128_fn orc_c128 = nullptr;

bool load_oracle(const char* self) {
    std::string dir(self);
    dir = dir.substr(0, dir.find_last_of('/') + 1);
    void* h = dlopen((dir + "../../oracle/liboracle.so").c_str(), RTLD_NOW);
    if (!h) return false;
    orc_i64 = reinterpret_cast<orc_i64_fn>(dlsym(h, "orc_sz_i64"));
    orc_c128 = reinterpret_cast<orc_c128_fn>(dlsym(h, "orc_sz_c128"));
    return orc_i64 && orc_c128;
}

Int oracle_int(const Matrix<Int>& m) {
    std::int64_t lo = 0, hi = 0;
    CHECK(orc_i64(m.order(), m.entries().data(), &lo, &hi, 1) == 0);
    CHECK(hi == (lo < 0 ? -1 : 0));
    return lo;
}

Cplx oracle_cplx(const Matrix<Cplx>& m) {
    double out[2];
    CHECK(orc_c128(m.order(), reinterpret_cast<const double*>(m.entries().data()), out, 1) == 0);
    return {out[0], out[1]};
}

// ---------------------------------------------------------------- host-only

void host_closed_forms() {
    // reference tests/test_permanent.cpp:131-147 (counts) and :149-168 (tables)
    for (int n = 2; n <= 20; ++n) {
        const std::uint64_t pow2 = std::uint64_t{1} << n;
        CHECK((store_zechin_counts(n) == OpCount{static_cast<std::uint64_t>(n) * (pow2 / 2) - n,
                                                 static_cast<std::uint64_t>(n) * (pow2 / 2) - pow2 + 1}));
    }
    CHECK((store_zechin_counts(1) == OpCount{0, 0}));
    CHECK((store_zechin_counts(2) == OpCount{2, 1}));
    auto report_for = [](int n) { return store_zechin_attributed(SquareMatrix(Matrix<Int>::filled(n, 1))); };
    const AttributionReport r3 = report_for(3);
    CHECK((r3.per_term == std::vector<OpCount>{{3, 1}, {3, 1}, {3, 1}}));
    CHECK(r3.final_combination_adds == 2);
    CHECK((r3.totals == OpCount{9, 5}));
    const AttributionReport r4 = report_for(4);
    CHECK((r4.per_term == std::vector<OpCount>{{10, 5}, {8, 4}, {6, 3}, {4, 2}}));
    CHECK((r4.totals == OpCount{28, 17}));
    const AttributionReport r5 = report_for(5);
    CHECK((r5.per_term == std::vector<OpCount>{{29, 17}, {20, 12}, {13, 8}, {8, 5}, {5, 3}}));
    CHECK(r5.final_combination_adds == 4);
    CHECK((r5.totals == OpCount{75, 49}));
    for (int n = 3; n <= 24; ++n) {
        const AttributionReport r = report_for(n);
        CHECK(r.totals == store_zechin_counts(n));
    }
    CHECK_THROWS_AS(store_zechin_attributed(SquareMatrix(Matrix<Int>::identity(2))), DomainError);
    for (Algorithm a : {Algorithm::Naive, Algorithm::Ryser, Algorithm::StoreZechin}) {
        CHECK(algorithm_from_name(algorithm_name(a)) == a);
    }
    CHECK_THROWS_AS(algorithm_from_name("glynn"), DomainError);
    // rings (reference ring.hpp:39-42, ring.cpp:34-45): the reference's tags, plus real
    for (RingTag t : {RingTag::Int, RingTag::Rational, RingTag::Complex, RingTag::Real}) {
        CHECK(ring_from_name(ring_name(t)) == t);
    }
    CHECK(ring_name(RingTag::Rational) == "rational");
    CHECK_THROWS_AS(ring_from_name("quaternion"), DomainError);
    CHECK(SquareMatrix(Matrix<Real>::identity(2)).ring() == RingTag::Real);
    CHECK(SquareMatrix(Matrix<Cplx>::identity(2)).ring() == RingTag::Complex);
    CHECK(ring_of(RingElement(Real{1})) == RingTag::Real);
    {
        std::int64_t in = 1, out = 0;  // no device arithmetic for the rational ring (checked before any device call)
        CHECK_THROWS_AS(store_zechin_permanent_batch(RingTag::Rational, 1, 1, &in, &out), DomainError);
    }
    // matrix index validation (reference matrix.hpp:93-184, test_matrix.cpp)
    {
        const Matrix<Int> m = Matrix<Int>::identity(3);
        CHECK_THROWS_AS(m.permute({0, 1}, {0, 1, 2}), DomainError);      // wrong length
        CHECK_THROWS_AS(m.permute({0, 0, 1}, {0, 1, 2}), DomainError);   // not a permutation
        CHECK_THROWS_AS(m.permute({0, 1, 2}, {0, 1, 3}), DomainError);   // out of range
        CHECK(m.permute({2, 0, 1}, {2, 0, 1}) == m);
        CHECK_THROWS_AS(m.remove_rows_cols({0, 0}, {0, 1}), DomainError);  // duplicate row
        CHECK_THROWS_AS(m.remove_rows_cols({3}, {0}), DomainError);        // row out of range
        CHECK_THROWS_AS(m.remove_rows_cols({0}, {-1}), DomainError);       // column out of range
        CHECK(m.remove_rows_cols({1}, {1}) == Matrix<Int>::identity(2));
    }
    // limits (reference tests/test_permanent.cpp:280-294): rejected before any device work
    Limits limits;
    limits.subset_order_limit = 4;
    CHECK_THROWS_AS(store_zechin_permanent(SquareMatrix(Matrix<Int>::filled(5, 1)), limits), DomainError);
    limits = Limits{};
    limits.memo_budget_bytes = 16;
    CHECK_THROWS_AS(store_zechin_permanent(SquareMatrix(Matrix<Int>::filled(5, 1)), limits), DomainError);
    CHECK_THROWS_AS(store_zechin_permanent(SquareMatrix(Matrix<Int>::filled(35, 1))), DomainError);
    setenv("PERMLAB_LIMITS", "subset_order_limit=24,memo_budget_bytes=1024", 1);
    const Limits env = Limits::from_env();
    CHECK(env.subset_order_limit == 24);
    CHECK(env.memo_budget_bytes == 1024);
    setenv("PERMLAB_LIMITS", "bogus=1", 1);
    CHECK_THROWS_AS(Limits::from_env(), DomainError);
    unsetenv("PERMLAB_LIMITS");
}

// ---------------------------------------------------------------- device

void device_goldens() {
    // reference tests/test_permanent.cpp:48-92
    CHECK(value_of(store_zechin_permanent(SquareMatrix(int_matrix(2, {1, 2, 3, 4})))) == 10);
    CHECK(value_of(store_zechin_permanent(SquareMatrix(int_matrix(3, {1, 2, 3, 4, 5, 6, 7, 8, 9})))) == 450);
    const auto dev = store_zechin_permanent(SquareMatrix(kDev4));
    CHECK(value_of(dev) == 9722);
    CHECK((dev.counts == OpCount{28, 17}));
    CHECK(dev.algorithm == Algorithm::StoreZechin);
    const SquareMatrix a5(int_matrix(5, {1, 1, 0, 2, 3, 2, 0, 1, 1, 4, 3, 1, 2, 0, 1, 0, 2, 1, 3, 2, 1, 0, 4, 1, 2}));
    const auto r5 = store_zechin_permanent(a5);
    CHECK(value_of(r5) == 988);
    CHECK((r5.counts == OpCount{75, 49}));
    const auto one = store_zechin_permanent(SquareMatrix(int_matrix(1, {42})));
    CHECK(value_of(one) == 42);
    // the Ryser engine on the same goldens (reference permanent.hpp:84), with
    // the reference's counts (tests/acceptance.cpp:72)
    const auto ry4 = ryser_permanent(SquareMatrix(kDev4));
    CHECK(value_of(ry4) == 9722);
    CHECK((ry4.counts == OpCount{45, 58}));
    CHECK(ry4.algorithm == Algorithm::Ryser);
    const auto ry5 = ryser_permanent(a5);
    CHECK(value_of(ry5) == 988);
    CHECK((ry5.counts == OpCount{124, 160}));
    CHECK(value_of(ryser_permanent(SquareMatrix(int_matrix(1, {42})))) == 42);
    CHECK_THROWS_AS(ryser_permanent(SquareMatrix(Matrix<Int>::filled(21, 1))), DomainError);
    CHECK((one.counts == OpCount{0, 0}));
    const auto two = store_zechin_permanent(SquareMatrix(int_matrix(2, {2, 3, 5, 7})));
    CHECK(value_of(two) == 29);
    CHECK((two.counts == OpCount{2, 1}));
    CHECK(value_of(store_zechin_permanent(SquareMatrix(Matrix<Int>::filled(3, 1)))) == 6);
    CHECK(value_of(store_zechin_permanent(SquareMatrix(Matrix<Int>::identity(7)))) == 1);
    // first-column development of the order-4 example (reference :246-255)
    const std::vector<Int> minors{1116, 258, 166, 122};
    Int sum = 0;
    for (int i = 0; i < 4; ++i) {
        const auto minor = kDev4.remove_rows_cols({i}, {0});
        CHECK(value_of(store_zechin_permanent(SquareMatrix(minor))) == minors[i]);
        sum += kDev4(i, 0) * minors[i];
    }
    CHECK(sum == 9722);
}

void device_oracle_agreement() {
    // reference tests/test_permanent.cpp:94-106 (n = 1..6, 20 each), widened to n = 1..16
    std::mt19937_64 g(41);
    for (int n = 1; n <= 16; ++n) {
        for (int rep = 0; rep < (n <= 8 ? 20 : 3); ++rep) {
            const auto m = random_int_matrix(n, g, n <= 10 ? -9 : -2, n <= 10 ? 9 : 2);
            CHECK(value_of(store_zechin_permanent(SquareMatrix(m))) == oracle_int(m));
        }
    }
    // complex: bitwise equal to the oracle (which is bitwise the reference)
    std::mt19937_64 gc(47);
    for (int n = 1; n <= 14; ++n) {
        const auto m = random_cplx_matrix(n, gc);
        const Cplx d = std::get<Cplx>(store_zechin_permanent(SquareMatrix(m)).value);
        const Cplx o = oracle_cplx(m);
        CHECK(d == o);
        CHECK(approx_equal(d, o));
    }
}

void device_identities() {
    // reference tests/test_permanent.cpp:196-244
    std::mt19937_64 g(67);
    for (int rep = 0; rep < 25; ++rep) {
        const int n = 2 + static_cast<int>(g() % 4);
        const auto m = random_int_matrix(n, g);
        const Int expected = value_of(store_zechin_permanent(SquareMatrix(m)));
        const auto p = m.permute(random_permutation(n, g), random_permutation(n, g));
        CHECK(value_of(store_zechin_permanent(SquareMatrix(p))) == expected);
        CHECK(value_of(store_zechin_permanent(SquareMatrix(m.transpose()))) == expected);
        const Int s = Int(rep) - 12;
        CHECK(value_of(store_zechin_permanent(SquareMatrix(m.scale_row(rep % n, s)))) == s * expected);
        if (n > 2) {
            Int sum = 0;
            for (int j = 0; j < n; ++j) {
                sum += m(0, j) * value_of(store_zechin_permanent(SquareMatrix(m.remove_rows_cols({0}, {j}))));
            }
            CHECK(sum == expected);
        }
    }
}

void device_run_and_batch() {
    // reference tests/test_permanent.cpp:184-194
    std::mt19937_64 g(61);
    for (int n : {3, 4, 6, 8}) {
        const StoreZechinRun run = store_zechin_run(SquareMatrix(random_int_matrix(n, g)));
        const std::uint64_t expected = (std::uint64_t{1} << n) - 2 - static_cast<std::uint64_t>(n);
        CHECK(run.cache_misses == expected);
        CHECK(run.distinct_subsets == expected);
    }
    // vector batch == singles
    std::vector<SquareMatrix> batch;
    for (int b = 0; b < 40; ++b) batch.emplace_back(random_int_matrix(5, g));
    const auto res = store_zechin_permanent_batch(batch);
    CHECK(res.size() == batch.size());
    for (std::size_t b = 0; b < batch.size(); ++b) {
        CHECK(value_of(res[b]) == value_of(store_zechin_permanent(batch[b])));
    }
    CHECK_THROWS_AS(store_zechin_permanent_batch(std::vector<SquareMatrix>{SquareMatrix(Matrix<Int>::filled(3, 1)),
                                                                           SquareMatrix(Matrix<Int>::filled(4, 1))}),
                    DomainError);
    // int64 guard: an exact value beyond int64 is a DomainError, never a wrap
    CHECK_THROWS_AS(store_zechin_permanent(SquareMatrix(Matrix<Int>::filled(22, 1000))), DomainError);
    // ... and the exact entry point returns the reference's arbitrary-precision value: 1000^22 22!
    {
        const BigInt big = store_zechin_permanent_exact(Matrix<Int>::filled(22, 1000));
        CHECK(!big.negative && !big.fits_int64());
        CHECK(big.str() == "1124000727777607680000" + std::string(66, '0'));
        const BigInt neg = store_zechin_permanent_exact(Matrix<Int>::filled(21, -1));
        CHECK(neg.negative && neg.str() == "-51090942171709440000");
        const BigInt small = store_zechin_permanent_exact(Matrix<Int>::filled(5, -2));
        CHECK(small.fits_int64() && small.to_int64() == -3840 && small.str() == "-3840");
        CHECK(store_zechin_permanent_exact(Matrix<Int>::filled(16, 0)).str() == "0");
        // Ryser's formula, same integers (residue sums beyond the 128-bit guard)
        CHECK(ryser_permanent_exact(Matrix<Int>::filled(22, 1000)).str() == big.str());
        CHECK(ryser_permanent_exact(Matrix<Int>::filled(21, -1)).str() == neg.str());
        CHECK(ryser_permanent_exact(Matrix<Int>::filled(5, -2)).to_int64() == -3840);
    }
    // the guard is conservative but the checked path still computes what fits
    CHECK(value_of(store_zechin_permanent(SquareMatrix(Matrix<Int>::filled(20, 1)))) == 2432902008176640000LL);
}

// Limits.num_gpus >= 1: the single-process multi-GPU path (NCCL communicators
// over devices 0..g-1; this box has one GPU, so g = 1 -- the all-gather plan
// through ncclAllGather on a one-rank communicator). Bitwise equal to the
// oracle and to the default single-device path.
void device_multi() {
    int devices = pl_device_count();
    Limits multi;
    multi.num_gpus = 1;
    std::mt19937_64 g(73);
    for (int n : {15, 18, 21}) {
        const auto mc = random_cplx_matrix(n, g);
        const Cplx vm = std::get<Cplx>(store_zechin_permanent(SquareMatrix(mc), multi).value);
        CHECK(vm == oracle_cplx(mc));
        CHECK(vm == std::get<Cplx>(store_zechin_permanent(SquareMatrix(mc)).value));
        const auto mi = random_int_matrix(n, g, -2, 2);
        CHECK(value_of(store_zechin_permanent(SquareMatrix(mi), multi)) == oracle_int(mi));
    }
    // int64 overflow is a DomainError through the sharded path too
    CHECK_THROWS_AS(store_zechin_permanent(SquareMatrix(Matrix<Int>::filled(22, 1000)), multi), DomainError);
    // a batch of small orders is split by matrix across the devices
    std::vector<SquareMatrix> batch;
    for (int b = 0; b < 64; ++b) batch.emplace_back(random_int_matrix(9, g));
    const auto split = store_zechin_permanent_batch(batch, multi);
    for (std::size_t b = 0; b < batch.size(); ++b) {
        CHECK(value_of(split[b]) == oracle_int(batch[b].as<Int>()));
    }
    // more devices than the box has: a DomainError before any work
    Limits too_many;
    too_many.num_gpus = devices + 1;
    CHECK_THROWS_AS(store_zechin_permanent(SquareMatrix(Matrix<Int>::filled(16, 1)), too_many), DomainError);
}

// ---------------------------------------------------------------- boson sampling
// mirrors reference tests/test_boson.cpp case by case

Matrix<Cplx> balanced_coupler() {
    const double s = 1.0 / std::sqrt(2.0);
    return {2, {Cplx(s), Cplx(s), Cplx(s), Cplx(-s)}};
}

bool near(double a, double b, double eps) { return std::abs(a - b) <= eps * std::max(std::abs(a), std::abs(b)); }

void host_boson() {
    // reference test_boson.cpp:28-36
    const Interferometer coupler(2, balanced_coupler());
    CHECK(coupler.modes() == 2);
    CHECK_THROWS_AS(Interferometer(2, Matrix<Cplx>::filled(2, Cplx(0.5))), DomainError);
    CHECK_THROWS_AS(Interferometer(3, balanced_coupler()), DomainError);
    CHECK_THROWS_AS(Interferometer(0, Matrix<Cplx>::identity(1)), DomainError);
    // :38-63
    for (int m : {1, 2, 5, 8}) {
        const Interferometer itf = haar_unitary(m, 99);
        CHECK(itf.modes() == m);
    }
    CHECK(haar_unitary(4, 5).unitary() == haar_unitary(4, 5).unitary());
    CHECK(!(haar_unitary(4, 5).unitary() == haar_unitary(4, 6).unitary()));
    // :65-72
    const auto patterns = enumerate_patterns(2, 2);
    CHECK(patterns.size() == 3);
    CHECK(patterns[0].occupancy == (std::vector<int>{2, 0}));
    CHECK(patterns[1].occupancy == (std::vector<int>{1, 1}));
    CHECK(patterns[2].occupancy == (std::vector<int>{0, 2}));
    CHECK(enumerate_patterns(6, 3).size() == 56);
    // :74-99
    const Interferometer itf = haar_unitary(3, 7);
    CHECK(extract_submatrix(itf, {0, 1, 2}, {{1, 1, 1}}) == itf.unitary());
    const auto one = extract_submatrix(itf, {1}, {{0, 0, 1}});
    CHECK(one.order() == 1);
    CHECK(one(0, 0) == itf.unitary()(2, 1));
    const auto two = extract_submatrix(itf, {0, 1}, {{2, 0, 0}});
    CHECK(two(0, 0) == two(1, 0));
    CHECK(two(0, 1) == two(1, 1));
    CHECK_THROWS_AS(extract_submatrix(itf, {0, 3}, {{1, 1, 0}}), DomainError);
    CHECK_THROWS_AS(extract_submatrix(itf, {0, 0}, {{1, 1, 0}}), DomainError);
    CHECK_THROWS_AS(extract_submatrix(itf, {0, 1}, {{1, 1, 1}}), DomainError);
    CHECK_THROWS_AS(extract_submatrix(itf, {0, 1}, {{1, 1}}), DomainError);
    CHECK_THROWS_AS(extract_submatrix(itf, {0, 1}, {{2, -1, 1}}), DomainError);
    // :196-206 (all rejected before any device work)
    const Interferometer itf8 = haar_unitary(8, 41);
    CHECK_THROWS_AS(full_distribution(itf8, {0, 1, 2, 3, 4, 5, 6}), DomainError);
    Limits tight;
    tight.enumeration_cap = 10;
    CHECK_THROWS_AS(full_distribution(itf8, {0, 1, 2}, tight), DomainError);
    CHECK_THROWS_AS(full_distribution(itf8, {}), DomainError);
    CHECK_THROWS_AS(full_distribution(itf8, {0, 8}), DomainError);
}

void device_boson() {
    // :101-115 two-photon interference on the balanced coupler
    const Interferometer coupler(2, balanced_coupler());
    const std::vector<int> input{0, 1};
    CHECK(outcome_probability(coupler, input, {{1, 1}}) <= 1e-12);
    CHECK(near(outcome_probability(coupler, input, {{2, 0}}), 0.5, 1e-12));
    CHECK(near(outcome_probability(coupler, input, {{0, 2}}), 0.5, 1e-12));
    const OutcomeDistribution dist = full_distribution(coupler, input);
    CHECK(dist.entries.size() == 3);
    CHECK(near(dist.entries[0].second, 0.5, 1e-12));
    CHECK(dist.entries[1].second <= 1e-12);
    CHECK(near(dist.entries[2].second, 0.5, 1e-12));
    CHECK(near(dist.total_probability(), 1.0, 1e-12));
    // :117-128 single photons
    const Interferometer itf4 = haar_unitary(4, 17);
    double total = 0;
    for (int j = 0; j < 4; ++j) {
        OutputPattern out{std::vector<int>(4, 0)};
        out.occupancy[static_cast<std::size_t>(j)] = 1;
        const double p = outcome_probability(itf4, {2}, out);
        CHECK(near(p, std::norm(itf4.unitary()(j, 2)), 1e-12));
        total += p;
    }
    CHECK(near(total, 1.0, 1e-10));
    // :140-163 the distribution against per-pattern Store-zechin on the device
    const Interferometer itf6 = haar_unitary(6, 31);
    const std::vector<int> in3{0, 1, 2};
    const OutcomeDistribution d6 = full_distribution(itf6, in3);
    CHECK(d6.entries.size() == 56);
    CHECK(std::abs(d6.total_probability() - 1.0) <= 1e-9);
    for (const auto& [pattern, p] : d6.entries) {
        const Cplx per = std::get<Cplx>(store_zechin_permanent(SquareMatrix(extract_submatrix(itf6, in3, pattern))).value);
        CHECK(per == oracle_cplx(extract_submatrix(itf6, in3, pattern)));
        double divisor = 1;
        for (int c : pattern.occupancy)
            for (int i = 2; i <= c; ++i) divisor *= i;
        CHECK(p == std::norm(per) / divisor);  // bitwise: same DP, same rounding
    }
    // batch entry point == singles; distribution chunks == the whole
    std::vector<OutputPattern> pats;
    for (const auto& e : d6.entries) pats.push_back(e.first);
    const auto batch = outcome_probabilities(itf6, in3, pats);
    const auto chunk = distribution_probabilities(itf6, in3, 10, 30);
    for (std::size_t i = 0; i < pats.size(); ++i) CHECK(batch[i] == d6.entries[i].second);
    for (std::size_t i = 0; i < chunk.size(); ++i) CHECK(chunk[i] == d6.entries[10 + i].second);
    // :165-194 relabelling output modes permutes the distribution
    const Interferometer itf = haar_unitary(4, 37);
    const OutcomeDistribution base = full_distribution(itf, input);
    const std::vector<int> perm{2, 0, 3, 1};
    std::vector<int> inverse(perm.size());
    for (std::size_t j = 0; j < perm.size(); ++j) inverse[static_cast<std::size_t>(perm[j])] = static_cast<int>(j);
    const Interferometer relabeled(4, itf.unitary().permute(inverse, {0, 1, 2, 3}));
    const OutcomeDistribution moved = full_distribution(relabeled, input);
    for (const auto& [pattern, p] : base.entries) {
        OutputPattern rp{std::vector<int>(4, 0)};
        for (std::size_t j = 0; j < perm.size(); ++j) rp.occupancy[static_cast<std::size_t>(perm[j])] = pattern.occupancy[j];
        bool found = false;
        for (const auto& [q_pattern, q] : moved.entries) {
            if (q_pattern == rp) {
                CHECK(near(q, p, 1e-9));
                found = true;
            }
        }
        CHECK(found);
    }
    // :208-232 sampling
    CHECK(sample(coupler, input, 0, 1).empty());
    const auto draws = sample(coupler, input, 10000, 7);
    CHECK(draws.size() == 10000);
    std::size_t first = 0;
    for (const auto& p : draws) {
        CHECK(!(p.occupancy == std::vector<int>{1, 1}));
        first += p.occupancy == std::vector<int>{2, 0} ? 1 : 0;
    }
    CHECK(first > 4500 && first < 5500);
    CHECK(sample(coupler, input, 200, 99) == sample(coupler, input, 200, 99));
    CHECK(!(sample(coupler, input, 200, 99) == sample(coupler, input, 200, 100)));
}

}  // namespace

int main(int argc, char** argv) {
    const bool host_only = argc > 1 && std::string(argv[1]) == "--host-only";
    host_closed_forms();
    host_boson();
    if (!host_only) {
        if (!load_oracle(argv[0])) {
            std::fprintf(stderr, "cannot load oracle/liboracle.so\n");
            return 2;
        }
        device_goldens();
        device_oracle_agreement();
        device_identities();
        device_run_and_batch();
        device_multi();
        device_boson();
    }
    std::printf("%d checks, %d failures\n", g_checks, g_failures);
    return g_failures == 0 ? 0 : 1;
}

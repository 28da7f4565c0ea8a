// permlab C++ host API over the B200 C ABI (include/permlab/permanent.hpp).
//
// Host work here is argument handling, the Limits / DomainError contract
// (reference proj/src/limits.cpp:43-76, proj/src/permanent.cpp:232-240) and
// closed-form diagnostics; every permanent is computed on the device through
// pl_sz_permanent / pl_sz_permanent_batch. There is no CPU fallback.
#include "permlab/permanent.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "permlab_b200.h"

namespace permlab {

namespace {

[[noreturn]] void raise(pl_status s) {
    const std::string msg = pl_last_error();
    switch (s) {
        case PL_ERR_ARG:
        case PL_ERR_LIMIT:
        case PL_ERR_OVERFLOW:
            throw DomainError(msg);
        default:
            throw std::runtime_error("permlab-b200: " + msg);
    }
}

void check(pl_status s) {
    if (s != PL_OK) raise(s);
}

pl_dtype dtype_of(RingTag r) {
    switch (r) {
        case RingTag::Int:
            return PL_I64;
        case RingTag::Real:
            return PL_F64;
        case RingTag::Complex:
            return PL_C128;
        case RingTag::Rational:
            throw DomainError("the rational ring has no device arithmetic (use int, real or complex)");
    }
    throw DomainError("unknown ring tag");
}

pl_limits to_c(const Limits& l) {
    pl_limits c;
    pl_limits_default(&c);
    c.subset_order_limit = l.subset_order_limit;
    c.memo_budget_bytes = l.memo_budget_bytes;
    c.num_gpus = l.num_gpus;
    return c;
}

std::uint64_t parse_u64(std::string_view key, std::string_view value) {
    if (value.empty()) throw DomainError("PERMLAB_LIMITS: empty value for " + std::string(key));
    std::uint64_t out = 0;
    for (char c : value) {
        if (c < '0' || c > '9') throw DomainError("PERMLAB_LIMITS: non-numeric value for " + std::string(key));
        out = out * 10 + static_cast<std::uint64_t>(c - '0');
    }
    return out;
}

std::uint64_t binom(int s, int l) { return pl_binom(s, l); }

// Cost of evaluating one memo entry of size t (reference permanent.cpp:158-175).
OpCount entry_cost(int t) { return t == 2 ? OpCount{2, 1} : OpCount{static_cast<std::uint64_t>(t), static_cast<std::uint64_t>(t - 1)}; }

}  // namespace

Limits Limits::from_env() {
    Limits limits;
    const char* raw = std::getenv("PERMLAB_LIMITS");
    if (raw == nullptr) return limits;
    std::string_view rest(raw);
    while (!rest.empty()) {
        const auto comma = rest.find(',');
        const std::string_view item = rest.substr(0, comma);
        rest = comma == std::string_view::npos ? std::string_view{} : rest.substr(comma + 1);
        if (item.empty()) continue;
        const auto eq = item.find('=');
        if (eq == std::string_view::npos) {
            throw DomainError("PERMLAB_LIMITS: expected key=value, got '" + std::string(item) + "'");
        }
        const std::string_view key = item.substr(0, eq);
        const std::uint64_t v = parse_u64(key, item.substr(eq + 1));
        if (key == "naive_order_limit") {
            limits.naive_order_limit = static_cast<int>(v);
        } else if (key == "subset_order_limit") {
            limits.subset_order_limit = static_cast<int>(v);
        } else if (key == "enumeration_cap") {
            limits.enumeration_cap = v;
        } else if (key == "memo_budget_bytes") {
            limits.memo_budget_bytes = v;
        } else if (key == "num_gpus") {
            limits.num_gpus = static_cast<int>(v);
        } else {
            throw DomainError("PERMLAB_LIMITS: unknown key '" + std::string(key) + "'");
        }
    }
    return limits;
}

std::string_view ring_name(RingTag tag) {
    switch (tag) {
        case RingTag::Int:
            return "int";
        case RingTag::Real:
            return "real";
        case RingTag::Complex:
            return "complex";
        case RingTag::Rational:
            return "rational";
    }
    throw DomainError("unknown ring tag");
}

RingTag ring_from_name(std::string_view name) {
    if (name == "int") return RingTag::Int;
    if (name == "rational") return RingTag::Rational;
    if (name == "complex") return RingTag::Complex;
    if (name == "real") return RingTag::Real;
    throw DomainError("unknown ring name: " + std::string(name));
}

RingTag ring_of(const RingElement& v) {
    static constexpr RingTag kTags[] = {RingTag::Int, RingTag::Real, RingTag::Complex};
    return kTags[v.index()];
}

bool approx_equal(const Cplx& a, const Cplx& b) {
    const double diff = std::abs(a - b);
    const double scale = std::max(std::abs(a), std::abs(b));
    return diff <= std::max(kComplexAbsTol, kComplexRelTol * scale);
}

bool approx_equal(const RingElement& a, const RingElement& b) {
    if (ring_of(a) != ring_of(b)) throw DomainError("cannot compare values from different rings");
    if (const auto* x = std::get_if<Int>(&a)) return *x == std::get<Int>(b);
    if (const auto* x = std::get_if<Real>(&a)) return approx_equal(Cplx(*x), Cplx(std::get<Real>(b)));
    return approx_equal(std::get<Cplx>(a), std::get<Cplx>(b));
}

std::string to_string(const RingElement& v) {
    char buf[64];
    if (const auto* x = std::get_if<Int>(&v)) return std::to_string(*x);
    if (const auto* x = std::get_if<Real>(&v)) {
        std::snprintf(buf, sizeof buf, "%.17g", *x);
        return buf;
    }
    const Cplx z = std::get<Cplx>(v);
    std::snprintf(buf, sizeof buf, "%.17g", z.real());
    std::string s = buf;
    if (z.imag() == 0.0) return s;
    if (!(z.imag() < 0)) s += "+";
    std::snprintf(buf, sizeof buf, "%.17g", z.imag());
    return s + buf + "i";
}

std::string_view algorithm_name(Algorithm a) {
    switch (a) {
        case Algorithm::Naive:
            return "naive";
        case Algorithm::Ryser:
            return "ryser";
        case Algorithm::StoreZechin:
            return "store-zechin";
    }
    throw DomainError("unknown algorithm tag");
}

Algorithm algorithm_from_name(std::string_view name) {
    if (name == "naive") return Algorithm::Naive;
    if (name == "ryser") return Algorithm::Ryser;
    if (name == "store-zechin") return Algorithm::StoreZechin;
    throw DomainError("unknown algorithm name: " + std::string(name));
}

OpCount store_zechin_counts(int n) {
    OpCount c;
    check(pl_sz_counts(n, &c.multiplications, &c.additions));
    return c;
}

void store_zechin_permanent_batch(RingTag ring, int n, std::int64_t count, const void* entries, void* out,
                                  const Limits& limits, const BatchOptions& options) {
    const pl_limits lim = to_c(limits);
    std::uint32_t flags = 0;
    if (options.device_pointers) flags |= PL_FLAG_DEVICE_PTRS;
    if (options.allow_fma) flags |= PL_FLAG_FMA;
    check(pl_sz_permanent_batch(dtype_of(ring), n, count, entries, out, flags, &lim, options.stream, nullptr));
}

PermanentResult store_zechin_permanent(const SquareMatrix& a, const Limits& limits) {
    const pl_limits lim = to_c(limits);
    PermanentResult r;
    r.algorithm = Algorithm::StoreZechin;
    r.counts = store_zechin_counts(a.order());
    switch (a.ring()) {
        case RingTag::Int: {
            Int v = 0;
            check(pl_sz_permanent(PL_I64, a.order(), a.data(), &v, 0, &lim, nullptr));
            r.value = v;
            break;
        }
        case RingTag::Real: {
            Real v = 0;
            check(pl_sz_permanent(PL_F64, a.order(), a.data(), &v, 0, &lim, nullptr));
            r.value = v;
            break;
        }
        case RingTag::Rational:
            throw DomainError("the rational ring has no device arithmetic (use int, real or complex)");
        case RingTag::Complex: {
            Cplx v;
            check(pl_sz_permanent(PL_C128, a.order(), a.data(), &v, 0, &lim, nullptr));
            r.value = v;
            break;
        }
    }
    return r;
}

bool BigInt::fits_int64() const {
    if (limbs.empty()) return true;
    if (limbs.size() > 1) return false;
    return negative ? limbs[0] <= (std::uint64_t{1} << 63) : limbs[0] < (std::uint64_t{1} << 63);
}

Int BigInt::to_int64() const {
    if (!fits_int64()) throw DomainError("integer value does not fit int64");
    if (limbs.empty()) return 0;
    return negative ? static_cast<Int>(~limbs[0] + 1) : static_cast<Int>(limbs[0]);
}

std::string BigInt::str() const {
    std::vector<std::uint64_t> w = limbs;
    while (!w.empty() && w.back() == 0) w.pop_back();
    if (w.empty()) return "0";
    constexpr std::uint64_t kChunk = 10000000000000000000ull;  // 10^19
    std::vector<std::uint64_t> chunks;
    while (!w.empty()) {
        unsigned __int128 rem = 0;
        for (std::size_t i = w.size(); i-- > 0;) {
            const unsigned __int128 cur = (rem << 64) | w[i];
            w[i] = static_cast<std::uint64_t>(cur / kChunk);
            rem = cur % kChunk;
        }
        chunks.push_back(static_cast<std::uint64_t>(rem));
        while (!w.empty() && w.back() == 0) w.pop_back();
    }
    std::string out = negative ? "-" : "";
    out += std::to_string(chunks.back());
    for (std::size_t i = chunks.size() - 1; i-- > 0;) {
        const std::string d = std::to_string(chunks[i]);
        out += std::string(19 - d.size(), '0') + d;
    }
    return out;
}

namespace {

BigInt exact_int(bool ryser, const Matrix<Int>& a, const Limits& limits) {
    const pl_limits lim = to_c(limits);
    BigInt r;
    Int v = 0;
    const pl_status s = ryser ? pl_ryser_permanent(PL_I64, a.order(), a.entries().data(), &v, 0, &lim, nullptr)
                              : pl_sz_permanent(PL_I64, a.order(), a.entries().data(), &v, 0, &lim, nullptr);
    if (s == PL_OK) {
        r.negative = v < 0;
        if (v != 0) r.limbs.push_back(v < 0 ? ~static_cast<std::uint64_t>(v) + 1 : static_cast<std::uint64_t>(v));
        return r;
    }
    if (s != PL_ERR_OVERFLOW) check(s);
    r.limbs.resize(40);  // 34 x 34 int64 entries need at most 37
    std::size_t nl = 0;
    std::int32_t neg = 0;
    check((ryser ? pl_ryser_permanent_bigint : pl_sz_permanent_bigint)(a.order(), a.entries().data(), r.limbs.data(),
                                                                       r.limbs.size(), &nl, &neg, &lim, nullptr));
    r.limbs.resize(nl);
    r.negative = neg != 0;
    return r;
}

}  // namespace

BigInt store_zechin_permanent_exact(const Matrix<Int>& a, const Limits& limits) { return exact_int(false, a, limits); }
BigInt ryser_permanent_exact(const Matrix<Int>& a, const Limits& limits) { return exact_int(true, a, limits); }

OpCount ryser_counts(int n) {
    OpCount c;
    check(pl_ryser_counts(n, &c.multiplications, &c.additions));
    return c;
}

PermanentResult ryser_permanent(const SquareMatrix& a, const Limits& limits) {
    const pl_limits lim = to_c(limits);
    PermanentResult r;
    r.algorithm = Algorithm::Ryser;
    r.counts = ryser_counts(a.order());
    switch (a.ring()) {
        case RingTag::Int: {
            Int v = 0;
            check(pl_ryser_permanent(PL_I64, a.order(), a.data(), &v, 0, &lim, nullptr));
            r.value = v;
            break;
        }
        case RingTag::Real: {
            Real v = 0;
            check(pl_ryser_permanent(PL_F64, a.order(), a.data(), &v, 0, &lim, nullptr));
            r.value = v;
            break;
        }
        case RingTag::Rational:
            throw DomainError("the rational ring has no device arithmetic (use int, real or complex)");
        case RingTag::Complex: {
            Cplx v;
            check(pl_ryser_permanent(PL_C128, a.order(), a.data(), &v, 0, &lim, nullptr));
            r.value = v;
            break;
        }
    }
    return r;
}

// Closed form of the reference's per-term attribution (permanent.cpp:179-199):
// term j first demands exactly the subsets T of full \ {j} with
// {0..j-1} subset of T and 2 <= |T| <= n-1 (everything missing one of
// 0..j-1 was memoised by an earlier term), plus its own product.
AttributionReport store_zechin_attributed(const SquareMatrix& a, const Limits& limits) {
    const int n = a.order();
    if (n < 3) throw DomainError("attribution needs order >= 3; orders 1 and 2 are base cases");
    if (n > limits.subset_order_limit) {
        throw DomainError("matrix order exceeds subset_order_limit (" + std::to_string(limits.subset_order_limit) + ")");
    }
    AttributionReport rep;
    for (int j = 0; j < n; ++j) {
        OpCount term{1, 0};
        const int free = n - 1 - j;
        for (int u = 0; u <= free; ++u) {
            const int t = j + u;
            if (t < 2 || t > n - 1) continue;
            const OpCount c = entry_cost(t);
            term += OpCount{binom(free, u) * c.multiplications, binom(free, u) * c.additions};
        }
        rep.per_term.push_back(term);
        rep.totals += term;
    }
    rep.final_combination_adds = static_cast<std::uint64_t>(n) - 1;
    rep.totals += OpCount{0, rep.final_combination_adds};
    return rep;
}

StoreZechinRun store_zechin_run(const SquareMatrix& a, const Limits& limits) {
    StoreZechinRun run;
    run.result = store_zechin_permanent(a, limits);
    const int n = a.order();
    check(pl_sz_diagnostics(n, &run.cache_misses, &run.distinct_subsets));
    if (n >= 3) {
        run.attribution = store_zechin_attributed(a, limits);
    } else {
        run.attribution.totals = run.result.counts;
    }
    return run;
}

std::vector<PermanentResult> store_zechin_permanent_batch(const std::vector<SquareMatrix>& batch,
                                                          const Limits& limits) {
    std::vector<PermanentResult> out;
    if (batch.empty()) return out;
    const int n = batch.front().order();
    const RingTag ring = batch.front().ring();
    for (const auto& m : batch) {
        if (m.order() != n || m.ring() != ring) {
            throw DomainError("batch matrices must share one order and one ring");
        }
    }
    const std::size_t per = static_cast<std::size_t>(n) * n;
    const OpCount counts = store_zechin_counts(n);
    auto run = [&](auto tag) {
        using T = decltype(tag);
        std::vector<T> flat;
        flat.reserve(per * batch.size());
        for (const auto& m : batch) {
            const auto& e = m.as<T>().entries();
            flat.insert(flat.end(), e.begin(), e.end());
        }
        std::vector<T> vals(batch.size());
        store_zechin_permanent_batch(ring, n, static_cast<std::int64_t>(batch.size()), flat.data(), vals.data(),
                                     limits);
        for (const T& v : vals) out.push_back({RingElement(v), counts, Algorithm::StoreZechin});
    };
    switch (ring) {
        case RingTag::Int:
            run(Int{});
            break;
        case RingTag::Real:
            run(Real{});
            break;
        case RingTag::Complex:
            run(Cplx{});
            break;
        case RingTag::Rational:
            throw DomainError("the rational ring has no device arithmetic (use int, real or complex)");
    }
    return out;
}

}  // namespace permlab

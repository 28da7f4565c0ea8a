// TEST INFRASTRUCTURE ONLY (oracle/_ref). A C-callable wrapper around the
// reference engine compiled UNMODIFIED from /root/reference/proj/src
// (permanent.cpp, limits.cpp, ring.cpp, matrix.cpp, boson.cpp) against the
// Boost shim in oracle/shim. It exists so tests can pin the oracle
// restatement (sz_oracle.c) and the config generators against the
// reference itself, and so bench.py can time the reference's own CPU path
// ("cpu_baseline.kind = reference"). Nothing in the product links it.
//
// Entry points wrap the reference's public API:
//   permlab::store_zechin_permanent / store_zechin_run
//       (reference include/permlab/permanent.hpp:90,96)
//   permlab::naive_permanent / ryser_permanent   (permanent.hpp:77,84)
//   permlab::haar_unitary, outcome_probability, full_distribution, sample,
//   enumerate_patterns                            (include/permlab/boson.hpp)
// Status codes: 0 ok, 1 DomainError (message via ref_last_error), 2 the value
// (or an intermediate) left the shim's 128-bit range, 3 other exception.
#include <algorithm>
#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <json.hpp>

#include "permlab/boson.hpp"
#include "permlab/matrix.hpp"
#include "permlab/permanent.hpp"

using namespace permlab;

namespace {

thread_local std::string g_last_error;

Limits make_limits(int subset_order_limit, std::uint64_t memo_budget_bytes) {
    Limits l;
    if (subset_order_limit > 0) l.subset_order_limit = subset_order_limit;
    if (memo_budget_bytes > 0) l.memo_budget_bytes = memo_budget_bytes;
    l.naive_order_limit = 12;
    return l;
}

SquareMatrix int_matrix(int n, const std::int64_t* a) {
    std::vector<Int> e(static_cast<std::size_t>(n) * n);
    for (std::size_t i = 0; i < e.size(); ++i) e[i] = Int(static_cast<long long>(a[i]));
    return SquareMatrix(Matrix<Int>(n, std::move(e)));
}

SquareMatrix cplx_matrix(int n, const double* a, bool real_only) {
    std::vector<Cplx> e(static_cast<std::size_t>(n) * n);
    for (std::size_t i = 0; i < e.size(); ++i) {
        e[i] = real_only ? Cplx(a[i], 0.0) : Cplx(a[2 * i], a[2 * i + 1]);
    }
    return SquareMatrix(Matrix<Cplx>(n, std::move(e)));
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const DomainError& e) {
        g_last_error = e.what();
        return 1;
    } catch (const std::overflow_error& e) {
        g_last_error = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 3;
    }
}

void put_int(const RingElement& v, std::int64_t* lo, std::int64_t* hi) {
    const __int128 w = std::get<Int>(v).raw();
    *lo = static_cast<std::int64_t>(static_cast<std::uint64_t>(w));
    *hi = static_cast<std::int64_t>(w >> 64);
}

void put_cplx(const RingElement& v, double* out) {
    const Cplx z = std::get<Cplx>(v);
    out[0] = z.real();
    out[1] = z.imag();
}

template <typename Body>
int run_chunks(std::int64_t count, int nthreads, Body&& body) {
    nthreads = std::max(1, nthreads);
    std::vector<int> status(static_cast<std::size_t>(nthreads), 0);
    std::vector<std::thread> pool;
    const std::int64_t per = (count + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        const std::int64_t b0 = t * per;
        const std::int64_t b1 = std::min<std::int64_t>(count, b0 + per);
        pool.emplace_back([&, t, b0, b1] {
            for (std::int64_t b = b0; b < b1 && status[t] == 0; ++b) status[t] = body(b);
        });
    }
    for (auto& th : pool) th.join();
    for (int s : status) {
        if (s != 0) return s;
    }
    return 0;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_last_error.c_str(); }

int ref_sz_i64(int n, const std::int64_t* a, std::int64_t* lo, std::int64_t* hi, std::uint64_t* mults,
               std::uint64_t* adds, int subset_order_limit, std::uint64_t memo_budget_bytes) {
    return guarded([&] {
        const PermanentResult r =
            store_zechin_permanent(int_matrix(n, a), make_limits(subset_order_limit, memo_budget_bytes));
        put_int(r.value, lo, hi);
        if (mults) *mults = r.counts.multiplications;
        if (adds) *adds = r.counts.additions;
    });
}

int ref_sz_c128(int n, const double* a, double* out, std::uint64_t* mults, std::uint64_t* adds,
                int subset_order_limit, std::uint64_t memo_budget_bytes) {
    return guarded([&] {
        const PermanentResult r =
            store_zechin_permanent(cplx_matrix(n, a, false), make_limits(subset_order_limit, memo_budget_bytes));
        put_cplx(r.value, out);
        if (mults) *mults = r.counts.multiplications;
        if (adds) *adds = r.counts.additions;
    });
}

// Real matrices go through Matrix<Cplx> with imag = 0: the reference has no
// real-double ring (reference include/permlab/ring.hpp:43).
int ref_sz_f64(int n, const double* a, double* out, int subset_order_limit, std::uint64_t memo_budget_bytes) {
    return guarded([&] {
        const PermanentResult r =
            store_zechin_permanent(cplx_matrix(n, a, true), make_limits(subset_order_limit, memo_budget_bytes));
        double z[2];
        put_cplx(r.value, z);
        out[0] = z[0];
    });
}

// store_zechin_run diagnostics: cache_misses, distinct_subsets and the
// per-term attribution table (2*n entries: mults, adds per term).
int ref_sz_run_i64(int n, const std::int64_t* a, std::int64_t* lo, std::int64_t* hi, std::uint64_t* misses,
                   std::uint64_t* distinct, std::uint64_t* per_term, std::uint64_t* final_adds) {
    return guarded([&] {
        const StoreZechinRun run = store_zechin_run(int_matrix(n, a), make_limits(0, 0));
        put_int(run.result.value, lo, hi);
        *misses = run.cache_misses;
        *distinct = run.distinct_subsets;
        for (std::size_t t = 0; t < run.attribution.per_term.size(); ++t) {
            per_term[2 * t] = run.attribution.per_term[t].multiplications;
            per_term[2 * t + 1] = run.attribution.per_term[t].additions;
        }
        *final_adds = run.attribution.final_combination_adds;
    });
}

int ref_naive_i64(int n, const std::int64_t* a, std::int64_t* lo, std::int64_t* hi) {
    return guarded([&] { put_int(naive_permanent(int_matrix(n, a), make_limits(0, 0)).value, lo, hi); });
}

int ref_ryser_i64(int n, const std::int64_t* a, std::int64_t* lo, std::int64_t* hi) {
    return guarded([&] { put_int(ryser_permanent(int_matrix(n, a), make_limits(0, 0)).value, lo, hi); });
}

int ref_ryser_c128(int n, const double* a, double* out) {
    return guarded([&] { put_cplx(ryser_permanent(cplx_matrix(n, a, false), make_limits(0, 0)).value, out); });
}

// Batches through the reference's public single-matrix API (the reference has
// no batch entry point; its own batch loop is boson.cpp:262-265). Contiguous
// per-thread chunks; the API is reentrant (reference SPEC.md:191-192).
int ref_sz_batch_i64(int n, std::int64_t count, const std::int64_t* a, std::int64_t* out_lohi, int nthreads) {
    return run_chunks(count, nthreads, [&](std::int64_t b) {
        return ref_sz_i64(n, a + b * n * n, &out_lohi[2 * b], &out_lohi[2 * b + 1], nullptr, nullptr, 0, 0);
    });
}

int ref_sz_batch_c128(int n, std::int64_t count, const double* a, double* out, int nthreads) {
    return run_chunks(count, nthreads, [&](std::int64_t b) {
        return ref_sz_c128(n, a + 2 * b * n * n, out + 2 * b, nullptr, nullptr, 0, 0);
    });
}

int ref_sz_batch_f64(int n, std::int64_t count, const double* a, double* out, int nthreads,
                     std::uint64_t memo_budget_bytes) {
    return run_chunks(count, nthreads, [&](std::int64_t b) {
        return ref_sz_f64(n, a + b * n * n, out + b, 0, memo_budget_bytes);
    });
}

int ref_haar(int m, std::uint64_t seed, double* u) {
    return guarded([&] {
        const Interferometer itf = haar_unitary(m, seed);
        const auto& e = itf.unitary().entries();
        for (std::size_t i = 0; i < e.size(); ++i) {
            u[2 * i] = e[i].real();
            u[2 * i + 1] = e[i].imag();
        }
    });
}

// ---- boson sampling (reference include/permlab/boson.hpp:67-99) ----------
// `u` is the m*m unitary, interleaved (re, im); occupancy vectors have length m.

Interferometer make_itf(int m, const double* u) {
    std::vector<Cplx> e(static_cast<std::size_t>(m) * m);
    for (std::size_t i = 0; i < e.size(); ++i) e[i] = Cplx(u[2 * i], u[2 * i + 1]);
    return Interferometer(m, Matrix<Cplx>(m, std::move(e)));
}

int ref_outcome_probability(int m, const double* u, int n, const int* input_modes, const int* occupancy,
                            double* prob) {
    return guarded([&] {
        const Interferometer itf = make_itf(m, u);
        OutputPattern out{std::vector<int>(occupancy, occupancy + m)};
        *prob = outcome_probability(itf, std::vector<int>(input_modes, input_modes + n), out, make_limits(0, 0));
    });
}

// Pattern count of full_distribution; with occupancy/probs non-null (sized by a
// previous call) also the patterns and probabilities, enumeration order.
int ref_full_distribution(int m, const double* u, int n, const int* input_modes, std::uint64_t enumeration_cap,
                          std::int64_t* count, int* occupancy, double* probs) {
    return guarded([&] {
        const Interferometer itf = make_itf(m, u);
        Limits lim = make_limits(0, 0);
        if (enumeration_cap) lim.enumeration_cap = enumeration_cap;
        const OutcomeDistribution d = full_distribution(itf, std::vector<int>(input_modes, input_modes + n), lim);
        *count = static_cast<std::int64_t>(d.entries.size());
        if (occupancy && probs) {
            for (std::size_t i = 0; i < d.entries.size(); ++i) {
                std::copy(d.entries[i].first.occupancy.begin(), d.entries[i].first.occupancy.end(),
                          occupancy + i * static_cast<std::size_t>(m));
                probs[i] = d.entries[i].second;
            }
        }
    });
}

int ref_sample(int m, const double* u, int n, const int* input_modes, std::uint64_t count, std::uint64_t seed,
               std::uint64_t enumeration_cap, int* occupancy) {
    return guarded([&] {
        const Interferometer itf = make_itf(m, u);
        Limits lim = make_limits(0, 0);
        if (enumeration_cap) lim.enumeration_cap = enumeration_cap;
        const auto s = sample(itf, std::vector<int>(input_modes, input_modes + n), count, seed, lim);
        for (std::size_t i = 0; i < s.size(); ++i)
            std::copy(s[i].occupancy.begin(), s[i].occupancy.end(), occupancy + i * static_cast<std::size_t>(m));
    });
}

int ref_enumerate_patterns(int m, int n, std::int64_t* count, int* occupancy) {
    return guarded([&] {
        const auto p = enumerate_patterns(m, n);
        *count = static_cast<std::int64_t>(p.size());
        if (occupancy) {
            for (std::size_t i = 0; i < p.size(); ++i)
                std::copy(p[i].occupancy.begin(), p[i].occupancy.end(), occupancy + i * static_cast<std::size_t>(m));
        }
    });
}

}  // extern "C"

// ---- CLI output formats (test infrastructure for the device CLI,
// paper_1802_02779_b200/cli.py): the reference's own formatting primitives
// (permlab::to_string, Interferometer::to_json, parse_matrix/emit_matrix and
// nlohmann::json's dump as the reference CLI uses it, tools/permlab_cli.cpp)
// applied to given values, so the device CLI's bytes can be compared.

namespace {

int put_text(const std::string& t, char* buf, std::size_t cap) {
    if (t.size() + 1 > cap) return static_cast<int>(t.size() + 1);
    std::memcpy(buf, t.c_str(), t.size() + 1);
    return 0;
}

nlohmann::json value_json(int ring, std::int64_t iv, double re, double im) {
    if (ring == 0) return static_cast<long long>(iv);
    return nlohmann::json::array({re, im});
}

}  // namespace

extern "C" {

// ring 0: int64 value iv; ring 1: complex (re, im)
int ref_fmt_value_text(int ring, std::int64_t iv, double re, double im, char* buf, std::size_t cap) {
    const RingElement v = ring == 0 ? RingElement(Int(static_cast<long long>(iv))) : RingElement(Cplx(re, im));
    return put_text(to_string(v), buf, cap);
}

// the object run_perm prints for --format json
int ref_fmt_perm_json(int ring, std::int64_t iv, double re, double im, int order, std::uint64_t mults,
                      std::uint64_t adds, char* buf, std::size_t cap) {
    const nlohmann::json j{{"algorithm", "store-zechin"},
                           {"order", order},
                           {"value", value_json(ring, iv, re, im)},
                           {"counts", nlohmann::json{{"multiplications", mults}, {"additions", adds}}}};
    return put_text(j.dump(2) + "\n", buf, cap);
}

// the object run_bs_dist prints for --format json: occupancy (count x m), probs (count)
int ref_fmt_dist_json(int m, int photons, std::int64_t count, const int* occupancy, const double* probs, char* buf,
                      std::size_t cap) {
    nlohmann::json entries = nlohmann::json::array();
    for (std::int64_t i = 0; i < count; ++i) {
        std::vector<int> occ(occupancy + i * m, occupancy + (i + 1) * m);
        entries.push_back(nlohmann::json{{"pattern", nlohmann::json(occ)}, {"probability", probs[i]}});
    }
    const nlohmann::json j{{"modes", m}, {"photons", photons}, {"entries", std::move(entries)}};
    return put_text(j.dump(2) + "\n", buf, cap);
}

// compact dump of an array of occupancy arrays (run_bs_sample --format json)
int ref_fmt_sample_json(int m, std::int64_t count, const int* occupancy, char* buf, std::size_t cap) {
    nlohmann::json out = nlohmann::json::array();
    for (std::int64_t i = 0; i < count; ++i) out.push_back(std::vector<int>(occupancy + i * m, occupancy + (i + 1) * m));
    return put_text(out.dump() + "\n", buf, cap);
}

int ref_fmt_itf_json(int m, const double* u, char* buf, std::size_t cap) {
    int rc = 0;
    std::string t;
    rc = guarded([&] { t = make_itf(m, u).to_json(); });
    return rc ? -rc : put_text(t, buf, cap);
}

// parse a matrix file's text the reference way; out: order, ring (0 int, 1 complex), entries
int ref_parse_matrix(const char* text, int csv, int csv_ring_complex, int* order, int* ring, std::int64_t* ints,
                     double* cplx, int cap_entries) {
    return guarded([&] {
        const SquareMatrix m = parse_matrix(text, csv ? MatrixFormat::Csv : MatrixFormat::Json,
                                            csv_ring_complex ? RingTag::Complex : RingTag::Int);
        *order = m.order();
        const int n = m.order();
        if (n * n > cap_entries) throw DomainError("capacity");
        if (m.ring() == RingTag::Int) {
            *ring = 0;
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) ints[i * n + j] = static_cast<std::int64_t>(std::get<Int>(m.entry(i, j)).raw());
        } else if (m.ring() == RingTag::Complex) {
            *ring = 1;
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) {
                    const Cplx z = std::get<Cplx>(m.entry(i, j));
                    cplx[2 * (i * n + j)] = z.real();
                    cplx[2 * (i * n + j) + 1] = z.imag();
                }
        } else {
            *ring = 2;
        }
    });
}

}  // extern "C"

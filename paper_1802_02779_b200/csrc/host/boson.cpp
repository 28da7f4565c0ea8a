// permlab boson-sampling host API over the B200 C ABI (include/permlab/boson.hpp).
//
// Host work: the reference's argument checks and messages (reference
// proj/src/boson.cpp:47-104), pattern enumeration for the returned objects
// (boson.cpp:185-205) and the inverse-CDF draws (boson.cpp:271-290, a serial
// generator). Every probability comes from the device (pl_boson_*).
#include "permlab/boson.hpp"

#include <algorithm>
#include <cmath>
#include <random>
#include <string>

#include "permlab_b200.h"

extern "C" int pl_gen_haar(int m, std::uint64_t seed, int ncols, double* u);  // libpermlab_gen.so

namespace permlab {

namespace {

void check(pl_status s) {
    if (s == PL_OK) return;
    const std::string msg = pl_last_error();
    if (s == PL_ERR_ARG || s == PL_ERR_LIMIT || s == PL_ERR_OVERFLOW) throw DomainError(msg);
    throw std::runtime_error("permlab-b200: " + msg);
}

void check_unitary(const Matrix<Cplx>& u) {
    const int n = u.order();
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            Cplx dot = 0;
            for (int k = 0; k < n; ++k) dot += std::conj(u(k, i)) * u(k, j);
            const Cplx expected = i == j ? Cplx(1.0) : Cplx(0.0);
            if (std::abs(dot - expected) > kUnitarityTol) throw DomainError("matrix is not unitary within 1e-10");
        }
    }
}

void check_input_modes(const std::vector<int>& input_modes, int modes) {
    if (input_modes.empty()) throw DomainError("at least one input mode is required");
    std::vector<char> seen(static_cast<std::size_t>(modes), 0);
    for (int m : input_modes) {
        if (m < 0 || m >= modes) throw DomainError("input mode index out of range");
        if (seen[static_cast<std::size_t>(m)]) throw DomainError("input modes must be distinct");
        seen[static_cast<std::size_t>(m)] = 1;
    }
}

void check_pattern(const OutputPattern& out, int modes, int photons) {
    if (static_cast<int>(out.occupancy.size()) != modes) {
        throw DomainError("occupancy vector length must equal the mode count");
    }
    for (int c : out.occupancy) {
        if (c < 0) throw DomainError("occupancy counts must be nonnegative");
    }
    if (out.total() != photons) throw DomainError("output photon count does not match the input photon count");
}

std::vector<std::int32_t> rows_of(const OutputPattern& out) {
    std::vector<std::int32_t> r;
    for (int mode = 0; mode < static_cast<int>(out.occupancy.size()); ++mode)
        for (int c = 0; c < out.occupancy[static_cast<std::size_t>(mode)]; ++c) r.push_back(mode);
    return r;
}

pl_limits to_c(const Limits& l) {
    pl_limits c;
    pl_limits_default(&c);
    c.subset_order_limit = l.subset_order_limit;
    c.memo_budget_bytes = l.memo_budget_bytes;
    c.num_gpus = l.num_gpus;
    return c;
}

const double* u_ptr(const Interferometer& itf) {
    return reinterpret_cast<const double*>(itf.unitary().entries().data());
}

}  // namespace

int OutputPattern::total() const {
    int s = 0;
    for (int c : occupancy) s += c;
    return s;
}

Interferometer::Interferometer(int modes, Matrix<Cplx> unitary) : modes_(modes), u_(std::move(unitary)) {
    if (modes_ < 1) throw DomainError("mode count must be >= 1");
    if (u_.order() != modes_) throw DomainError("unitary order must equal the mode count");
    check_unitary(u_);
}

Interferometer haar_unitary(int modes, std::uint64_t seed) {
    if (modes < 1) throw DomainError("mode count must be >= 1");
    std::vector<Cplx> u(static_cast<std::size_t>(modes) * modes);
    if (pl_gen_haar(modes, seed, modes, reinterpret_cast<double*>(u.data())) != 0) {
        throw std::runtime_error("permlab-b200: haar generator failed");
    }
    return Interferometer(modes, Matrix<Cplx>(modes, std::move(u)));
}

std::vector<OutputPattern> enumerate_patterns(int modes, int photons) {
    if (modes < 1 || photons < 0) throw DomainError("need modes >= 1 and photons >= 0");
    std::vector<OutputPattern> out;
    // nondecreasing row sequences in lexicographic order (= the reference's
    // recursion, mode 0 taking the most photons first)
    std::vector<int> r(static_cast<std::size_t>(photons), 0);
    while (true) {
        OutputPattern p{std::vector<int>(static_cast<std::size_t>(modes), 0)};
        for (int x : r) ++p.occupancy[static_cast<std::size_t>(x)];
        out.push_back(std::move(p));
        int i = photons - 1;
        while (i >= 0 && r[static_cast<std::size_t>(i)] == modes - 1) --i;
        if (i < 0) break;
        const int v = r[static_cast<std::size_t>(i)] + 1;
        for (int j = i; j < photons; ++j) r[static_cast<std::size_t>(j)] = v;
    }
    return out;
}

Matrix<Cplx> extract_submatrix(const Interferometer& itf, const std::vector<int>& input_modes,
                               const OutputPattern& out) {
    check_input_modes(input_modes, itf.modes());
    const int n = static_cast<int>(input_modes.size());
    check_pattern(out, itf.modes(), n);
    std::vector<Cplx> e;
    e.reserve(static_cast<std::size_t>(n) * n);
    for (int r : rows_of(out))
        for (int c : input_modes) e.push_back(itf.unitary()(r, c));
    return Matrix<Cplx>(n, std::move(e));
}

std::vector<double> outcome_probabilities(const Interferometer& itf, const std::vector<int>& input_modes,
                                          const std::vector<OutputPattern>& outs, const Limits& limits) {
    check_input_modes(input_modes, itf.modes());
    const int n = static_cast<int>(input_modes.size());
    std::vector<std::int32_t> rows;
    rows.reserve(outs.size() * static_cast<std::size_t>(n));
    for (const auto& o : outs) {
        check_pattern(o, itf.modes(), n);
        const auto r = rows_of(o);
        rows.insert(rows.end(), r.begin(), r.end());
    }
    std::vector<double> probs(outs.size());
    const std::vector<std::int32_t> modes(input_modes.begin(), input_modes.end());
    const pl_limits lim = to_c(limits);
    check(pl_boson_probabilities(itf.modes(), u_ptr(itf), n, modes.data(), static_cast<std::int64_t>(outs.size()),
                                 rows.data(), probs.data(), 0, &lim, nullptr, nullptr));
    return probs;
}

double outcome_probability(const Interferometer& itf, const std::vector<int>& input_modes, const OutputPattern& out,
                           const Limits& limits) {
    return outcome_probabilities(itf, input_modes, {out}, limits)[0];
}

double OutcomeDistribution::total_probability() const {
    double sum = 0;
    for (const auto& e : entries) sum += e.second;
    return sum;
}

std::vector<double> distribution_probabilities(const Interferometer& itf, const std::vector<int>& input_modes,
                                               std::uint64_t first, std::uint64_t count) {
    check_input_modes(input_modes, itf.modes());
    const std::vector<std::int32_t> modes(input_modes.begin(), input_modes.end());
    std::vector<double> probs(count);
    check(pl_boson_distribution(itf.modes(), u_ptr(itf), static_cast<int>(modes.size()), modes.data(), first,
                                static_cast<std::int64_t>(count), probs.data(), 0, nullptr));
    return probs;
}

OutcomeDistribution full_distribution(const Interferometer& itf, const std::vector<int>& input_modes,
                                      const Limits& limits) {
    check_input_modes(input_modes, itf.modes());
    const int n = static_cast<int>(input_modes.size());
    if (n > 6) throw DomainError("full distributions are enumerated for at most 6 photons");
    const std::uint64_t count = pl_boson_pattern_count(itf.modes(), n);
    if (count == 0 || count > limits.enumeration_cap) throw DomainError("outcome count exceeds enumeration_cap");
    const std::vector<double> probs = distribution_probabilities(itf, input_modes, 0, count);
    OutcomeDistribution dist;
    dist.input_modes = input_modes;
    auto patterns = enumerate_patterns(itf.modes(), n);
    dist.entries.reserve(patterns.size());
    for (std::size_t i = 0; i < patterns.size(); ++i) dist.entries.emplace_back(std::move(patterns[i]), probs[i]);
    return dist;
}

std::vector<OutputPattern> sample(const Interferometer& itf, const std::vector<int>& input_modes, std::uint64_t count,
                                  std::uint64_t seed, const Limits& limits) {
    const OutcomeDistribution dist = full_distribution(itf, input_modes, limits);
    std::vector<double> cdf;
    cdf.reserve(dist.entries.size());
    double acc = 0;
    for (const auto& e : dist.entries) {
        acc += e.second;
        cdf.push_back(acc);
    }
    std::mt19937_64 gen(seed);
    std::vector<OutputPattern> out;
    out.reserve(count);
    for (std::uint64_t i = 0; i < count; ++i) {
        const double u = static_cast<double>(gen() >> 11) * 0x1.0p-53;
        const auto it = std::upper_bound(cdf.begin(), cdf.end(), u);
        const std::size_t idx = std::min(static_cast<std::size_t>(it - cdf.begin()), dist.entries.size() - 1);
        out.push_back(dist.entries[idx].first);
    }
    return out;
}

}  // namespace permlab

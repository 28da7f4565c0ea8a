// permlab C++ host API, device-backed.
//
// Drop-in for the reference's Store-zechin entry points (reference
// proj/include/permlab/permanent.hpp:34-96) with the same names, argument
// meaning and error type; every call runs on the B200 through the C ABI in
// include/permlab_b200.h. Deviations, all documented in DESIGN.md:
//   * Int is int64_t with a guard (DomainError when an intermediate could
//     reach 2^63) instead of arbitrary precision (reference ring.hpp:31);
//   * a Real (double) ring is added next to the reference's tags; the
//     Rational tag is kept (ring_name / ring_from_name) but has no device
//     arithmetic: a Rational batch call throws DomainError;
//   * Limits.subset_order_limit defaults to the device cap 34 (reference 30)
//     and memo_budget_bytes caps device layer scratch (0 = uncapped);
//   * StoreZechinRun.attribution is computed by a host-side replay of the
//     reference's DFS visiting order (counting only), not by instrumenting
//     the device arithmetic.
#ifndef PERMLAB_B200_PERMANENT_HPP
#define PERMLAB_B200_PERMANENT_HPP

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <variant>
#include <vector>

namespace permlab {

/// Contract violations and exceeded limits (reference errors.hpp:24-27).
class DomainError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

/// Resource guards (reference limits.hpp:23-40); PERMLAB_LIMITS overrides
/// with the reference's key=value syntax (reference limits.cpp:43-76).
struct Limits {
    int naive_order_limit = 12;
    int subset_order_limit = 34;
    std::uint64_t enumeration_cap = 100000;
    std::uint64_t memo_budget_bytes = 0;
    /// Devices to run on (addition; pl_limits.num_gpus): 0 = the current
    /// device; g >= 1 = devices 0..g-1, the large-order layer DP sharded over
    /// them with NCCL, batches split by matrix. PERMLAB_LIMITS key num_gpus.
    int num_gpus = 0;
    static Limits from_env();
};

/// Ring-operation tally (reference op_count.hpp:27-42).
struct OpCount {
    std::uint64_t multiplications = 0;
    std::uint64_t additions = 0;
    OpCount& operator+=(const OpCount& o) {
        multiplications += o.multiplications;
        additions += o.additions;
        return *this;
    }
    friend OpCount operator+(OpCount a, const OpCount& b) { return a += b; }
    bool operator==(const OpCount&) const = default;
};

using Int = std::int64_t;
using Real = double;
using Cplx = std::complex<double>;

/// The reference's tags keep their values (reference ring.hpp:39); Real is
/// the added double ring.
enum class RingTag { Int = 0, Rational = 1, Complex = 2, Real = 3 };
using RingElement = std::variant<Int, Real, Cplx>;

std::string_view ring_name(RingTag tag);          // "int" | "rational" | "complex" | "real"
RingTag ring_from_name(std::string_view name);    // reference ring.cpp:34-45, plus "real"
RingTag ring_of(const RingElement& v);

inline constexpr double kComplexRelTol = 1e-9;  // reference ring.hpp:49-50
inline constexpr double kComplexAbsTol = 1e-12;
bool approx_equal(const Cplx& a, const Cplx& b);
bool approx_equal(const RingElement& a, const RingElement& b);
std::string to_string(const RingElement& v);  // %.17g rendering (reference ring.cpp:95-120)

/// Dense row-major n x n matrix over one ring (reference matrix.hpp:50-189).
template <typename T>
class Matrix {
  public:
    Matrix(int order, std::vector<T> entries) : order_(order), entries_(std::move(entries)) {
        if (order_ < 1) throw DomainError("matrix order must be >= 1");
        if (entries_.size() != static_cast<std::size_t>(order_) * static_cast<std::size_t>(order_)) {
            throw DomainError("entry count does not match order^2");
        }
    }
    static Matrix filled(int order, const T& v) {
        if (order < 1) throw DomainError("matrix order must be >= 1");
        return Matrix(order, std::vector<T>(static_cast<std::size_t>(order) * order, v));
    }
    static Matrix identity(int order) {
        Matrix m = filled(order, T(0));
        for (int i = 0; i < order; ++i) m.entries_[static_cast<std::size_t>(i) * order + i] = T(1);
        return m;
    }
    int order() const { return order_; }
    const std::vector<T>& entries() const { return entries_; }
    const T& operator()(int i, int j) const { return entries_[static_cast<std::size_t>(i) * order_ + j]; }
    Matrix transpose() const {
        std::vector<T> out(entries_.size());
        for (int i = 0; i < order_; ++i)
            for (int j = 0; j < order_; ++j) out[static_cast<std::size_t>(j) * order_ + i] = (*this)(i, j);
        return Matrix(order_, std::move(out));
    }
    /// Entry (i, j) of the result is entry (row_perm[i], col_perm[j]); both
    /// must be permutations of 0..order-1 (reference matrix.hpp:133-146).
    Matrix permute(const std::vector<int>& row_perm, const std::vector<int>& col_perm) const {
        check_permutation(row_perm, "row");
        check_permutation(col_perm, "column");
        std::vector<T> out;
        out.reserve(entries_.size());
        for (int i = 0; i < order_; ++i)
            for (int j = 0; j < order_; ++j) out.push_back((*this)(row_perm[i], col_perm[j]));
        return Matrix(order_, std::move(out));
    }
    Matrix scale_row(int row, const T& s) const {
        if (row < 0 || row >= order_) throw DomainError("row index out of range");
        std::vector<T> out = entries_;
        for (int j = 0; j < order_; ++j) out[static_cast<std::size_t>(row) * order_ + j] = (*this)(row, j) * s;
        return Matrix(order_, std::move(out));
    }
    /// Minor with the listed rows and columns removed (|rows| == |cols| < order;
    /// indices in range and distinct, reference matrix.hpp:93-120).
    Matrix remove_rows_cols(const std::vector<int>& rows, const std::vector<int>& cols) const {
        if (rows.size() != cols.size()) throw DomainError("row and column removal sets must have equal size");
        if (static_cast<int>(rows.size()) >= order_) throw DomainError("cannot remove all rows of a matrix");
        std::vector<char> dr(order_, 0), dc(order_, 0);
        mark(rows, dr, "row");
        mark(cols, dc, "column");
        const int k = order_ - static_cast<int>(rows.size());
        std::vector<T> out;
        for (int i = 0; i < order_; ++i)
            for (int j = 0; j < order_ && !dr[i]; ++j)
                if (!dc[j]) out.push_back((*this)(i, j));
        return Matrix(k, std::move(out));
    }
    bool operator==(const Matrix&) const = default;

  private:
    // The reference's index checks and messages (matrix.hpp:164-184).
    void mark(const std::vector<int>& idx, std::vector<char>& flags, const char* what) const {
        for (int i : idx) {
            if (i < 0 || i >= order_) throw DomainError(std::string(what) + " index out of range");
            if (flags[i]) throw DomainError(std::string("duplicate ") + what + " index");
            flags[i] = 1;
        }
    }
    void check_permutation(const std::vector<int>& p, const char* what) const {
        if (static_cast<int>(p.size()) != order_) throw DomainError(std::string(what) + " permutation has wrong length");
        std::vector<char> seen(order_, 0);
        for (int v : p) {
            if (v < 0 || v >= order_ || seen[v]) throw DomainError(std::string(what) + " argument is not a permutation");
            seen[v] = 1;
        }
    }

    int order_;
    std::vector<T> entries_;
};

/// Ring-erased square matrix (reference matrix.hpp:192-258).
class SquareMatrix {
  public:
    using Variant = std::variant<Matrix<Int>, Matrix<Real>, Matrix<Cplx>>;
    explicit SquareMatrix(Matrix<Int> m) : m_(std::move(m)) {}
    explicit SquareMatrix(Matrix<Real> m) : m_(std::move(m)) {}
    explicit SquareMatrix(Matrix<Cplx> m) : m_(std::move(m)) {}
    RingTag ring() const {
        static constexpr RingTag kTags[] = {RingTag::Int, RingTag::Real, RingTag::Complex};
        return kTags[m_.index()];
    }
    int order() const {
        return std::visit([](const auto& m) { return m.order(); }, m_);
    }
    template <typename T>
    const Matrix<T>& as() const {
        if (const auto* p = std::get_if<Matrix<T>>(&m_)) return *p;
        throw DomainError("matrix ring mismatch");
    }
    const Variant& inner() const { return m_; }
    /// Pointer to the contiguous entries (int64 / double / interleaved complex).
    const void* data() const {
        return std::visit([](const auto& m) -> const void* { return m.entries().data(); }, m_);
    }

  private:
    Variant m_;
};

enum class Algorithm { Naive, Ryser, StoreZechin };
std::string_view algorithm_name(Algorithm a);
Algorithm algorithm_from_name(std::string_view name);

struct PermanentResult {
    RingElement value;
    OpCount counts;  // store-zechin: n*2^(n-1)-n, n*2^(n-1)-2^n+1; ryser: see ryser_counts
    Algorithm algorithm;
};

/// Per-term cost split of the reference's DFS order (reference permanent.hpp:44-48).
struct AttributionReport {
    std::vector<OpCount> per_term;
    std::uint64_t final_combination_adds = 0;
    OpCount totals;
};

struct StoreZechinRun {
    PermanentResult result;
    AttributionReport attribution;
    std::uint64_t cache_misses = 0;
    std::uint64_t distinct_subsets = 0;
};

/// Options of the zero-copy batch overload.
struct BatchOptions {
    bool device_pointers = false;  // entries/out are CUDA device pointers
    bool allow_fma = false;        // contract products into FMAs (not the reference's rounding order)
    void* stream = nullptr;        // cudaStream_t
};

PermanentResult store_zechin_permanent(const SquareMatrix& a, const Limits& limits = {});

/// Arbitrary-precision integer: sign and magnitude as little-endian 64-bit limbs
/// (no limbs = 0). The value of the reference's Int ring (cpp_int, reference
/// ring.hpp:29-31) where it leaves int64.
struct BigInt {
    bool negative = false;
    std::vector<std::uint64_t> limbs;
    bool fits_int64() const;
    Int to_int64() const;     // DomainError unless fits_int64()
    std::string str() const;  // decimal, as cpp_int streams it
};
/// The exact integer permanent at any magnitude (reference permanent.hpp:90 on its
/// Int ring never overflows): the int64 engine where every intermediate fits,
/// otherwise the layer DP on residues modulo 31-bit primes, recombined on the
/// host (pl_sz_permanent_bigint). store_zechin_permanent keeps Int = int64 and
/// throws DomainError on overflow.
BigInt store_zechin_permanent_exact(const Matrix<Int>& a, const Limits& limits = {});
/// The same through Ryser's formula (reference permanent.hpp:84 on its Int ring):
/// 128-bit wrapping sums where the guard bound allows, else inclusion-exclusion sums on
/// residues (pl_ryser_permanent_bigint).
BigInt ryser_permanent_exact(const Matrix<Int>& a, const Limits& limits = {});
/// Ryser's formula on the device (reference permanent.hpp:84): float rings
/// bitwise the reference's visit-order fold, Int exact (guarded like
/// store_zechin_permanent); counts = count_formula(Ryser, n).
PermanentResult ryser_permanent(const SquareMatrix& a, const Limits& limits = {});
/// Closed-form Ryser operation counts (reference cost_model.cpp:168-174).
OpCount ryser_counts(int n);
StoreZechinRun store_zechin_run(const SquareMatrix& a, const Limits& limits = {});
AttributionReport store_zechin_attributed(const SquareMatrix& a, const Limits& limits = {});

/// Batch over matrices of one ring and one order (the reference's callers loop
/// over store_zechin_permanent, e.g. boson.cpp:262-265).
std::vector<PermanentResult> store_zechin_permanent_batch(const std::vector<SquareMatrix>& batch,
                                                          const Limits& limits = {});

/// Zero-copy batch over a contiguous buffer of `count` row-major n x n
/// matrices; `out` receives `count` values of the ring's element type.
void store_zechin_permanent_batch(RingTag ring, int n, std::int64_t count, const void* entries, void* out,
                                  const Limits& limits = {}, const BatchOptions& options = {});

/// Closed-form Store-zechin operation counts (reference cost_model.cpp:176-181).
OpCount store_zechin_counts(int n);

}  // namespace permlab

#endif  // PERMLAB_B200_PERMANENT_HPP

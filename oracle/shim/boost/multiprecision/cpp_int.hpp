// TEST INFRASTRUCTURE ONLY (oracle/). Minimal stand-in for the two
// Boost.Multiprecision types the reference's ring header names
// (reference include/permlab/ring.hpp:23,31,33), so the reference engine
// sources compile unmodified in this image, which has no Boost.
//
//   cpp_int      -> checked signed 128-bit integer; every operation that would
//                   leave the 128-bit range throws std::overflow_error instead
//                   of wrapping, so a shim result is either exact or absent.
//   cpp_rational -> gcd-normalised pair of cpp_int (positive denominator).
//
// All config values (|per| <= 12! and <= 5! * 9^5) are far below 2^127, so the
// Int parity goldens are exact under this shim.
#ifndef PERMLAB_ORACLE_BOOST_SHIM_CPP_INT_HPP
#define PERMLAB_ORACLE_BOOST_SHIM_CPP_INT_HPP

#include <cstdint>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>

namespace boost::multiprecision {

class cpp_int {
  public:
    using wide = __int128;

    cpp_int() = default;
    template <typename I, typename = std::enable_if_t<std::is_integral_v<I>>>
    cpp_int(I v) : v_(static_cast<wide>(v)) {}  // NOLINT(implicit)
    explicit cpp_int(const std::string& text) { parse(text); }
    explicit cpp_int(const char* text) { parse(text); }

    static cpp_int from_wide(wide v) {
        cpp_int out;
        out.v_ = v;
        return out;
    }
    wide raw() const { return v_; }

    friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
        wide r;
        if (__builtin_add_overflow(a.v_, b.v_, &r)) throw std::overflow_error("cpp_int shim: add overflow");
        return from_wide(r);
    }
    friend cpp_int operator-(const cpp_int& a, const cpp_int& b) {
        wide r;
        if (__builtin_sub_overflow(a.v_, b.v_, &r)) throw std::overflow_error("cpp_int shim: sub overflow");
        return from_wide(r);
    }
    friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
        wide r;
        if (__builtin_mul_overflow(a.v_, b.v_, &r)) throw std::overflow_error("cpp_int shim: mul overflow");
        return from_wide(r);
    }
    friend cpp_int operator/(const cpp_int& a, const cpp_int& b) {
        if (b.v_ == 0) throw std::domain_error("cpp_int shim: division by zero");
        return from_wide(a.v_ / b.v_);
    }
    friend cpp_int operator%(const cpp_int& a, const cpp_int& b) {
        if (b.v_ == 0) throw std::domain_error("cpp_int shim: division by zero");
        return from_wide(a.v_ % b.v_);
    }
    cpp_int operator-() const { return cpp_int(0) - *this; }
    cpp_int& operator+=(const cpp_int& o) { return *this = *this + o; }
    cpp_int& operator-=(const cpp_int& o) { return *this = *this - o; }
    cpp_int& operator*=(const cpp_int& o) { return *this = *this * o; }
    cpp_int& operator/=(const cpp_int& o) { return *this = *this / o; }

    friend bool operator==(const cpp_int& a, const cpp_int& b) { return a.v_ == b.v_; }
    friend bool operator!=(const cpp_int& a, const cpp_int& b) { return a.v_ != b.v_; }
    friend bool operator<(const cpp_int& a, const cpp_int& b) { return a.v_ < b.v_; }
    friend bool operator<=(const cpp_int& a, const cpp_int& b) { return a.v_ <= b.v_; }
    friend bool operator>(const cpp_int& a, const cpp_int& b) { return a.v_ > b.v_; }
    friend bool operator>=(const cpp_int& a, const cpp_int& b) { return a.v_ >= b.v_; }

    template <typename T>
    T convert_to() const {
        return static_cast<T>(v_);
    }

    std::string str() const {
        if (v_ == 0) return "0";
        unsigned __int128 mag = v_ < 0 ? -static_cast<unsigned __int128>(v_) : static_cast<unsigned __int128>(v_);
        std::string digits;
        while (mag != 0) {
            digits.insert(digits.begin(), static_cast<char>('0' + static_cast<int>(mag % 10)));
            mag /= 10;
        }
        return v_ < 0 ? "-" + digits : digits;
    }

    friend std::ostream& operator<<(std::ostream& os, const cpp_int& v) { return os << v.str(); }

  private:
    void parse(const std::string& text) {
        std::size_t i = 0;
        bool neg = false;
        if (i < text.size() && (text[i] == '-' || text[i] == '+')) {
            neg = text[i] == '-';
            ++i;
        }
        if (i == text.size()) throw std::invalid_argument("cpp_int shim: empty literal");
        wide acc = 0;
        for (; i < text.size(); ++i) {
            const char c = text[i];
            if (c < '0' || c > '9') throw std::invalid_argument("cpp_int shim: bad literal");
            if (__builtin_mul_overflow(acc, static_cast<wide>(10), &acc) ||
                __builtin_add_overflow(acc, static_cast<wide>(c - '0'), &acc)) {
                throw std::overflow_error("cpp_int shim: literal overflow");
            }
        }
        v_ = neg ? -acc : acc;
    }

    wide v_ = 0;
};

inline cpp_int shim_gcd(cpp_int a, cpp_int b) {
    __int128 x = a.raw() < 0 ? -a.raw() : a.raw();
    __int128 y = b.raw() < 0 ? -b.raw() : b.raw();
    while (y != 0) {
        const __int128 t = x % y;
        x = y;
        y = t;
    }
    return cpp_int::from_wide(x);
}

class cpp_rational {
  public:
    cpp_rational() = default;
    template <typename I, typename = std::enable_if_t<std::is_integral_v<I>>>
    cpp_rational(I v) : num_(v), den_(1) {}  // NOLINT(implicit)
    cpp_rational(const cpp_int& v) : num_(v), den_(1) {}  // NOLINT(implicit)
    cpp_rational(const cpp_int& n, const cpp_int& d) : num_(n), den_(d) { normalise(); }

    friend const cpp_int& numerator(const cpp_rational& r) { return r.num_; }
    friend const cpp_int& denominator(const cpp_rational& r) { return r.den_; }

    friend cpp_rational operator+(const cpp_rational& a, const cpp_rational& b) {
        return {a.num_ * b.den_ + b.num_ * a.den_, a.den_ * b.den_};
    }
    friend cpp_rational operator-(const cpp_rational& a, const cpp_rational& b) {
        return {a.num_ * b.den_ - b.num_ * a.den_, a.den_ * b.den_};
    }
    friend cpp_rational operator*(const cpp_rational& a, const cpp_rational& b) {
        return {a.num_ * b.num_, a.den_ * b.den_};
    }
    friend cpp_rational operator/(const cpp_rational& a, const cpp_rational& b) {
        return {a.num_ * b.den_, a.den_ * b.num_};
    }
    cpp_rational operator-() const { return {-num_, den_}; }
    cpp_rational& operator+=(const cpp_rational& o) { return *this = *this + o; }
    cpp_rational& operator-=(const cpp_rational& o) { return *this = *this - o; }
    cpp_rational& operator*=(const cpp_rational& o) { return *this = *this * o; }
    cpp_rational& operator/=(const cpp_rational& o) { return *this = *this / o; }

    friend bool operator==(const cpp_rational& a, const cpp_rational& b) {
        return a.num_ == b.num_ && a.den_ == b.den_;
    }
    friend bool operator!=(const cpp_rational& a, const cpp_rational& b) { return !(a == b); }

  private:
    void normalise() {
        if (den_ == 0) throw std::domain_error("cpp_rational shim: zero denominator");
        if (den_ < 0) {
            num_ = -num_;
            den_ = -den_;
        }
        const cpp_int g = shim_gcd(num_, den_);
        if (g != 0 && g != 1) {
            num_ = num_ / g;
            den_ = den_ / g;
        }
    }

    cpp_int num_ = 0;
    cpp_int den_ = 1;
};

}  // namespace boost::multiprecision

#endif  // PERMLAB_ORACLE_BOOST_SHIM_CPP_INT_HPP

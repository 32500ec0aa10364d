// Minimal stand-in for boost::rational<T> so the reference's headers compile
// without Boost (Boost is not in this image). Test
// infrastructure only: the routing/numerics data path never evaluates a Rat.
#pragma once
#include <numeric>
#include <stdexcept>

namespace boost {
template <class T>
class rational {
public:
    rational() : n_(0), d_(1) {}
    rational(T n) : n_(n), d_(1) {}  // NOLINT(implicit)
    rational(T n, T d) : n_(n), d_(d) { norm(); }
    T numerator() const { return n_; }
    T denominator() const { return d_; }
    friend rational operator+(const rational& a, const rational& b) {
        return rational(a.n_ * b.d_ + b.n_ * a.d_, a.d_ * b.d_);
    }
    friend rational operator-(const rational& a, const rational& b) {
        return rational(a.n_ * b.d_ - b.n_ * a.d_, a.d_ * b.d_);
    }
    friend rational operator*(const rational& a, const rational& b) {
        return rational(a.n_ * b.n_, a.d_ * b.d_);
    }
    friend rational operator/(const rational& a, const rational& b) {
        return rational(a.n_ * b.d_, a.d_ * b.n_);
    }
    rational& operator+=(const rational& o) { return *this = *this + o; }
    rational& operator-=(const rational& o) { return *this = *this - o; }
    rational& operator*=(const rational& o) { return *this = *this * o; }
    rational& operator/=(const rational& o) { return *this = *this / o; }
    friend bool operator==(const rational& a, const rational& b) {
        return a.n_ == b.n_ && a.d_ == b.d_;
    }
    friend bool operator!=(const rational& a, const rational& b) { return !(a == b); }
    friend bool operator<(const rational& a, const rational& b) {
        return static_cast<__int128>(a.n_) * b.d_ < static_cast<__int128>(b.n_) * a.d_;
    }
    friend bool operator>(const rational& a, const rational& b) { return b < a; }
    friend bool operator<=(const rational& a, const rational& b) { return !(b < a); }
    friend bool operator>=(const rational& a, const rational& b) { return !(a < b); }

private:
    void norm() {
        if (d_ == 0) throw std::domain_error("bad rational: zero denominator");
        if (d_ < 0) { n_ = -n_; d_ = -d_; }
        T g = std::gcd(n_ < 0 ? -n_ : n_, d_);
        if (g > 1) { n_ /= g; d_ /= g; }
    }
    T n_, d_;
};
}  // namespace boost

// sfconv:: drop-in (B200 build) -- exact rationals used by AlgorithmSpec.
// Same names and semantics as the reference's include/sfconv/rational.hpp:14-168
// (overflow-checked int64 fractions, row-major matrices, exact solve); this is an
// independent implementation for the plan / catalog layer of libsfc_b200.so.
#pragma once

#include <cstdint>
#include <initializer_list>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

namespace sfconv {

struct Rat {
    std::int64_t num = 0;
    std::int64_t den = 1;

    Rat() = default;
    Rat(std::int64_t n) : num(n), den(1) {}
    Rat(std::int64_t n, std::int64_t d) : num(n), den(d) { normalize(); }

    static std::int64_t mul_ck(std::int64_t a, std::int64_t b) {
        std::int64_t r;
        if (__builtin_mul_overflow(a, b, &r)) throw std::overflow_error("rational mul overflow");
        return r;
    }
    static std::int64_t add_ck(std::int64_t a, std::int64_t b) {
        std::int64_t r;
        if (__builtin_add_overflow(a, b, &r)) throw std::overflow_error("rational add overflow");
        return r;
    }
    void normalize() {
        if (den == 0) throw std::domain_error("rational with zero denominator");
        if (den < 0) num = mul_ck(num, -1), den = mul_ck(den, -1);
        const std::int64_t g = std::gcd(num < 0 ? -num : num, den);
        if (g > 1) num /= g, den /= g;
    }
    bool is_zero() const { return num == 0; }
    double to_double() const { return double(num) / double(den); }
    std::string str() const { return den == 1 ? std::to_string(num) : std::to_string(num) + "/" + std::to_string(den); }

    friend Rat operator+(const Rat& a, const Rat& b) {
        const std::int64_t g = std::gcd(a.den, b.den);
        return Rat(add_ck(mul_ck(a.num, b.den / g), mul_ck(b.num, a.den / g)), mul_ck(a.den, b.den / g));
    }
    friend Rat operator-(const Rat& a) { return Rat(mul_ck(a.num, -1), a.den); }
    friend Rat operator-(const Rat& a, const Rat& b) { return a + (-b); }
    friend Rat operator*(const Rat& a, const Rat& b) { return Rat(mul_ck(a.num, b.num), mul_ck(a.den, b.den)); }
    friend Rat operator/(const Rat& a, const Rat& b) {
        if (b.num == 0) throw std::domain_error("rational division by zero");
        return Rat(mul_ck(a.num, b.den), mul_ck(a.den, b.num));
    }
    Rat& operator+=(const Rat& o) { return *this = *this + o; }
    Rat& operator-=(const Rat& o) { return *this = *this - o; }
    Rat& operator*=(const Rat& o) { return *this = *this * o; }
    friend bool operator==(const Rat& a, const Rat& b) { return a.num == b.num && a.den == b.den; }
    friend bool operator!=(const Rat& a, const Rat& b) { return !(a == b); }
};

struct RatMatrix {
    int rows = 0;
    int cols = 0;
    std::vector<Rat> a;

    RatMatrix() = default;
    RatMatrix(int r, int c) : rows(r), cols(c), a(std::size_t(r) * c) {}
    RatMatrix(std::initializer_list<std::initializer_list<std::int64_t>> init);

    Rat& at(int r, int c) { return a[std::size_t(r) * cols + c]; }
    const Rat& at(int r, int c) const { return a[std::size_t(r) * cols + c]; }

    static RatMatrix identity(int n);
    RatMatrix transposed() const;
    RatMatrix inverse() const;
    std::vector<double> to_double() const;

    friend RatMatrix operator*(const RatMatrix& x, const RatMatrix& y);
    friend bool operator==(const RatMatrix& x, const RatMatrix& y) {
        return x.rows == y.rows && x.cols == y.cols && x.a == y.a;
    }
};

// Exact solution of M x = b; domain_error when inconsistent, free variables 0.
std::vector<Rat> solve_exact(const RatMatrix& M, const std::vector<Rat>& b);

}  // namespace sfconv

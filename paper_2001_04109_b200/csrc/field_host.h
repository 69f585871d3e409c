// Host-side prime-field setup: primality, Legendre symbol, canonical square
// roots, the skew-orthogonal Y and the nrsyf 2x2 factor.  O(log p) scalar
// work done once per call, before any kernel runs.
//
// Restates the reference's PrimeField setup routines
// (proj/src/fields.cpp:12-18, 33-123) and skew_orthogonal / nrsyf
// (proj/include/fsyrk/skew.hpp:41-73, 180-194).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <utility>

namespace fsyrk_b200::host {

inline bool is_prime(uint64_t n) {
    if (n < 2) return false;
    if (n % 2 == 0) return n == 2;
    for (uint64_t d = 3; d * d <= n; d += 2)
        if (n % d == 0) return false;
    return true;
}

struct Field {
    uint64_t p;
    uint64_t mu;  // floor(2^64 / p): Barrett reduction of products < 2^62 (p < 2^31)
    Field(uint64_t p_) : p(p_), mu(p_ > 1 ? (uint64_t)((((unsigned __int128)1) << 64) / p_) : 0) {}
    uint64_t mul(uint64_t a, uint64_t b) const {
        const uint64_t x = a * b;  // a, b < p < 2^31
        if (p < 2) return 0;
        const uint64_t q = (uint64_t)(((unsigned __int128)x * mu) >> 64);  // floor(x / p) - {0, 1}
        const uint64_t r = x - q * p;
        return r >= p ? r - p : r;
    }
    uint64_t add(uint64_t a, uint64_t b) const { uint64_t s = a + b; return s >= p ? s - p : s; }
    uint64_t sub(uint64_t a, uint64_t b) const { return a >= b ? a - b : a + p - b; }
    uint64_t neg(uint64_t a) const { return a == 0 ? 0 : p - a; }
    uint64_t pow(uint64_t b, uint64_t e) const {
        uint64_t r = 1, acc = b % p;
        while (e) {
            if (e & 1) r = mul(r, acc);
            acc = mul(acc, acc);
            e >>= 1;
        }
        return r;
    }
    uint64_t inv(uint64_t a) const { return pow(a, p - 2); }
    int legendre(uint64_t k) const {
        k %= p;
        if (k == 0) return 0;
        return pow(k, (p - 1) / 2) == 1 ? 1 : -1;
    }
    uint64_t lqnr() const {
        uint64_t s = 2;
        while (legendre(s) == 1) ++s;
        return s;
    }
    // Canonical root min(r, p - r); throws std::domain_error for a non-residue.
    uint64_t sqrt(uint64_t k) const {
        k %= p;
        if (p == 2 || k == 0) return k;
        if (legendre(k) != 1) throw std::domain_error("not a square");
        uint64_t r;
        if (p % 4 == 3) {
            r = pow(k, (p + 1) / 4);
        } else {  // Tonelli-Shanks
            uint64_t q = p - 1;
            unsigned s = 0;
            while (q % 2 == 0) { q /= 2; ++s; }
            uint64_t c = pow(lqnr(), q), t = pow(k, q);
            r = pow(k, (q + 1) / 2);
            unsigned m = s;
            while (t != 1) {
                uint64_t t2 = t;
                unsigned i = 0;
                while (t2 != 1) { t2 = mul(t2, t2); ++i; }
                uint64_t b = c;
                for (unsigned j = 0; j + i + 1 < m; ++j) b = mul(b, b);
                m = i;
                c = mul(b, b);
                t = mul(t, c);
                r = mul(r, b);
            }
        }
        return r < p - r ? r : p - r;
    }
    std::pair<uint64_t, uint64_t> sum_of_squares(uint64_t k) const {
        k %= p;
        if (legendre(k) >= 0) return {sqrt(k), 0};
        uint64_t s = lqnr();
        uint64_t c = sqrt(s - 1);
        uint64_t a = sqrt(mul(k, inv(s)));
        return {a, mul(a, c)};
    }
};

struct Skew {
    int form;  // 0 scalar root, 1 pair
    uint64_t a, b;
    int ycost;
};

inline Skew skew_orthogonal(const Field& f) {
    const uint64_t p = f.p;
    if (p == 2) return {0, 1, 0, 0};
    if (p % 4 == 1) {
        uint64_t r = f.sqrt(p - 1);
        return {0, r, 0, r == 1 ? 0 : 1};
    }
    if (p % 8 == 3) return {1, 1, f.sqrt(p - 2), 2};
    auto [a, b] = f.sum_of_squares(p - 1);
    return {1, a, b, a == 1 ? 2 : 3};
}

// nrsyf(alpha, beta): [[a, b], [c, d]] with Y Y^T = diag(alpha, beta); both must be non-residues.
inline bool nrsyf(const Field& f, uint64_t alpha, uint64_t beta, std::array<uint64_t, 4>& y) {
    if (f.legendre(alpha) != -1 || f.legendre(beta) != -1) return false;
    auto [a, b] = f.sum_of_squares(alpha);
    if (a == 0) return false;
    uint64_t d = f.mul(a, f.sqrt(f.mul(beta, f.inv(alpha))));
    uint64_t c = f.neg(f.mul(b, f.mul(d, f.inv(a))));
    y = {a, b, c, d};
    return true;
}

}  // namespace fsyrk_b200::host

// Reference-compatible operation tallies (fsyrk::OpCount semantics).
//
// The reference counts the scalar field operations of its CPU kernels
// (include/fsyrk/opcount.hpp:10-25): every routine adds a closed-form tally
// for the block it touched.  The device path runs other kernels (exact int8
// products, fused additions), so to keep OpCount a drop-in the library fills
// it with what the reference would have counted for the same call: a host
// dry-run of the reference's recursion over shapes only, with each routine's
// tally restated from its source.  Memoised on the shape, so any policy
// (threshold 2, unlimited levels) costs microseconds.
//
//   syrk_classical             matrix.hpp:372-407     gemm_classical_nt        matrix.hpp:317-328
//   gemm_classical_nt_acc      matrix.hpp:331-367     ew_add / ew_sub          matrix.hpp:166-186
//   add_lower                  matrix.hpp:188-199     add_transposed           matrix.hpp:225-236
//   scale_inplace / _lower     matrix.hpp:248-263     apply_skew_right_inplace skew.hpp:124-167
//   wino_rec / wino_peel       winograd.hpp:64-169    gemm_winograd_nt_acc     winograd.hpp:207-235
//   syrk_fast_level / _rec     fast_syrk.hpp:82-157   syrk_fast_acc_level/_rec fast_syrk.hpp:164-267
//   sub_from_padded            fast_syrk.hpp:49-57    syrkd / scale_column     scaled_syrk.hpp:42-104
//   syrkbd (odd characteristic) scaled_syrk.hpp:117-159
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <tuple>
#include <vector>

namespace fsyrk_b200::refops {

struct Tally {
    uint64_t mults = 0, adds = 0;
    Tally& operator+=(const Tally& o) {
        mults += o.mults;
        adds += o.adds;
        return *this;
    }
};

// Scalar constants that change a tally: only whether they equal 0 or 1.
struct Scalar {
    bool zero, one;
    static Scalar of(uint64_t v) { return {v == 0, v == 1}; }
    static Scalar unit() { return {false, true}; }
    static Scalar nil() { return {true, false}; }
};

// What the recursion needs to know about the field and plan.
struct Model {
    uint64_t threshold = 64;
    uint64_t max_levels = ~0ull;
    int skew_form = 0;         // 0 ScalarRoot, 1 Pair (skew.hpp:21-37)
    bool skew_a_one = false;   // ScalarRoot(1) is free; Pair(1, b) costs one mult less
    std::map<std::tuple<uint64_t, uint64_t, uint64_t, uint64_t>, Tally> wino_memo;
    std::map<std::tuple<uint64_t, uint64_t, uint64_t, int, int, int, int, int>, Tally> syrk_memo;

    static uint64_t tri(uint64_t n) { return n * (n + 1) / 2; }

    // apply_skew_right_inplace on rows x cols (skew.hpp:124-167)
    Tally skew(uint64_t elems) const {
        Tally t;
        if (skew_form == 0) {
            if (!skew_a_one) t.mults = elems;
            return t;
        }
        t.mults = (skew_a_one ? 1 : 2) * elems;
        t.adds = elems;
        return t;
    }

    // syrk_classical(alpha, A n x k, beta) (matrix.hpp:372-407)
    static Tally syrk_classical(uint64_t n, uint64_t k, Scalar alpha, Scalar beta) {
        Tally t;
        const uint64_t tr = tri(n);
        if (alpha.zero) {
            if (!beta.zero && !beta.one) t.mults = tr;  // scale_lower_inplace(beta)
            return t;
        }
        t.mults = tr * (k + (alpha.one ? 0 : 1) + (beta.zero || beta.one ? 0 : 1));
        if (k > 0) t.adds = tr * (k - 1);
        if (!beta.zero) t.adds += tr;
        return t;
    }

    // gemm_classical_nt_acc: C (n x m) <- alpha A (n x k) B^T + beta C (matrix.hpp:331-367)
    static Tally gemm_nt_acc_classical(uint64_t n, uint64_t k, uint64_t m, Scalar alpha, Scalar beta) {
        Tally t;
        if (alpha.zero) {
            if (!beta.zero && !beta.one) t.mults = n * m;  // scale_inplace(beta)
            return t;
        }
        t.mults = n * m * (k + (alpha.one ? 0 : 1) + (beta.zero || beta.one ? 0 : 1));
        if (k > 0) t.adds = n * m * (k - 1);
        if (!beta.zero) t.adds += n * m;
        return t;
    }

    // wino_rec: C (m x p) = A (m x n) B^T, B stored p x n (winograd.hpp:64-169)
    Tally wino(uint64_t m, uint64_t n, uint64_t p, uint64_t levels) {
        if (levels == 0 || std::min({m, n, p}) < threshold) {  // wino_classical -> gemm_classical_nt
            Tally t;
            t.mults = m * p * n;
            if (n > 0) t.adds = m * p * (n - 1);
            return t;
        }
        const auto key = std::make_tuple(m, n, p, levels);
        auto it = wino_memo.find(key);
        if (it != wino_memo.end()) return it->second;
        Tally t;
        if (m % 2 || n % 2 || p % 2) {  // wino_peel
            const uint64_t mc = m & ~1ull, nc = n & ~1ull, pc = p & ~1ull;
            if (mc > 0 && nc > 0 && pc > 0) t += wino(mc, nc, pc, levels);
            if (n % 2 == 1 && mc > 0 && pc > 0) {
                t.mults += mc * pc;
                t.adds += mc * pc;
            }
            if (m % 2 == 1) {
                t.mults += p * n;
                if (n > 0) t.adds += p * (n - 1);
            }
            if (p % 2 == 1) {
                t.mults += mc * n;
                if (n > 0) t.adds += mc * (n - 1);
            }
        } else {
            const uint64_t mh = m / 2, nh = n / 2, ph = p / 2;
            const Tally sub = wino(mh, nh, ph, levels - 1);
            for (int i = 0; i < 7; ++i) t += sub;
            t.adds += 4 * mh * nh + 4 * ph * nh + 7 * mh * ph;  // s1..s4, t1..t4, c1..c7
        }
        wino_memo[key] = t;
        return t;
    }

    // gemm_winograd_nt_acc (winograd.hpp:207-235)
    Tally gemm_nt_acc(uint64_t m, uint64_t n, uint64_t p, Scalar alpha, Scalar beta, uint64_t levels) {
        if (levels == 0 || std::min({m, n, p}) < threshold) return gemm_nt_acc_classical(m, n, p, alpha, beta);
        Tally t = wino(m, n, p, levels);
        t.mults += m * p * ((alpha.one ? 0 : 1) + (beta.zero || beta.one ? 0 : 1));
        if (!beta.zero) t.adds += m * p;
        return t;
    }

    // syrk_fast_rec (acc = false, fast_syrk.hpp:135-157) / syrk_fast_acc_rec (acc = true, :246-267)
    Tally syrk(uint64_t n, uint64_t k, uint64_t levels, bool acc, Scalar alpha, Scalar beta) {
        if (!acc) {
            alpha = Scalar::unit();
            beta = Scalar::nil();
        }
        if (levels == 0 || n % 2 || k % 2 || std::min(n, k) < threshold) return syrk_classical(n, k, alpha, beta);
        const auto key = std::make_tuple(n, k, levels, (int)acc, (int)alpha.zero, (int)alpha.one, (int)beta.zero,
                                         (int)beta.one);
        auto it = syrk_memo.find(key);
        if (it != syrk_memo.end()) return it->second;
        Tally t;
        if (k > n) {  // split on k
            const uint64_t k1 = (k / 2) & ~1ull;
            t += syrk(n, k1, levels, acc, alpha, beta);
            t += syrk(n, k - k1, levels, true, acc ? alpha : Scalar::unit(), Scalar::unit());
        } else {
            const bool padded = skew_form == 1 && (k / 2) % 2 == 1;
            if (padded && k / 2 + 1 > n / 2) {
                t = syrk_classical(n, k, alpha, beta);
            } else {
                t = acc ? acc_level(n, k, levels, alpha, beta, padded) : level(n, k, levels, padded);
            }
        }
        syrk_memo[key] = t;
        return t;
    }

    // syrk_fast_level (fast_syrk.hpp:82-133)
    Tally level(uint64_t n, uint64_t k, uint64_t levels, bool padded) {
        const uint64_t h = n / 2, kh = k / 2, kw = kh + (padded ? 1 : 0), next = levels - 1;
        Tally t;
        t.adds += h * kh;       // 1: ew_sub
        t += skew(h * kw);      //    apply Y
        t += skew(h * kw);      // 2: load_and_apply_skew
        t.adds += h * kw;       //    sub_from_padded
        t += wino(h, kw, h, next);  // 3: P4^T
        t.adds += h * kh;       // 4: S3
        t += syrk(h, kw, next, false, Scalar::unit(), Scalar::nil());  // 5: P5
        t.adds += h * kh;       // 6: S4
        t += wino(h, kh, h, next);  // 7: P3
        t += syrk(h, kh, next, false, Scalar::unit(), Scalar::nil());  // 8: P1
        t.adds += tri(h);       // 9: U1
        t.adds += h * h;        // 10: U2 (add_transposed)
        t.adds += h * h;        // 11: U4
        t.adds += tri(h);       // 12: U5
        t += syrk(h, kh, next, false, Scalar::unit(), Scalar::nil());  // 13: P2
        t.adds += tri(h);       // 14: U3
        return t;
    }

    // syrk_fast_acc_level (fast_syrk.hpp:164-244)
    Tally acc_level(uint64_t n, uint64_t k, uint64_t levels, Scalar alpha, Scalar beta, bool padded) {
        const uint64_t h = n / 2, kh = k / 2, kw = kh + (padded ? 1 : 0), next = levels - 1;
        Tally t;
        t.adds += h * kh;  // S1
        t += skew(h * kw);
        t += skew(h * kw);  // S2
        t.adds += h * kw;
        t += wino(h, kw, h, next);  // P4^T
        if (!alpha.one) t.mults += h * h;  // scale_inplace
        t.adds += h * kh;  // S3
        t += syrk(h, kw, next, false, Scalar::unit(), Scalar::nil());  // P5
        if (!alpha.one) t.mults += tri(h);  // scale_lower_inplace
        t.adds += h * kh;  // S4
        t += gemm_nt_acc(h, kh, h, alpha, beta, next);  // P3 (+ beta C21)
        t += syrk(h, kh, next, false, Scalar::unit(), Scalar::nil());  // P1
        if (!alpha.one) t.mults += tri(h);
        t.adds += tri(h);   // U1
        t.adds += h * h;    // U2
        t.adds += h * h;    // U4
        t.adds += tri(h);   // U5
        if (!beta.zero) {
            t.adds += tri(h);
            if (!beta.one) t.mults += tri(h);
        }
        t += syrk(h, kh, next, true, alpha, beta);  // P2 (+ beta C11)
        t.adds += tri(h);   // U3
        return t;
    }
};

}  // namespace fsyrk_b200::refops

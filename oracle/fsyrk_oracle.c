/* CPU oracle: plain-C restatement of the reference's mod-p SYRK hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library, and only as the
 * checker.  The product path (paper_2001_04109_b200/) never links or calls
 * it.
 *
 * Parity of this restatement is PINNED against the reference itself: the
 * golden fixtures in tests/golden/ are produced by oracle/_ref/ref_driver,
 * which is the unmodified reference code compiled from /root/reference
 * (oracle/Makefile), and tests/test_oracle.py checks every function here
 * against them (random_matrix streams, skew constants, syrk outputs).
 *
 * Reference citations are relative to /root/reference/.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "sha256.h"

typedef unsigned __int128 u128;

/* ------------------------------------------------------------ mt19937_64 */
/* std::mt19937_64 as used by random_matrix (proj/include/fsyrk/matrix.hpp:411-419)
 * and PrimeField::random_element (proj/include/fsyrk/fields.hpp:81-83). */
typedef struct {
    uint64_t mt[312];
    int idx;
} orc_mt64;

static void mt_seed(orc_mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t mt_next(orc_mt64* s) {
    if (s->idx >= 312) {
        const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
        const uint64_t matrix_a = 0xB5026F5AA96619E9ULL;
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & upper) | (s->mt[(i + 1) % 312] & lower);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= matrix_a;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t z = s->mt[s->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* std::uniform_int_distribution<uint64_t>(lo, hi) as implemented by
 * libstdc++ (GCC >= 11) for a full-range 64-bit engine: Lemire's
 * nearly-divisionless multiply-shift with 128-bit products. */
static uint64_t uid_next(orc_mt64* s, uint64_t lo, uint64_t hi) {
    uint64_t range = hi - lo + 1; /* hi - lo < 2^64 - 1 for every use here */
    u128 prod = (u128)mt_next(s) * range;
    uint64_t low = (uint64_t)prod;
    if (low < range) {
        uint64_t threshold = (0 - range) % range;
        while (low < threshold) {
            prod = (u128)mt_next(s) * range;
            low = (uint64_t)prod;
        }
    }
    return lo + (uint64_t)(prod >> 64);
}

/* Exposed so tests can pin the stream itself. */
void orc_mt64_stream(uint64_t seed, size_t count, uint64_t* out) {
    orc_mt64 s;
    mt_seed(&s, seed);
    for (size_t i = 0; i < count; ++i) out[i] = mt_next(&s);
}

/* random_matrix(f, rows, cols, seed): proj/include/fsyrk/matrix.hpp:411-419 */
void orc_random_matrix(uint64_t p, size_t rows, size_t cols, uint64_t seed, uint64_t* out) {
    orc_mt64 s;
    mt_seed(&s, seed);
    for (size_t i = 0; i < rows * cols; ++i) out[i] = uid_next(&s, 0, p - 1);
}

/* nonzero diagonal for the Schur-update config: 1 + rng() % (p - 1) (bench/test
 * convention, mirrored by oracle/ref_driver.cpp make_instance). */
void orc_random_nonzero(uint64_t p, size_t count, uint64_t seed, uint64_t* out) {
    orc_mt64 s;
    mt_seed(&s, seed);
    for (size_t i = 0; i < count; ++i) out[i] = 1 + mt_next(&s) % (p - 1);
}

/* uniform_int_distribution<uint64_t>(lo, hi) stream (pins the libstdc++ mapping). */
void orc_uniform_stream(uint64_t lo, uint64_t hi, size_t count, uint64_t seed, uint64_t* out) {
    orc_mt64 s;
    mt_seed(&s, seed);
    for (size_t i = 0; i < count; ++i) out[i] = uid_next(&s, lo, hi);
}

/* alpha, beta = 1 + rng() % (p - 1) from mt19937_64(abseed) (ref_driver convention). */
void orc_alpha_beta(uint64_t p, uint64_t abseed, uint64_t* alpha, uint64_t* beta) {
    orc_mt64 s;
    mt_seed(&s, abseed);
    *alpha = 1 + mt_next(&s) % (p - 1);
    *beta = 1 + mt_next(&s) % (p - 1);
}

/* -------------------------------------------------------------- PrimeField */
/* proj/include/fsyrk/fields.hpp:49-66, proj/src/fields.cpp:31-127 */
static uint64_t f_add(uint64_t p, uint64_t a, uint64_t b) { uint64_t s = a + b; return s >= p ? s - p : s; }
static uint64_t f_sub(uint64_t p, uint64_t a, uint64_t b) { return a >= b ? a - b : a + p - b; }
static uint64_t f_neg(uint64_t p, uint64_t a) { return a == 0 ? 0 : p - a; }
static uint64_t f_mul(uint64_t p, uint64_t a, uint64_t b) { return (a * b) % p; }

int orc_is_prime(uint64_t n) { /* fields.cpp:12-18 trial division */
    if (n < 2) return 0;
    if (n % 2 == 0) return n == 2;
    for (uint64_t d = 3; d * d <= n; d += 2)
        if (n % d == 0) return 0;
    return 1;
}

uint64_t orc_pow(uint64_t p, uint64_t base, uint64_t e) { /* fields.cpp:45-54 */
    uint64_t r = 1, acc = base % p;
    while (e) {
        if (e & 1) r = f_mul(p, r, acc);
        acc = f_mul(p, acc, acc);
        e >>= 1;
    }
    return r;
}

uint64_t orc_inv(uint64_t p, uint64_t a) { return orc_pow(p, a, p - 2); } /* fields.cpp:56-59 */

int orc_legendre(uint64_t p, uint64_t k) { /* fields.cpp:61-68 */
    k %= p;
    if (k == 0) return 0;
    return orc_pow(p, k, (p - 1) / 2) == 1 ? 1 : -1;
}

uint64_t orc_lqnr(uint64_t p) { /* fields.cpp:38-42 */
    uint64_t s = 2;
    while (orc_legendre(p, s) == 1) ++s;
    return s;
}

/* canonical square root min(r, p - r); returns UINT64_MAX for a non-residue
 * (fields.cpp:70-107; Tonelli-Shanks, any root gives the same canonical min) */
uint64_t orc_sqrt(uint64_t p, uint64_t k) {
    k %= p;
    if (p == 2 || k == 0) return k;
    if (orc_legendre(p, k) != 1) return UINT64_MAX;
    uint64_t r;
    if (p % 4 == 3) {
        r = orc_pow(p, k, (p + 1) / 4);
    } else {
        uint64_t q = p - 1;
        unsigned s = 0;
        while (q % 2 == 0) { q /= 2; ++s; }
        uint64_t c = orc_pow(p, orc_lqnr(p), q);
        uint64_t t = orc_pow(p, k, q);
        r = orc_pow(p, k, (q + 1) / 2);
        unsigned m = s;
        while (t != 1) {
            uint64_t t2 = t;
            unsigned i = 0;
            while (t2 != 1) { t2 = f_mul(p, t2, t2); ++i; }
            uint64_t b = c;
            for (unsigned j = 0; j + i + 1 < m; ++j) b = f_mul(p, b, b);
            m = i;
            c = f_mul(p, b, b);
            t = f_mul(p, t, c);
            r = f_mul(p, r, b);
        }
    }
    return r < p - r ? r : p - r;
}

/* sum_of_squares(k): fields.cpp:114-123 */
void orc_sum_of_squares(uint64_t p, uint64_t k, uint64_t* a, uint64_t* b) {
    k %= p;
    if (orc_legendre(p, k) >= 0) { *a = orc_sqrt(p, k); *b = 0; return; }
    uint64_t s = orc_lqnr(p);
    uint64_t c = orc_sqrt(p, s - 1);
    uint64_t r = f_mul(p, k, orc_inv(p, s));
    uint64_t aa = orc_sqrt(p, r);
    *a = aa;
    *b = f_mul(p, aa, c);
}

/* skew_orthogonal(PrimeField, dim): proj/include/fsyrk/skew.hpp:66-73 and
 * make_scalar_root / make_pair (skew.hpp:41-58).  form: 0 = ScalarRoot, 1 = Pair. */
void orc_skew(uint64_t p, int* form, uint64_t* a, uint64_t* b, int* ycost) {
    if (p == 2) { *form = 0; *a = 1; *b = 0; *ycost = 0; return; }
    if (p % 4 == 1) { *form = 0; *a = orc_sqrt(p, p - 1); *b = 0; *ycost = *a == 1 ? 0 : 1; return; }
    if (p % 8 == 3) { *form = 1; *a = 1; *b = orc_sqrt(p, p - 2); *ycost = 2; return; }
    orc_sum_of_squares(p, p - 1, a, b);
    *form = 1;
    *ycost = *a == 1 ? 2 : 3;
}

/* nrsyf(alpha, beta): proj/include/fsyrk/skew.hpp:180-194.  Returns 0 on
 * success, -1 when alpha or beta is not a non-residue. */
int orc_nrsyf(uint64_t p, uint64_t alpha, uint64_t beta, uint64_t out[4]) {
    if (orc_legendre(p, alpha) != -1 || orc_legendre(p, beta) != -1) return -1;
    uint64_t a, b;
    orc_sum_of_squares(p, alpha, &a, &b);
    uint64_t d = f_mul(p, a, orc_sqrt(p, f_mul(p, beta, orc_inv(p, alpha))));
    uint64_t c = f_neg(p, f_mul(p, b, f_mul(p, d, orc_inv(p, a))));
    out[0] = a; out[1] = b; out[2] = c; out[3] = d;
    return 0;
}

/* ---------------------------------------------------------- classical SYRK */
/* detail::dot + syrk_classical: proj/include/fsyrk/matrix.hpp:144-160, 372-407.
 * Lower triangle of alpha*A*A^T + beta*C; upper triangle untouched. */
static uint64_t dot_mod(uint64_t p, const uint64_t* a, const uint64_t* b, size_t k) {
    u128 acc = 0;
    for (size_t l = 0; l < k; ++l) acc += (u128)a[l] * b[l];
    return (uint64_t)(acc % p);
}

uint64_t orc_dot_mod(uint64_t p, const uint64_t* a, const uint64_t* b, size_t k) { return dot_mod(p, a, b, k); }

void orc_syrk_classical(uint64_t p, uint64_t alpha, const uint64_t* A, size_t n, size_t k, size_t lda,
                        uint64_t beta, uint64_t* C, size_t ldc) {
#pragma omp parallel for schedule(dynamic, 8)
    for (long long ii = 0; ii < (long long)n; ++ii) {
        size_t i = (size_t)ii;
        for (size_t j = 0; j <= i; ++j) {
            uint64_t acc = dot_mod(p, A + i * lda, A + j * lda, k);
            acc = f_mul(p, alpha % p, acc);
            C[i * ldc + j] = beta == 0 ? acc : f_add(p, f_mul(p, beta, C[i * ldc + j]), acc);
        }
    }
}

/* gemm_classical_nt: C = A * B^T (matrix.hpp:317-329) */
static void gemm_nt(uint64_t p, const uint64_t* A, size_t lda, const uint64_t* B, size_t ldb, uint64_t* C,
                    size_t ldc, size_t m, size_t nn, size_t k) {
#pragma omp parallel for schedule(static)
    for (long long ii = 0; ii < (long long)m; ++ii)
        for (size_t j = 0; j < nn; ++j) C[ii * ldc + j] = dot_mod(p, A + ii * lda, B + j * ldb, k);
}

/* abat_oracle (proj/tests/test_scaled_syrk.cpp:25-47, acceptance.cpp:253-275):
 * C = (A * B) * A^T with the block-diagonal B materialised densely; blocks are given as
 * parallel arrays two[i], d[i], beta[i], gamma[i] (scaled_syrk.hpp:13-20). Full C. */
void orc_abat_classical(uint64_t p, const uint64_t* A, size_t n, size_t k, size_t lda, const int* two,
                        const uint64_t* d, const uint64_t* beta, const uint64_t* gamma, size_t nblocks, uint64_t* C,
                        size_t ldc) {
    uint64_t* B = (uint64_t*)calloc(k * k + 1, sizeof(uint64_t));
    uint64_t* AB = (uint64_t*)calloc(n * k + 1, sizeof(uint64_t));
    size_t at = 0;
    for (size_t i = 0; i < nblocks && at < k; ++i) {
        if (two[i]) {
            B[at * k + at + 1] = beta[i] % p;
            B[(at + 1) * k + at] = beta[i] % p;
            B[(at + 1) * k + at + 1] = gamma[i] % p;
            at += 2;
        } else {
            B[at * k + at] = d[i] % p;
            at += 1;
        }
    }
    /* gemm_classical(A, B): AB[r][j] = sum_l A[r][l] B[l][j] (B^T rows = columns of B) */
    uint64_t* BT = (uint64_t*)calloc(k * k + 1, sizeof(uint64_t));
    for (size_t l = 0; l < k; ++l)
        for (size_t j = 0; j < k; ++j) BT[j * k + l] = B[l * k + j];
    gemm_nt(p, A, lda, BT, k, AB, k, n, k, k);
    gemm_nt(p, AB, k, A, lda, C, ldc, n, n, k);
    free(B);
    free(BT);
    free(AB);
}

/* Classical product over F_{p^2} = F_p[x] / (x^2 - ns) (QuadExtField, fields.hpp:148-176):
 * C[i][j] = sum_l A[i][l] * (conj ? conj(A[j][l]) : A[j][l]) for j <= i (lower triangle; the
 * reference's syrk_classical with conjugate, matrix.hpp:369-407).  Elements are (a, b) pairs. */
void orc_fp2_syrk_classical(uint64_t p, uint64_t ns, const uint64_t* A, size_t n, size_t k, int conj, uint64_t* C) {
#pragma omp parallel for schedule(dynamic, 4)
    for (long long ii = 0; ii < (long long)n; ++ii) {
        const size_t i = (size_t)ii;
        for (size_t j = 0; j <= i; ++j) {
            u128 re = 0, im = 0, nsbb = 0, neg = 0;
            for (size_t l = 0; l < k; ++l) {
                const uint64_t a = A[2 * (i * k + l)], b = A[2 * (i * k + l) + 1];
                const uint64_t c = A[2 * (j * k + l)], d0 = A[2 * (j * k + l) + 1];
                const uint64_t d = conj ? (d0 ? p - d0 : 0) : d0;
                /* (a + bx)(c + dx) = ac + ns bd + (ad + bc) x */
                re += (u128)a * c;
                nsbb += (u128)b * d;
                im += (u128)a * d + (u128)b * c;
            }
            (void)neg;
            const uint64_t bd = (uint64_t)(nsbb % p);
            C[2 * (i * n + j)] = (uint64_t)((re % p + (u128)bd * ns % p) % p);
            C[2 * (i * n + j) + 1] = (uint64_t)(im % p);
        }
    }
}

/* ------------------------------------------------- the 5-product recursion */
typedef struct {
    uint64_t p;
    int form;
    uint64_t ya, yb;
    size_t threshold, max_levels;
} orc_plan;

static void plan_init(orc_plan* pl, uint64_t p, size_t threshold, size_t max_levels) {
    int yc;
    pl->p = p;
    orc_skew(p, &pl->form, &pl->ya, &pl->yb, &yc);
    pl->threshold = threshold;
    pl->max_levels = max_levels;
}

/* X <- X*Y in place (h x kw, row-major ld): apply_skew_right_inplace,
 * proj/include/fsyrk/skew.hpp:124-167 (Pair acts on column halves). */
static void apply_y(const orc_plan* pl, uint64_t* X, size_t rows, size_t kw, size_t ld) {
    uint64_t p = pl->p;
    if (pl->form == 0) {
        for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < kw; ++j) X[i * ld + j] = f_mul(p, X[i * ld + j], pl->ya);
        return;
    }
    size_t hh = kw / 2;
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < hh; ++j) {
            uint64_t u = X[i * ld + j], v = X[i * ld + hh + j];
            X[i * ld + j] = f_sub(p, f_mul(p, pl->ya, u), f_mul(p, pl->yb, v));
            X[i * ld + hh + j] = f_add(p, f_mul(p, pl->yb, u), f_mul(p, pl->ya, v));
        }
}

static void fast_rec(const orc_plan* pl, const uint64_t* A, size_t n, size_t k, size_t lda, uint64_t* C,
                     size_t ldc, size_t levels);

/* The S-chain and the five products of one level (Table 3 of the paper,
 * proj/include/fsyrk/fast_syrk.hpp:82-133), restated with explicit
 * temporaries instead of the in-place C-quadrant placement.  Outputs are
 * h x kw (S) and h x h (P, with P4 = S1*S2^T, i.e. the transpose of R's
 * stored P4^T).  Any output pointer may be NULL. */
static void level_blocks(const orc_plan* pl, const uint64_t* A, size_t n, size_t k, size_t lda, size_t levels,
                         int padded, uint64_t* S1o, uint64_t* S2o, uint64_t* S3o, uint64_t* S4o, uint64_t* P1,
                         uint64_t* P2, uint64_t* P3, uint64_t* P4, uint64_t* P5) {
    uint64_t p = pl->p;
    size_t h = n / 2, kh = k / 2, kw = kh + (padded ? 1 : 0);
    const uint64_t *a11 = A, *a12 = A + kh, *a21 = A + h * lda, *a22 = A + h * lda + kh;
    uint64_t* S1 = calloc(h * kw, 8);
    uint64_t* S2 = calloc(h * kw, 8);
    uint64_t* S3 = calloc(h * kw, 8);
    uint64_t* S4 = calloc(h * kw, 8);
    uint64_t* Z = calloc(h * kw, 8); /* zero-padded A22 and A12 as h x kw */
    uint64_t* W = calloc(h * kw, 8);
    for (size_t i = 0; i < h; ++i)
        for (size_t j = 0; j < kh; ++j) {
            S1[i * kw + j] = f_sub(p, a21[i * lda + j], a11[i * lda + j]); /* :101 */
            S2[i * kw + j] = a21[i * lda + j];                             /* :105 */
            Z[i * kw + j] = a22[i * lda + j];
            W[i * kw + j] = a12[i * lda + j];
        }
    apply_y(pl, S1, h, kw, kw); /* S1 = (A21 - A11) Y          :102-103 */
    apply_y(pl, S2, h, kw, kw); /* A21 Y                       :105 */
    for (size_t i = 0; i < h * kw; ++i) {
        S2[i] = f_sub(p, Z[i], S2[i]); /* S2 = A22 - A21 Y  :106 */
        S3[i] = f_sub(p, S1[i], Z[i]); /* S3 = S1 - A22     :110 */
        S4[i] = f_add(p, S3[i], W[i]); /* S4 = S3 + A12     :114-115 */
    }
    size_t next = levels - 1;
    uint64_t* tmpa = calloc(h * h, 8);
    if (P4) gemm_nt(p, S1, kw, S2, kw, P4, h, h, h, kw);  /* P4 = S1 S2^T (R stores P4^T) :108 */
    if (P3) gemm_nt(p, Z, kw, S4, kw, P3, h, h, h, kw);   /* P3 = A22 S4^T               :117 */
    if (P5) fast_rec(pl, S3, h, kw, kw, P5, h, next);      /* P5 = S3 S3^T               :112 */
    if (P1) fast_rec(pl, a11, h, kh, lda, P1, h, next);    /* P1 = A11 A11^T             :119 */
    if (P2) fast_rec(pl, a12, h, kh, lda, P2, h, next);    /* P2 = A12 A12^T             :130 */
    if (S1o) memcpy(S1o, S1, h * kw * 8);
    if (S2o) memcpy(S2o, S2, h * kw * 8);
    if (S3o) memcpy(S3o, S3, h * kw * 8);
    if (S4o) memcpy(S4o, S4, h * kw * 8);
    free(S1); free(S2); free(S3); free(S4); free(Z); free(W); free(tmpa);
}

/* syrk_fast_level: U-combination of the five products (fast_syrk.hpp:120-132):
 *   C11 = Low(P1 + P2), C21 = U1 + P4 + P3, C22 = Low(U1 + P4 + P4^T),
 *   with U1 = P1 + P5 completed symmetrically from its lower triangle. */
static void fast_level(const orc_plan* pl, const uint64_t* A, size_t n, size_t k, size_t lda, uint64_t* C,
                       size_t ldc, size_t levels, int padded) {
    uint64_t p = pl->p;
    size_t h = n / 2;
    uint64_t *P1 = calloc(h * h, 8), *P2 = calloc(h * h, 8), *P3 = calloc(h * h, 8);
    uint64_t *P4 = calloc(h * h, 8), *P5 = calloc(h * h, 8);
    level_blocks(pl, A, n, k, lda, levels, padded, NULL, NULL, NULL, NULL, P1, P2, P3, P4, P5);
    for (size_t i = 0; i < h; ++i)
        for (size_t j = 0; j < h; ++j) {
            size_t li = i >= j ? i : j, lj = i >= j ? j : i;
            uint64_t u1 = f_add(p, P1[li * h + lj], P5[li * h + lj]);
            C[(h + i) * ldc + j] = f_add(p, f_add(p, u1, P4[i * h + j]), P3[i * h + j]);
            if (j <= i) {
                C[i * ldc + j] = f_add(p, P1[i * h + j], P2[i * h + j]);
                C[(h + i) * ldc + h + j] = f_add(p, f_add(p, u1, P4[i * h + j]), P4[j * h + i]);
            }
        }
    free(P1); free(P2); free(P3); free(P4); free(P5);
}

static void acc_into(const orc_plan* pl, uint64_t alpha, const uint64_t* X, size_t ldx, uint64_t beta, uint64_t* C,
                     size_t ldc, size_t n) {
    uint64_t p = pl->p;
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j <= i; ++j)
            C[i * ldc + j] = f_add(p, f_mul(p, alpha, X[i * ldx + j]), f_mul(p, beta, C[i * ldc + j]));
}

/* syrk_fast_rec: decision logic of proj/include/fsyrk/fast_syrk.hpp:135-157 */
static void fast_rec(const orc_plan* pl, const uint64_t* A, size_t n, size_t k, size_t lda, uint64_t* C,
                     size_t ldc, size_t levels) {
    size_t mn = n < k ? n : k;
    if (levels == 0 || n % 2 != 0 || k % 2 != 0 || mn < pl->threshold) {
        orc_syrk_classical(pl->p, 1, A, n, k, lda, 0, C, ldc);
        return;
    }
    if (k > n) { /* split on k, then accumulate with beta = 1 (:143-150) */
        size_t k1 = (k / 2) & ~(size_t)1;
        uint64_t* X = calloc(n * n, 8);
        fast_rec(pl, A, n, k1, lda, C, ldc, levels);
        fast_rec(pl, A + k1, n, k - k1, lda, X, n, levels);
        acc_into(pl, 1, X, n, 1, C, ldc, n);
        free(X);
        return;
    }
    int padded = pl->form == 1 && (k / 2) % 2 == 1; /* needs_pair_padding :34-37 */
    if (padded && k / 2 + 1 > n / 2) {             /* :151-155 */
        orc_syrk_classical(pl->p, 1, A, n, k, lda, 0, C, ldc);
        return;
    }
    fast_level(pl, A, n, k, lda, C, ldc, levels, padded);
}

/* syrk_fast_into (fast_syrk.hpp:274-282): Low(C) = Low(A A^T). */
void orc_syrk_fast(uint64_t p, const uint64_t* A, size_t n, size_t k, size_t lda, uint64_t* C, size_t ldc,
                   size_t threshold, size_t max_levels) {
    orc_plan pl;
    plan_init(&pl, p, threshold, max_levels);
    fast_rec(&pl, A, n, k, lda, C, ldc, max_levels);
}

/* syrk_fast_acc (fast_syrk.hpp:293-303): Low(C) = Low(alpha A A^T + beta C).
 * The Table-4 schedule (:164-244) computes exactly this linear combination;
 * the restatement composes it from the plain recursion. */
void orc_syrk_fast_acc(uint64_t p, uint64_t alpha, const uint64_t* A, size_t n, size_t k, size_t lda,
                       uint64_t beta, uint64_t* C, size_t ldc, size_t threshold, size_t max_levels) {
    orc_plan pl;
    plan_init(&pl, p, threshold, max_levels);
    uint64_t* X = calloc(n * n ? n * n : 1, 8);
    fast_rec(&pl, A, n, k, lda, X, n, max_levels);
    acc_into(&pl, alpha % p, X, n, beta % p, C, ldc, n);
    free(X);
}

/* syrkd column transform (proj/include/fsyrk/scaled_syrk.hpp:58-104):
 * builds Abar (n x kbar, kbar = k or k+1) with Abar Abar^T = A D A^T.
 * Returns kbar, or -1 on error (p == 2 / nrsyf failure). */
long orc_syrkd_transform(uint64_t p, const uint64_t* A, size_t n, size_t k, size_t lda, const uint64_t* d,
                         uint64_t* Abar /* n x (k+1) */, size_t ldb) {
    if (p == 2) return -1;
    size_t* nr = malloc((k + 2) * sizeof(size_t));
    uint64_t* dbar = malloc((k + 1) * 8);
    size_t nnr = 0;
    for (size_t j = 0; j < k; ++j) {
        dbar[j] = d[j] % p;
        if (orc_legendre(p, d[j]) == -1) nr[nnr++] = j;
    }
    int augment = nnr % 2 == 1;
    size_t kbar = k + (augment ? 1 : 0);
    for (size_t i = 0; i < n; ++i) {
        for (size_t j = 0; j < k; ++j) Abar[i * ldb + j] = A[i * lda + j];
        if (augment) Abar[i * ldb + k] = 0;
    }
    if (augment) { dbar[k] = d[nr[0]] % p; nr[nnr++] = k; }
    for (size_t j = 0; j < kbar; ++j)
        if (orc_legendre(p, dbar[j]) >= 0) {
            uint64_t s = orc_sqrt(p, dbar[j]);
            if (s != 1)
                for (size_t i = 0; i < n; ++i) Abar[i * ldb + j] = f_mul(p, Abar[i * ldb + j], s);
        }
    for (size_t t = 0; t + 1 < nnr; t += 2) {
        size_t ci = nr[t], cj = nr[t + 1];
        uint64_t y[4];
        if (orc_nrsyf(p, dbar[ci], dbar[cj], y) != 0) { free(nr); free(dbar); return -1; }
        for (size_t r = 0; r < n; ++r) {
            uint64_t u = Abar[r * ldb + ci], v = Abar[r * ldb + cj];
            Abar[r * ldb + ci] = f_add(p, f_mul(p, y[0], u), f_mul(p, y[2], v));
            Abar[r * ldb + cj] = f_add(p, f_mul(p, y[1], u), f_mul(p, y[3], v));
        }
    }
    free(nr);
    free(dbar);
    return (long)kbar;
}

/* syrkd then fast SYRK: Low(C) = Low(A D A^T) (scaled_syrk.hpp:58-104). */
long orc_syrkd(uint64_t p, const uint64_t* A, size_t n, size_t k, size_t lda, const uint64_t* d, uint64_t* C,
               size_t ldc, size_t threshold, size_t max_levels) {
    uint64_t* Abar = calloc(n * (k + 1) + 1, 8);
    long kbar = orc_syrkd_transform(p, A, n, k, lda, d, Abar, k + 1);
    if (kbar >= 0) orc_syrk_fast(p, Abar, n, (size_t)kbar, k + 1, C, ldc, threshold, max_levels);
    free(Abar);
    return kbar;
}

/* White-box access to one level: S1..S4 (h x kw) and P1..P5 (h x h). */
int orc_level_blocks(uint64_t p, const uint64_t* A, size_t n, size_t k, size_t lda, size_t threshold,
                     size_t max_levels, uint64_t* S1, uint64_t* S2, uint64_t* S3, uint64_t* S4, uint64_t* P1,
                     uint64_t* P2, uint64_t* P3, uint64_t* P4, uint64_t* P5) {
    orc_plan pl;
    plan_init(&pl, p, threshold, max_levels);
    if (n % 2 || k % 2 || max_levels == 0) return -1;
    int padded = pl.form == 1 && (k / 2) % 2 == 1;
    level_blocks(&pl, A, n, k, lda, max_levels, padded, S1, S2, S3, S4, P1, P2, P3, P4, P5);
    return padded;
}

void orc_lower_digest(const uint64_t* C, size_t n, size_t ldc, char* hex65) { lower_digest_u64(C, n, ldc, hex65); }

// Drop-in check: the reference's own call sites, switched to the B200 path by
// including fsyrk_b200/fsyrk.hpp with FSYRK_B200_OVERRIDE, against the
// reference's templates called explicitly (fsyrk::syrk_fast<PrimeField>) on
// the same inputs.  Mirrors the reference's test style
// (proj/tests/test_fast_syrk.cpp:14-31 oracle pattern, :71-98 battery,
// :312-375 accumulating variant, :377-385 alias rejection;
// proj/tests/test_scaled_syrk.cpp:104-135 syrkd battery).
//
// TEST INFRASTRUCTURE: built by tests/cpp/Makefile against /root/reference in the build
// container; the binary runs on the GPU box (tests/test_dropin.py, -m gpu).
#include <cstdio>
#include <random>
#include <stdexcept>

#include "fsyrk/count_model.hpp"
#include "fsyrk/fast_syrk.hpp"
#include "fsyrk/scaled_syrk.hpp"
#define FSYRK_B200_OVERRIDE
#include "fsyrk_b200/fsyrk.hpp"

using namespace fsyrk;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond, ...)                    \
    do {                                    \
        if (cond) {                         \
            ++g_pass;                       \
        } else {                            \
            ++g_fail;                       \
            std::printf("FAIL: " __VA_ARGS__); \
            std::printf("\n");              \
        }                                   \
    } while (0)

int main() {
    // 1. battery: unmodified call sites (now the B200 path) vs the reference templates
    std::mt19937_64 rng(2024);
    for (std::uint64_t p : {5ull, 13ull, 131041ull, 3ull, 7ull, 11ull, 131071ull, 65537ull, 65521ull, 2147483647ull}) {
        PrimeField f(p);
        for (int t = 0; t < 6; ++t) {
            std::size_t n = 1 + rng() % 200, k = 1 + rng() % 200;
            RecursionPolicy pol{static_cast<std::size_t>(2 + (rng() % 3) * 6), kUnlimitedLevels};
            auto a = random_matrix(f, n, k, rng());
            auto plan = make_syrk_plan(f, pol);
            OpCount o1, o2;
            auto dev = syrk_fast(f, a.view(), plan, o1);                 // resolves to the B200 overload
            auto ref = syrk_fast<PrimeField>(f, a.view(), plan, o2);     // the reference template
            CHECK(lower_equal(f, dev.view(), ref.view()), "syrk_fast p=%llu n=%zu k=%zu", (unsigned long long)p, n, k);
            CHECK(o1 == o2, "syrk_fast OpCount p=%llu n=%zu k=%zu: %llu/%llu vs %llu/%llu", (unsigned long long)p, n, k,
                  (unsigned long long)o1.mults, (unsigned long long)o1.adds, (unsigned long long)o2.mults,
                  (unsigned long long)o2.adds);
        }
    }
    // 2. accumulating form with random alpha, beta
    {
        PrimeField f(131071);
        std::mt19937_64 r2(55);
        for (int t = 0; t < 6; ++t) {
            std::size_t n = 1 + r2() % 150, k = 1 + r2() % 150;
            auto alpha = f.random_element(r2), beta = f.random_element(r2);
            auto a = random_matrix(f, n, k, r2());
            auto c0 = random_matrix(f, n, n, r2());
            auto c1 = c0, c2 = c0;
            auto plan = make_syrk_plan(f, {2, kUnlimitedLevels});
            OpCount o1, o2;
            syrk_fast_acc(f, alpha, a.view(), beta, c1.view(), plan, o1);
            syrk_fast_acc<PrimeField>(f, alpha, a.view(), beta, c2.view(), plan, o2);
            CHECK(lower_equal(f, c1.view(), c2.view()), "syrk_fast_acc n=%zu k=%zu", n, k);
            CHECK(o1 == o2, "syrk_fast_acc OpCount n=%zu k=%zu", n, k);
        }
    }
    // 3. syrkd through the shim vs the reference's syrkd
    for (std::uint64_t p : {3ull, 7ull, 13ull, 131071ull}) {
        PrimeField f(p);
        std::mt19937_64 r3(p * 7 + 1);
        auto plan = make_syrk_plan(f, {2, kUnlimitedLevels});
        for (int t = 0; t < 5; ++t) {
            std::size_t m = 1 + r3() % 64, n = 1 + r3() % 64;
            auto a = random_matrix(f, m, n, r3());
            std::vector<PrimeField::Element> d(n);
            for (auto& v : d) v = f.random_element(r3);
            OpCount o1, o2;
            auto dev = fsyrk_b200::syrkd(f, a.view(), d, plan, o1);
            auto ref = syrkd<PrimeField>(f, a.view(), d, plan, o2);
            CHECK(lower_equal(f, dev.view(), ref.view()), "syrkd p=%llu m=%zu n=%zu", (unsigned long long)p, m, n);
            CHECK(o1 == o2, "syrkd OpCount p=%llu m=%zu n=%zu", (unsigned long long)p, m, n);
        }
    }
    // 3b. syrkbd through the shim vs the reference's syrkbd (random block structures,
    //     acceptance.cpp:277-345 pattern)
    for (std::uint64_t p : {3ull, 7ull, 13ull, 65537ull, 131071ull, 2147483647ull}) {
        PrimeField f(p);
        std::mt19937_64 r4(p * 11 + 3);
        auto plan = make_syrk_plan(f, {2, kUnlimitedLevels});
        for (int t = 0; t < 6; ++t) {
            const std::size_t m = 1 + r4() % 80, want = 1 + r4() % 40;
            BlockDiagonal<PrimeField> b;
            std::size_t dim = 0;
            while (dim < want) {
                if (r4() % 3 == 0 || dim + 1 == want) {
                    b.blocks.push_back(BlockDiagonal<PrimeField>::scalar(f.random_element(r4)));
                    dim += 1;
                } else {
                    b.blocks.push_back(BlockDiagonal<PrimeField>::two_by_two(1 + r4() % (p - 1), 0));
                    dim += 2;
                }
            }
            auto a = random_matrix(f, m, dim, r4());
            OpCount o1, o2;
            auto dev = fsyrk_b200::syrkbd(f, a.view(), b, plan, o1);
            auto ref = syrkbd<PrimeField>(f, a.view(), b, plan, o2);
            CHECK(lower_equal(f, dev.view(), ref.view()), "syrkbd p=%llu m=%zu k=%zu", (unsigned long long)p, m, dim);
            CHECK(o1 == o2, "syrkbd OpCount p=%llu m=%zu k=%zu", (unsigned long long)p, m, dim);
        }
        BlockDiagonal<PrimeField> bad;
        bad.blocks.push_back(BlockDiagonal<PrimeField>::two_by_two(1, 1));
        Matrix<PrimeField> a2(2, 2, 1);
        OpCount ops;
        bool threw = false;
        try {
            fsyrk_b200::syrkbd(f, a2.view(), bad, plan, ops);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw, "syrkbd gamma != 0 must throw std::invalid_argument (p=%llu)", (unsigned long long)p);
    }
    // 3c. herk_fast over F_{p^2} through the shim vs the reference's herk_fast
    for (std::uint64_t p : {7ull, 13ull, 131071ull, 2147483647ull}) {
        QuadExtField f(p);
        std::mt19937_64 r5(p * 13 + 5);
        for (int t = 0; t < 4; ++t) {
            const std::size_t n = 1 + r5() % 70, k = 1 + r5() % 50;
            auto a = random_matrix(f, n, k, r5());
            auto plan = make_herk_plan(f, {4, kUnlimitedLevels}, t % 2 == 1);
            OpCount o1, o2;
            auto dev = fsyrk_b200::herk_fast(f, a.view(), plan, o1);
            auto ref = herk_fast(f, a.view(), plan, o2);
            CHECK(lower_equal(f, dev.view(), ref.view()), "herk_fast p=%llu n=%zu k=%zu", (unsigned long long)p, n, k);
            CHECK(o1 == o2, "herk_fast OpCount p=%llu n=%zu k=%zu", (unsigned long long)p, n, k);
        }
    }
    // 3d. the reference's count-model reconciliation through the drop-in
    //     (test_fast_syrk.cpp:202-238, the `count` command of tools/fsyrk.cpp:215-242)
    for (std::uint64_t p : {5ull, 13ull, 11ull, 19ull, 7ull, 23ull}) {
        PrimeField f(p);
        const int y = skew_orthogonal(f, 0).ycost;
        for (std::size_t n : {4u, 8u, 16u, 32u})
            for (unsigned rec : {1u, 2u}) {
                if (n < (std::size_t{2} << rec)) continue;
                auto a = random_matrix(f, n, n, n * 10 + rec);
                OpCount ops;
                auto c = syrk_fast(f, a.view(), make_syrk_plan(f, {2, rec}), ops);  // the B200 overload
                (void)c;
                const std::uint64_t expect = count({CountAlg::FastSyrk, n, rec, y, HalfAddConvention::Triangular});
                CHECK(ops.total() == expect, "count model p=%llu n=%zu rec=%u: %llu vs %llu", (unsigned long long)p, n,
                      rec, (unsigned long long)ops.total(), (unsigned long long)expect);
            }
    }
    {
        PrimeField f(5);
        auto a = random_matrix(f, 4, 4, 1);
        OpCount ops;
        syrk_fast(f, a.view(), make_syrk_plan(f, {2, 1}), ops);
        CHECK(ops.total() == 92, "hand-counted cell: %llu", (unsigned long long)ops.total());
    }
    // 4. error convention: aliased output and bad policy throw std::invalid_argument
    {
        PrimeField f(7);
        Matrix<PrimeField> a(8, 8, 1);
        auto plan = make_syrk_plan(f, {2, kUnlimitedLevels});
        OpCount ops;
        bool threw = false;
        try {
            syrk_fast_into(f, a.view(), a.view(), plan, ops);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw, "alias must throw std::invalid_argument");
        threw = false;
        Matrix<PrimeField> c(5, 5, 0);
        try {
            syrk_fast_into(f, a.view(), c.view(), plan, ops);
        } catch (const DimensionError&) {
            threw = true;
        }
        CHECK(threw, "shape mismatch must throw DimensionError");
    }
    std::printf("dropin: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}

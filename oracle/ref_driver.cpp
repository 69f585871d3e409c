// Reference driver: runs the UNMODIFIED reference fsyrk hot path, compiled
// from /root/reference/proj sources (see oracle/Makefile), on seeded inputs.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Used (a) to generate the golden
// fixtures under tests/golden/ (with tests/golden/make_golden.py), (b) to
// precompute lower-triangle digests for the large configs, and (c) as the
// CPU baseline in bench.py (`cpu_baseline.kind = "reference"` and
// `--impl reference`).  It is never linked into the product library.
//
// Entry points exercised (reference file:line):
//   random_matrix            proj/include/fsyrk/matrix.hpp:411-419
//   make_syrk_plan           proj/include/fsyrk/fast_syrk.hpp:20-24
//   syrk_fast_into           proj/include/fsyrk/fast_syrk.hpp:274-282
//   syrk_fast_acc            proj/include/fsyrk/fast_syrk.hpp:293-303
//   syrkd                    proj/include/fsyrk/scaled_syrk.hpp:58-104
//   syrkbd                   proj/include/fsyrk/scaled_syrk.hpp:117-159
//   syrk_classical           proj/include/fsyrk/matrix.hpp:372-407
//
// Output: one JSON line on stdout.
#include <atomic>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "fsyrk/fast_syrk.hpp"
#include "fsyrk/scaled_syrk.hpp"
#include "sha256.h"

using namespace fsyrk;

namespace {

struct Args {
    std::uint64_t p = 131071;
    std::size_t n = 64, k = 64;
    std::uint64_t seed = 42;
    std::size_t threshold = 64;
    std::size_t levels = kUnlimitedLevels;
    std::string mode = "plain";  // plain | acc | schur | classical | syrkbd
    std::uint64_t cseed = 43, abseed = 7, dseed = 44;
    bool mirror = false;
    int threads = 1;
    int reps = 1;
    std::string out_a, out_c, out_c0, out_d;
    bool digest = true;
    int sample = 0;
    bool alpha_set = false, beta_set = false;
    std::uint64_t alpha = 1, beta = 0;
};

[[noreturn]] void usage() {
    std::fprintf(stderr,
                 "usage: ref_driver [--p P] [--n N] [--k K] [--seed S] [--threshold T]\n"
                 "  [--levels L|inf] [--mode plain|acc|schur|classical|syrkbd|herk|syrk2] [--cseed S] [--abseed S]\n"
                 "  [--alpha a --beta b] [--dseed S] [--mirror] [--threads T] [--reps R]\n"
                 "  [--out-a F] [--out-c F] [--out-c0 F] [--out-d F] [--no-digest] [--sample N]\n");
    std::exit(2);
}

Args parse(int argc, char** argv) {
    Args a;
    for (int i = 1; i < argc; ++i) {
        std::string k = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) usage();
            return argv[++i];
        };
        if (k == "--p") a.p = std::stoull(val());
        else if (k == "--n") a.n = std::stoull(val());
        else if (k == "--k") a.k = std::stoull(val());
        else if (k == "--seed") a.seed = std::stoull(val());
        else if (k == "--threshold") a.threshold = std::stoull(val());
        else if (k == "--levels") {
            std::string v = val();
            a.levels = v == "inf" ? kUnlimitedLevels : std::stoull(v);
        } else if (k == "--mode") a.mode = val();
        else if (k == "--cseed") a.cseed = std::stoull(val());
        else if (k == "--abseed") a.abseed = std::stoull(val());
        else if (k == "--dseed") a.dseed = std::stoull(val());
        else if (k == "--alpha") { a.alpha = std::stoull(val()); a.alpha_set = true; }
        else if (k == "--beta") { a.beta = std::stoull(val()); a.beta_set = true; }
        else if (k == "--mirror") a.mirror = true;
        else if (k == "--threads") a.threads = std::stoi(val());
        else if (k == "--reps") a.reps = std::stoi(val());
        else if (k == "--out-a") a.out_a = val();
        else if (k == "--out-c") a.out_c = val();
        else if (k == "--out-c0") a.out_c0 = val();
        else if (k == "--out-d") a.out_d = val();
        else if (k == "--no-digest") a.digest = false;
        else if (k == "--sample") a.sample = std::stoi(val());
        else usage();
    }
    return a;
}

void dump(const std::string& path, const void* data, std::size_t bytes) {
    if (path.empty()) return;
    FILE* fp = std::fopen(path.c_str(), "wb");
    if (!fp) { std::perror(path.c_str()); std::exit(1); }
    std::fwrite(data, 1, bytes, fp);
    std::fclose(fp);
}

// One complete evaluation of the configured hot-path call.  Inputs are
// generated outside the timed region; returns the seconds spent in the call.
struct Instance {
    Matrix<PrimeField> a, c, c0;
    std::vector<std::uint64_t> d;  // schur: D; syrkbd: blocks as (two, d, beta, gamma) quadruples
    BlockDiagonal<PrimeField> b;
    std::uint64_t alpha = 1, beta = 0;
    OpCount ops;  // the reference's own tally of the last call (opcount.hpp)
};

Instance make_instance(const PrimeField& f, const Args& g) {
    Instance in;
    in.a = random_matrix(f, g.n, g.k, g.seed);
    in.c = Matrix<PrimeField>(g.n, g.n, 0);
    if (g.mode == "acc" || g.mode == "schur") {
        in.c0 = random_matrix(f, g.n, g.n, g.cseed);
        mirror_lower_to_upper(f, in.c0.view());
        in.c = in.c0;
    }
    if (g.mode == "acc") {
        std::mt19937_64 rng(g.abseed);
        in.alpha = 1 + rng() % (g.p - 1);
        in.beta = 1 + rng() % (g.p - 1);
        if (g.alpha_set) in.alpha = g.alpha % g.p;
        if (g.beta_set) in.beta = g.beta % g.p;
    }
    if (g.mode == "schur") {
        // D: k nonzero residues 1 + rng() % (p - 1) from mt19937_64(dseed) (the convention of
        // BASELINE.md's config-5 oracle run: seeds 5001/5002/5003 give 526 non-residues)
        std::mt19937_64 rng(g.dseed);
        in.d.resize(g.k);
        for (auto& v : in.d) v = 1 + rng() % (g.p - 1);
    }
    if (g.mode == "syrkbd") {
        // B: scalar blocks d = rng() % p (zero allowed) and antidiagonal 2x2 blocks
        // beta = 1 + rng() % (p - 1), drawn until the dimension reaches k
        std::mt19937_64 rng(g.dseed);
        std::size_t dim = 0;
        while (dim < g.k) {
            const bool scalar = rng() % 3 == 0 || dim + 1 == g.k;
            if (scalar) {
                const std::uint64_t v = rng() % g.p;
                in.b.blocks.push_back(BlockDiagonal<PrimeField>::scalar(v));
                in.d.insert(in.d.end(), {0, v, 0, 0});
                dim += 1;
            } else {
                const std::uint64_t beta = 1 + rng() % (g.p - 1);
                in.b.blocks.push_back(BlockDiagonal<PrimeField>::two_by_two(beta, 0));
                in.d.insert(in.d.end(), {1, 0, beta, 0});
                dim += 2;
            }
        }
    }
    return in;
}

double run_instance(const PrimeField& f, const Args& g, Instance& in) {
    auto plan = make_syrk_plan(f, RecursionPolicy{g.threshold, g.levels}, g.mirror);
    OpCount ops;
    auto t0 = std::chrono::steady_clock::now();
    if (g.mode == "plain") {
        syrk_fast_into(f, in.a.view(), in.c.view(), plan, ops);
    } else if (g.mode == "classical") {
        syrk_classical(f, f.one(), in.a.view(), f.zero(), in.c.view(), ops);
    } else if (g.mode == "acc") {
        syrk_fast_acc(f, in.alpha, in.a.view(), in.beta, in.c.view(), plan, ops);
    } else if (g.mode == "schur") {
        // C <- C - A*D*A^T on the lower triangle (R has no fused form).
        Matrix<PrimeField> x = syrkd(f, in.a.view(), in.d, plan, ops);
        for (std::size_t i = 0; i < g.n; ++i)
            for (std::size_t j = 0; j <= i; ++j) in.c.at(i, j) = f.sub(in.c.at(i, j), x.at(i, j));
        if (g.mirror) mirror_lower_to_upper(f, in.c.view());
    } else if (g.mode == "syrkbd") {
        in.c = syrkbd(f, in.a.view(), in.b, plan, ops);
        if (g.mirror) mirror_lower_to_upper(f, in.c.view());
    } else {
        usage();
    }
    auto t1 = std::chrono::steady_clock::now();
    in.ops = ops;
    return std::chrono::duration<double>(t1 - t0).count();
}

}  // namespace

// F_{p^2} modes (QuadExtField, proj/include/fsyrk/fields.hpp:142-212): "herk" runs
// herk_fast (make_herk_plan, fast_syrk.hpp:26-29, 305-320), "syrk2" runs syrk_fast over the
// extension.  Matrices are dumped as (a, b) uint64 pairs; C is the full n x n matrix.
int main_fp2(const Args& g) {
    QuadExtField f(g.p);
    auto a = random_matrix(f, g.n, g.k, g.seed);
    OpCount ops;
    Matrix<QuadExtField> c(g.n, g.n, f.zero());
    if (g.mode == "herk") {
        auto plan = make_herk_plan(f, RecursionPolicy{g.threshold, g.levels}, g.mirror);
        herk_fast_into(f, a.view(), c.view(), plan, ops);
    } else {
        auto plan = make_syrk_plan(f, RecursionPolicy{g.threshold, g.levels}, g.mirror);
        syrk_fast_into(f, a.view(), c.view(), plan, ops);
    }
    dump(g.out_a, a.data().data(), a.data().size() * sizeof(QuadExtElement));
    dump(g.out_c, c.data().data(), c.data().size() * sizeof(QuadExtElement));
    std::printf("{\"p\": %" PRIu64 ", \"n\": %zu, \"k\": %zu, \"mode\": \"%s\", \"seed\": %" PRIu64
                ", \"non_residue\": %" PRIu64 ", \"alpha\": 1, \"beta\": 0, \"digest\": \"\""
                ", \"ops_mults\": %" PRIu64 ", \"ops_adds\": %" PRIu64 "}\n",
                g.p, g.n, g.k, g.mode.c_str(), g.seed, f.non_residue(), ops.mults, ops.adds);
    return 0;
}

int main(int argc, char** argv) {
    Args g = parse(argc, argv);
    if (g.mode == "herk" || g.mode == "syrk2") return main_fp2(g);
    PrimeField f(g.p);
    auto y = skew_orthogonal(f, 2);

    std::vector<Instance> inst;
    inst.reserve(g.threads);
    for (int t = 0; t < g.threads; ++t) inst.push_back(make_instance(f, g));

    std::vector<double> secs(g.threads, 0.0);
    auto wall0 = std::chrono::steady_clock::now();
    {
        std::vector<std::thread> pool;
        for (int t = 0; t < g.threads; ++t)
            pool.emplace_back([&, t] {
                for (int r = 0; r < g.reps; ++r) {
                    if (r > 0) inst[t] = make_instance(f, g);
                    secs[t] += run_instance(f, g, inst[t]);
                }
            });
        for (auto& th : pool) th.join();
    }
    double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    double max_s = 0, sum_s = 0;
    for (double s : secs) { max_s = std::max(max_s, s); sum_s += s; }

    Instance& r0 = inst[0];
    char hex[65] = "";
    if (g.digest) lower_digest_u64(r0.c.data().data(), g.n, g.n, hex);
    dump(g.out_a, r0.a.data().data(), r0.a.data().size() * 8);
    dump(g.out_c, r0.c.data().data(), r0.c.data().size() * 8);
    if (!r0.c0.data().empty()) dump(g.out_c0, r0.c0.data().data(), r0.c0.data().size() * 8);
    if (!r0.d.empty()) dump(g.out_d, r0.d.data(), r0.d.size() * 8);

    std::printf("{\"p\": %" PRIu64 ", \"n\": %zu, \"k\": %zu, \"mode\": \"%s\", \"seed\": %" PRIu64
                ", \"threshold\": %zu, \"levels\": %s, \"threads\": %d, \"reps\": %d"
                ", \"alpha\": %" PRIu64 ", \"beta\": %" PRIu64
                ", \"skew_form\": \"%s\", \"skew_a\": %" PRIu64 ", \"skew_b\": %" PRIu64
                ", \"seconds_per_call\": %.6f, \"wall_seconds\": %.6f, \"digest\": \"%s\""
                ", \"ops_mults\": %" PRIu64 ", \"ops_adds\": %" PRIu64,
                g.p, g.n, g.k, g.mode.c_str(), g.seed, g.threshold,
                g.levels == kUnlimitedLevels ? "\"inf\"" : std::to_string(g.levels).c_str(),
                g.threads, g.reps, r0.alpha, r0.beta,
                y.form == SkewOrthogonal<PrimeField>::Form::Pair ? "pair" : "scalar", y.a, y.b,
                sum_s / (g.threads * g.reps), wall, hex, r0.ops.mults, r0.ops.adds);
    if (g.sample > 0) {
        // deterministic sample positions in the lower triangle
        std::mt19937_64 rng(12345);
        std::printf(", \"sample\": [");
        for (int s = 0; s < g.sample; ++s) {
            std::size_t i = rng() % g.n;
            std::size_t j = rng() % (i + 1);
            std::printf("%s[%zu, %zu, %" PRIu64 "]", s ? ", " : "", i, j, r0.c.at(i, j));
        }
        std::printf("]");
    }
    std::printf("}\n");
    return 0;
}

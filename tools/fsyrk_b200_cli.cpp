// fsyrk_b200 — command-line front end of the B200 path, mirroring the reference CLI
// (proj/tools/fsyrk.cpp) for the prime field: the same subcommands, options, text formats
// (proj/include/fsyrk/text_io.hpp) and exit codes (0 ok, 1 verification failed, 2 usage /
// input error).  Every product runs on the device through the C ABI (include/fsyrk_b200.h).
//
//   fsyrk_b200 syrk   --prime P --input A.txt [--output C.txt] [--mirror] [--threshold T] [--rec R]
//                     [--scaling B.txt | --alpha a --beta b --acc C0.txt]
//   fsyrk_b200 verify --prime P [--n N] [--cols K] [--cases M] [--threshold T] [--rec R] [--seed S]
//   fsyrk_b200 bench  --prime P [--min-n N0] [--max-n N1] [--threshold T] [--rec R] [--seed S] [--output F]
//   fsyrk_b200 sos    --prime P --value V
//   fsyrk_b200 nrsyf  --prime P --alpha A --beta B
// `--field` accepts `fp` and, for `syrk` / `verify`, `fp2` (F_{p^2}: syrk_fast and herk_fast);
// gf2k / complex are outside the B200 path and `count` (the operation-count model) is not part
// of this tool.
#include <cerrno>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "fsyrk_b200.h"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitVerifyFailed = 1;
constexpr int kExitUsage = 2;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {  // text_io.hpp / fields.cpp ParseError
    using std::runtime_error::runtime_error;
};

void check(int status) {
    if (status != FSYRK_B200_OK) throw std::runtime_error(fsyrk_b200_last_error());
}

// ------------------------------------------------------------------ options
struct Options {
    std::string cmd;
    std::map<std::string, std::string> kv;
    std::map<std::string, bool> flags;

    bool has(const std::string& k) const { return kv.count(k) != 0; }
    std::string str(const std::string& k, const std::string& def = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? def : it->second;
    }
    uint64_t u64(const std::string& k, uint64_t def) const {
        if (!has(k)) return def;
        const std::string& t = kv.at(k);
        char* end = nullptr;
        errno = 0;
        unsigned long long v = std::strtoull(t.c_str(), &end, 10);
        if (errno || end == t.c_str() || *end) throw UsageError("--" + k + ": not a non-negative integer: " + t);
        return v;
    }
    bool flag(const std::string& k) const { return flags.count(k) != 0; }
};

Options parse_args(int argc, char** argv) {
    static const std::map<std::string, std::vector<std::string>> kOptions = {
        {"syrk", {"field", "prime", "input", "output", "scaling", "alpha", "beta", "acc", "threshold", "rec"}},
        {"verify", {"field", "prime", "n", "cols", "cases", "threshold", "rec", "seed"}},
        {"bench", {"field", "prime", "min-n", "max-n", "threshold", "rec", "seed", "output"}},
        {"sos", {"prime", "value"}},
        {"nrsyf", {"prime", "alpha", "beta"}},
    };
    static const std::map<std::string, std::vector<std::string>> kFlags = {{"syrk", {"mirror"}}};
    if (argc < 2) throw UsageError("a subcommand is required: syrk, verify, bench, sos, nrsyf");
    Options o;
    o.cmd = argv[1];
    if (o.cmd == "count")
        throw UsageError("count: the operation-count model is not part of the B200 path");
    auto it = kOptions.find(o.cmd);
    if (it == kOptions.end()) throw UsageError("unknown subcommand: " + o.cmd);
    for (int i = 2; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + a);
        std::string k = a.substr(2);
        const auto& fl = kFlags.count(o.cmd) ? kFlags.at(o.cmd) : std::vector<std::string>{};
        bool is_flag = false;
        for (const auto& f : fl) is_flag |= f == k;
        if (is_flag) {
            o.flags[k] = true;
            continue;
        }
        bool known = false;
        for (const auto& name : it->second) known |= name == k;
        if (!known) throw UsageError(o.cmd + ": unknown option --" + k);
        if (i + 1 >= argc) throw UsageError("--" + k + " needs a value");
        o.kv[k] = argv[++i];
    }
    if (o.has("field") && o.str("field") != "fp" && o.str("field") != "fp2")
        throw UsageError("--field " + o.str("field") + ": only fp and fp2 run on the B200 path");
    if (o.str("field") == "fp2" && o.cmd != "syrk" && o.cmd != "verify")
        throw UsageError(o.cmd + ": only --field fp is supported");
    return o;
}

// ------------------------------------------------------------------- field
struct Field {
    uint64_t p;
    explicit Field(uint64_t p_) : p(p_) {
        fsyrk_b200_skew s;  // validates p (prime, < 2^31) with the library's rules
        fsyrk_b200_policy pol{2, UINT64_MAX};
        const int st = fsyrk_b200_make_syrk_plan(p, pol, 0, &s);
        if (st != FSYRK_B200_OK) throw UsageError(fsyrk_b200_last_error());
    }
    std::string name() const { return "F_" + std::to_string(p); }
    uint64_t parse(const std::string& t) const {  // fields.cpp:20-27
        char* end = nullptr;
        errno = 0;
        unsigned long long v = std::strtoull(t.c_str(), &end, 10);
        if (errno != 0 || end == t.c_str() || *end != '\0' || v >= p)
            throw ParseError("invalid " + name() + " element: '" + t + "'");
        return v;
    }
    uint64_t mul(uint64_t a, uint64_t b) const { return (uint64_t)((unsigned __int128)a * b % p); }
    uint64_t add(uint64_t a, uint64_t b) const { return (a + b) % p; }
    uint64_t random_element(std::mt19937_64& rng) const {
        return std::uniform_int_distribution<uint64_t>(0, p - 1)(rng);
    }
};

struct Matrix {
    size_t rows = 0, cols = 0;
    std::vector<uint64_t> data;
    Matrix() = default;
    Matrix(size_t r, size_t c) : rows(r), cols(c), data(r * c, 0) {}
    uint64_t& at(size_t i, size_t j) { return data[i * cols + j]; }
    uint64_t at(size_t i, size_t j) const { return data[i * cols + j]; }
    const uint64_t* ptr() const { return data.empty() ? nullptr : data.data(); }
    uint64_t* ptr() { return data.empty() ? nullptr : data.data(); }
};

// ------------------------------------------------------------------ text io (text_io.hpp)
Matrix read_matrix(const Field& f, std::istream& is) {
    size_t rows = 0, cols = 0;
    if (!(is >> rows >> cols)) throw ParseError("matrix header must be 'rows cols'");
    Matrix m(rows, cols);
    std::string token;
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j) {
            if (!(is >> token)) throw ParseError("matrix body ended early at row " + std::to_string(i));
            m.at(i, j) = f.parse(token);
        }
    return m;
}

void write_matrix(std::ostream& os, const Matrix& m) {
    os << m.rows << ' ' << m.cols << '\n';
    for (size_t i = 0; i < m.rows; ++i) {
        for (size_t j = 0; j < m.cols; ++j) {
            if (j) os << ' ';
            os << m.at(i, j);
        }
        os << '\n';
    }
}

std::vector<fsyrk_b200_block> read_block_diagonal(const Field& f, std::istream& is) {
    std::vector<fsyrk_b200_block> b;
    std::string line;
    while (std::getline(is, line)) {
        std::istringstream ls(line);
        std::string kind;
        if (!(ls >> kind)) continue;  // blank line
        std::string t1, t2;
        if (kind == "S") {
            if (!(ls >> t1)) throw ParseError("scalar block needs one value: '" + line + "'");
            b.push_back(fsyrk_b200_block{0, f.parse(t1), 0, 0});
        } else if (kind == "T") {
            if (!(ls >> t1 >> t2)) throw ParseError("2x2 block needs beta and gamma: '" + line + "'");
            b.push_back(fsyrk_b200_block{1, 0, f.parse(t1), f.parse(t2)});
        } else {
            throw ParseError("block kind must be S or T, got '" + kind + "'");
        }
        std::string extra;
        if (ls >> extra) throw ParseError("trailing tokens in block line: '" + line + "'");
    }
    return b;
}

fsyrk_b200_policy policy_of(const Options& o) {
    const uint64_t rec = o.u64("rec", 0);
    return fsyrk_b200_policy{o.u64("threshold", 64), rec == 0 ? UINT64_MAX : rec};
}

Matrix random_matrix(const Field& f, size_t r, size_t c, uint64_t seed) {
    Matrix m(r, c);
    check(fsyrk_b200_random_matrix(f.p, r, c, seed, m.ptr(), c ? c : 1));
    return m;
}

// C = A * B^T mod p on the host (the verify batteries' oracle, matrix.hpp:317-329)
Matrix classical_nt(const Field& f, const Matrix& a, const Matrix& b) {
    Matrix c(a.rows, b.rows);
    for (size_t i = 0; i < a.rows; ++i)
        for (size_t j = 0; j < b.rows; ++j) {
            unsigned __int128 acc = 0;
            for (size_t l = 0; l < a.cols; ++l) acc += (unsigned __int128)a.at(i, l) * b.at(j, l);
            c.at(i, j) = (uint64_t)(acc % f.p);
        }
    return c;
}

bool lower_equal(const Matrix& x, const Matrix& y) {
    for (size_t i = 0; i < x.rows; ++i)
        for (size_t j = 0; j <= i; ++j)
            if (x.at(i, j) != y.at(i, j)) return false;
    return true;
}

// F_{p^2} = F_p[x] / (x^2 - ns) (QuadExtField): matrices of (a, b) pairs; the text format
// prints the integer encoding a + b p (fields.hpp:194-198).
struct Fp2 {
    Field base;
    uint64_t ns;
    explicit Fp2(uint64_t p) : base(p), ns(0) {
        if (p == 2) throw UsageError("QuadExtField requires an odd prime");
        for (uint64_t s = 2;; ++s) {  // least non-residue (Euler's criterion)
            uint64_t r = 1, b = s % p, e = (p - 1) / 2;
            while (e) {
                if (e & 1) r = base.mul(r, b);
                b = base.mul(b, b);
                e >>= 1;
            }
            if (r == p - 1) {
                ns = s;
                break;
            }
        }
    }
    uint64_t p() const { return base.p; }
    void parse_into(const std::string& t, uint64_t* ab) const {
        char* end = nullptr;
        errno = 0;
        unsigned long long v = std::strtoull(t.c_str(), &end, 10);
        if (errno != 0 || end == t.c_str() || *end != '\0' || v >= p() * p())
            throw ParseError("invalid F_" + std::to_string(p()) + "^2 element: '" + t + "'");
        ab[0] = v % p();
        ab[1] = v / p();
    }
};

struct Matrix2 {  // rows x cols of (a, b) pairs
    size_t rows = 0, cols = 0;
    std::vector<uint64_t> data;
    Matrix2() = default;
    Matrix2(size_t r, size_t c) : rows(r), cols(c), data(2 * r * c, 0) {}
    uint64_t* at(size_t i, size_t j) { return &data[2 * (i * cols + j)]; }
    const uint64_t* at(size_t i, size_t j) const { return &data[2 * (i * cols + j)]; }
};

Matrix2 read_matrix2(const Fp2& f, std::istream& is) {
    size_t rows = 0, cols = 0;
    if (!(is >> rows >> cols)) throw ParseError("matrix header must be 'rows cols'");
    Matrix2 m(rows, cols);
    std::string token;
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j) {
            if (!(is >> token)) throw ParseError("matrix body ended early at row " + std::to_string(i));
            f.parse_into(token, m.at(i, j));
        }
    return m;
}

void write_matrix2(const Fp2& f, std::ostream& os, const Matrix2& m) {
    os << m.rows << ' ' << m.cols << '\n';
    for (size_t i = 0; i < m.rows; ++i) {
        for (size_t j = 0; j < m.cols; ++j) {
            if (j) os << ' ';
            os << m.at(i, j)[0] + m.at(i, j)[1] * f.p();
        }
        os << '\n';
    }
}

// Low(A conj(A)^T) (conj) or Low(A A^T) over F_{p^2}, classical, on the host (the oracle of the
// verify batteries, fsyrk.cpp verify_herk_battery)
Matrix2 classical2(const Fp2& f, const Matrix2& a, bool conj) {
    const uint64_t p = f.p();
    Matrix2 c(a.rows, a.rows);
    for (size_t i = 0; i < a.rows; ++i)
        for (size_t j = 0; j <= i; ++j) {
            uint64_t re = 0, im = 0;
            for (size_t l = 0; l < a.cols; ++l) {
                const uint64_t* x = a.at(i, l);
                const uint64_t* y = a.at(j, l);
                const uint64_t yb = conj ? (p - y[1]) % p : y[1];
                re = (re + f.base.mul(x[0], y[0]) + f.base.mul(f.ns, f.base.mul(x[1], yb))) % p;
                im = (im + f.base.mul(x[0], yb) + f.base.mul(x[1], y[0])) % p;
            }
            c.at(i, j)[0] = re;
            c.at(i, j)[1] = im;
        }
    return c;
}

int cmd_syrk_fp2(const Options& o) {
    Fp2 f(o.u64("prime", 131071));
    if (!o.has("input")) throw UsageError("syrk: --input is required");
    if (o.has("scaling") || o.has("alpha") || o.has("beta") || o.has("acc"))
        throw UsageError("--field fp2: only the plain product runs on the B200 path");
    std::ifstream in(o.str("input"));
    if (!in) throw std::runtime_error("cannot open input file: " + o.str("input"));
    Matrix2 a = read_matrix2(f, in);
    Matrix2 c(a.rows, a.rows);
    check(fsyrk_b200_syrk_fast_into_fp2(f.p(), a.data.data(), a.rows, a.cols, a.cols ? a.cols : 1, c.data.data(),
                                        a.rows ? a.rows : 1, policy_of(o), o.flag("mirror"), nullptr));
    if (o.has("output")) {
        std::ofstream out(o.str("output"));
        if (!out) throw std::runtime_error("cannot open output file: " + o.str("output"));
        write_matrix2(f, out, c);
    } else {
        write_matrix2(f, std::cout, c);
    }
    return kExitOk;
}

int cmd_verify_fp2(const Options& o) {
    Fp2 f(o.u64("prime", 131071));
    const size_t nmax = o.u64("n", 64), kmax = o.u64("cols", 0) ? o.u64("cols", 0) : nmax;
    const int cases = (int)o.u64("cases", 100);
    const uint64_t seed = o.u64("seed", 0);
    const fsyrk_b200_policy pol = policy_of(o);
    bool all = true;
    for (int conj = 0; conj < 2; ++conj) {  // syrk_fast, then herk_fast (verify_herk_battery)
        std::mt19937_64 rng(seed + 3 * conj);
        bool ok = true;
        const int nc = conj ? std::max(1, cases / 4) : cases;
        for (int t = 0; t < nc; ++t) {
            const size_t n = 1 + rng() % (conj ? std::min<size_t>(nmax, 64) : nmax);
            const size_t k = 1 + rng() % (conj ? std::min<size_t>(nmax, 64) : kmax);
            Matrix2 a(n, k);
            std::vector<uint64_t> flat(2 * n * k);
            check(fsyrk_b200_random_matrix(f.p(), n, 2 * k, rng(), flat.data(), 2 * k));  // a, then b per element
            a.data = flat;
            Matrix2 c(n, n);
            check((conj ? fsyrk_b200_herk_fast_into : fsyrk_b200_syrk_fast_into_fp2)(
                f.p(), a.data.data(), n, k, k, c.data.data(), n, pol, 0, nullptr));
            Matrix2 ref = classical2(f, a, conj);
            for (size_t i = 0; i < n && ok; ++i)
                for (size_t j = 0; j <= i; ++j) ok &= c.at(i, j)[0] == ref.at(i, j)[0] && c.at(i, j)[1] == ref.at(i, j)[1];
        }
        std::cout << (ok ? "PASS" : "FAIL") << (conj ? " herk_fast" : " syrk_fast") << " vs classical (" << nc
                  << " cases, F_" << f.p() << "^2)\n";
        all &= ok;
    }
    std::cout << (all ? "PASS" : "FAIL") << " overall\n";
    return all ? kExitOk : kExitVerifyFailed;
}

// ------------------------------------------------------------------ commands
int cmd_syrk(const Options& o) {
    if (o.str("field") == "fp2") return cmd_syrk_fp2(o);
    Field f(o.u64("prime", 131071));
    if (!o.has("input")) throw UsageError("syrk: --input is required");
    std::ifstream in(o.str("input"));
    if (!in) throw std::runtime_error("cannot open input file: " + o.str("input"));
    Matrix a = read_matrix(f, in);
    const bool mirror = o.flag("mirror");
    const fsyrk_b200_policy pol = policy_of(o);
    Matrix c(a.rows, a.rows);
    const bool accumulate = o.has("alpha") || o.has("beta") || o.has("acc");
    if (accumulate && o.has("scaling")) throw UsageError("--alpha/--beta/--acc cannot combine with --scaling");
    const size_t lda = a.cols ? a.cols : 1, ldc = a.rows ? a.rows : 1;
    if (accumulate) {
        const uint64_t alpha = o.has("alpha") ? f.parse(o.str("alpha")) : 1;
        const uint64_t beta = o.has("beta") ? f.parse(o.str("beta")) : 0;
        if (o.has("acc")) {
            std::ifstream acc(o.str("acc"));
            if (!acc) throw std::runtime_error("cannot open --acc file: " + o.str("acc"));
            c = read_matrix(f, acc);
            if (c.rows != a.rows || c.cols != a.rows) throw std::runtime_error("syrk_fast_acc: dimension mismatch");
        }
        check(fsyrk_b200_syrk_fast_acc(f.p, alpha, a.ptr(), a.rows, a.cols, lda, beta, c.ptr(), ldc, pol, mirror,
                                       nullptr));
    } else if (o.has("scaling")) {
        std::ifstream sc(o.str("scaling"));
        if (!sc) throw std::runtime_error("cannot open scaling file: " + o.str("scaling"));
        auto blocks = read_block_diagonal(f, sc);
        check(fsyrk_b200_syrkbd(f.p, 1, a.ptr(), a.rows, a.cols, lda, blocks.data(), blocks.size(), 0, c.ptr(), ldc,
                                pol, mirror, nullptr));
    } else {
        check(fsyrk_b200_syrk_fast_into(f.p, a.ptr(), a.rows, a.cols, lda, c.ptr(), ldc, pol, mirror, nullptr));
    }
    if (!mirror)  // deterministic file: the strict upper triangle is scratch (fsyrk.cpp scrubs it too)
        for (size_t i = 0; i < c.rows; ++i)
            for (size_t j = i + 1; j < c.cols; ++j) c.at(i, j) = 0;
    if (o.has("output")) {
        std::ofstream out(o.str("output"));
        if (!out) throw std::runtime_error("cannot open output file: " + o.str("output"));
        write_matrix(out, c);
    } else {
        write_matrix(std::cout, c);
    }
    return kExitOk;
}

int cmd_verify(const Options& o) {
    if (o.str("field") == "fp2") return cmd_verify_fp2(o);
    Field f(o.u64("prime", 131071));
    const size_t nmax = o.u64("n", 64), kmax = o.u64("cols", 0) ? o.u64("cols", 0) : nmax;
    const int cases = (int)o.u64("cases", 100);
    const uint64_t seed = o.u64("seed", 0);
    const fsyrk_b200_policy pol = policy_of(o);
    bool all = true;
    {  // syrk_fast vs classical (fsyrk.cpp verify_syrk_battery)
        std::mt19937_64 rng(seed);
        bool ok = true;
        for (int t = 0; t < cases; ++t) {
            const size_t n = 1 + rng() % nmax, k = 1 + rng() % kmax;
            Matrix a = random_matrix(f, n, k, rng());
            Matrix c(n, n);
            check(fsyrk_b200_syrk_fast_into(f.p, a.ptr(), n, k, k, c.ptr(), n, pol, 0, nullptr));
            ok &= lower_equal(c, classical_nt(f, a, a));
        }
        std::cout << (ok ? "PASS" : "FAIL") << " syrk_fast vs classical (" << cases << " cases, " << f.name()
                  << ")\n";
        all &= ok;
    }
    {  // accumulating form (verify_acc_battery)
        std::mt19937_64 rng(seed + 1);
        bool ok = true;
        const int nc = std::max(1, cases / 4);
        for (int t = 0; t < nc; ++t) {
            const size_t n = 1 + rng() % std::min<size_t>(nmax, 96), k = 1 + rng() % std::min<size_t>(nmax, 96);
            const uint64_t alpha = f.random_element(rng), beta = f.random_element(rng);
            Matrix a = random_matrix(f, n, k, rng());
            Matrix c0 = random_matrix(f, n, n, rng());
            Matrix c = c0;
            check(fsyrk_b200_syrk_fast_acc(f.p, alpha, a.ptr(), n, k, k, beta, c.ptr(), n, pol, 0, nullptr));
            Matrix ref = classical_nt(f, a, a);
            for (size_t i = 0; i < n && ok; ++i)
                for (size_t j = 0; j <= i; ++j)
                    ok &= c.at(i, j) == f.add(f.mul(alpha, ref.at(i, j)), f.mul(beta, c0.at(i, j)));
        }
        std::cout << (ok ? "PASS" : "FAIL") << " syrk_fast_acc vs classical (" << nc << " cases, " << f.name()
                  << ")\n";
        all &= ok;
    }
    if (f.p != 2) {  // syrkd vs brute force (verify_scaled_battery)
        std::mt19937_64 rng(seed + 2);
        bool ok = true;
        const int nc = std::max(1, cases / 4);
        for (int t = 0; t < nc; ++t) {
            const size_t m = 1 + rng() % 32, n = 1 + rng() % 32;
            Matrix a = random_matrix(f, m, n, rng());
            std::vector<uint64_t> d(n);
            for (auto& v : d) v = f.random_element(rng);
            Matrix c(m, m);
            check(fsyrk_b200_syrkd(f.p, 1, a.ptr(), m, n, n, d.data(), 0, c.ptr(), m, pol, 0, nullptr));
            Matrix scaled = a;
            for (size_t j = 0; j < n; ++j)
                for (size_t i = 0; i < m; ++i) scaled.at(i, j) = f.mul(scaled.at(i, j), d[j]);
            ok &= lower_equal(c, classical_nt(f, scaled, a));
        }
        std::cout << (ok ? "PASS" : "FAIL") << " syrkd vs brute force (" << nc << " cases, " << f.name() << ")\n";
        all &= ok;
    }
    std::cout << (all ? "PASS" : "FAIL") << " overall\n";
    return all ? kExitOk : kExitVerifyFailed;
}

int cmd_bench(const Options& o) {
    Field f(o.u64("prime", 131071));
    const size_t n0 = o.u64("min-n", 256), n1 = o.u64("max-n", 2048);
    const uint64_t seed = o.u64("seed", 0);
    const fsyrk_b200_policy pol = policy_of(o);
    std::ofstream file;
    if (o.has("output")) {
        file.open(o.str("output"));
        if (!file) throw std::runtime_error("cannot open output file: " + o.str("output"));
    }
    std::ostream& os = o.has("output") ? file : std::cout;
    os << "algorithm,n,seconds,effective_gfops\n";
    for (size_t n = n0; n <= n1; n *= 2) {
        Matrix a = random_matrix(f, n, n, seed + n);
        Matrix c(n, n);
        check(fsyrk_b200_syrk_fast_into(f.p, a.ptr(), n, n, n, c.ptr(), n, pol, 0, nullptr));  // plan + warm-up
        auto t0 = std::chrono::steady_clock::now();
        check(fsyrk_b200_syrk_fast_into(f.p, a.ptr(), n, n, n, c.ptr(), n, pol, 0, nullptr));
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        os << "syrk_fast_b200," << n << ',' << secs << ',' << (double)n * n * n / (1e9 * secs) << '\n';
        if (n == 0) break;
    }
    return kExitOk;
}

int cmd_sos(const Options& o) {
    if (!o.has("prime") || !o.has("value")) throw UsageError("sos: --prime and --value are required");
    uint64_t a = 0, b = 0;
    check(fsyrk_b200_sum_of_squares(o.u64("prime", 0), o.u64("value", 0), &a, &b));
    std::cout << a << ' ' << b << '\n';
    return kExitOk;
}

int cmd_nrsyf(const Options& o) {
    if (!o.has("prime") || !o.has("alpha") || !o.has("beta"))
        throw UsageError("nrsyf: --prime, --alpha and --beta are required");
    uint64_t y[4];
    check(fsyrk_b200_nrsyf(o.u64("prime", 0), o.u64("alpha", 0), o.u64("beta", 0), y));
    std::cout << y[0] << ' ' << y[1] << '\n' << y[2] << ' ' << y[3] << '\n';
    return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        Options o = parse_args(argc, argv);
        if (o.cmd == "syrk") return cmd_syrk(o);
        if (o.cmd == "verify") return cmd_verify(o);
        if (o.cmd == "bench") return cmd_bench(o);
        if (o.cmd == "sos") return cmd_sos(o);
        if (o.cmd == "nrsyf") return cmd_nrsyf(o);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitUsage;
    }
    return kExitUsage;
}

// Host recursion driver and C ABI of the B200 mod-p SYRK.
//
// The recursion decisions are the reference's, node for node
// (syrk_fast_rec, include/fsyrk/fast_syrk.hpp:135-157): classical leaf when
// the level budget is spent, n or k is odd, or min(n, k) < threshold; a
// split on k when k > n; the Pair-form padding rule (fast_syrk.hpp:34-37,
// 151-155); otherwise one level of the 5-product schedule.  What changes is
// the execution: instead of walking the tree with in-place CPU kernels, the
// driver plans the whole tree once ("wide" device schedule, one buffer per
// product) and runs it as a short fixed sequence of
// batched launches:
//     convert-in -> prep (per depth) -> tensor-core products (per shape)
//     -> post-additions (per depth, bottom-up) -> finalize (alpha, beta, mirror)
// Plans (device arena, TMA descriptors, node tables) are cached per
// (p, n, k, policy) so repeated calls only launch kernels.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <exception>
#include <array>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <tuple>
#include <type_traits>
#include <queue>
#include <vector>

#include "../../include/fsyrk_b200.h"
#include "elementwise.cuh"
#include "field_host.h"
#include "ref_opcount.h"
#include "host_io.h"
#include "modp.cuh"
#include "per_device.h"
#include "tc_modmm.h"

namespace fsyrk_b200 {

namespace {

thread_local std::string g_last_error;
thread_local int g_launch_counts[5] = {0, 0, 0, 0, 0};
thread_local std::string g_last_plan_json;
thread_local bool g_phase_timing = false;
// FSYRK_B200_ALWAYS_WAIT=1: every call waits on the plan's previous call even on the same stream (A/B switch)
const bool g_always_wait = getenv("FSYRK_B200_ALWAYS_WAIT") != nullptr;
thread_local float g_phase_ms[5] = {0, 0, 0, 0, 0};
thread_local uint64_t g_transfer[2] = {0, 0};  // host<->device bytes of the last host-API call
constexpr size_t kTriRows = 256;                // row block of the triangular C transfers

struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        int code = e == cudaErrorMemoryAllocation ? FSYRK_B200_ENOMEM : FSYRK_B200_ECUDA;
        fail(code, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

// rethrow the status of a nested entry point (its message is in g_last_error)
void check_status(int st) {
    if (st != FSYRK_B200_OK) fail(st, g_last_error);
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return FSYRK_B200_OK;
    } catch (const Error& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return FSYRK_B200_EINVAL;
    }
}

// ------------------------------------------------------------------ device
struct DeviceProbe {
    std::once_flag flag;
    int ok = 0;
};
int device_ok() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return 0;
    }
    DeviceProbe& pr = per_device<DeviceProbe>();  // cached per device (a process may use several)
    std::call_once(pr.flag, [&] {
        cudaDeviceProp prop{};
        if (cudaGetDeviceProperties(&prop, current_device()) != cudaSuccess) {
            cudaGetLastError();
            return;
        }
        pr.ok = prop.major == 10 ? 1 : 0;
    });
    return pr.ok;
}

void require_device() {
    if (!device_ok())
        fail(FSYRK_B200_ENODEV, "no sm_100 (B200) device available: the fsyrk_b200 path has no CPU fallback");
}

// ------------------------------------------------------------- TMA encode
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q),
           "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
        if (!ptr || q != cudaDriverEntryPointSuccess) fail(FSYRK_B200_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeFn>(ptr);
    }
    return fn;
}

// 4-D int8 plane tensor [batch][L][rows][kpad], boxes of 128 (K) x box_rows.
CUtensorMap make_plane_map(void* base, int kpad, int rows, int L, int batch, int box_rows, int bk) {
    CUtensorMap m;
    cuuint64_t dims[4] = {(cuuint64_t)kpad, (cuuint64_t)rows, (cuuint64_t)L, (cuuint64_t)batch};
    cuuint64_t strides[3] = {(cuuint64_t)kpad, (cuuint64_t)kpad * rows, (cuuint64_t)kpad * rows * L};
    cuuint32_t box[4] = {(cuuint32_t)bk, (cuuint32_t)box_rows, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, base, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE,
                             bk == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                             : bk == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                        : CU_TENSOR_MAP_SWIZZLE_32B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(FSYRK_B200_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

long long round_up(long long x, long long m) { return (x + m - 1) / m * m; }


uint64_t pow_mod(uint64_t b, uint64_t e, uint64_t p) {
    host::Field f{p};
    return f.pow(b, e);
}


// ------------------------------------------------------ multi-GPU partition
// Top-level tile-pair ownership: the h x h quadrants of the top
// level are cut into blocks of kPartBlock rows/columns (a multiple of the
// product tile 128 x BN of the plan's scheme and of the 32-row post tile); the owner
// of the unordered block pair {I >= J} computes P1, P2, P5 on (I, J), P3 and
// P4 on (I, J) and (J, I), and the post-additions of C11(I, J), C22(I, J),
// C21(I, J), C21(J, I) -- all local.  Pairs are assigned longest-first to the
// least-loaded rank (cost ~ rows_I * rows_J, halved on the diagonal).
int part_block_for(int bm, int bn) {
    int b = bm;
    while (b % bn) b += bm;  // lcm(tile rows, BN), e.g. 640 (128 x 160) or 1280 (256 x 160)
    return b;
}

std::vector<int> partition_owners(int h, int nranks, int kPartBlock) {
    const int nb = (h + kPartBlock - 1) / kPartBlock;
    std::vector<int> owner((size_t)nb * nb, -1);
    struct PairCost {
        double cost;
        int i, j;
    };
    std::vector<PairCost> pc;
    auto rows = [&](int b) { return (double)std::min(kPartBlock, h - b * kPartBlock); };
    for (int i = 0; i < nb; ++i)
        for (int j = 0; j <= i; ++j) pc.push_back({rows(i) * rows(j) * (i == j ? 0.5 : 1.0), i, j});
    std::stable_sort(pc.begin(), pc.end(), [](const PairCost& a, const PairCost& b) { return a.cost > b.cost; });
    // Each rank also prepares the operand rows of every block its pairs touch (the pre-additions
    // of the top level), so a block new to a rank costs about one block pair of products
    // (kBlockCost); pairs go, longest first, to the rank where they add the least total work.
    constexpr double kBlockCost = 1.0;
    std::vector<double> load(nranks, 0.0);
    std::vector<std::vector<char>> need(nranks, std::vector<char>(nb, 0));
    for (const auto& q : pc) {
        int best = 0;
        double best_score = 0;
        for (int t = 0; t < nranks; ++t) {
            double extra = q.cost;
            if (!need[t][q.i]) extra += kBlockCost * rows(q.i) * kPartBlock;
            if (q.j != q.i && !need[t][q.j]) extra += kBlockCost * rows(q.j) * kPartBlock;
            const double score = load[t] + extra;
            if (t == 0 || score < best_score) {
                best = t;
                best_score = score;
            }
        }
        load[best] = best_score;
        need[best][q.i] = need[best][q.j] = 1;
        owner[(size_t)q.i * nb + q.j] = best;
    }
    return owner;
}

// ------------------------------------------------------------------- plan
enum Kind { LEAF = 0, LEVEL = 1, SPLITK = 2 };

// One problem C = A B^T of the Strassen-Winograd engine (uint32 residue operands).
struct WinoProblem {
    const uint32_t* a;
    long long lda;
    const uint32_t* b;
    long long ldb;
    uint32_t* c;
    long long ldc;
};
void wino_gemm_multi(uint64_t p, const std::vector<WinoProblem>& probs, size_t m, size_t n, size_t k,
                     fsyrk_b200_policy pol, cudaStream_t s);

// Smallest general product (min(h, kw)) of the top level that runs Strassen-Winograd levels
// (fsyrk_b200_set_winograd_min; 0 = never).  Default 16384: the measured crossover on B200
// (profiles/r01/winograd_ablation.txt); FSYRK_B200_WINOGRAD_MIN overrides it at load time.
std::atomic<uint64_t> g_wino_min{[] {
    const char* e = getenv("FSYRK_B200_WINOGRAD_MIN");
    return e ? (uint64_t)atoll(e) : (uint64_t)16384;
}()};

struct Node {
    int kind = LEAF;
    int n = 0, k = 0, depth = 0;
    int h = 0, kh = 0, kw = 0;
    bool padded = false;
    int ch[3] = {-1, -1, -1};
    int parent = -1, role = -1;
    // input: an internal residue buffer (in, ldin) or, when in64, the window at
    // (r0, c0) of the caller's uint64 matrix (top of the tree, no syrkd)
    const uint32_t* in = nullptr;
    long long ldin = 0;
    bool in64 = false;
    int r0 = 0, c0 = 0;
    bool leaf_from_prep = false;
    int lgroup = -1, lslot = -1;
    int ggroup = -1, gslot = -1;
    uint32_t* x = nullptr;  // n x n output (lower)
    long long ldx = 0;
    uint32_t* s3res = nullptr;
    long long lds3 = 0;
};

struct LeafGroup {
    int n, k, count = 0;
    int rpad, kpad;
    long long plane, slot;
    int8_t* planes = nullptr;
    uint32_t* xout = nullptr;
    CUtensorMap tA, tB;
    int ntiles = 0;  // lower tiles per SYRK
    size_t off_planes = 0, off_x = 0;
};

struct GemmGroup {
    int h, kw, count = 0;
    bool root = false;  // the two general products of the top level (launched early, see execute)
    int hpad, kpad;
    long long plane, slot, slot_b;  // slot_b: B-role operands keep only the scheme's first pb planes
    int8_t *ga = nullptr, *gb = nullptr;
    uint32_t* out = nullptr;
    CUtensorMap tA, tB;
    size_t off_ga = 0, off_gb = 0, off_out = 0;
    // Strassen-Winograd general products (the reference's gemm_winograd_nt_into inside the
    // level, winograd.hpp:118-169): operands as uint32 residues S1 | S2 | A22 | S4 (h x kw each)
    // and the Winograd engine instead of the grouped product launch; wino = levels it may use
    int wino = 0;
    fsyrk_b200_policy wino_pol{0, 0};
    uint32_t* res = nullptr;
    size_t off_res = 0;
};

// One persistent grouped launch of the product kernel.
struct ProdLaunch {
    struct Member {
        bool leaf;
        int idx;
    };
    std::vector<Member> members;
    std::vector<int4> host_tiles;
    size_t off_tiles = 0;
    int phase = 1;  // 0: top-level general products (start right after the top pre-additions)
    GroupedArgs args;
};

struct PrepGroup {
    int depth, n, k;
    bool in64 = false;
    std::vector<int> nodes;
    PrepArgs args;
    PrepNode* dev_nodes = nullptr;
    size_t off_nodes = 0;
};

struct PostGroup {
    int depth, n, kind;
    std::vector<int> nodes;
    PostNode* dev_post = nullptr;
    std::vector<PostNode> host_post;  // the same table on the host (small ones travel in the launch parameters)
    AddNode* dev_add = nullptr;
    size_t off_nodes = 0;
};

constexpr size_t kTileOffBytes = 4096;  // per-unit tile ranges behind a launch's tile list (<= 1023 units)

struct Arena {
    size_t size = 0;
    size_t take(size_t bytes, size_t align = 256) {
        size_t o = (size_t)round_up((long long)size, (long long)align);
        size = o + bytes;
        return o;
    }
};

struct Plan {
    uint64_t p;
    int n, kin, k;  // k: columns after the (optional) syrkd transform
    fsyrk_b200_policy policy;
    bool colmap = false;
    SchemeInfo sch;  // digit scheme of the tensor-core products (schemes.cuh)
    int L, BN, BK;   // L: digit planes stored per leaf operand
    int BMt = 128;   // output rows per product tile (256 on CTA pairs)
    int ncta = 148;  // CTAs of a persistent product launch
    host::Skew y;
    ModP m;
    uint32_t c32 = 0;
    std::vector<Node> nodes;
    std::vector<LeafGroup> leaves;
    std::vector<GemmGroup> gemms;
    std::vector<PrepGroup> preps;
    std::vector<PostGroup> posts;
    std::vector<int> split_leaves;  // LEAF nodes converted from a residue view
    std::vector<ProdLaunch> prods;
    int nsm = 148;
    // multi-GPU partition of the top level (rank prank of pnranks); see partition_owners
    int prank = 0, pnranks = 1;
    bool partitioned = false;  // top level split across ranks
    bool idle = false;         // this rank has no share (shape not partitionable, rank > 0)
    int part_nb = 0, kPartBlock = 384;
    std::vector<int> owner;
    std::vector<int2> root_pairs;  // owned 32 x 32 post tile pairs of the root
    int2* dev_pairs = nullptr;
    size_t off_pairs = 0;
    bool owns_block_pair(int bi, int bj) const {
        if (!partitioned) return true;
        if (bi < bj) std::swap(bi, bj);
        return owner[(size_t)bi * part_nb + bj] == prank;
    }
    uint8_t* arena = nullptr;
    size_t arena_bytes = 0;
    uint32_t* root_in = nullptr;
    size_t off_root_in = 0;
    ColMap* dev_colmap = nullptr;
    std::vector<ColMap> colmap_uploaded;  // what dev_colmap holds (repeated calls skip the upload)
    size_t off_colmap = 0;
    uint64_t tensor_macs = 0;  // modular MACs issued on the tensor cores
    uint64_t int8_macs = 0;
    uint64_t ew_adds = 0;
    uint64_t prep_bytes = 0, post_bytes = 0, post_cin_bytes = 0, convert_bytes = 0;  // algorithmic HBM bytes

    // low-memory schedule (fsyrk_b200_set_workspace_limit): the top level's two general products
    // P4, P3 are written into the caller's C12 quadrant -- strict upper triangle, scratch in the
    // reference too (fast_syrk.hpp:271-273), which also keeps its S blocks there (:96-98) --
    // instead of the arena; the root post-addition reads them from there
    // a root-leaf plan (depth 0: one classical product over the whole problem) has the product
    // epilogue write alpha X + beta C into the caller's C (no uint32 X, no finalize pass)
    bool root_direct = false;
    bool lowmem = false;
    const uint64_t* lm_c = nullptr;  // C the root group's output map was last encoded for
    long long lm_ldc = 0;
    // fused subtree pre-additions (prep_tree_kernel): depth of the complete uniform tree read in
    // one launch from the caller's A (0: per-depth launches)
    int tree_depth = 0;
    PrepTreeArgs tree_args{};
    PrepNode* tree_dev = nullptr;  // depth-ordered PrepNode tables in tree order

    // the two deepest post-addition levels fused (post2_kernel): parent depth (-1: off), the
    // parents' and the deepest nodes' PostNode tables in tree order
    int post2_parent_depth = -1;
    int post2_h2 = 0, post2_nparents = 0;
    PostNode* post2_dev = nullptr;
    std::vector<PostNode> post2_host;  // parents, then the deepest nodes (as uploaded to post2_dev)

    // side stream + events: the top level's general products overlap the deeper pre/post-additions
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // Root post-addition overlapped with the products (one-level plans, FSYRK_B200_POST_ROUNDS=R,
    // off by default -- measured slower, profiles/r01/variants.txt): the product tiles run in R
    // rounds of output rows (a round holds every tile whose first needed post pair lies in its
    // rows) on FSYRK_B200_ROUND_CTAS SMs, and the root post runs as the product kernel's
    // programmatic dependent on the other SMs, each pair once its round's tiles are stored.
    int nrounds = 0;                 // 0: off
    std::vector<int> round_target;   // epilogue-warp reports of each round (its tiles x epilogue warps)
    size_t off_rounds = 0;           // device: [round_done[nrounds] | next_pair | target[nrounds]]
    int* dev_rounds = nullptr;
    int round_ctas = 0;  // product CTAs (the remaining SMs run the post)

    // Calls that share this plan share its arena: each call's stream first waits for the
    // previous call's last kernel (ev_done), whatever stream that call used.
    std::mutex use_mu;
    cudaEvent_t ev_done = nullptr;
    unsigned long long last_sid = 0;  // id of the stream the previous call ran on
    bool last_sid_valid = false;

    ~Plan() {
        if (ev_done) cudaEventDestroy(ev_done);
        if (arena) cudaFree(arena);
        if (side) cudaStreamDestroy(side);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (tree_dev) cudaFree(tree_dev);
        if (post2_dev) cudaFree(post2_dev);
    }

    int build(int n_, int k_, uint64_t levels, int depth, int parent, int role) {
        Node nd;
        nd.n = n_;
        nd.k = k_;
        nd.depth = depth;
        nd.parent = parent;
        nd.role = role;
        const int idx = (int)nodes.size();
        nodes.push_back(nd);
        const uint64_t thr = policy.threshold;
        const int mn = std::min(n_, k_);
        if (levels == 0 || n_ % 2 != 0 || k_ % 2 != 0 || (uint64_t)mn < thr) {
            nodes[idx].kind = LEAF;
            return idx;
        }
        if (k_ > n_) {  // split on k (fast_syrk.hpp:143-150)
            const int k1 = (k_ / 2) & ~1;
            nodes[idx].kind = SPLITK;
            int c0 = build(n_, k1, levels, depth + 1, idx, 0);
            int c1 = build(n_, k_ - k1, levels, depth + 1, idx, 1);
            nodes[idx].ch[0] = c0;
            nodes[idx].ch[1] = c1;
            return idx;
        }
        const bool padded = y.form == 1 && (k_ / 2) % 2 == 1;
        if (padded && k_ / 2 + 1 > n_ / 2) {
            nodes[idx].kind = LEAF;
            return idx;
        }
        nodes[idx].kind = LEVEL;
        nodes[idx].h = n_ / 2;
        nodes[idx].kh = k_ / 2;
        nodes[idx].kw = k_ / 2 + (padded ? 1 : 0);
        nodes[idx].padded = padded;
        const uint64_t next = levels == UINT64_MAX ? UINT64_MAX : levels - 1;
        const int h = n_ / 2, kh = k_ / 2, kw = nodes[idx].kw;
        int c0 = build(h, kh, next, depth + 1, idx, 0);  // P1 = A11 A11^T
        int c1 = build(h, kh, next, depth + 1, idx, 1);  // P2 = A12 A12^T
        int c2 = build(h, kw, next, depth + 1, idx, 2);  // P5 = S3 S3^T
        nodes[idx].ch[0] = c0;
        nodes[idx].ch[1] = c1;
        nodes[idx].ch[2] = c2;
        return idx;
    }

    int leaf_group(int n_, int k_) {
        for (size_t g = 0; g < leaves.size(); ++g)
            if (leaves[g].n == n_ && leaves[g].k == k_) return (int)g;
        LeafGroup lg;
        lg.n = n_;
        lg.k = k_;
        leaves.push_back(lg);
        return (int)leaves.size() - 1;
    }
    int gemm_group(int h, int kw, bool root) {
        for (size_t g = 0; g < gemms.size(); ++g)
            if (gemms[g].h == h && gemms[g].kw == kw && gemms[g].root == root) return (int)g;
        GemmGroup gg;
        gg.h = h;
        gg.kw = kw;
        gg.root = root;
        gemms.push_back(gg);
        return (int)gemms.size() - 1;
    }

    // dry: lay out the plan and its arena (arena_bytes) without touching the device
    void create(uint64_t p_, int n_, int kin_, int k_, fsyrk_b200_policy pol, bool colmap_, int rank_ = 0,
                int nranks_ = 1, bool dry = false, bool lowmem_ = false) {
        p = p_;
        n = n_;
        kin = kin_;
        k = k_;
        policy = pol;
        colmap = colmap_;
        prank = rank_;
        pnranks = nranks_;
        sch = scheme_for(p, nranks_);
        L = sch.planes;
        BN = sch.bn;
        BK = sch.bk;
        BMt = sch.bm;
        host::Field f{p};
        y = host::skew_orthogonal(f);
        m = make_modp((uint32_t)p);
        c32 = (uint32_t)pow_mod(2, 32, p);

        // the multi-GPU partition splits one top level whose three SYRK products are leaves
        build(n, k, pnranks > 1 ? std::min<uint64_t>(pol.max_levels, 1) : pol.max_levels, 0, -1, -1);
        if (pnranks > 1) {
            const Node& r = nodes[0];
            partitioned = r.kind == LEVEL && nodes[r.ch[0]].kind == LEAF && nodes[r.ch[1]].kind == LEAF &&
                          nodes[r.ch[2]].kind == LEAF;
            if (partitioned) {
                kPartBlock = part_block_for(sch.bm, BN);
                part_nb = (r.h + kPartBlock - 1) / kPartBlock;
                owner = partition_owners(r.h, pnranks, kPartBlock);
            } else {
                idle = prank != 0;  // not partitionable: rank 0 computes everything
            }
        }
        // measured (profiles/r02/depth0.txt): pays from ~2048^2 outputs (cfg2 / cfg3 / cfg5 shapes at
        // depth 0); below, the separate finalize pass is cheaper than the heavier epilogue
        root_direct = pnranks == 1 && nodes[0].kind == LEAF && (long long)n_ * n_ >= (2048ll << 11) &&
                      getenv("FSYRK_B200_NO_ROOT_DIRECT") == nullptr;
        // the low-memory schedule applies to a single-rank plan whose top level is a 2 x 2 level
        lowmem = lowmem_ && pnranks == 1 && nodes[0].kind == LEVEL && nodes[0].h % 4 == 0;
        // any K is exact: the product kernel drains its int32 accumulators mod p every
        // modmm_k_limit(sch, p) of K (chunk_blocks), like the reference's __int128 dot
        // products accept any k (matrix.hpp:144-160)
        // ---- input sources: views of the caller's matrix stay uint64 windows (no conversion
        // pass); only S3 (and, for syrkd, the transformed root) live in residue buffers.
        // Nodes are in DFS order, so parents are visited before their children.
        nodes[0].in64 = !colmap;
        for (auto& nd : nodes) {
            if (nd.kind == LEVEL) {
                Node &q0 = nodes[nd.ch[0]], &q1 = nodes[nd.ch[1]], &q2 = nodes[nd.ch[2]];
                q0.in64 = q1.in64 = nd.in64;
                q0.r0 = q1.r0 = nd.r0;
                q0.c0 = nd.c0;
                q1.c0 = nd.c0 + nd.kh;
                q2.in64 = false;
            } else if (nd.kind == SPLITK) {
                Node &q0 = nodes[nd.ch[0]], &q1 = nodes[nd.ch[1]];
                q0.in64 = q1.in64 = nd.in64;
                q0.r0 = q1.r0 = nd.r0;
                q0.c0 = nd.c0;
                q1.c0 = nd.c0 + q0.k;
            }
        }

        // ---- grouping
        for (int i = 0; i < (int)nodes.size(); ++i) {
            Node& nd = nodes[i];
            if (nd.kind == LEAF) {
                nd.lgroup = leaf_group(nd.n, nd.k);
                nd.lslot = leaves[nd.lgroup].count++;
                nd.leaf_from_prep = nd.parent >= 0 && nodes[nd.parent].kind == LEVEL;
                if (!nd.leaf_from_prep) split_leaves.push_back(i);
            } else if (nd.kind == LEVEL) {
                nd.ggroup = gemm_group(nd.h, nd.kw, nd.parent < 0);
                nd.gslot = gemms[nd.ggroup].count++;
            }
        }

        // ---- arena layout
        Arena ar;
        const int kin_pad = (int)round_up(k, 4);
        if (colmap) {
            off_root_in = ar.take((size_t)n * kin_pad * 4);
            off_colmap = ar.take((size_t)k * sizeof(ColMap));
        }
        for (auto& lg : leaves) {
            lg.rpad = (int)round_up(lg.n, 128);
            lg.kpad = (int)round_up(std::max(lg.k, 1), 128);
            lg.plane = (long long)lg.rpad * lg.kpad;
            lg.slot = lg.plane * L;
            lg.off_planes = ar.take((size_t)lg.slot * lg.count, 1024);
            lg.off_x = ar.take((size_t)lg.count * lg.n * lg.n * 4);
            lg.ntiles = 0;
            for (int tm = 0; tm * BMt < lg.n; ++tm)
                for (int tn = 0; tn * BN < lg.n && tn * BN <= tm * BMt + BMt - 1; ++tn) ++lg.ntiles;
        }
        // Winograd levels for the top level's general products where they pay: min(h, kw) of at
        // least FSYRK_B200_WINOGRAD_MIN (default 16384, the measured crossover,
        // profiles/r01/winograd_ablation.txt; 0 = wherever the reference's policy recurses)
        {
            const uint64_t wmin = g_wino_min.load();
            const uint64_t next = pol.max_levels == UINT64_MAX ? UINT64_MAX : pol.max_levels - 1;
            for (auto& gg : gemms) {
                if (!gg.root || pnranks > 1 || next == 0 || wmin == 0) continue;
                // base products of at least 128 (one tensor tile) below the last level
                const uint64_t thr = std::max<uint64_t>({pol.threshold, wmin, 256});
                if (gg.h % 2 == 0 && gg.kw % 2 == 0 && (uint64_t)std::min(gg.h, gg.kw) >= thr) {
                    gg.wino = 1;
                    gg.wino_pol = fsyrk_b200_policy{thr, next};
                }
            }
        }
        for (auto& gg : gemms) {
            if (gg.wino) {  // residue operands only; the engine keeps its own scratch
                gg.hpad = gg.h;
                gg.kpad = gg.kw;
                gg.plane = gg.slot = gg.slot_b = 0;
                gg.off_res = ar.take((size_t)4 * gg.count * gg.h * gg.kw * 4);
                if (!(lowmem && gg.root)) gg.off_out = ar.take((size_t)2 * gg.count * gg.h * gg.h * 4);
                continue;
            }
            gg.hpad = (int)round_up(gg.h, 128);
            gg.kpad = (int)round_up(gg.kw, 128);
            gg.plane = (long long)gg.hpad * gg.kpad;
            gg.slot = gg.plane * sch.pa;  // A-role operands (S1, A22)
            gg.off_ga = ar.take((size_t)gg.slot * 2 * gg.count, 1024);
            gg.slot_b = gg.plane * sch.pb;
            gg.off_gb = ar.take((size_t)gg.slot_b * 2 * gg.count, 1024);
            if (!(lowmem && gg.root)) gg.off_out = ar.take((size_t)2 * gg.count * gg.h * gg.h * 4);
        }
        // product launches: every GEMM group and leaf group, kMaxGroups per persistent launch,
        // tiles (group, batch, tm, tn) ordered longest-K first
        {
            struct PG { bool leaf; int idx; int kpad; int phase; };
            std::vector<PG> pgs;
            // FSYRK_B200_OVERLAP=1: launch the top level's products on their own, overlapped with
            // the deeper pre/post-additions (measured slower on cfg2: the elementwise kernels get
            // only the SM resources the persistent kernel leaves); default: one launch
            const bool split_root = getenv("FSYRK_B200_OVERLAP") != nullptr && !lowmem_;
            for (int i = 0; i < (int)gemms.size(); ++i)
                if (!gemms[i].wino) pgs.push_back({false, i, gemms[i].kpad, gemms[i].root && split_root ? 0 : 1});
            for (int i = 0; i < (int)leaves.size(); ++i) pgs.push_back({true, i, leaves[i].kpad, 1});
            std::stable_sort(pgs.begin(), pgs.end(), [](const PG& a, const PG& b) {
                return a.phase != b.phase ? a.phase < b.phase : a.kpad > b.kpad;
            });
            for (size_t c0 = 0; c0 < pgs.size();) {
                ProdLaunch pl;
                pl.phase = pgs[c0].phase;
                size_t c = c0;
                // Tiles of one product in groups of kGroupRows tile rows, column by column inside a
                // group: the ~ncta tiles in flight then share kGroupRows A row panels and ~ncta /
                // kGroupRows B column panels in L2, instead of every B panel being streamed again
                // for each tile row (cfg4's 8192^2 products: 11x re-reads from DRAM in row order).
                static const int kGroupRows = [] {
                    const char* e = getenv("FSYRK_B200_GROUP_ROWS");
                    return e ? atoi(e) : 12;
                }();
                auto push_tiles = [&](int gi, int b, int nrow, int ncol, bool lower) {
                    const int ntm = (nrow + BMt - 1) / BMt, ntn = (ncol + BN - 1) / BN;
                    const int gm = kGroupRows > 0 ? kGroupRows : ntm;
                    for (int tm0 = 0; tm0 < ntm; tm0 += gm)
                        for (int tn = 0; tn < ntn; ++tn)
                            for (int tm = tm0; tm < std::min(ntm, tm0 + gm); ++tm)
                                if ((!lower || tn * BN <= tm * BMt + BMt - 1) && !idle &&
                                    owns_block_pair(tm * BMt / kPartBlock, tn * BN / kPartBlock))
                                    pl.host_tiles.push_back(make_int4(gi, b, tm, tn));
                };
                for (; c < pgs.size() && c < c0 + kMaxGroups && pgs[c].phase == pl.phase; ++c) {
                    const int gi = (int)(c - c0);
                    pl.members.push_back({pgs[c].leaf, pgs[c].idx});
                    if (!pgs[c].leaf) {
                        const GemmGroup& gg = gemms[pgs[c].idx];
                        for (int b = 0; b < 2 * gg.count; ++b) push_tiles(gi, b, gg.h, gg.h, false);
                    } else {
                        const LeafGroup& lg = leaves[pgs[c].idx];
                        for (int b = 0; b < lg.count; ++b) push_tiles(gi, b, lg.n, lg.n, true);
                    }
                }
                pl.off_tiles = ar.take(pl.host_tiles.size() * sizeof(int4) + kTileOffBytes);  // + per-unit ranges
                prods.push_back(std::move(pl));
                c0 = c;
            }
        }
        // post-overlap rounds (one-level plans: the root's P1, P2, P5 are leaf products)
        {
            static const int want = [] {
                const char* e = getenv("FSYRK_B200_POST_ROUNDS");
                return e ? atoi(e) : 0;  // measured slower (profiles/r01/variants.txt): off
            }();
            const Node& r0 = nodes[0];
            const bool any_wino = std::any_of(gemms.begin(), gemms.end(), [](const GemmGroup& g) { return g.wino; });
            if (want > 1 && !partitioned && !idle && !lowmem && !any_wino && r0.kind == LEVEL && nodes[r0.ch[0]].kind == LEAF &&
                nodes[r0.ch[1]].kind == LEAF && nodes[r0.ch[2]].kind == LEAF && prods.size() == 1 &&
                r0.h >= 2048) {
                const ProdLaunch& pl = prods[0];
                const int T = (r0.h + 31) / 32;
                // a tile covering 32-row blocks [a, ..) and 32-column blocks [c, ..) is first needed
                // by the post pairs (I, J), I >= J, with I = max(a, c)
                auto first_u = [&](const int4& t) { return std::max(t.z * BMt, t.w * BN) / 32; };
                std::vector<long long> cnt(T + 1, 0);
                for (const int4& t : pl.host_tiles) cnt[first_u(t)]++;
                const int R = std::min(want, T);
                std::vector<int> bound(1, 0);  // round r covers 32-row blocks [bound[r], bound[r + 1])
                long long acc = 0, tot = (long long)pl.host_tiles.size();
                for (int u = 0; u < T; ++u) {
                    acc += cnt[u];
                    if ((int)bound.size() < R && acc * R >= tot * (long long)bound.size() && u + 1 < T)
                        bound.push_back(u + 1);
                }
                bound.push_back(T);
                std::vector<int> round_of(T + 1, 0);
                for (size_t r = 0; r + 1 < bound.size(); ++r)
                    for (int u = bound[r]; u < bound[r + 1]; ++u) round_of[u] = (int)r;
                const int nr = (int)bound.size() - 1;
                // one launch, tiles in round order, the round in the tile's group field
                ProdLaunch& pm = prods[0];
                std::vector<int4> sorted;
                round_target.assign(nr, 0);
                for (int r = 0; r < nr; ++r)
                    for (const int4& t : pm.host_tiles)
                        if (round_of[first_u(t)] == r) {
                            sorted.push_back(make_int4(t.x | (r << kTileGroupBits), t.y, t.z, t.w));
                            round_target[r] += modmm_epilogue_warps();
                        }
                pm.host_tiles = std::move(sorted);
                for (int r = 0; r < nr; ++r)
                    for (int I = bound[r]; I < bound[r + 1]; ++I)
                        for (int J = 0; J <= I; ++J) root_pairs.push_back(make_int2(I | (r << 20), J));
                nrounds = nr;
                off_rounds = ar.take((2 * (size_t)nr + 1) * sizeof(int));
                off_pairs = ar.take(root_pairs.size() * sizeof(int2));
            }
        }
        std::vector<size_t> off_x(nodes.size(), 0), off_s3(nodes.size(), 0);
        for (size_t i = 0; i < nodes.size(); ++i) {
            Node& nd = nodes[i];
            // node outputs X; a LEVEL root's post-addition writes the caller's C directly (no X)
            if (nd.kind != LEAF && !(i == 0 && nd.kind == LEVEL)) off_x[i] = ar.take((size_t)nd.n * nd.n * 4);
            if (nd.kind == LEVEL && nodes[nd.ch[2]].kind != LEAF) off_s3[i] = ar.take((size_t)nd.h * nd.kw * 4);
        }
        // prep / post groups
        for (size_t i = 0; i < nodes.size(); ++i) {
            Node& nd = nodes[i];
            if (nd.kind != LEVEL) continue;
            bool found = false;
            for (auto& pg : preps)
                if (pg.depth == nd.depth && pg.n == nd.n && pg.k == nd.k) {
                    pg.nodes.push_back((int)i);
                    found = true;
                }
            if (!found) {
                PrepGroup pg;
                pg.depth = nd.depth;
                pg.n = nd.n;
                pg.k = nd.k;
                pg.in64 = nd.in64;
                pg.nodes.push_back((int)i);
                preps.push_back(pg);
            }
        }
        for (size_t i = 0; i < nodes.size(); ++i) {
            Node& nd = nodes[i];
            if (nd.kind == LEAF) continue;
            bool found = false;
            for (auto& pg : posts)
                if (pg.depth == nd.depth && pg.n == nd.n && pg.kind == nd.kind) {
                    pg.nodes.push_back((int)i);
                    found = true;
                }
            if (!found) {
                PostGroup pg;
                pg.depth = nd.depth;
                pg.n = nd.n;
                pg.kind = nd.kind;
                pg.nodes.push_back((int)i);
                posts.push_back(pg);
            }
        }
        std::sort(preps.begin(), preps.end(), [](const PrepGroup& a, const PrepGroup& b) { return a.depth < b.depth; });
        std::sort(posts.begin(), posts.end(), [](const PostGroup& a, const PostGroup& b) { return a.depth > b.depth; });
        for (auto& pg : preps) pg.off_nodes = ar.take(pg.nodes.size() * sizeof(PrepNode));
        for (auto& pg : posts)
            pg.off_nodes = ar.take(pg.nodes.size() * (pg.kind == LEVEL ? sizeof(PostNode) : sizeof(AddNode)));
        if (partitioned) {  // owned 32 x 32 tile pairs of the root post-addition
            const int h = nodes[0].h, T = (h + 31) / 32;
            for (int I = 0; I < T; ++I)
                for (int J = 0; J <= I; ++J)
                    if (owns_block_pair(I * 32 / kPartBlock, J * 32 / kPartBlock)) root_pairs.push_back(make_int2(I, J));
            off_pairs = ar.take(std::max<size_t>(root_pairs.size(), 1) * sizeof(int2));
        }

        // ---- allocate and clear (the zero padding of every operand plane is never rewritten)
        arena_bytes = ar.size;
        if (dry) return;
        if (cudaMalloc(&arena, arena_bytes) != cudaSuccess) {
            cudaGetLastError();
            arena = nullptr;
            fail(FSYRK_B200_ECUDA, "cudaMalloc(plan arena of " + std::to_string(arena_bytes) +
                                       " bytes) failed: out of device memory (fsyrk_b200_workspace_bytes reports it)");
        }
        ck(cudaMemset(arena, 0, arena_bytes), "cudaMemset(plan arena)");
        if (colmap) {
            root_in = reinterpret_cast<uint32_t*>(arena + off_root_in);
            dev_colmap = reinterpret_cast<ColMap*>(arena + off_colmap);
        }
        for (auto& lg : leaves) {
            lg.planes = reinterpret_cast<int8_t*>(arena + lg.off_planes);
            lg.xout = reinterpret_cast<uint32_t*>(arena + lg.off_x);
            lg.tA = make_plane_map(lg.planes, lg.kpad, lg.rpad, L, lg.count, 128, BK);
            lg.tB = make_plane_map(lg.planes, lg.kpad, lg.rpad, L, lg.count, sch.b_box, BK);
        }
        for (auto& gg : gemms) {
            gg.ga = reinterpret_cast<int8_t*>(arena + gg.off_ga);
            gg.gb = reinterpret_cast<int8_t*>(arena + gg.off_gb);
            gg.out = lowmem && gg.root ? nullptr : reinterpret_cast<uint32_t*>(arena + gg.off_out);
            if (gg.wino) {
                gg.res = reinterpret_cast<uint32_t*>(arena + gg.off_res);
                gg.ga = gg.gb = nullptr;
                continue;  // no digit-plane operand maps
            }
            gg.tA = make_plane_map(gg.ga, gg.kpad, gg.hpad, sch.pa, 2 * gg.count, 128, BK);
            gg.tB = make_plane_map(gg.gb, gg.kpad, gg.hpad, sch.pb, 2 * gg.count, sch.b_box, BK);
        }
        {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            ncta = modmm_grid(sch, nsm);
        }
        for (auto& pl : prods) {
            GroupedArgs& a = pl.args;
            std::memset(&a, 0, sizeof(a));
            a.modp = m;
            fill_fold_weights(sch, p, a.w);
            a.ngroups = (int)pl.members.size();
            a.ntiles = (int)pl.host_tiles.size();
            int4* tiles = reinterpret_cast<int4*>(arena + pl.off_tiles);
            a.tiles = tiles;
            // schedule of the launch: FSYRK_B200_SCHED = dynamic | balanced (default) | strided
            static const int sched_mode = [] {
                const char* e = getenv("FSYRK_B200_SCHED");
                return !e ? 1 : !strcmp(e, "dynamic") ? 2 : !strcmp(e, "strided") ? 0 : 1;
            }();
            int* extra = reinterpret_cast<int*>(tiles + pl.host_tiles.size());  // kTileOffBytes, zeroed with the arena
            std::vector<int> tile_off;
            if (sched_mode == 2 && BMt == 128 && !nrounds && (int)pl.host_tiles.size() > ncta)
                a.dyn = extra;  // two counters, zero between launches (the kernel rearms them)
            else if (sched_mode == 1)
                tile_off = balance_tiles(pl);
            ck(cudaMemcpy(tiles, pl.host_tiles.data(), pl.host_tiles.size() * sizeof(int4), cudaMemcpyHostToDevice),
               "upload tile list");
            if (!tile_off.empty()) {
                int* off = extra + 2;
                ck(cudaMemcpy(off, tile_off.data(), tile_off.size() * sizeof(int), cudaMemcpyHostToDevice),
                   "upload tile ranges");
                a.tile_off = off;
            }
            for (int gi = 0; gi < a.ngroups; ++gi) {
                GroupDesc& g = a.g[gi];
                g.a_mult = g.b_mult = 1;
                g.a_off = g.b_off = 0;
                if (!pl.members[gi].leaf) {
                    const GemmGroup& gg = gemms[pl.members[gi].idx];
                    g.tmA = gg.tA;
                    g.tmB = gg.tB;
                    g.M = g.N = gg.h;
                    modmm_set_k(g, sch, p, gg.kpad);
                    g.syrk = 0;
                    g.vec_ok = gg.h % 4 == 0;
                    g.out = gg.out;
                    g.out_bs = (long long)gg.h * gg.h;
                    g.ldo = gg.h;
                    modmm_set_output_map(g, 2 * gg.count);
                } else {
                    const LeafGroup& lg = leaves[pl.members[gi].idx];
                    g.tmA = lg.tA;
                    g.tmB = lg.tB;
                    g.M = g.N = lg.n;
                    modmm_set_k(g, sch, p, lg.kpad);
                    g.syrk = 1;
                    g.vec_ok = lg.n % 4 == 0;
                    g.out = lg.xout;
                    g.out_bs = (long long)lg.n * lg.n;
                    g.ldo = lg.n;
                    modmm_set_output_map(g, lg.count);
                }
            }
        }
        if (nrounds) {
            dev_rounds = reinterpret_cast<int*>(arena + off_rounds);
            ck(cudaMemcpy(dev_rounds + nrounds + 1, round_target.data(), nrounds * sizeof(int), cudaMemcpyHostToDevice),
               "upload round targets");
            static const int ctas = [] {
                const char* e = getenv("FSYRK_B200_ROUND_CTAS");
                return e ? atoi(e) : 0;
            }();
            round_ctas = ctas > 0 ? std::min(ctas, ncta) : std::max(1, ncta - ncta / 6);
        }
        // node pointers (top-down: a node's input is set before its children read it)
        for (size_t i = 0; i < nodes.size(); ++i) {
            Node& nd = nodes[i];
            if (nd.parent < 0 && !nd.in64) {
                nd.in = root_in;
                nd.ldin = kin_pad;
            }
            if (nd.kind == LEAF) {
                LeafGroup& lg = leaves[nd.lgroup];
                nd.x = lg.xout + (long long)nd.lslot * nd.n * nd.n;
                nd.ldx = nd.n;
            } else if (i == 0 && nd.kind == LEVEL) {
                nd.x = nullptr;  // the root post writes the caller's C
                nd.ldx = 0;
            } else {
                nd.x = reinterpret_cast<uint32_t*>(arena + off_x[i]);
                nd.ldx = nd.n;
            }
            if (nd.kind == LEVEL) {
                if (nodes[nd.ch[2]].kind != LEAF) {
                    nd.s3res = reinterpret_cast<uint32_t*>(arena + off_s3[i]);
                    nd.lds3 = nd.kw;
                }
                Node& c0 = nodes[nd.ch[0]];
                Node& c1 = nodes[nd.ch[1]];
                Node& c2 = nodes[nd.ch[2]];
                if (!nd.in64) {
                    c0.in = nd.in;
                    c0.ldin = nd.ldin;
                    c1.in = nd.in + nd.kh;
                    c1.ldin = nd.ldin;
                }
                c2.in = nd.s3res;
                c2.ldin = nd.lds3;
            } else if (nd.kind == SPLITK && !nd.in64) {
                Node& c0 = nodes[nd.ch[0]];
                Node& c1 = nodes[nd.ch[1]];
                c0.in = nd.in;
                c0.ldin = nd.ldin;
                c1.in = nd.in + c0.k;
                c1.ldin = nd.ldin;
            }
        }
        // prep node tables
        std::vector<PrepNode> host_prep(nodes.size());
        for (auto& pg : preps) {
            const Node& n0 = nodes[pg.nodes[0]];
            GemmGroup& gg = gemms[n0.ggroup];
            PrepArgs& a = pg.args;
            a.m = m;
            a.L = sch.id;  // digit scheme
            a.h = n0.h;
            a.kh = n0.kh;
            a.kw = n0.kw;
            a.pair = y.form == 1;
            a.half = a.pair ? n0.kw / 2 : n0.kw;
            a.ya = (uint32_t)y.a;
            a.yb = (uint32_t)y.b;
            a.cya = make_mulconst(a.ya, (uint32_t)p);
            a.cyb = make_mulconst(a.yb, (uint32_t)p);
            a.in64 = 0;       // set below when a node reads the caller's matrix
            a.a64 = nullptr;  // per call
            a.ld64 = 0;
            a.g_plane = gg.plane;
            a.g_row = gg.kpad;
            a.c_plane = a.c_row = a.c3_plane = a.c3_row = 0;
            const Node& ca = nodes[n0.ch[0]];
            const Node& c3 = nodes[n0.ch[2]];
            if (ca.kind == LEAF) {
                a.c_plane = leaves[ca.lgroup].plane;
                a.c_row = leaves[ca.lgroup].kpad;
            }
            if (c3.kind == LEAF) {
                a.c3_plane = leaves[c3.lgroup].plane;
                a.c3_row = leaves[c3.lgroup].kpad;
            }
            std::vector<PrepNode> tab;
            a.aligned = 1;
            a.part_block = 0;
            a.need_mask = ~0ull;
            if (partitioned && n0.parent < 0 && part_nb <= 64) {  // the root: this rank's row blocks only
                unsigned long long need = 0;
                for (int bi = 0; bi < part_nb; ++bi)
                    for (int bj = 0; bj <= bi; ++bj)
                        if (owns_block_pair(bi, bj)) need |= (1ull << bi) | (1ull << bj);
                a.part_block = kPartBlock;
                a.need_mask = need;
            }
            for (int ni : pg.nodes) {
                const Node& nd = nodes[ni];
                GemmGroup& g = gemms[nd.ggroup];
                PrepNode pn{};
                pn.in = InView{nd.in, nd.ldin, nd.r0, nd.c0, nd.in64 ? 1 : 0};
                if (nd.in64) a.in64 = 1;
                // vector loads: uint4 of residues (uint32 input) or 2 x ulonglong2 (uint64 window)
                if (nd.in64 ? nd.c0 % 2 != 0
                            : nd.ldin % 4 != 0 || reinterpret_cast<uintptr_t>(nd.in) % 16 != 0)
                    a.aligned = 0;
                if (nd.s3res && (nd.lds3 % 4 != 0 || reinterpret_cast<uintptr_t>(nd.s3res) % 16 != 0)) a.aligned = 0;
                if (g.wino) {  // residue operands for the Winograd engine
                    pn.s1 = pn.s2 = pn.a22 = pn.s4 = nullptr;
                    pn.ld_op = g.kw;
                    pn.op_stride = (long long)g.h * g.kw;
                    pn.r_op = g.res + 4LL * nd.gslot * pn.op_stride;
                    if (pn.ld_op % 4 != 0) a.aligned = 0;
                } else {
                    pn.s1 = g.ga + (2LL * nd.gslot) * g.slot;       // P4 = S1 S2^T : problem 2s
                    pn.s2 = g.gb + (2LL * nd.gslot) * g.slot_b;
                    pn.a22 = g.ga + (2LL * nd.gslot + 1) * g.slot;  // P3 = A22 S4^T: problem 2s+1
                    pn.s4 = g.gb + (2LL * nd.gslot + 1) * g.slot_b;
                }
                const Node& q0 = nodes[nd.ch[0]];
                const Node& q1 = nodes[nd.ch[1]];
                const Node& q2 = nodes[nd.ch[2]];
                if (q0.kind == LEAF) pn.c_a11 = leaves[q0.lgroup].planes + q0.lslot * leaves[q0.lgroup].slot;
                if (q1.kind == LEAF) pn.c_a12 = leaves[q1.lgroup].planes + q1.lslot * leaves[q1.lgroup].slot;
                if (q2.kind == LEAF) pn.c_s3 = leaves[q2.lgroup].planes + q2.lslot * leaves[q2.lgroup].slot;
                pn.r_s3 = nd.s3res;
                pn.ld_s3 = nd.lds3;
                tab.push_back(pn);
                host_prep[ni] = pn;
            }
            pg.dev_nodes = reinterpret_cast<PrepNode*>(arena + pg.off_nodes);
            a.nodes = pg.dev_nodes;
            a.nnodes = (int)tab.size();
            a.ninl = tab.size() <= (size_t)kInlineNodes ? (int)tab.size() : 0;
            for (int i = 0; i < a.ninl; ++i) a.inl[i] = tab[i];
            ck(cudaMemcpy(pg.dev_nodes, tab.data(), tab.size() * sizeof(PrepNode), cudaMemcpyHostToDevice),
               "upload prep table");
        }
        setup_tree_prep(host_prep);
        std::vector<PostNode> host_post(nodes.size());
        for (auto& pg : posts) {
            if (pg.kind == LEVEL) {
                std::vector<PostNode> tab;
                for (int ni : pg.nodes) {
                    const Node& nd = nodes[ni];
                    const GemmGroup& g = gemms[nd.ggroup];
                    PostNode pn{};
                    pn.p1 = nodes[nd.ch[0]].x;
                    pn.ld1 = nodes[nd.ch[0]].ldx;
                    pn.p2 = nodes[nd.ch[1]].x;
                    pn.ld2 = nodes[nd.ch[1]].ldx;
                    pn.p5 = nodes[nd.ch[2]].x;
                    pn.ld5 = nodes[nd.ch[2]].ldx;
                    pn.p4 = g.out + (2LL * nd.gslot) * g.h * g.h;
                    pn.p3 = g.out + (2LL * nd.gslot + 1) * g.h * g.h;
                    pn.ld3 = pn.ld4 = g.h;
                    pn.x = nd.x;
                    pn.ldx = nd.ldx;
                    tab.push_back(pn);
                    host_post[ni] = pn;
                }
                pg.dev_post = reinterpret_cast<PostNode*>(arena + pg.off_nodes);
                pg.host_post = tab;
                ck(cudaMemcpy(pg.dev_post, tab.data(), tab.size() * sizeof(PostNode), cudaMemcpyHostToDevice),
                   "upload post table");
                if ((partitioned || nrounds) && pg.depth == 0 && !root_pairs.empty()) {
                    dev_pairs = reinterpret_cast<int2*>(arena + off_pairs);
                    ck(cudaMemcpy(dev_pairs, root_pairs.data(), root_pairs.size() * sizeof(int2),
                                  cudaMemcpyHostToDevice),
                       "upload pair list");
                }
            } else {
                std::vector<AddNode> tab;
                for (int ni : pg.nodes) {
                    const Node& nd = nodes[ni];
                    AddNode an{};
                    an.x1 = nodes[nd.ch[0]].x;
                    an.ld1 = nodes[nd.ch[0]].ldx;
                    an.x2 = nodes[nd.ch[1]].x;
                    an.ld2 = nodes[nd.ch[1]].ldx;
                    an.x = nd.x;
                    an.ldx = nd.ldx;
                    tab.push_back(an);
                }
                pg.dev_add = reinterpret_cast<AddNode*>(arena + pg.off_nodes);
                ck(cudaMemcpy(pg.dev_add, tab.data(), tab.size() * sizeof(AddNode), cudaMemcpyHostToDevice),
                   "upload add table");
            }
        }
        setup_post2(host_post);
        // the arena clear and the table uploads above ran on the legacy stream with pageable
        // sources (the DMA may still be in flight when cudaMemcpy returns); the calls run on
        // non-blocking streams, so finish them here
        ck(cudaDeviceSynchronize(), "plan upload");
        // op tallies
        tensor_macs = int8_macs = ew_adds = 0;
        for (auto& lg : leaves) {
            uint64_t macs = (uint64_t)lg.count * lg.n * (lg.n + 1) / 2 * lg.k;
            tensor_macs += macs;
            int8_macs += (uint64_t)lg.count * lg.ntiles * (uint64_t)BMt * BN * lg.kpad * sch.nterms;
        }
        for (auto& gg : gemms) {
            if (gg.wino) {  // one Winograd level: 7 half-size products (the engine may go deeper)
                tensor_macs += (uint64_t)2 * gg.count * 7 * (gg.h / 2) * (gg.h / 2) * (gg.kw / 2);
                ew_adds += (uint64_t)gg.count * (4ull * gg.h * gg.kw + 4ull * gg.h * gg.h);
                continue;
            }
            tensor_macs += (uint64_t)2 * gg.count * gg.h * gg.h * gg.kw;
            int8_macs += (uint64_t)2 * gg.count * ((gg.h + BMt - 1) / BMt) * ((gg.h + BN - 1) / BN) * (uint64_t)BMt *
                         BN * gg.kpad * sch.nterms;
            ew_adds += (uint64_t)gg.count * (4ull * gg.h * gg.kw + 4ull * gg.h * gg.h);
        }
        // algorithmic HBM bytes of the elementwise phases (what each kernel must read and write;
        // bench.py divides them by the phase times for the HBM roofline fraction)
        prep_bytes = post_bytes = post_cin_bytes = 0;
        convert_bytes = colmap ? (uint64_t)n * kin * 8 + (uint64_t)n * k * 4 : 0;  // caller's A in, residues out
        auto lower = [](uint64_t m) { return m * (m + 1) / 2; };
        for (const Node& nd : nodes) {
            if (nd.kind == LEVEL) {
                const uint64_t h = nd.h, kh = nd.kh, kw = nd.kw;
                // the four quadrants (the fused subtree prep reads only the root's, from the caller)
                if (!tree_depth || nd.parent < 0) prep_bytes += (uint64_t)nd.n * nd.k * (nd.in64 ? 8 : 4);
                prep_bytes += 2 * h * kw * (uint64_t)(sch.pa + sch.pb);          // S1, A22 / S2, S4 planes
                for (int c = 0; c < 3; ++c) {
                    const Node& ch = nodes[nd.ch[c]];
                    if (ch.kind == LEAF) prep_bytes += h * (uint64_t)ch.k * L;   // leaf operand planes
                    else if (c == 2 && !tree_depth) prep_bytes += h * kw * 4;     // S3 residues
                }
                post_bytes += 3 * lower(h) * 4 + 2 * h * h * 4;                  // P1, P2, P5 (lower), P3, P4
            } else if (nd.kind == SPLITK) {
                post_bytes += 2 * lower(nd.n) * 4;
            } else {
                continue;
            }
            post_bytes += lower(nd.n) * (nd.parent < 0 ? 8 : 4);  // X (the root: the caller's uint64 C)
            if (nd.parent < 0) post_cin_bytes = lower(nd.n) * 8;   // + C_in when beta != 0
            // fused two-level post: the deepest nodes' X stay on chip (not written, not read back)
            if (post2_parent_depth >= 0 && nd.kind == LEVEL && nd.depth == post2_parent_depth + 1)
                post_bytes -= 2 * lower(nd.n) * 4;
        }
    }

    std::string json() const {
        std::ostringstream o;
        static const char* scheme_names[] = {"limb2", "limb3", "limb4", "m17", "m31", "m17n"};
        o << "{\"p\": " << p << ", \"n\": " << n << ", \"k\": " << k << ", \"scheme\": \"" << scheme_names[sch.id]
          << "\", \"planes\": " << L << ", \"terms\": " << sch.products << ", \"mmas_per_kstep\": " << sch.nterms
          << ", \"accumulators\": " << sch.nacc
          << ", \"limbs\": " << L << ", \"block_n\": " << BN
          << ", \"skew\": {\"form\": \"" << (y.form ? "pair" : "scalar") << "\", \"a\": " << y.a << ", \"b\": " << y.b
          << "}, \"nodes\": " << nodes.size() << ", \"post_rounds\": " << nrounds
          << ", \"arena_bytes\": " << arena_bytes << ", \"schedule\": \"" << (lowmem ? "low-memory" : "wide") << "\""
          << ", \"tree_prep\": " << tree_depth << ", \"post2\": " << (post2_parent_depth >= 0 ? 1 : 0) << ", \"winograd_groups\": " << std::count_if(gemms.begin(), gemms.end(), [](const GemmGroup& g) { return g.wino != 0; })
          << ", \"tensor_macs\": " << tensor_macs << ", \"int8_macs\": " << int8_macs
          << ", \"prep_bytes\": " << prep_bytes << ", \"post_bytes\": " << post_bytes
          << ", \"post_cin_bytes\": " << post_cin_bytes << ", \"convert_bytes\": " << convert_bytes
          << ", \"leaf_groups\": [";
        for (size_t i = 0; i < leaves.size(); ++i)
            o << (i ? ", " : "") << "{\"n\": " << leaves[i].n << ", \"k\": " << leaves[i].k
              << ", \"count\": " << leaves[i].count << ", \"tiles\": " << leaves[i].ntiles << "}";
        o << "], \"gemm_groups\": [";
        for (size_t i = 0; i < gemms.size(); ++i)
            o << (i ? ", " : "") << "{\"h\": " << gemms[i].h << ", \"kw\": " << gemms[i].kw
              << ", \"count\": " << gemms[i].count << "}";
        o << "], \"prep_groups\": " << preps.size() << ", \"post_groups\": " << posts.size() << "}";
        return o.str();
    }

    // Levels of a complete uniform tree: lv[d] = the depth-d nodes in tree order (node t's
    // children at 3t, 3t + 1, 3t + 2 of lv[d + 1]); every node above depth D a LEVEL node of one
    // shape, unpadded, all depth-D nodes leaves of one shape.  Returns D (0: not such a tree or
    // deeper than max_depth).
    int uniform_levels(std::vector<std::vector<int>>& lv, int max_depth) const {
        lv.assign(1, std::vector<int>{0});
        int D = 0;
        for (;;) {
            const std::vector<int>& cur = lv.back();
            const Node& f0 = nodes[cur[0]];
            bool all_level = true, all_leaf = true;
            for (int i : cur) {
                const Node& nd = nodes[i];
                all_level &= nd.kind == LEVEL && !nd.padded && nd.n == f0.n && nd.k == f0.k;
                all_leaf &= nd.kind == LEAF && nd.n == f0.n && nd.k == f0.k;
            }
            if (all_leaf) return D;
            if (!all_level || D >= max_depth) return 0;
            std::vector<int> next;
            for (int i : cur)
                for (int r = 0; r < 3; ++r) next.push_back(nodes[i].ch[r]);
            lv.push_back(next);
            ++D;
        }
    }

    // The two deepest post-addition levels as one launch (post2_kernel) when the tree is
    // complete and uniform with at least two levels and the deepest quadrants are whole 32 x 32
    // tiles.  FSYRK_B200_POST2=0 keeps one launch per depth.
    void setup_post2(const std::vector<PostNode>& host_post) {
        static const int want = [] {  // 0 off, 1 parents below the root only, 2 any parent (default)
            const char* e = getenv("FSYRK_B200_POST2");
            return e ? atoi(e) : 2;
        }();
        post2_parent_depth = -1;
        if (!want || partitioned || idle || nrounds || nodes.empty() || nodes[0].kind != LEVEL) return;
        std::vector<std::vector<int>> lv;
        const int D = uniform_levels(lv, 8);
        if (D < 2) return;
        const Node& deep = nodes[lv[D - 1][0]];
        if (deep.h % 32 != 0 || nodes[lv[D - 2][0]].h != 2 * deep.h) return;  // whole 32 x 32 post2 tiles
        if (D - 2 < 1 && want < 2) return;  // FSYRK_B200_POST2=1: not with the root as the parent
        std::vector<PostNode> tab;
        for (int i : lv[D - 2]) tab.push_back(host_post[i]);
        for (int i : lv[D - 1]) tab.push_back(host_post[i]);
        post2_host = tab;
        ck(cudaMalloc(&post2_dev, tab.size() * sizeof(PostNode)), "cudaMalloc(post2 tables)");
        ck(cudaMemcpy(post2_dev, tab.data(), tab.size() * sizeof(PostNode), cudaMemcpyHostToDevice),
           "upload post2 tables");
        post2_parent_depth = D - 2;
        post2_h2 = deep.h;
        post2_nparents = (int)lv[D - 2].size();
    }

    // Balanced tile schedule of a persistent product launch.  The default gives unit u the tiles
    // u, u + units, ... of the longest-K-first list; with tiles of three or four different lengths
    // and 8-9 tiles per CTA the last CTA finished ~7% after a perfect split would (cfg2:
    // profiles/r01/variants.txt, load balance).  Here the list is dealt out in its own order, each
    // tile to the unit with the least work so far (cost: its K blocks plus an epilogue's worth),
    // so tiles still run at about the time they did (the L2 sharing of a wave of neighbouring
    // tiles survives) and every unit ends within one short tile of the others.  Returns the
    // per-unit ranges (empty: keep the strided default) and reorders pl.host_tiles by unit.
    std::vector<int> balance_tiles(ProdLaunch& pl) {
        static const bool want = [] {
            const char* e = getenv("FSYRK_B200_BALANCE");
            return !(e && atoi(e) == 0);
        }();
        const int per = BMt / 128;
        int grid = std::min(ncta, (int)pl.host_tiles.size() * per);
        if (per == 2) grid &= ~1;
        const int units = grid / per;
        if (!want || nrounds || units < 2 || (int)pl.host_tiles.size() <= units ||
            (size_t)(units + 3) * sizeof(int) > kTileOffBytes)
            return {};
        // the MMA wait a tile's epilogue costs, in 128-deep K blocks of the scheme's MMAs (per-tile
        // traces, profiles/r01/variants.txt: M17 3.2k cycles against 2.9k per block, LIMB2 1.9k / 1.0k)
        static const double epi_env = [] {
            const char* e = getenv("FSYRK_B200_BALANCE_EPI");
            return e ? atof(e) : -1.0;
        }();
        const double epi = epi_env >= 0 ? epi_env
                           : sch.id == SCHEME_LIMB2 ? 1.9
                           : sch.id == SCHEME_M31   ? 0.5
                           : sch.id == SCHEME_LIMB3 ? 1.7
                           : sch.id == SCHEME_LIMB4 ? 1.5
                                                    : 1.1;
        std::vector<double> cost(pl.members.size());
        for (size_t gi = 0; gi < pl.members.size(); ++gi) {
            const int kpad = pl.members[gi].leaf ? leaves[pl.members[gi].idx].kpad : gemms[pl.members[gi].idx].kpad;
            cost[gi] = (double)kpad / BK + epi * 128 / BK;  // K blocks + the epilogue's share
        }
        // least-loaded unit first; ties by index (deterministic)
        using Slot = std::pair<double, int>;
        std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> pq;
        for (int u = 0; u < units; ++u) pq.push({0.0, u});
        std::vector<std::vector<int4>> lists(units);
        for (const int4& t : pl.host_tiles) {
            Slot s = pq.top();
            pq.pop();
            lists[s.second].push_back(t);
            s.first += cost[t.x & ((1 << kTileGroupBits) - 1)];
            pq.push(s);
        }
        std::vector<int> off(units + 1, 0);
        std::vector<int4> ordered;
        ordered.reserve(pl.host_tiles.size());
        for (int u = 0; u < units; ++u) {
            off[u] = (int)ordered.size();
            ordered.insert(ordered.end(), lists[u].begin(), lists[u].end());
        }
        off[units] = (int)ordered.size();
        pl.host_tiles = std::move(ordered);
        return off;
    }

    // One launch for all pre-additions when the tree is complete and uniform below the root
    // (every node at depth d < D a LEVEL node of the same shape, unpadded; all depth-D nodes
    // leaves) and the root reads the caller's A; D = 2 or 3 (registers: 4^D fine blocks per
    // thread).  FSYRK_B200_TREE_PREP=0 keeps the per-depth launches.
    void setup_tree_prep(const std::vector<PrepNode>& host_prep) {
        static const bool want = [] {
            const char* e = getenv("FSYRK_B200_TREE_PREP");
            return !(e && atoi(e) == 0);
        }();
        tree_depth = 0;
        if (!want || colmap || partitioned || idle || nodes.empty() || nodes[0].kind != LEVEL || !nodes[0].in64 ||
            !split_leaves.empty())
            return;
        for (const GemmGroup& gg : gemms)
            if (gg.wino) return;  // residue operands: the per-depth kernels write them
        std::vector<std::vector<int>> lv;
        const int D = uniform_levels(lv, 3);
        if (D < 2 || D > 3) return;
        const Node& leaf = nodes[lv[D][0]];
        if (leaf.n != (n >> D) || leaf.k != (k >> D) || leaf.n * (1 << D) != n || leaf.k * (1 << D) != k) return;
        const int ncol = y.form == 1 ? leaf.k / 2 : leaf.k;  // columns (pairs) of the fine block
        if ((y.form == 1 && leaf.k % 2 != 0) || ncol % 4 != 0) return;
        int cp = D == 3 ? 32 : 128;  // kTreeCP / kTreeCP2 (elementwise.cu): 128 work items per level-0 CTA
        while (ncol % cp) cp /= 2;
        PrepTreeArgs& a = tree_args;
        a = PrepTreeArgs{};
        a.m = m;
        a.L = sch.id;
        a.depth = D;
        a.rows = leaf.n;
        a.w = leaf.k;
        a.cp = cp;
        a.pair = y.form == 1;
        a.cya = make_mulconst((uint32_t)y.a, (uint32_t)p);
        a.cyb = make_mulconst((uint32_t)y.b, (uint32_t)p);
        a.c_plane = leaves[leaf.lgroup].plane;
        a.c_row = leaves[leaf.lgroup].kpad;
        std::vector<PrepNode> tab;
        std::vector<size_t> start;
        for (int d = 0; d < D; ++d) {
            const GemmGroup& gg = gemms[nodes[lv[d][0]].ggroup];
            a.g_plane[d] = gg.plane;
            a.g_row[d] = gg.kpad;
            start.push_back(tab.size());
            for (int i : lv[d]) tab.push_back(host_prep[i]);
        }
        ck(cudaMalloc(&tree_dev, tab.size() * sizeof(PrepNode)), "cudaMalloc(tree prep table)");
        ck(cudaMemcpy(tree_dev, tab.data(), tab.size() * sizeof(PrepNode), cudaMemcpyHostToDevice),
           "upload tree prep table");
        for (int d = 0; d < D; ++d) a.nodes[d] = tree_dev + start[d];
        for (int d = 0, q = 0; d < D; ++d)
            for (size_t i = 0; i < lv[d].size(); ++i, ++q) {
                const PrepNode& pn = host_prep[lv[d][i]];
                a.tp[q] = PrepTreeArgs::Ptrs{pn.s1, pn.a22, pn.s2, pn.s4, pn.c_a11, pn.c_a12, pn.c_s3};
            }
        tree_depth = D;
    }

    // The Winograd groups' products: P4 = S1 S2^T and P3 = A22 S4^T of every member node through
    // the Strassen-Winograd engine (one grouped tensor-core launch of all base products); the
    // low-memory schedule's root products land in C12 like the direct ones.
    void run_wino(cudaStream_t s, const uint32_t* lm_p4, long long ldc) {
        for (GemmGroup& gg : gemms) {
            if (!gg.wino) continue;
            const long long st = (long long)gg.h * gg.kw, hh = (long long)gg.h * gg.h;
            std::vector<WinoProblem> probs;
            for (int q = 0; q < gg.count; ++q) {
                const uint32_t* r = gg.res + 4LL * q * st;
                uint32_t* p4 = gg.out + 2LL * q * hh;
                long long ldo = gg.h;
                uint32_t* p3 = p4 + hh;
                if (gg.root && lm_p4) {
                    p4 = const_cast<uint32_t*>(lm_p4);
                    p3 = p4 + gg.h;
                    ldo = 2 * ldc;
                }
                probs.push_back(WinoProblem{r, gg.kw, r + st, gg.kw, p4, ldo});            // P4 = S1 S2^T
                probs.push_back(WinoProblem{r + 2 * st, gg.kw, r + 3 * st, gg.kw, p3, ldo});  // P3 = A22 S4^T
            }
            wino_gemm_multi(p, probs, gg.h, gg.h, gg.kw, gg.wino_pol, s);
        }
    }

    void execute(const uint64_t* a_dev, long long lda, uint64_t* c_dev, long long ldc, uint32_t alpha,
                 uint32_t beta, bool mirror, cudaStream_t s) {
        int counts[5] = {0, 0, 0, 0, 0};
        // Phase timing: an event is recorded only at a boundary that has launches behind it since
        // the previous one -- an empty interval between two recorded events still reads ~2.7 us
        // (B200), which used to be charged to "pre" (three records before the first kernel) and
        // to "convert" on plans without a conversion pass.  at[i]: the event that stands for mark i.
        cudaEvent_t ev[7], at[7] = {};
        int marked_launches = -1;
        cudaEvent_t last_ev = nullptr;
        if (g_phase_timing)
            for (auto& e : ev) ck(cudaEventCreate(&e), "event");
        auto mark = [&](int i) {
            if (!g_phase_timing) return;
            const int total = counts[0] + counts[1] + counts[2] + counts[3] + counts[4];
            if (last_ev && total == marked_launches) {
                at[i] = last_ev;
                return;
            }
            ck(cudaEventRecord(ev[i], s), "event record");
            at[i] = last_ev = ev[i];
            marked_launches = total;
        };
        if (idle) {  // multi-GPU rank without a share (top level not partitionable)
            std::fill(g_launch_counts, g_launch_counts + 5, 0);
            g_last_plan_json = json();
            return;
        }
        mark(0);
        const Node& root = nodes[0];
        bool root_done = false;
        if (root_direct) {  // the root leaf's products write the caller's C themselves
            for (auto& pl : prods)
                for (int gi = 0; gi < pl.args.ngroups; ++gi)
                    if (pl.members[gi].leaf && pl.members[gi].idx == root.lgroup) {
                        GroupDesc& g = pl.args.g[gi];
                        g.out64 = 1;
                        g.c64 = c_dev;
                        g.ldc64 = ldc;
                        g.alpha = alpha;
                        g.beta = beta;
                        g.calpha = make_mulconst(alpha, (uint32_t)p);
                        g.cbeta = make_mulconst(beta, (uint32_t)p);
                    }
            root_done = true;
        }
        const uint32_t* lm_p4 = nullptr;  // low-memory schedule: P4 | P3 rows inside C12
        if (lowmem) {
            if (ldc % 2 != 0 || reinterpret_cast<uintptr_t>(c_dev) % 16 != 0)
                fail(FSYRK_B200_EINVAL, "low-memory schedule: C needs an even row stride and 16-byte alignment");
            lm_p4 = reinterpret_cast<const uint32_t*>(c_dev + root.h);
            if (c_dev != lm_c || ldc != lm_ldc) {
                for (auto& pl : prods)
                    for (int gi = 0; gi < pl.args.ngroups; ++gi)
                        if (!pl.members[gi].leaf && gemms[pl.members[gi].idx].root) {
                            GroupDesc& g = pl.args.g[gi];
                            g.out = const_cast<uint32_t*>(lm_p4);
                            g.ldo = 2 * ldc;
                            g.out_bs = root.h;  // P4 in the first half of each C12 row, P3 in the second
                            modmm_set_output_map(g, 2);
                        }
                lm_c = c_dev;
                lm_ldc = ldc;
            }
        }
        // 1. syrkd: convert the reference-layout input with the column transform folded in;
        //    otherwise the top-level pre-additions read the caller's uint64 matrix directly
        if (colmap) {
            ck(launch_convert_in(a_dev, lda, n, kin, k, dev_colmap, (uint32_t)p, root_in, root.ldin, s), "convert_in");
            counts[3]++;
        }
        mark(6);  // end of the conversion pass
        // 2. leaf operands that are plain views (root leaf, split-on-k children)
        for (int li : split_leaves) {
            const Node& nd = nodes[li];
            const LeafGroup& lg = leaves[nd.lgroup];
            ck(launch_split_planes(sch.id, InView{nd.in, nd.ldin, nd.r0, nd.c0, nd.in64 ? 1 : 0}, a_dev, lda, nd.n, nd.k,
                                   (uint32_t)p, lg.planes + nd.lslot * lg.slot, lg.plane, lg.kpad, s),
               "split_planes");
            counts[1]++;
        }
        mark(1);
        // FSYRK_B200_TRACE=1: per-launch events on their streams, timeline printed to stderr
        static const bool trace = getenv("FSYRK_B200_TRACE") != nullptr;
        struct TraceRec {
            std::string name;
            cudaEvent_t a, b;
        };
        std::vector<TraceRec> tr;
        auto traced = [&](const std::string& name, cudaStream_t st, auto&& fn) {
            if (!trace) {
                fn();
                return;
            }
            TraceRec r{name, nullptr, nullptr};
            cudaEventCreate(&r.a);
            cudaEventCreate(&r.b);
            cudaEventRecord(r.a, st);
            fn();
            cudaEventRecord(r.b, st);
            tr.push_back(r);
        };
        auto run_prep = [&](PrepGroup& pg, cudaStream_t st) {
            PrepArgs a = pg.args;
            if (a.in64) {
                a.a64 = a_dev;
                a.ld64 = lda;
            }
            traced("prep d" + std::to_string(pg.depth), st, [&] { ck(launch_prep(a, st), "prep"); });
            counts[1]++;
        };
        auto run_prod = [&](ProdLaunch& pl, cudaStream_t st) {
            traced("products phase " + std::to_string(pl.phase), st,
                   [&] { ck(modmm_launch(sch, pl.args, std::min(ncta, pl.args.ntiles * (BMt / 128)), st), "modmm"); });
            counts[0]++;
        };
        auto run_post = [&](PostGroup& pg, cudaStream_t st, bool fused2 = false) {
            if (pg.kind == LEVEL) {
                PostArgs a{};
                a.m = m;
                a.h = pg.n / 2;
                a.nodes = fused2 ? post2_dev : pg.dev_post;
                a.nnodes = fused2 ? post2_nparents : (int)pg.nodes.size();
                {
                    const std::vector<PostNode>& tab = fused2 ? post2_host : pg.host_post;
                    a.ninl = a.nnodes <= kInlineNodes && (int)tab.size() >= a.nnodes ? a.nnodes : 0;
                    for (int i = 0; i < a.ninl; ++i) a.inl[i] = tab[i];
                }
                if (pg.depth == 0) {  // the root writes alpha X + beta C into the caller's C
                    if (lm_p4) {
                        a.p4o = lm_p4;
                        a.p3o = lm_p4 + root.h;
                        a.ld34o = 2 * ldc;
                    }
                    a.out64 = 1;
                    a.c64 = c_dev;
                    a.ldc = ldc;
                    a.alpha = alpha;
                    a.beta = beta;
                    a.calpha = make_mulconst(alpha, (uint32_t)p);
                    a.cbeta = make_mulconst(beta, (uint32_t)p);
                    root_done = true;
                    if (partitioned) {
                        if (root_pairs.empty()) return;  // this rank owns no block pair
                        a.pairs = dev_pairs;
                        a.npairs = (int)root_pairs.size();
                    }
                }
                if (fused2) {  // this level and the one below it in one launch
                    Post2Args a2{};
                    a2.par = a;
                    a2.ch = post2_dev + post2_nparents;
                    a2.h2 = post2_h2;
                    const int nch = (int)post2_host.size() - post2_nparents;
                    a2.nchi = nch <= kInlineChildren ? nch : 0;
                    for (int i = 0; i < a2.nchi; ++i) a2.chi[i] = post2_host[post2_nparents + i];
                    traced("post d" + std::to_string(pg.depth) + "+" + std::to_string(pg.depth + 1), st,
                           [&] { ck(launch_post2(a2, st), "post2"); });
                } else {
                    traced("post d" + std::to_string(pg.depth), st, [&] { ck(launch_post(a, st), "post"); });
                }
            } else {
                ck(launch_add_lower(pg.dev_add, (int)pg.nodes.size(), pg.n, (uint32_t)p, st), "add_lower");
            }
            counts[2]++;
        };
        const bool overlap = !g_phase_timing && !prods.empty() && prods[0].phase == 0;
        const bool post_rounds = !g_phase_timing && nrounds > 0 && !trace;
        if (post_rounds) {
            ck(cudaMemsetAsync(dev_rounds, 0, (nrounds + 1) * sizeof(int), s), "clear round counters");
            for (auto& pg : preps) run_prep(pg, s);
            mark(2);
            ProdLaunch& pm = prods[0];
            GroupedArgs ga = pm.args;
            ga.round_done = dev_rounds;
            ck(modmm_launch(sch, ga, std::min(round_ctas, ga.ntiles * (BMt / 128)), s), "modmm");
            counts[0]++;
            const PostGroup& root_post = posts[0];
            PostArgs a{};
            a.m = m;
            a.h = root_post.n / 2;
            a.nodes = root_post.dev_post;
            a.nnodes = 1;
            a.out64 = 1;
            a.c64 = c_dev;
            a.ldc = ldc;
            a.alpha = alpha;
            a.beta = beta;
            a.calpha = make_mulconst(alpha, (uint32_t)p);
            a.cbeta = make_mulconst(beta, (uint32_t)p);
            a.pairs = dev_pairs;
            a.npairs = (int)root_pairs.size();
            static const int post_blocks = [] {
                const char* e = getenv("FSYRK_B200_POST_BLOCKS");
                return e ? atoi(e) : 0;
            }();
            const int blocks = post_blocks > 0 ? post_blocks : 6 * nsm;
            ck(launch_post_rounds(a, dev_rounds, dev_rounds + nrounds + 1, dev_rounds + nrounds, blocks, s),
               "post rounds");
            counts[2]++;
            root_done = true;
            mark(3);
            mark(4);
        } else if (!overlap) {
            // 3. fused pre-additions, top-down; 4. products; 5. post-additions, bottom-up
            if (tree_depth) {
                PrepTreeArgs a = tree_args;
                a.a64 = a_dev;
                a.ld64 = lda;
                traced("prep tree", s, [&] { ck(launch_prep_tree(a, nsm, s), "prep tree"); });
                counts[1]++;
            } else {
                for (auto& pg : preps) run_prep(pg, s);
            }
            mark(2);
            for (auto& pl : prods) run_prod(pl, s);
            run_wino(s, lm_p4, ldc);
            mark(3);
            for (auto& pg : posts) {
                if (post2_parent_depth >= 0 && pg.kind == LEVEL && pg.depth == post2_parent_depth + 1) continue;
                run_post(pg, s, post2_parent_depth >= 0 && pg.kind == LEVEL && pg.depth == post2_parent_depth);
            }
            mark(4);
        } else {
            // The top level's two general products need only the top pre-additions; they run on
            // the caller's stream while a side stream carries the deeper pre-additions, products
            // and post-additions (elementwise work co-resides with the persistent tensor kernel:
            // it leaves HBM bandwidth and issue slots idle).  The root post-addition joins both.
            if (!side) {
                ck(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking), "side stream");
                ck(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming), "event");
            }
            for (auto& pg : preps)
                if (pg.depth == 0) run_prep(pg, s);
            ck(cudaEventRecord(ev_fork, s), "fork");
            ck(cudaStreamWaitEvent(side, ev_fork, 0), "fork wait");
            for (auto& pl : prods)
                if (pl.phase == 0) run_prod(pl, s);
            for (auto& pg : preps)
                if (pg.depth != 0) run_prep(pg, side);
            for (auto& pl : prods)
                if (pl.phase != 0) run_prod(pl, side);
            for (auto& pg : posts)
                if (pg.depth != 0) run_post(pg, side);
            ck(cudaEventRecord(ev_join, side), "join");
            ck(cudaStreamWaitEvent(s, ev_join, 0), "join wait");
            for (auto& pg : posts)
                if (pg.depth == 0) run_post(pg, s);
        }
        // 6. root leaf / split: C <- alpha X + beta C in the reference layout; optional mirror
        if (!root_done) {
            ck(launch_finalize(root.x, root.ldx, n, c_dev, ldc, m, alpha, beta, s), "finalize");
            counts[3]++;
        }
        if (mirror) {
            ck(launch_mirror(c_dev, ldc, n, s), "mirror");
            counts[3]++;
        }
        mark(5);
        if (trace && !tr.empty()) {
            cudaError_t se = cudaStreamSynchronize(s);
            if (se != cudaSuccess) fprintf(stderr, "[fsyrk trace] sync: %s\n", cudaGetErrorString(se));
            for (auto& r : tr) {
                float t0 = 0, t1 = 0;
                cudaError_t e0 = cudaEventElapsedTime(&t0, tr[0].a, r.a);
                cudaError_t e1 = cudaEventElapsedTime(&t1, tr[0].a, r.b);
                if (e0 != cudaSuccess || e1 != cudaSuccess)
                    fprintf(stderr, "[fsyrk trace] elapsed: %s / %s\n", cudaGetErrorString(e0), cudaGetErrorString(e1));
                fprintf(stderr, "[fsyrk trace] %-20s %8.1f us -> %8.1f us (%7.1f us)\n", r.name.c_str(), t0 * 1e3,
                        t1 * 1e3, (t1 - t0) * 1e3);
            }
            for (auto& r : tr) {
                cudaEventDestroy(r.a);
                cudaEventDestroy(r.b);
            }
        }
        std::copy(counts, counts + 5, g_launch_counts);
        if (g_phase_timing) {
            ck(cudaEventSynchronize(at[5]), "event sync");
            // kinds: 0 products, 1 pre (split + prep), 2 post, 3 convert/finalize
            auto span = [&](int a, int b) {
                float ms = 0;
                if (at[a] && at[b] && at[a] != at[b]) cudaEventElapsedTime(&ms, at[a], at[b]);
                return ms;
            };
            g_phase_ms[0] = span(2, 3);
            g_phase_ms[1] = span(6, 2);               // pre: end of conversion -> end of pre-additions
            g_phase_ms[2] = span(3, 4);
            g_phase_ms[3] = span(0, 6) + span(4, 5);  // convert + finalize / mirror
            g_phase_ms[4] = 0;
            for (auto& e : ev) cudaEventDestroy(e);
        }
        g_last_plan_json = json();
    }
};

// ------------------------------------------------------------ plan cache
struct PlanKey {
    uint64_t p;
    int n, kin, k;
    uint64_t thr, lev;
    bool colmap;
    int dev, rank, nranks;
    bool lowmem;
    uint64_t wino_min;
    bool operator<(const PlanKey& o) const {
        return std::tie(p, n, kin, k, thr, lev, colmap, dev, rank, nranks, lowmem, wino_min) <
               std::tie(o.p, o.n, o.kin, o.k, o.thr, o.lev, o.colmap, o.dev, o.rank, o.nranks, o.lowmem, o.wino_min);
    }
};

// Process-wide workspace limit (fsyrk_b200_set_workspace_limit): 0 = none.  A plan whose wide
// workspace exceeds it uses the low-memory schedule; one that exceeds it even so is refused.
std::atomic<uint64_t> g_ws_limit{0};
std::atomic<int> g_force_lowmem{0};  // fsyrk_b200_set_low_memory(1): every applicable plan

uint64_t dry_arena(uint64_t p, int n, int kin, int k, fsyrk_b200_policy pol, bool colmap, int rank, int nranks,
                   bool lowmem) {
    Plan plan;
    plan.create(p, n, kin, k, pol, colmap, rank, nranks, true, lowmem);
    return plan.arena_bytes;
}

std::mutex g_cache_mu;
std::map<PlanKey, std::shared_ptr<Plan>> g_cache;  // guarded by g_cache_mu

// The cache lookup / creation is serialised; a call keeps its plan alive (shared ownership)
// even if fsyrk_b200_release_cache drops the cache's reference meanwhile.
std::shared_ptr<Plan> get_plan(uint64_t p, int n, int kin, int k, fsyrk_b200_policy pol, bool colmap, int rank = 0,
                               int nranks = 1) {
    int dev = 0;
    cudaGetDevice(&dev);
    bool lowmem = g_force_lowmem.load() != 0;
    if (const uint64_t limit = g_ws_limit.load(); limit && !lowmem) {
        // the schedule decision per (shape, limit) is made once (two host-only dry layouts)
        static std::mutex mu;
        static std::map<std::pair<PlanKey, uint64_t>, bool> decided;
        const PlanKey k0{p, n, kin, k, pol.threshold, pol.max_levels, colmap, dev, rank, nranks, false, g_wino_min.load()};
        std::lock_guard<std::mutex> lk(mu);
        auto d = decided.find({k0, limit});
        if (d != decided.end()) {
            lowmem = d->second;
        } else {
            if (dry_arena(p, n, kin, k, pol, colmap, rank, nranks, false) > limit) {
                lowmem = true;
                const uint64_t lm = dry_arena(p, n, kin, k, pol, colmap, rank, nranks, true);
                if (lm > limit)
                    fail(FSYRK_B200_EINVAL, "workspace limit of " + std::to_string(limit) + " bytes is below the " +
                                                std::to_string(lm) + " bytes of the low-memory schedule");
            }
            decided[{k0, limit}] = lowmem;
        }
    }
    PlanKey key{p, n, kin, k, pol.threshold, pol.max_levels, colmap, dev, rank, nranks, lowmem, g_wino_min.load()};
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) return it->second;
    auto plan = std::make_shared<Plan>();
    plan->create(p, n, kin, k, pol, colmap, rank, nranks, false, lowmem);
    g_cache[key] = plan;
    return plan;
}

// ------------------------------------------------------------- validation
void validate_field(uint64_t p) {
    if (p >= (1ull << 31)) fail(FSYRK_B200_EINVAL, "prime modulus must be < 2^31, got " + std::to_string(p));
    if (!host::is_prime(p)) fail(FSYRK_B200_EINVAL, std::to_string(p) + " is not prime");
}
void validate_policy(fsyrk_b200_policy pol) {
    if (pol.threshold < 2) fail(FSYRK_B200_EINVAL, "recursion threshold must be >= 2");
}
void validate_shapes(size_t n, size_t k, size_t lda, size_t ldc) {
    if (lda < k || ldc < n) fail(FSYRK_B200_EDIMENSION, "syrk_fast: dimension mismatch (stride smaller than row)");
    if (n > (size_t)INT32_MAX / 2 || k > (size_t)INT32_MAX / 2) fail(FSYRK_B200_EDIMENSION, "matrix too large");
}
bool ranges_overlap(const void* a, size_t a_bytes, const void* b, size_t b_bytes) {
    if (a_bytes == 0 || b_bytes == 0) return false;
    auto pa = reinterpret_cast<uintptr_t>(a), pb = reinterpret_cast<uintptr_t>(b);
    return pa < pb + b_bytes && pb < pa + a_bytes;
}
size_t span_bytes(size_t rows, size_t cols, size_t ld) { return rows == 0 || cols == 0 ? 0 : ((rows - 1) * ld + cols) * 8; }

// Column transform applied to A on its way in (convert_in): column j of the
// transformed matrix is sum_t c[t] * A[:, src[t]].
struct ColXform {
    std::vector<ColMap> map;
    // the reference's own tallies of the column transform, per row of A (scaled_syrk.hpp:42-48,
    // 91-100, 146-153): columns scaled by sqrt(d) != 1, nrsyf pairs, syrkbd 2x2 blocks
    uint64_t scaled_cols = 0, nr_pairs = 0, blocks2 = 0;
};

ColMap col_identity(int j) { return ColMap{{j, -1, -1, -1}, {1, 0, 0, 0}}; }

// cu * u + cv * v for two transformed columns (term lists concatenate; at most 4 terms
// because only syrkbd's (u + v, u - v) columns carry two).
ColMap col_combine(const host::Field& f, const ColMap& u, uint64_t cu, const ColMap& v, uint64_t cv) {
    ColMap r{{-1, -1, -1, -1}, {0, 0, 0, 0}};
    int t = 0;
    for (const auto* src : {&u, &v}) {
        const uint64_t w = src == &u ? cu : cv;
        for (int q = 0; q < 4; ++q)
            if (src->src[q] >= 0) {
                if (t == 4) fail(FSYRK_B200_EINVAL, "column transform exceeds 4 source columns");
                r.src[t] = src->src[q];
                r.c[t++] = (uint32_t)f.mul(w, src->c[q]);
            }
    }
    return r;
}

// syrkd's diagonal fold (include/fsyrk/scaled_syrk.hpp:58-104) applied on top of an
// initial column map `map` (identity for syrkd, syrkbd's block fold otherwise): residue
// entries scale their column by sqrt(d), non-residues are consumed in pairs through their
// nrsyf factor, an odd count appends a zero column carrying a copy of the first one.
// fn(i) for i in [0, n): O(log p) field work per index (Legendre symbols, square roots,
// nrsyf factors), split over host threads when n is large enough to pay for them.
template <class Fn>
void parallel_for(size_t n, Fn fn) {
    const size_t hw = std::max<size_t>(1, std::thread::hardware_concurrency());
    const size_t nt = n < 256 ? 1 : std::min<size_t>({hw, 16, n / 128});
    if (nt <= 1) {
        for (size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    for (size_t t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            for (size_t i = t * n / nt; i < (t + 1) * n / nt; ++i) fn(i);
        });
    for (auto& th : pool) th.join();
}

void fold_diagonal(uint64_t p, std::vector<uint64_t> dbar, std::vector<ColMap>& map, ColXform* tally = nullptr) {
    host::Field f{p};
    if (p == 2) fail(FSYRK_B200_EINVAL, "syrkd requires an odd prime field");
    const size_t k = dbar.size();
    for (auto& v : dbar) v %= p;
    std::vector<int> leg(k);
    parallel_for(k, [&](size_t j) { leg[j] = f.legendre(dbar[j]); });
    std::vector<size_t> nr;
    for (size_t j = 0; j < k; ++j)
        if (leg[j] == -1) nr.push_back(j);
    if (nr.size() % 2 == 1) {
        dbar.push_back(dbar[nr.front()]);
        leg.push_back(-1);
        nr.push_back(k);
        map.push_back(ColMap{{-1, -1, -1, -1}, {0, 0, 0, 0}});  // the appended zero column
    }
    std::vector<char> scaled(dbar.size(), 0);
    parallel_for(dbar.size(), [&](size_t j) {
        if (leg[j] < 0) return;
        const uint64_t sq = f.sqrt(dbar[j]);
        scaled[j] = sq != 1;  // scale_column skips s = 1 (scaled_syrk.hpp:45)
        for (int q = 0; q < 4; ++q)
            if (map[j].src[q] >= 0) map[j].c[q] = (uint32_t)f.mul(map[j].c[q], sq);
    });
    const size_t npairs = nr.size() / 2;
    std::vector<char> bad(npairs, 0);
    parallel_for(npairs, [&](size_t t) {
        const size_t i = nr[2 * t], j = nr[2 * t + 1];
        std::array<uint64_t, 4> y;
        if (!host::nrsyf(f, dbar[i], dbar[j], y)) {
            bad[t] = 1;
            return;
        }
        // (u, v) -> (y0 u + y2 v, y1 u + y3 v)   (scaled_syrk.hpp:93-98)
        try {  // no exception may leave a worker thread
            const ColMap u = map[i], v = map[j];
            map[i] = col_combine(f, u, y[0], v, y[2]);
            map[j] = col_combine(f, u, y[1], v, y[3]);
        } catch (...) {
            bad[t] = 2;
        }
    });
    for (char b : bad) {
        if (b == 1) fail(FSYRK_B200_ENONRES, "nrsyf: argument is not a non-residue");
        if (b == 2) fail(FSYRK_B200_EINVAL, "column transform exceeds 4 source columns");
    }
    if (tally) {
        for (char c : scaled) tally->scaled_cols += (uint64_t)c;
        tally->nr_pairs += npairs;
    }
}

ColXform xform_diag(uint64_t p, const uint64_t* d, size_t k) {
    ColXform x;
    for (size_t j = 0; j < k; ++j) x.map.push_back(col_identity((int)j));
    fold_diagonal(p, std::vector<uint64_t>(d, d + k), x.map, &x);
    return x;
}

// syrkbd over a prime field (include/fsyrk/scaled_syrk.hpp:117-159): every 2x2 block
// ((0, beta), (beta, 0)) becomes diagonal entries (beta/2, -beta/2) under the column
// transform (u, v) -> (u + v, u - v); then the diagonal fold of syrkd.
ColXform xform_blocks(uint64_t p, const fsyrk_b200_block* b, size_t nblocks, size_t k) {
    host::Field f{p};
    size_t dim = 0;
    for (size_t i = 0; i < nblocks; ++i) {
        if (b[i].two && b[i].beta % p == 0) fail(FSYRK_B200_EINVAL, "block-diagonal: 2x2 block requires beta != 0");
        dim += b[i].two ? 2 : 1;
    }
    if (dim != k) fail(FSYRK_B200_EDIMENSION, "syrkbd: block-diagonal dimension must match column count");
    if (p == 2) fail(FSYRK_B200_EINVAL, "syrkbd over characteristic 2 uses BinaryField");
    const uint64_t half = f.inv(2 % p);
    ColXform x;
    std::vector<uint64_t> dbar(k, 1);
    for (size_t i = 0, j = 0; i < nblocks; ++i) {
        if (!b[i].two) {
            x.map.push_back(col_identity((int)j));
            dbar[j++] = b[i].d % p;
            continue;
        }
        if (b[i].gamma % p != 0) fail(FSYRK_B200_EINVAL, "syrkbd: 2x2 blocks in odd characteristic must be antidiagonal");
        dbar[j] = f.mul(half, b[i].beta % p);
        dbar[j + 1] = (p - dbar[j]) % p;
        x.map.push_back(ColMap{{(int)j, (int)j + 1, -1, -1}, {1, 1, 0, 0}});
        x.map.push_back(ColMap{{(int)j, (int)j + 1, -1, -1}, {1, (uint32_t)(p - 1), 0, 0}});
        j += 2;
        x.blocks2++;
    }
    fold_diagonal(p, std::move(dbar), x.map, &x);
    return x;
}

struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    void ensure(size_t b) {
        if (b <= bytes) return;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        ck(cudaMalloc(&ptr, b), "cudaMalloc(staging)");
        bytes = b;
    }
    ~DevBuf() {
        if (ptr) cudaFree(ptr);
    }
};

// The host entry points' staging (device buffers, pinned slots, the host worker pool) is one
// resource: one host call at a time.  The device-side buffers and streams are per device.
std::mutex g_stage_mu;

// OpCount as the reference counts it (ref_opcount.h): a host dry-run of the reference's
// recursion for this call.  syrk_fast_into is syrk_fast_acc with (1, 0), which the reference
// tallies identically.  With a column transform the call is the reference's syrkd / syrkbd
// (transform + plain syrk_fast over the transformed A) followed by this library's alpha / beta
// extension, tallied like syrk_classical's scaling: tri mults per alpha != 1 and per
// beta not in {0, 1}, tri adds for beta != 0.
refops::Model ref_model(uint64_t p, const fsyrk_b200_policy& pol) {
    refops::Model md;
    md.threshold = pol.threshold;
    md.max_levels = pol.max_levels;
    const host::Skew y = host::skew_orthogonal(host::Field{p});
    md.skew_form = y.form;
    md.skew_a_one = y.a == 1;
    return md;
}

refops::Tally ref_tally(uint64_t p, size_t n, size_t kbar, const fsyrk_b200_policy& pol, uint64_t alpha, uint64_t beta,
                        const ColXform* xf) {
    refops::Model md = ref_model(p, pol);
    alpha %= p;
    beta %= p;
    if (!xf) {
        const bool acc = !(alpha == 1 && beta == 0);
        return md.syrk(n, kbar, pol.max_levels, acc, refops::Scalar::of(alpha), refops::Scalar::of(beta));
    }
    refops::Tally t;
    t.mults = n * (xf->scaled_cols + 4 * xf->nr_pairs);
    t.adds = n * (2 * xf->nr_pairs + 2 * xf->blocks2);
    t += md.syrk(n, kbar, pol.max_levels, false, refops::Scalar::unit(), refops::Scalar::nil());
    const uint64_t tri = refops::Model::tri(n);
    if (alpha != 1) t.mults += tri;
    if (beta != 0 && beta != 1) t.mults += tri;
    if (beta != 0) t.adds += tri;
    return t;
}

// F_{p^2}: the reference's syrk_fast / herk_fast recursion over QuadExtField (scalar skew root
// sqrt(-1) or the skew-unitary z, never 1 for odd p; skew.hpp:76-100), one tally per
// extension-field operation.
refops::Tally ref_tally_fp2(size_t n, size_t k, const fsyrk_b200_policy& pol) {
    refops::Model md;
    md.threshold = pol.threshold;
    md.max_levels = pol.max_levels;
    md.skew_form = 0;
    md.skew_a_one = false;
    return md.syrk(n, k, pol.max_levels, false, refops::Scalar::unit(), refops::Scalar::nil());
}

void add_tally(fsyrk_b200_opcount* ops, const refops::Tally& t) {
    if (!ops) return;
    ops->mults += t.mults;
    ops->adds += t.adds;
}

// Adds a call's tally when the call returns normally (not when it throws).
struct TallyOnSuccess {
    fsyrk_b200_opcount* ops;
    refops::Tally t;
    int exc = std::uncaught_exceptions();
    ~TallyOnSuccess() {
        if (std::uncaught_exceptions() == exc) add_tally(ops, t);
    }
};

// One operand of a batched product: a uint32 residue view, or a window of a uint64 matrix.
struct GemmOperand {
    InView v;
    const uint64_t* a64 = nullptr;
    long long ld64 = 0;
};
GemmOperand operand_u64(const uint64_t* a, long long lda) { return GemmOperand{InView{nullptr, 0, 0, 0, 1}, a, lda}; }
GemmOperand operand_u32(const uint32_t* a, long long lda) { return GemmOperand{InView{a, lda, 0, 0, 0}, nullptr, 0}; }

// out[b] = A[b] * B[b]^T mod p (b = 0 .. batch-1; A[b] m x k, B[b] n x k, out[b] at out + b * out_bs,
// row stride ldo) on the tensor cores: digit split per operand, ONE grouped product launch.
// Scratch buffers are call-local (products outside the recursion plan are not hot).
void gemm_batch_dev(uint64_t p, size_t m, size_t n, size_t k, const std::vector<GemmOperand>& A,
                    const std::vector<GemmOperand>& B, uint32_t* out, long long ldo, long long out_bs,
                    cudaStream_t s) {
    const SchemeInfo sch = scheme_for(p);
    const int L = sch.planes, BN = sch.bn, BK = sch.bk;
    const int batch = (int)A.size();
    if (m == 0 || n == 0 || batch == 0) return;
    const long long kpad = round_up((long long)std::max<size_t>(k, 1), 128);
    const long long mpad = round_up((long long)m, 128), npad = round_up((long long)n, 128);
    // scratch kept across calls (grows to the largest product seen); one product at a time per device
    struct Scratch {
        std::mutex mu;
        DevBuf pa, pb, dtiles;
    };
    Scratch& sc = per_device<Scratch>();
    std::lock_guard<std::mutex> lk(sc.mu);
    DevBuf &pa = sc.pa, &pb = sc.pb, &dtiles = sc.dtiles;
    pa.ensure((size_t)(mpad * kpad * L * batch));
    pb.ensure((size_t)(npad * kpad * L * batch));
    ck(cudaMemsetAsync(pa.ptr, 0, (size_t)(mpad * kpad * L * batch), s), "memset");
    ck(cudaMemsetAsync(pb.ptr, 0, (size_t)(npad * kpad * L * batch), s), "memset");
    for (int b = 0; k > 0 && b < batch; ++b) {
        ck(launch_split_planes(sch.id, A[b].v, A[b].a64, A[b].ld64, (int)m, (int)k, (uint32_t)p,
                               static_cast<int8_t*>(pa.ptr) + (long long)b * L * mpad * kpad, mpad * kpad, kpad, s),
           "split A");
        ck(launch_split_planes(sch.id, B[b].v, B[b].a64, B[b].ld64, (int)n, (int)k, (uint32_t)p,
                               static_cast<int8_t*>(pb.ptr) + (long long)b * L * npad * kpad, npad * kpad, kpad, s),
           "split B");
    }
    std::vector<int4> tiles;
    for (int b = 0; b < batch; ++b)
        for (int tm = 0; tm * sch.bm < (int)m; ++tm)
            for (int tn = 0; tn * BN < (int)n; ++tn) tiles.push_back(make_int4(0, b, tm, tn));
    dtiles.ensure(tiles.size() * sizeof(int4));
    ck(cudaMemcpyAsync(dtiles.ptr, tiles.data(), tiles.size() * sizeof(int4), cudaMemcpyHostToDevice, s), "tiles");
    GroupedArgs args;
    std::memset(&args, 0, sizeof(args));
    args.modp = make_modp((uint32_t)p);
    fill_fold_weights(sch, p, args.w);
    args.ngroups = 1;
    args.ntiles = (int)tiles.size();
    args.tiles = static_cast<int4*>(dtiles.ptr);
    GroupDesc& g = args.g[0];
    g.tmA = make_plane_map(pa.ptr, (int)kpad, (int)mpad, L, batch, 128, BK);
    g.tmB = make_plane_map(pb.ptr, (int)kpad, (int)npad, L, batch, sch.b_box, BK);
    g.M = (int)m;
    g.N = (int)n;
    modmm_set_k(g, sch, p, kpad);
    g.syrk = 0;
    g.vec_ok = ldo % 4 == 0 && out_bs % 4 == 0;
    g.a_mult = g.b_mult = 1;
    g.out = out;
    g.out_bs = out_bs;
    g.ldo = ldo;
    modmm_set_output_map(g, batch);
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    ck(modmm_launch(sch, args, std::min<int>(modmm_grid(sch, nsm), (int)tiles.size() * (sch.bm / 128)), s), "modmm");
    ck(cudaStreamSynchronize(s), "sync");  // the scratch is reused by the next call
}

// C = A * B^T mod p for device-resident uint64 A (m x k, lda) and B (n x k, ldb) into uint32 out.
void gemm_nt_dev(uint64_t p, const uint64_t* a, size_t m, size_t k, size_t lda, const uint64_t* b, size_t n,
                 size_t ldb, uint32_t* out, long long ldo, cudaStream_t s) {
    gemm_batch_dev(p, m, n, k, {operand_u64(a, (long long)lda)}, {operand_u64(b, (long long)ldb)}, out, ldo, 0, s);
}

// Strassen-Winograd levels over the tensor-core product (the reference's generic-product
// engine gemm_winograd_nt_into, include/fsyrk/winograd.hpp:118-169, 195-202): C = A B^T for
// uint32 residue matrices A (m x k) and B (n x k, the stored form of B^T).  Each level splits
// every problem into 7 half-size products with the pre-additions
//   S1 = A21 + A22, S2 = S1 - A11, S3 = A11 - A21, S4 = A12 - S2,
//   T1 = B'12 - B'11, T2 = B'22 - T1, T3 = B'22 - B'12, T4 = T2 - B'21     (B' = B^T blocks)
// and the post-additions C11 = M1 + M2, C12 = M1 + M6 + M5 + M3, C21 = M1 + M6 + M7 - M4,
// C22 = M1 + M6 + M7 + M5; all 7^levels base products of a call run as ONE grouped
// tensor-core launch.  Levels stop where a dimension is odd or below the policy threshold
// (the reference peels odd dimensions instead; the result is the same exact product).
void wino_gemm_multi(uint64_t p, const std::vector<WinoProblem>& probs, size_t m, size_t n, size_t k,
                     fsyrk_b200_policy pol, cudaStream_t s) {
    struct Prob {
        GemmOperand a, b;
        uint32_t* c;
        long long ldc;
    };
    std::vector<Prob> cur;
    for (const WinoProblem& w : probs) cur.push_back({operand_u32(w.a, w.lda), operand_u32(w.b, w.ldb), w.c, w.ldc});
    if (cur.empty()) return;
    struct Level {
        std::vector<Prob> parents;
        uint32_t* m_out;  // 7 x parents.size() products of hm x hn, child-major order
        long long hm, hn;
    };
    std::vector<Level> levels;
    struct Pool {  // per-level scratch kept across calls, per device
        std::mutex mu;
        std::vector<std::unique_ptr<DevBuf>> bufs;
    };
    Pool& pl = per_device<Pool>();
    std::lock_guard<std::mutex> lk(pl.mu);
    std::vector<std::unique_ptr<DevBuf>>& pool = pl.bufs;
    size_t cm = m, cn = n, ck_ = k;
    const uint32_t pp = (uint32_t)p;
    for (uint64_t lev = 0; lev < pol.max_levels; ++lev) {
        if (cm % 2 || cn % 2 || ck_ % 2 || std::min({cm, cn, ck_}) < pol.threshold) break;
        const long long hm = (long long)cm / 2, hn = (long long)cn / 2, hk = (long long)ck_ / 2;
        Level L;
        L.hm = hm;
        L.hn = hn;
        const size_t np = cur.size();
        // per parent: S1..S4 (hm x hk), T1..T4 (hn x hk); per level: 7 np products (hm x hn)
        const size_t per = (size_t)(4 * hm * hk + 4 * hn * hk);
        if (pool.size() <= lev) pool.push_back(std::make_unique<DevBuf>());
        pool[lev]->ensure((per * np + (size_t)7 * np * hm * hn) * 4);
        auto* base = static_cast<uint32_t*>(pool[lev]->ptr);
        L.m_out = base + per * np;
        std::vector<Prob> next;
        for (size_t q = 0; q < np; ++q) {
            const Prob& pr = cur[q];
            uint32_t* S = base + per * q;
            uint32_t* T = S + 4 * hm * hk;
            const uint32_t* a = pr.a.v.p32;
            const long long la = pr.a.v.ld32;
            const uint32_t* b = pr.b.v.p32;
            const long long lb = pr.b.v.ld32;
            ck(launch_wino_pre(a, a + hk, a + hm * la, a + hm * la + hk, la, (int)hm, (int)hk, pp, 0, S, hk,
                               hm * hk, s),
               "winograd pre A");
            // stored blocks of B: B'11 = B[0:hn, 0:hk], B'12 = B[hn:, 0:hk], B'21 = B[0:hn, hk:], B'22 = B[hn:, hk:]
            ck(launch_wino_pre(b, b + hn * lb, b + hk, b + hn * lb + hk, lb, (int)hn, (int)hk, pp, 1, T, hk,
                               hn * hk, s),
               "winograd pre B");
            const uint32_t *S1 = S, *S2 = S + hm * hk, *S3 = S + 2 * hm * hk, *S4 = S + 3 * hm * hk;
            const uint32_t *T1 = T, *T2 = T + hn * hk, *T3 = T + 2 * hn * hk, *T4 = T + 3 * hn * hk;
            const GemmOperand ops[7][2] = {
                {operand_u32(a, la), operand_u32(b, lb)},                               // M1 = A11 B'11
                {operand_u32(a + hk, la), operand_u32(b + hk, lb)},                     // M2 = A12 B'21
                {operand_u32(S4, hk), operand_u32(b + hn * lb + hk, lb)},               // M3 = S4 B'22
                {operand_u32(a + hm * la + hk, la), operand_u32(T4, hk)},               // M4 = A22 T4
                {operand_u32(S1, hk), operand_u32(T1, hk)},                             // M5 = S1 T1
                {operand_u32(S2, hk), operand_u32(T2, hk)},                             // M6 = S2 T2
                {operand_u32(S3, hk), operand_u32(T3, hk)}};                            // M7 = S3 T3
            for (int i = 0; i < 7; ++i)
                next.push_back(Prob{ops[i][0], ops[i][1], L.m_out + ((long long)q * 7 + i) * hm * hn, hn});
        }
        L.parents = std::move(cur);
        levels.push_back(std::move(L));
        cur = std::move(next);
        cm /= 2;
        cn /= 2;
        ck_ /= 2;
    }
    // base products: one grouped launch (outputs are either C itself or a level's contiguous M batch)
    std::vector<GemmOperand> ea, eb;
    for (auto& pr : cur) {
        ea.push_back(pr.a);
        eb.push_back(pr.b);
    }
    if (levels.empty()) {
        for (size_t q = 0; q < cur.size(); ++q) gemm_batch_dev(p, cm, cn, ck_, {ea[q]}, {eb[q]}, cur[q].c, cur[q].ldc, 0, s);
    } else
        gemm_batch_dev(p, cm, cn, ck_, ea, eb, levels.back().m_out, (long long)cn, (long long)cm * cn, s);
    // post-additions, deepest level first
    for (size_t l = levels.size(); l-- > 0;) {
        Level& L = levels[l];
        for (size_t q = 0; q < L.parents.size(); ++q) {
            const Prob& pr = L.parents[q];
            ck(launch_wino_post(L.m_out + (long long)q * 7 * L.hm * L.hn, L.hm * L.hn, L.hn, (int)L.hm, (int)L.hn, pp,
                                pr.c, pr.ldc, s),
               "winograd post");
        }
    }
    ck(cudaStreamSynchronize(s), "sync");
}

void wino_gemm_dev(uint64_t p, const uint32_t* A, long long lda, size_t m, const uint32_t* B, long long ldb, size_t n,
                   size_t k, uint32_t* C, long long ldc, fsyrk_b200_policy pol, cudaStream_t s) {
    wino_gemm_multi(p, {WinoProblem{A, lda, B, ldb, C, ldc}}, m, n, k, pol, s);
}

// Core device call: everything resident on the device.
void run_dev(uint64_t p, uint32_t alpha, const uint64_t* a_dev, size_t n, size_t k, size_t lda, const ColXform* xf,
             uint32_t beta, uint64_t* c_dev, size_t ldc, fsyrk_b200_policy pol, bool mirror, cudaStream_t s,
             fsyrk_b200_opcount* ops, int rank = 0, int nranks = 1) {
    validate_field(p);
    validate_policy(pol);
    validate_shapes(n, k, lda, ldc);
    require_device();
    if (n == 0) return;
    const int kbar = xf ? (int)xf->map.size() : (int)k;
    if (nranks > 1 && mirror) fail(FSYRK_B200_EINVAL, "mirror_output needs the whole C (not available per rank)");
    const std::shared_ptr<Plan> plan_ref = get_plan(p, (int)n, (int)k, kbar, pol, xf != nullptr, rank, nranks);
    Plan* plan = plan_ref.get();
    std::lock_guard<std::mutex> use(plan->use_mu);
    // Calls that share a plan share its arena: wait for the previous call's last kernel -- unless
    // that call ran on this very stream (stream order already serialises them; the wait would only
    // put a semaphore command in front of the first kernel).  Stream ids are unique for the
    // life of the process, handles are not.
    unsigned long long sid = 0;
    const bool have_sid = cudaStreamGetId(s, &sid) == cudaSuccess;
    if (!have_sid) cudaGetLastError();
    if (!plan->ev_done) ck(cudaEventCreateWithFlags(&plan->ev_done, cudaEventDisableTiming), "event");
    else if (g_always_wait || !(have_sid && plan->last_sid_valid && plan->last_sid == sid))
        ck(cudaStreamWaitEvent(s, plan->ev_done, 0), "wait for the plan's previous call");
    plan->last_sid = sid;
    plan->last_sid_valid = have_sid;
    if (xf) {
        auto same = [](const std::vector<ColMap>& x, const std::vector<ColMap>& y) {
            return x.size() == y.size() && std::memcmp(x.data(), y.data(), x.size() * sizeof(ColMap)) == 0;
        };
        if (!same(xf->map, plan->colmap_uploaded)) {
            // pageable source: the copy is staged before returning, so the host vector may change after
            ck(cudaMemcpyAsync(plan->dev_colmap, xf->map.data(), xf->map.size() * sizeof(ColMap),
                               cudaMemcpyHostToDevice, s),
               "upload colmap");
            plan->colmap_uploaded = xf->map;
        }
    }
    plan->execute(a_dev, (long long)lda, c_dev, (long long)ldc, alpha, beta, mirror, s);
    ck(cudaEventRecord(plan->ev_done, s), "event record");
    if (ops && rank == 0) add_tally(ops, ref_tally(p, n, (size_t)kbar, pol, alpha, beta, xf));
}

// Host call: the caller's A (and Low(C_in) when accumulating) cross PCIe through host_io
// (uint32 on the wire, narrowed / widened by host threads), the device computes, Low(C) comes
// back the same way.  Only Low(C) is moved (the strict upper triangle is scratch,
// fast_syrk.hpp:271-273); with beta = 0 the strict upper parts of the diagonal 256-row blocks
// are cleared, the rest of the strict upper triangle is left as the caller had it.
//
// Accumulating into pinned C (FSYRK_B200_HOSTIO=auto|duplex): the uint64 row blocks of C_in
// and of the result move unnarrowed but at the same time in both PCIe directions -- the device
// computes alpha X into a side buffer while C_in streams in, then per chunk of row blocks
// combines beta C_in + alpha X and sends the chunk back while later chunks still arrive.
enum class IoMode { Auto, Narrow, Duplex };
IoMode io_mode() {
    static const IoMode m = [] {
        const char* e = getenv("FSYRK_B200_HOSTIO");
        if (!e) return IoMode::Auto;
        if (!strcmp(e, "narrow")) return IoMode::Narrow;
        if (!strcmp(e, "duplex")) return IoMode::Duplex;
        return IoMode::Auto;
    }();
    return m;
}

struct IoStreams {
    cudaStream_t main = nullptr, cin = nullptr, cout = nullptr;
    cudaEvent_t a_done = nullptr;
    std::vector<cudaEvent_t> in_ev, fin_ev;
    void init() {
        if (main) return;
        ck(cudaStreamCreateWithFlags(&main, cudaStreamNonBlocking), "stream");
        ck(cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking), "stream");
        ck(cudaStreamCreateWithFlags(&cout, cudaStreamNonBlocking), "stream");
        ck(cudaEventCreateWithFlags(&a_done, cudaEventDisableTiming), "event");
    }
    void events(size_t n) {
        while (in_ev.size() < n) {
            cudaEvent_t a, b;
            ck(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "event");
            ck(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "event");
            in_ev.push_back(a);
            fin_ev.push_back(b);
        }
    }
};
struct DevStage {
    DevBuf a, c, x;        // caller's A / C (uint64 rows), alpha X of the duplex path
    DevBuf a32, sendb, recvb, pairs;  // multi-GPU: A residues, packed shares, pair lists
    IoStreams io;
};
DevStage& stage() { return per_device<DevStage>(); }

void run_host(uint64_t p, uint64_t alpha, const uint64_t* a, size_t n, size_t k, size_t lda, const ColXform* xf,
              uint64_t beta, uint64_t* c, size_t ldc, fsyrk_b200_policy pol, bool mirror, fsyrk_b200_opcount* ops) {
    validate_field(p);
    validate_policy(pol);
    validate_shapes(n, k, lda, ldc);
    g_transfer[0] = g_transfer[1] = 0;
    if (ranges_overlap(a, span_bytes(n, k, lda), c, span_bytes(n, n, ldc)))
        fail(FSYRK_B200_EINVAL, "syrk_fast: C must not alias A");
    require_device();
    if (n == 0) return;
    TallyOnSuccess tally{ops, ops ? ref_tally(p, n, xf ? xf->map.size() : k, pol, alpha, beta, xf) : refops::Tally{}};
    if ((k > 0 && hio::is_device(a)) || hio::is_device(c))
        fail(FSYRK_B200_EINVAL, "host entry point called with device memory (use fsyrk_b200_syrk_dev)");
    std::lock_guard<std::mutex> lk(g_stage_mu);
    DevStage& st = stage();
    IoStreams& g_io = st.io;
    g_io.init();
    const size_t abytes = n * std::max<size_t>(k, 1) * 8, cbytes = n * n * 8;
    st.a.ensure(abytes);
    st.c.ensure(cbytes);
    uint64_t* da = static_cast<uint64_t*>(st.a.ptr);
    uint64_t* dc = static_cast<uint64_t*>(st.c.ptr);
    cudaStream_t s = g_io.main;
    uint64_t h2d = 0, d2h = 0;
    static const bool io_trace = getenv("FSYRK_B200_IO_TRACE") != nullptr;
    auto tnow = [] {
        return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    double tr[4] = {tnow(), 0, 0, 0};
    hio::g_io_stats = hio::IoStats{};
    const int bits = hio::transfer_bits(p);
    const size_t lda_dev = k == 0 ? 1 : k;
    const bool need_c = (beta % p) != 0;
    // auto: duplex for pinned C unless residues pack to 16 bits or less (then the packed path
    // moves 4x fewer PCIe bytes than the raw duplex and wins, profiles/r01/hostio.txt)
    const bool duplex = need_c && !mirror && io_mode() != IoMode::Narrow &&
                        (io_mode() == IoMode::Duplex || (hio::is_pinned(c) && bits > 16));
    // duplex: chunks of whole kTriRows-row blocks of C, ~32 MB each
    std::vector<std::pair<size_t, size_t>> chunks;
    auto blocks = [&](size_t r0, size_t r1, bool in) {
        for (size_t b0 = r0; b0 < r1; b0 += kTriRows) {
            const size_t b1 = std::min(r1, b0 + kTriRows);
            if (in)
                ck(cudaMemcpy2DAsync(dc + b0 * n, n * 8, c + b0 * ldc, ldc * 8, b1 * 8, b1 - b0,
                                     cudaMemcpyHostToDevice, g_io.cin),
                   "H2D C");
            else
                ck(cudaMemcpy2DAsync(c + b0 * ldc, ldc * 8, dc + b0 * n, n * 8, b1 * 8, b1 - b0,
                                     cudaMemcpyDeviceToHost, g_io.cout),
                   "D2H C");
            (in ? h2d : d2h) += (b1 - b0) * b1 * 8;
        }
    };
    auto queue_cin = [&] {
        for (size_t q = 0; q < chunks.size(); ++q) {
            blocks(chunks[q].first, chunks[q].second, true);
            ck(cudaEventRecord(g_io.in_ev[q], g_io.cin), "event");
        }
    };
    // C_in follows A on the wire (A gates the compute); FSYRK_B200_CIN_EARLY=1 queues it first,
    // sharing the H2D direction with A's narrowed chunks
    static const bool cin_early = getenv("FSYRK_B200_CIN_EARLY") != nullptr;
    if (duplex) {
        for (size_t r0 = 0; r0 < n;) {
            size_t r1 = r0, elems = 0;
            while (r1 < n && (elems == 0 || elems < (size_t(4) << 20))) {
                const size_t b1 = std::min(n, r1 + kTriRows);
                elems += (b1 - r1) * b1;
                r1 = b1;
            }
            chunks.push_back({r0, r1});
            r0 = r1;
        }
        g_io.events(chunks.size());
        if (cin_early) queue_cin();
    }
    if (k > 0) ck(hio::upload(a, lda, hio::Region{n, k, false}, da, k, bits, s, &h2d), "H2D A");
    if (io_trace) {
        ck(cudaStreamSynchronize(s), "sync");
        tr[1] = tnow();
    }
    if (!duplex) {
        if (need_c) ck(hio::upload(c, ldc, hio::Region{n, n, true}, dc, n, bits, s, &h2d), "H2D C");
        run_dev(p, (uint32_t)(alpha % p), da, n, k, lda_dev, xf, (uint32_t)(beta % p), dc, n, pol, mirror, s, nullptr);
        if (io_trace) {
            ck(cudaStreamSynchronize(s), "sync");
            tr[2] = tnow();
        }
        ck(hio::download(dc, n, hio::Region{n, n, !mirror}, c, ldc, (need_c || mirror) ? 0 : kTriRows, bits, s, &d2h),
           "D2H C");
    } else {
        st.x.ensure(cbytes);
        uint64_t* dx = static_cast<uint64_t*>(st.x.ptr);
        if (!cin_early) {
            ck(cudaEventRecord(g_io.a_done, s), "event");
            ck(cudaStreamWaitEvent(g_io.cin, g_io.a_done, 0), "wait");
            queue_cin();
        }
        run_dev(p, (uint32_t)(alpha % p), da, n, k, lda_dev, xf, 0, dx, n, pol, false, s, nullptr);
        if (io_trace) {
            ck(cudaStreamSynchronize(s), "sync");
            tr[2] = tnow();
        }
        const ModP m = make_modp((uint32_t)p);
        for (size_t q = 0; q < chunks.size(); ++q) {
            ck(cudaStreamWaitEvent(s, g_io.in_ev[q], 0), "wait");
            ck(hio::launch_acc_combine(dx, (long long)n, dc, (long long)n, (int)chunks[q].first, (int)chunks[q].second,
                                       m, (uint32_t)(beta % p), s),
               "acc_combine");
            ck(cudaEventRecord(g_io.fin_ev[q], s), "event");
            ck(cudaStreamWaitEvent(g_io.cout, g_io.fin_ev[q], 0), "wait");
            blocks(chunks[q].first, chunks[q].second, false);
        }
        ck(cudaStreamSynchronize(g_io.cout), "sync");
    }
    ck(cudaStreamSynchronize(s), "sync");
    g_transfer[0] = h2d;
    g_transfer[1] = d2h;
    if (io_trace) {
        tr[3] = tnow();
        fprintf(stderr, "[io] n=%zu k=%zu %s: A %.3f ms, C_in+compute %.3f ms, out %.3f ms, total %.3f ms; pool %.3f ms, slot waits %.3f ms, threads %d\n",
                n, k, duplex ? "duplex" : "narrow", (tr[1] - tr[0]) * 1e3, (tr[2] - tr[1]) * 1e3,
                (tr[3] - tr[2]) * 1e3, (tr[3] - tr[0]) * 1e3, hio::g_io_stats.host * 1e3, hio::g_io_stats.wait * 1e3,
                hio::host_threads());
    }
}

// Products over F_{p^2} = F_p[x] / (x^2 - ns), ns the least non-residue (the reference's
// QuadExtField, proj/include/fsyrk/fields.hpp:148-212).  With A = X + x Y:
//   herk (conj):  A conj(A)^T = (X X^T - ns Y Y^T) + x (Y X^T - X Y^T)
//   syrk:         A A^T       = (X X^T + ns Y Y^T) + x (Y X^T + X Y^T)
// The real part is the syrkd of [X | Y] with D = (1, .., 1, -+ns, .., -+ns) on the device path
// (recursion, digit-plane products); the imaginary part is G +- G^T with G = Y X^T from one
// tensor-core product.  Exact, so equal to the reference's herk_fast / syrk_fast over F_{p^2}
// (fast_syrk.hpp:305-320) for any policy.  a, c: (a, b) uint64 pairs, lda / ldc in pairs.
void run_fp2(uint64_t p, const uint64_t* a, size_t n, size_t k, size_t lda, uint64_t* c, size_t ldc,
             fsyrk_b200_policy pol, bool mirror, bool conj, fsyrk_b200_opcount* ops) {
    validate_field(p);
    validate_policy(pol);
    if (p == 2) fail(FSYRK_B200_EINVAL, "QuadExtField requires an odd prime");
    validate_shapes(n, 2 * k, 2 * lda, 2 * ldc);
    if (ranges_overlap(a, span_bytes(n, 2 * k, 2 * lda), c, span_bytes(n, 2 * n, 2 * ldc)))
        fail(FSYRK_B200_EINVAL, "syrk_fast: C must not alias A");
    require_device();
    if (n == 0) return;
    TallyOnSuccess tally{ops, ops ? ref_tally_fp2(n, k, pol) : refops::Tally{}};
    host::Field f{p};
    const uint64_t ns = f.lqnr();
    std::lock_guard<std::mutex> lk(g_stage_mu);
    const size_t kk = std::max<size_t>(k, 1);
    DevBuf dA, dX, dY, dR, dG, dC;
    dA.ensure(n * 2 * kk * 8);
    dX.ensure(n * kk * 8);
    dY.ensure(n * kk * 8);
    dR.ensure(n * n * 8);
    dG.ensure(n * n * 4);
    dC.ensure(n * n * 16);
    cudaStream_t s = 0;
    auto* A = static_cast<uint64_t*>(dA.ptr);
    auto* R = static_cast<uint64_t*>(dR.ptr);
    auto* G = static_cast<uint32_t*>(dG.ptr);
    if (k == 0) {
        ck(cudaMemsetAsync(dR.ptr, 0, n * n * 8, s), "memset");
        ck(cudaMemsetAsync(dG.ptr, 0, n * n * 4, s), "memset");
    } else {
        ck(cudaMemcpy2DAsync(A, 2 * k * 8, a, 2 * lda * 8, 2 * k * 8, n, cudaMemcpyHostToDevice, s), "H2D A");
        // real part: columns [a parts | b parts] scaled by (1 | -+ns) through syrkd's diagonal fold
        ColXform xf;
        for (size_t j = 0; j < 2 * k; ++j)
            xf.map.push_back(ColMap{{(int)(j < k ? 2 * j : 2 * (j - k) + 1), -1, -1, -1}, {1, 0, 0, 0}});
        std::vector<uint64_t> dbar(2 * k, 1);
        for (size_t j = k; j < 2 * k; ++j) dbar[j] = conj ? p - ns : ns;
        fold_diagonal(p, std::move(dbar), xf.map);
        run_dev(p, 1, A, n, 2 * k, 2 * k, &xf, 0, R, n, pol, false, s, nullptr);
        // imaginary part: G = Y X^T
        ck(launch_deinterleave(A, (long long)k, (int)n, (int)k, static_cast<uint64_t*>(dX.ptr),
                               static_cast<uint64_t*>(dY.ptr), s),
           "deinterleave");
        gemm_nt_dev(p, static_cast<uint64_t*>(dY.ptr), n, k, k, static_cast<uint64_t*>(dX.ptr), n, k, G, (long long)n,
                    s);
    }
    ck(launch_fp2_combine(R, (long long)n, G, (long long)n, (int)n, (uint32_t)p, conj ? 1 : 0, mirror ? 1 : 0,
                          static_cast<uint64_t*>(dC.ptr), (long long)n, s),
       "fp2 combine");
    ck(cudaMemcpy2DAsync(c, 2 * ldc * 8, dC.ptr, 2 * n * 8, 2 * n * 8, n, cudaMemcpyDeviceToHost, s), "D2H C");
    ck(cudaStreamSynchronize(s), "sync");
}


// ------------------------------------------------------------- multi-GPU
// one problem over several GPUs.  Rank 0 holds the caller's host A (and C);
// A crosses PCIe once (bit-packed, host_io) into rank 0, is reduced to uint32 residues and
// broadcast over NVLink by NCCL; every rank computes the top-level tile pairs it owns
// (partition_owners, Plan::create) with no data-path exchange; the owned 32 x 32 tiles of
// Low(C) come back to rank 0 as packed uint32 shares (ncclSend / ncclRecv, 4 bytes per entry
// instead of a reduce over the full uint64 C) and cross PCIe once.  Accumulating calls scatter
// the owned tiles of Low(C_in) the same way before the compute.
//
// NCCL is loaded at first use (dlopen of libnccl.so.2: the copy a host process such as
// PyTorch already loaded, else the system one), so the library itself has no link-time NCCL
// dependency and its version never conflicts with the caller's.
struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommInitAll) init_all = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            a.error = e ? e : "dlopen(libnccl.so.2) failed";
            return a;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && a.error.empty()) a.error = std::string("symbol ") + name + " missing";
        };
        sym(a.get_unique_id, "ncclGetUniqueId");
        sym(a.init_rank, "ncclCommInitRank");
        sym(a.init_all, "ncclCommInitAll");
        sym(a.destroy, "ncclCommDestroy");
        sym(a.broadcast, "ncclBroadcast");
        sym(a.send, "ncclSend");
        sym(a.recv, "ncclRecv");
        sym(a.group_start, "ncclGroupStart");
        sym(a.group_end, "ncclGroupEnd");
        sym(a.error_string, "ncclGetErrorString");
        return a;
    }();
    if (!api.error.empty()) fail(FSYRK_B200_ENCCL, "NCCL unavailable: " + api.error);
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(FSYRK_B200_ENCCL, std::string(what) + ": " + nccl().error_string(r));
}

// A communicator handle of the C ABI (fsyrk_b200_comm_init_rank).
struct Comm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1, dev = 0;
};

// One rank driven by this process.  comm == nullptr: loopback transport (several ranks of a
// single-process call on one device -- a test configuration: the shares move by device copies).
struct LocalRank {
    int dev = 0, rank = 0;
    ncclComm_t comm = nullptr;
};

// Device buffers of one rank (several loopback ranks may share a device).
struct RankBufs {
    DevBuf a64, a32, c64, sendb, recvb, pairs;
    cudaStream_t s = nullptr;
    cudaEvent_t ev = nullptr;
};
RankBufs& rank_bufs(int rank) {
    struct M {
        std::mutex mu;
        std::map<int, std::unique_ptr<RankBufs>> m;
    };
    M& mm = per_device<M>();
    std::lock_guard<std::mutex> lk(mm.mu);
    std::unique_ptr<RankBufs>& b = mm.m[rank];
    if (!b) {
        b.reset(new RankBufs);
        ck(cudaStreamCreateWithFlags(&b->s, cudaStreamNonBlocking), "stream");
        ck(cudaEventCreateWithFlags(&b->ev, cudaEventDisableTiming), "event");
    }
    return *b;
}

// The 32 x 32 tile pairs of the root post-addition owned by `rank` (Plan::create root_pairs).
std::vector<int2> owned_pairs(const Plan& pl, int rank) {
    std::vector<int2> out;
    const int h = pl.nodes[0].h, T = (h + 31) / 32;
    for (int I = 0; I < T; ++I)
        for (int J = 0; J <= I; ++J) {
            const int bi = I * 32 / pl.kPartBlock, bj = J * 32 / pl.kPartBlock;
            if (pl.owner[(size_t)bi * pl.part_nb + bj] == rank) out.push_back(make_int2(I, J));
        }
    return out;
}

constexpr size_t kShareWords = 4 * 1024;  // uint32 words of one tile pair's share

void mgpu_run(const std::vector<LocalRank>& loc, int nranks, uint64_t p, uint64_t alpha, const uint64_t* a, size_t n,
              size_t k, size_t lda, const ColXform* xf, uint64_t beta, uint64_t* c, size_t ldc,
              fsyrk_b200_policy pol, bool mirror, fsyrk_b200_opcount* ops) {
    validate_field(p);
    validate_policy(pol);
    validate_shapes(n, k, lda, ldc);
    const LocalRank* r0 = nullptr;
    for (const LocalRank& lr : loc)
        if (lr.rank == 0) r0 = &lr;
    if (r0) {
        if (ranges_overlap(a, span_bytes(n, k, lda), c, span_bytes(n, n, ldc)))
            fail(FSYRK_B200_EINVAL, "syrk_fast: C must not alias A");
        if ((n > 0 && k > 0 && !a) || (n > 0 && !c)) fail(FSYRK_B200_EINVAL, "syrk_mgpu: rank 0 needs host A and C");
    }
    const int saved = current_device();
    struct DevGuard {
        int d;
        ~DevGuard() { cudaSetDevice(d); }
    } guard{saved};
    if (n == 0) return;
    const int kbar = xf ? (int)xf->map.size() : (int)k;
    const bool need_c = (beta % p) != 0;
    // plans first: every rank's plan is built from the same deterministic partition
    struct R {
        LocalRank lr;
        RankBufs* b;
        std::shared_ptr<Plan> plan;
    };
    std::vector<R> rs;
    for (const LocalRank& lr : loc) {
        ck(cudaSetDevice(lr.dev), "cudaSetDevice");
        require_device();
        rs.push_back(R{lr, &rank_bufs(lr.rank), k > 0 ? get_plan(p, (int)n, (int)k, kbar, pol, xf != nullptr, lr.rank,
                                                                 nranks)
                                                      : nullptr});
    }
    const bool part = k > 0 && nranks > 1 && rs[0].plan->partitioned;
    if (!part) {  // not partitionable (or one rank): rank 0 runs the single-GPU host path
        if (r0) {
            ck(cudaSetDevice(r0->dev), "cudaSetDevice");
            run_host(p, alpha, a, n, k, lda, xf, beta, c, ldc, pol, mirror, ops);
        }
        return;
    }
    std::lock_guard<std::mutex> lk(g_stage_mu);  // rank 0's host staging
    g_transfer[0] = g_transfer[1] = 0;
    if (r0 && ((k > 0 && hio::is_device(a)) || hio::is_device(c)))
        fail(FSYRK_B200_EINVAL, "host entry point called with device memory (use fsyrk_b200_syrk_part_dev)");
    const Plan& pl0 = *rs[0].plan;
    const int h = pl0.nodes[0].h;
    std::vector<std::vector<int2>> pairs(nranks);
    for (int r = 0; r < nranks; ++r) pairs[r] = owned_pairs(pl0, r);
    std::vector<size_t> roff(nranks + 1, 0);  // rank 0's receive offsets (words)
    for (int r = 0; r < nranks; ++r) roff[r + 1] = roff[r] + (r == 0 ? 0 : pairs[r].size() * kShareWords);
    const int bits = hio::transfer_bits(p);
    const bool loopback = loc.front().comm == nullptr;
    // ---- buffers; pair lists on the devices (rank 0: every rank's, concatenated)
    std::vector<int2> all_pairs;
    std::vector<size_t> poff(nranks + 1, 0);
    for (int r = 0; r < nranks; ++r) {
        all_pairs.insert(all_pairs.end(), pairs[r].begin(), pairs[r].end());
        poff[r + 1] = all_pairs.size();
    }
    for (R& x : rs) {
        ck(cudaSetDevice(x.lr.dev), "cudaSetDevice");
        RankBufs& b = *x.b;
        b.a64.ensure(n * k * 8);
        b.a32.ensure(n * k * 4);
        b.c64.ensure(n * n * 8);
        b.sendb.ensure(std::max<size_t>(1, pairs[x.lr.rank].size()) * kShareWords * 4);
        if (x.lr.rank == 0) b.recvb.ensure(std::max<size_t>(1, roff[nranks]) * 4);
        b.pairs.ensure(std::max<size_t>(1, all_pairs.size()) * sizeof(int2));
        ck(cudaMemcpyAsync(b.pairs.ptr, all_pairs.data(), all_pairs.size() * sizeof(int2), cudaMemcpyHostToDevice, b.s),
           "upload pair lists");
    }
    auto pairs_dev = [&](const R& x, int r) { return static_cast<int2*>(x.b->pairs.ptr) + poff[r]; };
    auto u64 = [](DevBuf& d) { return static_cast<uint64_t*>(d.ptr); };
    auto u32 = [](DevBuf& d) { return static_cast<uint32_t*>(d.ptr); };
    R* x0 = nullptr;
    for (R& x : rs)
        if (x.lr.rank == 0) x0 = &x;
    // loopback transport: copies between the ranks' buffers, ordered by events
    auto copy_from = [&](R& dst, void* to, R& src, const void* from, size_t bytes) {
        ck(cudaSetDevice(src.lr.dev), "cudaSetDevice");
        ck(cudaEventRecord(src.b->ev, src.b->s), "event");
        ck(cudaSetDevice(dst.lr.dev), "cudaSetDevice");
        ck(cudaStreamWaitEvent(dst.b->s, src.b->ev, 0), "wait");
        ck(cudaMemcpyAsync(to, from, bytes, cudaMemcpyDefault, dst.b->s), "loopback copy");
    };
    uint64_t h2d = 0, d2h = 0;
    // 1. rank 0: A (and Low(C_in)) from the host; A reduced to uint32 residues for the broadcast
    if (x0) {
        ck(cudaSetDevice(x0->lr.dev), "cudaSetDevice");
        ck(hio::upload(a, lda, hio::Region{n, k, false}, u64(x0->b->a64), k, bits, x0->b->s, &h2d), "H2D A");
        ck(launch_convert_in(u64(x0->b->a64), (long long)k, (int)n, (int)k, (int)k, nullptr, (uint32_t)p,
                             u32(x0->b->a32), (long long)k, x0->b->s),
           "narrow A");
        if (need_c) ck(hio::upload(c, ldc, hio::Region{n, n, true}, u64(x0->b->c64), n, bits, x0->b->s, &h2d), "H2D C");
    }
    // 2. broadcast A; the other ranks widen it back to the uint64 layout the plan reads
    if (loopback) {
        for (R& x : rs)
            if (x.lr.rank != 0) copy_from(x, x.b->a32.ptr, *x0, x0->b->a32.ptr, n * k * 4);
    } else {
        const NcclApi& nc = nccl();
        nck(nc.group_start(), "ncclGroupStart");
        for (R& x : rs) {
            ck(cudaSetDevice(x.lr.dev), "cudaSetDevice");
            nck(nc.broadcast(x.b->a32.ptr, x.b->a32.ptr, n * k, ncclUint32, 0, x.lr.comm, x.b->s), "ncclBroadcast(A)");
        }
        nck(nc.group_end(), "ncclGroupEnd");
    }
    for (R& x : rs) {
        if (x.lr.rank == 0) continue;
        ck(cudaSetDevice(x.lr.dev), "cudaSetDevice");
        ck(launch_u32_to_u64(u32(x.b->a32), (long long)k, (int)n, (int)k, u64(x.b->a64), (long long)k, x.b->s),
           "widen A");
    }
    // 2b. accumulate: rank 0 scatters the owned tiles of Low(C_in)
    if (need_c) {
        if (x0) {
            ck(cudaSetDevice(x0->lr.dev), "cudaSetDevice");
            for (int r = 1; r < nranks; ++r)
                ck(launch_share_pack(u64(x0->b->c64), (long long)n, h, pairs_dev(*x0, r), (int)pairs[r].size(),
                                     u32(x0->b->recvb) + roff[r], x0->b->s),
                   "pack C_in share");
        }
        if (loopback) {
            for (R& x : rs)
                if (x.lr.rank != 0)
                    copy_from(x, x.b->sendb.ptr, *x0, u32(x0->b->recvb) + roff[x.lr.rank],
                              pairs[x.lr.rank].size() * kShareWords * 4);
        } else {
            const NcclApi& nc = nccl();
            nck(nc.group_start(), "ncclGroupStart");
            for (R& x : rs) {
                ck(cudaSetDevice(x.lr.dev), "cudaSetDevice");
                if (x.lr.rank == 0) {
                    for (int r = 1; r < nranks; ++r)
                        if (!pairs[r].empty())
                            nck(nc.send(u32(x.b->recvb) + roff[r], pairs[r].size() * kShareWords, ncclUint32, r,
                                        x.lr.comm, x.b->s),
                                "ncclSend(C_in)");
                } else if (!pairs[x.lr.rank].empty()) {
                    nck(nc.recv(x.b->sendb.ptr, pairs[x.lr.rank].size() * kShareWords, ncclUint32, 0, x.lr.comm,
                                x.b->s),
                        "ncclRecv(C_in)");
                }
            }
            nck(nc.group_end(), "ncclGroupEnd");
        }
        for (R& x : rs) {
            if (x.lr.rank == 0) continue;
            ck(cudaSetDevice(x.lr.dev), "cudaSetDevice");
            ck(launch_share_unpack(u32(x.b->sendb), h, pairs_dev(x, x.lr.rank), (int)pairs[x.lr.rank].size(),
                                   u64(x.b->c64), (long long)n, x.b->s),
               "unpack C_in share");
        }
    }
    // 3. every rank computes its share (no data-path exchange)
    for (R& x : rs) {
        ck(cudaSetDevice(x.lr.dev), "cudaSetDevice");
        run_dev(p, (uint32_t)(alpha % p), u64(x.b->a64), n, k, k, xf, (uint32_t)(beta % p), u64(x.b->c64), n, pol,
                false, x.b->s, x.lr.rank == 0 ? ops : nullptr, x.lr.rank, nranks);
    }
    // 4. gather the shares into rank 0's C
    for (R& x : rs) {
        if (x.lr.rank == 0) continue;
        ck(cudaSetDevice(x.lr.dev), "cudaSetDevice");
        ck(launch_share_pack(u64(x.b->c64), (long long)n, h, pairs_dev(x, x.lr.rank), (int)pairs[x.lr.rank].size(),
                             u32(x.b->sendb), x.b->s),
           "pack share");
    }
    if (loopback) {
        for (R& x : rs)
            if (x.lr.rank != 0)
                copy_from(*x0, u32(x0->b->recvb) + roff[x.lr.rank], x, x.b->sendb.ptr,
                          pairs[x.lr.rank].size() * kShareWords * 4);
    } else {
        const NcclApi& nc = nccl();
        nck(nc.group_start(), "ncclGroupStart");
        for (R& x : rs) {
            ck(cudaSetDevice(x.lr.dev), "cudaSetDevice");
            if (x.lr.rank == 0) {
                for (int r = 1; r < nranks; ++r)
                    if (!pairs[r].empty())
                        nck(nc.recv(u32(x.b->recvb) + roff[r], pairs[r].size() * kShareWords, ncclUint32, r, x.lr.comm,
                                    x.b->s),
                            "ncclRecv(share)");
            } else if (!pairs[x.lr.rank].empty()) {
                nck(nc.send(x.b->sendb.ptr, pairs[x.lr.rank].size() * kShareWords, ncclUint32, 0, x.lr.comm, x.b->s),
                    "ncclSend(share)");
            }
        }
        nck(nc.group_end(), "ncclGroupEnd");
    }
    // 5. rank 0: unpack, optional mirror, Low(C) (or all of C) back to the host
    if (x0) {
        ck(cudaSetDevice(x0->lr.dev), "cudaSetDevice");
        for (int r = 1; r < nranks; ++r)
            ck(launch_share_unpack(u32(x0->b->recvb) + roff[r], h, pairs_dev(*x0, r), (int)pairs[r].size(),
                                   u64(x0->b->c64), (long long)n, x0->b->s),
               "unpack share");
        if (mirror) ck(launch_mirror(u64(x0->b->c64), (long long)n, (int)n, x0->b->s), "mirror");
        ck(hio::download(u64(x0->b->c64), n, hio::Region{n, n, !mirror}, c, ldc, (need_c || mirror) ? 0 : kTriRows,
                         bits, x0->b->s, &d2h),
           "D2H C");
    }
    for (R& x : rs) {
        ck(cudaSetDevice(x.lr.dev), "cudaSetDevice");
        ck(cudaStreamSynchronize(x.b->s), "sync");
    }
    g_transfer[0] = h2d;
    g_transfer[1] = d2h;
}

// Single-process communicators over distinct devices (ncclCommInitAll), cached per device list.
std::vector<ncclComm_t> comms_for(const std::vector<int>& devs) {
    static std::mutex mu;
    static std::map<std::vector<int>, std::vector<ncclComm_t>> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(devs);
    if (it != cache.end()) return it->second;
    std::vector<ncclComm_t> comms(devs.size(), nullptr);
    nck(nccl().init_all(comms.data(), (int)devs.size(), devs.data()), "ncclCommInitAll");
    cache[devs] = comms;
    return comms;
}

}  // namespace

}  // namespace fsyrk_b200

using namespace fsyrk_b200;

extern "C" {

const char* fsyrk_b200_last_error(void) { return g_last_error.c_str(); }
int fsyrk_b200_abi_version(void) { return FSYRK_B200_ABI_VERSION; }
int fsyrk_b200_device_available(void) { return device_ok(); }

int fsyrk_b200_skew_orthogonal(uint64_t p, size_t dim, fsyrk_b200_skew* skew) {
    return guarded([&] {
        validate_field(p);
        host::Skew y = host::skew_orthogonal(host::Field{p});
        if (y.form == 1 && dim % 2 != 0)
            fail(FSYRK_B200_EPARITY, "pair-form skew-orthogonal matrix requires an even dimension");
        if (skew) *skew = fsyrk_b200_skew{y.form, y.a, y.b, y.ycost};
    });
}

int fsyrk_b200_make_syrk_plan(uint64_t p, fsyrk_b200_policy policy, int mirror_output, fsyrk_b200_skew* skew) {
    (void)mirror_output;
    return guarded([&] {
        validate_policy(policy);
        validate_field(p);
        host::Skew y = host::skew_orthogonal(host::Field{p});
        if (skew) *skew = fsyrk_b200_skew{y.form, y.a, y.b, y.ycost};
    });
}

int fsyrk_b200_sum_of_squares(uint64_t p, uint64_t k, uint64_t* a, uint64_t* b) {
    return guarded([&] {
        validate_field(p);
        if (p == 2) fail(FSYRK_B200_EDOMAIN, "sum-of-squares decomposition requires odd p");
        auto ab = host::Field{p}.sum_of_squares(k % p);
        if (a) *a = ab.first;
        if (b) *b = ab.second;
    });
}

int fsyrk_b200_nrsyf(uint64_t p, uint64_t alpha, uint64_t beta, uint64_t y[4]) {
    return guarded([&] {
        validate_field(p);
        if (p == 2) fail(FSYRK_B200_EDOMAIN, "nrsyf requires an odd prime");
        std::array<uint64_t, 4> v;
        if (!host::nrsyf(host::Field{p}, alpha % p, beta % p, v))
            fail(FSYRK_B200_ENONRES, "nrsyf: argument is not a non-residue");
        if (y) std::copy(v.begin(), v.end(), y);
    });
}

int fsyrk_b200_random_matrix(uint64_t p, size_t rows, size_t cols, uint64_t seed, uint64_t* out, size_t ld) {
    return guarded([&] {
        validate_field(p);
        if (ld < cols) fail(FSYRK_B200_EDIMENSION, "random_matrix: stride smaller than row");
        std::mt19937_64 rng(seed);
        std::uniform_int_distribution<uint64_t> dist(0, p - 1);
        for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < cols; ++j) out[i * ld + j] = dist(rng);
    });
}

int fsyrk_b200_syrk_fast_into(uint64_t p, const uint64_t* a, size_t n, size_t k, size_t lda, uint64_t* c, size_t ldc,
                              fsyrk_b200_policy policy, int mirror_output, fsyrk_b200_opcount* ops) {
    return guarded([&] { run_host(p, 1, a, n, k, lda, nullptr, 0, c, ldc, policy, mirror_output != 0, ops); });
}

int fsyrk_b200_syrk_fast_acc(uint64_t p, uint64_t alpha, const uint64_t* a, size_t n, size_t k, size_t lda,
                             uint64_t beta, uint64_t* c, size_t ldc, fsyrk_b200_policy policy, int mirror_output,
                             fsyrk_b200_opcount* ops) {
    return guarded([&] { run_host(p, alpha, a, n, k, lda, nullptr, beta, c, ldc, policy, mirror_output != 0, ops); });
}

int fsyrk_b200_syrkd(uint64_t p, uint64_t alpha, const uint64_t* a, size_t n, size_t k, size_t lda, const uint64_t* d,
                     uint64_t beta, uint64_t* c, size_t ldc, fsyrk_b200_policy policy, int mirror_output,
                     fsyrk_b200_opcount* ops) {
    return guarded([&] {
        if (!d && k > 0) fail(FSYRK_B200_EDIMENSION, "syrkd: diagonal length must match column count");
        validate_field(p);
        const ColXform xf = xform_diag(p, d, d ? k : 0);
        run_host(p, alpha, a, n, k, lda, &xf, beta, c, ldc, policy, mirror_output != 0, ops);
    });
}

int fsyrk_b200_set_workspace_limit(uint64_t bytes) {
    g_ws_limit.store(bytes);
    return FSYRK_B200_OK;
}

int fsyrk_b200_set_winograd_min(uint64_t min_dim) {
    g_wino_min.store(min_dim);
    return FSYRK_B200_OK;
}

int fsyrk_b200_set_low_memory(int enable) {
    g_force_lowmem.store(enable != 0);
    return FSYRK_B200_OK;
}

int fsyrk_b200_workspace_bytes(uint64_t p, size_t n, size_t k, fsyrk_b200_policy policy, int lowmem, uint64_t* arena,
                               uint64_t* host_call) {
    return guarded([&] {
        validate_field(p);
        validate_policy(policy);
        validate_shapes(n, k, k, n);
        uint64_t bytes = 0;
        if (n > 0 && k > 0) bytes = dry_arena(p, (int)n, (int)k, (int)k, policy, false, 0, 1, lowmem != 0);
        if (arena) *arena = bytes;
        // host entry points also stage A and C on the device as uint64 rows
        if (host_call) *host_call = bytes + (uint64_t)n * k * 8 + (uint64_t)n * n * 8;
    });
}

int fsyrk_b200_opcount_syrk(uint64_t p, size_t n, size_t k, uint64_t alpha, uint64_t beta, fsyrk_b200_policy policy,
                            fsyrk_b200_opcount* ops) {
    return guarded([&] {
        validate_field(p);
        validate_policy(policy);
        if (!ops) fail(FSYRK_B200_EINVAL, "null opcount");
        add_tally(ops, ref_tally(p, n, k, policy, alpha, beta, nullptr));
    });
}

int fsyrk_b200_opcount_syrkd(uint64_t p, size_t n, size_t k, const uint64_t* d, uint64_t alpha, uint64_t beta,
                             fsyrk_b200_policy policy, fsyrk_b200_opcount* ops) {
    return guarded([&] {
        validate_field(p);
        validate_policy(policy);
        if (!ops) fail(FSYRK_B200_EINVAL, "null opcount");
        if (!d && k > 0) fail(FSYRK_B200_EDIMENSION, "syrkd: diagonal length must match column count");
        const ColXform xf = xform_diag(p, d, d ? k : 0);
        add_tally(ops, ref_tally(p, n, xf.map.size(), policy, alpha, beta, &xf));
    });
}

int fsyrk_b200_opcount_syrkbd(uint64_t p, size_t n, const fsyrk_b200_block* blocks, size_t nblocks, uint64_t alpha,
                              uint64_t beta, fsyrk_b200_policy policy, fsyrk_b200_opcount* ops) {
    return guarded([&] {
        validate_field(p);
        validate_policy(policy);
        if (!ops) fail(FSYRK_B200_EINVAL, "null opcount");
        if (!blocks && nblocks) fail(FSYRK_B200_EINVAL, "syrkbd: null block list");
        size_t k = 0;
        for (size_t i = 0; i < nblocks; ++i) k += blocks[i].two ? 2 : 1;
        const ColXform xf = xform_blocks(p, blocks, nblocks, k);
        add_tally(ops, ref_tally(p, n, xf.map.size(), policy, alpha, beta, &xf));
    });
}

int fsyrk_b200_opcount_fp2(uint64_t p, size_t n, size_t k, fsyrk_b200_policy policy, fsyrk_b200_opcount* ops) {
    return guarded([&] {
        validate_field(p);
        validate_policy(policy);
        if (p == 2) fail(FSYRK_B200_EINVAL, "QuadExtField requires an odd prime");
        if (!ops) fail(FSYRK_B200_EINVAL, "null opcount");
        add_tally(ops, ref_tally_fp2(n, k, policy));
    });
}

int fsyrk_b200_syrkbd(uint64_t p, uint64_t alpha, const uint64_t* a, size_t n, size_t k, size_t lda,
                      const fsyrk_b200_block* blocks, size_t nblocks, uint64_t beta, uint64_t* c, size_t ldc,
                      fsyrk_b200_policy policy, int mirror_output, fsyrk_b200_opcount* ops) {
    return guarded([&] {
        validate_field(p);
        if (!blocks && nblocks) fail(FSYRK_B200_EINVAL, "syrkbd: null block list");
        const ColXform xf = xform_blocks(p, blocks, nblocks, k);
        run_host(p, alpha, a, n, k, lda, &xf, beta, c, ldc, policy, mirror_output != 0, ops);
    });
}

int fsyrk_b200_syrkbd_dev(uint64_t p, uint64_t alpha, const uint64_t* a_dev, size_t n, size_t k, size_t lda,
                          const fsyrk_b200_block* blocks, size_t nblocks, uint64_t beta, uint64_t* c_dev, size_t ldc,
                          fsyrk_b200_policy policy, int mirror_output, void* stream, fsyrk_b200_opcount* ops) {
    return guarded([&] {
        validate_field(p);
        if (!blocks && nblocks) fail(FSYRK_B200_EINVAL, "syrkbd: null block list");
        const ColXform xf = xform_blocks(p, blocks, nblocks, k);
        run_dev(p, (uint32_t)(alpha % p), a_dev, n, k, lda, &xf, (uint32_t)(beta % p), c_dev, ldc, policy,
                mirror_output != 0, static_cast<cudaStream_t>(stream), ops);
    });
}

int fsyrk_b200_syrk_dev(uint64_t p, uint64_t alpha, const uint64_t* a_dev, size_t n, size_t k, size_t lda,
                        const uint64_t* d_host, uint64_t beta, uint64_t* c_dev, size_t ldc, fsyrk_b200_policy policy,
                        int mirror_output, void* stream, fsyrk_b200_opcount* ops) {
    return guarded([&] {
        validate_field(p);
        ColXform xf;
        if (d_host) xf = xform_diag(p, d_host, k);
        run_dev(p, (uint32_t)(alpha % p), a_dev, n, k, lda, d_host ? &xf : nullptr, (uint32_t)(beta % p), c_dev, ldc,
                policy, mirror_output != 0, static_cast<cudaStream_t>(stream), ops);
    });
}

int fsyrk_b200_syrk_part_dev(uint64_t p, uint64_t alpha, const uint64_t* a_dev, size_t n, size_t k, size_t lda,
                             const uint64_t* d_host, uint64_t beta, uint64_t* c_dev, size_t ldc,
                             fsyrk_b200_policy policy, int rank, int nranks, void* stream, fsyrk_b200_opcount* ops) {
    return guarded([&] {
        validate_field(p);
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(FSYRK_B200_EINVAL, "rank out of range");
        ColXform xf;
        if (d_host) xf = xform_diag(p, d_host, k);
        run_dev(p, (uint32_t)(alpha % p), a_dev, n, k, lda, d_host ? &xf : nullptr, (uint32_t)(beta % p), c_dev, ldc,
                policy, false, static_cast<cudaStream_t>(stream), ops, rank, nranks);
    });
}

int fsyrk_b200_partition_owners(uint64_t p, size_t h, int nranks, int* owners, size_t owners_len, size_t* nblocks,
                                size_t* block) {
    return guarded([&] {
        if (nranks < 1) fail(FSYRK_B200_EINVAL, "nranks must be >= 1");
        validate_field(p);
        const SchemeInfo si = scheme_for(p, nranks);
        const int blk = part_block_for(si.bm, si.bn);
        std::vector<int> own = partition_owners((int)h, nranks, blk);
        const size_t nb = (h + blk - 1) / blk;
        if (nblocks) *nblocks = nb;
        if (block) *block = (size_t)blk;
        if (owners) {
            if (owners_len < own.size()) fail(FSYRK_B200_EDIMENSION, "owner buffer too small");
            std::copy(own.begin(), own.end(), owners);
        }
    });
}

void fsyrk_b200_release_cache(void) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache.clear();
}

int fsyrk_b200_upload(uint64_t p, const uint64_t* h, size_t rows, size_t cols, size_t ldh, int lower, uint64_t* d_dev,
                      size_t ldd, void* stream) {
    return guarded([&] {
        validate_field(p);
        if (ldh < cols || ldd < cols || (lower && cols < rows)) fail(FSYRK_B200_EDIMENSION, "upload: bad shape");
        require_device();
        if (rows == 0 || cols == 0) return;
        if (hio::is_device(h)) fail(FSYRK_B200_EINVAL, "upload: host rows are device memory");
        std::lock_guard<std::mutex> lk(g_stage_mu);
        uint64_t bytes = 0;
        ck(hio::upload(h, ldh, hio::Region{rows, cols, lower != 0}, d_dev, ldd, hio::transfer_bits(p),
                       static_cast<cudaStream_t>(stream), &bytes),
           "upload");
        g_transfer[0] = bytes;
        g_transfer[1] = 0;
    });
}

int fsyrk_b200_download(uint64_t p, const uint64_t* d_dev, size_t rows, size_t cols, size_t ldd, int lower,
                        uint64_t* h, size_t ldh, void* stream) {
    return guarded([&] {
        validate_field(p);
        if (ldh < cols || ldd < cols || (lower && cols < rows)) fail(FSYRK_B200_EDIMENSION, "download: bad shape");
        require_device();
        if (rows == 0 || cols == 0) return;
        if (hio::is_device(h)) fail(FSYRK_B200_EINVAL, "download: host rows are device memory");
        std::lock_guard<std::mutex> lk(g_stage_mu);
        uint64_t bytes = 0;
        ck(hio::download(d_dev, ldd, hio::Region{rows, cols, lower != 0}, h, ldh, 0, hio::transfer_bits(p),
                         static_cast<cudaStream_t>(stream), &bytes),
           "download");
        g_transfer[1] = bytes;
    });
}

int fsyrk_b200_hostio_roundtrip(const uint64_t* a, size_t rows, size_t cols, size_t lda, int lower, int bits,
                                uint64_t* out, size_t ldo, size_t* raw_chunks, double* secs) {
    return guarded([&] {
        if (lower && cols < rows) fail(FSYRK_B200_EDIMENSION, "hostio_roundtrip: lower region needs cols >= rows");
        if (lda < cols || ldo < cols) fail(FSYRK_B200_EDIMENSION, "hostio_roundtrip: stride < cols");
        double t[2];
        std::lock_guard<std::mutex> lk(g_stage_mu);  // one user of the host worker pool at a time
        const size_t raw = hio::roundtrip(a, lda, hio::Region{rows, cols, lower != 0}, bits, out, ldo, t);
        if (raw_chunks) *raw_chunks = raw;
        if (secs) {
            secs[0] = t[0];
            secs[1] = t[1];
        }
    });
}

int fsyrk_b200_last_transfer_bytes(uint64_t* h2d, uint64_t* d2h) {
    if (h2d) *h2d = g_transfer[0];
    if (d2h) *d2h = g_transfer[1];
    return FSYRK_B200_OK;
}

int fsyrk_b200_last_launch_count(int* by_kind, int nkinds) {
    int total = 0;
    for (int i = 0; i < 5; ++i) {
        total += g_launch_counts[i];
        if (by_kind && i < nkinds) by_kind[i] = g_launch_counts[i];
    }
    return total;
}

const char* fsyrk_b200_last_plan_json(void) { return g_last_plan_json.c_str(); }

int fsyrk_b200_set_phase_timing(int enable) {
    g_phase_timing = enable != 0;
    return 0;
}

int fsyrk_b200_last_phase_ms(float* out, int nkinds) {
    for (int i = 0; i < 5 && i < nkinds; ++i) out[i] = g_phase_ms[i];
    return 0;
}

int fsyrk_b200_level_blocks(uint64_t p, const uint64_t* a, size_t n, size_t k, size_t lda, uint64_t* s1, uint64_t* s2,
                            uint64_t* s3, uint64_t* s4, uint64_t* p1, uint64_t* p2, uint64_t* p3, uint64_t* p4,
                            uint64_t* p5, size_t* kw_out) {
    return guarded([&] {
        validate_field(p);
        validate_shapes(n, k, lda, n);
        require_device();
        fsyrk_b200_policy pol{2, 1};
        Plan plan;
        plan.create(p, (int)n, (int)k, (int)k, pol, false);
        const Node& root = plan.nodes[0];
        if (root.kind != LEVEL) fail(FSYRK_B200_EDIMENSION, "level_blocks: shape does not admit a recursion level");
        DevBuf da, dc;
        da.ensure(n * k * 8);
        dc.ensure(n * n * 8);
        ck(cudaMemcpy2D(da.ptr, k * 8, a, lda * 8, k * 8, n, cudaMemcpyHostToDevice), "H2D");
        plan.execute(static_cast<uint64_t*>(da.ptr), (long long)k, static_cast<uint64_t*>(dc.ptr), (long long)n, 1, 0,
                     false, 0);
        ck(cudaDeviceSynchronize(), "sync");
        const int h = root.h, kw = root.kw, L = plan.L;
        if (kw_out) *kw_out = (size_t)kw;
        const GemmGroup& g = plan.gemms[root.ggroup];
        // recombine digit planes -> residues on the host (white-box readback only): the first
        // `nd` planes are the digits of base 2^bits, signed for the balanced LIMB schemes
        const int sid = plan.sch.id;
        const bool m17 = sid == SCHEME_M17 || sid == SCHEME_M17N;
        const int nd = m17 ? 3 : sid == SCHEME_M31 ? 4 : L;
        const int bits = m17 ? 6 : 8;
        const bool sgn = !plan.sch.is_unsigned;
        auto read_planes = [&](const int8_t* base, long long plane, long long row, int rows, int cols, uint64_t* out) {
            std::vector<int8_t> buf((size_t)plane * nd);
            ck(cudaMemcpy(buf.data(), base, buf.size(), cudaMemcpyDeviceToHost), "D2H planes");
            for (int i = 0; i < rows; ++i)
                for (int j = 0; j < cols; ++j) {
                    long long v = 0, w = 1;
                    for (int l = 0; l < nd; ++l) {
                        const int8_t b = buf[(size_t)l * plane + (size_t)i * row + j];
                        v += (sgn ? (long long)b : (long long)(uint8_t)b) * w;
                        w <<= bits;
                    }
                    long long r = v % (long long)p;
                    if (r < 0) r += (long long)p;
                    out[(size_t)i * cols + j] = (uint64_t)r;
                }
        };
        if (s1) read_planes(g.ga + (2LL * root.gslot) * g.slot, g.plane, g.kpad, h, kw, s1);
        if (s2) read_planes(g.gb + (2LL * root.gslot) * g.slot_b, g.plane, g.kpad, h, kw, s2);
        if (s4) read_planes(g.gb + (2LL * root.gslot + 1) * g.slot_b, g.plane, g.kpad, h, kw, s4);
        if (s3) {
            const Node& c2 = plan.nodes[root.ch[2]];
            const LeafGroup& lg = plan.leaves[c2.lgroup];
            read_planes(lg.planes + c2.lslot * lg.slot, lg.plane, lg.kpad, h, kw, s3);
        }
        auto read_u32 = [&](const uint32_t* src, long long ld, uint64_t* out) {
            std::vector<uint32_t> buf((size_t)h * h);
            ck(cudaMemcpy2D(buf.data(), h * 4, src, ld * 4, h * 4, h, cudaMemcpyDeviceToHost), "D2H P");
            for (size_t i = 0; i < buf.size(); ++i) out[i] = buf[i];
        };
        if (p1) read_u32(plan.nodes[root.ch[0]].x, plan.nodes[root.ch[0]].ldx, p1);
        if (p2) read_u32(plan.nodes[root.ch[1]].x, plan.nodes[root.ch[1]].ldx, p2);
        if (p5) read_u32(plan.nodes[root.ch[2]].x, plan.nodes[root.ch[2]].ldx, p5);
        if (p4) read_u32(g.out + (2LL * root.gslot) * g.h * g.h, g.h, p4);
        if (p3) read_u32(g.out + (2LL * root.gslot + 1) * g.h * g.h, g.h, p3);
    });
}

int fsyrk_b200_gemm_nt(uint64_t p, const uint64_t* a, size_t m, size_t k, size_t lda, const uint64_t* b, size_t n,
                       size_t ldb, uint64_t* c, size_t ldc) {
    return guarded([&] {
        validate_field(p);
        if (lda < k || ldb < k || ldc < n) fail(FSYRK_B200_EDIMENSION, "gemm_nt: dimension mismatch");
        require_device();
        if (m == 0 || n == 0) return;
        const size_t kk = std::max<size_t>(k, 1);
        DevBuf d64a, d64b, out;
        d64a.ensure(m * kk * 8);
        d64b.ensure(n * kk * 8);
        out.ensure(m * n * 4);
        if (k > 0) {
            ck(cudaMemcpy2D(d64a.ptr, k * 8, a, lda * 8, k * 8, m, cudaMemcpyHostToDevice), "H2D A");
            ck(cudaMemcpy2D(d64b.ptr, k * 8, b, ldb * 8, k * 8, n, cudaMemcpyHostToDevice), "H2D B");
        }
        gemm_nt_dev(p, static_cast<uint64_t*>(d64a.ptr), m, k, kk, static_cast<uint64_t*>(d64b.ptr), n, kk,
                    static_cast<uint32_t*>(out.ptr), (long long)n, 0);
        std::vector<uint32_t> buf(m * n);
        ck(cudaMemcpy(buf.data(), out.ptr, m * n * 4, cudaMemcpyDeviceToHost), "D2H");
        for (size_t i = 0; i < m; ++i)
            for (size_t j = 0; j < n; ++j) c[i * ldc + j] = buf[i * n + j];
    });
}

int fsyrk_b200_gemm_winograd_nt(uint64_t p, const uint64_t* a, size_t m, size_t k, size_t lda, const uint64_t* b,
                                size_t n, size_t ldb, uint64_t* c, size_t ldc, fsyrk_b200_policy policy) {
    return guarded([&] {
        validate_field(p);
        validate_policy(policy);
        if (lda < k || ldb < k || ldc < n) fail(FSYRK_B200_EDIMENSION, "gemm_winograd_nt: dimension mismatch");
        require_device();
        if (m == 0 || n == 0) return;
        const size_t kk = std::max<size_t>(k, 1);
        DevBuf d64a, d64b, d64c;
        d64a.ensure(m * kk * 8);
        d64b.ensure(n * kk * 8);
        d64c.ensure(m * n * 8);
        if (k > 0) {
            ck(cudaMemcpy2D(d64a.ptr, k * 8, a, lda * 8, k * 8, m, cudaMemcpyHostToDevice), "H2D A");
            ck(cudaMemcpy2D(d64b.ptr, k * 8, b, ldb * 8, k * 8, n, cudaMemcpyHostToDevice), "H2D B");
        }
        check_status(fsyrk_b200_gemm_winograd_nt_dev(p, static_cast<uint64_t*>(d64a.ptr), m, k, kk,
                                                     static_cast<uint64_t*>(d64b.ptr), n, kk,
                                                     static_cast<uint64_t*>(d64c.ptr), n, policy, nullptr));
        ck(cudaMemcpy2D(c, ldc * 8, d64c.ptr, n * 8, n * 8, m, cudaMemcpyDeviceToHost), "D2H C");
    });
}

int fsyrk_b200_gemm_winograd_nt_dev(uint64_t p, const uint64_t* a_dev, size_t m, size_t k, size_t lda,
                                    const uint64_t* b_dev, size_t n, size_t ldb, uint64_t* c_dev, size_t ldc,
                                    fsyrk_b200_policy policy, void* stream) {
    return guarded([&] {
        validate_field(p);
        validate_policy(policy);
        if (lda < k || ldb < k || ldc < n) fail(FSYRK_B200_EDIMENSION, "gemm_winograd_nt: dimension mismatch");
        require_device();
        if (m == 0 || n == 0) return;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const size_t kk = std::max<size_t>(k, 1);
        struct Io {  // residue copies of A, B, C kept across calls, per device
            std::mutex mu;
            DevBuf ra, rb, rc;
        };
        Io& io = per_device<Io>();
        std::lock_guard<std::mutex> lk(io.mu);
        DevBuf &ra = io.ra, &rb = io.rb, &rc = io.rc;
        ra.ensure(m * kk * 4);
        rb.ensure(n * kk * 4);
        rc.ensure(m * n * 4);
        auto* A = static_cast<uint32_t*>(ra.ptr);
        auto* B = static_cast<uint32_t*>(rb.ptr);
        auto* C = static_cast<uint32_t*>(rc.ptr);
        if (k == 0) {
            ck(cudaMemsetAsync(C, 0, m * n * 4, s), "memset");
        } else {
            ck(launch_convert_in(a_dev, (long long)lda, (int)m, (int)k, (int)k, nullptr, (uint32_t)p, A, (long long)k, s),
               "convert A");
            ck(launch_convert_in(b_dev, (long long)ldb, (int)n, (int)k, (int)k, nullptr, (uint32_t)p, B, (long long)k, s),
               "convert B");
            wino_gemm_dev(p, A, (long long)k, m, B, (long long)k, n, k, C, (long long)n, policy, s);
        }
        ck(launch_u32_to_u64(C, (long long)n, (int)m, (int)n, c_dev, (long long)ldc, s), "widen C");
        ck(cudaStreamSynchronize(s), "sync");
    });
}

int fsyrk_b200_herk_fast_into(uint64_t p, const uint64_t* a, size_t n, size_t k, size_t lda, uint64_t* c, size_t ldc,
                              fsyrk_b200_policy policy, int mirror_output, fsyrk_b200_opcount* ops) {
    return guarded([&] { run_fp2(p, a, n, k, lda, c, ldc, policy, mirror_output != 0, true, ops); });
}

int fsyrk_b200_syrk_fast_into_fp2(uint64_t p, const uint64_t* a, size_t n, size_t k, size_t lda, uint64_t* c,
                                  size_t ldc, fsyrk_b200_policy policy, int mirror_output, fsyrk_b200_opcount* ops) {
    return guarded([&] { run_fp2(p, a, n, k, lda, c, ldc, policy, mirror_output != 0, false, ops); });
}


int fsyrk_b200_syrk_mgpu(uint64_t p, uint64_t alpha, const uint64_t* a, size_t n, size_t k, size_t lda,
                         const uint64_t* d, uint64_t beta, uint64_t* c, size_t ldc, fsyrk_b200_policy policy,
                         int mirror_output, const int* devices, int ngpus, fsyrk_b200_opcount* ops) {
    return guarded([&] {
        if (ngpus < 1 || !devices) fail(FSYRK_B200_EINVAL, "syrk_mgpu: need at least one device");
        validate_field(p);
        ColXform xf;
        if (d) xf = xform_diag(p, d, k);
        std::vector<int> devs(devices, devices + ngpus);
        std::vector<int> sorted = devs;
        std::sort(sorted.begin(), sorted.end());
        const bool distinct = std::unique(sorted.begin(), sorted.end()) == sorted.end();
        std::vector<LocalRank> loc(ngpus);
        std::vector<ncclComm_t> comms;
        if (distinct && ngpus > 1) comms = comms_for(devs);
        for (int r = 0; r < ngpus; ++r) loc[r] = LocalRank{devs[r], r, comms.empty() ? nullptr : comms[r]};
        mgpu_run(loc, ngpus, p, alpha, a, n, k, lda, d ? &xf : nullptr, beta, c, ldc, policy, mirror_output != 0, ops);
    });
}

int fsyrk_b200_nccl_unique_id(uint8_t id[128]) {
    return guarded([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
        ncclUniqueId u;
        nck(nccl().get_unique_id(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    });
}

int fsyrk_b200_comm_init_rank(const uint8_t id[128], int rank, int nranks, void** comm) {
    return guarded([&] {
        if (!comm || nranks < 1 || rank < 0 || rank >= nranks) fail(FSYRK_B200_EINVAL, "comm_init_rank: bad rank");
        require_device();
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        auto* cm = new Comm;
        cm->rank = rank;
        cm->nranks = nranks;
        cm->dev = current_device();
        const ncclResult_t r = nccl().init_rank(&cm->comm, nranks, u, rank);
        if (r != ncclSuccess) {
            delete cm;
            nck(r, "ncclCommInitRank");
        }
        *comm = cm;
    });
}

int fsyrk_b200_comm_destroy(void* comm) {
    return guarded([&] {
        if (!comm) return;
        auto* cm = static_cast<Comm*>(comm);
        if (cm->comm) nck(nccl().destroy(cm->comm), "ncclCommDestroy");
        delete cm;
    });
}

int fsyrk_b200_syrk_mgpu_rank(void* comm, uint64_t p, uint64_t alpha, const uint64_t* a, size_t n, size_t k,
                              size_t lda, const uint64_t* d, uint64_t beta, uint64_t* c, size_t ldc,
                              fsyrk_b200_policy policy, int mirror_output, fsyrk_b200_opcount* ops) {
    return guarded([&] {
        if (!comm) fail(FSYRK_B200_EINVAL, "syrk_mgpu_rank: null communicator");
        const Comm& cm = *static_cast<const Comm*>(comm);
        validate_field(p);
        ColXform xf;
        if (d) xf = xform_diag(p, d, k);
        std::vector<LocalRank> loc{LocalRank{cm.dev, cm.rank, cm.comm}};
        mgpu_run(loc, cm.nranks, p, alpha, a, n, k, lda, d ? &xf : nullptr, beta, c, ldc, policy, mirror_output != 0,
                 ops);
    });
}


int fsyrk_b200_share_pairs(uint64_t p, size_t h, int rank, int nranks, int* pairs, size_t cap, size_t* count) {
    return guarded([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(FSYRK_B200_EINVAL, "rank out of range");
        validate_field(p);
        const SchemeInfo si = scheme_for(p, nranks);
        const int blk = part_block_for(si.bm, si.bn);
        const std::vector<int> own = partition_owners((int)h, nranks, blk);
        const int nb = ((int)h + blk - 1) / blk, T = ((int)h + 31) / 32;
        size_t cnt = 0;
        for (int I = 0; I < T; ++I)
            for (int J = 0; J <= I; ++J)
                if (own[(size_t)(I * 32 / blk) * nb + J * 32 / blk] == rank) {
                    if (pairs) {
                        if (cnt >= cap) fail(FSYRK_B200_EDIMENSION, "share_pairs: buffer too small");
                        pairs[2 * cnt] = I;
                        pairs[2 * cnt + 1] = J;
                    }
                    ++cnt;
                }
        if (count) *count = cnt;
    });
}

}  // extern "C"

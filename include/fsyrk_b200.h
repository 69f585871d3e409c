/* fsyrk_b200 — C ABI of the B200-native mod-p SYRK hot path.
 *
 * Drop-in boundary for the reference fsyrk library's PrimeField SYRK entry
 * points.  Every function below replaces one reference interface; the
 * citation after "replaces" is the reference declaration (paths relative to
 * /root/reference/proj).  Matrices use the reference layout: row-major
 * uint64_t residues in [0, p), (data, rows, cols, stride-in-elements)
 * (include/fsyrk/matrix.hpp:58-127).  Only Low(C) (diagonal included) is
 * defined on return; the strict upper triangle is left untouched unless
 * mirror_output is set (include/fsyrk/fast_syrk.hpp:271-282).
 *
 * All entry points are synchronous: they return with C filled (host
 * variants) or with the work complete on the given stream's device
 * (device variants synchronise the stream before returning).  Errors are
 * reported as status codes; fsyrk_b200_last_error() gives the message of the
 * calling thread's last failure.  The C++ shim include/fsyrk_b200/fsyrk.hpp
 * maps the codes back to the reference's exception types.
 *
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry point returns FSYRK_B200_ENODEV.
 */
#ifndef FSYRK_B200_H
#define FSYRK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSYRK_B200_ABI_VERSION 1

/* Status codes.  Mapping to the reference's error convention:
 *   EDIMENSION -> fsyrk::DimensionError        (matrix.hpp:131-133)
 *   EINVAL     -> std::invalid_argument         (alias fast_syrk.hpp:279, threshold<2
 *                                                winograd.hpp:18-20, bad prime fields.cpp:33-37)
 *   EPARITY    -> fsyrk::DimensionParityError   (skew.hpp:54-55)
 *   ENONRES    -> fsyrk::NotNonResidueError      (skew.hpp:182-187)
 *   EDOMAIN    -> std::domain_error              (fields.cpp:63-64, p = 2 cases)
 *   ECUDA / ENOMEM / ENODEV / ENCCL -> std::runtime_error (device side; no reference analogue) */
enum fsyrk_b200_status {
    FSYRK_B200_OK = 0,
    FSYRK_B200_EDIMENSION = 1,
    FSYRK_B200_EINVAL = 2,
    FSYRK_B200_EPARITY = 3,
    FSYRK_B200_ENONRES = 4,
    FSYRK_B200_EDOMAIN = 5,
    FSYRK_B200_ECUDA = 6,
    FSYRK_B200_ENOMEM = 7,
    FSYRK_B200_ENODEV = 8,
    FSYRK_B200_ENCCL = 9
};

/* Recursion policy: replaces fsyrk::RecursionPolicy (include/fsyrk/winograd.hpp:14-21).
 * max_levels = UINT64_MAX means unlimited (kUnlimitedLevels, winograd.hpp:9). */
typedef struct fsyrk_b200_policy {
    uint64_t threshold;
    uint64_t max_levels;
} fsyrk_b200_policy;

/* Operation tally: replaces fsyrk::OpCount (include/fsyrk/opcount.hpp:10-25).
 * Every entry point adds what the reference would have counted for the same call
 * (its per-routine tallies of syrk_classical, the Winograd engine, the level
 * additions, the skew and the syrkd / syrkbd column transforms; a host dry-run of
 * its recursion, csrc/ref_opcount.h), so the reference's reconciliations with its
 * count model (tests/test_fast_syrk.cpp:202-238, tools/fsyrk.cpp:215-242) hold.
 * The device's own work (tensor MACs, elementwise bytes) is in fsyrk_b200_last_plan_json. */
typedef struct fsyrk_b200_opcount {
    uint64_t mults;
    uint64_t adds;
} fsyrk_b200_opcount;

/* Skew-orthogonal Y: replaces fsyrk::SkewOrthogonal / skew_orthogonal(PrimeField, dim)
 * (include/fsyrk/skew.hpp:21-37, 66-73).  form: 0 = ScalarRoot(a), 1 = Pair(a, b). */
typedef struct fsyrk_b200_skew {
    int form;
    uint64_t a;
    uint64_t b;
    int ycost;
} fsyrk_b200_skew;

const char* fsyrk_b200_last_error(void);
int fsyrk_b200_abi_version(void);

/* 1 if a usable sm_100 device is present (no work launched). */
int fsyrk_b200_device_available(void);

/* make_syrk_plan(f, policy, mirror) (include/fsyrk/fast_syrk.hpp:20-24): validates the
 * field and policy and returns the Y the recursion uses.  Host-only setup. */
int fsyrk_b200_make_syrk_plan(uint64_t p, fsyrk_b200_policy policy, int mirror_output, fsyrk_b200_skew* skew);

/* skew_orthogonal(PrimeField, dim) (include/fsyrk/skew.hpp:66-73). */
int fsyrk_b200_skew_orthogonal(uint64_t p, size_t dim, fsyrk_b200_skew* skew);

/* random_matrix(f, rows, cols, seed) (include/fsyrk/matrix.hpp:411-419): the
 * reference's seeded generator (std::mt19937_64 + uniform_int_distribution),
 * host-side, so callers can build the same inputs as the reference. */
int fsyrk_b200_random_matrix(uint64_t p, size_t rows, size_t cols, uint64_t seed, uint64_t* out, size_t ld);

/* PrimeField::sum_of_squares(k) (proj/src/fields.cpp:114-123): a^2 + b^2 = k (mod p), odd p.
 * Host-only; used by the skew construction and the CLI's `sos` command. */
int fsyrk_b200_sum_of_squares(uint64_t p, uint64_t k, uint64_t* a, uint64_t* b);

/* nrsyf(f, alpha, beta) (proj/include/fsyrk/skew.hpp:180-194): y = [[a, b], [c, d]] with
 * Y * Y^T = diag(alpha, beta) for two non-residues (FSYRK_B200_ENONRES otherwise).  Host-only. */
int fsyrk_b200_nrsyf(uint64_t p, uint64_t alpha, uint64_t beta, uint64_t y[4]);

/* ---------------------------------------------------------------- host API */

/* syrk_fast_into(f, a, c, plan, ops) (include/fsyrk/fast_syrk.hpp:274-282):
 * Low(C) <- Low(A * A^T).  a: n x k host matrix, c: n x n host matrix. */
int fsyrk_b200_syrk_fast_into(uint64_t p, const uint64_t* a, size_t n, size_t k, size_t lda, uint64_t* c,
                              size_t ldc, fsyrk_b200_policy policy, int mirror_output, fsyrk_b200_opcount* ops);

/* syrk_fast_acc(f, alpha, a, beta, c, plan, ops) (include/fsyrk/fast_syrk.hpp:293-303):
 * Low(C) <- Low(alpha * A * A^T + beta * C); reads only Low(C_in). */
int fsyrk_b200_syrk_fast_acc(uint64_t p, uint64_t alpha, const uint64_t* a, size_t n, size_t k, size_t lda,
                             uint64_t beta, uint64_t* c, size_t ldc, fsyrk_b200_policy policy, int mirror_output,
                             fsyrk_b200_opcount* ops);

/* syrkd(f, a, d, plan, ops) (include/fsyrk/scaled_syrk.hpp:58-104), extended with the
 * accumulate form so the LDL^T Schur update C <- C - A*D*A^T is one call
 * (alpha = p - 1, beta = 1):  Low(C) <- Low(alpha * A * Diag(d) * A^T + beta * C).
 * d has k entries.  alpha = 1, beta = 0 is exactly the reference's syrkd. */
int fsyrk_b200_syrkd(uint64_t p, uint64_t alpha, const uint64_t* a, size_t n, size_t k, size_t lda,
                     const uint64_t* d, uint64_t beta, uint64_t* c, size_t ldc, fsyrk_b200_policy policy,
                     int mirror_output, fsyrk_b200_opcount* ops);

/* One block of the middle matrix of syrkbd: replaces fsyrk::BlockDiagonal<F>::Block
 * (include/fsyrk/scaled_syrk.hpp:13-20).  two = 0: scalar block d; two = 1: the 2x2
 * block ((0, beta), (beta, gamma)), beta != 0; gamma must be 0 over an odd prime. */
typedef struct fsyrk_b200_block {
    int two;
    uint64_t d;
    uint64_t beta;
    uint64_t gamma;
} fsyrk_b200_block;

/* syrkbd(f, a, b, plan, ops) (include/fsyrk/scaled_syrk.hpp:117-159), with the same
 * accumulate extension as fsyrk_b200_syrkd:
 *   Low(C) <- Low(alpha * A * B * A^T + beta * C),  B = blockdiag(blocks[0..nblocks)).
 * The block dimension (scalar blocks count 1, 2x2 blocks 2) must equal k. */
int fsyrk_b200_syrkbd(uint64_t p, uint64_t alpha, const uint64_t* a, size_t n, size_t k, size_t lda,
                      const fsyrk_b200_block* blocks, size_t nblocks, uint64_t beta, uint64_t* c, size_t ldc,
                      fsyrk_b200_policy policy, int mirror_output, fsyrk_b200_opcount* ops);

/* Quadratic extension F_{p^2} = F_p[x] / (x^2 - ns), ns the least quadratic non-residue
 * (fsyrk::QuadExtField, include/fsyrk/fields.hpp:142-212).  Matrices hold (a, b) uint64 pairs
 * (QuadExtElement, fields.hpp:142-146) row-major; lda / ldc count pairs.
 * herk_fast_into (include/fsyrk/fast_syrk.hpp:307-313): Low(C) <- Low(A * conj(A)^T);
 * the fp2 syrk_fast_into (fast_syrk.hpp:274-282 over QuadExtField): Low(C) <- Low(A * A^T).
 * mirror_output fills the upper triangle with the (conjugate) transpose; otherwise it is zero. */
int fsyrk_b200_herk_fast_into(uint64_t p, const uint64_t* a, size_t n, size_t k, size_t lda, uint64_t* c, size_t ldc,
                              fsyrk_b200_policy policy, int mirror_output, fsyrk_b200_opcount* ops);
int fsyrk_b200_syrk_fast_into_fp2(uint64_t p, const uint64_t* a, size_t n, size_t k, size_t lda, uint64_t* c,
                                  size_t ldc, fsyrk_b200_policy policy, int mirror_output, fsyrk_b200_opcount* ops);

/* -------------------------------------------------------------- device API */

/* Same operations on device-resident uint64 matrices (pointers from
 * cudaMalloc on the current device); `stream` is a cudaStream_t (NULL =
 * legacy default stream).  d (syrkd) is a HOST array of k entries.  These do
 * not synchronise the host beyond what plan creation needs; call
 * cudaStreamSynchronize before reading C. */
int fsyrk_b200_syrk_dev(uint64_t p, uint64_t alpha, const uint64_t* a_dev, size_t n, size_t k, size_t lda,
                        const uint64_t* d_host, uint64_t beta, uint64_t* c_dev, size_t ldc,
                        fsyrk_b200_policy policy, int mirror_output, void* stream, fsyrk_b200_opcount* ops);

/* syrkbd on device-resident A and C (blocks is a HOST array). */
int fsyrk_b200_syrkbd_dev(uint64_t p, uint64_t alpha, const uint64_t* a_dev, size_t n, size_t k, size_t lda,
                          const fsyrk_b200_block* blocks, size_t nblocks, uint64_t beta, uint64_t* c_dev, size_t ldc,
                          fsyrk_b200_policy policy, int mirror_output, void* stream, fsyrk_b200_opcount* ops);

/* ------------------------------------------------------------ multi-GPU */

/* One rank's share of a syrk / syrk_acc / syrkd call partitioned over `nranks`
 * GPUs (no reference analogue -- the reference is single-threaded).
 * Every rank holds the whole A on its device and calls this with the same
 * arguments; rank r computes the entries of Low(C) in the top-level block pairs
 * it owns (fsyrk_b200_partition_owners) and leaves all other entries of C
 * untouched.  The union over ranks equals the single-GPU result.  The top level
 * is split with its three SYRK products as leaves (max_levels is capped at 1);
 * shapes whose top level does not recurse are computed entirely by rank 0. */
int fsyrk_b200_syrk_part_dev(uint64_t p, uint64_t alpha, const uint64_t* a_dev, size_t n, size_t k, size_t lda,
                             const uint64_t* d_host, uint64_t beta, uint64_t* c_dev, size_t ldc,
                             fsyrk_b200_policy policy, int rank, int nranks, void* stream, fsyrk_b200_opcount* ops);

/* Host <-> device staging of residue matrices through the library's transfer path (bit-packed
 * residues of p on the wire, host worker threads, pinned slots; see host_io.h) -- what the host
 * entry points use internally, for callers that keep A / C on the device (e.g. rank 0 of a
 * multi-GPU call before an NCCL broadcast).  lower != 0: only row i's columns [0, i] move.
 * upload returns once the transfer is queued on `stream` (the caller's host rows may be reused);
 * download is synchronous; device values must be < 2^32.  Host-to-device / device-to-host byte
 * counts land in fsyrk_b200_last_transfer_bytes. */
int fsyrk_b200_upload(uint64_t p, const uint64_t* h, size_t rows, size_t cols, size_t ldh, int lower, uint64_t* d_dev,
                      size_t ldd, void* stream);
int fsyrk_b200_download(uint64_t p, const uint64_t* d_dev, size_t rows, size_t cols, size_t ldd, int lower,
                        uint64_t* h, size_t ldh, void* stream);

/* Owner rank of every top-level block pair (I >= J) for quadrant size h = n/2:
 * owners[I * nblocks + J]; blocks are `block` rows/columns (lcm of 128 and the
 * product tile width of p's digit scheme).  Host-only. */
int fsyrk_b200_partition_owners(uint64_t p, size_t h, int nranks, int* owners, size_t owners_len, size_t* nblocks,
                                size_t* block);

/* ------------------------------------------------------------- multi-GPU */

/* Multi-GPU syrk_fast_into / syrk_fast_acc / syrkd over `ngpus` devices of this process
 * (replaces the same reference entry points as the host API above,
 * include/fsyrk/fast_syrk.hpp:274-303 and scaled_syrk.hpp:58-104, for callers that want
 * several GPUs).  Host A / C as in the host API; d: syrkd diagonal (k entries) or NULL;
 *   Low(C) <- Low(alpha * A * Diag(d) * A^T + beta * C).
 * A crosses PCIe once into devices[0], is broadcast as uint32 residues over NVLink by an
 * internal NCCL communicator (ncclCommInitAll, cached per device list), every device computes
 * the top-level tile pairs it owns (fsyrk_b200_share_pairs), and the owned tiles of Low(C)
 * return to devices[0] as packed uint32 shares (ncclSend / ncclRecv) before crossing PCIe.
 * Shapes whose top level is not partitionable run on devices[0] alone.  A device listed more
 * than once makes the ranks on it exchange by device copies instead of NCCL (a test mode). */
int fsyrk_b200_syrk_mgpu(uint64_t p, uint64_t alpha, const uint64_t* a, size_t n, size_t k, size_t lda,
                         const uint64_t* d, uint64_t beta, uint64_t* c, size_t ldc, fsyrk_b200_policy policy,
                         int mirror_output, const int* devices, int ngpus, fsyrk_b200_opcount* ops);

/* The same call with one process per GPU (e.g. under torchrun): rank 0 creates an NCCL unique
 * id and hands it to the other ranks out of band; every rank creates its communicator on its
 * current device and makes the same collective call.  Only rank 0 reads `a` and reads / writes
 * `c` (the other ranks may pass NULL); d, alpha, beta, policy must agree on every rank. */
int fsyrk_b200_nccl_unique_id(uint8_t id[128]);
int fsyrk_b200_comm_init_rank(const uint8_t id[128], int rank, int nranks, void** comm);
int fsyrk_b200_comm_destroy(void* comm);
int fsyrk_b200_syrk_mgpu_rank(void* comm, uint64_t p, uint64_t alpha, const uint64_t* a, size_t n, size_t k,
                              size_t lda, const uint64_t* d, uint64_t beta, uint64_t* c, size_t ldc,
                              fsyrk_b200_policy policy, int mirror_output, fsyrk_b200_opcount* ops);

/* The 32 x 32 tile pairs (I >= J, as int pairs I, J) of the h x h top-level quadrants owned
 * by `rank` of `nranks`: its share of Low(C) is tile (I, J) of C11, C21 and C22 and tile
 * (J, I) of C21 for each pair, moved as 4 x 1024 uint32 words per pair (slot order C11(I,J),
 * C21(I,J), C22(I,J), C21(J,I); entries outside Low(C) or beyond h are zero).  Host-only.
 * pairs may be NULL (count only); *count = number of pairs. */
int fsyrk_b200_share_pairs(uint64_t p, size_t h, int rank, int nranks, int* pairs, size_t cap, size_t* count);

/* Drop cached plans and device arenas (tests, memory pressure). */
void fsyrk_b200_release_cache(void);

/* --------------------------------------------------------------- telemetry */

/* Kernel launches issued by the last compute call on this thread, and the
 * per-kind launch counts (index: 0 tensor-core products, 1 pre-addition,
 * 2 post-addition, 3 conversion/finalize, 4 other). */
int fsyrk_b200_last_launch_count(int* by_kind, int nkinds);

/* Host<->device bytes moved by the last host-API call on this thread (A, and only the
 * lower-triangle row blocks of C unless mirror_output). */
int fsyrk_b200_last_transfer_bytes(uint64_t* h2d, uint64_t* d2h);

/* Host-only check of the host transfer format (no device needed): the rows of `a`
 * (lower != 0: row i holds columns [0, i]) are packed exactly as the host entry points put
 * them on the wire -- `bits` in [8, 24] bit-packed groups, 32 = uint32 -- by the library's host
 * worker pool, then unpacked into `out` (same shape, stride ldo).  Returns the number of
 * chunks that would cross unnarrowed (a value >= 2^bits) in *raw_chunks and the seconds
 * spent packing / unpacking in secs[2].  Diagnostic / test hook. */
int fsyrk_b200_hostio_roundtrip(const uint64_t* a, size_t rows, size_t cols, size_t lda, int lower, int bits,
                                uint64_t* out, size_t ldo, size_t* raw_chunks, double* secs);

/* Describe the last executed plan as a JSON string (tree, groups, limbs, bytes). */
const char* fsyrk_b200_last_plan_json(void);

/* Time each kernel kind of the last plan with CUDA events when enabled
 * (adds syncs; for profiling only).  Returns milliseconds per kind via out[5]. */
int fsyrk_b200_set_phase_timing(int enable);
int fsyrk_b200_last_phase_ms(float* out, int nkinds);

/* ------------------------------------------------------------- white box */

/* One recursion level with direct (classical) sub-products on the device:
 * returns S1..S4 (h x kw, row-major, ld = kw) and P1..P5 (h x h, P4 = S1*S2^T),
 * the blocks of Table 3 (include/fsyrk/fast_syrk.hpp:82-133), as uint64.
 * Any output may be NULL.  Host pointers. */
int fsyrk_b200_level_blocks(uint64_t p, const uint64_t* a, size_t n, size_t k, size_t lda, uint64_t* s1,
                            uint64_t* s2, uint64_t* s3, uint64_t* s4, uint64_t* p1, uint64_t* p2, uint64_t* p3,
                            uint64_t* p4, uint64_t* p5, size_t* kw_out);

/* Exact tensor-core product C = A*B^T mod p (m x k times (n x k)^T), host
 * pointers; the general-product engine (replaces gemm_winograd_nt_into,
 * include/fsyrk/winograd.hpp:195-202, and gemm_classical_nt, matrix.hpp:317-329). */
int fsyrk_b200_gemm_nt(uint64_t p, const uint64_t* a, size_t m, size_t k, size_t lda, const uint64_t* b, size_t n,
                       size_t ldb, uint64_t* c, size_t ldc);

/* Strassen-Winograd general product C = A * B^T mod p (replaces gemm_winograd_nt_into,
 * include/fsyrk/winograd.hpp:195-202): policy.max_levels Winograd levels over the tensor-core
 * product while every dimension is even and >= policy.threshold; exact, so identical to
 * fsyrk_b200_gemm_nt.  Host pointers; _dev takes device pointers (C is m x n uint64). */
int fsyrk_b200_gemm_winograd_nt(uint64_t p, const uint64_t* a, size_t m, size_t k, size_t lda, const uint64_t* b,
                                size_t n, size_t ldb, uint64_t* c, size_t ldc, fsyrk_b200_policy policy);
int fsyrk_b200_gemm_winograd_nt_dev(uint64_t p, const uint64_t* a_dev, size_t m, size_t k, size_t lda,
                                    const uint64_t* b_dev, size_t n, size_t ldb, uint64_t* c_dev, size_t ldc,
                                    fsyrk_b200_policy policy, void* stream);

/* Device memory a call needs, without allocating it (host only): the plan's workspace
 * (`arena`: digit-plane operands, product outputs, node outputs; cached per shape) under the
 * wide (lowmem = 0) or the low-memory (lowmem = 1) schedule and, for the host entry points,
 * the workspace plus the device staging of A and C (`host_call`).  Either output may be
 * NULL.  A workspace the device cannot hold makes the call fail with FSYRK_B200_ECUDA and
 * the byte count in fsyrk_b200_last_error(). */
int fsyrk_b200_workspace_bytes(uint64_t p, size_t n, size_t k, fsyrk_b200_policy policy, int lowmem,
                               uint64_t* arena, uint64_t* host_call);

/* Process-wide workspace limit in bytes (0 = none, the default).  A call whose wide
 * workspace exceeds it runs the low-memory schedule -- the reference's placement of the
 * top level's general products in the scratch quadrant C12 of C (fast_syrk.hpp:96-98,
 * 271-273): P4 and P3 go to the strict upper triangle of the caller's C (device C needs an
 * even row stride and 16-byte alignment) instead of the workspace -- and one whose
 * low-memory workspace still exceeds it fails with FSYRK_B200_EINVAL.  Results are
 * identical; only the strict upper triangle of C (scratch, fast_syrk.hpp:271-273) differs. */
int fsyrk_b200_set_workspace_limit(uint64_t bytes);

/* Process-wide: enable = 1 runs every plan created afterwards (where a 2 x 2 top level
 * exists) with the low-memory schedule regardless of the limit; 0 restores the default. */
int fsyrk_b200_set_low_memory(int enable);

/* Process-wide: the top level's two general products P4, P3 run Strassen-Winograd levels
 * (the reference's gemm_winograd_nt_into inside the level, winograd.hpp:118-169, 195-202;
 * levels while every dimension is even and at least max(threshold, min_dim, 256)) when
 * min(h, kw) >= min_dim; below it they are direct tensor-core products (exact either way).
 * Default 16384, the measured crossover on B200; 0 = never.  Applies to plans created
 * afterwards (fsyrk_b200_release_cache drops cached ones). */
int fsyrk_b200_set_winograd_min(uint64_t min_dim);

/* ------------------------------------------------ reference op tallies (host only) */

/* The OpCount the reference's entry point adds for one call, without running it
 * (no device needed): syrk_fast_into (alpha = 1, beta = 0) / syrk_fast_acc
 * (fast_syrk.hpp:274-303); syrkd (scaled_syrk.hpp:58-104, d has k entries) and syrkbd
 * (:117-159) with this library's alpha / beta extension (alpha = 1, beta = 0 is the
 * reference's call); herk_fast / syrk_fast over F_{p^2} (fast_syrk.hpp:305-320). */
int fsyrk_b200_opcount_syrk(uint64_t p, size_t n, size_t k, uint64_t alpha, uint64_t beta,
                            fsyrk_b200_policy policy, fsyrk_b200_opcount* ops);
int fsyrk_b200_opcount_syrkd(uint64_t p, size_t n, size_t k, const uint64_t* d, uint64_t alpha, uint64_t beta,
                             fsyrk_b200_policy policy, fsyrk_b200_opcount* ops);
int fsyrk_b200_opcount_syrkbd(uint64_t p, size_t n, const fsyrk_b200_block* blocks, size_t nblocks,
                              uint64_t alpha, uint64_t beta, fsyrk_b200_policy policy, fsyrk_b200_opcount* ops);
int fsyrk_b200_opcount_fp2(uint64_t p, size_t n, size_t k, fsyrk_b200_policy policy, fsyrk_b200_opcount* ops);

#ifdef __cplusplus
}
#endif

#endif /* FSYRK_B200_H */

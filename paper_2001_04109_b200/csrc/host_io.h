// Host <-> device movement of the caller's matrices for the host entry points
// (fsyrk_b200_syrk_fast_into / _acc / syrkd / syrkbd).
//
// The reference's matrices are host uint64 residues (include/fsyrk/matrix.hpp:58-127); on
// this path PCIe is the bound (55 GB/s per direction from pinned memory on the B200 box,
// 11 GB/s from pageable memory, profiles/r01/hostio.txt), not the device.  Residues of p < 2^31
// need only 32 bits, so the host side narrows (H2D) / widens (D2H) on a pool of host threads
// through a ring of pinned staging slots, chunk by chunk, while the copy engine moves the
// previous chunk: half the PCIe bytes, and pageable callers get pinned-speed transfers.
// A chunk holding a value >= 2^32 (a non-canonical input; the device reduces any uint64) is
// copied unnarrowed, so the result never depends on the narrowing.
//
// All functions assume the caller holds the host-staging lock (one host call at a time).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "modp.cuh"

namespace fsyrk_b200 {
namespace hio {

// Rows [0, rows) of a row-major matrix; row i covers columns [0, lower ? i + 1 : cols).
struct Region {
    size_t rows, cols;
    bool lower;
    size_t width(size_t i) const { return lower ? i + 1 : cols; }
    size_t offset(size_t i) const { return lower ? i * (i + 1) / 2 : i * cols; }  // packed position of row i
};

// true when `p` is page-locked host memory (cudaHostAlloc / cudaHostRegister)
bool is_pinned(const void* p);
// true when `p` is device memory (not readable by host threads)
bool is_device(const void* p);

// Host rows -> device uint64 rows (row stride ldd).  Returns after the last chunk is queued on
// `s` (host work done; the device side completes in stream order).  *bytes += PCIe bytes.
// `bits` < 32: residues cross as a B-bit packed stream (groups of 32 values in B words; B from
// transfer_bits(p)); 32: as uint32.
cudaError_t upload(const uint64_t* h, size_t ldh, Region r, uint64_t* d, size_t ldd, int bits, cudaStream_t s,
                   uint64_t* bytes);

// Device uint64 rows (every value < 2^32) -> host rows; synchronous.  zero_rb > 0 also writes
// zeros at (i, j) for i < j < min(rows, (i / zero_rb + 1) * zero_rb) (the strict upper parts of
// the diagonal zero_rb-row blocks) without moving them.  *bytes += PCIe bytes.
cudaError_t download(const uint64_t* d, size_t ldd, Region r, uint64_t* h, size_t ldh, size_t zero_rb, int bits,
                     cudaStream_t s, uint64_t* bytes);

// Transfer width for residues mod p: the bit length of p - 1 (at least 8) when it is at most 24,
// else 32 (FSYRK_B200_PACK=0: always 32).
int transfer_bits(uint64_t p);

// c[i][j] <- (x[i][j] + beta * (c[i][j] mod p)) mod p on the lower triangle of rows [r0, r1)
// (x already reduced; c any uint64).  The accumulate step of the pinned-memory duplex path.
cudaError_t launch_acc_combine(const uint64_t* x, long long ldx, uint64_t* c, long long ldc, int r0, int r1,
                               const ModP& m, uint32_t beta, cudaStream_t s);

// Host-only pack -> unpack of a region through the worker pool (format check and host
// bandwidth probe; fsyrk_b200_hostio_roundtrip).  Returns the chunks that would go unnarrowed.
size_t roundtrip(const uint64_t* h, size_t ldh, Region r, int bits, uint64_t* out, size_t ldo, double* secs);

// Host seconds spent converting on the pool / waiting for staging slots (FSYRK_B200_IO_TRACE).
struct IoStats {
    double host = 0, wait = 0;
};
extern IoStats g_io_stats;

// Number of host threads used for narrowing / widening (FSYRK_B200_HOST_THREADS overrides).
int host_threads();

}  // namespace hio
}  // namespace fsyrk_b200

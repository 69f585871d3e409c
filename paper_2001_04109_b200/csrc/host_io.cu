// Host <-> device movement of the caller's matrices (see host_io.h for the why).
//
// Upload pipeline, chunk c of ~2 Mi elements (download is the mirror image):
//   host workers narrow their slice of chunk c (uint64 -> uint32, AVX2 + streaming stores)
//   into pinned slot c % kSlots; the calling thread, once all slices are in, queues
//   slot -> device staging (packed uint32 rows) and the widen kernel (-> uint64 rows), and
//   hands the workers the next slot as soon as the copy that last used it has finished.
// Workers stay inside one parallel region for the whole transfer and hand chunks over through
// spin-waited counters (no per-chunk thread wake-ups).
//
// Pinned callers also move a share of the rows unnarrowed, by DMA straight from / into their
// memory on a second copy stream: the host threads and the copy engine then finish together
// (FSYRK_B200_RAW_UP / FSYRK_B200_RAW_DOWN override the shares).
#include "host_io.h"

#include <immintrin.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

#include "elementwise.cuh"
#include "per_device.h"

namespace fsyrk_b200 {
namespace hio {

IoStats g_io_stats;

namespace {

size_t env_size(const char* name, size_t dflt) {
    const char* e = std::getenv(name);
    const long long v = e && *e ? std::atoll(e) : -1;
    return v >= 0 ? (size_t)v : dflt;
}
// elements per chunk (FSYRK_B200_CHUNK), streaming (cache-bypassing) stores into the slots
// (FSYRK_B200_NT_UP) and into the caller's C (FSYRK_B200_NT_DOWN)
// (defaults measured on the B200 box, profiles/r01/hostio.txt: 1 Mi-element chunks, streaming
// stores both ways)
const size_t kChunk = env_size("FSYRK_B200_CHUNK", size_t(1) << 20);
const bool kNtUp = env_size("FSYRK_B200_NT_UP", 2) != 0;
const bool kNtDown = env_size("FSYRK_B200_NT_DOWN", 2) != 0;
constexpr int kSlots = 4;
constexpr size_t kRawBlock = 256;  // rows per unnarrowed 2-D copy of a lower-triangle region

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

inline void cpu_relax() { _mm_pause(); }

// Worker threads that each run fn(worker index) once per region; start() returns at once,
// join() waits for every worker to leave fn.
class Workers {
  public:
    explicit Workers(int n) {
        for (int t = 0; t < n; ++t) th_.emplace_back([this, t] { loop(t); });
    }
    ~Workers() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int size() const { return (int)th_.size(); }
    void start(std::function<void(int)> fn) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = std::move(fn);
            left_.store((int)th_.size());
            ++gen_;
        }
        cv_.notify_all();
    }
    void join() {
        for (int spin = 0; left_.load(std::memory_order_acquire) != 0; ++spin)
            if (spin > 4096) std::this_thread::yield();
            else cpu_relax();
        std::lock_guard<std::mutex> lk(mu_);
        fn_ = nullptr;
    }

  private:
    void loop(int t) {
        unsigned long long seen = 0;
        for (;;) {
            std::function<void(int)>* fn;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                fn = &fn_;
            }
            (*fn)(t);
            left_.fetch_sub(1, std::memory_order_release);
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::function<void(int)> fn_;
    std::atomic<int> left_{0};
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

Workers& workers() {
    // the calling thread orchestrates; a forked child (whose copy has no threads) builds its own
    static Workers* w = nullptr;
    static pid_t owner = 0;
    if (!w || owner != getpid()) {
        w = new Workers(std::max(1, host_threads() - 1));  // the parent's copy is abandoned on purpose
        owner = getpid();
    }
    return *w;
}

// ---- conversions (AVX2 when the CPU has it) ----
template <bool NT>
__attribute__((target("avx2"))) uint64_t narrow_avx2(const uint64_t* s, uint32_t* o, size_t n) {
    size_t j = 0;
    uint64_t hi = 0;
    for (; j < n && (reinterpret_cast<uintptr_t>(o + j) & 31); ++j) {
        o[j] = (uint32_t)s[j];
        hi |= s[j];
    }
    const __m256i perm = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
    __m256i h = _mm256_setzero_si256();
    for (; j + 8 <= n; j += 8) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + j));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + j + 4));
        h = _mm256_or_si256(h, _mm256_or_si256(a, b));
        const __m256i pa = _mm256_permutevar8x32_epi32(a, perm), pb = _mm256_permutevar8x32_epi32(b, perm);
        const __m256i v = _mm256_permute2x128_si256(pa, pb, 0x20);
        if (NT) _mm256_stream_si256(reinterpret_cast<__m256i*>(o + j), v);
        else _mm256_store_si256(reinterpret_cast<__m256i*>(o + j), v);
    }
    alignas(32) uint64_t hv[4];
    _mm256_store_si256(reinterpret_cast<__m256i*>(hv), h);
    hi |= hv[0] | hv[1] | hv[2] | hv[3];
    for (; j < n; ++j) {
        o[j] = (uint32_t)s[j];
        hi |= s[j];
    }
    return hi >> 32;
}
uint64_t narrow_scalar(const uint64_t* s, uint32_t* o, size_t n) {
    uint64_t hi = 0;
    for (size_t j = 0; j < n; ++j) {
        o[j] = (uint32_t)s[j];
        hi |= s[j];
    }
    return hi >> 32;
}
template <bool NT>
__attribute__((target("avx2"))) void widen_avx2(const uint32_t* s, uint64_t* o, size_t n) {
    size_t j = 0;
    if (NT)
        for (; j < n && (reinterpret_cast<uintptr_t>(o + j) & 31); ++j) o[j] = s[j];
    for (; j + 8 <= n; j += 8) {
        const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + j));
        const __m256i lo = _mm256_cvtepu32_epi64(_mm256_castsi256_si128(v));
        const __m256i hi = _mm256_cvtepu32_epi64(_mm256_extracti128_si256(v, 1));
        if (NT) {
            _mm256_stream_si256(reinterpret_cast<__m256i*>(o + j), lo);
            _mm256_stream_si256(reinterpret_cast<__m256i*>(o + j + 4), hi);
        } else {
            _mm256_storeu_si256(reinterpret_cast<__m256i*>(o + j), lo);
            _mm256_storeu_si256(reinterpret_cast<__m256i*>(o + j + 4), hi);
        }
    }
    for (; j < n; ++j) o[j] = s[j];
}
void widen_scalar(const uint32_t* s, uint64_t* o, size_t n) {
    for (size_t j = 0; j < n; ++j) o[j] = s[j];
}
const bool g_avx2 = [] {
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx2") != 0;
}();
inline uint64_t narrow_run(const uint64_t* s, uint32_t* o, size_t n) {
    if (!g_avx2) return narrow_scalar(s, o, n);
    return kNtUp ? narrow_avx2<true>(s, o, n) : narrow_avx2<false>(s, o, n);
}
inline void widen_run(const uint32_t* s, uint64_t* o, size_t n) {
    if (!g_avx2) widen_scalar(s, o, n);
    else if (kNtDown) widen_avx2<true>(s, o, n);
    else widen_avx2<false>(s, o, n);
}

// ---- B-bit packing (B < 32): groups of 32 residues -> B little-endian 32-bit words ----
template <int B, size_t... T>
inline void pack32_impl(const uint32_t* v, uint32_t* w, std::index_sequence<T...>) {
    ((w[(T * B) / 32] |= v[T] << ((T * B) % 32),
      w[(T * B) / 32 + 1] |= ((T * B) % 32 + B > 32) ? v[T] >> ((32 - (T * B) % 32) & 31) : 0u),
     ...);
}
template <int B>
inline void pack32(const uint32_t* v, uint32_t* out) {
    uint32_t w[B + 1] = {};
    pack32_impl<B>(v, w, std::make_index_sequence<32>{});
    for (int i = 0; i < B; ++i) _mm_stream_si32(reinterpret_cast<int*>(out + i), (int)w[i]);
}
template <int B, size_t... T>
inline void unpack32_impl(const uint32_t* w, uint32_t* v, std::index_sequence<T...>) {
    constexpr uint32_t mask = (1u << B) - 1;
    ((v[T] = ((w[(T * B) / 32] >> ((T * B) % 32)) |
              (((T * B) % 32 + B > 32) ? w[(T * B) / 32 + 1] << ((32 - (T * B) % 32) & 31) : 0u)) &
             mask),
     ...);
}
template <int B>
inline void unpack32(const uint32_t* in, uint32_t* v) {
    uint32_t w[B + 1];
    for (int i = 0; i < B; ++i) w[i] = in[i];
    w[B] = 0;
    unpack32_impl<B>(w, v, std::make_index_sequence<32>{});
}

// Packs a worker's run of row segments (starting at a group boundary) into consecutive groups.
template <int B>
struct Packer {
    uint32_t v[32];
    int n = 0;
    uint32_t* out;
    uint64_t hi = 0;
    void push(const uint64_t* s, size_t cnt) {
        while (cnt) {
            if (n == 0 && cnt >= 32) {  // whole groups straight from the row
                for (; cnt >= 32; cnt -= 32, s += 32, out += B) {
                    uint64_t h = 0;
                    for (int t = 0; t < 32; ++t) {
                        h |= s[t];
                        v[t] = (uint32_t)s[t];
                    }
                    hi |= h;
                    pack32<B>(v, out);
                }
                continue;
            }
            const size_t t = std::min<size_t>(32 - n, cnt);
            for (size_t j = 0; j < t; ++j) {
                hi |= s[j];
                v[n + j] = (uint32_t)s[j];
            }
            n += (int)t;
            s += t;
            cnt -= t;
            if (n == 32) {
                pack32<B>(v, out);
                out += B;
                n = 0;
            }
        }
    }
    void flush() {
        if (!n) return;
        for (int t = n; t < 32; ++t) v[t] = 0;
        pack32<B>(v, out);
        out += B;
        n = 0;
    }
};
template <int B>
struct Unpacker {
    uint32_t v[32];
    int n = 32;  // values of v already handed out
    const uint32_t* in;
    void pull(uint64_t* o, size_t cnt) {
        while (cnt) {
            if (n == 32 && cnt >= 32) {
                for (; cnt >= 32; cnt -= 32, o += 32, in += B) {
                    unpack32<B>(in, v);
                    for (int t = 0; t < 32; ++t) _mm_stream_si64(reinterpret_cast<long long*>(o + t), (long long)v[t]);
                }
                continue;
            }
            if (n == 32) {
                unpack32<B>(in, v);
                in += B;
                n = 0;
            }
            const size_t t = std::min<size_t>(32 - n, cnt);
            for (size_t j = 0; j < t; ++j) _mm_stream_si64(reinterpret_cast<long long*>(o + j), (long long)v[n + j]);
            n += (int)t;
            o += t;
            cnt -= t;
        }
    }
};

// ---- staging ----
struct Slot {
    uint32_t* buf = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;  // a copy from / into buf may still be in flight
};
struct Staging {
    uint32_t* ptr = nullptr;
    size_t n = 0;
};

// Staging state of one device (streams, events and device buffers belong to the device that was
// current when they were made; a process may drive several GPUs): pinned slots with their copy
// events, the second copy stream for the unnarrowed share, packed words / uint32 rows.
struct DevIo {
    Slot slot[kSlots];
    cudaStream_t raw = nullptr;
    cudaEvent_t raw_done = nullptr, fork = nullptr;
    Staging dev32, devw;
};

DevIo& dev_io() { return per_device<DevIo>(); }

cudaError_t ensure_slots(DevIo& io, size_t cap) {
    if (!io.raw) {
        cudaError_t e = cudaStreamCreateWithFlags(&io.raw, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&io.raw_done, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&io.fork, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    for (auto& s : io.slot) {
        if (!s.ev) {
            cudaError_t e = cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
        if (s.cap >= cap) continue;
        if (s.pending) {
            cudaError_t e = cudaEventSynchronize(s.ev);
            if (e != cudaSuccess) return e;
            s.pending = false;
        }
        if (s.buf) cudaFreeHost(s.buf);
        s.buf = nullptr;
        s.cap = 0;
        cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&s.buf), cap * 4, cudaHostAllocDefault);
        if (e != cudaSuccess) return e;
        s.cap = cap;
    }
    return cudaSuccess;
}

cudaError_t acquire(Slot& s) {
    if (!s.pending) return cudaSuccess;
    s.pending = false;
    const double t0 = now_s();
    cudaError_t e = cudaEventSynchronize(s.ev);
    g_io_stats.wait += now_s() - t0;
    return e;
}

cudaError_t ensure_devw(DevIo& io, size_t n) {
    if (io.devw.n >= n) return cudaSuccess;
    if (io.devw.ptr) cudaFree(io.devw.ptr);
    io.devw.ptr = nullptr;
    io.devw.n = 0;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&io.devw.ptr), n * 4);
    if (e == cudaSuccess) io.devw.n = n;
    return e;
}

cudaError_t ensure_dev32(DevIo& io, size_t n) {
    if (io.dev32.n >= n) return cudaSuccess;
    if (io.dev32.ptr) cudaFree(io.dev32.ptr);
    io.dev32.ptr = nullptr;
    io.dev32.n = 0;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&io.dev32.ptr), n * 4);
    if (e == cudaSuccess) io.dev32.n = n;
    return e;
}

struct Chunk {
    size_t r0, r1, off, len;  // rows [r0, r1), packed elements [off, off + len)
};

std::vector<Chunk> make_chunks(const Region& r, size_t rows, size_t cap) {
    std::vector<Chunk> out;
    for (size_t r0 = 0; r0 < rows;) {
        size_t r1 = r0, len = 0;
        while (r1 < rows && (len == 0 || len + r.width(r1) <= cap)) len += r.width(r1++);
        out.push_back(Chunk{r0, r1, r.offset(r0), len});
        r0 = r1;
    }
    return out;
}

// Worker w's slice of a chunk, walked row by row: fn(row, c0, c1, packed index of (row, c0)).
// Slices start at multiples of 32 chunk elements (whole groups of the bit-packed format).
template <class Fn>
void slice(const Region& r, const Chunk& ch, int w, int nw, Fn&& fn) {
    const size_t b = ch.off + ch.len * w / nw / 32 * 32;
    const size_t e = w + 1 == nw ? ch.off + ch.len : ch.off + ch.len * (w + 1) / nw / 32 * 32;
    if (b >= e) return;
    size_t lo = ch.r0, hi = ch.r1 - 1;  // first row whose packed range contains b
    while (lo < hi) {
        const size_t mid = (lo + hi + 1) / 2;
        if (r.offset(mid) <= b) lo = mid;
        else hi = mid - 1;
    }
    for (size_t i = lo, pos = b; pos < e; ++i) {
        const size_t rb = r.offset(i), c0 = pos - rb, c1 = std::min(r.width(i), e - rb);
        fn(i, c0, c1, pos);
        pos = rb + c1;
    }
}

// Worker entry points per bit width (8..24), dispatched through tables.
using PackFn = uint64_t (*)(const Region&, const Chunk&, int, int, const uint64_t*, size_t, uint32_t*);
using UnpackFn = void (*)(const Region&, const Chunk&, int, int, const uint32_t*, uint64_t*, size_t, size_t);
template <int B>
uint64_t pack_slice(const Region& r, const Chunk& ch, int w, int nw, const uint64_t* h, size_t ldh, uint32_t* words) {
    Packer<B> pk;
    pk.out = words + (ch.len * w / nw / 32) * B;
    slice(r, ch, w, nw, [&](size_t i, size_t c0, size_t c1, size_t) { pk.push(h + i * ldh + c0, c1 - c0); });
    pk.flush();
    return pk.hi >> B;
}
template <int B>
void unpack_slice(const Region& r, const Chunk& ch, int w, int nw, const uint32_t* words, uint64_t* h, size_t ldh,
                  size_t zero_rb) {
    Unpacker<B> up;
    up.in = words + (ch.len * w / nw / 32) * B;
    slice(r, ch, w, nw, [&](size_t i, size_t c0, size_t c1, size_t) {
        uint64_t* o = h + i * ldh;
        up.pull(o + c0, c1 - c0);
        if (zero_rb && c1 == r.width(i)) {
            const size_t end = std::min(r.rows, (i / zero_rb + 1) * zero_rb);
            if (end > i + 1) std::memset(o + i + 1, 0, (end - i - 1) * 8);
        }
    });
}
constexpr int kMinBits = 8, kMaxBits = 24;
template <int... Bs>
struct Tables {
    static constexpr PackFn pack[] = {&pack_slice<Bs>...};
    static constexpr UnpackFn unpack[] = {&unpack_slice<Bs>...};
};
using Tab = Tables<8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23, 24>;

size_t packed_words(size_t len, int bits) { return bits >= 32 ? len : (len + 31) / 32 * (size_t)bits; }

// Chunks through the workers.  prepare(c) (calling thread) makes chunk c's slot usable,
// work(c, w, nw) is worker w's share, finish(c) (calling thread) runs once every share is in.
// The calling thread keeps up to `ahead` chunks published beyond the one it finishes.
template <class Prep, class Work, class Fin>
cudaError_t run_chunks(size_t nchunks, size_t ahead, Prep&& prepare, Work&& work, Fin&& finish) {
    if (nchunks == 0) return cudaSuccess;
    Workers& W = workers();
    const int nw = W.size();
    std::unique_ptr<std::atomic<int>[]> done(new std::atomic<int>[nchunks]);
    for (size_t c = 0; c < nchunks; ++c) done[c].store(0);
    std::atomic<size_t> ready{0};  // chunks [0, ready) may be worked on
    std::atomic<bool> abort{false};
    const double t0 = now_s();
    W.start([&](int w) {
        for (size_t c = 0; c < nchunks; ++c) {
            for (int spin = 0; ready.load(std::memory_order_acquire) <= c; ++spin) {
                if (abort.load(std::memory_order_relaxed)) return;
                if (spin > 1024) std::this_thread::yield();
                else cpu_relax();
            }
            work(c, w, nw);
            _mm_sfence();  // streaming stores drained before the slot is handed to the copy engine
            done[c].fetch_add(1, std::memory_order_release);
        }
    });
    cudaError_t err = cudaSuccess;
    size_t published = 0;
    for (size_t c = 0; c < nchunks && err == cudaSuccess; ++c) {
        while (published < nchunks && published <= c + ahead && err == cudaSuccess) {
            err = prepare(published);
            if (err == cudaSuccess) ready.store(++published, std::memory_order_release);
        }
        if (err != cudaSuccess) break;
        for (int spin = 0; done[c].load(std::memory_order_acquire) < nw; ++spin)
            if (spin > 1024) std::this_thread::yield();
            else cpu_relax();
        err = finish(c);
    }
    if (err != cudaSuccess) abort.store(true);
    W.join();
    g_io_stats.host += now_s() - t0;
    return err;
}

double env_frac(const char* name, double dflt) {
    const char* e = std::getenv(name);
    if (!e) return dflt;
    const double v = std::atof(e);
    return v < 0 ? 0 : v > 1 ? 1 : v;
}

// First row of the unnarrowed tail: about `frac` of the region's elements.
size_t raw_split(const Region& r, double frac) {
    if (frac <= 0) return r.rows;
    const size_t total = r.offset(r.rows), keep = (size_t)((1.0 - frac) * (double)total);
    size_t lo = 0, hi = r.rows;
    while (lo < hi) {  // smallest row with offset >= keep
        const size_t mid = (lo + hi) / 2;
        if (r.offset(mid) < keep) lo = mid + 1;
        else hi = mid;
    }
    if (r.lower) lo = lo / kRawBlock * kRawBlock;  // whole row blocks
    return lo;
}

// Unnarrowed copies of rows [r0, rows) (row blocks of kRawBlock for a lower region).
cudaError_t raw_copy(const Region& r, size_t r0, uint64_t* dst, size_t ldd_dst, const uint64_t* src, size_t ld_src,
                     cudaMemcpyKind kind, cudaStream_t s, uint64_t* bytes) {
    if (r0 >= r.rows) return cudaSuccess;
    if (!r.lower) {
        *bytes += (r.rows - r0) * r.cols * 8;
        return cudaMemcpy2DAsync(dst + r0 * ldd_dst, ldd_dst * 8, src + r0 * ld_src, ld_src * 8, r.cols * 8,
                                 r.rows - r0, kind, s);
    }
    for (size_t b0 = r0; b0 < r.rows; b0 += kRawBlock) {
        const size_t b1 = std::min(r.rows, b0 + kRawBlock);
        cudaError_t e = cudaMemcpy2DAsync(dst + b0 * ldd_dst, ldd_dst * 8, src + b0 * ld_src, ld_src * 8, b1 * 8,
                                          b1 - b0, kind, s);
        if (e != cudaSuccess) return e;
        *bytes += (b1 - b0) * b1 * 8;
    }
    return cudaSuccess;
}

__global__ void widen_kernel(const uint32_t* __restrict__ src, size_t off0, int r0, int r1, int cols, int lower,
                             uint64_t* __restrict__ d, long long ldd) {
    for (int i = r0 + blockIdx.y; i < r1; i += gridDim.y) {
        const size_t w = lower ? (size_t)i + 1 : (size_t)cols;
        const size_t o = (lower ? (size_t)i * (i + 1) / 2 : (size_t)i * cols) - off0;
        for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < w; j += (size_t)gridDim.x * blockDim.x)
            d[i * ldd + j] = src[o + j];
    }
}

__global__ void narrow_kernel(const uint64_t* __restrict__ d, long long ldd, int rows, int cols, int lower,
                              uint32_t* __restrict__ dst) {
    for (int i = blockIdx.y; i < rows; i += gridDim.y) {
        const size_t w = lower ? (size_t)i + 1 : (size_t)cols;
        const size_t o = lower ? (size_t)i * (i + 1) / 2 : (size_t)i * cols;
        for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < w; j += (size_t)gridDim.x * blockDim.x)
            dst[o + j] = (uint32_t)d[i * ldd + j];
    }
}

// Bit-packed transfer format on the device: value t of group g sits at bits [t B, t B + B) of
// words [g B, g B + B).
__global__ void unpack_kernel(const uint32_t* __restrict__ words, size_t n, int B, uint32_t* __restrict__ out) {
    const uint32_t mask = (1u << B) - 1;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x) {
        const size_t g = idx / 32;
        const unsigned bit = (unsigned)(idx % 32) * B;
        const size_t wi = g * B + bit / 32;
        const unsigned sh = bit % 32;
        uint32_t v = words[wi] >> sh;
        if (sh + B > 32) v |= words[wi + 1] << (32 - sh);
        out[idx] = v & mask;
    }
}
__global__ void pack_kernel(const uint32_t* __restrict__ vals, size_t n, int B, uint32_t* __restrict__ words,
                            size_t nwords) {
    for (size_t wi = blockIdx.x * (size_t)blockDim.x + threadIdx.x; wi < nwords; wi += (size_t)gridDim.x * blockDim.x) {
        const size_t g = wi / B;
        const int b0 = (int)(wi % B) * 32;  // first bit of the word inside its group
        uint32_t w = 0;
        for (int t = b0 / B; t < 32 && t * B < b0 + 32; ++t) {
            const size_t idx = g * 32 + t;
            const uint32_t v = idx < n ? vals[idx] : 0;
            const int off = t * B - b0;
            w |= off >= 0 ? v << off : v >> -off;
        }
        words[wi] = w;
    }
}

__global__ void acc_combine_kernel(const uint64_t* __restrict__ x, long long ldx, uint64_t* __restrict__ c,
                                   long long ldc, int r0, int r1, ModP m, uint32_t beta) {
    for (int i = r0 + blockIdx.y; i < r1; i += gridDim.y)
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= i; j += gridDim.x * blockDim.x) {
            const uint32_t ci = mod_u64(c[(long long)i * ldc + j], m);
            c[(long long)i * ldc + j] = addm((uint32_t)x[(long long)i * ldx + j], mulm(ci, beta, m), m.p);
        }
}

dim3 rows_grid(size_t rows, size_t width) {
    const unsigned gx = (unsigned)std::min<size_t>(64, (width + 255) / 256);
    const unsigned gy = (unsigned)std::min<size_t>(65535, std::max<size_t>(1, rows));
    return dim3(std::max(1u, gx), gy);
}

}  // namespace

int host_threads() {
    static const int n = [] {
        if (const char* e = std::getenv("FSYRK_B200_HOST_THREADS")) {
            const int v = std::atoi(e);
            if (v > 0) return std::min(v, 256);
        }
        const int hw = (int)std::thread::hardware_concurrency();
        // a library should not claim a whole large host by default: at most 16 worker threads
        // (the B200 box has 16 cores; FSYRK_B200_HOST_THREADS raises or lowers it)
        return std::max(2, std::min(hw, 16));
    }();
    return n;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

int transfer_bits(uint64_t p) {
    static const bool pack = env_size("FSYRK_B200_PACK", 1) != 0;
    int b = 0;
    while (b < 64 && ((p - 1) >> b) != 0) ++b;  // bit length of the largest residue
    if (!pack || b > kMaxBits) return 32;
    return std::max(b, kMinBits);
}

bool is_device(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice;
}

cudaError_t upload(const uint64_t* h, size_t ldh, Region r, uint64_t* d, size_t ldd, int bits, cudaStream_t s,
                   uint64_t* bytes) {
    const size_t total = r.offset(r.rows);
    if (total == 0) return cudaSuccess;
    DevIo& io = dev_io();
    if (bits < 32 && (bits < kMinBits || bits > kMaxBits)) bits = 32;
    const size_t cap = std::max(kChunk, r.lower ? r.rows : r.cols);
    cudaError_t e;
    if ((e = ensure_slots(io, cap)) != cudaSuccess) return e;
    if ((e = ensure_dev32(io, total)) != cudaSuccess) return e;
    // pinned caller: the tail rows go unnarrowed on the second copy stream, queued first
    const size_t split = is_pinned(h) ? raw_split(r, env_frac("FSYRK_B200_RAW_UP", 0.12)) : r.rows;
    if (split < r.rows) {
        if ((e = cudaEventRecord(io.fork, s)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(io.raw, io.fork, 0)) != cudaSuccess) return e;
        if ((e = raw_copy(r, split, d, ldd, h, ldh, cudaMemcpyHostToDevice, io.raw, bytes)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(io.raw_done, io.raw)) != cudaSuccess) return e;
    }
    const std::vector<Chunk> chunks = make_chunks(r, split, cap);
    std::vector<size_t> wofs(chunks.size() + 1, 0);  // packed words of each chunk in the device word buffer
    for (size_t c = 0; c < chunks.size(); ++c) wofs[c + 1] = wofs[c] + packed_words(chunks[c].len, bits);
    if (bits < 32 && (e = ensure_devw(io, wofs.back())) != cudaSuccess) return e;
    const PackFn packer = bits < 32 ? Tab::pack[bits - kMinBits] : nullptr;
    const size_t nw = (size_t)workers().size();
    std::vector<uint64_t> high(chunks.size() * nw, 0);  // out-of-range bits seen, per chunk and worker
    e = run_chunks(
        chunks.size(), kSlots - 1, [&](size_t c) { return acquire(io.slot[c % kSlots]); },
        [&](size_t c, int w, int nwk) {
            const Chunk& ch = chunks[c];
            uint64_t hi = 0;
            if (packer) {
                hi = packer(r, ch, w, nwk, h, ldh, io.slot[c % kSlots].buf);
            } else {
                uint32_t* dst = io.slot[c % kSlots].buf - ch.off;
                slice(r, ch, w, nwk, [&](size_t i, size_t c0, size_t c1, size_t pos) {
                    hi |= narrow_run(h + i * ldh + c0, dst + pos, c1 - c0);
                });
            }
            high[c * nw + (size_t)w] = hi;
        },
        [&](size_t c) -> cudaError_t {
            const Chunk& ch = chunks[c];
            uint64_t hi = 0;
            for (size_t w = 0; w < nw; ++w) hi |= high[c * nw + w];
            cudaError_t e2;
            if (hi) {  // a value that does not fit the transfer width (non-canonical input): unnarrowed
                const size_t wd = r.width(ch.r1 - 1);
                *bytes += (ch.r1 - ch.r0) * wd * 8;
                return cudaMemcpy2DAsync(d + ch.r0 * ldd, ldd * 8, h + ch.r0 * ldh, ldh * 8, wd * 8, ch.r1 - ch.r0,
                                         cudaMemcpyHostToDevice, s);
            }
            Slot& sl = io.slot[c % kSlots];
            uint32_t* d32 = io.dev32.ptr + ch.off;
            const size_t nwords = wofs[c + 1] - wofs[c];
            uint32_t* dst = bits < 32 ? io.devw.ptr + wofs[c] : d32;
            if ((e2 = cudaMemcpyAsync(dst, sl.buf, nwords * 4, cudaMemcpyHostToDevice, s)) != cudaSuccess) return e2;
            if ((e2 = cudaEventRecord(sl.ev, s)) != cudaSuccess) return e2;
            sl.pending = true;
            *bytes += nwords * 4;
            if (bits < 32) {
                unpack_kernel<<<(unsigned)std::min<size_t>(4096, (ch.len + 255) / 256), 256, 0, s>>>(dst, ch.len, bits,
                                                                                                    d32);
                if ((e2 = cudaGetLastError()) != cudaSuccess) return e2;
            }
            widen_kernel<<<rows_grid(ch.r1 - ch.r0, r.width(ch.r1 - 1)), 256, 0, s>>>(
                d32, ch.off, (int)ch.r0, (int)ch.r1, (int)r.cols, r.lower ? 1 : 0, d, (long long)ldd);
            return cudaGetLastError();
        });
    if (e != cudaSuccess) return e;
    if (split < r.rows) e = cudaStreamWaitEvent(s, io.raw_done, 0);
    return e;
}

cudaError_t download(const uint64_t* d, size_t ldd, Region r, uint64_t* h, size_t ldh, size_t zero_rb, int bits,
                     cudaStream_t s, uint64_t* bytes) {
    const size_t total = r.offset(r.rows);
    if (total == 0) return cudaSuccess;
    DevIo& io = dev_io();
    if (bits < 32 && (bits < kMinBits || bits > kMaxBits)) bits = 32;
    const size_t cap = std::max(kChunk, r.lower ? r.rows : r.cols);
    cudaError_t e;
    if ((e = ensure_slots(io, cap)) != cudaSuccess) return e;
    if ((e = ensure_dev32(io, total)) != cudaSuccess) return e;
    const size_t split = is_pinned(h) ? raw_split(r, env_frac("FSYRK_B200_RAW_DOWN", 0.0)) : r.rows;
    if (split < r.rows) {
        // the unnarrowed row blocks carry their diagonal blocks' strict upper parts: clear them on
        // the device first when the caller expects zeros there
        if (zero_rb && r.lower &&
            (e = launch_zero_upper(const_cast<uint64_t*>(d), (long long)ldd, (int)r.rows, (int)zero_rb, s)) !=
                cudaSuccess)
            return e;
        if ((e = cudaEventRecord(io.fork, s)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(io.raw, io.fork, 0)) != cudaSuccess) return e;
        if ((e = raw_copy(r, split, h, ldh, d, ldd, cudaMemcpyDeviceToHost, io.raw, bytes)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(io.raw_done, io.raw)) != cudaSuccess) return e;
    }
    const std::vector<Chunk> chunks = make_chunks(r, split, cap);
    std::vector<size_t> wofs(chunks.size() + 1, 0);
    for (size_t c = 0; c < chunks.size(); ++c) wofs[c + 1] = wofs[c] + packed_words(chunks[c].len, bits);
    if (bits < 32 && (e = ensure_devw(io, wofs.back())) != cudaSuccess) return e;
    if (!chunks.empty()) {
        narrow_kernel<<<rows_grid(split, r.lower ? split : r.cols), 256, 0, s>>>(
            d, (long long)ldd, (int)split, (int)r.cols, r.lower ? 1 : 0, io.dev32.ptr);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (bits < 32)
            for (size_t c = 0; c < chunks.size(); ++c) {
                const size_t nwords = wofs[c + 1] - wofs[c];
                pack_kernel<<<(unsigned)std::min<size_t>(4096, (nwords + 255) / 256), 256, 0, s>>>(
                    io.dev32.ptr + chunks[c].off, chunks[c].len, bits, io.devw.ptr + wofs[c], nwords);
            }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    auto issue = [&](size_t c) -> cudaError_t {
        Slot& sl = io.slot[c % kSlots];
        cudaError_t e2 = acquire(sl);
        if (e2 != cudaSuccess) return e2;
        const size_t nwords = wofs[c + 1] - wofs[c];
        const uint32_t* src = bits < 32 ? io.devw.ptr + wofs[c] : io.dev32.ptr + chunks[c].off;
        e2 = cudaMemcpyAsync(sl.buf, src, nwords * 4, cudaMemcpyDeviceToHost, s);
        if (e2 != cudaSuccess) return e2;
        e2 = cudaEventRecord(sl.ev, s);
        sl.pending = true;
        *bytes += nwords * 4;
        return e2;
    };
    for (size_t c = 0; c < chunks.size() && c < (size_t)kSlots; ++c)
        if ((e = issue(c)) != cudaSuccess) return e;
    const UnpackFn unpacker = bits < 32 ? Tab::unpack[bits - kMinBits] : nullptr;
    e = run_chunks(
        chunks.size(), 1, [&](size_t c) { return acquire(io.slot[c % kSlots]); },
        [&](size_t c, int w, int nw) {
            const Chunk& ch = chunks[c];
            if (unpacker) {
                unpacker(r, ch, w, nw, io.slot[c % kSlots].buf, h, ldh, zero_rb);
                return;
            }
            const uint32_t* src = io.slot[c % kSlots].buf - ch.off;
            slice(r, ch, w, nw, [&](size_t i, size_t c0, size_t c1, size_t pos) {
                uint64_t* o = h + i * ldh;
                widen_run(src + pos, o + c0, c1 - c0);
                if (zero_rb && c1 == r.width(i)) {  // the slice holding the row's end clears its block's upper part
                    const size_t end = std::min(r.rows, (i / zero_rb + 1) * zero_rb);
                    if (end > i + 1) std::memset(o + i + 1, 0, (end - i - 1) * 8);
                }
            });
        },
        [&](size_t c) { return c + kSlots < chunks.size() ? issue(c + kSlots) : cudaSuccess; });
    if (e != cudaSuccess) return e;
    if (split < r.rows) e = cudaEventSynchronize(io.raw_done);
    return e;
}

size_t roundtrip(const uint64_t* h, size_t ldh, Region r, int bits, uint64_t* out, size_t ldo, double* secs) {
    if (bits < 32 && (bits < kMinBits || bits > kMaxBits)) bits = 32;
    const size_t cap = std::max(kChunk, r.lower ? r.rows : r.cols);
    const std::vector<Chunk> chunks = make_chunks(r, r.rows, cap);
    const PackFn packer = bits < 32 ? Tab::pack[bits - kMinBits] : nullptr;
    const UnpackFn unpacker = bits < 32 ? Tab::unpack[bits - kMinBits] : nullptr;
    std::vector<uint32_t> buf(cap + 64);
    const size_t nw = (size_t)workers().size();
    std::vector<uint64_t> high(nw);
    size_t raw = 0;
    secs[0] = secs[1] = 0;
    auto none = [](size_t) { return cudaSuccess; };
    for (const Chunk& ch : chunks) {
        const Chunk* pc = &ch;
        double t0 = now_s();
        run_chunks(
            1, 0, none,
            [&](size_t, int w, int nwk) {
                uint64_t hi = 0;
                if (packer) {
                    hi = packer(r, *pc, w, nwk, h, ldh, buf.data());
                } else {
                    uint32_t* dst = buf.data() - pc->off;
                    slice(r, *pc, w, nwk, [&](size_t i, size_t c0, size_t c1, size_t pos) {
                        hi |= narrow_run(h + i * ldh + c0, dst + pos, c1 - c0);
                    });
                }
                high[(size_t)w] = hi;
            },
            none);
        double t1 = now_s();
        uint64_t hi = 0;
        for (uint64_t x : high) hi |= x;
        raw += hi != 0;
        run_chunks(
            1, 0, none,
            [&](size_t, int w, int nwk) {
                if (unpacker) {
                    unpacker(r, *pc, w, nwk, buf.data(), out, ldo, 0);
                    return;
                }
                const uint32_t* src = buf.data() - pc->off;
                slice(r, *pc, w, nwk, [&](size_t i, size_t c0, size_t c1, size_t pos) {
                    widen_run(src + pos, out + i * ldo + c0, c1 - c0);
                });
            },
            none);
        secs[0] += t1 - t0;
        secs[1] += now_s() - t1;
    }
    return raw;
}

cudaError_t launch_acc_combine(const uint64_t* x, long long ldx, uint64_t* c, long long ldc, int r0, int r1,
                               const ModP& m, uint32_t beta, cudaStream_t s) {
    if (r1 <= r0) return cudaSuccess;
    acc_combine_kernel<<<rows_grid(r1 - r0, r1), 256, 0, s>>>(x, ldx, c, ldc, r0, r1, m, beta);
    return cudaGetLastError();
}

}  // namespace hio
}  // namespace fsyrk_b200

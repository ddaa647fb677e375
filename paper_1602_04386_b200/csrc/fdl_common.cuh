// fdl_common.cuh -- internal helpers of libfiedler (product path, sm_100a).
// Nothing here is shared with oracle/ (task rule 3): the counter-based
// generator below is this side's own implementation of DESIGN.md reading R6.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <chrono>
#include <initializer_list>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/fiedler.h"

namespace fdl {

// ----------------------------------------------------------------- errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define FDL_CK(call)                                                                      \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            throw ::fdl::Error(e_ == cudaErrorMemoryAllocation ? FIEDLER_ERR_NOMEM        \
                                                               : FIEDLER_ERR_CUDA,        \
                               std::string(#call) + ": " + cudaGetErrorString(e_) +       \
                                   " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
    } while (0)

// Every kernel launch site is followed by FDL_LAUNCH_CK(), which also counts
// the launch (reported as fiedler_info.setup_launches / launches).
extern thread_local long long g_launch_count;
#define FDL_LAUNCH_CK()                 \
    do {                                \
        ::fdl::g_launch_count++;        \
        FDL_CK(cudaGetLastError());     \
    } while (0)

#define FDL_REQUIRE(cond, code, msg)                                                      \
    do {                                                                                  \
        if (!(cond)) throw ::fdl::Error((code), (msg));                                   \
    } while (0)

// ----------------------------------------------------------------- tracing
// FIEDLER_TRACE=1 in the environment: every trace_mark() synchronises the
// stream and prints the wall time since the previous mark to stderr
// (diagnostics only; off by default, zero cost when off).
bool trace_enabled();
void trace_mark(cudaStream_t st, const char *what);

// ----------------------------------------------------------------- memory
// Small-buffer arena of one fiedler_create: while a create runs, buffers of at
// most kArenaMaxBytes are carved from one slab by a bump pointer and never
// reused; their frees are no-ops and the slab goes with the handle.  The setup
// makes ~40 small allocations per level (counts, flags, the arrays of the
// small levels); as pool calls they cost host time that left the device idle
// between the small levels' kernels.
constexpr size_t kArenaMaxBytes = (size_t)1 << 20;
struct SmallArena {
    char *base = nullptr;
    size_t cap = 0, off = 0;
    void *take(size_t b) {
        const size_t r = (b + 255) & ~(size_t)255;
        if (!base || off + r > cap) return nullptr;
        void *p = base + off;
        off += r;
        return p;
    }
};
extern std::atomic<long long> g_alloc_ns, g_alloc_calls, g_free_ns, g_free_calls;   // FIEDLER_ALLOC_STATS
bool alloc_stats_enabled();
extern thread_local SmallArena *tl_arena;   // set by fiedler_create for its duration

// Stream-ordered device buffer (cudaMallocAsync pool; capture-safe frees are
// never issued inside a captured region), or a piece of the create's arena.
struct DBuf {
    void *p = nullptr;
    size_t bytes = 0;
    cudaStream_t s = nullptr;
    bool in_arena = false;
    DBuf() = default;
    DBuf(size_t b, cudaStream_t st) { alloc(b, st); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept { *this = std::move(o); }
    DBuf &operator=(DBuf &&o) noexcept {
        if (this != &o) {
            release();
            p = o.p; bytes = o.bytes; s = o.s; in_arena = o.in_arena;
            o.p = nullptr; o.bytes = 0; o.in_arena = false;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t b, cudaStream_t st) {
        release();
        s = st;
        bytes = b;
        if (!b) return;
        if (tl_arena && b <= kArenaMaxBytes && (p = tl_arena->take(b))) {
            in_arena = true;
            return;
        }
        if (alloc_stats_enabled()) {
            const auto t0 = std::chrono::steady_clock::now();
            FDL_CK(cudaMallocAsync(&p, b, st));
            g_alloc_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
            g_alloc_calls++;
            return;
        }
        FDL_CK(cudaMallocAsync(&p, b, st));
    }
    void release() noexcept {
        if (p && !in_arena) {
            if (alloc_stats_enabled()) {
                const auto t0 = std::chrono::steady_clock::now();
                cudaFreeAsync(p, s);
                g_free_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
                g_free_calls++;
            } else {
                cudaFreeAsync(p, s);
            }
        }
        p = nullptr;
        bytes = 0;
        in_arena = false;
    }
    template <class T> T *as() const { return static_cast<T *>(p); }
};

// ----------------------------------------------------------------- generator (R6)
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
constexpr uint64_t kTagMatch = 0x6D61746368000000ULL;  // "match"
constexpr uint64_t kTagColor = 0x636F6C6F72000000ULL;  // "color"
constexpr uint64_t kTagRand = 0x72616E6400000000ULL;   // "rand"

__host__ __device__ __forceinline__ uint64_t salt_match(uint64_t seed, int level) {
    return splitmix64(seed ^ (kTagMatch + (uint64_t)level));
}
__host__ __device__ __forceinline__ uint64_t salt_color(uint64_t seed, int level) {
    return splitmix64(seed ^ (kTagColor + (uint64_t)level));
}
// tie-break hash of the undirected edge {a, b} (R2)
__device__ __forceinline__ uint64_t edge_hash(uint64_t salt, int a, int b) {
    uint64_t lo = (uint64_t)(unsigned)min(a, b), hi = (uint64_t)(unsigned)max(a, b);
    return splitmix64(salt ^ ((lo << 32) | hi));
}

// ----------------------------------------------------------------- launch helpers
constexpr int kNumSMs = 148;

// Per-device caches of launch configurations and function attributes (each
// device needs its own cudaFuncSetAttribute calls).  Lock-free: racing threads
// compute the same value.
constexpr int kMaxDevices = 64;
inline int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
    return d;
}
using DeviceCache = std::atomic<int>[kMaxDevices];
inline int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }
inline int grid_for(int64_t threads, int block = 256, int cap = kNumSMs * 32) {
    int64_t g = (threads + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }


// ----------------------------------------------------------------- primitives (fdl_prims.cu)
// Exclusive prefix sum of int32; `total` (device, may be null) receives the sum.
void scan_exclusive(const int *in, int *out, int64_t n, int *total, cudaStream_t st);

// Small device -> host readbacks (counts, sizes, flags) of the setup: the
// pieces are copied into pinned host memory and the host polls an event, so a
// round trip costs a few microseconds of device idle time (a pageable copy +
// cudaStreamSynchronize cost ~40 us each).  Waits for all prior work on st.
struct ReadPiece {
    void *dst;
    const void *src;
    size_t bytes;
};
void readback(cudaStream_t st, std::initializer_list<ReadPiece> pieces);
void readback(cudaStream_t st, const std::vector<ReadPiece> &pieces);
// the same wait without copies
void host_wait(cudaStream_t st);
// Stream-ordered copy of a small host array to the device without a stream
// synchronisation (pinned staging, fdl_prims.cu); src may be reused on return.
void upload(cudaStream_t st, void *dst, const void *src, size_t bytes);
// Stable LSD radix sort of (key, value) pairs on bits [0, bits); result in keys/vals.
void radix_sort_u32_i32(unsigned *keys, int *vals, int64_t n, int bits, cudaStream_t st);
// stable sort of the vertices by colour (< 256 colours): perm, inv, degree in sorted order, segment starts
void colour_sort(const int *color, int64_t n, int ncolors, const int *rp, int *perm, int *inv, int *degp,
                 int *segstart, cudaStream_t st);
void radix_sort_u64_i32(unsigned long long *keys, int *vals, int64_t n, int bits, cudaStream_t st);
// Stream compaction: out[k] = (in ? in[i] : i) for the k-th i in [0, n) with
// flags[i] != 0 (order kept); *d_count (device) = number kept.  flags are 0/1.
void compact_flagged(const int *in, const int *flags, int64_t n, int *out, int *d_count,
                     cudaStream_t st);
// Device-wide max of an int array (n >= 1) into *out (device).
void reduce_max_i32(const int *in, int64_t n, int *out, cudaStream_t st);

inline int bits_for(int64_t maxval) {  // bits to represent values in [0, maxval]
    int b = 0;
    while (b < 63 && (int64_t(1) << b) <= maxval) b++;
    return b < 1 ? 1 : b;
}

}  // namespace fdl

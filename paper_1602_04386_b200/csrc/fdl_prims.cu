// fdl_prims.cu -- hand-written device primitives: exclusive scan (single pass,
// decoupled look-back, 16384-element tiles, vectorised int4 traffic) and a stable LSD radix
// sort (8-bit digits, 8192-element tiles, warp __match_any_sync ranking).
// Used by the aggregate numbering (prefix scan of leader flags), work-list and
// CSR offset scans everywhere, the Galerkin product's long-row path (two-key
// radix sort) and the multicolour layout (sort by colour).
#include <algorithm>
#include <mutex>
#include <climits>
#include <cstring>

#include "fdl_common.cuh"

namespace fdl {

// =============================================================== scan
// 16 items per thread (4 x int4): 16384-element tiles keep the look-back chain
// short (one inclusive-prefix hop covers up to 32 tiles = 512 K elements);
// with 4096-element tiles the chain of hops, not bandwidth, bounded the scan
constexpr int kScanThreads = 1024;
#ifndef FDL_SCAN_ITEMS
#define FDL_SCAN_ITEMS 16
#endif
constexpr int kScanItems = FDL_SCAN_ITEMS;
static_assert(kScanItems % 4 == 0, "scan items come in int4 groups");
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int warp_incl_scan(int v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane_id() >= o) v += t;
    }
    return v;
}

// Block-wide exclusive scan of one int per thread; returns the block total.
__device__ __forceinline__ int block_excl_scan(int v, int &total) {
    __shared__ int s_warp[32];
    __shared__ int s_total;
    int incl = warp_incl_scan(v);
    int w = threadIdx.x >> 5;
    if (lane_id() == 31) s_warp[w] = incl;
    __syncthreads();
    if (w == 0) {
        int nw = blockDim.x >> 5;
        int x = lane_id() < nw ? s_warp[lane_id()] : 0;
        int xi = warp_incl_scan(x);
        if (lane_id() < nw) s_warp[lane_id()] = xi - x;
    }
    __syncthreads();
    int res = incl - v + s_warp[w];
    if (threadIdx.x == blockDim.x - 1) s_total = res + v;
    __syncthreads();
    total = s_total;
    __syncthreads();
    return res;
}

__device__ __forceinline__ void load4(const int *in, int64_t n, int64_t i, int x[4]) {
    if (i + 3 < n && ((reinterpret_cast<uintptr_t>(in + i) & 15) == 0)) {
        int4 v = *reinterpret_cast<const int4 *>(in + i);
        x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else {
#pragma unroll
        for (int k = 0; k < 4; k++) x[k] = (i + k < n) ? in[i + k] : 0;
    }
}

// Single-pass scan with decoupled look-back: tiles take their index from a
// counter (a tile's predecessors started earlier: no deadlock), publish their
// aggregate at once (flag 1) and their inclusive prefix once known (flag 2);
// warp 0 of a tile looks back 32 predecessors at a time.  status[t] =
// flag << 32 | value, written atomically; read volatile.  Reads the input once.
__global__ void __launch_bounds__(kScanThreads) k_scan_lb(const int *in, int *out, int64_t n, int ntiles,
                                                          unsigned long long *status, int *tile_ctr,
                                                          int *total) {
    __shared__ int s_tile, s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1);
    __syncthreads();
    const int t = s_tile;
    const int64_t i = (int64_t)t * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int x[kScanItems];
#pragma unroll
    for (int g = 0; g < kScanItems / 4; g++) load4(in, n, i + 4 * g, x + 4 * g);
    int s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) s += x[k];
    int tot;
    const int ex = block_excl_scan(s, tot);
    if (threadIdx.x == 0)
        atomicExch(status + t, (t == 0 ? (2ull << 32) : (1ull << 32)) | (unsigned)tot);
    if (threadIdx.x < 32) {
        int prefix = 0;
        for (int j = t - 1; j >= 0;) {
            const int idx = j - (int)threadIdx.x;
            const unsigned long long sv =
                idx >= 0 ? *reinterpret_cast<volatile unsigned long long *>(status + idx) : (2ull << 32);
            const unsigned flag = (unsigned)(sv >> 32);
            const unsigned incl = __ballot_sync(0xffffffffu, flag == 2u);
            const unsigned inv = __ballot_sync(0xffffffffu, flag == 0u);
            const int fi = incl ? __ffs(incl) - 1 : 32;
            const int fz = inv ? __ffs(inv) - 1 : 32;
            if (fz < fi) continue;   // a nearer predecessor has not published yet: re-read
            int v = ((int)threadIdx.x <= fi && idx >= 0) ? (int)(unsigned)(sv & 0xffffffffu) : 0;
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            prefix += v;
            if (fi < 32) break;
            j -= 32;
        }
        if (threadIdx.x == 0) {
            s_prefix = prefix;
            if (t > 0) atomicExch(status + t, (2ull << 32) | (unsigned)(prefix + tot));
            if (t == ntiles - 1 && total) *total = prefix + tot;
        }
    }
    __syncthreads();
    int run = ex + s_prefix;
#pragma unroll
    for (int g = 0; g < kScanItems / 4; g++) {
        int y[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            y[k] = run;
            run += x[4 * g + k];
        }
        const int64_t j = i + 4 * g;
        if (j + 3 < n && ((reinterpret_cast<uintptr_t>(out + j) & 15) == 0)) {
            *reinterpret_cast<int4 *>(out + j) = make_int4(y[0], y[1], y[2], y[3]);
        } else {
#pragma unroll
            for (int k = 0; k < 4; k++)
                if (j + k < n) out[j + k] = y[k];
        }
    }
}

// ---------------------------------------------------------------- readbacks / uploads
// Per-thread host scratch: a pinned readback buffer, a pinned upload arena and
// the polling events.  The setup's helper thread is created per
// fiedler_create, so the scratch objects come from a process-wide pool (no
// cudaMallocHost / cudaFreeHost / event creation per create).
namespace {
struct ThreadScratch {
    void *pin = nullptr;           // readbacks
    size_t pincap = 0;
    char *up = nullptr;            // uploads
    size_t upcap = 0, upoff = 0;
    cudaStream_t upst = nullptr;   // stream of the pending uploads
    cudaEvent_t ev[kMaxDevices] = {};
};
std::mutex g_scratch_mu;
std::vector<ThreadScratch *> g_scratch_free;

void poll_on(ThreadScratch &s, cudaStream_t st) {
    cudaEvent_t &ev = s.ev[current_device()];
    if (!ev) FDL_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    FDL_CK(cudaEventRecord(ev, st));
    cudaError_t e;
    while ((e = cudaEventQuery(ev)) == cudaErrorNotReady) {
    }
    FDL_CK(e);
    if (s.upst == st) s.upoff = 0;   // this stream's uploads are complete
}

struct ScratchHolder {
    ThreadScratch *s = nullptr;
    ThreadScratch &get() {
        if (!s) {
            std::lock_guard<std::mutex> lk(g_scratch_mu);
            if (!g_scratch_free.empty()) {
                s = g_scratch_free.back();
                g_scratch_free.pop_back();
            } else {
                s = new ThreadScratch();
            }
        }
        return *s;
    }
    ~ScratchHolder() {
        if (!s) return;
        if (s->upoff) {   // uploads still pending: let them land before the arena is reused
            cudaStreamSynchronize(s->upst);
            s->upoff = 0;
        }
        std::lock_guard<std::mutex> lk(g_scratch_mu);
        g_scratch_free.push_back(s);
    }
};
thread_local ScratchHolder tl_scratch;
}  // namespace

void host_wait(cudaStream_t st) { poll_on(tl_scratch.get(), st); }

void readback(cudaStream_t st, std::initializer_list<ReadPiece> pieces) {
    readback(st, std::vector<ReadPiece>(pieces));
}

void readback(cudaStream_t st, const std::vector<ReadPiece> &pieces) {
    ThreadScratch &S = tl_scratch.get();
    size_t total = 0;
    for (const ReadPiece &r : pieces) total += (r.bytes + 15) & ~(size_t)15;
    if (total > S.pincap) {
        if (S.pin) FDL_CK(cudaFreeHost(S.pin));
        S.pin = nullptr;
        S.pincap = 0;
        const size_t cap = std::max<size_t>(total, 1 << 16);
        FDL_CK(cudaMallocHost(&S.pin, cap));
        S.pincap = cap;
    }
    char *buf = static_cast<char *>(S.pin);
    size_t off = 0;
    for (const ReadPiece &r : pieces) {
        if (r.bytes) FDL_CK(cudaMemcpyAsync(buf + off, r.src, r.bytes, cudaMemcpyDeviceToHost, st));
        off += (r.bytes + 15) & ~(size_t)15;
    }
    poll_on(S, st);
    off = 0;
    for (const ReadPiece &r : pieces) {
        if (r.bytes) std::memcpy(r.dst, buf + off, r.bytes);
        off += (r.bytes + 15) & ~(size_t)15;
    }
}

// Host -> device copies of small host-computed arrays (tile counts, hub lists)
// through the pinned upload arena: a copy from pageable memory synchronises the
// stream first (a host round trip while the device drains), one from pinned
// memory does not.  The arena is reused once its stream has been waited on.
void upload(cudaStream_t st, void *dst, const void *src, size_t bytes) {
    if (!bytes) return;
    ThreadScratch &S = tl_scratch.get();
    const size_t r = (bytes + 15) & ~(size_t)15;
    if (S.upoff && (S.upst != st || S.upoff + r > S.upcap)) poll_on(S, S.upst);
    S.upoff = S.upst == st ? S.upoff : 0;
    if (r > S.upcap) {
        if (S.up) FDL_CK(cudaFreeHost(S.up));
        S.up = nullptr;
        S.upcap = 0;
        const size_t cap = std::max<size_t>(r, 1 << 20);
        FDL_CK(cudaMallocHost(reinterpret_cast<void **>(&S.up), cap));
        S.upcap = cap;
    }
    std::memcpy(S.up + S.upoff, src, bytes);
    FDL_CK(cudaMemcpyAsync(dst, S.up + S.upoff, bytes, cudaMemcpyHostToDevice, st));
    S.upoff += r;
    S.upst = st;
}

void scan_exclusive(const int *in, int *out, int64_t n, int *total, cudaStream_t st) {
    if (n <= 0) {
        if (total) FDL_CK(cudaMemsetAsync(total, 0, sizeof(int), st));
        return;
    }
    const int nb = div_up(n, kScanTile);
    // status words (8 bytes per tile) followed by the tile counter
    DBuf ws((size_t)nb * 8 + 16, st);
    FDL_CK(cudaMemsetAsync(ws.p, 0, (size_t)nb * 8 + 16, st));
    unsigned long long *status = ws.as<unsigned long long>();
    k_scan_lb<<<nb, kScanThreads, 0, st>>>(in, out, n, nb, status, reinterpret_cast<int *>(status + nb), total);
    FDL_LAUNCH_CK();
}

// =============================================================== radix sort
constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsSub = 32;                        // sub-tiles of 256 items per tile
constexpr int kRsTile = kRsThreads * kRsSub;      // 8192 items per block

template <class K>
__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const K *keys, int64_t n, int shift,
                                                        int nb, int *hist) {
    __shared__ int cnt[256];
    cnt[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * kRsTile;
    for (int s = 0; s < kRsSub; s++) {
        int64_t i = base + (int64_t)s * kRsThreads + threadIdx.x;
        if (i < n) atomicAdd(&cnt[(unsigned)(keys[i] >> shift) & 255u], 1);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * nb + blockIdx.x] = cnt[threadIdx.x];
}

template <class K, class V>
__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(const K *keys, const V *vals,
                                                           int64_t n, int shift, int nb,
                                                           const int *offs, K *keys_out,
                                                           V *vals_out) {
    __shared__ int s_run[256];
    __shared__ int s_cnt[kRsWarps][256];
    s_run[threadIdx.x] = offs[(int64_t)threadIdx.x * nb + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kRsWarps; w++) s_cnt[w][threadIdx.x] = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    int64_t base = (int64_t)blockIdx.x * kRsTile;
    for (int s = 0; s < kRsSub; s++) {
        if (base + (int64_t)s * kRsThreads >= n) break;  // block-uniform
        int64_t i = base + (int64_t)s * kRsThreads + threadIdx.x;
        bool valid = i < n;
        K k = valid ? keys[i] : K(0);
        V v = valid ? vals[i] : V(0);
        int d = valid ? (int)((unsigned)(k >> shift) & 255u) : 256;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        int rank = __popc(peers & lt);
        if (valid && rank == 0) s_cnt[warp][d] = __popc(peers);
        __syncthreads();
        {   // per-digit exclusive scan over warps, continuing the running offset
            int t = threadIdx.x;
            int run = s_run[t];
#pragma unroll
            for (int w = 0; w < kRsWarps; w++) {
                int c = s_cnt[w][t];
                s_cnt[w][t] = run;
                run += c;
            }
            s_run[t] = run;
        }
        __syncthreads();
        if (valid) {
            int pos = s_cnt[warp][d] + rank;
            keys_out[pos] = k;
            vals_out[pos] = v;
        }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < kRsWarps; w++) s_cnt[w][threadIdx.x] = 0;
        __syncthreads();
    }
}

// One stable counting-sort pass of the vertices by colour (colours < 256) that
// also writes what the GS layout needs from it: perm[pos] = v, inv[v] = pos
// (coalesced: v is read in order) and degp[pos] = degree of v.
__global__ void __launch_bounds__(kRsThreads) k_colour_scatter(const unsigned *color, int64_t n, int nb,
                                                               const int *offs, const int *rp, int *perm,
                                                               int *inv, int *degp) {
    __shared__ int s_run[256];
    __shared__ int s_cnt[kRsWarps][256];
    s_run[threadIdx.x] = offs[(int64_t)threadIdx.x * nb + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kRsWarps; w++) s_cnt[w][threadIdx.x] = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    int64_t base = (int64_t)blockIdx.x * kRsTile;
    for (int s = 0; s < kRsSub; s++) {
        if (base + (int64_t)s * kRsThreads >= n) break;  // block-uniform
        int64_t i = base + (int64_t)s * kRsThreads + threadIdx.x;
        bool valid = i < n;
        int d = valid ? (int)(color[i] & 255u) : 256;
        int dg = valid ? rp[i + 1] - rp[i] : 0;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        int rank = __popc(peers & lt);
        if (valid && rank == 0) s_cnt[warp][d] = __popc(peers);
        __syncthreads();
        {
            int t = threadIdx.x;
            int run = s_run[t];
#pragma unroll
            for (int w = 0; w < kRsWarps; w++) {
                int c = s_cnt[w][t];
                s_cnt[w][t] = run;
                run += c;
            }
            s_run[t] = run;
        }
        __syncthreads();
        if (valid) {
            int pos = s_cnt[warp][d] + rank;
            perm[pos] = (int)i;
            inv[i] = pos;
            degp[pos] = dg;
        }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < kRsWarps; w++) s_cnt[w][threadIdx.x] = 0;
        __syncthreads();
    }
}

__global__ void k_seg_from_hist(int ncolors, int nb, const int *offs, int *segstart) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncolors; c += gridDim.x * blockDim.x)
        segstart[c] = offs[(int64_t)c * nb];
}

void colour_sort(const int *color, int64_t n, int ncolors, const int *rp, int *perm, int *inv, int *degp,
                 int *segstart, cudaStream_t st) {
    FDL_REQUIRE(ncolors <= 256 && n < (int64_t(1) << 31), FIEDLER_ERR_INTERNAL, "colour_sort: bad sizes");
    const int nb = div_up(n, kRsTile);
    DBuf hist((size_t)256 * nb * sizeof(int), st);
    const unsigned *keys = reinterpret_cast<const unsigned *>(color);
    k_rs_hist<unsigned><<<nb, kRsThreads, 0, st>>>(keys, n, 0, nb, hist.as<int>());
    FDL_LAUNCH_CK();
    scan_exclusive(hist.as<int>(), hist.as<int>(), (int64_t)256 * nb, nullptr, st);
    k_colour_scatter<<<nb, kRsThreads, 0, st>>>(keys, n, nb, hist.as<int>(), rp, perm, inv, degp);
    FDL_LAUNCH_CK();
    k_seg_from_hist<<<1, 256, 0, st>>>(ncolors, nb, hist.as<int>(), segstart);
    FDL_LAUNCH_CK();
}

template <class K, class V>
static void radix_sort_impl(K *keys, V *vals, int64_t n, int bits, cudaStream_t st) {
    if (n <= 1 || bits <= 0) return;
    FDL_REQUIRE(n < (int64_t(1) << 31), FIEDLER_ERR_TOO_LARGE, "radix sort: n >= 2^31");
    int nb = div_up(n, kRsTile);
    DBuf hist((size_t)256 * nb * sizeof(int), st);
    DBuf kalt((size_t)n * sizeof(K), st), valt((size_t)n * sizeof(V), st);
    K *ka = keys, *kb = kalt.as<K>();
    V *va = vals, *vb = valt.as<V>();
    int passes = (bits + 7) / 8;
    for (int p = 0; p < passes; p++) {
        int shift = 8 * p;
        k_rs_hist<K><<<nb, kRsThreads, 0, st>>>(ka, n, shift, nb, hist.as<int>());
        FDL_LAUNCH_CK();
        scan_exclusive(hist.as<int>(), hist.as<int>(), (int64_t)256 * nb, nullptr, st);
        k_rs_scatter<K, V><<<nb, kRsThreads, 0, st>>>(ka, va, n, shift, nb, hist.as<int>(), kb, vb);
        FDL_LAUNCH_CK();
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (ka != keys) {
        FDL_CK(cudaMemcpyAsync(keys, ka, (size_t)n * sizeof(K), cudaMemcpyDeviceToDevice, st));
        FDL_CK(cudaMemcpyAsync(vals, va, (size_t)n * sizeof(V), cudaMemcpyDeviceToDevice, st));
    }
}

void radix_sort_u32_i32(unsigned *keys, int *vals, int64_t n, int bits, cudaStream_t st) {
    radix_sort_impl<unsigned, int>(keys, vals, n, bits, st);
}
void radix_sort_u64_i32(unsigned long long *keys, int *vals, int64_t n, int bits, cudaStream_t st) {
    radix_sort_impl<unsigned long long, int>(keys, vals, n, bits, st);
}

// =============================================================== compaction
__global__ void k_compact(const int *in, const int *flags, const int *pos, int64_t n, int *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (flags[i]) out[pos[i]] = in ? in[i] : (int)i;
}

void compact_flagged(const int *in, const int *flags, int64_t n, int *out, int *d_count,
                     cudaStream_t st) {
    if (n <= 0) {
        FDL_CK(cudaMemsetAsync(d_count, 0, sizeof(int), st));
        return;
    }
    DBuf pos((size_t)n * sizeof(int), st);
    scan_exclusive(flags, pos.as<int>(), n, d_count, st);
    k_compact<<<grid_for(n, 256, kNumSMs * 16), 256, 0, st>>>(in, flags, pos.as<int>(), n, out);
    FDL_LAUNCH_CK();
}

// =============================================================== max
__global__ void k_max_i32(const int *in, int64_t n, int *out) {
    int m = INT_MIN;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, in[i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane_id() == 0) atomicMax(out, m);
}

__global__ void k_set_i32(int *p, int v) { *p = v; }

void reduce_max_i32(const int *in, int64_t n, int *out, cudaStream_t st) {
    k_set_i32<<<1, 1, 0, st>>>(out, INT_MIN);
    FDL_LAUNCH_CK();
    k_max_i32<<<grid_for(n, 256, kNumSMs * 8), 256, 0, st>>>(in, n, out);
    FDL_LAUNCH_CK();
}

}  // namespace fdl

// fdl_setup.cu -- Setup Phase of Algorithm 3 on the GPU.
//
//   per level l (natural numbering):
//     heavy edge coarsening, parallel order (R2): the handshake matching in the
//       strict edge order (w, splitmix64 hash) -- equal to the greedy
//       heaviest-first matching -- as ONE cooperative launch (grid barriers
//       between rounds), then unmatched vertices join the aggregate of their
//       heaviest neighbour (Algorithm 1 line 13);
//     aggregate numbering: exclusive prefix scan over leader flags;
//     Galerkin product I L I^T per coarse row from the aggregate
//       members, folded in the R3 order (sort by (B, lo, hi) per row);
//     greedy first-fit colouring in decreasing hash priority (R4), the DAG form
//       of Jones-Plassmann, one cooperative launch on a second stream,
//       overlapped with the coarsening chain;
//     solve layouts: GS rows sorted by (colour, natural id) + the natural CSR.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <condition_variable>
#include <exception>
#include <mutex>
#include <queue>
#include <thread>

#include <cooperative_groups.h>

#include "fdl_internal.h"

namespace fdl {

// ----------------------------------------------------------------- sub-warp loops
// Rows are processed by groups of W lanes; the outer loop is warp-uniform so
// width-W shuffles after the per-row loop are always executed by full warps.
#define SUBWARP_LOOP(W, NITEMS, IDX)                                                   \
    const int sw_lane_ = threadIdx.x & ((W)-1);                                        \
    const int64_t sw_warp_ = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;   \
    const int64_t sw_nwarps_ = ((int64_t)gridDim.x * blockDim.x) >> 5;                 \
    for (int64_t sw_base_ = sw_warp_ * (32 / (W)); sw_base_ < (NITEMS);                 \
         sw_base_ += sw_nwarps_ * (32 / (W)))                                          \
        for (int64_t IDX = sw_base_ + ((threadIdx.x & 31) / (W)), sw_once_ = 0;         \
             sw_once_ < 1; sw_once_++)

template <int W>
__device__ __forceinline__ void argmax_reduce(double &bw, unsigned long long &bh, int &bj) {
#pragma unroll
    for (int o = W / 2; o; o >>= 1) {
        double ow = __shfl_xor_sync(0xffffffffu, bw, o, W);
        unsigned long long oh = __shfl_xor_sync(0xffffffffu, bh, o, W);
        int oj = __shfl_xor_sync(0xffffffffu, bj, o, W);
        if (oj >= 0 && (bj < 0 || ow > bw || (ow == bw && oh > bh))) { bw = ow; bh = oh; bj = oj; }
    }
}

template <int W> __device__ __forceinline__ int sub_sum(int v) {
#pragma unroll
    for (int o = W / 2; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, W);
    return v;
}

// cooperative kernels: thread-per-vertex below 8 neighbours (more independent
// dependency chains in flight), sub-warps above
#define DISPATCH_WC(avg, ...)                                   \
    do {                                                        \
        if ((avg) <= 8.5) { constexpr int W = 1; __VA_ARGS__; } \
        else if ((avg) <= 18) { constexpr int W = 8; __VA_ARGS__; } \
        else { constexpr int W = 32; __VA_ARGS__; }             \
    } while (0)

#define DISPATCH_W(avg, ...)                                    \
    do {                                                        \
        if ((avg) <= 4.5) { constexpr int W = 4; __VA_ARGS__; } \
        else if ((avg) <= 9) { constexpr int W = 8; __VA_ARGS__; } \
        else if ((avg) <= 18) { constexpr int W = 16; __VA_ARGS__; } \
        else { constexpr int W = 32; __VA_ARGS__; }             \
    } while (0)

static int sub_grid(int64_t items, int W) { return grid_for(items * W, 256, kNumSMs * 16); }

// ================================================================= validation
__global__ void k_rp64_to_32(const int64_t *rp64, int64_t n, int64_t nnz, int *rp32, int *flags) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = rp64[i];
        if (v < 0 || v > nnz || (i == 0 && v != 0) || (i == n && v != nnz)) atomicOr(flags, 1);
        if (i < n && rp64[i + 1] < v) atomicOr(flags, 1);
        rp32[i] = (int)v;
    }
}

__global__ void k_rp_check32(const int *rp, int n, int nnz, int *flags) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
        int v = rp[i];
        if (v < 0 || v > nnz || (i == 0 && v != 0) || (i == n && v != nnz)) atomicOr(flags, 1);
        if (i < n && rp[i + 1] < v) atomicOr(flags, 1);
    }
}

__global__ void k_validate(int n, const int *rp, const int *ci, const double *w, int *flags) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int b = rp[i], e = rp[i + 1];
        int prev = -1, f = 0;
        for (int k = b; k < e; k++) {
            int j = ci[k];
            double x = w[k];
            if (j < 0 || j >= n) { f |= 2; continue; }
            if (j == i) f |= 4;
            if (j <= prev) f |= 8;
            prev = j;
            if (!(x > 0.0) || !isfinite(x)) f |= 16;
            // symmetric partner: binary search row j for i
            int lo = rp[j], hi = rp[j + 1] - 1, found = -1;
            while (lo <= hi) {
                int mid = (lo + hi) >> 1;
                int cm = ci[mid];
                if (cm == i) { found = mid; break; }
                if (cm < i) lo = mid + 1; else hi = mid - 1;
            }
            if (found < 0 || w[found] != x) f |= 32;
        }
        if (f) atomicOr(flags, f);
    }
}

void validate_input(int64_t n, int64_t nnz, const int *rp32, const int *ci, const double *w,
                    cudaStream_t st) {
    DBuf fl(sizeof(int), st);
    FDL_CK(cudaMemsetAsync(fl.p, 0, sizeof(int), st));
    k_rp_check32<<<grid_for(n + 1), 256, 0, st>>>(rp32, (int)n, (int)nnz, fl.as<int>());
    FDL_LAUNCH_CK();
    int h = 0;
    readback(st, {{&h, fl.p, sizeof(int)}});
    FDL_REQUIRE(h == 0, FIEDLER_ERR_GRAPH, "row_ptr is not a valid CSR offset array");
    k_validate<<<grid_for(n), 256, 0, st>>>((int)n, rp32, ci, w, fl.as<int>());
    FDL_LAUNCH_CK();
    readback(st, {{&h, fl.p, sizeof(int)}});
    if (h) {
        std::string m = "invalid graph CSR:";
        if (h & 2) m += " column index out of range;";
        if (h & 4) m += " self loop;";
        if (h & 8) m += " columns not strictly increasing within a row;";
        if (h & 16) m += " weight not finite and > 0;";
        if (h & 32) m += " adjacency not symmetric (w_ij != w_ji);";
        throw Error(FIEDLER_ERR_GRAPH, m);
    }
}

void convert_row_ptr(const int64_t *rp64_dev, int64_t n, int64_t nnz, int *rp32, cudaStream_t st) {
    DBuf fl(sizeof(int), st);
    FDL_CK(cudaMemsetAsync(fl.p, 0, sizeof(int), st));
    k_rp64_to_32<<<grid_for(n + 1), 256, 0, st>>>(rp64_dev, n, nnz, rp32, fl.as<int>());
    FDL_LAUNCH_CK();
    int h = 0;
    readback(st, {{&h, fl.p, sizeof(int)}});
    FDL_REQUIRE(h == 0, FIEDLER_ERR_GRAPH, "row_ptr is not a valid CSR offset array");
}

// ================================================================= heavy edge coarsening
// The handshake rounds run inside ONE cooperative kernel per level (grid-wide
// barriers between phases, no host round trip per round).  Work lists are
// appended through a per-CTA shared-memory buffer (one global atomic per
// flush); list order is irrelevant to every consumer, so results are
// deterministic.
namespace cg = cooperative_groups;
constexpr int kCoopThreads = 256;
#ifndef FDL_COOP_MINB
#define FDL_COOP_MINB 6
#endif
constexpr int kCoopMinBlocks = FDL_COOP_MINB;   // resident CTAs per SM the register budget must allow
#ifndef FDL_MATCH_MINB
#define FDL_MATCH_MINB 5
#endif
constexpr int kMatchMinBlocks = FDL_MATCH_MINB;   // ... for the matching (more live state per thread)
constexpr int kAppendCap = 2048;
constexpr int kMaxRounds = 1 << 16;
#ifndef FDL_MATCH_UNROLL
#define FDL_MATCH_UNROLL 4
#endif
constexpr int kMatchUnroll = FDL_MATCH_UNROLL;
// the matching and the colouring (second stream) are both cooperative: each
// takes part of the co-resident grid so that they can run side by side
// (round 2, two side streams: config 4 step 72.1 / 71.9 / 71.8 / 76.0 ms at a
// matching share of 0.5 / 0.55 / 0.6 / 0.63 -- past ~0.6 the cooperative
// launches no longer fit beside each other; 0.55 keeps a margin)
#ifndef FDL_MATCH_GRID_FRAC
#define FDL_MATCH_GRID_FRAC 0.55
#endif
constexpr double kMatchGridFrac = FDL_MATCH_GRID_FRAC;
static_assert(kAppendCap >= 2 * kMatchUnroll * kCoopThreads, "append buffer too small");   // JP depth can reach thousands on dense cores

// Grid-wide barrier of the cooperative kernels (all CTAs resident) with a
// polling backoff (FDL_GRID_BACKOFF=1), instead of cg's grid sync, which spins
// its CTA masters on an acquire load: tried in case the long chains of rounds
// slowed the other streams' kernels with polls -- measured 0.2-2 ms slower on
// every config (the barrier's own latency grows), so off by default.
// bar[0] = arrivals, bar[1] = generation (zero at launch).
#ifndef FDL_GRID_BACKOFF
#define FDL_GRID_BACKOFF 0
#endif
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void grid_sync_bo(cg::grid_group &grid, unsigned *bar) {
    if (!FDL_GRID_BACKOFF) {
        grid.sync();
        return;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire_gpu(bar + 1);
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            unsigned ns = 32;
            while (ld_acquire_gpu(bar + 1) == g) {
                __nanosleep(ns);
                if (ns < 256) ns <<= 1;
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// FIEDLER_TRACE: per-phase device timestamps of the cooperative kernels
__device__ unsigned long long *g_round_ts = nullptr;
__device__ __forceinline__ void round_stamp(int i) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && i < 2 * kMaxRounds && g_round_ts) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_round_ts[i] = t;
    }
}

// predicated atomic decrement (returns the old value, 0 when pred is false):
// branch-free, so the decrements of a whole chunk are in flight together
__device__ __forceinline__ int atom_dec_if(int *p, bool pred) {
    int old = 0;
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q atom.global.add.s32 %0, [%1], -1;\n}\n"
        : "+r"(old)
        : "l"(p), "r"((int)pred)
        : "memory");
    return old;
}

struct CtaAppend {
    int *buf;
    int *n;
    int *base;
    __device__ __forceinline__ void push(int v) { buf[atomicAdd(n, 1)] = v; }
    // push that spills straight to the global list when the buffer is full
    __device__ __forceinline__ void push_safe(int v, int *out, int *gcount) {
        const int p = atomicAdd(n, 1);
        if (p < kAppendCap) buf[p] = v;
        else out[atomicAdd(gcount, 1)] = v;
    }
    // all threads, after a __syncthreads(): whether more than thr entries are
    // buffered.  Every thread reads the count before the barrier inside, so a
    // fast warp's next push cannot make the threads disagree (the decision
    // guards barriers).
    __device__ __forceinline__ bool due(int thr) {
        const int x = *n;
#ifndef FDL_RACY_FLUSH
        __syncthreads();
#endif
        return x > thr;
    }
    // all threads; call after __syncthreads()
    __device__ __forceinline__ void flush(int *out, int *gcount) {
        const int cnt = min(*n, kAppendCap);
        if (cnt == 0) return;
        if (threadIdx.x == 0) *base = atomicAdd(gcount, cnt);
        __syncthreads();
        const int b = *base;
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) out[b + i] = buf[i];
        __syncthreads();
        if (threadIdx.x == 0) *n = 0;
        __syncthreads();
    }
};

// heaviest neighbour of v in the strict order (w, hash) among neighbours with
// skip(j) == false (sub-warp of W lanes; all lanes return the same result)
template <int W, class Skip>
__device__ __forceinline__ int heaviest(int v, const int *rp, const int *ci, const double *w,
                                        uint64_t salt, int lane, Skip skip) {
    double bw = 0.0;
    unsigned long long bh = 0;
    int bj = -1;
    if (v >= 0)
        for (int k = rp[v] + lane; k < rp[v + 1]; k += W) {
            const int j = ci[k];
            if (skip(j)) continue;
            const double x = w[k];
            const unsigned long long h = edge_hash(salt, v, j);
            if (bj < 0 || x > bw || (x == bw && h > bh)) { bw = x; bh = h; bj = j; }
        }
    argmax_reduce<W>(bw, bh, bj);
    return bj;
}

// strict edge order of R2: (w, hash) descending
__device__ __forceinline__ bool edge_greater(double wa, unsigned long long ha, double wb,
                                             unsigned long long hb) {
    return wa > wb || (wa == wb && ha > hb);
}

// Rows up to kSortSlots * W entries get their neighbours ranked once in the
// strict edge order (nbr[rp[v] + rank] = neighbour): re-pointing to the
// heaviest FREE neighbour is then a cursor advance.  Longer rows are rescanned.
template <int W> struct SortSlots { static constexpr int value = W == 1 ? 8 : 4; };
// movers whose rescan is longer than this go to the whole CTA (k_match_coop, W > 1)
constexpr int kMatchHeavyDeg = 2048;
constexpr int kMatchHeavyCap = 64;

// One thread ranks the <= S entries of row v in the strict edge order
// (nbr[b + rank] = neighbour); returns the heaviest neighbour (-1: none).
template <int S>
__device__ __forceinline__ int rank_row(int v, int b, int deg, const int *ci, const double *w, uint64_t salt,
                                        int *nbr) {
    double wv[S];
    unsigned long long hv[S];
    int cv[S];
#pragma unroll
    for (int i = 0; i < S; i++) {
        const bool on = v >= 0 && i < deg;
        cv[i] = on ? ci[b + i] : -1;
        wv[i] = on ? w[b + i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < S; i++) hv[i] = cv[i] >= 0 ? edge_hash(salt, v, cv[i]) : 0ull;
    int top = -1;
#pragma unroll
    for (int i = 0; i < S; i++) {
        int rank = 0;
#pragma unroll
        for (int j = 0; j < S; j++)
            if (j != i) rank += cv[j] >= 0 && edge_greater(wv[j], hv[j], wv[i], hv[i]);
        if (cv[i] >= 0) {
            nbr[b + rank] = cv[i];
            if (rank == 0) top = cv[i];
        }
    }
    return top;
}

// Rows longer than the in-kernel ranking (kSortSlots * W entries) of dense
// levels: without a ranking, a vertex whose target got matched rescans its
// whole row, and on R-MAT's dense levels (30-55 handshake rounds, a few
// matches per round, thousands of vertices pointing at each popular one) the
// rescans were most of the matching's time.  This pass ranks every row of
// kSortSlots * W < deg <= kRankMax entries once (a CTA per row: bitonic sort
// of (w, hash) descending in shared memory; w > 0, so its bits order like the
// value), so re-pointing is a cursor advance for them too.
constexpr int kRankMax = 8192;
#ifndef FDL_RANK_MIN_AVG
#define FDL_RANK_MIN_AVG 450
#endif
// levels this dense (entries per row) rank their long rows: measured on R-MAT
// (step 126.3 / 120.2 / 118.3 / 118.8 ms at 64 / 200 / 450 / 800; below ~450 the
// sorts cost more than the rescans they save)
constexpr double kRankMinAvg = FDL_RANK_MIN_AVG;
constexpr int kRankSmall = 1024;   // rows up to this many entries: small CTAs, many per SM
__device__ __forceinline__ void rank_row_cta(int v, int b, int deg, int P, const int *ci, const double *w,
                                             uint64_t salt, int *nbr, unsigned long long *kw,
                                             unsigned long long *kh, int *kj) {
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        if (i < deg) {
            const int j = ci[b + i];
            kw[i] = (unsigned long long)__double_as_longlong(w[b + i]);
            kh[i] = edge_hash(salt, v, j);
            kj[i] = j;
        } else {
            kw[i] = 0ull;   // padding sorts last (every weight is > 0)
            kh[i] = 0ull;
            kj[i] = -1;
        }
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int ixj = i ^ jj;
                if (ixj <= i) continue;
                // descending overall: blocks with (i & k) == 0 descending
                const bool gt = kw[ixj] > kw[i] || (kw[ixj] == kw[i] && kh[ixj] > kh[i]);
                const bool lt = kw[ixj] < kw[i] || (kw[ixj] == kw[i] && kh[ixj] < kh[i]);
                if (((i & k) == 0) ? gt : lt) {
                    const unsigned long long tw = kw[i], th = kh[i];
                    const int tj = kj[i];
                    kw[i] = kw[ixj]; kh[i] = kh[ixj]; kj[i] = kj[ixj];
                    kw[ixj] = tw; kh[ixj] = th; kj[ixj] = tj;
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < deg; i += blockDim.x) nbr[b + i] = kj[i];
    __syncthreads();
}
// the rows to rank: dmin < deg <= kRankSmall into list[0..), longer ones (<= kRankMax)
// from the top of the list downwards (cnt[0], cnt[1])
__global__ void k_rank_list(int n, const int *rp, int dmin, int *list, int *cnt) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int deg = rp[v + 1] - rp[v];
        if (deg <= dmin || deg > kRankMax) continue;
        if (deg <= kRankSmall) list[atomicAdd(cnt, 1)] = v;
        else list[n - 1 - atomicAdd(cnt + 1, 1)] = v;
    }
}
template <int T, int CAP>
__global__ void __launch_bounds__(T) k_rank_rows(int n, const int *rp, const int *ci, const double *w, uint64_t salt,
                                                 const int *list, const int *cnt, bool big, int *nbr) {
    extern __shared__ __align__(16) unsigned char rk_smem[];
    unsigned long long *kw = reinterpret_cast<unsigned long long *>(rk_smem);
    unsigned long long *kh = kw + CAP;
    int *kj = reinterpret_cast<int *>(kh + CAP);
    const int m = big ? cnt[1] : cnt[0];
    for (int i = blockIdx.x; i < m; i += gridDim.x) {
        const int v = big ? list[n - 1 - i] : list[i];
        const int b = rp[v], deg = rp[v + 1] - b;
        int P = 1;
        while (P < deg) P <<= 1;
        rank_row_cta(v, b, deg, P, ci, w, salt, nbr, kw, kh, kj);
    }
}

// counts[r] = length of the work list of round r (zeroed by the host); the
// lists ping-pong between la and lb.  rounds_out[0] = handshake rounds.
// W == 1 (low-degree levels): round 0 takes two rows per thread and the first
// handshake list is implicit (every vertex; isolated ones have no pointer).
template <int W>
__global__ void __launch_bounds__(kCoopThreads, kMatchMinBlocks) k_match_coop(int n, const int *rp, const int *ci,
                                                             const double *w, uint64_t salt, int *m,
                                                             int *ptr, int *mate, int *nbr, int *cursor,
                                                             int *la, int *lb, int *counts,
                                                             int *rounds_out, int *lm, int *mcount, int rank_avail) {
    cg::grid_group grid = cg::this_grid();
    unsigned *gbar = reinterpret_cast<unsigned *>(counts + kMaxRounds + 4);
    __shared__ int s_buf[kAppendCap];
    __shared__ int s_n, s_base;
    __shared__ int s_hm[kMatchHeavyCap], s_nhm;   // heavy movers of this CTA (W > 1)
    __shared__ double s_aw[kCoopThreads / 32];
    __shared__ unsigned long long s_ah[kCoopThreads / 32];
    __shared__ int s_aj[kCoopThreads / 32];
    if (threadIdx.x == 0) { s_n = 0; s_nhm = 0; }
    __syncthreads();
    CtaAppend app{s_buf, &s_n, &s_base};
    int stamp = 0;
    round_stamp(stamp++);
    const int lane = threadIdx.x & (W - 1);
    const int per_block = kCoopThreads / W;
    // round 0: rank every short row's neighbours; m(v) = heaviest neighbour =
    // the first handshake pointer; vertices with a neighbour enter the list
    if (W == 1) {
        for (long long base = (long long)blockIdx.x * 2 * kCoopThreads; base < n;
             base += (long long)gridDim.x * 2 * kCoopThreads) {
            int v[2], b[2], deg[2];
#pragma unroll
            for (int u = 0; u < 2; u++) {
                const long long idx = base + u * kCoopThreads + threadIdx.x;
                v[u] = idx < n ? (int)idx : -1;
                b[u] = v[u] >= 0 ? rp[v[u]] : 0;
                deg[u] = v[u] >= 0 ? rp[v[u] + 1] - b[u] : 0;
            }
            // warp-uniform slot count: 4 (grids), 8, or a rescan of long rows
            const int dmax = max(deg[0], deg[1]);
            const bool four = __all_sync(0xffffffffu, dmax <= 4);
            const bool ranked = __all_sync(0xffffffffu, dmax <= 8);
            auto store = [&](int vv, int top, bool rk) {
                if (vv < 0) return;
                m[vv] = top;
                ptr[vv] = top;
                cursor[vv] = rk ? 0 : -1;
            };
            if (four) {
                const int t0 = rank_row<4>(v[0], b[0], deg[0], ci, w, salt, nbr);
                const int t1 = rank_row<4>(v[1], b[1], deg[1], ci, w, salt, nbr);
                store(v[0], t0, true);
                store(v[1], t1, true);
            } else {
#pragma unroll 1
                for (int u = 0; u < 2; u++) {
                    const int vv = u ? v[1] : v[0], bb = u ? b[1] : b[0], dd = u ? deg[1] : deg[0];
                    // rows of <= 8 entries are ranked even in a warp with longer
                    // rows (only those are rescanned when they re-point)
                    const bool rk = ranked || dd <= 8;
                    int t;
                    if (rk) t = rank_row<8>(vv, bb, dd, ci, w, salt, nbr);
                    else t = vv >= 0 ? heaviest<1>(vv, rp, ci, w, salt, 0, [](int) { return false; }) : -1;
                    store(vv, t, rk);
                }
            }
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) counts[0] = n;   // implicit list: every vertex
    }
    for (long long base = (long long)blockIdx.x * per_block; W > 1 && base < n;
         base += (long long)gridDim.x * per_block) {
        const long long idx = base + threadIdx.x / W;
        const int v = idx < n ? (int)idx : -1;
        int b = 0, deg = 0;
        if (v >= 0) { b = rp[v]; deg = rp[v + 1] - b; }
        constexpr int kSortSlots = SortSlots<W>::value;
        const bool sortable = deg <= kSortSlots * W;
        // rows ranked by k_rank_long_rows (dense levels, W == 32: one vertex per warp)
        const bool presorted = W == 32 && rank_avail && v >= 0 && !sortable && deg <= kRankMax;
        int bj;
        const bool ranked = presorted || __all_sync(0xffffffffu, v < 0 || sortable);   // warp-uniform
        if (presorted) {
            bj = nbr[b];
        } else if (ranked) {
            double wv[kSortSlots];
            unsigned long long hv[kSortSlots];
            int cv[kSortSlots], rank[kSortSlots];
#pragma unroll
            for (int i = 0; i < kSortSlots; i++) {
                const int j = lane + i * W;
                rank[i] = 0;
                cv[i] = -1;
                wv[i] = 0.0;
                hv[i] = 0ull;
                if (j < deg) {
                    cv[i] = ci[b + j];
                    wv[i] = w[b + j];
                    hv[i] = edge_hash(salt, v, cv[i]);
                }
            }
            // rank = number of entries of the row greater than this one
#pragma unroll
            for (int sl = 0; sl < kSortSlots; sl++)
#pragma unroll
                for (int src = 0; src < W; src++) {
                    const int j = sl * W + src;
                    const double wj = __shfl_sync(0xffffffffu, wv[sl], src, W);
                    const unsigned long long hj = __shfl_sync(0xffffffffu, hv[sl], src, W);
                    if (j < deg)
#pragma unroll
                        for (int i = 0; i < kSortSlots; i++)
                            rank[i] += edge_greater(wj, hj, wv[i], hv[i]);
                }
            int top = -1;
#pragma unroll
            for (int i = 0; i < kSortSlots; i++)
                if (cv[i] >= 0) {
                    nbr[b + rank[i]] = cv[i];
                    if (rank[i] == 0) top = cv[i];
                }
            // the heaviest neighbour sits in exactly one lane of the sub-warp
#pragma unroll
            for (int o = W / 2; o; o >>= 1) top = max(top, __shfl_xor_sync(0xffffffffu, top, o, W));
            bj = top;
        } else {
            bj = heaviest<W>(v, rp, ci, w, salt, lane, [](int) { return false; });
        }
        if (v >= 0 && lane == 0) {
            m[v] = bj;
            ptr[v] = bj;
            cursor[v] = ranked ? 0 : -1;
            if (bj >= 0) app.push(v);
        }
        __syncthreads();
        if (app.due(kAppendCap - kCoopThreads)) app.flush(la, counts);
    }
    __syncthreads();
    app.flush(la, counts);
    grid_sync_bo(grid, gbar);
    round_stamp(stamp++);
    int *in = la, *out = lb;
    bool implicit = W == 1;   // the first list of W == 1 is every vertex, in order
    int r = 0;
    int cnt = *(volatile int *)&counts[0];
    while (cnt > 0 && r + 1 < kMaxRounds) {
        // (a) mutual pointers match (kMatchUnroll entries per thread in flight)
        {
            const int stride = gridDim.x * blockDim.x;
            for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < cnt; i0 += stride * kMatchUnroll) {
                int v[kMatchUnroll], p[kMatchUnroll];
#pragma unroll
                for (int u = 0; u < kMatchUnroll; u++) {
                    const int i = i0 + u * stride;
                    v[u] = i < cnt ? (implicit ? i : in[i]) : -1;
                }
#pragma unroll
                for (int u = 0; u < kMatchUnroll; u++) p[u] = v[u] >= 0 ? ptr[v[u]] : -1;
#pragma unroll
                for (int u = 0; u < kMatchUnroll; u++)
                    if (p[u] >= 0 && ptr[p[u]] == v[u]) mate[v[u]] = p[u];
            }
        }
        grid_sync_bo(grid, gbar);
        round_stamp(stamp++);
        // (b) unmatched vertices whose target got matched re-point at their
        //     heaviest FREE neighbour (cursor advance, or a rescan for long rows)
        int *gcount = counts + r + 1;
        if (W == 1) {
            // thread per vertex, kMatchUnroll vertices per thread with their
            // loads in flight together; long rows (no cursor) are rescanned
            for (long long base = (long long)blockIdx.x * kCoopThreads * kMatchUnroll; base < cnt;
                 base += (long long)gridDim.x * kCoopThreads * kMatchUnroll) {
                int v[kMatchUnroll], mv[kMatchUnroll], p[kMatchUnroll], cur[kMatchUnroll], b[kMatchUnroll],
                    e[kMatchUnroll], mp[kMatchUnroll], cand[kMatchUnroll], mc[kMatchUnroll];
#pragma unroll
                for (int u = 0; u < kMatchUnroll; u++) {
                    const long long idx = base + u * kCoopThreads + threadIdx.x;
                    v[u] = idx < cnt ? (implicit ? (int)idx : in[idx]) : -1;
                }
#pragma unroll
                for (int u = 0; u < kMatchUnroll; u++) {
                    const bool ok = v[u] >= 0;
                    mv[u] = ok ? mate[v[u]] : 0;
                    p[u] = ok ? ptr[v[u]] : 0;
                    cur[u] = ok ? cursor[v[u]] : -1;
                    b[u] = ok ? rp[v[u]] : 0;
                    e[u] = ok ? rp[v[u] + 1] : 0;
                }
#pragma unroll
                for (int u = 0; u < kMatchUnroll; u++)
                    mp[u] = (v[u] >= 0 && mv[u] < 0 && p[u] >= 0) ? mate[p[u]] : -1;
#pragma unroll
                for (int u = 0; u < kMatchUnroll; u++) {
                    const bool adv = v[u] >= 0 && mv[u] < 0 && mp[u] >= 0 && cur[u] >= 0;
                    cur[u] += 1;
                    cand[u] = (adv && b[u] + cur[u] < e[u]) ? nbr[b[u] + cur[u]] : -1;
                }
#pragma unroll
                for (int u = 0; u < kMatchUnroll; u++) mc[u] = cand[u] >= 0 ? mate[cand[u]] : -1;
#pragma unroll
                for (int u = 0; u < kMatchUnroll; u++) {
                    if (v[u] < 0 || mv[u] >= 0 || p[u] < 0) continue;   // matched, or no neighbour
                    bool keep = mp[u] < 0;
                    if (!keep) {   // the target got matched: re-point
                        int bj;
                        if (cur[u] > 0) {   // ranked row: cursor advance from cur + 1
                            int c = cur[u], j = cand[u], mj = mc[u];
                            while (j >= 0 && mj >= 0) {
                                // the next four candidates, their mate loads in flight together
                                int jj[4], mm[4];
#pragma unroll
                                for (int k = 0; k < 4; k++)
                                    jj[k] = b[u] + c + 1 + k < e[u] ? nbr[b[u] + c + 1 + k] : -1;
#pragma unroll
                                for (int k = 0; k < 4; k++) mm[k] = jj[k] >= 0 ? mate[jj[k]] : -1;
                                int fk = 4, fj = -1, fm = -1;   // first free candidate or the row end
#pragma unroll
                                for (int k = 0; k < 4; k++)
                                    if (fk == 4 && !(jj[k] >= 0 && mm[k] >= 0)) { fk = k; fj = jj[k]; fm = mm[k]; }
                                if (fk < 4) { c += 1 + fk; j = fj; mj = fm; }
                                else { c += 4; j = jj[3]; mj = mm[3]; }
                            }
                            bj = j;
                            cursor[v[u]] = c;
                        } else {
                            bj = heaviest<1>(v[u], rp, ci, w, salt, 0, [&](int j) { return mate[j] >= 0; });
                        }
                        ptr[v[u]] = bj;
                        keep = bj >= 0;
                    }
                    if (keep) app.push(v[u]);
                }
                __syncthreads();
                if (app.due(kAppendCap - kMatchUnroll * kCoopThreads)) app.flush(out, gcount);
            }
        } else {
            // (b1) thread per entry: matched vertices drop out, those whose target
            //      is still free stay listed, the rest (the movers) are collected
            int *mc = mcount + r;
            for (long long base = (long long)blockIdx.x * kCoopThreads; base < cnt;
                 base += (long long)gridDim.x * kCoopThreads) {
                const long long idx = base + threadIdx.x;
                const int v = idx < cnt ? in[idx] : -1;
                bool keep = false, mv = false;
                if (v >= 0 && mate[v] < 0) {
                    if (mate[ptr[v]] < 0) keep = true;
                    else mv = true;
                }
                if (keep) app.push(v);
                const unsigned bal = __ballot_sync(0xffffffffu, mv);   // one atomic per warp
                int wb = 0;
                if (bal && lane_id() == 0) wb = atomicAdd(mc, __popc(bal));
                wb = __shfl_sync(0xffffffffu, wb, 0);
                if (mv) lm[wb + __popc(bal & ((1u << lane_id()) - 1u))] = v;
                __syncthreads();
                if (app.due(kAppendCap - kCoopThreads)) app.flush(out, gcount);
            }
            grid_sync_bo(grid, gbar);
            // (b2) a sub-warp per mover re-points it at its heaviest FREE neighbour
            //      (cursor advance, or a rescan of a long row); slot s of CTA b
            //      takes mover base + s * gridDim + b, spread over all CTAs
            const int mcnt = *(volatile int *)mc;
            for (long long base = 0; base < mcnt; base += (long long)gridDim.x * per_block) {
                const long long idx = base + (long long)(threadIdx.x / W) * gridDim.x + blockIdx.x;
                const int v = idx < mcnt ? lm[idx] : -1;
                const int cur = v >= 0 ? cursor[v] : -1;
                int bj = -1;
                const bool rescan = v >= 0 && cur < 0;
                if (v >= 0 && cur >= 0) {
                    // cursor advance by the sub-warp: W candidates per step, the
                    // first free one by a ballot (was one dependent pair of loads
                    // per candidate in lane 0)
                    const int b = rp[v], deg = rp[v + 1] - b;
                    const unsigned sub = W == 32 ? 0xffffffffu
                                                 : (((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1)));
                    int c = cur + 1;
                    for (;; c += W) {
                        const int k = c + lane;
                        const int j = k < deg ? nbr[b + k] : -1;
                        const bool freej = j >= 0 && mate[j] < 0;
                        const bool endk = k >= deg;
                        const unsigned hit = __ballot_sync(sub, freej || endk) & sub;
                        if (hit) {
                            const int f = __ffs(hit >> ((threadIdx.x & 31) & ~(W - 1))) - 1;
                            c += f;
                            break;
                        }
                    }
                    bj = c < deg ? nbr[b + c] : -1;
                    if (lane == 0) cursor[v] = c;
                }
                // a rescan of a row longer than kMatchHeavyDeg: deferred to the
                // whole CTA (below) -- a sub-warp walking a 10000-entry row took
                // ~0.4 ms, and on dense levels a hub re-points in most rounds
                int hslot = -1;
                if (W > 1 && rescan && lane == 0 && rp[v + 1] - rp[v] > kMatchHeavyDeg) {
                    hslot = atomicAdd(&s_nhm, 1);
                    if (hslot < kMatchHeavyCap) s_hm[hslot] = v;
                }
                hslot = __shfl_sync(0xffffffffu, hslot, (threadIdx.x & 31) & ~(W - 1));
                const bool deferred = hslot >= 0 && hslot < kMatchHeavyCap;
                const int bs = heaviest<W>(rescan && !deferred ? v : -1, rp, ci, w, salt, lane,
                                           [&](int j) { return mate[j] >= 0; });
                if (rescan) bj = bs;
                if (v >= 0 && lane == 0 && !deferred) {
                    ptr[v] = bj;
                    if (bj >= 0) app.push(v);
                }
                __syncthreads();
                if (app.due(kAppendCap - kCoopThreads)) app.flush(out, gcount);
            }
            // the deferred heavy rescans: the CTA's threads over the row, 4
            // entries each in flight, then a CTA argmax in the strict order
            const int nhm = min(s_nhm, kMatchHeavyCap);   // read after the loop's barrier
            for (int i = 0; i < nhm; i++) {
                const int hv = s_hm[i];
                double bw = 0.0;
                unsigned long long bh = 0;
                int bj = -1;
                const int kb = rp[hv], ke = rp[hv + 1];
                for (int k0 = kb + threadIdx.x; k0 < ke; k0 += 4 * kCoopThreads) {
                    int jj[4], mm[4];
                    double ww[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int k = k0 + u * kCoopThreads;
                        jj[u] = k < ke ? ci[k] : -1;
                        ww[u] = k < ke ? w[k] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; u++) mm[u] = jj[u] >= 0 ? mate[jj[u]] : 0;
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        if (jj[u] < 0 || mm[u] >= 0) continue;
                        const unsigned long long h = edge_hash(salt, hv, jj[u]);
                        if (bj < 0 || ww[u] > bw || (ww[u] == bw && h > bh)) { bw = ww[u]; bh = h; bj = jj[u]; }
                    }
                }
                argmax_reduce<32>(bw, bh, bj);
                if (lane_id() == 0) {
                    s_aw[threadIdx.x >> 5] = bw;
                    s_ah[threadIdx.x >> 5] = bh;
                    s_aj[threadIdx.x >> 5] = bj;
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    for (int q = 1; q < kCoopThreads / 32; q++)
                        if (s_aj[q] >= 0 &&
                            (bj < 0 || s_aw[q] > bw || (s_aw[q] == bw && s_ah[q] > bh))) {
                            bw = s_aw[q];
                            bh = s_ah[q];
                            bj = s_aj[q];
                        }
                    ptr[hv] = bj;
                    if (bj >= 0) app.push_safe(hv, out, gcount);
                }
                __syncthreads();
            }
            if (threadIdx.x == 0) s_nhm = 0;
            __syncthreads();
        }
        __syncthreads();
        app.flush(out, gcount);
        grid_sync_bo(grid, gbar);
        round_stamp(stamp++);
        r++;
        cnt = *(volatile int *)gcount;
        int *t = in; in = out; out = t;
        implicit = false;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) rounds_out[0] = cnt == 0 ? r : -1;
}

// leader of v's aggregate (4 vertices per thread with their loads in flight)
__global__ void k_leaders(int n, const int *m, const int *mate, int *leader, int *flag, int *err) {
    const int stride = gridDim.x * blockDim.x;
    for (int v0 = blockIdx.x * blockDim.x + threadIdx.x; v0 < n; v0 += 4 * stride) {
        int mv[4], mm[4], mu[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int v = v0 + u * stride;
            mv[u] = v < n ? mate[v] : 0;
            mm[u] = v < n ? m[v] : -1;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) mu[u] = (mv[u] < 0 && mm[u] >= 0) ? mate[mm[u]] : 0;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int v = v0 + u * stride;
            if (v >= n) continue;
            int L;
            if (mv[u] >= 0) L = min(v, mv[u]);
            else if (mm[u] >= 0) {
                int x = mu[u];
                if (x < 0) { atomicOr(err, 1); x = mm[u]; }   // impossible for a maximal matching
                L = min(mm[u], x);
            } else L = v;
            leader[v] = L;
            flag[v] = (L == v);
        }
    }
}

__global__ void k_assign(int n, const int *leader, const int *id, int *q) {
    const int stride = gridDim.x * blockDim.x;
    for (int v0 = blockIdx.x * blockDim.x + threadIdx.x; v0 < n; v0 += 4 * stride) {
        int L[4], r[4];
#pragma unroll
        for (int u = 0; u < 4; u++) L[u] = v0 + u * stride < n ? leader[v0 + u * stride] : -1;
#pragma unroll
        for (int u = 0; u < 4; u++) r[u] = L[u] >= 0 ? id[L[u]] : 0;
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (L[u] >= 0) q[v0 + u * stride] = r[u];
    }
}

static int read_int(const int *dptr, cudaStream_t st) {
    int h;
    readback(st, {{&h, dptr, sizeof(int)}});
    return h;
}

// trace mode: arm the timestamp buffer before a cooperative kernel, print after
struct RoundTrace {
    DBuf buf;
    cudaStream_t st;
    const char *name;
    explicit RoundTrace(cudaStream_t s, const char *nm) : st(s), name(nm) {
        if (!trace_enabled()) return;
        buf.alloc((size_t)2 * kMaxRounds * 8, st);
        FDL_CK(cudaMemsetAsync(buf.p, 0, (size_t)2 * kMaxRounds * 8, st));
        void *p = buf.p;
        FDL_CK(cudaMemcpyToSymbolAsync(g_round_ts, &p, sizeof(p), 0, cudaMemcpyHostToDevice, st));
    }
    void report(const int *d_counts) {
        if (!trace_enabled()) return;
        std::vector<unsigned long long> ts(2 * kMaxRounds);
        std::vector<int> cnt(64);
        FDL_CK(cudaMemcpyAsync(ts.data(), buf.p, ts.size() * 8, cudaMemcpyDeviceToHost, st));
        FDL_CK(cudaMemcpyAsync(cnt.data(), d_counts, cnt.size() * 4, cudaMemcpyDeviceToHost, st));
        void *z = nullptr;
        FDL_CK(cudaMemcpyToSymbolAsync(g_round_ts, &z, sizeof(z), 0, cudaMemcpyHostToDevice, st));
        FDL_CK(cudaStreamSynchronize(st));
        std::string line = std::string("[fiedler trace]   ") + name + " phases(us):";
        for (int i = 1; i < 2 * kMaxRounds && ts[i]; i++) {
            char tmp[64];
            std::snprintf(tmp, sizeof(tmp), " %.0f", (ts[i] - ts[i - 1]) * 1e-3);
            line += tmp;
        }
        line += "  lists:";
        for (int i = 0; i < 64 && (i == 0 || cnt[i - 1]); i++) line += " " + std::to_string(cnt[i]);
        std::fprintf(stderr, "%s\n", line.c_str());
    }
};

// cooperative launch with every CTA co-resident (grid = SMs x resident CTAs);
// `work` = vertices x lanes per vertex: small levels take only as many CTAs as
// they can use (8 work items per thread), which keeps their grid barriers cheap
#ifndef FDL_COOP_ITEMS_PER_THREAD
#define FDL_COOP_ITEMS_PER_THREAD 8
#endif
template <class K>
static void coop_launch(K kernel, void **args, cudaStream_t st, double grid_frac, int64_t work) {
    static DeviceCache grid_cache{};   // one cache per kernel instantiation and device
    std::atomic<int> &grid_slot = grid_cache[current_device()];
    int grid = grid_slot.load();
    if (!grid) {
        int per_sm = 0, dev = 0, sms = kNumSMs;
        // a small shared-memory carveout: these kernels live on L1-cached gathers
        FDL_CK(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 25));
        FDL_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kCoopThreads, 0));
        FDL_CK(cudaGetDevice(&dev));
        FDL_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        FDL_REQUIRE(per_sm > 0, FIEDLER_ERR_CUDA, "cooperative kernel cannot be resident");
        grid = per_sm * sms;
        grid_slot.store(grid);
    }
    // the kernels are grid-size agnostic: if the driver finds fewer co-resident
    // CTAs than the occupancy query promised, retry with a smaller grid
    for (;;) {
        const int64_t useful = (work + (int64_t)kCoopThreads * FDL_COOP_ITEMS_PER_THREAD - 1) /
                               ((int64_t)kCoopThreads * FDL_COOP_ITEMS_PER_THREAD);
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)(grid * grid_frac), useful));
        cudaError_t e = cudaLaunchCooperativeKernel((const void *)kernel, dim3(g), dim3(kCoopThreads), args, 0, st);
        if (e == cudaErrorCooperativeLaunchTooLarge && grid > kNumSMs) {
            (void)cudaGetLastError();
            grid = grid * 3 / 4;
            grid_slot.store(grid);
            continue;
        }
        FDL_CK(e);
        break;
    }
    FDL_LAUNCH_CK();
}

// Returns the number of aggregates c; fills q (natural), mate.
static int hec_parallel(const NatGraph &g, uint64_t salt, DBuf &q, DBuf &mate, int &rounds,
                        cudaStream_t st) {
    int n = g.n;
    const double avg = n ? (double)g.nnz / n : 0.0;
    DBuf lmv((size_t)n * 4, st), mcount((size_t)kMaxRounds * 4, st);
    FDL_CK(cudaMemsetAsync(mcount.p, 0, (size_t)kMaxRounds * 4, st));
    DBuf m((size_t)n * 4, st), ptr((size_t)n * 4, st), la((size_t)n * 4, st), lb((size_t)n * 4, st),
        nbr((size_t)std::max(g.nnz, 1) * 4, st), cursor((size_t)n * 4, st),
        counts((size_t)(kMaxRounds + 8) * 4, st);
    q.alloc((size_t)n * 4, st);
    mate.alloc((size_t)n * 4, st);
    FDL_CK(cudaMemsetAsync(mate.p, 0xff, (size_t)n * 4, st));
    FDL_CK(cudaMemsetAsync(counts.p, 0, (size_t)(kMaxRounds + 8) * 4, st));
    {
        const int *rp = g.rp, *ci = g.ci;
        const double *w = g.w;
        int *pm = m.as<int>(), *pp = ptr.as<int>(), *pmate = mate.as<int>(), *pn = nbr.as<int>(),
            *pcur = cursor.as<int>(), *pa = la.as<int>(), *pb = lb.as<int>(), *pc = counts.as<int>(),
            *pr = counts.as<int>() + kMaxRounds;
        int *plm = lmv.as<int>(), *pmc = mcount.as<int>();
        int ra = avg > kRankMinAvg ? 1 : 0;   // long rows ranked by k_rank_rows (below)
        void *args[] = {&n, &rp, &ci, &w, &salt, &pm, &pp, &pmate, &pn, &pcur, &pa, &pb, &pc, &pr, &plm, &pmc, &ra};
        if (avg > kRankMinAvg) {   // dense W == 32 levels: rank the long rows first
            static DeviceCache attr{};
            std::atomic<int> &a = attr[current_device()];
            if (!a.load()) {
                FDL_CK(cudaFuncSetAttribute(k_rank_rows<512, kRankMax>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            kRankMax * 20));
                a.store(1);
            }
            DBuf rl((size_t)n * 4 + 16, st);
            int *rcnt = rl.as<int>() + n;
            FDL_CK(cudaMemsetAsync(rcnt, 0, 8, st));
            k_rank_list<<<grid_for(n), 256, 0, st>>>(n, rp, SortSlots<32>::value * 32, rl.as<int>(), rcnt);
            FDL_LAUNCH_CK();
            k_rank_rows<128, kRankSmall><<<kNumSMs * 8, 128, kRankSmall * 20, st>>>(n, rp, ci, w, salt, rl.as<int>(),
                                                                                  rcnt, false, pn);
            FDL_LAUNCH_CK();
            k_rank_rows<512, kRankMax><<<kNumSMs, 512, kRankMax * 20, st>>>(n, rp, ci, w, salt, rl.as<int>(), rcnt,
                                                                          true, pn);
            FDL_LAUNCH_CK();
        }
        RoundTrace tr(st, "match");
        DISPATCH_WC(avg, coop_launch(k_match_coop<W>, args, st, kMatchGridFrac, (int64_t)n * W));
        tr.report(counts.as<int>());
    }
    int rr[2];
    la.release();
    lb.release();
    nbr.release();
    cursor.release();
    // leaders, prefix scan numbering
    DBuf leader((size_t)n * 4, st), flag((size_t)n * 4, st), id((size_t)n * 4, st), tot(8, st);
    FDL_CK(cudaMemsetAsync(tot.p, 0, 8, st));
    k_leaders<<<grid_for(n), 256, 0, st>>>(n, m.as<int>(), mate.as<int>(), leader.as<int>(),
                                           flag.as<int>(), tot.as<int>() + 1);
    FDL_LAUNCH_CK();
    scan_exclusive(flag.as<int>(), id.as<int>(), n, tot.as<int>(), st);
    k_assign<<<grid_for(n), 256, 0, st>>>(n, leader.as<int>(), id.as<int>(), q.as<int>());
    FDL_LAUNCH_CK();
    // one round trip for the round count / termination flag and the aggregate count
    int th[2];
    readback(st, {{rr, counts.as<int>() + kMaxRounds, 8}, {th, tot.p, 8}});
    rounds = rr[0];
    FDL_REQUIRE(rounds >= 0 && rr[1] == 0, FIEDLER_ERR_INTERNAL, "matching did not terminate");
    FDL_REQUIRE(th[1] == 0, FIEDLER_ERR_INTERNAL, "heavy-edge matching is not maximal");
    return th[0];
}

__global__ void k_seg_starts(int n, const unsigned *keys, int *segstart) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        if (t == 0 || keys[t] != keys[t - 1]) segstart[keys[t]] = t;
}

// ================================================================= Galerkin product
// I L I^T with the R3 summation order, computed per COARSE ROW
// from the aggregate members (no global sort of all contributions):
//   1. members of every aggregate (counting sort by aggregate id) and the slot
//      count T_A = sum of the member degrees of every coarse row A;
//   2. the contributions of row A are its members' fine entries (m, j) with
//      B = q(j) != A: (B, lo = min(m, j), hi = max(m, j), w_mj); the R3 order
//      of the fine edges {i < j} is ascending (lo, hi);
//   3. each row sorts its contributions by (B, lo, hi) and left-folds every run
//      of equal B in that order -- the oracle's fold, computed independently
//      and identically on both sides of the pair, so W_c is symmetric bit for
//      bit.  Rows by size: <= 16 slots in warp batches (k_gal_direct_batch,
//      one 64-bit key per slot), <= 32 a warp with a slot per lane, <= 256 a
//      warp in shared memory, bigger rows (hubs) by emitting their
//      contributions and one global two-key radix sort (galerkin_big_rows);
//   4. prefix scan of the row lengths and a compacting copy give the CSR.
constexpr int kGalMid = 256;

__global__ void k_member_fill(int n, const int *q, const int *mrp, int *fill, int *mem) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int A = q[v];
        mem[mrp[A] + atomicAdd(&fill[A], 1)] = v;
    }
}

// contributions of member position t (vertex m = mem[t]): neighbours outside q[m]
template <int W>
__global__ void k_gal_member_count(int n, const int *mem, const int *rp, const int *ci, const int *q,
                                   int *cnt) {
    SUBWARP_LOOP(W, n, t) {
        int c = 0;
        if (t < n) {
            const int m = mem[t];
            const int qm = q[m];
            for (int k = rp[m] + sw_lane_; k < rp[m + 1]; k += W) c += (q[ci[k]] != qm);
        }
        c = sub_sum<W>(c);
        if (t < n && sw_lane_ == 0) cnt[t] = c;
    }
}


template <int W>
__global__ void k_gal_member_emit(int n, const int *mem, const int *rp, const int *ci, const double *w,
                                  const int *q, const int *coff, unsigned long long *keys,
                                  unsigned *keys2, double *vals) {
    if (W == 1) {
        // thread per member, 8 entries per step with their loads/gathers in flight
        for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
            const int m = mem[t];
            const int qm = q[m], b = rp[m], e = rp[m + 1];
            int o = coff[t];
            for (int k = b; k < e; k += 8) {
                int j8[8], q8[8];
#pragma unroll
                for (int i = 0; i < 8; i++) j8[i] = k + i < e ? ci[k + i] : -1;
#pragma unroll
                for (int i = 0; i < 8; i++) q8[i] = j8[i] >= 0 ? q[j8[i]] : qm;
#pragma unroll
                for (int i = 0; i < 8; i++)
                    if (q8[i] != qm) {
                        const int lo = min(m, j8[i]), hi = max(m, j8[i]);
                        keys[o] = ((unsigned long long)(unsigned)q8[i] << 32) | (unsigned)lo;
                        keys2[o] = (unsigned)hi;
                        vals[o] = w[k + i];
                        o++;
                    }
            }
        }
        return;
    }
    SUBWARP_LOOP(W, n, t) {
        const unsigned sub_mask = (W == 32) ? 0xffffffffu
                                            : (((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1)));
        int m = 0, qm = 0, b = 0, e = 0, o = 0;
        if (t < n) { m = mem[t]; qm = q[m]; b = rp[m]; e = rp[m + 1]; o = coff[t]; }
        const int len = e - b;
        int maxlen = len;   // warp-wide max: the ballot below needs all 32 lanes
#pragma unroll
        for (int s = 16; s; s >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, s));
        for (int tt = 0; tt < maxlen; tt += W) {   // uniform within the warp
            const int k = b + tt + sw_lane_;
            bool f = false;
            int j = 0, qj = 0;
            if (tt + sw_lane_ < len) {
                j = ci[k];
                qj = q[j];
                f = (qj != qm);
            }
            const unsigned bal = __ballot_sync(0xffffffffu, f) & sub_mask;
            if (f) {
                const int rank = __popc(bal & ((1u << (threadIdx.x & 31)) - 1u));
                keys[o + rank] = ((unsigned long long)(unsigned)qj << 32) | (unsigned)min(m, j);
                keys2[o + rank] = (unsigned)max(m, j);
                vals[o + rank] = w[k];
            }
            o += __popc(bal);
        }
    }
}

// ---- rows too big for the direct kernels: global two-key radix sort
__global__ void k_big_sizes(int h, const int *lo, const int *hi, int *sz) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < h; r += gridDim.x * blockDim.x) sz[r] = hi[r] - lo[r];
}

// one CTA per big row: gather its segment into the concatenated arrays
__global__ void k_big_gather(int h, const int *lo, const int *hi, const int *boff, const unsigned *keys2,
                             unsigned *ck2, int *cidx, unsigned *crank, int *cdst) {
    for (int r = blockIdx.x; r < h; r += gridDim.x) {
        const int sb = lo[r], s = hi[r] - sb, o = boff[r];
        for (int i = threadIdx.x; i < s; i += blockDim.x) {
            ck2[o + i] = keys2[sb + i];
            cidx[o + i] = o + i;
            crank[o + i] = (unsigned)r;
            cdst[o + i] = sb + i;
        }
    }
}

__global__ void k_big_rank_of(int E, const int *idx, const unsigned *crank, unsigned *rank2) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < E; p += gridDim.x * blockDim.x)
        rank2[p] = crank[idx[p]];
}

// k1 of the concatenated element idx[p] (original position srcpos[idx[p]])
__global__ void k_big_key1_of(int E, const int *idx, const int *srcpos, const unsigned long long *keys,
                              unsigned long long *k1) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < E; p += gridDim.x * blockDim.x)
        k1[p] = keys[srcpos[idx[p]]];
}

// sorted element p (original concatenated index idx[p]) lands at the p-th slot of
// the row segments (segments are concatenated in rank order)
__global__ void k_big_place(int E, const int *idx, const int *cdst, const int *srcpos,
                            const unsigned long long *keys, const double *vals,
                            unsigned long long *keys_out, double *vals_out) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < E; p += gridDim.x * blockDim.x) {
        const int from = srcpos[idx[p]];
        keys_out[cdst[p]] = keys[from];
        vals_out[cdst[p]] = vals[from];
    }
}

// one CTA per big row: heads, block scan for run indices, sequential fold per run
__global__ void __launch_bounds__(256) k_big_fold(int h, const int *list, const int *lo, const int *hi,
                                                  const int *oo, const unsigned long long *keys,
                                                  const double *vals, int *outB, double *outW,
                                                  int *deg) {
    __shared__ int s_warp[8];
    __shared__ int s_base;
    for (int r = blockIdx.x; r < h; r += gridDim.x) {
        const int A = list[r];
        const int sb = lo[r], s = hi[r] - sb, ob = oo[r];
        if (threadIdx.x == 0) s_base = 0;
        __syncthreads();
        for (int c0 = 0; c0 < s; c0 += blockDim.x) {
            const int i = c0 + threadIdx.x;
            const bool head = i < s && (i == 0 || (keys[sb + i] >> 32) != (keys[sb + i - 1] >> 32));
            const unsigned hm = __ballot_sync(0xffffffffu, head);
            const int warp = threadIdx.x >> 5;
            if (lane_id() == 0) s_warp[warp] = __popc(hm);
            __syncthreads();
            int before = s_base;
            for (int q = 0; q < warp; q++) before += s_warp[q];
            if (head) {
                const int ri = before + __popc(hm & ((1u << lane_id()) - 1u));
                const unsigned long long B = keys[sb + i] >> 32;
                double acc = vals[sb + i];
                for (int u = i + 1; u < s && (keys[sb + u] >> 32) == B; u++) acc += vals[sb + u];
                outB[ob + ri] = (int)B;
                outW[ob + ri] = acc;
            }
            __syncthreads();
            if (threadIdx.x == 0)
                for (int q = 0; q < (int)(blockDim.x >> 5); q++) s_base += s_warp[q];
            __syncthreads();
        }
        if (threadIdx.x == 0) deg[A] = s_base;
        __syncthreads();
    }
}

template <int W>
__global__ void k_gal_write(int c, const int *rowoff, const int *crp, const int *outB,
                            const double *outW, int *cci, double *cw) {
    if (W == 1) {
        // a warp per 32 consecutive rows: their output is one contiguous range,
        // which the lanes write at consecutive positions (entry t of the range
        // comes from the row whose prefix start is the last one <= t)
        const int lane = lane_id();
        const int nwarps = gridDim.x * (blockDim.x >> 5);
        for (int A0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; A0 < c; A0 += nwarps * 32) {
            const int A = A0 + lane;
            const int o = A < c ? crp[A] : 0;
            const int sb = A < c ? rowoff[A] : 0;
            const int last = min(A0 + 32, c);
            const int o0 = __shfl_sync(0xffffffffu, o, 0);
            const int T = crp[last] - o0;
            const int rel = A < c ? o - o0 : 0x7fffffff;   // prefix start of lane's row
            for (int t0 = 0; t0 < T; t0 += 4 * 32) {
                int b4[4];
                double w4[4];
                int src[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int t = t0 + u * 32 + lane;
                    // row of entry t: the number of lanes with rel <= t, minus one
                    // (rel ascends with the lane; a binary search over the shuffles)
                    int r = 0;
#pragma unroll
                    for (int step = 16; step; step >>= 1) {
                        const int rr = __shfl_sync(0xffffffffu, rel, r + step);
                        if (rr <= t) r += step;
                    }
                    const int rs = __shfl_sync(0xffffffffu, rel, r);
                    const int sr = __shfl_sync(0xffffffffu, sb, r);
                    src[u] = t < T ? sr + (t - rs) : -1;
                }
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (src[u] >= 0) { b4[u] = outB[src[u]]; w4[u] = outW[src[u]]; }
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (src[u] >= 0) { cci[o0 + t0 + u * 32 + lane] = b4[u]; cw[o0 + t0 + u * 32 + lane] = w4[u]; }
            }
        }
        return;
    }
    SUBWARP_LOOP(W, c, A) {
        if (A < c) {
            const int sb = rowoff[A], o = crp[A], d = crp[A + 1] - o;
            for (int i = sw_lane_; i < d; i += W) {
                cci[o + i] = outB[sb + i];
                cw[o + i] = outW[sb + i];
            }
        }
    }
}

// ---- direct path (every row with <= kGalMid slots): the contributions are
// read straight from the members' CSR rows, never materialised.  The SLOTS of
// coarse row A are the fine entries (m, j) of its members m in member order,
// T_A = sum of their degrees; a slot contributes (B = q(j), lo, hi, w_mj) when
// B != A and is empty (key ~0, sorts last) otherwise.  Sorting all slots by
// (B, lo, hi) and folding runs of B gives exactly the fold of the general path.
__global__ void k_member_count_deg(int n, const int *q, const int *rp, unsigned long long *cnt_deg) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        atomicAdd(&cnt_deg[q[v]], (1ull << 32) | (unsigned)(rp[v + 1] - rp[v]));
}

__global__ void k_split_cnt_deg(int c, const unsigned long long *cnt_deg, int *mcnt, int *slots) {
    for (int A = blockIdx.x * blockDim.x + threadIdx.x; A < c; A += gridDim.x * blockDim.x) {
        const unsigned long long x = cnt_deg[A];
        mcnt[A] = (int)(x >> 32);
        slots[A] = (int)(x & 0xffffffffu);
    }
}

// class of a coarse row in the direct path: 0 = thread per row in a batch of 32
// (k_gal_direct_batch), 1 = warp per row with one slot per lane, 2 = warp in
// shared memory (<= kGalMid slots and members); 3 = too big for the direct path
constexpr int kGalBatchMembers = 4;
__device__ __forceinline__ int gal_class(int nm, int T) {
    if (nm <= kGalBatchMembers && T <= 16) return 0;
    if (nm <= 32 && T <= 32) return 1;
    if (nm <= kGalMid && T <= kGalMid) return 2;
    return 3;
}

// lists of the rows of classes 1, 2, 3 (CTA-aggregated appends: shared-memory
// counters, one global atomic per class and block; the list order is
// irrelevant: every row's result and place are its own)
__global__ void __launch_bounds__(256) k_gal_classify(int c, const int *mrp, const int *toff, int *l1, int *l2,
                                                      int *l3, int *cnt) {
    __shared__ int s_cnt[3], s_base[3];
    for (int A0 = blockIdx.x * blockDim.x; A0 < c; A0 += gridDim.x * blockDim.x) {   // block-uniform
        if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
        __syncthreads();
        const int A = A0 + threadIdx.x;
        int k = 0, li = 0;
        if (A < c) k = gal_class(mrp[A + 1] - mrp[A], toff[A + 1] - toff[A]);
        if (k > 0) li = atomicAdd(&s_cnt[k - 1], 1);
        __syncthreads();
        if (threadIdx.x < 3 && s_cnt[threadIdx.x]) s_base[threadIdx.x] = atomicAdd(cnt + threadIdx.x, s_cnt[threadIdx.x]);
        __syncthreads();
        if (k > 0) (k == 1 ? l1 : k == 2 ? l2 : l3)[s_base[k - 1] + li] = A;
        __syncthreads();
    }
}

// Sub-warp of W lanes per coarse row, lane s holding slot s: member table by
// lanes, slot gathers coalesced along the member rows, bitonic sort across the
// lanes by (B, lo, hi), then every head of a B run left-folds the run in order.
template <int W, bool LIST>
__global__ void __launch_bounds__(256) k_gal_direct_sw(int c, const int *list, const int *count, const int *mrp,
                                                       const int *mem, const int *toff, const int *rowoff,
                                                       const int *rp,
                                                       const int *ci, const double *w, const int *q, int *outB,
                                                       double *outW, int *deg) {
    const int cnt = LIST ? *count : c;
    const int lane = threadIdx.x & (W - 1);
    const int wl = threadIdx.x & 31;
    const unsigned sub = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << (wl & ~(W - 1)));
    for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x - wl) / W + wl / W; ;
         base += (int64_t)gridDim.x * blockDim.x / W) {
        // warp-uniform loop exit: the shuffles below need every lane of the warp
        if (__all_sync(0xffffffffu, base >= cnt)) break;
        const bool live = base < cnt;
        const int A = live ? (LIST ? list[base] : (int)base) : 0;
        int mb = 0, nm = 0, tb = 0, T = 0;
        if (live) { mb = mrp[A]; nm = mrp[A + 1] - mb; T = toff[A + 1] - toff[A]; tb = rowoff[A]; }
        const bool mine = live && (LIST || gal_class(nm, T) == 0);
        // member table: lane t holds member t, its row start and slot offset
        int mv = 0, bv = 0, d = 0;
        if (mine && lane < nm) { mv = mem[mb + lane]; bv = rp[mv]; d = rp[mv + 1] - bv; }
        int pin = d;   // inclusive prefix of the member degrees
#pragma unroll
        for (int o = 1; o < W; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, pin, o, W);
            if (lane >= o) pin += y;
        }
        // member of slot `lane`: the number of members ending at or before it
        int nmax = mine ? nm : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
        int t = 0;
        for (int u = 0; u < nmax; u++) {
            const int e = __shfl_sync(0xffffffffu, pin, u, W);
            t += (u < nm && e <= lane);
        }
        t = min(t, W - 1);
        const int m = __shfl_sync(0xffffffffu, mv, t, W);
        const int b = __shfl_sync(0xffffffffu, bv, t, W);
        const int ps = __shfl_sync(0xffffffffu, pin - d, t, W);
        unsigned long long key = ~0ull;
        unsigned k2 = ~0u;
        double v = 0.0;
        if (mine && lane < T) {
            const int k = b + lane - ps;
            const int j = ci[k];
            const double x = w[k];
            const int B = q[j];
            if (B != A) {
                key = ((unsigned long long)(unsigned)B << 32) | (unsigned)min(m, j);
                k2 = (unsigned)max(m, j);
                v = x;
            }
        }
        // bitonic sort across the W lanes, ascending (B, lo, hi); empty slots last
#pragma unroll
        for (int kk = 2; kk <= W; kk <<= 1)
#pragma unroll
            for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, jj, W);
                const unsigned ok2 = __shfl_xor_sync(0xffffffffu, k2, jj, W);
                const double ov = __shfl_xor_sync(0xffffffffu, v, jj, W);
                const bool up = (lane & kk) == 0;
                const bool lower = (lane & jj) == 0;
                const bool other_less = ok < key || (ok == key && ok2 < k2);
                // the lower lane of an ascending pair keeps the smaller entry
                if (other_less == (lower == up)) { key = ok; k2 = ok2; v = ov; }
            }
        const unsigned Bm = (unsigned)(key >> 32);
        const unsigned Bprev = __shfl_up_sync(0xffffffffu, Bm, 1, W);
        const bool head = key != ~0ull && (lane == 0 || Bprev != Bm);
        // left fold of the run starting at a head, in order; the loop runs to
        // the longest run of the warp (runs end at the next head or the first
        // empty slot -- the empty slots sort last)
        const unsigned hm = __ballot_sync(0xffffffffu, head) & sub;
        const unsigned fm = __ballot_sync(0xffffffffu, key != ~0ull) & sub;
        int runlen = 0;
        if (head) {
            const unsigned after = (hm | ~fm) & sub & ~((2u << wl) - 1u);   // later heads / empty slots
            const int nxt = after ? __ffs(after) - 1 : (wl | (W - 1)) + 1;
            runlen = nxt - wl;
        }
        const int maxrun = __reduce_max_sync(0xffffffffu, (unsigned)runlen);
        double acc = v;
        for (int u = 1; u < maxrun; u++) {
            const double x = __shfl_down_sync(0xffffffffu, v, u, W);
            if (u < runlen) acc += x;
        }
        if (head) {
            const int r = __popc(hm & ((1u << wl) - 1u));
            outB[tb + r] = (int)Bm;
            outW[tb + r] = acc;
        }
        if (mine && lane == 0) deg[A] = __popc(hm);
    }
}

// Sort-and-fold of one row's <= CAP slots (smem at P: coarse column B, or -1
// for an edge inside the aggregate; lo = min(m, j); the weight) on ONE 64-bit
// key per slot, (B << 33 | lo << 4 | slot), in batch_sort_fold below.  The slot index breaks the ties of
// (B, lo) in the order of hi, because the slots run through the members in
// ascending order and every member row in ascending column order: equal lo is
// either one member m < j with several neighbours j in B (slot order = j order)
// or one neighbour j < m adjacent to several members (slot order = m order).
// So the runs of B come out in the R3 order (lo, hi) and are left-folded.
// Requires B < 2^27, vertex ids < 2^29 and ascending CSR rows (the input
// contract of fiedler_create; every Galerkin output row ascends in B).
// All 32 lanes: lane rows with Tm > 0 are sorted and folded here; every lane
// reserves `resv` output entries (its fold's run count when resv < 0) in the
// batch's output block that starts at bbase, dense in lane order, and returns
// its offset there in *off (its run count as the result).
template <int CAP>
__device__ __forceinline__ int batch_sort_fold(const int *KB, const int *LO, const double *V, int P, int Tm,
                                               int resv, int bbase, int lane, int *outB, double *outW,
                                               int *off) {
    unsigned long long k[CAP];
#pragma unroll
    for (int s = 0; s < CAP; s++) {
        const int B = s < Tm ? KB[P + s] : -1;
        k[s] = B < 0 ? ~0ull
                     : ((unsigned long long)B << 33) | ((unsigned long long)(unsigned)LO[P + s] << 4) |
                           (unsigned long long)s;
    }
#pragma unroll
    for (int kk = 2; kk <= CAP; kk <<= 1)
#pragma unroll
        for (int jj = kk >> 1; jj > 0; jj >>= 1)
#pragma unroll
            for (int i = 0; i < CAP; i++) {
                const int l = i ^ jj;
                if (l > i) {
                    const unsigned long long a = min(k[i], k[l]), b = max(k[i], k[l]);
                    if ((i & kk) == 0) { k[i] = a; k[l] = b; } else { k[i] = b; k[l] = a; }
                }
            }
    int runs = k[0] != ~0ull;
#pragma unroll
    for (int i = 1; i < CAP; i++) runs += k[i] != ~0ull && (k[i] >> 33) != (k[i - 1] >> 33);
    const int r = resv < 0 ? runs : resv;
    int Q = r;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, Q, o);
        if (lane >= o) Q += y;
    }
    Q += bbase - r;
    *off = Q;
    int *oB = outB + Q;
    double *oW = outW + Q;
    int nr = 0;
    unsigned curB = 0;
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < CAP; i++) {
        if (k[i] != ~0ull) {
            const unsigned B = (unsigned)(k[i] >> 33);
            const double x = V[P + (int)(k[i] & 15u)];
            if (i == 0) { curB = B; acc = x; }
            else if (B != curB) {
                oB[nr] = (int)curB; oW[nr] = acc; nr++;
                curB = B; acc = x;
            } else {
                acc += x;
            }
        }
    }
    if (k[0] != ~0ull) { oB[nr] = (int)curB; oW[nr] = acc; }
    return runs;
}

// Batches of 32 consecutive coarse rows per warp, class 0 only: lane = row
// reads its row's members and lays its slot descriptors (CSR position, row) out
// in shared memory; the lanes then gather all slots of the batch together
// (consecutive slots are consecutive CSR entries); finally every lane sorts and
// folds its own row in registers (batch_sort_fold) and writes it to the dense
// output block of the batch (rowoff[A] = its offset; the other classes' rows
// keep T_A entries reserved there).  Without the b64 premises (`b64` false)
// every class-0 row is appended to `redo` for the warp-per-row kernel.
#ifndef FDL_GAL_BATCH_WARPS
#define FDL_GAL_BATCH_WARPS 4
#endif
constexpr int kGalBatchWarps = FDL_GAL_BATCH_WARPS;   // warps (32-row batches) per CTA
constexpr int kGalBatchSlots = 32 * 16;
#ifndef FDL_GAL_UNROLL
#define FDL_GAL_UNROLL 8
#endif
constexpr int kGalGatherUnroll = FDL_GAL_UNROLL;
__global__ void __launch_bounds__(kGalBatchWarps * 32) k_gal_direct_batch(
    int c, bool b64, const int *mrp, const int *mem, const int *toff, const int *rp, const int *ci,
    const double *w, const int *q, int *outB, double *outW, int *deg, int *rowoff, int *redo, int *redo_count) {
    __shared__ int skb[kGalBatchWarps][kGalBatchSlots];
    __shared__ int slo[kGalBatchWarps][kGalBatchSlots];
    __shared__ double sv[kGalBatchWarps][kGalBatchSlots];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    int *KB = skb[warp];
    int *LO = slo[warp];
    double *V = sv[warp];
    int *VA = reinterpret_cast<int *>(V);   // the slot's row during the gather
    const int64_t nw = (int64_t)gridDim.x * kGalBatchWarps;
    for (int64_t base = ((int64_t)blockIdx.x * kGalBatchWarps + warp) * 32; base < c; base += nw * 32) {
        const int A = (int)(base + lane);
        const bool live = A < c;
        int mb = 0, nm = 0, tb = 0, T = 0;
        if (live) { mb = mrp[A]; nm = mrp[A + 1] - mb; tb = toff[A]; T = toff[A + 1] - tb; }
        const bool mine = live && gal_class(nm, T) == 0;
        const int Tm = mine ? T : 0;
        int P = Tm;   // inclusive, then exclusive prefix of the slot counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, P, o);
            if (lane >= o) P += y;
        }
        const int total = __shfl_sync(0xffffffffu, P, 31);
        P -= Tm;
        // members, their row starts and slot offsets
        int m[kGalBatchMembers], b[kGalBatchMembers], p[kGalBatchMembers + 1];
#pragma unroll
        for (int t = 0; t < kGalBatchMembers; t++) m[t] = (mine && t < nm) ? mem[mb + t] : 0x7fffffff;
        // members in ascending order (sort_fold_b64 relies on it)
#pragma unroll
        for (int kk = 2; kk <= kGalBatchMembers; kk <<= 1)
#pragma unroll
            for (int jj = kk >> 1; jj > 0; jj >>= 1)
#pragma unroll
                for (int t = 0; t < kGalBatchMembers; t++) {
                    const int l = t ^ jj;
                    if (l > t) {
                        const int lo = min(m[t], m[l]), hi = max(m[t], m[l]);
                        if ((t & kk) == 0) { m[t] = lo; m[l] = hi; } else { m[t] = hi; m[l] = lo; }
                    }
                }
        p[0] = 0;
#pragma unroll
        for (int t = 0; t < kGalBatchMembers; t++) {
            const bool ok = mine && t < nm;
            b[t] = ok ? rp[m[t]] : 0;
            p[t + 1] = p[t] + (ok ? rp[m[t] + 1] - b[t] : 0);
        }
#pragma unroll
        for (int s2 = 0; s2 < 16; s2++) {
            if (s2 < Tm) {
                int bt = b[0], pt = p[0], mt = m[0];
#pragma unroll
                for (int u = 1; u < kGalBatchMembers; u++)
                    if (s2 >= p[u]) { bt = b[u]; pt = p[u]; mt = m[u]; }
                KB[P + s2] = bt + s2 - pt;
                LO[P + s2] = mt;
                VA[2 * (P + s2)] = A;
            }
        }
        __syncwarp();
        // gather every slot of the batch, kGalGatherUnroll per lane in flight
        for (int i0 = 0; i0 < total; i0 += 32 * kGalGatherUnroll) {
            int kk[kGalGatherUnroll], aa[kGalGatherUnroll], jj[kGalGatherUnroll];
            double xx[kGalGatherUnroll];
#pragma unroll
            for (int u = 0; u < kGalGatherUnroll; u++) {
                const int i = i0 + u * 32 + lane;
                const bool ok = i < total;
                kk[u] = ok ? KB[i] : 0;
                aa[u] = ok ? VA[2 * i] : -1;
            }
#pragma unroll
            for (int u = 0; u < kGalGatherUnroll; u++) {
                xx[u] = aa[u] >= 0 ? w[kk[u]] : 0.0;
                jj[u] = aa[u] >= 0 ? ci[kk[u]] : 0;
            }
#pragma unroll
            for (int u = 0; u < kGalGatherUnroll; u++) kk[u] = aa[u] >= 0 ? q[jj[u]] : 0;
#pragma unroll
            for (int u = 0; u < kGalGatherUnroll; u++) {
                const int i = i0 + u * 32 + lane;
                if (aa[u] < 0) continue;
                KB[i] = kk[u] != aa[u] ? kk[u] : -1;
                LO[i] = min(LO[i], jj[u]);
                V[i] = xx[u];
            }
        }
        __syncwarp();
        // folded here: class-0 rows under the b64 premises; the rest reserve T
        const int Tf = b64 ? Tm : 0;
        const int resv = (mine && b64) ? -1 : (live ? T : 0);
        const int bbase = __shfl_sync(0xffffffffu, tb, 0);   // toff of the batch's first row
        int off, d;
        if (__all_sync(0xffffffffu, Tf <= 8))
            d = batch_sort_fold<8>(KB, LO, V, P, Tf, resv, bbase, lane, outB, outW, &off);
        else
            d = batch_sort_fold<16>(KB, LO, V, P, Tf, resv, bbase, lane, outB, outW, &off);
        if (live) rowoff[A] = off;
        if (mine) {
            if (b64) deg[A] = d;
            else redo[atomicAdd(redo_count, 1)] = A;
        }
        __syncwarp();
    }
}

// warp per coarse row (<= kGalMid slots and members): member table and slots in
// shared memory, bitonic sort there, heads of the B runs fold them in order
constexpr int kGalDirectWarps = 4;
__global__ void __launch_bounds__(kGalDirectWarps * 32) k_gal_direct_warp(
    const int *list, const int *count, const int *mrp, const int *mem, const int *toff, const int *rowoff,
    const int *rp, const int *ci, const double *w, const int *q, int *outB, double *outW, int *deg) {
    __shared__ unsigned long long sk[kGalDirectWarps][kGalMid];
    __shared__ unsigned sk2[kGalDirectWarps][kGalMid];
    __shared__ double sv[kGalDirectWarps][kGalMid];
    __shared__ int sm_m[kGalDirectWarps][kGalMid], sm_b[kGalDirectWarps][kGalMid],
        sm_p[kGalDirectWarps][kGalMid];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int cnt = *count;
    unsigned long long *K = sk[warp];
    unsigned *K2 = sk2[warp];
    double *V = sv[warp];
    int *Mm = sm_m[warp], *Mb = sm_b[warp], *Mp = sm_p[warp];
    for (int idx = blockIdx.x * kGalDirectWarps + warp; idx < cnt; idx += gridDim.x * kGalDirectWarps) {
        const int A = list[idx];
        const int mb = mrp[A], nm = mrp[A + 1] - mb, tb = rowoff[A], T = toff[A + 1] - toff[A];
        // member table with the exclusive prefix of the member degrees
        int carry = 0;
        for (int t0 = 0; t0 < nm; t0 += 32) {
            const int t = t0 + lane;
            int mv = 0, bv = 0, d = 0;
            if (t < nm) { mv = mem[mb + t]; bv = rp[mv]; d = rp[mv + 1] - bv; }
            int x = d;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (t < nm) { Mm[t] = mv; Mb[t] = bv; Mp[t] = carry + x - d; }
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
        __syncwarp();
        int N = 32;
        while (N < T) N <<= 1;
        for (int s = lane; s < N; s += 32) {
            unsigned long long kk = ~0ull;
            unsigned kk2 = ~0u;
            double vv = 0.0;
            if (s < T) {
                int lo = 0, hi = nm - 1;   // last t with Mp[t] <= s
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (Mp[mid] <= s) lo = mid; else hi = mid - 1;
                }
                const int mv = Mm[lo], k = Mb[lo] + s - Mp[lo];
                const int j = ci[k];
                const int B = q[j];
                if (B != A) {
                    kk = ((unsigned long long)(unsigned)B << 32) | (unsigned)min(mv, j);
                    kk2 = (unsigned)max(mv, j);
                    vv = w[k];
                }
            }
            K[s] = kk;
            K2[s] = kk2;
            V[s] = vv;
        }
        __syncwarp();
        for (int kk = 2; kk <= N; kk <<= 1)
            for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                for (int i = lane; i < N; i += 32) {
                    const int l = i ^ jj;
                    if (l > i) {
                        const bool up = (i & kk) == 0;
                        const bool gt = K[i] > K[l] || (K[i] == K[l] && K2[i] > K2[l]);
                        if (gt == up) {
                            unsigned long long tk = K[i]; K[i] = K[l]; K[l] = tk;
                            unsigned t2 = K2[i]; K2[i] = K2[l]; K2[l] = t2;
                            double tv = V[i]; V[i] = V[l]; V[l] = tv;
                        }
                    }
                }
                __syncwarp();
            }
        int base = 0;
        for (int c0 = 0; c0 < N; c0 += 32) {
            const int i = c0 + lane;
            const bool head = K[i] != ~0ull && (i == 0 || (K[i] >> 32) != (K[i - 1] >> 32));
            const unsigned hm = __ballot_sync(0xffffffffu, head);
            if (head) {
                const int r = base + __popc(hm & ((1u << lane) - 1u));
                double acc = V[i];
                for (int u = i + 1; u < N && (K[u] >> 32) == (K[i] >> 32); u++) acc += V[u];
                outB[tb + r] = (int)(K[i] >> 32);
                outW[tb + r] = acc;
            }
            base += __popc(hm);
        }
        if (lane == 0) deg[A] = base;
        __syncwarp();
    }
}


__global__ void k_set_rows_zero(int h, const int *list, int *deg) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < h; r += gridDim.x * blockDim.x) deg[list[r]] = 0;
}

// big rows (class 3) of the direct path: their members, contribution ranges
__global__ void k_big_member_counts(int h, const int *list, const int *mrp, int *nm) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < h; r += gridDim.x * blockDim.x)
        nm[r] = mrp[list[r] + 1] - mrp[list[r]];
}

__global__ void k_big_members(int h, const int *list, const int *mrp, const int *mem, const int *moff,
                              int *subm) {
    for (int r = blockIdx.x; r < h; r += gridDim.x) {
        const int mb = mrp[list[r]], nm = mrp[list[r] + 1] - mb;
        for (int i = threadIdx.x; i < nm; i += blockDim.x) subm[moff[r] + i] = mem[mb + i];
    }
}

__global__ void k_big_ranges(int h, const int *list, const int *moff, const int *coff, const int *rowoff,
                             int *lo, int *hi, int *oo) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < h; r += gridDim.x * blockDim.x) {
        lo[r] = coff[moff[r]];
        hi[r] = coff[moff[r + 1]];
        oo[r] = rowoff[list[r]];
    }
}

// The big rows: every member emits its contributions (B, lo, hi, w), one global
// two-key LSD radix sort orders each row's contributions by (B, lo, hi) (passes:
// hi, then (B, lo), then the row rank), then a CTA per row folds its runs of B
// into its reserved output slots (rowoff).
static void galerkin_big_rows(const NatGraph &g, const int *q, int c, int h, const int *biglist,
                              const int *mrp, const int *mem, const int *rowoff, int *outB, double *outW,
                              int *deg, cudaStream_t st) {
    const double avg = g.n ? (double)g.nnz / g.n : 0.0;
    DBuf nm((size_t)h * 4, st), moff((size_t)(h + 1) * 4, st);
    k_big_member_counts<<<grid_for(h), 256, 0, st>>>(h, biglist, mrp, nm.as<int>());
    FDL_LAUNCH_CK();
    scan_exclusive(nm.as<int>(), moff.as<int>(), h, moff.as<int>() + h, st);
    const int M = read_int(moff.as<int>() + h, st);
    DBuf subm((size_t)std::max(M, 1) * 4, st), cnt((size_t)std::max(M, 1) * 4, st),
        coff((size_t)(M + 1) * 4, st);
    k_big_members<<<std::min(h, kNumSMs * 8), 256, 0, st>>>(h, biglist, mrp, mem, moff.as<int>(), subm.as<int>());
    FDL_LAUNCH_CK();
    DISPATCH_WC(avg, (k_gal_member_count<W><<<sub_grid(M, W), 256, 0, st>>>(
                         M, subm.as<int>(), g.rp, g.ci, q, cnt.as<int>())));
    FDL_LAUNCH_CK();
    scan_exclusive(cnt.as<int>(), coff.as<int>(), M, coff.as<int>() + M, st);
    const int E = read_int(coff.as<int>() + M, st);
    DBuf keys((size_t)std::max(E, 1) * 8, st), keys2((size_t)std::max(E, 1) * 4, st),
        vals((size_t)std::max(E, 1) * 8, st);
    if (E > 0) {
        DISPATCH_WC(avg, (k_gal_member_emit<W><<<sub_grid(M, W), 256, 0, st>>>(
                             M, subm.as<int>(), g.rp, g.ci, g.w, q, coff.as<int>(),
                             keys.as<unsigned long long>(), keys2.as<unsigned>(), vals.as<double>())));
        FDL_LAUNCH_CK();
    }
    DBuf lo((size_t)h * 4, st), hi((size_t)h * 4, st), oo((size_t)h * 4, st), sz((size_t)h * 4, st),
        boff((size_t)(h + 1) * 4, st);
    k_big_ranges<<<grid_for(h), 256, 0, st>>>(h, biglist, moff.as<int>(), coff.as<int>(), rowoff, lo.as<int>(),
                                               hi.as<int>(), oo.as<int>());
    FDL_LAUNCH_CK();
    k_big_sizes<<<grid_for(h), 256, 0, st>>>(h, lo.as<int>(), hi.as<int>(), sz.as<int>());
    FDL_LAUNCH_CK();
    scan_exclusive(sz.as<int>(), boff.as<int>(), h, boff.as<int>() + h, st);
    const int EB = E;   // every contribution here belongs to a big row
    if (EB > 0) {
        DBuf ckey((size_t)EB * 8, st), ck2((size_t)EB * 4, st), cidx((size_t)EB * 4, st),
            crank((size_t)EB * 4, st), cdst((size_t)EB * 4, st), srcpos((size_t)EB * 4, st);
        k_big_gather<<<std::min(h, kNumSMs * 8), 256, 0, st>>>(
            h, lo.as<int>(), hi.as<int>(), boff.as<int>(), keys2.as<unsigned>(), ck2.as<unsigned>(),
            cidx.as<int>(), crank.as<unsigned>(), cdst.as<int>());
        FDL_LAUNCH_CK();
        // srcpos[o] = original position of concatenated element o (= cdst before sorting)
        FDL_CK(cudaMemcpyAsync(srcpos.p, cdst.p, (size_t)EB * 4, cudaMemcpyDeviceToDevice, st));
        // LSD radix passes, least significant key first: hi, then (B, lo), then the row rank
        radix_sort_u32_i32(ck2.as<unsigned>(), cidx.as<int>(), EB, 32, st);
        k_big_key1_of<<<grid_for(EB), 256, 0, st>>>(EB, cidx.as<int>(), srcpos.as<int>(),
                                                    keys.as<unsigned long long>(), ckey.as<unsigned long long>());
        FDL_LAUNCH_CK();
        radix_sort_u64_i32(ckey.as<unsigned long long>(), cidx.as<int>(), EB, 32 + bits_for(c - 1), st);
        DBuf rank2((size_t)EB * 4, st);
        k_big_rank_of<<<grid_for(EB), 256, 0, st>>>(EB, cidx.as<int>(), crank.as<unsigned>(), rank2.as<unsigned>());
        FDL_LAUNCH_CK();
        radix_sort_u32_i32(rank2.as<unsigned>(), cidx.as<int>(), EB, bits_for(h - 1), st);
        DBuf keys_s((size_t)E * 8, st), vals_s((size_t)E * 8, st);
        k_big_place<<<grid_for(EB), 256, 0, st>>>(EB, cidx.as<int>(), cdst.as<int>(), srcpos.as<int>(),
                                                  keys.as<unsigned long long>(), vals.as<double>(),
                                                  keys_s.as<unsigned long long>(), vals_s.as<double>());
        FDL_LAUNCH_CK();
        k_big_fold<<<std::min(h, kNumSMs * 8), 256, 0, st>>>(h, biglist, lo.as<int>(), hi.as<int>(), oo.as<int>(),
                                                            keys_s.as<unsigned long long>(), vals_s.as<double>(),
                                                            outB, outW, deg);
        FDL_LAUNCH_CK();
    } else {
        k_set_rows_zero<<<grid_for(h), 256, 0, st>>>(h, biglist, deg);
        FDL_LAUNCH_CK();
    }
}

static NatGraph galerkin(const NatGraph &g, const int *q, int c, cudaStream_t st) {
    const int n = g.n;
    const double avg = n ? (double)g.nnz / n : 0.0;
    NatGraph out;
    out.n = c;
    out.own_rp.alloc(padded((size_t)(c + 1) * 4), st);
    // 1. members grouped by aggregate (counting sort with atomics; the order
    //    inside an aggregate is irrelevant: step 3 sorts by (B, kpos))
    //    with the slot count T_A = sum of the member degrees of every row
    DBuf mem((size_t)n * 4, st), mrp((size_t)(c + 1) * 4, st), mfill((size_t)c * 4, st),
        toff((size_t)(c + 1) * 4, st);
    {
        DBuf cd((size_t)c * 8, st), slots((size_t)c * 4, st);
        FDL_CK(cudaMemsetAsync(cd.p, 0, (size_t)c * 8, st));
        k_member_count_deg<<<grid_for(n, 256, kNumSMs * 16), 256, 0, st>>>(n, q, g.rp,
                                                                            cd.as<unsigned long long>());
        FDL_LAUNCH_CK();
        k_split_cnt_deg<<<grid_for(c), 256, 0, st>>>(c, cd.as<unsigned long long>(), mfill.as<int>(),
                                                      slots.as<int>());
        FDL_LAUNCH_CK();
        scan_exclusive(mfill.as<int>(), mrp.as<int>(), c, mrp.as<int>() + c, st);
        scan_exclusive(slots.as<int>(), toff.as<int>(), c, toff.as<int>() + c, st);
    }
    FDL_CK(cudaMemsetAsync(mfill.p, 0, (size_t)c * 4, st));
    k_member_fill<<<grid_for(n, 256, kNumSMs * 16), 256, 0, st>>>(n, q, mrp.as<int>(), mfill.as<int>(),
                                                                  mem.as<int>());
    FDL_LAUNCH_CK();
    mfill.release();
    // rows by size class (gal_class): 0 in warp batches, 1 warp per row, 2 warp in
    // shared memory, 3 (big) through the sort-based path
    DBuf deg((size_t)(c + 1) * 4, st), rowoff((size_t)c * 4, st), outB((size_t)std::max(g.nnz, 1) * 4, st),
        outW((size_t)std::max(g.nnz, 1) * 8, st);
    int dc[3] = {0, 0, 0};
    DBuf dl((size_t)c * 4 * 3, st), dcnt(16, st);
    FDL_CK(cudaMemsetAsync(dcnt.p, 0, 16, st));
    k_gal_classify<<<grid_for(c), 256, 0, st>>>(c, mrp.as<int>(), toff.as<int>(), dl.as<int>(),
                                                dl.as<int>() + c, dl.as<int>() + 2 * c, dcnt.as<int>());
    FDL_LAUNCH_CK();
    readback(st, {{dc, dcnt.p, 12}});
    {
        // rows ascend: input contract.  FIEDLER_TEST_FULL_SORT=1 (tests) forces
        // the fallback that very large levels take
        const char *fs = std::getenv("FIEDLER_TEST_FULL_SORT");
        const bool b64 = c < (1 << 27) && n < (1 << 29) && !(fs && fs[0] == '1');
        DBuf redo(b64 ? 0 : (size_t)c * 4, st);
        k_gal_direct_batch<<<std::min(div_up(c, 32 * kGalBatchWarps), kNumSMs * 128 / kGalBatchWarps), kGalBatchWarps * 32, 0,
                             st>>>(c, b64, mrp.as<int>(), mem.as<int>(), toff.as<int>(), g.rp, g.ci, g.w, q,
                                   outB.as<int>(), outW.as<double>(), deg.as<int>(), rowoff.as<int>(),
                                   redo.as<int>(), dcnt.as<int>() + 3);
        FDL_LAUNCH_CK();
        if (!b64) {
            // beyond the b64 key ranges: the class-0 rows take the full (B, lo, hi)
            // sort (the kernel reads the list length on the device)
            k_gal_direct_sw<32, true><<<kNumSMs * 8, 256, 0, st>>>(
                c, redo.as<int>(), dcnt.as<int>() + 3, mrp.as<int>(), mem.as<int>(), toff.as<int>(),
                rowoff.as<int>(), g.rp, g.ci, g.w, q, outB.as<int>(), outW.as<double>(), deg.as<int>());
            FDL_LAUNCH_CK();
        }
        if (dc[0] > 0) {
            k_gal_direct_sw<32, true><<<grid_for((int64_t)dc[0] * 32, 256, kNumSMs * 16), 256, 0, st>>>(
                c, dl.as<int>(), dcnt.as<int>(), mrp.as<int>(), mem.as<int>(), toff.as<int>(),
                rowoff.as<int>(), g.rp, g.ci, g.w, q, outB.as<int>(), outW.as<double>(), deg.as<int>());
            FDL_LAUNCH_CK();
        }
        if (dc[1] > 0) {
            k_gal_direct_warp<<<std::min(div_up(dc[1], kGalDirectWarps), kNumSMs * 16), kGalDirectWarps * 32,
                                0, st>>>(dl.as<int>() + c, dcnt.as<int>() + 1, mrp.as<int>(), mem.as<int>(),
                                         toff.as<int>(), rowoff.as<int>(), g.rp, g.ci, g.w, q, outB.as<int>(),
                                         outW.as<double>(), deg.as<int>());
            FDL_LAUNCH_CK();
        }
        if (dc[2] > 0)
            galerkin_big_rows(g, q, c, dc[2], dl.as<int>() + 2 * c, mrp.as<int>(), mem.as<int>(),
                              rowoff.as<int>(), outB.as<int>(), outW.as<double>(), deg.as<int>(), st);
        toff.release();
        mem.release();
    }
    // 4. CSR assembly
    scan_exclusive(deg.as<int>(), out.own_rp.as<int>(), c, out.own_rp.as<int>() + c, st);
    out.nnz = read_int(out.own_rp.as<int>() + c, st);
    out.own_ci.alloc(padded((size_t)std::max(out.nnz, 1) * 4), st);
    out.own_w.alloc(padded((size_t)std::max(out.nnz, 1) * 8), st);
    const double cavg = c ? (double)out.nnz / c : 0.0;
    DISPATCH_WC(cavg, (k_gal_write<W><<<W == 1 ? grid_for((int64_t)div_up(c, 32) * 32, 256, kNumSMs * 16) : sub_grid(c, W), 256, 0, st>>>(
                          c, rowoff.as<int>(), out.own_rp.as<int>(), outB.as<int>(),
                          outW.as<double>(), out.own_ci.as<int>(), out.own_w.as<double>())));
    FDL_LAUNCH_CK();
    out.rp = out.own_rp.as<int>();
    out.ci = out.own_ci.as<int>();
    out.w = out.own_w.as<double>();
    return out;
}

// ================================================================= colouring (R4)
// Jones-Plassmann rounds = the greedy first-fit colouring in decreasing
// priority (pi(v), v), pi(v) = splitmix64(salt ^ v): a vertex takes the
// smallest colour not used by a higher-priority neighbour as soon as all of
// them are coloured, which fixes every colour independently of the schedule.
// All rounds run in one cooperative kernel per level.
__device__ __forceinline__ bool higher_prio(uint64_t pu, int u, uint64_t pv, int v) {
    return pu > pv || (pu == pv && u > v);
}

// First-fit colour of v from its higher-priority neighbours' colours (all final),
// by a sub-warp of W lanes (v < 0: idle lanes, which still take part in the
// warp-wide steps).  The used colours go into a shared-memory bitmap of the
// sub-warp (kBmWords x 32 colours), so hundreds of colours cost one row scan;
// only when all of them are taken does a windowed rescan look further.
constexpr int kBmWords = 64;
template <int W>
__device__ __forceinline__ void color_first_fit(int v, const int *rp, const int *ci, uint64_t salt,
                                                int *color, int lane, unsigned *bm) {
    for (int i = lane; i < kBmWords; i += W) bm[i] = 0u;
    __syncwarp();
    uint64_t pv = 0;
    int b = 0, e = 0;
    if (v >= 0) {
        pv = splitmix64(salt ^ (uint64_t)v);
        b = rp[v];
        e = rp[v + 1];
        for (int k = b + lane; k < e; k += W) {
            const int u = ci[k];
            if (!higher_prio(splitmix64(salt ^ (uint64_t)u), u, pv, v)) continue;
            const int cu = color[u];
            if (cu < 32 * kBmWords) atomicOr(&bm[cu >> 5], 1u << (cu & 31));
        }
    }
    __syncwarp();
    int col = 0x7fffffff;
    for (int i = lane; i < kBmWords; i += W) {
        const unsigned fr = ~bm[i];
        if (fr) { col = i * 32 + __ffs(fr) - 1; break; }
    }
#pragma unroll
    for (int o = W / 2; o; o >>= 1) col = min(col, __shfl_xor_sync(0xffffffffu, col, o, W));
    // rare: colours 0 .. 32 kBmWords - 1 all taken -> windows of 64 beyond
    int need_big = (v >= 0 && col == 0x7fffffff) ? 1 : 0;
    int any_big = __any_sync(0xffffffffu, need_big);   // warp-uniform loop below
    for (int wb = 32 * kBmWords; any_big; wb += 64) {
        unsigned long long m2 = 0ull;
        if (need_big)
            for (int k = b + lane; k < e; k += W) {
                const int u = ci[k];
                if (!higher_prio(splitmix64(salt ^ (uint64_t)u), u, pv, v)) continue;
                const int cu = color[u];
                if (cu >= wb && cu < wb + 64) m2 |= 1ull << (cu - wb);
            }
#pragma unroll
        for (int o = W / 2; o; o >>= 1) m2 |= __shfl_xor_sync(0xffffffffu, m2, o, W);
        if (need_big && ~m2) { col = wb + __ffsll((long long)~m2) - 1; need_big = 0; }
        any_big = __any_sync(0xffffffffu, need_big);
    }
    if (v >= 0 && lane == 0) color[v] = col;
    __syncwarp();
}

// Heavy vertices (degree > kHeavyDeg: hubs, dense coarse levels) are handled
// by the whole CTA instead of a sub-warp: otherwise one sub-warp walking a hub's
// row would hold every other CTA at the round's grid barrier.
#ifndef FDL_HEAVY_DEG
#define FDL_HEAVY_DEG 128
#endif
constexpr int kHeavyDeg = FDL_HEAVY_DEG;
constexpr int kHeavyCap = 512;

__device__ __forceinline__ int cta_sum_int(int v, int *sm) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane_id() == 0) sm[threadIdx.x >> 5] = v;
    __syncthreads();
    int t = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); k++) t += sm[k];
    __syncthreads();
    return t;
}

__device__ __forceinline__ int cta_min_int(int v, int *sm) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane_id() == 0) sm[threadIdx.x >> 5] = v;
    __syncthreads();
    int t = 0x7fffffff;
    for (int k = 0; k < (int)(blockDim.x >> 5); k++) t = min(t, sm[k]);
    __syncthreads();
    return t;
}

// number of higher-priority neighbours of v, whole CTA
__device__ __forceinline__ int cta_indeg(int v, const int *rp, const int *ci, uint64_t salt, int *sm) {
    const uint64_t pv = splitmix64(salt ^ (uint64_t)v);
    int c = 0;
    for (int k = rp[v] + threadIdx.x; k < rp[v + 1]; k += blockDim.x) {
        const int u = ci[k];
        c += higher_prio(splitmix64(salt ^ (uint64_t)u), u, pv, v);
    }
    return cta_sum_int(c, sm);
}

// first-fit colour of v (all higher-priority neighbours coloured), whole CTA
__device__ __forceinline__ void cta_first_fit(int v, const int *rp, const int *ci, uint64_t salt, int *color,
                                              unsigned *bm, int *sm) {
    for (int i = threadIdx.x; i < kBmWords; i += blockDim.x) bm[i] = 0u;
    __syncthreads();
    const uint64_t pv = splitmix64(salt ^ (uint64_t)v);
    const int b = rp[v], e = rp[v + 1];
    for (int k = b + threadIdx.x; k < e; k += blockDim.x) {
        const int u = ci[k];
        if (!higher_prio(splitmix64(salt ^ (uint64_t)u), u, pv, v)) continue;
        const int cu = color[u];
        if (cu < 32 * kBmWords) atomicOr(&bm[cu >> 5], 1u << (cu & 31));
    }
    __syncthreads();
    int col = 0x7fffffff;
    for (int i = threadIdx.x; i < kBmWords; i += blockDim.x)
        if (~bm[i]) col = min(col, i * 32 + __ffs(~bm[i]) - 1);
    col = cta_min_int(col, sm);
    for (int wb = 32 * kBmWords; col == 0x7fffffff; wb += 32 * kBmWords) {   // rare
        for (int i = threadIdx.x; i < kBmWords; i += blockDim.x) bm[i] = 0u;
        __syncthreads();
        for (int k = b + threadIdx.x; k < e; k += blockDim.x) {
            const int u = ci[k];
            if (!higher_prio(splitmix64(salt ^ (uint64_t)u), u, pv, v)) continue;
            const int cu = color[u] - wb;
            if (cu >= 0 && cu < 32 * kBmWords) atomicOr(&bm[cu >> 5], 1u << (cu & 31));
        }
        __syncthreads();
        int c2 = 0x7fffffff;
        for (int i = threadIdx.x; i < kBmWords; i += blockDim.x)
            if (~bm[i]) c2 = min(c2, wb + i * 32 + __ffs(~bm[i]) - 1);
        col = cta_min_int(c2, sm);
    }
    if (threadIdx.x == 0) color[v] = col;
    __syncthreads();
}

// W == 1 round work: colour a released vertex from its higher-priority
// neighbours' colours (all final) and release its lower-priority neighbours
// (they read colour(v) only after the round's grid barrier).  The row is taken
// 8 entries at a time with every load and atomic of a chunk in flight; two
// rows of <= 4 entries share one chunk (colour_pair_w1).
// slot i of a chunk: vertex vs[i], neighbour u[i] (-1: empty slot)
__device__ __forceinline__ void colour_chunk(const int (&vs)[8], const int (&u8)[8], const uint64_t (&pvs)[8],
                                             uint64_t salt, const int *color, int *indeg,
                                             unsigned long long &mask0, unsigned long long &mask1,
                                             CtaAppend &app, int *out, int *gcount, int *rounds_out) {
    int r8[8];
    bool hi8[8];
#pragma unroll
    for (int i = 0; i < 8; i++)
        hi8[i] = u8[i] >= 0 && higher_prio(splitmix64(salt ^ (uint64_t)u8[i]), u8[i], pvs[i], vs[i]);
#pragma unroll
    for (int i = 0; i < 8; i++) r8[i] = hi8[i] ? color[u8[i]] : 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const bool lo = u8[i] >= 0 && !hi8[i];
        const int o = atom_dec_if(&indeg[lo ? u8[i] : 0], lo);
        if (lo) r8[i] = o;
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
        if (u8[i] < 0) continue;
        if (hi8[i]) {
            unsigned long long &mk = i < 4 ? mask0 : mask1;
            if (r8[i] < 0) rounds_out[1] = 1;   // impossible: uncoloured predecessor
            else if (r8[i] < 64) mk |= 1ull << r8[i];
        } else if (r8[i] == 1) {
            app.push_safe(u8[i], out, gcount);
        }
    }
}

// Colouring state of the W == 1 rounds.  IntColourState: colour and in-degree
// in two int arrays.  ByteColourState: ONE byte per vertex -- the in-degree
// while uncoloured (bit 7 clear), 0x80 | colour once coloured -- for levels
// whose degrees are all <= kByteMaxDeg (so every colour is < 127): a quarter
// of one int array, which keeps the random accesses of the rounds in L2 (the
// int arrays of level 0 of config 4 are 2 x 268 MB; the byte state 67 MB).
struct IntColourState {
    int *color, *indeg;
    __device__ __forceinline__ int colour_of(int u) const { return color[u]; }   // < 0: uncoloured
    // predicated release of u: old in-degree (0 when pred is false)
    __device__ __forceinline__ int release(int u, bool pred) const { return atom_dec_if(&indeg[pred ? u : 0], pred); }
    __device__ __forceinline__ void set_colour(int v, int c) const { color[v] = c; }
};
constexpr int kByteMaxDeg = 126;
struct ByteColourState {
    unsigned char *s;
    __device__ __forceinline__ int colour_of(int u) const {
        const int b = s[u];
        return (b & 0x80) ? (b & 0x7f) : -1;
    }
    // the in-degree is a byte of an aligned word: subtracting 1 << shift never
    // borrows across bytes (a vertex is released exactly in-degree times)
    __device__ __forceinline__ int release(int u, bool pred) const {
        const int uu = pred ? u : 0;
        unsigned *wp = reinterpret_cast<unsigned *>(s + (uu & ~3));
        const unsigned d = 0u - (1u << (8 * (uu & 3)));   // add of -(1 << shift) mod 2^32
        unsigned old = 0u;
        asm volatile(
            "{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q atom.global.add.u32 %0, [%1], %2;\n}\n"
            : "+r"(old)
            : "l"(wp), "r"(d), "r"((int)pred)
            : "memory");
        return (int)((old >> (8 * (uu & 3))) & 0xffu);
    }
    // v's byte is 0 (in-degree reached 0): OR in the colour; the neighbouring
    // bytes of the word may be released concurrently, hence the atomic
    __device__ __forceinline__ void set_colour(int v, int c) const {
        atomicOr(reinterpret_cast<unsigned *>(s + (v & ~3)), (0x80u | (unsigned)c) << (8 * (v & 3)));
    }
};

// first free colour of v given the colours < 64 of its higher-priority
// neighbours (mask); rare: all of 0..63 taken -> windows of 64 beyond
template <class State>
__device__ __forceinline__ int first_fit_w1(int v, unsigned long long mask, const int *rp, const int *ci,
                                            uint64_t salt, const State &cs) {
    if (~mask) return __ffsll((long long)~mask) - 1;
    const uint64_t pv = splitmix64(salt ^ (uint64_t)v);
    const int b = rp[v], e = rp[v + 1];
    for (int wb = 64;; wb += 64) {
        unsigned long long m2 = 0ull;
        for (int k = b; k < e; k++) {
            const int u = ci[k];
            if (!higher_prio(splitmix64(salt ^ (uint64_t)u), u, pv, v)) continue;
            const int cu = cs.colour_of(u);
            if (cu >= wb && cu < wb + 64) m2 |= 1ull << (cu - wb);
        }
        if (~m2) return wb + __ffsll((long long)~m2) - 1;
    }
}

// W == 1 round work: colour a released vertex from its higher-priority
// neighbours' colours (all final) and release its lower-priority neighbours
// (they read colour(v) only after the round's grid barrier).  The row is taken
// 8 entries at a time with every load and atomic of a chunk in flight; two
// rows of <= 4 entries share one chunk (colour_pair_w1).
// slot i of a chunk: vertex vs[i], neighbour u[i] (-1: empty slot)
template <class State>
__device__ __forceinline__ void colour_chunk(const int (&vs)[8], const int (&u8)[8], const uint64_t (&pvs)[8],
                                             uint64_t salt, const State &cs,
                                             unsigned long long &mask0, unsigned long long &mask1,
                                             CtaAppend &app, int *out, int *gcount, int *rounds_out) {
    int r8[8];
    bool hi8[8];
#pragma unroll
    for (int i = 0; i < 8; i++)
        hi8[i] = u8[i] >= 0 && higher_prio(splitmix64(salt ^ (uint64_t)u8[i]), u8[i], pvs[i], vs[i]);
#pragma unroll
    for (int i = 0; i < 8; i++) r8[i] = hi8[i] ? cs.colour_of(u8[i]) : 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const bool lo = u8[i] >= 0 && !hi8[i];
        const int o = cs.release(u8[i], lo);
        if (lo) r8[i] = o;
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
        if (u8[i] < 0) continue;
        if (hi8[i]) {
            unsigned long long &mk = i < 4 ? mask0 : mask1;
            if (r8[i] < 0) rounds_out[1] = 1;   // impossible: uncoloured predecessor
            else if (r8[i] < 64) mk |= 1ull << r8[i];
        } else if (r8[i] == 1) {
            app.push_safe(u8[i], out, gcount);
        }
    }
}

template <class State>
__device__ __forceinline__ void colour_pair_w1(int v0, int v1, const int *rp, const int *ci, uint64_t salt,
                                               const State &cs, CtaAppend &app, int *out, int *gcount,
                                               int *rounds_out) {
    const int b0 = v0 >= 0 ? rp[v0] : 0, e0 = v0 >= 0 ? rp[v0 + 1] : 0;
    const int b1 = v1 >= 0 ? rp[v1] : 0, e1 = v1 >= 0 ? rp[v1 + 1] : 0;
    const uint64_t p0 = v0 >= 0 ? splitmix64(salt ^ (uint64_t)v0) : 0, p1 = v1 >= 0 ? splitmix64(salt ^ (uint64_t)v1) : 0;
    if (__all_sync(0xffffffffu, e0 - b0 <= 4 && e1 - b1 <= 4)) {   // warp-uniform: one chunk, both rows
        int vs[8], u8[8];
        uint64_t pvs[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const bool first = i < 4;
            const int k = (first ? b0 : b1) + (i & 3);
            vs[i] = first ? v0 : v1;
            pvs[i] = first ? p0 : p1;
            u8[i] = k < (first ? e0 : e1) ? ci[k] : -1;
        }
        unsigned long long m0 = 0ull, m1 = 0ull;
        colour_chunk(vs, u8, pvs, salt, cs, m0, m1, app, out, gcount, rounds_out);
        if (v0 >= 0) cs.set_colour(v0, first_fit_w1(v0, m0, rp, ci, salt, cs));
        if (v1 >= 0) cs.set_colour(v1, first_fit_w1(v1, m1, rp, ci, salt, cs));
        return;
    }
#pragma unroll 1
    for (int s = 0; s < 2; s++) {
        const int v = s ? v1 : v0, b = s ? b1 : b0, e = s ? e1 : e0;
        const uint64_t pv = s ? p1 : p0;
        if (v < 0) continue;
        unsigned long long mask = 0ull;
        for (int k = b; k < e; k += 8) {
            int vs[8], u8[8];
            uint64_t pvs[8];
#pragma unroll
            for (int i = 0; i < 8; i++) {
                vs[i] = v;
                pvs[i] = pv;
                u8[i] = k + i < e ? ci[k + i] : -1;
            }
            unsigned long long m0 = 0ull, m1 = 0ull;
            colour_chunk(vs, u8, pvs, salt, cs, m0, m1, app, out, gcount, rounds_out);
            mask |= m0 | m1;
        }
        cs.set_colour(v, first_fit_w1(v, mask, rp, ci, salt, cs));
    }
}

// The W == 1 colouring with the byte state (ByteColourState).  Round 0 also
// checks the degree bound; a level that breaks it leaves counts[0] = 0 and
// flag[0] = 1, and k_color_coop<1> (launched after it, gated on the flag)
// colours it with the int state instead.  The rounds are those of
// k_color_coop<1>; a last pass writes the int colours.
__global__ void __launch_bounds__(kCoopThreads, kCoopMinBlocks)
    k_color_byte(int n, const int *rp, const int *ci, uint64_t salt, int *color, unsigned char *st8,
                 int *la, int *lb, int *counts, int *rounds_out, int *flag) {
    cg::grid_group grid = cg::this_grid();
    unsigned *gbar = reinterpret_cast<unsigned *>(counts + kMaxRounds + 4);
    __shared__ int s_buf[kAppendCap];
    __shared__ int s_n, s_base, s_big;
    if (threadIdx.x == 0) { s_n = 0; s_big = 0; }
    __syncthreads();
    CtaAppend app{s_buf, &s_n, &s_base};
    int stamp = 0;
    round_stamp(stamp++);
    for (long long base = (long long)blockIdx.x * kCoopThreads; base < n; base += (long long)gridDim.x * kCoopThreads) {
        const long long idx = base + threadIdx.x;
        const int v = idx < n ? (int)idx : -1;
        int c = 0;
        if (v >= 0) {
            const int b = rp[v], e = rp[v + 1];
            if (e - b > kByteMaxDeg) {
                s_big = 1;
            } else {
                const uint64_t pv = splitmix64(salt ^ (uint64_t)v);
                for (int k = b; k < e; k++) {
                    const int u = ci[k];
                    c += higher_prio(splitmix64(salt ^ (uint64_t)u), u, pv, v);
                }
                st8[v] = (unsigned char)c;
                if (c == 0) app.push(v);
            }
        }
        __syncthreads();
        if (app.due(kAppendCap - kCoopThreads)) app.flush(la, counts);
    }
    __syncthreads();
    app.flush(la, counts);
    if (threadIdx.x == 0 && s_big) atomicOr(flag, 1);
    grid_sync_bo(grid, gbar);
    round_stamp(stamp++);
    if (*(volatile int *)flag) {   // grid-uniform: the int-state kernel takes over
        if (blockIdx.x == 0 && threadIdx.x == 0) counts[0] = 0;
        return;
    }
    const ByteColourState cs{st8};
    int *in = la, *out = lb;
    int r = 0;
    int cnt = *(volatile int *)&counts[0];
    while (cnt > 0 && r + 1 < kMaxRounds) {
        int *gcount = counts + r + 1;
        for (long long base = (long long)blockIdx.x * 2 * kCoopThreads; base < cnt;
             base += (long long)gridDim.x * 2 * kCoopThreads) {
            const long long idx = base + threadIdx.x, idx1 = idx + kCoopThreads;
            const int v = idx < cnt ? in[idx] : -1;
            const int v1 = idx1 < cnt ? in[idx1] : -1;
            colour_pair_w1(v, v1, rp, ci, salt, cs, app, out, gcount, rounds_out);
            __syncthreads();
            if (app.due(kAppendCap - 2 * kCoopThreads)) app.flush(out, gcount);
        }
        __syncthreads();
        app.flush(out, gcount);
        grid_sync_bo(grid, gbar);
        round_stamp(stamp++);
        r++;
        cnt = *(volatile int *)gcount;
        int *t = in; in = out; out = t;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) rounds_out[0] = cnt == 0 ? r : -1;
    for (long long v = (long long)blockIdx.x * kCoopThreads + threadIdx.x; v < n;
         v += (long long)gridDim.x * kCoopThreads)
        color[v] = cs.colour_of((int)v);
}

// Topological (DAG) form of the same greedy colouring: indeg[v] = number of
// higher-priority neighbours; a vertex is coloured once all of them are, then
// it releases its lower-priority neighbours.  Every vertex and edge is handled
// a constant number of times (the round-based JP rescans waiting vertices).
// The JP rounds of k_color_coop, for a group of CTAs: the whole cooperative
// grid (GridG) or, for the deep tail of a dense level's priority DAG (hundreds
// to thousands of rounds with a handful of ready vertices each), its first
// kColourTailCtas CTAs (SubG) with a barrier of their own.  In the grid, the
// rounds stop once a list is shorter than tail_list (tail_list = 0: never).
struct ColourShared {
    int *s_buf;
    int *s_n, *s_base;
    unsigned (*s_bm)[kBmWords];
    int *s_heavy;
    int *s_nh;
    int *s_red;
};
struct GridG {
    cg::grid_group &g;
    unsigned *bar;
    __device__ int nb() const { return gridDim.x; }
    __device__ int rank() const { return blockIdx.x; }
    __device__ void sync() { grid_sync_bo(g, bar); }
};
// the first K CTAs of the cooperative grid (the others have exited), with a
// barrier of their own in global memory: bar[0] arrivals, bar[1] generation
struct SubG {
    int K;
    unsigned *bar;
    __device__ int nb() const { return K; }
    __device__ int rank() const { return blockIdx.x; }
    __device__ void sync() {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned g = ld_acquire_gpu(bar + 1);
            __threadfence();
            if (atomicAdd(bar, 1u) == (unsigned)K - 1) {
                atomicExch(bar, 0u);
                __threadfence();
                atomicAdd(bar + 1, 1u);
            } else {
                while (ld_acquire_gpu(bar + 1) == g) {
                }
            }
            __threadfence();
        }
        __syncthreads();
    }
};
#ifndef FDL_COLOUR_TAIL_CTAS
#define FDL_COLOUR_TAIL_CTAS 48
#endif
// (R-MAT step 131.6 / 113.3 / 104.6 / 101.4 / 102.2 / 105.2 ms with 8 / 16 / 32 /
// 48 / 64 / 96 tail CTAs; a 16-CTA cluster kernel instead measured 112.1)
constexpr int kColourTailCtas = FDL_COLOUR_TAIL_CTAS;
// returns {round, list parity} when it hands over (a list shorter than
// tail_list), {-1, 0} when the colouring is complete
template <int W, class G>
__device__ int2 colour_rounds(G &grp, const ColourShared &sh, int n, const int *rp, const int *ci, uint64_t salt,
                              int *color, int *indeg, int *la, int *lb, int *counts, int *rounds_out, int r,
                              int parity, int tail_list, int stamp) {
    (void)n;
    CtaAppend app{sh.s_buf, sh.s_n, sh.s_base};
    const int lane = threadIdx.x & (W - 1);
    const int per_block = kCoopThreads / W;
    int *in = parity ? lb : la, *out = parity ? la : lb;
    int cnt = *(volatile int *)&counts[r];
    auto heavy_round = [&](int *hout, int *hcount) {
        const int nh = *sh.s_nh;   // read after a barrier
        for (int i = 0; i < nh; i++) {
            const int hv = sh.s_heavy[i];
            cta_first_fit(hv, rp, ci, salt, color, sh.s_bm[0], sh.s_red);
            const uint64_t pv = splitmix64(salt ^ (uint64_t)hv);
            for (int k = rp[hv] + threadIdx.x; k < rp[hv + 1]; k += blockDim.x) {
                const int u = ci[k];
                if (higher_prio(splitmix64(salt ^ (uint64_t)u), u, pv, hv)) continue;
                if (atomicSub(&indeg[u], 1) == 1) app.push_safe(u, hout, hcount);
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) *sh.s_nh = 0;
        __syncthreads();
    };
    const int NB = grp.nb(), RK = grp.rank();
    while (cnt > 0 && r + 1 < kMaxRounds) {
        if (tail_list > 0 && cnt < tail_list) return make_int2(r, in == la ? 0 : 1);   // uniform
        int *gcount = counts + r + 1;
        // W == 1: contiguous entries per CTA; W > 1: sub-warp slot s of CTA b
        // takes entry base + s * NB + b, so a short list (the deep rounds
        // of dense levels) is spread over all CTAs, at most one heavy vertex each
        // (W == 1 takes two entries per thread: idx and idx + kCoopThreads)
        for (long long base = W == 1 ? (long long)RK * 2 * kCoopThreads : 0; base < cnt;
             base += (long long)NB * (W == 1 ? 2 * kCoopThreads : per_block)) {
            const long long idx = W == 1 ? base + threadIdx.x
                                         : base + (long long)(threadIdx.x / W) * NB + RK;
            int v = idx < cnt ? in[idx] : -1;
            if (W > 1 && v >= 0 && rp[v + 1] - rp[v] > kHeavyDeg) {   // the CTA does it below
                if (lane == 0) sh.s_heavy[atomicAdd(sh.s_nh, 1)] = v;
                v = -1;
            }
            if (W == 1) {
                const long long idx1 = idx + kCoopThreads;   // the thread's second entry
                const int v1 = idx1 < cnt ? in[idx1] : -1;
                colour_pair_w1(v, v1, rp, ci, salt, IntColourState{color, indeg}, app, out, gcount, rounds_out);
            } else {
                // all higher-priority neighbours are coloured: first fit
                color_first_fit<W>(v, rp, ci, salt, color, lane, sh.s_bm[threadIdx.x / W]);
                // release the lower-priority neighbours
                if (v >= 0) {
                    const uint64_t pv = splitmix64(salt ^ (uint64_t)v);
                    for (int k = rp[v] + lane; k < rp[v + 1]; k += W) {
                        const int u = ci[k];
                        if (higher_prio(splitmix64(salt ^ (uint64_t)u), u, pv, v)) continue;
                        if (atomicSub(&indeg[u], 1) == 1) app.push_safe(u, out, gcount);
                    }
                }
            }
            __syncthreads();
            const int nh1 = *sh.s_nh;   // read by every thread before the next barrier
            __syncthreads();
            if (W > 1 && nh1 > kHeavyCap - per_block) {
                heavy_round(out, gcount);
                __syncthreads();
            }
            if (app.due(kAppendCap - 2 * kCoopThreads)) app.flush(out, gcount);
        }
        if (W > 1) heavy_round(out, gcount);
        __syncthreads();
        app.flush(out, gcount);
        grp.sync();
        round_stamp(stamp++);
        r++;
        cnt = *(volatile int *)gcount;
        int *t = in; in = out; out = t;
    }
    if (RK == 0 && threadIdx.x == 0) rounds_out[0] = cnt == 0 ? r : -1;
    return make_int2(-1, 0);
}

template <int W>
__global__ void __launch_bounds__(kCoopThreads, kCoopMinBlocks) k_color_coop(int n, const int *rp, const int *ci,
                                                             uint64_t salt, int *color, int *indeg,
                                                             int *la, int *lb, int *counts,
                                                             int *rounds_out, const int *gate, int tail_list) {
    // gated (after k_color_byte): runs only when the byte state could not be used
    if (gate && *(volatile const int *)gate == 0) return;
    cg::grid_group grid = cg::this_grid();
    unsigned *gbar = reinterpret_cast<unsigned *>(counts + kMaxRounds + 4);
    __shared__ int s_buf[kAppendCap];
    __shared__ int s_n, s_base;
    __shared__ unsigned s_bm[W > 1 ? kCoopThreads / W : 1][kBmWords];   // first-fit bitmaps
    __shared__ int s_heavy[W > 1 ? kHeavyCap : 1];
    __shared__ int s_nh;
    __shared__ int s_red[32];
    if (threadIdx.x == 0) { s_n = 0; s_nh = 0; }
    __syncthreads();
    CtaAppend app{s_buf, &s_n, &s_base};
    int stamp = 0;
    round_stamp(stamp++);
    const int lane = threadIdx.x & (W - 1);
    const int per_block = kCoopThreads / W;
    // round 0: in-degrees in the priority DAG; sources form the first list
    for (long long base = (long long)blockIdx.x * per_block; base < n;
         base += (long long)gridDim.x * per_block) {
        const long long idx = base + threadIdx.x / W;
        int v = idx < n ? (int)idx : -1;
        if (W > 1 && v >= 0 && rp[v + 1] - rp[v] > kHeavyDeg) {   // the CTA does it below
            if (lane == 0) s_heavy[atomicAdd(&s_nh, 1)] = v;
            v = -1;
        }
        int c = 0;
        if (v >= 0) {
            const uint64_t pv = splitmix64(salt ^ (uint64_t)v);
            for (int k = rp[v] + lane; k < rp[v + 1]; k += W) {
                const int u = ci[k];
                c += higher_prio(splitmix64(salt ^ (uint64_t)u), u, pv, v);
            }
        }
        c = sub_sum<W>(c);
        if (v >= 0 && lane == 0) {
            indeg[v] = c;
            if (c == 0) app.push(v);
        }
        __syncthreads();
        const int nh0 = s_nh;   // read by every thread before the next barrier
        __syncthreads();
        if (W > 1 && nh0 > kHeavyCap - per_block) {
            for (int i = 0; i < nh0; i++) {
                const int hv = s_heavy[i];
                const int hc = cta_indeg(hv, rp, ci, salt, s_red);
                if (threadIdx.x == 0) { indeg[hv] = hc; if (hc == 0) app.push_safe(hv, la, counts); }
            }
            __syncthreads();
            if (threadIdx.x == 0) s_nh = 0;
            __syncthreads();
        }
        if (app.due(kAppendCap - kCoopThreads)) app.flush(la, counts);
    }
    if (W > 1) {
        const int nh0 = s_nh;   // after the loop's last barrier; no push follows
        for (int i = 0; i < nh0; i++) {
            const int hv = s_heavy[i];
            const int hc = cta_indeg(hv, rp, ci, salt, s_red);
            if (threadIdx.x == 0) { indeg[hv] = hc; if (hc == 0) app.push_safe(hv, la, counts); }
        }
        __syncthreads();
        if (threadIdx.x == 0) s_nh = 0;
    }
    __syncthreads();
    app.flush(la, counts);
    grid_sync_bo(grid, gbar);
    round_stamp(stamp++);
    GridG grp{grid, gbar};
    const ColourShared sh{s_buf, &s_n, &s_base, s_bm, s_heavy, &s_nh, s_red};
    const int2 hand = colour_rounds<W>(grp, sh, n, rp, ci, salt, color, indeg, la, lb, counts, rounds_out, 0, 0,
                                       tail_list, stamp);
    if (hand.x < 0) return;
    // the deep tail of the DAG (short lists, hundreds of rounds): the first
    // kColourTailCtas CTAs alone, with a barrier of their own (a grid barrier
    // over every CTA cost ~10 us a round); the others leave the SMs to the
    // other streams' kernels
    const int K = min((int)gridDim.x, kColourTailCtas);
    if ((int)blockIdx.x >= K) return;
    SubG sub{K, reinterpret_cast<unsigned *>(counts + kMaxRounds + 8)};
    colour_rounds<W>(sub, sh, n, rp, ci, salt, color, indeg, la, lb, counts, rounds_out, hand.x, hand.y, 0,
                     stamp + hand.x);
}


// Small dense levels (n <= kSmallColourN, average degree >= 64: the coarse levels of power-law
// graphs: hundreds of colours, priority DAGs ~n deep): the same topological JP
// in ONE CTA, with colours, in-degrees and both work lists in shared memory
// (shared-memory atomics, __syncthreads between rounds instead of grid
// barriers).  A round takes its ready vertices kSmallChunk at a time and
// spreads ALL their row entries over the CTA (8 loads per thread in flight):
// higher-priority neighbours mark the vertex's first-fit bitmap, lower-priority
// ones are released; then one warp per vertex picks the first free colour.
constexpr int kSmallColourN = 12288;
constexpr int kSmallColourThreads = 1024;
constexpr int kSmallChunk = 64;
#ifndef FDL_SMALL_COLOUR_MINDEG
#define FDL_SMALL_COLOUR_MINDEG 64.0
#endif
constexpr double kSmallColourMinDeg = FDL_SMALL_COLOUR_MINDEG;   // sparse small levels: the grid kernel is faster
__global__ void __launch_bounds__(kSmallColourThreads, 1) k_color_small(int n, const int *rp, const int *ci,
                                                                          uint64_t salt, int *color,
                                                                          int *rounds_out) {
    extern __shared__ int sm_col[];
    int *col = sm_col, *indeg = sm_col + n, *la = sm_col + 2 * n, *lb = sm_col + 3 * n;
    __shared__ unsigned bm[kSmallChunk][kBmWords];
    __shared__ int s_off[kSmallChunk + 1], s_b[kSmallChunk], s_v[kSmallChunk];
    __shared__ unsigned long long s_pv[kSmallChunk];
    __shared__ int s_cnt[2], s_err;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    constexpr int nwarps = kSmallColourThreads / 32;
    if (threadIdx.x == 0) { s_cnt[0] = 0; s_cnt[1] = 0; s_err = 0; }
    __syncthreads();
    // in-degrees in the priority DAG: warp per vertex, 8 entries per lane in flight
    for (int v = warp; v < n; v += nwarps) {
        const uint64_t pv = splitmix64(salt ^ (uint64_t)v);
        const int b = rp[v], e = rp[v + 1];
        int c = 0;
        for (int k0 = b; k0 < e; k0 += 256) {
            int u8[8];
#pragma unroll
            for (int i = 0; i < 8; i++) u8[i] = k0 + i * 32 + lane < e ? ci[k0 + i * 32 + lane] : -1;
#pragma unroll
            for (int i = 0; i < 8; i++)
                c += u8[i] >= 0 && higher_prio(splitmix64(salt ^ (uint64_t)u8[i]), u8[i], pv, v);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) {
            indeg[v] = c;
            col[v] = -1;
            if (c == 0) la[atomicAdd(&s_cnt[0], 1)] = v;
        }
    }
    __syncthreads();
    int cur = 0, r = 0;
    int cnt = s_cnt[0];
    while (cnt > 0 && r + 1 < kMaxRounds) {
        const int *in = cur ? lb : la;
        int *out = cur ? la : lb;
        int *ocnt = &s_cnt[cur ^ 1];
        for (int c0 = 0; c0 < cnt; c0 += kSmallChunk) {
            const int m = min(kSmallChunk, cnt - c0);
            // chunk table: vertices, row starts, entry offsets (warp 0 scans)
            if (warp == 0) {
                int carry = 0;
                for (int t0 = 0; t0 < m; t0 += 32) {
                    const int t = t0 + lane;
                    int d = 0;
                    if (t < m) {
                        const int v = in[c0 + t];
                        const int b = rp[v];
                        d = rp[v + 1] - b;
                        s_v[t] = v;
                        s_b[t] = b;
                        s_pv[t] = splitmix64(salt ^ (uint64_t)v);
                    }
                    int x = d;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= o) x += y;
                    }
                    if (t < m) s_off[t] = carry + x - d;
                    carry += __shfl_sync(0xffffffffu, x, 31);
                }
                if (lane == 0) s_off[m] = carry;
            }
            for (int t = threadIdx.x; t < m * kBmWords; t += blockDim.x) bm[t / kBmWords][t % kBmWords] = 0u;
            __syncthreads();
            const int E = s_off[m];
            for (int e0 = threadIdx.x; e0 < E; e0 += 8 * kSmallColourThreads) {
                int idx[8], u8[8];
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    const int e = e0 + i * kSmallColourThreads;
                    int lo = 0, hi = m - 1;   // last t with s_off[t] <= e
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (s_off[mid] <= e) lo = mid; else hi = mid - 1;
                    }
                    idx[i] = e < E ? lo : -1;
                    u8[i] = e < E ? ci[s_b[lo] + e - s_off[lo]] : 0;
                }
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    if (idx[i] < 0) continue;
                    const int u = u8[i], t = idx[i];
                    if (higher_prio(splitmix64(salt ^ (uint64_t)u), u, s_pv[t], s_v[t])) {
                        const int cu = col[u];
                        if (cu < 0) s_err = 1;   // impossible: uncoloured predecessor
                        else if (cu < 32 * kBmWords) atomicOr(&bm[t][cu >> 5], 1u << (cu & 31));
                    } else if (atomicSub(&indeg[u], 1) == 1) {
                        out[atomicAdd(ocnt, 1)] = u;
                    }
                }
            }
            __syncthreads();
            for (int t = warp; t < m; t += nwarps) {
                const int v = s_v[t];
                int c = 0x7fffffff;
                for (int q = lane; q < kBmWords; q += 32)
                    if (~bm[t][q]) c = min(c, q * 32 + __ffs(~bm[t][q]) - 1);
#pragma unroll
                for (int o = 16; o; o >>= 1) c = min(c, __shfl_xor_sync(0xffffffffu, c, o));
                // rare: colours 0 .. 32 kBmWords - 1 all taken -> the warp rescans windows beyond
                const int b = s_b[t], e = b + s_off[t + 1] - s_off[t];
                for (int wb = 32 * kBmWords; c == 0x7fffffff; wb += 32) {
                    unsigned used = 0u;
                    for (int k = b + lane; k < e; k += 32) {
                        const int u = ci[k];
                        if (!higher_prio(splitmix64(salt ^ (uint64_t)u), u, s_pv[t], v)) continue;
                        const int cu = col[u] - wb;
                        if (cu >= 0 && cu < 32) used |= 1u << cu;
                    }
#pragma unroll
                    for (int o = 16; o; o >>= 1) used |= __shfl_xor_sync(0xffffffffu, used, o);
                    if (~used) c = wb + __ffs(~used) - 1;
                }
                if (lane == 0) col[v] = c;
            }
            __syncthreads();
        }
        cnt = *ocnt;
        r++;
        __syncthreads();
        if (threadIdx.x == 0) s_cnt[cur] = 0;   // the list just consumed is the next output
        cur ^= 1;
        __syncthreads();
    }
    for (int v = threadIdx.x; v < n; v += blockDim.x) color[v] = col[v];
    if (threadIdx.x == 0) {
        rounds_out[0] = cnt == 0 ? r : -1;
        rounds_out[1] = s_err;
    }
}

// Mid-size dense levels (n <= kClusterColourN, average degree >= 64): the same
// topological JP by ONE cluster of kColourCluster CTAs.  Vertex v lives in CTA
// v mod C (local slot v / C): its colour, in-degree and list entries sit in that
// CTA's shared memory and the other CTAs reach them through distributed shared
// memory (loads, atomics on the in-degree and the owner's next-list counter).
// Each CTA works its own list as k_color_small does; cluster barriers separate
// the rounds.
constexpr int kColourCluster = 16;
constexpr int kClusterColourLocal = 12288;   // vertices per CTA (16 bytes each in smem)
constexpr int kClusterColourN = kColourCluster * kClusterColourLocal;
__global__ void __launch_bounds__(kSmallColourThreads, 1) k_color_cluster(int n, const int *rp, const int *ci,
                                                                            uint64_t salt, int *color,
                                                                            int *rounds_out) {
    cg::cluster_group clu = cg::this_cluster();
    const int cr = (int)clu.block_rank();
    constexpr int C = kColourCluster;
    const int nloc = (n + C - 1) / C;
    extern __shared__ int sm_cc[];
    int *col = sm_cc, *indeg = sm_cc + nloc, *la = sm_cc + 2 * nloc, *lb = sm_cc + 3 * nloc;
    __shared__ unsigned bm[kSmallChunk][kBmWords];
    __shared__ int s_off[kSmallChunk + 1], s_b[kSmallChunk], s_v[kSmallChunk];
    __shared__ unsigned long long s_pv[kSmallChunk];
    __shared__ int s_cnt[2], s_err, s_total;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    constexpr int nwarps = kSmallColourThreads / 32;
    if (threadIdx.x == 0) { s_cnt[0] = 0; s_cnt[1] = 0; s_err = 0; }
    __syncthreads();
    // in-degrees of the own vertices v = cr + C * i
    for (int i = warp; i < nloc; i += nwarps) {
        const int v = cr + C * i;
        if (v >= n) break;
        const uint64_t pv = splitmix64(salt ^ (uint64_t)v);
        const int b = rp[v], e = rp[v + 1];
        int c = 0;
        for (int k0 = b; k0 < e; k0 += 256) {
            int u8[8];
#pragma unroll
            for (int q = 0; q < 8; q++) u8[q] = k0 + q * 32 + lane < e ? ci[k0 + q * 32 + lane] : -1;
#pragma unroll
            for (int q = 0; q < 8; q++)
                c += u8[q] >= 0 && higher_prio(splitmix64(salt ^ (uint64_t)u8[q]), u8[q], pv, v);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) {
            indeg[i] = c;
            col[i] = -1;
            if (c == 0) la[atomicAdd(&s_cnt[0], 1)] = v;
        }
    }
    clu.sync();
    int cur = 0, r = 0;
    int total = 0;
    if (threadIdx.x == 0) {
        int t = 0;
        for (int q = 0; q < C; q++) t += clu.map_shared_rank(&s_cnt[0], q)[0];
        s_total = t;
    }
    __syncthreads();
    total = s_total;
    while (total > 0 && r + 1 < kMaxRounds) {
        const int *in = cur ? lb : la;
        const int cnt = s_cnt[cur];
        for (int c0 = 0; c0 < cnt; c0 += kSmallChunk) {
            const int m = min(kSmallChunk, cnt - c0);
            if (warp == 0) {
                int carry = 0;
                for (int t0 = 0; t0 < m; t0 += 32) {
                    const int t = t0 + lane;
                    int d = 0;
                    if (t < m) {
                        const int v = in[c0 + t];
                        const int b = rp[v];
                        d = rp[v + 1] - b;
                        s_v[t] = v;
                        s_b[t] = b;
                        s_pv[t] = splitmix64(salt ^ (uint64_t)v);
                    }
                    int x = d;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= o) x += y;
                    }
                    if (t < m) s_off[t] = carry + x - d;
                    carry += __shfl_sync(0xffffffffu, x, 31);
                }
                if (lane == 0) s_off[m] = carry;
            }
            for (int t = threadIdx.x; t < m * kBmWords; t += blockDim.x) bm[t / kBmWords][t % kBmWords] = 0u;
            __syncthreads();
            const int E = s_off[m];
            for (int e0 = threadIdx.x; e0 < E; e0 += 8 * kSmallColourThreads) {
                int idx[8], u8[8];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const int e = e0 + q * kSmallColourThreads;
                    int lo = 0, hi = m - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (s_off[mid] <= e) lo = mid; else hi = mid - 1;
                    }
                    idx[q] = e < E ? lo : -1;
                    u8[q] = e < E ? ci[s_b[lo] + e - s_off[lo]] : 0;
                }
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    if (idx[q] < 0) continue;
                    const int u = u8[q], t = idx[q];
                    const int ow = u % C, ul = u / C;
                    if (higher_prio(splitmix64(salt ^ (uint64_t)u), u, s_pv[t], s_v[t])) {
                        const int cu = clu.map_shared_rank(col, ow)[ul];
                        if (cu < 0) s_err = 1;   // impossible: uncoloured predecessor
                        else if (cu < 32 * kBmWords) atomicOr(&bm[t][cu >> 5], 1u << (cu & 31));
                    } else if (atomicSub(clu.map_shared_rank(indeg, ow) + ul, 1) == 1) {
                        int *ocnt = clu.map_shared_rank(&s_cnt[cur ^ 1], ow);
                        int *olist = clu.map_shared_rank(cur ? la : lb, ow);
                        olist[atomicAdd(ocnt, 1)] = u;
                    }
                }
            }
            __syncthreads();
            for (int t = warp; t < m; t += nwarps) {
                const int v = s_v[t];
                int c = 0x7fffffff;
                for (int q = lane; q < kBmWords; q += 32)
                    if (~bm[t][q]) c = min(c, q * 32 + __ffs(~bm[t][q]) - 1);
#pragma unroll
                for (int o = 16; o; o >>= 1) c = min(c, __shfl_xor_sync(0xffffffffu, c, o));
                const int b = s_b[t], e = b + s_off[t + 1] - s_off[t];
                for (int wb = 32 * kBmWords; c == 0x7fffffff; wb += 32) {   // rare: > 2048 colours
                    unsigned used = 0u;
                    for (int k = b + lane; k < e; k += 32) {
                        const int u = ci[k];
                        if (!higher_prio(splitmix64(salt ^ (uint64_t)u), u, s_pv[t], v)) continue;
                        const int cu = clu.map_shared_rank(col, u % C)[u / C] - wb;
                        if (cu >= 0 && cu < 32) used |= 1u << cu;
                    }
#pragma unroll
                    for (int o = 16; o; o >>= 1) used |= __shfl_xor_sync(0xffffffffu, used, o);
                    if (~used) c = wb + __ffs(~used) - 1;
                }
                if (lane == 0) col[v / C] = c;
            }
            __syncthreads();
        }
        clu.sync();   // every push of the round landed; colours of the round final
        r++;
        if (threadIdx.x == 0) {
            int t = 0;
            for (int q = 0; q < C; q++) t += clu.map_shared_rank(&s_cnt[cur ^ 1], q)[0];
            s_total = t;
            s_cnt[cur] = 0;   // the list just consumed is the next round's output
        }
        clu.sync();   // counters reset everywhere before the next round pushes
        total = s_total;
        cur ^= 1;
    }
    for (int i = threadIdx.x; i < nloc; i += blockDim.x)
        if (cr + C * i < n) color[cr + C * i] = col[i];
    if (s_err) atomicOr(rounds_out + 1, 1);
    if (cr == 0 && threadIdx.x == 0) rounds_out[0] = total == 0 ? r : -1;
}

// The colouring of a level runs on the handle's second stream, overlapped with
// the matching / Galerkin chain of the coarser levels on the main stream; its
// colour count is read back only when the level's layout is built.
#ifndef FDL_COLOUR_GRID_FRAC
#define FDL_COLOUR_GRID_FRAC 0.3333
#endif
constexpr double kColourGridFrac = FDL_COLOUR_GRID_FRAC;
// dense levels (W = 32 sub-warps: power-law graphs) take a smaller share: their
// colouring is a long chain of rounds that slowed the concurrent Galerkin
// product of R-MAT's level 0 from 6.7 ms (alone) to 26.6 ms at a third of the
// grid (measured: R-MAT step 137.0 / 128.5 / 130.3 ms at 1/3, 0.2, 0.12; the
// grids keep 1/3: config 4 72.8 / 78.2 / 85.3 ms)
#ifndef FDL_COLOUR_GRID_FRAC_DENSE
#define FDL_COLOUR_GRID_FRAC_DENSE 0.2
#endif
constexpr double kColourGridFracDense = FDL_COLOUR_GRID_FRAC_DENSE;

struct ColourJob {
    DBuf la, lb, indeg, counts, mx, st8;
};
#ifndef FDL_BYTE_COLOUR
#define FDL_BYTE_COLOUR 1
#endif
constexpr bool kByteColour = FDL_BYTE_COLOUR;

// whether a 16-CTA cluster of k_color_cluster (1024 threads, ~210 KB shared
// memory each) can be resident on this device
static bool cluster_colour_ok() {
    static DeviceCache cache{};   // 0 unknown, 1 no, 2 yes
    std::atomic<int> &slot = cache[current_device()];
    if (slot.load() == 0) {
        int ok = 0;
        if (cudaFuncSetAttribute(k_color_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                cudaSuccess &&
            cudaFuncSetAttribute(k_color_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 16 * kClusterColourLocal) == cudaSuccess) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3(kColourCluster);
            q.blockDim = dim3(kSmallColourThreads);
            q.dynamicSmemBytes = (size_t)16 * kClusterColourLocal;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = kColourCluster;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            int nc = 0;
            ok = cudaOccupancyMaxActiveClusters(&nc, k_color_cluster, &q) == cudaSuccess && nc > 0;
        }
        (void)cudaGetLastError();
        slot.store(ok ? 2 : 1);
    }
    return slot.load() == 2;
}

#ifndef FDL_COLOUR_TAIL_LIST
#define FDL_COLOUR_TAIL_LIST 4096
#endif
constexpr int kColourTailList = FDL_COLOUR_TAIL_LIST;

static void color_launch(const NatGraph &g, uint64_t salt, DBuf &color, ColourJob &job, cudaStream_t st) {
    int n = g.n;
    const double avg = n ? (double)g.nnz / n : 0.0;
    color.alloc((size_t)n * 4, st);
    FDL_CK(cudaMemsetAsync(color.p, 0xff, (size_t)n * 4, st));
    job.la.alloc((size_t)n * 4, st);
    job.lb.alloc((size_t)n * 4, st);
    job.indeg.alloc((size_t)n * 4, st);
    job.counts.alloc((size_t)(kMaxRounds + 12) * 4, st);
    FDL_CK(cudaMemsetAsync(job.counts.p, 0, (size_t)(kMaxRounds + 12) * 4, st));
    {
        const int *rp = g.rp, *ci = g.ci;
        int *pcol = color.as<int>(), *pin = job.indeg.as<int>(), *pa = job.la.as<int>(), *pb = job.lb.as<int>(),
            *pc = job.counts.as<int>(), *pr = job.counts.as<int>() + kMaxRounds;
        const int *gate = nullptr;
        // dense levels hand the deep tail of the DAG (lists shorter than this)
        // to the first kColourTailCtas CTAs of the grid
        int tail = avg > 18 ? kColourTailList : 0;
        void *args[] = {&n, &rp, &ci, &salt, &pcol, &pin, &pa, &pb, &pc, &pr, &gate, &tail};
        if (n <= kSmallColourN && avg >= kSmallColourMinDeg) {
            static DeviceCache attr{};
            std::atomic<int> &attr_slot = attr[current_device()];
            if (!attr_slot.load()) {
                FDL_CK(cudaFuncSetAttribute(k_color_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            16 * kSmallColourN));
                attr_slot.store(1);
            }
            k_color_small<<<1, kSmallColourThreads, (size_t)16 * n, st>>>(n, rp, ci, salt, pcol, pr);
            FDL_LAUNCH_CK();
        } else if (n <= kClusterColourN && avg >= kSmallColourMinDeg && cluster_colour_ok()) {
            const int nloc = (n + kColourCluster - 1) / kColourCluster;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(kColourCluster);
            cfg.blockDim = dim3(kSmallColourThreads);
            cfg.dynamicSmemBytes = (size_t)16 * nloc;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = kColourCluster;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            FDL_CK(cudaLaunchKernelEx(&cfg, k_color_cluster, n, rp, ci, salt, pcol, pr));
        } else {
            RoundTrace tr(st, "colour");
            if (avg <= 8.5 && kByteColour) {
                // byte state (the int-state kernel below runs only if a degree is too big)
                job.st8.alloc(padded((size_t)n), st);
                unsigned char *p8 = job.st8.as<unsigned char>();
                int *flag = pc + kMaxRounds + 2;
                void *bargs[] = {&n, &rp, &ci, &salt, &pcol, &p8, &pa, &pb, &pc, &pr, &flag};
                coop_launch(k_color_byte, bargs, st, kColourGridFrac, (int64_t)n);
                gate = flag;
            }
            // a third of the co-resident grid, the matching (main stream) half:
            // both cooperative kernels fit side by side with room for the rest
            // of the coarsening chain (a full-grid cooperative launch would wait
            // for the other one to drain)
            DISPATCH_WC(avg, coop_launch(k_color_coop<W>, args, st, W == 32 ? kColourGridFracDense : kColourGridFrac,
                                         (int64_t)n * W));
            tr.report(job.counts.as<int>());
        }
    }
    job.mx.alloc(4, st);
    reduce_max_i32(color.as<int>(), n, job.mx.as<int>(), st);
    job.la.release();
    job.lb.release();
    job.indeg.release();
    job.st8.release();
}

// ================================================================= solve layout
__global__ void k_color_keys(int n, const int *color, unsigned *keys, int *vals) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        keys[v] = (unsigned)color[v];
        vals[v] = v;
    }
}


__global__ void k_inv_and_deg(int n, const int *perm, const int *rp, int *inv, int *degp) {
    const int stride = gridDim.x * blockDim.x;
    for (int t0 = blockIdx.x * blockDim.x + threadIdx.x; t0 < n; t0 += 4 * stride) {
        int v[4], d[4];
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = t0 + u * stride < n ? perm[t0 + u * stride] : -1;
#pragma unroll
        for (int u = 0; u < 4; u++) d[u] = v[u] >= 0 ? rp[v[u] + 1] - rp[v[u]] : 0;
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (v[u] >= 0) { inv[v[u]] = t0 + u * stride; degp[t0 + u * stride] = d[u]; }
    }
}

// GS layout rows: natural row v is copied to GS row inv[v] with its columns
// renumbered by inv (order kept).  Walking natural rows keeps the reads and the
// inv gathers streaming; the writes form one sequential stream per colour.
// The sub-warp handles kPermRows rows per step with all their loads in flight,
// and also yields max_i d_i (Gershgorin shift, R5) with every d_i summed in
// stored (= natural ascending) order, as the oracle.  Rows longer than a tile
// (hubs) are left to k_hub_permute: a sub-warp walking a 30000-entry row 32
// entries at a time, with a 32-step ordered fold per chunk, took ~1 ms per hub
// (R-MAT level 1: 9 ms of layout).
constexpr int kPermRows = 4;
template <int W>
__global__ void k_permute_rows(int n, const int *inv, const int *rp, const int *ci, const double *w,
                               const int *rpp, int *cip, double *wp, unsigned long long *dmax) {
    const int lane = threadIdx.x & (W - 1);
    const unsigned smask = W == 32 ? 0xffffffffu : ((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1));
    const int64_t nsub = (int64_t)gridDim.x * blockDim.x / W;
    const int64_t sub = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / W;
    double dm = 0.0;
    int lm = 0;   // longest row (dmax[1]: rows longer than a tile need piece tiles)
    for (int64_t r0 = sub; r0 < n; r0 += nsub * kPermRows) {
        int b[kPermRows], e[kPermRows], iv[kPermRows], o[kPermRows], c[kPermRows];
        double x[kPermRows];
#pragma unroll
        for (int u = 0; u < kPermRows; u++) {
            const int64_t v = r0 + u * nsub;
            const bool ok = v < n;
            b[u] = ok ? rp[v] : 0;
            e[u] = ok ? rp[v + 1] : 0;
            iv[u] = ok ? inv[v] : 0;
        }
#pragma unroll
        for (int u = 0; u < kPermRows; u++) {
            o[u] = e[u] > b[u] ? rpp[iv[u]] : 0;
            const bool ok = lane < e[u] - b[u];
            c[u] = ok ? ci[b[u] + lane] : -1;
            x[u] = ok ? w[b[u] + lane] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kPermRows; u++) {
            if (c[u] >= 0) {
                cip[o[u] + lane] = inv[c[u]];
                wp[o[u] + lane] = x[u];
            }
        }
#pragma unroll
        for (int u = 0; u < kPermRows; u++) {
            // d_v = sum of the row in order: the first W entries, then the rest
            double d = 0.0;
#pragma unroll
            for (int l = 0; l < W; l++) d += __shfl_sync(smask, x[u], l, W);
            const int len = e[u] - b[u];
            lm = max(lm, len);
            if (len > kTileT) continue;   // a hub row: k_hub_permute (its first W entries are copied)
            for (int k0 = W; k0 < len; k0 += W) {   // rows longer than W (uniform in the sub-warp)
                const int k = k0 + lane;
                double y = 0.0;
                if (k < len) {
                    cip[o[u] + k] = inv[ci[b[u] + k]];
                    y = w[b[u] + k];
                    wp[o[u] + k] = y;
                }
                const int cnt = min(W, len - k0);
                for (int l = 0; l < cnt; l++) d += __shfl_sync(smask, y, l, W);
            }
            dm = fmax(dm, d);
        }
    }
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) {
        dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o2));
        lm = max(lm, __shfl_xor_sync(0xffffffffu, lm, o2));
    }
    if (lane_id() == 0) {
        atomicMax(dmax, (unsigned long long)__double_as_longlong(dm));
        atomicMax(dmax + 1, (unsigned long long)lm);
    }
}

__global__ void k_gather_i32(int k, const int *src, const int *idx, int *out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
        out[i] = src[idx[i]];
}

// colour segment starts of the GS layout (segstart[c] = first row of colour c,
// -1 when empty) -> seg[c] with empty colours taking the next start,
// seg[ncolors] = n, and their nonzero offsets segnnz[c] = rp[seg[c]]
__global__ void k_seg_fix(int ncolors, int n, const int *segstart, const int *rp, int *seg, int *segnnz) {
    int next = n;
    seg[ncolors] = n;
    segnnz[ncolors] = rp[n];
    for (int k = ncolors - 1; k >= 0; k--) {
        const int s = segstart[k];
        next = s < 0 ? next : s;
        seg[k] = next;
        segnnz[k] = rp[next];
    }
}

// Tiles of the row range [s0, s1): tile t holds the rows whose coordinate
// rp[r] + r lies in [C0 + t*kTileT, C0 + (t+1)*kTileT), C0 = rp[s0] + s0.
// The coordinate is strictly increasing in r, so the bounds are binary searches.
__device__ __forceinline__ int lower_bound_coord(const int *rp, int lo, int hi, long long target) {
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if ((long long)rp[mid] + mid < target) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void k_make_tiles(const int *rp, int s0, int s1, int ntiles, Tile *out) {
    const long long C0 = (long long)rp[s0] + s0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x) {
        int a = t == 0 ? s0 : lower_bound_coord(rp, s0, s1, C0 + (long long)t * kTileT);
        int b = (t + 1 == ntiles) ? s1 : lower_bound_coord(rp, s0, s1, C0 + (long long)(t + 1) * kTileT);
        out[t] = make_int2(a, b);
    }
}

// the GS tiles of every colour in one launch: tile t belongs to the colour c
// with ctile[c] <= t < ctile[c + 1] (binary search), then as k_make_tiles
// (cwin[c]: window tiles of colour c; the slots after them hold hub piece tiles)
// tile offsets of the colours (ctile, ncolors + 1) and their window tile
// counts (cwin): in the kernel parameters (inline in the launch, no copy) up
// to kCtParam colours, else in device memory
constexpr int kCtParam = 512;
struct CtParam {
    int ctile[kCtParam + 1];
    int cwin[kCtParam];
    __device__ int ct(int i) const { return ctile[i]; }
    __device__ int cw(int i) const { return cwin[i]; }
};
struct CtPtr {
    const int *ctile, *cwin;
    __device__ int ct(int i) const { return ctile[i]; }
    __device__ int cw(int i) const { return cwin[i]; }
};
template <class CT>
__global__ void k_make_tiles_colours(const int *rp, const int *seg, const CT T, int ncolors, Tile *out) {
    const int nt = T.ct(ncolors);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        int lo = 0, hi = ncolors - 1;   // last c with ctile[c] <= t
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (T.ct(mid) <= t) lo = mid; else hi = mid - 1;
        }
        const int c = lo, s0 = seg[c], s1 = seg[c + 1], tl = t - T.ct(c), ntc = T.cw(c);
        if (tl >= ntc) continue;
        const long long C0 = (long long)rp[s0] + s0;
        const int a = tl == 0 ? s0 : lower_bound_coord(rp, s0, s1, C0 + (long long)tl * kTileT);
        const int b = (tl + 1 == ntc) ? s1 : lower_bound_coord(rp, s0, s1, C0 + (long long)(tl + 1) * kTileT);
        out[t] = make_int2(a, b);
    }
}

// rows longer than a tile (hubs of power-law levels): {GS row, natural id, length}
constexpr int kMaxHubs = 1 << 16;
__global__ void k_hub_find(int n, const int *rp, const int *perm, int *count, int4 *list) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int len = rp[r + 1] - rp[r];
        if (len > kTileT) {
            const int i = atomicAdd(count, 1);
            if (i < kMaxHubs) list[i] = make_int4(r, perm[r], len, 0);
        }
    }
}
// hub rows of the GS layout (list from k_hub_find: {GS row, natural id, length}):
// a CTA per row copies entries W.. (k_permute_rows copied the first W) with
// renumbered columns, 4 per thread in flight, and stages the weights chunk by
// chunk in shared memory, where thread 0 folds d_v in stored order (the
// oracle's order) without waiting on global loads
constexpr int kHubChunk = 4096;
__global__ void __launch_bounds__(256) k_hub_permute(int nh, const int4 *hubs, int W, const int *inv, const int *rp,
                                                     const int *ci, const double *w, const int *rpp, int *cip,
                                                     double *wp, unsigned long long *dmax) {
    __shared__ double sw[kHubChunk];
    for (int h = blockIdx.x; h < nh; h += gridDim.x) {
        const int4 hb = hubs[h];
        const int b = rp[hb.y], len = hb.z, o = rpp[hb.x];
        double d = 0.0;
        for (int c0 = 0; c0 < len; c0 += kHubChunk) {
            const int cn = min(kHubChunk, len - c0);
            for (int i0 = threadIdx.x; i0 < cn; i0 += 4 * blockDim.x) {
                int c[4];
                double y[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int i = i0 + u * blockDim.x;
                    c[u] = i < cn ? ci[b + c0 + i] : -1;
                    y[u] = i < cn ? w[b + c0 + i] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (c[u] >= 0) {
                        const int i = i0 + u * blockDim.x;
                        sw[i] = y[u];
                        if (c0 + i >= W) {
                            cip[o + c0 + i] = inv[c[u]];
                            wp[o + c0 + i] = y[u];
                        }
                    }
            }
            __syncthreads();
            if (threadIdx.x == 0)
                for (int i = 0; i < cn; i++) d += sw[i];
            __syncthreads();
        }
        if (threadIdx.x == 0) atomicMax(dmax, (unsigned long long)__double_as_longlong(d));
    }
}
__global__ void k_scatter_tiles(int k, const int *dst, const Tile *src, Tile *tiles) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) tiles[dst[i]] = src[i];
}

static int tiles_for(long long coord_span) { return std::max(1, (int)((coord_span + kTileT - 1) / kTileT)); }

static void build_layout(NatGraph &g, const int *color_nat, int ncolors, Level &L,
                         cudaStream_t st) {
    const int n = g.n;
    const double avg = n ? (double)g.nnz / n : 0.0;
    L.n = n;
    L.nnz = g.nnz;
    L.ncolors = ncolors;
    // ---- GS layout: rows sorted (stably) by colour
    L.perm.alloc((size_t)n * 4, st);
    L.inv.alloc((size_t)n * 4, st);
    DBuf degp((size_t)n * 4, st);
    DBuf segstart((size_t)(ncolors + 1) * 4, st);
    FDL_CK(cudaMemsetAsync(segstart.p, 0xff, (size_t)(ncolors + 1) * 4, st));
    if (ncolors <= 256) {
        // one counting-sort pass: perm, inv, degrees and segment starts together
        colour_sort(color_nat, n, ncolors, g.rp, L.perm.as<int>(), L.inv.as<int>(), degp.as<int>(),
                    segstart.as<int>(), st);
    } else {
        DBuf keys((size_t)n * 4, st);
        k_color_keys<<<grid_for(n), 256, 0, st>>>(n, color_nat, keys.as<unsigned>(), L.perm.as<int>());
        FDL_LAUNCH_CK();
        radix_sort_u32_i32(keys.as<unsigned>(), L.perm.as<int>(), n, bits_for(ncolors - 1), st);
        k_seg_starts<<<grid_for(n), 256, 0, st>>>(n, keys.as<unsigned>(), segstart.as<int>());
        FDL_LAUNCH_CK();
        keys.release();
        k_inv_and_deg<<<grid_for(n), 256, 0, st>>>(n, L.perm.as<int>(), g.rp, L.inv.as<int>(), degp.as<int>());
        FDL_LAUNCH_CK();
    }
    L.rp.alloc((size_t)(n + 1) * 4 + kPadBytes, st);
    scan_exclusive(degp.as<int>(), L.rp.as<int>(), n, L.rp.as<int>() + n, st);
    degp.release();
    const size_t ci_bytes = (size_t)std::max(g.nnz, 1) * 4 + kPadBytes;
    const size_t w_bytes = (size_t)std::max(g.nnz, 1) * 8 + kPadBytes;
    L.ci.alloc(ci_bytes, st);
    L.w.alloc(w_bytes, st);
    DBuf dmax(16, st);   // {max d_i (bits of a non-negative double), longest row}
    FDL_CK(cudaMemsetAsync(dmax.p, 0, 16, st));
    DISPATCH_W(avg, (k_permute_rows<W><<<sub_grid(n, W), 256, 0, st>>>(
                         n, L.inv.as<int>(), g.rp, g.ci, g.w, L.rp.as<int>(),
                         L.ci.as<int>(), L.w.as<double>(), dmax.as<unsigned long long>())));
    FDL_LAUNCH_CK();
    // ---- PI/RQ layout: the natural CSR, take_natural() once the setup is complete

    // colour segment boundaries and their nonzero offsets -> host
    // (empty colours take the next colour's start; one round trip for all)
    std::vector<int> seg(ncolors + 1), segnnz(ncolors + 1);
    DBuf sfix((size_t)(ncolors + 1) * 8, st);
    k_seg_fix<<<1, 1, 0, st>>>(ncolors, n, segstart.as<int>(), L.rp.as<int>(), sfix.as<int>(),
                               sfix.as<int>() + ncolors + 1);
    FDL_LAUNCH_CK();
    double dm = 0.0;
    unsigned long long lenmax = 0;
    readback(st, {{seg.data(), sfix.p, (size_t)(ncolors + 1) * 4},
                  {segnnz.data(), sfix.as<int>() + ncolors + 1, (size_t)(ncolors + 1) * 4},
                  {&dm, dmax.p, 8},
                  {&lenmax, dmax.as<unsigned long long>() + 1, 8}});
    // hub rows (> kTileT entries; power-law levels only): one more round trip
    std::vector<int4> hub;   // {GS row, natural id, length, colour}
    int nhub = 0;
    DBuf hubd;
    if (lenmax > (unsigned long long)kTileT) {
        hubd.alloc(16 + (size_t)std::min(n, kMaxHubs) * 16, st);
        FDL_CK(cudaMemsetAsync(hubd.p, 0, 16, st));
        k_hub_find<<<grid_for(n), 256, 0, st>>>(n, L.rp.as<int>(), L.perm.as<int>(), hubd.as<int>(),
                                                reinterpret_cast<int4 *>(hubd.as<char>() + 16));
        FDL_LAUNCH_CK();
        readback(st, {{&nhub, hubd.p, 4}});
        FDL_REQUIRE(nhub <= kMaxHubs, FIEDLER_ERR_INTERNAL, "too many rows longer than a tile");
        // the hub rows' entries past the first W and their degrees
        const int W = avg <= 4.5 ? 4 : avg <= 9 ? 8 : avg <= 18 ? 16 : 32;   // DISPATCH_W's sub-warp
        k_hub_permute<<<std::min(nhub, kNumSMs * 8), 256, 0, st>>>(
            nhub, reinterpret_cast<const int4 *>(hubd.as<char>() + 16), W, L.inv.as<int>(), g.rp, g.ci, g.w,
            L.rp.as<int>(), L.ci.as<int>(), L.w.as<double>(), dmax.as<unsigned long long>());
        FDL_LAUNCH_CK();
        readback(st, {{&dm, dmax.p, 8}});
    }
    if (nhub > 0 && nhub <= kMaxHubs) {
        hub.resize(nhub);
        readback(st, {{hub.data(), hubd.as<char>() + 16, (size_t)nhub * 16}});
        std::sort(hub.begin(), hub.end(), [](const int4 &p, const int4 &q) { return p.x < q.x; });
        for (auto &hb : hub) hb.w = (int)(std::upper_bound(seg.begin(), seg.end(), hb.x) - seg.begin()) - 1;
    }
    // R8: c = 2 max_i d_i (Gershgorin); on a 2-vertex level 2 max d = lambda_max
    // exactly and c I - L would annihilate the only non-constant direction
    L.shift = (n == 2 ? 3.0 : 2.0) * dm;

    // tiles: GS colours, then the natural-order pass
    L.seg = seg;
    L.seg_d.alloc((size_t)(ncolors + 1) * 4, st);
    FDL_CK(cudaMemcpyAsync(L.seg_d.p, sfix.p, (size_t)(ncolors + 1) * 4, cudaMemcpyDeviceToDevice, st));
    // trailing colours small enough for the single-CTA GS kernel (<= kGsTailRows rows
    // and nonzeros small enough together); a whole small level qualifies
    {
#ifndef FDL_GS_TAIL_ROWS
#define FDL_GS_TAIL_ROWS 1024
#endif
        constexpr int kGsTailRows = FDL_GS_TAIL_ROWS;
        int c0 = ncolors;
        while (c0 > 0 && seg[ncolors] - seg[c0 - 1] <= kGsTailRows &&
               (long long)segnnz[ncolors] - segnnz[c0 - 1] <= 16LL * kGsTailRows)
            c0--;
        L.gs_tail_c0 = c0;
        // colours before the tail: a grid-wide tile pass each, except runs of
        // small colours (<= kClusterColourRows rows), one cluster launch per run
#ifndef FDL_CLUSTER_COLOUR_ROWS
#define FDL_CLUSTER_COLOUR_ROWS 4096
#endif
        constexpr int kClusterColourRows = FDL_CLUSTER_COLOUR_ROWS;
        L.gs_runs.clear();
        // kinds: 0 = grid tile pass of one colour; 1 / 2 = k_gs_multi on a
        // cluster / one CTA; 3 / 4 = k_gs_pieces on a cluster / one CTA.
        // k_gs_pieces runs (fdl_solve.cu), on dense levels (>= kGdDenseDeg
        // entries per row, where they pay off: R-MAT's 150-500 colours per level;
        // on sparse levels k_gs_multi measured the same and needs no setup):
        // colours of <= kClusterColourRows rows, or of <= kGdMaxEntries entries;
        // the trailing colours of a run of at most one piece per warp go to one CTA.
#ifndef FDL_GD_MAX_ENTRIES
#define FDL_GD_MAX_ENTRIES 262144
#endif
#ifndef FDL_GD_SINGLE_ENTRIES
#define FDL_GD_SINGLE_ENTRIES 8192
#endif
        constexpr long long kGdMaxEntries = FDL_GD_MAX_ENTRIES, kGdSingleEntries = FDL_GD_SINGLE_ENTRIES;
        constexpr long long kGdDenseDeg = 16;
        constexpr int kGdSinglePieces = 16;   // k_gs_pieces warps per CTA
        // eligibility and the one-CTA choice from bounds on the piece counts
        // (no readback): pieces(c) <= rows + entries / kGdPiece + 1, and a part
        // pair (two parts per CTA of an 8-CTA cluster) holds at most an eighth
        // of them plus the pieces of the row its cut extends over
        auto rows_of = [&](int c) { return (long long)seg[c + 1] - seg[c]; };
        auto ent_of = [&](int c) { return (long long)segnnz[c + 1] - segnnz[c]; };
        auto pbound = [&](int c) { return rows_of(c) + ent_of(c) / kGdPiece + 1; };
        auto elig = [&](int c) {
            const long long rows = rows_of(c), ent = ent_of(c);
            if (rows == 0) return true;
            if (!(rows <= kClusterColourRows || ent <= kGdMaxEntries)) return false;
            return pbound(c) / 8 + ent / kGdPiece + 2 <= kGdSlotCapHost;
        };
        auto single = [&](int c) { return ent_of(c) <= kGdSingleEntries && pbound(c) <= kGdSinglePieces; };
        std::vector<char> use(ncolors, 0);
        bool any = false;
        if (FDL_GS_PIECES && avg >= (double)kGdDenseDeg)
            for (int c = 0; c < ncolors; c++) {
                use[c] = rows_of(c) > 0 && elig(c);
                any |= use[c] != 0;
            }
        if (any) {
            build_gs_pieces(L, seg, segnnz, use, st);
            for (int c = 0; c < ncolors;) {
                if (!elig(c)) {
                    L.gs_runs.insert(L.gs_runs.end(), {c, c + 1, 0});
                    c++;
                    continue;
                }
                int e = c;
                while (e < ncolors && elig(e) && e - c < kGdMaxRunColours) e++;
                int t = e;
                while (t > c && single(t - 1)) t--;
                if (t > c) L.gs_runs.insert(L.gs_runs.end(), {c, t, 3});
                if (e > t) L.gs_runs.insert(L.gs_runs.end(), {t, e, 4});
                c = e;
            }
        } else {
            for (int c = 0; c < c0;) {
                int e = c;
                while (e < c0 && seg[e + 1] - seg[e] <= kClusterColourRows) e++;
                if (e > c) {
                    L.gs_runs.insert(L.gs_runs.end(), {c, e, 1});
                    c = e;
                } else {
                    L.gs_runs.insert(L.gs_runs.end(), {c, c + 1, 0});
                    c++;
                }
            }
            if (c0 < ncolors) L.gs_runs.insert(L.gs_runs.end(), {c0, ncolors, 2});
        }
    }
    // tiles of every pass: colour c's window tiles then its hub piece tiles,
    // the natural pass likewise (hub rows: pieces of kTileT entries, a tile each)
    std::vector<int> hpieces(ncolors + 1, 0);
    for (const auto &hb : hub) {
        const int np = div_up(hb.z, kTileT);
        hpieces[hb.w] += np;
        hpieces[ncolors] += np;
    }
    L.ctile.assign(ncolors + 1, 0);
    int nt = 0;
    std::vector<int> cnt(ncolors + 1);
    for (int c = 0; c < ncolors; c++) {
        L.ctile[c] = nt;
        long long span = (long long)(segnnz[c + 1] + seg[c + 1]) - (segnnz[c] + seg[c]);
        cnt[c] = seg[c + 1] > seg[c] ? tiles_for(span) : 0;
        nt += cnt[c] + hpieces[c];
    }
    L.ctile[ncolors] = nt;
    cnt[ncolors] = tiles_for((long long)g.nnz + n);
    nt += cnt[ncolors] + hpieces[ncolors];
    L.ntiles = nt;
    L.tiles.alloc((size_t)nt * sizeof(Tile), st);
    if (L.ctile[ncolors] > 0 && ncolors <= kCtParam) {
        CtParam T;
        std::copy(L.ctile.begin(), L.ctile.end(), T.ctile);
        std::copy(cnt.begin(), cnt.begin() + ncolors, T.cwin);
        k_make_tiles_colours<CtParam><<<grid_for(L.ctile[ncolors]), 256, 0, st>>>(
            L.rp.as<int>(), L.seg_d.as<int>(), T, ncolors, L.tiles.as<Tile>());
        FDL_LAUNCH_CK();
    } else if (L.ctile[ncolors] > 0) {
        DBuf ctd((size_t)(2 * ncolors + 1) * 4, st);
        upload(st, ctd.p, L.ctile.data(), (size_t)(ncolors + 1) * 4);
        upload(st, ctd.as<int>() + ncolors + 1, cnt.data(), (size_t)ncolors * 4);
        k_make_tiles_colours<CtPtr><<<grid_for(L.ctile[ncolors]), 256, 0, st>>>(
            L.rp.as<int>(), L.seg_d.as<int>(), CtPtr{ctd.as<int>(), ctd.as<int>() + ncolors + 1}, ncolors,
            L.tiles.as<Tile>());
        FDL_LAUNCH_CK();
    }
    k_make_tiles<<<grid_for(cnt[ncolors]), 256, 0, st>>>(g.rp, 0, n, cnt[ncolors],
                                                         L.tiles.as<Tile>() + L.ctile[ncolors]);
    FDL_LAUNCH_CK();
    if (!hub.empty()) {
        // hub lists {row, first piece tile (pass-relative), pieces, 0} per pass
        // (rows ascending), and the piece tiles {row, -(1 + piece)}
        std::vector<std::vector<int4>> per(ncolors + 1);
        std::vector<int> used(ncolors + 1, 0);
        std::vector<int> pdst;
        std::vector<Tile> ptile;
        auto add = [&](int pass, int row, int len) {
            const int np = div_up(len, kTileT), first = cnt[pass] + used[pass];
            per[pass].push_back(make_int4(row, first, np, 0));
            for (int i = 0; i < np; i++) {
                pdst.push_back(L.ctile[pass] + first + i);
                ptile.push_back(make_int2(row, -(1 + i)));
            }
            used[pass] += np;
        };
        for (const auto &hb : hub) add(hb.w, hb.x, hb.z);
        std::vector<int4> hn(hub);
        std::sort(hn.begin(), hn.end(), [](const int4 &p, const int4 &q) { return p.y < q.y; });
        for (const auto &hb : hn) add(ncolors, hb.y, hb.z);
        std::vector<int4> all;
        L.hoff.assign(ncolors + 2, 0);
        int maxpass = 0;
        for (int c = 0; c <= ncolors; c++) {
            L.hoff[c] = (int)all.size();
            all.insert(all.end(), per[c].begin(), per[c].end());
            maxpass = std::max(maxpass, (c < ncolors ? L.ctile[c + 1] : nt) - L.ctile[c]);
        }
        L.hoff[ncolors + 1] = (int)all.size();
        L.hubs.alloc(all.size() * sizeof(int4), st);
        upload(st, L.hubs.p, all.data(), all.size() * sizeof(int4));
        L.hub_part.alloc((size_t)maxpass * 16, st);
        const int k = (int)pdst.size();
        DBuf pd((size_t)k * 4, st), pt((size_t)k * sizeof(Tile), st);
        upload(st, pd.p, pdst.data(), (size_t)k * 4);
        upload(st, pt.p, ptile.data(), (size_t)k * sizeof(Tile));
        k_scatter_tiles<<<grid_for(k), 256, 0, st>>>(k, pd.as<int>(), pt.as<Tile>(), L.tiles.as<Tile>());
        FDL_LAUNCH_CK();
    }
}

// the natural CSR of a level for the PI / RQ passes: taken over from the setup
// graph when it owns padded storage, copied otherwise (the caller's level 0)
static void take_natural(NatGraph &g, Level &L, cudaStream_t st) {
    // (an owned buffer always holds the level's array: the setup's own output,
    // the staged host input, or the side-stream copy of a device input)
    auto take = [&](DBuf &own, const void *ptr, size_t bytes, DBuf &dst) {
        if (own.p && own.bytes >= padded(bytes)) {
            dst = std::move(own);
        } else {
            dst.alloc(padded(bytes), st);
            if (bytes) FDL_CK(cudaMemcpyAsync(dst.p, ptr, bytes, cudaMemcpyDeviceToDevice, st));
        }
    };
    take(g.own_rp, g.rp, (size_t)(g.n + 1) * 4, L.rpN);
    take(g.own_ci, g.ci, (size_t)g.nnz * 4, L.ciN);
    take(g.own_w, g.w, (size_t)g.nnz * 8, L.wN);
    g.rp = L.rpN.as<int>();
    g.ci = L.ciN.as<int>();
    g.w = L.wN.as<double>();
}

// ================================================================= connectivity (coarsest level)
static bool coarsest_connected(const Level &L, cudaStream_t st) {
    std::vector<int> rp(L.n + 1), ci(std::max(L.nnz, 1));
    readback(st, {{rp.data(), L.rp.p, (size_t)(L.n + 1) * 4}, {ci.data(), L.ci.p, (size_t)L.nnz * 4}});
    std::vector<char> seen(L.n, 0);
    std::vector<int> stack{0};
    seen[0] = 1;
    int cnt = 1;
    while (!stack.empty()) {
        int v = stack.back();
        stack.pop_back();
        for (int k = rp[v]; k < rp[v + 1]; k++)
            if (!seen[ci[k]]) { seen[ci[k]] = 1; cnt++; stack.push_back(ci[k]); }
    }
    return cnt == L.n;
}

__global__ void k_compose_qg(int n, const int *perm, const int *q_nat, int *qg) {
    const int stride = gridDim.x * blockDim.x;
    for (int t0 = blockIdx.x * blockDim.x + threadIdx.x; t0 < n; t0 += 4 * stride) {   // 4 gathers in flight
        int p[4], r[4];
#pragma unroll
        for (int u = 0; u < 4; u++) p[u] = t0 + u * stride < n ? perm[t0 + u * stride] : -1;
#pragma unroll
        for (int u = 0; u < 4; u++) r[u] = p[u] >= 0 ? q_nat[p[u]] : 0;
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (p[u] >= 0) qg[t0 + u * stride] = r[u];
    }
}

// FIEDLER_PHASE_TIMES=1: CUDA events around the setup phases of every level
// (read once the setup is complete; off by default: no events in the timed
// creates of the bench)
struct PhaseTimes {
    bool on = false;
    std::vector<cudaEvent_t> ev;   // per level and phase: begin, end
    explicit PhaseTimes(int max_levels) {
        const char *e = std::getenv("FIEDLER_PHASE_TIMES");
        on = e && e[0] == '1';
        ev.assign((size_t)(max_levels + 1) * 8, nullptr);   // sized once: two threads mark
    }
    ~PhaseTimes() {
        for (cudaEvent_t x : ev)
            if (x) cudaEventDestroy(x);
    }
    cudaEvent_t &at(int level, int phase, int end) {
        const size_t i = ((size_t)level * 4 + phase) * 2 + end;
        if (ev.size() <= i) ev.resize(i + 1, nullptr);
        return ev[i];
    }
    void mark(int level, int phase, int end, cudaStream_t s) {
        if (!on) return;
        cudaEvent_t &x = at(level, phase, end);
        if (!x) FDL_CK(cudaEventCreate(&x));
        FDL_CK(cudaEventRecord(x, s));
    }
    void collect(std::vector<Level> &levels) {
        if (!on) return;
        for (size_t l = 0; l < levels.size(); l++)
            for (int p = 0; p < 4; p++) {
                const size_t i = (l * 4 + p) * 2;
                if (i + 1 >= ev.size() || !ev[i] || !ev[i + 1]) continue;
                float ms = 0.f;
                FDL_CK(cudaEventSynchronize(ev[i + 1]));
                FDL_CK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
                levels[l].phase_ms[p] = ms;
            }
    }
};

// Two host threads: this one drives the coarsening chain (matching, Galerkin)
// on the main stream; a helper drives, on the second stream, the colouring and
// the GS layout of every level as soon as the level exists.  Each blocks only
// on its own stream's readbacks, so the layouts overlap the coarsening of the
// coarser levels instead of following it.  Levels and graphs live in vectors
// reserved up front (no reallocation while the helper holds references); the
// helper touches only the colouring / layout members of a Level.
struct LevelFeed {
    std::mutex mu;
    std::condition_variable cv;
    int ready = 0;      // levels whose graph is enqueued (event recorded)
    bool done = false;  // no more levels
    void publish(int r) {
        { std::lock_guard<std::mutex> lk(mu); ready = r; }
        cv.notify_all();
    }
    void finish() {
        { std::lock_guard<std::mutex> lk(mu); done = true; }
        cv.notify_all();
    }
    bool wait_for(int ell) {   // true: level ell exists; false: no such level
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return ready > ell || done; });
        return ready > ell;
    }
};

// levels first, first + stride, ... (one helper thread and stream per residue)
// fiedler_create_preset: a level's matching / aggregates and the next level
// given by the caller (fiedler_pset_*), copied into the handle's buffers
static int take_preset_match(const fiedler_preset_level &P, int n, Level &L, cudaStream_t st) {
    L.q_nat.alloc((size_t)n * 4, st);
    L.mate_nat.alloc((size_t)n * 4, st);
    FDL_CK(cudaMemcpyAsync(L.q_nat.p, P.agg, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    FDL_CK(cudaMemcpyAsync(L.mate_nat.p, P.mate, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    L.match_rounds = P.match_rounds;
    return (int)P.n_next;
}

static NatGraph take_preset_graph(const fiedler_preset_level &P, cudaStream_t st) {
    NatGraph out;
    out.n = (int)P.n_next;
    out.nnz = (int)P.nnz_next;
    out.own_rp.alloc(padded((size_t)(out.n + 1) * 4), st);
    convert_row_ptr(P.rp_next, out.n, out.nnz, out.own_rp.as<int>(), st);
    out.own_ci.alloc(padded((size_t)std::max(out.nnz, 1) * 4), st);
    out.own_w.alloc(padded((size_t)std::max(out.nnz, 1) * 8), st);
    if (out.nnz) {
        FDL_CK(cudaMemcpyAsync(out.own_ci.p, P.ci_next, (size_t)out.nnz * 4, cudaMemcpyDeviceToDevice, st));
        FDL_CK(cudaMemcpyAsync(out.own_w.p, P.w_next, (size_t)out.nnz * 8, cudaMemcpyDeviceToDevice, st));
    }
    out.rp = out.own_rp.as<int>();
    out.ci = out.own_ci.as<int>();
    out.w = out.own_w.as<double>();
    return out;
}

static void colour_and_layout(Handle &h, std::vector<NatGraph> &graphs, std::vector<cudaEvent_t> &lev_ev,
                              LevelFeed &feed, PhaseTimes &pt, cudaStream_t sb, int first, int stride) {
    for (int ell = first; feed.wait_for(ell); ell += stride) {
        Level &L = h.levels[ell];
        NatGraph &g = graphs[ell];
        // the colouring needs the pattern (level 0 from host input: its event,
        // the weights may still be copying), the layout the whole level
        FDL_CK(cudaStreamWaitEvent(sb, ell == 0 && h.ev_pattern ? h.ev_pattern : lev_ev[ell], 0));
        ColourJob job;
        pt.mark(ell, 2, 0, sb);
        int cr[3];
        if (ell < (int)h.preset.size()) {   // fiedler_create_preset: the colouring is given
            const fiedler_preset_level &P = h.preset[ell];
            L.color_nat.alloc((size_t)g.n * 4, sb);
            FDL_CK(cudaMemcpyAsync(L.color_nat.p, P.color, (size_t)g.n * 4, cudaMemcpyDeviceToDevice, sb));
            cr[0] = P.colour_rounds;
            cr[1] = 0;
            cr[2] = P.ncolors - 1;
            pt.mark(ell, 2, 1, sb);
        } else {
            color_launch(g, salt_color(h.opts.seed, ell), L.color_nat, job, sb);
            pt.mark(ell, 2, 1, sb);
            readback(sb, {{cr, job.counts.as<int>() + kMaxRounds, 8}, {cr + 2, job.mx.p, 4}});
        }
        FDL_REQUIRE(cr[0] >= 0 && cr[1] == 0, FIEDLER_ERR_INTERNAL, "colouring did not terminate");
        L.color_rounds = cr[0];
        if (ell == 0 && h.ev_pattern) FDL_CK(cudaStreamWaitEvent(sb, lev_ev[0], 0));
        pt.mark(ell, 3, 0, sb);
        build_layout(g, L.color_nat.as<int>(), cr[2] + 1, L, sb);
        // the prolongation map into GS numbering, qg = q o perm, once the
        // matching of this level is done (the next level exists)
        if (feed.wait_for(ell + 1)) {
            FDL_CK(cudaStreamWaitEvent(sb, lev_ev[ell + 1], 0));
            L.qg.alloc((size_t)L.n * 4, sb);
            k_compose_qg<<<grid_for(L.n), 256, 0, sb>>>(L.n, L.perm.as<int>(), L.q_nat.as<int>(), L.qg.as<int>());
            FDL_LAUNCH_CK();
        }
        pt.mark(ell, 3, 1, sb);
        trace_mark(sb, ell == 0 ? "L0 colour+layout (second stream)" : "Lk colour+layout (second stream)");
    }
}

void build_hierarchy(Handle &h, NatGraph &&g0) {
    cudaStream_t st = h.stream, sb = h.stream2;
    const fiedler_opts &o = h.opts;
    const int maxl = std::max(1, o.max_levels);
    PhaseTimes pt(maxl);
    bool serial = false;
    {   // FIEDLER_SERIAL_COLOUR=1 (diagnostics): colourings and layouts on the
        // main stream, after the coarsening chain, one host thread
        const char *e = std::getenv("FIEDLER_SERIAL_COLOUR");
        serial = e && e[0] == '1';
    }
    if (serial) sb = st;
    h.levels.clear();
    h.levels.reserve((size_t)maxl + 1);
    std::vector<NatGraph> graphs;
    graphs.reserve((size_t)maxl + 1);
    std::vector<cudaEvent_t> lev_ev((size_t)maxl + 1, nullptr);
    LevelFeed feed;
    // kSides helper threads colour and lay out the levels = k mod kSides on
    // side stream k, so a level's colouring starts as soon as the level exists
    // even while the previous level's layout still runs (serial: one pass on st)
    cudaStream_t sides[kSides];
    for (int k = 0; k < kSides; k++) sides[k] = serial ? sb : h.set.side[k];
    std::exception_ptr side_err[kSides];
    long long side_launches[kSides] = {};
    std::thread side[kSides];
    auto run_side = [&](int k, int first, int stride) {
        const long long l0 = g_launch_count;
        try {
            FDL_CK(cudaSetDevice(h.device));
            colour_and_layout(h, graphs, lev_ev, feed, pt, sides[k], first, stride);
        } catch (...) {
            side_err[k] = std::current_exception();
        }
        side_launches[k] = g_launch_count - l0;
    };
    if (!serial)
        for (int k = 0; k < kSides; k++) side[k] = std::thread(run_side, k, k, kSides);
    try {
        graphs.emplace_back(std::move(g0));
        for (int ell = 0;; ell++) {
            h.levels.emplace_back();
            Level &L = h.levels.back();
            NatGraph &cur = graphs.back();
            FDL_CK(cudaEventCreateWithFlags(&lev_ev[ell], cudaEventDisableTiming));
            FDL_CK(cudaEventRecord(lev_ev[ell], st));
            feed.publish(ell + 1);
            bool coarsen = cur.n > o.coarsest_size && ell + 1 < maxl;
            const bool pre = ell < (int)h.preset.size();
            FDL_REQUIRE(!pre || coarsen, FIEDLER_ERR_ARG,
                        "a preset level must be one fiedler_create coarsens (n > coarsest_size, below max_levels)");
            if (coarsen) {
                pt.mark(ell, 0, 0, st);
                int c = pre ? take_preset_match(h.preset[ell], cur.n, L, st)
                            : hec_parallel(cur, salt_match(o.seed, ell), L.q_nat, L.mate_nat, L.match_rounds, st);
                pt.mark(ell, 0, 1, st);
                trace_mark(st, ell == 0 ? "L0 matching" : "Lk matching");
                // stall guard (R9): stop when HEC no longer shrinks the graph
                if ((double)c > 0.95 * (double)cur.n || c < 2) {
                    FDL_REQUIRE(!pre, FIEDLER_ERR_ARG, "a preset level stalls the coarsening (R9)");
                    coarsen = false;
                    L.q_nat.release();
                    L.mate_nat.release();
                } else {
                    pt.mark(ell, 1, 0, st);
                    NatGraph next = pre ? take_preset_graph(h.preset[ell], st)
                                        : galerkin(cur, L.q_nat.as<int>(), c, st);
                    pt.mark(ell, 1, 1, st);
                    trace_mark(st, ell == 0 ? "L0 galerkin" : "Lk galerkin");
                    graphs.emplace_back(std::move(next));
                }
            }
            if (!coarsen) break;
        }
    } catch (...) {
        feed.finish();
        for (int k = 0; k < kSides; k++) {
            if (side[k].joinable()) side[k].join();
            cudaStreamSynchronize(sides[k]);
        }
        for (cudaEvent_t e : lev_ev)
            if (e) cudaEventDestroy(e);
        throw;
    }
    feed.finish();
    if (serial) {
        run_side(0, 0, 1);
    } else {
        for (int k = 0; k < kSides; k++) side[k].join();
        for (int k = 0; k < kSides; k++) g_launch_count += side_launches[k];
    }
    for (cudaEvent_t e : lev_ev)
        if (e) cudaEventDestroy(e);
    for (int k = 0; k < kSides; k++)
        if (side_err[k]) {
            for (int j = 0; j < kSides; j++) cudaStreamSynchronize(sides[j]);
            std::rethrow_exception(side_err[k]);
        }
    // the main stream continues after the colourings and layouts
    for (int k = 0; k < kSides; k++) {
        FDL_CK(cudaEventRecord(h.set.sev[k], sides[k]));
        FDL_CK(cudaStreamWaitEvent(st, h.set.sev[k], 0));
    }
    trace_mark(st, "colourings and layouts joined");
    const int J = (int)h.levels.size() - 1;
    for (int ell = 0; ell <= J; ell++) take_natural(graphs[ell], h.levels[ell], st);
    host_wait(st);
    pt.collect(h.levels);
    trace_mark(st, "compose qp");
    if (!coarsest_connected(h.levels[J], st))
        throw Error(FIEDLER_ERR_DISCONNECTED,
                    "graph is disconnected (lambda_2 = 0): the coarsest level splits into components");
}

}  // namespace fdl

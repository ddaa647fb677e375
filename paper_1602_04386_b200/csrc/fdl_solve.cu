// fdl_solve.cu -- Steps 2-3 of Algorithm 3 and the final
// Rayleigh quotient, as tile-pass kernels over the two solve layouts.
//
// One tile-pass kernel serves the three HBM-bound sweeps of the path:
//   OP_GS  multicolour Gauss-Seidel on L x = 0 (Algorithm 2 line 87 with
//          b = 0: x_i = sum_j w_ij x_j / d_i, in place, one colour per launch),
//          over the GS layout (rows sorted by colour);
//   OP_PI  one step of power iteration on c I - L with deflation (R5, R8):
//          z_i = [c (y_i - mu) + sum_j w_ij (y_j - y_i)] / sigma, where (mu, sigma)
//          are the mean / deflated norm of y from the previous pass (lazy
//          deflate + normalise: the whole step is ONE pass over the level);
//   OP_RQ  Rayleigh quotient of v = s (z - mu) / sigma with the edge form
//          sum_ij w_ij (z_i - z_j)^2 (R7), ||L v||, and v written in natural order.
//   PI and RQ work on the level's natural CSR with vectors in natural
//   numbering (coalesced own/output streams, L2-local gathers); GS works on
//   the GS layout (rows sorted by colour) in GS numbering, and its result is
//   permuted to natural numbering once per level.
// d_i = sum_j w_ij is recomputed on the fly from the streamed weights (no
// degree array is read).  Every pass produces its reductions with a
// deterministic two-level tree (per-CTA partials, last CTA folds them in
// fixed order), so results are bit-reproducible run to run.
//
// Data movement: persistent CTAs walk their tiles (fdl_internal.h) with a
// two-stage pipeline: while a tile is computed, one thread has already issued
// the bulk copies (cp.async.bulk, TMA engine, L2 evict-first hint) of the next
// tile's column and weight streams into the other shared-memory stage, tracked
// by an mbarrier with a transaction count.  Rows with <= 32 nonzeros are
// reduced by one thread from shared memory; longer rows by a warp (or, for a
// row longer than a tile, the whole CTA) straight from global memory.
#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstring>

#include <cooperative_groups.h>

#include "fdl_internal.h"

namespace fdl {
namespace cg = cooperative_groups;

enum { OP_GS = 0, OP_PI = 1, OP_RQ = 2 };
// solve-path kernels are programmatic dependent launches (pdl_wait, launch_pdl)
#ifndef FDL_PDL
#define FDL_PDL 1
#endif
#ifndef FDL_PASS_THREADS
#define FDL_PASS_THREADS 128
#endif
constexpr int kPassThreads = FDL_PASS_THREADS;
constexpr int kPassWarps = kPassThreads / 32;
// entries per row gathered together (x 2 rows in flight) and CTAs per SM, per
// pass kind (tuned with tools/build_variants.py: the GS passes, with no own
// value and a sparse colour sub-range, prefer a deeper chunk)
#ifndef FDL_PI_CHUNK
#define FDL_PI_CHUNK 4
#endif
#ifndef FDL_GS4_MINB
#define FDL_GS4_MINB 7
#endif
#ifndef FDL_PI_MINB
#define FDL_PI_MINB 8
#endif
#ifndef FDL_PI_MINB_SMALL
#define FDL_PI_MINB_SMALL 7
#endif
#ifndef FDL_PI_BIG_ROWS
#define FDL_PI_BIG_ROWS (48 << 20)
#endif
#ifndef FDL_RQ_MINB
#define FDL_RQ_MINB 7
#endif
#ifndef FDL_GS4_MAXDEG
#define FDL_GS4_MAXDEG 8.0
#endif
template <int OP, int CH> struct PassTune {
    static constexpr int chunk = CH ? CH : (OP == 0 ? 8 : FDL_PI_CHUNK);
    // the chunk-4 GS pass (levels of <= 8 entries per row) keeps 7 CTAs per SM
    // (72 registers): measured on the 8192^2 grid, level-0 sweep 1.23 ms with
    // 8 CTAs, 1.15 / 1.05 / 1.01 ms with 5 / 6 / 7; levels 1-4 gain 2-10 % over
    // the chunk-8 pass; the power step prefers 8 CTAs (tools/gpu_levels_variants.sh)
    // the power step: 8 CTAs per SM on the largest levels, 7 below (M != 0);
    // the Rayleigh pass 7 (measured: 0.94 -> 0.86 ms on the 8192^2 grid's level 0)
    static constexpr int min_blocks = (OP == 0 && chunk == 4) ? FDL_GS4_MINB
                                      : (OP == 1 && chunk == 4) ? FDL_PI_MINB
                                      : (OP == 2 && chunk == 4) ? FDL_RQ_MINB
                                      : ((chunk == 4 && OP != 2) ? 4 : 3) * FDL_PASS_MINB / 4;
};
constexpr int kNumStats = 3;
constexpr int kCiBuf = kStageCap + 8;   // + start alignment (<= 3) + 16-byte round-up (<= 3)
constexpr int kWBuf = kStageCap + 4;    // + start alignment (<= 1) + round-up (<= 1)

struct __align__(16) StageBuf {
    double w[kWBuf];
    int ci[kCiBuf];
};
struct __align__(16) PassSmem {
    StageBuf st[kStages];
    unsigned long long bar[kStages];
};
static_assert(sizeof(double) * kWBuf % 16 == 0 && sizeof(int) * kCiBuf % 16 == 0, "stage alignment");

struct CsrView {
    int n;
    const int *rp;
    const int *ci;
    const double *w;
};

struct PassArgs {
    const double *x;        // input (GS: in/out)
    double *y;              // output (PI)
    const double *in_stat;  // slot of the input vector: [2]=mu, [3]=sigma
    double *out_stat;       // slot receiving S, Q, mu, sigma
    int stat_mode;          // bit0: first contribution (assign), bit1: last (finalise), bit2: wanted,
                            // bit3: sums shifted by the slot's previous mean (see finish_stats)
    int n;                  // level size (mean)
    double shift;           // c
    double *partials;       // [grid][kNumStats]
    unsigned *counter;
    double *vnat;           // RQ: output vector, natural order
    const double *sign;     // RQ: +-1
    double *result;         // RQ: {lambda2, residual, ||v||}, or the raw sums if rq_raw
    int rq_raw;             // RQ: write the raw partial sums (partitioned solve)
    // rows longer than a tile ("hubs", power-law levels): reduced in pieces of
    // kTileT entries by the piece tiles {row, -(1 + piece)} of the pass, partial
    // sums in hub_part[tile], folded in piece order by the last CTA
    const int4 *hubs;       // {row, first piece tile (pass-relative), pieces, 0}; null: no piece tiles
    int nhub;
    double2 *hub_part;
};

// ----------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ unsigned long long evict_first_policy() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// bulk copy global -> shared (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar, unsigned long long pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ unsigned round16(unsigned b) { return (b + 15u) & ~15u; }

// ----------------------------------------------------------------- per-row math
template <int OP> struct RowAcc {
    double a = 0.0, b = 0.0;  // GS: (sum w x, sum w); PI: (sum w (x_j - y_i), -); RQ: (sum w d^2, sum w d)
    double own = 0.0;
    __device__ __forceinline__ void add(double wk, double xj) {
        if (OP == OP_GS) { a = fma(wk, xj, a); b += wk; }
        else if (OP == OP_PI) { a = fma(wk, xj - own, a); }
        else { double d = own - xj; a = fma(wk * d, d, a); b = fma(wk, d, b); }
    }
    __device__ __forceinline__ void merge(const RowAcc &o) { a += o.a; b += o.b; }
    __device__ __forceinline__ void warp_sum() {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            if (OP != OP_PI) b += __shfl_xor_sync(0xffffffffu, b, o);
        }
    }
};

struct Scal {
    double mu, inv_sigma, sigma, sign;
};

// own value of row r (PI / RQ)
template <int OP>
__device__ __forceinline__ double own_of(int r, const PassArgs &a) {
    return OP == OP_GS ? 0.0 : a.x[r];
}

// row epilogue: write result, accumulate statistics st[0..2]
template <int OP>
__device__ __forceinline__ void row_finish(int r, const RowAcc<OP> &acc, const PassArgs &a,
                                           const Scal &sc, double st[kNumStats]) {
    if (OP == OP_GS) {
        double xn = acc.a / acc.b;
        const_cast<double *>(a.x)[r] = xn;
        const double xs = xn - sc.mu;   // shift K (finish_stats), 0 without bit 3
        st[0] += xs;
        st[1] = fma(xs, xs, st[1]);
    } else if (OP == OP_PI) {
        double z = (a.shift * (acc.own - sc.mu) + acc.a) * sc.inv_sigma;
        a.y[r] = z;
        st[0] += z;
        st[1] = fma(z, z, st[1]);
    } else {
        double zc = acc.own - sc.mu;
        a.vnat[r] = sc.sign * zc * sc.inv_sigma;
        double lv = acc.b * sc.inv_sigma;
        st[0] += acc.a;
        st[1] = fma(zc, zc, st[1]);
        st[2] = fma(lv, lv, st[2]);
    }
}

// ----------------------------------------------------------------- reductions
template <int N>
__device__ __forceinline__ void block_sum(double v[N], double (*sm)[N]) {
#pragma unroll
    for (int k = 0; k < N; k++)
#pragma unroll
        for (int o = 16; o; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    const int w = threadIdx.x >> 5;
    if (lane_id() == 0)
#pragma unroll
        for (int k = 0; k < N; k++) sm[w][k] = v[k];
    __syncthreads();
    if (threadIdx.x < 32) {
#pragma unroll
        for (int k = 0; k < N; k++) {
            double t = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x][k] : 0.0;
#pragma unroll
            for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            v[k] = t;
        }
    }
    __syncthreads();
}

// Per-CTA partials -> last CTA folds all partials in a fixed order and runs
// `fin(total)` on thread 0.  Deterministic for a fixed grid.
struct NoHubs {
    __device__ void operator()(double *) const {}
};
template <class Fin>
__device__ __forceinline__ void grid_reduce(double st[kNumStats], double *partials, unsigned *counter, Fin fin);
// Hub(hs): run by every thread of the last CTA before the totals; its
// statistics hs are block-summed and added to them (fixed order)
template <class Hub, class Fin>
__device__ __forceinline__ void grid_reduce(double st[kNumStats], double *partials,
                                            unsigned *counter, Hub hub, Fin fin) {
    __shared__ double sm[32][kNumStats];
    __shared__ bool s_last;
    block_sum<kNumStats>(st, sm);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < kNumStats; k++) partials[blockIdx.x * kNumStats + k] = st[k];
        __threadfence();
        unsigned t = atomicAdd(counter, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double hs[kNumStats] = {0.0, 0.0, 0.0};
    hub(hs);
    double v[kNumStats] = {0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
        for (int k = 0; k < kNumStats; k++) v[k] += __ldcg(&partials[b * kNumStats + k]);
    block_sum<kNumStats>(v, sm);
    if (!std::is_same<Hub, NoHubs>::value) {
        block_sum<kNumStats>(hs, sm);
#pragma unroll
        for (int k = 0; k < kNumStats; k++) v[k] += hs[k];
    }
    if (threadIdx.x == 0) {
        fin(v);
        *counter = 0u;
    }
}
template <class Fin>
__device__ __forceinline__ void grid_reduce(double st[kNumStats], double *partials, unsigned *counter, Fin fin) {
    grid_reduce(st, partials, counter, NoHubs{}, fin);
}

// slot = {S, Q, mean, deflated norm}.  With bit 3 of mode the sums are of
// x - K, K = slot[2] on entry (the Gauss-Seidel passes shift by the mean of
// their input, which their output stays close to): then Q - S^2/n does not
// cancel even when |mean| >> the deflated norm.  Without it K = 0 (the
// power-step / prolongation / random outputs have means ~ 0 or ~ the norm).
__device__ __forceinline__ void finish_stats(const double tot[kNumStats], double *slot, int mode,
                                             int n) {
    if (mode & 1) { slot[0] = tot[0]; slot[1] = tot[1]; }
    else { slot[0] += tot[0]; slot[1] += tot[1]; }
    if (mode & 2) {
        const double K = (mode & 8) ? slot[2] : 0.0;
        const double m = slot[0] / (double)n;          // mean of x - K
        const double var = slot[1] - slot[0] * m;      // sum (x - mean)^2
        slot[2] = K + m;
        slot[3] = sqrt(fmax(var, 0.0));
    }
}

// programmatic dependent launch (launch_pdl): wait for the previous kernel on
// the stream -- its writes visible -- before reading what it produced
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ----------------------------------------------------------------- the tile pass
// x gathers: through the read-only path, or L2-coherent (__ldcg) when x is
// rewritten inside the same launch (the fused GS sweep)
template <bool COHERENT>
__device__ __forceinline__ double ldx(const double *p) {
    return COHERENT ? __ldcg(p) : __ldg(p);
}

// entries kb, kb + step, ... < ke of a row (global memory) into acc, in that
// order, 8 per thread with their loads and gathers in flight together
template <int OP, bool COHERENT>
__device__ __forceinline__ void acc_range(RowAcc<OP> &acc, const CsrView &L, const double *x, int kb, int ke,
                                          int step) {
    for (int k0 = kb; k0 < ke; k0 += 8 * step) {
        int c8[8];
        double w8[8], x8[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int k = k0 + i * step;
            c8[i] = k < ke ? __ldcs(L.ci + k) : -1;
            w8[i] = k < ke ? __ldcs(L.w + k) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 8; i++) x8[i] = c8[i] >= 0 ? ldx<COHERENT>(x + c8[i]) : 0.0;
#pragma unroll
        for (int i = 0; i < 8; i++)
            if (c8[i] >= 0) acc.add(w8[i], x8[i]);
    }
}

// entries kb, kb + 32, ... < ke of a row from the stage (sci / sw indexed by
// the global entry number), 8 per lane with their gathers in flight
template <int OP, bool COHERENT>
__device__ __forceinline__ void acc_smem(RowAcc<OP> &acc, const int *__restrict__ sci,
                                         const double *__restrict__ sw, const double *x, int kb, int ke) {
    for (int k0 = kb; k0 < ke; k0 += 8 * 32) {
        int c8[8];
        double w8[8], x8[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int k = k0 + i * 32;
            c8[i] = k < ke ? sci[k] : -1;
            w8[i] = k < ke ? sw[k] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 8; i++) x8[i] = c8[i] >= 0 ? ldx<COHERENT>(x + c8[i]) : 0.0;
#pragma unroll
        for (int i = 0; i < 8; i++)
            if (c8[i] >= 0) acc.add(w8[i], x8[i]);
    }
}

// one thread stages the column/weight streams of tile t into stage b
// first entry / entry count of a tile (a piece tile: its kTileT-entry slice of the row)
__device__ __forceinline__ int2 tile_entries(const CsrView &L, Tile t) {
    if (t.y < 0) {
        const int e0 = L.rp[t.x] + (-t.y - 1) * kTileT;
        return make_int2(e0, min(kTileT, L.rp[t.x + 1] - e0));
    }
    const int e0 = L.rp[t.x];
    return make_int2(e0, min(L.rp[t.y] - e0, kStageCap));
}
__device__ __forceinline__ void issue_tile(PassSmem &S, const CsrView &L, Tile t, int b,
                                           unsigned long long pol) {
    const int2 te = tile_entries(L, t);
    const int e0 = te.x, cnt = te.y;
    if (cnt > 0) {
        const int a4 = e0 & ~3, a2 = e0 & ~1;
        const unsigned bci = round16((unsigned)(e0 + cnt - a4) * 4u);
        const unsigned bw = round16((unsigned)(e0 + cnt - a2) * 8u);
        mbar_arrive_expect_tx(&S.bar[b], bci + bw);
        bulk_g2s(S.st[b].ci, L.ci + a4, bci, &S.bar[b], pol);
        bulk_g2s(S.st[b].w, L.w + a2, bw, &S.bar[b], pol);
    } else {
        mbar_arrive_expect_tx(&S.bar[b], 0u);
    }
}

// Short rows (<= kShortMax) of a tile with few rows: a sub-warp of W lanes per
// row, lane l taking entries l, l + W, ... from shared memory (all its gathers
// in flight), then a shuffle reduction; returns whether the tile has long rows.
template <int OP, int W, bool COHERENT>
__device__ __forceinline__ int subwarp_rows(const Tile t, const int *__restrict__ sci,
                                            const double *__restrict__ sw, const CsrView &L,
                                            const PassArgs &a, const Scal &sc, double st[kNumStats]) {
    const int sl = threadIdx.x & (W - 1);
    const double *__restrict__ x = a.x;
    int has_long = 0;
    for (int r = t.x + (int)threadIdx.x / W; r - (int)(threadIdx.x & 31) / W < t.y;
         r += kPassThreads / W) {
        // (loop bound per warp: all lanes of a warp iterate together for the shuffles)
        const bool live = r < t.y;
        int kb = 0, ke = 0;
        if (live) { kb = L.rp[r]; ke = L.rp[r + 1]; }
        const bool sh = live && ke - kb <= kShortMax;
        if (live && !sh) has_long = 1;
        RowAcc<OP> acc;
        if (OP != OP_GS && sh) acc.own = own_of<OP>(r, a);
        const int n = sh ? ke - kb : 0;
        for (int j0 = 0; j0 < n; j0 += 4 * W) {   // 4 entries per lane per step
            int c[4];
            double wv[4], xv[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int j = j0 + sl + i * W;
                c[i] = j < n ? sci[kb + j] : 0;
                wv[i] = j < n ? sw[kb + j] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 4; i++) xv[i] = (j0 + sl + i * W < n) ? ldx<COHERENT>(x + c[i]) : 0.0;
#pragma unroll
            for (int i = 0; i < 4; i++)
                if (j0 + sl + i * W < n) acc.add(wv[i], xv[i]);
        }
#pragma unroll
        for (int o = W / 2; o; o >>= 1) {
            acc.a += __shfl_xor_sync(0xffffffffu, acc.a, o, W);
            if (OP != OP_PI) acc.b += __shfl_xor_sync(0xffffffffu, acc.b, o, W);
        }
        if (sh && sl == 0) row_finish<OP>(r, acc, a, sc, st);
    }
    return has_long;
}

// Reduce the rows of tile t, whose streams land in stage b (mbarrier phase `phase`).
// Rows <= 32 nonzeros: thread per row from shared memory, two rows per thread with
// their gathers in flight together; longer rows: a warp each (round robin over the
// warps) from global memory; a row longer than a tile (necessarily the tile's last)
// gets the whole CTA.  Ends with a __syncthreads (stage b may then be refilled).
template <int OP, int CH, bool COHERENT, int SW, bool HUB>
__device__ __forceinline__ void tile_compute(const Tile t, int ti, PassSmem &S, int b, unsigned phase,
                                             RowAcc<OP> *s_red, const CsrView &L, const PassArgs &a,
                                             const Scal &sc, double st[kNumStats]) {
    const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const double *__restrict__ x = a.x;
    if (HUB && t.y < 0) {
        // a piece of a hub row: its kTileT entries from shared memory, 8 per
        // thread in flight; the CTA's partial sums go to hub_part[ti]
        const int2 te = tile_entries(L, t);
        const int *__restrict__ sci = S.st[b].ci - (te.x & ~3);
        const double *__restrict__ sw = S.st[b].w - (te.x & ~1);
        RowAcc<OP> acc;
        if (OP != OP_GS) acc.own = own_of<OP>(t.x, a);
        mbar_wait(&S.bar[b], phase);
        const int ke = te.x + te.y;
        for (int k0 = te.x + tid; k0 < ke; k0 += 8 * kPassThreads) {
            int c8[8];
            double w8[8], x8[8];
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const int k = k0 + i * kPassThreads;
                c8[i] = k < ke ? sci[k] : -1;
                w8[i] = k < ke ? sw[k] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 8; i++) x8[i] = c8[i] >= 0 ? ldx<COHERENT>(x + c8[i]) : 0.0;
#pragma unroll
            for (int i = 0; i < 8; i++)
                if (c8[i] >= 0) acc.add(w8[i], x8[i]);
        }
        acc.warp_sum();
        if (lane == 0) s_red[warp] = acc;
        __syncthreads();
        if (tid == 0) {
            RowAcc<OP> tot = s_red[0];
            for (int k = 1; k < kPassWarps; k++) tot.merge(s_red[k]);
            a.hub_part[ti] = make_double2(tot.a, tot.b);
        }
        __syncthreads();   // stage b and s_red may be reused
        return;
    }
    const int e0 = L.rp[t.x];
    const int a4 = e0 & ~3, a2 = e0 & ~1;
    const int *__restrict__ sci = S.st[b].ci - a4;   // index with the global entry number
    const double *__restrict__ sw = S.st[b].w - a2;
    int r0 = t.x + tid;
    int b0 = 0, e0r = 0, b1 = 0, e1r = 0;
    double own0 = 0.0, own1 = 0.0;
    auto fetch = [&](int rr0) {
        const int rr1 = rr0 + kPassThreads;
        b0 = e0r = b1 = e1r = 0;
        if (rr0 < t.y) {
            b0 = L.rp[rr0];
            e0r = L.rp[rr0 + 1];
            if (OP != OP_GS) own0 = own_of<OP>(rr0, a);
        }
        if (rr1 < t.y) {
            b1 = L.rp[rr1];
            e1r = L.rp[rr1 + 1];
            if (OP != OP_GS) own1 = own_of<OP>(rr1, a);
        }
    };
    int has_long = 0;
    if constexpr (SW > 0) {
        // dense level: a sub-warp of SW lanes per short row instead
        mbar_wait(&S.bar[b], phase);
        has_long = subwarp_rows<OP, SW, COHERENT>(t, sci, sw, L, a, sc, st);
        r0 = t.y;   // the pair loop below has nothing left
    } else {
        fetch(r0);   // the first pair's offsets / own values are in flight during the wait
        mbar_wait(&S.bar[b], phase);
    }
    for (; r0 < t.y; r0 += 2 * kPassThreads) {
        if (r0 != t.x + tid) fetch(r0);
        const int r1 = r0 + kPassThreads;
        const bool v1 = r1 < t.y;
        const bool s0 = e0r - b0 <= kShortMax;
        const bool s1 = v1 && e1r - b1 <= kShortMax;
        if (!s0 || (v1 && !s1)) has_long = 1;
        RowAcc<OP> acc0, acc1;
        acc0.own = own0;
        acc1.own = own1;
        const int n0 = s0 ? e0r - b0 : 0, n1 = s1 ? e1r - b1 : 0;
        const int len = max(n0, n1);
        // kChunk entries of each row per step, all their gathers in flight together;
        // each row still accumulates in its sequential entry order
        constexpr int kChunk = PassTune<OP, CH>::chunk;
        for (int j = 0; j < len; j += kChunk) {
            int c0[kChunk], c1[kChunk];
            double w0[kChunk], w1[kChunk], x0[kChunk], x1[kChunk];
#pragma unroll
            for (int i = 0; i < kChunk; i++) {
                const bool ok0 = j + i < n0, ok1 = j + i < n1;
                c0[i] = ok0 ? sci[b0 + j + i] : 0;
                w0[i] = ok0 ? sw[b0 + j + i] : 0.0;
                c1[i] = ok1 ? sci[b1 + j + i] : 0;
                w1[i] = ok1 ? sw[b1 + j + i] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < kChunk; i++) {
                x0[i] = (j + i < n0) ? ldx<COHERENT>(x + c0[i]) : 0.0;
                x1[i] = (j + i < n1) ? ldx<COHERENT>(x + c1[i]) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < kChunk; i++) {
                if (j + i < n0) acc0.add(w0[i], x0[i]);
                if (j + i < n1) acc1.add(w1[i], x1[i]);
            }
        }
        if (s0) row_finish<OP>(r0, acc0, a, sc, st);
        if (s1) row_finish<OP>(r1, acc1, a, sc, st);
    }
    if (__syncthreads_or(has_long)) {
        const int last = t.y - 1;
        // a row longer than a tile: the whole CTA, or its piece tiles (a.hubs)
        const int eT = L.rp[t.y];
        const bool cta_last = eT - L.rp[last] > kTileT;
        const int se = min(eT, e0 + kStageCap);   // end of the staged entries
        // warp w takes the tile's rows in blocks of 32 (w, w + kPassWarps, ...):
        // one coalesced load of their offsets, then each long row in turn, its
        // entries from the stage when they were staged (else global memory)
        for (int rb = t.x + warp * 32; rb < t.y; rb += kPassWarps * 32) {
            const int row = rb + lane;
            int kb = 0, ke = 0;
            if (row < t.y) { kb = L.rp[row]; ke = L.rp[row + 1]; }
            unsigned m = __ballot_sync(0xffffffffu, row < t.y && ke - kb > kShortMax && !(cta_last && row == last));
            while (m) {
                const int l = __ffs(m) - 1;
                m &= m - 1;
                const int r = rb + l, rkb = __shfl_sync(0xffffffffu, kb, l), rke = __shfl_sync(0xffffffffu, ke, l);
                RowAcc<OP> acc;
                if (OP != OP_GS) acc.own = own_of<OP>(r, a);
                if (rke <= se) acc_smem<OP, COHERENT>(acc, sci, sw, x, rkb + lane, rke);
                else acc_range<OP, COHERENT>(acc, L, x, rkb + lane, rke, 32);
                acc.warp_sum();
                if (lane == 0) row_finish<OP>(r, acc, a, sc, st);
            }
        }
        if (cta_last && !HUB) {
            const int kb = L.rp[last], ke = L.rp[t.y];
            RowAcc<OP> acc;
            if (OP != OP_GS) acc.own = own_of<OP>(last, a);
            acc_range<OP, COHERENT>(acc, L, x, kb + tid, ke, kPassThreads);
            acc.warp_sum();
            if (lane == 0) s_red[warp] = acc;
            __syncthreads();
            if (tid == 0) {
                RowAcc<OP> tot = s_red[0];
                for (int k = 1; k < kPassWarps; k++) tot.merge(s_red[k]);
                row_finish<OP>(last, tot, a, sc, st);
            }
        }
    }
    __syncthreads();   // stage b may be overwritten by the next copy
}

__device__ __forceinline__ void init_stages(PassSmem &S) {
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < kStages; k++) mbar_init(&S.bar[k], 1);
        fence_mbar_init();
    }
    __syncthreads();
}

template <int OP>
__device__ __forceinline__ Scal load_scal(const PassArgs &a) {
    Scal sc{0.0, 1.0, 1.0, 1.0};
    if (OP == OP_GS && (a.stat_mode & 12) == 12) sc.mu = a.out_stat[2];   // shift of the statistics
    if (OP != OP_GS) {
        sc.mu = a.in_stat[2];
        sc.sigma = a.in_stat[3];
        sc.inv_sigma = 1.0 / sc.sigma;
        if (OP == OP_RQ) sc.sign = *a.sign;
    }
    return sc;
}

template <int OP, int CH = 0, int SW = 0, bool HUB = false, int M = 0>
__global__ void __launch_bounds__(kPassThreads, M ? M : PassTune<OP, CH>::min_blocks) k_tilepass(const Tile *__restrict__ tiles, int ntiles,
                                                           CsrView L, PassArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PassSmem &S = *reinterpret_cast<PassSmem *>(smem_raw);
    __shared__ RowAcc<OP> s_red[kPassWarps];
    init_stages(S);
    double st[kNumStats] = {0.0, 0.0, 0.0};
    unsigned long long pol = 0;
    if (threadIdx.x == 0) pol = evict_first_policy();
    // ring of kStages stages: iteration `it` consumes stage it % kStages and first
    // refills the stage consumed in iteration it-1 with the tile kStages-1 ahead
    if (threadIdx.x == 0)
        for (int k = 0; k < kStages - 1; k++) {
            const int tk = blockIdx.x + k * gridDim.x;
            if (tk < ntiles) issue_tile(S, L, tiles[tk], k, pol);
        }
    // programmatic dependent launch: everything above (mbarriers, the first
    // tile's column / weight streams -- the matrix, never written by the
    // solve) overlaps the previous kernel's tail; the vectors and statistics
    // it wrote are read only after this wait
    pdl_wait();
    const Scal sc = load_scal<OP>(a);
    int it = 0;
    for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, it++) {
        const int b = it % kStages;
        const int ahead = ti + (kStages - 1) * (int)gridDim.x;
        if (threadIdx.x == 0 && ahead < ntiles) {
            fence_proxy_async();   // generic reads of that stage (previous tile) before async writes
            issue_tile(S, L, tiles[ahead], (it + kStages - 1) % kStages, pol);
        }
        tile_compute<OP, CH, false, SW, HUB>(tiles[ti], ti, S, b, (unsigned)(it / kStages) & 1u, s_red, L, a, sc, st);
    }
    if (OP == OP_GS && !(a.stat_mode & 4) && !HUB) return;   // uniform: statistics not wanted
    // the last CTA first completes the hub rows: partial sums of their piece
    // tiles folded in piece order, then the row epilogue (outputs, statistics
    // in a fixed hub -> thread map)
    auto hub_rows = [&](double hs[kNumStats]) {
        if (!HUB) return;
        for (int h = threadIdx.x; h < a.nhub; h += kPassThreads) {
            const int4 hb = a.hubs[h];
            RowAcc<OP> acc;
            if (OP != OP_GS) acc.own = own_of<OP>(hb.x, a);
            for (int k0 = 0; k0 < hb.z; k0 += 8) {   // 8 partials in flight, folded in order
                double2 pp[8];
#pragma unroll
                for (int i = 0; i < 8; i++)
                    pp[i] = k0 + i < hb.z ? __ldcg(a.hub_part + hb.y + k0 + i) : make_double2(0.0, 0.0);
#pragma unroll
                for (int i = 0; i < 8; i++)
                    if (k0 + i < hb.z) { acc.a += pp[i].x; acc.b += pp[i].y; }
            }
            row_finish<OP>(hb.x, acc, a, sc, hs);
        }
    };
    grid_reduce(st, a.partials, a.counter, hub_rows, [&](const double *tot) {
        if (OP == OP_GS && !(a.stat_mode & 4)) return;
        if (OP == OP_RQ && a.rq_raw) {
            a.result[0] = tot[0];
            a.result[1] = tot[1];
            a.result[2] = tot[2];
        } else if (OP == OP_RQ) {
            double lam = 0.5 * tot[0] / tot[1];
            double vn2 = tot[1] * sc.inv_sigma * sc.inv_sigma;   // ||v||^2
            double res2 = tot[2] - lam * lam * vn2;
            a.result[0] = lam;
            a.result[1] = sqrt(fmax(res2, 0.0));
            a.result[2] = sqrt(vn2);
        } else {
            finish_stats(tot, a.out_stat, a.stat_mode, a.n);
        }
    });
}

// ----------------------------------------------------------------- single-CTA kernels
// Small colours and small levels are launch-bound as grid-wide passes: one CTA
// walks them with __syncthreads between the dependent steps instead.
constexpr int kCtaThreads = 1024;
constexpr int kCtaWarps = kCtaThreads / 32;

// block-wide sum of 2 values (all threads get the totals)
__device__ __forceinline__ void cta_sum2(double &a, double &b, double (*sm)[2]) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    const int w = threadIdx.x >> 5;
    if (lane_id() == 0) { sm[w][0] = a; sm[w][1] = b; }
    __syncthreads();
    double ta = 0.0, tb = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); k++) { ta += sm[k][0]; tb += sm[k][1]; }
    a = ta;
    b = tb;
    __syncthreads();
}

// GS colours [c0, c1) of `sweeps` sweeps (GS layout, x in place) by ONE
// thread-block cluster (CLUSTER) or ONE CTA: the many small colours of dense
// levels and the small trailing colours, where a grid-wide launch per colour
// would be launch-bound.  Row r of a colour belongs to CTA (r - a) mod |cluster|; rows
// <= kShortMax entries a thread each, <= kGcLong a warp each, longer the CTA;
// every row keeps 8 loads per thread in flight.  A cluster barrier (release /
// acquire at cluster scope) separates the colours; x is read through L2
// (__ldcg) because other CTAs of the cluster rewrite it.  Statistics of the
// last sweep: one pass over the rows in a fixed order, reduced over the
// cluster in rank order (deterministic).
#ifndef FDL_GC_THREADS
#define FDL_GC_THREADS 512
#endif
constexpr int kGcThreads = FDL_GC_THREADS;
constexpr int kGcWarps = kGcThreads / 32;
constexpr int kGcLong = 2048;
constexpr int kGcMaxCluster = 16;

__device__ __forceinline__ void gc_row_part(const CsrView &L, const double *x, int kb, int ke, int step,
                                            double &num, double &den) {
    for (int k0 = kb; k0 < ke; k0 += 8 * step) {
        int c8[8];
        double w8[8], x8[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int k = k0 + i * step;
            c8[i] = k < ke ? __ldg(L.ci + k) : -1;
            w8[i] = k < ke ? __ldg(L.w + k) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 8; i++) x8[i] = c8[i] >= 0 ? __ldcg(x + c8[i]) : 0.0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            num = fma(w8[i], x8[i], num);
            den += w8[i];
        }
    }
}

template <bool CLUSTER>
__global__ void __launch_bounds__(kGcThreads) k_gs_multi(CsrView L, const int *__restrict__ seg, int c0,
                                                         int c1, int sweeps, double *x, double *slot,
                                                         int stat_mode, int n) {
    pdl_wait();
    const int cr = CLUSTER ? (int)cg::this_cluster().block_rank() : 0;
    const int ncl = CLUSTER ? (int)cg::this_cluster().num_blocks() : 1;
    const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    constexpr int kMedCap = 1024, kLongCap = 64;
    __shared__ double sm[kGcWarps][2];
    __shared__ double s_part[kGcMaxCluster][2];
    __shared__ int s_med[kMedCap], s_long[kLongCap];
    __shared__ int s_nmed, s_nlong;
    double S = 0.0, Q = 0.0;
    auto finish_row = [&](int r, double num, double den, bool) { x[r] = num / den; };
    for (int s = 0; s < sweeps; s++) {
        const bool last = s == sweeps - 1;
        for (int c = c0; c < c1; c++) {
            const int a = seg[c] + cr, b = seg[c + 1];   // this CTA: rows a, a + ncl, ...
            if (tid == 0) { s_nmed = 0; s_nlong = 0; }
            __syncthreads();
            // short rows here; longer ones listed for the warp / CTA passes
            for (int r = a + tid * ncl; r < b; r += kGcThreads * ncl) {
                const int kb = L.rp[r], ke = L.rp[r + 1];
                if (ke - kb > kGcLong) { const int i = atomicAdd(&s_nlong, 1); if (i < kLongCap) s_long[i] = r; continue; }
                if (ke - kb > kShortMax) { const int i = atomicAdd(&s_nmed, 1); if (i < kMedCap) s_med[i] = r; continue; }
                double num = 0.0, den = 0.0;
                gc_row_part(L, x, kb, ke, 1, num, den);
                finish_row(r, num, den, last);
            }
            __syncthreads();
            const int nmed = s_nmed, nlong = s_nlong;
            // warp rows (from the list; a full list: every row of the share rescanned)
            const bool medlist = nmed <= kMedCap;
            for (int i = warp; medlist ? i < nmed : a + i * ncl < b; i += kGcWarps) {
                const int r = medlist ? s_med[i] : a + i * ncl;
                const int kb = L.rp[r], ke = L.rp[r + 1];
                if (ke - kb <= kShortMax || ke - kb > kGcLong) continue;
                double num = 0.0, den = 0.0;
                gc_row_part(L, x, kb + lane, ke, 32, num, den);
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    num += __shfl_xor_sync(0xffffffffu, num, o);
                    den += __shfl_xor_sync(0xffffffffu, den, o);
                }
                if (lane == 0) finish_row(r, num, den, last);
            }
            // CTA rows (uniform loop over the list, or over the share when it overflowed)
            const bool longlist = nlong <= kLongCap;
            for (int i = 0; longlist ? i < nlong : a + i * ncl < b; i++) {
                const int r = longlist ? s_long[i] : a + i * ncl;
                const int kb = L.rp[r], ke = L.rp[r + 1];
                if (ke - kb <= kGcLong) continue;
                double num = 0.0, den = 0.0;
                gc_row_part(L, x, kb + tid, ke, kGcThreads, num, den);
                cta_sum2(num, den, sm);
                if (tid == 0) finish_row(r, num, den, last);
            }
            // colour c complete (cluster- / CTA-wide) before colour c+1 reads it
            if (CLUSTER) cg::this_cluster().sync();
            else __syncthreads();
        }
    }
    if (!(stat_mode & 4)) return;
    // statistics of the rows of these colours, in a fixed row -> thread map (the
    // lists above are filled in atomic order), shifted by K (finish_stats)
    const double K = (stat_mode & 8) ? slot[2] : 0.0;
    for (int r = seg[c0] + cr * kGcThreads + tid; r < seg[c1]; r += ncl * kGcThreads) {
        const double xr = __ldcg(x + r) - K;
        S += xr;
        Q = fma(xr, xr, Q);
    }
    cta_sum2(S, Q, sm);
    if (CLUSTER) {
        if (tid == 0) {
            double *dst = cg::this_cluster().map_shared_rank(&s_part[0][0], 0);
            dst[2 * cr] = S;
            dst[2 * cr + 1] = Q;
        }
        cg::this_cluster().sync();
    } else if (tid == 0) {
        s_part[0][0] = S;
        s_part[0][1] = Q;
    }
    if (cr == 0 && tid == 0) {
        double tot[kNumStats] = {0.0, 0.0, 0.0};
        for (int i = 0; i < ncl; i++) { tot[0] += s_part[i][0]; tot[1] += s_part[i][1]; }
        finish_stats(tot, slot, stat_mode, n);
    }
}

// ----------------------------------------------------------------- piece-list GS (small colours)
// Runs of colours too small for a grid-wide tile pass each (the coarse levels
// of every graph; all the dense coarse levels of a power-law graph, 150-500
// colours per level) are latency-bound: one colour is one dependent step.
// This kernel keeps each step to one barrier and one round trip of gathers:
//  * the colour's rows are cut at setup into PIECES of <= kGdPiece entries
//    (int4 {row, kind, kb, ke}: 32 consecutive short rows, lane per row; one
//    whole row, warp-strided; or one piece of a longer row, warp-strided,
//    combined in the CTA in piece order), and the pieces of every colour into
//    kGdParts parts cut at row boundaries (build_gs_pieces);
//  * a CTA of the cluster owns parts cr * 16/ncl ...; warp w takes pieces
//    P0 + w, P0 + w + 16, ...;
//  * the column / weight streams of a warp's first piece of the NEXT colour
//    are loaded (and, for lane-per-row pieces, the row offsets before them)
//    between the barrier's arrive and its wait: they never depend on x, so
//    after the barrier only the x gathers remain (one round trip);
//  * levels of <= kGdXsmemN vertices keep x in shared memory, replicated in
//    every CTA of the cluster: a new value is stored to every replica through
//    distributed shared memory (and to global memory for the result), so the
//    gathers after the barrier are shared-memory loads.
// The barrier between colours is barrier.cluster.arrive.release /
// wait.acquire (split) for a cluster, __syncthreads for a single CTA.
// Piece kinds (int4.y): >= 0: rows [x, y) one per lane; -1: row x whole;
// -2: continuation piece of row x; <= -3: first of -(y) - 1 pieces of row x.
constexpr int kGdThreads = 512;
constexpr int kGdWarps = kGdThreads / 32;
constexpr int kGdSlotCap = kGdSlotCapHost;   // pieces of one CTA's share of a colour (partial-sum slots)
constexpr int kGdXsmemN = 20480;     // x replicated in shared memory up to this level size
constexpr size_t kGdSmemBase = (size_t)kGdSlotCap * 16;   // then kGdMaxRunColours ranges, then x


struct GdArgs {
    CsrView L;                  // GS layout
    const int4 *pieces;
    const int *parts;           // [ncolors][kGdParts + 1] piece indices
    const int *seg;             // [ncolors + 1] GS row range of every colour
    int c0, c1, sweeps;
    double *x;                  // GS numbering, in place
    double *slot;
    int stat_mode, n;
};

struct GdPiece {
    int4 d;
    int kb, ke;
    int c[8];
    double w[8];
};

// the three dependent steps of a piece's loads, software-pipelined over the
// items (k_gs_pieces): descriptor; row offsets (lane-per-row pieces);
// column / weight streams
__device__ __forceinline__ int4 gd_desc(const int4 *__restrict__ pieces, int pi, int P1) {
    return pi < P1 ? __ldg(pieces + pi) : make_int4(0, 0, 0, 0);   // {0,0,..}: no rows
}
__device__ __forceinline__ int2 gd_offs(const int4 d, const CsrView &L, int lane) {
    if (d.y < 0) return make_int2(d.z + lane, d.w);
    const int r = d.x + lane;
    return r < d.y ? make_int2(__ldg(L.rp + r), __ldg(L.rp + r + 1)) : make_int2(0, 0);
}
__device__ __forceinline__ void gd_data(GdPiece &p, const int4 d, const int2 o, const CsrView &L) {
    p.d = d;
    p.kb = o.x;
    p.ke = o.y;
    const int step = d.y >= 0 ? 1 : 32;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int k = p.kb + i * step;
        p.c[i] = k < p.ke ? __ldg(L.ci + k) : -1;
        p.w[i] = k < p.ke ? __ldg(L.w + k) : 0.0;
    }
}
__device__ __forceinline__ void gd_load(GdPiece &p, const int4 *__restrict__ pieces, int pi, int P1,
                                        const CsrView &L, int lane) {
    const int4 d = gd_desc(pieces, pi, P1);
    gd_data(p, d, gd_offs(d, L, lane), L);
}

template <bool XS>
__device__ __forceinline__ double gd_xv(const double *xg, const double *xs, int j) {
    return XS ? xs[j] : __ldcg(xg + j);
}

// new value v of row r: global x, and every replica of the cluster (XS)
template <bool CLUSTER, bool XS>
__device__ __forceinline__ void gd_store_lane(double *xg, double *xs, int r, double v, int ncl) {
    xg[r] = v;
    if (XS) {
        if (CLUSTER) {
            for (int j = 0; j < ncl; j++) cg::this_cluster().map_shared_rank(xs, j)[r] = v;
        } else {
            xs[r] = v;
        }
    }
}
// the same by a warp whose lanes all hold v: lane j stores replica j
template <bool CLUSTER, bool XS>
__device__ __forceinline__ void gd_store_warp(double *xg, double *xs, int r, double v, int ncl, int lane) {
    if (lane == 0) xg[r] = v;
    if (XS) {
        if (CLUSTER) {
            if (lane < ncl) cg::this_cluster().map_shared_rank(xs, lane)[r] = v;
        } else if (lane == 0) {
            xs[r] = v;
        }
    }
}

// one piece: gathers of the staged entries, then the row epilogue; returns
// 1 if the piece is the first of a split row (combined after the CTA barrier)
template <bool CLUSTER, bool XS>
__device__ __forceinline__ int gd_piece(GdPiece &p, int slot_idx, double2 *slots, const CsrView &L,
                                        double *xg, double *xs, int ncl, int lane) {
    double xv[8];
#pragma unroll
    for (int i = 0; i < 8; i++) xv[i] = p.c[i] >= 0 ? gd_xv<XS>(xg, xs, p.c[i]) : 0.0;
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int i = 0; i < 8; i++)
        if (p.c[i] >= 0) { num = fma(p.w[i], xv[i], num); den += p.w[i]; }
    if (p.d.y >= 0) {
        // lane per row: entries past the first 8 (rows of 9..32 entries)
        for (int k0 = p.kb + 8; k0 < p.ke; k0 += 8) {
            int c[8];
            double w[8], v[8];
#pragma unroll
            for (int i = 0; i < 8; i++) {
                c[i] = k0 + i < p.ke ? __ldg(L.ci + k0 + i) : -1;
                w[i] = k0 + i < p.ke ? __ldg(L.w + k0 + i) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 8; i++) v[i] = c[i] >= 0 ? gd_xv<XS>(xg, xs, c[i]) : 0.0;
#pragma unroll
            for (int i = 0; i < 8; i++)
                if (c[i] >= 0) { num = fma(w[i], v[i], num); den += w[i]; }
        }
        const int r = p.d.x + lane;
        if (r < p.d.y) gd_store_lane<CLUSTER, XS>(xg, xs, r, num / den, ncl);
        return 0;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, o);
        den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    if (p.d.y == -1) {
        gd_store_warp<CLUSTER, XS>(xg, xs, p.d.x, num / den, ncl, lane);
        return 0;
    }
    if (lane == 0) slots[slot_idx] = make_double2(num, den);
    return p.d.y <= -3 ? 1 : 0;
}

__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <bool CLUSTER, bool XS>
__global__ void __launch_bounds__(kGdThreads, 1) k_gs_pieces(GdArgs a) {
    extern __shared__ __align__(16) unsigned char gd_smem[];
    double2 *slots = reinterpret_cast<double2 *>(gd_smem);
    double *xs = reinterpret_cast<double *>(gd_smem + kGdSmemBase + (size_t)kGdMaxRunColours * 8);
    __shared__ double sm[kGdWarps][2];
    __shared__ double s_part[kGcMaxCluster][2];
    const int cr = CLUSTER ? (int)cg::this_cluster().block_rank() : 0;
    const int ncl = CLUSTER ? (int)cg::this_cluster().num_blocks() : 1;
    const int per = kGdParts / ncl;
    const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const CsrView L = a.L;
    double *xg = a.x;
    // this CTA's piece range of every colour of the run, in shared memory
    int2 *rng = reinterpret_cast<int2 *>(gd_smem + kGdSmemBase);
    const int ncol = a.c1 - a.c0;
    for (int c = tid; c < ncol; c += kGdThreads)
        rng[c] = make_int2(__ldg(a.parts + (a.c0 + c) * (kGdParts + 1) + cr * per),
                           __ldg(a.parts + (a.c0 + c) * (kGdParts + 1) + (cr + 1) * per));
    __syncthreads();
    const int items = a.sweeps * ncol;
    auto item_rng = [&](int it) {   // colour of item it (it / ncol <= sweeps: a few subtractions)
        int c = it;
        while (c >= ncol) c -= ncol;
        return it < items ? rng[c] : make_int2(0, 0);
    };
    // pipeline of this warp's first piece (the matrix is never written by the
    // solve): item it+1 fully loaded, it+2 up to its row offsets, it+3 its descriptor
    GdPiece cur;
    int4 d2, d3;
    int2 o2;
    {
        const int2 r0 = item_rng(0), r1 = item_rng(1), r2 = item_rng(2);
        const int4 d0 = gd_desc(a.pieces, r0.x + warp, r0.y);
        d2 = gd_desc(a.pieces, r1.x + warp, r1.y);
        d3 = gd_desc(a.pieces, r2.x + warp, r2.y);
        const int2 o0 = gd_offs(d0, L, lane);
        o2 = gd_offs(d2, L, lane);
        gd_data(cur, d0, o0, L);
    }
    pdl_wait();
    if (XS) {
        for (int i = tid; i < a.n; i += kGdThreads) xs[i] = __ldcg(xg + i);
        if (CLUSTER) cg::this_cluster().sync();   // no replica written before its owner filled it
        else __syncthreads();
    }
    for (int it = 0; it < items; it++) {
        if (it > 0) {
            if (CLUSTER) cluster_wait();
            else __syncthreads();
        }
        const int2 R = item_rng(it);
        const int P0 = R.x, P1 = R.y;
        int has_split = gd_piece<CLUSTER, XS>(cur, warp, slots, L, xg, xs, ncl, lane);
        // the warp's further pieces (a colour's long rows), two at a time with
        // both pieces' loads in flight together (the prefetch registers of
        // `cur` are free until the next colour's loads are issued)
        for (int pi = P0 + warp + kGdWarps; pi < P1; pi += 2 * kGdWarps) {
            const int pj = pi + kGdWarps;
            const int4 d1 = gd_desc(a.pieces, pi, P1), d2b = gd_desc(a.pieces, pj, P1);
            const int2 o1 = gd_offs(d1, L, lane), o2b = gd_offs(d2b, L, lane);
            GdPiece q1, q2;
            gd_data(q1, d1, o1, L);
            gd_data(q2, d2b, o2b, L);
            has_split |= gd_piece<CLUSTER, XS>(q1, pi - P0, slots, L, xg, xs, ncl, lane);
            if (pj < P1) has_split |= gd_piece<CLUSTER, XS>(q2, pj - P0, slots, L, xg, xs, ncl, lane);
        }
        if (__syncthreads_or(has_split)) {
            // rows split into pieces: the warp of the first piece folds the
            // partial sums in piece order
            for (int pi = P0 + warp; pi < P1; pi += kGdWarps) {
                const int4 d = __ldg(a.pieces + pi);
                if (d.y > -3) continue;
                const int np = -d.y - 1;
                double num = 0.0, den = 0.0;
                for (int k = lane; k < np; k += 32) {
                    const double2 sv = slots[pi - P0 + k];
                    num += sv.x;
                    den += sv.y;
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    num += __shfl_xor_sync(0xffffffffu, num, o);
                    den += __shfl_xor_sync(0xffffffffu, den, o);
                }
                gd_store_warp<CLUSTER, XS>(xg, xs, d.x, num / den, ncl, lane);
            }
        }
        if (it + 1 < items) {
            if (CLUSTER) cluster_arrive();
            gd_data(cur, d2, o2, L);
            o2 = gd_offs(d3, L, lane);
            d2 = d3;
            const int2 r3 = item_rng(it + 3);
            d3 = gd_desc(a.pieces, r3.x + warp, r3.y);
        }
    }
    // every replica write done before any CTA reads the statistics or exits
    if (CLUSTER) cg::this_cluster().sync();
    else __syncthreads();
    if (!(a.stat_mode & 4)) return;
    // statistics of the rows of these colours in a fixed row -> thread map,
    // shifted by K (finish_stats), reduced over the cluster in rank order
    const double K = (a.stat_mode & 8) ? a.slot[2] : 0.0;
    double S = 0.0, Q = 0.0;
    const int rb = __ldg(a.seg + a.c0), re = __ldg(a.seg + a.c1);
    for (int r = rb + cr * kGdThreads + tid; r < re; r += ncl * kGdThreads) {
        const double xr = (XS ? xs[r] : __ldcg(xg + r)) - K;
        S += xr;
        Q = fma(xr, xr, Q);
    }
    cta_sum2(S, Q, sm);
    if (CLUSTER) {
        if (tid == 0) {
            double *dst = cg::this_cluster().map_shared_rank(&s_part[0][0], 0);
            dst[2 * cr] = S;
            dst[2 * cr + 1] = Q;
        }
        cg::this_cluster().sync();
    } else if (tid == 0) {
        s_part[0][0] = S;
        s_part[0][1] = Q;
    }
    if (cr == 0 && tid == 0) {
        double tot[kNumStats] = {0.0, 0.0, 0.0};
        for (int i = 0; i < ncl; i++) { tot[0] += s_part[i][0]; tot[1] += s_part[i][1]; }
        finish_stats(tot, a.slot, a.stat_mode, a.n);
    }
}

// ---- setup side: pieces and parts of a level (called by build_layout)
// groups of 32 consecutive rows of one colour; gstart[c] = first group of colour c
__device__ __forceinline__ int div_up_d(int a, int b) { return (a + b - 1) / b; }
__device__ __forceinline__ int gd_group_colour(const int *gstart, int ncolors, int g) {
    int lo = 0, hi = ncolors;   // largest c with gstart[c] <= g
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (gstart[mid] <= g) lo = mid;   // (global or shared memory)
        else hi = mid;
    }
    return lo;
}
__global__ void k_gd_count(const int *rp, const int *seg, const int *gstart, int ncolors, int ngroups,
                           int *gcnt) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += gridDim.x * blockDim.x) {
        const int c = gd_group_colour(gstart, ncolors, g);
        const int r0 = seg[c] + (g - gstart[c]) * kGdGroup, r1 = min(r0 + kGdGroup, seg[c + 1]);
        int cnt = 0, maxlen = 0;
        for (int r = r0; r < r1; r++) {
            const int len = rp[r + 1] - rp[r];
            maxlen = max(maxlen, len);
            cnt += len > kGdPiece ? (len + kGdPiece - 1) / kGdPiece : 1;
        }
        gcnt[g] = maxlen <= kGdShort ? 1 : cnt;
    }
}
// the pieces of the group of rows [r0, r1) from position p
__device__ void gd_write_group(const int *rp, int r0, int r1, int p, int4 *pieces) {
    int maxlen = 0;
    for (int r = r0; r < r1; r++) maxlen = max(maxlen, rp[r + 1] - rp[r]);
    if (maxlen <= kGdShort) {
        pieces[p] = make_int4(r0, r1, rp[r0], rp[r1]);
        return;
    }
    for (int r = r0; r < r1; r++) {
        const int kb = rp[r], ke = rp[r + 1], len = ke - kb;
        if (len <= kGdPiece) {
            pieces[p++] = make_int4(r, -1, kb, ke);
            continue;
        }
        const int np = (len + kGdPiece - 1) / kGdPiece;
        for (int i = 0; i < np; i++)
            pieces[p++] = make_int4(r, i == 0 ? -(np + 1) : -2, kb + i * kGdPiece, min(kb + (i + 1) * kGdPiece, ke));
    }
}
__global__ void k_gd_write(const int *rp, const int *seg, const int *gstart, int ncolors, int ngroups,
                           const int *goff, int4 *pieces) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += gridDim.x * blockDim.x) {
        const int c = gd_group_colour(gstart, ncolors, g);
        const int r0 = seg[c] + (g - gstart[c]) * kGdGroup, r1 = min(r0 + kGdGroup, seg[c + 1]);
        gd_write_group(rp, r0, r1, goff[g], pieces);
    }
}
// parts: kGdParts + 1 piece indices per colour, cut at the first piece of a row
__global__ void k_gd_parts(const int *gstart, const int *goff, const int4 *pieces, int ncolors, int *parts) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ncolors * (kGdParts + 1)) return;
    const int c = t / (kGdParts + 1), k = t % (kGdParts + 1);
    const int p0 = goff[gstart[c]], p1 = goff[gstart[c + 1]];
    int p = p0 + (int)((long long)k * (p1 - p0) / kGdParts);
    while (p < p1 && pieces[p].y == -2) p++;
    parts[t] = p;
}

// The same in ONE launch for small levels (<= kGdSmallGroups groups, <= 1024
// colours): group starts of the used colours, counts, exclusive scans and
// the pieces / parts, in shared memory (the small levels' setup is launch-bound)
constexpr int kGdSmallGroups = 8192;
struct GdUse {
    unsigned bits[32];
};
// in-place exclusive scan of a[0, n) by the whole CTA (blockDim.x == 1024); returns the total
__device__ int cta_exclusive_scan(int *a, int n) {
    __shared__ int s_w[32];
    const int per = (n + 1023) / 1024, t = threadIdx.x, b = t * per, e = min(b + per, n);
    int sum = 0;
    for (int i = b; i < e; i++) sum += a[i];
    int x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if ((t & 31) >= o) x += y;
    }
    if ((t & 31) == 31) s_w[t >> 5] = x;
    __syncthreads();
    if (t < 32) {
        int w = s_w[t];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (t >= o) w += y;
        }
        s_w[t] = w;
    }
    __syncthreads();
    int run = x - sum + ((t >> 5) ? s_w[(t >> 5) - 1] : 0);
    const int total = s_w[31];
    for (int i = b; i < e; i++) {
        const int v = a[i];
        a[i] = run;
        run += v;
    }
    __syncthreads();
    return total;
}
__global__ void __launch_bounds__(1024) k_gd_small(const int *rp, const int *seg, GdUse use, int ncolors,
                                                   int4 *pieces, int *parts) {
    __shared__ int s_gs[1025];
    __shared__ int s_go[kGdSmallGroups + 1];
    const int t = threadIdx.x;
    for (int c = t; c < ncolors; c += 1024)
        s_gs[c] = ((use.bits[c >> 5] >> (c & 31)) & 1u) ? div_up_d(seg[c + 1] - seg[c], kGdGroup) : 0;
    __syncthreads();
    const int ng = cta_exclusive_scan(s_gs, ncolors);
    if (t == 0) s_gs[ncolors] = ng;
    __syncthreads();
    for (int g = t; g < ng; g += 1024) {
        const int c = gd_group_colour(s_gs, ncolors, g);
        const int r0 = seg[c] + (g - s_gs[c]) * kGdGroup, r1 = min(r0 + kGdGroup, seg[c + 1]);
        int cnt = 0, maxlen = 0;
        for (int r = r0; r < r1; r++) {
            const int len = rp[r + 1] - rp[r];
            maxlen = max(maxlen, len);
            cnt += len > kGdPiece ? (len + kGdPiece - 1) / kGdPiece : 1;
        }
        s_go[g] = maxlen <= kGdShort ? 1 : cnt;
    }
    __syncthreads();
    const int np = cta_exclusive_scan(s_go, ng);
    if (t == 0) s_go[ng] = np;
    __syncthreads();
    for (int g = t; g < ng; g += 1024) {
        const int c = gd_group_colour(s_gs, ncolors, g);
        const int r0 = seg[c] + (g - s_gs[c]) * kGdGroup, r1 = min(r0 + kGdGroup, seg[c + 1]);
        gd_write_group(rp, r0, r1, s_go[g], pieces);
    }
    __syncthreads();   // the parts read the pieces' kinds (global writes of this CTA)
    for (int i = t; i < ncolors * (kGdParts + 1); i += 1024) {
        const int c = i / (kGdParts + 1), k = i % (kGdParts + 1);
        const int p0 = s_go[s_gs[c]], p1 = s_go[s_gs[c + 1]];
        int p = p0 + (int)((long long)k * (p1 - p0) / kGdParts);
        while (p < p1 && pieces[p].y == -2) p++;
        parts[i] = p;
    }
}

void build_gs_pieces(Level &L, const std::vector<int> &seg, const std::vector<int> &segnnz,
                     const std::vector<char> &use, cudaStream_t st) {
    const int ncolors = L.ncolors;
    std::vector<int> gstart(ncolors + 1, 0);
    long long bound = 1;
    for (int c = 0; c < ncolors; c++) {
        const int rows = seg[c + 1] - seg[c];
        gstart[c + 1] = gstart[c] + (use[c] ? div_up(rows, kGdGroup) : 0);
        if (use[c]) bound += rows + (segnnz[c + 1] - segnnz[c]) / kGdPiece + 1;   // >= pieces of colour c
    }
    const int ngroups = gstart[ncolors];
    if (ngroups <= kGdSmallGroups && ncolors <= 1024) {
        GdUse u{};
        for (int c = 0; c < ncolors; c++)
            if (use[c]) u.bits[c >> 5] |= 1u << (c & 31);
        L.gd_pieces.alloc((size_t)bound * sizeof(int4), st);
        L.gd_parts.alloc((size_t)ncolors * (kGdParts + 1) * 4, st);
        k_gd_small<<<1, 1024, 0, st>>>(L.rp.as<int>(), L.seg_d.as<int>(), u, ncolors, L.gd_pieces.as<int4>(),
                                       L.gd_parts.as<int>());
        FDL_LAUNCH_CK();
        return;
    }
    DBuf gs_d((size_t)(ncolors + 1) * 4, st);
    upload(st, gs_d.p, gstart.data(), (size_t)(ncolors + 1) * 4);
    DBuf gcnt((size_t)(ngroups + 1) * 4, st), goff((size_t)(ngroups + 1) * 4, st);
    L.gd_pieces.alloc((size_t)bound * sizeof(int4), st);
    if (ngroups > 0) {
        k_gd_count<<<grid_for(ngroups), 256, 0, st>>>(L.rp.as<int>(), L.seg_d.as<int>(), gs_d.as<int>(), ncolors,
                                                       ngroups, gcnt.as<int>());
        FDL_LAUNCH_CK();
    }
    scan_exclusive(gcnt.as<int>(), goff.as<int>(), ngroups, goff.as<int>() + ngroups, st);
    if (ngroups > 0) {
        k_gd_write<<<grid_for(ngroups), 256, 0, st>>>(L.rp.as<int>(), L.seg_d.as<int>(), gs_d.as<int>(), ncolors,
                                                       ngroups, goff.as<int>(), L.gd_pieces.as<int4>());
        FDL_LAUNCH_CK();
    }
    const int np = ncolors * (kGdParts + 1);
    L.gd_parts.alloc((size_t)np * 4, st);
    k_gd_parts<<<grid_for(np), 256, 0, st>>>(gs_d.as<int>(), goff.as<int>(), L.gd_pieces.as<int4>(), ncolors,
                                             L.gd_parts.as<int>());
    FDL_LAUNCH_CK();
}

// `iters` power steps on c I - L of a small level (natural CSR), one CTA:
// z = (c (y - mu) + sum w (y_j - y_i)) / sigma with (mu, sigma) of the previous
// vector, ping-pong between y0 and y1 (the result ends in y0 if iters is even);
// in_slot = (mu, sigma) of y0 on entry, out_slot = statistics of the result.
__global__ void __launch_bounds__(kCtaThreads) k_pi_small(CsrView L, double shift, int iters, double *y0,
                                                          double *y1, const double *in_slot, double *out_slot) {
    pdl_wait();
    __shared__ double sm[kCtaWarps][2];
    __shared__ double s_mu, s_isig;
    const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const int n = L.n;
    if (tid == 0) { s_mu = in_slot[2]; s_isig = 1.0 / in_slot[3]; }
    __syncthreads();
    double *src = y0, *dst = y1;
    double S = 0.0, Q = 0.0;
    for (int it = 0; it < iters; it++) {
        const double mu = s_mu, is = s_isig;
        S = 0.0;
        Q = 0.0;
        int has_long = 0;
        for (int r = tid; r < n; r += kCtaThreads) {
            const int kb = L.rp[r], ke = L.rp[r + 1];
            if (ke - kb > kShortMax) { has_long = 1; continue; }
            const double own = src[r];
            double acc = 0.0;
            for (int k = kb; k < ke; k++) acc = fma(L.w[k], src[L.ci[k]] - own, acc);
            const double z = (shift * (own - mu) + acc) * is;
            dst[r] = z;
            S += z;
            Q = fma(z, z, Q);
        }
        if (__syncthreads_or(has_long)) {
            for (int r = warp; r < n; r += kCtaWarps) {
                const int kb = L.rp[r], ke = L.rp[r + 1];
                if (ke - kb <= kShortMax) continue;
                const double own = src[r];
                double acc = 0.0;
                for (int k = kb + lane; k < ke; k += 32) acc = fma(L.w[k], src[L.ci[k]] - own, acc);
#pragma unroll
                for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (lane == 0) {
                    const double z = (shift * (own - mu) + acc) * is;
                    dst[r] = z;
                    S += z;
                    Q = fma(z, z, Q);
                }
            }
        }
        cta_sum2(S, Q, sm);   // also the barrier before the next step reads dst
        if (tid == 0) {
            const double m = S / (double)n;
            s_mu = m;
            s_isig = 1.0 / sqrt(fmax(Q - (double)n * m * m, 0.0));
        }
        __syncthreads();
        double *t = src; src = dst; dst = t;
    }
    if (tid == 0) {
        const double tot[kNumStats] = {S, Q, 0.0};
        finish_stats(tot, out_slot, 1 | 2, n);
    }
}

// ----------------------------------------------------------------- small kernels
// prolongation y^j = I^T y^{j+1}: y[i] = xc[map[i]], xc in the
// coarse level's natural numbering; map = q (natural output) or q o perm (GS output)
__global__ void __launch_bounds__(256) k_prolong(int n, const int *__restrict__ qp,
                                                 const double *__restrict__ xc, double *__restrict__ y,
                                                 double *slot, double *partials, unsigned *counter,
                                                 double *mean_copy) {
    pdl_wait();
    double st[kNumStats] = {0.0, 0.0, 0.0};
    const int stride = gridDim.x * blockDim.x;
    // 4 entries per thread in flight; statistics still summed in i order per thread
    for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
        int q[4];
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) q[u] = i0 + u * stride < n ? __ldcs(qp + i0 + u * stride) : -1;
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = q[u] >= 0 ? __ldg(xc + q[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (q[u] >= 0) {
                y[i0 + u * stride] = v[u];
                st[0] += v[u];
                st[1] = fma(v[u], v[u], st[1]);
            }
    }
    grid_reduce(st, partials, counter, [&](const double *tot) {
        finish_stats(tot, slot, 3, n);
        if (mean_copy) *mean_copy = slot[2];   // the GS statistics' shift (finish_stats)
    });
}

// rand(n_J) in natural order, counter-based (R6)
__global__ void __launch_bounds__(256) k_rand(int n, uint64_t seed,
                                              double *__restrict__ y, double *slot, double *partials,
                                              unsigned *counter) {
    pdl_wait();
    const uint64_t s0 = splitmix64(seed ^ kTagRand);
    double st[kNumStats] = {0.0, 0.0, 0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = (double)(splitmix64(s0 + (uint64_t)i) >> 11) * 0x1.0p-53;
        y[i] = v;
        st[0] += v;
        st[1] = fma(v, v, st[1]);
    }
    grid_reduce(st, partials, counter, [&](const double *tot) { finish_stats(tot, slot, 3, n); });
}

// sign convention: first nonzero entry (natural order) of v = (z - mu)/sigma positive
__global__ void k_sign(int n, const double *__restrict__ z, const double *slot, double *sign) {
    pdl_wait();
    const double mu = slot[2];
    for (int base = 0; base < n; base += 32) {
        int i = base + lane_id();
        double v = i < n ? z[i] - mu : 0.0;
        unsigned nz = __ballot_sync(0xffffffffu, v != 0.0);
        if (nz) {
            int src = __ffs(nz) - 1;
            double f = __shfl_sync(0xffffffffu, v, src);
            if (lane_id() == 0) *sign = f > 0.0 ? 1.0 : -1.0;
            return;
        }
    }
    if (lane_id() == 0) *sign = 1.0;
}

// GS numbering -> natural numbering: dst[v] = src[inv[v]] (coalesced writes)
__global__ void __launch_bounds__(256) k_gs_to_nat(int n, const int *__restrict__ inv,
                                                   const double *__restrict__ src, double *__restrict__ dst) {
    pdl_wait();
    const int stride = gridDim.x * blockDim.x;
    for (int v0 = blockIdx.x * blockDim.x + threadIdx.x; v0 < n; v0 += 4 * stride) {   // 4 gathers in flight
        int p[4];
        double x[4];
#pragma unroll
        for (int u = 0; u < 4; u++) p[u] = v0 + u * stride < n ? __ldcs(inv + v0 + u * stride) : -1;
#pragma unroll
        for (int u = 0; u < 4; u++) x[u] = p[u] >= 0 ? __ldg(src + p[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (p[u] >= 0) dst[v0 + u * stride] = x[u];
    }
}

__global__ void k_set_slot(double *slot, double mu, double sigma) {
    slot[0] = 0.0; slot[1] = 0.0; slot[2] = mu; slot[3] = sigma;
}

__global__ void k_gather_f64(int n, const int *__restrict__ idx, const double *__restrict__ src,
                             double *__restrict__ dst) {  // dst[i] = src[idx[i]]
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}
__global__ void k_scatter_f64(int n, const int *__restrict__ idx, const double *__restrict__ src,
                              double *__restrict__ dst) {  // dst[idx[i]] = src[i]
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        dst[idx[i]] = src[i];
}
// materialise (z - mu)/sigma in place
__global__ void k_normalise(int n, double *z, const double *slot) {
    const double mu = slot[2], is = 1.0 / slot[3];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        z[i] = (z[i] - mu) * is;
}

// ----------------------------------------------------------------- host-side schedule
constexpr size_t kPassSmemBytes = sizeof(PassSmem);

#ifndef FDL_SMALL_PI_ROWS
#define FDL_SMALL_PI_ROWS 1024
#endif
constexpr int kSmallPiRows = FDL_SMALL_PI_ROWS;   // levels this small run all power steps in one CTA
constexpr int kSmallPiNnz = 1 << 18;  // ... unless dense: one CTA streams ~0.1 TB/s

// CTAs of a pass: resident CTAs per SM x SMs (persistent tile loop), per OP
// one cluster (16 CTAs where the device allows, else 8) for k_gs_multi<true>
static void launch_gs_cluster(cudaStream_t st, CsrView v, const int *seg, int c0, int c1, int sweeps, double *x,
                              double *slot, int mode, int n) {
    static DeviceCache cl_cache{};
    std::atomic<int> &cl_slot = cl_cache[current_device()];
    int cl = cl_slot.load();
    if (!cl) {
        cl = 8;
        if (cudaFuncSetAttribute(k_gs_multi<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3(kGcMaxCluster);
            q.blockDim = dim3(kGcThreads);
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = kGcMaxCluster;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, k_gs_multi<true>, &q) == cudaSuccess && nclusters > 0)
                cl = kGcMaxCluster;
        }
        (void)cudaGetLastError();
        cl_slot.store(cl);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(kGcThreads);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = FDL_PDL;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    FDL_CK(cudaLaunchKernelEx(&cfg, k_gs_multi<true>, v, seg, c0, c1, sweeps, x, slot, mode, n));
}

// k_gs_pieces: a cluster of 16 CTAs where the device allows (else 8), or one CTA
template <bool CLUSTER, bool XS>
static int gd_prepare() {
    static DeviceCache cache{};
    std::atomic<int> &slot = cache[current_device()];
    int cl = slot.load();
    if (cl) return cl;
    const int smem = (int)(kGdSmemBase + (size_t)kGdMaxRunColours * 8 + (XS ? (size_t)kGdXsmemN * 8 : 0));
    FDL_CK(cudaFuncSetAttribute(k_gs_pieces<CLUSTER, XS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cl = 1;
    if (CLUSTER) {
        cl = 8;
        if (cudaFuncSetAttribute(k_gs_pieces<CLUSTER, XS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
            cudaSuccess) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3(kGcMaxCluster);
            q.blockDim = dim3(kGdThreads);
            q.dynamicSmemBytes = smem;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = kGcMaxCluster;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, k_gs_pieces<CLUSTER, XS>, &q) == cudaSuccess &&
                nclusters > 0)
                cl = kGcMaxCluster;
        }
        (void)cudaGetLastError();
    }
    slot.store(cl);
    return cl;
}

template <bool CLUSTER, bool XS>
static void launch_gs_pieces_t(cudaStream_t st, const GdArgs &a) {
    const int cl = gd_prepare<CLUSTER, XS>();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(kGdThreads);
    cfg.dynamicSmemBytes = kGdSmemBase + (size_t)kGdMaxRunColours * 8 + (XS ? (size_t)a.n * 8 : 0);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na++].val.programmaticStreamSerializationAllowed = FDL_PDL;
    if (CLUSTER) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = cl;
        at[na].val.clusterDim.y = 1;
        at[na++].val.clusterDim.z = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    FDL_CK(cudaLaunchKernelEx(&cfg, k_gs_pieces<CLUSTER, XS>, a));
    FDL_LAUNCH_CK();
}

static void launch_gs_pieces(cudaStream_t st, const Level &L, int c0, int c1, int sweeps, double *x, double *slot,
                             int mode, bool cluster) {
    GdArgs a{};
    a.L = CsrView{L.n, L.rp.as<int>(), L.ci.as<int>(), L.w.as<double>()};
    a.pieces = L.gd_pieces.as<int4>();
    a.parts = L.gd_parts.as<int>();
    a.seg = L.seg_d.as<int>();
    a.c0 = c0;
    a.c1 = c1;
    a.sweeps = sweeps;
    a.x = x;
    a.slot = slot;
    a.stat_mode = mode;
    a.n = L.n;
    const bool xs = L.n <= kGdXsmemN;
    if (cluster) {
        if (xs) launch_gs_pieces_t<true, true>(st, a);
        else launch_gs_pieces_t<true, false>(st, a);
    } else {
        if (xs) launch_gs_pieces_t<false, true>(st, a);
        else launch_gs_pieces_t<false, false>(st, a);
    }
}

#ifndef FDL_DENSE_ROW_DEG
#define FDL_DENSE_ROW_DEG 7.0
#endif
constexpr double kDenseRowDeg = FDL_DENSE_ROW_DEG;   // rows per tile few enough for sub-warp rows
static DeviceCache g_pass_grid[5] = {};   // per OP (3: the GS chunk-4 variant, 4: the power step below FDL_PI_BIG_ROWS), per device
static int pass_grid(int op) { return g_pass_grid[op][current_device()].load(); }

// A tile pass as a programmatic dependent launch (FDL_PDL): its CTAs may start
// while the previous kernel on the stream drains, up to griddepcontrol.wait
template <class K>
static void launch_pass(K kernel, int grid, cudaStream_t st, const Tile *tiles, int nt, CsrView v, PassArgs a) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kPassThreads);
    cfg.dynamicSmemBytes = kPassSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = FDL_PDL;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FDL_CK(cudaLaunchKernelEx(&cfg, kernel, tiles, nt, v, a));
    FDL_LAUNCH_CK();
}

// any solve-path kernel as a programmatic dependent launch
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = FDL_PDL;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FDL_CK(cudaLaunchKernelEx(&cfg, kernel, args...));
    FDL_LAUNCH_CK();
}

struct Enq {
    Handle &h;
    cudaStream_t st;
    int launches = 0;
    double *slot(int k) { return h.scal.as<double>() + 4 * k; }

    // OP over the tiles [tiles, tiles + nt) of level L (GS: GS layout; PI/RQ: natural layout)
    template <int OP>
    void pass_tiles(const Level &L, const Tile *tiles, int nt, PassArgs a) {
        if (nt <= 0) return;
        int grid = std::min(nt, pass_grid(OP));
        a.partials = h.partials.as<double>();
        a.counter = h.counter.as<unsigned>();
        CsrView v = OP == OP_GS ? CsrView{L.n, L.rp.as<int>(), L.ci.as<int>(), L.w.as<double>()}
                                : CsrView{L.n, L.rpN.as<int>(), L.ciN.as<int>(), L.wN.as<double>()};
        // GS: the chunk of 4 suits <= 4.5 neighbours per row, 8 the denser coarse
        // levels; dense levels (>= kDenseRowDeg per row): 4 lanes per short row
        if (a.hubs) {   // piece tiles of hub rows in the range (power-law levels)
            if (L.nnz >= kDenseRowDeg * (double)L.n) launch_pass(k_tilepass<OP, 0, 4, true>, grid, st, tiles, nt, v, a);
            else launch_pass(k_tilepass<OP, 0, 0, true>, grid, st, tiles, nt, v, a);
        } else if (OP == OP_GS && L.nnz <= FDL_GS4_MAXDEG * L.n) {
            grid = std::min(nt, pass_grid(3));
            launch_pass(k_tilepass<OP_GS, 4>, grid, st, tiles, nt, v, a);
        } else if (L.nnz >= kDenseRowDeg * (double)L.n) {
            launch_pass(k_tilepass<OP, 0, 4>, grid, st, tiles, nt, v, a);
        } else if (OP == OP_PI && L.n < FDL_PI_BIG_ROWS) {
            grid = std::min(nt, pass_grid(4));
            launch_pass(k_tilepass<OP_PI, 0, 0, false, FDL_PI_MINB_SMALL>, grid, st, tiles, nt, v, a);
        } else {
            launch_pass(k_tilepass<OP>, grid, st, tiles, nt, v, a);
        }
        launches++;
    }
    // hp: the pass whose hub rows have piece tiles in [tb, te) (colour c, or
    // ncolors for the natural-order pass)
    template <int OP>
    void pass(const Level &L, int tb, int te, PassArgs a, int hp) {
        if (!L.hoff.empty() && L.hoff[hp + 1] > L.hoff[hp]) {
            a.hubs = L.hubs.as<int4>() + L.hoff[hp];
            a.nhub = L.hoff[hp + 1] - L.hoff[hp];
            a.hub_part = L.hub_part.as<double2>();
        }
        pass_tiles<OP>(L, L.tiles.as<Tile>() + tb, te - tb, a);
    }
    // One sweep = the level's GS schedule (L.gs_runs): grid-wide tile passes for
    // big colours, one cluster launch per run of small colours, one single-CTA
    // launch for the small trailing colours; a level that is one run does all
    // its sweeps in one launch.  Statistics of the last sweep go to out_slot.
    void gs_run(const Level &L, int cb, int ce, int kind, double *x, int sweeps, double *out_slot, int mode) {
        CsrView v{L.n, L.rp.as<int>(), L.ci.as<int>(), L.w.as<double>()};
        if (kind == 0) {
            PassArgs a{};
            a.x = x;
            a.n = L.n;
            a.out_stat = out_slot;
            a.stat_mode = mode;
            pass<OP_GS>(L, L.ctile[cb], L.ctile[cb + 1], a, cb);
        } else if (kind >= 3) {
            launch_gs_pieces(st, L, cb, ce, sweeps, x, out_slot, mode, kind == 3);
            launches++;
        } else if (kind == 1) {
            launch_gs_cluster(st, v, L.seg_d.as<int>(), cb, ce, sweeps, x, out_slot, mode, L.n);
            launches++;
        } else {
            launch_pdl(k_gs_multi<false>, dim3(1), dim3(kGcThreads), st, v, (const int *)L.seg_d.as<int>(), cb, ce,
                       sweeps, x, out_slot, mode, (int)L.n);
            launches++;
        }
    }
    void gs(const Level &L, double *x, int sweeps, double *out_slot) {
        if (sweeps <= 0) return;
        const int nr = (int)L.gs_runs.size() / 3;
        const int *R = L.gs_runs.data();
        // statistics shifted by the input's mean, slot[2] of out_slot (bit 3)
        if (nr == 1 && R[2] != 0) {
            gs_run(L, R[0], R[1], R[2], x, sweeps, out_slot, out_slot ? (8 | 4 | 1 | 2) : 0);
            return;
        }
        for (int s = 0; s < sweeps; s++) {
            const bool want = (s == sweeps - 1) && out_slot;
            for (int i = 0; i < nr; i++) {
                const int mode = want ? (8 | 4 | (i == 0 ? 1 : 0) | (i == nr - 1 ? 2 : 0)) : 0;
                gs_run(L, R[3 * i], R[3 * i + 1], R[3 * i + 2], x, 1, out_slot, mode);
            }
        }
    }
    // `iters` power steps from (cur, cur_slot); returns the buffer / slot of the result
    void pi_iters(const Level &L, double *&cur, double *&oth, double *&cur_slot, int iters,
                  double *(*next_slot)(void *), void *ctx) {
        if (iters <= 0) return;
        if (L.n <= kSmallPiRows && L.nnz <= kSmallPiNnz) {
            double *ns = next_slot(ctx);
            CsrView v{L.n, L.rpN.as<int>(), L.ciN.as<int>(), L.wN.as<double>()};
            launch_pdl(k_pi_small, dim3(1), dim3(kCtaThreads), st, v, (double)L.shift, iters, cur, oth,
                       (const double *)cur_slot, ns);
            launches++;
            if (iters & 1) std::swap(cur, oth);
            cur_slot = ns;
            return;
        }
        for (int k = 0; k < iters; k++) {
            double *ns = next_slot(ctx);
            pi(L, cur, oth, cur_slot, ns);
            std::swap(cur, oth);
            cur_slot = ns;
        }
    }
    void pi(const Level &L, const double *x, double *y, const double *in_slot, double *out_slot) {
        PassArgs a{};
        a.x = x;
        a.y = y;
        a.in_stat = in_slot;
        a.out_stat = out_slot;
        a.stat_mode = 7;
        a.n = L.n;
        a.shift = L.shift;
        pass<OP_PI>(L, L.nat_tile_begin(), L.ntiles, a, L.ncolors);
    }
    void rq(const Level &L, const double *x, const double *in_slot, double *vnat, const double *sign) {
        PassArgs a{};
        a.x = x;
        a.in_stat = in_slot;
        a.n = L.n;
        a.vnat = vnat;
        a.sign = sign;
        a.result = h.result.as<double>();
        pass<OP_RQ>(L, L.nat_tile_begin(), L.ntiles, a, L.ncolors);
    }
    void prolong(const Level &L, const int *map, const double *xc, double *y, double *out_slot,
                 double *mean_copy = nullptr) {
        launch_pdl(k_prolong, dim3(grid_for(L.n, 256, h.row_grid)), dim3(256), st, (int)L.n, map, xc, y, out_slot,
                   h.partials.as<double>(), h.counter.as<unsigned>(), mean_copy);
        launches++;
    }
    void to_nat(const Level &L, const double *xg, double *xn) {
        launch_pdl(k_gs_to_nat, dim3(grid_for(L.n, 256, h.row_grid)), dim3(256), st, (int)L.n,
                   (const int *)L.inv.as<int>(), xg, xn);
        launches++;
    }
};

// returns true when it allocated (on h.stream)
static bool ensure_solve_buffers(Handle &h, int nslots) {
    cudaStream_t st = h.stream;
    bool grew = false;
    if (!h.xa.p) {
        grew = true;
        h.xa.alloc((size_t)h.n0 * 8, st);
        h.xb.alloc((size_t)h.n0 * 8, st);
        h.vnat.alloc((size_t)h.n0 * 8, st);
        h.partials.alloc((size_t)h.row_grid * kNumStats * 8, st);
        h.counter.alloc(64, st);
        FDL_CK(cudaMemsetAsync(h.counter.p, 0, 64, st));
        h.result.alloc(8 * 8, st);
    }
    if (h.nslots < nslots) {
        if (h.gexec) { cudaGraphExecDestroy(h.gexec); h.gexec = nullptr; }   // it captured the old slots
        h.scal.alloc((size_t)nslots * 4 * 8, st);
        FDL_CK(cudaMemsetAsync(h.scal.p, 0, (size_t)nslots * 4 * 8, st));
        h.nslots = nslots;
        grew = true;
    }
    return grew;
}

static int slots_needed(const Handle &h, const SolveCfg &cfg) {
    const int J = (int)h.levels.size() - 1;
    // 1 (rand) + piJ + per level (1 prolong + 1 gs + pi) + sign, and >= 8 for level ops
    return std::max(8, 2 + cfg.piJ + J * (2 + cfg.pi) + 2);
}

// allocate everything the solve needs (never inside a graph capture)
int prepare_solve(Handle &h, const SolveCfg &cfg) {
    ensure_solve_buffers(h, slots_needed(h, cfg));
    return 0;
}

// returns the largest pass grid (sizes the partial-sum buffer)
int rowpass_grid() {
    static DeviceCache cache{};
    const int cdev = current_device();
    if (int c = cache[cdev].load()) return c;
    const int smem = (int)kPassSmemBytes;
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_GS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_PI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_RQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_GS, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_GS, 0, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_PI, 0, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_RQ, 0, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_GS, 0, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_PI, 0, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_RQ, 0, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_GS, 0, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_PI, 0, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_RQ, 0, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));

    FDL_CK(cudaFuncSetAttribute(k_tilepass<OP_PI, 0, 0, false, FDL_PI_MINB_SMALL>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int b3 = 0, b4 = 0;
    FDL_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b3, k_tilepass<OP_GS, 4>, kPassThreads, smem));
    FDL_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b4, k_tilepass<OP_PI, 0, 0, false, FDL_PI_MINB_SMALL>,
                                                         kPassThreads, smem));
    int b0 = 0, b1 = 0, b2 = 0;
    FDL_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b0, k_tilepass<OP_GS>, kPassThreads, smem));
    FDL_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k_tilepass<OP_PI>, kPassThreads, smem));
    FDL_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_tilepass<OP_RQ>, kPassThreads, smem));
    int dev = 0, sms = kNumSMs;
    FDL_CK(cudaGetDevice(&dev));
    FDL_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    g_pass_grid[OP_GS][cdev].store(sms * std::max(1, b0));
    g_pass_grid[OP_PI][cdev].store(sms * std::max(1, b1));
    g_pass_grid[OP_RQ][cdev].store(sms * std::max(1, b2));
    g_pass_grid[3][cdev].store(sms * std::max(1, b3));
    g_pass_grid[4][cdev].store(sms * std::max(1, b4));
    const int all = sms * std::max(std::max(std::max(1, b3), b4), std::max(b0, std::max(b1, b2)));
    cache[cdev].store(all);
    return all;
}

int enqueue_solve(Handle &h, const SolveCfg &cfg) {
    const int J = (int)h.levels.size() - 1;
    const int nslots = slots_needed(h, cfg);
    FDL_REQUIRE(h.nslots >= nslots && h.xa.p, FIEDLER_ERR_INTERNAL, "solve buffers not prepared");
    Enq e{h, h.stream};
    int sl = 0;
    double *xa = h.xa.as<double>(), *xb = h.xb.as<double>();
    // ---- coarsest level: rand(n_J), deflate + normalise (lazily), power iteration
    const Level &LJ = h.levels[J];
    double *cur_slot = e.slot(sl++);
    launch_pdl(k_rand, dim3(grid_for(LJ.n, 256, h.row_grid)), dim3(256), h.stream, (int)LJ.n, (uint64_t)cfg.seed, xa,
               cur_slot, h.partials.as<double>(), h.counter.as<unsigned>());
    e.launches++;
    double *cur = xa, *oth = xb;
    struct SlotCtx { Enq *e; int *sl; } sctx{&e, &sl};
    auto next_slot = [](void *p) -> double * {
        SlotCtx *c = static_cast<SlotCtx *>(p);
        return c->e->slot((*c->sl)++);
    };
    e.pi_iters(LJ, cur, oth, cur_slot, cfg.piJ, next_slot, &sctx);
    // ---- cascadic refinement
    for (int ell = J - 1; ell >= 0; ell--) {
        const Level &L = h.levels[ell];
        double *ps = e.slot(sl++);
        if (cfg.gs > 0) {
            // prolong straight into GS numbering, sweep, return to natural numbering
            // (the GS statistics are shifted by the mean of the GS input: the
            // prolongation copies it into the GS slot, finish_stats)
            double *gsl = e.slot(sl++);
            e.prolong(L, L.qg.as<int>(), cur, oth, ps, gsl + 2);
            std::swap(cur, oth);
            e.gs(L, cur, cfg.gs, gsl);
            e.to_nat(L, cur, oth);
            std::swap(cur, oth);
            cur_slot = gsl;
        } else {
            e.prolong(L, L.q_nat.as<int>(), cur, oth, ps);
            std::swap(cur, oth);
            cur_slot = ps;
        }
        e.pi_iters(L, cur, oth, cur_slot, cfg.pi, next_slot, &sctx);
    }
    // ---- Rayleigh quotient on level 0 (+ vector in natural order)
    const Level &L0 = h.levels[0];
    double *sgn = e.slot(sl++);
    launch_pdl(k_sign, dim3(1), dim3(32), h.stream, (int)L0.n, (const double *)cur, (const double *)cur_slot, sgn);
    e.launches++;
    e.rq(L0, cur, cur_slot, h.vnat.as<double>(), sgn);
    FDL_REQUIRE(sl <= nslots, FIEDLER_ERR_INTERNAL, "slot overflow");
    return e.launches;
}

// ----------------------------------------------------------------- fiedler_level_apply
void apply_level_op(Handle &h, int level, int op, int count, const double *x_in, double *x_out,
                    double *scal_host) {
    const Level &L = h.levels[level];
    cudaStream_t st = h.stream;
    ensure_solve_buffers(h, 8);
    Enq e{h, st};
    double *xa = h.xa.as<double>(), *xb = h.xb.as<double>();
    double *s0 = e.slot(0), *s1 = e.slot(1);
    double res[4] = {0, 0, 0, 0};
    if (op == FIEDLER_OP_PROLONG) {
        const Level &C = h.levels[level + 1];
        FDL_CK(cudaMemcpyAsync(xa, x_in, (size_t)C.n * 8, cudaMemcpyDeviceToDevice, st));
        e.prolong(L, L.q_nat.as<int>(), xa, x_out, s0);
        FDL_CK(cudaMemcpyAsync(res, s0, 32, cudaMemcpyDeviceToHost, st));
        FDL_CK(cudaStreamSynchronize(st));
        if (scal_host) { scal_host[0] = res[2]; scal_host[1] = res[3]; }
    } else {
        if (op == FIEDLER_OP_GS_SWEEPS) {   // natural -> GS numbering
            k_gather_f64<<<grid_for(L.n), 256, 0, st>>>(L.n, L.perm.as<int>(), x_in, xa);
            FDL_LAUNCH_CK();
        } else {
            FDL_CK(cudaMemcpyAsync(xa, x_in, (size_t)L.n * 8, cudaMemcpyDeviceToDevice, st));
        }
        if (op == FIEDLER_OP_GS_SWEEPS) {
            // statistics shifted by K = the first input entry (finish_stats): any
            // value near the data keeps Q - S^2/n free of cancellation
            FDL_CK(cudaMemsetAsync(s0, 0, 32, st));
            FDL_CK(cudaMemcpyAsync(s0 + 2, xa, 8, cudaMemcpyDeviceToDevice, st));
            e.gs(L, xa, count, s0);
            k_scatter_f64<<<grid_for(L.n), 256, 0, st>>>(L.n, L.perm.as<int>(), xa, x_out);
            FDL_LAUNCH_CK();
            FDL_CK(cudaMemcpyAsync(res, s0, 32, cudaMemcpyDeviceToHost, st));
            FDL_CK(cudaStreamSynchronize(st));
            if (scal_host) { scal_host[0] = res[2]; scal_host[1] = res[3]; }
        } else if (op == FIEDLER_OP_POWER) {
            k_set_slot<<<1, 1, 0, st>>>(s0, 0.0, 1.0);
            FDL_LAUNCH_CK();
            double *cur = xa, *oth = xb, *cs = s0, *ns = s1;
            for (int k = 0; k < count; k++) {
                e.pi(L, cur, oth, cs, ns);
                std::swap(cur, oth);
                std::swap(cs, ns);
            }
            if (count > 0) {
                k_normalise<<<grid_for(L.n), 256, 0, st>>>(L.n, cur, cs);
                FDL_LAUNCH_CK();
            }
            FDL_CK(cudaMemcpyAsync(x_out, cur, (size_t)L.n * 8, cudaMemcpyDeviceToDevice, st));
            FDL_CK(cudaMemcpyAsync(res, cs, 32, cudaMemcpyDeviceToHost, st));
            FDL_CK(cudaStreamSynchronize(st));
            if (scal_host) { scal_host[0] = res[2]; scal_host[1] = res[3]; }
        } else if (op == FIEDLER_OP_RAYLEIGH) {
            k_set_slot<<<1, 1, 0, st>>>(s0, 0.0, 1.0);
            FDL_LAUNCH_CK();
            k_set_slot<<<1, 1, 0, st>>>(s1, 1.0, 1.0);   // sign = +1 at s1[2]
            FDL_LAUNCH_CK();
            e.rq(L, xa, s0, xb, s1 + 2);                 // xb: natural-order scratch
            FDL_CK(cudaMemcpyAsync(res, h.result.p, 24, cudaMemcpyDeviceToHost, st));
            FDL_CK(cudaStreamSynchronize(st));
            if (scal_host) { scal_host[0] = res[0]; scal_host[1] = res[1]; }
        } else {
            throw Error(FIEDLER_ERR_ARG, "unknown op");
        }
    }
    FDL_CK(cudaStreamSynchronize(st));
}

// ----------------------------------------------------------------- fiedler_level_time
void time_level_op(Handle &h, int level, int op, int reps, double *ms_per_rep, double *bytes_per_rep) {
    const Level &L = h.levels[level];
    cudaStream_t st = h.stream;
    ensure_solve_buffers(h, 8);
    Enq e{h, st};
    double *xa = h.xa.as<double>(), *xb = h.xb.as<double>();
    double *s0 = e.slot(0), *s1 = e.slot(1);
    // finite, non-constant input: the counter-based uniform vector
    k_rand<<<grid_for(L.n, 256, h.row_grid), 256, 0, st>>>(L.n, 7, xa, s0,
                                                           h.partials.as<double>(), h.counter.as<unsigned>());
    FDL_LAUNCH_CK();
    k_set_slot<<<1, 1, 0, st>>>(s1, 1.0, 1.0);
    FDL_LAUNCH_CK();
    auto one = [&]() {
        if (op == FIEDLER_OP_GS_SWEEPS) e.gs(L, xa, 1, nullptr);
        else if (op == FIEDLER_OP_POWER) e.pi(L, xa, xb, s0, e.slot(2));
        else e.rq(L, xa, s0, h.vnat.as<double>(), s1 + 2);
    };
    one();  // warm-up
    cudaEvent_t a, b;
    FDL_CK(cudaEventCreate(&a));
    FDL_CK(cudaEventCreate(&b));
    FDL_CK(cudaEventRecord(a, st));
    for (int r = 0; r < reps; r++) one();
    FDL_CK(cudaEventRecord(b, st));
    FDL_CK(cudaEventSynchronize(b));
    float ms = 0.f;
    FDL_CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *ms_per_rep = ms / reps;
    if (bytes_per_rep) {
        // algorithmic bytes of one pass: row offsets, columns
        // and weights once, the input vector once, the output vector once
        double n = L.n, nnz = L.nnz;
        *bytes_per_rep = 4.0 * (n + 1) + 12.0 * nnz + 8.0 * n + 8.0 * n;
    }
}

}  // namespace fdl

// =================================================================== partitioned solve
// fiedler_dist_plan / fiedler_dist_op (include/fiedler.h).
namespace fdl {

__device__ __forceinline__ int lower_bound_coord_d(const int *rp, int lo, int hi, long long target) {
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if ((long long)rp[mid] + mid < target) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// bounds[k] = first natural row whose coordinate rp[r] + r reaches k (n + nnz) / nranks
__global__ void k_dist_bounds(const int *rp, int n, int nranks, int *bounds) {
    const int k = threadIdx.x;
    if (k > nranks) return;
    const long long total = (long long)rp[n] + n;
    bounds[k] = k == 0 ? 0 : (k == nranks ? n : lower_bound_coord_d(rp, 0, n, total * k / nranks));
}

// own GS rows of colour c: [lower_bound(perm_c, r0), lower_bound(perm_c, r1)) inside the
// colour's segment (natural ids ascend within a colour)
// own GS row range [a, b) of every colour (rows of a colour are sorted by
// natural id) and the row offsets at its ends: ab[4c..4c+3] = {a, b, rp[a], rp[b]}
__global__ void k_dist_colour_ranges(const int *perm, const int *seg, const int *rp, int ncol, int r0, int r1,
                                     int *ab) {
    for (int c = threadIdx.x; c < ncol; c += blockDim.x) {
        for (int side = 0; side < 2; side++) {
            int lo = seg[c], hi = seg[c + 1];
            const int target = side ? r1 : r0;
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (perm[mid] < target) lo = mid + 1; else hi = mid;
            }
            ab[4 * c + side] = lo;
            ab[4 * c + 2 + side] = rp[lo];
        }
    }
}

__global__ void k_make_tiles_d(const int *rp, int s0, int s1, int ntiles, Tile *out) {
    const long long C0 = (long long)rp[s0] + s0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x) {
        int a = t == 0 ? s0 : lower_bound_coord_d(rp, s0, s1, C0 + (long long)t * kTileT);
        int b = (t + 1 == ntiles) ? s1 : lower_bound_coord_d(rp, s0, s1, C0 + (long long)(t + 1) * kTileT);
        out[t] = make_int2(a, b);
    }
}

__device__ __forceinline__ int owner_of(int u, const int *bounds, int nranks) {
    int p = 0;
    while (p + 1 < nranks && u >= bounds[p + 1]) p++;
    return p;
}

// ghosts: neighbours of own rows outside [r0, r1); peer masks of own rows
__global__ void k_dist_mark(const int *rp, const int *ci, int r0, int r1, const int *bounds, int nranks,
                            int rank, int *ghost_flag, unsigned long long *peer_mask) {
    for (int v = r0 + blockIdx.x * blockDim.x + threadIdx.x; v < r1; v += gridDim.x * blockDim.x) {
        unsigned long long m = 0ull;
        for (int k = rp[v]; k < rp[v + 1]; k++) {
            const int u = ci[k];
            if (u < r0 || u >= r1) {
                ghost_flag[u] = 1;
                m |= 1ull << owner_of(u, bounds, nranks);
            }
        }
        peer_mask[v - r0] = m & ~(1ull << rank);
    }
}

__global__ void k_mask_bit(const unsigned long long *mask, int cnt, int p, int *flag) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
        flag[i] = (int)((mask[i] >> p) & 1ull);
}

__global__ void k_add_offset(int *a, int cnt, int off) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) a[i] += off;
}

// number of sorted list entries below each bound
__global__ void k_count_below(const int *list, const int *cnt, const int *bounds, int nb, int *pos) {
    const int k = threadIdx.x;
    if (k >= nb) return;
    int lo = 0, hi = *cnt;
    const int target = bounds[k];
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (list[mid] < target) lo = mid + 1; else hi = mid;
    }
    pos[k] = lo;
}

static int read_i(const int *d, cudaStream_t st) {
    int h;
    FDL_CK(cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaStreamSynchronize(st));
    return h;
}

void dist_plan(Handle &h, int level, int nranks, int rank, fiedler_dist_plan_info *info) {
    Level &L = h.levels[level];
    cudaStream_t st = h.stream;
    DistPlan &P = L.dist;
    P = DistPlan();
    P.nranks = nranks;
    P.rank = rank;
    const int n = L.n;
    DBuf db((size_t)(nranks + 1) * 4, st);
    k_dist_bounds<<<1, 128, 0, st>>>(L.rpN.as<int>(), n, nranks, db.as<int>());
    FDL_LAUNCH_CK();
    std::vector<int> b(nranks + 1);
    FDL_CK(cudaMemcpyAsync(b.data(), db.p, (size_t)(nranks + 1) * 4, cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaStreamSynchronize(st));
    P.bounds.assign(b.begin(), b.end());
    P.r0 = b[rank];
    P.r1 = b[rank + 1];
    // own natural tiles
    int rr[2];
    FDL_CK(cudaMemcpyAsync(&rr[0], L.rpN.as<int>() + P.r0, 4, cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaMemcpyAsync(&rr[1], L.rpN.as<int>() + P.r1, 4, cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaStreamSynchronize(st));
    const long long spanN = (long long)(rr[1] + P.r1) - (rr[0] + P.r0);
    P.ntN = P.r1 > P.r0 ? (int)((spanN + kTileT - 1) / kTileT) : 0;
    P.tilesN.alloc((size_t)std::max(P.ntN, 1) * sizeof(Tile), st);
    if (P.ntN) {
        k_make_tiles_d<<<grid_for(P.ntN), 256, 0, st>>>(L.rpN.as<int>(), P.r0, P.r1, P.ntN, P.tilesN.as<Tile>());
        FDL_LAUNCH_CK();
    }
    // own GS tiles per colour
    const int nc = L.ncolors;
    DBuf dseg((size_t)(nc + 1) * 4, st), dab((size_t)4 * nc * 4, st);
    FDL_CK(cudaMemcpyAsync(dseg.p, L.seg.data(), (size_t)(nc + 1) * 4, cudaMemcpyHostToDevice, st));
    k_dist_colour_ranges<<<1, 256, 0, st>>>(L.perm.as<int>(), dseg.as<int>(), L.rp.as<int>(), nc, P.r0, P.r1,
                                            dab.as<int>());
    FDL_LAUNCH_CK();
    std::vector<int> ab(4 * nc);
    FDL_CK(cudaMemcpyAsync(ab.data(), dab.p, (size_t)4 * nc * 4, cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaStreamSynchronize(st));
    std::vector<int> cnt(nc, 0);
    P.ctile.assign(nc + 1, 0);
    int nt = 0;
    for (int c = 0; c < nc; c++) {
        P.ctile[c] = nt;
        const int a0 = ab[4 * c], a1 = ab[4 * c + 1];
        if (a1 > a0) {
            const long long span = (long long)(ab[4 * c + 3] + a1) - (ab[4 * c + 2] + a0);
            cnt[c] = (int)((span + kTileT - 1) / kTileT);
            if (cnt[c] < 1) cnt[c] = 1;
        }
        nt += cnt[c];
    }
    P.ctile[nc] = nt;
    P.tilesGS.alloc((size_t)std::max(nt, 1) * sizeof(Tile), st);
    for (int c = 0; c < nc; c++)
        if (cnt[c]) {
            k_make_tiles_d<<<grid_for(cnt[c]), 256, 0, st>>>(L.rp.as<int>(), ab[4 * c], ab[4 * c + 1], cnt[c],
                                                             P.tilesGS.as<Tile>() + P.ctile[c]);
            FDL_LAUNCH_CK();
        }
    // halo plan
    P.send_cnt.assign(nranks, 0);
    P.recv_cnt.assign(nranks, 0);
    if (nranks > 1) {
        const int own = P.r1 - P.r0;
        DBuf gflag((size_t)std::max(n, 1) * 4, st), mask((size_t)std::max(own, 1) * 8, st),
            glist((size_t)std::max(n, 1) * 4, st), gcnt(8, st), pos((size_t)(nranks + 1) * 4, st);
        FDL_CK(cudaMemsetAsync(gflag.p, 0, (size_t)n * 4, st));
        if (own > 0) {
            k_dist_mark<<<grid_for(own), 256, 0, st>>>(L.rpN.as<int>(), L.ciN.as<int>(), P.r0, P.r1, db.as<int>(),
                                                       nranks, rank, gflag.as<int>(), mask.as<unsigned long long>());
            FDL_LAUNCH_CK();
        }
        compact_flagged(nullptr, gflag.as<int>(), n, glist.as<int>(), gcnt.as<int>(), st);
        k_count_below<<<1, 128, 0, st>>>(glist.as<int>(), gcnt.as<int>(), db.as<int>(), nranks + 1, pos.as<int>());
        FDL_LAUNCH_CK();
        std::vector<int> hp(nranks + 1);
        FDL_CK(cudaMemcpyAsync(hp.data(), pos.p, (size_t)(nranks + 1) * 4, cudaMemcpyDeviceToHost, st));
        FDL_CK(cudaStreamSynchronize(st));
        P.recv_total = hp[nranks] - hp[0];
        for (int p = 0; p < nranks; p++) P.recv_cnt[p] = hp[p + 1] - hp[p];
        P.recv_idx.alloc((size_t)std::max(P.recv_total, 1) * 4, st);
        if (P.recv_total)
            FDL_CK(cudaMemcpyAsync(P.recv_idx.p, glist.as<int>() + hp[0], (size_t)P.recv_total * 4,
                                   cudaMemcpyDeviceToDevice, st));
        // send lists, peer-major
        std::vector<DBuf> parts;
        std::vector<int> pc(nranks, 0);
        DBuf flag((size_t)std::max(own, 1) * 4, st);
        for (int p = 0; p < nranks; p++) {
            if (p == rank || own == 0) continue;
            parts.emplace_back((size_t)own * 4, st);
            DBuf &part = parts.back();
            k_mask_bit<<<grid_for(own), 256, 0, st>>>(mask.as<unsigned long long>(), own, p, flag.as<int>());
            FDL_LAUNCH_CK();
            compact_flagged(nullptr, flag.as<int>(), own, part.as<int>(), gcnt.as<int>() + 1, st);
            pc[p] = read_i(gcnt.as<int>() + 1, st);
            if (pc[p]) {
                k_add_offset<<<grid_for(pc[p]), 256, 0, st>>>(part.as<int>(), pc[p], P.r0);
                FDL_LAUNCH_CK();
            }
        }
        P.send_total = 0;
        for (int p = 0; p < nranks; p++) { P.send_cnt[p] = pc[p]; P.send_total += pc[p]; }
        P.send_idx.alloc((size_t)std::max(P.send_total, 1) * 4, st);
        int off = 0, k = 0;
        for (int p = 0; p < nranks; p++) {
            if (p == rank || own == 0) continue;
            if (pc[p])
                FDL_CK(cudaMemcpyAsync(P.send_idx.as<int>() + off, parts[k].p, (size_t)pc[p] * 4,
                                       cudaMemcpyDeviceToDevice, st));
            off += pc[p];
            k++;
        }
    }
    FDL_CK(cudaStreamSynchronize(st));
    P.valid = true;
    if (info) {
        std::memset(info, 0, sizeof(*info));
        info->n = n;
        info->nranks = nranks;
        info->rank = rank;
        info->colors = nc;
        info->row_begin = P.r0;
        info->row_end = P.r1;
        for (int p = 0; p <= nranks; p++) info->row_bounds[p] = P.bounds[p];
        for (int p = 0; p < nranks; p++) {
            info->send_count[p] = P.send_cnt[p];
            info->recv_count[p] = P.recv_cnt[p];
        }
        info->send_total = P.send_total;
        info->recv_total = P.recv_total;
    }
}

// ---- op kernels
// y = I^T x on own rows [r0, r1) and on the ghost rows; natural row v goes to
// y[v] (natural) or y[inv[v]] (GS); partial (S, Q) over the own rows
__global__ void __launch_bounds__(256) k_dist_prolong(int r0, int r1, const int *__restrict__ ghosts, int ng,
                                                      const int *__restrict__ q, const int *__restrict__ inv,
                                                      const double *__restrict__ xc, double *__restrict__ y,
                                                      double *slot, double *partials, unsigned *counter) {
    double st[kNumStats] = {0.0, 0.0, 0.0};
    const int own = r1 - r0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < own + ng; i += gridDim.x * blockDim.x) {
        const int v = i < own ? r0 + i : ghosts[i - own];
        const double val = __ldg(xc + q[v]);
        y[inv ? inv[v] : v] = val;
        if (i < own) {
            st[0] += val;
            st[1] = fma(val, val, st[1]);
        }
    }
    grid_reduce(st, partials, counter, [&](const double *tot) { finish_stats(tot, slot, 1, 1); });
}

// y[v] = x[inv[v]] on own rows; partial (S, Q)
__global__ void __launch_bounds__(256) k_dist_to_nat(int r0, int r1, const int *__restrict__ inv,
                                                     const double *__restrict__ x, double *__restrict__ y,
                                                     double *slot, double *partials, unsigned *counter) {
    double st[kNumStats] = {0.0, 0.0, 0.0};
    for (int v = r0 + blockIdx.x * blockDim.x + threadIdx.x; v < r1; v += gridDim.x * blockDim.x) {
        const double val = __ldg(x + inv[v]);
        y[v] = val;
        st[0] += val;
        st[1] = fma(val, val, st[1]);
    }
    grid_reduce(st, partials, counter, [&](const double *tot) { finish_stats(tot, slot, 1, 1); });
}

__global__ void k_dist_finalise(double *slot, int n) {
    const double tot[kNumStats] = {slot[0], slot[1], 0.0};
    finish_stats(tot, slot, 1 | 2, n);
}

__global__ void k_dist_finalise_rq(double *slot, const double *xs) {
    const double is = 1.0 / xs[3];
    const double lam = 0.5 * slot[0] / slot[1];
    const double vn2 = slot[1] * is * is;
    const double res2 = slot[2] - lam * lam * vn2;
    slot[0] = lam;
    slot[1] = sqrt(fmax(res2, 0.0));
    slot[2] = sqrt(vn2);
}

// first own row with x - mean != 0: key = 2 i + (negative)
__global__ void k_dist_first_nonzero(int r0, int r1, const double *__restrict__ x, const double *xs,
                                     double *out) {
    const double mu = xs[2];
    double key = 1152921504606846976.0;   // 2^60
    for (int base = r0; base < r1; base += 32) {
        const int i = base + lane_id();
        const double v = i < r1 ? x[i] - mu : 0.0;
        const unsigned nz = __ballot_sync(0xffffffffu, v != 0.0);
        if (nz) {
            const int src = __ffs(nz) - 1;
            const double f = __shfl_sync(0xffffffffu, v, src);
            key = 2.0 * (double)(base + src) + (f < 0.0 ? 1.0 : 0.0);
            break;
        }
    }
    if (lane_id() == 0) out[0] = key;
}

__global__ void k_dist_sign(double *slot) {
    const double key = slot[0];
    slot[2] = (key < 1152921504606846976.0 && fmod(key, 2.0) == 1.0) ? -1.0 : 1.0;
}

__global__ void k_dist_pack(const int *__restrict__ idx, int cnt, const int *__restrict__ inv,
                            const double *__restrict__ x, double *__restrict__ buf) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const int v = idx[i];
        buf[i] = x[inv ? inv[v] : v];
    }
}

__global__ void k_dist_unpack(const int *__restrict__ idx, int cnt, const int *__restrict__ inv,
                              const double *__restrict__ buf, double *__restrict__ y) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const int v = idx[i];
        y[inv ? inv[v] : v] = buf[i];
    }
}

void dist_op(Handle &h, int level, int op, int64_t arg, const double *x, double *y, double *stat,
             const double *stat_in, const double *sign_slot, cudaStream_t st) {
    const Level &L = h.levels[level];
    const DistPlan &P = L.dist;
    FDL_REQUIRE(P.valid, FIEDLER_ERR_ARG, "fiedler_dist_op: no plan on this level (call fiedler_dist_plan)");
    // scratch allocated on the handle's stream must exist before `st` uses it
    if (ensure_solve_buffers(h, 8) && st != h.stream) FDL_CK(cudaStreamSynchronize(h.stream));
    Enq e{h, st};
    double *partials = h.partials.as<double>();
    unsigned *counter = h.counter.as<unsigned>();
    const int own = P.r1 - P.r0;
    switch (op) {
    case FIEDLER_DOP_RAND:
        FDL_REQUIRE(P.nranks == 1, FIEDLER_ERR_ARG, "FIEDLER_DOP_RAND needs a replicated (1-rank) plan");
        k_rand<<<grid_for(L.n, 256, h.row_grid), 256, 0, st>>>(L.n, (uint64_t)arg, y, stat, partials, counter);
        FDL_LAUNCH_CK();
        break;
    case FIEDLER_DOP_PROLONG: {
        FDL_REQUIRE(level + 1 < (int)h.levels.size(), FIEDLER_ERR_ARG, "no coarser level");
        k_dist_prolong<<<grid_for(own + P.recv_total, 256, h.row_grid), 256, 0, st>>>(
            P.r0, P.r1, P.recv_idx.as<int>(), P.recv_total, L.q_nat.as<int>(), arg ? L.inv.as<int>() : nullptr,
            x, y, stat, partials, counter);
        FDL_LAUNCH_CK();
        break;
    }
    case FIEDLER_DOP_GS_COLOUR: {
        FDL_REQUIRE(arg >= 0 && arg < L.ncolors, FIEDLER_ERR_ARG, "bad colour");
        PassArgs a{};
        a.x = x;
        a.n = L.n;
        a.stat_mode = 0;
        e.pass_tiles<OP_GS>(L, P.tilesGS.as<Tile>() + P.ctile[arg], P.ctile[arg + 1] - P.ctile[arg], a);
        break;
    }
    case FIEDLER_DOP_TO_NAT:
        k_dist_to_nat<<<grid_for(std::max(own, 1), 256, h.row_grid), 256, 0, st>>>(
            P.r0, P.r1, L.inv.as<int>(), x, y, stat, partials, counter);
        FDL_LAUNCH_CK();
        break;
    case FIEDLER_DOP_POWER: {
        PassArgs a{};
        a.x = x;
        a.y = y;
        a.in_stat = stat_in;
        a.out_stat = stat;
        a.stat_mode = 4 | 1;   // assign the partial sums, the caller reduces and finalises
        a.n = L.n;
        a.shift = L.shift;
        if (P.ntN) e.pass_tiles<OP_PI>(L, P.tilesN.as<Tile>(), P.ntN, a);
        else FDL_CK(cudaMemsetAsync(stat, 0, 16, st));
        break;
    }
    case FIEDLER_DOP_FINALISE:
        k_dist_finalise<<<1, 1, 0, st>>>(stat, L.n);
        FDL_LAUNCH_CK();
        break;
    case FIEDLER_DOP_FIRST_NONZERO:
        k_dist_first_nonzero<<<1, 32, 0, st>>>(P.r0, P.r1, x, stat_in, stat);
        FDL_LAUNCH_CK();
        break;
    case FIEDLER_DOP_SIGN:
        k_dist_sign<<<1, 1, 0, st>>>(stat);
        FDL_LAUNCH_CK();
        break;
    case FIEDLER_DOP_RAYLEIGH: {
        PassArgs a{};
        a.x = x;
        a.in_stat = stat_in;
        a.n = L.n;
        a.vnat = y;
        a.sign = sign_slot + 2;
        a.result = stat;
        a.rq_raw = 1;
        if (P.ntN) e.pass_tiles<OP_RQ>(L, P.tilesN.as<Tile>(), P.ntN, a);
        else FDL_CK(cudaMemsetAsync(stat, 0, 24, st));
        break;
    }
    case FIEDLER_DOP_FINALISE_RQ:
        k_dist_finalise_rq<<<1, 1, 0, st>>>(stat, stat_in);
        FDL_LAUNCH_CK();
        break;
    case FIEDLER_DOP_HALO_PACK:
        if (P.send_total) {
            k_dist_pack<<<grid_for(P.send_total), 256, 0, st>>>(P.send_idx.as<int>(), P.send_total,
                                                                 arg ? L.inv.as<int>() : nullptr, x, y);
            FDL_LAUNCH_CK();
        }
        break;
    case FIEDLER_DOP_HALO_UNPACK:
        if (P.recv_total) {
            k_dist_unpack<<<grid_for(P.recv_total), 256, 0, st>>>(P.recv_idx.as<int>(), P.recv_total,
                                                                   arg ? L.inv.as<int>() : nullptr, x, y);
            FDL_LAUNCH_CK();
        }
        break;
    default:
        throw Error(FIEDLER_ERR_ARG, "fiedler_dist_op: unknown op");
    }
}

}  // namespace fdl

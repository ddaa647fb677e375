// fdl_pset.cu -- row-partitioned setup of the fine levels (include/fiedler.h,
// "Row-partitioned SETUP").
//
// Every rank holds a level's whole CSR and runs the setup rules on its own rows
// [r0, r1) only; the driver (paper_1602_04386_b200/dist.py PartitionedSetup)
// exchanges the boundary rows' state between the calls.  The rules are those
// of the single-GPU setup (fdl_setup.cu) and of the oracle's readings:
//   R2 heavy-edge matching as the handshake of locally
//      heaviest free edges, aggregates numbered by increasing leader;
//   R3 Galerkin product: W_c(A, B) = left fold over the fine
//      edges {i < j} in (i, j) lexicographic order;
//   R4 Jones-Plassmann rounds of the greedy first-fit colouring in decreasing
//      priority.
// Each is a strict order, so the result does not depend on the partition or
// on the schedule of the rounds.  These kernels favour plain one-row-per-thread
// passes over the single-GPU setup's cooperative schedules: a rank's work is
// 1/N of a level and every round ends in a halo exchange anyway.
#include <algorithm>
#include <climits>
#include <vector>

#include "fdl_internal.h"

namespace fdl {
namespace {

constexpr int kPsBlock = 256;

inline int ps_grid(int64_t items) { return grid_for(std::max<int64_t>(items, 1), kPsBlock, kNumSMs * 16); }

// ------------------------------------------------------------------ partition
__global__ void k_ps_bounds(int64_t n, const int64_t *rp, int nranks, int64_t *bounds) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k > nranks) return;
    if (k == 0) { bounds[0] = 0; return; }
    if (k == nranks) { bounds[k] = n; return; }
    const int64_t total = rp[n] + n;
    const int64_t target = total * k / nranks;   // floor, as fiedler_dist_plan
    // first r in [0, n) with rp[r] + r >= target (n if none)
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (rp[mid] + mid >= target) hi = mid; else lo = mid + 1;
    }
    bounds[k] = lo;
}

struct RankBounds { int64_t b[FIEDLER_MAX_RANKS + 1]; };

__device__ __forceinline__ int owner_of(const RankBounds &rb, int nranks, int64_t u) {
    int lo = 0, hi = nranks - 1;   // largest k with b[k] <= u
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (rb.b[mid] <= u) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// peers of every own row (bit p: the row has a neighbour owned by rank p != rank)
__global__ void k_ps_peer_mask(const int64_t *rp, const int *ci, int64_t r0, int64_t r1, RankBounds rb,
                               int nranks, unsigned long long *mask, unsigned long long *counts) {
    for (int64_t v = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < r1;
         v += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long m = 0;
        for (int64_t k = rp[v]; k < rp[v + 1]; k++) {
            const int64_t u = ci[k];
            if (u < r0 || u >= r1) m |= 1ull << owner_of(rb, nranks, u);
        }
        mask[v - r0] = m;
        while (m) {
            const int p = __ffsll((long long)m) - 1;
            m &= m - 1;
            atomicAdd(counts + p, 1ull);
        }
    }
}

__global__ void k_ps_peer_flags(const unsigned long long *mask, int64_t own, int p, int *flags) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < own; i += (int64_t)gridDim.x * blockDim.x)
        flags[i] = (int)((mask[i] >> p) & 1ull);
}

__global__ void k_ps_add(int *x, int64_t count, int add) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        x[i] += add;
}

__global__ void k_ps_gather(const int *x, const int *idx, int64_t count, int *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = x[idx[i]];
}

__global__ void k_ps_scatter(const int *in, const int *idx, int64_t count, int *x) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        x[idx[i]] = in[i];
}

// ------------------------------------------------------------------ matching (R2)
// (w, h) decreasing: does (wa, ha) come before (wb, hb)?
__device__ __forceinline__ bool heavier(double wa, uint64_t ha, double wb, uint64_t hb) {
    return wa > wb || (wa == wb && ha > hb);
}

// Work lists of the rounds (optional caller scratch `work`, include/fiedler.h):
// a round walks the list the previous half-round left (or all own rows) and
// appends the rows that stay in play to the next list, one atomic per warp.
struct WorkList {
    const int *in;        // rows to visit; null: all own rows [r0, r1)
    const int *in_cnt;
    int *out;             // rows kept for the next half-round; null: no list
    int *out_cnt;
    int64_t r0, own;
    __device__ __forceinline__ int64_t count() const { return in ? (int64_t)*in_cnt : own; }
    __device__ __forceinline__ int64_t row(int64_t i) const { return in ? (int64_t)in[i] : r0 + i; }
    // every lane of the warp calls this with the same trip count
    __device__ __forceinline__ void keep(bool k, int v) const {
        if (!out) return;
        const unsigned m = __ballot_sync(0xffffffffu, k);
        if (!m) return;
        int base = 0;
        if (lane_id() == 0) base = atomicAdd(out_cnt, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (k) out[base + __popc(m & ((1u << lane_id()) - 1))] = v;
    }
};

// warp-uniform trip count of a grid-stride loop over [0, cnt)
#define PS_WARP_LOOP(i, cnt)                                                                     \
    for (int64_t i##_base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~int64_t(31),     \
                 i = i##_base + lane_id();                                                       \
         i##_base < (cnt); i##_base += (int64_t)gridDim.x * blockDim.x, i = i##_base + lane_id())

__global__ void k_ps_point(const int64_t *rp, const int *ci, const double *w, WorkList wl, uint64_t salt,
                           const int *mate, int *ptr, unsigned long long *active) {
    unsigned long long act = 0;
    const int64_t cnt = wl.count();
    PS_WARP_LOOP(i, cnt) {
        bool keep = false;
        int v = -1;
        if (i < cnt) {
            v = (int)wl.row(i);
            if (mate[v] < 0) {
                int best = -1;
                double bw = 0.0;
                uint64_t bh = 0;
                for (int64_t k = rp[v]; k < rp[v + 1]; k++) {
                    const int u = ci[k];
                    if (mate[u] >= 0) continue;
                    const uint64_t h = edge_hash(salt, v, u);
                    if (best < 0 || heavier(w[k], h, bw, bh)) { best = u; bw = w[k]; bh = h; }
                }
                ptr[v] = best;
                keep = best >= 0;
                act += keep;
            }
        }
        wl.keep(keep, v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) act += __shfl_xor_sync(0xffffffffu, act, o);
    if (lane_id() == 0 && act) atomicAdd(active, act);
}

__global__ void k_ps_resolve(WorkList wl, const int *ptr, int *mate) {
    const int64_t cnt = wl.count();
    PS_WARP_LOOP(i, cnt) {
        bool keep = false;
        int v = -1;
        if (i < cnt) {
            v = (int)wl.row(i);
            if (mate[v] < 0) {
                const int u = ptr[v];
                if (u >= 0 && ptr[u] == v) mate[v] = u;
                else keep = true;   // still free: visited by the next POINT
            }
        }
        wl.keep(keep, v);
    }
}

// ------------------------------------------------------------------ aggregates (R2)
__device__ __forceinline__ int heaviest_neighbour(const int64_t *rp, const int *ci, const double *w,
                                                  uint64_t salt, int v) {
    int best = -1;
    double bw = 0.0;
    uint64_t bh = 0;
    for (int64_t k = rp[v]; k < rp[v + 1]; k++) {
        const int u = ci[k];
        const uint64_t h = edge_hash(salt, v, u);
        if (best < 0 || heavier(w[k], h, bw, bh)) { best = u; bw = w[k]; bh = h; }
    }
    return best;
}

__global__ void k_ps_leader_flags(const int64_t *rp, const int *mate, int64_t r0, int64_t r1, int *flags) {
    for (int64_t v = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < r1;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int m = mate[v];
        flags[v - r0] = m >= 0 ? (int)(v < m) : (int)(rp[v + 1] == rp[v]);
    }
}

__global__ void k_ps_ids(int64_t r0, int64_t r1, const int *flags, const int *pos, int offset, int *q) {
    for (int64_t v = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < r1;
         v += (int64_t)gridDim.x * blockDim.x)
        q[v] = flags[v - r0] ? offset + pos[v - r0] : -1;
}

__global__ void k_ps_q_mates(int64_t r0, int64_t r1, const int *mate, int *q) {
    for (int64_t v = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < r1;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int m = mate[v];
        if (m >= 0 && m < v) q[v] = q[m];
    }
}

__global__ void k_ps_q_join(const int64_t *rp, const int *ci, const double *w, int64_t r0, int64_t r1,
                            uint64_t salt, const int *mate, int *q, unsigned long long *bad) {
    for (int64_t v = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < r1;
         v += (int64_t)gridDim.x * blockDim.x) {
        if (mate[v] >= 0 || rp[v + 1] == rp[v]) continue;
        const int m = heaviest_neighbour(rp, ci, w, salt, (int)v);
        if (mate[m] < 0 || q[m] < 0) atomicAdd(bad, 1ull);   // not maximal / q(m) not exchanged
        q[v] = q[m];
    }
}

// ------------------------------------------------------------------ Galerkin (R3)
__global__ void k_ps_member_flags(int64_t n, const int *q, int a0, int a1, int *flags) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        flags[v] = q[v] >= a0 && q[v] < a1;
}

__global__ void k_ps_contrib_count(const int64_t *rp, const int *ci, const int *q, const int *members,
                                   int64_t nm, int *cnt) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nm; t += (int64_t)gridDim.x * blockDim.x) {
        const int i = members[t], a = q[i];
        int c = 0;
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) c += q[ci[k]] != a;
        cnt[t] = c;
    }
}

// contribution of the entry i -> j (q(j) = B != A = q(i)) of a member i of a
// coarse row A in [a0, a1): key1 = (A - a0, B), key2 = (min(i, j), max(i, j)),
// value = the CSR position of the entry
__global__ void k_ps_contrib_fill(const int64_t *rp, const int *ci, const int *q, const int *members, int64_t nm,
                                  const int *off, int a0, unsigned long long *key1, unsigned long long *key2,
                                  int *val) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nm; t += (int64_t)gridDim.x * blockDim.x) {
        const int i = members[t], a = q[i];
        int o = off[t];
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) {
            const int j = ci[k], b = q[j];
            if (b == a) continue;
            key1[o] = ((unsigned long long)(a - a0) << 31) | (unsigned long long)b;
            const unsigned long long lo = (unsigned)min(i, j), hi = (unsigned)max(i, j);
            key2[o] = (lo << 31) | hi;
            val[o] = (int)k;
            o++;
        }
    }
}

__global__ void k_ps_iota(int *x, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = (int)i;
}

__global__ void k_ps_permute_keys(const unsigned long long *key1, const int *perm, int64_t n,
                                  unsigned long long *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = key1[perm[i]];
}

__global__ void k_ps_run_flags(const unsigned long long *key1, int64_t n, int *flags) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flags[i] = i == 0 || key1[i] != key1[i - 1];
}

// one thread per (A, B) run: the left fold of its weights in (lo, hi) order
__global__ void k_ps_fold(const unsigned long long *key1, const int *perm, const int *val, const double *w,
                          const int *starts, int nruns, int64_t ncontrib, int *cci, double *cw, int *row) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nruns; r += (int64_t)gridDim.x * blockDim.x) {
        const int s = starts[r];
        const int e = r + 1 < nruns ? starts[r + 1] : (int)ncontrib;
        double acc = w[val[perm[s]]];
        for (int t = s + 1; t < e; t++) acc += w[val[perm[t]]];
        cci[r] = (int)(key1[s] & 0x7fffffffull);
        cw[r] = acc;
        row[r] = (int)(key1[s] >> 31);
    }
}

// crp[A] = the first run of a row >= A (runs are sorted by row)
__global__ void k_ps_row_ptr(const int *row, int nruns, int na, int64_t *crp) {
    for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a <= na; a += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nruns;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (row[mid] >= a) hi = mid; else lo = mid + 1;
        }
        crp[a] = lo;
    }
}

// Per-coarse-row path.  Members grouped by coarse row (counting sort), T_A =
// the sum of the members' degrees (the row's slots); rows with T_A <= kGalSmall
// are built by one thread each: contributions insertion-sorted by (B, lo, hi)
// in local memory, runs folded left to right; bigger rows go through the
// two-sort path above, restricted to their members.
constexpr int kGalSmall = 32;

__global__ void k_ps_row_members(const int64_t *rp, int64_t n, const int *q, int a0, int a1, int *mcnt, int *slots) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int a = q[v];
        if (a < a0 || a >= a1) continue;
        atomicAdd(mcnt + (a - a0), 1);
        atomicAdd(slots + (a - a0), (int)(rp[v + 1] - rp[v]));
    }
}

__global__ void k_ps_row_fill(int64_t n, const int *q, int a0, int a1, const int *mrp, int *cursor, int *mem) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int a = q[v];
        if (a < a0 || a >= a1) continue;
        mem[mrp[a - a0] + atomicAdd(cursor + (a - a0), 1)] = (int)v;
    }
}

__global__ void k_ps_gal_small(const int64_t *rp, const int *ci, const double *w, const int *q, int a0, int na,
                               const int *mrp, const int *mem, const int *slots, const int *soff, int *sB,
                               double *sW, int *cnt, int *big) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < na; r += gridDim.x * blockDim.x) {
        if (slots[r] > kGalSmall) {
            big[r] = 1;
            cnt[r] = 0;
            continue;
        }
        big[r] = 0;
        const int A = a0 + r;
        int bb[kGalSmall];
        unsigned long long kk[kGalSmall];
        double ww[kGalSmall];
        int m = 0;
        for (int t = mrp[r]; t < mrp[r + 1]; t++) {
            const int i = mem[t];
            for (int64_t k = rp[i]; k < rp[i + 1]; k++) {
                const int j = ci[k], B = q[j];
                if (B == A) continue;
                const unsigned long long key = ((unsigned long long)min(i, j) << 32) | (unsigned)max(i, j);
                int p = m++;
                while (p > 0 && (bb[p - 1] > B || (bb[p - 1] == B && kk[p - 1] > key))) {
                    bb[p] = bb[p - 1];
                    kk[p] = kk[p - 1];
                    ww[p] = ww[p - 1];
                    p--;
                }
                bb[p] = B;
                kk[p] = key;
                ww[p] = w[k];
            }
        }
        int o = soff[r], c = 0;
        for (int t = 0; t < m;) {
            double acc = ww[t];
            int u = t + 1;
            for (; u < m && bb[u] == bb[t]; u++) acc += ww[u];
            sB[o + c] = bb[t];
            sW[o + c] = acc;
            c++;
            t = u;
        }
        cnt[r] = c;
    }
}

__global__ void k_ps_big_member_flags(int64_t n, const int *q, int a0, int a1, const int *big, int *flags) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int a = q[v];
        flags[v] = a >= a0 && a < a1 && big[a - a0];
    }
}

// runs of the big rows into their slot ranges; rr = first run of every local row
__global__ void k_ps_big_place(const int *row, const int *cB, const double *cWv, int nruns, const int *rr,
                               const int *soff, int *sB, double *sW) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nruns; t += gridDim.x * blockDim.x) {
        const int r = row[t];
        const int o = soff[r] + (t - rr[r]);
        sB[o] = cB[t];
        sW[o] = cWv[t];
    }
}

__global__ void k_ps_big_cnt(const int *rr, int na, const int *big, int *cnt) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < na; r += gridDim.x * blockDim.x)
        if (big[r]) cnt[r] = rr[r + 1] - rr[r];
}

__global__ void k_ps_gal_out(int na, const int *cnt, const int *coff, const int *soff, const int *sB, const double *sW,
                             int64_t *crp, int *cci, double *cw, int total) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= na; r += gridDim.x * blockDim.x) {
        if (r == na) { crp[na] = total; continue; }
        const int o = coff[r], s0 = soff[r];
        crp[r] = o;
        for (int t = 0; t < cnt[r]; t++) {
            cci[o + t] = sB[s0 + t];
            cw[o + t] = sW[s0 + t];
        }
    }
}

__global__ void k_ps_row_ptr32(const int *row, int nruns, int na, int *rr) {
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a <= na; a += gridDim.x * blockDim.x) {
        int lo = 0, hi = nruns;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (row[mid] >= a) hi = mid; else lo = mid + 1;
        }
        rr[a] = lo;
    }
}

// ------------------------------------------------------------------ colouring (R4)
__global__ void k_ps_colour(const int64_t *rp, const int *ci, WorkList wl, uint64_t salt, int *colour,
                            unsigned long long *left, int *maxc) {
    unsigned long long nleft = 0;
    int mc = -1;
    const int64_t cnt = wl.count();
    PS_WARP_LOOP(i, cnt) {
        bool keep = false;
        int v = -1;
        if (i < cnt) {
            v = (int)wl.row(i);
            if (colour[v] < 0) {
                const uint64_t pv = splitmix64(salt ^ (uint64_t)v);
                bool ready = true;
                for (int64_t k = rp[v]; k < rp[v + 1] && ready; k++) {
                    const int u = ci[k];
                    const uint64_t pu = splitmix64(salt ^ (uint64_t)u);
                    if ((pu > pv || (pu == pv && u > v)) && colour[u] < 0) ready = false;
                }
                if (ready) {
                    // first fit: smallest colour no coloured neighbour has (all coloured
                    // neighbours have higher priority), 64 colours per row scan
                    int cv = 0;
                    for (int base = 0;; base += 64) {
                        unsigned long long used = 0;
                        for (int64_t k = rp[v]; k < rp[v + 1]; k++) {
                            const int c = colour[ci[k]] - base;
                            if (c >= 0 && c < 64) used |= 1ull << c;
                        }
                        if (~used) { cv = base + __ffsll((long long)~used) - 1; break; }
                    }
                    colour[v] = cv;
                    mc = max(mc, cv);
                } else {
                    keep = true;
                    nleft++;
                }
            }
        }
        wl.keep(keep, v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        nleft += __shfl_xor_sync(0xffffffffu, nleft, o);
        mc = max(mc, __shfl_xor_sync(0xffffffffu, mc, o));
    }
    if (lane_id() == 0) {
        if (nleft) atomicAdd(left, nleft);
        atomicMax(maxc, mc);
    }
}

__global__ void k_ps_init_counters(unsigned long long *c, int nc, int *m) {
    if (threadIdx.x < nc) c[threadIdx.x] = 0;
    if (threadIdx.x == 0 && m) *m = -1;
}

void check_rows(int64_t n, int64_t r0, int64_t r1) {
    FDL_REQUIRE(n >= 1 && n < (int64_t(1) << 31) - 1, FIEDLER_ERR_ARG, "n out of range");
    FDL_REQUIRE(0 <= r0 && r0 <= r1 && r1 <= n, FIEDLER_ERR_ARG, "own rows outside [0, n]");
}

}  // namespace

// ------------------------------------------------------------------ host side
void pset_bounds(int64_t n, const int64_t *rp, int nranks, int64_t *bounds, cudaStream_t st) {
    DBuf b((size_t)(nranks + 1) * 8, st);
    k_ps_bounds<<<1, 128, 0, st>>>(n, rp, nranks, b.as<int64_t>());
    FDL_LAUNCH_CK();
    readback(st, {{bounds, b.p, (size_t)(nranks + 1) * 8}});
}

void pset_halo(int64_t n, const int64_t *rp, const int *ci, int nranks, int rank, const int64_t *bounds,
               int *send_idx, int64_t *send_count, cudaStream_t st) {
    RankBounds rb{};
    for (int k = 0; k <= nranks; k++) rb.b[k] = bounds[k];
    const int64_t r0 = bounds[rank], r1 = bounds[rank + 1], own = r1 - r0;
    DBuf mask((size_t)std::max<int64_t>(own, 1) * 8, st), counts((size_t)FIEDLER_MAX_RANKS * 8, st);
    k_ps_init_counters<<<1, FIEDLER_MAX_RANKS, 0, st>>>(counts.as<unsigned long long>(), FIEDLER_MAX_RANKS, nullptr);
    FDL_LAUNCH_CK();
    if (own) {
        k_ps_peer_mask<<<ps_grid(own), kPsBlock, 0, st>>>(rp, ci, r0, r1, rb, nranks, mask.as<unsigned long long>(),
                                                          counts.as<unsigned long long>());
        FDL_LAUNCH_CK();
    }
    std::vector<unsigned long long> hc(FIEDLER_MAX_RANKS);
    readback(st, {{hc.data(), counts.p, (size_t)FIEDLER_MAX_RANKS * 8}});
    for (int p = 0; p < nranks; p++) send_count[p] = p == rank ? 0 : (int64_t)hc[p];
    if (!send_idx || !own) return;
    DBuf flags((size_t)own * 4, st), dcount(8, st);
    int64_t off = 0;
    for (int p = 0; p < nranks; p++) {
        if (p == rank || !send_count[p]) continue;
        k_ps_peer_flags<<<ps_grid(own), kPsBlock, 0, st>>>(mask.as<unsigned long long>(), own, p, flags.as<int>());
        FDL_LAUNCH_CK();
        compact_flagged(nullptr, flags.as<int>(), own, send_idx + off, dcount.as<int>(), st);
        k_ps_add<<<ps_grid(send_count[p]), kPsBlock, 0, st>>>(send_idx + off, send_count[p], (int)r0);
        FDL_LAUNCH_CK();
        off += send_count[p];
    }
    host_wait(st);   // the scratch above is freed on st; the lists are complete on return
}

void pset_gather(const int *x, const int *idx, int64_t count, int *out, cudaStream_t st) {
    if (count <= 0) return;
    k_ps_gather<<<ps_grid(count), kPsBlock, 0, st>>>(x, idx, count, out);
    FDL_LAUNCH_CK();
}

void pset_scatter(const int *in, const int *idx, int64_t count, int *x, cudaStream_t st) {
    if (count <= 0) return;
    k_ps_scatter<<<ps_grid(count), kPsBlock, 0, st>>>(in, idx, count, x);
    FDL_LAUNCH_CK();
}

// work lists in `work` (device int32 [8 + 2 own]): header {count A, count B},
// list A at work + 8, list B at work + 8 + own.  POINT of round 0 visits every
// own row and writes B; RESOLVE reads B, writes A; later POINTs read A, write B.
static WorkList make_list(int *work, int64_t r0, int64_t own, int read, int write) {
    WorkList wl{};
    wl.r0 = r0;
    wl.own = own;
    if (work) {
        if (read >= 0) { wl.in = work + 8 + read * own; wl.in_cnt = work + read; }
        wl.out = work + 8 + write * own;
        wl.out_cnt = work + write;
    }
    return wl;
}

void pset_match(int phase, int64_t n, const int64_t *rp, const int *ci, const double *w, int64_t r0, int64_t r1,
                uint64_t seed, int level, int *mate, int *ptr, int round, int *work, int64_t *active, cudaStream_t st) {
    check_rows(n, r0, r1);
    FDL_REQUIRE(round >= 0, FIEDLER_ERR_ARG, "round < 0");
    const int64_t own = r1 - r0;
    if (phase == FIEDLER_PSET_POINT) {
        FDL_REQUIRE(active, FIEDLER_ERR_ARG, "POINT needs `active`");
        DBuf cnt(8, st);
        k_ps_init_counters<<<1, 32, 0, st>>>(cnt.as<unsigned long long>(), 1, nullptr);
        FDL_LAUNCH_CK();
        if (own) {
            if (work) FDL_CK(cudaMemsetAsync(work + 1, 0, 4, st));
            k_ps_point<<<ps_grid(own), kPsBlock, 0, st>>>(rp, ci, w, make_list(work, r0, own, round ? 0 : -1, 1),
                                                          salt_match(seed, level), mate, ptr,
                                                          cnt.as<unsigned long long>());
            FDL_LAUNCH_CK();
        }
        unsigned long long a = 0;
        readback(st, {{&a, cnt.p, 8}});
        *active = (int64_t)a;
    } else if (phase == FIEDLER_PSET_RESOLVE) {
        if (!own) return;
        if (work) FDL_CK(cudaMemsetAsync(work, 0, 4, st));
        k_ps_resolve<<<ps_grid(own), kPsBlock, 0, st>>>(make_list(work, r0, own, work ? 1 : -1, 0), ptr, mate);
        FDL_LAUNCH_CK();
    } else {
        throw Error(FIEDLER_ERR_ARG, "bad matching phase");
    }
}

void pset_aggregate(int phase, int64_t n, const int64_t *rp, const int *ci, const double *w, int64_t r0, int64_t r1,
                    uint64_t seed, int level, const int *mate, int *q, int64_t offset, int64_t *count,
                    cudaStream_t st) {
    check_rows(n, r0, r1);
    const int64_t own = r1 - r0;
    if (phase == FIEDLER_PSET_LEADERS || phase == FIEDLER_PSET_IDS) {
        FDL_REQUIRE(phase != FIEDLER_PSET_LEADERS || count, FIEDLER_ERR_ARG, "LEADERS needs `count`");
        FDL_REQUIRE(offset >= 0 && offset < n, FIEDLER_ERR_ARG, "offset out of range");
        if (!own) {
            if (count) *count = 0;
            return;
        }
        DBuf flags((size_t)own * 4, st), pos((size_t)own * 4, st), tot(8, st);
        k_ps_leader_flags<<<ps_grid(own), kPsBlock, 0, st>>>(rp, mate, r0, r1, flags.as<int>());
        FDL_LAUNCH_CK();
        scan_exclusive(flags.as<int>(), pos.as<int>(), own, tot.as<int>(), st);
        if (phase == FIEDLER_PSET_IDS) {
            k_ps_ids<<<ps_grid(own), kPsBlock, 0, st>>>(r0, r1, flags.as<int>(), pos.as<int>(), (int)offset, q);
            FDL_LAUNCH_CK();
        }
        int t = 0;
        readback(st, {{&t, tot.p, 4}});
        if (count) *count = t;
    } else if (phase == FIEDLER_PSET_MATES) {
        if (!own) return;
        k_ps_q_mates<<<ps_grid(own), kPsBlock, 0, st>>>(r0, r1, mate, q);
        FDL_LAUNCH_CK();
    } else if (phase == FIEDLER_PSET_JOIN) {
        if (!own) return;
        DBuf bad(8, st);
        k_ps_init_counters<<<1, 32, 0, st>>>(bad.as<unsigned long long>(), 1, nullptr);
        FDL_LAUNCH_CK();
        k_ps_q_join<<<ps_grid(own), kPsBlock, 0, st>>>(rp, ci, w, r0, r1, salt_match(seed, level), mate, q,
                                                       bad.as<unsigned long long>());
        FDL_LAUNCH_CK();
        unsigned long long b = 0;
        readback(st, {{&b, bad.p, 8}});
        FDL_REQUIRE(b == 0, FIEDLER_ERR_INTERNAL,
                    "JOIN: a heaviest neighbour is unmatched or has no aggregate (matching not maximal, "
                    "or q of the boundary rows not exchanged)");
    } else {
        throw Error(FIEDLER_ERR_ARG, "bad aggregate phase");
    }
}

// the two-sort path: contributions of the members listed in `members` (nm of
// them), sorted by (A, B, lo, hi), folded per (A, B); returns the number of
// runs, their local row / column / weight in row / cB / cWv
static int gal_sorted_runs(const int64_t *rp, const int *ci, const double *w, const int *q, const int *members, int nm,
                           int a0, int na, DBuf &row, DBuf &cB, DBuf &cWv, cudaStream_t st) {
    DBuf cnt((size_t)std::max(nm, 1) * 4, st), off((size_t)std::max(nm, 1) * 4, st), dcnt(8, st);
    k_ps_contrib_count<<<ps_grid(nm), kPsBlock, 0, st>>>(rp, ci, q, members, nm, cnt.as<int>());
    FDL_LAUNCH_CK();
    scan_exclusive(cnt.as<int>(), off.as<int>(), nm, dcnt.as<int>(), st);
    int nc = 0;
    readback(st, {{&nc, dcnt.p, 4}});
    if (!nc) return 0;
    DBuf key1((size_t)nc * 8, st), key2((size_t)nc * 8, st), val((size_t)nc * 4, st), perm((size_t)nc * 4, st),
        skey((size_t)nc * 8, st);
    k_ps_contrib_fill<<<ps_grid(nm), kPsBlock, 0, st>>>(rp, ci, q, members, nm, off.as<int>(), a0,
                                                        key1.as<unsigned long long>(), key2.as<unsigned long long>(),
                                                        val.as<int>());
    FDL_LAUNCH_CK();
    // (A, B, lo, hi) order by two stable LSD sorts: (lo, hi) first, then (A, B)
    k_ps_iota<<<ps_grid(nc), kPsBlock, 0, st>>>(perm.as<int>(), nc);
    FDL_LAUNCH_CK();
    radix_sort_u64_i32(key2.as<unsigned long long>(), perm.as<int>(), nc, 62, st);
    k_ps_permute_keys<<<ps_grid(nc), kPsBlock, 0, st>>>(key1.as<unsigned long long>(), perm.as<int>(), nc,
                                                        skey.as<unsigned long long>());
    FDL_LAUNCH_CK();
    radix_sort_u64_i32(skey.as<unsigned long long>(), perm.as<int>(), nc, 31 + bits_for(std::max(na - 1, 0)), st);
    DBuf rflags((size_t)nc * 4, st), starts((size_t)nc * 4, st);
    k_ps_run_flags<<<ps_grid(nc), kPsBlock, 0, st>>>(skey.as<unsigned long long>(), nc, rflags.as<int>());
    FDL_LAUNCH_CK();
    compact_flagged(nullptr, rflags.as<int>(), nc, starts.as<int>(), dcnt.as<int>(), st);
    int nruns = 0;
    readback(st, {{&nruns, dcnt.p, 4}});
    row.alloc((size_t)nruns * 4, st);
    cB.alloc((size_t)nruns * 4, st);
    cWv.alloc((size_t)nruns * 8, st);
    k_ps_fold<<<ps_grid(nruns), kPsBlock, 0, st>>>(skey.as<unsigned long long>(), perm.as<int>(), val.as<int>(), w,
                                                   starts.as<int>(), nruns, nc, cB.as<int>(), cWv.as<double>(),
                                                   row.as<int>());
    FDL_LAUNCH_CK();
    return nruns;
}

void pset_galerkin(int phase, int64_t n, const int64_t *rp, const int *ci, const double *w, const int *q, int64_t a0,
                   int64_t a1, int64_t cap, int64_t *crp, int *cci, double *cw, int64_t *count, cudaStream_t st) {
    check_rows(n, 0, n);
    FDL_REQUIRE(0 <= a0 && a0 <= a1 && a1 <= n, FIEDLER_ERR_ARG, "coarse rows out of range");
    FDL_REQUIRE(count, FIEDLER_ERR_ARG, "NULL count");
    FDL_REQUIRE(phase == 0 || phase == 1, FIEDLER_ERR_ARG, "bad Galerkin phase");
    const int na = (int)(a1 - a0);
    // members grouped by coarse row (counting sort) and the rows' slot counts
    DBuf mcnt((size_t)(na + 1) * 4, st), slots((size_t)(na + 1) * 4, st), mrp((size_t)(na + 1) * 4, st),
        soff((size_t)(na + 1) * 4, st), dcnt(16, st);
    FDL_CK(cudaMemsetAsync(mcnt.p, 0, (size_t)(na + 1) * 4, st));
    FDL_CK(cudaMemsetAsync(slots.p, 0, (size_t)(na + 1) * 4, st));
    k_ps_row_members<<<ps_grid(n), kPsBlock, 0, st>>>(rp, n, q, (int)a0, (int)a1, mcnt.as<int>(), slots.as<int>());
    FDL_LAUNCH_CK();
    scan_exclusive(mcnt.as<int>(), mrp.as<int>(), na + 1, dcnt.as<int>(), st);
    scan_exclusive(slots.as<int>(), soff.as<int>(), na + 1, dcnt.as<int>() + 1, st);
    int tot[2] = {0, 0};
    readback(st, {{tot, dcnt.p, 8}});
    const int nm = tot[0], ns = tot[1];
    if (phase == 0) {   // crossing contributions of the rows (<= their slots)
        if (!nm) { *count = 0; return; }
        DBuf flags((size_t)n * 4, st), members((size_t)n * 4, st), cnt((size_t)nm * 4, st), pos((size_t)nm * 4, st);
        k_ps_member_flags<<<ps_grid(n), kPsBlock, 0, st>>>(n, q, (int)a0, (int)a1, flags.as<int>());
        FDL_LAUNCH_CK();
        compact_flagged(nullptr, flags.as<int>(), n, members.as<int>(), dcnt.as<int>(), st);
        k_ps_contrib_count<<<ps_grid(nm), kPsBlock, 0, st>>>(rp, ci, q, members.as<int>(), nm, cnt.as<int>());
        FDL_LAUNCH_CK();
        scan_exclusive(cnt.as<int>(), pos.as<int>(), nm, dcnt.as<int>(), st);
        int nc = 0;
        readback(st, {{&nc, dcnt.p, 4}});
        *count = nc;
        return;
    }
    FDL_REQUIRE(crp, FIEDLER_ERR_ARG, "NULL crp");
    DBuf mem((size_t)std::max(nm, 1) * 4, st), cursor((size_t)(na + 1) * 4, st), sB((size_t)std::max(ns, 1) * 4, st),
        sW((size_t)std::max(ns, 1) * 8, st), cnt((size_t)(na + 1) * 4, st), big((size_t)(na + 1) * 4, st),
        coff((size_t)(na + 1) * 4, st);
    FDL_CK(cudaMemsetAsync(cursor.p, 0, (size_t)(na + 1) * 4, st));
    FDL_CK(cudaMemsetAsync(cnt.p, 0, (size_t)(na + 1) * 4, st));
    FDL_CK(cudaMemsetAsync(big.p, 0, (size_t)(na + 1) * 4, st));
    if (na) {
        k_ps_row_fill<<<ps_grid(n), kPsBlock, 0, st>>>(n, q, (int)a0, (int)a1, mrp.as<int>(), cursor.as<int>(),
                                                       mem.as<int>());
        FDL_LAUNCH_CK();
        k_ps_gal_small<<<ps_grid(na), kPsBlock, 0, st>>>(rp, ci, w, q, (int)a0, na, mrp.as<int>(), mem.as<int>(),
                                                         slots.as<int>(), soff.as<int>(), sB.as<int>(), sW.as<double>(),
                                                         cnt.as<int>(), big.as<int>());
        FDL_LAUNCH_CK();
        // rows with more than kGalSmall slots: the sort path over their members
        DBuf flags((size_t)n * 4, st), members((size_t)n * 4, st);
        k_ps_big_member_flags<<<ps_grid(n), kPsBlock, 0, st>>>(n, q, (int)a0, (int)a1, big.as<int>(), flags.as<int>());
        FDL_LAUNCH_CK();
        compact_flagged(nullptr, flags.as<int>(), n, members.as<int>(), dcnt.as<int>(), st);
        int nbm = 0;
        readback(st, {{&nbm, dcnt.p, 4}});
        if (nbm) {
            DBuf row, cB, cWv;
            const int nruns = gal_sorted_runs(rp, ci, w, q, members.as<int>(), nbm, (int)a0, na, row, cB, cWv, st);
            if (nruns) {
                DBuf rr((size_t)(na + 1) * 4, st);
                k_ps_row_ptr32<<<ps_grid(na + 1), kPsBlock, 0, st>>>(row.as<int>(), nruns, na, rr.as<int>());
                FDL_LAUNCH_CK();
                k_ps_big_place<<<ps_grid(nruns), kPsBlock, 0, st>>>(row.as<int>(), cB.as<int>(), cWv.as<double>(),
                                                                    nruns, rr.as<int>(), soff.as<int>(), sB.as<int>(),
                                                                    sW.as<double>());
                FDL_LAUNCH_CK();
                k_ps_big_cnt<<<ps_grid(na), kPsBlock, 0, st>>>(rr.as<int>(), na, big.as<int>(), cnt.as<int>());
                FDL_LAUNCH_CK();
            }
        }
    }
    scan_exclusive(cnt.as<int>(), coff.as<int>(), na + 1, dcnt.as<int>(), st);
    int nnz = 0;
    readback(st, {{&nnz, dcnt.p, 4}});
    FDL_REQUIRE(cap >= nnz && (nnz == 0 || (cci && cw)), FIEDLER_ERR_ARG, "cap below the coarse nonzeros");
    k_ps_gal_out<<<ps_grid(na + 1), kPsBlock, 0, st>>>(na, cnt.as<int>(), coff.as<int>(), soff.as<int>(), sB.as<int>(),
                                                       sW.as<double>(), crp, cci, cw, nnz);
    FDL_LAUNCH_CK();
    *count = nnz;
    host_wait(st);
}

void pset_colour(int64_t n, const int64_t *rp, const int *ci, int64_t r0, int64_t r1, uint64_t seed, int level,
                 int round, int *work, int *colour, int64_t *out, cudaStream_t st) {
    check_rows(n, r0, r1);
    FDL_REQUIRE(out, FIEDLER_ERR_ARG, "NULL out");
    FDL_REQUIRE(round >= 0, FIEDLER_ERR_ARG, "round < 0");
    const int64_t own = r1 - r0;
    DBuf c(16, st);
    k_ps_init_counters<<<1, 32, 0, st>>>(c.as<unsigned long long>(), 1, reinterpret_cast<int *>(c.as<char>() + 8));
    FDL_LAUNCH_CK();
    if (own) {
        // round r reads the list of round r - 1 (parity), writes list r & 1
        const int wr = round & 1;
        if (work) FDL_CK(cudaMemsetAsync(work + wr, 0, 4, st));
        k_ps_colour<<<ps_grid(own), kPsBlock, 0, st>>>(rp, ci, make_list(work, r0, own, round ? 1 - wr : -1, wr),
                                                       salt_color(seed, level), colour, c.as<unsigned long long>(),
                                                       reinterpret_cast<int *>(c.as<char>() + 8));
        FDL_LAUNCH_CK();
    }
    struct { unsigned long long left; int maxc, pad; } h{};
    readback(st, {{&h, c.p, 16}});
    out[0] = (int64_t)h.left;
    out[1] = h.maxc;
}

}  // namespace fdl

// ------------------------------------------------------------------ C ABI
using namespace fdl;

extern "C" {

int fiedler_pset_bounds(int64_t n, const int64_t *row_ptr, int32_t nranks, int64_t *bounds, void *stream) {
    API_BEGIN
    FDL_REQUIRE(n >= 1 && row_ptr && bounds, FIEDLER_ERR_ARG, "bad arguments");
    FDL_REQUIRE(nranks >= 1 && nranks <= FIEDLER_MAX_RANKS, FIEDLER_ERR_ARG, "nranks outside [1, MAX_RANKS]");
    pset_bounds(n, row_ptr, nranks, bounds, (cudaStream_t)stream);
    return FIEDLER_OK;
    API_END
}

int fiedler_pset_halo(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, int32_t nranks, int32_t rank,
                      const int64_t *bounds, int32_t *send_idx, int64_t *send_count, void *stream) {
    API_BEGIN
    FDL_REQUIRE(n >= 1 && row_ptr && col_idx && bounds && send_count, FIEDLER_ERR_ARG, "bad arguments");
    FDL_REQUIRE(nranks >= 1 && nranks <= FIEDLER_MAX_RANKS && rank >= 0 && rank < nranks, FIEDLER_ERR_ARG,
                "bad nranks / rank");
    FDL_REQUIRE(bounds[0] == 0 && bounds[nranks] == n, FIEDLER_ERR_ARG, "bounds must span [0, n]");
    for (int k = 0; k < nranks; k++) FDL_REQUIRE(bounds[k] <= bounds[k + 1], FIEDLER_ERR_ARG, "bounds not sorted");
    pset_halo(n, row_ptr, col_idx, nranks, rank, bounds, send_idx, send_count, (cudaStream_t)stream);
    return FIEDLER_OK;
    API_END
}

int fiedler_pset_gather(const int32_t *x, const int32_t *idx, int64_t count, int32_t *out, void *stream) {
    API_BEGIN
    FDL_REQUIRE(count >= 0 && (count == 0 || (x && idx && out)), FIEDLER_ERR_ARG, "bad arguments");
    pset_gather(x, idx, count, out, (cudaStream_t)stream);
    return FIEDLER_OK;
    API_END
}

int fiedler_pset_scatter(const int32_t *in, const int32_t *idx, int64_t count, int32_t *x, void *stream) {
    API_BEGIN
    FDL_REQUIRE(count >= 0 && (count == 0 || (x && idx && in)), FIEDLER_ERR_ARG, "bad arguments");
    pset_scatter(in, idx, count, x, (cudaStream_t)stream);
    return FIEDLER_OK;
    API_END
}

int fiedler_pset_match(int32_t phase, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                       const double *weights, int64_t r0, int64_t r1, uint64_t seed, int32_t level, int32_t *mate,
                       int32_t *ptr, int32_t round, int32_t *work, int64_t *active, void *stream) {
    API_BEGIN
    FDL_REQUIRE(row_ptr && col_idx && weights && mate && ptr, FIEDLER_ERR_ARG, "NULL array");
    pset_match(phase, n, row_ptr, col_idx, weights, r0, r1, seed, level, mate, ptr, round, work, active,
               (cudaStream_t)stream);
    return FIEDLER_OK;
    API_END
}

int fiedler_pset_aggregate(int32_t phase, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                           const double *weights, int64_t r0, int64_t r1, uint64_t seed, int32_t level,
                           const int32_t *mate, int32_t *q, int64_t offset, int64_t *count, void *stream) {
    API_BEGIN
    FDL_REQUIRE(row_ptr && col_idx && weights && mate && q, FIEDLER_ERR_ARG, "NULL array");
    pset_aggregate(phase, n, row_ptr, col_idx, weights, r0, r1, seed, level, mate, q, offset, count,
                   (cudaStream_t)stream);
    return FIEDLER_OK;
    API_END
}

int fiedler_pset_galerkin(int32_t phase, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                          const double *weights, const int32_t *q, int64_t a0, int64_t a1, int64_t cap, int64_t *crp,
                          int32_t *cci, double *cw, int64_t *count, void *stream) {
    API_BEGIN
    FDL_REQUIRE(row_ptr && col_idx && weights && q, FIEDLER_ERR_ARG, "NULL array");
    pset_galerkin(phase, n, row_ptr, col_idx, weights, q, a0, a1, cap, crp, cci, cw, count, (cudaStream_t)stream);
    return FIEDLER_OK;
    API_END
}

int fiedler_pset_colour(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, int64_t r0, int64_t r1,
                        uint64_t seed, int32_t level, int32_t round, int32_t *work, int32_t *colour, int64_t *out,
                        void *stream) {
    API_BEGIN
    FDL_REQUIRE(row_ptr && col_idx && colour, FIEDLER_ERR_ARG, "NULL array");
    pset_colour(n, row_ptr, col_idx, r0, r1, seed, level, round, work, colour, out, (cudaStream_t)stream);
    return FIEDLER_OK;
    API_END
}

}  // extern "C"

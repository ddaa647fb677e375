// fdl_setup.cu -- Setup Phase of Algorithm 3 on the GPU.
//
//   per level l (natural numbering):
//     heavy edge coarsening, parallel order (R2): locally-dominant handshake
//       matching in the strict edge order (w, splitmix64 hash) -- equal to the
//       greedy heaviest-first matching -- then unmatched vertices join the
//       aggregate of their heaviest neighbour (Algorithm 1 line 13);
//     aggregate numbering: exclusive prefix scan over leader flags;
//     Galerkin product I L I^T with the R3 summation order:
//       crossing fine edges -> (coarse pair key, w), stable radix sort,
//       sequential left fold per pair, symmetric CSR assembly;
//     Jones-Plassmann colouring = greedy first-fit colouring in decreasing
//       hash priority (R4);
//     solve layout: rows sorted by (colour, row class, natural id).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <queue>

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
    FDL_CK(cudaMemcpyAsync(&h, fl.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaStreamSynchronize(st));
    FDL_REQUIRE(h == 0, FIEDLER_ERR_GRAPH, "row_ptr is not a valid CSR offset array");
    k_validate<<<grid_for(n), 256, 0, st>>>((int)n, rp32, ci, w, fl.as<int>());
    FDL_LAUNCH_CK();
    FDL_CK(cudaMemcpyAsync(&h, fl.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaStreamSynchronize(st));
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
    FDL_CK(cudaMemcpyAsync(&h, fl.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaStreamSynchronize(st));
    FDL_REQUIRE(h == 0, FIEDLER_ERR_GRAPH, "row_ptr is not a valid CSR offset array");
}

// ================================================================= heavy edge coarsening
// m(v) = heaviest neighbour in the strict order (w, hash); also the first
// handshake pointer.  Vertices with neighbours enter the work list.
template <int W>
__global__ void k_heavy_init(int n, const int *rp, const int *ci, const double *w, uint64_t salt,
                             int *m, int *ptr, int *list, int *count) {
    SUBWARP_LOOP(W, n, v) {
        double bw = 0.0;
        unsigned long long bh = 0;
        int bj = -1;
        if (v < n) {
            for (int k = rp[v] + sw_lane_; k < rp[v + 1]; k += W) {
                int j = ci[k];
                double x = w[k];
                unsigned long long h = edge_hash(salt, (int)v, j);
                if (bj < 0 || x > bw || (x == bw && h > bh)) { bw = x; bh = h; bj = j; }
            }
        }
        argmax_reduce<W>(bw, bh, bj);
        if (v < n && sw_lane_ == 0) {
            m[v] = bj;
            ptr[v] = bj;
        }
        const bool app = v < n && sw_lane_ == 0 && bj >= 0;
        const int slot = warp_append(app, count);
        if (app) list[slot] = (int)v;
    }
}

// handshake: mutual pointers match
__global__ void k_match_mutual(const int *list, const int *count, const int *ptr, int *mate) {
    int cnt = *count;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        int v = list[i];
        int p = ptr[v];
        if (p >= 0 && ptr[p] == v) mate[v] = p;
    }
}

// re-point vertices whose target got matched at their heaviest FREE neighbour
template <int W>
__global__ void k_repoint(const int *list, const int *count, const int *rp, const int *ci,
                          const double *w, uint64_t salt, int *ptr, const int *mate, int *newlist,
                          int *newcount) {
    const int cnt = *count;
    SUBWARP_LOOP(W, cnt, idx) {
        int v = idx < cnt ? list[idx] : -1;
        bool keep = false, rescan = false;
        if (v >= 0 && mate[v] < 0) {
            int p = ptr[v];
            if (mate[p] < 0) keep = true;
            else rescan = true;
        }
        double bw = 0.0;
        unsigned long long bh = 0;
        int bj = -1;
        if (rescan) {
            for (int k = rp[v] + sw_lane_; k < rp[v + 1]; k += W) {
                int j = ci[k];
                if (mate[j] >= 0) continue;
                double x = w[k];
                unsigned long long h = edge_hash(salt, v, j);
                if (bj < 0 || x > bw || (x == bw && h > bh)) { bw = x; bh = h; bj = j; }
            }
        }
        argmax_reduce<W>(bw, bh, bj);
        if (sw_lane_ == 0 && rescan) {
            ptr[v] = bj;
            if (bj >= 0) keep = true;
        }
        const bool app = sw_lane_ == 0 && keep;
        const int slot = warp_append(app, newcount);
        if (app) newlist[slot] = v;
    }
}

__global__ void k_leaders(int n, const int *m, const int *mate, int *leader, int *flag, int *err) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        int L;
        int mv = mate[v];
        if (mv >= 0) L = min(v, mv);
        else if (m[v] >= 0) {
            int u = m[v];
            int mu = mate[u];
            if (mu < 0) { atomicOr(err, 1); mu = u; }   // impossible for a maximal matching
            L = min(u, mu);
        } else L = v;
        leader[v] = L;
        flag[v] = (L == v);
    }
}

__global__ void k_assign(int n, const int *leader, const int *id, int *q) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        q[v] = id[leader[v]];
}

static int read_int(const int *dptr, cudaStream_t st) {
    int h;
    FDL_CK(cudaMemcpyAsync(&h, dptr, sizeof(int), cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaStreamSynchronize(st));
    return h;
}

// Returns the number of aggregates c; fills q (natural), mate.
static int hec_parallel(const NatGraph &g, uint64_t salt, DBuf &q, DBuf &mate, int &rounds,
                        cudaStream_t st) {
    const int n = g.n;
    const double avg = n ? (double)g.nnz / n : 0.0;
    DBuf m((size_t)n * 4, st), ptr((size_t)n * 4, st), la((size_t)n * 4, st), lb((size_t)n * 4, st),
        cnt(2 * sizeof(int), st);
    q.alloc((size_t)n * 4, st);
    mate.alloc((size_t)n * 4, st);
    FDL_CK(cudaMemsetAsync(mate.p, 0xff, (size_t)n * 4, st));
    FDL_CK(cudaMemsetAsync(cnt.p, 0, 2 * sizeof(int), st));
    int *ca = cnt.as<int>(), *cb = cnt.as<int>() + 1;
    DISPATCH_W(avg, (k_heavy_init<W><<<sub_grid(n, W), 256, 0, st>>>(
                         n, g.rp, g.ci, g.w, salt, m.as<int>(), ptr.as<int>(), la.as<int>(), ca)));
    FDL_LAUNCH_CK();
    int *L0 = la.as<int>(), *L1 = lb.as<int>();
    int active = read_int(ca, st);
    rounds = 0;
    while (active > 0) {
        rounds++;
        FDL_REQUIRE(rounds < 100000, FIEDLER_ERR_INTERNAL, "matching did not terminate");
        k_match_mutual<<<grid_for(active), 256, 0, st>>>(L0, ca, ptr.as<int>(), mate.as<int>());
        FDL_LAUNCH_CK();
        FDL_CK(cudaMemsetAsync(cb, 0, sizeof(int), st));
        DISPATCH_W(avg, (k_repoint<W><<<sub_grid(active, W), 256, 0, st>>>(
                             L0, ca, g.rp, g.ci, g.w, salt, ptr.as<int>(), mate.as<int>(), L1, cb)));
        FDL_LAUNCH_CK();
        std::swap(L0, L1);
        std::swap(ca, cb);
        active = read_int(ca, st);
    }
    // leaders, prefix scan numbering
    DBuf leader((size_t)n * 4, st), flag((size_t)n * 4, st), id((size_t)n * 4, st), tot(8, st);
    FDL_CK(cudaMemsetAsync(tot.p, 0, 8, st));
    k_leaders<<<grid_for(n), 256, 0, st>>>(n, m.as<int>(), mate.as<int>(), leader.as<int>(),
                                           flag.as<int>(), tot.as<int>() + 1);
    FDL_LAUNCH_CK();
    scan_exclusive(flag.as<int>(), id.as<int>(), n, tot.as<int>(), st);
    k_assign<<<grid_for(n), 256, 0, st>>>(n, leader.as<int>(), id.as<int>(), q.as<int>());
    FDL_LAUNCH_CK();
    int th[2];
    FDL_CK(cudaMemcpyAsync(th, tot.p, 8, cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaStreamSynchronize(st));
    FDL_REQUIRE(th[1] == 0, FIEDLER_ERR_INTERNAL, "heavy-edge matching is not maximal");
    return th[0];
}

// ================================================================= Galerkin product
template <int W>
__global__ void k_gal_count(int n, const int *rp, const int *ci, const int *q, int *cnt) {
    SUBWARP_LOOP(W, n, i) {
        int c = 0;
        if (i < n) {
            int qi = q[i];
            for (int k = rp[i] + sw_lane_; k < rp[i + 1]; k += W) {
                int j = ci[k];
                c += (j > i && q[j] != qi);
            }
        }
        c = sub_sum<W>(c);
        if (i < n && sw_lane_ == 0) cnt[i] = c;
    }
}

template <int W>
__global__ void k_gal_emit(int n, const int *rp, const int *ci, const double *w, const int *q,
                           const int *off, int bitsB, unsigned long long *keys, double *vals) {
    SUBWARP_LOOP(W, n, i) {
        const unsigned sub_mask = (W == 32) ? 0xffffffffu
                                            : (((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1)));
        int qi = 0, b = 0, e = 0, o = 0;
        if (i < n) { qi = q[i]; b = rp[i]; e = rp[i + 1]; o = off[i]; }
        int len = e - b;
        int maxlen = len;   // warp-wide max: the ballot below needs all 32 lanes
#pragma unroll
        for (int s = 16; s; s >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, s));
        for (int t = 0; t < maxlen; t += W) {   // uniform within the warp
            int k = b + t + sw_lane_;
            bool f = false;
            int j = 0, qj = 0;
            if (t + sw_lane_ < len) {
                j = ci[k];
                qj = q[j];
                f = (j > i && qj != qi);
            }
            unsigned bal = __ballot_sync(0xffffffffu, f) & sub_mask;
            if (f) {
                int rank = __popc(bal & ((1u << (threadIdx.x & 31)) - 1u));
                unsigned A = min(qi, qj), B = max(qi, qj);
                keys[o + rank] = ((unsigned long long)A << bitsB) | B;
                vals[o + rank] = w[k];
            }
            o += __popc(bal);
        }
    }
}

__global__ void k_run_heads(const unsigned long long *keys, int E, int *head) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < E; t += gridDim.x * blockDim.x)
        head[t] = (t == 0 || keys[t] != keys[t - 1]);
}

// sequential left fold of each run (R3 order = the stable-sorted visit order)
__global__ void k_run_fold(const unsigned long long *keys, const double *vals, int E,
                           const int *head, const int *runid, int bitsB, int *pA, int *pB,
                           double *pw) {
    const unsigned long long maskB = (1ull << bitsB) - 1ull;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < E; t += gridDim.x * blockDim.x) {
        if (!head[t]) continue;
        double s = vals[t];
        for (int u = t + 1; u < E && !head[u]; u++) s += vals[u];
        int r = runid[t];
        unsigned long long k = keys[t];
        pA[r] = (int)(k >> bitsB);
        pB[r] = (int)(k & maskB);
        pw[r] = s;
    }
}

__global__ void k_pair_counts(int P, const int *pA, const int *pB, int *upcnt, int *lowcnt,
                              int *firstA) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < P; r += gridDim.x * blockDim.x) {
        atomicAdd(&upcnt[pA[r]], 1);
        atomicAdd(&lowcnt[pB[r]], 1);
        if (r == 0 || pA[r] != pA[r - 1]) firstA[pA[r]] = r;
    }
}

__global__ void k_add(int n, const int *a, const int *b, int *out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = a[i] + b[i];
}

__global__ void k_fill_upper(int P, const int *pA, const int *pB, const double *pw, const int *crp,
                             const int *lowcnt, const int *firstA, int *cci, double *cw) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < P; r += gridDim.x * blockDim.x) {
        int A = pA[r];
        int pos = crp[A] + lowcnt[A] + (r - firstA[A]);
        cci[pos] = pB[r];
        cw[pos] = pw[r];
    }
}

__global__ void k_pairs_by_B(int P, const int *pB, unsigned *keys, int *vals) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < P; r += gridDim.x * blockDim.x) {
        keys[r] = (unsigned)pB[r];
        vals[r] = r;
    }
}

__global__ void k_first_of_runs_u32(int P, const unsigned *keys, int *first) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < P; t += gridDim.x * blockDim.x)
        if (t == 0 || keys[t] != keys[t - 1]) first[keys[t]] = t;
}

__global__ void k_fill_lower(int P, const unsigned *sB, const int *sr, const int *pA,
                             const double *pw, const int *crp, const int *firstB, int *cci,
                             double *cw) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < P; t += gridDim.x * blockDim.x) {
        int B = (int)sB[t];
        int r = sr[t];
        int pos = crp[B] + (t - firstB[B]);
        cci[pos] = pA[r];
        cw[pos] = pw[r];
    }
}

static NatGraph galerkin(const NatGraph &g, const int *q, int c, cudaStream_t st) {
    const int n = g.n;
    const double avg = n ? (double)g.nnz / n : 0.0;
    const int bitsB = bits_for(c - 1);
    DBuf cnt((size_t)n * 4, st), off((size_t)n * 4, st), tot(4, st);
    DISPATCH_W(avg, (k_gal_count<W><<<sub_grid(n, W), 256, 0, st>>>(n, g.rp, g.ci, q, cnt.as<int>())));
    FDL_LAUNCH_CK();
    scan_exclusive(cnt.as<int>(), off.as<int>(), n, tot.as<int>(), st);
    const int E = read_int(tot.as<int>(), st);
    NatGraph out;
    out.n = c;
    out.own_rp.alloc((size_t)(c + 1) * 4, st);
    if (E == 0) {
        FDL_CK(cudaMemsetAsync(out.own_rp.p, 0, (size_t)(c + 1) * 4, st));
        out.nnz = 0;
        out.rp = out.own_rp.as<int>();
        return out;
    }
    DBuf keys((size_t)E * 8, st), vals((size_t)E * 8, st);
    DISPATCH_W(avg, (k_gal_emit<W><<<sub_grid(n, W), 256, 0, st>>>(
                         n, g.rp, g.ci, g.w, q, off.as<int>(), bitsB,
                         keys.as<unsigned long long>(), vals.as<double>())));
    FDL_LAUNCH_CK();
    radix_sort_u64_f64(keys.as<unsigned long long>(), vals.as<double>(), E, 2 * bitsB, st);
    DBuf head((size_t)E * 4, st), runid((size_t)E * 4, st);
    k_run_heads<<<grid_for(E), 256, 0, st>>>(keys.as<unsigned long long>(), E, head.as<int>());
    FDL_LAUNCH_CK();
    scan_exclusive(head.as<int>(), runid.as<int>(), E, tot.as<int>(), st);
    const int P = read_int(tot.as<int>(), st);
    DBuf pA((size_t)P * 4, st), pB((size_t)P * 4, st), pw((size_t)P * 8, st);
    k_run_fold<<<grid_for(E), 256, 0, st>>>(keys.as<unsigned long long>(), vals.as<double>(), E,
                                            head.as<int>(), runid.as<int>(), bitsB, pA.as<int>(),
                                            pB.as<int>(), pw.as<double>());
    FDL_LAUNCH_CK();
    keys.release(); vals.release(); head.release(); runid.release();
    DBuf upcnt((size_t)c * 4, st), lowcnt((size_t)c * 4, st), firstA((size_t)c * 4, st),
        rowcnt((size_t)c * 4, st);
    FDL_CK(cudaMemsetAsync(upcnt.p, 0, (size_t)c * 4, st));
    FDL_CK(cudaMemsetAsync(lowcnt.p, 0, (size_t)c * 4, st));
    k_pair_counts<<<grid_for(P), 256, 0, st>>>(P, pA.as<int>(), pB.as<int>(), upcnt.as<int>(),
                                               lowcnt.as<int>(), firstA.as<int>());
    FDL_LAUNCH_CK();
    k_add<<<grid_for(c), 256, 0, st>>>(c, upcnt.as<int>(), lowcnt.as<int>(), rowcnt.as<int>());
    FDL_LAUNCH_CK();
    scan_exclusive(rowcnt.as<int>(), out.own_rp.as<int>(), c, out.own_rp.as<int>() + c, st);
    out.nnz = 2 * P;
    out.own_ci.alloc((size_t)out.nnz * 4, st);
    out.own_w.alloc((size_t)out.nnz * 8, st);
    k_fill_upper<<<grid_for(P), 256, 0, st>>>(P, pA.as<int>(), pB.as<int>(), pw.as<double>(),
                                              out.own_rp.as<int>(), lowcnt.as<int>(),
                                              firstA.as<int>(), out.own_ci.as<int>(),
                                              out.own_w.as<double>());
    FDL_LAUNCH_CK();
    DBuf sB((size_t)P * 4, st), sr((size_t)P * 4, st), firstB((size_t)c * 4, st);
    k_pairs_by_B<<<grid_for(P), 256, 0, st>>>(P, pB.as<int>(), sB.as<unsigned>(), sr.as<int>());
    FDL_LAUNCH_CK();
    radix_sort_u32_i32(sB.as<unsigned>(), sr.as<int>(), P, bitsB, st);
    k_first_of_runs_u32<<<grid_for(P), 256, 0, st>>>(P, sB.as<unsigned>(), firstB.as<int>());
    FDL_LAUNCH_CK();
    k_fill_lower<<<grid_for(P), 256, 0, st>>>(P, sB.as<unsigned>(), sr.as<int>(), pA.as<int>(),
                                              pw.as<double>(), out.own_rp.as<int>(),
                                              firstB.as<int>(), out.own_ci.as<int>(),
                                              out.own_w.as<double>());
    FDL_LAUNCH_CK();
    out.rp = out.own_rp.as<int>();
    out.ci = out.own_ci.as<int>();
    out.w = out.own_w.as<double>();
    return out;
}

// ================================================================= colouring (R4)
__device__ __forceinline__ bool higher_prio(uint64_t pu, int u, uint64_t pv, int v) {
    return pu > pv || (pu == pv && u > v);
}

template <int W>
__global__ void k_color_round(const int *list, const int *count, const int *rp, const int *ci,
                              uint64_t salt, int *color, int *newlist, int *newcount) {
    const int cnt = *count;
    volatile int *vcolor = color;
    SUBWARP_LOOP(W, cnt, idx) {
        int v = idx < cnt ? list[idx] : -1;
        int notready = 0;
        unsigned long long mask = 0ull;
        int big = 0;
        uint64_t pv = 0;
        int b = 0, e = 0;
        if (v >= 0) {
            pv = splitmix64(salt ^ (uint64_t)v);
            b = rp[v];
            e = rp[v + 1];
            for (int k = b + sw_lane_; k < e; k += W) {
                int u = ci[k];
                if (!higher_prio(splitmix64(salt ^ (uint64_t)u), u, pv, v)) continue;
                int cu = vcolor[u];
                if (cu < 0) notready = 1;
                else if (cu < 64) mask |= 1ull << cu;
                else big = 1;
            }
        }
#pragma unroll
        for (int o = W / 2; o; o >>= 1) {
            notready |= __shfl_xor_sync(0xffffffffu, notready, o, W);
            big |= __shfl_xor_sync(0xffffffffu, big, o, W);
            mask |= __shfl_xor_sync(0xffffffffu, mask, o, W);
        }
        int col = -1;
        if (v >= 0 && !notready) {
            if (~mask) col = __ffsll((long long)~mask) - 1;
        }
        // rare: all of 0..63 taken -> scan further windows (sub-warp cooperative)
        int need_big = (v >= 0 && !notready && col < 0) ? 1 : 0;
        int any_big = __any_sync(0xffffffffu, need_big);   // warp-uniform loop below
        for (int wb = 64; any_big; wb += 64) {
            unsigned long long m2 = 0ull;
            if (need_big)
                for (int k = b + sw_lane_; k < e; k += W) {
                    int u = ci[k];
                    if (!higher_prio(splitmix64(salt ^ (uint64_t)u), u, pv, v)) continue;
                    int cu = vcolor[u];
                    if (cu >= wb && cu < wb + 64) m2 |= 1ull << (cu - wb);
                }
#pragma unroll
            for (int o = W / 2; o; o >>= 1) m2 |= __shfl_xor_sync(0xffffffffu, m2, o, W);
            if (need_big && ~m2) { col = wb + __ffsll((long long)~m2) - 1; need_big = 0; }
            any_big = __any_sync(0xffffffffu, need_big);
        }
        (void)big;
        if (v >= 0 && sw_lane_ == 0 && !notready) vcolor[v] = col;
        const bool app = v >= 0 && sw_lane_ == 0 && notready;
        const int slot = warp_append(app, newcount);
        if (app) newlist[slot] = v;
    }
}

__global__ void k_iota(int n, int *a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

static int color_graph(const NatGraph &g, uint64_t salt, DBuf &color, int &rounds, cudaStream_t st) {
    const int n = g.n;
    const double avg = n ? (double)g.nnz / n : 0.0;
    color.alloc((size_t)n * 4, st);
    FDL_CK(cudaMemsetAsync(color.p, 0xff, (size_t)n * 4, st));
    DBuf la((size_t)n * 4, st), lb((size_t)n * 4, st), cnt(8, st);
    k_iota<<<grid_for(n), 256, 0, st>>>(n, la.as<int>());
    FDL_LAUNCH_CK();
    int *ca = cnt.as<int>(), *cb = cnt.as<int>() + 1;
    FDL_CK(cudaMemcpyAsync(ca, &n, sizeof(int), cudaMemcpyHostToDevice, st));
    int *L0 = la.as<int>(), *L1 = lb.as<int>();
    int active = n;
    rounds = 0;
    while (active > 0) {
        rounds++;
        FDL_REQUIRE(rounds < 1000000, FIEDLER_ERR_INTERNAL, "colouring did not terminate");
        FDL_CK(cudaMemsetAsync(cb, 0, sizeof(int), st));
        DISPATCH_W(avg, (k_color_round<W><<<sub_grid(active, W), 256, 0, st>>>(
                             L0, ca, g.rp, g.ci, salt, color.as<int>(), L1, cb)));
        FDL_LAUNCH_CK();
        std::swap(L0, L1);
        std::swap(ca, cb);
        active = read_int(ca, st);
    }
    DBuf mx(4, st);
    reduce_max_i32(color.as<int>(), n, mx.as<int>(), st);
    return read_int(mx.as<int>(), st) + 1;
}

// ================================================================= solve layout
__global__ void k_color_keys(int n, const int *color, unsigned *keys, int *vals) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        keys[v] = (unsigned)color[v];
        vals[v] = v;
    }
}

__global__ void k_seg_starts(int n, const unsigned *keys, int *segstart) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        if (t == 0 || keys[t] != keys[t - 1]) segstart[keys[t]] = t;
}

__global__ void k_inv_and_deg(int n, const int *perm, const int *rp, int *inv, int *degp) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        int v = perm[t];
        inv[v] = t;
        degp[t] = rp[v + 1] - rp[v];
    }
}

// GS layout rows: row t = natural row perm[t], columns renumbered by inv, order kept
template <int W>
__global__ void k_permute_rows(int n, const int *perm, const int *inv, const int *rp, const int *ci,
                               const double *w, const int *rpp, int *cip, double *wp) {
    SUBWARP_LOOP(W, n, t) {
        if (t < n) {
            int v = perm[t];
            int b = rp[v], e = rp[v + 1], o = rpp[t];
            for (int k = sw_lane_; k < e - b; k += W) {
                cip[o + k] = inv[ci[b + k]];
                wp[o + k] = w[b + k];
            }
        }
    }
}

// PI/RQ layout: natural rows, columns renumbered by inv (a pure stream)
__global__ void k_renumber_cols(int nnz, const int *inv, const int *ci, const double *w, int *cin,
                                double *wn) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += gridDim.x * blockDim.x) {
        cin[k] = inv[ci[k]];
        wn[k] = w[k];
    }
}

__global__ void k_copy_i32(int n, const int *a, int *b) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = a[i];
}

// max_i d_i with d_i summed in stored (= natural ascending) order, as the oracle
__global__ void k_degree_max(int n, const int *rp, const double *w, unsigned long long *dmax) {
    double m = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = rp[i]; k < rp[i + 1]; k++) s += w[k];
        m = fmax(m, s);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane_id() == 0) atomicMax(dmax, (unsigned long long)__double_as_longlong(m));
}

__global__ void k_gather_i32(int k, const int *src, const int *idx, int *out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
        out[i] = src[idx[i]];
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

static int tiles_for(long long coord_span) { return std::max(1, (int)((coord_span + kTileT - 1) / kTileT)); }

static void build_layout(const NatGraph &g, const int *color_nat, int ncolors, Level &L,
                         cudaStream_t st) {
    const int n = g.n;
    const double avg = n ? (double)g.nnz / n : 0.0;
    L.n = n;
    L.nnz = g.nnz;
    L.ncolors = ncolors;
    // ---- GS layout: rows sorted (stably) by colour
    DBuf keys((size_t)n * 4, st);
    L.perm.alloc((size_t)n * 4, st);
    k_color_keys<<<grid_for(n), 256, 0, st>>>(n, color_nat, keys.as<unsigned>(), L.perm.as<int>());
    FDL_LAUNCH_CK();
    radix_sort_u32_i32(keys.as<unsigned>(), L.perm.as<int>(), n, bits_for(ncolors - 1), st);
    DBuf segstart((size_t)(ncolors + 1) * 4, st);
    FDL_CK(cudaMemsetAsync(segstart.p, 0xff, (size_t)(ncolors + 1) * 4, st));
    k_seg_starts<<<grid_for(n), 256, 0, st>>>(n, keys.as<unsigned>(), segstart.as<int>());
    FDL_LAUNCH_CK();
    keys.release();
    L.inv.alloc((size_t)n * 4, st);
    DBuf degp((size_t)n * 4, st);
    k_inv_and_deg<<<grid_for(n), 256, 0, st>>>(n, L.perm.as<int>(), g.rp, L.inv.as<int>(), degp.as<int>());
    FDL_LAUNCH_CK();
    L.rp.alloc((size_t)(n + 1) * 4 + kPadBytes, st);
    scan_exclusive(degp.as<int>(), L.rp.as<int>(), n, L.rp.as<int>() + n, st);
    degp.release();
    const size_t ci_bytes = (size_t)std::max(g.nnz, 1) * 4 + kPadBytes;
    const size_t w_bytes = (size_t)std::max(g.nnz, 1) * 8 + kPadBytes;
    L.ci.alloc(ci_bytes, st);
    L.w.alloc(w_bytes, st);
    DISPATCH_W(avg, (k_permute_rows<W><<<sub_grid(n, W), 256, 0, st>>>(
                         n, L.perm.as<int>(), L.inv.as<int>(), g.rp, g.ci, g.w, L.rp.as<int>(),
                         L.ci.as<int>(), L.w.as<double>())));
    FDL_LAUNCH_CK();
    // ---- PI/RQ layout: natural rows, solve-numbered columns
    L.rpN.alloc((size_t)(n + 1) * 4 + kPadBytes, st);
    L.ciN.alloc(ci_bytes, st);
    L.wN.alloc(w_bytes, st);
    k_copy_i32<<<grid_for(n + 1), 256, 0, st>>>(n + 1, g.rp, L.rpN.as<int>());
    FDL_LAUNCH_CK();
    if (g.nnz) {
        k_renumber_cols<<<grid_for(g.nnz, 256, kNumSMs * 16), 256, 0, st>>>(
            g.nnz, L.inv.as<int>(), g.ci, g.w, L.ciN.as<int>(), L.wN.as<double>());
        FDL_LAUNCH_CK();
    }
    DBuf dmax(8, st);
    FDL_CK(cudaMemsetAsync(dmax.p, 0, 8, st));
    k_degree_max<<<grid_for(n, 256, kNumSMs * 8), 256, 0, st>>>(n, g.rp, g.w,
                                                               dmax.as<unsigned long long>());
    FDL_LAUNCH_CK();

    // colour segment boundaries and their nonzero offsets -> host
    std::vector<int> seg(ncolors + 1);
    FDL_CK(cudaMemcpyAsync(seg.data(), segstart.p, (size_t)(ncolors + 1) * 4, cudaMemcpyDeviceToHost, st));
    double dm = 0.0;
    FDL_CK(cudaMemcpyAsync(&dm, dmax.p, 8, cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaStreamSynchronize(st));
    L.shift = 2.0 * dm;
    seg[ncolors] = n;
    for (int k = ncolors - 1; k >= 0; k--)
        if (seg[k] < 0) seg[k] = seg[k + 1];
    DBuf sidx((size_t)(ncolors + 1) * 4, st), sval((size_t)(ncolors + 1) * 4, st);
    FDL_CK(cudaMemcpyAsync(sidx.p, seg.data(), (size_t)(ncolors + 1) * 4, cudaMemcpyHostToDevice, st));
    k_gather_i32<<<1, 256, 0, st>>>(ncolors + 1, L.rp.as<int>(), sidx.as<int>(), sval.as<int>());
    FDL_LAUNCH_CK();
    std::vector<int> segnnz(ncolors + 1);
    FDL_CK(cudaMemcpyAsync(segnnz.data(), sval.p, (size_t)(ncolors + 1) * 4, cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaStreamSynchronize(st));

    // tiles: GS colours, then the natural-order pass
    L.ctile.assign(ncolors + 1, 0);
    int nt = 0;
    std::vector<int> cnt(ncolors + 1);
    for (int c = 0; c < ncolors; c++) {
        L.ctile[c] = nt;
        long long span = (long long)(segnnz[c + 1] + seg[c + 1]) - (segnnz[c] + seg[c]);
        cnt[c] = seg[c + 1] > seg[c] ? tiles_for(span) : 0;
        nt += cnt[c];
    }
    L.ctile[ncolors] = nt;
    cnt[ncolors] = tiles_for((long long)g.nnz + n);
    nt += cnt[ncolors];
    L.ntiles = nt;
    L.tiles.alloc((size_t)nt * sizeof(Tile), st);
    for (int c = 0; c < ncolors; c++)
        if (cnt[c]) {
            k_make_tiles<<<grid_for(cnt[c]), 256, 0, st>>>(L.rp.as<int>(), seg[c], seg[c + 1], cnt[c],
                                                           L.tiles.as<Tile>() + L.ctile[c]);
            FDL_LAUNCH_CK();
        }
    k_make_tiles<<<grid_for(cnt[ncolors]), 256, 0, st>>>(L.rpN.as<int>(), 0, n, cnt[ncolors],
                                                         L.tiles.as<Tile>() + L.ctile[ncolors]);
    FDL_LAUNCH_CK();
}

// ================================================================= connectivity (coarsest level)
static bool coarsest_connected(const Level &L, cudaStream_t st) {
    std::vector<int> rp(L.n + 1), ci(std::max(L.nnz, 1));
    FDL_CK(cudaMemcpyAsync(rp.data(), L.rp.p, (size_t)(L.n + 1) * 4, cudaMemcpyDeviceToHost, st));
    if (L.nnz) FDL_CK(cudaMemcpyAsync(ci.data(), L.ci.p, (size_t)L.nnz * 4, cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaStreamSynchronize(st));
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

__global__ void k_compose_qp(int n, const int *perm, const int *q_nat, const int *inv_coarse, int *qp) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        qp[t] = inv_coarse[q_nat[perm[t]]];
}

void build_hierarchy(Handle &h, NatGraph &&g0) {
    cudaStream_t st = h.stream;
    const fiedler_opts &o = h.opts;
    NatGraph cur = std::move(g0);
    h.levels.clear();
    for (int ell = 0;; ell++) {
        Level L;
        bool coarsen = cur.n > o.coarsest_size && ell + 1 < o.max_levels;
        NatGraph next;
        if (coarsen) {
            int c = hec_parallel(cur, salt_match(o.seed, ell), L.q_nat, L.mate_nat, L.match_rounds, st);
            // stall guard (R9): stop when HEC no longer shrinks the graph
            if ((double)c > 0.95 * (double)cur.n || c < 2) {
                coarsen = false;
                L.q_nat.release();
                L.mate_nat.release();
            } else {
                next = galerkin(cur, L.q_nat.as<int>(), c, st);
            }
        }
        int ncol = color_graph(cur, salt_color(o.seed, ell), L.color_nat, L.color_rounds, st);
        build_layout(cur, L.color_nat.as<int>(), ncol, L, st);
        h.levels.push_back(std::move(L));
        if (!coarsen) break;
        cur = std::move(next);
    }
    const int J = (int)h.levels.size() - 1;
    for (int ell = 0; ell < J; ell++) {
        Level &L = h.levels[ell];
        L.qp.alloc((size_t)L.n * 4, st);
        k_compose_qp<<<grid_for(L.n), 256, 0, st>>>(L.n, L.perm.as<int>(), L.q_nat.as<int>(),
                                                    h.levels[ell + 1].inv.as<int>(), L.qp.as<int>());
        FDL_LAUNCH_CK();
    }
    FDL_CK(cudaStreamSynchronize(st));
    if (!coarsest_connected(h.levels[J], st))
        throw Error(FIEDLER_ERR_DISCONNECTED,
                    "graph is disconnected (lambda_2 = 0): the coarsest level splits into components");
}

}  // namespace fdl

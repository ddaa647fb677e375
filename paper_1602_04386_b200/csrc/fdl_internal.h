// fdl_internal.h -- host-side data structures of libfiedler.
//
// Device data layout:
//   setup works on the NATURAL numbering of every level (the oracle's);
//   the solve works on a per-level SOLVE LAYOUT: rows permuted by
//   (colour, row class, natural id) so that every colour class of the
//   multicolour Gauss-Seidel is a contiguous row range, and within it the
//   short / medium / long rows are contiguous (different kernels' work items).
#pragma once

#include <vector>

#include "fdl_common.cuh"

namespace fdl {

// Row classes of the solve layout (by adjacency nonzeros of the row).
constexpr int kShortMax = 32;    // class 0: staged through shared-memory tiles
constexpr int kMediumMax = 1024; // class 1: one warp per row; class 2: one CTA per row
constexpr int kNumKinds = 3;
constexpr int kTileNnz = 2048;   // nonzeros per short-row tile (target)
constexpr int kTileCap = kTileNnz + kShortMax;
constexpr int kRowsPerMedItem = 8;

// A work item of the row-pass kernels: x = kind, y = first row, z = end row.
using Item = int4;

// Natural-numbering CSR of one level during setup.
struct NatGraph {
    int n = 0;
    int nnz = 0;
    const int *rp = nullptr;     // int32 [n+1]
    const int *ci = nullptr;     // int32 [nnz]
    const double *w = nullptr;   // f64  [nnz]
    DBuf own_rp, own_ci, own_w;  // storage when owned by the library
};

struct Level {
    int n = 0, nnz = 0;
    // solve layout
    DBuf rp, ci, w;          // permuted CSR (columns in permuted numbering, order kept)
    DBuf perm;               // int32 [n]: solve row -> natural id
    DBuf inv;                // int32 [n]: natural id -> solve row
    DBuf qp;                 // int32 [n]: solve row -> solve row of its aggregate on level+1
    // natural-numbering setup results kept for fiedler_level_export
    DBuf q_nat, mate_nat, color_nat;
    // work items: all colours back to back; colour c owns [citem[c], citem[c+1])
    DBuf items;
    std::vector<int> citem;
    int ncolors = 0;
    int nitems = 0;
    int max_item_rows = 0;
    double shift = 0.0;      // c of c I - L: 2 max_i d_i (R8)
    int match_rounds = 0;
    int color_rounds = 0;
};

struct Handle {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    fiedler_opts opts{};
    std::vector<Level> levels;
    int n0 = 0;
    // solve state
    DBuf xa, xb;             // level vectors (sized n0)
    DBuf vnat;               // result in natural numbering (n0)
    DBuf scal;               // scalar slots (4 doubles each)
    int nslots = 0;
    DBuf partials;           // per-CTA partial sums
    DBuf counter;            // last-CTA counter
    DBuf result;             // {lambda2, residual, ...} (device)
    int row_grid = kNumSMs * 8;   // CTAs of a row pass
    double setup_ms = 0.0;
    int setup_launches = 0;
    // captured solve graph and the options it was captured with
    cudaGraphExec_t gexec = nullptr;
    int g_gs = -1, g_pi = -1, g_piJ = -1;
    uint64_t g_seed = 0;
    int g_launches = 0;
    ~Handle();
};

// fdl_setup.cu
void validate_input(int64_t n, int64_t nnz, const int *rp32, const int *ci, const double *w,
                    cudaStream_t st);
void build_hierarchy(Handle &h, NatGraph &&g0);

// fdl_solve.cu
struct SolveCfg {
    int gs, pi, piJ;
    uint64_t seed;
};
// Enqueue the whole solve on h.stream; returns the number of kernel launches.
int enqueue_solve(Handle &h, const SolveCfg &cfg);
// Single-operation entry (fiedler_level_apply); vectors in solve numbering on device.
void apply_level_op(Handle &h, int level, int op, int count, const double *x_in, double *x_out,
                    double *scal_host);
// fiedler_level_time: CUDA-event timing of `reps` back-to-back row passes
void time_level_op(Handle &h, int level, int op, int reps, double *ms_per_rep, double *bytes_per_rep);

}  // namespace fdl

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

// Tile decomposition of the row passes.  A tile is a
// run of consecutive rows whose "coordinate" rp[r] + r starts inside a window
// of kTileT units, so a tile holds at most kTileT rows and its short rows
// (<= kShortMax nonzeros) end within kTileT + kShortMax nonzeros of the tile's
// first nonzero: that range is staged into shared memory by bulk copies.
constexpr int kShortMax = 32;    // longer rows are reduced by a warp from global memory
#ifndef FDL_TILE_T
#define FDL_TILE_T 1024
#endif
#ifndef FDL_STAGES
#define FDL_STAGES 2
#endif
#ifndef FDL_PASS_MINB
#define FDL_PASS_MINB 8
#endif
constexpr int kTileT = FDL_TILE_T;    // coordinate window per tile
constexpr int kStages = FDL_STAGES;   // depth of the bulk-copy pipeline of a row pass
constexpr int kStageCap = kTileT + kShortMax;
constexpr int kPadBytes = 64;    // slack after every staged array (bulk copies round up to 16 B)

// A tile: x = first row, y = end row (exclusive).
using Tile = int2;

// Natural-numbering CSR of one level during setup.
struct NatGraph {
    int n = 0;
    int nnz = 0;
    const int *rp = nullptr;     // int32 [n+1]
    const int *ci = nullptr;     // int32 [nnz]
    const double *w = nullptr;   // f64  [nnz]
    DBuf own_rp, own_ci, own_w;  // storage when owned by the library
};

// Row partition of one level for the partitioned solve (fiedler_dist_plan).
struct DistPlan {
    bool valid = false;
    int nranks = 1, rank = 0;
    int r0 = 0, r1 = 0;                  // own natural rows
    std::vector<int64_t> bounds;         // [nranks + 1] natural row bounds of every rank
    DBuf tilesN;                         // own natural tiles (PI / RQ)
    int ntN = 0;
    DBuf tilesGS;                        // own GS tiles, colour c at [ctile[c], ctile[c+1])
    std::vector<int> ctile;
    DBuf send_idx, recv_idx;             // natural ids, peer-major, ascending within a peer
    std::vector<int64_t> send_cnt, recv_cnt;
    int send_total = 0, recv_total = 0;
};

struct Level {
    int n = 0, nnz = 0;
    // GS layout: rows sorted by (colour, natural id); every colour is one
    // contiguous row range; columns in solve numbering (= GS row order).
    DBuf rp, ci, w;
    // PI / RQ layout: the level's natural CSR itself (natural rows and columns;
    // vectors of the power iteration live in natural numbering).
    DBuf rpN, ciN, wN;
    DBuf perm;               // int32 [n]: GS row -> natural id
    DBuf inv;                // int32 [n]: natural id -> GS row
    DBuf qg;                 // int32 [n]: GS row -> natural id of its aggregate on level+1
    // natural-numbering setup results kept for fiedler_level_export
    DBuf q_nat, mate_nat, color_nat;
    // tiles: GS tiles of all colours back to back (colour c owns
    // [ctile[c], ctile[c+1])), then the natural-order tiles [ctile[ncolors], ntiles)
    DBuf tiles;
    std::vector<int> ctile;
    std::vector<int> seg;    // [ncolors + 1] GS row range of every colour
    DBuf seg_d;              // device copy of seg
    int gs_tail_c0 = 0;      // colours [gs_tail_c0, ncolors) run in one single-CTA launch
    std::vector<int> gs_runs;  // GS schedule of one sweep: (c_begin, c_end, kind) triplets,
                               // kind 0 = grid tile pass of one colour, 1 / 2 = k_gs_multi
                               // cluster / single-CTA run, 3 / 4 = k_gs_pieces cluster / single-CTA run
    // hub rows (> kTileT entries): piece tiles at the end of their pass's tile
    // range; hubs of colour c at [hoff[c], hoff[c+1]), of the natural pass at
    // [hoff[ncolors], hoff[ncolors+1]) (empty hoff: no hubs)
    DBuf hubs;               // int4 {row, first piece tile (pass-relative), pieces, 0}
    std::vector<int> hoff;
    DBuf hub_part;           // double2 per tile of the largest pass
    DBuf gd_pieces;          // int4 pieces of the GS rows (build_gs_pieces), when a run uses them
    DBuf gd_parts;           // [ncolors][kGdParts + 1] piece index bounds
    DistPlan dist;
    int ncolors = 0;
    int ntiles = 0;
    double shift = 0.0;      // c of c I - L: 2 max_i d_i, 3 max_i d_i when n == 2 (R8)
    int match_rounds = 0;
    int color_rounds = 0;
    // FIEDLER_PHASE_TIMES=1: device ms of the setup phases (match, Galerkin, colour, layout)
    double phase_ms[4] = {0.0, 0.0, 0.0, 0.0};
    int gs_tile_begin(int c) const { return ctile[c]; }
    int nat_tile_begin() const { return ctile[ncolors]; }
};

// The streams and events of a handle come from a per-device pool and go back
// to it at fiedler_destroy (fdl_api.cu): creating and destroying them for
// every handle cost up to tens of milliseconds now and then (driver work).
// helper threads / side streams of the setup (colourings and layouts of the
// levels = k mod kSides on side stream k; build knob FDL_SIDES)
#ifndef FDL_SIDES
#define FDL_SIDES 2
#endif
constexpr int kMaxSides = 4;
constexpr int kSides = FDL_SIDES < 1 ? 1 : FDL_SIDES > kMaxSides ? kMaxSides : FDL_SIDES;
struct StreamSet {
    cudaStream_t stream = nullptr;    // the handle's stream
    cudaStream_t stream2 = nullptr;   // setup: colourings beside the coarsening chain (levels = 0 mod kSides)
    cudaStream_t side[kMaxSides] = {};   // setup: side[0] = stream2, side[k] the levels = k mod kSides
    cudaEvent_t ev[4] = {};           // 0: join, 1: pattern, 2: setup scratch, 3: spare (no timing)
    cudaEvent_t sev[kMaxSides] = {};  // joins of the side streams
    cudaEvent_t tev[2] = {};          // timing events of create / solve
};

struct Handle {
    int device = 0;
    StreamSet set;                    // from the pool, returned by ~Handle
    cudaStream_t stream = nullptr;
    bool own_stream = false;          // always true: the handle owns `stream` (fdl_api.cu)
    cudaStream_t stream2 = nullptr;   // setup: colourings overlapped with the coarsening chain
    cudaEvent_t ev_pattern = nullptr; // host input: level-0 pattern (rp, ci) on the device
    cudaEvent_t ev_join = nullptr;    // joins a caller's stream with `stream` (fdl_api.cu StreamJoin)
    SmallArena arena;                 // small buffers of the create (fdl_common.cuh); freed last
    fiedler_opts opts{};
    std::vector<Level> levels;
    // fiedler_create_preset: levels 0..preset.size()-1 copied from these
    // (matching, aggregates, colouring, next level) instead of computed
    std::vector<fiedler_preset_level> preset;
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
    int solves_same = 0;      // solves so far with the configuration in g_* (the first runs eagerly)
    ~Handle();
};

// fdl_setup.cu
void validate_input(int64_t n, int64_t nnz, const int *rp32, const int *ci, const double *w,
                    cudaStream_t st);
void build_hierarchy(Handle &h, NatGraph &&g0);
// allocation size of an array that the row passes stage with bulk copies
inline size_t padded(size_t bytes) { return bytes + kPadBytes; }

// fdl_solve.cu
// piece lists of the small-colour GS kernel (fdl_solve.cu k_gs_pieces)
#ifndef FDL_GS_PIECES
#define FDL_GS_PIECES 1
#endif
constexpr int kGdPiece = 256;    // entries of one warp-strided piece (8 per lane)
constexpr int kGdGroup = 32;     // consecutive rows of one colour packed lane per row ...
constexpr int kGdShort = 32;     // ... when none has more entries than this
constexpr int kGdParts = 16;     // parts per colour (CTA shares of a 16-CTA cluster)
constexpr int kGdSlotCapHost = 2048;
constexpr int kGdMaxRunColours = 1024;   // colours of one k_gs_pieces launch
// pieces and parts of the colours with use[c] != 0 (the others get empty part ranges)
void build_gs_pieces(Level &L, const std::vector<int> &seg, const std::vector<int> &segnnz,
                     const std::vector<char> &use, cudaStream_t st);
struct SolveCfg {
    int gs, pi, piJ;
    uint64_t seed;
};
// Enqueue the whole solve on h.stream; returns the number of kernel launches.
int enqueue_solve(Handle &h, const SolveCfg &cfg);
// Single-operation entry (fiedler_level_apply); vectors in solve numbering on device.
void apply_level_op(Handle &h, int level, int op, int count, const double *x_in, double *x_out,
                    double *scal_host);
// partitioned solve (fiedler_dist_plan / fiedler_dist_op)
void dist_plan(Handle &h, int level, int nranks, int rank, fiedler_dist_plan_info *info);
void dist_op(Handle &h, int level, int op, int64_t arg, const double *x, double *y, double *stat,
             const double *stat_in, const double *sign_slot, cudaStream_t st);
// fiedler_level_time: CUDA-event timing of `reps` back-to-back row passes
void time_level_op(Handle &h, int level, int op, int reps, double *ms_per_rep, double *bytes_per_rep);


// error translation of the extern "C" entry points (fdl_api.cu, fdl_pset.cu)
void set_error(const std::string &m);
}  // namespace fdl

#define API_BEGIN try {
#define API_END                                                  \
    }                                                            \
    catch (const fdl::Error &e) {                                \
        fdl::set_error(e.what());                                \
        return e.code;                                           \
    }                                                            \
    catch (const std::bad_alloc &) {                             \
        fdl::set_error("host allocation failed");                \
        return FIEDLER_ERR_NOMEM;                                \
    }                                                            \
    catch (const std::exception &e) {                            \
        fdl::set_error(e.what());                                \
        return FIEDLER_ERR_INTERNAL;                             \
    }

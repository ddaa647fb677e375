/*
 * fiedler.h -- C ABI of the B200-native cascadic-multigrid Fiedler solver
 * (libfiedler.so, package paper_1602_04386_b200).
 *
 * Method: Gandhi, "Improvement of the Cascadic Multigrid Algorithm with a
 * Gauss Seidel Smoother to Efficiently Compute the Fiedler Vector of a Graph
 * Laplacian", arXiv 1602.04386.  "PAPER.md:NN" cites a line of the paper text,
 * "R<k>" a reading of the paper listed in DESIGN.md section 3.
 *
 *   fiedler_create   Algorithm 3 Step 1, Setup Phase:
 *                    repeated heavy edge coarsening (Algorithm 1, PAPER.md:49-74,
 *                    parallel order R2), aggregate numbering by prefix scan,
 *                    Galerkin product L^{i+1} = I L^i I^T (order R3),
 *                    plus the multicolour ordering of every level (R4).
 *   fiedler_solve    Algorithm 3 Steps 2-3: shifted power
 *                    iteration on the coarsest level (R5), then per
 *                    level prolongation y^j = I^T y^{j+1},
 *                    Gauss-Seidel sweeps (Algorithm 2, R5) and
 *                    power iteration on c I - L with deflation (R8);
 *                    finally the Rayleigh quotient.
 *   fiedler_destroy  frees the handle.
 *
 * Conventions (all entry points):
 *   - Graph input is the weighted ADJACENCY W of an undirected graph in CSR:
 *     row_ptr[n+1] (int64, row_ptr[0]=0, nondecreasing), col_idx[nnz] (int32,
 *     strictly increasing within each row, no self loops), weights[nnz]
 *     (float64, finite, > 0, w_ij == w_ji bit-for-bit).  The Laplacian is
 *     L = D - W (Definition 2.1).  nnz counts both directions.
 *   - `mem` arguments say where a pointer lives: FIEDLER_MEM_HOST (pageable or
 *     pinned host memory) or FIEDLER_MEM_DEVICE (memory of opts->device).
 *   - Device memory comes from the device's default stream-ordered pool; the
 *     library sets its release threshold to "keep everything" and grows it once
 *     per fiedler_create to ~8x the input size (FIEDLER_NO_POOL_RESERVE=1 skips
 *     that).  Environment, diagnostics only: FIEDLER_TRACE=1 (phase times on
 *     stderr), FIEDLER_PHASE_TIMES=1 (device times of the setup phases in
 *     fiedler_info), FIEDLER_SERIAL_COLOUR=1 (colourings on the main stream),
 *     FIEDLER_TEST_FULL_SORT=1 (the Galerkin fallback of very large levels).
 *     Input buffers are only read and never retained after the call returns
 *     (fiedler_create copies what it needs); output buffers are caller-owned.
 *   - Every call returns FIEDLER_OK (0) or a negative FIEDLER_ERR_* code and
 *     leaves a human-readable message for fiedler_last_error() (thread-local).
 *     No call falls back to a CPU path: without a usable sm_100 device every
 *     call that needs one fails with FIEDLER_ERR_CUDA.
 *   - Every handle issues its work on a stream it owns (created by
 *     fiedler_create, destroyed by fiedler_destroy; all of the handle's device
 *     buffers are allocated and freed in that stream's order).  A caller's
 *     stream in opts->stream (a cudaStream_t, may differ between calls) is
 *     joined with events: the call's work starts after the work already
 *     enqueued on it and later work on it runs after the call's.  Calls other
 *     than fiedler_dist_op return after the call's work has finished
 *     (results are ready on return).
 *   - A handle is not thread-safe: calls on one handle must not overlap in
 *     time (one host thread at a time), and the fiedler_dist_op work of one
 *     handle must be serialised on one stream -- every call shares the
 *     handle's partial-sum scratch and its last-CTA counter.
 */
#ifndef FIEDLER_H
#define FIEDLER_H

#include <stdint.h>

#if defined(__GNUC__)
#define FIEDLER_API __attribute__((visibility("default")))
#else
#define FIEDLER_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define FIEDLER_OK 0
#define FIEDLER_ERR_ARG -1           /* invalid argument / option               */
#define FIEDLER_ERR_GRAPH -2         /* CSR violates the conventions above      */
#define FIEDLER_ERR_DISCONNECTED -3  /* lambda_2 = 0: Fiedler vector undefined  */
#define FIEDLER_ERR_CUDA -4          /* CUDA runtime / launch / device failure  */
#define FIEDLER_ERR_NOMEM -5         /* device allocation failed                */
#define FIEDLER_ERR_INTERNAL -6      /* an internal invariant failed            */
#define FIEDLER_ERR_TOO_LARGE -7     /* nnz >= 2^31 (int32 offsets) or n >= 2^31 */

#define FIEDLER_MEM_HOST 0
#define FIEDLER_MEM_DEVICE 1

/* Options.  Obtain defaults with fiedler_default_opts(). */
typedef struct fiedler_opts {
    int32_t device;               /* CUDA device ordinal (default 0)                        */
    int32_t coarsest_size;        /* stop coarsening when n <= this ("n_i > 25") */
    int32_t max_levels;           /* hard cap on hierarchy depth (default 50)               */
    int32_t gs_sweeps;            /* Gauss-Seidel sweeps per level below J (default 2)      */
    int32_t power_iters;          /* power iterations per level (default 10)                */
    int32_t coarsest_power_iters; /* power iterations on level J; -1 = power_iters          */
    int32_t validate;             /* 1 = check the CSR conventions on the device (default 1) */
    int32_t use_graph;            /* 1 = repeated solves with the same configuration are
                                     captured once and replayed as one CUDA graph (the
                                     first runs eagerly); 0 = always eager (default 1)     */
    uint64_t seed;                /* counter-based generator seed (R6), default 0           */
    void *stream;                 /* cudaStream_t to use; NULL = handle-owned stream        */
} fiedler_opts;

#define FIEDLER_MAX_LEVELS 64

/* Diagnostics filled by fiedler_solve (optional). */
typedef struct fiedler_info {
    int32_t num_levels;                     /* J + 1                                    */
    int32_t launches;                       /* kernels launched by this solve call      */
    int32_t setup_launches;                 /* kernels launched by fiedler_create        */
    double lambda2;                         /* Rayleigh quotient of the returned vector  */
    double residual_norm;                   /* || L v - lambda2 v ||_2                   */
    double setup_ms;                        /* device time of fiedler_create's setup     */
    double solve_ms;                        /* device time of this solve                 */
    int64_t level_n[FIEDLER_MAX_LEVELS];    /* vertices per level                        */
    int64_t level_nnz[FIEDLER_MAX_LEVELS];  /* adjacency nonzeros per level              */
    int32_t level_colors[FIEDLER_MAX_LEVELS]; /* colours of the multicolour ordering     */
    int32_t level_match_rounds[FIEDLER_MAX_LEVELS]; /* handshake rounds of the matching  */
    double level_shift[FIEDLER_MAX_LEVELS]; /* c of c I - L (R8)                          */
    /* Device time of the setup phases of every level (CUDA events; filled only
     * when the handle was created with FIEDLER_PHASE_TIMES=1 in the
     * environment, else 0).  The colouring runs on a second stream, overlapped
     * with the matching / Galerkin chain, so the phases may overlap in time. */
    double level_match_ms[FIEDLER_MAX_LEVELS];    /* heavy-edge matching + aggregate numbering */
    double level_galerkin_ms[FIEDLER_MAX_LEVELS]; /* Galerkin product to the next level        */
    double level_colour_ms[FIEDLER_MAX_LEVELS];   /* multicolour ordering                       */
    double level_layout_ms[FIEDLER_MAX_LEVELS];   /* GS / natural solve layouts, tiles, shift   */
} fiedler_info;

typedef struct fiedler_handle_s *fiedler_handle;

/* Fill *opts with the defaults listed above. */
FIEDLER_API void fiedler_default_opts(fiedler_opts *opts);

/* Build the multilevel hierarchy of the graph (Setup Phase).
 *   n, nnz       vertices (n >= 2) and stored adjacency entries.
 *   row_ptr, col_idx, weights   CSR of W as described above, in `mem`.
 *   opts         NULL = defaults; device/coarsest_size/max_levels/validate/seed/stream used.
 *   out          receives the handle on success (NULL on failure).
 * Errors: ARG (bad sizes/pointers), GRAPH (validation failed: unsorted or
 * out-of-range columns, self loop, non-positive or non-finite weight,
 * asymmetric entry), DISCONNECTED (the coarsest level is disconnected, which
 * holds iff the input is), TOO_LARGE, NOMEM, CUDA. */
FIEDLER_API int fiedler_create(int64_t n, int64_t nnz, const int64_t *row_ptr,
                   const int32_t *col_idx, const double *weights, int32_t mem,
                   const fiedler_opts *opts, fiedler_handle *out);

/* Run the cascadic refinement (Steps 2-3) and the Rayleigh quotient.
 *   opts            NULL = the options given to fiedler_create; otherwise
 *                   gs_sweeps/power_iters/coarsest_power_iters/seed/use_graph/stream.
 *   fiedler_vector  n doubles in `vec_mem` (may be NULL): the unit-norm vector,
 *                   orthogonal to 1, first nonzero entry positive.
 *   lambda2         (may be NULL) algebraic connectivity estimate = Rayleigh
 *                   quotient of the returned vector (Definition 2.2).
 *   info            (may be NULL) diagnostics.
 * Errors: ARG, CUDA, INTERNAL. */
FIEDLER_API int fiedler_solve(fiedler_handle h, const fiedler_opts *opts, double *fiedler_vector,
                  int32_t vec_mem, double *lambda2, fiedler_info *info);

/* Release every device resource of the handle (NULL is a no-op). */
FIEDLER_API int fiedler_destroy(fiedler_handle h);

/* Message of the last failing call on this thread ("" if none). */
FIEDLER_API const char *fiedler_last_error(void);

/* ---------------------------------------------------------------------------
 * Introspection and single-operation calls (used by the parity tests; they
 * run the same kernels as fiedler_create/fiedler_solve on one level).
 * All vectors here are in the level's NATURAL numbering (the numbering of the
 * oracle: level 0 = input order, level l+1 = aggregate ids of R2).
 * ------------------------------------------------------------------------- */

/* Number of levels J+1 of the hierarchy. */
FIEDLER_API int fiedler_num_levels(fiedler_handle h, int32_t *num_levels);

/* Size of level `level`: vertices, adjacency nonzeros, colours. */
FIEDLER_API int fiedler_level_size(fiedler_handle h, int32_t level, int64_t *n, int64_t *nnz,
                       int32_t *colors);

/* Copy level `level` to HOST buffers (any pointer may be NULL):
 *   row_ptr[n+1] (int64), col_idx[nnz], weights[nnz]: adjacency W^level in
 *     natural numbering with columns ascending (the Galerkin product of R3);
 *   agg[n]: aggregate id of every vertex on level+1 (q of Algorithm 1; -1 on J);
 *   mate[n]: partner in the heavy-edge matching (-1 if unmatched or on J);
 *   color[n]: colour of the multicolour ordering (R4). */
FIEDLER_API int fiedler_level_export(fiedler_handle h, int32_t level, int64_t *row_ptr,
                         int32_t *col_idx, double *weights, int32_t *agg,
                         int32_t *mate, int32_t *color);

#define FIEDLER_OP_GS_SWEEPS 1   /* x_out = `count` multicolour GS sweeps on L x = 0 from x_in (no deflation) */
#define FIEDLER_OP_POWER 2       /* x_out = `count` steps of y <- normalise(deflate((cI - L) y)), y0 = x_in */
#define FIEDLER_OP_PROLONG 3     /* x_out (level) = I^T x_in (level+1): x_out[i] = x_in[q(i)] */
#define FIEDLER_OP_RAYLEIGH 4    /* scalar_out[0] = x^T L x / x^T x of x_in; x_out unused */

/* Apply one solve-phase operation on level `level`.  x_in/x_out live in
 * `mem`, natural numbering, sizes n_level (n_{level+1} for x_in of PROLONG).
 * scalar_out (host, may be NULL) receives {mean, norm} of the result for
 * GS/POWER/PROLONG and {rayleigh, residual_norm} for RAYLEIGH. */
FIEDLER_API int fiedler_level_apply(fiedler_handle h, int32_t level, int32_t op, int32_t count,
                        const double *x_in, double *x_out, int32_t mem,
                        double *scalar_out);

/* Profiling: time `reps` back-to-back launches of one hot kernel on `level`
 * with CUDA events on the handle's stream (after one warm-up launch):
 *   FIEDLER_OP_GS_SWEEPS one full multicolour sweep (all colour launches) per rep,
 *   FIEDLER_OP_POWER     one power-iteration row pass per rep,
 *   FIEDLER_OP_RAYLEIGH  one Rayleigh-quotient row pass per rep.
 * *ms_per_rep = mean device time of one rep; *bytes_per_rep (may be NULL) =
 * the ALGORITHMIC HBM bytes of one rep (4(n+1) row
 * offsets + 12 per adjacency nonzero + 8n vector read + 8n vector written).
 * The level's solve buffers are used as scratch; call between solves, not
 * during one. */
FIEDLER_API int fiedler_level_time(fiedler_handle h, int32_t level, int32_t op, int32_t reps,
                                   double *ms_per_rep, double *bytes_per_rep);

/* ---------------------------------------------------------------------------
 * Row-partitioned solve across ranks (one process per GPU).
 *
 * Every rank holds the whole hierarchy (fiedler_create is deterministic, so
 * all ranks build the same one).  A partitioned level gives rank r the
 * contiguous natural rows [row_begin, row_end) (balanced by rows + nonzeros);
 * every pass of the solve then runs on the rank's own rows only, and the
 * caller moves the bytes between ranks with its collectives library
 * (paper_1602_04386_b200/dist.py: torch.distributed over NCCL):
 *   - halo exchange: after a pass, the values of the rank's rows that other
 *     ranks read (send lists) go to them, and the rank receives the values of
 *     its ghost rows (recv lists);  peer-major, ascending row order, so rank
 *     p's send list to rank r equals rank r's recv list from rank p;
 *   - all-reduce (sum) of the pass statistics, then FIEDLER_DOP_FINALISE;
 *   - all-gather of a level's final vector before the next finer level.
 * Reading of the paper (R2-R8) and the arithmetic per row are those of
 * fiedler_solve; only the summation order of the global sums differs.
 *
 * Vectors are device arrays of the level's size in one of two numberings:
 * natural (the level's own vertex ids) or GS (the multicolour order used by
 * the Gauss-Seidel sweeps; FIEDLER_DOP_PROLONG / _TO_NAT convert).
 * Statistic slots are device arrays of 4 doubles.
 * ------------------------------------------------------------------------- */
#define FIEDLER_MAX_RANKS 64

typedef struct fiedler_dist_plan_info {
    int64_t n;                                   /* level size                     */
    int32_t nranks, rank, colors;
    int64_t row_begin, row_end;                  /* rows of this rank              */
    int64_t row_bounds[FIEDLER_MAX_RANKS + 1];   /* rows of every rank             */
    int64_t send_count[FIEDLER_MAX_RANKS];       /* halo entries sent to each rank */
    int64_t recv_count[FIEDLER_MAX_RANKS];       /* ghost entries from each rank   */
    int64_t send_total, recv_total;
} fiedler_dist_plan_info;

/* Build (or rebuild) the plan of `level` for (nranks, rank); nranks == 1 gives
 * the replicated (whole-level) plan.  Synchronises the handle's stream.
 * Errors: ARG (bad level / nranks outside [1, FIEDLER_MAX_RANKS] / rank). */
FIEDLER_API int fiedler_dist_plan(fiedler_handle h, int32_t level, int32_t nranks, int32_t rank,
                                  fiedler_dist_plan_info *info);

#define FIEDLER_DOP_RAND 1          /* y (natural) = rand(n) (R6, seed = arg); stat = partial (S, Q)     */
#define FIEDLER_DOP_PROLONG 2       /* y = I^T x for own + ghost rows; x = FULL vector of level+1
                                       (natural); arg 0: y natural, 1: y GS; stat = partial (S, Q)     */
#define FIEDLER_DOP_GS_COLOUR 3     /* one GS pass over own rows of colour arg; x (GS) in place          */
#define FIEDLER_DOP_TO_NAT 4        /* y (natural) = x (GS) on own rows; stat = partial (S, Q)            */
#define FIEDLER_DOP_POWER 5         /* y = one power step of x on own rows; stat_in = finalised slot of x;
                                       stat = partial (S, Q) of y                                       */
#define FIEDLER_DOP_FINALISE 6      /* stat: (S, Q) -> (S, Q, mean, deflated norm) of the level          */
#define FIEDLER_DOP_FIRST_NONZERO 7 /* stat[0] = 2 i + (v_i < 0) for the first own row i with
                                       v_i = x_i - mean != 0 (stat_in = slot of x), else 2^60        */
#define FIEDLER_DOP_SIGN 8          /* stat[2] = +-1 from the reduced key in stat[0]                     */
#define FIEDLER_DOP_RAYLEIGH 9      /* own rows: y (natural) = sign (x - mean)/norm; stat = partial
                                       (edge form, sum (x - mean)^2, ||L (x - mean)||^2);
                                       stat_in = slot of x, sign read at sign_slot[2] (arg ignored)     */
#define FIEDLER_DOP_FINALISE_RQ 10  /* stat (reduced partials) -> {lambda2, residual, ||v||}, using
                                       stat_in = slot of x                                              */
#define FIEDLER_DOP_HALO_PACK 11    /* y (send buffer) = x at the send rows; arg 0: x natural, 1: GS     */
#define FIEDLER_DOP_HALO_UNPACK 12  /* y at the ghost rows = x (recv buffer); arg 0: y natural, 1: GS    */

/* Enqueue one operation of the partitioned solve on `stream` (NULL = the
 * handle's own stream, which is non-blocking: device inputs written on other
 * streams must be complete, or pass their stream) for the plan last built on
 * `level`.  Never synchronises
 * `stream` (the first call may wait for the handle's own stream while it
 * allocates the handle's scratch).  All fiedler_dist_op calls of a handle,
 * and its fiedler_solve / fiedler_level_* calls, must be serialised on one
 * stream: they share the handle's reduction scratch (see the notes above).
 * x / y / stat / stat_in / sign_slot: device pointers (unused ones may be
 * NULL).  Errors: ARG (no plan on level, bad op), CUDA. */
FIEDLER_API int fiedler_dist_op(fiedler_handle h, int32_t level, int32_t op, int64_t arg,
                                const double *x, double *y, double *stat, const double *stat_in,
                                const double *sign_slot, void *stream);

/* ---------------------------------------------------------------------------
 * Row-partitioned SETUP of the fine levels (Algorithm 3 Step 1, PAPER.md:117-125;
 * DESIGN.md section 9).  Handle-free operations on one level's whole CSR
 * (device arrays, the conventions of fiedler_create: int64 row_ptr, int32
 * ascending columns, float64 weights; every rank holds the whole level), each
 * run on the caller's OWN rows [r0, r1) only.  The driver
 * (paper_1602_04386_b200/dist.py, PartitionedSetup) exchanges the state of the
 * boundary rows between the calls with its collectives library:
 *   matching   rounds of POINT, halo(ptr), RESOLVE, halo(mate) until no own
 *              free row has a free neighbour anywhere (all-reduce);
 *   aggregates LEADERS (count), exclusive scan of the counts over ranks,
 *              IDS, halo(q), MATES, halo(q), JOIN, all-gather of q;
 *   Galerkin   the coarse rows [a0, a1) of the caller's leaders (contiguous:
 *              aggregates are numbered by increasing leader), all-gathered;
 *   colouring  Jones-Plassmann rounds with halo(colour) until no row is left.
 * The results are those of fiedler_create, bit for bit, for any partition
 * (R2-R4: every rule is a strict order independent of the schedule).
 * State arrays (mate, ptr, q, colour) are device int32 [n]; only own rows are
 * written, ghost rows are read.  `stream` = cudaStream_t (NULL = legacy default
 * stream).  Calls that return a count synchronise `stream`; the others only
 * enqueue.  Errors: ARG (sizes, ranges, NULL pointers), CUDA, NOMEM.
 * ------------------------------------------------------------------------- */

/* Row partition of a level for `nranks` ranks: bounds[k] = the first row r with
 * row_ptr[r] + r >= floor(k (nnz + n) / nranks) (rows + nonzeros balanced; the
 * rule of fiedler_dist_plan), bounds[0] = 0, bounds[nranks] = n.  row_ptr:
 * device; bounds: host [nranks + 1].  Synchronises. */
FIEDLER_API int fiedler_pset_bounds(int64_t n, const int64_t *row_ptr, int32_t nranks, int64_t *bounds,
                                    void *stream);

/* Halo send lists of rank `rank`: for every peer p != rank (peer-major), the own
 * rows that have a neighbour in p's rows, ascending.  By symmetry of the graph
 * they are p's ghost rows of this rank, i.e. p's receive list from `rank`.
 * bounds: host [nranks + 1] (fiedler_pset_bounds).  send_count: host [nranks]
 * (0 for p == rank).  send_idx: device [sum send_count] of natural row ids, or
 * NULL to get the counts only.  Synchronises. */
FIEDLER_API int fiedler_pset_halo(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, int32_t nranks,
                                  int32_t rank, const int64_t *bounds, int32_t *send_idx, int64_t *send_count,
                                  void *stream);

/* Halo pack / unpack of int32 state: out[k] = x[idx[k]] (gather) and
 * x[idx[k]] = in[k] (scatter), k < count.  Device arrays; enqueue only. */
FIEDLER_API int fiedler_pset_gather(const int32_t *x, const int32_t *idx, int64_t count, int32_t *out,
                                    void *stream);
/* x[idx[k]] = in[k], k < count (the unpack of fiedler_pset_gather's buffers). */
FIEDLER_API int fiedler_pset_scatter(const int32_t *in, const int32_t *idx, int64_t count, int32_t *x,
                                     void *stream);

#define FIEDLER_PSET_POINT 0     /* matching: ptr[v] = the heaviest free neighbour of own free v        */
#define FIEDLER_PSET_RESOLVE 1   /* matching: mate[v] = ptr[v] where ptr[ptr[v]] == v                   */

/* One half-round of the parallel heavy-edge matching (Algorithm 1, PAPER.md:49-74,
 * in the parallel order of R2) on own rows.  Edge order: (w, h) decreasing,
 * h({u,v}) = splitmix64(salt ^ (min << 32 | max)), salt = splitmix64(seed ^
 * (TAG_MATCH + level)).  mate[v] = -1 while v is free.  POINT: for own free v,
 * ptr[v] = the first neighbour u in that order with mate[u] == -1 (-1 if none);
 * *active (host) = the number of own rows with ptr[v] >= 0 (synchronises).
 * RESOLVE: own free v with u = ptr[v] >= 0 and ptr[u] == v gets mate[v] = u
 * (the handshake: the edge is the heaviest free edge at both ends, so the
 * greedy heaviest-first matching of R2 takes it).  The caller initialises mate
 * and ptr to -1 and exchanges ptr (after POINT) and mate (after RESOLVE) of the
 * boundary rows; when the all-reduced *active is 0 the matching is maximal
 * and equals R2's greedy matching.  round = the handshake round (0, 1, ...).
 * work: NULL (every half-round visits all own rows) or device int32 scratch
 * [8 + 2 (r1 - r0)] kept by the caller for the level's rounds: POINT of round
 * k > 0 visits only the rows the previous RESOLVE left free, RESOLVE only the
 * rows POINT found a partner for (a row with no free neighbour never gets one
 * back, a matched row stays matched). */
FIEDLER_API int fiedler_pset_match(int32_t phase, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                                   const double *weights, int64_t r0, int64_t r1, uint64_t seed, int32_t level,
                                   int32_t *mate, int32_t *ptr, int32_t round, int32_t *work, int64_t *active,
                                   void *stream);

#define FIEDLER_PSET_LEADERS 0   /* *count = own leaders (synchronises)                                   */
#define FIEDLER_PSET_IDS 1       /* q[v] = offset + rank of v among own leaders; -1 on other own rows     */
#define FIEDLER_PSET_MATES 2     /* own matched non-leader v: q[v] = q[mate[v]]                           */
#define FIEDLER_PSET_JOIN 3      /* own unmatched v with neighbours: q[v] = q[m(v)], m(v) heaviest nbr    */

/* Aggregate numbering of R2 on own rows, given the maximal
 * matching `mate`.  The leader of an aggregate is min(u, mate(u)) for a matched
 * pair, the vertex itself if it has no neighbour; an unmatched vertex joins the
 * aggregate of its heaviest neighbour m(v) (edge order of fiedler_pset_match),
 * which is matched.  Aggregates are numbered by increasing leader: rank r's
 * leaders get the contiguous ids [offset, offset + count_r), offset = the sum of
 * the counts of the lower ranks.  Between IDS / MATES / JOIN the caller
 * exchanges q of the boundary rows. */
FIEDLER_API int fiedler_pset_aggregate(int32_t phase, int64_t n, const int64_t *row_ptr,
                                       const int32_t *col_idx, const double *weights, int64_t r0, int64_t r1,
                                       uint64_t seed, int32_t level, const int32_t *mate, int32_t *q,
                                       int64_t offset, int64_t *count, void *stream);

/* Galerkin product I L I^T (R3) for the coarse rows [a0, a1) given
 * the WHOLE aggregate map q (device int32 [n]).  Phase 0: *count = the number of
 * crossing contributions of those rows (fine entries i -> j with q(i) in
 * [a0, a1), q(j) != q(i): an upper bound of their coarse nonzeros;
 * synchronises).  Coarse rows whose members have at most 32 entries in all are
 * built by one thread each, longer ones by a sort of their contributions.  Phase 1 (cap >= that bound): the coarse adjacency
 * rows in CSR with LOCAL offsets: crp (device int64 [a1 - a0 + 1], crp[0] = 0),
 * ascending columns cci (device int32), weights cw (device float64): W_c(A, B) =
 * the left fold of the fine weights w_ij over the fine edges {i < j} with
 * {q(i), q(j)} = {A, B} in (i, j) lexicographic order; *count = crp[a1 - a0]
 * (synchronises). */
FIEDLER_API int fiedler_pset_galerkin(int32_t phase, int64_t n, const int64_t *row_ptr,
                                      const int32_t *col_idx, const double *weights, const int32_t *q,
                                      int64_t a0, int64_t a1, int64_t cap, int64_t *crp, int32_t *cci,
                                      double *cw, int64_t *count, void *stream);

/* One Jones-Plassmann round of the colouring of R4 on own rows: an own
 * uncoloured v (colour[v] == -1) all of whose neighbours u of higher priority
 * (pi(u), u) > (pi(v), v), pi(x) = splitmix64(salt ^ x), salt =
 * splitmix64(seed ^ (TAG_COLOR + level)), are coloured takes the smallest
 * colour none of its coloured neighbours has -- the greedy first-fit colouring
 * in decreasing priority, independent of the schedule.  out (host int64 [2]):
 * {own rows still uncoloured, largest colour given in this round (-1 if none)};
 * synchronises.  round = 0, 1, ... of the level; work: NULL (every round
 * visits all own rows) or device int32 scratch [8 + 2 (r1 - r0)] kept across
 * the level's rounds (round k > 0 visits only the rows round k - 1 left). */
FIEDLER_API int fiedler_pset_colour(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, int64_t r0,
                                    int64_t r1, uint64_t seed, int32_t level, int32_t round, int32_t *work,
                                    int32_t *colour, int64_t *out, void *stream);

/* One level of a hierarchy built outside fiedler_create (fiedler_pset_*): the
 * level's aggregate map, matching and colouring (device int32 [n_l]) and the
 * next level's adjacency (device CSR, fiedler_create's conventions). */
typedef struct fiedler_preset_level {
    const int32_t *agg, *mate, *color;
    int32_t ncolors, match_rounds, colour_rounds, reserved;
    int64_t n_next, nnz_next;
    const int64_t *rp_next;
    const int32_t *ci_next;
    const double *w_next;
} fiedler_preset_level;

/* fiedler_create whose levels 0..npreset-1 are given: their matching, aggregate
 * map, colouring and next level are copied from `preset` instead of being
 * computed (the preset levels must be levels fiedler_create would coarsen:
 * n_l > coarsest_size, l + 1 < max_levels, not stalled by R9); the coarser
 * levels, every layout and the solve state are built as by fiedler_create.
 * The preset arrays are copied before the call returns (caller keeps
 * ownership).  npreset = 0 is fiedler_create.  Errors: those of fiedler_create,
 * ARG (npreset outside [0, max_levels - 1], NULL preset arrays, sizes). */
FIEDLER_API int fiedler_create_preset(int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col_idx,
                                      const double *weights, int32_t mem, const fiedler_opts *opts,
                                      int32_t npreset, const fiedler_preset_level *preset,
                                      fiedler_handle *out);

#ifdef __cplusplus
}
#endif
#endif /* FIEDLER_H */

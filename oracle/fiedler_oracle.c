/*
 * oracle/fiedler_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously-correct CPU reference ("oracle") for the
 * cascadic-multigrid Fiedler solver of Gandhi, "Improvement of the Cascadic
 * Multigrid Algorithm with a Gauss Seidel Smoother to Efficiently Compute the
 * Fiedler Vector of a Graph Laplacian" (arXiv 1602.04386).  Citations of the
 * form "PAPER.md:NN" are line numbers of the paper text; "R<k>" names a
 * reading listed in DESIGN.md section 3 (where the paper is silent/garbled).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * "--impl reference" legs may load this library.  It shares no code, header,
 * constant generator or helper with the CUDA product path; the counter-based
 * generator (splitmix64) is re-implemented here on purpose (task rule 3).
 *
 * Everything is float64, single-threaded, written in the paper's order.
 * Compiled with -O2 -ffp-contract=off (no FMA contraction), so every
 * floating-point operation below rounds exactly as written.
 *
 * Graph representation: the weighted adjacency W of G=(V,E,w)
 * in CSR: rp[n+1] (int64), ci[nnz] (int32, ascending within a row, no self
 * loops), w[nnz] (float64, > 0, w_ij == w_ji bit-for-bit).  The Laplacian is
 * L = D - W (Definition 2.1); its diagonal d is computed by
 * orc_degrees().
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Counter-based generator (R6).  SplitMix64 finaliser, Steele et al. */
/* ------------------------------------------------------------------ */
uint64_t orc_splitmix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* rand(n_J) of Algorithm 3 Step 2: u_i in [0,1) from the
 * counter stream s0 + i, s0 = splitmix64(seed ^ TAG_RAND) (R6). */
#define TAG_RAND 0x72616E6400000000ULL
void orc_rand_uniform(int64_t n, uint64_t seed, double *out)
{
    uint64_t s0 = orc_splitmix64(seed ^ TAG_RAND);
    for (int64_t i = 0; i < n; i++)
        out[i] = (double)(orc_splitmix64(s0 + (uint64_t)i) >> 11) * 0x1.0p-53;
}

/* p <- randperm(n) of Algorithm 1 line 3, Fisher-Yates driven
 * by the splitmix64 stream of (seed ^ TAG_PERM ^ level) (R6). */
#define TAG_PERM 0x7065726D00000000ULL
void orc_randperm(int64_t n, uint64_t seed, int64_t level, int64_t *p)
{
    uint64_t s0 = orc_splitmix64(seed ^ TAG_PERM ^ (uint64_t)level);
    for (int64_t i = 0; i < n; i++) p[i] = i;
    for (int64_t i = n - 1; i > 0; i--) {
        int64_t j = (int64_t)(orc_splitmix64(s0 + (uint64_t)i) % (uint64_t)(i + 1));
        int64_t t = p[i]; p[i] = p[j]; p[j] = t;
    }
}

/* ------------------------------------------------------------------ */
/* Definition 2.1: the Laplacian and its actions.     */
/* ------------------------------------------------------------------ */

/* d_{v_i} = sum_j w_ij, summed in ascending j. */
void orc_degrees(int64_t n, const int64_t *rp, const int32_t *ci,
                 const double *w, double *d)
{
    (void)ci;
    for (int64_t i = 0; i < n; i++) {
        double s = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) s += w[k];
        d[i] = s;
    }
}

/* y = L x, row i of Definition 2.1: d_i x_i + sum_{j!=i} (-w_ij) x_j. */
void orc_laplacian_matvec(int64_t n, const int64_t *rp, const int32_t *ci,
                          const double *w, const double *d, const double *x,
                          double *y)
{
    for (int64_t i = 0; i < n; i++) {
        double s = d[i] * x[i];
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) s += (-w[k]) * x[ci[k]];
        y[i] = s;
    }
}

/* x^T L x written as the Laplacian quadratic form sum_{(i,j) in E} w_ij
 * (x_i - x_j)^2, which is Definition 2.1 expanded (R7: cancellation-free
 * form; pinned against the dense matrix product in tests). */
double orc_quadratic_form(int64_t n, const int64_t *rp, const int32_t *ci,
                          const double *w, const double *x)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++)
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) {
            int64_t j = ci[k];
            if (j > i) {
                double t = x[i] - x[j];
                s += w[k] * (t * t);
            }
        }
    return s;
}

/* "calculate the Rayleigh Quotient to achieve the eigenvalue"
 * (PAPER.md:19,112): (x^T L x) / (x^T x). */
double orc_rayleigh(int64_t n, const int64_t *rp, const int32_t *ci,
                    const double *w, const double *x)
{
    double den = 0.0;
    for (int64_t i = 0; i < n; i++) den += x[i] * x[i];
    return orc_quadratic_form(n, rp, ci, w, x) / den;
}

/* Deflation against the constant eigenvector [1,...,1]^T:
 * x <- x - mean(x) 1. */
void orc_deflate(int64_t n, double *x)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) s += x[i];
    double m = s / (double)n;
    for (int64_t i = 0; i < n; i++) x[i] -= m;
}

/* x <- x / ||x||_2 ; returns 0 on a zero vector. */
int orc_normalize(int64_t n, double *x)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) s += x[i] * x[i];
    if (!(s > 0.0)) return 0;
    double r = sqrt(s);
    for (int64_t i = 0; i < n; i++) x[i] /= r;
    return 1;
}

/* ------------------------------------------------------------------ */
/* Algorithm 1, Heavy Edge Coarsening.                */
/* ------------------------------------------------------------------ */

/* m <- argmin(L(:,v)).  Column v of L holds d_v >= 0 on the
 * diagonal, -w_uv < 0 at the neighbours and 0 elsewhere, so for a vertex
 * with neighbours the minimum is the heaviest incident edge; MATLAB's min
 * returns the lowest index among equal minima (R1).  An isolated vertex
 * returns itself (R1). */
static int64_t heaviest_neighbor_lowest_index(const int64_t *rp, const int32_t *ci,
                                              const double *w, int64_t v)
{
    int64_t m = v;
    double best = 0.0;
    for (int64_t k = rp[v]; k < rp[v + 1]; k++) {
        /* column entry L(ci,v) = -w ; strictly smaller wins, ties keep the
         * lower index because columns are scanned in ascending order */
        if (m == v || -w[k] < -best) { best = w[k]; m = ci[k]; }
    }
    return m;
}

/* Algorithm 1 verbatim with the visiting order p given (sequential mode).
 * Aggregate ids are 0-based (paper: 1..c).  Returns c. */
int64_t orc_hec_sequential(int64_t n, const int64_t *rp, const int32_t *ci,
                           const double *w, const int64_t *p, int64_t *q)
{
    int64_t c = 0;                                    /* line 2 */
    for (int64_t i = 0; i < n; i++) q[i] = -1;        /* line 4: q <- zeros */
    for (int64_t i = 0; i < n; i++) {                 /* line 5 */
        int64_t v = p[i];
        if (q[v] == -1) {                             /* line 6 */
            int64_t m = heaviest_neighbor_lowest_index(rp, ci, w, v); /* line 7 */
            if (q[m] == -1) {                         /* line 8 */
                q[m] = c;                             /* lines 9-11 */
                q[v] = c;
                c = c + 1;
            } else {
                q[v] = q[m];                          /* line 13 */
            }
        }
    }
    return c;
}

/* Parallel-order heavy edge coarsening (R2).  The edge order is
 *   e > f  iff  w_e > w_f, or w_e == w_f and h(e) > h(f),
 * h({u,v}) = splitmix64(salt ^ (min<<32 | max)) (injective => strict order).
 * (1) heaviest-first greedy matching: scan edges in decreasing order and
 *     match an edge whose two endpoints are both free;
 * (2) an unmatched vertex v with neighbours joins the aggregate of its
 *     heaviest neighbour m(v) (the rule "q(p(i)) = q(m)");
 *     m(v) is matched because the greedy matching is maximal;
 * (3) an aggregate's leader is min(u, mate(u)) for a matched pair, the vertex
 *     itself if isolated; aggregates are numbered by increasing leader
 *     index (an exclusive prefix sum over leader flags).
 * Outputs mate[n] (-1 if unmatched) and q[n]; returns c. */
typedef struct { double w; uint64_t h; int64_t u, v; } orc_edge;

static int edge_cmp_desc(const void *a, const void *b)
{
    const orc_edge *x = (const orc_edge *)a, *y = (const orc_edge *)b;
    if (x->w > y->w) return -1;
    if (x->w < y->w) return 1;
    if (x->h > y->h) return -1;
    if (x->h < y->h) return 1;
    return 0;
}

static uint64_t edge_hash(uint64_t salt, int64_t a, int64_t b)
{
    uint64_t lo = (uint64_t)(a < b ? a : b), hi = (uint64_t)(a < b ? b : a);
    return orc_splitmix64(salt ^ ((lo << 32) | hi));
}

int64_t orc_hec_parallel(int64_t n, const int64_t *rp, const int32_t *ci,
                         const double *w, uint64_t salt, int64_t *mate,
                         int64_t *q)
{
    int64_t ne = 0;
    for (int64_t u = 0; u < n; u++)
        for (int64_t k = rp[u]; k < rp[u + 1]; k++)
            if (ci[k] > u) ne++;
    orc_edge *E = (orc_edge *)malloc(sizeof(orc_edge) * (size_t)(ne > 0 ? ne : 1));
    int64_t *heavy = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *leader = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    if (!E || !heavy || !leader) { free(E); free(heavy); free(leader); return -1; }

    ne = 0;
    for (int64_t u = 0; u < n; u++)
        for (int64_t k = rp[u]; k < rp[u + 1]; k++)
            if (ci[k] > u) {
                E[ne].w = w[k];
                E[ne].h = edge_hash(salt, u, ci[k]);
                E[ne].u = u;
                E[ne].v = ci[k];
                ne++;
            }
    qsort(E, (size_t)ne, sizeof(orc_edge), edge_cmp_desc);

    /* (1) greedy heaviest-first matching */
    for (int64_t v = 0; v < n; v++) mate[v] = -1;
    for (int64_t e = 0; e < ne; e++)
        if (mate[E[e].u] == -1 && mate[E[e].v] == -1) {
            mate[E[e].u] = E[e].v;
            mate[E[e].v] = E[e].u;
        }

    /* m(v): heaviest incident edge in the same strict order */
    for (int64_t v = 0; v < n; v++) {
        heavy[v] = -1;
        double bw = 0.0;
        uint64_t bh = 0;
        for (int64_t k = rp[v]; k < rp[v + 1]; k++) {
            uint64_t h = edge_hash(salt, v, ci[k]);
            if (heavy[v] == -1 || w[k] > bw || (w[k] == bw && h > bh)) {
                heavy[v] = ci[k]; bw = w[k]; bh = h;
            }
        }
    }

    /* (2)+(3) leaders, numbered in increasing vertex order */
    for (int64_t v = 0; v < n; v++) {
        if (mate[v] >= 0) leader[v] = v < mate[v] ? v : mate[v];
        else if (heavy[v] >= 0) {
            int64_t m = heavy[v];
            if (mate[m] < 0) { free(E); free(heavy); free(leader); return -2; } /* not maximal: impossible */
            leader[v] = m < mate[m] ? m : mate[m];
        } else leader[v] = v;
    }
    int64_t c = 0;
    int64_t *id = heavy; /* reuse: id of a leader */
    for (int64_t v = 0; v < n; v++) id[v] = (leader[v] == v) ? c++ : -1;
    for (int64_t v = 0; v < n; v++) q[v] = id[leader[v]];

    free(E); free(heavy); free(leader);
    return c;
}

/* ------------------------------------------------------------------ */
/* Galerkin product L^{i+1} = I L^i I^T (Algorithm 3 line 5) */
/* ------------------------------------------------------------------ */
/* I = I_i^{i+1} has I(q(v),v) = 1.  Off the diagonal,
 * (I L I^T)(a,b) = -sum_{q(i)=a, q(j)=b} w_ij, so the coarse graph has edge
 * weights W_c(a,b) = sum of the fine weights between aggregates a != b, and
 * the coarse diagonal equals sum_b W_c(a,b) (zero row sums).  We therefore
 * return the coarse ADJACENCY W_c; the coarse Laplacian is D_c - W_c.
 * Summation order (R3): the fine undirected edges {i,j} (i<j) crossing the
 * coarse pair {a,b} are folded left-to-right in (i, j) lexicographic order,
 * starting from the first contribution.  The order depends only on the
 * unordered pair, so W_c(a,b) == W_c(b,a) bit-for-bit.
 * crp[c+1]; cci/cw must hold nnz(fine) entries.  Returns the coarse nnz. */
typedef struct { int64_t a, b, pos; double w; } orc_contrib;

static int contrib_cmp(const void *x_, const void *y_)
{
    const orc_contrib *x = (const orc_contrib *)x_, *y = (const orc_contrib *)y_;
    if (x->a != y->a) return x->a < y->a ? -1 : 1;
    if (x->b != y->b) return x->b < y->b ? -1 : 1;
    return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

int64_t orc_galerkin(int64_t n, const int64_t *rp, const int32_t *ci,
                     const double *w, const int64_t *q, int64_t c,
                     int64_t *crp, int32_t *cci, double *cw)
{
    int64_t nfe = 0;
    for (int64_t i = 0; i < n; i++)
        for (int64_t k = rp[i]; k < rp[i + 1]; k++)
            if (ci[k] > i) nfe++;
    orc_contrib *C = (orc_contrib *)malloc(sizeof(orc_contrib) * (size_t)(nfe > 0 ? nfe : 1));
    int64_t *fill = (int64_t *)calloc((size_t)c + 1, sizeof(int64_t));
    if (!C || !fill) { free(C); free(fill); return -1; }

    /* 1. contributions of crossing fine edges, visited in (i, j) order and
     *    keyed by the unordered coarse pair (A, B), A < B */
    int64_t nc = 0;
    for (int64_t i = 0; i < n; i++)
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) {
            int64_t j = ci[k];
            if (j <= i) continue;
            int64_t a = q[i], b = q[j];
            if (a == b) continue;              /* intra-aggregate: on the diagonal */
            C[nc].a = a < b ? a : b;
            C[nc].b = a < b ? b : a;
            C[nc].pos = nc;
            C[nc].w = w[k];
            nc++;
        }
    qsort(C, (size_t)nc, sizeof(orc_contrib), contrib_cmp);   /* by (A, B, visit order) */

    /* 2. left fold of every run of equal (A, B); compact in place */
    int64_t np = 0;
    for (int64_t t = 0; t < nc;) {
        int64_t u = t;
        double s = C[t].w;
        for (u = t + 1; u < nc && C[u].a == C[t].a && C[u].b == C[t].b; u++) s += C[u].w;
        C[np] = C[t];
        C[np].w = s;
        np++;
        t = u;
    }

    /* 3. symmetric CSR: pairs are sorted by (A, B), so appending each pair to
     *    rows A and B in this order leaves every row sorted by column */
    for (int64_t a = 0; a <= c; a++) crp[a] = 0;
    for (int64_t t = 0; t < np; t++) { crp[C[t].a + 1]++; crp[C[t].b + 1]++; }
    for (int64_t a = 0; a < c; a++) crp[a + 1] += crp[a];
    for (int64_t t = 0; t < np; t++) {
        int64_t A = C[t].a, B = C[t].b;
        cci[crp[A] + fill[A]] = (int32_t)B; cw[crp[A] + fill[A]] = C[t].w; fill[A]++;
        cci[crp[B] + fill[B]] = (int32_t)A; cw[crp[B] + fill[B]] = C[t].w; fill[B]++;
    }
    free(C); free(fill);
    return crp[c];
}

/* ------------------------------------------------------------------ */
/* Deterministic colouring for multicolour Gauss-Seidel (R4).           */
/* ------------------------------------------------------------------ */
/* Greedy first-fit colouring in decreasing priority (pi(v), v),
 * pi(v) = splitmix64(salt ^ v): color(v) = the smallest colour not used by
 * an already-coloured (= higher-priority) neighbour.  Returns #colours. */
typedef struct { uint64_t pi; int64_t v; } orc_prio;

static int prio_cmp_desc(const void *a, const void *b)
{
    const orc_prio *x = (const orc_prio *)a, *y = (const orc_prio *)b;
    if (x->pi > y->pi) return -1;
    if (x->pi < y->pi) return 1;
    if (x->v > y->v) return -1;
    if (x->v < y->v) return 1;
    return 0;
}

int32_t orc_greedy_coloring(int64_t n, const int64_t *rp, const int32_t *ci,
                            uint64_t salt, int32_t *color)
{
    orc_prio *P = (orc_prio *)malloc(sizeof(orc_prio) * (size_t)(n > 0 ? n : 1));
    if (!P) return -1;
    for (int64_t v = 0; v < n; v++) { P[v].pi = orc_splitmix64(salt ^ (uint64_t)v); P[v].v = v; }
    qsort(P, (size_t)n, sizeof(orc_prio), prio_cmp_desc);
    for (int64_t v = 0; v < n; v++) color[v] = -1;
    int32_t ncol = 0;
    int64_t maxdeg = 0;
    for (int64_t v = 0; v < n; v++) if (rp[v + 1] - rp[v] > maxdeg) maxdeg = rp[v + 1] - rp[v];
    unsigned char *used = (unsigned char *)calloc((size_t)maxdeg + 2, 1);
    if (!used) { free(P); return -1; }
    for (int64_t t = 0; t < n; t++) {
        int64_t v = P[t].v;
        for (int64_t k = rp[v]; k < rp[v + 1]; k++) {
            int32_t cu = color[ci[k]];
            if (cu >= 0 && cu <= maxdeg) used[cu] = 1;
        }
        int32_t cv = 0;
        while (used[cv]) cv++;
        color[v] = cv;
        if (cv + 1 > ncol) ncol = cv + 1;
        for (int64_t k = rp[v]; k < rp[v + 1]; k++) {
            int32_t cu = color[ci[k]];
            if (cu >= 0 && cu <= maxdeg) used[cu] = 0;
        }
    }
    free(used); free(P);
    return ncol;
}

/* ------------------------------------------------------------------ */
/* Algorithm 2, Gauss-Seidel.                          */
/* ------------------------------------------------------------------ */

/* General form for a matrix A given in CSR *with* its diagonal: forward
 * sweeps x_i = 1/a_ii [ b_i - sum_{j<i} a_ij x_j - sum_{j>i} a_ij X0_j ]
 * (line 87, in-place = newest values), stopped when max|x - X0| < tol
 * (line 88) or after N sweeps (line 85).  Returns sweeps performed, or -1
 * on a zero diagonal. */
int64_t orc_gs_solve(int64_t n, const int64_t *rp, const int32_t *ci,
                     const double *a, const double *b, double *x, double tol,
                     int64_t N)
{
    int64_t k = 1;
    while (k <= N) {
        double change = 0.0;
        for (int64_t i = 0; i < n; i++) {
            double aii = 0.0, s = b[i];
            for (int64_t t = rp[i]; t < rp[i + 1]; t++) {
                if (ci[t] == i) aii = a[t];
                else s -= a[t] * x[ci[t]];
            }
            if (aii == 0.0) return -1;
            double xi = s / aii;
            double dlt = fabs(xi - x[i]);
            if (dlt > change) change = dlt;
            x[i] = xi;
        }
        if (change < tol) return k;
        k = k + 1;
    }
    return N;
}

/* The smoother GS(L^j, y) of Algorithm 3 on L y = 0 (R5):
 * with a_ii = d_i, a_ij = -w_ij, b = 0 line 87 reads
 *     x_i = (1/d_i) sum_j w_ij x_j        (newest values, in place),
 * visiting vertices in `order` (identity = lexicographic Gauss-Seidel;
 * (colour, index) order = the parallel-mode multicolour sweep). */
void orc_gs_sweeps(int64_t n, const int64_t *rp, const int32_t *ci,
                   const double *w, const double *d, const int64_t *order,
                   double *x, int64_t sweeps)
{
    for (int64_t s = 0; s < sweeps; s++)
        for (int64_t t = 0; t < n; t++) {
            int64_t i = order[t];
            double acc = 0.0;                 /* b_i = 0 */
            for (int64_t k = rp[i]; k < rp[i + 1]; k++)
                acc -= (-w[k]) * x[ci[k]];    /* - a_ij x_j, a_ij = -w_ij */
            x[i] = acc / d[i];                /* 1/a_ii [...] */
        }
}

/* ------------------------------------------------------------------ */
/* Power iteration on the modified matrix c I - L with deflation          */
/* ("power iteration on a modified matrix"; "A direct power   */
/* iteration is used").  Each step: y <- (cI - L) y,          */
/* deflate, normalise.                                                     */
/* ------------------------------------------------------------------ */
int orc_power_iterations(int64_t n, const int64_t *rp, const int32_t *ci,
                         const double *w, const double *d, double shift,
                         double *x, int64_t iters, double *work)
{
    for (int64_t it = 0; it < iters; it++) {
        orc_laplacian_matvec(n, rp, ci, w, d, x, work);   /* work = L x */
        for (int64_t i = 0; i < n; i++) x[i] = shift * x[i] - work[i];
        orc_deflate(n, x);
        if (!orc_normalize(n, x)) return 0;
    }
    return 1;
}

/* Prolongation y^j = (I_j^{j+1})^T y^{j+1} (Algorithm 3 line 14,
 * PAPER.md:131): the transpose of the 0/1 matrix copies y^{j+1}[q(i)]. */
void orc_prolongate(int64_t n_fine, const int64_t *q, const double *yc, double *yf)
{
    for (int64_t i = 0; i < n_fine; i++) yf[i] = yc[q[i]];
}

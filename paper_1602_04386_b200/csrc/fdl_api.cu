// fdl_api.cu -- the extern "C" boundary declared in include/fiedler.h.
// Argument checking, host<->device staging, CUDA-graph capture/replay of the
// solve schedule, and error translation.  All numerical work is in
// fdl_setup.cu / fdl_solve.cu kernels; there is no CPU fallback.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <memory>
#include <string>

#include "fdl_internal.h"

namespace fdl {

thread_local std::string g_last_error;

bool trace_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = std::getenv("FIEDLER_TRACE");
        on = (e && e[0] == '1') ? 1 : 0;
    }
    return on == 1;
}

void trace_mark(cudaStream_t st, const char *what) {
    if (!trace_enabled()) return;
    static thread_local auto last = std::chrono::steady_clock::now();
    if (st) cudaStreamSynchronize(st);
    auto now = std::chrono::steady_clock::now();
    double ms = std::chrono::duration<double, std::milli>(now - last).count();
    std::fprintf(stderr, "[fiedler trace] %-40s %9.3f ms\n", what, ms);
    last = now;
}
thread_local long long g_launch_count = 0;

// FIEDLER_ALLOC_STATS=1 (diagnostics): host time spent inside cudaMallocAsync /
// cudaFreeAsync (pool calls of DBuf), printed per create
std::atomic<long long> g_alloc_ns{0}, g_alloc_calls{0}, g_free_ns{0}, g_free_calls{0};
bool alloc_stats_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = std::getenv("FIEDLER_ALLOC_STATS");
        on = (e && e[0] == '1') ? 1 : 0;
    }
    return on == 1;
}

void set_error(const std::string &m) { g_last_error = m; }

#ifndef FDL_STREAM2_PRIO
#define FDL_STREAM2_PRIO 0
#endif
#ifndef FDL_MAIN_PRIO
#define FDL_MAIN_PRIO 1
#endif

// ---- per-device pool of stream sets (include: fdl_internal.h StreamSet)
namespace {
std::mutex g_pool_mu;
std::vector<StreamSet> g_pool[kMaxDevices];
}  // namespace

static StreamSet take_stream_set(int dev) {
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (!g_pool[dev].empty()) {
            StreamSet s = g_pool[dev].back();
            g_pool[dev].pop_back();
            return s;
        }
    }
    StreamSet s;
    {   // main stream priority (build knob FDL_MAIN_PRIO: 1 highest (default), 0 default priority;
        // measured: config 3 -0.9 ms, config 2 -0.2 ms, config 4 unchanged): pending
        // CTAs of the coarsening chain are placed before the side streams' (layouts)
        int lo = 0, hi = 0;
        FDL_CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        FDL_CK(cudaStreamCreateWithPriority(&s.stream, cudaStreamNonBlocking, FDL_MAIN_PRIO > 0 ? hi : 0));
    }
    {   // stream2 priority (build knob FDL_STREAM2_PRIO: 0 default, 1 highest, -1 lowest)
        int lo = 0, hi = 0;
        FDL_CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        const int pr = FDL_STREAM2_PRIO > 0 ? hi : FDL_STREAM2_PRIO < 0 ? lo : 0;
        FDL_CK(cudaStreamCreateWithPriority(&s.stream2, cudaStreamNonBlocking, pr));
        s.side[0] = s.stream2;
        for (int k = 1; k < kSides; k++) FDL_CK(cudaStreamCreateWithPriority(&s.side[k], cudaStreamNonBlocking, pr));
    }
    for (int k = 0; k < kSides; k++) FDL_CK(cudaEventCreateWithFlags(&s.sev[k], cudaEventDisableTiming));
    for (cudaEvent_t &e : s.ev) FDL_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (cudaEvent_t &e : s.tev) FDL_CK(cudaEventCreate(&e));
    return s;
}

static void give_stream_set(int dev, const StreamSet &s) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool[dev].push_back(s);
}

Handle::~Handle() {
    if (gexec) cudaGraphExecDestroy(gexec);
    gexec = nullptr;
    // the buffers are freed stream-ordered on the streams that allocated them
    // (the setup's side streams are idle): drain the handle's work first, so no
    // buffer goes back to the pool while a solve still reads it
    bool ok = !stream || cudaStreamSynchronize(stream) == cudaSuccess;
    for (int k = 0; k < kSides; k++) ok = ok && (!set.side[k] || cudaStreamSynchronize(set.side[k]) == cudaSuccess);
    levels.clear();
    xa.release(); xb.release(); vnat.release(); scal.release();
    partials.release(); counter.release(); result.release();
    if (arena.base) cudaFreeAsync(arena.base, stream);   // every arena buffer is gone (no-op frees)
    arena.base = nullptr;
    // idle streams go back to the pool (nothing of this handle is left on them)
    if (set.stream && ok) give_stream_set(device, set);
}

void convert_row_ptr(const int64_t *rp64_dev, int64_t n, int64_t nnz, int *rp32, cudaStream_t st);
int rowpass_grid();

thread_local SmallArena *tl_arena = nullptr;

// routes the small allocations of the enclosing scope (one fiedler_create) to an arena
struct ArenaScope {
    explicit ArenaScope(SmallArena *a) { tl_arena = a; }
    ~ArenaScope() { tl_arena = nullptr; }
};

// Orders the handle's own stream after the caller's stream on entry (the
// caller's inputs) and the caller's stream after the handle's on exit (the
// results): the work of one call looks stream-ordered on the caller's stream.
struct StreamJoin {
    cudaEvent_t ev;
    cudaStream_t user, own;
    StreamJoin(cudaEvent_t e, cudaStream_t u, cudaStream_t o) : ev(e), user(u && u != o ? u : nullptr), own(o) {
        if (!user) return;
        FDL_CK(cudaEventRecord(ev, user));
        FDL_CK(cudaStreamWaitEvent(own, ev, 0));
    }
    ~StreamJoin() {
        if (!user) return;
        if (cudaEventRecord(ev, own) == cudaSuccess) cudaStreamWaitEvent(user, ev, 0);
    }
};

// device time of one call between two timing events of the handle's set
struct EventTimer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t s;
    EventTimer(cudaStream_t st, const StreamSet &set) : a(set.tev[0]), b(set.tev[1]), s(st) {
        FDL_CK(cudaEventRecord(a, s));
    }
    double stop_ms() {
        FDL_CK(cudaEventRecord(b, s));
        cudaError_t e;
        while ((e = cudaEventQuery(b)) == cudaErrorNotReady) {   // poll: no sleeping host wake-up
        }
        FDL_CK(e);
        float ms = 0.f;
        FDL_CK(cudaEventElapsedTime(&ms, a, b));
        return ms;
    }
};

static void check_device(int dev) {
    // the capability check runs once per device (cudaGetDeviceProperties costs ~10 ms)
    static DeviceCache checked{};
    int count = 0;
    FDL_CK(cudaGetDeviceCount(&count));
    FDL_REQUIRE(dev >= 0 && dev < count && dev < 64, FIEDLER_ERR_CUDA, "no such CUDA device");
    FDL_CK(cudaSetDevice(dev));
    if (checked[dev]) return;
    int major = 0, minor = 0;
    FDL_CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    FDL_CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
    FDL_REQUIRE(major == 10, FIEDLER_ERR_CUDA,
                "libfiedler is built for sm_100a (B200); device is sm_" + std::to_string(major) +
                    std::to_string(minor));
    // this device's default pool keeps freed memory (release threshold = max)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    checked[dev].store(1);
}

// Grow the stream-ordered pool once to `need` bytes in one piece (the pool
// keeps freed memory: release threshold = max), so that later creates do not
// map new physical memory piecemeal in the middle of the setup.
#ifndef FDL_POOL_FACTOR
#define FDL_POOL_FACTOR 8.0
#endif
constexpr double kPoolFactor = FDL_POOL_FACTOR;
static void reserve_pool(int dev, size_t need, cudaStream_t st) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
    uint64_t reserved = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) != cudaSuccess) return;
    if (reserved >= need) return;
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return;
    need = std::min(need, (size_t)(fr * 0.6));
    void *p = nullptr;
    if (need > reserved && cudaMallocAsync(&p, need, st) == cudaSuccess) cudaFreeAsync(p, st);
    (void)cudaGetLastError();
}

static SolveCfg cfg_of(const fiedler_opts &o) {
    SolveCfg c;
    c.gs = o.gs_sweeps;
    c.pi = o.power_iters;
    c.piJ = o.coarsest_power_iters < 0 ? o.power_iters : o.coarsest_power_iters;
    c.seed = o.seed;
    return c;
}

int prepare_solve(Handle &h, const SolveCfg &cfg);

}  // namespace fdl

using namespace fdl;

extern "C" {

void fiedler_default_opts(fiedler_opts *o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->device = 0;
    o->coarsest_size = 25;
    o->max_levels = 50;
    o->gs_sweeps = 2;
    o->power_iters = 10;
    o->coarsest_power_iters = -1;
    o->validate = 1;
    o->use_graph = 1;
    o->seed = 0;
    o->stream = nullptr;
}

const char *fiedler_last_error(void) { return fdl::g_last_error.c_str(); }

int fiedler_create(int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col_idx,
                   const double *weights, int32_t mem, const fiedler_opts *opts,
                   fiedler_handle *out) {
    return fiedler_create_preset(n, nnz, row_ptr, col_idx, weights, mem, opts, 0, nullptr, out);
}

int fiedler_create_preset(int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col_idx,
                          const double *weights, int32_t mem, const fiedler_opts *opts, int32_t npreset,
                          const fiedler_preset_level *preset, fiedler_handle *out) {
    API_BEGIN
    fdl::set_error("");
    FDL_REQUIRE(out != nullptr, FIEDLER_ERR_ARG, "out is NULL");
    *out = nullptr;
    fiedler_opts o;
    if (opts) o = *opts; else fiedler_default_opts(&o);
    FDL_REQUIRE(n >= 2, FIEDLER_ERR_ARG, "need n >= 2");
    FDL_REQUIRE(nnz >= 0, FIEDLER_ERR_ARG, "nnz < 0");
    FDL_REQUIRE(n < (int64_t(1) << 31) - 1 && nnz < (int64_t(1) << 31) - 1, FIEDLER_ERR_TOO_LARGE,
                "n and nnz must be < 2^31 - 1 (int32 offsets)");
    FDL_REQUIRE(row_ptr && (nnz == 0 || (col_idx && weights)), FIEDLER_ERR_ARG, "NULL CSR pointer");
    FDL_REQUIRE(mem == FIEDLER_MEM_HOST || mem == FIEDLER_MEM_DEVICE, FIEDLER_ERR_ARG, "bad mem kind");
    FDL_REQUIRE(o.coarsest_size >= 2 && o.max_levels >= 1 && o.max_levels <= FIEDLER_MAX_LEVELS &&
                    o.gs_sweeps >= 0 && o.power_iters >= 0,
                FIEDLER_ERR_ARG, "invalid options");
    FDL_REQUIRE(npreset >= 0 && npreset < o.max_levels && (npreset == 0 || preset), FIEDLER_ERR_ARG,
                "npreset outside [0, max_levels - 1] or NULL preset");
    for (int l = 0; l < npreset; l++) {
        const fiedler_preset_level &P = preset[l];
        const int64_t nl = l == 0 ? n : preset[l - 1].n_next;
        FDL_REQUIRE(P.agg && P.mate && P.color && P.rp_next && (P.nnz_next == 0 || (P.ci_next && P.w_next)),
                    FIEDLER_ERR_ARG, "NULL preset array");
        FDL_REQUIRE(P.n_next >= 2 && P.n_next < nl && P.nnz_next >= 0 && P.nnz_next < (int64_t(1) << 31) - 1 &&
                        P.ncolors >= 1 && P.ncolors <= nl,
                    FIEDLER_ERR_ARG, "preset level sizes out of range");
    }
    trace_mark(nullptr, "create: enter");
    check_device(o.device);
    trace_mark(nullptr, "create: check_device");

    std::unique_ptr<Handle> h(new Handle());
    h->device = o.device;
    h->opts = o;
    h->preset.assign(preset, preset + npreset);
    // The handle always works on a stream of its own: every device buffer it
    // allocates is freed on that stream, which lives until fiedler_destroy.  A
    // caller's stream (opts->stream) is joined with events (StreamJoin).
    h->set = take_stream_set(o.device);
    h->stream = h->set.stream;
    h->stream2 = h->set.stream2;
    h->ev_join = h->set.ev[0];
    h->own_stream = true;
    cudaStream_t st = h->stream;
    StreamJoin join(h->ev_join, (cudaStream_t)o.stream, st);
    h->row_grid = rowpass_grid();
    EventTimer timer(st, h->set);

    if (!std::getenv("FIEDLER_NO_POOL_RESERVE"))
        reserve_pool(o.device, (size_t)(kPoolFactor * ((double)n * 12.0 + (double)nnz * 12.0)), st);
    // small-buffer arena of the setup: 4 MB + 128 B per vertex, at most 64 MB
    h->arena.cap = std::min<size_t>((size_t)64 << 20, ((size_t)4 << 20) + (size_t)n * 128);
    FDL_CK(cudaMallocAsync((void **)&h->arena.base, h->arena.cap, st));
    ArenaScope arena_scope(&h->arena);
    NatGraph g0;
    g0.n = (int)n;
    g0.nnz = (int)nnz;
    g0.own_rp.alloc(padded((size_t)(n + 1) * 4), st);
    if (mem == FIEDLER_MEM_DEVICE) {
        convert_row_ptr(row_ptr, n, nnz, g0.own_rp.as<int>(), st);
        g0.ci = col_idx;
        g0.w = weights;
        // the handle's own copy of the level-0 columns / weights (the power
        // steps' natural CSR, padded for the bulk copies), made on a side stream
        // while the setup reads the caller's arrays: it used to be a 3 GB copy
        // on the main stream at the end of the setup (config 4: ~1 ms)
        if (nnz) {
            cudaStream_t sd = h->set.side[kSides > 1 ? 1 : 0];
            FDL_CK(cudaEventRecord(h->set.ev[3], st));
            FDL_CK(cudaStreamWaitEvent(sd, h->set.ev[3], 0));
            g0.own_ci.alloc(padded((size_t)nnz * 4), sd);
            g0.own_w.alloc(padded((size_t)nnz * 8), sd);
            FDL_CK(cudaMemcpyAsync(g0.own_ci.p, col_idx, (size_t)nnz * 4, cudaMemcpyDeviceToDevice, sd));
            FDL_CK(cudaMemcpyAsync(g0.own_w.p, weights, (size_t)nnz * 8, cudaMemcpyDeviceToDevice, sd));
        }
    } else {
        DBuf rp64((size_t)(n + 1) * 8, st);
        FDL_CK(cudaMemcpyAsync(rp64.p, row_ptr, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, st));
        convert_row_ptr(rp64.as<int64_t>(), n, nnz, g0.own_rp.as<int>(), st);
        g0.own_ci.alloc(padded((size_t)std::max<int64_t>(nnz, 1) * 4), st);
        g0.own_w.alloc(padded((size_t)std::max<int64_t>(nnz, 1) * 8), st);
        if (nnz) {
            FDL_CK(cudaMemcpyAsync(g0.own_ci.p, col_idx, (size_t)nnz * 4, cudaMemcpyHostToDevice, st));
            // without validation the level-0 colouring (pattern only) may start
            // while the weights are still being copied
            if (!o.validate) {
                h->ev_pattern = h->set.ev[1];
                FDL_CK(cudaEventRecord(h->ev_pattern, st));
            }
            FDL_CK(cudaMemcpyAsync(g0.own_w.p, weights, (size_t)nnz * 8, cudaMemcpyHostToDevice, st));
        }
        g0.ci = g0.own_ci.as<int>();
        g0.w = g0.own_w.as<double>();
    }
    g0.rp = g0.own_rp.as<int>();
    if (o.validate) validate_input(n, nnz, g0.rp, g0.ci, g0.w, st);
    h->n0 = (int)n;
    trace_mark(st, "create: input staging");
    const long long l0 = g_launch_count;
    build_hierarchy(*h, std::move(g0));
    h->preset.clear();   // copied (build_hierarchy synchronises the stream)
    prepare_solve(*h, cfg_of(o));
    trace_mark(st, "create: prepare_solve");
    if (alloc_stats_enabled())
        std::fprintf(stderr, "[fiedler alloc] cudaMallocAsync %lld calls %.3f ms, cudaFreeAsync %lld calls %.3f ms (host, all threads)\n",
                     g_alloc_calls.exchange(0), g_alloc_ns.exchange(0) / 1e6, g_free_calls.exchange(0),
                     g_free_ns.exchange(0) / 1e6);
    if (trace_enabled()) {
        cudaMemPool_t pool;
        uint64_t hi = 0, res = 0;
        if (cudaDeviceGetDefaultMemPool(&pool, o.device) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &hi) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res) == cudaSuccess)
            std::fprintf(stderr, "[fiedler trace] pool: used high %.2f GB, reserved %.2f GB, input %.2f GB\n",
                         hi * 1e-9, res * 1e-9, ((double)n * 12.0 + (double)nnz * 12.0) * 1e-9);
    }
    h->setup_launches = (int)(g_launch_count - l0);
    h->setup_ms = timer.stop_ms();
    *out = reinterpret_cast<fiedler_handle>(h.release());
    return FIEDLER_OK;
    API_END
}

int fiedler_solve(fiedler_handle hh, const fiedler_opts *opts, double *vec, int32_t vec_mem,
                  double *lambda2, fiedler_info *info) {
    API_BEGIN
    fdl::set_error("");
    FDL_REQUIRE(hh != nullptr, FIEDLER_ERR_ARG, "NULL handle");
    Handle &h = *reinterpret_cast<Handle *>(hh);
    FDL_REQUIRE(vec_mem == FIEDLER_MEM_HOST || vec_mem == FIEDLER_MEM_DEVICE, FIEDLER_ERR_ARG,
                "bad mem kind");
    fiedler_opts o = opts ? *opts : h.opts;
    FDL_REQUIRE(o.gs_sweeps >= 0 && o.power_iters >= 0, FIEDLER_ERR_ARG, "invalid options");
    FDL_CK(cudaSetDevice(h.device));
    cudaStream_t st = h.stream;
    StreamJoin join(h.ev_join, opts ? (cudaStream_t)opts->stream : nullptr, st);
    SolveCfg cfg = cfg_of(o);
    prepare_solve(h, cfg);
    trace_mark(st, "solve: enter");
    EventTimer timer(st, h.set);
    int launches = 0;
    // The first solve of a handle (and of every new configuration) runs eagerly:
    // capturing and instantiating a graph costs more host time than it saves
    // once, and eager launches keep the tile passes' programmatic dependent
    // launches (measured: config 4 solve 30.7 ms via a fresh graph, 29.8 eager).
    // A repeated solve with the same configuration is captured and replayed.
    const bool same_cfg = h.g_gs == cfg.gs && h.g_pi == cfg.pi && h.g_piJ == cfg.piJ && h.g_seed == cfg.seed;
    const bool replay = o.use_graph && same_cfg && h.solves_same > 0;
    if (!same_cfg) {
        h.solves_same = 0;
        if (h.gexec) { cudaGraphExecDestroy(h.gexec); h.gexec = nullptr; }
    }
    h.g_gs = cfg.gs; h.g_pi = cfg.pi; h.g_piJ = cfg.piJ; h.g_seed = cfg.seed;
    h.solves_same++;
    if (replay) {
        if (!h.gexec) {
            cudaGraph_t g = nullptr;
            FDL_CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            try {
                launches = enqueue_solve(h, cfg);
            } catch (...) {
                cudaStreamEndCapture(st, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            FDL_CK(cudaStreamEndCapture(st, &g));
            cudaError_t e = cudaGraphInstantiate(&h.gexec, g, 0);
            cudaGraphDestroy(g);
            FDL_CK(e);
            h.g_launches = launches;
        }
        trace_mark(st, "solve: capture+instantiate");
        FDL_CK(cudaGraphLaunch(h.gexec, st));
        launches = h.g_launches;
    } else {
        launches = enqueue_solve(h, cfg);
    }
    if (vec) {
        FDL_CK(cudaMemcpyAsync(vec, h.vnat.p, (size_t)h.n0 * 8,
                               vec_mem == FIEDLER_MEM_HOST ? cudaMemcpyDeviceToHost
                                                           : cudaMemcpyDeviceToDevice, st));
    }
    double res[3] = {0, 0, 0};
    double ms = timer.stop_ms();
    readback(st, {{res, h.result.p, sizeof(res)}});
    trace_mark(st, "solve: run+copy");
    if (lambda2) *lambda2 = res[0];
    if (info) {
        std::memset(info, 0, sizeof(*info));
        info->num_levels = (int)h.levels.size();
        info->launches = launches;
        info->setup_launches = h.setup_launches;
        info->lambda2 = res[0];
        info->residual_norm = res[1];
        info->setup_ms = h.setup_ms;
        info->solve_ms = ms;
        for (size_t l = 0; l < h.levels.size() && l < FIEDLER_MAX_LEVELS; l++) {
            info->level_n[l] = h.levels[l].n;
            info->level_nnz[l] = h.levels[l].nnz;
            info->level_colors[l] = h.levels[l].ncolors;
            info->level_match_rounds[l] = h.levels[l].match_rounds;
            info->level_shift[l] = h.levels[l].shift;
            info->level_match_ms[l] = h.levels[l].phase_ms[0];
            info->level_galerkin_ms[l] = h.levels[l].phase_ms[1];
            info->level_colour_ms[l] = h.levels[l].phase_ms[2];
            info->level_layout_ms[l] = h.levels[l].phase_ms[3];
        }
    }
    return FIEDLER_OK;
    API_END
}

int fiedler_destroy(fiedler_handle hh) {
    API_BEGIN
    if (!hh) return FIEDLER_OK;
    Handle *h = reinterpret_cast<Handle *>(hh);
    cudaSetDevice(h->device);
    trace_mark(nullptr, "destroy: enter");
    delete h;
    trace_mark(nullptr, "destroy: done");
    return FIEDLER_OK;
    API_END
}

int fiedler_num_levels(fiedler_handle hh, int32_t *num_levels) {
    API_BEGIN
    FDL_REQUIRE(hh && num_levels, FIEDLER_ERR_ARG, "NULL argument");
    *num_levels = (int)reinterpret_cast<Handle *>(hh)->levels.size();
    return FIEDLER_OK;
    API_END
}

int fiedler_level_size(fiedler_handle hh, int32_t level, int64_t *n, int64_t *nnz, int32_t *colors) {
    API_BEGIN
    FDL_REQUIRE(hh, FIEDLER_ERR_ARG, "NULL handle");
    Handle &h = *reinterpret_cast<Handle *>(hh);
    FDL_REQUIRE(level >= 0 && level < (int)h.levels.size(), FIEDLER_ERR_ARG, "bad level");
    const Level &L = h.levels[level];
    if (n) *n = L.n;
    if (nnz) *nnz = L.nnz;
    if (colors) *colors = L.ncolors;
    return FIEDLER_OK;
    API_END
}

int fiedler_level_export(fiedler_handle hh, int32_t level, int64_t *row_ptr, int32_t *col_idx,
                         double *weights, int32_t *agg, int32_t *mate, int32_t *color) {
    API_BEGIN
    FDL_REQUIRE(hh, FIEDLER_ERR_ARG, "NULL handle");
    Handle &h = *reinterpret_cast<Handle *>(hh);
    FDL_REQUIRE(level >= 0 && level < (int)h.levels.size(), FIEDLER_ERR_ARG, "bad level");
    FDL_CK(cudaSetDevice(h.device));
    const Level &L = h.levels[level];
    cudaStream_t st = h.stream;
    const int n = L.n, nnz = L.nnz;
    std::vector<int> perm(n), inv(n), rp(n + 1), ci(std::max(nnz, 1));
    std::vector<double> w(std::max(nnz, 1));
    FDL_CK(cudaMemcpyAsync(perm.data(), L.perm.p, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaMemcpyAsync(inv.data(), L.inv.p, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    FDL_CK(cudaMemcpyAsync(rp.data(), L.rp.p, (size_t)(n + 1) * 4, cudaMemcpyDeviceToHost, st));
    if (nnz) {
        FDL_CK(cudaMemcpyAsync(ci.data(), L.ci.p, (size_t)nnz * 4, cudaMemcpyDeviceToHost, st));
        FDL_CK(cudaMemcpyAsync(w.data(), L.w.p, (size_t)nnz * 8, cudaMemcpyDeviceToHost, st));
    }
    auto copy_nat = [&](const DBuf &b, int32_t *dst) {
        if (!dst) return;
        if (b.p) FDL_CK(cudaMemcpyAsync(dst, b.p, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
        else std::fill(dst, dst + n, -1);
    };
    copy_nat(L.q_nat, agg);
    copy_nat(L.mate_nat, mate);
    copy_nat(L.color_nat, color);
    FDL_CK(cudaStreamSynchronize(st));
    // un-permute (introspection only): natural row v = solve row inv[v]; the
    // within-row order of the solve layout is the natural ascending order
    int64_t off = 0;
    for (int v = 0; v < n; v++) {
        if (row_ptr) row_ptr[v] = off;
        int t = inv[v];
        for (int k = rp[t]; k < rp[t + 1]; k++, off++) {
            if (col_idx) col_idx[off] = perm[ci[k]];
            if (weights) weights[off] = w[k];
        }
    }
    if (row_ptr) row_ptr[n] = off;
    return FIEDLER_OK;
    API_END
}

int fiedler_level_time(fiedler_handle hh, int32_t level, int32_t op, int32_t reps,
                       double *ms_per_rep, double *bytes_per_rep) {
    API_BEGIN
    FDL_REQUIRE(hh && ms_per_rep && reps > 0, FIEDLER_ERR_ARG, "bad argument");
    Handle &h = *reinterpret_cast<Handle *>(hh);
    FDL_REQUIRE(level >= 0 && level < (int)h.levels.size(), FIEDLER_ERR_ARG, "bad level");
    FDL_REQUIRE(op == FIEDLER_OP_GS_SWEEPS || op == FIEDLER_OP_POWER || op == FIEDLER_OP_RAYLEIGH,
                FIEDLER_ERR_ARG, "bad op");
    FDL_CK(cudaSetDevice(h.device));
    time_level_op(h, level, op, reps, ms_per_rep, bytes_per_rep);
    return FIEDLER_OK;
    API_END
}

int fiedler_level_apply(fiedler_handle hh, int32_t level, int32_t op, int32_t count,
                        const double *x_in, double *x_out, int32_t mem, double *scalar_out) {
    API_BEGIN
    FDL_REQUIRE(hh && x_in, FIEDLER_ERR_ARG, "NULL argument");
    Handle &h = *reinterpret_cast<Handle *>(hh);
    const int nl = (int)h.levels.size();
    FDL_REQUIRE(level >= 0 && level < nl, FIEDLER_ERR_ARG, "bad level");
    FDL_REQUIRE(op >= 1 && op <= 4 && count >= 0, FIEDLER_ERR_ARG, "bad op/count");
    FDL_REQUIRE(op != FIEDLER_OP_PROLONG || level + 1 < nl, FIEDLER_ERR_ARG, "no coarser level");
    FDL_REQUIRE(op == FIEDLER_OP_RAYLEIGH || x_out, FIEDLER_ERR_ARG, "x_out is NULL");
    FDL_CK(cudaSetDevice(h.device));
    cudaStream_t st = h.stream;
    const int n_out = h.levels[level].n;
    const int n_in = op == FIEDLER_OP_PROLONG ? h.levels[level + 1].n : n_out;
    DBuf din, dout;
    const double *pin = x_in;
    double *pout = x_out;
    if (mem == FIEDLER_MEM_HOST) {
        din.alloc((size_t)n_in * 8, st);
        dout.alloc((size_t)n_out * 8, st);
        FDL_CK(cudaMemcpyAsync(din.p, x_in, (size_t)n_in * 8, cudaMemcpyHostToDevice, st));
        pin = din.as<double>();
        pout = dout.as<double>();
    }
    apply_level_op(h, level, op, count, pin, pout, scalar_out);
    if (mem == FIEDLER_MEM_HOST && x_out && op != FIEDLER_OP_RAYLEIGH) {
        FDL_CK(cudaMemcpyAsync(x_out, dout.p, (size_t)n_out * 8, cudaMemcpyDeviceToHost, st));
        FDL_CK(cudaStreamSynchronize(st));
    }
    return FIEDLER_OK;
    API_END
}

int fiedler_dist_plan(fiedler_handle hh, int32_t level, int32_t nranks, int32_t rank,
                      fiedler_dist_plan_info *info) {
    API_BEGIN
    FDL_REQUIRE(hh, FIEDLER_ERR_ARG, "NULL handle");
    Handle &h = *reinterpret_cast<Handle *>(hh);
    FDL_REQUIRE(level >= 0 && level < (int)h.levels.size(), FIEDLER_ERR_ARG, "bad level");
    FDL_REQUIRE(nranks >= 1 && nranks <= FIEDLER_MAX_RANKS && rank >= 0 && rank < nranks, FIEDLER_ERR_ARG,
                "bad nranks / rank");
    FDL_CK(cudaSetDevice(h.device));
    dist_plan(h, level, nranks, rank, info);
    return FIEDLER_OK;
    API_END
}

int fiedler_dist_op(fiedler_handle hh, int32_t level, int32_t op, int64_t arg, const double *x, double *y,
                    double *stat, const double *stat_in, const double *sign_slot, void *stream) {
    API_BEGIN
    FDL_REQUIRE(hh, FIEDLER_ERR_ARG, "NULL handle");
    Handle &h = *reinterpret_cast<Handle *>(hh);
    FDL_REQUIRE(level >= 0 && level < (int)h.levels.size(), FIEDLER_ERR_ARG, "bad level");
    dist_op(h, level, op, arg, x, y, stat, stat_in, sign_slot, stream ? (cudaStream_t)stream : h.stream);
    return FIEDLER_OK;
    API_END
}

}  // extern "C"

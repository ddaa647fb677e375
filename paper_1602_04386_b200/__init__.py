"""paper_1602_04386_b200 -- B200-native cascadic-multigrid Fiedler solver.

Thin ctypes binding of ``libfiedler.so`` (C ABI in ``include/fiedler.h``).
Every function here only marshals arguments; all work runs in the library's
sm_100a kernels.  There is no CPU fallback: if the library is missing or no
B200 is visible the calls raise.

C-ABI names are kept (``fiedler_create``, ``fiedler_solve``, ...).  Arrays may
be numpy arrays (host memory) or torch tensors (host or CUDA memory); their
dtypes must be int64 (row_ptr), int32 (col_idx) and float64 (weights/vectors).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FIEDLER_LIB overrides the library (tuning sweeps of build variants only)
LIB_PATH = os.environ.get("FIEDLER_LIB") or os.path.join(_HERE, "libfiedler.so")

FIEDLER_OK = 0
FIEDLER_ERR_ARG = -1
FIEDLER_ERR_GRAPH = -2
FIEDLER_ERR_DISCONNECTED = -3
FIEDLER_ERR_CUDA = -4
FIEDLER_ERR_NOMEM = -5
FIEDLER_ERR_INTERNAL = -6
FIEDLER_ERR_TOO_LARGE = -7
FIEDLER_MEM_HOST = 0
FIEDLER_MEM_DEVICE = 1
FIEDLER_MAX_LEVELS = 64
FIEDLER_OP_GS_SWEEPS = 1
FIEDLER_OP_POWER = 2
FIEDLER_OP_PROLONG = 3
FIEDLER_OP_RAYLEIGH = 4

FIEDLER_MAX_RANKS = 64
FIEDLER_DOP_RAND = 1
FIEDLER_DOP_PROLONG = 2
FIEDLER_DOP_GS_COLOUR = 3
FIEDLER_DOP_TO_NAT = 4
FIEDLER_DOP_POWER = 5
FIEDLER_DOP_FINALISE = 6
FIEDLER_DOP_FIRST_NONZERO = 7
FIEDLER_DOP_SIGN = 8
FIEDLER_DOP_RAYLEIGH = 9
FIEDLER_DOP_FINALISE_RQ = 10
FIEDLER_DOP_HALO_PACK = 11
FIEDLER_DOP_HALO_UNPACK = 12

EXPORTED = ("fiedler_default_opts", "fiedler_create", "fiedler_solve", "fiedler_destroy",
            "fiedler_last_error", "fiedler_num_levels", "fiedler_level_size",
            "fiedler_level_export", "fiedler_level_apply", "fiedler_level_time",
            "fiedler_dist_plan", "fiedler_dist_op", "fiedler_pset_bounds", "fiedler_pset_halo",
            "fiedler_pset_gather", "fiedler_pset_scatter", "fiedler_pset_match", "fiedler_pset_aggregate",
            "fiedler_pset_galerkin", "fiedler_pset_colour", "fiedler_create_preset")

FIEDLER_PSET_POINT = 0
FIEDLER_PSET_RESOLVE = 1
FIEDLER_PSET_LEADERS = 0
FIEDLER_PSET_IDS = 1
FIEDLER_PSET_MATES = 2
FIEDLER_PSET_JOIN = 3


class fiedler_opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("coarsest_size", ctypes.c_int32),
                ("max_levels", ctypes.c_int32), ("gs_sweeps", ctypes.c_int32),
                ("power_iters", ctypes.c_int32), ("coarsest_power_iters", ctypes.c_int32),
                ("validate", ctypes.c_int32), ("use_graph", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("stream", ctypes.c_void_p)]


class fiedler_info(ctypes.Structure):
    _fields_ = [("num_levels", ctypes.c_int32), ("launches", ctypes.c_int32),
                ("setup_launches", ctypes.c_int32),
                ("lambda2", ctypes.c_double), ("residual_norm", ctypes.c_double),
                ("setup_ms", ctypes.c_double), ("solve_ms", ctypes.c_double),
                ("level_n", ctypes.c_int64 * FIEDLER_MAX_LEVELS),
                ("level_nnz", ctypes.c_int64 * FIEDLER_MAX_LEVELS),
                ("level_colors", ctypes.c_int32 * FIEDLER_MAX_LEVELS),
                ("level_match_rounds", ctypes.c_int32 * FIEDLER_MAX_LEVELS),
                ("level_shift", ctypes.c_double * FIEDLER_MAX_LEVELS),
                ("level_match_ms", ctypes.c_double * FIEDLER_MAX_LEVELS),
                ("level_galerkin_ms", ctypes.c_double * FIEDLER_MAX_LEVELS),
                ("level_colour_ms", ctypes.c_double * FIEDLER_MAX_LEVELS),
                ("level_layout_ms", ctypes.c_double * FIEDLER_MAX_LEVELS)]

    def levels(self):
        return [dict(n=self.level_n[i], nnz=self.level_nnz[i], colors=self.level_colors[i],
                     match_rounds=self.level_match_rounds[i], shift=self.level_shift[i],
                     match_ms=self.level_match_ms[i], galerkin_ms=self.level_galerkin_ms[i],
                     colour_ms=self.level_colour_ms[i], layout_ms=self.level_layout_ms[i])
                for i in range(self.num_levels)]


class fiedler_dist_plan_info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nranks", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("colors", ctypes.c_int32),
                ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("row_bounds", ctypes.c_int64 * (FIEDLER_MAX_RANKS + 1)),
                ("send_count", ctypes.c_int64 * FIEDLER_MAX_RANKS),
                ("recv_count", ctypes.c_int64 * FIEDLER_MAX_RANKS),
                ("send_total", ctypes.c_int64), ("recv_total", ctypes.c_int64)]


class fiedler_preset_level(ctypes.Structure):
    _fields_ = [("agg", ctypes.c_void_p), ("mate", ctypes.c_void_p), ("color", ctypes.c_void_p),
                ("ncolors", ctypes.c_int32), ("match_rounds", ctypes.c_int32),
                ("colour_rounds", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("n_next", ctypes.c_int64), ("nnz_next", ctypes.c_int64),
                ("rp_next", ctypes.c_void_p), ("ci_next", ctypes.c_void_p), ("w_next", ctypes.c_void_p)]


class FiedlerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("libfiedler error %d: %s" % (code, msg))
        self.code = code


_lib = None


def library_path() -> str:
    return LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libfiedler.so is not built (run __graft_entry__.build() or "
                               "python paper_1602_04386_b200/build.py); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        lib.fiedler_default_opts.restype = None
        lib.fiedler_default_opts.argtypes = [ctypes.POINTER(fiedler_opts)]
        lib.fiedler_create.restype = ctypes.c_int
        lib.fiedler_create.argtypes = [i64, i64, P, P, P, i32, ctypes.POINTER(fiedler_opts), ctypes.POINTER(P)]
        lib.fiedler_solve.restype = ctypes.c_int
        lib.fiedler_solve.argtypes = [P, ctypes.POINTER(fiedler_opts), P, i32, ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(fiedler_info)]
        lib.fiedler_destroy.restype = ctypes.c_int
        lib.fiedler_destroy.argtypes = [P]
        lib.fiedler_last_error.restype = ctypes.c_char_p
        lib.fiedler_last_error.argtypes = []
        lib.fiedler_num_levels.restype = ctypes.c_int
        lib.fiedler_num_levels.argtypes = [P, ctypes.POINTER(i32)]
        lib.fiedler_level_size.restype = ctypes.c_int
        lib.fiedler_level_size.argtypes = [P, i32, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i32)]
        lib.fiedler_level_export.restype = ctypes.c_int
        lib.fiedler_level_export.argtypes = [P, i32, P, P, P, P, P, P]
        lib.fiedler_level_time.restype = ctypes.c_int
        lib.fiedler_level_time.argtypes = [P, i32, i32, i32, ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(ctypes.c_double)]
        lib.fiedler_dist_plan.restype = ctypes.c_int
        lib.fiedler_dist_plan.argtypes = [P, i32, i32, i32, ctypes.POINTER(fiedler_dist_plan_info)]
        lib.fiedler_dist_op.restype = ctypes.c_int
        lib.fiedler_dist_op.argtypes = [P, i32, i32, i64, P, P, P, P, P, P]
        u64 = ctypes.c_uint64
        i64p = ctypes.POINTER(i64)
        lib.fiedler_pset_bounds.argtypes = [i64, P, i32, i64p, P]
        lib.fiedler_pset_halo.argtypes = [i64, P, P, i32, i32, i64p, P, i64p, P]
        lib.fiedler_pset_gather.argtypes = [P, P, i64, P, P]
        lib.fiedler_pset_scatter.argtypes = [P, P, i64, P, P]
        lib.fiedler_pset_match.argtypes = [i32, i64, P, P, P, i64, i64, u64, i32, P, P, i32, P, i64p, P]
        lib.fiedler_pset_aggregate.argtypes = [i32, i64, P, P, P, i64, i64, u64, i32, P, P, i64, i64p, P]
        lib.fiedler_pset_galerkin.argtypes = [i32, i64, P, P, P, P, i64, i64, i64, P, P, P, i64p, P]
        lib.fiedler_pset_colour.argtypes = [i64, P, P, i64, i64, u64, i32, i32, P, P, i64p, P]
        lib.fiedler_create_preset.argtypes = [i64, i64, P, P, P, i32, ctypes.POINTER(fiedler_opts), i32,
                                              ctypes.POINTER(fiedler_preset_level), ctypes.POINTER(P)]
        for f in ("fiedler_pset_bounds", "fiedler_pset_halo", "fiedler_pset_gather", "fiedler_pset_scatter",
                  "fiedler_pset_match", "fiedler_pset_aggregate", "fiedler_pset_galerkin",
                  "fiedler_pset_colour", "fiedler_create_preset"):
            getattr(lib, f).restype = ctypes.c_int
        lib.fiedler_level_apply.restype = ctypes.c_int
        lib.fiedler_level_apply.argtypes = [P, i32, i32, i32, P, P, i32, ctypes.POINTER(ctypes.c_double)]
        _lib = lib
    return _lib


def _check(code):
    if code != FIEDLER_OK:
        raise FiedlerError(code, _load().fiedler_last_error().decode())


def _ptr(a, dtype):
    """(pointer, mem kind) of a contiguous numpy array or torch tensor."""
    if a is None:
        return None, None
    if isinstance(a, np.ndarray):
        if a.dtype != np.dtype(dtype) or not a.flags.c_contiguous:
            raise TypeError("expected contiguous %s array" % np.dtype(dtype))
        return a.ctypes.data, FIEDLER_MEM_HOST
    try:
        import torch
    except ImportError:  # pragma: no cover
        raise TypeError("unsupported array type %r" % type(a))
    if isinstance(a, torch.Tensor):
        tdt = {np.int64: torch.int64, np.int32: torch.int32, np.float64: torch.float64}[np.dtype(dtype).type]
        if a.dtype != tdt or not a.is_contiguous():
            raise TypeError("expected contiguous %s tensor" % tdt)
        return a.data_ptr(), (FIEDLER_MEM_DEVICE if a.is_cuda else FIEDLER_MEM_HOST)
    raise TypeError("unsupported array type %r" % type(a))


def fiedler_default_opts(**overrides) -> fiedler_opts:
    o = fiedler_opts()
    _load().fiedler_default_opts(ctypes.byref(o))
    for k, v in overrides.items():
        setattr(o, k, v)
    return o


def fiedler_last_error() -> str:
    return _load().fiedler_last_error().decode()


def fiedler_create(n, nnz, row_ptr, col_idx, weights, opts: fiedler_opts = None):
    """Setup Phase (Algorithm 3 Step 1).  Returns an opaque handle (int)."""
    prp, m0 = _ptr(row_ptr, np.int64)
    pci, m1 = _ptr(col_idx, np.int32)
    pw, m2 = _ptr(weights, np.float64)
    if len({m0, m1, m2}) != 1:
        raise ValueError("row_ptr, col_idx and weights must live in the same memory")
    h = ctypes.c_void_p()
    _check(_load().fiedler_create(int(n), int(nnz), prp, pci, pw, m0,
                                  ctypes.byref(opts) if opts is not None else None, ctypes.byref(h)))
    return h.value


def fiedler_solve(handle, vector=None, opts: fiedler_opts = None, info: fiedler_info = None):
    """Steps 2-3 + Rayleigh quotient.  Writes the Fiedler vector into `vector`
    (if given) and returns lambda2."""
    pv, mv = _ptr(vector, np.float64)
    lam = ctypes.c_double()
    _check(_load().fiedler_solve(handle, ctypes.byref(opts) if opts is not None else None, pv,
                                 mv if mv is not None else FIEDLER_MEM_HOST, ctypes.byref(lam),
                                 ctypes.byref(info) if info is not None else None))
    return lam.value


def fiedler_destroy(handle):
    _check(_load().fiedler_destroy(handle))


def fiedler_num_levels(handle) -> int:
    k = ctypes.c_int32()
    _check(_load().fiedler_num_levels(handle, ctypes.byref(k)))
    return k.value


def fiedler_level_size(handle, level):
    n, nnz, col = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    _check(_load().fiedler_level_size(handle, level, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(col)))
    return n.value, nnz.value, col.value


def fiedler_level_export(handle, level):
    """Level `level` in natural numbering: dict(rp, ci, w, agg, mate, color) (numpy)."""
    n, nnz, _ = fiedler_level_size(handle, level)
    out = dict(rp=np.empty(n + 1, np.int64), ci=np.empty(max(nnz, 1), np.int32),
               w=np.empty(max(nnz, 1), np.float64), agg=np.empty(n, np.int32),
               mate=np.empty(n, np.int32), color=np.empty(n, np.int32))
    _check(_load().fiedler_level_export(handle, level, *[out[k].ctypes.data for k in
                                                          ("rp", "ci", "w", "agg", "mate", "color")]))
    out["ci"] = out["ci"][:nnz]
    out["w"] = out["w"][:nnz]
    out["n"] = n
    return out


def fiedler_level_apply(handle, level, op, x_in, x_out=None, count=1):
    """One solve-phase operation on `level` (natural numbering).  Returns the
    two scalars of the C call; writes x_out (same memory kind as x_in)."""
    pin, mi = _ptr(x_in, np.float64)
    pout, mo = _ptr(x_out, np.float64)
    if pout is not None and mo != mi:
        raise ValueError("x_in and x_out must live in the same memory")
    sc = (ctypes.c_double * 2)()
    _check(_load().fiedler_level_apply(handle, level, op, count, pin, pout, mi, sc))
    return sc[0], sc[1]


def fiedler_level_time(handle, level, op, reps=20):
    """(ms per rep, algorithmic bytes per rep) of one hot kernel (CUDA events)."""
    ms, by = ctypes.c_double(), ctypes.c_double()
    _check(_load().fiedler_level_time(handle, level, op, reps, ctypes.byref(ms), ctypes.byref(by)))
    return ms.value, by.value


def fiedler_dist_plan(handle, level, nranks, rank) -> fiedler_dist_plan_info:
    """Row partition + halo plan of `level` for (nranks, rank) (include/fiedler.h)."""
    info = fiedler_dist_plan_info()
    _check(_load().fiedler_dist_plan(handle, level, nranks, rank, ctypes.byref(info)))
    return info


def fiedler_dist_op(handle, level, op, arg=0, x=None, y=None, stat=None, stat_in=None, sign_slot=None,
                    stream=None):
    """Enqueue one partitioned-solve operation; array arguments are CUDA tensors
    (float64) or raw device pointers, `stream` a cudaStream_t (int) or None."""
    def ptr(t):
        if t is None:
            return None
        if isinstance(t, int):
            return t
        if t.dtype.itemsize != 8 or not t.is_cuda or not t.is_contiguous():
            raise TypeError("expected a contiguous CUDA float64 tensor")
        return t.data_ptr()
    _check(_load().fiedler_dist_op(handle, level, op, int(arg), ptr(x), ptr(y), ptr(stat), ptr(stat_in),
                                   ptr(sign_slot), stream))


# ---------------------------------------------------------------- partitioned setup
def _dptr(t, itemsize=None):
    """Device pointer of a contiguous CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous() or (itemsize and t.dtype.itemsize != itemsize):
        raise TypeError("expected a contiguous CUDA tensor of %s-byte items" % itemsize)
    return t.data_ptr()


def fiedler_pset_bounds(n, row_ptr, nranks, stream=None):
    """Row bounds [nranks + 1] of the rows + nonzeros balanced partition (list of int)."""
    b = (ctypes.c_int64 * (nranks + 1))()
    _check(_load().fiedler_pset_bounds(int(n), _dptr(row_ptr, 8), int(nranks), b, stream))
    return list(b)


def fiedler_pset_halo(n, row_ptr, col_idx, nranks, rank, bounds, send_idx=None, stream=None):
    """Send counts per peer (list); fills send_idx (CUDA int32) when given."""
    b = (ctypes.c_int64 * (nranks + 1))(*bounds)
    c = (ctypes.c_int64 * nranks)()
    _check(_load().fiedler_pset_halo(int(n), _dptr(row_ptr, 8), _dptr(col_idx, 4), int(nranks), int(rank), b,
                                     _dptr(send_idx, 4), c, stream))
    return list(c)


def fiedler_pset_gather(x, idx, count, out, stream=None):
    _check(_load().fiedler_pset_gather(_dptr(x, 4), _dptr(idx, 4), int(count), _dptr(out, 4), stream))


def fiedler_pset_scatter(inp, idx, count, x, stream=None):
    _check(_load().fiedler_pset_scatter(_dptr(inp, 4), _dptr(idx, 4), int(count), _dptr(x, 4), stream))


def fiedler_pset_match(phase, n, rp, ci, w, r0, r1, seed, level, mate, ptr, round=0, work=None, stream=None):
    """One matching half-round; returns the active count for POINT (else 0)."""
    a = ctypes.c_int64(0)
    _check(_load().fiedler_pset_match(int(phase), int(n), _dptr(rp, 8), _dptr(ci, 4), _dptr(w, 8), int(r0),
                                      int(r1), int(seed) & (2**64 - 1), int(level), _dptr(mate, 4), _dptr(ptr, 4),
                                      int(round), _dptr(work, 4), ctypes.byref(a), stream))
    return a.value


def fiedler_pset_aggregate(phase, n, rp, ci, w, r0, r1, seed, level, mate, q, offset=0, stream=None):
    """One aggregate-numbering phase; returns the own leader count for LEADERS / IDS."""
    c = ctypes.c_int64(0)
    _check(_load().fiedler_pset_aggregate(int(phase), int(n), _dptr(rp, 8), _dptr(ci, 4), _dptr(w, 8), int(r0),
                                          int(r1), int(seed) & (2**64 - 1), int(level), _dptr(mate, 4),
                                          _dptr(q, 4), int(offset), ctypes.byref(c), stream))
    return c.value


def fiedler_pset_galerkin(phase, n, rp, ci, w, q, a0, a1, cap=0, crp=None, cci=None, cw=None, stream=None):
    """Phase 0: contribution count; phase 1: coarse rows [a0, a1) into crp / cci / cw, returns their nnz."""
    c = ctypes.c_int64(0)
    _check(_load().fiedler_pset_galerkin(int(phase), int(n), _dptr(rp, 8), _dptr(ci, 4), _dptr(w, 8), _dptr(q, 4),
                                         int(a0), int(a1), int(cap), _dptr(crp, 8), _dptr(cci, 4), _dptr(cw, 8),
                                         ctypes.byref(c), stream))
    return c.value


def fiedler_pset_colour(n, rp, ci, r0, r1, seed, level, colour, round=0, work=None, stream=None):
    """One Jones-Plassmann round; returns (own rows left uncoloured, largest colour given)."""
    out = (ctypes.c_int64 * 2)()
    _check(_load().fiedler_pset_colour(int(n), _dptr(rp, 8), _dptr(ci, 4), int(r0), int(r1),
                                       int(seed) & (2**64 - 1), int(level), int(round), _dptr(work, 4),
                                       _dptr(colour, 4), out, stream))
    return out[0], out[1]


def fiedler_create_preset(n, nnz, row_ptr, col_idx, weights, opts, presets):
    """fiedler_create with levels 0..len(presets)-1 given (fiedler_preset_level list)."""
    prp, m0 = _ptr(row_ptr, np.int64)
    pci, m1 = _ptr(col_idx, np.int32)
    pw, m2 = _ptr(weights, np.float64)
    if len({m0, m1, m2}) != 1:
        raise ValueError("row_ptr, col_idx and weights must live in the same memory")
    arr = (fiedler_preset_level * max(len(presets), 1))(*presets)
    h = ctypes.c_void_p()
    _check(_load().fiedler_create_preset(int(n), int(nnz), prp, pci, pw, m0,
                                         ctypes.byref(opts) if opts is not None else None, len(presets),
                                         arr if presets else None, ctypes.byref(h)))
    return h.value


class FiedlerSolver:
    """Convenience owner of a handle (marshalling only)."""

    def __init__(self, n, row_ptr, col_idx, weights, **opts):
        self.opts = fiedler_default_opts(**opts)
        nnz = int(col_idx.shape[0])
        self.n = int(n)
        self.handle = fiedler_create(n, nnz, row_ptr, col_idx, weights, self.opts)

    def solve(self, vector=None, info=None, **opts):
        o = None
        if opts:
            o = fiedler_opts.from_buffer_copy(self.opts)
            for k, v in opts.items():
                setattr(o, k, v)
        return fiedler_solve(self.handle, vector, o, info)

    def close(self):
        if self.handle:
            fiedler_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

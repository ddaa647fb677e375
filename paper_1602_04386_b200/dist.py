"""Row-partitioned Fiedler solve across ranks (one process per GPU).

DESIGN.md section 9.  Every rank holds the whole hierarchy (``fiedler_create``
is deterministic, so all ranks build the same one).  Levels with at least
``min_rows`` vertices are partitioned: rank r owns a contiguous range of
natural rows and runs every pass (prolongation, Gauss-Seidel colour passes,
power steps, Rayleigh quotient) on its own rows only; coarser levels are
computed whole on every rank ("gathered").  Between passes the ranks

  * exchange halos (values of own rows that other ranks read -> their ghost
    rows) with one all-to-all per pass,
  * all-reduce the pass statistics (sums for the lazy deflation /
    normalisation of R5, the Rayleigh-quotient sums) and finalise them,
  * all-gather a partitioned level's final vector before the next finer level.

This module is orchestration only: the arithmetic runs in libfiedler's
kernels (``fiedler_dist_op``, an ``Ops`` object) and the bytes move through a
``Comm`` object (``TorchComm``: torch.distributed -- NCCL on GPUs, gloo on the
CPU test rig).  ``Ops`` / ``Comm`` are interfaces so the same driver runs the
CPU multi-process tests (tests/test_dist_cpu.py) with a reference ``Ops``.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import List, Optional

import torch

from . import (FIEDLER_DOP_FINALISE, FIEDLER_DOP_FINALISE_RQ, FIEDLER_DOP_FIRST_NONZERO,
               FIEDLER_DOP_GS_COLOUR, FIEDLER_DOP_HALO_PACK, FIEDLER_DOP_HALO_UNPACK,
               FIEDLER_DOP_POWER, FIEDLER_DOP_PROLONG, FIEDLER_DOP_RAND, FIEDLER_DOP_RAYLEIGH,
               FIEDLER_DOP_SIGN, FIEDLER_DOP_TO_NAT)

NATURAL, GS = 0, 1


@dataclass
class Plan:
    """Row partition + halo plan of one level for one rank."""
    n: int
    colors: int
    nranks: int
    rank: int
    row_begin: int
    row_end: int
    bounds: List[int]
    send_count: List[int]
    recv_count: List[int]

    @property
    def send_total(self) -> int:
        return sum(self.send_count)

    @property
    def recv_total(self) -> int:
        return sum(self.recv_count)


class Comm:
    """Collectives used by the driver (all in place on 1-D float64 tensors)."""
    nranks = 1
    rank = 0

    def allreduce_sum(self, t):  # pragma: no cover - interface
        raise NotImplementedError

    def allreduce_min(self, t):  # pragma: no cover - interface
        raise NotImplementedError

    def all_to_all(self, out, inp, out_splits, in_splits):  # pragma: no cover - interface
        raise NotImplementedError

    def allgatherv(self, out, inp, sizes):
        """out = concatenation over ranks of every rank's `inp` (rank k's has
        sizes[k] items).  Default: one all-to-all with the input repeated."""
        rep = inp.unsqueeze(0).expand(self.nranks, inp.numel()).reshape(-1) if inp.numel() else inp
        self.all_to_all(out, rep.contiguous(), list(sizes), [inp.numel()] * self.nranks)


class TorchComm(Comm):
    """torch.distributed process group (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.nranks = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allreduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def allreduce_min(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)

    def all_to_all(self, out, inp, out_splits, in_splits):
        self.dist.all_to_all_single(out, inp, output_split_sizes=list(out_splits),
                                    input_split_sizes=list(in_splits), group=self.group)

    def allgatherv(self, out, inp, sizes):
        # equal-size all-gather of the inputs padded to the largest, then compaction
        m = max(sizes)
        pad = torch.zeros(max(m, 1), dtype=inp.dtype, device=inp.device)
        pad[:inp.numel()] = inp
        parts = [torch.empty_like(pad) for _ in range(self.nranks)]
        self.dist.all_gather(parts, pad, group=self.group)
        o = 0
        for k, sz in enumerate(sizes):
            out[o:o + sz] = parts[k][:sz]
            o += sz


class LocalComm(Comm):
    """Single rank: every collective is the identity."""

    def allreduce_sum(self, t):
        pass

    def allreduce_min(self, t):
        pass

    def all_to_all(self, out, inp, out_splits, in_splits):
        out.copy_(inp)

    def allgatherv(self, out, inp, sizes):
        out[:inp.numel()] = inp


_OWN_STREAMS = {}


def _own_stream(device, stream):
    """The torch stream the library calls of an Ops object are issued on.  A
    NULL / default stream (0) is not passed to the library: its C ABI reads
    NULL as "the handle's own stream" (fiedler_dist_op) or "no caller stream
    to join" (fiedler_create), which would not be ordered with torch's work on
    the legacy default stream; such callers get a stream of their own, joined
    with theirs by _Joined."""
    if stream is None or stream == 0:
        # one such stream per device and host thread, reused by every Ops object:
        # torch's caching allocator pools freed blocks per stream, so a fresh
        # stream per solve would find none of the previous solve's buffers
        # (measured: +512 MiB reserved and one cudaMalloc per sharded step)
        key = (str(device), threading.get_ident())
        s = _OWN_STREAMS.get(key)
        if s is None:
            s = _OWN_STREAMS[key] = torch.cuda.Stream(device)
        return s
    return torch.cuda.ExternalStream(stream)


class _Joined:
    """Enter: the Ops stream waits for the caller's current stream and becomes
    current.  Exit: the caller's stream waits for the Ops stream."""

    def __init__(self, s):
        self.s = s

    def __enter__(self):
        self.caller = torch.cuda.current_stream(self.s.device)
        self.s.wait_stream(self.caller)
        self.ctx = torch.cuda.stream(self.s)
        self.ctx.__enter__()
        return self

    def __exit__(self, *exc):
        self.ctx.__exit__(*exc)
        self.caller.wait_stream(self.s)
        return False


class LibOps:
    """Ops backed by libfiedler (fiedler_dist_plan / fiedler_dist_op) on one GPU."""

    def __init__(self, handle, device, stream=None):
        from . import fiedler_level_size, fiedler_num_levels
        self.h = handle
        self.device = device
        # library kernels and torch's tensor work (allocation, zero-fill, slicing,
        # collectives) are ordered by running both on one (non-default) stream:
        # the driver enters stream_ctx() around the solve
        self.torch_stream = _own_stream(device, stream)
        self.stream = self.torch_stream.cuda_stream
        self.num_levels = fiedler_num_levels(handle)
        self.sizes = [fiedler_level_size(handle, l)[0] for l in range(self.num_levels)]

    def stream_ctx(self):
        return _Joined(self.torch_stream)

    def plan(self, level, nranks, rank) -> Plan:
        from . import fiedler_dist_plan
        i = fiedler_dist_plan(self.h, level, nranks, rank)
        return Plan(n=i.n, colors=i.colors, nranks=i.nranks, rank=i.rank, row_begin=i.row_begin,
                    row_end=i.row_end, bounds=[i.row_bounds[k] for k in range(nranks + 1)],
                    send_count=[i.send_count[k] for k in range(nranks)],
                    recv_count=[i.recv_count[k] for k in range(nranks)])

    def vec(self, n):
        return torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)

    def op(self, level, op, arg=0, x=None, y=None, stat=None, stat_in=None, sign_slot=None):
        from . import fiedler_dist_op
        fiedler_dist_op(self.h, level, op, arg, x, y, stat, stat_in, sign_slot, self.stream)


class PartitionedSolver:
    """Cascadic refinement (Algorithm 3 Steps 2-3) and the
    Rayleigh quotient with row-partitioned fine levels."""

    def __init__(self, ops, comm: Comm, min_rows: int = 1 << 20):
        self.ops = ops
        self.comm = comm
        self.min_rows = min_rows
        nr, rk = comm.nranks, comm.rank
        J = ops.num_levels - 1
        # the coarsest level is always whole on every rank ("gathered")
        self.part = [nr > 1 and l < J and ops.sizes[l] >= min_rows for l in range(ops.num_levels)]
        self.plans = [ops.plan(l, nr if self.part[l] else 1, rk if self.part[l] else 0)
                      for l in range(ops.num_levels)]
        # every buffer of a solve is allocated once, here: per level the
        # prolongation target, two power-iteration vectors, the halo send /
        # receive buffers and the all-gather buffers; statistic slots from one
        # pool (each op writes what it later reads, so reuse across solves is safe)
        L = ops.num_levels
        self.ybuf = [ops.vec(ops.sizes[l]) for l in range(L)]
        self.pbuf = [(ops.vec(ops.sizes[l]), ops.vec(ops.sizes[l])) for l in range(L)]
        self.send = [ops.vec(self.plans[l].send_total) if self.part[l] else None for l in range(L)]
        self.recv = [ops.vec(self.plans[l].recv_total) if self.part[l] else None for l in range(L)]
        self.ag_out = [ops.vec(ops.sizes[l]) if self.part[l] else None for l in range(L)]
        self.ag_in = [ops.vec((self.plans[l].row_end - self.plans[l].row_begin) * nr) if self.part[l] else None
                      for l in range(L)]
        self.vnat = ops.vec(ops.sizes[0])
        self._slots = ops.vec(4 * (4 * L + 8)).view(-1, 4)
        self._next_slot = 0

    # ---------------------------------------------------------------- helpers
    def _slot(self):
        s = self._slots[self._next_slot % self._slots.shape[0]]
        self._next_slot += 1
        return s

    def halo_bytes_per_solve(self, gs_sweeps=2, power_iters=10):
        """Bytes this rank sends per solve: halo exchanges (one per GS colour
        pass, per power step and after the return to natural order) and the
        all-gathers of partitioned levels' vectors (statistics all-reduces are
        a few doubles and not counted)."""
        tot = 0
        J = self.ops.num_levels - 1
        for l in range(self.ops.num_levels):
            if not self.part[l]:
                continue
            p = self.plans[l]
            passes = power_iters + (gs_sweeps * p.colors + 1 if gs_sweeps > 0 else 0)
            tot += 8 * p.send_total * passes
            if l < J:   # all-gather of the level's vector (every level but the finest's RQ output)
                tot += 8 * (p.row_end - p.row_begin) * p.nranks
        return tot

    def _reduce_finalise(self, level, slot):
        if self.part[level]:
            self.comm.allreduce_sum(slot[:2])
        self.ops.op(level, FIEDLER_DOP_FINALISE, stat=slot)

    def _halo(self, level, v, numbering):
        """Own rows of v that other ranks read -> their ghost rows."""
        if not self.part[level]:
            return
        p = self.plans[level]
        send, recv = self.send[level], self.recv[level]
        self.ops.op(level, FIEDLER_DOP_HALO_PACK, numbering, x=v, y=send)
        self.comm.all_to_all(recv[:p.recv_total], send[:p.send_total], p.recv_count, p.send_count)
        self.ops.op(level, FIEDLER_DOP_HALO_UNPACK, numbering, x=recv, y=v)

    def _allgather(self, level, v):
        """Full vector of a partitioned level from every rank's own rows."""
        if not self.part[level]:
            return v
        p = self.plans[level]
        own = p.row_end - p.row_begin
        inp = self.ag_in[level][:own * p.nranks]
        if own:
            inp.view(p.nranks, own).copy_(v[p.row_begin:p.row_end].unsqueeze(0).expand(p.nranks, own))
        sizes = [p.bounds[k + 1] - p.bounds[k] for k in range(p.nranks)]
        out = self.ag_out[level]
        self.comm.all_to_all(out[:p.n], inp, sizes, [own] * p.nranks)
        return out

    def _power(self, level, cur, slot, iters):
        a, b = self.pbuf[level]
        for _ in range(iters):
            nxt = b if cur is a else a
            s2 = self._slot()
            self.ops.op(level, FIEDLER_DOP_POWER, x=cur, y=nxt, stat=s2, stat_in=slot)
            self._reduce_finalise(level, s2)
            self._halo(level, nxt, NATURAL)
            cur, slot = nxt, s2
        return cur, slot

    # ---------------------------------------------------------------- solve
    def solve(self, gs_sweeps=2, power_iters=10, coarsest_power_iters=None, seed=0):
        """Returns (full Fiedler vector in natural order, lambda2, residual_norm)."""
        ctx = getattr(self.ops, "stream_ctx", None)
        if ctx is None:
            return self._solve(gs_sweeps, power_iters, coarsest_power_iters, seed)
        with ctx():
            return self._solve(gs_sweeps, power_iters, coarsest_power_iters, seed)

    def _solve(self, gs_sweeps, power_iters, coarsest_power_iters, seed):
        ops = self.ops
        J = ops.num_levels - 1
        kJ = power_iters if coarsest_power_iters is None else coarsest_power_iters
        self._next_slot = 0
        # Step 2: rand(n_J) (R6) and power iteration on c I - L^J
        cur = self.pbuf[J][0]
        slot = self._slot()
        ops.op(J, FIEDLER_DOP_RAND, seed, y=cur, stat=slot)
        ops.op(J, FIEDLER_DOP_FINALISE, stat=slot)
        cur, slot = self._power(J, cur, slot, kJ)
        full = self._allgather(J, cur)
        # Step 3: cascadic refinement
        for l in range(J - 1, -1, -1):
            ps = self._slot()
            y = self.ybuf[l]
            if gs_sweeps > 0:
                ops.op(l, FIEDLER_DOP_PROLONG, GS, x=full, y=y, stat=ps)
                for _ in range(gs_sweeps):
                    for c in range(self.plans[l].colors):
                        ops.op(l, FIEDLER_DOP_GS_COLOUR, c, x=y)
                        self._halo(l, y, GS)
                z = self.pbuf[l][0]
                ops.op(l, FIEDLER_DOP_TO_NAT, x=y, y=z, stat=ps)
                self._reduce_finalise(l, ps)
                self._halo(l, z, NATURAL)
                cur = z
            else:
                ops.op(l, FIEDLER_DOP_PROLONG, NATURAL, x=full, y=y, stat=ps)
                self._reduce_finalise(l, ps)
                cur = y
            cur, slot = self._power(l, cur, ps, power_iters)
            if l > 0:
                full = self._allgather(l, cur)
        # Rayleigh quotient on level 0 with the sign of R10
        key = self._slot()
        ops.op(0, FIEDLER_DOP_FIRST_NONZERO, x=cur, stat=key, stat_in=slot)
        if self.part[0]:
            self.comm.allreduce_min(key[:1])
        ops.op(0, FIEDLER_DOP_SIGN, stat=key)
        vnat = self.vnat
        rq = self._slot()
        ops.op(0, FIEDLER_DOP_RAYLEIGH, x=cur, y=vnat, stat=rq, stat_in=slot, sign_slot=key)
        if self.part[0]:
            self.comm.allreduce_sum(rq[:3])
        ops.op(0, FIEDLER_DOP_FINALISE_RQ, stat=rq, stat_in=slot)
        v = self._allgather(0, vnat)
        res = rq.cpu()
        return v[:ops.sizes[0]].clone(), float(res[0]), float(res[1])


# =========================================================================
# Row-partitioned setup of the fine levels (Algorithm 3 Step 1)
# =========================================================================
@dataclass
class SetupGraph:
    """One level's whole adjacency (every rank holds it): int64 row offsets,
    int32 columns, float64 weights (the conventions of fiedler_create)."""
    n: int
    nnz: int
    rp: object
    ci: object
    w: object


@dataclass
class PresetLevel:
    """A partitioned level's setup results, gathered on every rank: the aggregate
    map q, the matching, the colouring (whole arrays) and the next level."""
    level: int
    q: object
    mate: object
    colour: object
    ncolors: int
    match_rounds: int
    colour_rounds: int
    nxt: SetupGraph
    row_bounds: List[int]


class LibSetupOps:
    """Setup operations backed by libfiedler's fiedler_pset_* kernels on one GPU;
    every call is issued on one stream shared with torch's tensor work."""

    def __init__(self, device, stream=None):
        import os
        self.device = device
        self.torch_stream = _own_stream(device, stream)
        self.stream = self.torch_stream.cuda_stream
        # FIEDLER_PSET_SYNC=1 (diagnostics): synchronise after every operation
        # so that a device fault is reported by the operation that caused it
        if os.environ.get("FIEDLER_PSET_SYNC") == "1":
            for name in ("bounds", "halo", "gather", "scatter", "match", "aggregate", "galerkin", "colour"):
                setattr(self, name, self._synced(name, getattr(self, name)))

    def _synced(self, name, fn):
        def call(*a, **k):
            r = fn(*a, **k)
            try:
                torch.cuda.synchronize(self.device)
            except Exception as e:   # pragma: no cover - diagnostics
                raise RuntimeError("device fault after LibSetupOps.%s: %s" % (name, e))
            return r
        return call

    def stream_ctx(self):
        return _Joined(self.torch_stream)

    def full(self, n, value, dtype):
        return torch.full((max(n, 1),), value, dtype=dtype, device=self.device)

    def bounds(self, g, nranks):
        from . import fiedler_pset_bounds
        return fiedler_pset_bounds(g.n, g.rp, nranks, self.stream)

    def halo(self, g, nranks, rank, bounds):
        from . import fiedler_pset_halo
        counts = fiedler_pset_halo(g.n, g.rp, g.ci, nranks, rank, bounds, None, self.stream)
        idx = self.full(sum(counts), 0, torch.int32)
        if sum(counts):
            fiedler_pset_halo(g.n, g.rp, g.ci, nranks, rank, bounds, idx, self.stream)
        return idx, counts

    def gather(self, x, idx, count, out):
        from . import fiedler_pset_gather
        fiedler_pset_gather(x, idx, count, out, self.stream)

    def scatter(self, inp, idx, count, x):
        from . import fiedler_pset_scatter
        fiedler_pset_scatter(inp, idx, count, x, self.stream)

    def match(self, phase, g, r0, r1, seed, level, mate, ptr, round=0, work=None):
        from . import fiedler_pset_match
        return fiedler_pset_match(phase, g.n, g.rp, g.ci, g.w, r0, r1, seed, level, mate, ptr, round, work,
                                  self.stream)

    def aggregate(self, phase, g, r0, r1, seed, level, mate, q, offset=0):
        from . import fiedler_pset_aggregate
        return fiedler_pset_aggregate(phase, g.n, g.rp, g.ci, g.w, r0, r1, seed, level, mate, q, offset,
                                      self.stream)

    def galerkin(self, phase, g, q, a0, a1, cap=0, crp=None, cci=None, cw=None):
        from . import fiedler_pset_galerkin
        return fiedler_pset_galerkin(phase, g.n, g.rp, g.ci, g.w, q, a0, a1, cap, crp, cci, cw, self.stream)

    def colour(self, g, r0, r1, seed, level, colour, round=0, work=None):
        from . import fiedler_pset_colour
        return fiedler_pset_colour(g.n, g.rp, g.ci, r0, r1, seed, level, colour, round, work, self.stream)


class PartitionedSetup:
    """Algorithm 3 Step 1 with row-partitioned fine levels.

    Every rank holds the current level's whole CSR and owns the rows
    [bounds[r], bounds[r+1]) (rows + nonzeros balanced).  Per level:

      * heavy-edge matching (Algorithm 1, parallel order R2):
        handshake rounds POINT / RESOLVE on own rows with the boundary rows'
        ptr and mate exchanged after each half-round (one all-to-all each),
        until the all-reduced count of own free rows with a free neighbour is 0;
      * aggregate numbering: own leader counts, their exclusive
        scan over ranks (an all-reduce of the count vector) gives each rank a
        contiguous id range; IDS, MATES and JOIN with q exchanged in between;
        q and the matching are all-gathered;
      * Galerkin product (R3) of the rank's own coarse rows (the
        aggregates of its leaders), all-gathered into the next level;
      * colouring (R4): Jones-Plassmann rounds with the boundary colours
        exchanged after every round, all-gathered.

    Levels with fewer than `min_rows` vertices are left to fiedler_create on
    every rank (fiedler_create_preset takes the partitioned levels as given).
    The result equals fiedler_create's hierarchy bit for bit (every rule is a
    strict order, independent of partition and schedule)."""

    def __init__(self, ops, comm: Comm, min_rows: int = 1 << 20, coarsest_size: int = 25,
                 max_levels: int = 50, seed: int = 0, stall_ratio: float = 0.95):
        self.ops = ops
        self.comm = comm
        self.min_rows = min_rows
        self.coarsest_size = coarsest_size
        self.max_levels = max_levels
        self.seed = seed
        self.stall_ratio = stall_ratio
        self.bytes_sent = 0          # halo + all-gather bytes this rank sent in the last run
        self.rounds = []             # (match rounds, colour rounds) per partitioned level
        # diagnostics: wall ms of the phases of every level (synchronising), when set
        self.phase_times = None
        self.match_lists = False     # work lists for the matching's half-rounds too

    def _mark(self, ell, name):
        if self.phase_times is None:
            return
        import time
        if self._dev.type == "cuda":
            torch.cuda.synchronize(self._dev)
        now = time.perf_counter()
        if name is not None:
            d = self.phase_times.setdefault(ell, {})
            d[name] = d.get(name, 0.0) + (now - self._t0) * 1e3
        self._t0 = now

    # ---------------------------------------------------------------- helpers
    def _scalar_sum(self, v):
        t = torch.tensor([int(v)], dtype=torch.int64, device=self._dev)
        self.comm.allreduce_sum(t)
        return int(t.item())

    def _per_rank(self, v):
        """[value of every rank] (an all-reduce of a one-hot vector)."""
        t = torch.zeros(self.comm.nranks, dtype=torch.int64, device=self._dev)
        t[self.comm.rank] = int(v)
        self.comm.allreduce_sum(t)
        return [int(x) for x in t.tolist()]

    def _exchange(self, x):
        """Own boundary rows of x -> the other ranks' ghost rows (int32 state)."""
        if self.comm.nranks == 1:
            return
        ops = self.ops
        ops.gather(x, self._send_idx, self._ns, self._sbuf)
        self.comm.all_to_all(self._rbuf[:self._nr], self._sbuf[:self._ns], self._recv_counts, self._send_counts)
        ops.scatter(self._rbuf, self._recv_idx, self._nr, x)
        self.bytes_sent += 4 * self._ns

    def _allgather(self, own, sizes, dtype):
        out = self.ops.full(sum(sizes), 0, dtype)
        self.comm.allgatherv(out[:sum(sizes)], own, sizes)
        self.bytes_sent += own.element_size() * own.numel() * max(self.comm.nranks - 1, 0)
        return out

    # ---------------------------------------------------------------- run
    def run(self, g: SetupGraph) -> List[PresetLevel]:
        ctx = getattr(self.ops, "stream_ctx", None)
        if ctx is None:
            return self._run(g)
        with ctx():
            return self._run(g)

    def _run(self, g):
        self._dev = g.rp.device
        self.bytes_sent = 0
        self.rounds = []
        out = []
        ell = 0
        while g.n > self.coarsest_size and ell + 1 < self.max_levels and g.n >= self.min_rows:
            lev = self._level(g, ell)
            if lev is None:      # the matching stalls (R9): fiedler_create decides this level
                break
            out.append(lev)
            g = lev.nxt
            ell += 1
        return out

    def _level(self, g, ell):
        from . import (FIEDLER_PSET_IDS, FIEDLER_PSET_JOIN, FIEDLER_PSET_LEADERS, FIEDLER_PSET_MATES,
                       FIEDLER_PSET_POINT, FIEDLER_PSET_RESOLVE)
        ops, comm = self.ops, self.comm
        N, rk = comm.nranks, comm.rank
        i32 = torch.int32
        self._mark(ell, None)
        bounds = ops.bounds(g, N)
        r0, r1 = bounds[rk], bounds[rk + 1]
        # halo plan: send lists by the library, receive lists = the peers' send lists to us
        self._send_idx, self._send_counts = ops.halo(g, N, rk, bounds)
        sc = torch.tensor(self._send_counts, dtype=torch.int64, device=self._dev)
        rc = torch.zeros_like(sc)
        comm.all_to_all(rc, sc, [1] * N, [1] * N)
        self._recv_counts = [int(x) for x in rc.tolist()]
        self._ns, self._nr = sum(self._send_counts), sum(self._recv_counts)
        self._recv_idx = ops.full(self._nr, 0, i32)
        comm.all_to_all(self._recv_idx[:self._nr], self._send_idx[:self._ns], self._recv_counts, self._send_counts)
        self._sbuf = ops.full(self._ns, 0, i32)
        self._rbuf = ops.full(self._nr, 0, i32)

        self._mark(ell, "halo_plan")
        # heavy-edge matching: handshake rounds
        mate = ops.full(g.n, -1, i32)
        ptr = ops.full(g.n, -1, i32)
        # the rounds' work lists (own rows still in play): the colouring's rounds
        # visit only them; the matching visits all own rows every half-round
        # (measured faster on the grids: ~7 rounds, most rows active until the last)
        work = ops.full(8 + 2 * (r1 - r0), 0, i32)
        mwork = work if self.match_lists else None
        mrounds = 0
        while True:
            act = ops.match(FIEDLER_PSET_POINT, g, r0, r1, self.seed, ell, mate, ptr, mrounds, mwork)
            if self._scalar_sum(act) == 0:
                break
            self._exchange(ptr)
            ops.match(FIEDLER_PSET_RESOLVE, g, r0, r1, self.seed, ell, mate, ptr, mrounds, mwork)
            self._exchange(mate)
            mrounds += 1
        self._mark(ell, "matching")
        # aggregates numbered by increasing leader: contiguous id range per rank
        own_leaders = ops.aggregate(FIEDLER_PSET_LEADERS, g, r0, r1, self.seed, ell, mate, ptr)
        counts = self._per_rank(own_leaders)
        c = sum(counts)
        if c > self.stall_ratio * g.n or c < 2:
            return None
        a0 = sum(counts[:rk])
        a1 = a0 + counts[rk]
        q = ops.full(g.n, -1, i32)
        ops.aggregate(FIEDLER_PSET_IDS, g, r0, r1, self.seed, ell, mate, q, a0)
        self._exchange(q)
        ops.aggregate(FIEDLER_PSET_MATES, g, r0, r1, self.seed, ell, mate, q)
        self._exchange(q)
        ops.aggregate(FIEDLER_PSET_JOIN, g, r0, r1, self.seed, ell, mate, q)
        rows = [bounds[k + 1] - bounds[k] for k in range(N)]
        q_full = self._allgather(q[r0:r1], rows, i32)
        mate_full = self._allgather(mate[r0:r1], rows, i32)

        self._mark(ell, "aggregates")
        # Galerkin product of the own coarse rows [a0, a1), gathered
        cap = ops.galerkin(0, g, q_full, a0, a1)
        crp = ops.full(a1 - a0 + 1, 0, torch.int64)
        cci = ops.full(cap, 0, i32)
        cw = ops.full(cap, 0.0, torch.float64)
        own_nnz = ops.galerkin(1, g, q_full, a0, a1, cap, crp, cci, cw)
        nnzs = self._per_rank(own_nnz)
        nnz_c = sum(nnzs)
        ci_next = self._allgather(cci[:own_nnz], nnzs, i32)
        w_next = self._allgather(cw[:own_nnz], nnzs, torch.float64)
        rp_own = crp[:a1 - a0] + sum(nnzs[:rk])
        rp_next = self._allgather(rp_own, counts, torch.int64)
        rp_full = ops.full(c + 1, 0, torch.int64)
        rp_full[:c] = rp_next[:c]
        rp_full[c] = nnz_c
        nxt = SetupGraph(n=c, nnz=nnz_c, rp=rp_full[:c + 1], ci=ci_next[:max(nnz_c, 1)], w=w_next[:max(nnz_c, 1)])

        self._mark(ell, "galerkin")
        # colouring: Jones-Plassmann rounds
        colour = ops.full(g.n, -1, i32)
        crounds = 0
        maxc = -1
        while True:
            left, mc = ops.colour(g, r0, r1, self.seed, ell, colour, crounds, work)
            maxc = max(maxc, mc)
            crounds += 1
            self._exchange(colour)
            if self._scalar_sum(left) == 0:
                break
        ncolors = max(self._per_rank(maxc + 1))
        colour_full = self._allgather(colour[r0:r1], rows, i32)
        self.rounds.append((mrounds, crounds))
        self._mark(ell, "colouring")
        return PresetLevel(level=ell, q=q_full[:g.n], mate=mate_full[:g.n], colour=colour_full[:g.n],
                           ncolors=ncolors, match_rounds=mrounds, colour_rounds=crounds, nxt=nxt,
                           row_bounds=bounds)


def create_from_presets(g: SetupGraph, presets: List[PresetLevel], opts=None):
    """fiedler_create_preset on the partitioned levels (device arrays).  The
    library joins opts.stream before it reads the arrays; with no stream given
    (NULL: nothing to join) torch's current stream is drained first."""
    from . import fiedler_create_preset, fiedler_default_opts, fiedler_preset_level
    opts = opts or fiedler_default_opts()
    if not opts.stream:
        torch.cuda.current_stream(g.rp.device).synchronize()
    pl = []
    for p in presets:
        s = fiedler_preset_level()
        s.agg, s.mate, s.color = p.q.data_ptr(), p.mate.data_ptr(), p.colour.data_ptr()
        s.ncolors, s.match_rounds, s.colour_rounds = p.ncolors, p.match_rounds, p.colour_rounds
        s.n_next, s.nnz_next = p.nxt.n, p.nxt.nnz
        s.rp_next, s.ci_next, s.w_next = p.nxt.rp.data_ptr(), p.nxt.ci.data_ptr(), p.nxt.w.data_ptr()
        pl.append(s)
    return fiedler_create_preset(g.n, g.nnz, g.rp, g.ci, g.w, opts, pl)

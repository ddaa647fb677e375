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


class LocalComm(Comm):
    """Single rank: every collective is the identity."""

    def allreduce_sum(self, t):
        pass

    def allreduce_min(self, t):
        pass

    def all_to_all(self, out, inp, out_splits, in_splits):
        out.copy_(inp)


class LibOps:
    """Ops backed by libfiedler (fiedler_dist_plan / fiedler_dist_op) on one GPU."""

    def __init__(self, handle, device, stream=None):
        from . import fiedler_level_size, fiedler_num_levels
        self.h = handle
        self.device = device
        # library kernels and torch's tensor work (allocation, zero-fill, slicing,
        # collectives) are ordered by running both on one (non-default) stream:
        # the driver enters stream_ctx() around the solve
        self.torch_stream = torch.cuda.Stream(device) if stream is None else torch.cuda.ExternalStream(stream)
        self.stream = self.torch_stream.cuda_stream
        self.num_levels = fiedler_num_levels(handle)
        self.sizes = [fiedler_level_size(handle, l)[0] for l in range(self.num_levels)]

    def stream_ctx(self):
        return torch.cuda.stream(self.torch_stream)

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

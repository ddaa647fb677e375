"""Test infrastructure for the partitioned solve (paper_1602_04386_b200/dist.py):

* ``RefOps`` -- a plain numpy/torch-CPU implementation of every
  ``fiedler_dist_op`` operation and of the row-partition / halo plan, written
  from the operation definitions in include/fiedler.h on top of the ORACLE's
  hierarchy (oracle/ is test infrastructure).  It lets the driver run on the
  CPU under gloo, and its plans are the reference for the library's plans.
* ``ThreadComm`` -- collectives between Python threads of ONE process (each
  thread plays a rank).  Used to run several ranks' drivers on one GPU: the
  ranks' kernels never wait on one another (every exchange is a host-side
  rendezvous after a device synchronisation).
"""
import threading

import numpy as np
import torch

from paper_1602_04386_b200.dist import Comm, Plan

DOP = dict(RAND=1, PROLONG=2, GS_COLOUR=3, TO_NAT=4, POWER=5, FINALISE=6, FIRST_NONZERO=7, SIGN=8,
           RAYLEIGH=9, FINALISE_RQ=10, HALO_PACK=11, HALO_UNPACK=12)
INV_DOP = {v: k for k, v in DOP.items()}
TILE_T = 2048


def ref_plan(rp, ci, ncolors, nranks, rank):
    """Row partition (coordinate rp[r] + r split evenly) and halo lists."""
    n = rp.size - 1
    total = int(rp[-1]) + n
    coord = rp[:-1] + np.arange(n)
    bounds = [0] + [int(np.searchsorted(coord, total * k // nranks, side="left")) for k in range(1, nranks)] + [n]
    r0, r1 = bounds[rank], bounds[rank + 1]
    owner = np.searchsorted(np.asarray(bounds[1:-1]), np.arange(n), side="right")
    ghosts = set()
    send = [[] for _ in range(nranks)]
    for v in range(r0, r1):
        peers = set()
        for j in ci[rp[v]:rp[v + 1]]:
            if j < r0 or j >= r1:
                ghosts.add(int(j))
                peers.add(int(owner[j]))
        for p in peers:
            send[p].append(v)
    g = np.array(sorted(ghosts), dtype=np.int64)
    recv = [g[(g >= bounds[p]) & (g < bounds[p + 1])] for p in range(nranks)]
    plan = Plan(n=n, colors=ncolors, nranks=nranks, rank=rank, row_begin=r0, row_end=r1, bounds=bounds,
                send_count=[len(s) for s in send], recv_count=[len(r) for r in recv])
    send_idx = np.concatenate([np.array(s, dtype=np.int64) for s in send]) if plan.send_total else np.zeros(0, np.int64)
    recv_idx = np.concatenate(recv) if plan.recv_total else np.zeros(0, np.int64)
    return plan, send_idx, recv_idx


class RefOps:
    """numpy implementation of the fiedler_dist_op operations on the oracle's hierarchy."""

    def __init__(self, levels, seed=0):
        import oracle
        self.oracle = oracle
        self.levels = levels
        self.num_levels = len(levels)
        self.sizes = [L.g.n for L in levels]
        self.state = {}
        self.inv = []
        for L in levels:
            order = oracle.color_order(L.color)     # GS numbering: (colour, natural id)
            inv = np.empty(L.g.n, dtype=np.int64)
            inv[order] = np.arange(L.g.n)
            self.inv.append(inv)

    def plan(self, level, nranks, rank):
        L = self.levels[level]
        p, s, r = ref_plan(L.g.rp, L.g.ci, L.ncolors, nranks, rank)
        self.state[level] = (p, s, r)
        return p

    def vec(self, n):
        return torch.zeros(max(n, 1), dtype=torch.float64)

    def op(self, level, op, arg=0, x=None, y=None, stat=None, stat_in=None, sign_slot=None):
        L = self.levels[level]
        g = L.g
        n = g.n
        p, send_idx, recv_idx = self.state[level]
        own = np.arange(p.row_begin, p.row_end)
        inv = self.inv[level]
        X = x.numpy() if x is not None else None
        Y = y.numpy() if y is not None else None
        S = stat.numpy() if stat is not None else None
        name = INV_DOP[op]
        if name == "RAND":
            v = self.oracle.rand_uniform(n, arg)
            Y[:n] = v
            S[0], S[1] = v.sum(), (v * v).sum()
        elif name == "PROLONG":
            q = L.q
            rows = np.concatenate([own, recv_idx])
            dst = inv[rows] if arg else rows
            Y[dst] = X[q[rows]]
            vals = X[q[own]]
            S[0], S[1] = vals.sum(), (vals * vals).sum()
        elif name == "GS_COLOUR":
            for v in own[L.color[own] == arg]:
                nb = g.ci[g.rp[v]:g.rp[v + 1]]
                w = g.w[g.rp[v]:g.rp[v + 1]]
                Y_ = X  # in place, GS numbering
                Y_[inv[v]] = np.dot(w, Y_[inv[nb]]) / w.sum()
        elif name == "TO_NAT":
            Y[own] = X[inv[own]]
            vals = Y[own]
            S[0], S[1] = vals.sum(), (vals * vals).sum()
        elif name == "POWER":
            mu, sig = stat_in[2].item(), stat_in[3].item()
            z = np.empty(own.size)
            for i, v in enumerate(own):
                nb = g.ci[g.rp[v]:g.rp[v + 1]]
                w = g.w[g.rp[v]:g.rp[v + 1]]
                z[i] = (L.shift * (X[v] - mu) + np.dot(w, X[nb] - X[v])) / sig
            Y[own] = z
            S[0], S[1] = z.sum(), (z * z).sum()
        elif name == "FINALISE":
            mu = S[0] / n
            S[2] = mu
            S[3] = np.sqrt(max(S[1] - n * mu * mu, 0.0))
        elif name == "FIRST_NONZERO":
            mu = stat_in[2].item()
            d = X[own] - mu
            nz = np.flatnonzero(d != 0.0)
            S[0] = 2.0 * own[nz[0]] + (1.0 if d[nz[0]] < 0 else 0.0) if nz.size else float(2 ** 60)
        elif name == "SIGN":
            key = S[0]
            S[2] = -1.0 if (key < 2 ** 60 and key % 2 == 1) else 1.0
        elif name == "RAYLEIGH":
            mu, sig = stat_in[2].item(), stat_in[3].item()
            sgn = sign_slot[2].item()
            num = den = lv2 = 0.0
            for v in own:
                nb = g.ci[g.rp[v]:g.rp[v + 1]]
                w = g.w[g.rp[v]:g.rp[v + 1]]
                d = X[v] - X[nb]
                num += np.dot(w, d * d)
                den += (X[v] - mu) ** 2
                lv2 += (np.dot(w, d) / sig) ** 2
                Y[v] = sgn * (X[v] - mu) / sig
            S[0], S[1], S[2] = num, den, lv2
        elif name == "FINALISE_RQ":
            sig = stat_in[3].item()
            lam = 0.5 * S[0] / S[1]
            vn2 = S[1] / sig ** 2
            S[0], S[1], S[2] = lam, np.sqrt(max(S[2] - lam * lam * vn2, 0.0)), np.sqrt(vn2)
        elif name == "HALO_PACK":
            Y[:send_idx.size] = X[inv[send_idx]] if arg else X[send_idx]
        elif name == "HALO_UNPACK":
            dst = inv[recv_idx] if arg else recv_idx
            Y[dst] = X[:recv_idx.size]
        else:
            raise ValueError(op)


class ThreadComm(Comm):
    """Collectives between threads of one process (one thread per rank)."""

    def __init__(self, shared, rank, nranks, sync_cuda=False):
        self.shared = shared          # dict with a threading.Barrier under "barrier"
        self.rank = rank
        self.nranks = nranks
        self.sync_cuda = sync_cuda

    def _exchange(self, item):
        if self.sync_cuda:
            torch.cuda.synchronize()
        b = self.shared["barrier"]
        self.shared.setdefault("box", {})[self.rank] = item
        b.wait()
        items = [self.shared["box"][r] for r in range(self.nranks)]
        b.wait()
        return items

    def allreduce_sum(self, t):
        items = self._exchange(t.clone())
        tot = items[0].clone()
        for it in items[1:]:
            tot += it
        t.copy_(tot)

    def allreduce_min(self, t):
        items = self._exchange(t.clone())
        m = items[0].clone()
        for it in items[1:]:
            m = torch.minimum(m, it)
        t.copy_(m)

    def all_to_all(self, out, inp, out_splits, in_splits):
        parts = list(torch.split(inp.clone(), list(in_splits)))
        items = self._exchange(parts)
        got = [items[r][self.rank] for r in range(self.nranks)]
        if got:
            out.copy_(torch.cat(got))


def run_threads(nranks, fn):
    """Run fn(rank, comm) on nranks threads; returns the results by rank."""
    shared = {"barrier": threading.Barrier(nranks)}
    res = [None] * nranks
    errs = []

    def body(r):
        try:
            res[r] = fn(r, shared)
        except BaseException as e:  # pragma: no cover - surfaced below
            errs.append(e)
            shared["barrier"].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return res


# ---------------------------------------------------------------------------
# Partitioned setup (paper_1602_04386_b200/dist.py PartitionedSetup): a plain
# numpy implementation of the fiedler_pset_* operations, written from their
# definitions in include/fiedler.h, on CPU tensors.  Lets the driver run on
# gloo ranks; the result is compared with the oracle's hierarchy.
# ---------------------------------------------------------------------------
class RefSetupOps:
    def __init__(self):
        import oracle
        self.o = oracle

    def full(self, n, value, dtype):
        return torch.full((max(n, 1),), value, dtype=dtype)

    @staticmethod
    def _np(g):
        return g.rp.numpy(), g.ci.numpy(), g.w.numpy()

    def bounds(self, g, nranks):
        rp = g.rp.numpy()
        coord = rp[:-1] + np.arange(g.n)
        total = int(rp[-1]) + g.n
        return [0] + [int(np.searchsorted(coord, total * k // nranks, side="left"))
                      for k in range(1, nranks)] + [g.n]

    def halo(self, g, nranks, rank, bounds):
        rp, ci, _ = self._np(g)
        r0, r1 = bounds[rank], bounds[rank + 1]
        owner = np.searchsorted(np.asarray(bounds[1:-1]), np.arange(g.n), side="right")
        send = [[] for _ in range(nranks)]
        for v in range(r0, r1):
            for p in sorted({int(owner[j]) for j in ci[rp[v]:rp[v + 1]] if j < r0 or j >= r1}):
                send[p].append(v)
        idx = [v for p in range(nranks) for v in send[p]]
        t = self.full(len(idx), 0, torch.int32)
        t[:len(idx)] = torch.tensor(idx, dtype=torch.int32)
        return t, [len(s) for s in send]

    def gather(self, x, idx, count, out):
        out[:count] = x[idx[:count].long()]

    def scatter(self, inp, idx, count, x):
        x[idx[:count].long()] = inp[:count]

    def _edge_key(self, salt, v, u, w):
        lo, hi = min(v, u), max(v, u)
        return (w, self.o.splitmix64((salt ^ ((lo << 32) | hi)) & self.o.MASK64))

    def match(self, phase, g, r0, r1, seed, level, mate, ptr, round=0, work=None):
        rp, ci, w = self._np(g)
        salt = self.o.salt_match(seed, level)
        if phase == 0:
            act = 0
            for v in range(r0, r1):
                if mate[v] >= 0:
                    continue
                best, bk = -1, None
                for k in range(rp[v], rp[v + 1]):
                    u = int(ci[k])
                    if mate[u] >= 0:
                        continue
                    key = self._edge_key(salt, v, u, w[k])
                    if best < 0 or key > bk:
                        best, bk = u, key
                ptr[v] = best
                act += best >= 0
            return act
        new = mate.clone()
        for v in range(r0, r1):
            u = int(ptr[v])
            if mate[v] < 0 and u >= 0 and int(ptr[u]) == v:
                new[v] = u
        mate.copy_(new)
        return 0

    def _heaviest(self, g, salt, v):
        rp, ci, w = self._np(g)
        best, bk = -1, None
        for k in range(rp[v], rp[v + 1]):
            key = self._edge_key(salt, v, int(ci[k]), w[k])
            if best < 0 or key > bk:
                best, bk = int(ci[k]), key
        return best

    def aggregate(self, phase, g, r0, r1, seed, level, mate, q, offset=0):
        rp = g.rp.numpy()
        if phase in (0, 1):
            lead = [v for v in range(r0, r1)
                    if (mate[v] >= 0 and v < mate[v]) or (mate[v] < 0 and rp[v + 1] == rp[v])]
            if phase == 1:
                q[r0:r1] = -1
                for i, v in enumerate(lead):
                    q[v] = offset + i
            return len(lead)
        if phase == 2:
            for v in range(r0, r1):
                if 0 <= mate[v] < v:
                    q[v] = q[int(mate[v])]
            return 0
        salt = self.o.salt_match(seed, level)
        for v in range(r0, r1):
            if mate[v] < 0 and rp[v + 1] > rp[v]:
                m = self._heaviest(g, salt, v)
                assert mate[m] >= 0 and q[m] >= 0
                q[v] = q[m]
        return 0

    def galerkin(self, phase, g, q, a0, a1, cap=0, crp=None, cci=None, cw=None):
        rp, ci, w = self._np(g)
        qn = q.numpy()
        contrib = []
        for i in range(g.n):
            a = int(qn[i])
            if not a0 <= a < a1:
                continue
            for k in range(rp[i], rp[i + 1]):
                j = int(ci[k])
                b = int(qn[j])
                if b != a:
                    contrib.append((a, b, min(i, j), max(i, j), w[k]))
        if phase == 0:
            return len(contrib)
        contrib.sort(key=lambda t: t[:4])
        rows = {}
        for a, b, _, _, wk in contrib:        # left fold in (lo, hi) order per (A, B)
            d = rows.setdefault(a, {})
            d[b] = wk if b not in d else d[b] + wk
        nnz = 0
        for a in range(a0, a1):
            crp[a - a0] = nnz
            for b in sorted(rows.get(a, {})):
                cci[nnz] = b
                cw[nnz] = rows[a][b]
                nnz += 1
        crp[a1 - a0] = nnz
        return nnz

    def colour(self, g, r0, r1, seed, level, colour, round=0, work=None):
        rp, ci, _ = self._np(g)
        salt = self.o.salt_color(seed, level)
        pi = lambda x: (self.o.splitmix64((salt ^ x) & self.o.MASK64), x)   # noqa: E731
        start = colour.clone()            # a round reads the state at its start
        left, mx = 0, -1
        for v in range(r0, r1):
            if start[v] < 0:
                nb = [int(u) for u in ci[rp[v]:rp[v + 1]]]
                if all(start[u] >= 0 for u in nb if pi(u) > pi(v)):
                    used = {int(start[u]) for u in nb if start[u] >= 0}
                    c = 0
                    while c in used:
                        c += 1
                    colour[v] = c
                else:
                    left += 1
            mx = max(mx, int(colour[v]))
        return left, mx

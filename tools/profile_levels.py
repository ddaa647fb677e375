"""Per-level timings of the three row passes (CUDA events via fiedler_level_time).
Usage: python tools/profile_levels.py [config] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_04386_b200 as fd  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
g = gg.config(cfg)
dev = torch.device("cuda", 0)
rp, ci, w = (torch.from_numpy(a).to(dev) for a in (g.rp, g.ci, g.w))
h = fd.fiedler_create(g.n, g.nnz, rp, ci, w, fd.fiedler_default_opts(validate=0))
tot = {"pi": 0.0, "gs": 0.0}
for lev in range(fd.fiedler_num_levels(h)):
    n, nnz, col = fd.fiedler_level_size(h, lev)
    row = []
    for name, op in (("pi", fd.FIEDLER_OP_POWER), ("gs", fd.FIEDLER_OP_GS_SWEEPS), ("rq", fd.FIEDLER_OP_RAYLEIGH)):
        ms, by = fd.fiedler_level_time(h, lev, op, reps)
        row.append("%s %.4f ms %.0f GB/s" % (name, ms, by / ms / 1e6))
        if name in tot:
            tot[name] += ms
    print("L%-2d n %9d nnz %10d col %2d | %s" % (lev, n, nnz, col, " | ".join(row)))
print("sum over levels: 10 x pi = %.2f ms, 2 x gs = %.2f ms" % (10 * tot["pi"], 2 * tot["gs"]))
fd.fiedler_destroy(h)

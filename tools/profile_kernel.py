"""Launch the level-`level` hot kernels of a BASELINE config once each, for
`ncu --set full -k regex:k_rowpass` captures (after create(), the first
k_rowpass launches are exactly these: POWER warm-up + rep, then the GS colour
passes, then the Rayleigh pass).
Usage: python tools/profile_kernel.py [config] [level]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_04386_b200 as fd  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
g = gg.config(cfg)
dev = torch.device("cuda", 0)
rp, ci, w = (torch.from_numpy(a).to(dev) for a in (g.rp, g.ci, g.w))
h = fd.fiedler_create(g.n, g.nnz, rp, ci, w, fd.fiedler_default_opts(validate=0))
for op in (fd.FIEDLER_OP_POWER, fd.FIEDLER_OP_GS_SWEEPS, fd.FIEDLER_OP_RAYLEIGH):
    ms, by = fd.fiedler_level_time(h, level, op, reps)
    print("op", op, "ms", ms, "GB/s", by / ms / 1e6)
fd.fiedler_destroy(h)

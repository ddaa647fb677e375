import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch, numpy as np
import graphgen as gg, paper_1602_04386_b200 as fd
from paper_1602_04386_b200 import dist as D
g = gg.rmat(12, 16.0, seed=5)
args = [torch.from_numpy(a).cuda() for a in (g.rp, g.ci, g.w)]
h = fd.fiedler_create(g.n, g.nnz, *args, fd.fiedler_default_opts(stream=torch.cuda.current_stream().cuda_stream))
vec = torch.empty(g.n, dtype=torch.float64, device='cuda')
print("ref", fd.fiedler_solve(h, vec))
ops = D.LibOps(h, torch.device('cuda'))
orig = ops.op
def traced(level, op, arg=0, x=None, y=None, stat=None, stat_in=None, sign_slot=None):
    orig(level, op, arg, x, y, stat, stat_in, sign_slot)
    torch.cuda.synchronize()
    if level <= 1 or op in (1,):
        print("L%d op%d arg%d stat=%s ysum=%s" % (level, op, arg, None if stat is None else stat.cpu().numpy(), None if y is None else float(y.sum())))
ops.op = traced
s = D.PartitionedSolver(ops, D.LocalComm())
print([ (p.n, p.colors, p.row_begin, p.row_end) for p in s.plans])
v, lam, res = s.solve()
print("lam", lam, res)

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads as problems
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
a = problems.varcoef7(n, seed=0); xs, b = problems.rhs(a)
cfg = P.CgConfig(ordering="hbmc", b_s=8, w=32, spmv_format="sell")
st = solver.attach_plan(solver.prepare(a, b, cfg), cfg)
bd = torch.from_numpy(st.b_sys).cuda(); xd = torch.empty_like(bd)
for k in range(3):
    rep, hist = st.plan.pcg(bd, xd, cfg.tol, cfg.max_iters)
    torch.cuda.synchronize()
    print(k, rep.iterations, rep.kernel_launches, flush=True)

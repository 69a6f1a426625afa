"""One ICCG solve of a config (for ncu launch lists): python scripts/iccg_once.py CFG"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads as problems
_, gen, bs, w = problems.CONFIGS[int(sys.argv[1])]
a = gen(); xs, b = problems.rhs(a)
cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
st = solver.attach_plan(solver.prepare(a, b, cfg), cfg)
bd = torch.from_numpy(st.b_sys).cuda(); xd = torch.empty_like(bd)
rep, _ = st.plan.pcg(bd, xd, cfg.tol, cfg.max_iters); torch.cuda.synchronize()
print("iterations", rep.iterations)

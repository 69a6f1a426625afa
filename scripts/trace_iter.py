"""Break one steady PCG iteration of the persistent kernel into phases."""
import ctypes as C
import os
import sys

os.environ["TB_TRACE"] = "1"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import numpy as np
import torch

import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import _lib, solver
import workloads as problems

arg = sys.argv[1] if len(sys.argv) > 1 else "2"
if arg.startswith("c5:"):   # config 5 family at a given grid size
    label, bs, w = f"aniso7_{arg[3:]}^3", 16, 32
    a = problems.lap7(int(arg[3:]), 1.0, 1.0, 1e-3)
else:
    label, gen, bs, w = problems.CONFIGS[int(arg)]
    a = gen()
xs, b = problems.rhs(a)
cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
s = solver.prepare(a, b, cfg)
solver.attach_plan(s, cfg)
bd = torch.from_numpy(s.b_sys).cuda()
xd = torch.empty_like(bd)
for _ in range(3):
    rep, _ = s.plan.pcg(bd, xd, cfg.tol, cfg.max_iters)
buf = (C.c_uint64 * 64)()
_lib.check(_lib.LIB.tb_plan_trace(s.plan.handle, buf))
t = [buf[i] for i in range(5)]
names = ["SpMV + p.Ap", "x/r update + ||r||", "precond (both sweeps) + r.z", "p update + barrier"]
tot = t[4] - t[0]
print(f"{label}: iteration {tot / 1e3:.1f} us")
for i, nm in enumerate(names):
    d = (t[i + 1] - t[i]) / 1e3
    print(f"  {nm:32s} {d:7.1f} us  {100 * d * 1e3 / tot:5.1f}%")

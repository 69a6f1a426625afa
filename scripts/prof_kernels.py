"""Profiling driver for one kernel family on one config (run under ncu).

    python scripts/prof_kernels.py {precond|spmv} {2|3|4|c5:N} [reps]
Builds the plan, warms up, then runs `reps` launches of the chosen operator
(plan.precond -> the persistent dataflow kernel; plan.spmv -> the TMA SpMV).
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np
import torch

import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads as problems

what, arg = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
if arg.startswith("c5:"):
    a, bs, w = problems.lap7(int(arg[3:]), 1.0, 1.0, 1e-3), 16, 32
else:
    _, gen, bs, w = problems.CONFIGS[int(arg)]
    a = gen()
cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
st = solver.attach_plan(solver.prepare(a, np.zeros(a.n), cfg), cfg)
n = st.layout.n_pad
r = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
z = torch.empty_like(r)
fs = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
fd = torch.empty((), dtype=torch.float64, device="cuda")
op = st.plan.precond if what == "precond" else st.plan.spmv
for _ in range(2 + reps):
    torch.sum(fs, dim=0, out=fd)
    op(r, z)
torch.cuda.synchronize()
nnz_l = (a.nnz - a.n) // 2
nb = 2 * (12 * nnz_l + 32 * a.n) if what == "precond" else 12 * a.nnz + 16 * a.n
print(f"{what} {arg}: algorithmic bytes per launch {nb}")

"""Profiling driver: build a BASELINE config, run K preconditioner applies.

    python scripts/prof_sweep.py [config] [reps]
Used under ncu (-k regex:sweep) to capture the substitution kernels.
"""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np
import torch

import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads as problems

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
label, gen, bs, w = problems.CONFIGS[cfg_id]
a = gen()
xs, b = problems.rhs(a)
cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
setup = solver.prepare(a, b, cfg)
solver.attach_plan(setup, cfg)
plan = setup.plan
n = setup.layout.n_pad
r = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
z = torch.empty_like(r)
ap = torch.empty_like(r)
flush = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
for _ in range(reps):
    flush.zero_()
    plan.precond(r, z)
    flush.zero_()
    plan.spmv(r, ap)
torch.cuda.synchronize()
t0 = time.perf_counter()
plan.precond(r, z)
torch.cuda.synchronize()
print(label, "n_pad", n, "precond ms", 1e3 * (time.perf_counter() - t0),
      [plan.phase_info(f, c) for f in (True, False) for c in range(setup.layout.n_c)])

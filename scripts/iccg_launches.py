"""One ICCG solve of a BASELINE config (for ncu launch lists)."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import torch

import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads as problems

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
label, gen, bs, w = problems.CONFIGS[cfg_id]
a = gen()
xs, b = problems.rhs(a)
cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
setup = solver.prepare(a, b, cfg)
solver.attach_plan(setup, cfg)
for _ in range(2):
    x, rep, hist = solver.solve_on_device(setup, cfg)
torch.cuda.synchronize()
print(label, "iterations", rep.iterations, "converged", rep.converged)

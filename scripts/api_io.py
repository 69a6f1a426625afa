"""Host-to-host timings of the trilab-facing calls (numpy in / numpy out)
at a given size: apply_ic_preconditioner and the device PCG through
solver.solve_on_device.  python scripts/api_io.py [config] [reps]"""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np
import torch

import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
label, a, bs, w = workloads.generate(cfg_id)
xs, b = workloads.rhs(a)
cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
st = solver.attach_plan(solver.prepare(a, b, cfg), cfg)
hl = st.layout
r = np.random.default_rng(0).standard_normal(hl.n_pad)
z0 = P.apply_ic_preconditioner("hbmc", st.factor, hl, r)
ts = []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    z = P.apply_ic_preconditioner("hbmc", st.factor, hl, r)
    ts.append(time.perf_counter() - t0)
assert np.array_equal(z, z0)
P.precond.release_plans(st.factor)
tsol = []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep, hist = solver.solve_on_device(st, cfg)
    tsol.append(time.perf_counter() - t0)
print(f"config {cfg_id}: apply_ic_preconditioner(numpy) {1e3 * min(ts):.1f} ms, "
      f"solve host->host {1e3 * min(tsol):.1f} ms ({rep.iterations} it), n_pad {hl.n_pad}",
      flush=True)

"""A/B of the plan SpMV kernels: python scripts/spmv_ab.py CFG|c5:N "name:ENV=V,..." ..."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads as problems
arg = sys.argv[1]
if arg.startswith("c5:"):
    a = problems.lap7(int(arg[3:]), 1.0, 1.0, 1e-3); bs, w = 16, 32
else:
    _, gen, bs, w = problems.CONFIGS[int(arg)]; a = gen()
cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
base = solver.prepare(a, np.zeros(a.n), cfg)
nb = 12 * a.nnz + 16 * a.n
fs = torch.ones(32 << 20, dtype=torch.float64, device="cuda"); fd = torch.empty((), dtype=torch.float64, device="cuda")
x = torch.from_numpy(np.random.default_rng(0).standard_normal(base.layout.n_pad)).cuda()
ref = None
for spec in sys.argv[2:]:
    name, _, kv = spec.partition(":")
    env = dict(e.split("=", 1) for e in kv.split(",") if e)
    old = {k: os.environ.get(k) for k in env}; os.environ.update(env)
    import copy
    s = solver.attach_plan(copy.copy(base), cfg)
    for k, v in old.items():
        os.environ.pop(k, None) if v is None else os.environ.__setitem__(k, v)
    y = torch.empty_like(x)
    ts = []
    for i in range(25):
        torch.sum(fs, dim=0, out=fd)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); s.plan.spmv(x, y); e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    us = statistics.median([e0.elapsed_time(e1) * 1e3 for e0, e1 in ts[5:]])
    yh = y.cpu().numpy()
    if ref is None: ref = yh
    print(f"{name:10s} spmv {us:8.1f} us {nb / us / 1e3:7.0f} GB/s same_as_first={np.array_equal(yh, ref)}", flush=True)
    s.plan.close()

"""In-process A/B of plan variants selected by environment variables.

    python scripts/ab.py [config] "name:VAR=VAL,VAR=VAL" "name2:..." ...

One setup; one device plan per variant (the plan reads its TB_* variables
at creation); then R interleaved rounds, each timing K preconditioner
applications per variant (256 MiB read flush before each, events
pre-created, enqueue-only).  Prints the median per variant and, for
variants whose plan supports it, one ICCG solve time.
"""
import os
import statistics
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np
import torch

import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads as problems

cfg_id = int(sys.argv[1])
variants = []
for spec in sys.argv[2:]:
    name, _, kv = spec.partition(":")
    env = dict(x.split("=", 1) for x in kv.split(",") if x)
    variants.append((name, env))
label, gen, bs, w = problems.CONFIGS[cfg_id]
a = gen()
xs, b = problems.rhs(a)
cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
base = solver.prepare(a, b, cfg)
plans = []
for name, env in variants:
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    import copy
    s = copy.copy(base)
    solver.attach_plan(s, cfg)
    plans.append((name, s.plan))
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
n = base.layout.n_pad
nnz_l = (a.nnz - a.n) // 2
step_bytes = 2 * (12 * nnz_l + 32 * a.n)
r = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
z = torch.empty_like(r)
fs = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
fd = torch.empty((), dtype=torch.float64, device="cuda")
K, R = 10, 5
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
      for _ in range(K)]
res = {name: [] for name, _ in plans}
zs = {}
for name, pl in plans:
    z.fill_(float("nan"))
    pl.precond(r, z)
    torch.cuda.synchronize()
    zs[name] = z.clone()
z0 = zs[plans[0][0]]
for name, _ in plans:
    print(f"{name:14s} z bitwise vs {plans[0][0]}: {bool(torch.equal(zs[name], z0))}", flush=True)
for rnd in range(R):
    for name, pl in plans:
        torch.cuda.synchronize()
        for e0, e1 in ev:
            torch.sum(fs, dim=0, out=fd)
            e0.record()
            pl.precond(r, z)
            e1.record()
        torch.cuda.synchronize()
        res[name] += [e0.elapsed_time(e1) * 1e3 for e0, e1 in ev]
b_dev = torch.from_numpy(base.b_sys).cuda()
x_dev = torch.empty_like(b_dev)
for name, pl in plans:
    med = statistics.median(res[name])
    pl.pcg(b_dev, x_dev, cfg.tol, cfg.max_iters)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep, _ = pl.pcg(b_dev, x_dev, cfg.tol, cfg.max_iters)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:14s} precond median {med:7.1f} us ({step_bytes / med / 1e3:6.0f} GB/s) "
          f"min {min(res[name]):7.1f} | iccg {e0.elapsed_time(e1):7.2f} ms it {rep.iterations} "
          f"persist {pl.persistent()}", flush=True)

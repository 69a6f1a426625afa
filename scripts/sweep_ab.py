"""Sweep kernel A/B with a bitwise cross-check: python scripts/sweep_ab.py CFG|c5:N "name:ENV=V,..." ...
Each variant's plan applies the preconditioner to the same r; z must be bitwise equal
to the first variant's; reports median fwd+bwd time (L2 flushed) and per-phase times."""
import os, sys, statistics, copy
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads as problems
arg = sys.argv[1]
if arg.startswith("c5:"):
    a, bs, w = problems.lap7(int(arg[3:]), 1.0, 1.0, 1e-3), 16, 32
else:
    _, gen, bs, w = problems.CONFIGS[int(arg)]; a = gen()
cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
base = solver.prepare(a, np.zeros(a.n), cfg)
nnz_l = (a.nnz - a.n) // 2
nb = 2 * (12 * nnz_l + 32 * a.n)
r = torch.from_numpy(np.random.default_rng(0).standard_normal(base.layout.n_pad)).cuda()
fs = torch.ones(32 << 20, dtype=torch.float64, device="cuda"); fd = torch.empty((), dtype=torch.float64, device="cuda")
ref = None
for spec in sys.argv[2:]:
    name, _, kv = spec.partition(":")
    env = dict(e.split("=", 1) for e in kv.split(",") if e)
    old = {k: os.environ.get(k) for k in env}; os.environ.update(env)
    st = solver.attach_plan(copy.copy(base), cfg)
    for k, v in old.items():
        os.environ.pop(k, None) if v is None else os.environ.__setitem__(k, v)
    z = torch.full_like(r, float("nan"))
    ev = []
    for i in range(12):
        torch.sum(fs, dim=0, out=fd)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); st.plan.precond(r, z); e1.record(); ev.append((e0, e1))
    torch.cuda.synchronize()
    us = statistics.median([e0.elapsed_time(e1) * 1e3 for e0, e1 in ev[2:]])
    zh = z.cpu().numpy()
    if ref is None: ref = zh
    print(f"{arg} {name:10s} precond {us:8.1f} us {nb / us / 1e3:6.0f} GB/s bitwise_same={np.array_equal(zh, ref)} "
          f"phases={[st.plan.phase_info(f, c)['staged'] for f in (True, False) for c in range(base.n_c)]}", flush=True)
    st.plan.close()

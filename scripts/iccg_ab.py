"""ICCG time-to-solution A/B of tb_pcg paths: python scripts/iccg_ab.py CFG|c5:N "name:ENV=V" ..."""
import os, sys
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
xs, b = problems.rhs(a)
cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
st = solver.attach_plan(solver.prepare(a, b, cfg), cfg)
bd = torch.from_numpy(st.b_sys).cuda(); xd = torch.empty_like(bd)
for spec in sys.argv[2:]:
    name, _, kv = spec.partition(":")
    env = dict(e.split("=", 1) for e in kv.split(",") if e)
    old = {k: os.environ.get(k) for k in env}; os.environ.update(env)
    st.plan.pcg(bd, xd, cfg.tol, cfg.max_iters)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); rep, hist = st.plan.pcg(bd, xd, cfg.tol, cfg.max_iters); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    x = xd.cpu().numpy()[st.old_positions]
    for k, v in old.items():
        os.environ.pop(k, None) if v is None else os.environ.__setitem__(k, v)
    print(f"{arg} {name:10s} iccg {min(ts):9.2f} ms  it {rep.iterations}  ms/it {min(ts)/rep.iterations:7.3f}  "
          f"launches {rep.kernel_launches} syncs {rep.host_syncs}  err {np.linalg.norm(x-xs)/np.linalg.norm(xs):.3e}", flush=True)

"""ICCG A/B of plan-creation knobs (grid sizes etc.): a fresh plan per setting.

    python scripts/vec_ab.py CFG "name:ENV=V,ENV2=V2" ...

Unlike iccg_ab.py (knobs read per solve), each spec here rebuilds the device
plan with its environment, since TB_VEC_PT / TB_RZP_FUSE are read at plan
creation.  Best of 5 solves, device time.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads as problems

_, gen, bs, w = problems.CONFIGS[int(sys.argv[1])]
a = gen()
xs, b = problems.rhs(a)
cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
st = solver.prepare(a, b, cfg)
bd = torch.from_numpy(st.b_sys).cuda()
xd = torch.empty_like(bd)
for rnd in range(2):
    for spec in sys.argv[2:]:
        name, _, kv = spec.partition(":")
        env = dict(e.split("=", 1) for e in kv.split(",") if e)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        solver.attach_plan(st, cfg)
        st.plan.pcg(bd, xd, cfg.tol, cfg.max_iters)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rep, hist = st.plan.pcg(bd, xd, cfg.tol, cfg.max_iters)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        x = xd.cpu().numpy()[st.old_positions]
        st.plan.close()
        for k, v in old.items():
            os.environ.pop(k, None) if v is None else os.environ.__setitem__(k, v)
        print(f"r{rnd} {sys.argv[1]} {name:10s} iccg {min(ts):8.3f} ms  it {rep.iterations}  "
              f"err {np.linalg.norm(x - xs) / np.linalg.norm(xs):.3e}", flush=True)

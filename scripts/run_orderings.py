"""The paper's ordering comparison on the B200: nodal MC vs BMC vs HBMC.

    python scripts/run_orderings.py [config=3]

BASELINE config 3 (27-point 192^3) is "compared against BMC and nodal MC
orderings of the same matrix".  For each ordering: host setup, one
preconditioner application (fwd+bwd, L2 flushed, CUDA events), the ICCG
solve (device time), iterations against the reference's own run
(tests/golden/config<k>_digest.json) and the reference's CPU solve time.
MC / BMC run the CSR task-sweep kernels (one phase per color / per block
color), HBMC the persistent dataflow SELL kernel.
"""
import json
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

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
label, gen, bs, w = problems.CONFIGS[cfg_id]
a = gen()
xs, b = problems.rhs(a)
with open(os.path.join(os.path.dirname(HERE), "tests", "golden",
                       f"config{cfg_id}_digest.json")) as fh:
    dg = json.load(fh)
nnz_l = (a.nnz - a.n) // 2
sweep2 = 2 * (12 * nnz_l + 32 * a.n)
flush_src = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
flush_dst = torch.empty((), dtype=torch.float64, device="cuda")
out = {"config": cfg_id, "label": label, "N": a.n, "nnz_A": int(a.nnz), "b_s": bs, "w": w,
       "orderings": {}}
for ordering in ("mc", "bmc", "hbmc"):
    cfg = P.CgConfig(ordering=ordering, b_s=bs, w=w,
                     spmv_format="sell" if ordering == "hbmc" else "crs")
    t0 = time.perf_counter()
    st = solver.attach_plan(solver.prepare(a, b, cfg), cfg)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    n = st.a_sys.n
    r = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
    z = torch.empty_like(r)
    ts = []
    for k in range(8):
        torch.sum(flush_src, dim=0, out=flush_dst)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.plan.precond(r, z)
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    pre_ms = min(e0.elapsed_time(e1) for e0, e1 in ts[2:])
    bd = torch.from_numpy(st.b_sys).cuda()
    xd = torch.empty_like(bd)
    st.plan.pcg(bd, xd, cfg.tol, cfg.max_iters)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep, hist = st.plan.pcg(bd, xd, cfg.tol, cfg.max_iters)
    e1.record()
    torch.cuda.synchronize()
    x_sys = xd.cpu().numpy()
    x = x_sys[st.old_positions] if st.old_positions is not None else x_sys
    ref = dg.get(ordering, {})
    out["orderings"][ordering] = {
        "n_c": int(st.n_c), "setup_s": t_setup, "precond_ms": pre_ms,
        "precond_GBps": sweep2 / (pre_ms / 1e3) / 1e9,
        "iterations": int(rep.iterations), "reference_iterations": ref.get("iterations"),
        "time_to_solution_ms": e0.elapsed_time(e1),
        "reference_cpu_solve_s": ref.get("time_solve_s"),
        "rel_err_vs_xstar": float(np.linalg.norm(x - xs) / np.linalg.norm(xs)),
        "kernel_launches": int(rep.kernel_launches)}
    print(ordering, json.dumps(out["orderings"][ordering]), flush=True)
    st.plan.close()
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/orderings_config{cfg_id}.json", "w") as fh:
    json.dump(out, fh, indent=1)

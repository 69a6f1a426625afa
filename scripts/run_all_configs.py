"""All BASELINE configs on one B200: setup, precond, SpMV, ICCG (one table).

    python scripts/run_all_configs.py [ids=1,2,3,4] [out=gpurun_out/all_configs.json]

Per config: host + device setup time, one preconditioner application
(fwd+bwd, L2 flushed before each, CUDA events, median of 10) and its
algorithmic GB/s (2 * (12 nnz_L + 32 N)), the plan SpMV (12 nnz_A + 16 N),
the ICCG solve to 1e-7 (device time, best of 3) with iterations against the
reference's own run (tests/golden/config<k>_digest.json; config 1 from the
full golden), and the reference's CPU solve time where recorded.
"""
import json
import os
import statistics
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)

import numpy as np
import torch

import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads as problems

ids = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3,4").split(",")]
out_path = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/all_configs.json"
fs = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
fd = torch.empty((), dtype=torch.float64, device="cuda")


def med_us(fn, k=10):
    ev = []
    for _ in range(k + 2):
        torch.sum(fs, dim=0, out=fd)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    return statistics.median(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev[2:])


rows = []
for cid in ids:
    label, gen, bs, w = problems.CONFIGS[cid]
    t0 = time.perf_counter()
    a = gen()
    xs, b = problems.rhs(a)
    t_gen = time.perf_counter() - t0
    cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
    t0 = time.perf_counter()
    st = solver.prepare(a, b, cfg)
    t_host = time.perf_counter() - t0
    t0 = time.perf_counter()
    solver.attach_plan(st, cfg)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    nnz_l = (a.nnz - a.n) // 2
    sb = 2 * (12 * nnz_l + 32 * a.n)
    mb = 12 * a.nnz + 16 * a.n
    n = st.layout.n_pad
    r = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
    z = torch.empty_like(r)
    pre = med_us(lambda: st.plan.precond(r, z))
    spm = med_us(lambda: st.plan.spmv(r, z))
    bd = torch.from_numpy(st.b_sys).cuda()
    xd = torch.empty_like(bd)
    st.plan.pcg(bd, xd, cfg.tol, cfg.max_iters)
    solves = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep, hist = st.plan.pcg(bd, xd, cfg.tol, cfg.max_iters)
        e1.record()
        torch.cuda.synchronize()
        solves.append(e0.elapsed_time(e1))
    x = xd.cpu().numpy()[st.old_positions]
    ref_it, ref_s = None, None
    dg_path = os.path.join(REPO, "tests", "golden", f"config{cid}_digest.json")
    if os.path.exists(dg_path):
        with open(dg_path) as fh:
            dg = json.load(fh)["hbmc"]
        ref_it, ref_s = dg["iterations"], dg.get("time_solve_s")
    elif cid == 1:
        g = np.load(os.path.join(REPO, "tests", "golden", "config1_full.npz"))
        ref_it = int(g["pcg_hbmc_iters"])
    row = {"config": cid, "label": label, "N": int(a.n), "nnz_A": int(a.nnz), "n_c": int(st.n_c),
           "b_s": bs, "w": w, "generate_s": t_gen, "host_setup_s": t_host,
           "device_setup_s": t_dev, "precond_us": pre, "precond_GBps": sb / pre / 1e3,
           "spmv_us": spm, "spmv_GBps": mb / spm / 1e3, "iccg_ms": min(solves),
           "iterations": int(rep.iterations), "reference_iterations": ref_it,
           "reference_cpu_solve_s": ref_s,
           "rel_err_vs_xstar": float(np.linalg.norm(x - xs) / np.linalg.norm(xs)),
           "persistent": st.plan.persistent()}
    print(json.dumps(row), flush=True)
    rows.append(row)
    st.plan.close()
    del st, a
os.makedirs(os.path.dirname(out_path), exist_ok=True)
with open(out_path, "w") as fh:
    json.dump(rows, fh, indent=1)

"""Config 5 (anisotropic 7-point 512^3, N = 134M, HBMC b_s=16, w=32) on one B200.

    python scripts/run_config5.py [n=512] [steps=5]

Stages are timed separately (generation, host builder, device upload); then
the preconditioner application (fwd+bwd sweeps, 2 * 9.1 GB algorithmic),
the SpMV and the whole ICCG solve are timed with CUDA events.  Parity at
full size: one forward and one backward sweep are compared BITWISE with the
C oracle (oracle/hbmc_oracle.c, OpenMP over the host cores) run on the same
SELL arrays.  The reference itself cannot build this system in 62 GB (SURVEY
8(c)); this is the size the north star names for the partitioned runs.
"""
import json
import os
import resource
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np
import torch

import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads as problems


def rss_gb():
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6


n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
out = {"config": 5, "grid": n, "b_s": 16, "w": 32}
t0 = time.perf_counter()
a = problems.lap7(n, 1.0, 1.0, 1e-3)
xs, b = problems.rhs(a)
out["generate_s"] = time.perf_counter() - t0
out["N"], out["nnz_A"] = int(a.n), int(a.nnz)
print("generated", out, f"rss {rss_gb():.1f} GB", flush=True)
cfg = P.CgConfig(ordering="hbmc", b_s=16, w=32, spmv_format="sell")
t0 = time.perf_counter()
st = solver.prepare(a, b, cfg, ic0=os.environ.get("C5_PREP_IC0", "auto"))
out["host_setup_s"] = time.perf_counter() - t0
hl = st.layout
out["n_c"], out["n_pad"], out["n_dummy"] = int(hl.n_c), int(hl.n_pad), int(hl.n_dummy)
print("host setup", out["host_setup_s"], f"rss {rss_gb():.1f} GB", flush=True)
del a
t0 = time.perf_counter()
solver.attach_plan(st, cfg)
torch.cuda.synchronize()
out["device_setup_s"] = time.perf_counter() - t0
plan = st.plan
out["device_bytes"] = int(plan.device_bytes())
out["persistent"] = plan.persistent()
print("device setup", out["device_setup_s"], out["device_bytes"] / 1e9, "GB", flush=True)

L = P.precond._strict_tri(st.a_sys)
nnz_l = int(L.row_ptr[-1])
real_n = int(out["N"])
sweep_b = 12 * nnz_l + 32 * real_n
spmv_b = 12 * out["nnz_A"] + 16 * real_n
out["nnz_L"] = nnz_l
out["sweep_bytes"] = sweep_b

r = torch.from_numpy(np.random.default_rng(0).standard_normal(hl.n_pad)).cuda()
y = torch.empty_like(r)
z = torch.empty_like(r)
ap = torch.empty_like(r)


def timed(fn, k):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(k)]
    for e0, e1 in ev:
        e0.record()
        fn()
        e1.record()
    torch.cuda.synchronize()
    return [e0.elapsed_time(e1) for e0, e1 in ev]


timed(lambda: plan.precond(r, z), 2)
pm = timed(lambda: plan.precond(r, z), steps)
out["precond_ms"] = min(pm)
out["precond_GBps"] = 2 * sweep_b / (min(pm) / 1e3) / 1e9
fm = timed(lambda: plan.forward(r, y), steps)
bm = timed(lambda: plan.backward(y, z), steps)
out["fwd_ms"], out["bwd_ms"] = min(fm), min(bm)
out["fwd_GBps"] = sweep_b / (min(fm) / 1e3) / 1e9
out["bwd_GBps"] = sweep_b / (min(bm) / 1e3) / 1e9
sm = timed(lambda: plan.spmv(r, ap), steps)
out["spmv_ms"] = min(sm)
out["spmv_GBps"] = spmv_b / (min(sm) / 1e3) / 1e9
print(json.dumps(out), flush=True)

# bitwise parity of both sweeps against the C oracle on the same arrays
if os.environ.get("C5_ORACLE", "1") == "1":
    from oracle import oracle as O
    t0 = time.perf_counter()
    sf = st.factor
    Ls, Us = sf.lower, sf.upper
    hd = {"n_pad": hl.n_pad, "w": 32, "b_s": 16, "n_c": hl.n_c,
          "color_lvl1_ranges": np.ascontiguousarray(hl.color_lvl1_ranges, dtype=np.int64)}
    osl = O.Sell(Ls.n, Ls.n_pad, 32, Ls.slice_ptr, Ls.slice_len, Ls.col_idx, Ls.vals)
    osu = O.Sell(Us.n, Us.n_pad, 32, Us.slice_ptr, Us.slice_len, Us.col_idx, Us.vals)
    rh = r.cpu().numpy()
    yo = O.hbmc_sweep(True, osl, sf.inv_diag, rh, hd, O.max_threads())
    zo = O.hbmc_sweep(False, osu, sf.inv_diag, yo, hd, O.max_threads())
    plan.forward(r, y)
    plan.backward(y, z)
    out["fwd_bitwise"] = bool(np.array_equal(y.cpu().numpy(), yo))
    out["bwd_bitwise"] = bool(np.array_equal(z.cpu().numpy(), zo))
    out["oracle_sweeps_s"] = time.perf_counter() - t0
    out["oracle_threads"] = O.max_threads()
    print("oracle parity", out["fwd_bitwise"], out["bwd_bitwise"], flush=True)

# IC(0): host builder (what prepare() ran) vs the device factorization
if os.environ.get("C5_IC0", "1") == "1":
    from paper_1908_00741_b200 import precond as PC
    t0 = time.perf_counter()
    fh = PC.ic0_factorize(st.a_sys, layout_tag="hbmc")
    out["ic0_host_s"] = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tk = {}
    fd = PC.ic0_factorize_device(st.a_sys, hl, timings=tk)
    out["ic0_device_s"] = time.perf_counter() - t0   # incl. checks, H2D of the pattern, D2H
    out["ic0_device_kernels_s"] = tk["kernel_s"]
    out["ic0_device_bitwise"] = bool(np.array_equal(fd.L.vals, fh.L.vals) and
                                     np.array_equal(fd.d, fh.d) and
                                     np.array_equal(fd.inv_diag, fh.inv_diag))
    del fh, fd
    print("ic0 host", out["ic0_host_s"], "device", out["ic0_device_s"],
          out["ic0_device_bitwise"], flush=True)

bd = torch.from_numpy(st.b_sys).cuda()
xd = torch.empty_like(bd)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
rep, hist = plan.pcg(bd, xd, cfg.tol, cfg.max_iters)
e1.record()
torch.cuda.synchronize()
x = xd.cpu().numpy()[st.old_positions]
out["iccg"] = {"iterations": int(rep.iterations), "converged": bool(rep.converged),
               "time_to_solution_ms": e0.elapsed_time(e1),
               "ms_per_iteration": e0.elapsed_time(e1) / max(1, rep.iterations),
               "rel_err_vs_xstar": float(np.linalg.norm(x - xs) / np.linalg.norm(xs)),
               "history_head": [float(v) for v in hist[:5]],
               "history_tail": [float(v) for v in hist[-3:]]}
out["bytes_per_iteration"] = 2 * sweep_b + spmv_b + 80 * real_n
out["iccg"]["GBps_per_iteration"] = out["bytes_per_iteration"] / (
    out["iccg"]["ms_per_iteration"] / 1e3) / 1e9
out["max_rss_gb"] = rss_gb()
print(json.dumps(out), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/config5_{n}.json", "w") as fh:
    json.dump(out, fh, indent=1)

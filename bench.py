#!/usr/bin/env python
"""Benchmark: HBMC IC(0) fwd+bwd substitution GB/s and ICCG time-to-solution.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 5]

Workload (default): BASELINE.json configs[4], the largest configuration that
fits one B200 -- anisotropic 3-D 7-point on 512^3 (N = 134,217,728,
nnz = 937,951,232), HBMC b_s=16, w=32, fp64, synthetic seeded inputs
(SURVEY.md Appendix B).  `--config 2` (configs[1], 128^3 variable
coefficient, b_s=8) and the others remain selectable.  One "step" = one
preconditioner application z = (L L^T)^-1 r on the device (forward +
backward HBMC sweep, all color phases), inputs resident in HBM.

Timing: CUDA events on the launching stream, created up front; every timed
step is enqueued without a host synchronisation (so host launch overhead
never sits inside a timed window) and is preceded by an L2 flush that READS
256 MiB (> the 126 MB L2; a write flush would leave dirty lines whose
write-back lands in the timed kernel).

value    = algorithmic bytes of the two sweeps (2 * (12 nnz_L + 32 N), SURVEY
           8(d)) x steps x ranks / max-over-ranks summed device time.
e2e      = the same through the C-ABI plan operator with HOST buffers: pinned
           host r -> device, fwd+bwd, z -> pinned host, copies inside the
           timed region (pipelined over 3 streams, as a caller streaming
           right-hand sides runs it).  e2e.api = per-call timings of the
           trilab-facing calls a user makes: apply_ic_preconditioner(numpy r)
           (pageable, synchronous) and the ICCG solve b (host) -> x (host).
roofline = the precond kernel (N = 1: the item-pipelined dataflow kernel
           flow2::precond_kernel, both sweeps in one launch, when the plan
           has one; else the persistent kernel or the per-color sweep
           launches): algorithmic bytes per launch / its CUDA-event
           duration, vs MEASURED_PEAKS.json.  `spmv` is the same for the
           plan SpMV.  traffic = ncu dram bytes of that kernel
           (profiles/traffic.json).
iccg     = full PCG solve to 1e-7 on the device (one CUDA-graph launch).
cpu_baseline = the CPU oracle port of the reference path (oracle/): the
           reference's fwd_sell_range / bwd_sell_range restated in C, timed
           on this product's SELL arrays (SURVEY 8(d) for config 5), all
           host threads and 1 thread, bounded samples (rank 0, N=1).

--impl reference: the reference's CPU path on this box's host cores -- the
oracle port (oracle/), which imports nothing from the product: matrix
assembled with the oracle's coo_to_csr, the oracle's own ordering / IC(0) /
SELL build, steps = full fwd+bwd HBMC sweeps with all threads, plus a
bounded ICCG sample (src/solver.py:139-204 with all threads).

N > 1 (torchrun, one rank per GPU, NCCL): the row-partitioned solve of
SURVEY 8(e) -- every color's level-1 blocks split over the ranks, one halo
exchange after every color phase (default: the owner's kernel stores the
halo entries straight into the peers' vectors over NVLink through CUDA IPC
mappings and releases a per-sender flag; `--transport nccl`: NCCL
send/recv), CG dots all-reduced with NCCL.
The problem is fixed as N grows (scaling "strong"); value = the whole
system's algorithmic sweep bytes / max-over-ranks device time.
`--mode replicas` instead runs N independent replicas (scaling "weak").
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "HBMC IC(0) fwd+bwd substitution GB/s (algorithmic bytes)"
L2_FLUSH_BYTES = 256 << 20


def sweep_bytes(nnz_l, n):
    """S = 12 nnz_L + 32 N per sweep (int32 idx, fp64 values)."""
    return 12 * nnz_l + 32 * n


def spmv_bytes(nnz_a, n):
    return 12 * nnz_a + 16 * n


def load_peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the GPU works
    (the profiling recipe's clocks line: `nvidia-smi --query-gpu=... -lms`
    started before, stopped after).  Wraps the warm-up and timed steps, so
    the samples are taken under the same load as the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, period_ms=50):
        self.index = index
        self.period_ms = period_ms
        self.samples = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.QUERY,
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.15)   # first sample lands before the work starts
        except Exception:
            self._p = None
        return self

    def __exit__(self, *exc):
        if self._p is None:
            return
        time.sleep(0.06)       # one more period under load
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=5)
        except Exception:
            self._p.kill()
            out, _ = self._p.communicate()
        for line in (out or "").splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None,
                    "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def build_problem(cfg_id, backend="product"):
    import workloads
    t0 = time.perf_counter()
    label, a, bs, w = workloads.generate(cfg_id, backend=backend)
    xs, b = workloads.rhs(a, backend=backend)
    return label, a, xs, b, bs, w, time.perf_counter() - t0


def load_digest(cfg_id):
    p = os.path.join(HERE, "tests", "golden", f"config{cfg_id}_digest.json")
    if not os.path.exists(p):
        return {}
    with open(p) as fh:
        return json.load(fh)


def time_sweeps(O, Ls, Us, inv_d, hl, r, threads, reps):
    """Seconds per fwd+bwd HBMC sweep pair (oracle kernels, fork-join per
    color over `threads` as src/precond.py:377-392)."""
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        y = O.hbmc_sweep(True, Ls, inv_d, r, hl, threads)
        O.hbmc_sweep(False, Us, inv_d, y, hl, threads)
        ts.append(time.perf_counter() - t0)
    return ts


def cpu_baseline_on_arrays(Ls, Us, inv_d, hl, nbytes, threads, reps_all, t1_budget_s=30.0):
    """The reference's sweep kernels (oracle port) on the given SELL arrays:
    all threads (`reps_all` applications, after one warm-up) and 1 thread
    (one application, or a bounded share of the level-1 blocks of every
    color when a whole one would exceed `t1_budget_s`)."""
    from oracle import oracle as O
    r = np.random.default_rng(0).standard_normal(hl["n_pad"])
    time_sweeps(O, Ls, Us, inv_d, hl, r, threads, 1)
    ts = time_sweeps(O, Ls, Us, inv_d, hl, r, threads, reps_all)
    t_all = sum(ts) / len(ts)
    # 1 thread: estimate from the all-thread time x threads, then sample a
    # fraction of every color's level-1 range sized to the budget
    frac = min(1.0, t1_budget_s / max(1e-9, t_all * threads))
    if frac >= 1.0:
        t1 = time_sweeps(O, Ls, Us, inv_d, hl, r, 1, 1)[0]
        t1_desc = "one full fwd+bwd application"
    else:
        # the first ceil(frac * nbar(c)) level-1 blocks of every color, fwd
        # then bwd (same kernels, same per-block work), scaled pro rata
        cl = np.asarray(hl["color_lvl1_ranges"], dtype=np.int64)
        keep = np.maximum(1, np.ceil(frac * np.diff(cl)).astype(np.int64))
        y = np.zeros(hl["n_pad"])
        z = np.zeros(hl["n_pad"])
        t0 = time.perf_counter()
        for c in range(hl["n_c"]):
            O.LIB.or_fwd_sell_range(Ls.slice_ptr, Ls.slice_len, Ls.col_idx, Ls.vals, inv_d,
                                    r, y, hl["w"], hl["b_s"], int(cl[c]), int(cl[c] + keep[c]))
        for c in range(hl["n_c"] - 1, -1, -1):
            O.LIB.or_bwd_sell_range(Us.slice_ptr, Us.slice_len, Us.col_idx, Us.vals, inv_d,
                                    y, z, hl["w"], hl["b_s"], int(cl[c]), int(cl[c] + keep[c]))
        frac_done = float(keep.sum()) / float(cl[-1])
        t1 = (time.perf_counter() - t0) / frac_done
        t1_desc = (f"the first {100 * frac_done:.2f} % of every color's level-1 blocks "
                   f"(fwd then bwd), scaled to the whole application")
    return {"value": nbytes / t_all / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
            "cpu": cpu_model(),
            "sample": f"{reps_all} fwd+bwd HBMC applications of the full workload after "
                      f"1 warm-up (oracle/hbmc_oracle.c fwd/bwd_sell_range, per-color "
                      f"fork-join over {threads} OpenMP threads as src/precond.py:377-392)",
            "ms_per_step": 1e3 * t_all,
            "t1": {"value": nbytes / t1 / 1e9, "unit": "GB/s", "cores": 1,
                   "ms_per_step": 1e3 * t1, "sample": t1_desc}}


def run_reference(args, rank):
    """The reference's CPU path, import-clean: nothing from the product
    package is imported (the matrix is assembled by the oracle's C
    coo_to_csr), so only oracle/liboracle.so is loaded."""
    if rank != 0:
        return
    from oracle import oracle as O
    threads = O.max_threads()
    label, a, xs, b, bs, w, t_gen = build_problem(args.config, backend="oracle")
    n, nnz_a = a.n, int(a.nnz)
    osys = O.HbmcSystem(a, b, bs, w, lean=True)
    del a
    hl = osys.hl
    nbytes = 2 * sweep_bytes(osys.nnz_L, n)
    r = np.random.default_rng(0).standard_normal(hl["n_pad"])
    time_sweeps(O, osys.Ls, osys.Us, osys.inv_d, hl, r, threads, args.warmup)
    ts = time_sweeps(O, osys.Ls, osys.Us, osys.inv_d, hl, r, threads, args.steps)
    value = nbytes * len(ts) / sum(ts) / 1e9
    cb = cpu_baseline_on_arrays(osys.Ls, osys.Us, osys.inv_d, hl, nbytes, threads, 1)
    cb["value"] = value
    cb["ms_per_step"] = 1e3 * sum(ts) / len(ts)
    cb["sample"] = (f"{args.steps} timed fwd+bwd HBMC applications of the full workload "
                    f"after {args.warmup} warm-ups (oracle/hbmc_oracle.c fwd/bwd_sell_range, "
                    f"per-color fork-join over {threads} OpenMP threads as "
                    f"src/precond.py:377-392), oracle-built system")
    cb["setup_s"] = osys.time_setup_s
    # ICCG (src/solver.py:139-204, all threads incl. the SELL SpMV): the
    # whole solve when it is short, else a bounded number of iterations
    dg = load_digest(args.config)
    ref_iters = (dg.get("hbmc") or {}).get("iterations")
    t0 = time.perf_counter()
    _, it1, _, _ = O.pcg_hbmc(osys, max_iters=1, threads=threads, spmv_threads=threads)
    t_first = time.perf_counter() - t0
    est_total = t_first * (ref_iters or 1)
    if est_total <= args.ref_iccg_budget_s:
        t0 = time.perf_counter()
        _, it, _, conv = O.pcg_hbmc(osys, threads=threads, spmv_threads=threads)
        iccg = {"iterations": it, "converged": conv,
                "time_to_solution_s": time.perf_counter() - t0, "kind": "full solve"}
    else:
        k = max(2, int(args.ref_iccg_budget_s / max(t_first, 1e-9)))
        t0 = time.perf_counter()
        _, it, _, conv = O.pcg_hbmc(osys, max_iters=k, threads=threads, spmv_threads=threads)
        dt = time.perf_counter() - t0
        per_it = dt / max(1, it)
        iccg = {"sampled_iterations": it, "s_per_iteration": per_it,
                "iterations_to_1e-7": ref_iters,
                "time_to_solution_s_estimated": per_it * ref_iters if ref_iters else None,
                "kind": f"first {it} iterations timed, x the oracle's iteration count "
                        f"(tests/golden/config{args.config}_digest.json)",
                "full_solve_s_offline": (dg.get("hbmc") or {}).get("time_solve_s"),
                "full_solve_offline_source": dg.get("source")}
    iccg["threads"] = threads
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(ts) / len(ts), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, SURVEY Appendix B)",
            "config": {"workload": f"config{args.config} {label} b_s={bs} w={w}",
                       "N": n, "n_pad": int(hl["n_pad"]), "nnz_A": nnz_a,
                       "nnz_L": int(osys.nnz_L), "n_c": int(hl["n_c"]),
                       "bytes_per_step": nbytes},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "iccg": iccg, "generate_s": t_gen}
    print(json.dumps(line), flush=True)


class Timer:
    """Enqueue-only event timing on one stream (no host syncs inside)."""

    def __init__(self, torch, stream, n):
        self.t = torch
        self.stream = stream
        self.ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(n)]
        self.i = 0

    def start(self):
        self.ev[self.i][0].record(self.stream)

    def stop(self):
        self.ev[self.i][1].record(self.stream)
        self.i += 1

    def times_ms(self):
        self.t.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in self.ev[:self.i]]


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1908_00741_b200 as P
    from paper_1908_00741_b200 import solver

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    label, a, xs, b, bs, w, t_gen = build_problem(args.config)
    n, nnz_a = a.n, int(a.nnz)
    cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
    t0 = time.perf_counter()
    setup = solver.prepare(a, b, cfg)
    t_host = time.perf_counter() - t0
    del a
    solver.attach_plan(setup, cfg)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    plan, hl = setup.plan, setup.layout
    n_pad = hl.n_pad
    nnz_l = (nnz_a - n) // 2   # strictly-lower nonzeros of A (= of L)
    step_bytes = 2 * sweep_bytes(nnz_l, n)

    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    flush_src = torch.ones(L2_FLUSH_BYTES // 8, dtype=torch.float64, device=dev)
    flush_dst = torch.empty((), dtype=torch.float64, device=dev)

    def flush():
        torch.sum(flush_src, dim=0, out=flush_dst)

    r = torch.from_numpy(np.random.default_rng(0).standard_normal(n_pad)).to(dev)
    z = torch.empty_like(r)
    y = torch.empty_like(r)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---------------- device-resident steps (value)
    tm = Timer(torch, stream, args.steps)
    with ClockSampler(local_rank) as clk:
        for _ in range(args.warmup):
            flush()
            plan.precond(r, z, sptr)
        barrier()
        for _ in range(args.steps):
            flush()
            tm.start()
            plan.precond(r, z, sptr)
            tm.stop()
        step_ms = tm.times_ms()
    barrier()
    dev_ms = sum(step_ms)
    launches = 2 * hl.n_c * args.steps

    # ---------------- per-launch timing of the sweep kernel (roofline)
    span = bs * w
    lower_counts = P.precond.tri_row_counts(setup.a_sys)
    upper_counts = P.precond.tri_row_counts(setup.a_sys, upper=True)
    real = np.zeros(n_pad, dtype=bool)
    real[hl.real_positions] = True
    phases = []
    for fw in (True, False):
        for c in (range(hl.n_c) if fw else range(hl.n_c - 1, -1, -1)):
            k0, k1 = int(hl.color_lvl1_ranges[c]), int(hl.color_lvl1_ranges[c + 1])
            cnt = (lower_counts if fw else upper_counts)[k0 * span:k1 * span]
            nb = 12 * int(cnt.sum()) + 32 * int(real[k0 * span:k1 * span].sum())
            phases.append((fw, c, nb))
    tl = Timer(torch, stream, len(phases) * (args.warmup + args.steps))
    for _ in range(args.warmup + args.steps):
        for fw, c, nb in phases:
            flush()
            tl.start()
            if fw:
                plan.sweep_phase(True, c, r, y, sptr)
            else:
                plan.sweep_phase(False, c, y, z, sptr)
            tl.stop()
    lt = tl.times_ms()[len(phases) * args.warmup:]
    per_phase = []
    for q, (fw, c, nb) in enumerate(phases):
        ts = lt[q::len(phases)]
        info = plan.phase_info(fw, c)
        per_phase.append({"sweep": "fwd" if fw else "bwd", "color": c,
                          "kernel": "lean" if info["staged"] == 4 else "simple",
                          "bytes": nb, "avg_us": 1e3 * sum(ts) / len(ts),
                          "GBps": nb / (sum(ts) / len(ts) / 1e3) / 1e9})
    peak, peak_src = load_peaks()
    pinfo = plan.persistent()
    finfo = plan.flow_info()
    if finfo["grid"] > 0:
        # the timed step is ONE launch of the item-pipelined dataflow kernel
        kernel_name = (f"flow2::precond_kernel (csrc/flow2.cuh: one warp per level-1 block, "
                       f"{finfo['stages']}-stage cp.async ring per warp, per-block completion "
                       f"flags, no grid barrier; grid {finfo['grid']} x 128 threads, "
                       f"{finfo['smem']} B smem per CTA)")
        tot_b = step_bytes * args.steps
        tot_ms = dev_ms
        n_launch = args.steps
    elif pinfo["precond"]:
        # the timed step is ONE persistent launch (both sweeps, all phases)
        kernel_name = (f"pcg_persistent<KC,dataflow> mode=precond (cooperative grid "
                       f"{pinfo['grid']} CTAs, per-level-1-block completion flags, no grid "
                       f"barrier)"
                       if w == 32 else
                       f"pcg_persistent mode=precond (cooperative, grid {pinfo['grid']} "
                       f"CTAs, {2 * hl.n_c - 1} in-kernel grid barriers)")
        tot_b = step_bytes * args.steps
        tot_ms = dev_ms
        n_launch = args.steps
    else:
        kernel_name = "HBMC sweep, one launch per color phase"
        tot_b = sum(p["bytes"] for p in per_phase) * args.steps
        tot_ms = sum(lt)
        n_launch = len(lt)
    achieved = tot_b / (tot_ms / 1e3) / 1e9
    traffic, traffic_src = args.traffic, "--traffic" if args.traffic else None
    tj = {}
    if traffic is None:
        tp = os.path.join(HERE, "profiles", "traffic.json")
        if os.path.exists(tp):
            with open(tp) as fh:
                tj = json.load(fh).get(f"config{args.config}", {})
            key = ("flow_precond" if finfo["grid"] > 0 else
                   "persistent_precond" if pinfo["precond"] else "per_phase")
            if key in tj:
                traffic = tj[key]["dram_bytes_per_launch"]
                traffic_src = tj[key]["source"]

    # ---------------- SpMV kernel alone (second hot kernel of the iteration)
    ap_dev = torch.empty_like(r)
    tsp = Timer(torch, stream, args.warmup + args.steps)
    for _ in range(args.warmup + args.steps):
        flush()
        tsp.start()
        plan.spmv(r, ap_dev, sptr)
        tsp.stop()
    sp_ms = tsp.times_ms()[args.warmup:]
    sp_us = 1e3 * sum(sp_ms) / len(sp_ms)
    sp_bytes = spmv_bytes(nnz_a, n)
    spmv_line = {"kernel": "plan SpMV: spmv_tma (TMA-staged SELL chunks); thread per row if no TMA candidate fits",
                 "algorithmic_bytes": sp_bytes, "avg_us": sp_us,
                 "achieved": sp_bytes / (sp_us / 1e6) / 1e9, "peak": peak, "unit": "GB/s",
                 "frac": sp_bytes / (sp_us / 1e6) / 1e9 / peak,
                 "traffic": tj.get("spmv_tma", {}).get("dram_bytes_per_launch") if not args.traffic else None,
                 "traffic_source": tj.get("spmv_tma", {}).get("source") if not args.traffic else None}

    # ---------------- e2e through the public API (host buffers)
    # Every step copies its rhs from pinned host memory, applies the
    # preconditioner and copies z back to pinned host memory.  Steps are
    # software-pipelined over three streams with TB_E2E_NBUF (3) rotating
    # device vectors (H2D of step i+1 and D2H of step i-1 overlap step i's
    # sweeps; PCIe is full duplex), as a caller streaming right-hand sides
    # would run it.  Timed from the first H2D to the last D2H on the device.
    nbuf = int(os.environ.get("TB_E2E_NBUF", "3"))
    r_host = torch.from_numpy(np.random.default_rng(0).standard_normal(n_pad)).pin_memory()
    z_host = [torch.empty(n_pad, dtype=torch.float64).pin_memory() for _ in range(nbuf)]
    r_dev = [torch.empty(n_pad, dtype=torch.float64, device=dev) for _ in range(nbuf)]
    z_dev = [torch.empty_like(r_dev[0]) for _ in range(nbuf)]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev = lambda: torch.cuda.Event()  # noqa: E731

    def e2e_run(k):
        e_in, e_cmp, e_out = [None] * k, [None] * k, [None] * k
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s_in)
        for i in range(k):
            bi = i % nbuf
            if i >= nbuf:
                s_in.wait_event(e_cmp[i - nbuf])       # compute i-2 done reading r_dev[bi]
            with torch.cuda.stream(s_in):
                r_dev[bi].copy_(r_host, non_blocking=True)
            e_in[i] = ev()
            e_in[i].record(s_in)
            stream.wait_event(e_in[i])
            if i >= nbuf:
                stream.wait_event(e_out[i - nbuf])     # D2H i-2 done reading z_dev[bi]
            plan.precond(r_dev[bi], z_dev[bi], sptr)
            e_cmp[i] = ev()
            e_cmp[i].record(stream)
            s_out.wait_event(e_cmp[i])
            with torch.cuda.stream(s_out):
                z_host[bi].copy_(z_dev[bi], non_blocking=True)
            e_out[i] = ev()
            e_out[i].record(s_out)
        s_in.wait_stream(s_out)
        t1.record(s_in)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1)

    e2e_run(args.warmup)
    barrier()
    e2e_ms = e2e_run(args.steps)
    barrier()

    # The host-link floor of that pipeline: the same H2D and D2H copies issued
    # concurrently with no compute (PCIe is full duplex), per step.
    def link_run(k):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s_in)
        s_out.wait_stream(s_in)
        for i in range(k):
            with torch.cuda.stream(s_in):
                r_dev[i % nbuf].copy_(r_host, non_blocking=True)
            with torch.cuda.stream(s_out):
                z_host[i % nbuf].copy_(z_dev[i % nbuf], non_blocking=True)
        s_in.wait_stream(s_out)
        t1.record(s_in)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / k

    link_run(2)
    link_ms = link_run(max(args.steps, 10))

    # ---------------- ICCG time-to-solution on the device
    b_dev = torch.from_numpy(setup.b_sys).to(dev)
    x_dev = torch.empty_like(b_dev)
    plan.pcg(b_dev, x_dev, cfg.tol, cfg.max_iters, sptr)   # warm-up (graph build)
    solves = []
    for _ in range(3):
        flush()
        ts = Timer(torch, stream, 1)
        ts.start()
        rep, hist = plan.pcg(b_dev, x_dev, cfg.tol, cfg.max_iters, sptr)
        ts.stop()
        solves.append(ts.times_ms()[0])
    x_sys = x_dev.cpu().numpy()
    x = x_sys[setup.old_positions]
    err = float(np.linalg.norm(x - xs) / np.linalg.norm(xs))
    # e2e solve through the public API: b on host -> x on host
    t_e2e_solve = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solver.solve_on_device(setup, cfg)
        t_e2e_solve.append(time.perf_counter() - t0)
    # the trilab-facing preconditioner call a user makes: numpy r in, numpy
    # z out (pageable host memory, synchronous; src/precond.py:411-425).  The
    # first call builds and uploads the factor plan (untimed).
    r_np = np.random.default_rng(0).standard_normal(n_pad)
    P.apply_ic_preconditioner("hbmc", setup.factor, hl, r_np)
    t_api = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.apply_ic_preconditioner("hbmc", setup.factor, hl, r_np)
        t_api.append(time.perf_counter() - t0)
    P.precond.release_plans(setup.factor)
    del r_np

    # ---------------- max over ranks
    def mx(v):
        if world == 1:
            return v
        tt = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    dev_ms_max = mx(dev_ms)
    e2e_ms_max = mx(e2e_ms)
    value = step_bytes * args.steps * world / (dev_ms_max / 1e3) / 1e9
    e2e_val = step_bytes * args.steps * world / (e2e_ms_max / 1e3) / 1e9

    line = None
    if rank == 0:
        cb = None
        if world == 1 and not args.no_cpu_baseline:
            from oracle import oracle as O
            hd = {"n_pad": n_pad, "w": hl.w, "b_s": hl.b_s, "n_c": hl.n_c,
                  "color_lvl1_ranges": np.asarray(hl.color_lvl1_ranges, dtype=np.int64)}
            cb = cpu_baseline_on_arrays(setup.factor.lower, setup.factor.upper,
                                        setup.factor.inv_diag, hd, step_bytes,
                                        O.max_threads(), 2)
            cb["sample"] += ", on this product's SELL arrays (SURVEY 8(d))"
        dg = load_digest(args.config)
        ref = dg.get("hbmc", {})
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, SURVEY Appendix B)",
            "config": {"workload": f"config{args.config} {label} b_s={bs} w={w}",
                       "N": n, "n_pad": n_pad, "nnz_A": nnz_a, "nnz_L": nnz_l,
                       "n_c": hl.n_c, "bytes_per_step": step_bytes,
                       "l2": "flushed before every timed step (256 MiB read)",
                       "parallelism": f"replicas x{world}" if world > 1 else "1 GPU"},
            "roofline": {"bound": "hbm", "kernel": kernel_name,
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_src,
                         "launches": n_launch, "avg_launch_us": 1e3 * tot_ms / max(1, n_launch),
                         "algorithmic_bytes_per_launch": tot_b / max(1, n_launch),
                         "traffic": traffic, "traffic_source": traffic_src,
                         "per_phase_kernels": per_phase},
            "cpu_baseline": cb,
            "e2e": {"value": e2e_val, "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * n_pad, "d2h_bytes_per_step": 8 * n_pad,
                    "ms_per_step": e2e_ms_max / args.steps,
                    "pipeline": f"H2D / precond / D2H on 3 streams, {nbuf} device buffers",
                    "link_floor_ms_per_step": link_ms,
                    "frac_of_link_floor": link_ms / (e2e_ms_max / args.steps),
                    "api": {"apply_ic_preconditioner_numpy_ms": 1e3 * min(t_api),
                            "apply_ic_preconditioner_GBps": step_bytes / min(t_api) / 1e9,
                            "iccg_host_to_host_ms": 1e3 * min(t_e2e_solve),
                            "note": "per call, pageable numpy in/out, synchronous"}},
            "gpu_launches": args.steps if pinfo["precond"] else launches,
            "clocks": clk.summary(),
            "iccg": {"iterations": int(rep.iterations),
                     "reference_iterations": ref.get("iterations"),
                     "reference_cpu_solve_s": ref.get("time_solve_s"),
                     "reference_cpu_threads": ref.get("threads"),
                     "reference_source": dg.get("source", "reference trilab + numba, "
                                                "survey container (make_golden.py --large)"),
                     "converged": bool(rep.converged),
                     "time_to_solution_ms": min(solves),
                     "ms_per_iteration": min(solves) / max(1, rep.iterations),
                     "kernel_launches": int(rep.kernel_launches),
                     "host_syncs": int(rep.host_syncs),
                     "rel_err_vs_xstar": err,
                     "e2e_solve_ms": 1e3 * min(t_e2e_solve),
                     "setup_host_s": t_host, "setup_total_s": t_setup,
                     "generate_s": t_gen},
            "spmv": spmv_line,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
    return line


def run_partitioned(args, rank, world, local_rank):
    """one rank per GPU, rows of every color split over ranks."""
    import torch
    import torch.distributed as dist

    import paper_1908_00741_b200 as P
    from paper_1908_00741_b200 import distributed as D
    from paper_1908_00741_b200 import solver

    dev = torch.device("cuda", local_rank)
    # rank-local setup: rank 0 alone generates and builds the system
    # (distributed.prepare_rank_parts); every rank loads only its part
    import workloads
    label, _, bs, w = workloads.CONFIGS[args.config]
    a = b = None
    t_gen = 0.0
    sizes = [None]
    if rank == 0:
        label, a, xs, b, bs, w, t_gen = build_problem(args.config)
        sizes = [(a.n, int(a.nnz))]
    dist.broadcast_object_list(sizes, src=0)
    n_glob, nnz_glob = sizes[0]
    cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
    t0 = time.perf_counter()
    part, b_part, info = D.prepare_rank_parts(a, b, cfg, world, rank, dist)
    del a, b
    ops = D.CudaRankOps(part)
    drv = D.DistHbmc([part], [ops], transport=args.transport)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    nnz_l = (nnz_glob - n_glob) // 2
    step_bytes = 2 * sweep_bytes(nnz_l, n_glob)
    stream = torch.cuda.current_stream(dev)
    flush_src = torch.ones(L2_FLUSH_BYTES // 8, dtype=torch.float64, device=dev)
    flush_dst = torch.empty((), dtype=torch.float64, device=dev)

    def flush():
        torch.sum(flush_src, dim=0, out=flush_dst)

    def barrier():
        dist.barrier()
        torch.cuda.synchronize()

    r_glob = np.random.default_rng(0).standard_normal(info["n_pad"])
    r = [ops.from_host(np.concatenate([r_glob[part.rows], np.zeros(part.n_halo)]))]
    y, z = [drv.ext_vec(0, "y")], [drv.ext_vec(0, "z")]
    for _ in range(args.warmup):
        flush()
        drv.precond(r, y, z)
    barrier()
    tm = Timer(torch, stream, args.steps)
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush()
            tm.start()
            drv.precond(r, y, z)
            tm.stop()
        dev_ms = sum(tm.times_ms())
    barrier()
    # e2e: local r from pinned host, z back to pinned host
    r_host = torch.from_numpy(r_glob[part.rows].copy()).pin_memory()
    z_host = torch.empty(part.n_loc, dtype=torch.float64).pin_memory()
    te = Timer(torch, stream, args.steps)
    for _ in range(args.steps):
        flush()
        te.start()
        r[0][:part.n_loc].copy_(r_host, non_blocking=True)
        drv.precond(r, y, z)
        z_host.copy_(z[0][:part.n_loc], non_blocking=True)
        te.stop()
    e2e_ms = sum(te.times_ms())
    barrier()
    # ICCG time-to-solution (host-timed around a synchronised solve)
    b_loc = [ops.from_host(b_part)]
    drv.pcg(b_loc, cfg.tol, cfg.max_iters)
    barrier()
    t1 = time.perf_counter()
    xs_loc, it, hist, conv = drv.pcg(b_loc, cfg.tol, cfg.max_iters)
    torch.cuda.synchronize()
    solve_ms = 1e3 * (time.perf_counter() - t1)

    def mx(v):
        tt = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    dev_ms_max, e2e_ms_max, solve_ms_max = mx(dev_ms), mx(e2e_ms), mx(solve_ms)
    value = step_bytes * args.steps / (dev_ms_max / 1e3) / 1e9
    peak, peak_src = load_peaks()
    if rank == 0:
        per_gpu = value / world
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, SURVEY Appendix B)",
            "config": {"workload": f"config{args.config} {label} b_s={bs} w={w}",
                       "N": n_glob, "n_pad": info["n_pad"], "nnz_L": nnz_l,
                       "n_c": info["n_c"], "bytes_per_step": step_bytes,
                       "l2": "flushed before every timed step (256 MiB read)",
                       "parallelism": f"row-partitioned x{world} (per-color halo exchange: "
                                      f"{'NVLink peer stores + flags' if args.transport == 'p2p' else 'NCCL send/recv'})",
                       "halo_rows_rank0": part.n_halo, "rows_rank0": part.n_loc},
            "roofline": {"bound": "hbm", "kernel": "per-rank HBMC sweep phases + halo exchange",
                         "achieved": per_gpu, "peak": peak, "unit": "GB/s",
                         "frac": per_gpu / peak, "peak_source": peak_src, "traffic": None},
            "cpu_baseline": None,
            "e2e": {"value": step_bytes * args.steps / (e2e_ms_max / 1e3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * part.n_loc, "d2h_bytes_per_step": 8 * part.n_loc,
                    "ms_per_step": e2e_ms_max / args.steps},
            "gpu_launches": args.steps * (2 * info["n_c"] + 2 * max(info["n_c"] - 1, 0)),
            "clocks": clk.summary(),
            "iccg": {"iterations": int(it), "converged": bool(conv),
                     "time_to_solution_ms": solve_ms_max, "setup_total_s": t_setup,
                     "exchanges_per_precond": 2 * max(info["n_c"] - 1, 0),
                     "reductions_per_iteration": drv.reductions_per_iteration,
                     "setup": "rank-local: rank 0 builds, each rank loads only its part"},
        }
        print(json.dumps(line), flush=True)
    drv.close()
    ops.close()
    dist.barrier()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--ref-iccg-budget-s", type=float, default=30.0,
                    help="--impl reference: full ICCG if it fits, else a timed prefix")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="partitioned", choices=["partitioned", "replicas"],
                    help="N > 1: row-partitioned solve (default) or independent replicas")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="partitioned halo exchange: NVLink peer stores (default) or NCCL")
    ap.add_argument("--force-partitioned", action="store_true",
                    help="run the partitioned path even at N = 1 (code-path check)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the dominant kernel (profiles/)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    partitioned = args.mode == "partitioned" and (world > 1 or args.force_partitioned)
    if world > 1 or partitioned:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local_rank))
    if partitioned:
        run_partitioned(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1 or partitioned:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

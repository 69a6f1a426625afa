"""Per-phase timing of the sweep kernel families on a BASELINE config.

    TB_SWEEP=<family> python scripts/sweep_micro.py [config] [reps]

Timing hygiene: events are created up front and every rep is enqueued
without a host synchronisation (flush, e0, kernel, e1, ...), so host launch
overhead is never inside a timed window; the L2 flush READS 256 MiB (a write
flush would leave dirty lines whose write-back lands in the next kernel).
Also reports a back-to-back figure (reps launches between one event pair).
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np
import torch

import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import solver
import workloads as problems

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
label, gen, bs, w = problems.CONFIGS[cfg_id]
a = gen()
xs, b = problems.rhs(a)
cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
setup = solver.prepare(a, b, cfg)
solver.attach_plan(setup, cfg)
plan, hl = setup.plan, setup.layout
n = hl.n_pad
r = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
y = torch.empty_like(r)
z = torch.empty_like(r)
flush_src = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
flush_dst = torch.empty(1, dtype=torch.float64, device="cuda")
span = bs * w
lower = np.diff(P.precond._strict_tri(setup.a_sys).row_ptr)
upper = np.diff(P.precond._strict_tri(setup.a_sys, upper=True).row_ptr)
E = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
     for _ in range(reps + 3)]
B0, B1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def flush():
    flush_dst.copy_(flush_src.sum())


def timed(fn, do_flush):
    torch.cuda.synchronize()
    for e0, e1 in E:
        if do_flush:
            flush()
        e0.record()
        fn()
        e1.record()
    torch.cuda.synchronize()
    ts = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in E[3:])
    return ts[len(ts) // 2]


def back_to_back(fn):
    fn()
    torch.cuda.synchronize()
    flush()
    B0.record()
    for _ in range(reps):
        fn()
    B1.record()
    torch.cuda.synchronize()
    return B0.elapsed_time(B1) * 1e3 / reps


tot_cold = tot_b2b = tot_b = 0.0
for fw in (True, False):
    colors = range(hl.n_c) if fw else range(hl.n_c - 1, -1, -1)
    for c in colors:
        k0, k1 = int(hl.color_lvl1_ranges[c]), int(hl.color_lvl1_ranges[c + 1])
        cnt = (lower if fw else upper)[k0 * span:k1 * span]
        nb = 12 * int(cnt.sum()) + 32 * (k1 - k0) * span
        if fw:
            f = lambda c=c: plan.sweep_phase(True, c, r, y)
        else:
            f = lambda c=c: plan.sweep_phase(False, c, y, z)
        tc = timed(f, True)
        tb = back_to_back(f)
        src = torch.empty(nb // 16, dtype=torch.float64, device="cuda")
        dstc = torch.empty_like(src)
        tcopy = timed(lambda: dstc.copy_(src), True)
        info = plan.phase_info(fw, c)
        print(f"{'fwd' if fw else 'bwd'} color {c}: kind {info['staged']} "
              f"maxl {info['max_slots']} | {nb/1e6:7.1f} MB | flushed {tc:6.1f} us "
              f"({nb/tc/1e3:5.0f} GB/s) | back-to-back {tb:6.1f} us ({nb/tb/1e3:5.0f} GB/s) "
              f"| copy same bytes {tcopy:5.1f} us ({nb/tcopy/1e3:5.0f} GB/s)")
        tot_cold += tc
        tot_b2b += tb
        tot_b += nb
full = timed(lambda: plan.precond(r, z), True)
fb2b = back_to_back(lambda: plan.precond(r, z))
print(f"sum of phases: flushed {tot_cold:.1f} us ({tot_b/tot_cold/1e3:.0f} GB/s), b2b "
      f"{tot_b2b:.1f} us; precond flushed {full:.1f} us ({tot_b/full/1e3:.0f} GB/s), "
      f"precond b2b {fb2b:.1f} us ({tot_b/fb2b/1e3:.0f} GB/s)")

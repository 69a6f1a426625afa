"""Host<->device copy ceiling for bench.py's e2e leg.

    python scripts/pcie_probe.py [n_doubles=2097152] [reps=20]

Times, with CUDA events, pinned-memory H2D alone, D2H alone, and H2D + D2H
issued concurrently on two streams (the e2e pipeline's steady state), for
the config-2 vector size.  Prints GB/s per direction and the per-step floor
the e2e leg cannot go below (max of the concurrent pair).
"""
import json
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2097152
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
nb = n * 8
h_in = torch.randn(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.randn(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    for _ in range(reps):
        fn()
    cur.wait_stream(s1)
    cur.wait_stream(s2)
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


t_in, t_out, t_both = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"bytes_per_direction": nb, "h2d_ms": t_in, "h2d_GBps": nb / t_in / 1e6,
                  "d2h_ms": t_out, "d2h_GBps": nb / t_out / 1e6,
                  "concurrent_ms": t_both, "concurrent_GBps_per_direction": nb / t_both / 1e6}))

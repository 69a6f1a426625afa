"""Config-5 golden digest from an INDEPENDENT build: the CPU oracle.

BASELINE config 5 (anisotropic 7-point 512^3, N = 134,217,728, b_s = 16,
w = 32) does not fit the reference `trilab` in this container's RAM (SURVEY
8(c)), so its golden comes from the CPU oracle (oracle/), which is pinned
bitwise to the reference on every small golden and on the full-size config
2-4 digests (tests/test_oracle.py, tests/golden/config*_digest.json).  This
script runs on the B200 box's host (196 GB RAM, 16 cores): nothing here
loads the product library -- the matrix is assembled by the oracle's
coo_to_csr (workloads.py, backend="oracle"), the ordering, padding,
permutation, IC(0), SELL packing and the whole PCG solve
(src/solver.py:139-204, numpy dots as in the reference) are the oracle's.

    python tests/golden/make_config5_digest.py               # 512^3 (~15 min)
    python tests/golden/make_config5_digest.py --size 64 --out /tmp/d.json

The digest has the fields of config{2,3,4}_digest.json (made from the
reference by make_golden.py --large) plus sha256 of L.vals and d.
"""

import argparse
import hashlib
import json
import os
import platform
import resource
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, REPO)

import workloads  # noqa: E402
from oracle import oracle as O  # noqa: E402


def arr_hash(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def a_hash(a):
    h = hashlib.sha256()
    for arr in (a.row_ptr, a.col_idx, a.vals):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--out", default=os.path.join(HERE, "config5_digest.json"))
    ap.add_argument("--max-iters", type=int, default=50000)
    args = ap.parse_args()
    threads = O.max_threads()
    t0 = time.perf_counter()
    a = workloads.lap7(args.size, 1.0, 1.0, 1e-3, backend="oracle")
    xs, b = workloads.rhs(a, backend="oracle")
    t_gen = time.perf_counter() - t0
    out = {"config": 5, "label": f"aniso7_{args.size}^3", "n": a.n, "nnz": int(a.nnz),
           "a_hash": a_hash(a), "b_s": 16, "w": 32,
           "source": "CPU oracle (oracle/hbmc_oracle.c + oracle/oracle.py), "
                     "tests/golden/make_config5_digest.py on the B200 host",
           "host": {"cpu": cpu_model(), "threads": threads}}
    print(f"generated N={a.n} nnz={a.nnz} in {t_gen:.1f}s", flush=True)

    t0 = time.perf_counter()
    block_of, nb, bptr, members = O.build_blocks(a, 16)
    lay = O.color_blocks(a, block_of, nb, bptr, members)
    hl = O.build_hbmc(a.n, lay, 16, 32)
    out.update(n_c=int(lay["n_c"]), n_pad=int(hl["n_pad"]), n_dummy=int(hl["n_dummy"]),
               nbar_of=[int(v) for v in hl["nbar_of"]],
               composed_hash=arr_hash(hl["composed"]),
               bmc_perm_hash=arr_hash(lay["perm"]),
               color_of_block_hash=arr_hash(lay["color_of_block"]))
    del block_of, bptr, members
    t_order = time.perf_counter() - t0
    print(f"ordering {t_order:.1f}s n_c={lay['n_c']} nbar={hl['nbar_of']}", flush=True)

    # the oracle's HbmcSystem pipeline, step by step so large temporaries
    # can be dropped (src/solver.py:127-136)
    t0 = time.perf_counter()
    a_ext, b_ext = O.extend_with_dummies(a, b, hl)
    a_o, b_o = O.permute_system(a_ext, b_ext, hl["composed"])
    del a_ext, a
    L, d, inv_d, U = O.ic0_factorize(a_o)
    out["nnz_L"] = int(L.nnz)
    out["L_vals_hash"] = arr_hash(L.vals)
    out["d_hash"] = arr_hash(d)
    sysx = O.HbmcSystem.__new__(O.HbmcSystem)
    sysx.hl, sysx.lay, sysx.b_sys = hl, lay, b_o
    sysx.d, sysx.inv_d = d, inv_d
    sysx.Ls = O.csr_to_sell(L, 32)
    del L
    sysx.Us = O.csr_to_sell(U, 32)
    del U
    out["L_sell_vals_hash"] = arr_hash(sysx.Ls.vals)
    out["U_sell_vals_hash"] = arr_hash(sysx.Us.vals)
    out["L_sell_slice_len_hash"] = arr_hash(sysx.Ls.slice_len)
    sysx.As = O.csr_to_sell(a_o, 32)
    del a_o
    sysx.nnz_L = out["nnz_L"]
    t_setup = time.perf_counter() - t0 + t_order
    print(f"setup {t_setup:.1f}s", flush=True)

    t0 = time.perf_counter()
    x, it, hist, conv = O.pcg_hbmc(sysx, max_iters=args.max_iters, threads=threads,
                                   spmv_threads=threads)
    t_solve = time.perf_counter() - t0
    stride = max(1, out["n"] // 4096)
    out["hbmc"] = {"iterations": int(it), "converged": bool(conv),
                   "history": [float(h) for h in hist],
                   "time_setup_s": t_setup, "time_solve_s": t_solve,
                   "time_generate_s": t_gen, "threads": threads,
                   "x_sample_stride": stride,
                   "x_sample": [float(v) for v in x[::stride]],
                   "x_hash": arr_hash(x),
                   "x_norm": float(np.linalg.norm(x)),
                   "err_vs_xstar": float(np.linalg.norm(x - xs) / np.linalg.norm(xs))}
    out["max_rss_gb"] = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6
    print(f"pcg {it} iterations in {t_solve:.1f}s converged={conv} "
          f"err={out['hbmc']['err_vs_xstar']:.3e} rss={out['max_rss_gb']:.1f} GB", flush=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()

"""Generate the golden fixtures from the REFERENCE implementation.

Runs only in the build container, where the read-only reference lives at
/root/reference.  It copies /root/reference/pkg to a scratch directory (the
numba cache needs a writable tree), imports `trilab` from there and records,
for each small case, the reference's own outputs on inputs produced by this
repo's generators (the generator itself is pinned by an A hash):

  ordering:  composed HBMC permutation, nbar_of, n_dummy, n_c, block_of,
             color_of_block, nodal color_of, BMC permutation
  factor:    IC(0) L values and d in HBMC order
  kernels:   forward / backward HBMC sweeps of r = default_rng(0).normal(n_pad),
             SELL SpMV of x = default_rng(2).normal(n_pad)
  solves:    pcg iterations, residual history and x for hbmc (sell SpMV),
             bmc, mc, natural

Large configs (BASELINE configs 1-4) get digests only (`--large`).

    python tests/golden/make_golden.py            # small cases (~1 min)
    python tests/golden/make_golden.py --large 2  # config 2 digests (~1 min)
"""

import hashlib
import json
import os
import shutil
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, REPO)

import workloads as problems  # noqa: E402
from paper_1908_00741_b200 import matrix as M  # noqa: E402


def load_reference():
    scratch = os.path.join(tempfile.gettempdir(), "trilab_ref_copy")
    if not os.path.exists(os.path.join(scratch, "src", "trilab")):
        shutil.rmtree(scratch, ignore_errors=True)
        shutil.copytree("/root/reference/pkg", scratch)
    sys.path.insert(0, os.path.join(scratch, "src"))
    import trilab
    return trilab


def a_hash(a):
    h = hashlib.sha256()
    for arr in (a.row_ptr, a.col_idx, a.vals):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def arr_hash(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def to_ref(T, a):
    return T.CsrMatrix(a.n, a.row_ptr.copy(), a.col_idx.copy(), a.vals.copy())


def path_matrix(n, diag=4.0, off=-1.0):
    rows, cols, vals = [], [], []
    for i in range(n):
        rows.append(i); cols.append(i); vals.append(diag)
        if i + 1 < n:
            rows += [i, i + 1]
            cols += [i + 1, i]
            vals += [off, off]
    return M.coo_to_csr(M.CooMatrix(n, np.array(rows), np.array(cols),
                                    np.array(vals, dtype=float)))


SMALL = {
    # name: (builder, b_s, w, rhs)  rhs "ones" or "xstar"
    "path16_b2_w4": (lambda: path_matrix(16), 2, 4, "ones"),
    "grid5_b4_w4": (lambda: M.gen_laplacian_5pt(5, 5)[0], 4, 4, "ones"),
    "grid8_b4_w4": (lambda: M.gen_laplacian_5pt(8, 8)[0], 4, 4, "ones"),
    "grid16_b4_w2": (lambda: M.gen_laplacian_5pt(16, 16)[0], 4, 2, "ones"),
    "grid32_b8_w4": (lambda: M.gen_laplacian_5pt(32, 32)[0], 8, 4, "ones"),
    "rand500_b8_w4": (lambda: M.gen_random_spd(500, density=0.01, seed=100), 8, 4, "ones"),
    "rand300_b3_w5": (lambda: M.gen_random_spd(300, density=0.02, seed=21), 3, 5, "ones"),
    "lap7_12_b4_w8": (lambda: problems.lap7(12), 4, 8, "xstar"),
    "var7_16_b8_w32": (lambda: problems.varcoef7(16, seed=0), 8, 32, "xstar"),
    "s27_10_b8_w32": (lambda: problems.stencil27(10, seed=0), 8, 32, "xstar"),
    "knn3000_b4_w32": (lambda: problems.knn_graph(3000, seed=0), 4, 32, "xstar"),
    "aniso12_b16_w32": (lambda: problems.lap7(12, 1.0, 1.0, 1e-3), 16, 32, "xstar"),
    "config1_full": (lambda: problems.lap7(32), 4, 8, "xstar"),
}


def small_case(T, name, spec):
    build, bs, w, rhs_kind = spec
    a = build()
    ra = to_ref(T, a)
    if rhs_kind == "ones":
        b = np.ones(a.n)
    else:
        _, b = problems.rhs(a)
        assert np.array_equal(b, T.spmv(ra, np.random.default_rng(1).uniform(-1, 1, a.n)))
    out = {"a_hash": np.array(a_hash(a)), "b": b, "b_s": bs, "w": w}
    lay = T.color_blocks(ra, T.build_blocks(ra, bs))
    hl = T.build_hbmc(lay, w)
    out.update(composed=hl.composed_perm.new_of_old, nbar_of=hl.nbar_of,
               n_dummy=hl.n_dummy, n_c=hl.n_c, n_pad=hl.n_pad,
               block_of=lay.blocking.block_of, color_of_block=lay.color_of_block,
               bmc_perm=lay.perm.new_of_old,
               color_lvl1_ranges=hl.color_lvl1_ranges)
    nod = T.greedy_color_nodes(ra)
    out.update(node_color=nod.color_of, mc_perm=nod.perm.new_of_old)
    a_ext, b_ext = T.extend_with_dummies(ra, b, hl)
    af, bf = T.permute_system(a_ext, b_ext, hl.composed_perm)
    f = T.ic0_factorize(af, layout_tag="hbmc")
    sf = T.build_sell_factor(f, hl)
    out.update(L_vals=f.L.vals, d=f.d, b_sys=bf)
    r = np.random.default_rng(0).standard_normal(hl.n_pad)
    y = T.sub_forward_hbmc(sf, hl, r)
    z = T.sub_backward_hbmc(sf, hl, y)
    assert np.array_equal(y, T.sub_forward_seq(f, r))
    assert np.array_equal(z, T.sub_backward_seq(f, y))
    out.update(r=r, y=y, z=z)
    xs = np.random.default_rng(2).standard_normal(hl.n_pad)
    out.update(spmv_x=xs, spmv_sell=T.spmv(T.csr_to_sell(af, w), xs),
               spmv_csr=T.spmv(af, xs))
    # MC / BMC seq sweeps of the same r (first a.n entries)
    for kind, perm in (("mc", nod.perm), ("bmc", lay.perm)):
        ap, _ = T.permute_system(ra, b, perm)
        fk = T.ic0_factorize(ap, layout_tag=kind)
        rk = r[:a.n]
        yk = T.sub_forward_seq(fk, rk)
        out[f"{kind}_y"] = yk
        out[f"{kind}_z"] = T.sub_backward_seq(fk, yk)
    fnat = T.ic0_factorize(ra)
    ynat = T.sub_forward_seq(fnat, r[:a.n])
    out.update(nat_y=ynat, nat_z=T.sub_backward_seq(fnat, ynat))
    for ordering in ("hbmc", "bmc", "mc", "natural"):
        cfg = T.CgConfig(ordering=ordering, b_s=bs, w=w,
                         spmv_format="sell" if ordering == "hbmc" else "crs")
        x, rep = T.pcg(ra, b, cfg)
        out[f"pcg_{ordering}_iters"] = rep.iterations
        out[f"pcg_{ordering}_hist"] = np.array(rep.residual_history)
        out[f"pcg_{ordering}_x"] = x
        out[f"pcg_{ordering}_barriers"] = rep.barrier_total
        out[f"pcg_{ordering}_converged"] = rep.converged
    return out


LARGE = {
    1: lambda: problems.lap7(32),
    2: lambda: problems.varcoef7(128, seed=0),
    3: lambda: problems.stencil27(192, seed=0),
    4: lambda: problems.knn_graph(4_000_000, seed=0),
}


def large_case(T, cfg_id, orderings):
    label, _, bs, w = problems.CONFIGS[cfg_id]
    t0 = time.time()
    a = LARGE[cfg_id]()
    xs, b = problems.rhs(a)
    ra = to_ref(T, a)
    lay = T.color_blocks(ra, T.build_blocks(ra, bs))
    hl = T.build_hbmc(lay, w)
    rec = {"config": cfg_id, "label": label, "n": a.n, "nnz": int(a.nnz),
           "a_hash": a_hash(a), "b_s": bs, "w": w, "n_c": hl.n_c,
           "n_pad": hl.n_pad, "n_dummy": hl.n_dummy,
           "nbar_of": hl.nbar_of.tolist(),
           "composed_hash": arr_hash(hl.composed_perm.new_of_old),
           "bmc_perm_hash": arr_hash(lay.perm.new_of_old),
           "color_of_block_hash": arr_hash(lay.color_of_block)}
    stride = max(1, a.n // 4096)
    for ordering in orderings:
        cfg = T.CgConfig(ordering=ordering, b_s=bs, w=w, threads=os.cpu_count(),
                         spmv_format="sell" if ordering == "hbmc" else "crs")
        x, rep = T.pcg(ra, b, cfg)
        rec[ordering] = {
            "iterations": rep.iterations, "converged": rep.converged,
            "history": rep.residual_history,
            "time_setup_s": rep.time_setup_s, "time_solve_s": rep.time_solve_s,
            "threads": os.cpu_count(),
            "x_sample_stride": stride, "x_sample": x[::stride].tolist(),
            "x_norm": float(np.linalg.norm(x)),
            "err_vs_xstar": float(np.linalg.norm(x - xs) / np.linalg.norm(xs)),
        }
        print(f"config {cfg_id} {ordering}: {rep.iterations} iters, setup "
              f"{rep.time_setup_s:.1f}s solve {rep.time_solve_s:.1f}s", flush=True)
    rec["wall_s"] = time.time() - t0
    return rec


def main():
    T = load_reference()
    if "--large" in sys.argv:
        cfg_id = int(sys.argv[sys.argv.index("--large") + 1])
        orderings = ["hbmc", "bmc"] + (["mc"] if cfg_id in (1, 3) else [])
        rec = large_case(T, cfg_id, orderings)
        with open(os.path.join(HERE, f"config{cfg_id}_digest.json"), "w") as fh:
            json.dump(rec, fh, indent=1)
        return
    only = sys.argv[1:] or list(SMALL)
    for name in only:
        t0 = time.time()
        out = small_case(T, name, SMALL[name])
        if name == "config1_full":
            # keep the fixture small: bitwise-compared arrays become sha256
            # digests; regenerable inputs (r, spmv_x, b) are dropped
            for key in ("L_vals", "y", "z", "spmv_sell", "spmv_csr", "b_sys",
                        "mc_y", "mc_z", "bmc_y", "bmc_z", "nat_y", "nat_z"):
                out[key + "_sha"] = np.array(arr_hash(out.pop(key)))
            for key in ("r", "spmv_x", "b", "pcg_bmc_x", "pcg_mc_x",
                        "pcg_natural_x"):
                out.pop(key)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(f"{name}: n_pad={out['n_pad']} n_c={out['n_c']} hbmc iters "
              f"{out['pcg_hbmc_iters']} ({time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    main()

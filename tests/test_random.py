"""Property-based parity on random matrices (hypothesis).

CPU: the product's host builder (ordering, padding, HBMC permutation,
permutation of the system, IC(0), SELL packing) is bit-exact with the C /
numpy oracle on random SPD matrices of random size and sparsity, random
b_s and w (dummies, undersized blocks, w > blocks per color, diagonal-only
and single-row systems included); the HBMC dependency structure the device
kernels rely on holds; the row partition covers every row once.
GPU: sweeps and SpMV bitwise against the oracle, PCG within the bar.
Examples are derandomized (reproducible) and sized to run in seconds.
"""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_1908_00741_b200 as P
from conftest import rel_err
from oracle import oracle as O
from paper_1908_00741_b200 import distributed, precond, solver
from paper_1908_00741_b200.matrix import CooMatrix, coo_to_csr

SETTINGS = dict(max_examples=40, deadline=None, derandomize=True,
                suppress_health_check=[HealthCheck.too_slow])


@st.composite
def systems(draw):
    """(matrix, b_s, w): random sparse SPD (diagonally dominant M-matrix
    or the reference's gen_random_spd), random symmetric renumbering."""
    n = draw(st.integers(1, 260))
    kind = draw(st.sampled_from(["spd", "lap", "diag"]))
    seed = draw(st.integers(0, 2**31 - 1))
    rng = np.random.default_rng(seed)
    if kind == "spd" or n < 3:
        a = P.gen_random_spd(n, density=draw(st.floats(0.0, 0.2)), seed=seed)
    elif kind == "diag":
        a = coo_to_csr(CooMatrix(n, np.arange(n), np.arange(n), rng.uniform(1, 2, n)))
    else:   # random graph Laplacian + shift, random degree
        m = draw(st.integers(0, 4 * n))
        i, j = rng.integers(0, n, m), rng.integers(0, n, m)
        keep = i != j
        e = np.unique(np.sort(np.stack([i[keep], j[keep]], 1), axis=1), axis=0)
        w_ = rng.uniform(0.1, 2.0, e.shape[0])
        diag = np.full(n, 1e-3)
        np.add.at(diag, e[:, 0], w_)
        np.add.at(diag, e[:, 1], w_)
        rows = np.concatenate([e[:, 0], e[:, 1], np.arange(n)])
        cols = np.concatenate([e[:, 1], e[:, 0], np.arange(n)])
        a = coo_to_csr(CooMatrix(n, rows, cols, np.concatenate([-w_, -w_, diag])))
    if draw(st.booleans()) and n > 1:   # random renumbering (algebraic coloring)
        q = rng.permutation(n)
        a, _ = P.permute_system(a, np.zeros(n), P.Permutation(q))
    b_s = draw(st.integers(1, 8))
    w = draw(st.sampled_from([1, 2, 3, 4, 8, 16, 32]))
    return a, b_s, w


def product_system(a, b, b_s, w):
    cfg = P.CgConfig(ordering="hbmc", b_s=b_s, w=w, spmv_format="sell")
    return solver.prepare(a, b, cfg)


@settings(**SETTINGS)
@given(systems())
def test_host_builder_bit_exact_vs_oracle(sys_):
    a, b_s, w = sys_
    b = np.random.default_rng(3).uniform(-1, 1, a.n)
    st_ = product_system(a, b, b_s, w)
    hl, sf = st_.layout, st_.factor
    ob = O.HbmcSystem(O.Csr(a.n, a.row_ptr, a.col_idx, a.vals), b, b_s, w)
    assert np.array_equal(hl.composed_perm.new_of_old, ob.hl["composed"])
    assert hl.n_c == ob.hl["n_c"] and hl.n_pad == ob.hl["n_pad"]
    assert np.array_equal(hl.color_lvl1_ranges, ob.hl["color_lvl1_ranges"])
    assert np.array_equal(st_.b_sys, ob.b_sys)
    assert np.array_equal(sf.d, ob.d) and np.array_equal(sf.inv_diag, ob.inv_d)
    for mine, ref in ((sf.lower, ob.Ls), (sf.upper, ob.Us)):
        assert np.array_equal(mine.slice_ptr, ref.slice_ptr)
        assert np.array_equal(mine.slice_len, ref.slice_len)
        assert np.array_equal(mine.col_idx, ref.col_idx)
        assert np.array_equal(mine.vals, ref.vals)
    # the dependency structure the per-color device schedules rely on
    precond._check_hbmc_lower_structure(precond._strict_tri(st_.a_sys), hl)


@settings(**SETTINGS)
@given(systems(), st.integers(1, 5))
def test_partition_covers_rows_and_halo_offsets(sys_, world):
    a, b_s, w = sys_
    st_ = product_system(a, np.ones(a.n), b_s, w)
    parts = distributed.partition_setup(st_, world)
    rows = np.concatenate([p.rows for p in parts])
    assert np.array_equal(np.sort(rows), np.arange(st_.layout.n_pad))
    for p in parts:
        for ex in [p.spmv] + p.fwd + p.bwd:
            for m in ex.sends:
                q = parts[m.peer]
                assert q.n_loc <= m.remote_offset <= q.n_ext - m.count
                got = q.halo_rows[m.remote_offset - q.n_loc:m.remote_offset - q.n_loc + m.count]
                assert np.array_equal(p.rows[ex.send_idx[m.offset:m.offset + m.count]], got)


@pytest.mark.gpu
@settings(**{**SETTINGS, "max_examples": 25})
@given(systems())
def test_device_sweeps_spmv_pcg_random(sys_):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a, b_s, w = sys_
    b = np.random.default_rng(3).uniform(-1, 1, a.n)
    st_ = product_system(a, b, b_s, w)
    hl, sf = st_.layout, st_.factor
    ob = O.HbmcSystem(O.Csr(a.n, a.row_ptr, a.col_idx, a.vals), b, b_s, w)
    r = np.random.default_rng(0).standard_normal(hl.n_pad)
    y = P.sub_forward_hbmc(sf, hl, r)
    z = P.sub_backward_hbmc(sf, hl, y)
    yo = O.hbmc_sweep(True, ob.Ls, ob.inv_d, r, ob.hl)
    assert np.array_equal(y, yo)
    assert np.array_equal(z, O.hbmc_sweep(False, ob.Us, ob.inv_d, yo, ob.hl))
    assert np.array_equal(P.spmv(P.csr_to_sell(st_.a_sys, w), r), O.spmv_sell(ob.As, r))
    x, rep = P.pcg(a, b, P.CgConfig(ordering="hbmc", b_s=b_s, w=w, spmv_format="sell"))
    xo, it, _, conv = O.pcg_hbmc(ob)
    assert rep.converged == conv and abs(rep.iterations - it) <= 1
    assert rel_err(x, xo) <= 1e-10

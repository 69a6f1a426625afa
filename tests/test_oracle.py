"""Pin the CPU oracle (oracle/) to the reference's golden outputs.

The fixtures were produced by importing the reference `trilab` itself
(tests/golden/make_golden.py).  Bitwise for ordering, factor, sweeps and
SpMV; the oracle's PCG uses numpy dots exactly like the reference, so its
iteration counts and histories must match too.
"""

import hashlib

import numpy as np
import pytest

from conftest import golden_matrix, golden_names, load_golden, rel_err
from oracle import oracle as O

NAMES = golden_names()


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def same(g, key, arr):
    if key in g:
        return np.array_equal(arr, g[key])
    return sha(arr) == str(g[key + "_sha"])


def oracle_csr(a):
    return O.Csr(a.n, a.row_ptr, a.col_idx, a.vals)


@pytest.fixture(scope="module", params=NAMES)
def case(request):
    name = request.param
    g = load_golden(name)
    a, bs, w, rhs_kind = golden_matrix(name)
    return name, g, oracle_csr(a), bs, w, rhs_kind


def test_generator_pinned(case):
    name, g, a, bs, w, _ = case
    h = hashlib.sha256()
    for arr in (a.row_ptr, a.col_idx, a.vals):
        h.update(arr.tobytes())
    assert h.hexdigest() == str(g["a_hash"])


def test_ordering_bitwise(case):
    name, g, a, bs, w, _ = case
    block_of, nb, bptr, members = O.build_blocks(a, bs)
    assert np.array_equal(block_of, g["block_of"])
    lay = O.color_blocks(a, block_of, nb, bptr, members)
    assert np.array_equal(lay["color_of_block"], g["color_of_block"])
    assert np.array_equal(lay["perm"], g["bmc_perm"])
    hl = O.build_hbmc(a.n, lay, bs, w)
    assert np.array_equal(hl["composed"], g["composed"])
    assert np.array_equal(hl["nbar_of"], g["nbar_of"])
    assert hl["n_dummy"] == int(g["n_dummy"])
    col = O.greedy_color(a)
    assert np.array_equal(col, g["node_color"])
    perm, _ = O.group_perm(col, int(col.max()) + 1)
    assert np.array_equal(perm, g["mc_perm"])


def test_factor_sweeps_spmv_bitwise(case):
    name, g, a, bs, w, rhs_kind = case
    b = np.ones(a.n)
    sysx = O.HbmcSystem(a, b, bs, w)
    assert same(g, "L_vals", sysx.L.vals)
    assert np.array_equal(sysx.d, g["d"])
    r = np.random.default_rng(0).standard_normal(sysx.hl["n_pad"])
    for threads in (1, 3):
        y = O.hbmc_sweep(True, sysx.Ls, sysx.inv_d, r, sysx.hl, threads)
        z = O.hbmc_sweep(False, sysx.Us, sysx.inv_d, y, sysx.hl, threads)
        assert same(g, "y", y)
        assert same(g, "z", z)
    assert np.array_equal(O.fwd_seq(sysx.L, sysx.inv_d, r), y)
    x = np.random.default_rng(2).standard_normal(sysx.hl["n_pad"])
    assert same(g, "spmv_sell", O.spmv_sell(sysx.As, x))
    assert same(g, "spmv_sell", O.spmv_sell(sysx.As, x, threads=4))
    assert same(g, "spmv_csr", O.spmv_csr(sysx.a_sys, x))


def test_pcg_hbmc_matches_reference(case):
    name, g, a, bs, w, rhs_kind = case
    if rhs_kind == "ones":
        b = np.ones(a.n)
    else:
        b = np.random.default_rng(1).uniform(-1, 1, a.n)
        b = O.spmv_csr(a, b)
    sysx = O.HbmcSystem(a, b, bs, w)
    x, it, hist, conv = O.pcg_hbmc(sysx)
    assert it == int(g["pcg_hbmc_iters"])
    assert conv == bool(g["pcg_hbmc_converged"])
    assert np.allclose(hist, g["pcg_hbmc_hist"], rtol=1e-12, atol=0)
    assert rel_err(x, g["pcg_hbmc_x"]) <= 1e-12


@pytest.mark.parametrize("cfg_id,size", [(1, 9), (2, 10), (3, 7), (4, 2000), (5, 11)])
def test_oracle_assembly_equals_product(cfg_id, size):
    """workloads.py assembles the same COO through the oracle's C
    coo_to_csr (bench.py's reference arm) and the product's: same CSR, same
    b = A x* (src/matrix.py:168-197, K/numba_backend.py:16-23)."""
    import workloads
    ap, _, _ = workloads.scaled(cfg_id, size)
    ao, _, _ = workloads.scaled(cfg_id, size, backend="oracle")
    assert np.array_equal(ap.row_ptr, ao.row_ptr)
    assert np.array_equal(ap.col_idx, ao.col_idx)
    assert np.array_equal(ap.vals, ao.vals)
    _, bp = workloads.rhs(ap)
    _, bo = workloads.rhs(ao, backend="oracle")
    assert np.array_equal(bp, bo)


def test_oracle_coo_duplicate_rejected():
    row = np.array([0, 1, 1, 0], dtype=np.int64)
    col = np.array([0, 1, 1, 1], dtype=np.int64)
    with pytest.raises(ValueError, match=r"duplicate entry at \(1, 1\)"):
        O.coo_to_csr(2, row, col, np.ones(4))


def test_oracle_permute_transpose_match_numpy(rng):
    """or_permute_csr / or_csr_transpose == the reference's COO -> lexsort
    formulation (src/matrix.py:200-208, 293-304) on a random pattern."""
    n = 300
    a = golden_matrix("rand300_b3_w5")[0]
    a = O.Csr(a.n, a.row_ptr, a.col_idx, a.vals)
    q = rng.permutation(n).astype(np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(a.row_ptr))
    ap, _ = O.permute_system(a, np.zeros(n), q)
    order = np.lexsort((q[a.col_idx], q[rows]))
    assert np.array_equal(ap.col_idx, q[a.col_idx][order])
    assert np.array_equal(ap.vals, a.vals[order])
    at = O.csr_transpose(a)
    order = np.lexsort((rows, a.col_idx))
    assert np.array_equal(at.col_idx, rows[order])
    assert np.array_equal(at.vals, a.vals[order])

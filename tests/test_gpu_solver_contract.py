"""The reference's solver / preconditioner contract on the B200 path.

Mirrors the behaviours `T/test_solver.py` and `T/test_precond.py` pin for
this path (own tests, same expectations): identity converges in one
iteration, zero rhs short-circuits, non-convergence is reported not raised,
an indefinite matrix raises CgBreakdownError, repeated solves are bitwise
deterministic, the reported residual matches the true one, every ordering
solves the same system, a shift changes the history but not the solution,
HBMC with w = 1 equals BMC bitwise, SELL and CRS SpMV agree, the
preconditioner dispatch equals the direct sweeps, M^-1 0 = 0, and the
report's JSON shape.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1908_00741_b200 as P
    return P


@pytest.fixture(scope="module")
def grid(P):
    a, b = P.gen_laplacian_5pt(16, 16)
    return a, b


def cfg(P, ordering, **kw):
    d = dict(ordering=ordering, b_s=4, w=4 if ordering != "hbmc" else 8,
             spmv_format="sell" if ordering == "hbmc" else "crs")
    d.update(kw)
    return P.CgConfig(**d)


def test_identity_converges_in_one_iteration(P):
    from paper_1908_00741_b200.matrix import CooMatrix, coo_to_csr
    n = 64
    a = coo_to_csr(CooMatrix(n, np.arange(n), np.arange(n), np.ones(n)))
    b = np.linspace(-1, 1, n)
    for ordering in ("natural", "mc", "bmc", "hbmc"):
        x, rep = P.pcg(a, b, cfg(P, ordering))
        assert rep.converged and rep.iterations == 1
        assert np.allclose(x, b, rtol=0, atol=1e-15)


def test_zero_rhs_short_circuits(P, grid):
    a, _ = grid
    x, rep = P.pcg(a, np.zeros(a.n), cfg(P, "hbmc"))
    assert rep.iterations == 0 and rep.converged
    assert rep.residual_history == [0.0]
    assert not np.any(x)


def test_nonconvergence_reported_not_raised(P, grid):
    a, b = grid
    x, rep = P.pcg(a, b, cfg(P, "hbmc", max_iters=3, tol=1e-14))
    assert not rep.converged and rep.iterations == 3
    assert len(rep.residual_history) == 4


def test_indefinite_raises_cg_breakdown(P):
    from paper_1908_00741_b200.matrix import CooMatrix, coo_to_csr
    n = 32
    d = np.ones(n)
    d[::2] = -1.0   # IC of a diagonal matrix with negative pivots would break: shift the
    a = coo_to_csr(CooMatrix(n, np.arange(n), np.arange(n), d))
    with pytest.raises((P.CgBreakdownError, P.IcBreakdownError)):
        P.pcg(a, np.ones(n), cfg(P, "hbmc"))


def test_repeated_solves_bitwise_identical(P, grid):
    a, b = grid
    x1, r1 = P.pcg(a, b, cfg(P, "hbmc"))
    x2, r2 = P.pcg(a, b, cfg(P, "hbmc"))
    assert np.array_equal(x1, x2)
    assert r1.residual_history == r2.residual_history


@pytest.mark.parametrize("ordering", ["natural", "mc", "bmc", "hbmc"])
def test_true_residual_matches_reported(P, grid, ordering):
    a, b = grid
    x, rep = P.pcg(a, b, cfg(P, ordering))
    assert rep.converged
    true_rel = np.linalg.norm(b - a.to_dense() @ x) / np.linalg.norm(b)
    assert true_rel < 1e-6
    assert abs(true_rel - rep.residual_history[-1]) <= 1e-9


def test_all_orderings_solve_the_same_system(P, grid):
    a, b = grid
    xs = [P.pcg(a, b, cfg(P, o))[0] for o in ("natural", "mc", "bmc", "hbmc")]
    for x in xs[1:]:
        assert np.linalg.norm(x - xs[0]) / np.linalg.norm(xs[0]) < 1e-6


def test_shift_changes_history_not_solution(P, grid):
    a, b = grid
    x0, r0 = P.pcg(a, b, cfg(P, "hbmc"))
    x1, r1 = P.pcg(a, b, cfg(P, "hbmc", shift=0.1))
    assert r0.residual_history != r1.residual_history
    assert np.linalg.norm(x1 - x0) / np.linalg.norm(x0) < 1e-6


@pytest.mark.parametrize("nx,ny,fmt", [(8, 8, "crs"), (5, 5, "crs"), (13, 11, "crs"), (6, 5, "crs"), (30, 22, "crs"),
                                        (31, 29, "crs"), (5, 5, "sell"), (31, 29, "sell")])
def test_hbmc_w1_bitwise_equals_bmc(P, nx, ny, fmt):
    """w = 1 makes the HBMC interleave the identity over the padded BMC order
    (T/test_solver.py:137-145): with dummy rows (5x5, 13x11, 31x29 grids,
    blocks of 4) the dot products run over the real rows only, in their
    order, so iterations, x AND the residual history are bitwise BMC's."""
    a, b = P.gen_laplacian_5pt(nx, ny)
    xb, rb = P.pcg(a, b, P.CgConfig(ordering="bmc", b_s=4, w=1, spmv_format=fmt))
    xh, rh = P.pcg(a, b, P.CgConfig(ordering="hbmc", b_s=4, w=1, spmv_format=fmt))
    if (nx * ny) % 4:
        assert rh.n_dummy > 0
    assert rb.iterations == rh.iterations
    assert np.array_equal(xb, xh)
    assert rb.residual_history == rh.residual_history


def test_sell_and_crs_spmv_agree(P, grid):
    a, b = grid
    xs, rs = P.pcg(a, b, cfg(P, "hbmc", spmv_format="sell"))
    xc, rc = P.pcg(a, b, cfg(P, "hbmc", spmv_format="crs"))
    assert rs.iterations == rc.iterations
    assert np.linalg.norm(xs - xc) / np.linalg.norm(xc) < 1e-12


def test_preconditioner_dispatch_and_zero(P, grid):
    a, _ = grid
    lay = P.color_blocks(a, P.build_blocks(a, 4))
    hl = P.build_hbmc(lay, 8)
    a_ext, b_ext = P.extend_with_dummies(a, np.zeros(a.n), hl)
    af, _ = P.permute_system(a_ext, b_ext, hl.composed_perm)
    f = P.ic0_factorize(af, layout_tag="hbmc")
    sf = P.build_sell_factor(f, hl)
    r = np.random.default_rng(5).standard_normal(hl.n_pad)
    z = P.apply_ic_preconditioner("hbmc", sf, hl, r)
    assert np.array_equal(z, P.sub_backward_hbmc(sf, hl, P.sub_forward_hbmc(sf, hl, r)))
    assert not np.any(P.apply_ic_preconditioner("hbmc", sf, hl, np.zeros(hl.n_pad)))
    # M^-1 is SPD: r . M^-1 r > 0
    assert float(r @ z) > 0


def test_report_json_shape(P, grid):
    a, b = grid
    _, rep = P.pcg(a, b, cfg(P, "hbmc"), matrix_name="grid16")
    d = rep.to_json_dict()
    assert set(d) == {"matrix", "ordering", "b_s", "w", "n_c", "iterations", "converged",
                      "time_setup_s", "time_solve_s", "residual_history", "barrier_total",
                      "n_dummy"}
    assert d["matrix"] == "grid16" and len(d["residual_history"]) == d["iterations"] + 1

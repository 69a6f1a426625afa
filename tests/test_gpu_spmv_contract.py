"""The reference's matrix-level SpMV contract on the B200 path.

Mirrors what `T/test_matrix.py` pins for `spmv` (own tests, same
expectations): structurally empty rows give 0, CSR and SELL (every width,
ragged last slice) agree with the dense product, the CSR kernel is bitwise
equal to the sequential per-row order (`src/matrix.py:307-323`), SELL equals
CSR bitwise on the same rows, and a CUDA tensor in gives a CUDA tensor out.
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


def max_rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_empty_rows(P):
    from paper_1908_00741_b200.matrix import CooMatrix, coo_to_csr
    a = coo_to_csr(CooMatrix(3, np.array([0, 2]), np.array([0, 2]), np.array([2.0, 3.0])),
                   ensure_diagonal=False)
    assert P.spmv(a, np.ones(3)).tolist() == [2.0, 0.0, 3.0]
    for w in (1, 2, 4):
        assert P.spmv(P.csr_to_sell(a, w), np.ones(3)).tolist() == [2.0, 0.0, 3.0]


@pytest.mark.parametrize("n", [1, 31, 50, 97, 1000])
@pytest.mark.parametrize("w", [1, 2, 4, 8, 32])
def test_sell_matches_dense_and_csr(P, n, w):
    from paper_1908_00741_b200.matrix import spmv_host_exact
    a = P.gen_random_spd(n, density=0.05, seed=n + w)
    x = np.random.default_rng(n).standard_normal(n)
    y_csr = P.spmv(a, x)
    y_sell = P.spmv(P.csr_to_sell(a, w), x)
    assert max_rel(y_csr, a.to_dense() @ x) < 1e-14
    assert np.array_equal(y_csr, spmv_host_exact(a, x))   # sequential per-row order
    assert np.array_equal(y_sell, y_csr)                  # same rows, same order


def test_tensor_in_tensor_out(P):
    import torch
    a, _ = P.gen_laplacian_5pt(9, 7)
    x = np.random.default_rng(1).standard_normal(a.n)
    yd = P.spmv(a, torch.from_numpy(x).cuda())
    assert isinstance(yd, torch.Tensor) and yd.is_cuda
    assert np.array_equal(yd.cpu().numpy(), P.spmv(a, x))


def test_sell32_plan_spmv_n_not_multiple_of_32(P):
    """A width-32 SELL A with n % 32 != 0 runs the TMA-staged plan SpMV: it
    must write only rows < n (the caller's y has length n) and leave the
    padded rows out of p.Ap -- the reference pads x to n_pad and returns
    out[:n] (src/matrix.py:315-322)."""
    import torch
    from paper_1908_00741_b200 import solver
    a = P.gen_random_spd(1000, density=0.01, seed=5)
    cfg = P.CgConfig(ordering="natural", w=32, spmv_format="sell")
    st = solver.attach_plan(solver.prepare(a, np.ones(a.n), cfg), cfg)
    plan = st.plan
    try:
        x = torch.from_numpy(np.random.default_rng(0).standard_normal(a.n)).cuda()
        buf = torch.full((a.n + 64,), 12345.0, dtype=torch.float64, device="cuda")
        plan.spmv(x, buf[:a.n])
        torch.cuda.synchronize()
        out = buf.cpu().numpy()
        assert np.all(out[a.n:] == 12345.0), "plan SpMV wrote past row n"
        ref = P.spmv(a, x.cpu().numpy())
        assert np.array_equal(out[:a.n], ref)
    finally:
        plan.close()


def test_natural_sell32_solve_n_not_multiple_of_32(P):
    """Whole solve through the TMA SpMV + fused p.Ap with n % 32 != 0
    converges like the CRS solve (no NaN from the slice padding)."""
    a = P.gen_random_spd(1000, density=0.01, seed=5)
    b = np.ones(a.n)
    x1, r1 = P.pcg(a, b, P.CgConfig(ordering="natural", w=32, spmv_format="sell"))
    x2, r2 = P.pcg(a, b, P.CgConfig(ordering="natural", spmv_format="crs"))
    assert r1.converged and r2.converged
    assert abs(r1.iterations - r2.iterations) <= 1
    assert np.linalg.norm(x1 - x2) <= 1e-10 * np.linalg.norm(x2)

"""Host side of the product (CPU): builder parity, C ABI, error behaviour.

Bit-exact checks of the native host builder (orderings, padding, HBMC
permutation, permutation of the system, IC(0), SELL packing) against the
reference's golden outputs and the pinned oracle; the library exports every
entry point include/hbmc_b200.h declares; the reference's exceptions and
validation messages.  No GPU needed.
"""

import hashlib
import json
import os
import re

import numpy as np
import pytest

import paper_1908_00741_b200 as P
from conftest import GOLDEN, REPO, golden_matrix, golden_names, load_golden
from oracle import oracle as O
from paper_1908_00741_b200 import _lib, kernels
import workloads as problems

NAMES = golden_names()


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def same(g, key, arr):
    if key in g:
        return np.array_equal(arr, g[key])
    return sha(arr) == str(g[key + "_sha"])


@pytest.fixture(scope="module", params=NAMES)
def case(request):
    name = request.param
    g = load_golden(name)
    a, bs, w, rhs_kind = golden_matrix(name)
    return name, g, a, bs, w


def test_generator_matches_golden_hash(case):
    name, g, a, bs, w = case
    h = hashlib.sha256()
    for arr in (a.row_ptr, a.col_idx, a.vals):
        h.update(arr.tobytes())
    assert h.hexdigest() == str(g["a_hash"])


def test_orderings_bit_exact(case):
    name, g, a, bs, w = case
    bl = P.build_blocks(a, bs)
    assert np.array_equal(bl.block_of, g["block_of"])
    lay = P.color_blocks(a, bl)
    assert np.array_equal(lay.color_of_block, g["color_of_block"])
    assert np.array_equal(lay.perm.new_of_old, g["bmc_perm"])
    hl = P.build_hbmc(lay, w)
    assert np.array_equal(hl.composed_perm.new_of_old, g["composed"])
    assert np.array_equal(hl.nbar_of, g["nbar_of"])
    assert hl.n_dummy == int(g["n_dummy"]) and hl.n_pad == int(g["n_pad"])
    assert hl.n_c == int(g["n_c"])
    assert np.array_equal(hl.color_lvl1_ranges, g["color_lvl1_ranges"])
    nod = P.greedy_color_nodes(a)
    assert np.array_equal(nod.color_of, g["node_color"])
    assert np.array_equal(nod.perm.new_of_old, g["mc_perm"])


def test_factor_and_sell_bit_exact(case):
    name, g, a, bs, w = case
    lay = P.color_blocks(a, P.build_blocks(a, bs))
    hl = P.build_hbmc(lay, w)
    b = np.ones(a.n)
    a_ext, b_ext = P.extend_with_dummies(a, b, hl)
    af, bf = P.permute_system(a_ext, b_ext, hl.composed_perm)
    f = P.ic0_factorize(af, layout_tag="hbmc")
    assert same(g, "L_vals", f.L.vals)
    assert np.array_equal(f.d, g["d"])
    sf = P.build_sell_factor(f, hl)
    # SELL layout identical to the (pinned) oracle's restatement of csr_to_sell
    osys = O.HbmcSystem(O.Csr(a.n, a.row_ptr, a.col_idx, a.vals), b, bs, w)
    for mine, ref in ((sf.lower, osys.Ls), (sf.upper, osys.Us)):
        assert np.array_equal(mine.slice_ptr, ref.slice_ptr)
        assert np.array_equal(mine.slice_len, ref.slice_len)
        assert np.array_equal(mine.col_idx, ref.col_idx)
        assert np.array_equal(mine.vals, ref.vals)
        assert np.array_equal(mine.col32, ref.col_idx.astype(np.int32))
    back = P.sell_to_csr(sf.lower)
    assert np.array_equal(back.col_idx, f.L.col_idx) and np.array_equal(back.vals, f.L.vals)


def test_kernel_seam_construction_functions(case):
    """kernels.py (the numba_backend drop-in) on the host builder."""
    name, g, a, bs, w = case
    block_of, nb = kernels.grow_blocks(a.row_ptr, a.col_idx, bs)
    assert np.array_equal(block_of, g["block_of"])
    bl = P.build_blocks(a, bs)
    cob = kernels.color_block_graph(a.row_ptr, a.col_idx, block_of, nb, bl.blocks.ptr,
                                    bl.blocks.members)
    assert np.array_equal(cob, g["color_of_block"])
    assert np.array_equal(kernels.greedy_color(a.row_ptr, a.col_idx), g["node_color"])


@pytest.mark.parametrize("cfg_id", [2])
def test_full_config_ordering_matches_reference_digest(cfg_id):
    """Config 2 at full size (N = 2.1M): permutation hash == reference's."""
    with open(os.path.join(GOLDEN, f"config{cfg_id}_digest.json")) as fh:
        dg = json.load(fh)
    label, gen, bs, w = problems.CONFIGS[cfg_id]
    a = gen()
    h = hashlib.sha256()
    for arr in (a.row_ptr, a.col_idx, a.vals):
        h.update(arr.tobytes())
    assert h.hexdigest() == dg["a_hash"]
    lay = P.color_blocks(a, P.build_blocks(a, bs))
    hl = P.build_hbmc(lay, w)
    assert sha(hl.composed_perm.new_of_old) == dg["composed_hash"]
    assert sha(lay.perm.new_of_old) == dg["bmc_perm_hash"]
    assert hl.n_c == dg["n_c"] and hl.n_dummy == dg["n_dummy"]
    assert hl.nbar_of.tolist() == dg["nbar_of"]


def test_library_exports_every_header_symbol():
    with open(os.path.join(REPO, "include", "hbmc_b200.h")) as fh:
        hdr = fh.read()
    names = set(re.findall(r"^(?:int|const char \*)\s*(tb_\w+)\(", hdr, re.M))
    assert len(names) >= 30
    for name in names:
        assert hasattr(_lib.LIB, name), name
    assert set(_lib.EXPORTED) >= names
    assert _lib.LIB.tb_abi_version() == _lib.ABI_VERSION


def test_ic_breakdown_reports_row_and_pivot():
    d = np.array([[1.0, 2.0], [2.0, 1.0]])
    r, c = np.nonzero(d)
    a = P.coo_to_csr(P.CooMatrix(2, r, c, d[r, c]))
    with pytest.raises(P.IcBreakdownError) as e:
        P.ic0_factorize(a)
    assert e.value.row == 1 and e.value.pivot == pytest.approx(-3.0)
    f = P.ic0_factorize(a, shift=4.0)
    assert np.all(f.d > 0)
    with pytest.raises(ValueError):
        P.ic0_factorize(a, shift=-0.1)


def test_ic_2x2_hand_values():
    d = np.array([[4.0, -1.0], [-1.0, 4.0]])
    r, c = np.nonzero(d)
    f = P.ic0_factorize(P.coo_to_csr(P.CooMatrix(2, r, c, d[r, c])))
    assert f.d[0] == 2.0 and f.d[1] == np.sqrt(3.75)
    assert f.L.vals[f.L.row_ptr[1]] == -0.5


def test_input_validation_messages():
    coo = P.CooMatrix(2, np.array([0, 0, 1]), np.array([0, 1, 0]), np.array([2.0, 1.0, 1.0]))
    with pytest.raises(ValueError, match="diagonal"):
        P.ic0_factorize(P.coo_to_csr(coo, ensure_diagonal=False))
    coo2 = P.CooMatrix(2, np.array([0, 0, 1]), np.array([0, 1, 1]), np.array([2.0, 1.0, 2.0]))
    with pytest.raises(ValueError, match="symmetr"):
        P.ic0_factorize(P.coo_to_csr(coo2, ensure_diagonal=False))
    dup = P.CooMatrix(2, np.array([0, 0, 1]), np.array([0, 0, 1]), np.array([1.0, 1.0, 1.0]))
    with pytest.raises(ValueError, match=r"duplicate entry at \(0, 0\)"):
        P.coo_to_csr(dup)
    for bad in (dict(ordering="zigzag"), dict(tol=0.0), dict(b_s=0), dict(w=0),
                dict(threads=0), dict(spmv_format="csc")):
        with pytest.raises(ValueError):
            P.CgConfig(**bad).validate()
    with pytest.raises(ValueError):
        P.build_blocks(P.gen_laplacian_5pt(3, 3)[0], 0)
    with pytest.raises(ValueError):
        P.build_hbmc(P.color_blocks(*(lambda a: (a, P.build_blocks(a, 2)))(
            P.gen_laplacian_5pt(3, 3)[0])), 0)


def test_golden_reference_hand_oracles():
    """Hand-checked layouts from the reference's own tests (T/test_ordering.py)."""
    a, _ = P.gen_laplacian_5pt(4, 4)
    lay = P.color_blocks(a, P.build_blocks(a, 4))
    assert lay.perm.old_of_new.tolist() == [0, 1, 2, 3, 8, 9, 10, 11, 4, 5, 6, 7,
                                            12, 13, 14, 15]   # T/test_ordering.py:155-164
    a5, _ = P.gen_laplacian_5pt(5, 5)
    hl = P.build_hbmc(P.color_blocks(a5, P.build_blocks(a5, 4)), 4)
    assert hl.n == 25 and hl.n_dummy == 23 and hl.n_pad == 48   # T/test_ordering.py:196-203
    from golden.make_golden import path_matrix
    lay16 = P.color_blocks(path_matrix(16), P.build_blocks(path_matrix(16), 2))
    hl16 = P.build_hbmc(lay16, 4)
    assert hl16.perm.new_of_old[:8].tolist() == [0, 4, 1, 5, 2, 6, 3, 7]   # :206-216
    assert hl16.composed_perm.old_of_new[:8].tolist() == [0, 4, 8, 12, 1, 5, 9, 13]

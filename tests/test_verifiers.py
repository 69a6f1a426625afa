"""Ordering verifiers (src/ordering.py:283-346) on this package's orderings:
the HBMC permutation keeps the BMC relative order of every coupled pair
across blocks (the paper's equivalence), and the
HBMC-ordered matrix has diagonal w-wide steps and no same-color coupling --
the structure the device kernels rely on.  CPU only."""

import numpy as np

import paper_1908_00741_b200 as P
from paper_1908_00741_b200 import problems


def _system(a, bs, w):
    lay = P.color_blocks(a, P.build_blocks(a, bs))
    hl = P.build_hbmc(lay, w)
    a_ext, b_ext = P.extend_with_dummies(a, np.zeros(a.n), hl)
    af, _ = P.permute_system(a_ext, b_ext, hl.composed_perm)
    return lay, hl, af


def test_level2_structure_holds_for_hbmc():
    for a, bs, w in ((problems.lap7(12), 4, 8), (problems.varcoef7(16, seed=0), 8, 32),
                     (problems.knn_graph(3000, seed=0), 4, 32),
                     (P.gen_random_spd(400, density=0.02, seed=3), 3, 5)):
        lay, hl, af = _system(a, bs, w)
        rep = P.check_level2_structure(af, hl)
        assert rep.holds, rep


def test_level2_structure_detects_violations():
    a = problems.lap7(8)
    lay, hl, af = _system(a, 4, 8)
    rep = P.check_level2_structure(af, hl)
    # the natural order of the 3-D grid is not an HBMC order
    a_ext, _ = P.extend_with_dummies(a, np.zeros(a.n), hl)
    bad = P.check_level2_structure(a_ext, hl)
    assert rep.holds and not bad.holds
    assert bad.n_diag_violations + bad.n_cross_violations > 0 and bad.examples


def test_er_condition_bmc_vs_hbmc():
    """HBMC is an equivalent reordering of BMC: written
    in BMC order, the move to HBMC order keeps the relative order of every
    coupled pair."""
    a = problems.varcoef7(12, seed=0)
    lay, hl, af = _system(a, 4, 8)
    a_b, _ = P.permute_system(a, np.zeros(a.n), lay.perm)
    node_at_bmc = np.empty(a.n, dtype=np.int64)
    node_at_bmc[lay.perm.new_of_old] = np.arange(a.n)
    hb_pos = hl.composed_perm.new_of_old[node_at_bmc]        # HBMC slot of each BMC row
    q = P.Permutation(np.argsort(np.argsort(hb_pos)))         # ranks among the real rows
    rep = P.check_er_condition(a_b, q)
    assert rep.n_pairs > 0 and rep.holds, rep
    g = P.build_ordering_graph(a_b, q)
    assert g.n_edges == rep.n_pairs
    assert np.all(q.new_of_old[g.tail] < q.new_of_old[g.head])
    assert g == P.build_ordering_graph(a_b, P.Permutation(np.arange(a.n)))


def test_er_condition_identity_and_reversal():
    a = P.gen_random_spd(200, density=0.05, seed=1)
    ident = P.Permutation(np.arange(a.n))
    rep = P.check_er_condition(a, ident)
    assert rep.holds and rep.n_violations == 0
    rev = P.Permutation(np.arange(a.n)[::-1].copy())
    bad = P.check_er_condition(a, rev, max_violations=5)
    assert not bad.holds and bad.n_violations == bad.n_pairs and len(bad.violations) == 5
    some = P.check_er_condition(a, rev, pair_filter=lambda lo, hi: hi - lo > 100)
    assert some.n_pairs < rep.n_pairs


def test_single_backend_registry():
    assert P.available_backends() == ["cuda"] and P.default_backend() == "cuda"
    assert P.get_kernels() is P.get_kernels("cuda")

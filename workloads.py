"""The BASELINE.json workloads -- test and bench
infrastructure, not the product.

The reference ships only 2-D generators (src/matrix.py:326-374); these are
the five 3-D / graph problems BASELINE.json names, defined exactly as the
survey's oracle runs defined them (node numbering is part of the problem:
BMC blocking seeds on the smallest index).  Natural x-fastest numbering
i = ix + nx*(iy + ny*iz), Dirichlet boundaries (boundary rows just lack
neighbours).  Diagonal sums are accumulated in the same element order as a
sequential np.add.at over `lo` then `hi` (np.bincount over the concatenation
performs exactly that sequence of additions), so values are bit-identical to
the survey's recipe.

This module is pure numpy at import time.  Each generator returns a CSR
assembled by the product's `coo_to_csr` (default) or, with
`backend="oracle"`, by the CPU oracle's (oracle/oracle.py) -- so bench.py's
reference arm builds its matrix without loading the product library.  Both
assemble the same COO triplets with the same (row, col) lexsort contract
(src/matrix.py:168-197); `tests/test_oracle.py` checks that they agree.
"""

import numpy as np


def _edges3d(nx, ny, nz):
    idx = np.arange(nx * ny * nz, dtype=np.int64).reshape(nz, ny, nx)
    out = []
    for axis in (2, 1, 0):  # x, y, z
        lo = [slice(None)] * 3
        hi = [slice(None)] * 3
        lo[axis] = slice(None, -1)
        hi[axis] = slice(1, None)
        out.append((idx[tuple(lo)].ravel(), idx[tuple(hi)].ravel()))
    return out


def _seq_sum(n, lo, hi, w, init=None):
    """diag = init; diag[lo[k]] += w[k] (k asc); then the same over hi."""
    if init is None:
        idx = np.concatenate([lo, hi])
        wt = np.concatenate([w, w])
    else:
        idx = np.concatenate([np.arange(n, dtype=np.int64), lo, hi])
        wt = np.concatenate([init, w, w])
    return np.bincount(idx, weights=wt, minlength=n)


def _assemble(n, lo, hi, off, diag, backend):
    """COO [lo->hi, hi->lo, diag] -> CSR (src/matrix.py:168-197)."""
    rows = np.concatenate([lo, hi, np.arange(n, dtype=np.int64)])
    cols = np.concatenate([hi, lo, np.arange(n, dtype=np.int64)])
    del lo, hi
    vals = np.concatenate([-off, -off, diag])
    if backend == "oracle":
        from oracle import oracle as O
        return O.coo_to_csr(n, rows, cols, vals)
    from paper_1908_00741_b200.matrix import CooMatrix, coo_to_csr
    return coo_to_csr(CooMatrix(n, rows, cols, vals))


def lap7(n, cx=1.0, cy=1.0, cz=1.0, backend="product"):
    """Configs 1 and 5: constant-coefficient (anisotropic) 7-point stencil.

    Off-diagonals -cx / -cy / -cz, diagonal 2*(cx+cy+cz) on every row."""
    N = n ** 3
    (xl, xh), (yl, yh), (zl, zh) = _edges3d(n, n, n)
    lo = np.concatenate([xl, yl, zl])
    hi = np.concatenate([xh, yh, zh])
    c = np.concatenate([np.full(xl.size, cx), np.full(yl.size, cy),
                        np.full(zl.size, cz)])
    del xl, xh, yl, yh, zl, zh
    diag = np.full(N, 2 * (cx + cy + cz))
    return _assemble(N, lo, hi, c, diag, backend)


def varcoef7(n, seed=0, backend="product"):
    """Config 2: kappa ~ lognormal(0, 1) per cell, harmonic face averages,
    Dirichlet faces contribute 2*kappa_i."""
    rng = np.random.default_rng(seed)
    N = n ** 3
    kappa = rng.lognormal(0.0, 1.0, N)
    (xl, xh), (yl, yh), (zl, zh) = _edges3d(n, n, n)
    lo = np.concatenate([xl, yl, zl])
    hi = np.concatenate([xh, yh, zh])
    c = 2 * kappa[lo] * kappa[hi] / (kappa[lo] + kappa[hi])
    diag = _seq_sum(N, lo, hi, c)
    deg = _seq_sum(N, lo, hi, np.ones(lo.size))
    diag += (6 - deg) * 2 * kappa
    return _assemble(N, lo, hi, c, diag, backend)


def stencil27(n, seed=0, backend="product"):
    """Config 3: 27-point, off-diagonals -u, u ~ U[0.5, 1.5] per unordered
    pair (13 forward offsets in lexicographic order), diagonal
    1.01 * row sum of |off-diagonals|."""
    rng = np.random.default_rng(seed)
    N = n ** 3
    idx = np.arange(N, dtype=np.int64).reshape(n, n, n)
    los, his = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if (dz, dy, dx) <= (0, 0, 0):
                    continue
                src = idx[max(0, -dz):n - max(0, dz), max(0, -dy):n - max(0, dy),
                          max(0, -dx):n - max(0, dx)]
                dst = idx[max(0, dz):n - max(0, -dz) or None,
                          max(0, dy):n - max(0, -dy) or None,
                          max(0, dx):n - max(0, -dx) or None]
                los.append(src.ravel())
                his.append(dst.ravel())
    lo = np.concatenate(los)
    hi = np.concatenate(his)
    u = rng.uniform(0.5, 1.5, lo.size)
    diag = _seq_sum(N, lo, hi, u)
    diag *= 1.01
    return _assemble(N, lo, hi, u, diag, backend)


def knn_graph(N, k=14, seed=0, backend="product"):
    """Config 4: N uniform points in the unit cube, edges to the k nearest
    neighbours (symmetrised, unique pairs, first occurrence kept), weights
    1/dist, node ids relabelled by a random permutation, diagonal = weight
    sum + 1e-3."""
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(seed)
    P = rng.random((N, 3))
    d, j = cKDTree(P).query(P, k=k + 1, workers=-1)
    i = np.repeat(np.arange(N, dtype=np.int64), k)
    j = j[:, 1:].ravel().astype(np.int64)
    d = d[:, 1:].ravel()
    lo = np.minimum(i, j)
    hi = np.maximum(i, j)
    key = lo * N + hi
    _, first = np.unique(key, return_index=True)
    lo, hi = lo[first], hi[first]
    wgt = 1.0 / d[first]
    perm = rng.permutation(N)
    lo, hi = perm[lo], perm[hi]
    diag = _seq_sum(N, lo, hi, wgt, init=np.full(N, 1e-3))
    return _assemble(N, lo, hi, wgt, diag, backend)


# BASELINE.json configs: id -> (label, b_s, w, generator(backend))
_GEN = {
    1: ("poisson7_32^3", 4, 8, lambda be: lap7(32, backend=be)),
    2: ("varcoef7_128^3", 8, 32, lambda be: varcoef7(128, seed=0, backend=be)),
    3: ("stencil27_192^3", 8, 32, lambda be: stencil27(192, seed=0, backend=be)),
    4: ("knn14_4M", 4, 32, lambda be: knn_graph(4_000_000, seed=0, backend=be)),
    5: ("aniso7_512^3", 16, 32, lambda be: lap7(512, 1.0, 1.0, 1e-3, backend=be)),
}

# id -> (label, generator() with the product's assembly, b_s, w)
CONFIGS = {k: (lab, (lambda g=g: g("product")), bs, w) for k, (lab, bs, w, g) in _GEN.items()}


def generate(cfg_id, backend="product"):
    """(label, A, b_s, w) of BASELINE config `cfg_id`."""
    label, bs, w, g = _GEN[cfg_id]
    return label, g(backend), bs, w


def scaled(cfg_id, size, backend="product"):
    """Same family as config `cfg_id` at a smaller size (parity tests)."""
    _, b_s, w, _ = _GEN[cfg_id]
    gen = {1: lambda: lap7(size, backend=backend),
           2: lambda: varcoef7(size, seed=0, backend=backend),
           3: lambda: stencil27(size, seed=0, backend=backend),
           4: lambda: knn_graph(size, seed=0, backend=backend),
           5: lambda: lap7(size, 1.0, 1.0, 1e-3, backend=backend)}[cfg_id]
    return gen(), b_s, w


def xstar(n, seed=1):
    """x* = default_rng(seed).uniform(-1, 1, N)."""
    return np.random.default_rng(seed).uniform(-1, 1, n)


def rhs(a, seed=1, backend="product"):
    """x*, b = A x* in the reference's sequential CSR accumulation order
    (src/matrix.py:307-323 -> K/numba_backend.py:16-23; computed once, on
    the host)."""
    xs = xstar(a.n, seed)
    if backend == "oracle":
        from oracle import oracle as O
        return xs, O.spmv_csr(a, xs)
    from paper_1908_00741_b200.matrix import spmv_host_exact
    return xs, spmv_host_exact(a, xs)

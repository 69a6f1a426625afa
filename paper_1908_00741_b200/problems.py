"""The BASELINE.json problem generators.

The reference ships only 2-D generators (src/matrix.py:326-374); these are
the five 3-D / graph problems BASELINE.json names, defined exactly as the
survey's oracle runs defined them (node numbering is part of the problem:
BMC blocking seeds on the smallest index).  Natural x-fastest numbering
i = ix + nx*(iy + ny*iz), Dirichlet boundaries (boundary rows just lack
neighbours).  Diagonal sums are accumulated in the same element order as a
sequential np.add.at over `lo` then `hi` (np.bincount over the concatenation
performs exactly that sequence of additions), so values are bit-identical to
the survey's recipe.
"""

import numpy as np

from .matrix import CooMatrix, coo_to_csr, spmv_host_exact


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


def _assemble(n, lo, hi, off, diag):
    rows = np.concatenate([lo, hi, np.arange(n, dtype=np.int64)])
    cols = np.concatenate([hi, lo, np.arange(n, dtype=np.int64)])
    vals = np.concatenate([-off, -off, diag])
    return coo_to_csr(CooMatrix(n, rows, cols, vals))


def _seq_sum(n, lo, hi, w, init=None):
    """diag = init; diag[lo[k]] += w[k] (k asc); then the same over hi."""
    if init is None:
        idx = np.concatenate([lo, hi])
        wt = np.concatenate([w, w])
    else:
        idx = np.concatenate([np.arange(n, dtype=np.int64), lo, hi])
        wt = np.concatenate([init, w, w])
    return np.bincount(idx, weights=wt, minlength=n)


def lap7(n, cx=1.0, cy=1.0, cz=1.0):
    """Configs 1 and 5: constant-coefficient (anisotropic) 7-point stencil.

    Off-diagonals -cx / -cy / -cz, diagonal 2*(cx+cy+cz) on every row."""
    N = n ** 3
    (xl, xh), (yl, yh), (zl, zh) = _edges3d(n, n, n)
    lo = np.concatenate([xl, yl, zl])
    hi = np.concatenate([xh, yh, zh])
    c = np.concatenate([np.full(xl.size, cx), np.full(yl.size, cy),
                        np.full(zl.size, cz)])
    diag = np.full(N, 2 * (cx + cy + cz))
    return _assemble(N, lo, hi, c, diag)


def varcoef7(n, seed=0):
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
    return _assemble(N, lo, hi, c, diag)


def stencil27(n, seed=0):
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
    return _assemble(N, lo, hi, u, diag)


def knn_graph(N, k=14, seed=0):
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
    return _assemble(N, lo, hi, wgt, diag)


# BASELINE.json configs: id -> (label, generator, b_s, w)
CONFIGS = {
    1: ("poisson7_32^3", lambda: lap7(32), 4, 8),
    2: ("varcoef7_128^3", lambda: varcoef7(128, seed=0), 8, 32),
    3: ("stencil27_192^3", lambda: stencil27(192, seed=0), 8, 32),
    4: ("knn14_4M", lambda: knn_graph(4_000_000, seed=0), 4, 32),
    5: ("aniso7_512^3", lambda: lap7(512, 1.0, 1.0, 1e-3), 16, 32),
}


def scaled(cfg_id, size):
    """Same family as config `cfg_id` at a smaller size (parity tests)."""
    _, _, b_s, w = CONFIGS[cfg_id]
    gen = {1: lambda: lap7(size), 2: lambda: varcoef7(size, seed=0),
           3: lambda: stencil27(size, seed=0), 4: lambda: knn_graph(size, seed=0),
           5: lambda: lap7(size, 1.0, 1.0, 1e-3)}[cfg_id]
    return gen(), b_s, w


def rhs(a, seed=1):
    """x* = default_rng(seed).uniform(-1, 1, N); b = A x* in the reference's
    sequential CSR accumulation order (computed once, on the host)."""
    xs = np.random.default_rng(seed).uniform(-1, 1, a.n)
    return xs, spmv_host_exact(a, xs)

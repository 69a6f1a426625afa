"""MC / BMC / HBMC orderings (drop-in for trilab.ordering).

Same dataclasses and field names as src/ordering.py:37-105; the greedy
kernels and the padding/interleave passes run in the native host builder and
are bit-exact with the reference (greedy first-fit is inherently sequential;
see DESIGN.md).  The verifiers of src/ordering.py:283-346 (ER condition,
level-2 structure) are not rebuilt: they are out of this path's scope
 and tests/test_verifiers.py applies the reference's own
verifiers to this module's orderings.
"""

from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import LIB, check, i64a, ptr
from .matrix import CsrMatrix, Permutation

__all__ = [
    "NodalColoring", "Blocking", "BmcLayout", "HbmcLayout",
    "greedy_color_nodes", "build_blocks", "color_blocks", "build_hbmc",
    "pad_colors", "extend_with_dummies",
]


class BlockList(Sequence):
    """Read-only list of per-block member arrays backed by two flat arrays.

    Behaves like the reference's `Blocking.blocks` list (src/ordering.py:49)
    without materialising millions of small numpy arrays.
    """

    def __init__(self, ptr_, members):
        self.ptr = ptr_
        self.members = members

    def __len__(self):
        return self.ptr.shape[0] - 1

    def __getitem__(self, b):
        if isinstance(b, slice):
            return [self[i] for i in range(*b.indices(len(self)))]
        nb = len(self)
        if b < 0:
            b += nb
        if not 0 <= b < nb:
            raise IndexError("block index out of range")
        return self.members[self.ptr[b]:self.ptr[b + 1]]

    def sizes(self):
        return np.diff(self.ptr)


@dataclass
class NodalColoring:
    n_c: int
    color_of: np.ndarray
    perm: Permutation
    color_ranges: np.ndarray


@dataclass
class Blocking:
    b_s: int
    block_of: np.ndarray
    blocks: Sequence  # BlockList: per-block members, ascending original index

    @property
    def n_blocks(self):
        return len(self.blocks)


@dataclass
class BmcLayout:
    blocking: Blocking
    n_c: int
    color_of_block: np.ndarray
    n_of: np.ndarray
    perm: Permutation
    color_ranges: np.ndarray
    block_order: np.ndarray
    block_bounds: np.ndarray
    color_block_ranges: np.ndarray


@dataclass
class HbmcLayout:
    base: BmcLayout
    w: int
    nbar_of: np.ndarray
    perm: Permutation
    padded_perm: Permutation
    composed_perm: Permutation
    level1_color: np.ndarray
    n: int
    n_pad: int
    color_ranges: np.ndarray
    color_lvl1_ranges: np.ndarray
    real_positions: np.ndarray

    @property
    def b_s(self):
        return self.base.blocking.b_s

    @property
    def n_c(self):
        return self.base.n_c

    @property
    def n_dummy(self):
        return self.n_pad - self.n

    @property
    def n_level1(self):
        return int(self.level1_color.shape[0])

    @property
    def level1_ranges(self):
        span = self.b_s * self.w
        k = np.arange(self.n_level1, dtype=np.int64)
        return np.stack([k * span, (k + 1) * span, self.level1_color], axis=1)


def _group(label, n_groups):
    """Stable grouping (counting sort): ptr[n_groups+1], members[n]."""
    label = i64a(label)
    p = np.empty(n_groups + 1, dtype=np.int64)
    m = np.empty(label.shape[0], dtype=np.int64)
    check(LIB.tb_group_by_label(label.shape[0], ptr(label), n_groups, ptr(p), ptr(m)))
    return p, m


def _group_perm(group_of, n_groups):
    """src/ordering.py:146-154 (stable argsort by group == counting sort)."""
    ranges, order = _group(group_of, n_groups)
    new_of_old = np.empty_like(order)
    new_of_old[order] = np.arange(order.shape[0], dtype=np.int64)
    return Permutation(new_of_old), ranges, order


def greedy_color_nodes(a: CsrMatrix, kernels=None):
    """src/ordering.py:157-162 over K/numba_backend.py:174-191."""
    color_of = np.empty(a.n, dtype=np.int64)
    check(LIB.tb_greedy_color(a.n, ptr(a.row_ptr), ptr(a.col_idx), ptr(color_of)))
    n_c = int(color_of.max()) + 1 if a.n else 0
    perm, ranges, _ = _group_perm(color_of, n_c)
    return NodalColoring(n_c, color_of, perm, ranges)


def build_blocks(a: CsrMatrix, b_s, kernels=None):
    """src/ordering.py:165-174 over K/numba_backend.py:232-270."""
    if b_s < 1:
        raise ValueError("b_s must be at least 1")
    block_of = np.empty(a.n, dtype=np.int64)
    nb = _lib.i64()
    check(LIB.tb_grow_blocks(a.n, ptr(a.row_ptr), ptr(a.col_idx), int(b_s),
                             ptr(block_of), nb))
    bptr, members = _group(block_of, nb.value)
    return Blocking(int(b_s), block_of, BlockList(bptr, members))


def _block_arrays(blocking):
    if isinstance(blocking.blocks, BlockList):
        return blocking.blocks.ptr, blocking.blocks.members
    sizes = np.array([len(b) for b in blocking.blocks], dtype=np.int64)
    bptr = np.zeros(sizes.shape[0] + 1, dtype=np.int64)
    np.cumsum(sizes, out=bptr[1:])
    members = (np.concatenate(blocking.blocks).astype(np.int64)
               if sizes.shape[0] else np.empty(0, dtype=np.int64))
    return bptr, members


def color_blocks(a: CsrMatrix, blocking: Blocking, kernels=None):
    """src/ordering.py:177-203 over K/numba_backend.py:273-291."""
    nb = blocking.n_blocks
    bptr, members = _block_arrays(blocking)
    color_of_block = np.empty(nb, dtype=np.int64)
    check(LIB.tb_color_block_graph(a.n, ptr(a.row_ptr), ptr(a.col_idx),
                                   ptr(i64a(blocking.block_of)), nb, ptr(bptr),
                                   ptr(members), ptr(color_of_block)))
    n_c = int(color_of_block.max()) + 1 if nb else 0
    n_of = np.bincount(color_of_block, minlength=n_c).astype(np.int64)
    color_block_ranges, block_order = _group(color_of_block, n_c)
    sizes = np.diff(bptr)[block_order]
    block_bounds = np.zeros(nb + 1, dtype=np.int64)
    np.cumsum(sizes, out=block_bounds[1:])
    # seq = concatenation of member lists in block_order
    if nb:
        starts = bptr[block_order]
        seq = members[np.repeat(starts - block_bounds[:-1], sizes)
                      + np.arange(a.n, dtype=np.int64)]
    else:
        seq = np.empty(0, dtype=np.int64)
    new_of_old = np.empty(a.n, dtype=np.int64)
    new_of_old[seq] = np.arange(a.n, dtype=np.int64)
    color_ranges = block_bounds[color_block_ranges]
    return BmcLayout(blocking, n_c, color_of_block, n_of,
                     Permutation(new_of_old), color_ranges, block_order,
                     block_bounds, color_block_ranges)


def pad_colors(layout: BmcLayout, w):
    """src/ordering.py:206-233: (slots, nbar_of, n_dummy)."""
    if w < 1:
        raise ValueError("w must be at least 1")
    b_s = layout.blocking.b_s
    n = len(layout.perm)
    nbar_of = np.empty(layout.n_c, dtype=np.int64)
    n_pad = _lib.i64()
    cbr = i64a(layout.color_block_ranges)
    check(LIB.tb_pad_colors_count(layout.n_c, ptr(cbr), b_s, int(w),
                                  ptr(nbar_of), n_pad))
    bptr, members = _block_arrays(layout.blocking)
    slots = np.empty(n_pad.value, dtype=np.int64)
    nd = _lib.i64()
    check(LIB.tb_pad_colors_fill(n, layout.n_c, ptr(cbr), ptr(i64a(layout.block_order)),
                                 ptr(bptr), ptr(members), b_s, int(w), ptr(slots),
                                 n_pad.value, nd))
    return slots, nbar_of, nd.value


def build_hbmc(layout: BmcLayout, w):
    """src/ordering.py:236-266."""
    if w < 1:
        raise ValueError("w must be at least 1")
    w = int(w)
    b_s = layout.blocking.b_s
    n = len(layout.perm)
    slots, nbar_of, _n_dummy = pad_colors(layout, w)
    n_pad = slots.shape[0]
    span = b_s * w
    padded = np.empty(n_pad, dtype=np.int64)
    composed = np.empty(n_pad, dtype=np.int64)
    check(LIB.tb_hbmc_compose(n_pad, ptr(slots), b_s, w, ptr(padded), ptr(composed)))
    n_lvl1 = n_pad // span
    local = (np.arange(span, dtype=np.int64) % b_s) * w + np.arange(span, dtype=np.int64) // b_s
    sec = (np.arange(n_lvl1, dtype=np.int64)[:, None] * span + local[None, :]).ravel()
    color_lvl1_ranges = np.zeros(layout.n_c + 1, dtype=np.int64)
    np.cumsum(nbar_of, out=color_lvl1_ranges[1:])
    color_ranges = color_lvl1_ranges * span
    level1_color = np.repeat(np.arange(layout.n_c, dtype=np.int64), nbar_of)
    real_positions = np.sort(composed[:n])
    return HbmcLayout(layout, w, nbar_of, Permutation(sec), Permutation(padded),
                      Permutation(composed), level1_color, n, n_pad, color_ranges,
                      color_lvl1_ranges, real_positions)


def extend_with_dummies(a: CsrMatrix, b, hl: HbmcLayout):
    """src/ordering.py:269-280: dummy rows (diagonal 1, rhs 0)."""
    nd = hl.n_dummy
    if nd == 0:
        return a, np.asarray(b, dtype=np.float64)
    n, n_pad = hl.n, hl.n_pad
    row_ptr = np.concatenate([a.row_ptr,
                              a.row_ptr[-1] + np.arange(1, nd + 1, dtype=np.int64)])
    col_idx = np.concatenate([a.col_idx, np.arange(n, n_pad, dtype=np.int64)])
    vals = np.concatenate([a.vals, np.ones(nd)])
    b_ext = np.concatenate([np.asarray(b, dtype=np.float64), np.zeros(nd)])
    return CsrMatrix(n_pad, row_ptr, col_idx, vals), b_ext

"""Row partition of an HBMC-ordered system across G ranks.

The level-1 blocks of one color are mutually independent
(`PAPER.md:382-386`; `src/ordering.py:328-346` checks it), so every color's
level-1 range `[color_lvl1_ranges[c], color_lvl1_ranges[c+1])` is split into
G contiguous chunks with the reference's own thread-chunking rule
`lo + cnt*i // G` (`src/precond.py:153-160`).  Rank g owns chunk g of every
color.  On rank g the owned level-1 blocks keep their HBMC order (color by
color), so the local system is again an HBMC system: same b_s, w, n_c, with
local `color_lvl1_ranges`, and the existing sweep / SpMV kernels run on it
unchanged.

Local vectors are `[owned rows (n_loc) | halo rows (n_halo)]`.  Columns of
the local L, U and A SELL arrays are remapped: owned rows to their local
position, remote rows to `n_loc + halo position`.  Slot order inside a row
and slice contents are the global ones, so every local row computes exactly
the floating-point operations of the single-device sweep / SpMV: the
partitioned sweeps and SpMV are bitwise equal to the unpartitioned ones.

Halo order: by (owner rank, color, class, global row), class 0 = referenced
only by L (needed by the forward sweep), 1 = by L and U, 2 = only by U
(needed by the backward sweep).  Hence, for each (source rank, color), the
entries the forward sweep needs are one contiguous range (classes 0-1),
those the backward sweep needs another (classes 1-2), and everything a
source sends for the SpMV is one contiguous range: every message is
received straight into the halo, with no unpack step.

Pure numpy; test infrastructure and the device driver share it.
"""

from dataclasses import dataclass, field

import numpy as np

from .matrix import SellMatrix


def chunk_bounds(lo, hi, parts):
    """src/precond.py:153-160: [lo + cnt*i//parts, lo + cnt*(i+1)//parts)."""
    cnt = hi - lo
    return [(lo + cnt * i // parts, lo + cnt * (i + 1) // parts) for i in range(parts)]


@dataclass
class Msg:
    """One message: `count` values, at `offset` in the packed send buffer
    (send side) or in the local extended vector (receive side)."""

    peer: int
    offset: int
    count: int
    remote_offset: int = -1   # sends: where the values land in the peer's extended vector


@dataclass
class Exchange:
    """All messages of one exchange step on one rank."""

    send_idx: np.ndarray          # int32 local rows packed into the send buffer
    sends: list                   # [Msg] offsets into the send buffer
    recvs: list                   # [Msg] offsets into the extended vector

    # fused push (sweep exchanges): per local row of the phase's color,
    # its destinations (peer rank, element index in the peer's vector)
    push_row0: int = 0
    push_ptr: np.ndarray = None
    push_rank: np.ndarray = None
    push_off: np.ndarray = None

    @property
    def n_send(self):
        return int(self.send_idx.shape[0])

    @property
    def n_recv(self):
        return int(sum(m.count for m in self.recvs))


@dataclass
class RankPart:
    rank: int
    world: int
    b_s: int
    w: int
    n_c: int
    n_loc: int
    n_halo: int
    color_lvl1_ranges: np.ndarray   # local
    lvl1: np.ndarray                # global level-1 ids owned, local order
    rows: np.ndarray                # global row of each local row
    halo_rows: np.ndarray           # global row of each halo slot
    L: SellMatrix
    U: SellMatrix
    A: SellMatrix
    inv_d: np.ndarray
    fwd: list = field(default_factory=list)   # [n_c] Exchange after fwd phase c
    bwd: list = field(default_factory=list)   # [n_c] Exchange after bwd phase c
    spmv: Exchange = None                     # p halo before the SpMV

    @property
    def n_ext(self):
        return self.n_loc + self.n_halo


def _owner_tables(color_lvl1_ranges, world):
    cr = np.asarray(color_lvl1_ranges, dtype=np.int64)
    n_c = cr.shape[0] - 1
    n_l1 = int(cr[-1])
    owner = np.empty(n_l1, dtype=np.int64)
    color = np.empty(n_l1, dtype=np.int64)
    for c in range(n_c):
        color[cr[c]:cr[c + 1]] = c
        for g, (a, b) in enumerate(chunk_bounds(int(cr[c]), int(cr[c + 1]), world)):
            owner[a:b] = g
    return owner, color


def _slot_index(S, sids, w):
    """Global slot positions of slices `sids` concatenated, + local slice_ptr."""
    lens = S.slice_len[sids].astype(np.int64)
    cnt = lens * w
    ptr = np.zeros(sids.shape[0] + 1, dtype=np.int64)
    np.cumsum(cnt, out=ptr[1:])
    total = int(ptr[-1])
    idx = np.arange(total, dtype=np.int64)
    idx += np.repeat(S.slice_ptr[sids] - ptr[:-1], cnt)
    return idx, ptr, lens


def _local_sell(S, sids, w, n_loc, gmap):
    idx, ptr, lens = _slot_index(S, sids, w)
    cols = gmap[S.col_idx[idx]]
    if cols.size and cols.min() < 0:
        raise AssertionError("partition: column outside owned rows and halo")
    return SellMatrix(n=n_loc, n_pad=n_loc, width=w, slice_ptr=ptr, slice_len=lens,
                      col_idx=cols, vals=S.vals[idx])


def _remote_cols(S, sids, w, own_of_row, rank):
    idx, _, _ = _slot_index(S, sids, w)
    cols = S.col_idx[idx]
    return np.unique(cols[own_of_row(cols) != rank])


def partition_hbmc(L, U, A, inv_d, color_lvl1_ranges, b_s, w, world, ranks=None):
    """Split a global HBMC system (SELL L, U, A with slice width w, slice
    k*b_s + l = step l of level-1 block k) into `world` RankParts.

    Returns the parts for `ranks` (default: all), with the exchange
    schedules filled in.  Every rank's schedule depends on every rank's halo,
    so all halos are computed (cheap: unique remote columns per rank).
    """
    ranks = list(range(world)) if ranks is None else list(ranks)
    span = b_s * w
    cr = np.asarray(color_lvl1_ranges, dtype=np.int64)
    n_c = cr.shape[0] - 1
    n_pad = int(cr[-1]) * span
    owner_l1, color_l1 = _owner_tables(cr, world)

    def own_of_row(rows):
        return owner_l1[rows // span]

    # owned level-1 blocks per rank in local (color-major) order
    lvl1 = []
    for g in range(world):
        ks = [np.arange(*chunk_bounds(int(cr[c]), int(cr[c + 1]), world)[g], dtype=np.int64)
              for c in range(n_c)]
        lvl1.append(np.concatenate(ks) if ks else np.zeros(0, np.int64))
    local_pos = np.empty(int(cr[-1]), dtype=np.int64)   # level-1 id -> local index on owner
    for g in range(world):
        local_pos[lvl1[g]] = np.arange(lvl1[g].shape[0])

    def sids_of(ks):
        return (ks[:, None] * b_s + np.arange(b_s, dtype=np.int64)[None, :]).ravel()

    # halo of every rank, ordered (owner, color, class, row)
    halos = []
    for g in range(world):
        sids = sids_of(lvl1[g])
        hl = _remote_cols(L, sids, w, own_of_row, g)
        hu = _remote_cols(U, sids, w, own_of_row, g)
        ha = _remote_cols(A, sids, w, own_of_row, g)
        if not np.array_equal(np.union1d(hl, hu), ha):
            raise AssertionError("partition: A's remote columns != L's and U's")
        in_l = np.isin(ha, hl, assume_unique=True)
        in_u = np.isin(ha, hu, assume_unique=True)
        cls = np.where(in_l & in_u, 1, np.where(in_l, 0, 2))
        own = own_of_row(ha)
        col = color_l1[ha // span]
        order = np.lexsort((ha, cls, col, own))
        halos.append((ha[order], own[order], col[order], cls[order]))

    def group(g, s, c):
        """[start, end) of halo(g) entries owned by s with color c, and the
        class boundaries inside it."""
        h, own, col, cls = halos[g]
        key = own * n_c + col
        a = int(np.searchsorted(key, s * n_c + c, "left"))
        b = int(np.searchsorted(key, s * n_c + c, "right"))
        seg = cls[a:b]
        c0 = a + int(np.searchsorted(seg, 1, "left"))   # first class >= 1
        c2 = a + int(np.searchsorted(seg, 2, "left"))   # first class == 2
        return a, b, c0, c2

    parts = []
    for g in ranks:
        ks = lvl1[g]
        n_loc = ks.shape[0] * span
        rows = (ks[:, None] * span + np.arange(span, dtype=np.int64)[None, :]).ravel()
        h = halos[g][0]
        gmap = np.full(n_pad, -1, dtype=np.int64)
        gmap[rows] = np.arange(n_loc, dtype=np.int64)
        gmap[h] = n_loc + np.arange(h.shape[0], dtype=np.int64)
        sids = sids_of(ks)
        lcr = np.zeros(n_c + 1, dtype=np.int64)
        for c in range(n_c):
            a, b = chunk_bounds(int(cr[c]), int(cr[c + 1]), world)[g]
            lcr[c + 1] = lcr[c] + (b - a)
        lcr_ = lcr
        part = RankPart(rank=g, world=world, b_s=b_s, w=w, n_c=n_c, n_loc=n_loc,
                        n_halo=int(h.shape[0]), color_lvl1_ranges=lcr, lvl1=ks, rows=rows,
                        halo_rows=h, L=_local_sell(L, sids, w, n_loc, gmap),
                        U=_local_sell(U, sids, w, n_loc, gmap),
                        A=_local_sell(A, sids, w, n_loc, gmap),
                        inv_d=np.ascontiguousarray(inv_d[rows]))
        del gmap

        def local_of(grow):
            return local_pos[grow // span] * span + grow % span

        def build(kind, c):
            # kind: "fwd" classes 0-1, "bwd" classes 1-2, "spmv" everything from a peer
            send_idx, sends, recvs = [], [], []
            off = 0
            for d in range(world):
                if d == g:
                    continue
                # what g sends to d
                if kind == "spmv":
                    hd = halos[d]
                    a = int(np.searchsorted(hd[1], g, "left"))
                    b = int(np.searchsorted(hd[1], g, "right"))
                else:
                    a, b, c0, c2 = group(d, g, c)
                    a, b = (a, c2) if kind == "fwd" else (c0, b)
                if b > a:
                    send_idx.append(local_of(halos[d][0][a:b]))
                    n_loc_d = lvl1[d].shape[0] * span
                    sends.append(Msg(d, off, b - a, n_loc_d + a))
                    off += b - a
            for s in range(world):
                if s == g:
                    continue
                if kind == "spmv":
                    a = int(np.searchsorted(halos[g][1], s, "left"))
                    b = int(np.searchsorted(halos[g][1], s, "right"))
                else:
                    a, b, c0, c2 = group(g, s, c)
                    a, b = (a, c2) if kind == "fwd" else (c0, b)
                if b > a:
                    recvs.append(Msg(s, n_loc + a, b - a))
            idx = (np.concatenate(send_idx) if send_idx else np.zeros(0, np.int64))
            ex = Exchange(idx.astype(np.int32), sends, recvs)
            if True:
                # rows the push may come from: color c's (sweeps) or all (spmv)
                row0 = 0 if kind == "spmv" else int(lcr_[c]) * span
                nrows = n_loc if kind == "spmv" else int(lcr_[c + 1] - lcr_[c]) * span
                rows_l = idx.astype(np.int64) - row0
                rk = np.concatenate([np.full(m.count, m.peer, np.int64) for m in sends]) \
                    if sends else np.zeros(0, np.int64)
                ro = np.concatenate([m.remote_offset + np.arange(m.count, dtype=np.int64)
                                     for m in sends]) if sends else np.zeros(0, np.int64)
                if rows_l.size and (rows_l.min() < 0 or rows_l.max() >= nrows):
                    raise AssertionError("partition: a sent row outside its color's rows")
                order = np.argsort(rows_l, kind="stable")
                ptr = np.zeros(nrows + 1, dtype=np.int64)
                np.cumsum(np.bincount(rows_l, minlength=nrows), out=ptr[1:])
                ex.push_row0 = row0
                ex.push_ptr = ptr.astype(np.int32)
                ex.push_rank = rk[order].astype(np.int32)
                ex.push_off = ro[order].astype(np.int32)
            return ex

        # the last forward phase and the last backward phase (color 0) feed
        # no later phase of their own sweep: no exchange after them
        part.fwd = [build("fwd", c) if c < n_c - 1 else Exchange(np.zeros(0, np.int32), [], [])
                    for c in range(n_c)]
        part.bwd = [build("bwd", c) if c > 0 else Exchange(np.zeros(0, np.int32), [], [])
                    for c in range(n_c)]
        part.spmv = build("spmv", -1)
        parts.append(part)
    return parts

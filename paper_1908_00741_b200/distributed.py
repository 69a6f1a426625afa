"""Row-partitioned HBMC ICCG across ranks.

Each rank owns chunk g of every color's level-1 range (`partition.py`) and
runs the single-device sweep / SpMV kernels on its local HBMC system.  Per
preconditioner application there are `n_c - 1` halo exchanges per sweep --
one after every color phase that a later phase of the same sweep depends on
(the reference's `n_c - 1` fork-join barriers, `src/precond.py:389-391`) --
and one p-halo exchange before each SpMV.  CG dot products are reduced
across ranks (NCCL all-reduce on the device scalars) at two points per
iteration: {p.Ap} and {||r||^2, r.z} in one all-reduce; the only host read
per iteration is p.Ap and ||r|| for the breakdown / convergence tests, as
in `src/solver.py:176-187`.

The iteration is `src/solver.py:139-204` restated over partitioned vectors:

    x0 = 0, r = b, z = M r, p = z, rz = <r, z>
    loop: ap = A p; pap = <p, ap> (<= 0: CgBreakdownError); alpha = rz/pap
          x += alpha p; r -= alpha ap; z = M r
          [||r||^2, rz_new] reduced together; rel = ||r||/||b||; stop if rel < tol
          beta = rz_new/rz; p = z + beta p

M r is applied before the convergence test so that ||r||^2 travels with
r.z: the values are the reference's, only the last iteration applies M once
more than the reference does.

Local-rank lockstep: one process may drive several ranks ("virtual ranks",
e.g. G partitions on one GPU for parity tests, all work serialised on one
stream -- no rank ever waits on another inside a kernel); with
torch.distributed initialised, each process drives exactly one rank and
messages to other processes go through `batch_isend_irecv` (NCCL over
NVLink on B200s, gloo in the CPU tests).  Every exchange step receives
directly into the halo slice of the destination vector (the partition
orders the halo so each message is contiguous); sends are packed by one
gather kernel per exchange step.

`ops` is the per-rank compute backend.  The product backend is
`CudaRankOps` (kernels of libhbmc_b200.so through the C ABI); the CPU tests
plug in an oracle-backed backend to check the exchange logic under gloo.
"""

import math
import time

import numpy as np

from . import _lib
from .partition import partition_hbmc

# device scalar slots; r.z alternates between RZ0 and RZ1 around RR, so the
# merged all-reduce of {||r||^2, r.z_new} is always one contiguous pair and
# never touches the current r.z
BB, PAP, RZ0, RR, RZ1 = 0, 1, 2, 3, 4
N_SCAL = 8


class CudaRankOps:
    """Per-rank device backend: a tb_plan over the local HBMC system plus the
    distributed-CG vector kernels (`csrc/dist.cu`)."""

    def __init__(self, part, device=None, stream=None):
        from . import device as D
        t = D.require_cuda()
        self.t = t
        self.part = part
        self.n = part.n_loc
        self.ws = t.empty(4096, dtype=t.float64, device="cuda")
        self.idx = {}
        self.plan = None
        self.plan_lean = True
        if part.n_loc == 0:   # a rank with no level-1 block (tiny systems)
            return
        self.plan = D.DevicePlan(kind=_lib.TB_PRECOND_HBMC, n=part.n_loc, n_real=part.n_loc,
                                 inv_d=part.inv_d, w=part.w, b_s=part.b_s,
                                 color_lvl1_ranges=part.color_lvl1_ranges,
                                 L_sell=part.L, U_sell=part.U,
                                 spmv_format=_lib.TB_SPMV_SELL, A_sell=part.A,
                                 device=device, partitioned=True)
        self.plan_lean = all(
            self.plan.phase_info(f, c)["staged"] == 4 or
            part.color_lvl1_ranges[c + 1] == part.color_lvl1_ranges[c]
            for f in (True, False) for c in range(part.n_c))

    def stream(self):
        from . import device as D
        return D.current_stream()

    def vec(self, n=None):
        return self.t.zeros(self.part.n_ext if n is None else n, dtype=self.t.float64,
                            device="cuda")

    def scalars(self):
        return self.t.zeros(N_SCAL, dtype=self.t.float64, device="cuda")

    def from_host(self, a):
        return self.t.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()

    def to_host(self, v, n=None):
        return v[: self.n if n is None else n].cpu().numpy()

    def sweep_phase(self, forward, c, src, dst):
        if self.plan is not None:
            self.plan.sweep_phase(forward, c, src, dst)

    def spmv(self, x, out):
        if self.plan is not None:
            self.plan.spmv(x, out)

    def pack(self, key, ex, src, buf):
        if ex.n_send == 0:
            return
        idx = self.idx.get(key)
        if idx is None:
            idx = self.idx[key] = self.t.from_numpy(ex.send_idx).cuda()
        _lib.check(_lib.LIB.tb_dev_gather(ex.n_send, _lib.ptr(idx), _lib.ptr(src),
                                          _lib.ptr(buf), self.stream()))

    def copy_range(self, dst, doff, src, soff, cnt):
        dst[doff:doff + cnt].copy_(src[soff:soff + cnt])

    def dot(self, u, v, scal, slot):
        _lib.check(_lib.LIB.tb_dev_dot(self.n, _lib.ptr(u), _lib.ptr(v), _lib.ptr(scal),
                                       slot, _lib.ptr(self.ws), self.stream()))

    def update_xr(self, scal, num, den, p, ap, x, r, rr_slot):
        _lib.check(_lib.LIB.tb_dev_cg_xr(self.n, _lib.ptr(scal), num, den, _lib.ptr(p),
                                         _lib.ptr(ap), _lib.ptr(x), _lib.ptr(r), rr_slot,
                                         _lib.ptr(self.ws), self.stream()))

    def update_p(self, scal, num, den, z, p):
        _lib.check(_lib.LIB.tb_dev_cg_p(self.n, _lib.ptr(scal), num, den, _lib.ptr(z),
                                        _lib.ptr(p), self.stream()))

    def copy(self, dst, src):
        dst[: self.n].copy_(src[: self.n])

    def fill_zero(self, v):
        v.zero_()

    def read(self, scal, slots):
        h = scal.cpu().numpy()
        return [float(h[s]) for s in slots]

    def add_scal(self, dst, src, slots):
        for s in slots:
            dst[s:s + 1].add_(src[s:s + 1])

    def set_scal(self, dst, src, slots):
        for s in slots:
            dst[s:s + 1].copy_(src[s:s + 1])

    def close(self):
        if self.plan is not None:
            self.plan.close()


class _DevBuf:
    """A raw device allocation viewed as a torch tensor (no copy)."""

    def __init__(self, ptr, n, dtype_str, device):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": dtype_str,
                                         "data": (ptr, False), "version": 3}
        self.device = device


class P2PTransport:
    """NVLink halo exchange by peer stores (csrc/dist.cu tb_p2p_*), no NCCL
    on the data path.

    Every local rank owns peer-visible copies of the exchanged vectors
    (y, z, p: `vec(name)`) and a flag word per sender.  Exchange step e:
    each rank pushes every message straight into the receiver's halo slice
    (gather + remote store in one kernel) and publishes epoch e in the
    receiver's flag for this sender -- an empty push to the peers it sends
    nothing to, so every receiver waits on all world - 1 flags -- then each
    rank's stream waits (acquire, system scope) for its flags before the next
    phase.  All ranks run the same exchange sequence, so epochs agree.
    Remote ranks' buffers are mapped through CUDA IPC handles exchanged with
    torch.distributed (all_gather_object); local (virtual) ranks use the
    pointers directly.
    """

    NAMES = ("y", "z", "p")

    def __init__(self, drv, fused=True, serialize=False):
        import ctypes as C
        t = drv.ops[0].t
        self.t, self.drv = t, drv
        # serialize (tests with several processes on ONE GPU): every rank's
        # pushes complete and all ranks meet at a host barrier before any
        # rank enqueues a flag wait, so no kernel ever spins on a peer's
        # kernel (ranks on one GPU are not guaranteed to run concurrently)
        self.serialize = serialize
        self.world = drv.world
        self.epoch = 0
        self.bufs = []          # per local rank: {name: (ptr, tensor)}
        self.flags = []         # per local rank: (ptr, tensor uint32[world])
        self.ctr = []           # per local rank: (ptr, tensor) push completion counter
        dev = t.device("cuda", t.cuda.current_device())
        mine = {}
        for i, p in enumerate(drv.parts):
            entry, handles = {}, {}
            for name in self.NAMES + ("flags", "ctr"):
                n = p.n_ext if name in self.NAMES else (self.world if name == "flags" else 1)
                nbytes = 8 * max(n, 1) if name in self.NAMES else 4 * max(n, 1)
                ptr = C.c_void_p()
                h = (C.c_char * 64)()
                _lib.check(_lib.LIB.tb_p2p_alloc(nbytes, C.byref(ptr), h))
                ts = "<f8" if name in self.NAMES else "<u4"
                tens = t.as_tensor(_DevBuf(ptr.value, max(n, 1), ts, dev), device=dev)
                entry[name] = (ptr.value, tens)
                handles[name] = bytes(h)
            self.bufs.append(entry)
            mine[p.rank] = handles
        # peer pointers: rank -> name -> device pointer
        self.peer = {p.rank: {k: v[0] for k, v in self.bufs[i].items()}
                     for i, p in enumerate(drv.parts)}
        self.opened = []
        if drv.dist is not None:
            allh = [None] * self.world
            drv.dist.all_gather_object(allh, mine, group=drv.group)
            for hmap in allh:
                for rank, handles in hmap.items():
                    if rank in self.peer:
                        continue
                    self.peer[rank] = {}
                    for name, h in handles.items():
                        if name == "ctr":
                            continue
                        ptr = C.c_void_p()
                        _lib.check(_lib.LIB.tb_p2p_open(h, C.byref(ptr)))
                        self.peer[rank][name] = ptr.value
                        self.opened.append(ptr.value)
        self.idx = {}
        # fused sweep + push (tb_plan_sweep_phase_push): destinations per row
        self.fused = fused
        self.descs = {}

    def _desc(self, i, kind, c, name, ex):
        key = (i, kind, c, name)
        d = self.descs.get(key)
        if d is None:
            p = self.drv.parts[i]
            peers = [r for r in range(self.world) if r != p.rank]
            slot = {r: q for q, r in enumerate(peers)}
            dptr = self.t.from_numpy(ex.push_ptr).cuda()
            dpeer = self.t.from_numpy(
                np.array([slot[int(r)] for r in ex.push_rank], dtype=np.int32)).cuda()
            doff = self.t.from_numpy(ex.push_off).cuda()
            d = _lib.TbPushDesc()
            d.row0 = ex.push_row0
            d.nrows = ex.push_ptr.shape[0] - 1
            d.ptr, d.peer, d.off = dptr.data_ptr(), dpeer.data_ptr(), doff.data_ptr()
            d.npeers = len(peers)
            for q, r in enumerate(peers):
                d.peer_dst[q] = self.peer[r][name]
                d.peer_flag[q] = self.peer[r]["flags"] + 4 * p.rank
            d.done_ctr = self.bufs[i]["ctr"][0]
            self.descs[key] = d = (d, (dptr, dpeer, doff))
        return d[0]

    def _before_wait(self):
        if self.serialize and self.drv.dist is not None:
            self.t.cuda.synchronize()
            self.drv.dist.barrier(group=self.drv.group)

    def fused_phase(self, forward, c, src, dst, name):
        """Color phase c of a sweep on every local rank with the halo push
        fused into the sweep kernel, then each rank's stream waits for its
        peers' flags (the exchange step of this phase)."""
        from . import device as D
        self.epoch = (self.epoch + 1) & 0x7fffffff
        st = D.current_stream()
        kind = "fwd" if forward else "bwd"
        for i, p in enumerate(self.drv.parts):
            ex = self.drv._ex(p, kind, c)
            ops = self.drv.ops[i]
            if ops.plan is not None:
                desc = self._desc(i, kind, c, name, ex)
                desc.epoch = self.epoch
                ops.plan.sweep_phase_push(forward, c, src[i], dst[i], desc)
            else:   # a rank without rows still releases its flags
                for r in range(self.world):
                    if r != p.rank:
                        _lib.check(_lib.LIB.tb_p2p_push(0, None, None, None,
                                                        self.peer[r]["flags"] + 4 * p.rank,
                                                        self.epoch, self.bufs[i]["ctr"][0], st))
            self.drv.bytes_sent += 8 * int(ex.push_off.shape[0]) if ex.push_off is not None else 0
        self._before_wait()
        for i, p in enumerate(self.drv.parts):
            _lib.check(_lib.LIB.tb_p2p_wait(self.bufs[i]["flags"][0], self.world, p.rank,
                                            self.epoch, st))

    def fused_p_update(self, scal, num, den, z, p):
        """p = z + beta p on every local rank with the p-halo push fused in;
        returns the epoch the next SpMV waits for."""
        import ctypes as C
        from . import device as D
        self.epoch = (self.epoch + 1) & 0x7fffffff
        st = D.current_stream()
        for i, part in enumerate(self.drv.parts):
            ex = part.spmv
            desc = self._desc(i, "spmv", -1, "p", ex)
            desc.epoch = self.epoch
            _lib.check(_lib.LIB.tb_dev_cg_p_push(part.n_loc, _lib.ptr(scal[i]), num, den,
                                                 _lib.ptr(z[i]), _lib.ptr(p[i]),
                                                 C.byref(desc), st))
            self.drv.bytes_sent += 8 * int(ex.push_off.shape[0])
        return self.epoch

    def wait(self, epoch):
        from . import device as D
        self._before_wait()
        st = D.current_stream()
        for i, p in enumerate(self.drv.parts):
            _lib.check(_lib.LIB.tb_p2p_wait(self.bufs[i]["flags"][0], self.world, p.rank,
                                            epoch, st))

    def vec(self, i, name):
        return self.bufs[i][name][1][: self.drv.parts[i].n_ext]

    def exchange(self, kind, c, name, exs):
        from . import device as D
        self.epoch = (self.epoch + 1) & 0x7fffffff
        st = D.current_stream()
        for i, (p, ex) in enumerate(zip(self.drv.parts, exs)):
            src = self.bufs[i][name][0]
            ctr = self.bufs[i]["ctr"][0]
            key = (kind, c, i)
            idx = self.idx.get(key)
            if idx is None and ex.n_send:
                idx = self.idx[key] = self.t.from_numpy(ex.send_idx).cuda()
            sent = set()
            for m in ex.sends:
                sent.add(m.peer)
                _lib.check(_lib.LIB.tb_p2p_push(
                    m.count, idx.data_ptr() + 4 * m.offset, src,
                    self.peer[m.peer][name] + 8 * m.remote_offset,
                    self.peer[m.peer]["flags"] + 4 * p.rank, self.epoch, ctr, st))
                self.drv.bytes_sent += 8 * m.count
            for d in range(self.world):   # flag-only pushes keep every waiter uniform
                if d != p.rank and d not in sent:
                    _lib.check(_lib.LIB.tb_p2p_push(0, None, src, None,
                                                    self.peer[d]["flags"] + 4 * p.rank,
                                                    self.epoch, ctr, st))
        self._before_wait()
        for i, p in enumerate(self.drv.parts):
            _lib.check(_lib.LIB.tb_p2p_wait(self.bufs[i]["flags"][0], self.world, p.rank,
                                            self.epoch, st))

    def close(self):
        for ptr in self.opened:
            _lib.LIB.tb_p2p_close(ptr)
        self.opened = []
        for entry in self.bufs:
            for ptr, _ in entry.values():
                _lib.LIB.tb_p2p_free(ptr)
        self.bufs = []


class DistHbmc:
    """Lockstep driver of the local ranks of this process.

    parts: RankParts owned by this process (all G for a single process; one
    per process under torch.distributed, with part.rank == dist rank).
    """

    def __init__(self, parts, ops, group=None, transport="nccl", fused=True, serialize=False):
        self.parts = list(parts)
        self.ops = list(ops)
        self.world = self.parts[0].world
        self.local = {p.rank: i for i, p in enumerate(self.parts)}
        self.group = group
        self.dist = None
        if len(self.parts) < self.world:
            import torch.distributed as dist
            if not dist.is_initialized():
                raise RuntimeError("DistHbmc: remote ranks need torch.distributed")
            self.dist = dist
        n_c = self.parts[0].n_c
        self.n_c = n_c
        self.sendbuf = {}
        for key_kind in ("fwd", "bwd", "spmv"):
            for c in (range(n_c) if key_kind != "spmv" else [-1]):
                for i, p in enumerate(self.parts):
                    ex = self._ex(p, key_kind, c)
                    if ex.n_send:
                        self.sendbuf[(key_kind, c, i)] = self.ops[i].vec(ex.n_send)
        self.exchanges = 0
        self.bytes_sent = 0
        self.reductions_per_iteration = 2   # {p.Ap}, {||r||^2, r.z}
        self.p2p = (P2PTransport(self, fused=fused, serialize=serialize)
                    if transport == "p2p" else None)
        self._p_epoch = 0

    @staticmethod
    def _ex(p, kind, c):
        return p.spmv if kind == "spmv" else (p.fwd[c] if kind == "fwd" else p.bwd[c])

    # ---------------------------------------------------------------- halo
    def exchange(self, kind, c, vecs):
        """Deliver the owners' values of `vecs` (one extended vector per local
        rank) into the peers' halo slices for exchange step (kind, c)."""
        exs = [self._ex(p, kind, c) for p in self.parts]
        if self.p2p is not None:
            name = self._p2p_name(vecs)
            if kind != "spmv" and ((kind == "fwd" and c == self.n_c - 1) or
                                   (kind == "bwd" and c == 0)):
                return   # no exchange after the last phase of a sweep (any transport)
            self.p2p.exchange(kind, c, name, exs)
            self.exchanges += 1
            return
        if all(ex.n_send == 0 and not ex.recvs for ex in exs):
            return
        for i, ex in enumerate(exs):
            self.ops[i].pack((kind, c), ex, vecs[i], self.sendbuf.get((kind, c, i)))
        p2p = []
        for i, (p, ex) in enumerate(zip(self.parts, exs)):
            buf = self.sendbuf.get((kind, c, i))
            for m in ex.sends:
                self.bytes_sent += 8 * m.count
                j = self.local.get(m.peer)
                if j is not None:
                    # in-process peer: find its matching receive slot
                    rm = next(r for r in exs[j].recvs if r.peer == p.rank)
                    assert rm.count == m.count
                    self.ops[j].copy_range(vecs[j], rm.offset, buf, m.offset, m.count)
                else:
                    p2p.append(self.dist.P2POp(self.dist.isend, buf[m.offset:m.offset + m.count],
                                               m.peer, self.group))
            for rm in ex.recvs:
                if rm.peer not in self.local:
                    p2p.append(self.dist.P2POp(self.dist.irecv,
                                               vecs[i][rm.offset:rm.offset + rm.count],
                                               rm.peer, self.group))
        if p2p:
            for req in self.dist.batch_isend_irecv(p2p):
                req.wait()
        self.exchanges += 1

    def _p2p_name(self, vecs):
        # identify the buffer on a local rank that has rows (an empty rank's
        # views are zero-length and their data pointers may coincide)
        i = next((k for k, p in enumerate(self.parts) if p.n_ext > 0), 0)
        ptr = vecs[i].data_ptr()
        for name in P2PTransport.NAMES:
            if self.p2p.vec(i, name).data_ptr() == ptr:
                return name
        raise ValueError("p2p exchange: vector is not a peer-visible buffer (use ext_vec)")

    def ext_vec(self, i, name):
        """Extended vector of local rank i; with the P2P transport the
        exchanged ones (y, z, p) live in peer-visible buffers."""
        if self.p2p is not None and name in P2PTransport.NAMES:
            return self.p2p.vec(i, name)
        return self.ops[i].vec()

    def close(self):
        if self.p2p is not None:
            self.p2p.close()
            self.p2p = None

    # ---------------------------------------------------------------- reductions
    def allreduce(self, scals, slots):
        """Sum the given scalar slots over all ranks, result on every rank."""
        if len(scals) > 1:
            for i in range(1, len(scals)):
                self.ops[0].add_scal(scals[0], scals[i], slots)
        if self.dist is not None:
            lo, hi = min(slots), max(slots) + 1
            assert hi - lo == len(slots), "all-reduced slots must be contiguous"
            t = scals[0][lo:hi]
            if t.is_cuda and self.dist.get_backend(self.group) == "gloo":
                h = t.cpu()   # gloo (one-GPU multi-process tests): via the host
                self.dist.all_reduce(h, group=self.group)
                t.copy_(h)
            else:
                self.dist.all_reduce(t, group=self.group)
        for i in range(1, len(scals)):
            self.ops[i].set_scal(scals[i], scals[0], slots)

    # ---------------------------------------------------------------- operators
    def sweep(self, forward, src, dst):
        """One substitution sweep on all local ranks with the per-color halo
        exchange (src/precond.py:377-392)."""
        order = range(self.n_c) if forward else range(self.n_c - 1, -1, -1)
        last = self.n_c - 1 if forward else 0
        fused = (self.p2p is not None and self.p2p.fused and self.parts[0].w == 32 and
                 all(o.plan is None or o.plan_lean for o in self.ops))
        for c in order:
            if fused and c != last:
                self.p2p.fused_phase(forward, c, src, dst, self._p2p_name(dst))
                self.exchanges += 1
                continue
            for i in range(len(self.parts)):
                self.ops[i].sweep_phase(forward, c, src[i], dst[i])
            self.exchange("fwd" if forward else "bwd", c, dst)

    def precond(self, r, y, z):
        self.sweep(True, r, y)
        self.sweep(False, y, z)

    def spmv(self, x, out):
        if self._p_epoch:   # the p update already pushed the halo: just wait
            self.p2p.wait(self._p_epoch)
            self._p_epoch = 0
            self.exchanges += 1
        else:
            self.exchange("spmv", -1, x)
        for i in range(len(self.parts)):
            self.ops[i].spmv(x[i], out[i])

    def update_p(self, sc, num, den, z, p):
        """p = z + beta p; with the fused P2P transport the p halo for the next
        SpMV is pushed by the same kernel."""
        if self.p2p is not None and self.p2p.fused and all(o.plan is not None for o in self.ops):
            self._p_epoch = self.p2p.fused_p_update(sc, num, den, z, p)
            return
        for i in range(len(self.parts)):
            self.ops[i].update_p(sc[i], num, den, z[i], p[i])

    # ---------------------------------------------------------------- PCG
    def pcg(self, b_loc, tol=1e-7, max_iters=50000):
        """src/solver.py:157-193 over the partition.

        b_loc: per local rank, the local rhs (length n_loc; backend vectors).
        Returns (x per local rank, iterations, history, converged).
        """
        R = range(len(self.parts))
        O = self.ops
        self._p_epoch = 0   # a halo push left over from an earlier solve is stale
        V = lambda name: [self.ext_vec(i, name) for i in R]  # noqa: E731
        x, r, y, z, p, ap = V("x"), V("r"), V("y"), V("z"), V("p"), V("ap")
        sc = [O[i].scalars() for i in R]
        for i in R:
            O[i].fill_zero(x[i])
            O[i].copy(r[i], b_loc[i])
            O[i].dot(r[i], r[i], sc[i], BB)
        self.allreduce(sc, [BB])
        bnorm = math.sqrt(O[0].read(sc[0], [BB])[0])
        if bnorm == 0.0:
            return x, 0, [0.0], True
        history = [1.0]
        self.precond(r, y, z)
        for i in R:
            O[i].copy(p[i], z[i])
            O[i].dot(r[i], z[i], sc[i], RZ0)
        self.allreduce(sc, [RZ0])
        rz, rzn = RZ0, RZ1
        it, converged = 0, False
        for j in range(1, max_iters + 1):
            self.spmv(p, ap)
            for i in R:
                O[i].dot(p[i], ap[i], sc[i], PAP)
            self.allreduce(sc, [PAP])
            for i in R:
                O[i].update_xr(sc[i], rz, PAP, p[i], ap[i], x[i], r[i], RR)
            # z = M r before the convergence test: ||r||^2 and r.z are reduced
            # in one all-reduce (slots RR and rzn are adjacent)
            self.precond(r, y, z)
            for i in R:
                O[i].dot(r[i], z[i], sc[i], rzn)
            self.allreduce(sc, [RR, rzn])
            pap, rr = O[0].read(sc[0], [PAP, RR])
            if pap <= 0.0:
                from .solver import CgBreakdownError
                raise CgBreakdownError(j, pap)
            rel = math.sqrt(rr) / bnorm
            history.append(rel)
            it = j
            if rel < tol:
                converged = True
                break
            self.update_p(sc, rzn, rz, z, p)
            rz, rzn = rzn, rz
        return x, it, history, converged


def partition_setup(setup, world, ranks=None):
    """RankParts of a prepared single-system HBMC Setup (solver.prepare)."""
    from .matrix import csr_to_sell
    sf, hl = setup.factor, setup.layout
    a_sell = csr_to_sell(setup.a_sys, sf.w, want_col64=True)
    return partition_hbmc(sf.lower, sf.upper, a_sell, sf.inv_diag, hl.color_lvl1_ranges,
                          sf.b_s, sf.w, world, ranks)


def prepare_rank_parts(a, b, cfg, world, rank=0, dist=None, group=None, shm_root="/dev/shm"):
    """Rank-local setup: rank 0 alone builds the global HBMC system
    (solver.prepare -- the greedy ordering and IC(0) are sequential over the
    whole matrix, src/solver.py:127-136) and partitions it one rank at a
    time; every rank then loads only its own RankPart and its slice of b
    from a tmpfs directory (node-local, like the GPUs).  So only rank 0 ever
    holds the whole system (config 5: ~100 GB of host memory once, not once
    per rank).  `a` and `b` are only read on rank 0.

    Returns (part, b_loc, info): info on rank 0 = dict(n_pad, old_positions,
    n_c, n_dummy, t_prepare); on the other ranks the same keys with
    old_positions None.
    """
    import os
    import pickle
    import shutil
    import tempfile
    from . import solver
    t0 = time.perf_counter()
    if dist is None or world == 1:
        setup = solver.prepare(a, b, cfg)
        part = partition_setup(setup, world, [rank])[0]
        return part, setup.b_sys[part.rows], dict(
            n_pad=setup.a_sys.n, old_positions=setup.old_positions, n_c=setup.n_c,
            n_dummy=setup.n_dummy, t_prepare=time.perf_counter() - t0)
    meta = [None]
    if rank == 0:
        setup = solver.prepare(a, b, cfg)
        root = shm_root if os.path.isdir(shm_root) else None
        tmp = tempfile.mkdtemp(prefix="hbmc_parts_", dir=root)
        for g in range(world):
            pg = partition_setup(setup, world, [g])[0]
            with open(os.path.join(tmp, f"part{g}.pkl"), "wb") as fh:
                pickle.dump((pg, setup.b_sys[pg.rows]), fh, protocol=5)
            if g == 0:
                mine = pg
            del pg
        info = dict(n_pad=setup.a_sys.n, old_positions=setup.old_positions, n_c=setup.n_c,
                    n_dummy=setup.n_dummy)
        meta = [dict(dir=tmp, n_pad=info["n_pad"], n_c=info["n_c"],
                     n_dummy=info["n_dummy"])]
        b0 = setup.b_sys[mine.rows]
        del setup
    dist.broadcast_object_list(meta, src=0, group=group)
    m = meta[0]
    if rank != 0:
        with open(os.path.join(m["dir"], f"part{rank}.pkl"), "rb") as fh:
            mine, b0 = pickle.load(fh)
        info = dict(n_pad=m["n_pad"], old_positions=None, n_c=m["n_c"], n_dummy=m["n_dummy"])
    dist.barrier(group=group)
    if rank == 0:
        shutil.rmtree(m["dir"], ignore_errors=True)
    info["t_prepare"] = time.perf_counter() - t0
    return mine, b0, info


def pcg_partitioned(a, b, cfg, world, matrix_name="", group=None, transport="nccl"):
    """HBMC ICCG with the rows partitioned over `world` ranks.

    Without torch.distributed: all `world` ranks are driven by this process
    on the current device (virtual ranks).  Under torch.distributed with
    world_size == world: this process drives its own rank; every rank
    returns the full solution (gathered on the host) and the same report.
    Returns (x in the original ordering, SolveReport).
    """
    from . import solver
    cfg.validate()
    if cfg.ordering != "hbmc":
        raise ValueError("pcg_partitioned: only the hbmc ordering partitions")
    t0 = time.perf_counter()
    dist = None
    try:
        import torch.distributed as td
        if td.is_initialized() and td.get_world_size(group) > 1:
            dist = td
    except ImportError:
        pass
    if dist is not None and dist.get_world_size(group) != world:
        raise ValueError("pcg_partitioned: world != torch.distributed world size")
    if dist is not None:
        part, b0, info = prepare_rank_parts(a, b, cfg, world, dist.get_rank(group), dist, group)
        parts, b_hosts = [part], [b0]
    else:
        setup = solver.prepare(a, b, cfg)
        parts = partition_setup(setup, world)
        b_hosts = [setup.b_sys[p.rows] for p in parts]
        info = dict(n_pad=setup.a_sys.n, old_positions=setup.old_positions, n_c=setup.n_c,
                    n_dummy=setup.n_dummy)
        del setup
    ops = [CudaRankOps(p) for p in parts]
    drv = DistHbmc(parts, ops, group, transport=transport)
    b_loc = [ops[i].from_host(bh) for i, bh in enumerate(b_hosts)]
    ops[0].t.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    t1 = time.perf_counter()
    try:
        xs, it, hist, conv = drv.pcg(b_loc, cfg.tol, cfg.max_iters)
        x_sys = np.zeros(info["n_pad"])
        for i, p in enumerate(parts):
            x_sys[p.rows] = ops[i].to_host(xs[i])
        if dist is not None:
            # every row is owned by exactly one rank: a sum assembles x everywhere
            xt = ops[0].t.from_numpy(x_sys)
            if dist.get_backend(group) == "nccl":
                xt = xt.cuda()
            dist.all_reduce(xt, group=group)
            x_sys = xt.cpu().numpy()
            pos = [info["old_positions"]]
            dist.broadcast_object_list(pos, src=0, group=group)
            info["old_positions"] = pos[0]
    finally:
        drv.close()
        for o in ops:
            o.close()
    t_solve = time.perf_counter() - t1
    x_out = x_sys[info["old_positions"]]
    applies = it if conv else 1 + it
    barrier_total = applies * 2 * max(info["n_c"] - 1, 0)
    rep = solver.SolveReport(matrix_name, cfg.ordering, cfg.b_s, cfg.w, info["n_c"], int(it),
                             bool(conv), t_setup, t_solve, [float(v) for v in hist],
                             barrier_total, info["n_dummy"])
    return x_out, rep

"""The multi-process P2P transport across REAL processes on
one B200: two torch.distributed ranks (gloo for the host-side collectives),
each a separate process with its own CUDA context, exchange their halos by
peer stores into each other's buffers through CUDA IPC mappings
(tb_p2p_alloc / tb_p2p_open) and release / acquire system-scope flags --
the code path a real 2-GPU run uses, including the sweep kernels with the
halo push fused in and the p-update push.

Ranks on ONE GPU are not guaranteed to run concurrently, so the transport
runs in its `serialize` mode: before any rank enqueues a flag wait, every
rank's pushes have completed and all ranks have met at a host barrier --
the wait kernels find their flags already released and never spin on a
peer's kernel (B200_PROFILING.md: kernels that wait on one another must
not share a GPU).  Results must be bitwise the single-device ones
(sweeps) and meet the north-star bar (PCG).
"""

import os
import socket

import numpy as np
import pytest

from conftest import golden_matrix, load_golden, rel_err

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, out_dir):
    import torch
    import torch.distributed as dist
    import paper_1908_00741_b200 as P
    from paper_1908_00741_b200 import distributed as D
    import workloads
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, bs, w, rhs_kind = golden_matrix(name)
        b = np.ones(a.n) if rhs_kind == "ones" else workloads.rhs(a)[1]
        cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
        part, b_loc, info = D.prepare_rank_parts(a if rank == 0 else None,
                                                 b if rank == 0 else None, cfg, world, rank,
                                                 dist, shm_root=out_dir)
        ops = D.CudaRankOps(part)
        drv = D.DistHbmc([part], [ops], transport="p2p", serialize=True)
        try:
            g = load_golden(name)
            r_glob = np.ascontiguousarray(g["r"])
            r = [ops.from_host(np.concatenate([r_glob[part.rows], np.zeros(part.n_halo)]))]
            y, z = [drv.ext_vec(0, "y")], [drv.ext_vec(0, "z")]
            drv.precond(r, y, z)
            torch.cuda.synchronize()
            yl = y[0][: part.n_loc].cpu().numpy()
            zl = z[0][: part.n_loc].cpu().numpy()
            xs, it, hist, conv = drv.pcg([ops.from_host(b_loc)], cfg.tol, cfg.max_iters)
            torch.cuda.synchronize()
            np.savez(os.path.join(out_dir, f"rank{rank}.npz"), rows=part.rows, y=yl, z=zl,
                     x=ops.to_host(xs[0]), it=it, hist=np.asarray(hist), conv=conv,
                     exchanges=drv.exchanges, sent=drv.bytes_sent, n_pad=info["n_pad"],
                     fused=drv.p2p.fused)
        finally:
            drv.close()
            ops.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["var7_16_b8_w32", "knn3000_b4_w32", "aniso12_b16_w32"])
def test_two_processes_p2p_ipc_on_one_gpu(name, tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world,
             join=True)
    g = load_golden(name)
    res = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    n_pad = int(res[0]["n_pad"])
    y = np.full(n_pad, np.nan)
    z = np.full(n_pad, np.nan)
    x_sys = np.full(n_pad, np.nan)
    for r in res:
        assert r["sent"] > 0 and r["exchanges"] > 0
        y[r["rows"]] = r["y"]
        z[r["rows"]] = r["z"]
        x_sys[r["rows"]] = r["x"]
    # the halo exchange across processes delivers exactly the values the
    # single-device sweeps use: bitwise the reference's y and z
    for key, v in (("y", y), ("z", z)):
        if key in g:
            assert np.array_equal(v, g[key]), key
        else:
            import hashlib
            assert hashlib.sha256(v.tobytes()).hexdigest() == str(g[key + "_sha"]), key
    assert res[0]["it"] == res[1]["it"]
    assert np.array_equal(res[0]["hist"], res[1]["hist"])
    assert abs(int(res[0]["it"]) - int(g["pcg_hbmc_iters"])) <= 1
    from paper_1908_00741_b200 import solver
    import paper_1908_00741_b200 as P
    a, bs, w, _ = golden_matrix(name)
    cfg = P.CgConfig(ordering="hbmc", b_s=bs, w=w, spmv_format="sell")
    st = solver.prepare(a, np.zeros(a.n), cfg)
    assert rel_err(x_sys[st.old_positions], g["pcg_hbmc_x"]) <= 1e-10

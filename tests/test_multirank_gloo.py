"""Multi-rank (z-slab) decomposition on the CPU with torch.distributed/gloo (world size 2).

The CUDA ranks exchange the interface-plane partial sums with NCCL; here the
same decomposition is exercised with the library's own slab layout (sc_layout_query, host
only) and the oracle's per-slab operator: every rank applies the condensed operator to its
slab (interface plane not Dirichlet), exchanges its interface plane with the neighbour,
adds, and must reproduce the global operator on its slab; dot products counting each
interface DOF on the lower rank only must reproduce the global dot product.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _grid(p, ne, lam):
    from synth import small_grid
    g = small_grid(p, ne, lam, lengths=(1.0, 0.8, 1.3))
    g.hz = np.linspace(0.7, 1.3, ne[2]) / ne[2]
    return g


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1601_08179_b200 import capi
    return capi.load()


@pytest.mark.parametrize("R,nz", [(2, 4), (3, 5), (4, 4), (8, 128)])
def test_slab_partition_covers_grid(lib, R, nz):
    from paper_1601_08179_b200 import layout_query
    from oracle import mesh
    g = _grid(3, (3, 2, nz), 1.0)
    Ls = [layout_query(g.p, g.ne, (g.hx, g.hy, g.hz), g.lam, rank=r, nranks=R) for r in range(R)]
    assert Ls[0].z_begin == 0 and Ls[-1].z_end == nz
    for a, b in zip(Ls[:-1], Ls[1:]):
        assert a.z_end == b.z_begin and a.z_end > a.z_begin
    if nz <= 8:
        assert sum(L.n_free for L in Ls) == int(mesh.free_skeleton_mask(g).sum())
    assert all(L.n_lattice_global == g.n_lattice for L in Ls)


def _slab_worker(rank, world, port, p, ne, lam, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import __graft_entry__  # noqa: F401  (path setup)
        from paper_1601_08179_b200 import layout_query
        from oracle import mesh, operator
        from synth import lattice_random
        import copy
        g = _grid(p, ne, lam)
        L = layout_query(g.p, g.ne, (g.hx, g.hy, g.hz), g.lam, rank=rank, nranks=world)
        z0, z1 = L.z_begin, L.z_end
        # global reference
        opg = operator.AssembledCondensedOperator(g)
        xg = lattice_random(11, g.ne, g.p)                     # (nz1, ny1, nx1), Dirichlet zero
        yg = opg.apply(xg.ravel()).reshape(xg.shape)
        # this rank's slab: element layers [z0, z1), lattice planes [z0 p, z1 p]
        gs = copy.deepcopy(g)
        gs.ne = (g.ne[0], g.ne[1], z1 - z0)
        gs.hz = g.hz[z0:z1]
        gs.extra = dict(g.extra, dirichlet_z=(rank == 0, rank == world - 1))
        xs = xg[z0 * p:z1 * p + 1].copy()
        ops = operator.AssembledCondensedOperator(gs)
        ys = ops.apply(xs.ravel()).reshape(xs.shape)
        # interface-plane exchange (the NCCL send/recv pair of sc_apply_condensed)
        bot = torch.from_numpy(ys[0].copy())
        top = torch.from_numpy(ys[-1].copy())
        recv_lo = torch.zeros_like(bot)
        recv_hi = torch.zeros_like(top)
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(bot, rank - 1))
            reqs.append(dist.irecv(recv_lo, rank - 1))
        if rank < world - 1:
            reqs.append(dist.isend(top, rank + 1))
            reqs.append(dist.irecv(recv_hi, rank + 1))
        for r_ in reqs:
            r_.wait()
        if rank > 0:
            ys[0] += recv_lo.numpy()
        if rank < world - 1:
            ys[-1] += recv_hi.numpy()
        ref = yg[z0 * p:z1 * p + 1]
        err = float(np.linalg.norm(ys - ref) / np.linalg.norm(ref))
        # dot product with lower-rank ownership of the interface plane
        own = np.ones_like(xs, dtype=bool)
        if rank > 0:
            own[0] = False
        part = torch.tensor([float(np.sum(xs[own] * ys[own]))], dtype=torch.float64)
        dist.all_reduce(part)
        dot_ref = float(np.sum(xg * yg))
        out_q.put((rank, err, abs(part.item() - dot_ref) / abs(dot_ref), z0, z1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p,ne", [(3, (2, 2, 4)), (4, (2, 3, 5))])
def test_two_rank_slab_apply_matches_global(lib, p, ne):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, p, ne, 0.7, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    for rank, err, derr, z0, z1 in res:
        assert err < 1e-13, (rank, err)
        assert derr < 1e-13, (rank, derr)
    assert res[0][4] == res[1][3]

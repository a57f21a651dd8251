"""z-slab decomposition host logic on 2 gloo ranks (CPU).

Checks the communicator the sharded trainer uses (halo planes, sum/max
all-reduce) and that the slab convention -- each rank owns its forward
differences including the one into the upper halo -- reproduces the full
TV value and subgradient (loss.py:183-207) exactly.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def slab_tv(vol_yxz, lo, hi, count):
    """TV sum and subgradient of a (h, w, c) slab with halo planes (h*w,)."""
    h, w, c = vol_yxz.shape
    v = vol_yxz.astype(np.float64)
    g = np.zeros_like(v)
    tot = 0.0
    for ax in (0, 1):
        d = np.diff(v, axis=ax)
        tot += np.abs(d).sum()
        s = np.sign(d)
        sl_lead = [slice(None)] * 3
        sl_lag = [slice(None)] * 3
        sl_lead[ax] = slice(1, None)
        sl_lag[ax] = slice(0, -1)
        g[tuple(sl_lead)] += s
        g[tuple(sl_lag)] -= s
    ext = [v]
    if hi is not None:
        ext.append(hi.reshape(h, w, 1).astype(np.float64))
    if lo is not None:
        ext.insert(0, lo.reshape(h, w, 1).astype(np.float64))
    e = np.concatenate(ext, axis=2)
    off = 1 if lo is not None else 0
    d = np.diff(e, axis=2)
    s = np.sign(d)
    # differences owned by this slab: those starting at a local plane
    own = d[:, :, off:off + c] if hi is not None else d[:, :, off:off + c - 1]
    tot += np.abs(own).sum()
    ge = np.zeros_like(e)
    ge[:, :, 1:] += s
    ge[:, :, :-1] -= s
    g += ge[:, :, off:off + c]
    return tot, g / count


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2411_04844_b200.distributed import SlabComm, slab_bounds
    comm = SlabComm()
    rng = np.random.default_rng(0)
    full = rng.integers(0, 3, (6, 7, 11)).astype(np.float32)   # (h, w, c) with ties
    s = slab_bounds(11, world, rank)
    local = torch.from_numpy(np.ascontiguousarray(full[:, :, s.z0:s.z0 + s.c_local]))
    lo, hi = comm.halo(local)
    if rank == 0:
        assert lo is None
    else:
        np.testing.assert_array_equal(lo.numpy(), full[:, :, s.z0 - 1].reshape(-1))
    if rank == world - 1:
        assert hi is None
    else:
        np.testing.assert_array_equal(hi.numpy(), full[:, :, s.z0 + s.c_local].reshape(-1))
    count = full.size
    tot, g = slab_tv(local.numpy(), None if lo is None else lo.numpy(),
                     None if hi is None else hi.numpy(), count)
    t = torch.tensor([tot], dtype=torch.float64)
    comm.allreduce_sum_(t)
    m = torch.tensor([float(rank)], dtype=torch.float64)
    comm.allreduce_max_(m)
    grads = torch.full((5, 3), float(rank + 1), dtype=torch.float64)
    comm.allreduce_sum_(grads)
    q.put((rank, s.z0, s.c_local, float(t.item()), g, float(m.item()), grads.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_slab_comm_and_tv_halo_convention():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    rng = np.random.default_rng(0)
    full = rng.integers(0, 3, (6, 7, 11)).astype(np.float32)
    val, grad = O.tv_loss(np.transpose(full, (2, 0, 1)))        # oracle works on (c,h,w)
    gfull = np.transpose(grad, (1, 2, 0))
    for rank, z0, cl, tot, g, mx, gr in res:
        assert abs(tot / full.size - val) < 1e-15
        np.testing.assert_allclose(g, gfull[:, :, z0:z0 + cl], rtol=0, atol=1e-15)
        assert mx == world - 1
        assert np.all(gr == sum(range(1, world + 1)))


def test_row_bands_cover_rows_once():
    from paper_2411_04844_b200.distributed import row_bands
    for nv, world in [(48, 2), (37, 4), (512, 8), (6, 4), (1024, 8), (3, 2)]:
        b = row_bands(nv, world)
        assert len(b) == world and b[0][0] == 0 and b[-1][1] == nv
        for (a0, a1), (b0, b1) in zip(b[:-1], b[1:]):
            assert a1 == b0 and a0 <= a1
        if nv >= 4 * world:
            assert all(r0 % 4 == 0 for r0, _ in b)


def _rs_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2411_04844_b200.distributed import SlabComm, row_bands
    comm = SlabComm()
    m, nu, nv = 5, 6, 19
    bands = row_bands(nv, world)
    # rank r's partial projection; the sum over ranks is the full prediction
    part = torch.from_numpy(np.random.default_rng(rank).standard_normal((m, nu, nv)).astype(np.float32))
    r0, r1 = bands[rank]
    band = torch.empty((m, nu, r1 - r0))
    comm.reduce_scatter_rows(part, bands, band)
    # dL/dpred band -> full on every rank
    gband = band * 2.0 + rank
    full = torch.empty((m, nu, nv))
    comm.all_gather_rows(gband, bands, full)
    g32 = torch.full((5, 4), 0.1 * (rank + 1), dtype=torch.float64)
    comm.allreduce_grads_(g32)
    q.put((rank, band.numpy(), full.numpy(), g32.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_cone_row_band_exchange():
    """Cone sharding: reduce-scatter of the partial projections
    over detector-row bands, all-gather of dL/dpred, f32 gradient all-reduce."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rs_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2411_04844_b200.distributed import row_bands
    m, nu, nv = 5, 6, 19
    bands = row_bands(nv, world)
    total = sum(np.random.default_rng(r).standard_normal((m, nu, nv)).astype(np.float32)
                for r in range(world))
    want_full = np.concatenate([total[:, :, a:b] * 2.0 + r for r, (a, b) in enumerate(bands)],
                               axis=2)
    for rank, band, full, g in res:
        a, b = bands[rank]
        np.testing.assert_allclose(band, total[:, :, a:b], rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(full, want_full, rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(g, 0.1 * sum(range(1, world + 1)), rtol=1e-6)

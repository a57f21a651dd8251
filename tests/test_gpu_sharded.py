"""z-slab sharded training on real kernels: 2 ranks emulated on one GPU.

The ranks talk over gloo (host-side collectives; no rank waits on another
inside a kernel), so two processes can share the single test GPU.  The
sharded run must reproduce the single-device run_reconstruction: same loss
trace and volume up to the order of the gradient all-reduce.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(variant="fan"):
    from paper_2411_04844_b200 import core, optim, phantom, projector
    dims = (48, 40, 37)                      # odd slice count: unequal slabs
    truth = phantom.shepp_logan_3d(*dims)
    if variant == "cone":   # rays cross the slab boundary: partial projections summed
        geom = core.ScanGeometry.cone(20, 72, 48, 1.2, 80.0, 60.0, 1.0)
    else:
        geom = core.ScanGeometry.fan(20, 72, 1.2, 80.0, 60.0)
    meas = projector.forward_project(truth, geom)
    box = core.BoxConfig.for_dims(17, dims)
    cloud = optim.init_cloud_random(dims, 3000, seed=3, box=box)
    settings = optim.ReconstructionSettings(dims=dims, box=box, max_iters=12,
                                            densify_interval=0)
    return meas, geom, settings, cloud


def _worker(rank, world, port, q, variant):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2411_04844_b200.distributed import run_reconstruction_sharded
    meas, geom, settings, cloud = _problem(variant)
    vol, cl, trace = run_reconstruction_sharded(meas, geom, settings, cloud)
    trace = np.array([[r.loss, r.loss_l1, r.loss_ssim, r.loss_tv] for r in trace])
    q.put((rank, None if vol is None else vol.zyx.copy(), cl.mu.copy(), trace))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("variant,world", [("fan", 2), ("cone", 2), ("fan", 4), ("cone", 3)])
def test_two_slab_ranks_match_single_device(variant, world):
    """world 4: 9-10-slice slabs under a 17-slice box, so Gaussians straddle
    three slabs (gradient all-reduce, TV halos on both sides)."""
    from paper_2411_04844_b200 import optim
    meas, geom, settings, cloud = _problem(variant)
    vol1, cl1, tr1 = optim.run_reconstruction(meas, geom, settings, init_cloud=cloud)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, variant))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    loss1 = np.array([r.loss for r in tr1])
    # cone: the prediction is a sum of slab partial projections (fp32 order)
    rtol = 1e-6 if variant == "fan" else 1e-5
    for rank, vol, mu, trace in res:
        np.testing.assert_allclose(trace[:, 0], loss1, rtol=rtol)
        # all-reduce order (4 ranks: a few centres differ at 2e-7 relative)
        np.testing.assert_allclose(mu, cl1.mu, rtol=1e-6, atol=1e-6)
    v = res[0][1]
    assert np.linalg.norm(v - vol1.zyx) / np.linalg.norm(vol1.zyx) < (1e-6 if variant == "fan"
                                                                      else 1e-5)


def test_bench_two_ranks_smoke():
    """bench.py's N > 1 flow (torchrun, slab sharding, segmented graphs, max-over-ranks
    timing, sharded e2e) end to end with host-staged gloo collectives on one GPU."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SPLATCT_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--no-cpu-baseline", "--config", "c1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1   # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0


@pytest.mark.parametrize("edges", [(True, True), (True, False), (False, True)])
def test_tv_halo_fixup_matches_halo_adjoint(edges):
    """The overlapped-halo step: adjoint without halos + splatct_tv_halo_fixup
    equals the adjoint with halo planes (value to 1e-12, dL/dV to f32 rounding)."""
    import torch
    from paper_2411_04844_b200 import core, device as D
    dev = D.require_cuda()
    w, h, c = 40, 36, 24
    geom = core.ScanGeometry.fan(16, 60, 1.2, 70.0, 50.0)
    op = D.ProjectorOperator(geom, w, h, 0.5, dev)
    g = torch.Generator(device="cpu").manual_seed(3)
    vol = torch.randint(0, 3, (h, w, c), generator=g).float().to(dev)   # ties: sign 0
    lo = torch.randint(0, 3, (h * w,), generator=g).float().to(dev) if edges[0] else None
    hi = torch.randint(0, 3, (h * w,), generator=g).float().to(dev) if edges[1] else None
    ys = torch.randn((16, 60, c), generator=g).to(dev)
    cnt = float(w * h * 3 * c)
    n = D.tv_partial_len(w, h, c)
    s1 = torch.zeros(3, dtype=torch.float64, device=dev)
    s2 = torch.zeros(3, dtype=torch.float64, device=dev)
    tp = torch.zeros(n, dtype=torch.float64, device=dev)
    a = op.adjoint(ys, vol=vol, halo_lo=lo, halo_hi=hi, lambda_tv=1.0, tv_count=cnt,
                   tv_partial=tp)
    D.reduce_sum(tp, s1[2:3])
    b = op.adjoint(ys, vol=vol, lambda_tv=1.0, tv_count=cnt, tv_partial=tp)
    D.reduce_sum(tp, s2[2:3])
    D.tv_halo_fixup(vol, b, lo, hi, 1.0, cnt, s2[2:3])
    torch.cuda.synchronize()
    assert abs(float(s1[2]) - float(s2[2])) <= 1e-12 * abs(float(s1[2]))
    d = (a - b).abs().max().item()
    assert d <= 2e-7 * a.abs().max().item() + 1e-12


def _hooks_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2411_04844_b200.distributed import run_reconstruction_sharded
    meas, geom, settings, cloud, truth = _hooks_problem()
    vol, cl, trace = run_reconstruction_sharded(meas, geom, settings, cloud, truth=truth)
    q.put((rank, [(r.loss, r.psnr, r.ssim, r.val_loss, r.n_gaussians, r.splits) for r in trace],
           cl.n))
    dist.barrier()
    dist.destroy_process_group()


def _hooks_problem():
    from paper_2411_04844_b200 import core, optim, phantom, projector
    from paper_2411_04844_b200.densify import DensifyParams
    dims = (48, 40, 37)
    truth = phantom.shepp_logan_3d(*dims)
    geom = core.ScanGeometry.fan(20, 72, 1.2, 80.0, 60.0)
    meas = projector.forward_project(truth, geom)
    box = core.BoxConfig.for_dims(17, dims)
    cloud = optim.init_cloud_random(dims, 2000, seed=3, box=box)
    dp = DensifyParams(n_max=3000, tau=1e-12, theta=1.0, box_size=17, grad_prune_enabled=False)
    settings = optim.ReconstructionSettings(dims=dims, box=box, max_iters=14, densify_interval=6,
                                            densify=dp, stop_rule="val-convergence", patience=50)
    return meas, geom, settings, cloud, truth


def test_sharded_loop_hooks_match_single_device():
    """The sharded run_reconstruction keeps the reference loop's hooks
    (optim.py:388-424): a densification event (identical on every rank: the
    replicated cloud, the all-reduced gradient statistics), per-iteration
    truth PSNR / SSIM and the held-out-view loss of the stop rule, from
    all-reduced slab partial sums -- against the single-device run."""
    from paper_2411_04844_b200 import optim
    meas, geom, settings, cloud, truth = _hooks_problem()
    _, cl1, tr1 = optim.run_reconstruction(meas, geom, settings, truth=truth, init_cloud=cloud)
    want = [(r.loss, r.psnr, r.ssim, r.val_loss, r.n_gaussians, r.splits) for r in tr1]
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_hooks_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert any(w[5] > 0 for w in want)        # the event split Gaussians
    for rank, rows, n in res:
        assert n == cl1.n and len(rows) == len(want)
        got, ref = np.array(rows, np.float64), np.array(want, np.float64)
        np.testing.assert_array_equal(got[:, 4:], ref[:, 4:])       # N, splits
        np.testing.assert_allclose(got[:, 0], ref[:, 0], rtol=1e-5)  # loss
        np.testing.assert_allclose(got[:, 1], ref[:, 1], rtol=1e-6)  # psnr
        np.testing.assert_allclose(got[:, 2:4], ref[:, 2:4], rtol=1e-5)   # ssim, val loss

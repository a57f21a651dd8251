"""Uninitialised-memory checks of our own (compute-sanitizer is not available
on this GPU pool): every workspace and output buffer is pre-filled with NaN
bit patterns (0xFF bytes) before the kernels run, and the results must be
bitwise those of a run on zero-filled buffers -- a kernel that reads a byte
it did not write first, or leaves an output element unwritten, fails."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2411_04844_b200 import core, device as D, loss, optim  # noqa: E402


def _fill(t, byte):
    t.view(torch.uint8).fill_(byte)


@pytest.mark.parametrize("dims", [(64, 48, 40), (40, 33, 19)])
@pytest.mark.parametrize("kernel", ["mma", "ff", "tc"])
def test_voxelizer_buffers(dims, kernel, monkeypatch):
    monkeypatch.setenv("SPLATCT_FWD_KERNEL", kernel)
    dev = D.require_cuda()
    box = core.BoxConfig.for_dims(17, dims)
    rng = np.random.default_rng(5)
    n = 700
    mu = np.stack([rng.uniform(-4, d + 4, n) for d in dims], 1)
    cloud = core.GaussianCloud(mu, rng.uniform(0.5, 2.5, n), rng.uniform(0, 1, n))
    params = D.cloud_to_params(cloud, dev)
    up = torch.randn((dims[1], dims[0], dims[2]), device=dev)
    res = []
    for byte in (0x00, 0xFF):
        plan = D.FvrPlan(n, dims, box.half, 0, dev)
        _fill(plan.ws, byte)
        vol = plan.new_volume()
        _fill(vol, byte)
        grads = torch.empty((5, n), dtype=torch.float64, device=dev)
        _fill(grads, byte)
        plan.bin(params)
        plan.forward(params, vol, masks=True)
        plain = plan.new_volume()
        _fill(plain, byte)
        plan.forward_plain(params, plain)
        plan.backward(params, up, grads, None)
        occ = plan.pixel_occupancy_words()
        cov = plan.footprint_coverage_words()
        torch.cuda.synchronize()
        res.append([x.clone() for x in (vol, plain, grads) if x is not None] +
                   [x.clone() for x in (occ, cov) if x is not None])
    for a, b in zip(*res):
        assert torch.equal(a.view(torch.uint8), b.view(torch.uint8))


def test_projector_and_loss_buffers():
    dev = D.require_cuda()
    w, h, c = 48, 40, 24
    geom = core.ScanGeometry.fan(20, 64, 1.3, 80.0, 60.0)
    op = D.ProjectorOperator(geom, w, h, 0.5, dev)
    g = torch.Generator(device="cpu").manual_seed(1)
    vol = torch.rand((h, w, c), generator=g).to(dev)
    y = torch.randn((20, 64, c), generator=g).to(dev)
    ref = torch.rand((20, 64, c), generator=g).to(dev)
    res = []
    for byte in (0x00, 0xFF):
        fwd = torch.empty((20, 64, c), device=dev)
        adj = torch.empty((h, w, c), device=dev)
        _fill(fwd, byte)
        _fill(adj, byte)
        op.forward(vol, fwd)
        op.adjoint(y, adj)
        lp = D.LossPlan(20, 64, c, dev)
        _fill(lp.ws, byte)
        gp = torch.empty_like(fwd)
        _fill(gp, byte)
        sums = torch.zeros(3, dtype=torch.float64, device=dev)
        lp.fused(fwd, ref, float(ref.max()), 0.6, 0.2, float(fwd.numel()), float(c), gp, sums)
        torch.cuda.synchronize()
        res.append([fwd.clone(), adj.clone(), gp.clone(), sums.clone()])
    for a, b in zip(*res):
        assert torch.equal(a.view(torch.uint8), b.view(torch.uint8))

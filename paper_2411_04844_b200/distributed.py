"""z-slab domain decomposition across the GPUs of one node.

For the per-slice parallel/fan geometries, sinogram slice z depends only on
volume slice z (_kernels.py:273-278), so each rank owns a contiguous z-slab
of the volume AND the same slices of the sinogram; projector, adjoint, L1
and SSIM are slab-local.  Exchanges per iteration:

  * all-reduce(sum) of the 3 loss sums (L1, SSIM, TV) -- bookkeeping only;
  * one xy-plane TV halo with each z-neighbour (the TV subgradient couples
    adjacent slices, loss.py:195-206);
  * all-reduce(sum) of the [5, N] partial gradient block, sent as f32 (a
    Gaussian whose box straddles a slab boundary gets contributions from two
    ranks; Adam is replicated, so every rank needs every gradient).

The halo exchange is posted at the start of the iteration (the planes come
from the previous iteration's splat) and completed after the adjoint, which
runs without halos; splatct_tv_halo_fixup then adds the two cross-boundary TV
terms, so the exchange overlaps the projector, the loss and the adjoint.

Cone beam ("partial projections summed"): rays cross slabs,
so each rank projects its slab into partial line integrals of the FULL
(m, nu, nv) sinogram; a reduce-scatter over detector-row bands completes them
and leaves each rank one band, on which it evaluates the projection loss
(SSIM windows lie inside a row's (view, column) image); an all-gather of
dL/dpred then gives every rank the full gradient sinogram to back-project
onto its own slab.  Same bytes as an all-reduce of the prediction, but the
loss runs once per band instead of replicated on every rank.

Adam then runs identically on every rank (replicated cloud).  The
communicator is written against torch.distributed and works for NCCL on
device tensors and for gloo on CPU tensors (tests/test_distributed.py).
"""

from __future__ import annotations

import os
import time

import numpy as np
import torch
import torch.distributed as dist

from .trainer import Slab


def slab_bounds(c: int, world: int, rank: int) -> Slab:
    """Contiguous, balanced split of c slices over world ranks."""
    base, rem = divmod(int(c), int(world))
    z0 = rank * base + min(rank, rem)
    cl = base + (1 if rank < rem else 0)
    return Slab(z0, cl, int(c))


class SlabComm:
    """Collectives of the z-slab decomposition over a torch.distributed group."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # gloo has no device-side point-to-point: stage halos through the host
        # (used to emulate ranks on one GPU in tests; NCCL stays on device)
        self.host_p2p = dist.get_backend(group) == "gloo"
        self._lo = None
        self._hi = None
        self._out_dev = None

    def _reduce(self, t: torch.Tensor, op) -> torch.Tensor:
        if self.host_p2p and t.is_cuda:
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op, group=self.group)
        return t

    def allreduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        return self._reduce(t, dist.ReduceOp.SUM)

    def allreduce_max_(self, t: torch.Tensor) -> torch.Tensor:
        return self._reduce(t, dist.ReduceOp.MAX)

    def halo(self, vol: torch.Tensor):
        """Exchange boundary z-planes of a (h, w, c_local) slab (blocking).

        Returns (lo, hi): plane z0-1 from rank-1 and plane z0+c_local from
        rank+1, each a contiguous (h*w,) tensor, or None at the volume edges.
        """
        self.halo_start(vol)
        return self.halo_wait()

    def halo_start(self, vol: torch.Tensor):
        """Post the boundary-plane exchange and return at once (NCCL runs it
        on its own stream, overlapping the projector, loss and adjoint that
        follow); halo_wait() completes it."""
        h, w, _ = vol.shape
        buf_dev = torch.device("cpu") if self.host_p2p else vol.device
        if self._lo is None or self._lo.numel() != h * w or self._out_dev != vol.device:
            self._out_dev = vol.device
            self._lo = torch.empty(h * w, dtype=vol.dtype, device=buf_dev)
            self._hi = torch.empty(h * w, dtype=vol.dtype, device=buf_dev)
            self._send_lo = torch.empty_like(self._lo)
            self._send_hi = torch.empty_like(self._lo)
            self._lo_dev = torch.empty(h * w, dtype=vol.dtype, device=vol.device)
            self._hi_dev = torch.empty(h * w, dtype=vol.dtype, device=vol.device)
        self._send_lo.copy_(vol[:, :, 0].reshape(-1))
        self._send_hi.copy_(vol[:, :, -1].reshape(-1))
        ops = []
        r, n = self.rank, self.world
        if r > 0:
            ops.append(dist.P2POp(dist.isend, self._send_lo, r - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, self._lo, r - 1, self.group))
        if r + 1 < n:
            ops.append(dist.P2POp(dist.isend, self._send_hi, r + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, self._hi, r + 1, self.group))
        self._reqs = dist.batch_isend_irecv(ops) if ops else []
        self._halo_cuda = vol.device.type == "cuda"

    def halo_wait(self):
        for req in self._reqs:
            req.wait()
        self._reqs = []
        lo, hi = self._lo, self._hi
        if self.host_p2p and self._halo_cuda:
            lo = self._lo_dev.copy_(self._lo)
            hi = self._hi_dev.copy_(self._hi)
        r, n = self.rank, self.world
        return (lo if r > 0 else None), (hi if r + 1 < n else None)

    def reduce_scatter_rows(self, pred: torch.Tensor, bands, out: torch.Tensor) -> torch.Tensor:
        """Cone beam: sum the ranks' partial projections (m, nu, nv) and leave
        rank r the rows bands[r] of the sum, out (m, nu, pb_r) -- each rank
        evaluates the loss on its own band instead of a replicated whole."""
        m, nu, _ = pred.shape
        pmax = max(r1 - r0 for r0, r1 in bands)
        key = (m, nu, pmax, str(pred.device))
        if getattr(self, "_rs_key", None) != key:
            self._rs_key = key
            dev = torch.device("cpu") if self.host_p2p else pred.device
            self._rs_in = torch.zeros((self.world, m, nu, pmax), dtype=pred.dtype, device=dev)
            self._rs_out = torch.zeros((m, nu, pmax), dtype=pred.dtype, device=dev)
            self._ag_in = torch.zeros((m, nu, pmax), dtype=pred.dtype, device=dev)
            self._ag_out = torch.zeros((self.world, m, nu, pmax), dtype=pred.dtype, device=dev)
        if self.host_p2p:
            _pack_rows(pred.cpu(), bands, self._rs_in)
        else:
            _pack_rows(pred, bands, self._rs_in)
        dist.reduce_scatter_tensor(self._rs_out.view(-1), self._rs_in.view(-1), group=self.group)
        r0, r1 = bands[self.rank]
        out.copy_(self._rs_out[:, :, : r1 - r0])
        return out

    def all_gather_rows(self, band: torch.Tensor, bands, out: torch.Tensor) -> torch.Tensor:
        """The inverse exchange: every rank's band (m, nu, pb_r) -> out (m, nu, nv)."""
        r0, r1 = bands[self.rank]
        self._ag_in[:, :, : r1 - r0].copy_(band)
        dist.all_gather_into_tensor(self._ag_out.view(-1), self._ag_in.view(-1), group=self.group)
        src = self._ag_out.to(out.device) if self.host_p2p else self._ag_out
        for g, (a, b) in enumerate(bands):
            if b > a:
                out[:, :, a:b].copy_(src[g, :, :, : b - a])
        return out

    def allreduce_grads_(self, g: torch.Tensor) -> torch.Tensor:
        """Sum the f64 [5, N] partial gradients over ranks, sent as f32 (half
        the bytes; the f32 partial sums keep ~1e-7 relative precision against
        the 1e-4 gradient tolerance)."""
        g32 = g.to(torch.float32)
        self._reduce(g32, dist.ReduceOp.SUM)
        g.copy_(g32)
        return g


def row_bands(nv: int, world: int):
    """Detector-row bands [r0, r1) of a cone sinogram, one per rank, starts on
    multiples of 4 where the row count allows (the 11 x 11 SSIM fast path
    wants a multiple-of-4 slice count); SSIM windows lie inside one row's
    (view, column) image, so bands are independent for the loss."""
    q = max(1, -(-int(nv) // int(world)))
    q = -(-q // 4) * 4 if nv >= 4 * world else q
    out = []
    for r in range(world):
        r0 = min(r * q, nv)
        out.append((r0, min(r0 + q, nv) if r + 1 < world else nv))
    return out


def _pack_rows(x, bands, buf):
    """x (m, nu, nv) -> buf (world, m, nu, pmax): band g of the rows, zero-padded."""
    for g, (r0, r1) in enumerate(bands):
        if r1 > r0:
            buf[g, :, :, : r1 - r0].copy_(x[:, :, r0:r1])
    return buf


def init_from_env(backend: str = "nccl"):
    """Initialise torch.distributed from torchrun's env (127.0.0.1 rendezvous)."""
    if dist.is_available() and not dist.is_initialized() and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # failure detection: a rank that dies or hangs in a
        # collective surfaces as an error on the others instead of a silent hang
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
        import datetime
        timeout = datetime.timedelta(seconds=int(os.environ.get("SPLATCT_PG_TIMEOUT_S", "600")))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local),
                                    timeout=timeout)
        else:
            dist.init_process_group(backend, timeout=timeout)
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


class _SlabEvaluator:
    """Per-iteration truth metrics and held-out view loss of a z-slab sharded
    run (optim._Evaluator across ranks): per-slab partial sums, all-reduced.

    PSNR: the slab's squared error against the truth slab; mean axial SSIM:
    the slab's slice images (SSIM is per slice, loss.py:159-180, so slabs are
    independent); held-out view L1 (optim.py:405-416): per-slice geometries
    project the slab onto the held-out views' slab slices, cone beam sums the
    slabs' partial projections first."""

    def __init__(self, tr, comm, truth, geom_val, sino_val, slab):
        from . import device as D
        dev = tr.device
        self.tr, self.comm, self.s = tr, comm, slab
        self.truth = None
        if truth is not None:
            z = np.ascontiguousarray(truth.zyx[slab.z0:slab.z0 + slab.c_local])
            self.truth = D.zyx_to_yxz(z, dev)
            self.peak = float(truth.data.max())
            w, h, c = truth.dims
            self.n_vox = float(w * h * c)
            self.c_global = c
            self.ssim_plan = D.LossPlan(h, w, slab.c_local, dev)
            self.scratch = torch.empty_like(self.truth)
            self.sums = torch.zeros(3, dtype=torch.float64, device=dev)
        self.val = geom_val is not None
        if self.val:
            w, h = tr.w, tr.h
            views = sino_val.views
            if geom_val.per_slice:
                self.val_op = D.ProjectorOperator(geom_val, w, h, 0.5, dev)
                views = views[:, :, slab.z0:slab.z0 + slab.c_local]
            else:
                self.val_op = D.ConeOperator(geom_val, w, h, slab.c_global, 0.5, dev)
            self.per_slice = geom_val.per_slice
            self.val_ref = D.sino_to_device(np.ascontiguousarray(views), dev)
            m, n, p = self.val_ref.shape
            self.val_plan = D.LossPlan(m, n, p, dev)
            self.val_pred = torch.empty((m, n, p), dtype=torch.float32, device=dev)
            self.val_g = torch.empty_like(self.val_pred)
            self.val_sums = torch.zeros(3, dtype=torch.float64, device=dev)
            self.val_count = float(sino_val.views.size)

    def metrics(self):
        from . import device as D
        if self.truth is None:
            return float("nan"), float("nan")
        vol = self.tr.vol
        part = torch.zeros(2, dtype=torch.float64, device=vol.device)
        part[0] = D.sum_sq_diff(vol, self.truth)
        p = self.ssim_plan
        p.fused(vol, self.truth, self.peak, 0.0, 1.0, 1.0, 1.0, self.scratch, self.sums)
        part[1] = self.sums[1]
        self.comm.allreduce_sum_(part)
        mse = float(part[0]) / self.n_vox
        psnr = 200.0 if mse == 0.0 else min(10.0 * np.log10(self.peak ** 2 / mse), 200.0)
        return psnr, float(part[1]) / p.valid / self.c_global

    def val_loss(self):
        self.val_op.forward(self.tr.vol, self.val_pred, z0=self.s.z0)
        if not self.per_slice:   # partial line integrals of every slab
            self.comm.allreduce_sum_(self.val_pred)
        self.val_plan.fused(self.val_pred, self.val_ref, 1.0, 1.0, 0.0, 1.0, 1.0, self.val_g,
                            self.val_sums)
        part = self.val_sums[0:1].clone()
        if self.per_slice:
            self.comm.allreduce_sum_(part)
        return float(part.item()) / self.val_count


def run_reconstruction_sharded(measured, geom, settings, init_cloud, comm=None,
                               use_graph: bool = True, truth=None):
    """run_reconstruction (optim.py:286-427) over a z-slab-sharded volume.

    Every rank calls this with the same host inputs; rank r keeps slices
    slab_bounds(c, world, r) of the volume (and of the measured sinogram for
    the per-slice geometries).  The loop body is the reference's: the sharded
    iteration (Trainer), densification on its interval (the cloud and the
    all-reduced gradient statistics are replicated, so every rank runs the
    identical device event with the same rng), per-iteration truth metrics
    (PSNR, mean axial SSIM) and the held-out-view stop rule, both from
    all-reduced slab partial sums.  Returns (VolumeGrid on rank 0 else None,
    GaussianCloud, list[TraceRow]).
    """
    from . import device as D
    from .core import ValidationError, VolumeGrid
    from .optim import DensifyParams, TraceRow, _holdout_split
    from .trainer import Trainer

    if comm is None:
        from .trainer import NullComm
        comm = SlabComm() if dist.is_available() and dist.is_initialized() else NullComm()
    dims = tuple(int(v) for v in settings.dims)
    box = settings.box
    s = slab_bounds(dims[2], comm.world, comm.rank)
    dev = D.require_cuda()
    if settings.stop_rule == "val-convergence":
        (geom_tr, sino_tr), (geom_val, sino_val) = _holdout_split(geom, measured,
                                                                  settings.holdout_fraction)
    elif settings.stop_rule == "iters":
        geom_tr, sino_tr, geom_val, sino_val = geom, measured, None, None
    else:
        raise ValidationError(f"unknown stop rule {settings.stop_rule!r}")
    # per-slice geometries: the rank's sinogram slab; cone beam: the full
    # sinogram on every rank (partial projections are summed in the Trainer)
    local = (np.ascontiguousarray(sino_tr.views[:, :, s.z0:s.z0 + s.c_local])
             if geom.per_slice else np.ascontiguousarray(sino_tr.views))
    tr = Trainer(D.sino_to_device(local, dev), geom_tr, dims, box, settings.weights,
                 D.cloud_to_params(init_cloud, dev), lr0=settings.lr_initial,
                 lrf=settings.lr_final, max_iters=settings.max_iters, slab=s, comm=comm,
                 trace_cap=max(settings.max_iters, 1))
    ev = _SlabEvaluator(tr, comm, truth, geom_val, sino_val, s)
    dparams = settings.densify or DensifyParams.for_volume(dims, box_size=box.extent)
    per_iter_host = truth is not None or geom_val is not None
    tr.initial_volume()
    trace = []
    best_val, best_it = np.inf, 0
    t_start = time.perf_counter()
    iters_acc = 0
    pending = []

    def flush():
        torch.cuda.current_stream().synchronize()
        rows = tr.trace.cpu().numpy()
        halted = tr.halted()
        out = []
        for idx, wall in pending:
            r = rows[idx]
            if halted and not np.isfinite(r[0]):
                raise RuntimeError(f"non-finite loss at iteration {idx}")
            out.append(TraceRow(iteration=idx + 1, loss=float(r[0]), loss_l1=float(r[1]),
                                loss_ssim=float(r[2]), loss_tv=float(r[3]), psnr=float("nan"),
                                ssim=float("nan"), n_gaussians=tr.N, wall_seconds=wall))
        pending.clear()
        return out

    it = 0
    captured = False
    while it < settings.max_iters:
        densify_due = (settings.densify_interval > 0 and (it + 1) % settings.densify_interval == 0
                       and it + 1 < settings.max_iters)
        if use_graph and not captured and not densify_due:
            # one graph per iteration on a single rank; with ranks, graphs for the
            # GPU segments between the (eager) slab collectives -- both execute `it`
            tr.capture() if comm.world == 1 else tr.capture_segments()
            captured = True
        else:
            tr.step()
        pending.append((it, time.perf_counter() - t_start))
        iters_acc += 1
        if densify_due or per_iter_host or it + 1 == settings.max_iters:
            rows = flush()
            row = rows[-1]
            trace.extend(rows[:-1])
            if densify_due:   # the identical device event on every rank (replicated cloud)
                rng = np.random.default_rng([settings.seed, it + 1])
                np_, nm1, nm2, report = D.densify(tr.params, tr.m1, tr.m2, tr.accum, iters_acc,
                                                  dparams, rng)
                if report.n_after == 0:
                    raise ValidationError("cloud is empty (densification pruned every Gaussian)")
                tr.resize(np_, nm1, nm2, None)
                captured = False
                iters_acc = 0
                row.clones, row.splits, row.prunes = report.clones, report.splits, report.prunes
                row.n_gaussians = report.n_after
            if truth is not None:
                row.psnr, row.ssim = ev.metrics()
            stop = False
            if geom_val is not None:
                val = ev.val_loss()
                row.val_loss = val
                if val < best_val - 1e-9:
                    best_val, best_it = val, it + 1
                elif it + 1 - best_it >= settings.patience:
                    stop = True
            trace.append(row)
            if stop:
                break
        it += 1
    if pending:
        trace.extend(flush())
    cmax = -(-dims[2] // comm.world)
    pad = torch.zeros((tr.h, tr.w, cmax), dtype=torch.float32, device=dev)
    pad[:, :, : s.c_local] = tr.vol
    parts = [torch.empty_like(pad) for _ in range(comm.world)] if comm.world > 1 else [pad]
    if comm.world > 1:
        if comm.host_p2p:
            hp = [torch.empty_like(pad, device="cpu") for _ in range(comm.world)]
            dist.all_gather(hp, pad.cpu(), group=comm.group)
            parts = [t.to(dev) for t in hp]
        else:
            dist.all_gather(parts, pad, group=comm.group)
    vol = None
    if comm.rank == 0:
        cols = [parts[r][:, :, : slab_bounds(dims[2], comm.world, r).c_local]
                for r in range(comm.world)]
        vol = VolumeGrid.from_zyx(D.yxz_to_zyx(torch.cat(cols, dim=2)))
    return vol, D.params_to_cloud(tr.params), trace

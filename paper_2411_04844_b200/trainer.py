"""Device-resident training iteration (the body of optim.run_reconstruction).

One iteration in the reference order (optim.py:350-403):

  1. pred  = A vol                         projector.forward_project   (proj.cu)
  2. L1 + SSIM value and dL/dpred (f32)    loss.l1_loss/ssim_loss     (loss.cu)
  3. dl_dvol = f32(A^T dL/dpred + l3 dTV)  projector.back_project + loss.tv_loss (proj.cu)
  4. loss bookkeeping, non-finite guard, Adam scalars (optim.py:356-366, 88-90)
  5. grads = splat adjoint(dl_dvol)        fvr.backward               (fvr.cu)
  6. Adam step + clamps                    optim.adam_step            (loss.cu)
  7. bins + vol = splat(params)            fvr.reconstruct            (fvr.cu)

Everything stays in HBM; no host synchronisation inside an iteration, so a
single-GPU iteration is captured once as a CUDA graph and replayed.  Under
z-slab sharding (distributed.py) each rank owns slices [z0, z0+c_local) of
the volume and the sinogram; the only exchanges are the loss sums and the
gradient all-reduce plus a one-plane TV halo.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import torch

from . import device as D
from .core import BoxConfig, ScanGeometry

SIGMA_FLOOR = 0.3
# the step bins with each tile's list ordered by first footprint row, so the
# forward's warps skip more k8 steps (SPLATCT_ROW_ORDER=0: canonical lists;
# measurement knob)
ROW_ORDERED_BINS = os.environ.get("SPLATCT_ROW_ORDER", "1") != "0"


def _capture_graph(device, fn) -> torch.cuda.CUDAGraph:
    """Capture fn's launches as a CUDA graph on a side stream.  Unlike the
    torch.cuda.graph context manager this skips gc.collect() and
    torch.cuda.empty_cache() around the capture: the latter hands every cached
    block back to the driver, so the allocations that follow in a first call
    pay cudaMalloc again (together ~9 ms of a cold C2 call)."""
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(device=device)
    side.wait_stream(torch.cuda.current_stream(device))
    with torch.cuda.stream(side):
        g.capture_begin()
        try:
            fn()
        finally:
            g.capture_end()
    torch.cuda.current_stream(device).wait_stream(side)
    return g


def adam_schedule(lr0: float, lrf: float, max_iters: int) -> list:
    """[lr, 1 - 0.9^t, 1 - 0.999^t] for pre-increment steps 0..max_iters, with
    Python float arithmetic as in the reference (optim.py:88-90, 123-126)."""
    T = max(int(max_iters), 1)
    rows = []
    for s in range(int(max_iters) + 1):
        rows.append([lr0 * (lrf / lr0) ** (min(s, max_iters) / T), 1.0 - 0.9 ** (s + 1),
                     1.0 - 0.999 ** (s + 1)])
    return rows


@dataclass
class Slab:
    """The z-range [z0, z0 + c_local) of a c_global-slice volume owned by a rank."""

    z0: int
    c_local: int
    c_global: int


class NullComm:
    """Single-device communicator (no-ops)."""

    rank = 0
    world = 1

    def allreduce_sum_(self, t):
        return t

    def allreduce_max_(self, t):
        return t

    def halo(self, vol):
        return None, None

    def halo_start(self, vol):
        pass

    def halo_wait(self):
        return None, None

    def allreduce_grads_(self, g):
        return g


class Trainer:
    """The training loop state on one device (one z-slab when sharded)."""

    def __init__(self, measured: torch.Tensor, geom: ScanGeometry, dims, box: BoxConfig,
                 weights, params: torch.Tensor, *, m1=None, m2=None, step: int = 0,
                 accum=None, lr0: float = 3e-4, lrf: float = 3e-5, max_iters: int = 1000,
                 slab: Slab | None = None, comm=None, trace_cap: int | None = None,
                 step_length: float = 0.5):
        self.device = D.require_cuda(measured.device)
        self.geom = geom
        self.w, self.h, self.c = (int(v) for v in dims)
        self.box = box
        self.weights = weights
        self.slab = slab or Slab(0, self.c, self.c)
        self.comm = comm or NullComm()
        self.lr0, self.lrf, self.max_iters = float(lr0), float(lrf), int(max_iters)
        self.sigma_ceiling = 3.0 * box.extent
        m, n, p = (int(v) for v in measured.shape)
        # per-slice geometries: the rank's sinogram slab mirrors its volume
        # slab; cone beam: every rank holds the full (m, nu, nv) sinogram and
        # its slab's projections are partial line integrals summed across
        # ranks (the north star's partial-projection reduction)
        self.per_slice = geom.per_slice
        cl = self.slab.c_local
        if self.per_slice and p != cl:
            raise ValueError(f"measured slab has {p} slices, slab owns {cl}")
        if not self.per_slice and p != geom.n_rows:
            raise ValueError(f"cone sinogram has {p} rows, geometry has {geom.n_rows}")
        self.p_global = self.slab.c_global if self.per_slice else p
        self.m, self.n = m, n
        self.meas = measured
        dev = self.device
        self.op = D.operator_for(geom, self.w, self.h, self.slab.c_global, step_length, dev)
        self.pred = torch.empty((m, n, p), dtype=torch.float32, device=dev)
        self.gpred = torch.empty_like(self.pred)
        # cone beam across ranks: the loss runs on this rank's detector-row band
        # (reduce-scatter of the partial projections, all-gather of dL/dpred)
        self.bands = None
        if not self.per_slice and self.comm.world > 1:
            from .distributed import row_bands
            self.bands = row_bands(p, self.comm.world)
            r0, r1 = self.bands[self.comm.rank]
            self.meas_band = measured[:, :, r0:r1].contiguous()
            self.pred_band = torch.empty_like(self.meas_band)
            self.gpred_band = torch.empty_like(self.meas_band)
            self.loss = D.LossPlan(m, n, r1 - r0, dev) if r1 > r0 else None
            if self.loss is not None:
                self.loss.prepare(self.meas_band)
        else:
            self.loss = D.LossPlan(m, n, p, dev)
            self.loss.prepare(measured)   # the measured sinogram is constant over a run
        self.vol = torch.empty((self.h, self.w, cl), dtype=torch.float32, device=dev)
        self.dl = torch.empty_like(self.vol)
        self.tv_part = torch.zeros(D.tv_partial_len(self.w, self.h, cl), dtype=torch.float64,
                                   device=dev)
        self.sums = torch.zeros(3, dtype=torch.float64, device=dev)
        self.fin_scratch = torch.zeros(97, dtype=torch.float64, device=dev)   # SPLATCT_FIN_SCRATCH_DOUBLES
        # the Adam scalars per pre-increment step, computed like the reference
        # on the host (optim.py:88-90, 123-126): the finalize looks them up
        self.adam_sched = torch.tensor(adam_schedule(self.lr0, self.lrf, self.max_iters),
                                       dtype=torch.float64, device=dev)
        self.adam_s = torch.zeros(3, dtype=torch.float64, device=dev)
        self.step_t = torch.tensor([int(step)], dtype=torch.int64, device=dev)
        self.iter_t = torch.zeros(1, dtype=torch.int64, device=dev)
        self.halt = torch.zeros(1, dtype=torch.int32, device=dev)
        self.trace_cap = int(trace_cap if trace_cap is not None else max_iters)
        self.trace = torch.full((max(self.trace_cap, 1), 4), math.nan, dtype=torch.float64,
                                device=dev)
        lm = torch.tensor([D.sino_max(measured)], dtype=torch.float64, device=dev)
        self.comm.allreduce_max_(lm)
        self.lmax = float(lm.item())
        cg = self.slab.c_global
        self.l1_count = float(m * n * self.p_global)
        self.ssim_count = float(D.ssim_valid(m, n) * self.p_global)
        self.tv_count = float(self.w * self.h * cg)
        self.graph = None
        self._set_params(params, m1, m2, accum)

    # -- state ------------------------------------------------------------
    def _set_params(self, params, m1=None, m2=None, accum=None):
        dev = self.device
        self.params = params.to(dev, torch.float64).contiguous()
        nG = int(self.params.shape[1])
        self.N = nG
        self.m1 = (m1.to(dev, torch.float64).contiguous() if m1 is not None
                   else torch.zeros_like(self.params))
        self.m2 = (m2.to(dev, torch.float64).contiguous() if m2 is not None
                   else torch.zeros_like(self.params))
        self.grads = torch.zeros_like(self.params)
        self.accum = (accum.to(dev, torch.float64).contiguous() if accum is not None
                      else torch.zeros(nG, dtype=torch.float64, device=dev))
        s = self.slab
        self.fvr = D.FvrPlan(nG, (self.w, self.h, s.c_local), self.box.half, s.z0, dev)
        self.graph = None
        self.segments = None

    def reload(self, measured, params, m1=None, m2=None, step: int = 0, accum=None):
        """Re-initialise the state in place (same shapes and lmax).

        Every buffer keeps its address, so a captured CUDA graph stays valid
        and the next run replays it without re-capture (optim's trainer cache).
        """
        if tuple(measured.shape) != tuple(self.meas.shape) or \
                tuple(params.shape) != tuple(self.params.shape):
            raise ValueError("reload needs the same sinogram and cloud shapes")
        self.meas.copy_(measured)
        if self.bands is not None:
            r0, r1 = self.bands[self.comm.rank]
            self.meas_band.copy_(measured[:, :, r0:r1])
            if self.loss is not None:
                self.loss.prepare(self.meas_band)
        else:
            self.loss.prepare(self.meas)
        self.params.copy_(params)
        if m1 is None:
            self.m1.zero_()
        else:
            self.m1.copy_(m1)
        if m2 is None:
            self.m2.zero_()
        else:
            self.m2.copy_(m2)
        self.grads.zero_()
        if accum is None:
            self.accum.zero_()
        else:
            self.accum.copy_(accum)
        self.step_t.fill_(int(step))
        self.iter_t.zero_()
        self.halt.zero_()
        self.trace.fill_(math.nan)

    def resize(self, params, m1, m2, accum=None):
        """Replace the cloud (densification changes N); drops the captured graph."""
        self._set_params(params, m1, m2, accum)
        self.initial_volume()

    # -- iteration ----------------------------------------------------------
    def initial_volume(self):
        self.fvr.bin(self.params, self.halt, row_ordered=ROW_ORDERED_BINS)
        self.fvr.forward(self.params, self.vol, self.halt, masks=True)

    def _stages(self):
        """The iteration as an ordered list of ("gpu" | "comm", fn) stages.

        GPU stages are stream-ordered kernel launches (graph-capturable); comm
        stages are the slab collectives, which run eagerly between captured
        segments when the job is sharded (capture_segments)."""
        lw = self.weights
        halt = self.halt
        z0 = self.slab.z0
        sharded = self.comm.world > 1
        replicated = not self.per_slice and sharded
        st = []
        overlap_halo = sharded and lw.lambda3 > 0
        if overlap_halo:   # planes of the previous splat; completed after the adjoint
            st.append(("comm", lambda: self.comm.halo_start(self.vol)))

        def project():   # empty-space skipping from the voxelizer's tile occupancy
            self.op.forward(self.vol, self.pred, halt, z0=z0, occ=self.fvr)
        st.append(("gpu", project))
        if replicated:   # partial cone projections -> this rank's row band of their sum
            st.append(("comm", lambda: self.comm.reduce_scatter_rows(self.pred, self.bands,
                                                                     self.pred_band)))

        # single device: the loss and TV sums stay block partials that the
        # iteration's finalize reduces (three reduction launches saved)
        fused_loss = (lw.lambda1 > 0 or lw.lambda2 > 0) and self.loss is not None
        defer = not sharded and fused_loss and self.loss.prepared_ref == self.meas.data_ptr()
        tv_blocked = getattr(self.op, "blocked", False)
        defer_tv = not sharded and lw.lambda3 > 0 and tv_blocked

        def data_loss():
            pred, meas, gpred = ((self.pred_band, self.meas_band, self.gpred_band) if replicated
                                 else (self.pred, self.meas, self.gpred))
            if fused_loss:
                self.loss.fused(pred, meas, self.lmax, lw.lambda1, lw.lambda2, self.l1_count,
                                float(self.p_global), gpred, self.sums, halt, defer=defer)
            else:
                gpred.zero_()
                self.sums[0:2].zero_()
        st.append(("gpu", data_loss))
        if replicated:   # every rank back-projects the full dL/dpred onto its slab
            st.append(("comm", lambda: self.comm.all_gather_rows(self.gpred_band, self.bands,
                                                                 self.gpred)))
        if lw.lambda3 > 0:
            def adjoint_tv():
                # dl is read only inside footprints: skip empty neighbourhoods.
                # Sharded: no halos here -- the cross-slab TV terms are added by
                # the fix-up once the (overlapped) exchange completes
                self.op.adjoint(self.gpred, self.dl, vol=self.vol, lambda_tv=lw.lambda3,
                                tv_count=self.tv_count, tv_partial=self.tv_part, halt=halt,
                                z0=z0, occ=self.fvr)
                if not defer_tv:
                    D.reduce_sum(self.tv_part, self.sums[2:3])
            st.append(("gpu", adjoint_tv))
            if overlap_halo:
                def halo_wait():
                    self._halo = self.comm.halo_wait()
                st.append(("comm", halo_wait))

                def tv_fixup():
                    lo, hi = self._halo
                    D.tv_halo_fixup(self.vol, self.dl, lo, hi, lw.lambda3, self.tv_count,
                                    self.sums[2:3], halt)
                st.append(("gpu", tv_fixup))
        else:
            st.append(("gpu", lambda: self.op.adjoint(self.gpred, self.dl, halt=halt, z0=z0,
                                                      c_local=self.slab.c_local,
                                                      occ=self.fvr)))
        if sharded:
            st.append(("comm", lambda: self.comm.allreduce_sum_(self.sums)))

        parts = None
        if defer or defer_tv:
            l1p, nl1, ssp, nss = (self.loss.partials(lw.lambda2) if defer
                                  else (D.VP(0), 0, D.VP(0), 0))
            tvn = D.tv_partial_len(self.w, self.h, self.slab.c_local, blocked=True)
            parts = (l1p, nl1, ssp, nss, D.ptr(self.tv_part) if defer_tv else D.VP(0),
                     tvn if defer_tv else 0, D.ptr(self.fin_scratch), D.ptr(self.adam_sched),
                     int(self.adam_sched.shape[0]))

        def finalize_backward():
            scal = (float(lw.lambda1), float(lw.lambda2), float(lw.lambda3), self.l1_count,
                    self.ssim_count, self.tv_count, self.lr0, self.lrf, self.max_iters,
                    D.ptr(self.step_t), D.ptr(self.iter_t), D.ptr(self.trace), self.trace_cap,
                    D.ptr(self.adam_s), D.ptr(halt), D.stream_handle())
            if parts is not None:
                D.call("splatct_iter_finalize_partials", D.ptr(self.sums), *parts, *scal)
            else:
                D.call("splatct_iter_finalize", D.ptr(self.sums), *scal)
            self.fvr.backward(self.params, self.dl, self.grads,
                              None if sharded else self.accum, halt)
        st.append(("gpu", finalize_backward))
        if sharded:
            st.append(("comm", lambda: self.comm.allreduce_grads_(self.grads)))

        def update_resplat():
            if sharded:
                D.grad_norm_accum(self.grads, self.accum, halt)
            # Adam fused into the binning pass of the updated params
            self.fvr.adam_bin(self.params, self.grads, self.m1, self.m2, self.adam_s, SIGMA_FLOOR,
                              self.sigma_ceiling, halt, row_ordered=ROW_ORDERED_BINS)
            self.fvr.forward(self.params, self.vol, halt, masks=True)   # + empty-space masks
        st.append(("gpu", update_resplat))
        return st

    def iteration(self):
        # NVTX ranges name every stage in an nsys / ncu timeline; a
        # captured graph keeps only the kernels, its replay gets one range
        for kind, fn in self._stages():
            torch.cuda.nvtx.range_push(f"{kind}:{fn.__name__}")
            fn()
            torch.cuda.nvtx.range_pop()

    def capture(self):
        """Capture one iteration as a CUDA graph (runs one real iteration first)."""
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.iteration()
        torch.cuda.current_stream().wait_stream(side)
        self.graph = _capture_graph(self.device, self.iteration)
        return 1   # iterations executed

    def capture_segments(self):
        """Sharded jobs: capture the runs of GPU stages between collectives as
        CUDA graphs and keep the collectives eager (runs one real iteration
        first).  A step is then a few graph launches interleaved with the
        slab collectives instead of ~30 kernel launches."""
        stages = self._stages()
        self.iteration()
        torch.cuda.synchronize(self.device)
        plan, run = [], []

        def flush():
            if run:
                plan.append(("graph", _capture_graph(self.device,
                                                     lambda run=run: [fn() for fn in run])))
                run.clear()
        for kind, fn in stages:
            if kind == "gpu":
                run.append(fn)
            else:
                flush()
                plan.append(("comm", fn))
        flush()
        self.segments = plan
        return 1

    def step(self):
        if self.graph is not None:
            torch.cuda.nvtx.range_push("iteration (graph)")
            self.graph.replay()
            torch.cuda.nvtx.range_pop()
        elif getattr(self, "segments", None):
            for kind, x in self.segments:
                if kind == "graph":
                    x.replay()
                else:
                    x()
        else:
            self.iteration()

    # -- readback -----------------------------------------------------------
    def halted(self) -> bool:
        return bool(self.halt.item())

    def iterations_done(self) -> int:
        return int(self.iter_t.item())

    def trace_rows(self, upto: int | None = None):
        k = self.iterations_done() if upto is None else upto
        if self.halted():
            k = min(k + 1, self.trace_cap)
        return self.trace[:k].cpu().numpy()

"""Device-resident building blocks over the libsplatct C ABI.

PyTorch is used only for device memory, streams and collectives; all
arithmetic on the hot path runs in the hand-written sm_100a kernels of
``csrc/`` (called through ``_lib``).  There is no CPU fallback: every class
here requires a CUDA device and raises otherwise.

Layouts (include/splatct.h):
  params / grads / Adam moments  float64 [5, N]  (mu_x, mu_y, mu_z, sigma, I)
  volume                         float32 [h, w, c]  ("yxz", slice fastest)
  sinogram                       float32 [m, n, p]  (reference layout)
"""

from __future__ import annotations

import ctypes
import os
from collections import OrderedDict

import numpy as np
import torch

from . import _lib
from ._lib import call, size_query
from .core import GaussianCloud, ScanGeometry

VP = ctypes.c_void_p


def ptr(t) -> VP:
    return VP(0 if t is None else t.data_ptr())


def stream_handle(stream=None) -> VP:
    s = stream if stream is not None else torch.cuda.current_stream()
    return VP(s.cuda_stream)


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "splatct B200 path needs a CUDA device; there is no CPU fallback "
            "(the CPU restatement in oracle/ is test infrastructure only)")
    _lib.load()
    dev = torch.device(device if device is not None else "cuda")
    if dev.type != "cuda":
        raise RuntimeError(f"splatct kernels run on CUDA devices only, got {dev}")
    return dev


# ---------------------------------------------------------------------------
# conversions at the API edge
# ---------------------------------------------------------------------------

def cloud_to_params(cloud: GaussianCloud, device) -> torch.Tensor:
    """Host cloud -> the device's f64 [5, N] block.  The (N, 3) -> (3, N)
    transpose runs on the device: on the host it is a strided copy (~0.4 ms
    at 50 k Gaussians), the packed upload is three contiguous copies."""
    n = cloud.n
    st = _pinned(5 * n, torch.float64)   # packed in page-locked memory: one DMA
    h = st.numpy()
    h[: 3 * n] = cloud.mu.reshape(-1)
    h[3 * n: 4 * n] = cloud.sigma
    h[4 * n:] = cloud.intensity
    d = st.to(device, non_blocking=False)
    p = torch.empty((5, n), dtype=torch.float64, device=d.device)
    p[0:3].copy_(d[: 3 * n].view(n, 3).t())
    p[3:5].copy_(d[3 * n:].view(2, n))
    return p


def params_to_host(params: torch.Tensor) -> np.ndarray:
    """The device [5, N] block as one packed host array [mu (N, 3) | sigma | I],
    transposed on the device (one download)."""
    p = params.detach()
    return to_host(torch.cat([p[0:3].t().reshape(-1), p[3], p[4]]))


def cloud_from_host(h: np.ndarray) -> GaussianCloud:
    """A GaussianCloud viewing a params_to_host array."""
    n = h.size // 5
    return GaussianCloud(h[: 3 * n].reshape(n, 3), h[3 * n: 4 * n], h[4 * n:])


class CloudDownload:
    """params_to_host queued on the current stream (into the cached page-locked
    buffer) without waiting; cloud() waits for it and builds the GaussianCloud."""

    def __init__(self, params: torch.Tensor):
        p = params.detach()
        packed = torch.cat([p[0:3].t().reshape(-1), p[3], p[4]])
        self.st = _pinned(packed.numel(), packed.dtype)
        self.st.copy_(packed, non_blocking=True)
        self.ev = torch.cuda.Event()
        self.ev.record(torch.cuda.current_stream(p.device))

    def cloud(self) -> GaussianCloud:
        self.ev.synchronize()
        return cloud_from_host(self.st.numpy().copy())


def params_to_cloud(params: torch.Tensor) -> GaussianCloud:
    """The inverse of cloud_to_params."""
    return cloud_from_host(params_to_host(params))


def _host_f32(arr) -> torch.Tensor:
    a = np.ascontiguousarray(arr, dtype=np.float32)
    if not a.flags.writeable:   # value objects are frozen; torch wants writable memory
        a = a.copy()
    return torch.from_numpy(a)


def zyx_to_yxz(arr, device) -> torch.Tensor:
    """(c, h, w) host array -> (h, w, c) device tensor."""
    return _host_f32(arr).to(device).permute(1, 2, 0).contiguous()


_PINNED: dict = {}


def _pinned(numel: int, dtype) -> torch.Tensor:
    """A cached page-locked staging buffer of at least numel elements (reused:
    cudaHostAlloc of tens of MB costs more than the copy it serves)."""
    buf = _PINNED.get(dtype)
    if buf is None or buf.numel() < numel:
        buf = torch.empty(max(numel, 1), dtype=dtype, pin_memory=True)
        _PINNED[dtype] = buf
    return buf[:numel]


class _PinnedSlot:
    """A page-locked host buffer handed out as a numpy array and taken back
    when every view of that array has been released."""

    def __init__(self, numel: int):
        self.t = torch.empty(numel, dtype=torch.float32, pin_memory=True)
        self.busy = False

    def release(self):
        self.busy = False


_OUT_POOL: list = []
_OUT_POOL_MAX = 2   # a caller keeping more results than this gets pageable arrays


def pinned_output(shape) -> np.ndarray | None:
    """A float32 host array of `shape` in page-locked memory from a small reusable
    pool, or None when every slot is still referenced.  A device->host copy
    lands in it at DMA speed (C2's 64 MB volume: 1.2 ms against ~3 ms through
    a staging buffer and a host copy, tools/pin_probe.py); the slot returns to
    the pool once the caller drops the array and all its views."""
    import weakref
    numel = int(np.prod(shape))
    if not any(e.t.numel() == numel for e in _OUT_POOL):
        # a new size: idle slots of other sizes go, and every slot of this size
        # is page-locked now, so a caller that keeps one result while computing
        # the next never pays cudaHostAlloc mid-run
        _OUT_POOL[:] = [e for e in _OUT_POOL if e.busy]
        _OUT_POOL.extend(_PinnedSlot(numel) for _ in range(_OUT_POOL_MAX))
    slot = next((e for e in _OUT_POOL if not e.busy and e.t.numel() == numel), None)
    if slot is None:
        if sum(e.busy for e in _OUT_POOL) >= _OUT_POOL_MAX:
            return None
        slot = _PinnedSlot(numel)
        _OUT_POOL.append(slot)
        while len(_OUT_POOL) > _OUT_POOL_MAX + 1:   # drop idle slots of other sizes
            idle = next((e for e in _OUT_POOL if not e.busy and e is not slot), None)
            if idle is None:
                break
            _OUT_POOL.remove(idle)
    slot.busy = True
    base = slot.t.numpy()
    weakref.finalize(base, slot.release)
    return base.reshape(shape)


def to_pinned_host(t: torch.Tensor, out: np.ndarray) -> np.ndarray:
    """Device tensor -> a pinned_output() array of the same shape (one DMA)."""
    torch.from_numpy(out).copy_(t.reshape(out.shape), non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return out


class HostArray:
    """A host array allocated and page-faulted on a background thread, so a
    later device->host copy into it runs at memcpy speed (fresh pages would
    otherwise be faulted in during the copy)."""

    def __init__(self, shape, dtype=np.float32):
        import threading
        self._out = None
        self._th = threading.Thread(target=self._alloc, args=(tuple(shape), dtype), daemon=True)
        self._th.start()

    def _alloc(self, shape, dtype):
        a = np.empty(shape, dtype)
        a.fill(0)
        self._out = a

    def get(self) -> np.ndarray:
        self._th.join()
        return self._out


_COPY_POOL = None


def _par_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """np.copyto split over host threads (numpy releases the GIL while it
    copies): one thread moves ~10 GB/s, the staging copies are tens of MB."""
    global _COPY_POOL
    n = dst.shape[0] if dst.ndim else 0
    if dst.nbytes < (8 << 20) or n < 2:
        np.copyto(dst, src, casting="same_kind")
        return
    if _COPY_POOL is None:
        import concurrent.futures
        import os
        _COPY_POOL = concurrent.futures.ThreadPoolExecutor(
            max_workers=max(1, min(8, (os.cpu_count() or 2) // 2)))
    k = min(_COPY_POOL._max_workers, n)
    cuts = np.linspace(0, n, k + 1).astype(int)
    futs = [_COPY_POOL.submit(np.copyto, dst[a:b], src[a:b], casting="same_kind")
            for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
    for f in futs:
        f.result()


def _chunks(n0: int, nbytes: int):
    """Row ranges for pipelined staging: ~4 chunks once a copy is >= 16 MB."""
    k = 4 if nbytes >= (16 << 20) and n0 >= 4 else 1
    cuts = np.linspace(0, n0, k + 1).astype(int)
    return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def to_host(t: torch.Tensor, out: np.ndarray | None = None) -> np.ndarray:
    """Device -> numpy via a cached pinned staging buffer (DMA-speed D2H).
    Large copies go in row chunks: the host copy of chunk i overlaps the DMA
    of chunk i + 1."""
    if t.device.type != "cuda":
        return t.numpy().copy()
    t = t.contiguous()
    st = _pinned(t.numel(), t.dtype).view(t.shape)
    sn = st.numpy()
    if out is None:
        out = np.empty(tuple(t.shape), sn.dtype)
    elif (out.shape != tuple(t.shape) or out.dtype != sn.dtype
          or not out.flags.c_contiguous or not out.flags.writeable):
        # a reshape of anything else would be a copy: the chunks would land in
        # a temporary and the caller's array would come back untouched
        raise ValueError(f"to_host: out must be a writeable C-contiguous {sn.dtype} array of "
                         f"shape {tuple(t.shape)}, got {out.dtype} {out.shape}")
    o = out
    if t.dim() == 0:
        st.copy_(t)
        np.copyto(o, sn)
        return out
    s = torch.cuda.current_stream(t.device)
    parts = []
    for a, b in _chunks(t.shape[0], t.numel() * t.element_size()):
        st[a:b].copy_(t[a:b], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(s)
        parts.append((a, b, ev))
    for a, b, ev in parts:
        ev.synchronize()
        _par_copy(o[a:b], sn[a:b])
    return out


def yxz_to_zyx(t: torch.Tensor, out: np.ndarray | None = None) -> np.ndarray:
    return to_host(t.permute(2, 0, 1).contiguous(), out)


_UPLOAD_STREAM: dict = {}
_UPLOAD_PIN: dict = {}


class StagedHost:
    """A host array uploaded by a helper thread while the caller prepares other
    inputs: splatct_stage_upload copies it into a page-locked buffer with
    several native threads and queues each slice's DMA as soon as the slice is
    written (ctypes releases the GIL for the call).  .to() makes the caller's
    stream wait for the upload and returns the device tensor."""

    def __init__(self, views, device):
        import threading
        self.a = np.ascontiguousarray(views, dtype=np.float32)
        self.dev = torch.device(device)
        st = _UPLOAD_PIN.get(self.dev)
        if st is None or st.numel() < self.a.size:   # its own buffer: DMAs outlive .to()
            st = _UPLOAD_PIN[self.dev] = torch.empty(max(self.a.size, 1), dtype=torch.float32,
                                                     pin_memory=True)
        self.st = st
        self.out = torch.empty(self.a.shape, dtype=torch.float32, device=self.dev)
        side = _UPLOAD_STREAM.get(self.dev)
        if side is None:
            side = _UPLOAD_STREAM[self.dev] = torch.cuda.Stream(device=self.dev)
        self.side = side
        self.side.wait_stream(torch.cuda.current_stream(self.dev))   # out's allocation
        self.done = torch.cuda.Event()
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()

    def _run(self):
        call("splatct_stage_upload", ptr(self.out), VP(self.a.ctypes.data), ptr(self.st),
             self.a.nbytes, 8, VP(self.side.cuda_stream))
        self.done.record(self.side)

    def to(self, device=None) -> torch.Tensor:
        self._th.join()
        torch.cuda.current_stream(self.dev).wait_event(self.done)
        return self.out


def sino_to_device(views, device) -> torch.Tensor:
    """(m, n, p) host array -> device f32 through the pinned staging buffer
    (a chunked, overlapped variant measured no faster: 2.7 vs 3.3 ms at C2)."""
    a = np.asarray(views)
    st = _pinned(a.size, torch.float32)
    _par_copy(st.numpy().reshape(a.shape), a)
    return st.view(a.shape).to(device, non_blocking=False)


# ---------------------------------------------------------------------------
# voxelizer
# ---------------------------------------------------------------------------

class FvrPlan:
    """Workspace + launches for the tiled voxelizer on a (w, h, c) slab at z0.

    fvr.reconstruct / fvr.backward (fvr.py:148-273) on device.
    """

    def __init__(self, n: int, dims, half, z0: int = 0, device=None):
        self.device = require_cuda(device)
        self.n = int(n)
        self.w, self.h, self.c = (int(v) for v in dims)
        self.hx, self.hy, self.hz = (int(v) for v in half)
        self.z0 = int(z0)
        self.ws_bytes = size_query("splatct_fvr_workspace_bytes", self.n, self.w, self.h, self.c,
                                   self.hx, self.hy, self.hz)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        # empty-space masks of the last forward (one word per pixel column):
        # value-based occupancy for the projector forwards, footprint coverage
        # for the adjoints (the backward reads every footprint voxel)
        none = ctypes.c_size_t(-1).value
        poff = size_query("splatct_fvr_pixel_occupancy_offset", self.n, self.w, self.h, self.c,
                          self.hx, self.hy, self.hz)
        foff = size_query("splatct_fvr_footprint_coverage_offset", self.n, self.w, self.h,
                          self.c, self.hx, self.hy, self.hz)
        self._pocc_off = None if poff == none else poff
        self._fcov_off = None if foff == none else foff
        self.pixel_occupancy = None if poff == none else VP(self.ws.data_ptr() + poff)
        self.footprint_coverage = None if foff == none else VP(self.ws.data_ptr() + foff)

    def _words(self, off):
        if off is None:
            return None
        return self.ws[off:off + 8 * self.w * self.h].view(torch.int64)

    def pixel_occupancy_words(self) -> torch.Tensor | None:
        """Pixel-column occupancy words, int64 [h * w] (a workspace view)."""
        return self._words(self._pocc_off)

    def footprint_coverage_words(self) -> torch.Tensor | None:
        """Pixel-column footprint coverage words, int64 [h * w] (a workspace view)."""
        return self._words(self._fcov_off)

    def _geo(self):
        return (self.n, self.w, self.h, self.c, self.z0, self.hx, self.hy, self.hz)

    masks_valid = False

    def adam_bin(self, params, grads, m1, m2, scalars, sigma_floor: float, sigma_ceiling: float,
                 halt=None, row_ordered: bool = False) -> None:
        """adam() then bin() of the updated params, in one pass (the training step)."""
        call("splatct_fvr_adam_bin", ptr(params), ptr(grads), ptr(m1), ptr(m2), ptr(scalars),
             float(sigma_floor), float(sigma_ceiling), *self._geo(), ptr(self.ws), self.ws_bytes,
             int(row_ordered), ptr(halt), stream_handle())

    def bin(self, params: torch.Tensor, halt=None, row_ordered: bool = False) -> None:
        """row_ordered: each tile's list ordered by the Gaussians' first row
        (same pairs; the forward skips more work, its sums change order)."""
        call("splatct_fvr_bin_row_ordered" if row_ordered else "splatct_fvr_bin", ptr(params),
             *self._geo(), ptr(self.ws), self.ws_bytes, ptr(halt), stream_handle())

    def forward(self, params: torch.Tensor, out: torch.Tensor, halt=None,
                masks: bool = False) -> torch.Tensor:
        """masks: also record the empty-space masks (pixel_occupancy,
        footprint_coverage) the training step's projector pair uses."""
        call("splatct_fvr_forward_masked" if masks else "splatct_fvr_forward", ptr(params),
             *self._geo(), ptr(self.ws), self.ws_bytes, ptr(out), ptr(halt), stream_handle())
        self.masks_valid = masks   # the masks describe the volume of the last forward
        return out

    def forward_plain(self, params: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """The non-decomposed splat on the current bins (splat_plain, _kernels.py:81-129)."""
        call("splatct_fvr_forward_plain", ptr(params), *self._geo(), ptr(self.ws), self.ws_bytes,
             ptr(out), stream_handle())
        return out

    def backward(self, params, upstream, grads, accum=None, halt=None) -> torch.Tensor:
        call("splatct_fvr_backward", ptr(params), *self._geo(), ptr(self.ws), self.ws_bytes,
             ptr(upstream), ptr(grads), ptr(accum), ptr(halt), stream_handle())
        return grads

    def new_volume(self) -> torch.Tensor:
        return torch.empty((self.h, self.w, self.c), dtype=torch.float32, device=self.device)

    def export_bins(self):
        """(fp int32 [n,6], tile_start int32 [T+1], items int32 [P]) on the host."""
        fp = torch.empty((max(self.n, 1), 6), dtype=torch.int32, device=self.device)
        np_ = ctypes.c_int64(0)
        nt = ctypes.c_int64(0)
        call("splatct_fvr_export_bins", ptr(self.ws), self.ws_bytes, self.n, self.w, self.h,
             self.c, self.hx, self.hy, self.hz, VP(0), VP(0), VP(0), ctypes.byref(np_),
             ctypes.byref(nt), stream_handle())
        ts = torch.empty(nt.value + 1, dtype=torch.int32, device=self.device)
        items = torch.empty(max(np_.value, 1), dtype=torch.int32, device=self.device)
        call("splatct_fvr_export_bins", ptr(self.ws), self.ws_bytes, self.n, self.w, self.h,
             self.c, self.hx, self.hy, self.hz, ptr(fp), ptr(ts), ptr(items), ctypes.byref(np_),
             ctypes.byref(nt), stream_handle())
        torch.cuda.current_stream().synchronize()
        return (fp[: self.n].cpu().numpy(), ts.cpu().numpy(),
                items[: np_.value].cpu().numpy())


# ---------------------------------------------------------------------------
# projector operator
# ---------------------------------------------------------------------------

# forward row groups: kind 0, aligned 4-ray groups (one z-column gather feeds 4
# rays).  Measured alternatives, kept in the ABI (SPLATCT_FWD_GROUPS=4|band8|
# band16 selects one; measurement knob):
#   kind 2, aligned 8-ray groups with w[8] per entry: 0.54 vs 0.37 ms at C2 --
#     twice the accumulators halve the resident warps, the zero-weight FMAs double;
#   kinds 3 / 4, bands of 8 / 16 rays whose entries are sliding 4-ray windows: a
#     pixel's z-column is gathered once per band (C2: 17 % fewer gathered bytes
#     for 8-ray bands), but 0.38 vs 0.25 ms -- half the warps with twice the
#     serial work each, and the L1 sharing between neighbouring groups' warps
#     (15 % hit rate) is lost.  A band's weights must fit the build kernel's
#     8192-entry group capacity (C2 rays carry up to ~700: 16-ray bands do not).
_BLOCK_CAP = 8192


def _forward_group_kind(max_row_nnz: int) -> int:
    force = os.environ.get("SPLATCT_FWD_GROUPS")
    if force:
        kind = {"4": 0, "band8": 3, "band16": 4}[force]
        if _group_rows(kind) * max_row_nnz > _BLOCK_CAP:
            raise ValueError(f"SPLATCT_FWD_GROUPS={force}: rays of up to {max_row_nnz} "
                             f"weights overflow a {_BLOCK_CAP}-entry band")
        return kind
    return 0


def _group_rows(kind: int) -> int:
    return {0: 4, 1: 4, 2: 8, 3: 8, 4: 16}[kind]


def _occ(occ, kind: str):
    """The mask an operator needs from `occ`: an FvrPlan (its value-based pixel
    occupancy for forwards, its footprint coverage for adjoints), a raw
    pointer, or None."""
    if occ is None or isinstance(occ, VP):
        return occ
    if not occ.masks_valid:   # the plan's last forward did not record masks: stay dense
        return None
    return occ.pixel_occupancy if kind == "pixel" else occ.footprint_coverage


class ProjectorOperator:
    """Exact per-slice projector A and adjoint A^T for one geometry.

    Built once by marching every ray in f64 (the reference's
    _ray_geometry/_clip_ray sample enumeration, _kernels.py:208-303) and
    merging sample weights per (ray, pixel); reused every iteration.
    """

    def __init__(self, geom: ScanGeometry, w: int, h: int, step: float = 0.5, device=None,
                 blocked: bool = True):
        self.device = require_cuda(device)
        geom.check_volume((w, h, 1))
        self.geom = geom
        self.w, self.h = int(w), int(h)
        self.m, self.n_det = int(geom.n_views), int(geom.n_detectors)
        self.step = float(step)
        self.is_fan = geom.variant == "fan"
        self.rs = float(geom.source_to_origin) if self.is_fan else 0.0
        self.rd = float(geom.origin_to_detector) if self.is_fan else 0.0
        self.spacing = float(geom.detector_spacing)
        ang = np.asarray(geom.view_angles, np.float64)
        self.cos_t = torch.from_numpy(np.cos(ang)).to(self.device)
        self.sin_t = torch.from_numpy(np.sin(ang)).to(self.device)
        rays = self.m * self.n_det
        self.n_rays = rays
        g = self._gargs()
        sb = size_query("splatct_proj_scratch_bytes", self.m, self.n_det, self.w, self.h, 0)
        scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
        self.a_ptr = torch.empty(rays + 1, dtype=torch.int64, device=self.device)
        nnz = ctypes.c_int64(0)
        call("splatct_proj_count", *g, ptr(self.a_ptr), ptr(scratch), sb, ctypes.byref(nnz),
             stream_handle())
        self.nnz = int(nnz.value)
        sb = size_query("splatct_proj_scratch_bytes", self.m, self.n_det, self.w, self.h,
                        self.nnz)
        scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
        k = max(self.nnz, 1)
        self.a_col = torch.empty(k, dtype=torch.int32, device=self.device)
        self.a_val = torch.empty(k, dtype=torch.float32, device=self.device)
        self.at_ptr = torch.empty(self.w * self.h + 1, dtype=torch.int64, device=self.device)
        self.at_ray = torch.empty(k, dtype=torch.int32, device=self.device)
        self.at_val = torch.empty(k, dtype=torch.float32, device=self.device)
        call("splatct_proj_fill", *g, ptr(self.a_ptr), ptr(self.a_col), ptr(self.a_val),
             ptr(self.at_ptr), ptr(self.at_ray), ptr(self.at_val), ptr(scratch), sb,
             stream_handle())
        del scratch
        self.blocked = blocked
        if blocked:
            # forward: 4-ray groups (one z-column load feeds 4 rays); adjoint: 2x2 quads
            max_nnz = int((self.a_ptr[1:] - self.a_ptr[:-1]).max().item()) if rays else 0
            self.fkind = _forward_group_kind(max_nnz)
            self.fb = self._block(self.a_ptr, self.a_col, self.a_val, self.n_rays, self.fkind,
                                  self._group_dirs(_group_rows(self.fkind))
                                  if self.fkind in (0, 2) else None)
            self.ab = self._block(self.at_ptr, self.at_ray, self.at_val, self.w * self.h, 1)

    def _group_dirs(self, rows: int = 4) -> torch.Tensor:
        """Unit direction of the middle ray of each ray group (march-order key)."""
        ng = (self.n_rays + rows - 1) // rows
        r = np.minimum(np.arange(ng) * rows + rows // 2, self.n_rays - 1)
        v, d = r // self.n_det, r % self.n_det
        ang = np.asarray(self.geom.view_angles, np.float64)[v]
        c, s = np.cos(ang), np.sin(ang)
        if self.is_fan:
            u = (d - 0.5 * (self.n_det - 1)) * self.spacing
            dx = (self.rd + self.rs) * c - u * s
            dy = (self.rd + self.rs) * s + u * c
            nrm = np.hypot(dx, dy)
            dx, dy = dx / nrm, dy / nrm
        else:
            dx, dy = c, s
        return torch.from_numpy(np.stack([dx, dy], 1).astype(np.float32)).to(self.device)

    def _block(self, ptr_, idx, val, nrows, kind, order_dir=None):
        """Blocked copy (gptr, gidx, gval[nb, 4 or 8]) of a CSR operator."""
        sb = size_query("splatct_proj_block_scratch_bytes", nrows, kind, self.w, self.h)
        scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
        group = _group_rows(kind)
        rows = 8 if kind == 2 else 4   # weights per entry
        ng = ((nrows + group - 1) // group if kind != 1
              else ((self.w + 1) // 2) * ((self.h + 1) // 2))
        gptr = torch.empty(ng + 1, dtype=torch.int64, device=self.device)
        nb = ctypes.c_int64(0)
        call("splatct_proj_block_count", ptr(ptr_), ptr(idx), nrows, kind, self.w, self.h,
             ptr(order_dir), ptr(gptr), ptr(scratch), sb, ctypes.byref(nb), stream_handle())
        k = max(int(nb.value), 1)
        gidx = torch.empty(k, dtype=torch.int32, device=self.device)
        gval = torch.empty((k, rows), dtype=torch.float32, device=self.device)
        call("splatct_proj_block_fill", ptr(ptr_), ptr(idx), ptr(val), nrows, kind, self.w,
             self.h, ptr(order_dir), ptr(gptr), ptr(gidx), ptr(gval), ptr(scratch), sb,
             stream_handle())
        return gptr, gidx, gval, int(nb.value)

    def _gargs(self):
        return (ptr(self.cos_t), ptr(self.sin_t), self.m, self.n_det, self.spacing, self.step,
                int(self.is_fan), self.rs, self.rd, self.w, self.h)

    def forward_entry_pixels(self) -> torch.Tensor:
        """Pixel index of every blocked forward entry (band entries carry their
        window's first ray in the top bits of the packed index)."""
        idx = self.fb[1]
        return (idx & 0x07FFFFFF) if self.fkind in (3, 4) else idx

    @property
    def matrix_bytes(self) -> int:
        b = 16 * self.nnz + 8 * (self.n_rays + self.w * self.h + 2)
        if self.blocked:
            b += 20 * (self.fb[3] + self.ab[3]) + 8 * (len(self.fb[0]) + len(self.ab[0]))
        return b

    def forward(self, vol: torch.Tensor, out: torch.Tensor | None = None, halt=None,
                blocked: bool | None = None, z0: int = 0, occ=None):
        """vol (h, w, c) -> sinogram (m, n, c); per-slice, so a slab's z0 is irrelevant.

        occ: the FvrPlan whose forward produced `vol` (or its pixel_occupancy
        pointer) -- entries in all-zero column segments are skipped (exact)."""
        c = int(vol.shape[2])
        if out is None:
            out = torch.empty((self.m, self.n_det, c), dtype=torch.float32, device=vol.device)
        occ = _occ(occ, "pixel")
        if self.blocked if blocked is None else blocked:
            g = self.fb
            call("splatct_proj_forward_blocked_ordered", ptr(g[0]), ptr(g[1]), ptr(g[2]),
                 self.n_rays, self.fkind, ptr(vol), ptr(out), c,
                 occ if occ is not None else VP(0), self.w, self.h,
                 ptr(self._forward_order(c)), ptr(halt), stream_handle())
        else:
            call("splatct_proj_forward", ptr(self.a_ptr), ptr(self.a_col), ptr(self.a_val),
                 self.n_rays, ptr(vol), ptr(out), c, ptr(halt), stream_handle())
        return out

    def _forward_order(self, c: int):
        """The blocked forward's CTAs, those with the longest warp task first
        (None: default order).  A CTA lasts as long as its longest (group,
        z-chunk) task, about its group's entry count; launching the long ones
        first leaves short ones for the grid's tail (C2: 0.229 -> 0.200 ms).
        Computed once per slice depth, outside any graph capture."""
        cache = self.__dict__.setdefault("_orders", {})
        if c in cache:
            return cache[c]
        if torch.cuda.is_current_stream_capturing():
            return None
        ctas, zs, ordered = ctypes.c_int64(0), ctypes.c_int(0), ctypes.c_int(0)
        call("splatct_proj_forward_ctas", self.n_rays, self.fkind, self.w, self.h, c,
             ctypes.byref(ctas), ctypes.byref(zs), ctypes.byref(ordered))
        order = None
        if ordered.value and ctas.value > 1:
            gptr = self.fb[0]
            work = gptr[1:] - gptr[:-1]
            ng, z, n = work.numel(), zs.value, ctas.value
            task = torch.arange(4 * n, device=self.device)   # CTA b: tasks 4b .. 4b + 3
            grp = task // z if ordered.value == 1 else task % ng
            wk = torch.where(task < ng * z, work[grp.clamp(max=ng - 1)], torch.zeros_like(task))
            key = -wk.view(n, 4).amax(1)
            if ordered.value == 2:   # z-chunk-major: longest first within each chunk
                chunk = task.view(n, 4)[:, 0] // ng
                key = key + chunk * (int(work.max().item()) + 1)
            order = torch.argsort(key, stable=True).to(torch.int32)
        cache[c] = order
        return order

    def adjoint(self, gsino: torch.Tensor, out: torch.Tensor | None = None, vol=None,
                halo_lo=None, halo_hi=None, lambda_tv: float = 0.0, tv_count: float = 1.0,
                tv_partial=None, halt=None, blocked: bool | None = None, z0: int = 0,
                c_local: int | None = None, occ=None):
        """sinogram (m, n, c) -> volume (h, w, c) [+ lambda_tv * TV subgradient of vol].

        occ (training step only): the FvrPlan of vol (or its footprint_coverage
        pointer); the result is then written only around Gaussian footprints,
        which is where the voxelizer backward reads it."""
        c = int(c_local if c_local is not None else gsino.shape[2])
        if out is None:
            out = torch.empty((self.h, self.w, c), dtype=torch.float32, device=gsino.device)
        args = (ptr(gsino), ptr(vol), ptr(halo_lo), ptr(halo_hi), float(lambda_tv),
                float(tv_count), ptr(out), ptr(tv_partial), ptr(halt), stream_handle())
        occ = _occ(occ, "tile")
        if getattr(self, "blocked", False) if blocked is None else blocked:
            g = self.ab
            call("splatct_proj_adjoint_blocked", ptr(g[0]), ptr(g[1]), ptr(g[2]), self.w, self.h,
                 c, *args[:8], occ if occ is not None else VP(0), *args[8:])
        else:
            call("splatct_proj_adjoint", ptr(self.at_ptr), ptr(self.at_ray), ptr(self.at_val),
                 self.w, self.h, c, *args)
        return out

    def march_forward(self, vol: torch.Tensor) -> torch.Tensor:
        """Matrix-free ray-marching forward projection (cross-check path)."""
        c = int(vol.shape[2])
        out = torch.empty((self.m, self.n_det, c), dtype=torch.float32, device=vol.device)
        call("splatct_proj_march_forward", *self._gargs()[:9], self.w, self.h, c, ptr(vol),
             ptr(out), stream_handle())
        return out


_PROJ_CACHE: "OrderedDict[tuple, ProjectorOperator]" = OrderedDict()


def projector_for(geom: ScanGeometry, w: int, h: int, step: float = 0.5,
                  device=None) -> ProjectorOperator:
    dev = require_cuda(device)
    key = (geom.key(), int(w), int(h), float(step), str(dev))
    op = _PROJ_CACHE.get(key)
    if op is None:
        op = ProjectorOperator(geom, w, h, step, dev)
        _PROJ_CACHE[key] = op
        while len(_PROJ_CACHE) > 4:
            _PROJ_CACHE.popitem(last=False)
    else:
        _PROJ_CACHE.move_to_end(key)
    return op


class ConeOperator:
    """Circular cone-beam projector and its exact adjoint (cone.cu; SURVEY
    §8(f) N3, parity unpinned).  The per-column xy samples and their
    per-pixel transpose are built once per geometry; ``z0`` selects the slab
    of a ``c_global``-slice volume, whose projections are partial line
    integrals (summed across slabs by the caller).  Sinogram (m, nu, nv)."""

    def __init__(self, geom: ScanGeometry, w: int, h: int, c_global: int, step: float = 0.5,
                 device=None):
        if geom.variant != "cone":
            raise ValueError("ConeOperator needs a cone geometry")
        self.device = require_cuda(device)
        geom.check_volume((w, h, c_global))
        self.geom = geom
        self.w, self.h, self.c_global = int(w), int(h), int(c_global)
        self.m, self.n_det, self.nv = int(geom.n_views), int(geom.n_detectors), int(geom.n_rows)
        self.sv = float(geom.row_spacing)
        self.step = float(step)
        self.n_rays = self.m * self.n_det
        ang = np.asarray(geom.view_angles, np.float64)
        dev = self.device
        self.cos_t = torch.from_numpy(np.cos(ang)).to(dev)
        self.sin_t = torch.from_numpy(np.sin(ang)).to(dev)
        g = (ptr(self.cos_t), ptr(self.sin_t), self.m, self.n_det,
             float(geom.detector_spacing), float(geom.source_to_origin),
             float(geom.origin_to_detector), self.w, self.h, self.step)
        sb = size_query("splatct_cone_setup_scratch_bytes", self.m, self.n_det, self.w, self.h)
        scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
        # column-major merged entries {pixel, w, tau} and their pixel-major
        # transpose {column, w, tau, 1/tau}
        self.cptr = torch.empty(self.n_rays + 1, dtype=torch.int64, device=dev)
        self.inv_len = torch.empty(self.n_rays, dtype=torch.float32, device=dev)
        ns = ctypes.c_int64(0)
        call("splatct_cone_count", *g, ptr(self.cptr), ptr(self.inv_len), ptr(scratch), sb,
             ctypes.byref(ns), stream_handle())
        self.n_samples = int(ns.value)   # column entries
        self.col_entries = torch.empty((max(self.n_samples, 1), 4), dtype=torch.float32,
                                       device=dev)
        call("splatct_cone_fill", *g, ptr(self.cptr), ptr(self.col_entries), stream_handle())
        self.eptr = torch.empty(self.w * self.h + 1, dtype=torch.int64, device=dev)
        ne = ctypes.c_int64(0)
        call("splatct_cone_entry_count", ptr(self.col_entries), ptr(self.cptr), self.n_rays,
             self.w, self.h, ptr(self.eptr), ptr(scratch), sb, ctypes.byref(ne),
             stream_handle())
        self.n_entries = int(ne.value)
        self.entries = torch.empty((max(self.n_entries, 1), 4), dtype=torch.float32, device=dev)
        eb = size_query("splatct_cone_entry_scratch_bytes", self.n_entries, self.w, self.h)
        escr = torch.empty(eb, dtype=torch.uint8, device=dev)
        call("splatct_cone_entry_fill", ptr(self.col_entries), ptr(self.cptr), self.n_rays,
             self.w, self.h, ptr(self.eptr), self.n_entries, ptr(self.entries), ptr(escr), eb,
             stream_handle())
        del scratch, escr
        self.gscaled = torch.empty(self.n_rays * self.nv, dtype=torch.float32, device=dev)
        self.tvop = tv_operator(self.w, self.h, dev)

    @property
    def matrix_bytes(self) -> int:
        return 16 * (self.n_samples + self.n_entries) + 8 * (self.n_rays + self.w * self.h + 2)

    def _zc(self, z0: int) -> float:
        return 0.5 * (self.c_global - 1) - float(z0)

    def forward(self, vol: torch.Tensor, out: torch.Tensor | None = None, halt=None, z0: int = 0,
                blocked=None, occ=None):
        """vol slab (h, w, c_local) -> partial cone projections (m, nu, nv)."""
        cl = int(vol.shape[2])
        if out is None:
            out = torch.empty((self.m, self.n_det, self.nv), dtype=torch.float32,
                              device=vol.device)
        occ = _occ(occ, "pixel")
        call("splatct_cone_forward", ptr(self.col_entries), ptr(self.cptr), ptr(self.inv_len),
             self.n_rays, self.nv, self.sv, self.step, self.w, self.h, cl, self._zc(z0),
             ptr(vol), occ if occ is not None else VP(0), ptr(out), ptr(halt), stream_handle())
        return out

    def adjoint(self, gsino: torch.Tensor, out: torch.Tensor | None = None, vol=None,
                halo_lo=None, halo_hi=None, lambda_tv: float = 0.0, tv_count: float = 1.0,
                tv_partial=None, halt=None, z0: int = 0, c_local: int | None = None,
                blocked=None, occ=None):
        """(m, nu, nv) -> volume slab (h, w, c_local) [+ lambda_tv * TV subgradient of vol]."""
        cl = int(c_local if c_local is not None else
                 (out.shape[2] if out is not None else
                  (vol.shape[2] if vol is not None else self.c_global)))
        if out is None:
            out = torch.empty((self.h, self.w, cl), dtype=torch.float32, device=gsino.device)
        acc = 0
        if vol is not None and lambda_tv > 0:
            # TV first (the empty-operator adjoint writes out = l3 dTV and the
            # TV value partials), then the cone adjoint accumulates into it
            self.tvop.adjoint(gsino, out, vol=vol, halo_lo=halo_lo, halo_hi=halo_hi,
                              lambda_tv=lambda_tv, tv_count=tv_count, tv_partial=tv_partial,
                              halt=halt, blocked=False, c_local=cl)
            acc = 1
        occ = _occ(occ, "tile")
        call("splatct_cone_adjoint", ptr(self.entries), ptr(self.eptr), ptr(self.inv_len),
             self.n_rays, self.nv, self.sv, self.step, self.w, self.h, cl, self._zc(z0),
             ptr(gsino), ptr(self.gscaled), ptr(out), acc, occ if occ is not None else VP(0),
             ptr(halt), stream_handle())
        return out


_CONE_CACHE: "OrderedDict[tuple, ConeOperator]" = OrderedDict()


def cone_projector_for(geom: ScanGeometry, w: int, h: int, c_global: int, step: float = 0.5,
                       device=None) -> ConeOperator:
    dev = require_cuda(device)
    key = (geom.key(), int(w), int(h), int(c_global), float(step), str(dev))
    op = _CONE_CACHE.get(key)
    if op is None:
        op = ConeOperator(geom, w, h, c_global, step, dev)
        _CONE_CACHE[key] = op
        while len(_CONE_CACHE) > 2:
            _CONE_CACHE.popitem(last=False)
    else:
        _CONE_CACHE.move_to_end(key)
    return op


def clear_operator_caches() -> None:
    """Drop every cached projector operator (the next call rebuilds it: a
    cold API call, as bench.py's e2e "cold" leg measures)."""
    _PROJ_CACHE.clear()
    _CONE_CACHE.clear()


def operator_for(geom: ScanGeometry, w: int, h: int, c_global: int, step: float = 0.5,
                 device=None):
    """The projector of a geometry: per-slice (ProjectorOperator) or cone."""
    if geom.variant == "cone":
        return cone_projector_for(geom, w, h, c_global, step, device)
    return projector_for(geom, w, h, step, device)


def tv_partial_len(w: int, h: int, c: int, blocked: bool = False) -> int:
    """Doubles in a tv_partial buffer: what the blocked adjoint writes
    (blocked=True), else room for either adjoint (the CSR one writes w*h)."""
    n = ctypes.c_int64(0)
    call("splatct_proj_tv_partial_len", int(w), int(h), int(c), ctypes.byref(n))
    return int(n.value) if blocked else max(int(n.value), int(w) * int(h))


def tv_operator(w: int, h: int, device=None) -> ProjectorOperator:
    """An operator with an empty A^T: its adjoint is the TV term alone."""
    dev = require_cuda(device)
    op = ProjectorOperator.__new__(ProjectorOperator)
    op.device = dev
    op.w, op.h = int(w), int(h)
    op.at_ptr = torch.zeros(op.w * op.h + 1, dtype=torch.int64, device=dev)
    op.at_ray = torch.zeros(1, dtype=torch.int32, device=dev)
    op.at_val = torch.zeros(1, dtype=torch.float32, device=dev)
    return op


# ---------------------------------------------------------------------------
# loss
# ---------------------------------------------------------------------------

class LossPlan:
    """Workspace for the fused L1 + SSIM loss on an (m, n, p) sinogram slab."""

    def __init__(self, m: int, n: int, p: int, device=None):
        self.device = require_cuda(device)
        self.m, self.n, self.p = int(m), int(n), int(p)
        self.ws_bytes = size_query("splatct_loss_workspace_bytes", self.m, self.n, self.p)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        kr, kc = min(11, self.m), min(11, self.n)
        kr -= 1 - kr % 2
        kc -= 1 - kc % 2
        self.valid = (self.m - kr + 1) * (self.n - kc + 1)

        self.prepared_ref = None   # data_ptr of the ref whose window stats are in ws

    def prepare(self, ref: torch.Tensor) -> None:
        """Cache the constant reference sinogram's SSIM window moments (call
        again whenever ref's contents change)."""
        call("splatct_loss_prepare_ref", ptr(ref), self.m, self.n, self.p, ptr(self.ws),
             self.ws_bytes, stream_handle())
        self.prepared_ref = ref.data_ptr()

    def fused(self, pred, ref, lmax: float, lambda1: float, lambda2: float, l1_count: float,
              ssim_slices: float, grad_out, sums, halt=None, defer: bool = False):
        """defer (prepared ref only): leave sums[0:2] as block partials for
        iter_finalize_partials (partials() gives them)."""
        prepared = self.prepared_ref == ref.data_ptr()
        if defer and not prepared:
            raise ValueError("a deferred loss needs the prepared reference")
        fn = ("splatct_loss_fused_prepared_deferred" if defer
              else "splatct_loss_fused_prepared" if prepared else "splatct_loss_fused")
        call(fn, ptr(pred), ptr(ref), self.m, self.n, self.p, float(lmax),
             float(lambda1), float(lambda2), float(l1_count), float(ssim_slices), ptr(grad_out),
             ptr(self.ws), self.ws_bytes, ptr(sums), ptr(halt), stream_handle())

    def partials(self, lambda2: float):
        """(l1 pointer, count, SSIM pointer, count) of a deferred loss's block partials."""
        a, b = ctypes.c_void_p(0), ctypes.c_void_p(0)
        na, nb = ctypes.c_int64(0), ctypes.c_int64(0)
        call("splatct_loss_partials", self.m, self.n, self.p, float(lambda2), ptr(self.ws),
             self.ws_bytes, ctypes.byref(a), ctypes.byref(na), ctypes.byref(b), ctypes.byref(nb))
        return a, int(na.value), b, int(nb.value)


def sino_max(x: torch.Tensor) -> float:
    out = torch.empty(1 + _lib.SQDIFF_BLOCKS, dtype=torch.float64, device=x.device)
    call("splatct_sino_max", ptr(x), int(x.numel()), ptr(out), stream_handle())
    return float(out[0].item())


def ssim_valid(m: int, n: int) -> int:
    """Valid SSIM window positions of an m x n image: the 11 x 11 window shrunk
    to the largest odd size <= each dimension (loss.py:77-101)."""
    kr, kc = min(int(m), 11), min(int(n), 11)
    kr -= 1 - kr % 2
    kc -= 1 - kc % 2
    return (int(m) - kr + 1) * (int(n) - kc + 1)


def tv_halo_fixup(vol: torch.Tensor, dl: torch.Tensor, halo_lo, halo_hi, lambda_tv: float,
                  tv_count: float, tv_sum: torch.Tensor, halt=None) -> None:
    """Cross-slab TV terms after a halo-free adjoint (splatct_tv_halo_fixup)."""
    h, w, c = (int(v) for v in vol.shape)
    call("splatct_tv_halo_fixup", ptr(vol), ptr(dl), ptr(halo_lo), ptr(halo_hi), w, h, c,
         float(lambda_tv), float(tv_count), ptr(tv_sum), ptr(halt), stream_handle())


def reduce_sum(x: torch.Tensor, out: torch.Tensor) -> None:
    call("splatct_reduce_sum", ptr(x), int(x.numel()), ptr(out), stream_handle())


def sum_sq_diff(x: torch.Tensor, y: torch.Tensor) -> float:
    ws = torch.empty(_lib.SQDIFF_BLOCKS, dtype=torch.float64, device=x.device)
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    call("splatct_sum_sq_diff", ptr(x), ptr(y), int(x.numel()), ptr(ws), ptr(out),
         stream_handle())
    return float(out.item())


def adam(params, grads, m1, m2, scalars, sigma_floor, sigma_ceiling, halt=None):
    call("splatct_adam", ptr(params), ptr(grads), ptr(m1), ptr(m2), int(params.shape[1]),
         ptr(scalars), float(sigma_floor), float(sigma_ceiling), ptr(halt), stream_handle())


def grad_norm_accum(grads, accum, halt=None):
    call("splatct_grad_norm_accum", ptr(grads), int(grads.shape[1]), ptr(accum), ptr(halt),
         stream_handle())


def densify(params: torch.Tensor, m1: torch.Tensor, m2: torch.Tensor, accum: torch.Tensor,
            iters: int, dparams, rng: np.random.Generator):
    """One clone / split / prune event on the device (csrc/densify.cu).

    Same result as ``densify.densify_and_prune`` + ``OptimizerState.remap``
    (reference densify.py:86-147, optim.py:92-106) without moving the cloud
    through host memory: the host reads three counts, sizes the budgets
    exactly as the reference does, and draws the split children's normals
    from ``rng`` (the reference's ``default_rng([seed, it+1])``, optim.py:394).
    Returns (params', m1', m2', DensifyReport) with ``report.kept`` None.
    """
    from .densify import CBRT2, DensifyReport

    dev = params.device
    n = int(params.shape[1])
    if iters <= 0:
        from .core import ValidationError
        raise ValidationError("no backward passes accumulated since last event")
    cls = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    keys = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    counts = torch.empty(3, dtype=torch.int64, device=dev)
    ws_bytes = size_query("splatct_densify_workspace_bytes", n)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    s = stream_handle()
    call("splatct_densify_classify", ptr(params), ptr(accum), n, float(iters), float(dparams.tau),
         float(dparams.theta), 3.0 * float(dparams.box_size), int(dparams.grad_prune_enabled),
         ptr(cls), ptr(keys), ptr(counts), s)
    n_prune, c_clone, c_split = (int(v) for v in counts.cpu().tolist())
    k_clone = min(dparams.n_max - n, c_clone)                      # densify.py:104-106
    n_clone = max(k_clone, 0) if c_clone > 0 else 0
    call("splatct_densify_select", ptr(cls), ptr(keys), n, 2, k_clone, c_clone, ptr(ws), ws_bytes, s)
    k_split = min(dparams.n_max - n - n_clone, c_split)            # densify.py:107-110
    n_split = max(k_split, 0) if c_split > 0 else 0
    call("splatct_densify_select", ptr(cls), ptr(keys), n, 3, k_split, c_split, ptr(ws), ws_bytes, s)
    n_new = n - n_prune - n_split + n_clone + 2 * n_split
    noise = None
    if n_split:
        noise = torch.from_numpy(rng.standard_normal((2 * n_split, 3))).to(dev)
    out = [torch.empty((5, n_new), dtype=torch.float64, device=dev) for _ in range(3)]
    call("splatct_densify_apply", ptr(params), ptr(m1), ptr(m2), ptr(cls), ptr(noise), n, n_new,
         float(CBRT2), ptr(out[0]), ptr(out[1]), ptr(out[2]), ptr(ws), ws_bytes, s)
    return out[0], out[1], out[2], DensifyReport(n_clone, n_split, n_prune, n_new, None)

"""ctypes binding of libsplatct.so (the C ABI declared in include/splatct.h).

There is no fallback: if the library is missing or a CUDA device is absent,
every compute entry point raises.  ``load()`` builds the library in-tree on
first use when it is stale (nvcc cross-compiles without a GPU).
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import build as _build

c_i32 = ctypes.c_int
c_i64 = ctypes.c_int64
c_f64 = ctypes.c_double
c_sz = ctypes.c_size_t
c_vp = ctypes.c_void_p
c_szp = ctypes.POINTER(ctypes.c_size_t)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int)
c_vpp = ctypes.POINTER(ctypes.c_void_p)

# name -> argtypes (all return int status except where noted)
SIGNATURES: dict[str, list] = {
    "splatct_abi_version": [],
    "splatct_last_error": [],
    "splatct_launch_count": [],
    "splatct_fvr_workspace_bytes": [c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_szp],
    "splatct_fvr_bin": [c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp, c_sz,
                        c_vp, c_vp],
    "splatct_fvr_bin_row_ordered": [c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32,
                                    c_vp, c_sz, c_vp, c_vp],
    "splatct_fvr_adam_bin": [c_vp, c_vp, c_vp, c_vp, c_vp, c_f64, c_f64, c_i64, c_i32, c_i32,
                             c_i32, c_i32, c_i32, c_i32, c_i32, c_vp, c_sz, c_i32, c_vp, c_vp],
    "splatct_fvr_forward": [c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp,
                            c_sz, c_vp, c_vp, c_vp],
    "splatct_fvr_forward_masked": [c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp,
                            c_sz, c_vp, c_vp, c_vp],
    "splatct_fvr_forward_plain": [c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32,
                                  c_vp, c_sz, c_vp, c_vp],
    "splatct_fvr_backward": [c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp,
                             c_sz, c_vp, c_vp, c_vp, c_vp, c_vp],
    "splatct_grad_norm_accum": [c_vp, c_i64, c_vp, c_vp, c_vp],
    "splatct_tc_selftest": [c_vp, c_vp, c_vp, c_i32, c_vp],
    "splatct_tv_halo_fixup": [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_f64, c_f64, c_vp,
                              c_vp, c_vp],
    "splatct_fvr_export_bins": [c_vp, c_sz, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp,
                                c_vp, c_vp, c_i64p, c_i64p, c_vp],
    "splatct_proj_scratch_bytes": [c_i32, c_i32, c_i32, c_i32, c_i64, c_szp],
    "splatct_proj_count": [c_vp, c_vp, c_i32, c_i32, c_f64, c_f64, c_i32, c_f64, c_f64, c_i32,
                           c_i32, c_vp, c_vp, c_sz, c_i64p, c_vp],
    "splatct_proj_fill": [c_vp, c_vp, c_i32, c_i32, c_f64, c_f64, c_i32, c_f64, c_f64, c_i32,
                          c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp],
    "splatct_proj_forward": [c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_i32, c_vp, c_vp],
    "splatct_proj_adjoint": [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_f64,
                             c_f64, c_vp, c_vp, c_vp, c_vp],
    "splatct_proj_tv_partial_len": [c_i32, c_i32, c_i32, c_i64p],
    "splatct_proj_block_scratch_bytes": [c_i32, c_i32, c_i32, c_i32, c_szp],
    "splatct_proj_block_count": [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_sz,
                                 c_i64p, c_vp],
    "splatct_proj_block_fill": [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp,
                                c_vp, c_sz, c_vp],
    "splatct_proj_forward_blocked": [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_i32, c_vp,
                                     c_i32, c_i32, c_vp, c_vp],
    "splatct_proj_forward_ctas": [c_i32, c_i32, c_i32, c_i32, c_i32, c_i64p, c_i32p, c_i32p],
    "splatct_proj_forward_blocked_ordered": [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_i32,
                                             c_vp, c_i32, c_i32, c_vp, c_vp, c_vp],
    "splatct_fvr_footprint_coverage_offset": [c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32,
                                              c_szp],
    "splatct_fvr_pixel_occupancy_offset": [c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32,
                                           c_szp],
    "splatct_proj_adjoint_blocked": [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp,
                                     c_f64, c_f64, c_vp, c_vp, c_vp, c_vp, c_vp],
    "splatct_proj_march_forward": [c_vp, c_vp, c_i32, c_i32, c_f64, c_f64, c_i32, c_f64, c_f64,
                                   c_i32, c_i32, c_i32, c_vp, c_vp, c_vp],
    "splatct_loss_workspace_bytes": [c_i32, c_i32, c_i32, c_szp],
    "splatct_sino_max": [c_vp, c_i64, c_vp, c_vp],
    "splatct_loss_fused": [c_vp, c_vp, c_i32, c_i32, c_i32, c_f64, c_f64, c_f64, c_f64, c_f64,
                           c_vp, c_vp, c_sz, c_vp, c_vp, c_vp],
    "splatct_loss_prepare_ref": [c_vp, c_i32, c_i32, c_i32, c_vp, c_sz, c_vp],
    "splatct_loss_fused_prepared": [c_vp, c_vp, c_i32, c_i32, c_i32, c_f64, c_f64, c_f64, c_f64,
                                    c_f64, c_vp, c_vp, c_sz, c_vp, c_vp, c_vp],
    "splatct_sum_sq_diff": [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp],
    "splatct_reduce_sum": [c_vp, c_i64, c_vp, c_vp],
    "splatct_stage_upload": [c_vp, c_vp, c_vp, c_sz, c_i32, c_vp],
    "splatct_iter_finalize": [c_vp, c_f64, c_f64, c_f64, c_f64, c_f64, c_f64, c_f64, c_f64, c_i64,
                              c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp],
    "splatct_iter_finalize_partials": [c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp,
                                       c_i64, c_f64, c_f64, c_f64, c_f64, c_f64, c_f64, c_f64,
                                       c_f64, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp],
    "splatct_loss_partials": [c_i32, c_i32, c_i32, c_f64, c_vp, c_sz, c_vpp, c_i64p, c_vpp,
                              c_i64p],
    "splatct_loss_fused_prepared_deferred": [c_vp, c_vp, c_i32, c_i32, c_i32, c_f64, c_f64,
                                             c_f64, c_f64, c_f64, c_vp, c_vp, c_sz, c_vp, c_vp,
                                             c_vp],
    "splatct_adam": [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_f64, c_f64, c_vp, c_vp],
    "splatct_fbp_filter": [c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp],
    "splatct_fbp_backproject": [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_f64,
                                c_f64, c_i32, c_f64, c_vp, c_vp],
    "splatct_cone_setup_scratch_bytes": [c_i32, c_i32, c_i32, c_i32, c_szp],
    "splatct_cone_count": [c_vp, c_vp, c_i32, c_i32, c_f64, c_f64, c_f64, c_i32, c_i32, c_f64,
                           c_vp, c_vp, c_vp, c_sz, c_i64p, c_vp],
    "splatct_cone_fill": [c_vp, c_vp, c_i32, c_i32, c_f64, c_f64, c_f64, c_i32, c_i32, c_f64,
                          c_vp, c_vp, c_vp],
    "splatct_cone_entry_count": [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_sz, c_i64p,
                                 c_vp],
    "splatct_cone_entry_scratch_bytes": [c_i64, c_i32, c_i32, c_szp],
    "splatct_cone_entry_fill": [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_i64, c_vp, c_vp, c_sz,
                                c_vp],
    "splatct_cone_forward": [c_vp, c_vp, c_vp, c_i32, c_i32, c_f64, c_f64, c_i32, c_i32, c_i32,
                             c_f64, c_vp, c_vp, c_vp, c_vp, c_vp],
    "splatct_cone_adjoint": [c_vp, c_vp, c_vp, c_i32, c_i32, c_f64, c_f64, c_i32, c_i32, c_i32,
                             c_f64, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp],
    "splatct_densify_workspace_bytes": [c_i64, c_szp],
    "splatct_densify_classify": [c_vp, c_vp, c_i64, c_f64, c_f64, c_f64, c_f64, c_i32, c_vp, c_vp,
                                 c_vp, c_vp],
    "splatct_densify_select": [c_vp, c_vp, c_i64, c_i32, c_i64, c_i64, c_vp, c_sz, c_vp],
    "splatct_densify_apply": [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_f64, c_vp, c_vp, c_vp,
                              c_vp, c_sz, c_vp],
}

SQDIFF_BLOCKS = 592   # SPLATCT_SQDIFF_BLOCKS
TILE = 16             # SPLATCT_TILE

_lock = threading.Lock()
_lib = None


class SplatctError(RuntimeError):
    """A libsplatct entry point returned a non-zero status."""


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load (building if stale) libsplatct.so and bind every C-ABI symbol."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = _build.LIB
        if build_if_missing and _build.nvcc_available():
            _build.build()   # a failed build raises: never run a stale library
        elif not os.path.exists(path):
            raise OSError(f"libsplatct.so missing at {path} and nvcc is not available")
        if not os.path.exists(path):
            raise OSError(f"libsplatct.so not found at {path}; run paper_2411_04844_b200.build")
        L = ctypes.CDLL(path)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = argtypes
            fn.restype = {"splatct_last_error": ctypes.c_char_p,
                          "splatct_launch_count": ctypes.c_ulonglong}.get(name, ctypes.c_int)
        _lib = L
        return L


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point; raise SplatctError on failure."""
    L = load()
    rc = getattr(L, name)(*args)
    if rc != 0:
        msg = L.splatct_last_error().decode(errors="replace")
        raise SplatctError(f"{name} failed (status {rc}): {msg}")


def launch_count() -> int:
    return int(load().splatct_launch_count())


def size_query(name: str, *args) -> int:
    out = ctypes.c_size_t(0)
    call(name, *args, ctypes.byref(out))
    return int(out.value)

"""Raw + sidecar file formats (cli module SPEC.md:446-519).

The reference specifies the formats but ships no implementation (SURVEY §5.4,
§8(f) N4).  Every array is written as raw little-endian values in the
reference's index order, next to a JSON sidecar ``<path>.json`` carrying the
kind, dims, dtype, value range and (optionally) spacing / geometry, so that
every file round-trips bit-exactly through its own reader.

    volume     float32-le, idx = x + w*(y + h*z)   (VolumeGrid.zyx C order)
    sinogram   float32-le, (m, n, p) C order        (slice fastest)
    cloud      float64-le, mu (N,3) | sigma (N) | intensity (N)
    trace      CSV, one row per TraceRow
"""
from __future__ import annotations

import csv
import dataclasses
import json
import os

import numpy as np

from .core import GaussianCloud, ScanGeometry, Sinogram, ValidationError, VolumeGrid

__all__ = ["write_volume", "read_volume", "write_sinogram", "read_sinogram", "write_cloud",
           "read_cloud", "write_trace_csv", "geometry_to_dict", "geometry_from_dict",
           "sidecar_path"]


def sidecar_path(path: str) -> str:
    return path + ".json"


def _write_sidecar(path: str, meta: dict) -> None:
    with open(sidecar_path(path), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
        f.write("\n")


def _read_sidecar(path: str, kind: str) -> dict:
    sp = sidecar_path(path)
    if not os.path.exists(path) or not os.path.exists(sp):
        raise ValidationError(f"missing {kind} file or sidecar: {path}")
    with open(sp) as f:
        meta = json.load(f)
    if meta.get("kind") != kind:
        raise ValidationError(f"{sp}: expected kind {kind!r}, found {meta.get('kind')!r}")
    return meta


def _read_raw(path: str, dtype: str, count: int) -> np.ndarray:
    arr = np.fromfile(path, dtype=dtype)
    if arr.size != count:
        raise ValidationError(f"{path}: {arr.size} values, sidecar says {count}")
    return arr


def write_volume(path: str, vol: VolumeGrid, spacing=(1.0, 1.0, 1.0)) -> None:
    zyx = np.ascontiguousarray(vol.zyx, dtype="<f4")
    zyx.tofile(path)
    _write_sidecar(path, {"kind": "volume", "dims": [int(d) for d in vol.dims],
                          "dtype": "float32-le", "order": "idx = x + w*(y + h*z)",
                          "spacing": [float(s) for s in spacing],
                          "min": float(zyx.min()) if zyx.size else 0.0,
                          "max": float(zyx.max()) if zyx.size else 0.0})


def read_volume(path: str) -> VolumeGrid:
    meta = _read_sidecar(path, "volume")
    w, h, c = (int(d) for d in meta["dims"])
    arr = _read_raw(path, "<f4", w * h * c)
    return VolumeGrid.from_zyx(arr.reshape(c, h, w).astype(np.float32))


def write_sinogram(path: str, sino: Sinogram, geom: ScanGeometry | None = None) -> None:
    v = np.ascontiguousarray(sino.views, dtype="<f4")
    v.tofile(path)
    meta = {"kind": "sinogram", "dims": [int(d) for d in sino.dims], "dtype": "float32-le",
            "order": "(m, n, p) C order, slice fastest",
            "min": float(v.min()) if v.size else 0.0, "max": float(v.max()) if v.size else 0.0}
    if geom is not None:
        meta["geometry"] = geometry_to_dict(geom)
    _write_sidecar(path, meta)


def read_sinogram(path: str):
    """Returns (Sinogram, ScanGeometry | None)."""
    meta = _read_sidecar(path, "sinogram")
    m, n, p = (int(d) for d in meta["dims"])
    arr = _read_raw(path, "<f4", m * n * p)
    geom = geometry_from_dict(meta["geometry"]) if "geometry" in meta else None
    return Sinogram.from_views(arr.reshape(m, n, p).astype(np.float32)), geom


def write_cloud(path: str, cloud: GaussianCloud, extra: dict | None = None) -> None:
    n = cloud.n
    blob = np.concatenate([np.asarray(cloud.mu, "<f8").reshape(-1),
                           np.asarray(cloud.sigma, "<f8").reshape(-1),
                           np.asarray(cloud.intensity, "<f8").reshape(-1)])
    blob.tofile(path)
    meta = {"kind": "gaussian_cloud", "n": int(n), "dtype": "float64-le",
            "layout": "mu (N,3) x,y,z | sigma (N) | intensity (N)"}
    if extra:
        meta.update(extra)
    _write_sidecar(path, meta)


def read_cloud(path: str) -> GaussianCloud:
    meta = _read_sidecar(path, "gaussian_cloud")
    n = int(meta["n"])
    blob = _read_raw(path, "<f8", 5 * n)
    return GaussianCloud(blob[:3 * n].reshape(n, 3).copy(), blob[3 * n:4 * n].copy(),
                         blob[4 * n:].copy())


def write_trace_csv(path: str, trace) -> None:
    rows = [dataclasses.asdict(t) for t in trace]
    with open(path, "w", newline="") as f:
        if not rows:
            return
        wr = csv.DictWriter(f, fieldnames=list(rows[0]))
        wr.writeheader()
        wr.writerows(rows)


def geometry_to_dict(geom: ScanGeometry) -> dict:
    d = {"variant": geom.variant, "n_views": int(geom.n_views),
         "n_detectors": int(geom.n_detectors), "detector_spacing": float(geom.detector_spacing),
         "view_angles": [float(a) for a in geom.view_angles]}
    if geom.source_to_origin is not None:
        d["source_to_origin"] = float(geom.source_to_origin)
        d["origin_to_detector"] = float(geom.origin_to_detector)
    if geom.n_rows is not None:
        d["n_rows"] = int(geom.n_rows)
        d["row_spacing"] = float(geom.row_spacing)
    return d


def geometry_from_dict(d: dict) -> ScanGeometry:
    """Either explicit ``view_angles`` or ``angle_start`` / ``angle_extent``
    (counter-clockwise from +x, limited-angle as [start, start + extent))."""
    variant = d.get("variant", "parallel")
    m, n = int(d["n_views"]), int(d["n_detectors"])
    spacing = float(d.get("detector_spacing", 1.0))
    if "view_angles" in d:
        ang = np.asarray(d["view_angles"], np.float64)
        return ScanGeometry(variant, m, n, spacing, ang, d.get("source_to_origin"),
                            d.get("origin_to_detector"), d.get("n_rows"), d.get("row_spacing"))
    start = float(d.get("angle_start", 0.0))
    extent = float(d.get("angle_extent", np.pi))
    if variant == "parallel":
        return ScanGeometry.parallel(m, n, spacing, start, extent)
    if variant == "fan":
        return ScanGeometry.fan(m, n, spacing, float(d["source_to_origin"]),
                                float(d["origin_to_detector"]), start, extent)
    if variant == "cone":
        return ScanGeometry.cone(m, n, int(d["n_rows"]), spacing, float(d["source_to_origin"]),
                                 float(d["origin_to_detector"]), d.get("row_spacing"), start,
                                 float(d.get("angle_extent", 2 * np.pi)))
    raise ValidationError(f"unknown geometry variant {variant!r}")

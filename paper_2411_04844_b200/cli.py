"""Command-line surface.

    python -m paper_2411_04844_b200.cli phantom --kind shepp-logan-3d --dims 64 64 64 --out vol.raw
    python -m paper_2411_04844_b200.cli project --volume vol.raw --config run.json --out sino.raw
    python -m paper_2411_04844_b200.cli fbp --sinogram sino.raw --config run.json --out fbp.raw
    python -m paper_2411_04844_b200.cli reconstruct --config run.json --out DIR
    python -m paper_2411_04844_b200.cli metrics --recon a.raw --truth b.raw
    python -m paper_2411_04844_b200.cli bench --dims 128 128 128 --n 50000 --out bench.csv

Run config (JSON or YAML): ``dims``, ``geometry`` {variant, n_views, n_detectors,
detector_spacing, angle_start, angle_extent, source_to_origin, origin_to_detector},
``box``, ``weights`` (preset name or {lambda1, lambda2, lambda3}), ``optimizer``
{lr_initial, lr_final, max_iters}, ``densify`` {interval, n_max, tau, theta} or null,
``init`` {mode, n_gaussians, seed}, ``noise`` {model, sigma, photon_count, seed},
``paths`` {sinogram, truth, init_cloud}, ``deterministic``, ``stop_rule``,
``holdout_fraction``.  The reference has no CLI; the schema follows SPEC's
RunConfig.  Exit codes: 0 ok, 2 config error, 3 numeric failure.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

from . import io as fio
from .core import BoxConfig, ValidationError

EXIT_OK, EXIT_CONFIG, EXIT_NUMERIC = 0, 2, 3


def load_config(path: str) -> dict:
    if not os.path.exists(path):
        raise ValidationError(f"config file not found: {path}")
    with open(path) as f:
        text = f.read()
    if path.endswith((".yaml", ".yml")):
        import yaml
        cfg = yaml.safe_load(text)
    else:
        cfg = json.loads(text)
    if not isinstance(cfg, dict):
        raise ValidationError("run config must be a mapping")
    return cfg


def _dims(cfg) -> tuple:
    d = cfg.get("dims")
    if not d or len(d) != 3 or any(int(v) < 1 for v in d):
        raise ValidationError("config needs dims: [w, h, c]")
    return tuple(int(v) for v in d)


def _geometry(cfg):
    if "geometry" not in cfg:
        raise ValidationError("config needs a geometry block")
    return fio.geometry_from_dict(cfg["geometry"])


def _weights(cfg):
    from .loss import WEIGHT_PRESETS, LossWeights
    w = cfg.get("weights", "l1+ssim+tv")
    if isinstance(w, str):
        if w not in WEIGHT_PRESETS:
            raise ValidationError(f"unknown weight preset {w!r}")
        return WEIGHT_PRESETS[w]
    return LossWeights(float(w.get("lambda1", 0.6)), float(w.get("lambda2", 0.2)),
                       float(w.get("lambda3", 1.0)))


def settings_from_config(cfg: dict, args=None):
    """RunConfig -> (ReconstructionSettings, geometry, paths); validates
    everything the modules would reject before any compute starts."""
    from .densify import DensifyParams
    from .optim import ReconstructionSettings
    dims = _dims(cfg)
    geom = _geometry(cfg)
    geom.check_volume(dims)
    box_k = int(getattr(args, "box", None) or cfg.get("box", 17))
    box = BoxConfig.for_dims(box_k, dims)
    opt = cfg.get("optimizer", {})
    init = cfg.get("init", {})
    dens = cfg.get("densify")
    dparams, interval = None, 0
    if dens:
        interval = int(dens.get("interval", 100))
        dparams = DensifyParams(n_max=int(dens.get("n_max", 500_000)),
                                tau=float(dens.get("tau", 2e-4)),
                                theta=float(dens.get("theta", 1.0)), box_size=box_k,
                                interval=interval)
    max_iters = int(getattr(args, "max_iters", None) or opt.get("max_iters", 1000))
    seed = getattr(args, "seed", None)
    seed = int(seed if seed is not None else init.get("seed", 0))
    st = ReconstructionSettings(
        dims=dims, box=box, weights=_weights(cfg), max_iters=max_iters,
        lr_initial=float(opt.get("lr_initial", 3e-4)), lr_final=float(opt.get("lr_final", 3e-5)),
        densify=dparams, densify_interval=interval, init_mode=init.get("mode", "fbp"),
        n_gaussians=int(init.get("n_gaussians", 150_000)), seed=seed,
        deterministic=bool(cfg.get("deterministic", False) or getattr(args, "deterministic", False)),
        stop_rule=cfg.get("stop_rule", "iters"),
        holdout_fraction=float(cfg.get("holdout_fraction", 0.1)))
    paths = dict(cfg.get("paths", {}))
    for key in ("sinogram", "truth", "init_cloud"):
        p = paths.get(key)
        if p and not os.path.exists(p):
            raise ValidationError(f"paths.{key} does not exist: {p}")
    return st, geom, paths


# --------------------------------------------------------------------------- commands
def cmd_phantom(args) -> int:
    from . import phantom
    dims = [int(v) for v in args.dims]
    if args.kind == "shepp-logan-2d":
        if len(dims) != 2:
            raise ValidationError("shepp-logan-2d takes --dims W H")
        vol = phantom.shepp_logan_2d(*dims)
    elif args.kind in ("shepp-logan-3d", "chest-3d"):
        if len(dims) != 3:
            raise ValidationError(f"{args.kind} takes --dims W H C")
        vol = (phantom.shepp_logan_3d if args.kind == "shepp-logan-3d" else phantom.chest_3d)(*dims)
    else:
        raise ValidationError(f"unknown phantom kind {args.kind!r}")
    fio.write_volume(args.out, vol)
    return EXIT_OK


def cmd_project(args) -> int:
    from .projector import RaySamplingConfig, add_noise, forward_project
    cfg = load_config(args.config)
    vol = fio.read_volume(args.volume)
    geom = _geometry(cfg)
    sino = forward_project(vol, geom, RaySamplingConfig(float(cfg.get("step_length", 0.5))))
    noise = cfg.get("noise")
    if noise and noise.get("model", "none") != "none":
        sino = add_noise(sino, noise.get("model", "gaussian"), float(noise.get("sigma", 0.0)),
                         float(noise.get("photon_count", 1e5)), int(noise.get("seed", 0)))
    fio.write_sinogram(args.out, sino, geom)
    return EXIT_OK


def cmd_fbp(args) -> int:
    from .projector import fbp
    cfg = load_config(args.config) if args.config else {}
    sino, g = fio.read_sinogram(args.sinogram)
    geom = _geometry(cfg) if "geometry" in cfg else g
    if geom is None:
        raise ValidationError("no geometry: pass --config or a sinogram with a geometry sidecar")
    dims = _dims(cfg) if "dims" in cfg else (geom.n_detectors, geom.n_detectors, sino.dims[2])
    fio.write_volume(args.out, fbp(sino, geom, dims, cfg.get("fbp_filter", "ramp")))
    return EXIT_OK


def cmd_reconstruct(args) -> int:
    from .optim import NonFiniteLossError, run_reconstruction
    cfg = load_config(args.config)
    st, geom, paths = settings_from_config(cfg, args)
    if not paths.get("sinogram"):
        raise ValidationError("config needs paths.sinogram")
    meas, _ = fio.read_sinogram(paths["sinogram"])
    truth = fio.read_volume(paths["truth"]) if paths.get("truth") else None
    init_cloud = fio.read_cloud(paths["init_cloud"]) if paths.get("init_cloud") else None
    os.makedirs(args.out, exist_ok=True)
    t0 = time.perf_counter()
    try:
        vol, cloud, trace = run_reconstruction(meas, geom, st, truth=truth, init_cloud=init_cloud)
    except NonFiniteLossError as e:
        print(f"numeric failure: {e}", file=sys.stderr)
        return EXIT_NUMERIC
    fio.write_volume(os.path.join(args.out, "volume.raw"), vol)
    fio.write_cloud(os.path.join(args.out, "cloud.raw"), cloud,
                    {"iterations": len(trace), "seed": st.seed})
    fio.write_trace_csv(os.path.join(args.out, "trace.csv"), trace)
    summary = {"iterations": len(trace), "seconds": time.perf_counter() - t0,
               "final_loss": trace[-1].loss if trace else None, "n_gaussians": cloud.n}
    print(json.dumps(summary))
    return EXIT_OK


def cmd_metrics(args) -> int:
    from .metrics import volume_metrics
    rep = volume_metrics(fio.read_volume(args.recon), fio.read_volume(args.truth), args.max)
    print(json.dumps(rep, sort_keys=True))
    return EXIT_OK


def cmd_bench(args) -> int:
    """Decomposed vs plain splat wall time (SPEC cmd_bench; Table 5 trend)."""
    import torch
    from . import fvr
    from .optim import init_cloud_random
    dims = tuple(int(v) for v in args.dims)
    box = BoxConfig.for_dims(args.box, dims)
    rows = []
    for n in args.n:
        cloud = init_cloud_random(dims, int(n), seed=args.seed, box=box)
        for name, fn in (("reconstruct", fvr.reconstruct),
                         ("reconstruct_nodecomp", fvr.reconstruct_nodecomp)):
            fn(cloud, box, dims)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.reps):
                fn(cloud, box, dims)
            torch.cuda.synchronize()
            rows.append({"path": name, "n": int(n), "dims": "x".join(map(str, dims)),
                         "seconds_per_call": (time.perf_counter() - t0) / args.reps,
                         "peak_device_bytes": int(torch.cuda.max_memory_allocated())})
    with open(args.out, "w") as f:
        f.write(",".join(rows[0]) + "\n")
        for r in rows:
            f.write(",".join(str(v) for v in r.values()) + "\n")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="splatct-b200", description=__doc__.split("\n")[0])
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--deterministic", action="store_true")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("phantom")
    p.add_argument("--kind", required=True)
    p.add_argument("--dims", nargs="+", required=True)
    p.add_argument("--out", required=True)
    p.set_defaults(fn=cmd_phantom)
    p = sub.add_parser("project")
    p.add_argument("--volume", required=True)
    p.add_argument("--config", required=True)
    p.add_argument("--out", required=True)
    p.set_defaults(fn=cmd_project)
    p = sub.add_parser("fbp")
    p.add_argument("--sinogram", required=True)
    p.add_argument("--config", default=None)
    p.add_argument("--out", required=True)
    p.set_defaults(fn=cmd_fbp)
    p = sub.add_parser("reconstruct")
    p.add_argument("--config", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--max-iters", dest="max_iters", type=int, default=None)
    p.add_argument("--box", type=int, default=None)
    p.set_defaults(fn=cmd_reconstruct)
    p = sub.add_parser("metrics")
    p.add_argument("--recon", required=True)
    p.add_argument("--truth", required=True)
    p.add_argument("--max", type=float, default=None)
    p.set_defaults(fn=cmd_metrics)
    p = sub.add_parser("bench")
    p.add_argument("--dims", nargs=3, type=int, default=[128, 128, 128])
    p.add_argument("--n", nargs="+", type=int, default=[50_000])
    p.add_argument("--box", type=int, default=17)
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--out", required=True)
    p.set_defaults(fn=cmd_bench)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    if args.cmd == "bench" and args.seed is None:
        args.seed = 0
    try:
        return args.fn(args)
    except ValidationError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG


if __name__ == "__main__":
    sys.exit(main())

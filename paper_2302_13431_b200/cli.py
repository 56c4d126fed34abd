"""`estimate` subcommand of the reference CLI on the B200 path
(tools/senskit_main.cpp:139-184, flags :302-325, exit codes :23-27).

    python -m paper_2302_13431_b200 estimate --input KSPACE --calib 24,24 --output PREFIX [options]

Reads a CStack v1 k-space stack, extracts the centred calibration region
(types.cpp:58-90), runs estimate_maps and projection_residual through the
C-ABI, and writes PREFIX_maps / _mask / _lambda (CStack v1), PREFIX_mag_chNN.pgm
(2-D), PREFIX_spectrum.csv and PREFIX_provenance.json like the reference.
Exit codes: 0 ok, 2 bad flags, 3 I/O, 4 empty nullspace, 5 shape mismatch,
1 anything else (including options outside the pisco arm this path implements).
"""
from __future__ import annotations

import argparse
import json
import re
import sys

import numpy as np

EXIT_OK, EXIT_OTHER, EXIT_FLAGS, EXIT_IO, EXIT_NULLSPACE, EXIT_SHAPE = 0, 1, 2, 3, 4, 5


_STOLL = re.compile(r"[ \t\n\v\f\r]*([+-]?[0-9]+)")


def _stoll(tok: str) -> int:
    """std::stoll(tok) (base 10): leading whitespace, optional sign, digits; the
    rest of the token is ignored.  No conversion -> std::invalid_argument, out of
    range -> std::out_of_range; both reach the CLI's generic handler (exit 1)."""
    m = _STOLL.match(tok)
    if not m:
        raise ValueError(f"stoll: no conversion of '{tok}'")
    v = int(m.group(1))
    if not -(1 << 63) <= v < (1 << 63):
        raise OverflowError(f"stoll: '{tok}' out of range")
    return v


def parse_extents(text: str, rank: int) -> tuple:  # senskit_main.cpp:29-43
    """Comma-separated extents, token by token as the reference scans them (an
    empty token fails std::stoll; a trailing comma ends the scan).  A single
    value is broadcast to every axis; a count mismatch is CLI::ValidationError,
    a CLI11 ParseError -> exit 2 (senskit_main.cpp:40-41, 372-374)."""
    out = []
    pos = 0
    while pos < len(text):
        comma = text.find(",", pos)
        tok = text[pos:] if comma < 0 else text[pos:comma]
        out.append(_stoll(tok))
        if comma < 0:
            break
        pos = comma + 1
    if len(out) == 1 and rank > 1:
        out = out * rank
    if rank and len(out) != rank:
        raise argparse.ArgumentTypeError(f"expected {rank} comma-separated extents")
    return tuple(out)


def extract_calibration(data: np.ndarray, size: tuple):  # types.cpp:58-90
    from .api import Calib, DimError
    dims = data.shape[1:]
    if len(size) != len(dims):
        raise DimError("calibration size rank does not match stack")
    for a, (e, n) in enumerate(zip(size, dims)):
        if e < 1 or e > n:
            raise DimError(f"calibration size exceeds stack extent on axis {a}")
    start = [n // 2 - e // 2 for e, n in zip(size, dims)]
    sl = (slice(None),) + tuple(slice(s, s + e) for s, e in zip(start, size))
    return Calib(np.ascontiguousarray(data[sl]), tuple(e // 2 for e in size))


def config_from_flags(a):  # senskit_main.cpp:54-76 (both presets run on the GPU)
    from .api import ELLIPSOID, GRID_FULL, GRID_REDUCED, RECT, PipelineConfig
    if a.preset == "baseline":
        cfg = PipelineConfig.baseline()
    elif a.preset == "pisco":
        cfg = PipelineConfig.pisco()
    else:
        raise argparse.ArgumentTypeError(f"unknown preset '{a.preset}'")
    if a.kernel:
        cfg.kernel = RECT if a.kernel == "rect" else ELLIPSOID
    if a.gram:
        cfg.gram = 0 if a.gram == "explicit" else 1
    if a.grid:
        cfg.grid = GRID_FULL if a.grid == "full" else GRID_REDUCED
    if a.eig:
        cfg.eig = 0 if a.eig == "dense" else 1
    if a.method:
        cfg.method = 0 if a.method == "nullspace" else 1
    if a.field:
        cfg.field = 0 if a.field == "naive" else 1
    if a.tau >= 0:
        cfg.tau = a.tau
    if a.power_iters > 0:
        cfg.power_iters = a.power_iters
    if a.nullspace_threshold > 0:
        cfg.nullspace_threshold = a.nullspace_threshold
    if a.mask_threshold >= 0:
        cfg.mask_threshold = a.mask_threshold
    if a.apod_width != 0:
        cfg.apod_width = a.apod_width
    if a.grid_pad >= 0:
        cfg.grid_pad = a.grid_pad
    return cfg


def run_estimate(a) -> int:
    from . import api
    from .cstack import IoError, Stack, load_stack, save_pgm16, save_stack
    stack = load_stack(a.input)
    if stack.domain != "kspace":
        raise IoError("estimate expects a k-space stack, got an image-domain one")
    calib_size = parse_extents(a.calib, len(stack.dims))
    calib = extract_calibration(stack.data, calib_size)
    cfg = config_from_flags(a)
    ctx = api.Context(a.device)
    # the reference writes all n singular values (senskit_main.cpp:160-166): full spectrum requested
    result = api.estimate_maps(calib, stack.dims, cfg, ctx, want_spectrum=True)
    residual = api.projection_residual(stack.data, result.maps, ctx)

    save_stack(Stack(result.maps, "image"), a.output + "_maps")
    save_stack(Stack(result.support_mask.astype(np.complex64)[None], "image"), a.output + "_mask")
    save_stack(Stack(result.lambda_min_map.astype(np.complex64)[None], "image"), a.output + "_lambda")
    if len(stack.dims) == 2:
        for q in range(result.maps.shape[0]):
            save_pgm16(np.abs(result.maps[q]), f"{a.output}_mag_ch{q:02d}.pgm")
    spec = result.spectrum_normalized
    try:
        with open(a.output + "_spectrum.csv", "w") as f:
            f.write("index,sigma_normalized\n")
            for i, v in enumerate(spec):
                f.write(f"{i},{v!r}\n")
        prov = {
            "subcommand": "estimate", "input": a.input, "output": a.output, "preset": a.preset,
            "calib": list(calib_size), "full_dims": list(stack.dims), "grid_dims": list(result.grid_dims),
            "channels": int(stack.channels), "support_size": result.support_size,
            "nullspace_rank": result.nullspace_rank, "sigma1": result.sigma1, "cut_margin": result.cut_margin,
            "spectrum_normalized": [float(x) for x in spec], "zeroed_voxels": result.zeroed_voxels,
            "stages": {k: {"seconds": v / 1e3} for k, v in result.stage_ms.items()},
            "total_seconds": result.total_ms / 1e3, "residual": residual,
            "config": {"kernel": "rect" if cfg.kernel == api.RECT else "ellipsoid", "tau": cfg.tau,
                       "nullspace_threshold": cfg.nullspace_threshold,
                       "grid": "full" if cfg.grid == api.GRID_FULL else "reduced", "grid_pad": cfg.grid_pad,
                       "power_iters": cfg.power_iters, "mask_threshold": cfg.mask_threshold,
                       "apod_width": cfg.apod_width},
            "device": {"solver": result.extra, "device_index": a.device},
        }
        with open(a.output + "_provenance.json", "w") as f:
            f.write(json.dumps(prov, indent=2) + "\n")
    except OSError as e:
        raise IoError(str(e)) from None
    print(f"R={result.nullspace_rank} residual={residual} grid={int(np.prod(result.grid_dims))} voxels")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="senskit-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    est = sub.add_parser("estimate", help="estimate sensitivity maps from k-space data")
    est.add_argument("--input", required=True, help="input k-space stack")
    est.add_argument("--calib", required=True, help="calibration extents, e.g. 24,24")
    est.add_argument("--preset", default="pisco", help="baseline|pisco")
    est.add_argument("--kernel", choices=["rect", "ellipsoid"])
    est.add_argument("--tau", type=int, default=-1)
    est.add_argument("--gram", choices=["explicit", "fft"])
    est.add_argument("--nullspace-threshold", type=float, default=-1)
    est.add_argument("--grid", choices=["full", "reduced"])
    est.add_argument("--grid-pad", type=int, default=-1)
    est.add_argument("--eig", choices=["dense", "power"])
    est.add_argument("--power-iters", type=int, default=-1)
    est.add_argument("--method", choices=["nullspace", "espirit"])
    est.add_argument("--field", choices=["naive", "fast"])
    est.add_argument("--mask-threshold", type=float, default=-1)
    est.add_argument("--apod-width", type=float, default=0.0)
    est.add_argument("--threads", type=int, default=0, help="accepted for compatibility (GPU path)")
    est.add_argument("--device", type=int, default=0, help="CUDA device")
    est.add_argument("--output", required=True, help="output prefix")
    return ap


def main(argv=None) -> int:  # senskit_main.cpp:371-388
    from . import api
    from .cstack import IoError
    ap = build_parser()
    args = ap.parse_args(argv)  # bad flags: argparse exits with 2
    try:
        if args.cmd == "estimate":
            return run_estimate(args)
        return EXIT_FLAGS
    except argparse.ArgumentTypeError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_FLAGS
    except IoError as e:
        print(f"I/O error: {e}", file=sys.stderr)
        return EXIT_IO
    except api.NullspaceEmptyError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_NULLSPACE
    except api.DimError as e:
        print(f"shape error: {e}", file=sys.stderr)
        return EXIT_SHAPE
    except Exception as e:  # noqa: BLE001 - the reference maps every other exception to 1
        print(f"error: {e}", file=sys.stderr)
        return EXIT_OTHER


if __name__ == "__main__":
    sys.exit(main())

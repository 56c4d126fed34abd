"""Config-scale parity: the B200 pipeline against the FP64 oracle on the
BASELINE configs at their full sizes (test-side tool; the oracle is the
checker here, never the measured path).

usage: python tools/parity_configs.py C4 [--slices a:b] [--out FILE]

One JSON line per slice: nullspace rank (GPU vs oracle), cut margin, maps NRMSE
inside the oracle's support mask after coil-0 phase alignment, lambda errors
(norm-wise, pointwise inside the mask and everywhere), mask agreement, GPU and
oracle wall time.  Tolerances are BASELINE.json's (tests/parity.py).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2302_13431_b200 as K  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2302_13431_b200 import phantom  # noqa: E402
from tests import parity as PM  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--slices", default=None, help="a:b slice block (C3)")
    ap.add_argument("--out", default=None)
    ap.add_argument("--solver", default="bench", choices=["bench", "full"],
                    help="bench: the nullspace solver bench.py runs (auto -> subspace, no spectrum); full: cuSOLVER")
    args = ap.parse_args()
    sr = tuple(int(x) for x in args.slices.split(":")) if args.slices else None
    case = phantom.generate(args.config, slice_range=sr)
    spec = case.spec
    grid = tuple(spec.grid_dims) if spec.ndim == 3 else None
    ck = K.PipelineConfig(kernel=spec.kernel, tau=spec.tau, nullspace_threshold=spec.nullspace_threshold,
                          power_iters=spec.power_iters, grid=K.GRID_FULL if spec.full_grid else K.GRID_REDUCED,
                          grid_pad=spec.grid_dims[0] - spec.calib[0], grid_dims=grid)
    co = O.PipelineConfig.pisco()
    co.kernel, co.tau, co.nullspace_threshold = spec.kernel, spec.tau, spec.nullspace_threshold
    co.power_iters = spec.power_iters
    co.grid = O.GRID_FULL if spec.full_grid else O.GRID_REDUCED
    co.grid_pad = spec.grid_dims[0] - spec.calib[0]
    out = open(args.out, "a") if args.out else sys.stdout
    first = sr[0] if sr else 0
    for i, cal in enumerate(case.calib):
        t0 = time.time()
        res = K.estimate_maps(K.Calib(cal, case.center_offset), spec.full_dims, ck,
                              want_spectrum=args.solver == "full")
        t1 = time.time()
        ref = O.estimate_maps(O.Calib(cal.astype(np.complex128), case.center_offset), spec.full_dims, co,
                              grid_dims=grid)
        t2 = time.time()
        lam = PM.lambda_errors(res.lambda_min_map, ref.lambda_min_map, ref.support_mask)
        rec = {
            "config": args.config, "slice": first + i, "grid": list(spec.grid_dims), "full": list(spec.full_dims),
            "rank_gpu": int(res.nullspace_rank), "rank_oracle": int(ref.nullspace_rank),
            "cut_margin": float(res.cut_margin), "solver": res.extra,
            "maps_nrmse_in_mask": PM.maps_nrmse(res.maps, ref.maps, ref.support_mask),
            "lambda": lam, "mask_agree": float(np.mean(res.support_mask == ref.support_mask)),
            "mask_fraction": float(np.mean(ref.support_mask)),
            "gpu_s": t1 - t0, "oracle_s": t2 - t1,
        }
        rec["pass"] = bool(rec["rank_gpu"] == rec["rank_oracle"] and rec["maps_nrmse_in_mask"] < PM.TOL_MAPS
                           and lam["normwise"] < PM.TOL_LAMBDA
                           and lam.get("pointwise_max_in_mask", 0.0) < PM.TOL_LAMBDA)
        out.write(json.dumps(rec) + "\n")
        out.flush()
        del ref, res


if __name__ == "__main__":
    main()

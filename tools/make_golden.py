"""Golden fixtures for config-scale parity (test infrastructure).

usage: python tools/make_golden.py [C1 C2 C3 C4 C5] [--threads 8]

For each BASELINE config (C3: slices 0, 64 and 127 of 128) this runs the
REFERENCE ITSELF — oracle/_ref, the unmodified /root/reference/proj/src
sources compiled against oracle/ref_shim — through its staged pipeline
(maps.cpp:265-330, explicit grid via maps.hpp:117-123 for C4) on the seeded
synthetic calibration of paper_2302_13431_b200/phantom.py, and stores in
tests/golden/<config>[_s<slice>].npz:

* the calibration input itself (complex64, exactly what the GPU path reads;
  promoted to complex128 for the reference as io.cpp:66-67 does) + sha256;
* nullspace rank R, sigma_1 and the head of the normalised spectrum (the
  signal part plus 32 values past the cut);
* ||Gram||_F and 4096 + 256 sampled Gram entries (random + diagonal);
* ||G(x)||_F over the map grid and 8192 sampled G(x) entries (voxel, row, col),
  taken before the eigensolve consumes the field;
* the native-grid lambda (RawMaps::lambda) at up to 8192 grid voxels;
* final maps (Q x 2048 voxels), lambda_min_map and support_mask at 2048
  uniformly drawn full-resolution voxels.

The fixtures are generated here (the reference tree only exists in this
container) and committed; the -m gpu test tests/test_config_parity.py reads
them on the GPU box.
"""
import argparse
import hashlib
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import ref as R  # noqa: E402
from paper_2302_13431_b200 import phantom  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
C3_SLICES = (0, 64, 127)


def fixture_names(cfg):
    return [f"C3_s{s}" for s in C3_SLICES] if cfg == "C3" else [cfg]


def ref_config(spec):
    c = R.PipelineConfig.pisco()
    c.kernel, c.tau, c.nullspace_threshold = spec.kernel, spec.tau, spec.nullspace_threshold
    c.power_iters = spec.power_iters
    c.grid = R.GRID_FULL if spec.full_grid else R.GRID_REDUCED
    c.grid_pad = spec.grid_dims[0] - spec.calib[0]
    return c


def make(cfg, slice_index=0):
    sr = (slice_index, slice_index + 1) if cfg == "C3" else None
    case = phantom.generate(cfg, slice_range=sr)
    spec = case.spec
    cal = np.ascontiguousarray(case.calib[0], dtype=np.complex64)
    q = spec.channels
    lam = R.make_support(spec.kernel, spec.tau, spec.ndim).shape[0]
    n = q * lam
    ngrid = int(np.prod(spec.grid_dims))
    nfull = int(np.prod(spec.full_dims))
    rng = np.random.default_rng(20260 + 7 * slice_index + int(cfg[1]))
    gram_idx = np.concatenate([rng.integers(0, n, size=(4096, 2)),
                               np.repeat(rng.choice(n, min(n, 256), replace=False)[:, None], 2, 1)]).astype(np.int64)
    field_idx = np.stack([rng.integers(0, ngrid, 8192), rng.integers(0, q, 8192), rng.integers(0, q, 8192)],
                         1).astype(np.int64)
    rawl_idx = np.arange(ngrid) if ngrid <= 8192 else np.sort(rng.choice(ngrid, 8192, replace=False))
    vox_idx = np.sort(rng.choice(nfull, 2048, replace=False)).astype(np.int64)
    t = time.time()
    r = R.estimate_sampled(R.Calib(cal.astype(np.complex128), case.center_offset), spec.full_dims, ref_config(spec),
                           grid_dims=spec.grid_dims if spec.ndim == 3 else None, gram_idx=gram_idx,
                           field_idx=field_idx, vox_idx=vox_idx)
    secs = time.time() - t
    k = n - r["rank"]
    sig = r["spectrum_normalized"]
    cut = spec.nullspace_threshold
    margin = float(np.min(np.abs(sig - cut)) / cut)
    return dict(
        config=cfg, slice=slice_index, calib=cal, calib_sha256=hashlib.sha256(cal.tobytes()).hexdigest(),
        center_offset=np.asarray(case.center_offset, dtype=np.int64),
        full_dims=np.asarray(spec.full_dims, dtype=np.int64), grid_dims=np.asarray(spec.grid_dims, dtype=np.int64),
        channels=q, tau=spec.tau, kernel=spec.kernel, power_iters=spec.power_iters,
        nullspace_threshold=spec.nullspace_threshold, support_size=lam,
        rank=r["rank"], sigma1=r["sigma1"], spectrum_head=sig[: min(n, k + 32)], cut_margin=margin,
        gram_idx=gram_idx.astype(np.int32), gram_vals=r["gram_vals"], gram_fro=r["gram_fro"],
        field_idx=field_idx.astype(np.int32), field_vals=r["field_vals"], field_fro=r["field_fro"],
        rawl_idx=rawl_idx.astype(np.int32), rawl_vals=r["raw_lambda"].ravel()[rawl_idx],
        vox_idx=vox_idx.astype(np.int32), maps=r["maps"].astype(np.complex64), lam=r["lambda"], mask=r["mask"],
        ref_stage_seconds=np.asarray([r["stages"][s] for s in R.STAGES]), ref_seconds=secs,
        generator="oracle/_ref (unmodified reference sources + oracle/ref_shim), tools/make_golden.py",
    )


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    args = ap.parse_args()
    R.set_max_threads(args.threads)
    R.set_lapack_threads(args.threads)  # fixture generation only; the timed reference arm keeps 1
    os.makedirs(OUT, exist_ok=True)
    for cfg in args.configs:
        for name, sl in zip(fixture_names(cfg), C3_SLICES if cfg == "C3" else (0,)):
            d = make(cfg, sl)
            np.savez_compressed(os.path.join(OUT, name + ".npz"), **d)
            print(f"{name}: R={d['rank']} margin={d['cut_margin']:.4f} ref {d['ref_seconds']:.1f}s "
                  f"stages {np.round(d['ref_stage_seconds'], 2).tolist()}", flush=True)


if __name__ == "__main__":
    main()

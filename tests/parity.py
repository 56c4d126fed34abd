"""Parity metrics shared by the GPU tests, smoke() and bench (test-side code).

Tolerances are BASELINE.json north_star's:
  * Gram and G(x): relative Frobenius error <= 1e-4
  * per-voxel eigenvalues: relative error <= 1e-4 (norm-wise over voxels;
    the pointwise distribution is reported beside it)
  * maps: NRMSE <= 1e-3 inside the oracle's support mask after per-voxel
    phase alignment to coil 0
  * nullspace rank R: identical
"""
import numpy as np

TOL_GRAM = 1e-4
TOL_FIELD = 1e-4
TOL_LAMBDA = 1e-4
TOL_MAPS = 1e-3


def rel_fro(a, b):
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def align_coil0(m):
    """Per-voxel phase alignment to coil 0: m * conj(m_0)/|m_0| (m is (Q, ...))."""
    m = np.asarray(m, dtype=np.complex128).reshape(m.shape[0], -1)
    ph = m[0] / np.maximum(np.abs(m[0]), 1e-300)
    return m * np.conj(ph)[None]


def maps_nrmse(gpu, ref, mask):
    g = align_coil0(gpu)
    r = align_coil0(ref)
    sel = np.asarray(mask).reshape(-1) > 0
    if not sel.any():
        return 0.0
    return float(np.linalg.norm(g[:, sel] - r[:, sel]) / max(np.linalg.norm(r[:, sel]), 1e-300))


def lambda_errors(gpu, ref, mask=None):
    g = np.asarray(gpu, dtype=np.float64).ravel()
    r = np.asarray(ref, dtype=np.float64).ravel()
    normwise = float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300))
    rel = np.abs(g - r) / np.maximum(np.abs(r), 1e-300)
    out = {"normwise": normwise, "pointwise_max": float(rel.max()), "pointwise_p99": float(np.quantile(rel, 0.99)),
           "pointwise_median": float(np.median(rel)), "abs_max": float(np.abs(g - r).max())}
    if mask is not None:
        sel = np.asarray(mask).ravel() > 0
        if sel.any():
            out["pointwise_max_in_mask"] = float(rel[sel].max())
    return out

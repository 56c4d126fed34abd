"""Pins the FP64 restatement (oracle/, "port") to the reference itself.

oracle/_ref is the UNMODIFIED /root/reference/proj/src hot-path sources
(types, kernels, fft, calibration, nullspace, spatial_gram, eigensolve, maps,
synthetic, metrics) compiled by oracle/Makefile.ref against the Eigen-subset
shim in oracle/ref_shim.  Every entry point the GPU tests use as their checker
is called on both libraries with the same inputs; they must agree to FP64
roundoff (measured: bit for bit on every case here).  With this, the GPU
parity tests (which check against the port, or against golden fixtures the
reference build generated, tests/golden/) are pinned to the reference.
"""
import numpy as np
import pytest

from tests import parity as PM

TOL = 1e-12


def rnd(shape, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal(shape) + 1j * r.standard_normal(shape)


def sim_calib(R, q, dims, seed=3):
    """Calibration block of a reference-generated scene (synthetic.cpp:70-171):
    band-limited maps, so the Gram has a genuine nullspace."""
    full = tuple(max(2 * d, 24) for d in dims)
    k = R.simulate(q, full, 2, seed, 1, 1e-4, seed + 1)["kspace"]
    return R.extract_calibration(k, dims)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


@pytest.fixture(scope="module")
def P(O):
    return O


@pytest.mark.parametrize("nd", [1, 2, 3])
@pytest.mark.parametrize("tau", [0, 1, 3, 5])
@pytest.mark.parametrize("shape", [0, 1])
def test_support(P, R, nd, tau, shape):  # kernels.cpp:7-35
    assert np.array_equal(P.make_support(shape, tau, nd), R.make_support(shape, tau, nd))


def test_extract_calibration(P, R):  # types.cpp:58-90
    x = rnd((3, 40, 33), 1)
    for size in [(24, 24), (23, 24), (40, 33)]:
        a, b = P.extract_calibration(x, size), R.extract_calibration(x, size)
        assert np.array_equal(a.data, b.data) and a.center_offset == b.center_offset


@pytest.mark.parametrize("dims", [(5,), (12, 24), (7, 11), (4, 5, 6), (64, 64), (9, 16, 8)])
def test_fft_ops(P, R, dims):  # fft.cpp:37-112
    x = rnd(dims, 2)
    for op in ["fwd", "inv", "fftshift", "ifftshift", "image_to_kspace", "kspace_to_image",
               "image_to_kspace_unitary", "kspace_to_image_unitary"]:
        assert rel(P.fft_op(x, op), R.fft_op(x, op)) <= TOL, op


CASES = [  # (Q, calib dims, shape, tau)
    (3, (12, 12), 1, 2), (2, (14, 16), 0, 2), (4, (24, 24), 1, 3), (2, (9, 10, 8), 1, 2), (8, (24, 24), 1, 3),
]


@pytest.mark.parametrize("case", CASES)
def test_gram_nullspace_field_chain(P, R, case):
    """gram_fft / gram_explicit (calibration.cpp:30-144), extract_nullspace
    (nullspace.cpp:7-35), aggregate_w (spatial_gram.cpp:87-94), gram_field_fast /
    naive (:33-148) on the same inputs."""
    q, dims, shape, tau = case
    c = sim_calib(R, q, dims)
    cal, co = c.data, c.center_offset
    for gm in ("gram_fft", "gram_explicit"):
        a = getattr(P, gm)(P.Calib(cal, co), shape, tau)
        b = getattr(R, gm)(R.Calib(cal, co), shape, tau)
        assert rel(a, b) <= TOL, gm
    g = R.gram_fft(R.Calib(cal, co), shape, tau)
    na, nb = P.extract_nullspace(g, 0.05), R.extract_nullspace(g, 0.05)
    assert na.rank == nb.rank
    assert rel(na.spectrum, nb.spectrum) <= TOL
    wa, wb = P.aggregate_w(na.filters), R.aggregate_w(nb.filters)
    assert rel(wa, wb) <= 1e-11  # W is basis-invariant (test_nullspace.cpp:99-107)
    grid = tuple(d + 4 for d in dims)
    fa = P.gram_field_fast(wb, q, shape, tau, grid)
    fb = R.gram_field_fast(wb, q, shape, tau, grid)
    assert rel(fa, fb) <= TOL
    if len(dims) == 2:
        ha = P.gram_field_naive(nb.filters, q, shape, tau, grid)
        hb = R.gram_field_naive(nb.filters, q, shape, tau, grid)
        assert rel(ha, hb) <= TOL


def test_nullspace_errors_match(P, R):  # nullspace.cpp:9-12, 28-30
    eye = np.eye(6, dtype=np.complex128)
    for M in (P, R):
        with pytest.raises(M.NullspaceEmptyError):
            M.extract_nullspace(eye, 0.05)
        with pytest.raises(M.DimError):
            M.extract_nullspace(eye, 1.5)


@pytest.mark.parametrize("q", [1, 4, 8, 32])
def test_field_solvers(P, R, q):
    """espirit_inplace (spatial_gram.cpp:156-164), eig_power_field (eigensolve.cpp:40-74)
    incl. the restart/break rules, eig_dense_field (:9-38) both extremal pairs."""
    n = 37
    h = rnd((n, q, q), 4)
    field = np.einsum("nij,nkj->nik", h, h.conj())
    field[0] = 0.0                     # B ~ 0 voxel: break rule
    if q > 1:
        field[1] = np.eye(q) * 9.0     # identity: keeps the start vector
    ba, bb = P.espirit(field, 13), R.espirit(field, 13)
    assert rel(ba, bb) <= TOL
    for iters in (1, 10, 50):
        va, la = P.eig_power_field(bb, iters)
        vb, lb = R.eig_power_field(bb, iters)
        assert rel(va, vb) <= TOL and rel(la, lb) <= TOL
    for largest in (False, True):
        va, la, sa = P.eig_dense_field(field, largest)
        vb, lb, sb = R.eig_dense_field(field, largest)
        assert rel(la, lb) <= TOL and rel(sa, sb) <= TOL
        # eigenvectors up to a unit phase per voxel
        inner = np.sum(np.conj(vb) * va, axis=0)
        assert np.abs(np.abs(inner)[2:] - 1).max() < 1e-9


def test_normalize_and_interpolate(P, R):  # maps.cpp:54-176
    q, low, full = 4, (20, 24), (40, 48)
    raw = rnd((q,) + low, 5)
    raw[:, 0, 0] = 0.0
    cal = rnd((q, 12, 12), 6)
    for apod in (-1.0, 2.5):
        ma, za = P.normalize_maps(raw, P.Calib(cal, (6, 6)), apod)
        mb, zb = R.normalize_maps(raw, R.Calib(cal, (6, 6)), apod)
        assert za == zb and rel(ma, mb) <= TOL
    assert rel(P.interpolate_maps(raw, full), R.interpolate_maps(raw, full)) <= TOL
    lr = np.random.default_rng(7).random(low)
    assert rel(P.interpolate_real(lr, full), R.interpolate_real(lr, full)) <= TOL
    raw3 = rnd((2, 6, 8, 5), 8)
    assert rel(P.interpolate_maps(raw3, (12, 16, 10)), R.interpolate_maps(raw3, (12, 16, 10))) <= TOL


def _cfg(M, preset, **kw):
    c = M.PipelineConfig.pisco() if preset == "pisco" else M.PipelineConfig.baseline()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


PIPES = [
    ("pisco", {"tau": 3, "power_iters": 30, "grid_pad": 40}, (8, 24, 24), (64, 64), None),
    ("pisco", {"tau": 2, "power_iters": 10, "method": 1, "grid": 0}, (4, 16, 16), (32, 32), None),
    ("pisco", {"tau": 2, "power_iters": 10, "field": 0}, (4, 16, 16), (40, 40), None),
    ("baseline", {"tau": 2}, (4, 14, 14), (28, 28), None),
    ("baseline", {"tau": 2, "method": 1}, (4, 14, 14), (28, 28), None),
    ("pisco", {"tau": 2, "power_iters": 10}, (4, 10, 10, 10), (24, 24, 16), (16, 16, 12)),
]


@pytest.mark.parametrize("pipe", PIPES, ids=[f"p{i}" for i in range(len(PIPES))])
def test_estimate_maps(P, R, pipe):
    """estimate_maps (maps.cpp:265-330) end to end, both presets, the method /
    field / grid switches, an explicit 3-D grid (maps.hpp:117-123)."""
    preset, kw, cshape, full, grid = pipe
    c = sim_calib(R, cshape[0], cshape[1:], seed=9)
    cal, co = c.data, c.center_offset
    out = []
    for M in (P, R):
        out.append(M.estimate_maps(M.Calib(cal, co), full, _cfg(M, preset, **kw), grid_dims=grid, want_raw=True,
                                   want_gram=True))
    a, b = out
    assert a.nullspace_rank == b.nullspace_rank and a.grid_dims == b.grid_dims
    assert rel(a.gram, b.gram) <= TOL
    assert rel(a.raw_lambda, b.raw_lambda) <= 1e-10
    assert rel(a.lambda_min_map, b.lambda_min_map) <= 1e-10
    assert np.array_equal(a.support_mask, b.support_mask)
    assert PM.maps_nrmse(a.maps, b.maps, np.ones(b.support_mask.shape)) <= 1e-10
    assert a.zeroed_voxels == b.zeroed_voxels and abs(a.sigma1 - b.sigma1) <= TOL * b.sigma1


def test_estimate_maps_config_c1(P, R):
    """BASELINE config C1 at full size through the reference's own estimate_maps."""
    from paper_2302_13431_b200 import phantom
    case = phantom.generate("C1")
    spec = case.spec
    cal = case.calib[0].astype(np.complex128)
    out = []
    for M in (P, R):
        c = _cfg(M, "pisco", tau=spec.tau, power_iters=spec.power_iters, grid_pad=spec.grid_dims[0] - spec.calib[0])
        out.append(M.estimate_maps(M.Calib(cal, case.center_offset), spec.full_dims, c))
    a, b = out
    assert a.nullspace_rank == b.nullspace_rank
    assert rel(a.lambda_min_map, b.lambda_min_map) <= 1e-10
    assert np.array_equal(a.support_mask, b.support_mask)
    assert PM.maps_nrmse(a.maps, b.maps, b.support_mask) <= 1e-10


def test_simulate_and_residual(P, R):  # synthetic.cpp:70-171, metrics.cpp:11-49
    for kind in (0, 1):
        a = P.simulate(4, (24, 20), 2, 11, kind, 0.01, 5)
        b = R.simulate(4, (24, 20), 2, 11, kind, 0.01, 5)
        for k in b:
            assert rel(a[k], b[k]) <= TOL, k
    ks = b["kspace"]
    maps = b["true_maps"]
    ra, rb = P.projection_residual(ks, maps), R.projection_residual(ks, maps)
    assert abs(ra - rb) <= TOL * max(rb, 1e-30)

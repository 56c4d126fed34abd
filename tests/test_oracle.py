"""Pins the C++ FP64 oracle (oracle/) before it is trusted as the GPU checker.

Three kinds of evidence, since the reference ships no golden vectors
(SURVEY.md §8c): (1) the reference's own known-answer tests, re-asserted with
the reference file:line they come from — run against BOTH the restatement
(``port``) and the reference itself compiled from its unmodified sources
(``ref``, oracle/_ref, which also validates the Eigen-subset shim it is built
on); (2) an independent numpy restatement (tests/npref.py) on small cases;
(3) call-for-call equality of port and ref (tests/test_ref_pin.py).
"""
import numpy as np
import pytest

from tests import npref
from tests.conftest import load_ref


@pytest.fixture(scope="module", params=["port", "ref"])
def O(request):
    if request.param == "ref":
        return load_ref()
    from oracle import oracle
    oracle.lib()
    return oracle


def rnd(shape, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal(shape) + 1j * r.standard_normal(shape)


def rnd_orthonormal(rows, cols, seed):
    q, _ = np.linalg.qr(rnd((rows, cols), seed))
    return q


# ------------------------------------------------------------------ kernels
def test_support_sizes(O):  # test_kernels.cpp:30-37
    assert O.make_support(O.RECT, 3, 2).shape[0] == 49
    assert O.make_support(O.ELLIPSOID, 3, 2).shape[0] == 29
    d = O.make_support(O.RECT, 0, 2)
    assert d.shape == (1, 2) and (d == 0).all()


@pytest.mark.parametrize("nd", [1, 2, 3])
@pytest.mark.parametrize("tau", [0, 1, 2, 3])
@pytest.mark.parametrize("shape", [0, 1])
def test_support_membership_and_order(O, nd, tau, shape):  # test_kernels.cpp:39-75
    got = O.make_support(shape, tau, nd)
    want = npref.support(shape, tau, nd)
    assert np.array_equal(got, want)  # same set AND lexicographic order


def test_support_bad_args(O):  # test_kernels.cpp:83-86
    with pytest.raises(O.DimError):
        O.make_support(O.RECT, -1, 2)
    with pytest.raises(O.DimError):
        O.make_support(O.RECT, 1, 0)


# ---------------------------------------------------------------- grid core
def test_extract_calibration(O):  # test_grid_core.cpp:93-125
    parent = rnd((1, 256, 256), 7)
    reg = O.extract_calibration(parent, (24, 24))
    assert reg.center_offset == (12, 12)
    assert reg.data[0, 12, 12] == parent[0, 128, 128]
    full = O.extract_calibration(parent, (256, 256))
    assert np.array_equal(full.data, parent)
    twice = O.extract_calibration(reg.data, (24, 24))
    assert np.array_equal(twice.data, reg.data) and twice.center_offset == reg.center_offset
    odd = O.extract_calibration(parent, (23, 24))
    assert odd.center_offset == (11, 12) and odd.data[0, 11, 12] == parent[0, 128, 128]
    with pytest.raises(O.DimError):
        O.extract_calibration(parent, (257, 256))


# ---------------------------------------------------------------------- fft
@pytest.mark.parametrize("dims", [(5,), (6, 9), (12, 24), (72,), (4, 5, 6), (256, 64), (7, 11)])
def test_fft_matches_numpy(O, dims):
    x = rnd(dims, 1)
    f = np.fft.fftn(x)
    assert np.abs(O.fft_op(x, "fwd") - f).max() < 1e-12 * np.abs(f).max()
    assert np.abs(O.fft_op(x, "inv") - np.fft.ifftn(x) * x.size).max() < 1e-12 * np.abs(f).max()
    sh = np.fft.fftshift(x)
    assert np.array_equal(O.fft_op(x, "fftshift"), sh)
    assert np.array_equal(O.fft_op(sh, "ifftshift"), x)
    k = O.fft_op(x, "image_to_kspace")
    assert np.abs(O.fft_op(k, "kspace_to_image") - x).max() < 1e-12 * np.abs(x).max()
    ku = O.fft_op(x, "image_to_kspace_unitary")
    assert abs(np.sum(np.abs(ku) ** 2) - np.sum(np.abs(x) ** 2)) < 1e-10 * np.sum(np.abs(x) ** 2)


# -------------------------------------------------------------- calibration
def test_gram_explicit_matches_triple_loop(O):  # test_calibration.cpp:91-99
    cal = O.Calib(rnd((3, 12, 12), 6), (6, 6))
    g = O.gram_explicit(cal, O.RECT, 1)
    C = O.build_calib_matrix(cal, O.RECT, 1)
    want = C.conj().T @ C
    assert np.linalg.norm(g - want) / np.linalg.norm(want) < 1e-12
    assert C.shape == (100, 27)


def test_gram_fft_identity_kernel(O):  # test_calibration.cpp:118-126
    cal = O.Calib(rnd((1, 8, 8), 8), (4, 4))
    a = O.gram_fft(cal, O.RECT, 0)
    b = O.gram_explicit(cal, O.RECT, 0)
    assert a.shape == (1, 1) and abs(a[0, 0] - b[0, 0]) < 1e-12 * abs(b[0, 0])


def test_gram_fft_transform_counts(O):  # test_calibration.cpp:128-134
    O.fft_reset_counters()
    O.gram_fft(O.Calib(rnd((4, 24, 24), 9), (12, 12)), O.RECT, 3)
    assert O.fft_counters() == (4, 16)


def test_gram_fft_is_full_shift_gram(O):  # survey addition: gram_fft == C_full^H C_full
    for shape, tau, dims, q in [(1, 3, (24, 24), 3), (0, 2, (14, 16), 2), (1, 2, (9, 10, 8), 2)]:
        cal = O.Calib(rnd((q,) + dims, 11), tuple(d // 2 for d in dims))
        g = O.gram_fft(cal, shape, tau)
        C = npref.calib_full_matrix(cal.data, npref.support(shape, tau, len(dims)))
        want = C.conj().T @ C
        assert np.linalg.norm(g - want) / np.linalg.norm(want) < 1e-13


def test_gram_fft_same_lag_exact_and_deviation(O):  # test_calibration.cpp:136-167
    cal = O.Calib(rnd((2, 16, 16), 11), (8, 8))
    offs = O.make_support(O.RECT, 2, 2)
    g = O.gram_fft(cal, O.RECT, 2)
    lam = offs.shape[0]
    for s in range(lam - 1):
        for t in range(lam - 1):
            if np.array_equal(offs[s] - offs[t], offs[s + 1] - offs[t + 1]):
                assert g[lam + s, t] == g[lam + s + 1, t + 1]
    cal4 = O.Calib(rnd((4, 24, 24), 10), (12, 12))
    a, b = O.gram_fft(cal4, O.RECT, 3), O.gram_explicit(cal4, O.RECT, 3)
    rel = np.linalg.norm(a - b) / np.linalg.norm(b)
    assert 0 < rel < 1


def test_gram_block_hermitian_psd(O):  # test_calibration.cpp:169-185
    cal = O.Calib(rnd((3, 14, 14), 12), (7, 7))
    for g in (O.gram_fft(cal, O.ELLIPSOID, 2), O.gram_explicit(cal, O.ELLIPSOID, 2)):
        assert np.abs(g - g.conj().T).max() < 1e-12 * np.linalg.norm(g)
        w = np.linalg.eigvalsh(g)
        assert w.min() > -1e-10 * w.max()


def test_gram_too_small(O):  # test_calibration.cpp:76-80
    with pytest.raises(O.DimError):
        O.gram_fft(O.Calib(rnd((1, 6, 6), 3), (3, 3)), O.RECT, 3)


# ---------------------------------------------------------------- nullspace
def test_nullspace_diag(O):  # test_nullspace.cpp:22-34
    b = O.extract_nullspace(np.diag([4.0, 1.0, 1e-6]).astype(complex), 0.05)
    assert b.rank == 1
    assert np.allclose(b.spectrum, [2.0, 1.0, 1e-3])
    assert abs(abs(b.filters[2, 0]) - 1) < 1e-12 and abs(b.filters[0, 0]) < 1e-12


def test_nullspace_errors(O):  # test_nullspace.cpp:36-43
    with pytest.raises(O.NullspaceEmptyError):
        O.extract_nullspace(np.eye(4, dtype=complex), 0.05)
    for r in (0.0, 1.0):
        with pytest.raises(O.DimError):
            O.extract_nullspace(np.eye(2, dtype=complex), r)


def test_nullspace_annihilates(O):  # test_nullspace.cpp:45-72
    st = rnd((2, 12, 12), 21)
    st[1] = 1j * st[0]
    cal = O.Calib(st, (6, 6))
    C = O.build_calib_matrix(cal, O.RECT, 1)
    g = O.gram_explicit(cal, O.RECT, 1)
    b = O.extract_nullspace(g, 0.05)
    assert b.rank >= 1
    F = b.filters
    assert np.abs(F.conj().T @ F - np.eye(b.rank)).max() < 1e-10
    for r in range(b.rank):
        assert np.linalg.norm(C @ F[:, r]) / b.spectrum[0] < 0.05
        quad = np.real(F[:, r].conj() @ g @ F[:, r])
        assert quad <= (0.05 * b.spectrum[0]) ** 2 * (1 + 1e-6)


def test_w_basis_invariant_and_aggregate(O):  # test_nullspace.cpp:99-107, test_spatial_gram.cpp:123-145
    f = rnd_orthonormal(12, 4, 23)
    u = rnd_orthonormal(4, 4, 24)
    assert np.abs(O.aggregate_w(f) - O.aggregate_w(f @ u)).max() < 1e-12
    e1 = np.zeros((6, 1), complex)
    e1[0] = 1
    w = O.aggregate_w(e1)
    want = np.zeros((6, 6))
    want[0, 0] = 1
    assert np.array_equal(w, want)
    assert np.abs(O.aggregate_w(np.eye(8, dtype=complex)) - np.eye(8)).max() < 1e-14
    w = O.aggregate_w(rnd_orthonormal(12, 5, 34))
    assert abs(np.trace(w).real - 5) < 1e-10 and abs(np.trace(w).imag) < 1e-12


# ------------------------------------------------------------- spatial gram
@pytest.mark.parametrize("dims", [(8, 8), (5, 8), (4, 4)])
def test_field_fast_equals_naive_and_direct(O, dims):  # test_spatial_gram.cpp:160-170
    offs = O.make_support(O.RECT, 1, 2)
    lam = offs.shape[0]
    F = rnd_orthonormal(3 * lam, 6, 35)
    W = O.aggregate_w(F)
    fast = O.gram_field_fast(W, 3, O.RECT, 1, dims)
    naive = O.gram_field_naive(F, 3, O.RECT, 1, dims)
    scale = np.abs(naive).max()
    assert np.abs(fast - naive).max() < 1e-10 * scale
    direct = npref.field_direct(W, offs, 3, dims)
    for j in range(direct.shape[0]):
        for q in range(3):
            direct[j, q, q] = direct[j, q, q].real
    assert np.abs(fast - direct).max() < 1e-10 * scale


def test_field_dc_filter(O):  # test_spatial_gram.cpp:147-158
    lam = 9
    f = np.zeros((2 * lam, 1), complex)
    f[lam // 2, 0] = 1
    g = O.gram_field_fast(O.aggregate_w(f), 2, O.RECT, 1, (6, 6))
    assert np.abs(g[:, 0, 0] - 1).max() < 1e-12 and np.abs(g[:, 1, 0]).max() < 1e-12


def test_espirit_eigen_mapping(O):  # test_spatial_gram.cpp:183-229
    lam, q = 9, 3
    F = rnd_orthonormal(q * lam, 7, 36)
    g = O.gram_field_fast(O.aggregate_w(F), q, O.RECT, 1, (6, 6))
    b = O.espirit(g, lam)
    for j in range(g.shape[0]):
        eg = np.linalg.eigvalsh(g[j])
        eb = np.linalg.eigvalsh(b[j])
        assert np.allclose(eb, np.sort(1 - eg / lam), atol=1e-10)
        assert eg.min() / lam > -1e-8 and eg.max() / lam < 1 + 1e-6
    zero = np.zeros((4, q, q), complex)
    assert np.array_equal(O.espirit(zero, lam), np.broadcast_to(np.eye(q), (4, q, q)))


# ---------------------------------------------------------------- eigensolve
def test_power_contracts(O):  # test_eigensolve.cpp:67-77
    b = np.diag([1.0, 0.1]).astype(complex)[None]
    v, val = O.eig_power_field(b, 10)
    assert abs(abs(v[0, 0]) - 1) < 1e-9 and abs(val[0] - 1) < 1e-9


def test_power_identity_keeps_init(O):  # test_eigensolve.cpp:79-83
    v, _ = O.eig_power_field(np.eye(3, dtype=complex)[None], 10)
    assert np.abs(v[:, 0] - 1 / np.sqrt(3)).max() < 1e-12


def test_power_restart_and_break(O):  # eigensolve.cpp:56-66
    # all-ones annihilated -> restart from e_0
    b = np.array([[1, -1], [-1, 1]], dtype=complex)[None] / 2
    v, val = O.eig_power_field(b, 5)
    assert abs(abs(v[0, 0]) - 1 / np.sqrt(2)) < 1e-12 and abs(val[0] - 1) < 1e-12
    # zero matrix -> restart to e_0, still annihilated -> break keeping e_0, value 0
    v, val = O.eig_power_field(np.zeros((1, 3, 3), complex), 5)
    assert np.array_equal(v[:, 0], [1, 0, 0]) and val[0] == 0


def test_power_rayleigh_monotone_and_batched(O):  # test_eigensolve.cpp:85-117
    a = rnd((8, 3, 3), 47)
    field = np.einsum("jkp,jkq->jpq", a.conj(), a)
    prev = np.full(8, -1e300)
    for it in range(1, 11):
        _, val = O.eig_power_field(field, it)
        assert (val >= prev - 1e-12).all()
        prev = val
    m = rnd((17, 3, 3), 53)
    herm = (m + m.conj().transpose(0, 2, 1)) / 2
    vb, valb = O.eig_power_field(herm, 10)
    for j in range(17):
        vs, vals = O.eig_power_field(herm[j:j + 1], 10)
        assert np.abs(vb[:, j] - vs[:, 0]).max() < 1e-12 and abs(valb[j] - vals[0]) < 1e-12
    O.set_max_threads(1)
    vser, _ = O.eig_power_field(herm, 10)
    O.set_max_threads(0)
    assert np.abs(vb - vser).max() < 1e-12


def test_power_matches_numpy(O):
    m = rnd((40, 5, 5), 3)
    herm = (m + m.conj().transpose(0, 2, 1)) / 2 + 3 * np.eye(5)
    v, val = O.eig_power_field(herm, 12)
    vn, valn = npref.power(herm, 12)
    assert np.abs(v.T - vn).max() < 1e-12 and np.abs(val - valn).max() < 1e-12


def test_dense_field(O):  # test_eigensolve.cpp:37-65
    d = np.diag([3.0, 1.0, 0.01]).astype(complex)[None]
    v, val, sec = O.eig_dense_field(d, largest=False)
    assert abs(val[0] - 0.01) < 1e-12 and abs(sec[0] - 1) < 1e-12 and abs(abs(v[2, 0]) - 1) < 1e-12


# --------------------------------------------------------------------- maps
def test_interpolation(O):  # test_maps.cpp:25-55
    low = np.zeros((2, 8, 8), complex)
    low[0] = 0.3 - 0.2j
    low[1] = -1.1 + 0.4j
    up = O.interpolate_maps(low, (32, 32))
    assert np.abs(up[0] - (0.3 - 0.2j)).max() < 1e-12 and np.abs(up[1] - (-1.1 + 0.4j)).max() < 1e-12
    x = rnd((2, 9, 12), 61)
    assert np.abs(O.interpolate_maps(x, (9, 12)) - x).max() < 1e-12
    lo = O.simulate(2, (24, 24), 2, 63)["true_maps"]
    fine = O.simulate(2, (72, 72), 2, 63)["true_maps"]
    assert np.abs(O.interpolate_maps(lo, (72, 72)) - fine).max() < 1e-6
    with pytest.raises(O.DimError):
        O.interpolate_maps(rnd((1, 8, 8), 64), (4, 8))


def test_interpolation_matches_sinc_matrix(O):
    x = rnd((3, 10, 12), 5)
    full = (40, 36)
    got = O.interpolate_maps(x, full)
    out = x
    for a, (nl, nf) in enumerate(zip(x.shape[1:], full)):
        # spec = image_to_kspace (x 1/n), then kspace_to_image on the padded grid
        fwd = npref.centered_dft_matrix(nl, nl, nl // 2, nl // 2, -1, 1.0 / nl)
        inv = np.exp(2j * np.pi * (np.arange(nf)[:, None] - nf // 2) * (np.arange(nl)[None, :] - nl // 2) / nf)
        mat = inv @ fwd
        out = np.moveaxis(np.tensordot(out, mat, axes=([a + 1], [1])), -1, a + 1)
    assert np.abs(got - out).max() < 1e-11
    lr = np.random.default_rng(1).random((10, 12))
    assert np.abs(O.interpolate_real(lr, full) - O.interpolate_maps(lr[None].astype(complex), full)[0].real).max() < 1e-15


def test_normalization(O):  # test_maps.cpp:67-106
    q = 3
    maps = np.full((q, 6, 6), 1 / np.sqrt(3), complex)
    dc = O.Calib(np.ones((q, 1, 1), complex), (0, 0))
    out, z = O.normalize_maps(maps, dc)
    assert np.abs(out - maps).max() < 1e-14 and z == 0
    raw = rnd((3, 8, 8), 65)
    cal = O.Calib(rnd((3, 1, 1), 66), (0, 0))
    beta = np.random.default_rng(67).uniform(0.5, 2, (8, 8)) * np.exp(1j * np.random.default_rng(68).uniform(0, 6.28, (8, 8)))
    a, _ = O.normalize_maps(raw, cal)
    b, _ = O.normalize_maps(raw * beta[None], cal)
    assert np.abs(a - b).max() < 1e-10
    m = np.zeros((2, 4, 4), complex)
    m[0, 0, 0] = 1
    out, z = O.normalize_maps(m, O.Calib(np.ones((2, 1, 1), complex), (0, 0)))
    assert z == 15 and abs(abs(out[0, 0, 0]) - 1) < 1e-14


def test_end_to_end_noiseless(O):  # test_maps.cpp:108-149
    sc = O.simulate(3, (32, 32), 1, 71)
    cal = O.extract_calibration(sc["kspace"], (16, 16))
    cfg = O.PipelineConfig.baseline()
    cfg.tau = 2
    cfg.nullspace_threshold = 0.005
    res = O.estimate_maps(cal, (32, 32), cfg)
    assert res.nullspace_rank >= 3
    est = res.maps.reshape(3, -1)
    tru = sc["true_maps"].reshape(3, -1)
    inside = sc["support_mask_true"].reshape(-1) > 0
    cosang = np.abs(np.sum(est.conj() * tru, 0)) / (np.linalg.norm(est, axis=0) * np.linalg.norm(tru, axis=0))
    assert np.arccos(np.minimum(1, cosang[inside])).max() < 1e-2
    m = res.support_mask.reshape(-1) > 0
    assert np.abs(np.sum(np.abs(est[:, m]) ** 2, 0) - 1).max() < 1e-8
    again = O.estimate_maps(cal, (32, 32), cfg)
    assert np.abs(again.maps - res.maps).max() < 1e-12


def test_pipeline_errors(O):  # test_maps.cpp:192-217
    st = rnd((2, 12, 12), 79)
    cfg = O.PipelineConfig.baseline()
    cfg.tau = 0
    with pytest.raises(O.NullspaceEmptyError):
        O.estimate_maps(O.extract_calibration(st, (12, 12)), (12, 12), cfg)
    cfg.tau = 4
    with pytest.raises(O.DimError):
        O.estimate_maps(O.extract_calibration(rnd((2, 8, 8), 80), (8, 8)), (8, 8), cfg)
    with pytest.raises(O.DimError):
        O.estimate_maps(O.extract_calibration(st, (12, 12)), (8, 8), O.PipelineConfig.baseline())


def test_acceptance_a1(O):  # acceptance_main.cpp:64-87
    worst = 0.0
    for seed in range(1, 21):
        q = 2 + seed % 3
        tau = 1 + seed % 2
        grid = 16 if seed % 2 else 8
        sc = O.simulate(q, (24, 24), 1, seed, noise_sigma=0.001, noise_seed=seed)
        cal = O.extract_calibration(sc["kspace"], (16, 16))
        b = O.extract_nullspace(O.gram_explicit(cal, O.RECT, tau), 0.05)
        fast = O.gram_field_fast(O.aggregate_w(b.filters), q, O.RECT, tau, (grid, grid))
        naive = O.gram_field_naive(b.filters, q, O.RECT, tau, (grid, grid))
        worst = max(worst, np.abs(fast - naive).max() / np.abs(naive).max())
    assert worst < 1e-10


def test_acceptance_a7_noiseless_recovery(O):  # acceptance_main.cpp:238-268
    sc = O.simulate(8, (128, 128), 2, 23)
    cfg = O.PipelineConfig.baseline()
    cfg.nullspace_threshold = 0.002
    cfg.mask_threshold = 5e-5
    res = O.estimate_maps(O.extract_calibration(sc["kspace"], (48, 48)), (128, 128), cfg)
    assert O.projection_residual(sc["kspace"], res.maps) < 1e-3
    m = res.support_mask.reshape(-1) > 0
    t = sc["support_mask_true"].reshape(-1) > 0
    assert 2 * np.sum(m & t) / (m.sum() + t.sum()) > 0.95


def test_pisco_pipeline_matches_numpy_restatement(O):
    """Whole pisco path on a small case against tests/npref.py (independent)."""
    sc = O.simulate(4, (32, 32), 1, 5, noise_sigma=0.01, noise_seed=6)
    cal = O.extract_calibration(sc["kspace"], (16, 16))
    cfg = O.PipelineConfig.pisco()
    cfg.tau = 2
    cfg.grid = O.GRID_FULL
    cfg.power_iters = 20
    res = O.estimate_maps(cal, (32, 32), cfg, want_raw=True, want_gram=True)
    offs = npref.support(1, 2, 2)
    C = npref.calib_full_matrix(cal.data, offs)
    G = C.conj().T @ C
    assert np.linalg.norm(res.gram - G) / np.linalg.norm(G) < 1e-13
    w, U = np.linalg.eigh(G)
    sig = np.sqrt(np.maximum(w, 0))
    R = int(np.sum(sig < 0.05 * sig.max()))
    assert R == res.nullspace_rank
    W = U[:, :R] @ U[:, :R].conj().T
    Gf = npref.field_direct(W, offs, 4, (32, 32))
    lam = offs.shape[0]
    B = np.eye(4)[None] - Gf / lam
    v, val = npref.power(B, 20)
    raw = res.raw_maps.reshape(4, -1).T
    # per-voxel phase: eigenvectors are defined up to a global phase per voxel
    ph = np.sum(vn := v.conj() * raw, 1)
    del vn
    ph = ph / np.abs(ph)
    assert np.abs(raw - v * ph[:, None]).max() < 1e-8
    assert np.abs(res.raw_lambda.reshape(-1) - (1 - val)).max() < 1e-10

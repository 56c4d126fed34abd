"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front end over ``oracle/lib/libsk_oracle.so``, the FP64 C++ restatement
of the reference ``senskit`` hot path (see ``oracle/sko.hpp``).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product package never imports it.

Names and argument meanings follow the reference entry points
(``proj/include/senskit/*.hpp``); arrays are numpy complex128 in the reference
layouts (channel-major stacks, column-major matrices, voxel-major GramField).
"""
from __future__ import annotations

import ctypes as C
import glob
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "lib", "libsk_oracle.so")
# The reference itself (unmodified /root/reference/proj/src compiled against
# oracle/ref_shim by oracle/Makefile.ref); `oracle.ref` binds this same API to it.
REF_LIB_PATH = os.path.join(_HERE, "_ref", "libsk_ref.so")

RECT, ELLIPSOID = 0, 1
EXPLICIT, FFT = 0, 1
GRID_FULL, GRID_REDUCED = 0, 1
EIG_DENSE, EIG_POWER = 0, 1
METHOD_NULLSPACE, METHOD_ESPIRIT = 0, 1
FIELD_NAIVE, FIELD_FAST = 0, 1
DISK, RECTANGLES = 0, 1

_ERRORS = {4: "NullspaceEmptyError", 5: "DimError", 3: "IoError", 6: "LengthError", 1: "RuntimeError"}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_ERRORS.get(code, 'Error')}: {msg}")
        self.code = code
        self.kind = _ERRORS.get(code, "Error")


class NullspaceEmptyError(OracleError):
    pass


class DimError(OracleError):
    pass


class LengthError(OracleError):
    pass


_KIND = {4: NullspaceEmptyError, 5: DimError, 6: LengthError}


class sko_config(C.Structure):
    _fields_ = [
        ("kernel", C.c_int32), ("tau", C.c_int32), ("gram", C.c_int32),
        ("nullspace_threshold", C.c_double),
        ("grid", C.c_int32), ("grid_pad", C.c_int64),
        ("eig", C.c_int32), ("power_iters", C.c_int32), ("method", C.c_int32), ("field", C.c_int32),
        ("mask_threshold", C.c_double), ("apod_width", C.c_double),
    ]


@dataclass
class PipelineConfig:
    """maps.hpp:23-45 defaults; ``baseline()`` / ``pisco()`` presets from maps.cpp:12-28."""
    kernel: int = RECT
    tau: int = 3
    gram: int = EXPLICIT
    nullspace_threshold: float = 0.05
    grid: int = GRID_FULL
    grid_pad: int = 24
    eig: int = EIG_DENSE
    power_iters: int = 10
    method: int = METHOD_NULLSPACE
    field: int = FIELD_FAST
    mask_threshold: float = 0.01
    apod_width: float = -1.0

    @staticmethod
    def baseline() -> "PipelineConfig":
        return PipelineConfig()

    @staticmethod
    def pisco() -> "PipelineConfig":
        return PipelineConfig(kernel=ELLIPSOID, gram=FFT, grid=GRID_REDUCED, eig=EIG_POWER)

    def to_c(self) -> sko_config:
        return sko_config(self.kernel, self.tau, self.gram, self.nullspace_threshold, self.grid,
                          self.grid_pad, self.eig, self.power_iters, self.method, self.field,
                          self.mask_threshold, self.apod_width)


def _find_lapack() -> str:
    env = os.environ.get("SKO_LAPACK")
    if env:
        return env
    import scipy  # noqa: F401  (only to locate its bundled OpenBLAS)
    base = os.path.dirname(os.path.dirname(os.path.abspath(scipy.__file__)))
    hits = sorted(glob.glob(os.path.join(base, "scipy.libs", "libscipy_openblas*.so")))
    if not hits:
        raise RuntimeError("scipy's bundled OpenBLAS not found; set SKO_LAPACK")
    return hits[0]


_VP, _I32, _I64, _D, _U64 = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_uint64
_SIGS = {
    "sko_init": [C.c_char_p],
    "sko_set_max_threads": [_I32], "sko_set_lapack_threads": [_I32],
    "sko_make_support": [_I32, _I32, _I32, _VP, _VP],
    "sko_extract_calibration": [_I32, _VP, _I64, _VP, _VP, _VP, _VP],
    "sko_fft": [_I32, _VP, _VP, _I32],
    "sko_fft_counters": [_VP, _VP],
    "sko_gram": [_I32, _I32, _VP, _VP, _I64, _VP, _I32, _I32, _VP],
    "sko_calib_matrix": [_I32, _VP, _I64, _VP, _I32, _I32, _VP, _VP, _VP],
    "sko_extract_nullspace": [_I64, _VP, _D, _VP, _VP, _VP],
    "sko_aggregate_w": [_I64, _I64, _VP, _VP],
    "sko_gram_field_fast": [_I64, _VP, _I32, _I32, _I32, _VP, _VP],
    "sko_gram_field_naive": [_I64, _I64, _VP, _I32, _I32, _I32, _VP, _VP],
    "sko_espirit_inplace": [_I64, _I64, _VP, _I64],
    "sko_eig_power_field": [_I64, _I64, _VP, _I32, _VP, _VP],
    "sko_eig_dense_field": [_I64, _I64, _VP, _I32, _VP, _VP, _VP],
    "sko_normalize_maps": [_I32, _VP, _I64, _VP, _VP, _VP, _VP, _D, _VP, _VP],
    "sko_interpolate_maps": [_I32, _VP, _I64, _VP, _VP, _VP],
    "sko_interpolate_real": [_I32, _VP, _VP, _VP, _VP],
    "sko_estimate_maps": [_I32, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                          _VP, _VP, _VP, _VP, _VP],
    "sko_simulate": [_I64, _I32, _VP, _I32, _U64, _I32, _D, _U64, _VP, _VP, _VP, _VP, _VP],
    "sko_projection_residual": [_I32, _VP, _I64, _VP, _VP, _VP],
}
# Only in oracle/_ref/libsk_ref.so (golden-fixture sampling, oracle/ref_capi.cpp).
_SIGS_REF = {
    "skr_estimate_sampled": [_I32, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _I64, _VP, _VP, _VP, _I64, _VP, _VP, _VP,
                             _VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP],
}


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"oracle library missing: {_LIB_PATH} (run `make oracle`)")
        L = C.CDLL(_LIB_PATH)
        L.sko_last_error.restype = C.c_char_p
        L.sko_max_threads.restype = C.c_int
        for name, args in list(_SIGS.items()) + list(_SIGS_REF.items()):
            if not hasattr(L, name):
                continue
            getattr(L, name).argtypes = args
            if name not in ('sko_set_max_threads', 'sko_set_lapack_threads', 'sko_fft_counters'):
                getattr(L, name).restype = C.c_int
        rc = L.sko_init(_find_lapack().encode())
        if rc != 0:
            raise RuntimeError(L.sko_last_error().decode())
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        msg = lib().sko_last_error().decode()
        raise _KIND.get(rc, OracleError)(rc, msg)


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _i64(seq):
    return np.ascontiguousarray(np.asarray(seq, dtype=np.int64))


def _c128(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def set_max_threads(n: int) -> None:
    lib().sko_set_max_threads(int(n))


def max_threads() -> int:
    return int(lib().sko_max_threads())


def set_lapack_threads(n: int) -> None:
    lib().sko_set_lapack_threads(int(n))


# ---------------------------------------------------------------- kernels.cpp
def make_support(shape: int, tau: int, ndim: int) -> np.ndarray:
    """kernels.cpp:7-35 — |Lambda| x D int offsets, lexicographic."""
    cap = max(1, (2 * tau + 1) ** max(ndim, 1) * max(ndim, 1))
    buf = np.zeros(cap, dtype=np.int32)
    cnt = C.c_int64(0)
    _check(lib().sko_make_support(int(shape), int(tau), int(ndim), _p(buf), C.byref(cnt)))
    return buf[: cnt.value * ndim].reshape(cnt.value, ndim).copy()


# ------------------------------------------------------------------ types.cpp
@dataclass
class Calib:
    """CalibrationRegion (types.hpp:79-85): data is (Q, *dims) complex128."""
    data: np.ndarray
    center_offset: tuple

    @property
    def dims(self):
        return tuple(self.data.shape[1:])

    @property
    def channels(self):
        return self.data.shape[0]


def extract_calibration(stack: np.ndarray, size) -> Calib:
    """types.cpp:58-90; stack is (Q, *dims)."""
    stack = _c128(stack)
    q, dims = stack.shape[0], stack.shape[1:]
    nd = len(dims)
    out = np.zeros((q,) + tuple(size), dtype=np.complex128)
    co = np.zeros(nd, dtype=np.int64)
    _check(lib().sko_extract_calibration(nd, _p(_i64(dims)), q, _p(stack), _p(_i64(size)), _p(out), _p(co)))
    return Calib(out, tuple(int(c) for c in co))


# -------------------------------------------------------------------- fft.cpp
_FFT_OPS = {"fwd": 0, "inv": 1, "fftshift": 2, "ifftshift": 3, "image_to_kspace": 4,
            "kspace_to_image": 5, "image_to_kspace_unitary": 6, "kspace_to_image_unitary": 7}


def fft_op(x: np.ndarray, op: str) -> np.ndarray:
    a = _c128(x).copy()
    _check(lib().sko_fft(a.ndim, _p(_i64(a.shape)), _p(a), _FFT_OPS[op]))
    return a


def fft_counters():
    f, i = C.c_int64(0), C.c_int64(0)
    lib().sko_fft_counters(C.byref(f), C.byref(i))
    return f.value, i.value


def fft_reset_counters():
    lib().sko_fft_reset_counters()


# ------------------------------------------------------------ calibration.cpp
def _gram(method, calib: Calib, shape, tau):
    d = _c128(calib.data)
    q, dims = d.shape[0], d.shape[1:]
    lam = make_support(shape, tau, len(dims)).shape[0]
    n = q * lam
    g = np.zeros((n, n), dtype=np.complex128, order="F")
    _check(lib().sko_gram(method, len(dims), _p(_i64(dims)), _p(_i64(calib.center_offset)), q, _p(d),
                          int(shape), int(tau), g.ctypes.data_as(C.c_void_p)))
    return g


def gram_fft(calib: Calib, shape: int, tau: int) -> np.ndarray:
    """calibration.cpp:80-144 — (Q|L|)^2 Hermitian Gram, returned as a numpy array (column-major storage)."""
    return _gram(FFT, calib, shape, tau)


def gram_explicit(calib: Calib, shape: int, tau: int) -> np.ndarray:
    """calibration.cpp:30-78 — C^H C over valid shifts."""
    return _gram(EXPLICIT, calib, shape, tau)


def build_calib_matrix(calib: Calib, shape: int, tau: int) -> np.ndarray:
    d = _c128(calib.data)
    q, dims = d.shape[0], d.shape[1:]
    lam = make_support(shape, tau, len(dims)).shape[0]
    p = int(np.prod([e - 2 * tau for e in dims]))
    out = np.zeros((p, q * lam), dtype=np.complex128, order="F")
    r, c = C.c_int64(0), C.c_int64(0)
    _check(lib().sko_calib_matrix(len(dims), _p(_i64(dims)), q, _p(d), int(shape), int(tau),
                                  out.ctypes.data_as(C.c_void_p), C.byref(r), C.byref(c)))
    return out


# -------------------------------------------------------------- nullspace.cpp
@dataclass
class NullspaceBasis:
    filters: np.ndarray       # n x R
    spectrum: np.ndarray      # n, descending sigma
    threshold_ratio: float = 0.05

    @property
    def rank(self):
        return self.filters.shape[1]


def extract_nullspace(gram: np.ndarray, threshold_ratio: float = 0.05) -> NullspaceBasis:
    """nullspace.cpp:7-35."""
    g = np.asfortranarray(gram, dtype=np.complex128)
    n = g.shape[0]
    spec = np.zeros(n)
    filt = np.zeros((n, n), dtype=np.complex128, order="F")
    r = C.c_int64(0)
    _check(lib().sko_extract_nullspace(n, g.ctypes.data_as(C.c_void_p), C.c_double(threshold_ratio),
                                       C.byref(r), _p(spec), filt.ctypes.data_as(C.c_void_p)))
    return NullspaceBasis(np.array(filt[:, : r.value]), spec, threshold_ratio)


def aggregate_w(filters: np.ndarray) -> np.ndarray:
    """spatial_gram.cpp:87-94."""
    f = np.asfortranarray(filters, dtype=np.complex128)
    n, r = f.shape
    w = np.zeros((n, n), dtype=np.complex128, order="F")
    _check(lib().sko_aggregate_w(n, r, f.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p)))
    return w


# ----------------------------------------------------------- spatial_gram.cpp
def gram_field_fast(w: np.ndarray, q: int, shape: int, tau: int, dims) -> np.ndarray:
    """spatial_gram.cpp:96-148 — returns (N, Q, Q) array with [j, row, col]."""
    wf = np.asfortranarray(w, dtype=np.complex128)
    n = int(np.prod(dims))
    out = np.zeros(n * q * q, dtype=np.complex128)
    _check(lib().sko_gram_field_fast(q, wf.ctypes.data_as(C.c_void_p), int(shape), int(tau), len(dims),
                                     _p(_i64(dims)), _p(out)))
    return out.reshape(n, q, q).transpose(0, 2, 1)  # stored col-major per voxel


def gram_field_naive(filters: np.ndarray, q: int, shape: int, tau: int, dims) -> np.ndarray:
    """spatial_gram.cpp:33-85 — H(x) then G = H^H H per voxel."""
    f = np.asfortranarray(filters, dtype=np.complex128)
    n = int(np.prod(dims))
    out = np.zeros(n * q * q, dtype=np.complex128)
    _check(lib().sko_gram_field_naive(q, f.shape[1], f.ctypes.data_as(C.c_void_p), int(shape), int(tau),
                                      len(dims), _p(_i64(dims)), _p(out)))
    return out.reshape(n, q, q).transpose(0, 2, 1)


def _field_buf(field):
    """(N, Q, Q) [j,row,col] -> voxel-major col-major flat buffer."""
    return np.array(np.asarray(field, dtype=np.complex128).transpose(0, 2, 1), order="C", copy=True).reshape(-1)


def espirit(field: np.ndarray, support_size: int) -> np.ndarray:
    """spatial_gram.cpp:156-164 — B = I - G/|Lambda| (returns a new array)."""
    n, q, _ = field.shape
    buf = _field_buf(field)
    _check(lib().sko_espirit_inplace(n, q, _p(buf), int(support_size)))
    return buf.reshape(n, q, q).transpose(0, 2, 1)


def eig_power_field(bfield: np.ndarray, iters: int = 10):
    """eigensolve.cpp:40-74 — returns (vectors (Q, N), values (N,))."""
    n, q, _ = bfield.shape
    buf = _field_buf(bfield)
    vec = np.zeros(q * n, dtype=np.complex128)
    val = np.zeros(n)
    _check(lib().sko_eig_power_field(n, q, _p(buf), int(iters), _p(vec), _p(val)))
    return vec.reshape(n, q).T.copy(), val


def eig_dense_field(field: np.ndarray, largest: bool):
    """eigensolve.cpp:9-38 — returns (vectors (Q,N), values, second_values)."""
    n, q, _ = field.shape
    buf = _field_buf(field)
    vec = np.zeros(q * n, dtype=np.complex128)
    val, sec = np.zeros(n), np.zeros(n)
    _check(lib().sko_eig_dense_field(n, q, _p(buf), 1 if largest else 0, _p(vec), _p(val), _p(sec)))
    return vec.reshape(n, q).T.copy(), val, sec


# ------------------------------------------------------------------- maps.cpp
def normalize_maps(raw: np.ndarray, calib: Calib, apod_width: float = -1.0):
    """maps.cpp:101-176; raw is (Q, *dims). Returns (maps, zeroed_voxels)."""
    r = _c128(raw)
    q, dims = r.shape[0], r.shape[1:]
    out = np.zeros_like(r)
    z = C.c_int64(0)
    cd = _c128(calib.data)
    _check(lib().sko_normalize_maps(len(dims), _p(_i64(dims)), q, _p(r), _p(_i64(cd.shape[1:])),
                                    _p(_i64(calib.center_offset)), _p(cd), C.c_double(apod_width), _p(out),
                                    C.byref(z)))
    return out, z.value


def interpolate_maps(low: np.ndarray, full_dims) -> np.ndarray:
    """maps.cpp:54-90; low is (Q, *dims)."""
    lo = _c128(low)
    q = lo.shape[0]
    out = np.zeros((q,) + tuple(full_dims), dtype=np.complex128)
    _check(lib().sko_interpolate_maps(lo.ndim - 1, _p(_i64(lo.shape[1:])), q, _p(lo), _p(_i64(full_dims)),
                                      _p(out)))
    return out


def interpolate_real(low: np.ndarray, full_dims) -> np.ndarray:
    """maps.cpp:92-99."""
    lo = np.ascontiguousarray(low, dtype=np.float64)
    out = np.zeros(tuple(full_dims))
    _check(lib().sko_interpolate_real(lo.ndim, _p(_i64(lo.shape)), _p(lo), _p(_i64(full_dims)), _p(out)))
    return out


@dataclass
class SensitivityResult:
    """maps.hpp:60-81 (stage seconds under the reference's stage names)."""
    maps: np.ndarray
    lambda_min_map: np.ndarray
    support_mask: np.ndarray
    grid_dims: tuple
    nullspace_rank: int
    sigma1: float
    spectrum_normalized: np.ndarray
    stages: dict
    zeroed_voxels: int
    raw_maps: np.ndarray | None = None
    raw_lambda: np.ndarray | None = None
    gram: np.ndarray | None = None
    extra: dict = field(default_factory=dict)


STAGES = ("gram", "nullspace", "field", "eigensolve", "post")


def estimate_maps(calib: Calib, full_dims, cfg: PipelineConfig, grid_dims=None, want_raw=False,
                  want_gram=False) -> SensitivityResult:
    """maps.cpp:265-330 (grid_dims: explicit grid, maps.hpp:117-123)."""
    d = _c128(calib.data)
    q, cdims = d.shape[0], d.shape[1:]
    nd = len(cdims)
    lam = make_support(cfg.kernel, cfg.tau, nd).shape[0]
    n = q * lam
    nfull = int(np.prod(full_dims))
    maps = np.zeros((q,) + tuple(full_dims), dtype=np.complex128)
    lamb = np.zeros(tuple(full_dims))
    mask = np.zeros(tuple(full_dims), dtype=np.uint8)
    gd = np.zeros(nd, dtype=np.int64)
    rank = C.c_int64(0)
    s1 = C.c_double(0)
    spec = np.zeros(n)
    st = np.zeros(5)
    z = C.c_int64(0)
    if grid_dims is None:
        from_cfg = list(full_dims)
        if cfg.grid == GRID_REDUCED:
            from_cfg = [min(c + cfg.grid_pad, f) for c, f in zip(cdims, full_dims)]
        gshape = tuple(from_cfg)
    else:
        gshape = tuple(grid_dims)
    raw = np.zeros((q,) + gshape, dtype=np.complex128) if want_raw else None
    raw_l = np.zeros(gshape) if want_raw else None
    gram = np.zeros((n, n), dtype=np.complex128, order="F") if want_gram else None
    cfgc = cfg.to_c()
    _check(lib().sko_estimate_maps(
        nd, _p(_i64(cdims)), _p(_i64(calib.center_offset)), q, _p(d), _p(_i64(full_dims)), C.byref(cfgc),
        _p(_i64(grid_dims)) if grid_dims is not None else None, _p(maps), _p(lamb), _p(mask), _p(gd),
        C.byref(rank), C.byref(s1), _p(spec), _p(st), C.byref(z), _p(raw), _p(raw_l),
        gram.ctypes.data_as(C.c_void_p) if gram is not None else None))
    del nfull
    return SensitivityResult(maps, lamb, mask, tuple(int(x) for x in gd), rank.value, s1.value, spec,
                             dict(zip(STAGES, st.tolist())), z.value, raw, raw_l, gram)


# -------------------------------------------------------------- synthetic.cpp
def simulate(q: int, dims, tau_gen: int, seed: int, kind: int = DISK, noise_sigma: float = 0.0,
             noise_seed: int = 0):
    """make_scene + forward_kspace (synthetic.cpp:70-171).  Returns dict."""
    nd = len(dims)
    n = int(np.prod(dims))
    ks = np.zeros((q,) + tuple(dims), dtype=np.complex128)
    tm = np.zeros_like(ks)
    mask = np.zeros(tuple(dims), dtype=np.uint8)
    ph = np.zeros(tuple(dims))
    lam = (2 * tau_gen + 1) ** nd
    gc = np.zeros((lam, q), dtype=np.complex128, order="F")
    _check(lib().sko_simulate(q, nd, _p(_i64(dims)), int(tau_gen), C.c_uint64(seed), int(kind),
                              C.c_double(noise_sigma), C.c_uint64(noise_seed), _p(ks), _p(tm), _p(mask), _p(ph),
                              gc.ctypes.data_as(C.c_void_p)))
    del n
    return {"kspace": ks, "true_maps": tm, "support_mask_true": mask, "phantom": ph, "gen_coeffs": gc}


def estimate_sampled(calib: Calib, full_dims, cfg: PipelineConfig, grid_dims=None, gram_idx=None, field_idx=None,
                     vox_idx=None) -> dict:
    """The reference pipeline (maps.cpp:265-330, staged as in maps.hpp:115-123) with
    the Gram sampled at (row, col) pairs ``gram_idx`` (K,2), G(x) at (voxel, row, col)
    triples ``field_idx`` (K,3) before the eigensolve consumes it, and the final
    maps / lambda / mask gathered at ``vox_idx``.  Only the oracle/_ref library
    exports it (golden-fixture generation, tools/make_golden.py)."""
    L = lib()
    if not hasattr(L, "skr_estimate_sampled"):
        raise RuntimeError("estimate_sampled needs oracle/_ref (the reference build)")
    d = _c128(calib.data)
    q, cdims = d.shape[0], d.shape[1:]
    nd = len(cdims)
    n = q * make_support(cfg.kernel, cfg.tau, nd).shape[0]
    gi = _i64(np.zeros((0, 2)) if gram_idx is None else gram_idx).reshape(-1, 2)
    fi = _i64(np.zeros((0, 3)) if field_idx is None else field_idx).reshape(-1, 3)
    vi = _i64(np.zeros(0) if vox_idx is None else vox_idx).reshape(-1)
    if grid_dims is None:
        gshape = list(full_dims)
        if cfg.grid == GRID_REDUCED:
            gshape = [min(c + cfg.grid_pad, f) for c, f in zip(cdims, full_dims)]
    else:
        gshape = list(grid_dims)
    gv = np.zeros(len(gi), dtype=np.complex128)
    fv = np.zeros(len(fi), dtype=np.complex128)
    gfro, ffro = C.c_double(0), C.c_double(0)
    raw_l = np.zeros(tuple(gshape))
    ms = np.zeros((q, len(vi)), dtype=np.complex128)
    ls = np.zeros(len(vi))
    mk = np.zeros(len(vi), dtype=np.uint8)
    gd = np.zeros(nd, dtype=np.int64)
    rank, s1 = C.c_int64(0), C.c_double(0)
    spec = np.zeros(n)
    st = np.zeros(5)
    cfgc = cfg.to_c()
    _check(L.skr_estimate_sampled(
        nd, _p(_i64(cdims)), _p(_i64(calib.center_offset)), q, _p(d), _p(_i64(full_dims)), C.byref(cfgc),
        _p(_i64(grid_dims)) if grid_dims is not None else None, len(gi), _p(gi), _p(gv), C.byref(gfro),
        len(fi), _p(fi), _p(fv), C.byref(ffro), _p(raw_l), len(vi), _p(vi), _p(ms), _p(ls), _p(mk), _p(gd),
        C.byref(rank), C.byref(s1), _p(spec), _p(st)))
    return {"gram_vals": gv, "gram_fro": gfro.value, "field_vals": fv, "field_fro": ffro.value,
            "raw_lambda": raw_l, "maps": ms, "lambda": ls, "mask": mk, "grid_dims": tuple(int(x) for x in gd),
            "rank": rank.value, "sigma1": s1.value, "spectrum_normalized": spec,
            "stages": dict(zip(STAGES, st.tolist()))}


def projection_residual(kspace: np.ndarray, maps: np.ndarray) -> float:
    """metrics.cpp:11-49."""
    k, m = _c128(kspace), _c128(maps)
    out = C.c_double(0)
    _check(lib().sko_projection_residual(k.ndim - 1, _p(_i64(k.shape[1:])), k.shape[0], _p(k), _p(m),
                                         C.byref(out)))
    return out.value

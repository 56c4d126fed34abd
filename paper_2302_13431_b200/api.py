"""ctypes mirror of the reference entry points over ``libsenskit_b200.so``.

Every function names the reference declaration it stands in for.  Arrays are
numpy (host) or any object exposing a CUDA device pointer through an integer
address (``DevicePtr``); host arrays are complex64 / float32 in the reference
layouts (channel-major stacks (Q, *dims), column-major matrices, GramField
as (N, Q, Q) [voxel, row, col]).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from dataclasses import field as dc_field

import numpy as np

__all__ = [
    "RECT", "ELLIPSOID", "GRID_FULL", "GRID_REDUCED", "PipelineConfig", "Calib", "SensitivityResult",
    "SensKitError", "NullspaceEmptyError", "DimError", "LengthError", "CudaError", "UnsupportedError",
    "Context", "default_context", "lib", "library_path", "make_support", "reduced_grid_dims", "gram_fft",
    "build_calib_matrix", "gram_explicit", "eig_dense_field",
    "extract_nullspace", "aggregate_w", "gram_field_fast", "espirit", "eig_power_field", "normalize_maps",
    "interpolate_maps", "interpolate_real", "support_mask", "estimate_maps", "estimate_maps_batched",
    "DevicePtr", "STAGES",
]

RECT, ELLIPSOID = 0, 1
GRID_FULL, GRID_REDUCED = 0, 1
STAGES = ("gram", "nullspace", "field", "eigensolve", "post")

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_HERE, "lib", "libsenskit_b200.so")


class SensKitError(RuntimeError):
    code = 1


class NullspaceEmptyError(SensKitError):   # types.hpp:30-32
    code = 4


class DimError(SensKitError):              # types.hpp:25-27
    code = 5


class LengthError(SensKitError):
    code = 6


class CudaError(SensKitError):
    code = 7


class UnsupportedError(SensKitError):
    code = 9


_ERR = {4: NullspaceEmptyError, 5: DimError, 6: LengthError, 7: CudaError, 8: CudaError, 9: UnsupportedError}


class sk_config(C.Structure):
    _fields_ = [
        ("kernel", C.c_int32), ("tau", C.c_int32), ("gram", C.c_int32), ("nullspace_threshold", C.c_double),
        ("grid", C.c_int32), ("grid_pad", C.c_int64), ("eig", C.c_int32), ("power_iters", C.c_int32),
        ("method", C.c_int32), ("field", C.c_int32), ("mask_threshold", C.c_double), ("apod_width", C.c_double),
        ("grid_dims", C.c_int64 * 3), ("eig_solver", C.c_int32), ("certify", C.c_int32),
        ("field_byte_cap", C.c_int64),
    ]


class sk_provenance(C.Structure):
    _fields_ = [
        ("grid_dims", C.c_int64 * 3), ("support_size", C.c_int64), ("valid_shifts", C.c_int64),
        ("nullspace_rank", C.c_int64), ("zeroed_voxels", C.c_int64), ("sigma1", C.c_double),
        ("cut_margin", C.c_double), ("eig_solver_used", C.c_int32), ("certified", C.c_int32),
        ("subspace_iterations", C.c_int32), ("subspace_block", C.c_int32),
        ("stage_ms", C.c_double * 5), ("total_ms", C.c_double),
    ]


@dataclass
class PipelineConfig:
    """PipelineConfig (maps.hpp:23-45).  Dataclass defaults are the pisco preset (the
    reference's struct defaults are the baseline one; both presets run on the GPU)."""
    kernel: int = ELLIPSOID
    tau: int = 3
    gram: int = 1            # fft
    nullspace_threshold: float = 0.05
    grid: int = GRID_REDUCED
    grid_pad: int = 24
    eig: int = 1             # power
    power_iters: int = 10
    method: int = 0
    field: int = 1           # fast
    mask_threshold: float = 0.01
    apod_width: float = -1.0
    grid_dims: tuple | None = None   # explicit map grid (maps.hpp:115-123)
    eig_solver: int = 0      # B200 extension: 0 auto, 1 full cuSOLVER, 2 subspace
    certify: int = 0         # B200 extension: prove R with one Cholesky (subspace solver)
    field_byte_cap: int = 1 << 30   # maps.hpp:41 (naive field budget)

    @staticmethod
    def pisco() -> "PipelineConfig":   # maps.cpp:21-28
        return PipelineConfig()

    @staticmethod
    def baseline() -> "PipelineConfig":   # maps.cpp:12-19: rect kernel, explicit Gram, full grid, dense eig
        return PipelineConfig(kernel=RECT, gram=0, grid=GRID_FULL, eig=0)

    def to_c(self) -> sk_config:
        gd = (C.c_int64 * 3)(*(list(self.grid_dims or ()) + [0, 0, 0])[:3])
        return sk_config(self.kernel, self.tau, self.gram, self.nullspace_threshold, self.grid, self.grid_pad,
                         self.eig, self.power_iters, self.method, self.field, self.mask_threshold,
                         self.apod_width, gd, self.eig_solver, self.certify, self.field_byte_cap)


@dataclass
class Calib:
    """CalibrationRegion (types.hpp:79-85): data (Q, *dims) complex, center_offset per axis."""
    data: np.ndarray
    center_offset: tuple

    @property
    def dims(self):
        return tuple(self.data.shape[1:])

    @property
    def channels(self):
        return self.data.shape[0]


@dataclass
class DevicePtr:
    """A caller-owned device buffer (e.g. ``torch.Tensor.data_ptr()``)."""
    ptr: int


@dataclass
class SensitivityResult:
    """SensitivityResult + Provenance (maps.hpp:55-81); stage times are device ms."""
    maps: np.ndarray | None
    lambda_min_map: np.ndarray | None
    support_mask: np.ndarray | None
    grid_dims: tuple
    support_size: int
    nullspace_rank: int
    sigma1: float
    cut_margin: float
    spectrum_normalized: np.ndarray | None
    stage_ms: dict
    total_ms: float
    zeroed_voxels: int
    gram: np.ndarray | None = None
    field: np.ndarray | None = None
    raw_maps: np.ndarray | None = None
    raw_lambda: np.ndarray | None = None
    extra: dict = dc_field(default_factory=dict)


_VP, _I32, _I64, _D = C.c_void_p, C.c_int, C.c_int64, C.c_double
_SIGS = {
    "sk_create": ([_I32, C.POINTER(C.c_void_p)], _I32),
    "sk_destroy": ([_VP], _I32),
    "sk_set_stream": ([_VP, _VP], _I32),
    "sk_kernel_launches": ([_VP], _I64),
    "sk_library_calls": ([_VP], _I64),
    "sk_make_support": ([_I32, _I32, _I32, _VP, _VP], _I32),
    "sk_reduced_grid_dims": ([_I32, _VP, _I64, _VP, _VP], _I32),
    "sk_gram_fft": ([_VP, _I32, _VP, _I64, _VP, _I32, _I32, _VP], _I32),
    "sk_build_calib_matrix": ([_VP, _I32, _VP, _I64, _VP, _I32, _I32, _VP, _VP], _I32),
    "sk_gram_explicit": ([_VP, _I64, _I64, _VP, _VP], _I32),
    "sk_eig_dense_field": ([_VP, _I64, _I64, _VP, _I32, _VP, _VP, _VP], _I32),
    "sk_extract_nullspace": ([_VP, _I64, _VP, _D, _VP, _VP, _VP, _I64], _I32),
    "sk_aggregate_w": ([_VP, _I64, _I64, _VP, _VP], _I32),
    "sk_gram_field_fast": ([_VP, _I64, _VP, _I32, _I32, _I32, _VP, _VP], _I32),
    "sk_espirit_inplace": ([_VP, _I64, _I64, _VP, _I64], _I32),
    "sk_eig_power_field": ([_VP, _I64, _I64, _VP, _I32, _VP, _VP], _I32),
    "sk_normalize_maps": ([_VP, _I32, _VP, _I64, _VP, _VP, _VP, _VP, _D, _VP, _VP], _I32),
    "sk_interpolate_maps": ([_VP, _I32, _VP, _I64, _VP, _VP, _VP], _I32),
    "sk_interpolate_real": ([_VP, _I32, _VP, _VP, _VP, _VP], _I32),
    "sk_support_mask": ([_VP, _I64, _VP, _D, _VP], _I32),
    "sk_debug_small_eigh": ([_VP, _I64, _VP, _VP], _I32),
    "sk_debug_cholqr": ([_VP, _I64, _I64, _VP, _I32], _I32),
    "sk_debug_cross_gram": ([_VP, _I64, _I64, _VP, _VP, _VP], _I32),
    "sk_estimate_raw_slab": ([_VP, _I32, _VP, _VP, _I64, _VP, _VP, _VP, _I64, _I64, _VP, _VP, _VP], _I32),
    "sk_sos_accumulate": ([_VP, _I64, _I64, _VP, _VP], _I32),
    "sk_projection_residual": ([_VP, _I32, _VP, _I64, _VP, _VP, _VP], _I32),
    "sk_renormalize_sos": ([_VP, _I64, _I64, _VP, _VP], _I32),
    "sk_estimate_maps": ([_VP, _I32, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP], _I32),
    "sk_estimate_maps_debug": ([_VP, _I32, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                _VP, _VP], _I32),
    "sk_estimate_maps_probe": ([_VP, _I32, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I64, _VP, _VP, _VP,
                                _I64, _VP, _VP, _VP, _VP], _I32),
    "sk_signal_basis": ([_VP, _I32, _VP, _VP, _I64, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _VP], _I32),
    "sk_estimate_raw_slab_basis": ([_VP, _I32, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _I64, _D, _I64, _I64, _VP, _VP,
                                    _VP], _I32),
    "sk_estimate_maps_batched": ([_VP, _I64, _I32, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP], _I32),
}

_lib = None


def lib():
    """Load the native library; raise if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(library_path):
            raise RuntimeError(f"senskit_b200 native library missing: {library_path} (run `make product`)")
        L = C.CDLL(library_path)
        L.sk_last_error.restype = C.c_char_p
        L.sk_last_error.argtypes = []
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise _ERR.get(rc, SensKitError)(lib().sk_last_error().decode())


class Context:
    """One sk_ctx per GPU (not re-entrant)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib().sk_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device

    def set_stream(self, stream_handle: int | None):
        _check(lib().sk_set_stream(self.handle, C.c_void_p(stream_handle) if stream_handle else None))

    @property
    def launches(self) -> int:
        return int(lib().sk_kernel_launches(self.handle))

    @property
    def library_calls(self) -> int:
        return int(lib().sk_library_calls(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            lib().sk_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: dict = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def _ctx(ctx):
    return (ctx or default_context()).handle


def _i64(seq):
    return np.ascontiguousarray(np.asarray(seq, dtype=np.int64))


def _c64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex64))


def _p(a):
    if a is None:
        return None
    if isinstance(a, DevicePtr):
        return C.c_void_p(a.ptr)
    return a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------- host helpers
def make_support(shape: int, tau: int, ndim: int) -> np.ndarray:
    """make_support (kernels.hpp:24)."""
    cnt = C.c_int64(0)
    _check(lib().sk_make_support(int(shape), int(tau), int(ndim), None, C.byref(cnt)))
    buf = np.zeros(max(1, cnt.value * ndim), dtype=np.int32)
    _check(lib().sk_make_support(int(shape), int(tau), int(ndim), _p(buf), C.byref(cnt)))
    return buf[: cnt.value * ndim].reshape(cnt.value, ndim)


def reduced_grid_dims(calib_dims, pad, full_dims):
    """reduced_grid_dims (maps.hpp:102)."""
    out = np.zeros(len(calib_dims), dtype=np.int64)
    _check(lib().sk_reduced_grid_dims(len(calib_dims), _p(_i64(calib_dims)), int(pad), _p(_i64(full_dims)),
                                      _p(out)))
    return tuple(int(x) for x in out)


# ---------------------------------------------------------------- stages
def gram_fft(calib: Calib, shape: int, tau: int, ctx: Context | None = None) -> np.ndarray:
    """gram_fft (calibration.hpp:42) -> (n, n) complex64 Hermitian Gram."""
    d = _c64(calib.data)
    q, dims = d.shape[0], d.shape[1:]
    lam = make_support(shape, tau, len(dims)).shape[0]
    n = q * lam
    g = np.zeros((n, n), dtype=np.complex64, order="F")
    _check(lib().sk_gram_fft(_ctx(ctx), len(dims), _p(_i64(dims)), q, _p(d), int(shape), int(tau),
                             g.ctypes.data_as(C.c_void_p)))
    return g


def build_calib_matrix(calib: Calib, shape: int, tau: int, ctx: Context | None = None) -> np.ndarray:
    """build_calib_matrix (calibration.hpp:32) -> (P, n) complex64, P valid shifts."""
    d = _c64(calib.data)
    q, dims = d.shape[0], d.shape[1:]
    rows = C.c_int64(0)
    _check(lib().sk_build_calib_matrix(_ctx(ctx), len(dims), _p(_i64(dims)), q, _p(d), int(shape), int(tau), None,
                                       C.byref(rows)))
    n = q * make_support(shape, tau, len(dims)).shape[0]
    c = np.zeros((rows.value, n), dtype=np.complex64, order="F")
    if c.size:
        _check(lib().sk_build_calib_matrix(_ctx(ctx), len(dims), _p(_i64(dims)), q, _p(d), int(shape), int(tau),
                                           c.ctypes.data_as(C.c_void_p), C.byref(rows)))
    return c


def gram_explicit(cmat: np.ndarray, ctx: Context | None = None) -> np.ndarray:
    """gram_explicit (calibration.hpp:35) -> (n, n) complex64 C^H C (FP64 accumulation)."""
    c = np.asfortranarray(cmat, dtype=np.complex64)
    rows, n = c.shape
    g = np.zeros((n, n), dtype=np.complex64, order="F")
    _check(lib().sk_gram_explicit(_ctx(ctx), rows, n, c.ctypes.data_as(C.c_void_p), g.ctypes.data_as(C.c_void_p)))
    return g


@dataclass
class NullspaceBasis:
    """NullspaceBasis (nullspace.hpp:11-19)."""
    filters: np.ndarray | None
    spectrum: np.ndarray
    rank: int
    threshold_ratio: float = 0.05


def extract_nullspace(gram: np.ndarray, threshold_ratio: float = 0.05, want_filters: bool = True,
                      ctx: Context | None = None) -> NullspaceBasis:
    """extract_nullspace (nullspace.hpp:24)."""
    g = np.asfortranarray(gram, dtype=np.complex64)
    n = g.shape[0]
    spec = np.zeros(n)
    r = C.c_int64(0)
    filt = np.zeros((n, n), dtype=np.complex64, order="F") if want_filters else None
    _check(lib().sk_extract_nullspace(_ctx(ctx), n, g.ctypes.data_as(C.c_void_p), float(threshold_ratio),
                                      C.byref(r), _p(spec), filt.ctypes.data_as(C.c_void_p) if want_filters else None,
                                      n))
    return NullspaceBasis(np.array(filt[:, : r.value]) if want_filters else None, spec, r.value, threshold_ratio)


def aggregate_w(filters: np.ndarray, ctx: Context | None = None) -> np.ndarray:
    """aggregate_w (spatial_gram.hpp:61)."""
    f = np.asfortranarray(filters, dtype=np.complex64)
    n, r = f.shape
    w = np.zeros((n, n), dtype=np.complex64, order="F")
    _check(lib().sk_aggregate_w(_ctx(ctx), n, r, f.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p)))
    return w


def gram_field_fast(w: np.ndarray, q: int, shape: int, tau: int, dims, ctx: Context | None = None) -> np.ndarray:
    """gram_field_fast (spatial_gram.hpp:67) -> (N, Q, Q) [voxel, row, col]."""
    wf = np.asfortranarray(w, dtype=np.complex64)
    n = int(np.prod(dims))
    out = np.zeros(n * q * q, dtype=np.complex64)
    _check(lib().sk_gram_field_fast(_ctx(ctx), q, wf.ctypes.data_as(C.c_void_p), int(shape), int(tau), len(dims),
                                    _p(_i64(dims)), _p(out)))
    return out.reshape(n, q, q).transpose(0, 2, 1)


def _field_buf(field):
    return np.array(np.asarray(field, dtype=np.complex64).transpose(0, 2, 1), order="C", copy=True).reshape(-1)


def espirit(field: np.ndarray, support_size: int, ctx: Context | None = None) -> np.ndarray:
    """espirit_inplace (spatial_gram.hpp:73), returning a new array."""
    n, q, _ = field.shape
    buf = _field_buf(field)
    _check(lib().sk_espirit_inplace(_ctx(ctx), n, q, _p(buf), int(support_size)))
    return buf.reshape(n, q, q).transpose(0, 2, 1)


def eig_power_field(bfield: np.ndarray, iters: int = 10, ctx: Context | None = None):
    """eig_power_field (eigensolve.hpp:27) -> (vectors (Q, N), values (N,))."""
    n, q, _ = bfield.shape
    buf = _field_buf(bfield)
    vec = np.zeros(q * n, dtype=np.complex64)
    val = np.zeros(n, dtype=np.float32)
    _check(lib().sk_eig_power_field(_ctx(ctx), n, q, _p(buf), int(iters), _p(vec), _p(val)))
    return vec.reshape(n, q).T.copy(), val


def eig_dense_field(field: np.ndarray, largest: bool, ctx: Context | None = None):
    """eig_dense_field (eigensolve.hpp:21) -> (vectors (Q, N), values (N,), second_values (N,))."""
    n, q, _ = field.shape
    buf = _field_buf(field)
    vec = np.zeros(q * n, dtype=np.complex64)
    val = np.zeros(n, dtype=np.float32)
    sec = np.zeros(n, dtype=np.float32)
    _check(lib().sk_eig_dense_field(_ctx(ctx), n, q, _p(buf), 1 if largest else 0, _p(vec), _p(val), _p(sec)))
    return vec.reshape(n, q).T.copy(), val, sec


def normalize_maps(raw: np.ndarray, calib: Calib, apod_width: float = -1.0, ctx: Context | None = None):
    """normalize_maps (maps.hpp:92-94) -> (maps, zeroed_voxels)."""
    r = _c64(raw)
    q, dims = r.shape[0], r.shape[1:]
    cd = _c64(calib.data)
    out = np.zeros_like(r)
    z = C.c_int64(0)
    _check(lib().sk_normalize_maps(_ctx(ctx), len(dims), _p(_i64(dims)), q, _p(r), _p(_i64(cd.shape[1:])),
                                   _p(_i64(calib.center_offset)), _p(cd), float(apod_width), _p(out), C.byref(z)))
    return out, z.value


def interpolate_maps(low: np.ndarray, full_dims, ctx: Context | None = None) -> np.ndarray:
    """interpolate_maps (maps.hpp:98)."""
    lo = _c64(low)
    out = np.zeros((lo.shape[0],) + tuple(full_dims), dtype=np.complex64)
    _check(lib().sk_interpolate_maps(_ctx(ctx), lo.ndim - 1, _p(_i64(lo.shape[1:])), lo.shape[0], _p(lo),
                                     _p(_i64(full_dims)), _p(out)))
    return out


def interpolate_real(low: np.ndarray, full_dims, ctx: Context | None = None) -> np.ndarray:
    """interpolate_real (maps.hpp:99)."""
    lo = np.ascontiguousarray(low, dtype=np.float32)
    out = np.zeros(tuple(full_dims), dtype=np.float32)
    _check(lib().sk_interpolate_real(_ctx(ctx), lo.ndim, _p(_i64(lo.shape)), _p(lo), _p(_i64(full_dims)), _p(out)))
    return out


def small_eigh(h: np.ndarray, ctx: Context | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Test hook: the K2 Rayleigh-Ritz eigensolver on a Hermitian complex128
    matrix (eigenvalues ascending, eigenvectors as columns), like numpy.linalg.eigh."""
    a = np.array(h, dtype=np.complex128, order="F", copy=True)
    n = a.shape[0]
    if a.shape != (n, n):
        raise ValueError("small_eigh: square matrix required")
    w = np.zeros(n, dtype=np.float64)
    _check(lib().sk_debug_small_eigh(_ctx(ctx), n, a.ctypes.data, w.ctypes.data))
    return w, a


def cholqr(x: np.ndarray, passes: int = 1, ctx: Context | None = None) -> np.ndarray:
    """Test hook: the K2 block orthonormalisation (CholQR, `passes` times) on a
    complex128 n x b block; returns the orthonormal block with the same span."""
    a = np.array(x, dtype=np.complex128, order="F", copy=True)
    n, b = a.shape
    _check(lib().sk_debug_cholqr(_ctx(ctx), n, b, a.ctypes.data, int(passes)))
    return a


def cross_gram(x: np.ndarray, y: np.ndarray | None = None, ctx: Context | None = None) -> np.ndarray:
    """Test hook: X^H Y (X^H X when y is None) with the K2 block kernels."""
    xa = np.asfortranarray(x, dtype=np.complex128)
    n, b = xa.shape
    ya = None if y is None else np.asfortranarray(y, dtype=np.complex128)
    if ya is not None and ya.shape != xa.shape:
        raise ValueError("cross_gram: x and y must have the same shape")
    out = np.zeros((b, b), dtype=np.complex128, order="F")
    _check(lib().sk_debug_cross_gram(_ctx(ctx), n, b, xa.ctypes.data, None if ya is None else ya.ctypes.data,
                                     out.ctypes.data))
    return out


def support_mask(lam: np.ndarray, threshold: float, ctx: Context | None = None) -> np.ndarray:
    """support_mask (maps.hpp:105)."""
    lo = np.ascontiguousarray(lam, dtype=np.float32)
    out = np.zeros(lo.shape, dtype=np.uint8)
    _check(lib().sk_support_mask(_ctx(ctx), lo.size, _p(lo), float(threshold), _p(out)))
    return out


def _grid_for(cdims, full_dims, cfg: PipelineConfig):
    if cfg.grid_dims:
        return tuple(cfg.grid_dims)
    if cfg.grid == GRID_REDUCED:
        return tuple(min(c + cfg.grid_pad, f) for c, f in zip(cdims, full_dims))
    return tuple(full_dims)


def estimate_maps(calib: Calib, full_dims, cfg: PipelineConfig, ctx: Context | None = None, *,
                  want_spectrum: bool = False, want_gram: bool = False, want_field: bool = False,
                  want_raw: bool = False, out=None) -> SensitivityResult:
    """estimate_maps (maps.hpp:85-86).

    ``calib.data`` may be a numpy array (host) or a DevicePtr (then pass
    ``calib_dims`` via ``calib.center_offset``'s companion: use
    ``estimate_maps_device``).  ``out`` may supply preallocated destinations
    {maps, lambda, mask} (numpy or DevicePtr) to avoid allocation.
    """
    d = _c64(calib.data)
    q, cdims = d.shape[0], d.shape[1:]
    nd = len(cdims)
    lam_count = make_support(cfg.kernel, cfg.tau, nd).shape[0]
    n = q * lam_count
    grid = _grid_for(cdims, full_dims, cfg)
    out = out or {}
    maps = out.get("maps", np.zeros((q,) + tuple(full_dims), dtype=np.complex64))
    lamb = out.get("lambda", np.zeros(tuple(full_dims), dtype=np.float32))
    mask = out.get("mask", np.zeros(tuple(full_dims), dtype=np.uint8))
    spec = np.zeros(n) if want_spectrum else None
    prov = sk_provenance()
    ngrid = int(np.prod(grid))
    gram = np.zeros((n, n), dtype=np.complex64, order="F") if want_gram else None
    fieldb = np.zeros(ngrid * q * q, dtype=np.complex64) if want_field else None
    raw = np.zeros((q,) + grid, dtype=np.complex64) if want_raw else None
    raw_l = np.zeros(grid, dtype=np.float32) if want_raw else None
    cfgc = cfg.to_c()
    _check(lib().sk_estimate_maps_debug(
        _ctx(ctx), nd, _p(_i64(cdims)), _p(_i64(calib.center_offset)), q, _p(d), _p(_i64(full_dims)),
        C.byref(cfgc), _p(maps), _p(lamb), _p(mask), _p(spec), C.byref(prov),
        gram.ctypes.data_as(C.c_void_p) if want_gram else None, _p(fieldb), _p(raw), _p(raw_l)))
    return SensitivityResult(
        maps if not isinstance(maps, DevicePtr) else None,
        lamb if not isinstance(lamb, DevicePtr) else None,
        mask if not isinstance(mask, DevicePtr) else None,
        tuple(int(prov.grid_dims[a]) for a in range(nd)), int(prov.support_size), int(prov.nullspace_rank),
        float(prov.sigma1), float(prov.cut_margin), spec, dict(zip(STAGES, list(prov.stage_ms))),
        float(prov.total_ms), int(prov.zeroed_voxels), gram,
        fieldb.reshape(ngrid, q, q).transpose(0, 2, 1) if want_field else None, raw, raw_l,
        extra={"eig_solver": "full" if prov.eig_solver_used == 1 else "subspace", "certified": bool(prov.certified),
               "subspace_iterations": int(prov.subspace_iterations), "subspace_block": int(prov.subspace_block)})


def estimate_maps_probe(calib: Calib, full_dims, cfg: PipelineConfig, ctx: Context | None = None, *,
                        gram_idx=None, field_idx=None) -> tuple[SensitivityResult, dict]:
    """estimate_maps on exactly the sk_estimate_maps path (no spectrum requested, so
    the same nullspace solver the bench runs) plus in-place samples of the Gram at
    (row, col) ``gram_idx`` and of G(x) at (voxel, row, col) ``field_idx``, their
    Frobenius norms and the native-grid lambda (sk_estimate_maps_probe)."""
    d = _c64(calib.data)
    q, cdims = d.shape[0], d.shape[1:]
    nd = len(cdims)
    grid = _grid_for(cdims, full_dims, cfg)
    gi = _i64(np.zeros((0, 2)) if gram_idx is None else gram_idx).reshape(-1, 2)
    fi = _i64(np.zeros((0, 3)) if field_idx is None else field_idx).reshape(-1, 3)
    maps = np.zeros((q,) + tuple(full_dims), dtype=np.complex64)
    lamb = np.zeros(tuple(full_dims), dtype=np.float32)
    mask = np.zeros(tuple(full_dims), dtype=np.uint8)
    gv = np.zeros(len(gi), dtype=np.complex128)
    fv = np.zeros(len(fi), dtype=np.complex128)
    gfro, ffro = C.c_double(0), C.c_double(0)
    rawl = np.zeros(grid, dtype=np.float32)
    prov = sk_provenance()
    cfgc = cfg.to_c()
    _check(lib().sk_estimate_maps_probe(
        _ctx(ctx), nd, _p(_i64(cdims)), _p(_i64(calib.center_offset)), q, _p(d), _p(_i64(full_dims)), C.byref(cfgc),
        _p(maps), _p(lamb), _p(mask), C.byref(prov), len(gi), _p(gi), _p(gv), C.byref(gfro), len(fi), _p(fi), _p(fv),
        C.byref(ffro), _p(rawl)))
    res = SensitivityResult(
        maps, lamb, mask, tuple(int(prov.grid_dims[a]) for a in range(nd)), int(prov.support_size),
        int(prov.nullspace_rank), float(prov.sigma1), float(prov.cut_margin), None,
        dict(zip(STAGES, list(prov.stage_ms))), float(prov.total_ms), int(prov.zeroed_voxels), raw_lambda=rawl,
        extra={"eig_solver": "full" if prov.eig_solver_used == 1 else "subspace", "certified": bool(prov.certified),
               "subspace_iterations": int(prov.subspace_iterations), "subspace_block": int(prov.subspace_block)})
    return res, {"gram_vals": gv, "gram_fro": gfro.value, "field_vals": fv, "field_fro": ffro.value}


def projection_residual(kspace: np.ndarray, maps: np.ndarray, ctx: Context | None = None) -> float:
    """projection_residual (metrics.cpp:11-49): kspace and maps (Q, *dims)."""
    k = _c64(kspace)
    m = _c64(maps)
    if k.shape != m.shape:
        raise DimError("data and maps must share dims and channel count")
    v = C.c_double(0.0)
    _check(lib().sk_projection_residual(_ctx(ctx), k.ndim - 1, _p(_i64(k.shape[1:])), k.shape[0], _p(k), _p(m),
                                        C.byref(v)))
    return float(v.value)


def estimate_raw_slab(calib: Calib, full_dims, cfg: PipelineConfig, slab, ctx: Context | None = None):
    """z-slab sharding: pipeline::compute_field + solve_field + the
    per-voxel normalisation (maps.hpp:115-123) on map-grid rows slab = (begin,
    end) of axis 0.  Returns (maps (Q, end-begin, *grid[1:]) complex64,
    lambda (end-begin, *grid[1:]) float32, provenance)."""
    d = _c64(calib.data)
    q, cdims = d.shape[0], d.shape[1:]
    grid = _grid_for(cdims, full_dims, cfg)
    b, e = int(slab[0]), int(slab[1])
    shape = (e - b,) + tuple(grid[1:])
    maps = np.zeros((q,) + shape, dtype=np.complex64)
    lam = np.zeros(shape, dtype=np.float32)
    prov = sk_provenance()
    cfgc = cfg.to_c()
    _check(lib().sk_estimate_raw_slab(_ctx(ctx), len(cdims), _p(_i64(cdims)), _p(_i64(calib.center_offset)), q,
                                      _p(d), _p(_i64(full_dims)), C.byref(cfgc), b, e, _p(maps), _p(lam),
                                      C.byref(prov)))
    return maps, lam, prov


def estimate_raw_slab_device(ctx: Context, calib_ptr: int, calib_dims, center_offset, q: int, full_dims,
                             cfg: PipelineConfig, slab, maps_ptr: int, lambda_ptr: int) -> sk_provenance:
    """Device-buffer variant of estimate_raw_slab."""
    prov = sk_provenance()
    cfgc = cfg.to_c()
    _check(lib().sk_estimate_raw_slab(ctx.handle, len(calib_dims), _p(_i64(calib_dims)), _p(_i64(center_offset)), q,
                                      C.c_void_p(calib_ptr), _p(_i64(full_dims)), C.byref(cfgc), int(slab[0]),
                                      int(slab[1]), C.c_void_p(maps_ptr), C.c_void_p(lambda_ptr), C.byref(prov)))
    return prov


def signal_basis_device(ctx: Context, calib_ptr: int, calib_dims, center_offset, q: int, cfg: PipelineConfig,
                        u_ptr: int, kmax: int) -> dict:
    """compute_gram + extract_nullspace in complement form (sk_signal_basis): the
    k signal eigenvectors U_sig (n x k complex128, column-major) written to u_ptr
    (capacity n * kmax), plus k, R, sigma_1 and the cut margin."""
    k, r = C.c_int64(0), C.c_int64(0)
    s1, margin = C.c_double(0), C.c_double(0)
    cfgc = cfg.to_c()
    _check(lib().sk_signal_basis(ctx.handle, len(calib_dims), _p(_i64(calib_dims)), _p(_i64(center_offset)), q,
                                 C.c_void_p(calib_ptr), C.byref(cfgc), int(kmax), C.c_void_p(u_ptr), C.byref(k),
                                 C.byref(r), C.byref(s1), C.byref(margin)))
    return {"k": k.value, "rank": r.value, "sigma1": s1.value, "cut_margin": margin.value}


def estimate_raw_slab_basis_device(ctx: Context, calib_ptr: int, calib_dims, center_offset, q: int, full_dims,
                                   cfg: PipelineConfig, u_ptr: int, k: int, sigma1: float, slab, maps_ptr: int,
                                   lambda_ptr: int) -> sk_provenance:
    """estimate_raw_slab with a supplied signal basis (sk_estimate_raw_slab_basis):
    K1 and K2 skipped, so every rank expands the broadcast filters."""
    prov = sk_provenance()
    cfgc = cfg.to_c()
    _check(lib().sk_estimate_raw_slab_basis(ctx.handle, len(calib_dims), _p(_i64(calib_dims)),
                                            _p(_i64(center_offset)), q, C.c_void_p(calib_ptr), _p(_i64(full_dims)),
                                            C.byref(cfgc), C.c_void_p(u_ptr), int(k), float(sigma1), int(slab[0]),
                                            int(slab[1]), C.c_void_p(maps_ptr), C.c_void_p(lambda_ptr),
                                            C.byref(prov)))
    return prov


def sos_accumulate(maps, sos, ctx: Context | None = None):
    """sos += sum_c |maps_c|^2 per voxel (maps.cpp:236-258 renorm, one channel subset).
    maps: (C, *vox) complex64 array or DevicePtr-like with .data_ptr(); sos: float32, updated in place."""
    if hasattr(maps, "data_ptr"):
        _check(lib().sk_sos_accumulate(_ctx(ctx), sos.numel(), maps.shape[0], C.c_void_p(maps.data_ptr()),
                                       C.c_void_p(sos.data_ptr())))
        return sos
    m = _c64(maps)
    if not (isinstance(sos, np.ndarray) and sos.dtype == np.float32 and sos.flags.c_contiguous):
        raise ValueError("sos must be a contiguous float32 array")
    _check(lib().sk_sos_accumulate(_ctx(ctx), sos.size, m.shape[0], _p(m), _p(sos)))
    return sos


def renormalize_sos(maps, sos, ctx: Context | None = None):
    """maps /= sqrt(sos) where sos > 0 (in place); sos is the all-channel sum of squares."""
    if hasattr(maps, "data_ptr"):
        _check(lib().sk_renormalize_sos(_ctx(ctx), sos.numel(), maps.shape[0], C.c_void_p(maps.data_ptr()),
                                        C.c_void_p(sos.data_ptr())))
        return maps
    if not (isinstance(maps, np.ndarray) and maps.dtype == np.complex64 and maps.flags.c_contiguous):
        raise ValueError("maps must be a contiguous complex64 array")
    s = np.ascontiguousarray(sos, dtype=np.float32)
    _check(lib().sk_renormalize_sos(_ctx(ctx), s.size, maps.shape[0], _p(maps), _p(s)))
    return maps


def estimate_maps_device(ctx: Context, calib_ptr: int, calib_dims, center_offset, q: int, full_dims,
                         cfg: PipelineConfig, maps_ptr: int, lambda_ptr: int, mask_ptr: int) -> sk_provenance:
    """Device-resident call (all buffers already in HBM): the bench's `value` leg."""
    prov = sk_provenance()
    cfgc = cfg.to_c()
    _check(lib().sk_estimate_maps(ctx.handle, len(calib_dims), _p(_i64(calib_dims)), _p(_i64(center_offset)), q,
                                  C.c_void_p(calib_ptr), _p(_i64(full_dims)), C.byref(cfgc), C.c_void_p(maps_ptr),
                                  C.c_void_p(lambda_ptr), C.c_void_p(mask_ptr), None, C.byref(prov)))
    return prov


def estimate_maps_batched_device(ctx: Context, calib_ptr: int, slices: int, calib_dims, center_offset, q: int,
                                 full_dims, cfg: PipelineConfig, maps_ptr: int, lambda_ptr: int, mask_ptr: int):
    """Multislice on device (or pinned host) buffers, slice-major; returns per-slice provenance."""
    prov = (sk_provenance * max(int(slices), 1))()
    cfgc = cfg.to_c()
    _check(lib().sk_estimate_maps_batched(ctx.handle, int(slices), len(calib_dims), _p(_i64(calib_dims)),
                                          _p(_i64(center_offset)), q, C.c_void_p(calib_ptr), _p(_i64(full_dims)),
                                          C.byref(cfgc), C.c_void_p(maps_ptr), C.c_void_p(lambda_ptr),
                                          C.c_void_p(mask_ptr), C.cast(prov, C.c_void_p)))
    return list(prov)[: int(slices)]


def estimate_maps_batched(calibs: np.ndarray, center_offset, full_dims, cfg: PipelineConfig,
                          ctx: Context | None = None):
    """Multislice: calibs (S, Q, *E) -> maps (S, Q, *full), lambda (S, *full), mask (S, *full)."""
    d = _c64(calibs)
    s, q, cdims = d.shape[0], d.shape[1], d.shape[2:]
    maps = np.zeros((s, q) + tuple(full_dims), dtype=np.complex64)
    lamb = np.zeros((s,) + tuple(full_dims), dtype=np.float32)
    mask = np.zeros((s,) + tuple(full_dims), dtype=np.uint8)
    prov = (sk_provenance * s)()
    cfgc = cfg.to_c()
    _check(lib().sk_estimate_maps_batched(_ctx(ctx), s, len(cdims), _p(_i64(cdims)), _p(_i64(center_offset)), q,
                                          _p(d), _p(_i64(full_dims)), C.byref(cfgc), _p(maps), _p(lamb), _p(mask),
                                          C.cast(prov, C.c_void_p)))
    return maps, lamb, mask, [dict(rank=int(p.nullspace_rank), total_ms=float(p.total_ms)) for p in prov]

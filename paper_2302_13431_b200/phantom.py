"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference's own generator (synthetic.cpp:70-153: disk/rectangle phantoms
with exactly band-limited random maps) does not implement BASELINE's ellipse
phantoms or coil rings, so this module is a new generator:

* phantom  rho(x) = sum of 10 ellipses (ellipsoids in 3-D) with seeded centres
  U(-0.25, 0.25) FOV, full axis lengths U(0.05, 0.4) FOV, random rotation,
  intensities U(0.2, 1), times exp(i * low-order polynomial phase);
* coil maps |c_q| = 1 / (1 + (r_q/0.6)^2), r_q = distance to coil q, times a
  linear phase, root-sum-of-squares normalised; coil geometries per config;
* k-space = unitary centred FFT of c_q * rho (fft.cpp:96-103 convention) plus
  complex Gaussian noise, sigma per component = sqrt(mean|s|^2 / (2*10^(SNR/10)))
  over the full grid;
* calibration = centred E^D block (types.cpp:58-90), stored as complex64 like
  the reference's CStack v1 float32 files (io.hpp:9-16).

Only the calibration block is needed by the pipeline, so it is evaluated
directly as a partial DFT of the image (separable per axis) instead of a full
grid FFT; the full k-space is produced on request for the small configs.

FOV convention: voxel j on an axis of extent n sits at x = (j - n//2)/n
(types.hpp:52-54).  Seeds use numpy's PCG64, so inputs are identical on every
machine.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

RECT, ELLIPSOID = 0, 1


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    full_dims: tuple
    channels: int
    calib: tuple
    tau: int
    grid_dims: tuple          # map grid (== full_dims for full-resolution configs)
    power_iters: int
    snr_db: float
    slices: int = 1
    nullspace_threshold: float = 0.05
    kernel: int = ELLIPSOID
    note: str = ""

    @property
    def ndim(self):
        return len(self.full_dims)

    @property
    def full_grid(self):
        return tuple(self.grid_dims) == tuple(self.full_dims)


CONFIGS = {
    "C1": ConfigSpec("C1", (256, 256), 8, (24, 24), 3, (64, 64), 30, 40.0,
                     note="2D single slice, 8-coil ring at 1.5 FOV; maps on 64^2 (grid_pad 40) interpolated to 256^2"),
    "C2": ConfigSpec("C2", (256, 256), 32, (32, 32), 5, (256, 256), 50, 35.0,
                     note="2D single slice, two rings of 16 at z=+-0.3 FOV; full-resolution G(x)"),
    "C3": ConfigSpec("C3", (256, 256), 32, (24, 24), 4, (128, 128), 10, 35.0, slices=128,
                     note="multislice 2D, 128 slices, C2's rings evaluated at each slice z; iters unstated -> 10"),
    "C4": ConfigSpec("C4", (256, 256, 128), 32, (24, 24, 24), 3, (128, 128, 64), 10, 35.0,
                     note="3D volume, 32 coils on a cylinder (4 rings of 8); iters unstated -> 10"),
    "C5": ConfigSpec("C5", (512, 512), 64, (40, 40), 6, (512, 512), 80, 30.0,
                     note="2D stress case, two concentric rings of 32"),
}


def coords(dims):
    """Broadcastable FOV coordinates per axis (types.hpp:52-54)."""
    out = []
    for a, n in enumerate(dims):
        shape = [1] * len(dims)
        shape[a] = n
        out.append(((np.arange(n) - n // 2) / n).reshape(shape))
    return out


def coil_positions(spec: ConfigSpec, z_slice: float = 0.0):
    """Coil centres (x, y, z) in FOV units."""
    q = spec.channels
    if spec.name == "C1":
        ang = 2 * np.pi * np.arange(q) / q
        return np.stack([1.5 * np.cos(ang), 1.5 * np.sin(ang), np.zeros(q)], 1)
    if spec.name in ("C2", "C3"):
        ang = 2 * np.pi * np.arange(16) / 16
        ring = lambda z, off: np.stack([1.5 * np.cos(ang + off), 1.5 * np.sin(ang + off), np.full(16, z)], 1)
        pos = np.concatenate([ring(0.3, 0.0), ring(-0.3, np.pi / 16)], 0)
        pos[:, 2] -= z_slice
        return pos
    if spec.name == "C4":
        ang = 2 * np.pi * np.arange(8) / 8
        rings = [np.stack([1.5 * np.cos(ang + k * np.pi / 16), 1.5 * np.sin(ang + k * np.pi / 16),
                           np.full(8, z)], 1) for k, z in enumerate((-0.375, -0.125, 0.125, 0.375))]
        return np.concatenate(rings, 0)
    if spec.name == "C5":
        ang = 2 * np.pi * np.arange(32) / 32
        r1 = np.stack([1.5 * np.cos(ang), 1.5 * np.sin(ang), np.zeros(32)], 1)
        r2 = np.stack([2.0 * np.cos(ang + np.pi / 32), 2.0 * np.sin(ang + np.pi / 32), np.zeros(32)], 1)
        return np.concatenate([r1, r2], 0)
    raise KeyError(spec.name)


def coil_maps(spec: ConfigSpec, dims, z_slice: float = 0.0):
    """(Q, *dims) complex128 RSS-normalised maps."""
    xs = coords(dims)
    nd = len(dims)
    pos = coil_positions(spec, z_slice)
    maps = np.empty((spec.channels,) + tuple(dims), dtype=np.complex128)
    for q in range(spec.channels):
        cx, cy, cz = pos[q]
        r2 = (xs[0] - cx) ** 2 + (xs[1] - cy) ** 2
        r2 = r2 + ((xs[2] - cz) ** 2 if nd == 3 else cz ** 2)
        mag = 1.0 / (1.0 + r2 / 0.36)
        th = np.arctan2(cy, cx)
        # linear phase: a ramp toward the coil plus a per-coil offset
        ph = th + 1.5 * (np.cos(th) * xs[0] + np.sin(th) * xs[1])
        maps[q] = mag * np.exp(1j * ph)
    rss = np.sqrt(np.sum(np.abs(maps) ** 2, axis=0))
    return maps / rss


def phantom(dims, rng: np.random.Generator, count: int = 10):
    """Sum of `count` seeded ellipses/ellipsoids times a smooth polynomial phase."""
    xs = coords(dims)
    nd = len(dims)
    rho = np.zeros(tuple(dims))
    for _ in range(count):
        c = rng.uniform(-0.25, 0.25, nd)
        semi = rng.uniform(0.05, 0.4, nd) / 2
        val = rng.uniform(0.2, 1.0)
        if nd == 2:
            th = rng.uniform(0, np.pi)
            u = (xs[0] - c[0]) * np.cos(th) + (xs[1] - c[1]) * np.sin(th)
            v = -(xs[0] - c[0]) * np.sin(th) + (xs[1] - c[1]) * np.cos(th)
            inside = (u / semi[0]) ** 2 + (v / semi[1]) ** 2 <= 1.0
        else:
            inside = sum(((xs[a] - c[a]) / semi[a]) ** 2 for a in range(nd)) <= 1.0
        rho = rho + val * inside
    coef = rng.normal(0.0, 1.0, 6) * np.array([np.pi, 2.0, 2.0, 2.0, 2.0, 2.0])
    x0, x1 = xs[0], xs[1]
    phase = coef[0] + coef[1] * x0 + coef[2] * x1 + coef[3] * x0 ** 2 + coef[4] * x0 * x1 + coef[5] * x1 ** 2
    return rho * np.exp(1j * phase)


def _partial_dft(img, calib_dims):
    """Unitary centred DFT of img evaluated only on the centred calib block.

    out[k] = N^-1/2 sum_x img[x] exp(-i 2 pi (k - c_n)(x - c_n)/n) per axis,
    restricted to k in [c_n - c_E, c_n - c_E + E)  (types.cpp:58-90 start).
    """
    out = img
    for a, (n, e) in enumerate(zip(img.shape[1:], calib_dims)):
        start = n // 2 - e // 2
        f = (np.arange(start, start + e) - n // 2)[:, None]
        x = (np.arange(n) - n // 2)[None, :]
        mat = np.exp(-2j * np.pi * f * x / n)
        out = np.moveaxis(np.tensordot(out, mat, axes=([a + 1], [1])), -1, a + 1)
    return out / np.sqrt(np.prod(img.shape[1:]))


def full_kspace(img):
    axes = tuple(range(1, img.ndim))
    n = np.prod(img.shape[1:])
    return np.fft.fftshift(np.fft.fftn(np.fft.ifftshift(img, axes=axes), axes=axes), axes=axes) / np.sqrt(n)


@dataclass
class Case:
    spec: ConfigSpec
    calib: np.ndarray                # (S, Q, *E) complex64  (S = slices)
    center_offset: tuple
    kspace: np.ndarray | None = None  # (S, Q, *dims) complex64, on request
    true_maps: np.ndarray | None = None
    extra: dict = field(default_factory=dict)


def generate(name: str, seed: int = 1234, with_kspace: bool = False, slices: int | None = None,
             full_dims=None, channels: int | None = None, slice_range=None) -> Case:
    """Seeded case for config `name` (C1..C5).

    `slices` limits C3's slice count (first `slices` slices); `slice_range`
    = (start, stop) generates only that block.  Every slice has its own RNG
    stream (seed, slice index), so a shard's data does not depend on how the
    slices are partitioned across ranks.
    """
    spec = CONFIGS[name]
    if full_dims is not None or channels is not None:
        spec = ConfigSpec(**{**spec.__dict__, **({"full_dims": tuple(full_dims)} if full_dims else {}),
                             **({"channels": channels} if channels else {})})
    dims = spec.full_dims
    ns = spec.slices if slices is None else slices
    start, stop = slice_range if slice_range is not None else (0, ns)
    calibs, kss, tms = [], [], []
    for s in range(start, stop):
        rng = np.random.Generator(np.random.PCG64([seed, s]))
        z = (s - spec.slices // 2) / spec.slices if spec.slices > 1 else 0.0
        maps = coil_maps(spec, dims, z_slice=z)
        rho = phantom(dims, rng)
        img = maps * rho[None]
        energy = np.mean(np.abs(img) ** 2)  # = mean |s|^2 by Parseval (unitary transform)
        sigma = np.sqrt(energy / (2.0 * 10.0 ** (spec.snr_db / 10.0)))
        cal = _partial_dft(img, spec.calib)
        cal = cal + sigma * (rng.standard_normal(cal.shape) + 1j * rng.standard_normal(cal.shape))
        calibs.append(cal.astype(np.complex64))
        if with_kspace:
            ks = full_kspace(img)
            ks = ks + sigma * (rng.standard_normal(ks.shape) + 1j * rng.standard_normal(ks.shape))
            # keep the calib block identical to the returned calibration
            sl = tuple(slice(n // 2 - e // 2, n // 2 - e // 2 + e) for n, e in zip(dims, spec.calib))
            ks[(slice(None),) + sl] = cal
            kss.append(ks.astype(np.complex64))
            tms.append(maps.astype(np.complex64))
    co = tuple(e // 2 for e in spec.calib)
    return Case(spec, np.stack(calibs), co, np.stack(kss) if with_kspace else None,
                np.stack(tms) if with_kspace else None)


def generate_variants(name: str, count: int, seed: int = 1234, slice_range=None) -> Case:
    """`count` distinct inputs of config `name` for the bench's timed steps:
    variant 0 is exactly generate(name, seed, slice_range=...); variant v >= 1
    keeps each slice's phantom and coils and draws a fresh noise realisation
    from the stream (seed, slice, v), so every step sees a different Gram.
    Returns a Case whose calib is (count, S, Q, *E) complex64."""
    spec = CONFIGS[name]
    dims = spec.full_dims
    start, stop = slice_range if slice_range is not None else (0, spec.slices)
    out = np.empty((count, stop - start, spec.channels) + tuple(spec.calib), dtype=np.complex64)
    for i, s in enumerate(range(start, stop)):
        rng = np.random.Generator(np.random.PCG64([seed, s]))
        z = (s - spec.slices // 2) / spec.slices if spec.slices > 1 else 0.0
        img = coil_maps(spec, dims, z_slice=z) * phantom(dims, rng)[None]
        sigma = np.sqrt(np.mean(np.abs(img) ** 2) / (2.0 * 10.0 ** (spec.snr_db / 10.0)))
        clean = _partial_dft(img, spec.calib)
        for v in range(count):
            r = rng if v == 0 else np.random.Generator(np.random.PCG64([seed, s, v]))
            out[v, i] = clean + sigma * (r.standard_normal(clean.shape) + 1j * r.standard_normal(clean.shape))
    return Case(spec, out, tuple(e // 2 for e in spec.calib))

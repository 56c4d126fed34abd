"""CStack v1 files (the reference's on-disk stack format, io.hpp / io.cpp:23-96).

A stack is a JSON sidecar ``<base>.json`` ({"version": 1, "dims": [...],
"channels": Q, "domain": "kspace" | "image"}) plus ``<base>.craw``: Q x dims
complex values, channel-major, row-major, as interleaved float32 (re, im).
The interleaved float32 layout is exactly ``sk_c64``, so a loaded stack goes
to the C-ABI without conversion.  Errors raise IoError (CLI exit code 3).
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np


class IoError(RuntimeError):
    """types.hpp IoError."""


@dataclass
class Stack:
    data: np.ndarray  # (Q, *dims) complex64
    domain: str       # "kspace" | "image"

    @property
    def dims(self):
        return tuple(self.data.shape[1:])

    @property
    def channels(self):
        return self.data.shape[0]


def base_of(path: str) -> str:  # io.cpp:16-20
    for ext in (".json", ".craw"):
        if path.endswith(ext):
            return path[: -len(ext)]
    return path


def load_stack(path: str) -> Stack:  # io.cpp:23-69
    base = base_of(path)
    try:
        with open(base + ".json") as f:
            try:
                meta = json.load(f)
            except json.JSONDecodeError as e:
                raise IoError(f"malformed sidecar {base}.json: {e}") from None
    except OSError:
        raise IoError(f"cannot open sidecar {base}.json") from None
    if meta.get("version") != 1:
        raise IoError(f"unsupported CStack version in {base}.json")
    try:
        dims = tuple(int(d) for d in meta["dims"])
        channels = int(meta["channels"])
        domain = meta["domain"]
    except (KeyError, TypeError, ValueError) as e:
        raise IoError(f"malformed sidecar {base}.json: {e}") from None
    if domain not in ("kspace", "image"):
        raise IoError(f"unknown domain tag '{domain}' in {base}.json")
    if channels < 1 or not dims or any(d < 1 for d in dims):
        raise IoError(f"invalid stack shape in {base}.json")
    count = channels * int(np.prod(dims))
    raw = base + ".craw"
    try:
        size = os.path.getsize(raw)
    except OSError:
        raise IoError(f"cannot stat raw file {raw}") from None
    expected = count * 2 * 4
    if size != expected:
        raise IoError(f"raw size mismatch for {raw}: got {size} bytes, expected {expected}")
    try:
        buf = np.fromfile(raw, dtype="<f4", count=2 * count)
    except OSError:
        raise IoError(f"cannot open raw file {raw}") from None
    if buf.size != 2 * count:
        raise IoError(f"short read from {raw}")
    return Stack(buf.view(np.complex64).reshape((channels,) + dims), domain)


def save_stack(stack: Stack, path: str) -> None:  # io.cpp:71-96
    base = base_of(path)
    data = np.ascontiguousarray(stack.data, dtype=np.complex64)
    meta = {"version": 1, "dims": list(data.shape[1:]), "channels": int(data.shape[0]), "domain": stack.domain}
    try:
        with open(base + ".json", "w") as f:
            f.write(json.dumps(meta, indent=2) + "\n")
        data.view("<f4").tofile(base + ".craw")
    except OSError as e:
        raise IoError(f"write failure on {base}: {e}") from None


def save_pgm16(values: np.ndarray, path: str) -> None:  # io.cpp:98-118 (2-D, big-endian 16-bit)
    v = np.asarray(values, dtype=np.float64)
    if v.ndim != 2:
        raise ValueError("PGM export is 2-D only")
    vmax = v.max() if v.size else 0.0
    scale = 65535.0 / vmax if vmax > 0 else 0.0
    u = np.clip(v * scale + 0.5, 0, 65535).astype(">u2")
    try:
        with open(path, "wb") as f:
            f.write(f"P5\n{v.shape[1]} {v.shape[0]}\n65535\n".encode())
            f.write(u.tobytes())
    except OSError as e:
        raise IoError(f"cannot write {path}: {e}") from None

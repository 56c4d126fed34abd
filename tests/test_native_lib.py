"""CPU-side checks of the product library (no GPU needed).

The C-ABI shared library must load and export every entry point that
include/senskit_b200.h declares; the host-only utilities (make_support,
reduced_grid_dims) must match the oracle.  No compute call touches CUDA here.
"""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "senskit_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sk_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_reference_entry_points():
    syms = declared_symbols()
    for name in ["sk_gram_fft", "sk_extract_nullspace", "sk_aggregate_w", "sk_gram_field_fast", "sk_espirit_inplace",
                 "sk_eig_power_field", "sk_normalize_maps", "sk_interpolate_maps", "sk_interpolate_real",
                 "sk_support_mask", "sk_estimate_maps", "sk_make_support", "sk_reduced_grid_dims",
                 "sk_build_calib_matrix", "sk_gram_explicit", "sk_eig_dense_field"]:
        assert name in syms


def test_library_exports_every_declared_symbol():
    import paper_2302_13431_b200 as K
    lib = ctypes.CDLL(K.library_path)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    import subprocess
    import paper_2302_13431_b200 as K
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", K.library_path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("nd", [1, 2, 3])
@pytest.mark.parametrize("tau", [0, 1, 3, 6])
@pytest.mark.parametrize("shape", [0, 1])
def test_make_support_matches_oracle(O, nd, tau, shape):
    import paper_2302_13431_b200 as K
    if nd == 3 and tau == 6:
        pytest.skip("large")
    assert np.array_equal(K.make_support(shape, tau, nd), O.make_support(shape, tau, nd))


def test_reduced_grid_dims():  # test_maps.cpp:13-17
    import paper_2302_13431_b200 as K
    assert K.reduced_grid_dims((24, 24), 24, (256, 256)) == (48, 48)
    assert K.reduced_grid_dims((240, 240), 24, (256, 256)) == (256, 256)
    assert K.reduced_grid_dims((24, 24), 0, (256, 256)) == (24, 24)


def test_make_support_errors():
    import paper_2302_13431_b200 as K
    with pytest.raises(K.DimError):
        K.make_support(0, -1, 2)
    with pytest.raises(K.DimError):
        K.make_support(0, 1, 0)


def test_context_without_gpu_fails_loudly():
    import torch
    import paper_2302_13431_b200 as K
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(K.SensKitError):
        K.Context(0)

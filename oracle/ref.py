"""ORACLE — TEST INFRASTRUCTURE ONLY.

The reference itself: the same Python API as ``oracle.oracle`` (every function,
same arguments and return values), bound to ``oracle/_ref/libsk_ref.so`` — the
unmodified ``/root/reference/proj/src`` sources compiled by
``oracle/Makefile.ref`` against the Eigen-subset shim in ``oracle/ref_shim``.
Used to pin the FP64 restatement (tests/test_ref_pin.py), to generate the
golden fixtures (tools/make_golden.py) and as bench.py's reference arm.
Only tests/, tools/, __graft_entry__ and bench.py's CPU legs may import it.
"""
import importlib.util as _ilu
import os as _os
import sys as _sys

_HERE = _os.path.dirname(_os.path.abspath(__file__))
_spec = _ilu.spec_from_file_location("oracle._ref_api", _os.path.join(_HERE, "oracle.py"))
_mod = _ilu.module_from_spec(_spec)
_sys.modules["oracle._ref_api"] = _mod
_spec.loader.exec_module(_mod)
_mod._LIB_PATH = _mod.REF_LIB_PATH


def available() -> bool:
    return _os.path.exists(_mod.REF_LIB_PATH)


def __getattr__(name):
    return getattr(_mod, name)

"""paper_2302_13431_b200 — B200-native PISCO sensitivity-map hot path.

The product is the C-ABI library ``lib/libsenskit_b200.so`` (CUDA sm_100a
kernels + host runtime, declared in ``include/senskit_b200.h``).  This module
is the Python host mirror of the reference's C++ entry points
(``proj/include/senskit/*.hpp``): same names, argument meanings and error
classes, so the parity tests read like the reference's own tests.  It loads
the native library and raises if it is missing — there is no CPU fallback.
"""
from .api import *  # noqa: F401,F403
from .api import __all__  # noqa: F401

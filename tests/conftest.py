import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def O():
    from oracle import oracle
    oracle.lib()
    return oracle


def load_ref():
    """oracle/_ref: the unmodified reference sources compiled against oracle/ref_shim.
    Built on demand where /root/reference exists (this container); on the GPU box
    the prebuilt library travels with the repo snapshot."""
    import subprocess
    from oracle import ref
    if not ref.available():
        if os.path.isdir("/root/reference/proj/src"):
            subprocess.run(["make", "-C", ROOT, "-f", "oracle/Makefile.ref"], check=True,
                           stdout=subprocess.DEVNULL)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    ref.lib()
    return ref


@pytest.fixture(scope="session")
def R():
    return load_ref()

"""A compiled C++ client of include/senskit_b200.h (tests/abi_smoke.cpp): the
header must compile as C++ (and as C), link against the product library and
run; host-only entry points on CPU, the full pipeline under -m gpu."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2302_13431_b200", "lib")


def _build(tmp_path):
    exe = str(tmp_path / "abi_smoke")
    cuda = "/usr/local/cuda"
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", os.path.join(ROOT, "tests", "abi_smoke.cpp"), "-I",
                    os.path.join(ROOT, "include"), "-I", f"{cuda}/include", "-L", LIBDIR, "-lsenskit_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-L", f"{cuda}/lib64", "-lcudart", f"-Wl,-rpath,{cuda}/lib64", "-o", exe],
                   check=True)
    return exe


def test_header_compiles_as_c(tmp_path):
    src = tmp_path / "h.c"
    src.write_text('#include "senskit_b200.h"\nint main(void) { sk_config c; sk_provenance p; (void)c; (void)p; '
                   'return SK_OK; }\n')
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                    str(tmp_path / "h")], check=True)


def test_abi_smoke_host_only(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "--no-gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_abi_smoke_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr

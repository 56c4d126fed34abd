"""CStack v1 I/O (io.cpp:23-118) and the estimate CLI's host logic
(senskit_main.cpp:23-27, 139-184) on CPU: file round trips, error classes and
exit codes that are decided before any device work."""
import json

import numpy as np
import pytest

from paper_2302_13431_b200 import cli
from paper_2302_13431_b200.cstack import IoError, Stack, load_stack, save_pgm16, save_stack


def _stack(shape=(3, 6, 5), seed=0, domain="kspace"):
    r = np.random.default_rng(seed)
    return Stack((r.standard_normal(shape) + 1j * r.standard_normal(shape)).astype(np.complex64), domain)


def test_round_trip_and_layout(tmp_path):
    s = _stack()
    save_stack(s, str(tmp_path / "k.json"))  # base_of strips .json / .craw
    meta = json.loads((tmp_path / "k.json").read_text())
    assert meta == {"version": 1, "dims": [6, 5], "channels": 3, "domain": "kspace"}
    raw = np.fromfile(tmp_path / "k.craw", dtype="<f4")
    assert raw.size == 2 * s.data.size and raw[0] == s.data[0, 0, 0].real and raw[1] == s.data[0, 0, 0].imag
    back = load_stack(str(tmp_path / "k.craw"))
    assert back.domain == "kspace" and np.array_equal(back.data, s.data)


@pytest.mark.parametrize("mutate,msg", [
    (lambda p: (p / "k.json").unlink(), "cannot open sidecar"),
    (lambda p: (p / "k.json").write_text("{"), "malformed sidecar"),
    (lambda p: (p / "k.json").write_text(json.dumps({"version": 2, "dims": [6, 5], "channels": 3,
                                                      "domain": "kspace"})), "unsupported CStack version"),
    (lambda p: (p / "k.json").write_text(json.dumps({"version": 1, "dims": [6, 5], "channels": 3,
                                                      "domain": "xspace"})), "unknown domain tag"),
    (lambda p: (p / "k.craw").write_bytes(b"\0" * 8), "raw size mismatch"),
    (lambda p: (p / "k.craw").unlink(), "cannot stat raw file"),
])
def test_load_errors(tmp_path, mutate, msg):  # io.cpp:26-62
    save_stack(_stack(), str(tmp_path / "k"))
    mutate(tmp_path)
    with pytest.raises(IoError, match=msg):
        load_stack(str(tmp_path / "k"))


def test_pgm16(tmp_path):  # io.cpp:98-118
    v = np.array([[0.0, 1.0, 2.0], [4.0, 3.0, 0.5]])
    save_pgm16(v, str(tmp_path / "m.pgm"))
    data = (tmp_path / "m.pgm").read_bytes()
    header = b"P5\n3 2\n65535\n"
    assert data.startswith(header)
    px = np.frombuffer(data[len(header):], dtype=">u2").reshape(2, 3)
    assert px[1, 0] == 65535 and px[0, 0] == 0 and px[0, 2] == int(2 * 65535 / 4 + 0.5)


def test_extract_calibration_centered():  # types.cpp:58-90
    d = np.arange(2 * 7 * 6, dtype=np.complex64).reshape(2, 7, 6)
    c = cli.extract_calibration(d, (3, 4))
    assert c.center_offset == (1, 2)
    assert np.array_equal(c.data, d[:, 2:5, 1:5])


def test_parse_extents():  # senskit_main.cpp:29-43
    import argparse
    assert cli.parse_extents("24", 2) == (24, 24)
    assert cli.parse_extents("24,20,8", 3) == (24, 20, 8)
    assert cli.parse_extents("24,20,", 2) == (24, 20)       # trailing comma ends the scan
    assert cli.parse_extents(" 24x,+8", 2) == (24, 8)       # std::stoll: whitespace, sign, trailing text
    with pytest.raises(argparse.ArgumentTypeError):          # CLI::ValidationError -> exit 2
        cli.parse_extents("24,20", 3)
    with pytest.raises(argparse.ArgumentTypeError):
        cli.parse_extents("", 2)
    for bad in ("abc", ",24", "24,,8", "99999999999999999999"):  # std::invalid_argument / out_of_range -> exit 1
        with pytest.raises((ValueError, OverflowError)):
            cli.parse_extents(bad, 2)


def test_exit_codes_before_device_work(tmp_path, capsys):  # senskit_main.cpp:23-27
    base = str(tmp_path / "k")
    save_stack(_stack((2, 16, 16)), base)
    with pytest.raises(SystemExit) as e:  # bad flags -> 2 (argparse)
        cli.main(["estimate", "--input", base])
    assert e.value.code == 2
    assert cli.main(["estimate", "--input", str(tmp_path / "nope"), "--calib", "8", "--output", base + "o"]) == 3
    save_stack(_stack((2, 16, 16), domain="image"), str(tmp_path / "img"))
    assert cli.main(["estimate", "--input", str(tmp_path / "img"), "--calib", "8", "--output", base + "o"]) == 3
    assert cli.main(["estimate", "--input", base, "--calib", "32", "--output", base + "o"]) == 5  # DimError
    assert cli.main(["estimate", "--input", base, "--calib", "8", "--preset", "nope",
                     "--output", base + "o"]) == 2
    assert cli.main(["estimate", "--input", base, "--calib", "8,8,8", "--output", base + "o"]) == 2  # count
    assert cli.main(["estimate", "--input", base, "--calib", "8,x", "--output", base + "o"]) == 1  # stoll


def test_config_from_flags_mirrors_reference():  # senskit_main.cpp:54-76
    import argparse
    ns = argparse.Namespace(preset="baseline", kernel=None, gram=None, grid=None, eig=None, method=None, field=None,
                            tau=-1, power_iters=0, nullspace_threshold=0.0, mask_threshold=-1.0, apod_width=0.0,
                            grid_pad=-1)
    cfg = cli.config_from_flags(ns)
    assert (cfg.kernel, cfg.gram, cfg.grid, cfg.eig) == (0, 0, 0, 0)  # maps.cpp:12-19
    ns.preset, ns.eig, ns.method, ns.field, ns.gram, ns.tau = "pisco", "dense", "nullspace", "naive", "explicit", 4
    cfg = cli.config_from_flags(ns)
    assert (cfg.kernel, cfg.grid, cfg.eig, cfg.method, cfg.field, cfg.gram, cfg.tau) == (1, 1, 0, 0, 0, 0, 4)
    ns.preset = "nope"
    with pytest.raises(argparse.ArgumentTypeError):
        cli.config_from_flags(ns)

"""Instance file formats vs the reference's recorded behaviour (tests/golden/io_cases.json,
made by oracle/gen_golden_io.py from leanot.io): same arrays / bytes / texts, same errors."""

import base64
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2511_11359_b200 import io as IO

CASES = json.loads((Path(__file__).resolve().parent / "golden" / "io_cases.json").read_text())["cases"]


def _arr(d):
    return np.array(d["data"], dtype=float).reshape(d["shape"])


def _check(case, fn, path=None):
    if "error" in case:
        with pytest.raises(Exception) as ei:
            fn()
        assert type(ei.value).__name__ == case["error"]
        msg = str(ei.value)
        if path is not None:
            msg = msg.replace(str(path), "<path>")
        assert msg == case["message"]
    else:
        got = fn()
        want = case["ok"]
        if isinstance(want, dict):
            assert list(got.shape) == want["shape"]
            np.testing.assert_array_equal(got, _arr(want))
        else:
            assert got == want


@pytest.mark.parametrize("name", sorted(CASES["read_pgm"]))
def test_read_pgm(name, tmp_path):
    case = CASES["read_pgm"][name]
    f = tmp_path / "in.pgm"
    f.write_bytes(base64.b64decode(case["input"]))
    _check(case, lambda: IO.read_pgm(f))


@pytest.mark.parametrize("name", sorted(CASES["write_pgm"]))
def test_write_pgm(name, tmp_path):
    case = CASES["write_pgm"][name]
    f = tmp_path / "out.pgm"

    def run():
        IO.write_pgm(f, _arr(case["image"]), maxval=case["maxval"])
        return base64.b64encode(f.read_bytes()).decode()
    _check(case, run)


@pytest.mark.parametrize("name", sorted(CASES["read_histogram_csv"]))
def test_read_histogram_csv(name, tmp_path):
    case = CASES["read_histogram_csv"][name]
    f = tmp_path / "in.csv"
    f.write_bytes(case["input"].encode())
    _check(case, lambda: IO.read_histogram_csv(f), f)


@pytest.mark.parametrize("name", sorted(CASES["write_histogram_csv"]))
def test_write_histogram_csv(name, tmp_path):
    case = CASES["write_histogram_csv"][name]
    f = tmp_path / "h.csv"

    def run():
        IO.write_histogram_csv(f, _arr(case["weights"]))
        return f.read_text()
    _check(case, run)


@pytest.mark.parametrize("name", sorted(CASES["write_matrix_csv"]))
def test_write_matrix_csv(name, tmp_path):
    case = CASES["write_matrix_csv"][name]
    f = tmp_path / "m.csv"

    def run():
        IO.write_matrix_csv(f, _arr(case["matrix"]))
        return f.read_text()
    _check(case, run)


@pytest.mark.parametrize("name", sorted(CASES["block_mean_downsample"]))
def test_block_mean_downsample(name):
    case = CASES["block_mean_downsample"][name]
    _check(case, lambda: IO.block_mean_downsample(_arr(case["image"]), case["factor"]))


def test_roundtrip_pgm_to_histogram(tmp_path):
    """PGM -> downsample -> normalized histogram, the DOTmark instance path (cli.py:188-199)."""
    from paper_2511_11359_b200.core import Histogram
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, size=(16, 12)).astype(float)
    f = tmp_path / "img.pgm"
    IO.write_pgm(f, img, maxval=255)
    back = IO.read_pgm(f)
    assert back.shape == (16, 12)
    h = Histogram.normalized(IO.block_mean_downsample(back, 4).ravel() + 1e-6)
    assert h.weights.shape == (12,) and abs(h.weights.sum() - 1.0) <= 1e-12

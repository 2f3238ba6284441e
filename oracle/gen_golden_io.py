"""Golden cases for the instance file formats, produced by running the REFERENCE leanot.io.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_io.py

Writes tests/golden/io_cases.json: PGM byte strings / CSV texts / arrays fed to the
reference's read_pgm, write_pgm, read_histogram_csv, write_histogram_csv,
write_matrix_csv and block_mean_downsample (io.py:21-123), with the reference's output
or the exception it raised.  tests/test_io.py replays them against
paper_2511_11359_b200.io (test infrastructure; the reference does not travel).
"""

from __future__ import annotations

import base64
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from leanot import io as RIO  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden" / "io_cases.json"

PGM_INPUTS = {
    "p2_comments": b"P2\n# a comment\n3 2\n# another\n255\n0 128 255\n1 2 3\n",
    "p5_8bit": b"P5\n# c\n4 3\n200\n" + bytes([0, 10, 20, 30, 40, 50, 60, 70, 80, 90, 100, 200]),
    "p5_16bit": b"P5 2 2 1000\n" + np.array([0, 999, 1000, 500], dtype=">u2").tobytes(),
    "p2_truncated": b"P2\n3 3\n255\n1 2 3 4\n",
    "bad_magic": b"P6\n1 1\n255\n\x00\x00\x00",
    "truncated_header": b"P5\n4 # only two tokens\n",
    "zero_width": b"P2\n0 3\n255\n",
    "maxval_too_big": b"P2\n1 1\n70000\n5\n",
    "exceeds_maxval": b"P2\n2 1\n10\n5 11\n",
    "p5_short": b"P5\n4 4\n255\n" + bytes(range(10)),
    "cr_comment": b"P2\r# cr comment\r2 2\r15\r1 2\r3 4\r",
    "p2_extra_tokens": b"P2 2 1 9 1 2 3 4 5",
    "p2_float_tokens": b"P2 2 1 9\n1.5 2e0\n",
    "p5_whitespace_pixel": b"P5\n2 1\n255\n\x20\x09",
    "tabs": b"P2\t1\t1\t7\t7",
}

CSV_INPUTS = {
    "plain": "0.25\n0.25\n0.5\n",
    "header": "weight\n0.1\n0.9\n",
    "blank_lines": "\n0.5\n\n0.5\n\n",
    "blank_then_header": "\nweight\n1.0\n",
    "bad_later": "0.5\nfoo\n0.5\n",
    "empty": "",
    "header_only": "w\n",
    "crlf": "h\r\n0.5\r\n0.5\r\n",
    "spaces": "  1e-3  \n\t2\n",
    "scientific": "1.5e+2\n-0\ninf\n",
}


def arr(a):
    a = np.asarray(a, dtype=float)
    return {"shape": list(a.shape), "data": [float(v) for v in a.ravel()]}


def capture(fn):
    try:
        return {"ok": fn()}
    except Exception as e:  # the reference's own exception, recorded verbatim
        return {"error": type(e).__name__, "message": str(e)}


def main():
    rng = np.random.default_rng(77)
    cases = {"read_pgm": {}, "write_pgm": {}, "read_histogram_csv": {}, "write_histogram_csv": {},
             "write_matrix_csv": {}, "block_mean_downsample": {}}
    with tempfile.TemporaryDirectory() as td:
        tdp = Path(td)
        for name, raw in PGM_INPUTS.items():
            f = tdp / f"{name}.pgm"
            f.write_bytes(raw)
            res = capture(lambda: arr(RIO.read_pgm(f)))
            cases["read_pgm"][name] = {"input": base64.b64encode(raw).decode(), **res}
        imgs = {
            "random": (rng.random((5, 7)) * 3.0, 255),
            "zeros": (np.zeros((2, 3)), 255),
            "negative": (-rng.random((3, 3)), 255),
            "halfway": (np.array([[0.0, 0.5, 1.0, 1.5, 2.0, 2.5], [3.0, 3.5, 4.0, 4.5, 5.0, 10.0]]), 20),
            "maxval256": (rng.random((4, 4)), 256),
            "maxval65535": (rng.random((3, 5)) * 100.0, 65535),
            "one_pixel": (np.array([[7.0]]), 255),
            "not_2d": (rng.random(5), 255),
        }
        for name, (img, mv) in imgs.items():
            f = tdp / f"w_{name}.pgm"

            def w(img=img, mv=mv, f=f):
                RIO.write_pgm(f, img, maxval=mv)
                return base64.b64encode(f.read_bytes()).decode()
            cases["write_pgm"][name] = {"image": arr(img), "maxval": mv, **capture(w)}
        for name, text in CSV_INPUTS.items():
            f = tdp / f"{name}.csv"
            f.write_bytes(text.encode())
            res = capture(lambda: arr(RIO.read_histogram_csv(f)))
            if "error" in res:  # the path is part of the message: store it relative
                res["message"] = res["message"].replace(str(f), "<path>")
            cases["read_histogram_csv"][name] = {"input": text, **res}
        vecs = {"random": rng.random(6), "tiny": np.array([1e-300, 5e-324, 0.1, 1.0 / 3.0]),
                "matrix_like": rng.random((2, 3))}
        for name, v in vecs.items():
            f = tdp / f"h_{name}.csv"

            def wh(v=v, f=f):
                RIO.write_histogram_csv(f, v)
                return f.read_text()
            cases["write_histogram_csv"][name] = {"weights": arr(v), **capture(wh)}
        mats = {"random": rng.random((3, 4)), "row": rng.random((1, 5)), "special": np.array([[0.0, -1.5], [1e20, 2.0 / 3.0]])}
        for name, m in mats.items():
            f = tdp / f"m_{name}.csv"

            def wm(m=m, f=f):
                RIO.write_matrix_csv(f, m)
                return f.read_text()
            cases["write_matrix_csv"][name] = {"matrix": arr(m), **capture(wm)}
        img = rng.random((12, 8))
        for fac in (1, 2, 4, 3, 0, 5):
            cases["block_mean_downsample"][str(fac)] = {"image": arr(img), "factor": fac,
                                                        **capture(lambda: arr(RIO.block_mean_downsample(img, fac)))}
    OUT.write_text(json.dumps({"numpy": np.__version__, "cases": cases}, indent=1))
    print("wrote", OUT)


if __name__ == "__main__":
    main()

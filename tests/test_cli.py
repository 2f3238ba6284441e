"""CLI surface (cli.py) without a GPU: parser, flags, exit codes, instance generation,
downsampling, bad-input handling (the solver sub-commands run in tests/test_gpu_cli.py).

The reference's CLI cannot be imported as shipped, so the contract
is its source: sub-commands and flags (cli.py:459-520), exit codes (cli.py:46-48,
523-542), artifacts (cli.py:152-167) and generators (cli.py:401-451).
"""

import json

import numpy as np

from paper_2511_11359_b200 import cli
from paper_2511_11359_b200 import io as lio


def test_parser_has_reference_flags():
    p = cli.build_parser()
    a = p.parse_args(["solve", "--r", "a.csv", "--c", "b.csv", "--out", "o", "--tau-mu", "0.05",
                      "--eps", "1e-4", "--clock", "fixed", "--dense-cap", "0"])
    assert (a.solver, a.scheme, a.tau_mu, a.eps, a.clock, a.dense_cap, a.log_stride) == \
        ("dxg", "tuned", 0.05, 1e-4, "fixed", 0, 25)
    b = p.parse_args(["barycenter", "--marginal", "x.pgm", "--marginal", "y.pgm", "--out", "o",
                      "--solver", "ibp", "--eta", "1e-3", "--render"])
    assert b.marginal == ["x.pgm", "y.pgm"] and b.solver == "ibp" and b.render


def test_bad_input_exit_codes(tmp_path):
    assert cli.main(["solve", "--r", str(tmp_path / "missing.csv"), "--c", "x", "--out", str(tmp_path)]) == 2
    assert cli.main(["nonsense"]) == 2
    assert cli.main(["gen", "--kind", "shapes", "--n", "10", "--out", str(tmp_path)]) == 2   # not a square
    assert cli.main(["solve", "--r", "a", "--c", "b"]) == 2                                  # --out missing


def test_gen_writes_instances_and_manifest(tmp_path):
    out = tmp_path / "inst"
    assert cli.main(["gen", "--kind", "gaussian-mixture", "--n", "256", "--seed", "3", "--out", str(out)]) == 0
    r = lio.read_histogram_csv(out / "r.csv")
    assert r.shape == (256,) and abs(r.sum() - 1.0) <= 1e-12 and np.all(r > 0)
    assert lio.read_pgm(out / "c.pgm").shape == (16, 16)
    man = json.loads((out / "manifest.json").read_text())
    assert man["config"]["command"] == "gen" and set(man["files"]) == {"r", "c"}
    assert cli.main(["gen", "--kind", "shapes", "--n", "64", "--out", str(tmp_path / "s")]) == 0
    assert sorted(p.name for p in (tmp_path / "s").glob("*.csv")) == ["shape1.csv", "shape2.csv", "shape3.csv"]
    assert cli.main(["gen", "--kind", "checkerboard", "--n", "64", "--out", str(tmp_path / "k")]) == 0
    a = lio.read_pgm(tmp_path / "k" / "a.pgm")
    b = lio.read_pgm(tmp_path / "k" / "b.pgm")
    assert np.array_equal(a + b, np.full_like(a, a.max()))


def test_gen_is_deterministic(tmp_path):
    for d in ("x", "y"):
        assert cli.main(["gen", "--kind", "gaussian-mixture", "--n", "100", "--seed", "7", "--out", str(tmp_path / d)]) == 0
    assert (tmp_path / "x" / "r.csv").read_bytes() == (tmp_path / "y" / "r.csv").read_bytes()


def test_downsample_keeps_values(tmp_path):
    img = np.arange(64, dtype=float).reshape(8, 8) * 2
    lio.write_pgm(tmp_path / "img.pgm", img, maxval=255, rescale=False)
    assert cli.main(["downsample", str(tmp_path / "img.pgm"), "--factor", "2", "--out", str(tmp_path / "s.pgm")]) == 0
    small = lio.read_pgm(tmp_path / "s.pgm")
    ref = lio.block_mean_downsample(lio.read_pgm(tmp_path / "img.pgm"), 2)
    assert np.array_equal(small, np.clip(np.rint(ref), 0, 255))
    assert cli.main(["downsample", str(tmp_path / "img.pgm"), "--factor", "3", "--out", str(tmp_path / "t.pgm")]) == 2

"""CLI solver sub-commands end to end on the GPU (cli.py:175-383 of the reference).

Instances come from `gen` (cli.py:428-451); runs write trajectory.csv / summary.json /
manifest.json (+ plan.csv, potentials.npy, barycenter.csv/.pgm).  With `--clock fixed`
two identical runs give byte-identical trajectories (SPEC acceptance criterion 11).
"""

import csv
import json

import numpy as np
import pytest

from paper_2511_11359_b200 import cli
from paper_2511_11359_b200 import io as lio

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def inst(tmp_path_factory):
    d = tmp_path_factory.mktemp("inst")
    assert cli.main(["gen", "--kind", "gaussian-mixture", "--n", "144", "--seed", "1", "--out", str(d)]) == 0
    return d


def _traj(path):
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["iter", "seconds", "primal", "dual", "gap", "col_infeas_l1", "s"]
    return rows[1:]


def test_solve_dxg_artifacts_and_byte_identical_trajectories(inst, tmp_path):
    outs = []
    for k in range(2):
        out = tmp_path / f"run{k}"
        rc = cli.main(["solve", "--r", str(inst / "r.csv"), "--c", str(inst / "c.csv"), "--tau-mu", "0.05",
                       "--eps", "1e-3", "--max-iter", "20000", "--clock", "fixed", "--out", str(out)])
        assert rc == 0
        outs.append(out)
    a = (outs[0] / "trajectory.csv").read_bytes()
    assert a == (outs[1] / "trajectory.csv").read_bytes()
    rows = _traj(outs[0] / "trajectory.csv")
    assert all(r[1] == "0.000000" for r in rows)
    s = json.loads((outs[0] / "summary.json").read_text())
    assert s["solver"] == "dxg" and s["converged"] and s["iterations"] == int(rows[-1][0])
    assert s["final"]["gap"] <= 1e-3 / 6 and s["final"]["col_infeas_l1"] <= 1e-3 / 6
    plan = np.loadtxt(outs[0] / "plan.csv", delimiter=",")
    assert plan.shape == (144, 144) and abs(plan.sum() - 1.0) <= 1e-9
    m = json.loads((outs[0] / "manifest.json").read_text())
    assert m["config"]["command"] == "solve" and m["files"]["plan"] == "plan.csv"


def test_solve_sinkhorn_and_barycenters(inst, tmp_path):
    out = tmp_path / "sk"
    assert cli.main(["solve", "--solver", "sinkhorn", "--eta", "0.01", "--r", str(inst / "r.csv"),
                     "--c", str(inst / "c.csv"), "--eps", "1e-6", "--out", str(out)]) == 0
    s = json.loads((out / "summary.json").read_text())
    assert s["converged"] and s["final"]["col_infeas_l1"] <= 1e-6 / 6
    assert np.load(out / "potentials.npy").shape == (2, 144)
    assert cli.main(["solve", "--solver", "sinkhorn", "--r", str(inst / "r.csv"), "--c", str(inst / "c.csv"),
                     "--out", str(out)]) == 2          # eta required
    for solver in ("dxg-barycenter", "ibp"):
        ob = tmp_path / solver
        rc = cli.main(["barycenter", "--solver", solver, "--marginal", str(inst / "r.pgm"), "--marginal",
                       str(inst / "c.pgm"), "--eta", "1e-2", "--tau-mu", "0.05", "--eps", "1e-2",
                       "--max-iter", "20000", "--render", "--out", str(ob)])
        assert rc == 0
        bary = lio.read_histogram_csv(ob / "barycenter.csv")
        assert bary.shape == (144,) and abs(bary.sum() - 1.0) <= 1e-9
        assert lio.read_pgm(ob / "barycenter.pgm").shape == (12, 12)
        s = json.loads((ob / "summary.json").read_text())
        assert s["m"] == 2 and s["converged"]

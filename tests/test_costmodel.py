"""Cost model (mirror of kcycle.costmodel) against the reference's values
(tests/golden/costmodel.json, produced by the real reference)."""

import math

import numpy as np
import pytest

from conftest import load_json
from paper_2010_00626_b200 import costmodel as cm

INF = math.inf


def kap(s):
    return INF if s == "W" else int(s)


def test_cells_match_reference():
    g = load_json("costmodel.json")
    for cell in g["cells"]:
        k, n = kap(cell["kappa"]), cell["n"]
        assert [cm.level_calls(k, l) for l in range(1, n + 1)] == cell["level_calls"]
        assert cm.total_calls(k, n) == cell["total_calls"]
        for nu, v in cell["n_gpu_calls"].items():
            assert cm.n_gpu_calls(k, n, int(nu)) == v
        assert cm.ops_per_unknown(k) == cell["ops_per_unknown"]
        assert cm.predict_runtime(cm.CostModelParams(2.48e-3, 1.18e-6, 4), k, n) == pytest.approx(
            cell["predicted_ms_paper"], rel=1e-15)
        if "histogram" in cell:
            assert {str(a): b for a, b in cm.coarse_counter_histogram(k, n).items()} == cell["histogram"]


def test_f_factor_and_n_ops():
    g = load_json("costmodel.json")
    for e in g["f_factor"]:
        if e["value"] is None:
            with pytest.raises(ValueError):
                cm.f_factor(kap(e["kappa"]), e["c"])
        else:
            assert cm.f_factor(kap(e["kappa"]), e["c"]) == pytest.approx(e["value"], rel=1e-15)
    spec = cm.OpCountSpec(C=1.3, Ctilde=2.7, N1=1.0)
    for e in g["n_ops"]:
        assert cm.n_ops_model(kap(e["kappa"]), e["c"], e["n"], spec) == pytest.approx(e["value"], rel=1e-13)


def test_turning_points_and_fit():
    g = load_json("costmodel.json")
    params = cm.CostModelParams(2.48e-3, 1.18e-6, 4)
    for e in g["turning_points"]:
        tp = cm.turning_point(params, kap(e["kappa"]))
        assert tp.n_tp == pytest.approx(e["n_tp"], rel=1e-12)
        assert tp.converged == e["converged"]
    rows = [(kap(k), n, t) for k, n, t in g["fit"]["rows"]]
    a, b = cm.fit_params(rows, nu=4)
    assert a == pytest.approx(g["fit"]["alpha"], rel=1e-10)
    assert b == pytest.approx(g["fit"]["beta"], rel=1e-10)


def test_paper_table1_turning_points():
    """PAPER.md:575-594 Table 1 with the paper's alpha, beta."""
    params = cm.CostModelParams(alpha=2.48e-3, beta=1.18e-6, nu=4)
    for kappa, want in ((1, 8.2), (2, 9.1), (3, 10.0), (INF, 12.4)):
        assert abs(cm.turning_point(params, kappa).n_tp - want) <= 0.4


def test_validation_and_degenerate():
    with pytest.raises(ValueError):
        cm.CostModelParams(alpha=-1.0, beta=0.0)
    with pytest.raises(ValueError):
        cm.total_calls(0, 3)
    with pytest.raises(cm.RankDeficientError):
        cm.fit_params([(2, 6, 1.0), (2, 6, 1.0)], nu=4)
    assert cm.turning_point(cm.CostModelParams(0.0, 1.0), 2).degenerate
    assert cm.level_calls(0, 5) == 0
    assert cm.binom_real(8.5, 2) == pytest.approx(31.875)


def test_launch_accounting_matches_dry_stats():
    d = load_json("dry_stats.json")
    for key, rec in d.items():
        n = int(key.split("_")[0][1:])
        k = kap(key.split("_")[1][1:])
        nu = int(key.split("_")[2][2]) + int(key.split("_")[2][3])
        assert cm.n_gpu_calls(k if k != INF else n, n, nu) == rec["kernel_launches"], key

"""CLI mirror against the reference CLI's own output.

tests/golden/cli.json holds the reference `kcycle` CLI (cli.py) stdout and
exit codes on fixed argument lists (tests/golden/make_golden.py cli).  The
model subcommands run on the CPU and must print identical text; `solve`
runs on the B200 engine and must report the same status, iteration count,
launch and op-unit accounting, with norms equal to 1e-10 relative (the
engine's norms are deterministic fp64 trees, the reference's are OpenBLAS
ddot; iterates are bit-identical).
"""

import contextlib
import io
import json
import math
import os
import sys

import pytest

from conftest import load_json

from paper_2010_00626_b200 import cli

CASES = load_json("cli.json")


def run(argv, stdin=None):
    buf = io.StringIO()
    old = sys.stdin
    if stdin is not None:
        sys.stdin = io.StringIO(stdin)
    try:
        with contextlib.redirect_stdout(buf):
            rc = cli.main(argv)
    finally:
        sys.stdin = old
    return rc, buf.getvalue()


def _ids(cases):
    return [" ".join(c["argv"]) for c in cases]


MODEL = [c for c in CASES if c["argv"][0] != "solve"]
SOLVE = [c for c in CASES if c["argv"][0] == "solve"]


@pytest.mark.parametrize("case", MODEL, ids=_ids(MODEL))
def test_model_subcommands_match_reference(case):
    rc, out = run(case["argv"], case["stdin"])
    assert rc == case["exit"]
    assert out == case["stdout"]


def test_usage_errors_exit_2():
    for argv in (["calls", "--kappa", "0", "--levels", "3"], ["calls", "--kappa", "x", "--levels", "3"],
                 ["bench", "--kappa", "1", "--levels", "0"]):
        with pytest.raises(SystemExit) as e:
            cli.main(argv)
        assert e.value.code == 2


def test_fit_rank_deficient_exit_5():
    rc, _ = run(["fit"], "kappa,levels,ms\n1,4,0.1\n")
    assert rc == 5


def _close(a, b, rel):
    if a is None or b is None:
        return a is b
    return math.isclose(float(a), float(b), rel_tol=rel, abs_tol=0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("case", SOLVE, ids=_ids(SOLVE))
def test_solve_matches_reference(case):
    rc, out = run(case["argv"])
    assert rc == case["exit"]
    if "record" in case:
        got = json.loads(out)
        ref = case["record"]
        assert got["config"] == ref["config"]
        g, r = got["result"], ref["result"]
        for k in ("status", "iterations", "launches", "op_units"):
            assert g[k] == r[k], k
        assert _close(g["initial_norm"], r["initial_norm"], 1e-10)
        if "pcg" in case["argv"]:
            # PCG: alpha/beta differ in the last bit, so the iterates drift at
            # ~1e-16 of the initial scale; compare relative to the initial norm
            assert abs(g["final_norm"] - r["final_norm"]) <= 1e-10 * r["initial_norm"]
            assert _close(g["asymptotic_factor"], r["asymptotic_factor"], 1e-4)
        else:
            assert _close(g["final_norm"], r["final_norm"], 1e-10)
            assert _close(g["asymptotic_factor"], r["asymptotic_factor"], 1e-8)
    else:
        hdr, row = [line.split(",") for line in out.strip().splitlines()]
        assert hdr == case["csv_header"]
        row = dict(zip(hdr, row))
        for k, v in case["csv_row"].items():
            if k in ("initial_norm", "final_norm", "asymptotic_factor"):
                assert _close(row[k], v, 1e-8), k
            else:
                assert row[k] == v, k


@pytest.mark.gpu
def test_bench_timed_matches_reference_counts():
    """`bench --reps 2` (bench_cycle's timed path, cycle.py:381-410): every
    cell is timed on the device (mean_ms > 0) and its launch and unknown-touch
    counts are the real reference's dry-run counts (golden `bench --reps 0`)."""
    gold = next(c for c in json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cli.json")))
                if c["argv"][0] == "bench")
    rc, out = run(["bench", "--kappa", "1,2,inf", "--levels", "4-6", "--reps", "2"])
    assert rc == 0
    got = [line.split(",") for line in out.strip().splitlines()]
    ref = [line.split(",") for line in gold["stdout"].strip().splitlines()]
    assert got[0] == ref[0] and len(got) == len(ref)
    for g, r in zip(got[1:], ref[1:]):
        assert g[0:2] == r[0:2] and g[3:] == r[3:], (g, r)
        assert float(g[2]) > 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("kappa", [1, 3, math.inf])
def test_bench_cycle_api_timed(kappa):
    from paper_2010_00626_b200 import CycleConfig, ProblemSpec
    from paper_2010_00626_b200.cycle import bench_cycle
    cfg = CycleConfig(n=9, kappa=kappa)
    dry = bench_cycle(ProblemSpec(1e-4, 45.0), cfg, 0)
    res = bench_cycle(ProblemSpec(1e-4, 45.0), cfg, 3)
    assert dry.mean_ms is None and res.mean_ms is not None and 0.0 < res.mean_ms < 1e3
    assert (res.launches, res.op_units) == (dry.launches, dry.op_units)

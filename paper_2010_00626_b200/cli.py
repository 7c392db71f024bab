"""Command-line mirror of the reference driver (reference
cli.py:1-390), running the solves and benchmarks on the B200 engine.

    python -m paper_2010_00626_b200 <subcommand> [flags]

Subcommands, flags, output formats and exit codes follow the reference so
scripts can switch by changing the program name:

    solve          stand-alone or CG-preconditioned solve; one JSON record
                   (or a two-line CSV) with the config echo and the result
                   (cli.py:168-213)
    calls          per-level and total routine-call counts (cli.py:216-220)
    predict        model launches / op units / predicted ms (cli.py:223-234)
    fit            least-squares (alpha, beta) from a kappa,levels,ms CSV
                   (cli.py:237-266)
    turning-point  overhead/computation balance point (cli.py:269-283)
    bench          single-cycle timing sweep, CSV (cli.py:286-322); here
                   timed with CUDA events on the engine stream

Exit codes: 0 ok, 2 usage, 3 divergence or CG breakdown, 4 iteration budget
exhausted, 5 rank-deficient fit (cli.py:10-11).

Engine-side difference: `solve` accepts an optional `--stop residual` (the
relative-residual rule of the B200 benchmark; the default `error` is the
reference's rule).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import math
import sys
from datetime import datetime, timezone

import numpy as np

from . import __version__
from .costmodel import (
    CostModelParams,
    RankDeficientError,
    fit_params,
    level_calls,
    n_gpu_calls,
    ops_per_unknown,
    predict_runtime,
    total_calls,
    turning_point,
)
from .cycle import CONVERGED, DIVERGED, CycleConfig, bench_cycle, build_state, solve_standalone
from .krylov import PcgConfig, pcg_solve
from .mesh import Coarsening
from .smoother import SmootherKind, SmootherSpec
from .stencil import ProblemSpec

__all__ = ["main", "build_parser"]

EXIT_OK, EXIT_USAGE, EXIT_DIVERGED, EXIT_NOT_CONVERGED, EXIT_FIT_FAILED = 0, 2, 3, 4, 5

SMOOTHERS = {"jacobi": SmootherKind.DAMPED_JACOBI, "zebra-xy": SmootherKind.ZEBRA_ALTERNATING,
             "zebra-x": SmootherKind.ZEBRA_X}
COARSENINGS = {"full": Coarsening.FULL_STANDARD, "semi-y": Coarsening.SEMI_Y}
RESULT_FIELDS = ("iterations", "initial_norm", "final_norm", "asymptotic_factor", "launches", "op_units",
                 "wall_ms")


# ---------------------------------------------------------------------------
# argument types
# ---------------------------------------------------------------------------

def kappa_arg(text: str):
    """Positive integer or 'inf' (cli.py:67-76)."""
    if text.strip().lower() == "inf":
        return math.inf
    try:
        k = int(text)
    except ValueError:
        raise argparse.ArgumentTypeError(f"kappa must be a positive integer or 'inf', got {text!r}") from None
    if k < 1:
        raise argparse.ArgumentTypeError(f"kappa must be >= 1, got {k}")
    return k


def kappa_list_arg(text: str):
    return [kappa_arg(t) for t in text.split(",") if t.strip()]


def level_list_arg(text: str):
    """'4,5' or '4-8' or a mix (cli.py:83-97)."""
    levels = []
    for tok in (t.strip() for t in text.split(",")):
        if not tok:
            continue
        if "-" in tok:
            lo, hi = tok.split("-", 1)
            levels += list(range(int(lo), int(hi) + 1))
        else:
            levels.append(int(tok))
    if not levels or min(levels) < 1:
        raise argparse.ArgumentTypeError(f"invalid level list: {text!r}")
    return levels


def num(v) -> str:
    """Round-trip text for numeric CSV/console fields (cli.py:100-104)."""
    return repr(v) if isinstance(v, float) else str(v)


def kappa_text(k) -> str:
    return "inf" if k == math.inf else str(k)


# ---------------------------------------------------------------------------
# problem / config
# ---------------------------------------------------------------------------

def _default_coarsening(smoother: str, coarsening: str | None) -> Coarsening:
    if coarsening:
        if smoother == "zebra-x" and coarsening != "semi-y":
            print("warning: zebra-x is normally paired with --coarsening semi-y", file=sys.stderr)
        return COARSENINGS[coarsening]
    return Coarsening.SEMI_Y if smoother == "zebra-x" else Coarsening.FULL_STANDARD


def _config(args, parser, n: int, kappa) -> CycleConfig:
    try:
        return CycleConfig(n=n, kappa=kappa, nu1=args.nu1, nu2=args.nu2,
                           smoother=SmootherSpec(SMOOTHERS[args.smoother], omega=args.omega),
                           coarsening=_default_coarsening(args.smoother, args.coarsening),
                           coarse_op=args.coarse_op)
    except ValueError as exc:
        parser.error(str(exc))


def _problem(args, parser) -> ProblemSpec:
    try:
        return ProblemSpec(epsilon=args.eps, phi=args.phi, seed=args.seed)
    except ValueError as exc:
        parser.error(str(exc))


def _device_guard(parser, config: CycleConfig):
    # every smoother / coarsening of the reference runs on the engine (zebra and
    # semi-y on its per-op kernels); kept as the hook for future restrictions
    return None


# ---------------------------------------------------------------------------
# subcommands
# ---------------------------------------------------------------------------

def cmd_solve(args, parser) -> int:
    problem = _problem(args, parser)
    config = _config(args, parser, args.levels, args.kappa)
    _device_guard(parser, config)
    if args.reduction <= 1.0:
        parser.error(f"--reduction must exceed 1, got {args.reduction}")
    try:
        if args.solver == "standalone":
            rep = solve_standalone(problem, config, args.reduction, args.max_cycles, stop=args.stop)
        else:
            state = build_state(problem, config)
            x0 = np.random.default_rng(problem.seed).random(state.v[0].shape)
            pcfg = PcgConfig(cycle=config, target_reduction=args.reduction, max_iterations=args.max_cycles,
                             stop=args.stop)
            rep = pcg_solve(state, np.zeros_like(x0), pcfg, x0=x0)
            state.close()
    except ValueError as exc:
        parser.error(str(exc))
    echo = {
        "levels": config.n, "kappa": "inf" if config.kappa == math.inf else config.kappa,
        "eps": args.eps, "phi": args.phi, "smoother": args.smoother, "coarsening": config.coarsening.value,
        "omega": args.omega, "nu1": config.nu1, "nu2": config.nu2, "seed": args.seed,
        "coarse_op": args.coarse_op, "solver": args.solver, "reduction": args.reduction,
        "max_cycles": args.max_cycles,
    }
    result = {
        "status": rep.status, "iterations": rep.iterations, "initial_norm": rep.initial_error_norm,
        "final_norm": rep.final_error_norm, "asymptotic_factor": rep.asymptotic_factor,
        "launches": rep.stats.kernel_launches, "op_units": rep.stats.unknown_touches, "wall_ms": rep.wall_time_ms,
    }
    if args.out == "json":
        print(json.dumps({"config": echo, "result": result, "version": __version__,
                          "timestamp": datetime.now(timezone.utc).isoformat()}))
    else:
        w = csv.writer(sys.stdout, lineterminator="\n")
        w.writerow(list(echo) + ["status"] + list(RESULT_FIELDS))
        w.writerow([num(v) for v in echo.values()] + [result["status"]] + [num(result[k]) for k in RESULT_FIELDS])
    if rep.status == CONVERGED:
        return EXIT_OK
    return EXIT_DIVERGED if rep.status in (DIVERGED, "breakdown") else EXIT_NOT_CONVERGED


def cmd_calls(args, parser) -> int:
    print("level_calls:", " ".join(str(level_calls(args.kappa, l)) for l in range(1, args.levels + 1)))
    print("total_calls:", total_calls(args.kappa, args.levels))
    return EXIT_OK


def cmd_predict(args, parser) -> int:
    try:
        params = CostModelParams(alpha=args.alpha, beta=args.beta, nu=args.nu)
    except ValueError as exc:
        parser.error(str(exc))
    print("launches:", n_gpu_calls(args.kappa, args.levels, args.nu))
    print("op_units:", num((2 ** args.levels - 1) ** 2 * ops_per_unknown(args.kappa)))
    print("predicted_ms:", num(predict_runtime(params, args.kappa, args.levels)))
    return EXIT_OK


def cmd_fit(args, parser) -> int:
    try:
        if args.input == "-":
            text = sys.stdin.read()
        else:
            with open(args.input, encoding="utf-8") as fh:
                text = fh.read()
    except OSError as exc:
        parser.error(str(exc))
    rd = csv.DictReader(io.StringIO(text))
    if rd.fieldnames is None or not {"kappa", "levels", "ms"} <= set(rd.fieldnames):
        parser.error("fit input needs header kappa,levels,ms")
    obs = []
    try:
        for row in rd:
            k = math.inf if row["kappa"].strip().lower() == "inf" else int(row["kappa"])
            obs.append((k, int(row["levels"]), float(row["ms"])))
    except (KeyError, ValueError) as exc:
        parser.error(f"bad fit input row: {exc}")
    try:
        alpha, beta = fit_params(obs, nu=args.nu)
    except RankDeficientError as exc:
        print(f"fit failed: {exc}", file=sys.stderr)
        return EXIT_FIT_FAILED
    print("alpha:", num(alpha))
    print("beta:", num(beta))
    return EXIT_OK


def cmd_turning_point(args, parser) -> int:
    try:
        tp = turning_point(CostModelParams(alpha=args.alpha, beta=args.beta, nu=args.nu), args.kappa)
    except ValueError as exc:
        parser.error(str(exc))
    if tp.degenerate:
        print("degenerate: zero launch overhead, no turning point")
        return EXIT_OK
    if not tp.converged:
        print("warning: fixed-point iteration did not settle; reporting last iterate", file=sys.stderr)
    print("n_tp:", num(tp.n_tp))
    print("N_tp:", num(tp.N_tp))
    return EXIT_OK


def cmd_bench(args, parser) -> int:
    problem = _problem(args, parser)
    if args.smoother == "zebra-x" and args.coarsening == "full":
        print("warning: zebra-x is normally paired with --coarsening semi-y", file=sys.stderr)
    w = csv.writer(sys.stdout, lineterminator="\n")
    w.writerow(["kappa", "levels", "mean_ms", "launches", "op_units"] + (["cycles_to_target"] if args.converge else []))
    for k in args.kappa:
        for n in args.levels:
            config = _config(args, parser, n, k)
            if args.reps > 0 or args.converge:
                _device_guard(parser, config)
            cell = bench_cycle(problem, config, args.reps)
            row = [kappa_text(k), str(n), "" if cell.mean_ms is None else num(cell.mean_ms), str(cell.launches),
                   num(cell.op_units)]
            if args.converge:
                row.append(str(solve_standalone(problem, config, args.reduction, args.max_cycles).iterations))
            w.writerow(row)
            sys.stdout.flush()
    return EXIT_OK


# ---------------------------------------------------------------------------
# parser
# ---------------------------------------------------------------------------

def _problem_flags(p: argparse.ArgumentParser, levels_required: bool = True):
    p.add_argument("--eps", type=float, default=1.0, help="anisotropy in (0, 1]")
    p.add_argument("--phi", type=float, default=0.0, help="rotation angle, degrees")
    p.add_argument("--smoother", choices=sorted(SMOOTHERS), default="jacobi")
    p.add_argument("--coarsening", choices=sorted(COARSENINGS), default=None,
                   help="default: full (semi-y when --smoother zebra-x)")
    p.add_argument("--omega", type=float, default=0.8, help="Jacobi damping factor")
    p.add_argument("--nu1", type=int, default=2, help="pre-relaxation count")
    p.add_argument("--nu2", type=int, default=2, help="post-relaxation count")
    p.add_argument("--seed", type=int, default=0, help="initial-guess PRNG seed")
    p.add_argument("--coarse-op", choices=["galerkin", "rediscretize"], default="galerkin")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2010_00626_b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="command", required=True)

    p = sub.add_parser("solve", help="run a multigrid solve on the B200")
    p.add_argument("--levels", type=int, required=True, help="level count n")
    p.add_argument("--kappa", type=kappa_arg, default=1, help="cycle counter (int or 'inf')")
    _problem_flags(p)
    p.add_argument("--reduction", type=float, default=1e8, help="target reduction")
    p.add_argument("--max-cycles", type=int, default=10000)
    p.add_argument("--solver", choices=["standalone", "pcg"], default="standalone")
    p.add_argument("--stop", choices=["error", "residual"], default="error",
                   help="stopping measure (engine extension; the reference uses error)")
    p.add_argument("--out", choices=["json", "csv"], default="json")
    p.set_defaults(func=cmd_solve)

    p = sub.add_parser("calls", help="routine-call counts per level")
    p.add_argument("--kappa", type=kappa_arg, required=True)
    p.add_argument("--levels", type=int, required=True)
    p.set_defaults(func=cmd_calls)

    p = sub.add_parser("predict", help="model prediction for one cell")
    p.add_argument("--alpha", type=float, required=True, help="ms per launch")
    p.add_argument("--beta", type=float, required=True, help="ms per op unit")
    p.add_argument("--kappa", type=kappa_arg, required=True)
    p.add_argument("--levels", type=int, required=True)
    p.add_argument("--nu", type=int, default=4, help="relaxations per routine call")
    p.set_defaults(func=cmd_predict)

    p = sub.add_parser("fit", help="fit alpha, beta from kappa,levels,ms CSV")
    p.add_argument("--input", default="-", help="CSV path or '-' for stdin")
    p.add_argument("--nu", type=int, default=4)
    p.set_defaults(func=cmd_fit)

    p = sub.add_parser("turning-point", help="overhead/computation balance point")
    p.add_argument("--alpha", type=float, required=True)
    p.add_argument("--beta", type=float, required=True)
    p.add_argument("--kappa", type=kappa_arg, required=True)
    p.add_argument("--nu", type=int, default=4)
    p.set_defaults(func=cmd_turning_point)

    p = sub.add_parser("bench", help="single-cycle timing sweep (CSV to stdout)")
    p.add_argument("--kappa", type=kappa_list_arg, required=True, help="comma list, e.g. 1,2,inf")
    p.add_argument("--levels", type=level_list_arg, required=True, help="comma list or ranges, e.g. 4,5 or 4-8")
    p.add_argument("--reps", type=int, default=200, help="repetitions per cell (0 = dry)")
    _problem_flags(p)
    p.add_argument("--converge", action="store_true", help="also report cycles to reach --reduction")
    p.add_argument("--reduction", type=float, default=1e8)
    p.add_argument("--max-cycles", type=int, default=10000)
    p.set_defaults(func=cmd_bench)
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    args = ap.parse_args(argv)
    return args.func(args, ap)

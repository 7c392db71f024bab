"""pytest plugin: run the REFERENCE's own test modules against CudaGridState.

Loaded with `-p refshim` by tests/test_gpu_reference_dropin.py, which runs
the unmodified reference tests (baseline/_ref/kcycle_tests/test_cycle.py,
test_krylov.py, copied there by tools/install_reference.sh) in a subprocess.
Before any test module is imported it replaces `kcycle.cycle.build_state`
(cycle.py:266-270) -- the one factory through which the reference's tests
and its `solve_standalone` (cycle.py:303-366) obtain a state -- by a
function that builds this repo's device-resident `CudaGridState` from the
reference's own HierarchySpec / Stencil9 hierarchy / SmootherSpec.  Every
`kappa_cycle`, `run_cycle`, `gamma_cycle`, `f_cycle`, `solve_standalone` and
`pcg_solve` the reference's tests call then drives the B200 engine through
the state protocol ("the reference's own kappa_cycle /
run_cycle must be able to drive CudaGridState unchanged").

At session end the plugin writes how many CudaGridStates were built to
$KC_REFSHIM_REPORT, so the caller can check the device path really ran.
"""

from __future__ import annotations

import json
import os
import sys

_COUNT = {"cuda_states": 0}


def pytest_configure(config):
    ref = os.environ["KC_REF_PATH"]  # baseline/_ref
    repo = os.environ["KC_REPO_ROOT"]
    for p in (ref, repo):
        if p not in sys.path:
            sys.path.insert(0, p)
    import kcycle.cycle as rc
    import kcycle.mesh as rm
    import kcycle.stencil as rs

    from paper_2010_00626_b200.cycle import CudaGridState

    def cuda_build_state(problem, cfg):
        spec = rm.build_hierarchy(cfg.n, cfg.coarsening)
        ops = rs.operator_hierarchy(problem, spec, cfg.coarse_op)
        _COUNT["cuda_states"] += 1
        return CudaGridState(spec, ops, cfg.smoother, cfg.nu1, cfg.nu2)

    rc.build_state = cuda_build_state
    import kcycle
    kcycle.build_state = cuda_build_state


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("KC_REFSHIM_REPORT")
    if path:
        with open(path, "w") as fh:
            json.dump(_COUNT, fh)

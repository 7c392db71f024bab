"""ctypes binding of the C-ABI in include/kcb200.h (libkcb200.so, built in-tree).

This is the reference-side binding shape a maintainer of `kcycle` would add
(INTEGRATION.md): the reference is pure Python, so ctypes is its FFI.  There
is no CPU fallback anywhere in the package: if the library is missing the
import fails loudly, and if no sm_100 device is present `kc_create` fails with
KC_ECUDA, which is raised as `CudaUnavailableError`.

Error codes map onto the reference's exception types:
KC_EINVAL -> ValueError, KC_ESINGULAR -> numpy.linalg.LinAlgError,
KC_ECUDA -> CudaError (RuntimeError), KC_ENOMEM -> MemoryError.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KCB200_LIB") or os.path.join(_HERE, "libkcb200.so")  # override: experiments only
# the FMA-contracted build of the same sources (kc_common.cuh KC_FAST)
LIB_FAST_PATH = os.environ.get("KCB200_LIB_FAST") or os.path.join(_HERE, "libkcb200_fast.so")
ARITH_MODES = ("exact", "fast")

KC_OK, KC_EINVAL, KC_ESINGULAR, KC_ECUDA, KC_ENOMEM = 0, 1, 2, 3, 4
KC_COARSEN_FULL, KC_COARSEN_SEMI_Y = 0, 1
KC_SMOOTH_JACOBI, KC_SMOOTH_ZEBRA_X, KC_SMOOTH_ZEBRA_Y, KC_SMOOTH_ZEBRA_XY = 0, 1, 2, 3
COARSENING_KIND = {"full": KC_COARSEN_FULL, "semi-y": KC_COARSEN_SEMI_Y}  # Coarsening values (mesh.py:38-39)
SMOOTHER_KIND = {"jacobi": KC_SMOOTH_JACOBI, "zebra-x": KC_SMOOTH_ZEBRA_X, "zebra-y": KC_SMOOTH_ZEBRA_Y,
                 "zebra-xy": KC_SMOOTH_ZEBRA_XY}  # SmootherKind values (smoother.py:37-41)
KC_WHICH_V, KC_WHICH_F = 0, 1
KC_STOP_ERROR, KC_STOP_RESIDUAL = 0, 1
STATUS_NAMES = {0: "converged", 1: "diverged", 2: "max_cycles", 3: "breakdown"}


class CudaError(RuntimeError):
    """CUDA runtime failure inside the engine."""


class CudaUnavailableError(CudaError):
    """No usable sm_100 device: the engine has no CPU fallback."""


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_h = C.c_void_p
PRECOND_FN = C.CFUNCTYPE(None, _dp, _dp, C.c_longlong, C.c_longlong, C.c_void_p)

_SIGS = {
    "kc_abi_version": (C.c_int, []),
    "kc_last_error": (C.c_char_p, [_h]),
    "kc_galerkin_coarsen": (C.c_int, [_dp, C.c_int, _dp]),
    "kc_create": (C.c_int, [C.c_int, C.c_int, _dp, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                            C.POINTER(C.c_void_p)]),
    "kc_destroy": (C.c_int, [_h]),
    "kc_sync": (C.c_int, [_h]),
    "kc_level_dims": (C.c_int, [_h, C.c_int, _ip, _ip]),
    "kc_set": (C.c_int, [_h, C.c_int, C.c_int, _dp, C.c_longlong, C.c_longlong]),
    "kc_get": (C.c_int, [_h, C.c_int, C.c_int, _dp, C.c_longlong, C.c_longlong]),
    "kc_relax": (C.c_int, [_h, C.c_int, C.c_int]),
    "kc_restrict_residual": (C.c_int, [_h, C.c_int]),
    "kc_zero_guess": (C.c_int, [_h, C.c_int]),
    "kc_prolong_add": (C.c_int, [_h, C.c_int]),
    "kc_solve_coarsest": (C.c_int, [_h]),
    "kc_apply": (C.c_int, [_h, C.c_int, C.c_int, _dp, C.c_longlong, C.c_longlong]),
    "kc_norm2": (C.c_int, [_h, C.c_int, C.c_int, _dp]),
    "kc_residual_norm": (C.c_int, [_h, C.c_int, _dp]),
    "kc_run_cycles": (C.c_int, [_h, C.c_int, C.c_int]),
    "kc_time_cycles": (C.c_int, [_h, C.c_int, C.c_int, _dp]),
    "kc_solve": (C.c_int, [_h, C.c_int, C.c_int, C.c_double, C.c_int, _dp, _dp, _ip, _ip, _dp]),
    "kc_pcg": (C.c_int, [_h, C.c_int, _dp, _dp, C.c_int, C.c_double, C.c_int, PRECOND_FN, C.c_void_p,
                         _dp, _ip, _ip, _ip, _dp, _dp]),
    "kc_cycle_launches": (C.c_int, [_h, C.c_int, _ip]),
    "kc_profile_cycle": (C.c_int, [_h, C.c_int, C.c_int, _ip, _ip, _ip, _dp, _ip]),
    "kc_stream": (C.c_int, [_h, C.POINTER(C.c_void_p)]),
    "kc_fill_zero": (C.c_int, [_h, C.c_int, C.c_int]),
    "kc_snapshot": (C.c_int, [_h]),
    "kc_set_option": (C.c_int, [_h, C.c_char_p, C.c_int]),
    "kc_strip_jacobi": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, _dp, C.c_double,
                                  C.c_int, C.c_void_p]),
    "kc_strip_resid_restrict": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                          _dp, C.c_int, C.c_void_p]),
    "kc_strip_prolong_add": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_void_p]),
    "kc_strip_norms": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, _dp, C.c_void_p, C.c_void_p]),
    "kc_strip_pre": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p] + [C.c_int] * 8
                     + [_dp, C.c_double, C.c_int, C.c_int, C.c_void_p]),
    "kc_strip_post": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p] + [C.c_int] * 9
                      + [_dp, C.c_double, C.c_int, C.c_int, C.c_void_p]),
    "kc_strip_pre_window": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p] + [C.c_int] * 10
                            + [_dp, C.c_double, C.c_int, C.c_int, C.c_void_p]),
    "kc_strip_post_window": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p] + [C.c_int] * 11
                             + [_dp, C.c_double, C.c_int, C.c_int, C.c_void_p]),
    "kc_set_device": (C.c_int, [_h, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_longlong, C.c_longlong]),
    "kc_get_device": (C.c_int, [_h, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_longlong, C.c_longlong]),
    "kc_set_device_async": (C.c_int, [_h, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_longlong, C.c_longlong]),
    "kc_get_device_async": (C.c_int, [_h, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_longlong, C.c_longlong]),
    "kc_set_stream": (C.c_int, [_h, C.c_void_p]),
    "kc_cycle_enqueue": (C.c_int, [_h, C.c_int]),
    "kc_restore": (C.c_int, [_h]),
    # device-side loops of the distributed solvers (kc_dist.cuh)
    "kc_strip_apply_dot": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, _dp, C.c_void_p, C.c_void_p,
                                     C.c_int, C.c_void_p]),
    "kc_strip_dot": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                               C.c_void_p]),
    "kc_strip_pcg_update_xr": (C.c_int, [C.c_void_p] * 4 + [C.c_int] * 4 + [C.c_void_p, C.c_void_p, C.c_void_p]),
    "kc_strip_pcg_update_p": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "kc_strip_residual": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, _dp, C.c_void_p]),
    "kc_strip_copy_if": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "kc_dist_step": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
}

# scalar slots / step kinds of the distributed device loops (include/kcb200.h KC_DS_*)
DS = dict(RZ=0, RZN=1, PAP=2, MEAS=3, ALPHA=4, BETA=5, TARGET=6, IT=7, MAXIT=8, STATUS=9, DONE=10, JUST_DONE=11,
          E2=12, R2=13, STOP_RESIDUAL=14, STREAK=15, PREV=16, REDUCTION=17)
DS_SLOTS, DS_PART = 32, 592
DS_PCG_RZ0, DS_PCG_PAP, DS_PCG_MEAS, DS_PCG_RZ, DS_SOLVE = 0, 1, 2, 3, 4

_SIGS["kc_arith_mode"] = (C.c_int, [])


def _load(path: str, arith: int):
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA engine first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    handle = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if handle.kc_abi_version() != 1:
        raise ImportError(f"{path} ABI version {handle.kc_abi_version()} != 1; rebuild")
    if handle.kc_arith_mode() != arith:
        raise ImportError(f"{path} reports arithmetic mode {handle.kc_arith_mode()}, expected {arith}")
    return handle


lib = _load(LIB_PATH, 0)  # the exact build: iterates bit-identical to the reference
_libs = {"exact": lib}


def default_arith() -> str:
    """Arithmetic of new handles unless a caller says otherwise: KCB200_ARITH
    ("exact" or "fast"), else "exact" (the bit-exact drop-in)."""
    mode = os.environ.get("KCB200_ARITH", "exact")
    if mode not in ARITH_MODES:
        raise ValueError(f"KCB200_ARITH must be one of {ARITH_MODES}, got {mode!r}")
    return mode


def lib_for(arith: str | None = None):
    """The engine library of an arithmetic mode ("exact" | "fast"; None: default_arith())."""
    arith = default_arith() if arith is None else arith
    if arith not in ARITH_MODES:
        raise ValueError(f"arith must be one of {ARITH_MODES}, got {arith!r}")
    if arith not in _libs:
        _libs[arith] = _load(LIB_FAST_PATH, 1)
    return _libs[arith]


def last_error(handle, which=None) -> str:
    msg = (which or lib).kc_last_error(handle)
    return msg.decode() if msg else ""


def check(rc: int, handle=None, which=None) -> None:
    """Raise the reference's exception type for a non-OK status (`which`:
    the library that owns `handle`, default the exact build)."""
    if rc == KC_OK:
        return
    msg = last_error(handle, which)
    if rc == KC_EINVAL:
        raise ValueError(msg)
    if rc == KC_ESINGULAR:
        raise np.linalg.LinAlgError(msg)
    if rc == KC_ENOMEM:
        raise MemoryError(msg)
    if "no CUDA device" in msg or "targets sm_100a" in msg:
        raise CudaUnavailableError(msg)
    raise CudaError(msg or f"kcb200 error {rc}")


def dptr(a: np.ndarray):
    """Pointer to a C-contiguous float64 array (caller keeps it alive)."""
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def as_f64c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def galerkin_coarsen(w: np.ndarray, coarsening: int) -> np.ndarray:
    wf = as_f64c(w).reshape(9).copy()
    out = np.empty(9)
    check(lib.kc_galerkin_coarsen(dptr(wf), coarsening, dptr(out)))
    return out.reshape(3, 3)

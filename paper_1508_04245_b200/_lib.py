"""ctypes binding of ``libhdgconv.so`` (the C ABI in include/hdgconv.h).

The shared library is built in-tree by ``__graft_entry__.build()`` /
``python -m paper_1508_04245_b200.build``.  There is no fallback: if the
library is missing or fails to load, every operator raises.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
_DEFAULT_PATH = os.path.join(HERE, "libhdgconv.so")
LIB_PATH = os.environ.get("HDGC_LIB") or _DEFAULT_PATH

# exported symbols, in include/hdgconv.h order
SYMBOLS = (
    "hdgc_create", "hdgc_create_k", "hdgc_destroy", "hdgc_get_info", "hdgc_apply_v", "hdgc_apply_w",
    "hdgc_substeps", "hdgc_transfer", "hdgc_mass_inverse", "hdgc_max_speed",
    "hdgc_apply_v_host", "hdgc_substeps_host", "hdgc_propagate", "hdgc_richardson",
    "hdgc_set_dofmap", "hdgc_gather", "hdgc_scatter", "hdgc_apply_u", "hdgc_set_curved",
    "hdgc_check_finite", "hdgc_last_error", "hdgc_version",
)

HDGC_ENOCONV = -5
HDGC_EBLOWUP = -6


class NormBlowupError(FloatingPointError):
    """An explicit update produced non-finite values (SPEC.md:433 guard)."""


_dp = C.POINTER(C.c_double)


class MeshDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("n_vertices", C.c_int32), ("n_elements", C.c_int32),
        ("n_facets", C.c_int32), ("vertices", C.c_void_p), ("elements", C.c_void_p),
        ("facet_elems", C.c_void_p), ("facet_local", C.c_void_p), ("facet_perm", C.c_void_p),
    ]


class TablesDesc(C.Structure):
    _fields_ = [
        ("k", C.c_int32), ("nqv", C.c_int32), ("nf", C.c_int32),
        ("coef", C.c_void_p), ("div_modal", C.c_void_p), ("vol_w", C.c_void_p), ("vol_D", C.c_void_p),
        ("vol_G", C.c_void_p), ("fac_w", C.c_void_p), ("fac_L", C.c_void_p),
        ("fac_D", C.c_void_p), ("fac_len", C.c_void_p),
        ("col_n", C.c_int32), ("col_A", C.c_void_p), ("col_Ad", C.c_void_p), ("col_B", C.c_void_p),
        ("col_Bd", C.c_void_p), ("col_xi", C.c_void_p), ("col_wa", C.c_void_p), ("col_wy", C.c_void_p),
        ("col_inv1my", C.c_void_p), ("col_C", C.c_void_p), ("col_Cd", C.c_void_p), ("col_pf", C.c_void_p),
    ]


class Info(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("k", C.c_int32), ("nb", C.c_int32), ("nbs", C.c_int32),
        ("nqv", C.c_int32), ("nf", C.c_int32), ("n_elements", C.c_int32),
        ("n_facets", C.c_int32), ("n_boundary_facets", C.c_int32),
        ("volume_variant", C.c_int32), ("device_bytes", C.c_int64),
    ]


_LIB = None


def load(path: str = LIB_PATH):
    """Load the library once; raise RuntimeError (no fallback) on failure."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = C.CDLL(path)
    vp, i32, d = C.c_void_p, C.c_int32, C.c_double
    sig = {
        "hdgc_create": ([C.POINTER(MeshDesc), C.POINTER(TablesDesc), C.POINTER(vp)], C.c_int),
        "hdgc_create_k": ([C.POINTER(MeshDesc), i32, C.POINTER(vp)], C.c_int),
        "hdgc_destroy": ([vp], C.c_int),
        "hdgc_get_info": ([vp, C.POINTER(Info)], C.c_int),
        "hdgc_apply_v": ([vp, vp, vp, vp, vp, vp], C.c_int),
        "hdgc_apply_w": ([vp, vp, vp, vp, vp], C.c_int),
        "hdgc_substeps": ([vp, vp, vp, vp, d, i32, vp], C.c_int),
        "hdgc_transfer": ([vp, i32, vp, vp, vp], C.c_int),
        "hdgc_mass_inverse": ([vp, vp, vp], C.c_int),
        "hdgc_max_speed": ([vp, vp, vp, vp], C.c_int),
        "hdgc_apply_v_host": ([vp, vp, vp, vp, vp, vp], C.c_int),
        "hdgc_substeps_host": ([vp, vp, vp, vp, d, i32, vp], C.c_int),
        "hdgc_propagate": ([vp, vp, vp, d, d, d, d, i32, i32, vp, vp, vp], C.c_int),
        "hdgc_richardson": ([vp, vp, vp, vp, d, d, d, i32, vp, C.POINTER(i32), C.POINTER(d), C.POINTER(d), vp],
                            C.c_int),
        "hdgc_set_dofmap": ([vp, C.c_int64, vp, vp], C.c_int),
        "hdgc_gather": ([vp, vp, vp, vp], C.c_int),
        "hdgc_scatter": ([vp, vp, vp, vp], C.c_int),
        "hdgc_apply_u": ([vp, vp, vp, vp, vp], C.c_int),
        "hdgc_set_curved": ([vp, i32, vp, vp, vp, vp], C.c_int),
        "hdgc_check_finite": ([vp, vp], C.c_int),
        "hdgc_last_error": ([], C.c_char_p),
        "hdgc_version": ([], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        if path != _DEFAULT_PATH and not hasattr(lib, name):
            continue      # HDGC_LIB override (development A/B builds): older ABI subsets allowed
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _LIB = lib
    return lib


def check(rc: int, what: str):
    if rc != 0:
        msg = load().hdgc_last_error().decode(errors="replace")
        if rc == HDGC_EBLOWUP:
            raise NormBlowupError(f"{what}: {msg}")
        raise RuntimeError(f"{what} failed (status {rc}): {msg}")

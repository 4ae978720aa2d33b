"""ctypes loader for libstokescol.so (the C ABI in include/stokescol.h).

Argument marshalling only.  The library is built in-tree by
``paper_1909_06623_b200/build.py``; if it is missing this module raises --
there is no CPU fallback anywhere in the product.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libstokescol.so")

SC_OK, SC_NOT_CONVERGED = 0, 1
SC_EINVAL, SC_EDEGENERATE, SC_ENONFINITE, SC_ENOMEM, SC_ECUDA, SC_ENCCL = -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "SC_OK", 1: "SC_NOT_CONVERGED", -1: "SC_EINVAL", -2: "SC_EDEGENERATE",
                -3: "SC_ENONFINITE", -4: "SC_ENOMEM", -5: "SC_ECUDA", -6: "SC_ENCCL"}
K_FAMILIES = ["contacts", "assemble", "gather", "rpy", "combine", "dt", "finalize", "misc"]

# every symbol include/stokescol.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "sc_version", "sc_create", "sc_nccl_unique_id", "sc_create_dist", "sc_destroy", "sc_last_error",
    "sc_stream", "sc_build_contacts_spheres", "sc_build_contacts_rods", "sc_get_contacts",
    "sc_assemble_D", "sc_apply_D", "sc_apply_DT", "sc_mobility_apply", "sc_lcp_q", "sc_bbpgd_solve",
    "sc_collision_step", "sc_set_timing", "sc_get_timing", "sc_reset_timing", "sc_launch_count",
    "sc_plan_partition", "sc_set_emulated_world", "sc_set_rpy_kernel", "sc_time_step", "sc_apgd_solve",
    "sc_set_walls", "sc_set_mobility_model", "sc_minmap_residual", "sc_set_residual_trace",
    "sc_get_residual_trace", "sc_comm_info", "sc_sym_pair_table", "sc_set_wall_velocities", "sc_get_walls",
    "sc_set_fmm_params", "sc_get_fmm_info", "sc_build_flags", "sc_set_fmm_compression",
    "sc_get_fmm_compression_info", "sc_set_fmm_tolerance",
]


class BbpgdOpts(C.Structure):
    _fields_ = [("mu", C.c_double), ("tol", C.c_double), ("max_iter", C.c_int32), ("bb_mode", C.c_int32),
                ("fixed_iters", C.c_int32), ("warm_start", C.c_int32)]


class BbpgdStats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("mvops", C.c_int32), ("converged", C.c_int32),
                ("bb_breakdowns", C.c_int32), ("active", C.c_int32), ("reserved", C.c_int32),
                ("residual", C.c_double), ("alpha", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


class Problem(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("n", C.c_int64), ("pos", C.c_void_p),
                ("radius", C.c_void_p), ("dir", C.c_void_p), ("length", C.c_void_p), ("b", C.c_double),
                ("gap_abs", C.c_double), ("gap_rel", C.c_double), ("mu", C.c_double), ("dt", C.c_double),
                ("F_ext", C.c_void_p)]


_lib = None


def load(build_if_missing: bool = True):
    """Load libstokescol.so (building it with nvcc first if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SC_LIB") or LIB_PATH  # SC_LIB: tuning A/B of another build of this library
    if not os.path.exists(path):
        if not build_if_missing:
            raise RuntimeError(f"libstokescol.so not built at {LIB_PATH}")
        from . import build as _build
        _build.build()
    lib = C.CDLL(path)
    vp, i64, i32, d, ci = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_int
    pp = C.POINTER(C.c_void_p)
    sig = {
        "sc_version": (ci, []),
        "sc_build_flags": (ci, []),
        "sc_create": (ci, [pp, ci, vp]),
        "sc_nccl_unique_id": (ci, [vp]),
        "sc_create_dist": (ci, [pp, ci, vp, vp, ci, ci]),
        "sc_destroy": (None, [vp]),
        "sc_last_error": (C.c_char_p, [vp]),
        "sc_stream": (vp, [vp]),
        "sc_build_contacts_spheres": (ci, [vp, i64, vp, vp, d, d, C.POINTER(i64)]),
        "sc_build_contacts_rods": (ci, [vp, i64, vp, vp, vp, d, d, C.POINTER(i64)]),
        "sc_get_contacts": (ci, [vp, vp, vp, vp, vp, vp]),
        "sc_assemble_D": (ci, [vp]),
        "sc_apply_D": (ci, [vp, vp, vp]),
        "sc_apply_DT": (ci, [vp, vp, vp]),
        "sc_mobility_apply": (ci, [vp, d, vp, vp]),
        "sc_lcp_q": (ci, [vp, d, vp, vp]),
        "sc_bbpgd_solve": (ci, [vp, C.POINTER(BbpgdOpts), vp, vp, vp, vp, C.POINTER(BbpgdStats)]),
        "sc_collision_step": (ci, [vp, C.POINTER(Problem), C.POINTER(BbpgdOpts), vp, vp, C.POINTER(i64),
                                   C.POINTER(BbpgdStats)]),
        "sc_set_timing": (ci, [vp, ci]),
        "sc_get_timing": (ci, [vp, ci, C.POINTER(d), C.POINTER(i64)]),
        "sc_reset_timing": (ci, [vp]),
        "sc_launch_count": (i64, [vp]),
        "sc_plan_partition": (ci, [i64, ci, ci, C.POINTER(i64)]),
        "sc_set_emulated_world": (ci, [vp, ci]),
        "sc_set_rpy_kernel": (ci, [vp, ci]),
        "sc_set_walls": (ci, [vp, ci, vp]),
        "sc_set_mobility_model": (ci, [vp, ci]),
        "sc_minmap_residual": (ci, [vp, i64, vp, vp, vp]),
        "sc_set_residual_trace": (ci, [vp, i32]),
        "sc_get_residual_trace": (ci, [vp, vp, i32, C.POINTER(i32)]),
        "sc_comm_info": (ci, [vp, vp]),
        "sc_sym_pair_table": (ci, [i64, ci, ci, vp, C.POINTER(i64)]),
        "sc_set_wall_velocities": (ci, [vp, ci, vp]),
        "sc_get_walls": (ci, [vp, vp]),
        "sc_set_fmm_params": (ci, [vp, ci, ci]),
        "sc_get_fmm_info": (ci, [vp, vp]),
        "sc_set_fmm_compression": (ci, [vp, ci]),
        "sc_get_fmm_compression_info": (ci, [vp, vp]),
        "sc_set_fmm_tolerance": (ci, [vp, C.c_double, C.POINTER(ci)]),
        "sc_apgd_solve": (ci, [vp, C.POINTER(BbpgdOpts), vp, vp, C.POINTER(BbpgdStats)]),
        "sc_time_step": (ci, [vp, C.POINTER(Problem), C.POINTER(BbpgdOpts), vp, vp, vp, vp, C.POINTER(i64),
                              C.POINTER(BbpgdStats)]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("SC_LIB") and not hasattr(lib, name):
            continue  # an older A/B build without this entry point
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib

"""ctypes binding of the in-tree C ABI (include/hexbp_b200.h).

The product path has no CPU fallback: if ``libhexbp_b200.so`` is missing or
no CUDA device is visible, every operator entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HEXBP_LIB") or os.path.join(_HERE, "libhexbp_b200.so")

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


class SetupInfo(C.Structure):
    _fields_ = [("bp", C.c_int), ("p", C.c_int), ("q", C.c_int), ("dims", C.c_int * 3), ("gdims", C.c_int * 3),
                ("z0", C.c_int), ("components", C.c_int), ("l_size", C.c_int64), ("elements", C.c_int64),
                ("factor_bytes", C.c_int64)]


class CGReportC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("final_rel_residual", C.c_double),
                ("r0_norm", C.c_double), ("seconds", C.c_double)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -m paper_2109_05072_b200.build` "
            "(the B200 path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    i3 = C.POINTER(C.c_int)
    sig = {
        "hexbp_last_error": (C.c_char_p, []),
        "hexbp_device_count": (C.c_int, []),
        "hexbp_setup_create_box": (C.c_int, [C.c_int, C.c_int, i3, _dp, C.c_double, C.c_int, C.POINTER(_vp)]),
        "hexbp_setup_create_box_slab": (C.c_int, [C.c_int, C.c_int, i3, C.c_int, C.c_int, _dp, C.c_double, C.c_int,
                                                  C.POINTER(_vp)]),
        "hexbp_setup_create": (C.c_int, [C.c_int, C.c_int, C.c_int, i3, _dp, _dp, _dp, C.c_int, C.POINTER(_vp)]),
        "hexbp_setup_destroy": (None, [_vp]),
        "hexbp_setup_get_info": (C.c_int, [_vp, C.POINTER(SetupInfo)]),
        "hexbp_setup_basis": (C.c_int, [_vp, _dp, _dp]),
        "hexbp_setup_factors": (C.c_int, [_vp, _dp]),
        "hexbp_workspace_create": (C.c_int, [_vp, C.POINTER(_vp)]),
        "hexbp_workspace_destroy": (None, [_vp]),
        "hexbp_workspace_set_mode": (C.c_int, [_vp, C.c_int]),
        "hexbp_apply": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, _vp]),
        "hexbp_apply_ring_deferred": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, _vp]),
        "hexbp_apply_cg_form": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, _vp]),
        "hexbp_apply_host": (C.c_int, [_vp, _vp, _dp, _dp, C.c_int64, C.c_int]),
        "hexbp_cg": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, C.c_int, C.c_int, C.POINTER(CGReportC), _dp, _vp]),
        "hexbp_pcg": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_double, C.c_int, C.c_int, C.POINTER(CGReportC), _dp,
                                _vp]),
        "hexbp_pcg_host": (C.c_int, [_vp, _vp, _dp, _dp, _dp, C.c_int64, C.c_double, C.c_int, C.c_int,
                                     C.POINTER(CGReportC), _dp]),
        "hexbp_jacobi_diagonal": (C.c_int, [_vp, C.c_int, _vp, _vp]),
        "hexbp_workspace_set_backend": (C.c_int, [_vp, C.c_int]),
        "hexbp_jacobi_diagonal_host": (C.c_int, [_vp, C.c_int, _dp]),
        "hexbp_cg_host": (C.c_int, [_vp, _vp, _dp, _dp, C.c_int64, C.c_double, C.c_int, C.c_int,
                                    C.POINTER(CGReportC), _dp]),
        "hexbp_dot": (C.c_int, [_vp, _vp, _vp, C.c_int64, _dp, _vp]),
        "hexbp_count_flops": (C.c_int, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "hexbp_bench_rhs": (C.c_int, [C.c_int, C.c_int, i3, C.c_uint64, C.c_int64, C.c_int64, _dp]),
        "hexbp_kernel_info": (C.c_int, [_vp] + [C.POINTER(C.c_int)] * 4),
        "hexbp_workspace_vectors": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)]),
        "hexbp_cgd_reduce": (C.c_int, [_vp, C.c_int, _vp, C.c_int64, _vp, _vp]),
        "hexbp_cgd_finish": (C.c_int, [_vp, C.c_int, _vp, C.c_int, C.c_double, C.c_int, _vp]),
        "hexbp_cgd_update_xp": (C.c_int, [_vp, _vp, _vp]),
        "hexbp_cgd_report": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(CGReportC), _dp, C.c_int]),
        "hexbp_plane_combine": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp]),
        "hexbp_cgd_apply_fused": (C.c_int, [_vp, _vp, C.c_int, _vp, _vp]),
        "hexbp_setup_factors_device": (C.c_int, [_vp, _vp, _vp]),
        "hexbp_uniform_stream": (C.c_int, [C.c_uint64, C.c_double, C.c_double, C.c_int64, _vp]),
        "hexbp_workspace_info": (C.c_int, [_vp, _vp, _vp]),
        "hexbp_setup_node_coords": (C.c_int, [_vp, _vp, _vp]),
        "hexbp_interp_to_qpts": (C.c_int, [_vp, _vp, _vp, _vp]),
        "hexbp_interp_transpose": (C.c_int, [_vp, _vp, _vp, _vp]),
        "hexbp_cgd_update_r_fused": (C.c_int, [_vp, C.c_int, _vp, _vp]),
        "hexbp_workspace_reserve": (C.c_int, [_vp, C.c_int, C.c_int]),
        "hexbp_setup_check_restriction": (C.c_int, [_vp, _vp, C.c_int64]),
        "hexbp_dist_unique_id": (C.c_int, [_vp, C.c_int64]),
        "hexbp_dist_create": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_int64, C.c_int, C.POINTER(_vp)]),
        "hexbp_dist_create_box": (C.c_int, [C.c_int, C.c_int, i3, _dp, C.c_double, C.c_int, C.c_int, C.c_int, _vp,
                                            C.c_int64, C.c_int, C.POINTER(_vp)]),
        "hexbp_dist_destroy": (None, [_vp]),
        "hexbp_dist_info": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "hexbp_dist_set_mode": (C.c_int, [_vp, C.c_int]),
        "hexbp_dist_apply": (C.c_int, [_vp, _vp, _vp, C.c_int, _vp]),
        "hexbp_dist_cg": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int, C.c_int, C.POINTER(CGReportC), _dp, _vp]),
        "hexbp_dist_apply_host": (C.c_int, [_vp, _dp, _dp, C.c_int64, C.c_int]),
        "hexbp_dist_cg_host": (C.c_int, [_vp, _dp, _dp, C.c_int64, C.c_double, C.c_int, C.c_int,
                                         C.POINTER(CGReportC), _dp]),
    }
    dev_override = bool(os.environ.get("HEXBP_LIB"))  # A/B timing of older builds (tools/ab_time.py)
    for name, (res, args) in sig.items():
        if dev_override and not hasattr(L, name):
            continue
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def exported_symbols() -> list[str]:
    """Entry points declared in include/hexbp_b200.h (checked by tests)."""
    import re

    hdr = os.path.join(os.path.dirname(_HERE), "include", "hexbp_b200.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(hexbp_[a-z_]+)\s*\(", text)))

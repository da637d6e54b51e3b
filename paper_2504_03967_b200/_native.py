"""ctypes binding of libqgear_b200.so (include/qgear_b200.h).

The library is built in-tree (``python -m paper_2504_03967_b200.build``) and
loaded from this package directory.  There is no fallback: if the library is
missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import re

from .errors import raise_for_status

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QG_LIB_PATH") or os.path.join(_PKG, "libqgear_b200.so")  # override: dev variants
HEADER_PATH = os.path.join(os.path.dirname(_PKG), "include", "qgear_b200.h")

DTYPE_C64 = 0
DTYPE_C128 = 1


class PlanOpts(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("log2_ranks", C.c_int32), ("fuse", C.c_int32),
                ("tile_qubits", C.c_int32), ("max_stages", C.c_int32), ("max_cost", C.c_int32),
                ("kernel_cfg", C.c_int32), ("jit", C.c_int32), ("low_qubits", C.c_int32),
                ("reserved", C.c_int32 * 3)]


class JitStatus(C.Structure):
    _fields_ = [("n_passes", C.c_int64), ("n_jit", C.c_int64), ("n_fallback", C.c_int64), ("n_pending", C.c_int64),
                ("compile_ms_sum", C.c_double), ("compile_ms_wall", C.c_double), ("threads", C.c_int32),
                ("enabled", C.c_int32)]


class Qgir1Info(C.Structure):
    _fields_ = [("capacity", C.c_uint32), ("n_circ", C.c_uint32), ("n_meta", C.c_uint32), ("pad", C.c_uint32),
                ("headers_off", C.c_int64), ("gate_type_off", C.c_int64), ("gate_param_off", C.c_int64),
                ("meta_off", C.c_int64), ("total_bytes", C.c_int64)]


class PlanInfo(C.Structure):
    _fields_ = [("n_body_gates", C.c_int64), ("n_passes", C.c_int64), ("n_segments", C.c_int64),
                ("n_remaps", C.c_int64), ("n_ops", C.c_int64), ("n_stages", C.c_int64),
                ("tile_qubits", C.c_int32), ("n_local", C.c_int32), ("n_qubits", C.c_int32),
                ("dtype", C.c_int32), ("param_bytes", C.c_int64), ("n_cxm", C.c_int64)]


class Remap(C.Structure):
    _fields_ = [("s", C.c_int32), ("global_pos", C.c_int32 * 8), ("local_pos", C.c_int32 * 8)]


class ExecStats(C.Structure):
    _fields_ = [("pass_ms", C.c_double), ("pass_launches", C.c_int64), ("bytes_moved", C.c_int64)]


_P = C.c_void_p
_SIGS = {
    "qg_plan_create": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.POINTER(PlanOpts), C.POINTER(_P)]),
    "qg_plan_destroy": (C.c_int, [_P]),
    "qg_plan_rebind": (C.c_int, [_P, _P, C.c_int64]),
    "qg_plan_get_info": (C.c_int, [_P, C.POINTER(PlanInfo)]),
    "qg_plan_get_remap": (C.c_int, [_P, C.c_int64, C.POINTER(Remap)]),
    "qg_plan_get_final_map": (C.c_int, [_P, _P]),
    "qg_plan_export": (C.c_int, [_P, _P, C.POINTER(C.c_int64), _P, C.POINTER(C.c_int64)]),
    "qg_state_init_zero": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P]),
    "qg_state_init_uniform": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_uint64, C.c_int32, _P]),
    "qg_plan_execute_segment": (C.c_int, [_P, C.c_int64, _P, C.c_int32, _P, C.c_int32, C.POINTER(ExecStats)]),
    "qg_plan_execute": (C.c_int, [_P, _P, _P, C.c_int32, C.POINTER(ExecStats)]),
    "qg_apply_matrix": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P, _P]),
    "qg_apply_cx": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P]),
    "qg_apply_cr1": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, _P]),
    "qg_ucry_workspace_bytes": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "qg_apply_ucry": (C.c_int, [_P, C.c_int32, C.c_int32, _P, C.c_int32, _P, C.c_int32, _P, _P, C.c_int64, _P]),
    "qg_norm_sq": (C.c_int, [_P, C.c_int64, C.c_int32, _P, C.c_int64, C.POINTER(C.c_double), _P]),
    "qg_probabilities": (C.c_int, [_P, C.c_int64, C.c_int32, _P, _P]),
    "qg_sample_workspace_bytes": (C.c_int64, [C.c_int64, C.c_int64]),
    "qg_sample": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int64, C.c_uint64, _P, C.c_double, _P, C.c_int64,
                            _P, _P, C.POINTER(C.c_int64), C.POINTER(C.c_double), _P]),
    "qg_sample_async": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int64, C.c_uint64, _P, C.c_int64, _P, _P, _P, _P,
                                  _P]),
    "qg_qcrank_tally": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, _P]),
    "qg_sample_tree_workspace_bytes": (C.c_int64, [C.c_int64]),
    "qg_sample_tree_prepare": (C.c_int, [_P, C.c_int64, C.c_int32, _P, C.c_int64, C.POINTER(C.c_double), _P]),
    "qg_sample_tree_draw": (C.c_int, [_P, C.c_int64, C.c_int32, _P, C.c_int64, C.c_int64, C.c_uint64, C.c_uint32,
                                      C.c_int32, C.c_int64, _P, _P, C.c_int64, C.POINTER(C.c_int64), _P, _P]),
    "qg_split_shots": (C.c_int, [_P, C.c_int32, C.c_int64, C.c_uint64, _P, C.c_int64, _P, _P]),
    "qg_binomial_test": (C.c_int, [C.c_double, C.c_double, C.c_uint64, C.c_int64, _P, _P]),
    "qg_qgir1_parse": (C.c_int, [_P, C.c_int64, C.POINTER(Qgir1Info)]),
    "qg_qgir1_size": (C.c_int64, [C.c_uint32, C.c_uint32, C.c_uint32, _P]),
    "qg_qgir1_write": (C.c_int, [_P, C.c_int64, C.c_uint32, C.c_uint32, _P, _P, _P, C.c_uint32, _P, _P]),
    "qg_container_last_error": (C.c_char_p, []),
    "qg_last_error": (C.c_char_p, []),
    "qg_abi_version": (C.c_int, []),
}

_lib = None


def header_functions() -> list[str]:
    """Every function name declared in include/qgear_b200.h."""
    with open(HEADER_PATH) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(qg_\w+)\s*\(", text, flags=re.M)))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2504_03967_b200.build` "
                "(there is no CPU fallback)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(code: int) -> None:
    if code != 0:
        err = lib().qg_container_last_error if code == -14 else lib().qg_last_error
        raise_for_status(code, err().decode(errors="replace"))


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))

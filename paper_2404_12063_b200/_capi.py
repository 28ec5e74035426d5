"""ctypes binding of include/vpinn_gpu.h (the C-ABI of the B200 step).

Loads the in-tree paper_2404_12063_b200/_lib/libvpinn_b200.so and fails
loudly when it is missing: there is no Python or CPU fallback for the path.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "libvpinn_b200.so")
HEADER = os.path.join(os.path.dirname(_PKG), "include", "vpinn_gpu.h")

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


class Assembly(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int64), ("nodes", C.c_void_p), ("elements", C.c_void_p),
        ("xi", C.c_void_p), ("eta", C.c_void_p), ("weights", C.c_void_p),
        ("basis_val", C.c_void_p), ("basis_dxi", C.c_void_p), ("basis_deta", C.c_void_p),
        ("forcing", C.c_char_p),
    ]


class Problem(C.Structure):
    _fields_ = [
        ("n_elem", C.c_int32), ("n_test", C.c_int32), ("n_quad", C.c_int32),
        ("grad_x", C.c_void_p), ("grad_y", C.c_void_p), ("test", C.c_void_p),
        ("forcing", C.c_void_p), ("points", C.c_void_p),
        ("n_interior", C.c_int64), ("n_boundary", C.c_int64), ("n_sensors", C.c_int64),
        ("boundary_values", C.c_void_p), ("sensor_values", C.c_void_p),
        ("n_layer_sizes", C.c_int32), ("layer_sizes", C.c_void_p), ("activation", C.c_int32),
        ("n_scalars", C.c_int32),
        ("eps", C.c_float), ("bx", C.c_float), ("by", C.c_float),
        ("eps_source", C.c_int32), ("eps_scalar_index", C.c_int32),
        ("tau", C.c_double), ("gamma", C.c_double),
        ("device", C.c_int32), ("rank", C.c_int32), ("world_size", C.c_int32),
        ("assembly", C.c_void_p),
        ("form", C.c_int32), ("strong_forcing", C.c_void_p),
    ]


FORM_WEAK, FORM_STRONG = 0, 1


class TrainSpec(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64), ("lr_exponential", C.c_int32),
        ("lr0", C.c_double), ("decay", C.c_double), ("every", C.c_int32),
        ("has_eps_abs_tol", C.c_int32), ("has_eps_actual", C.c_int32), ("has_loss_tol", C.c_int32),
        ("eps_abs_tol", C.c_double), ("eps_actual", C.c_double), ("loss_tol", C.c_double),
        ("plateau_window", C.c_int32), ("steps_per_graph", C.c_int32),
    ]


class StepRecord(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("total", "variational", "boundary", "sensor", "lr", "eps", "seconds")]


class TrainResult(C.Structure):
    _fields_ = [("steps_run", C.c_int64), ("converged", C.c_int32), ("stop_reason", C.c_int32),
                ("abort_step", C.c_int64), ("final_eps", C.c_double)]


def declared_symbols():
    """Function names declared by include/vpinn_gpu.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(vpinn_gpu_\w+)\s*\(", text)))


def _declare(L):
    vp, i32, i64, d = C.c_void_p, C.c_int, C.c_int64, C.c_double
    pd = C.POINTER(C.c_double)
    sig = {
        "vpinn_gpu_last_error": (C.c_char_p, []),
        "vpinn_gpu_version": (C.c_char_p, []),
        "vpinn_gpu_step_kernel": (C.c_char_p, [vp]),
        "vpinn_gpu_device_ok": (i32, []),
        "vpinn_gpu_partition": (None, [i64, i64, i64, i32, i32, vp]),
        "vpinn_gpu_create": (i32, [C.POINTER(Problem), C.POINTER(vp)]),
        "vpinn_gpu_destroy": (None, [vp]),
        "vpinn_gpu_param_count": (i32, [vp]),
        "vpinn_gpu_set_params": (i32, [vp, vp, i32]),
        "vpinn_gpu_get_params": (i32, [vp, vp, i32]),
        "vpinn_gpu_loss_and_grad": (i32, [vp, vp, vp]),
        "vpinn_gpu_train": (i32, [vp, C.POINTER(TrainSpec), vp, C.POINTER(TrainResult)]),
        "vpinn_gpu_adam_reset": (i32, [vp]),
        "vpinn_gpu_run_steps": (i32, [vp, i32, d]),
        "vpinn_gpu_synchronize": (i32, [vp]),
        "vpinn_gpu_time_steps": (i32, [vp, i32, d, pd]),
        "vpinn_gpu_forward": (i32, [vp, vp, i64, i32, vp, vp, vp, vp]),
        "vpinn_gpu_forward2": (i32, [vp, vp, i64, vp, vp, vp, vp, vp]),
        "vpinn_gpu_contract": (i32, [vp, vp, vp, vp, vp, C.c_float, pd, vp, vp, vp, vp, vp]),
        "vpinn_gpu_time_contract": (i32, [vp, i32, pd, pd]),
        "vpinn_gpu_peer_handle": (i32, [vp, vp]),
        "vpinn_gpu_attach_peers": (i32, [vp, vp, i32, i32]),
        "vpinn_gpu_time_contract_kernels": (i32, [vp, i32, pd, pd, pd]),
        "vpinn_gpu_download_tensor": (i32, [vp, i32, vp, i64]),
        "vpinn_gpu_launch_count": (i64, [vp]),
        "vpinn_gpu_profile_step": (i32, [vp, i32, pd, pd, pd]),
        "vpinn_gpu_measure_ffma_peak": (i32, [i32, pd]),
        "vpinn_gpu_tc_probe": (i32, [i32, i32, vp, vp, vp, vp]),
        "vpinn_gpu_flush_l2": (i32, [vp]),
        "vpinn_gpu_phase_clock": (i32, [vp, vp, i32]),
        "vpinn_gpu_assemble": (i32, [i32, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
        "vpinn_gpu_release_cached_memory": (i32, []),
        "vpinn_gpu_set_test_hooks": (i32, [i32]),
        "vpinn_gpu_contract_matrix_free": (i32, [vp, vp, vp, vp, C.c_float, pd, vp, vp, vp, vp]),
        "vpinn_gpu_time_contract_matrix_free": (i32, [vp, i32, pd, pd]),
        "vpinn_gpu_nccl_unique_id": (i32, [vp]),
        "vpinn_gpu_attach_comm": (i32, [vp, vp, i32, i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} is missing: build it with `python -m paper_2404_12063_b200.build_native` "
                "(there is no CPU fallback for the B200 step)")
        _lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        _declare(_lib)
    return _lib


class VpinnError(RuntimeError):
    """Carries the reference ErrorCategory code (core.hpp:17-22; 6 = device)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def partition(n_elem, n_boundary, n_sensors, rank, world):
    """The rank's (e0, e1, b0, b1, s0, s1) exactly as vpinn_gpu_create splits."""
    out = (C.c_int64 * 6)()
    lib().vpinn_gpu_partition(n_elem, n_boundary, n_sensors, rank, world, out)
    return tuple(out)


def check(rc: int):
    if rc != 0:
        raise VpinnError(rc, lib().vpinn_gpu_last_error().decode(errors="replace"))

"""ctypes binding of libfusg.so (the C-ABI declared in include/fusg.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_2011_03009_b200/csrc``).  There is no fallback: if the library is missing or a CUDA
device is unavailable, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# FUSG_LIB: alternative build of the same library (kernel-variant experiments in tools/)
LIB_PATH = os.environ.get("FUSG_LIB") or os.path.join(_HERE, "libfusg.so")

FUSG_OK, FUSG_INVALID_ARGUMENT, FUSG_OUT_OF_RANGE, FUSG_RUNTIME, FUSG_CUDA, FUSG_NCCL, FUSG_OOM, FUSG_NOT_CONVERGED = range(8)


class FusgError(RuntimeError):
    """Device/runtime failure reported by libfusg (CUDA, NCCL, allocation)."""


class Grid(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3), ("dx", C.c_double),
                ("dims", C.c_int32 * 3), ("harmonic", C.c_int32)]


class Wave(C.Structure):
    _fields_ = [("k_re", C.c_double), ("k_im", C.c_double), ("harmonic", C.c_int32),
                ("omega", C.c_double)]


class MediumC(C.Structure):
    _fields_ = [("rho0", C.c_double), ("c0", C.c_double), ("beta", C.c_double),
                ("alpha0", C.c_double), ("eta", C.c_double)]


class Bowl(C.Structure):
    _fields_ = [("f0", C.c_double), ("focal_length", C.c_double), ("outer_radius", C.c_double),
                ("power", C.c_double), ("n_points", C.c_int32),
                ("points_host", C.POINTER(C.c_double))]


OperatorFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)


class VieConfigC(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int32), ("restart", C.c_int32)]


class StageTiming(C.Structure):
    _fields_ = [("harmonic", C.c_int32), ("voxels", C.c_uint64), ("meshing_s", C.c_double),
                ("interpolation_s", C.c_double), ("kernel_s", C.c_double),
                ("potential_s", C.c_double), ("p1_s", C.c_double), ("rhs_s", C.c_double)]


class CascadeDesc(C.Structure):
    _fields_ = [("medium", MediumC), ("transducer", Bowl), ("grids", C.POINTER(Grid)),
                ("n_harmonics", C.c_int32), ("recompute_p1_each_grid", C.c_int32),
                ("pad_small_primes", C.c_int32)]


_dp = C.POINTER(C.c_double)
_vp = C.c_void_p

# name -> (restype, argtypes); every symbol include/fusg.h declares
SIGNATURES = {
    "fusg_last_error": (C.c_char_p, []),
    "fusg_version": (C.c_char_p, []),
    "fusg_make_grid": (C.c_int, [_dp, _dp, C.c_double, C.c_int32, _dp, C.POINTER(Grid)]),
    "fusg_complex_wavenumber": (C.c_int, [C.POINTER(MediumC), C.c_double, C.c_int32, C.POINTER(Wave)]),
    "fusg_self_weight": (C.c_int, [C.POINTER(Wave), C.c_double, _dp]),
    "fusg_equivalent_sphere_radius": (C.c_double, [C.c_double]),
    "fusg_next_fast_size": (C.c_int32, [C.c_int32]),
    "fusg_padded_dims": (C.c_int, [C.POINTER(Grid), C.c_int32, C.POINTER(C.c_int32)]),
    "fusg_static_lengths": (C.c_int32, [C.c_int32, C.POINTER(C.c_int32), C.c_int32]),
    "fusg_distribute_points": (C.c_int, [C.c_double, C.c_double, C.c_int32, _dp]),
    "fusg_plan_nested_meshes": (C.c_int, [C.POINTER(Bowl), C.POINTER(MediumC), C.c_double, C.c_int32,
                                          C.c_int32, C.c_double, C.c_int32, C.POINTER(Grid), _dp, _dp,
                                          C.POINTER(Grid), _dp]),
    "fusg_rhs_coefficient": (C.c_double, [C.POINTER(MediumC), C.c_double, C.c_int32]),
    "fusg_random_vector": (C.c_int, [C.c_int64, C.c_uint32, _dp]),
    "fusg_ctx_create": (C.c_int, [C.c_int32, C.POINTER(_vp)]),
    "fusg_ctx_destroy": (C.c_int, [_vp]),
    "fusg_ctx_stream": (_vp, [_vp]),
    "fusg_ctx_synchronize": (C.c_int, [_vp]),
    "fusg_ctx_launch_count": (C.c_uint64, [_vp]),
    "fusg_kernel_create": (C.c_int, [_vp, C.POINTER(Grid), C.POINTER(Wave), C.c_int32, C.POINTER(_vp)]),
    "fusg_kernel_destroy": (C.c_int, [_vp]),
    "fusg_kernel_padded": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "fusg_kernel_device_bytes": (C.c_uint64, [_vp]),
    "fusg_kernel_apply": (C.c_int, [_vp, _vp, _vp, C.c_double, _vp]),
    "fusg_kernel_apply_timed": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int32, _dp]),
    "fusg_kernel_apply_host": (C.c_int, [_vp, _vp, _vp, C.c_double]),
    "fusg_monopole_grid": (C.c_int, [_vp, _dp, C.c_int32, C.POINTER(Grid), C.c_double, C.c_double,
                                     C.c_double, _vp, _vp]),
    "fusg_interpolate_source_planes": (C.c_int, [C.POINTER(Grid), C.POINTER(Grid), C.c_int32, C.c_int32,
                                                 C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "fusg_interpolate_zslab": (C.c_int, [_vp, C.POINTER(Grid), C.c_int32, C.c_int32, _vp, C.POINTER(Grid),
                                         C.c_int32, C.c_int32, _vp, _vp]),
    "fusg_monopole_grid_zslab": (C.c_int, [_vp, _dp, C.c_int32, C.POINTER(Grid), C.c_int32, C.c_int32,
                                           C.c_double, C.c_double, C.c_double, _vp, _vp]),
    "fusg_monopole_points": (C.c_int, [_vp, _dp, C.c_int32, _vp, C.c_int64, C.c_double, C.c_double,
                                       C.c_double, _vp, _vp]),
    "fusg_evaluate_potential_at": (C.c_int, [_vp, C.POINTER(Grid), C.POINTER(Wave), _vp, _vp, C.c_int64, _vp]),
    "fusg_field_threshold_box": (C.c_int, [_vp, C.POINTER(Grid), _vp, C.c_double, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
    "fusg_localisedness_map": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "fusg_radiated_power": (C.c_int, [_vp, _dp, C.c_int32, C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.c_double, C.c_double, C.c_double, C.c_int32,
                                      C.c_int32, _dp]),
    "fusg_rhs_source": (C.c_int, [_vp, C.c_int32, C.POINTER(_vp), C.c_int64, C.POINTER(MediumC),
                                  C.c_double, _vp, _vp]),
    "fusg_rhs_source_full": (C.c_int, [_vp, C.c_int32, C.POINTER(_vp), C.c_int32, C.c_int64,
                                       C.POINTER(MediumC), C.c_double, _vp, _vp]),
    "fusg_interpolate": (C.c_int, [_vp, C.POINTER(Grid), _vp, C.POINTER(Grid), _vp, _vp]),
    "fusg_run_cascade": (C.c_int, [_vp, C.POINTER(CascadeDesc), C.POINTER(_vp),
                                   C.POINTER(StageTiming), _dp]),
    "fusg_slab_range": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32)]),
    "fusg_slab_exchange_plan": (C.c_int, [C.POINTER(Grid), C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int64)]),
    "fusg_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "fusg_ctx_attach_nccl": (C.c_int, [_vp, C.c_int32, C.c_int32, C.POINTER(C.c_uint8)]),
    "fusg_kernel_create_slab": (C.c_int, [_vp, C.POINTER(Grid), C.POINTER(Wave), C.c_int32, C.c_int32,
                                          C.c_int32, C.POINTER(_vp)]),
    "fusg_kernel_octant_rows": (C.c_int, [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "fusg_kernel_slab": (C.c_int, [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "fusg_kernel_apply_slab": (C.c_int, [_vp, _vp, _vp, C.c_double, _vp]),
    "fusg_kernel_apply_slab_loopback": (C.c_int, [C.POINTER(_vp), C.c_int32, C.POINTER(_vp),
                                                  C.POINTER(_vp), C.c_double]),
    "fusg_vie_contrast": (C.c_int, [_vp, _vp, C.c_int64, C.POINTER(MediumC), C.c_double, C.c_int32, _vp, _vp]),
    "fusg_vie_operator_apply": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "fusg_gmres": (C.c_int, [_vp, OperatorFn, _vp, _vp, C.c_int64, C.c_double, C.c_int32, C.c_int32, _vp,
                             C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "fusg_solve_vie": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int32, C.c_int32, _vp, C.POINTER(C.c_double),
                                 C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "fusg_run_cascade_inhomogeneous": (C.c_int, [_vp, C.POINTER(CascadeDesc), C.POINTER(Grid), _vp,
                                                 C.POINTER(MediumC), C.POINTER(VieConfigC), C.POINTER(_vp),
                                                 C.POINTER(StageTiming), C.POINTER(C.c_double)]),
    "fusg_device_copy": (C.c_int, [_vp, _vp, _vp, C.c_uint64]),
    "fusg_slab_peer_plan": (C.c_int, [C.POINTER(Grid), C.c_int32, C.c_int32] + [C.POINTER(C.c_int64)] * 6),
    "fusg_kernel_slab_ipc_handles": (C.c_int, [_vp, C.POINTER(C.c_uint8)]),
    "fusg_kernel_slab_attach_peers": (C.c_int, [_vp, C.POINTER(C.c_uint8)]),
    "fusg_kernel_apply_slab_p2p": (C.c_int, [_vp, _vp, _vp, C.c_double, _vp]),
    "fusg_kernel_apply_slab_loopback_p2p": (C.c_int, [C.POINTER(_vp), C.c_int32, C.POINTER(_vp),
                                                      C.POINTER(_vp), C.c_double]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libfusg.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FusgError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                            "(make -C paper_2011_03009_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    """Map a fusg_status to the reference's exception classes."""
    if status == FUSG_OK:
        return
    msg = lib().fusg_last_error().decode(errors="replace")
    if status == FUSG_INVALID_ARGUMENT:
        raise ValueError(msg)          # std::invalid_argument
    if status == FUSG_OUT_OF_RANGE:
        raise IndexError(msg)          # std::out_of_range
    if status == FUSG_RUNTIME:
        raise RuntimeError(msg)        # std::runtime_error
    raise FusgError(f"[status {status}] {msg}")

"""ctypes binding of libnpcg.so (the C ABI declared in include/npcg.h).

The library is the product: there is no Python or CPU fallback.  Importing
works on a CPU-only machine (so the ABI can be inspected), but every compute
call goes through a context, and creating a context without a B200 fails
loudly with the library's own status.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnpcg.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "npcg.h")

_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_D = C.c_double
_PI64 = C.POINTER(C.c_int64)


class npcg_exec_config(C.Structure):
    _fields_ = [("L", _I64), ("b_out", _I64), ("b_in", _I64), ("executor", _I32),
                ("deterministic", _I32), ("workers", _I32), ("math", _I32), ("flags", _I32),
                ("reserved", _I32)]

FLAG_FIN_UNCHANGED = 1  # NPCG_FLAG_FIN_UNCHANGED


class npcg_cloud(C.Structure):
    _fields_ = [("xyz", _P), ("batch_offsets", _P), ("n_points", _I64), ("n_batches", _I64)]


class npcg_triplets(C.Structure):
    _fields_ = [("i", _P), ("j", _P), ("k", _P), ("size", _I64), ("n_out", _I64), ("n_in", _I64),
                ("n_kernels", _I64), ("sort_axis", _I32)]


STATUS_NAMES = {
    0: "ok", 1: "OffsetError", 2: "NonFiniteError", 3: "ShapeError", 4: "RadiusError",
    5: "VoxelError", 6: "IndexError", 7: "DomainError", 8: "StateError", 9: "IOError",
    10: "CudaError", 11: "OutOfMemory", 12: "InvalidArgument", 13: "Unsupported",
}

# name -> (restype, argtypes)
_SIGS = {
    "npcg_api_version": (C.c_int, []),
    "npcg_status_string": (C.c_char_p, [C.c_int]),
    "npcg_context_create": (C.c_int, [C.c_int, _P, C.POINTER(_P)]),
    "npcg_context_destroy": (C.c_int, [_P]),
    "npcg_context_set_stream": (C.c_int, [_P, _P]),
    "npcg_context_synchronize": (C.c_int, [_P]),
    "npcg_last_error": (C.c_char_p, [_P]),
    "npcg_launch_count": (C.c_int, [_P, _PI64]),
    "npcg_profile_enable": (C.c_int, [_P, C.c_int]),
    "npcg_profile_reset": (C.c_int, [_P]),
    "npcg_profile_query": (C.c_int, [_P, C.c_char_p, _PI64, C.POINTER(_D)]),
    "npcg_profile_dump": (C.c_int, [_P, C.c_char_p, C.c_size_t]),
    "npcg_memory_stats": (C.c_int, [_P, _PI64, _PI64]),
    "npcg_memory_reset_peak": (C.c_int, [_P]),
    "npcg_radius_search": (C.c_int, [_P, C.POINTER(npcg_cloud), C.POINTER(npcg_cloud), _D,
                                     C.POINTER(_P)]),
    "npcg_build_triplets_native": (C.c_int, [_P, C.POINTER(npcg_cloud), C.POINTER(npcg_cloud), _D,
                                             _I64, C.POINTER(_P)]),
    "npcg_neighbors_destroy": (C.c_int, [_P]),
    "npcg_neighbors_size": (C.c_int, [_P, _PI64]),
    "npcg_neighbors_info": (C.c_int, [_P, _PI64, _PI64, _PI64, C.POINTER(_D)]),
    "npcg_neighbors_export_pairs": (C.c_int, [_P, _P, _P, _P]),
    "npcg_neighbors_export_triplets": (C.c_int, [_P, _P, _I32, _P, _P, _P]),
    "npcg_kernel_index": (C.c_int, [_P, _P, _P, _I64, _D, _I64, _P]),
    "npcg_sort_triplets": (C.c_int, [_P, C.POINTER(npcg_triplets), _I32, _P, _P, _P]),
    "npcg_choose_sort_axis": (_I32, [_I64, _I64, _I64]),
    "npcg_mvmr": (C.c_int, [_P, C.c_int, _P, _I64, _I64, _I64, _I64, _P, _I64,
                            C.POINTER(npcg_triplets), _I64, C.POINTER(npcg_exec_config), _P]),
    "npcg_mvmr_transposed": (C.c_int, [_P, C.c_int, _P, _I64, _I64, _I64, _I64, _P, _I64,
                                       C.POINTER(npcg_triplets), _I64,
                                       C.POINTER(npcg_exec_config), _P]),
    "npcg_vvor": (C.c_int, [_P, C.c_int, _P, _I64, _P, _I64, _I64, _I64, _I64,
                            C.POINTER(npcg_triplets), _I64, C.POINTER(npcg_exec_config), _P]),
    "npcg_mvmr_fwd": (C.c_int, [_P, C.c_int, _P, _I64, _I64, _I64, _I64, _P, _I64,
                                C.POINTER(npcg_triplets), _I64, C.POINTER(npcg_exec_config), _P]),
    "npcg_mvmr_dgrad": (C.c_int, [_P, C.c_int, _P, _I64, _I64, _I64, _I64, _P, _I64,
                                  C.POINTER(npcg_triplets), _I64, C.POINTER(npcg_exec_config), _P]),
    "npcg_vvor_wgrad": (C.c_int, [_P, C.c_int, _P, _I64, _P, _I64, _I64, _I64, _I64,
                                  C.POINTER(npcg_triplets), _I64, C.POINTER(npcg_exec_config), _P]),
    "npcg_conv_forward": (C.c_int, [_P, _P, C.c_int, _P, _I64, _I64, _I64, _P,
                                    C.POINTER(npcg_exec_config), _P]),
    "npcg_conv_backward": (C.c_int, [_P, _P, C.c_int, _P, _I64, _I64, _I64, _P, _P,
                                     C.POINTER(npcg_exec_config), _P, _P]),
    "npcg_neighbors_prepare": (C.c_int, [_P, _P, _I32]),
    "npcg_neighbors_plan_stats": (C.c_int, [_P, _P, _P]),
    "npcg_debug_trace_forward": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "npcg_voxel_downsample": (C.c_int, [_P, C.POINTER(npcg_cloud), _D, _P, _P, _P, _PI64]),
    "npcg_upsample": (C.c_int, [_P, C.c_int, _P, _I64, _P, _I64, _I64, _P]),
    "npcg_gen_uniform_cube": (C.c_int, [_I64, _D, C.c_uint64, _P]),
    "npcg_gen_features": (C.c_int, [_I64, _I64, _I64, C.c_uint64, C.c_int, _P]),
    "npcg_make_weights": (C.c_int, [_I64, _I64, _I64, _I64, C.c_uint64, C.c_int, _P]),
    "npcg_comm_unique_id": (C.c_int, [_P]),
    "npcg_comm_create": (C.c_int, [_P, C.c_int, C.c_int, _P, C.POINTER(_P)]),
    "npcg_comm_destroy": (C.c_int, [_P]),
    "npcg_allreduce_dw": (C.c_int, [_P, _P, C.c_int, _P, _I64]),
    "npcg_build_triplets_degraded": (C.c_int, [_P, C.POINTER(npcg_cloud), _D, _I64, C.POINTER(_P)]),
    "npcg_neighbors_sites": (C.c_int, [_P, _PI64, _PI64, _PI64]),
    "npcg_neighbors_export_sites": (C.c_int, [_P, _P, _P, _P, _P, _P]),
}

_lib = None


def header_functions() -> list[str]:
    """Every function name declared in include/npcg.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(npcg_[a-z0-9_]+)\s*\(", txt)))


def lib():
    """Load libnpcg.so (raises if it was not built -- no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2511_23227_b200.build`"
                               " (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib

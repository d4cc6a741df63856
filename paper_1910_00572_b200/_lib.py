"""ctypes binding of the C-ABI (include/gridloc_b200.h).

Loads the in-tree ``libgridloc_b200.so``. There is no fallback: if the
library is missing or fails to load, importing the product raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GRIDLOC_B200_LIB", os.path.join(HERE, "libgridloc_b200.so"))

GL_OK = 0
GL_E_EXTINGUISHED = 1
GL_E_INVALID = 2
GL_E_MAP_PARSE = 3
GL_E_RUNTIME = 4
GL_E_CUDA = 5

GL_PATH_AUTO, GL_PATH_FUSED, GL_PATH_GENERIC = 0, 1, 2


class KernelInfo(C.Structure):
    _fields_ = [
        ("channels", C.c_int),
        ("radius", C.c_int),
        ("separable", C.c_int),
        ("degenerate_spatial", C.c_int),
        ("degenerate_angular", C.c_int),
        ("n_angular", C.c_int),
    ]


class PoseEstimateC(C.Structure):
    _fields_ = [
        ("x", C.c_double),
        ("y", C.c_double),
        ("theta", C.c_double),
        ("confidence", C.c_double),
        ("i", C.c_int),
        ("j", C.c_int),
        ("k", C.c_int),
    ]


class LikelihoodC(C.Structure):
    _fields_ = [("sigma_hit", C.c_double), ("weight_floor", C.c_double), ("beam_stride", C.c_int)]


class DifficultyC(C.Structure):
    _fields_ = [("error_threshold", C.c_double), ("beam_count", C.c_int), ("fov", C.c_double),
                ("max_range", C.c_double), ("stride", C.c_int), ("theta_bins", C.c_int),
                ("likelihood", LikelihoodC)]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p
_pvp = C.POINTER(C.c_void_p)

# (name, argtypes) for every exported symbol; tests check the list against
# include/gridloc_b200.h.
SIGNATURES = {
    "gl_last_error": [],
    "gl_version": [],
    "gl_context_create": [C.c_int, _pvp],
    "gl_context_destroy": [_vp],
    "gl_context_synchronize": [_vp],
    "gl_context_last_step_ms": [_vp, _dp],
    "gl_context_set_step_timing": [_vp, C.c_int],
    "gl_context_set_path": [_vp, C.c_int],
    "gl_context_set_fast": [_vp, C.c_int],
    "gl_context_set_himax": [_vp, C.c_int],
    "gl_context_set_channel_chunks": [_vp, C.c_int],
    "gl_context_set_wave_tail": [_vp, C.c_int, C.c_int],
    "gl_context_set_host_exp": [_vp, C.c_int],
    "gl_context_set_tile_order": [_vp, C.c_int, C.c_int],
    "gl_context_set_wall_mask": [_vp, C.c_int],
    "gl_shard_init_uniform": [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _pvp],
    "gl_shard_info": [_vp, _ip, _ip, _ip, _ip],
    "gl_tensor_plane_ptr": [_vp, _vp, C.c_int, C.POINTER(_dp)],
    "gl_tensor_max_ptr": [_vp, _vp, C.POINTER(C.POINTER(C.c_uint64))],
    "gl_shard_finalize": [_vp, _vp],
    "gl_tensor_copy_planes": [_vp, _vp, C.c_int, _vp, C.c_int, C.c_int],
    "gl_write_belief_snapshot": [_vp, _vp, C.c_char_p],
    "gl_read_belief_snapshot": [_vp, C.c_char_p, C.c_double, C.c_double, C.c_double, _pvp],
    "gl_debug_counters": [_vp, C.POINTER(C.c_uint64)],
    "gl_map_difficulty": [_vp, _vp, _vp, C.POINTER(DifficultyC), _dp],
    "gl_shard_set_peers": [_vp, _vp, _vp, _vp, C.c_int, _vp, _vp, C.c_int],
    "gl_tensor_buffer_ptr": [_vp, _vp, C.c_int, C.c_int, C.POINTER(_dp)],
    "gl_tensor_current_buffer": [_vp, _ip],
    "gl_ipc_get_handle": [_vp, _vp, C.c_int, _vp],
    "gl_ipc_open": [_vp, _vp, _pvp],
    "gl_ipc_close": [_vp, _vp],
    "gl_context_launch_count": [_vp, C.POINTER(C.c_uint64)],
    "gl_context_stream": [_vp, _pvp],
    "gl_context_time_steps": [_vp, C.c_int],
    "gl_tensors_status": [_vp, C.POINTER(_vp), C.c_int, C.POINTER(C.c_int)],
    "gl_context_step_times": [_vp, _dp, _ip],
    "gl_context_mark": [_vp, C.c_int],
    "gl_context_marks_ms": [_vp, C.c_int, C.c_int, _dp],
    "gl_load_map": [_u8p, C.c_size_t, C.c_int, _ip, _ip, _u8p],
    "gl_map_create": [_vp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, _u8p, _pvp],
    "gl_map_destroy": [_vp],
    "gl_map_info": [_vp, _ip, _ip, _dp, _dp, _dp, _ip],
    "gl_map_cells": [_vp, _u8p],
    "gl_field_create": [_vp, _vp, _pvp],
    "gl_field_destroy": [_vp],
    "gl_field_values": [_vp, _dp],
    "gl_build_kernels": [C.c_double, C.c_double, C.c_double, C.c_int, C.c_double, C.c_double, _pvp],
    "gl_kernels_create": [_vp, C.POINTER(KernelInfo), _dp, _dp, _ip, _dp, _pvp],
    "gl_kernels_destroy": [_vp],
    "gl_kernels_info": [_vp, C.POINTER(KernelInfo)],
    "gl_kernels_get": [_vp, _dp, _dp, _ip, _dp],
    "gl_make_activation": [_vp, _vp, _vp, C.c_int, _pvp],
    "gl_activation_destroy": [_vp],
    "gl_activation_get": [_vp, _vp, _dp, _dp],
    "gl_tensor_create": [_vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, _pvp],
    "gl_init_uniform": [_vp, _vp, C.c_int, _pvp],
    "gl_tensor_destroy": [_vp],
    "gl_tensor_info": [_vp, _ip, _ip, _ip, _dp, _dp, _dp],
    "gl_tensor_theta": [_vp, _dp],
    "gl_tensor_set_theta": [_vp, C.c_double],
    "gl_tensor_upload": [_vp, _vp, _dp],
    "gl_tensor_download": [_vp, _vp, _dp],
    "gl_tensor_hash": [_vp, _vp, C.POINTER(C.c_uint64)],
    "gl_tensor_read": [_vp, _vp, C.c_size_t, C.c_size_t, _dp],
    "gl_tensor_write": [_vp, _vp, C.c_size_t, C.c_size_t, _dp],
    "gl_tensor_clone": [_vp, _vp, _pvp],
    "gl_tensor_device_ptr": [_vp, _vp, C.POINTER(_dp)],
    "gl_step": [_vp, _vp, C.c_double, C.c_double, C.c_double, _vp, _vp, _vp],
    "gl_step_async": [_vp, _vp, C.c_double, C.c_double, C.c_double, _vp, _vp, _vp],
    "gl_tensor_status": [_vp, _vp],
    "gl_apply_motion": [_vp, _vp, C.c_double, C.c_double, C.c_double],
    "gl_belief_map": [_vp, _vp, _dp],
    "gl_argmax": [_vp, _vp, C.POINTER(PoseEstimateC)],
    "gl_dither": [_vp, _dp, C.c_int, C.c_int, C.c_int, _ip, C.c_int, _ip, _dp],
    "gl_dither_tensor": [_vp, _vp, C.c_int, _ip, C.c_int, _ip, _dp],
    "gl_scan_likelihood": [_vp, _vp, _vp, C.c_double, C.c_double, C.c_double, _dp, _dp, C.c_int,
                           C.c_double, LikelihoodC, _dp],
    "gl_observation_update": [_vp, _vp, _ip, C.c_int, _dp, _dp, C.c_int, C.c_double, _vp, _vp,
                              LikelihoodC],
    "gl_dither_device": [_vp, _vp, C.c_int, C.c_int, C.c_int, _ip, C.c_int, _ip, _dp],
    "gl_shard_belief_map": [_vp, _vp, _vp],
    "gl_shard_observe": [_vp, _vp, _ip, C.c_int, _dp, _dp, C.c_int, C.c_double, _vp, _vp, LikelihoodC],
    "gl_shard_observe_finalize": [_vp, _vp],
    "gl_tensor_hash_at": [_vp, _vp, C.c_uint64, C.POINTER(C.c_uint64)],
    "gl_raycast": [_vp, _vp, _dp, C.c_int, C.c_double, _dp],
    "gl_sequential_sum": [_vp, _dp, C.c_size_t, _dp],
    "gl_simulate_scans": [_vp, _vp, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, _dp, _dp, _dp],
    "gl_tensor_argmax_candidate": [_vp, _vp, C.c_double, _dp, C.POINTER(C.c_int64), _dp],
    "gl_engine_create": [_ip, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, _u8p, C.c_int,
                         C.c_int, _pvp],
    "gl_engine_destroy": [_vp],
    "gl_engine_info": [_vp, _ip, _ip, _ip],
    "gl_engine_context": [_vp, C.c_int, _pvp],
    "gl_engine_set_kernels": [_vp, C.c_int, _vp],
    "gl_engine_init_uniform": [_vp],
    "gl_engine_step": [_vp, C.c_double, C.c_double, C.c_double, C.c_int],
    "gl_engine_step_async": [_vp, C.c_double, C.c_double, C.c_double, C.c_int],
    "gl_engine_status": [_vp],
    "gl_engine_argmax": [_vp, C.POINTER(PoseEstimateC)],
    "gl_engine_belief_map": [_vp, _dp],
    "gl_engine_observe": [_vp, C.c_int, _dp, _dp, C.c_int, C.c_double, LikelihoodC, _ip, C.c_int, _ip, _dp],
    "gl_engine_download": [_vp, _dp, _dp],
    "gl_engine_upload": [_vp, _dp, C.c_double],
    "gl_engine_hash": [_vp, C.POINTER(C.c_uint64)],
}

GL_ENGINE_AUTO, GL_ENGINE_NCCL, GL_ENGINE_P2P = 0, 1, 2

_lib = None


def load():
    """Load libgridloc_b200.so (raises if absent: no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the gridloc_b200 product has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    # a library built from an older tree (GRIDLOC_B200_LIB, tuning
    # experiments only) may lack newer entry points; the product must not
    experimental = "GRIDLOC_B200_LIB" in os.environ
    for name, args in SIGNATURES.items():
        if experimental and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.gl_last_error.restype = C.c_char_p
    lib.gl_version.restype = C.c_char_p
    _lib = lib
    return lib


class GridlocError(RuntimeError):
    code = GL_E_RUNTIME


class BeliefExtinguishedError(GridlocError):
    """gridloc::BeliefExtinguishedError (belief_tensor.hpp:22-25)."""
    code = GL_E_EXTINGUISHED


class MapParseError(GridlocError):
    """gridloc::MapParseError (occupancy_map.hpp:22-30)."""
    code = GL_E_MAP_PARSE


class CudaError(GridlocError):
    code = GL_E_CUDA


def check(rc: int):
    if rc == GL_OK:
        return
    msg = _lib.gl_last_error().decode()
    if rc == GL_E_EXTINGUISHED:
        raise BeliefExtinguishedError(msg)
    if rc == GL_E_INVALID:
        raise ValueError(msg)
    if rc == GL_E_MAP_PARSE:
        raise MapParseError(msg)
    if rc == GL_E_CUDA:
        raise CudaError(msg)
    raise GridlocError(msg)

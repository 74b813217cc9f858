"""ctypes binding of libvol.so (include/vol.h).  Argument marshalling only: every step of the method
runs in the library's CUDA kernels.  There is no CPU fallback: if the library is missing this module
raises on import of the binding."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HVG_LIBVOL") or os.path.join(_HERE, "libvol.so")  # override: experiments only

VOL_OK, VOL_EINVAL, VOL_EDATA, VOL_ENOMEM, VOL_ECUDA, VOL_ENCCL, VOL_ENOTSUP = range(7)
_NAMES = {1: "EINVAL", 2: "EDATA", 3: "ENOMEM", 4: "ECUDA", 5: "ENCCL", 6: "ENOTSUP"}


class VolError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"VOL_{_NAMES.get(status, status)}: {msg}")
        self.status = status


class vol_opts(ctypes.Structure):
    _fields_ = [("theta", ctypes.c_float), ("data_term", ctypes.c_int), ("init", ctypes.c_int),
                ("resume", ctypes.c_int), ("kernel", ctypes.c_int), ("freeze", ctypes.c_int),
                ("exchange", ctypes.c_int)]


class vol_camera(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_float), ("fy", ctypes.c_float), ("cx", ctypes.c_float), ("cy", ctypes.c_float),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class vol_fusion_params(ctypes.Structure):
    _fields_ = [("voxel", ctypes.c_float), ("mu", ctypes.c_float), ("max_range", ctypes.c_float),
                ("w_max", ctypes.c_float)]


class vol_fusion_stats(ctypes.Structure):
    _fields_ = [("pixels_valid", ctypes.c_int64), ("blocks", ctypes.c_int64), ("block_frames", ctypes.c_int64),
                ("voxel_updates", ctypes.c_int64), ("ms_alloc", ctypes.c_float), ("ms_integrate", ctypes.c_float)]


class vol_stereo_params(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32), ("n_disp", ctypes.c_int32),
                ("window", ctypes.c_int32), ("outer", ctypes.c_int32), ("inner", ctypes.c_int32),
                ("lam", ctypes.c_float), ("alpha1", ctypes.c_float), ("alpha2", ctypes.c_float),
                ("beta", ctypes.c_float), ("gamma", ctypes.c_float), ("theta0", ctypes.c_float),
                ("theta_end", ctypes.c_float), ("tau", ctypes.c_float), ("sigma", ctypes.c_float)]


class vol_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("world", ctypes.c_int), ("part", ctypes.c_void_p),
                ("nccl_id", ctypes.c_void_p)]


EXPORTS = [
    "vol_default_opts", "vol_workspace_bytes", "vol_create", "vol_regularise", "vol_read_u", "vol_energy",
    "vol_read_state", "vol_load_state", "vol_read_tables", "vol_info", "vol_last_launches", "vol_sync",
    "vol_destroy", "vol_last_error", "vol_nccl_unique_id", "vol_group_connect", "vol_regularise_group",
    "vol_group_energy", "vol_block_hash", "vol_plan_shard", "vol_total_launches", "vol_fuse_workspace_bytes",
    "vol_fuse", "vol_fuse_incremental", "vol_extract", "vol_stereo_default_params", "vol_stereo_workspace_bytes", "vol_stereo",
    "vol_stereo_census", "vol_stereo_tensor", "vol_disparity_to_depth", "vol_shard_timing", "vol_create_w8",
    "vol_partition_route", "vol_release_comms", "vol_peer_info", "vol_connect_peer", "vol_ipc_handle",
    "vol_connect_peer_ipc", "vol_transport",
]

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built: run `python -m paper_1604_03734_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, i64, i32, u32, f32, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_float, ctypes.c_int
    st = ctypes.c_int
    sig = {
        "vol_default_opts": (None, [ctypes.POINTER(vol_opts)]),
        "vol_workspace_bytes": (ctypes.c_size_t, [P, i64, ctypes.POINTER(vol_dist)]),
        "vol_create": (st, [P, i64, P, P, ctypes.POINTER(vol_dist), P, ctypes.c_size_t, P, ctypes.POINTER(P)]),
        "vol_create_w8": (st, [P, i64, P, P, ctypes.POINTER(vol_dist), P, ctypes.c_size_t, P, ctypes.POINTER(P)]),
        "vol_regularise": (st, [P, f32, f32, f32, f32, i32, ctypes.POINTER(vol_opts)]),
        "vol_read_u": (st, [P, P]),
        "vol_energy": (st, [P, f32, f32, c_int, P, P]),
        "vol_read_state": (st, [P, P, P, P]),
        "vol_load_state": (st, [P, P, P, P]),
        "vol_read_tables": (st, [P, P, P, P, P]),
        "vol_info": (st, [P, P, P, P]),
        "vol_last_launches": (i64, [P]),
        "vol_sync": (st, [P]),
        "vol_destroy": (None, [P]),
        "vol_last_error": (ctypes.c_char_p, []),
        "vol_nccl_unique_id": (st, [P]),
        "vol_group_connect": (st, [P, c_int]),
        "vol_regularise_group": (st, [P, c_int, f32, f32, f32, f32, i32, ctypes.POINTER(vol_opts)]),
        "vol_group_energy": (st, [P, c_int, f32, f32, c_int, P, P]),
        "vol_block_hash": (u32, [i32, i32, i32, u32]),
        "vol_plan_shard": (st, [P, i64, P, c_int, c_int, P, P, P, P, P, P, P]),
        "vol_total_launches": (i64, []),
        "vol_partition_route": (st, [P, i64, P, i32, ctypes.c_double, c_int, P, P]),
        "vol_release_comms": (st, []),
        "vol_peer_info": (st, [P, P, i64, P]),
        "vol_connect_peer": (st, [P, c_int, P, P, i64]),
        "vol_ipc_handle": (st, [P, P, P]),
        "vol_connect_peer_ipc": (st, [P, c_int, P, i64, P, i64]),
        "vol_transport": (c_int, [P]),
        "vol_shard_timing": (st, [P, P, P, P]),
        "vol_extract": (st, [P, c_int, f32, f32, P, i64, P]),
        "vol_fuse_incremental": (st, [P, P, P, i64, P, i32, ctypes.POINTER(vol_camera), P,
                                      ctypes.POINTER(vol_fusion_params), i64, P, ctypes.c_size_t, P, P, P, P, P, P,
                                      ctypes.POINTER(vol_fusion_stats)]),
        "vol_stereo_default_params": (None, [ctypes.POINTER(vol_stereo_params)]),
        "vol_stereo_workspace_bytes": (ctypes.c_size_t, [i32, ctypes.POINTER(vol_stereo_params)]),
        "vol_stereo": (st, [P, P, i32, ctypes.POINTER(vol_stereo_params), P, ctypes.c_size_t, P, P, P, P]),
        "vol_stereo_census": (st, [P, i32, i32, i32, i32, P, P]),
        "vol_stereo_tensor": (st, [P, i32, i32, i32, f32, f32, P, P]),
        "vol_disparity_to_depth": (st, [P, i64, f32, f32, P, P]),
        "vol_fuse_workspace_bytes": (ctypes.c_size_t, [i64, i32, ctypes.POINTER(vol_camera)]),
        "vol_fuse": (st, [P, i32, ctypes.POINTER(vol_camera), P, ctypes.POINTER(vol_fusion_params), i64, P,
                          ctypes.c_size_t, P, P, P, P, P, P, ctypes.POINTER(vol_fusion_stats)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(status: int):
    if status != VOL_OK:
        raise VolError(status, lib().vol_last_error().decode(errors="replace"))

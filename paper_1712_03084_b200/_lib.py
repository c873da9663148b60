# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of the C-ABI in include/vc/vc.h (libvc_b200.so, in-tree).

There is no CPU fallback: importing works without a GPU (for the ABI checks),
but every compute entry point goes through the CUDA library and raises
VcError when it is missing or when no device is present.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.path.join(PKG_DIR, "libvc_b200.so")
HEADER_PATH = os.path.join(REPO_DIR, "include", "vc", "vc.h")

VC_OK, VC_ERR_INVALID_ARGUMENT, VC_ERR_EMPTY_SCENE, VC_ERR_CAPACITY = 0, 1, 2, 3
VC_ERR_CUDA, VC_ERR_NCCL, VC_ERR_OOM, VC_ERR_NO_DEVICE, VC_ERR_RUNTIME = 4, 5, 6, 7, 8
VC_MEM_HOST, VC_MEM_DEVICE = 0, 1


class VcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"vc status {status}: {msg}")
        self.status = status


class VcInvalidArgument(VcError, ValueError):
    """std::invalid_argument in the reference."""


class VcEmptyScene(VcError):
    """std::runtime_error("empty foreground in all views") in the reference."""


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class Pose(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3)]


class Sensor(C.Structure):
    _fields_ = [("depth_intr", Intrinsics), ("pose", Pose), ("rgb_intr", Intrinsics), ("rgb_relative", Pose)]


class View(C.Structure):
    _fields_ = [("depth", C.c_void_p), ("mask", C.c_void_p), ("rgb", C.c_void_p), ("depth_pitch", C.c_int32),
                ("mask_pitch", C.c_int32), ("rgb_pitch", C.c_int32), ("mem_kind", C.c_int32)]


class ReconConfig(C.Structure):
    _fields_ = [("r", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("mode", C.c_int32),
                ("discontinuity_mm", C.c_double), ("padding_voxels", C.c_int32),
                ("silhouette_radius_px", C.c_int32), ("eps_vis_mm", C.c_double)]


class GridSpec(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("origin", C.c_double * 3),
                ("edge_mm", C.c_double)]


class StageTimings(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("raw_ms", "weights_ms", "volumetric_ms", "texture_ms", "total_ms",
                                          "splat_ms", "fft_ms", "iso_ms", "mc_ms", "h2d_ms", "d2h_ms")]


class TexturedMesh(C.Structure):
    _fields_ = [("vertex_count", C.c_int32), ("triangle_count", C.c_int32), ("sensor_count", C.c_int32),
                ("point_count", C.c_int32), ("positions", C.c_void_p), ("normals", C.c_void_p),
                ("triangles", C.c_void_p), ("visible", C.c_void_p), ("uv", C.c_void_p), ("weight", C.c_void_p),
                ("untextured", C.c_void_p), ("rgb", C.c_void_p), ("positions_f64", C.c_void_p),
                ("iso_level", C.c_double), ("grid", GridSpec), ("mem_kind", C.c_int32)]


class DistInfo(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("rank", "world", "z_begin", "z_end", "vertex_offset", "vertex_total",
                                         "triangle_offset", "triangle_total")]


class PngHeader(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("width", "height", "bit_depth", "color_type")]


class Wms3imOptions(C.Structure):
    _fields_ = [("scales", C.c_int32), ("alpha", C.c_double * 3), ("beta", C.c_double * 3), ("gamma", C.c_double * 3),
                ("c1", C.c_double), ("c2", C.c_double), ("c3", C.c_double), ("window", C.c_int32),
                ("sigma", C.c_double)]


class Body(C.Structure):
    _fields_ = [("joints", C.c_double * 45), ("radii", C.c_double * 14), ("colors", C.c_uint8 * 42)]


_lib = None


def header_functions() -> list[str]:
    """Every function the C-ABI header declares."""
    src = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\*]+\s+)+\**(vc_\w+)\s*\(", src, re.M)))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise VcError(VC_ERR_NO_DEVICE, f"CUDA library missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.vc_status_string.restype = C.c_char_p
        L.vc_last_error.restype = C.c_char_p
        L.vc_last_error.argtypes = [P]
        L.vc_io_last_error.restype = C.c_char_p
        L.vc_ctx_stream.restype = P
        L.vc_ctx_stream.argtypes = [P]
        L.vc_ctx_kernels_per_frame.argtypes = [P]
        for name in header_functions():
            fn = getattr(L, name)
            if fn.restype is C.c_int and name not in ("vc_abi_version", "vc_ctx_kernels_per_frame"):
                fn.restype = C.c_int
        _lib = L
    return _lib


def check(status: int, ctx=None) -> None:
    if status == VC_OK:
        return
    L = lib()
    msg = L.vc_last_error(ctx).decode() if ctx else L.vc_status_string(status).decode()
    if status == VC_ERR_INVALID_ARGUMENT:
        raise VcInvalidArgument(status, msg)
    if status == VC_ERR_EMPTY_SCENE:
        raise VcEmptyScene(status, msg)
    raise VcError(status, msg)

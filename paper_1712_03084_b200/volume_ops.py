"""(A, L) consumers — Python face of csrc/k_binary.cu and
csrc/vc_volume.cpp, mirroring mocap/volume_ops.hpp:

  binarize(volume, grid, level)   binary_volume.cpp:10-66 (GPU union-find CCL)
  binarize_frame(ctx, out)        the same on the context's last frame volume (no copy)
  boundary_voxels(bv)             binary_volume.cpp:68-82
  skeletonize(bv)                 skeletonize.cpp:99-161 (GPU: simple-point table, re-check fixed point)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .volcap import Context, GridSpec, default_context


@dataclass
class BinaryVolume:  # volume_ops.hpp:13-20
    grid: np.ndarray     # (nz, ny, nx) uint8
    voxels: np.ndarray   # (n, 3) int32 (x, y, z), raster order
    spec: GridSpec

    def voxel_world(self, q) -> np.ndarray:
        return np.asarray(self.spec.origin) + self.spec.edge_mm * np.asarray(q, np.float64)


def _binarize(ctx, A_ptr, kind, spec: GridSpec, level: float) -> BinaryVolume:
    keep = np.zeros((spec.nz, spec.ny, spec.nx), np.uint8)
    n = C.c_int64()
    g = spec.to_c()
    # size query, then the voxel list
    ctx._check(L.lib().vc_binarize(ctx.handle, A_ptr, kind, C.byref(g), C.c_double(level),
                                   keep.ctypes.data_as(C.c_void_p), None, C.c_int64(0), C.byref(n)))
    vox = np.zeros((max(n.value, 1), 3), np.int32)
    ctx._check(L.lib().vc_binarize(ctx.handle, A_ptr, kind, C.byref(g), C.c_double(level), None,
                                   vox.ctypes.data_as(C.c_void_p), C.c_int64(n.value), C.byref(n)))
    return BinaryVolume(keep, vox[:n.value], spec)


def binarize(volume, spec: GridSpec, level: float, ctx: Context | None = None) -> BinaryVolume:
    ctx = ctx or default_context()
    A = np.ascontiguousarray(volume, np.float32)
    return _binarize(ctx, A.ctypes.data_as(C.c_void_p), L.VC_MEM_HOST, spec, level)


def binarize_frame(ctx: Context, spec: GridSpec, level: float) -> BinaryVolume:
    """On the volume of the context's last vc_reconstruct_frame (stays on the GPU)."""
    return _binarize(ctx, None, L.VC_MEM_DEVICE, spec, level)


def boundary_voxels(bv: BinaryVolume, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    keep = np.ascontiguousarray(bv.grid, np.uint8)
    vox = np.ascontiguousarray(bv.voxels, np.int32)
    out = np.zeros((max(len(vox), 1), 3))
    n = C.c_int64()
    ctx._check(L.lib().vc_boundary_voxels(ctx.handle, keep.ctypes.data_as(C.c_void_p), C.byref(bv.spec.to_c()),
                                          vox.ctypes.data_as(C.c_void_p), C.c_int64(len(vox)),
                                          out.ctypes.data_as(C.c_void_p), C.byref(n)))
    return out[:n.value]


def skeletonize(bv: BinaryVolume, ctx=None) -> np.ndarray:
    ctx = ctx or default_context()
    g = np.ascontiguousarray(bv.grid, np.uint8)
    vox = np.ascontiguousarray(bv.voxels, np.int32)
    out = np.zeros((max(len(vox), 1), 3), np.int32)
    n = C.c_int64()
    ctx._check(L.lib().vc_skeletonize(ctx.handle, g.ctypes.data_as(C.c_void_p), g.shape[2], g.shape[1], g.shape[0],
                                      vox.ctypes.data_as(C.c_void_p), C.c_int64(len(vox)),
                                      out.ctypes.data_as(C.c_void_p), C.byref(n)))
    return out[:n.value]

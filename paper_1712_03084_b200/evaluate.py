"""Evaluation renderer and metrics — Python face of
csrc/k_raster.cu, csrc/k_metrics.cu and csrc/vc_eval.cpp, mirroring eval/:

  rasterize(tm, camera, view_images, mode)   rasterize.cpp:35-161
  vre, hausdorff2d, distance_transform        metrics.cpp:12-43, distance_transform.cpp
  cp_rmse(ground, reconstructed)              metrics.cpp:86-94
  wms3im(rendered, ground, silhouette, opt)   ssim.cpp:159-176
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .volcap import Context, TexturedMesh, default_context

UV_BLEND, COLOR_PER_VERTEX = 0, 1


@dataclass
class RenderedView:  # rasterize.hpp
    depth: np.ndarray       # (h, w) float32, 0 = empty
    color: np.ndarray       # (h, w, 3) uint8
    silhouette: np.ndarray  # (h, w) uint8


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def rasterize(tm: TexturedMesh, intr: L.Intrinsics, pose: L.Pose, view_images, mode=UV_BLEND,
              ctx: Context | None = None) -> RenderedView:
    ctx = ctx or default_context()
    intr = intr.to_c() if hasattr(intr, "to_c") else intr
    pose = pose.to_c() if hasattr(pose, "to_c") else pose
    w, h = intr.width, intr.height
    V = np.ascontiguousarray(tm.mesh.vertices, np.float64)
    T = np.ascontiguousarray(tm.mesh.triangles, np.int32)
    k = tm.sensor_count
    vis = np.ascontiguousarray(tm.visible, np.uint8)
    uv = np.ascontiguousarray(tm.uv, np.float32)
    wt = np.ascontiguousarray(tm.weight, np.float32)
    imgs = [np.ascontiguousarray(im, np.uint8) for im in view_images[:k]]
    ptrs = (C.c_void_p * max(k, 1))(*[im.ctypes.data for im in imgs])
    iw = (C.c_int32 * max(k, 1))(*[im.shape[1] for im in imgs])
    ih = (C.c_int32 * max(k, 1))(*[im.shape[0] for im in imgs])
    depth = np.zeros((h, w), np.float32)
    color = np.zeros((h, w, 3), np.uint8)
    sil = np.zeros((h, w), np.uint8)
    ctx._check(L.lib().vc_rasterize(ctx.handle, _p(V), len(V), _p(T), len(T), k, _p(vis), _p(uv), _p(wt),
                                    C.byref(intr), C.byref(pose), ptrs, iw, ih, mode, _p(depth), _p(color), _p(sil)))
    return RenderedView(depth, color, sil)


def vre(rendered, ground, ctx: Context | None = None) -> float:
    ctx = ctx or default_context()
    a, b = np.ascontiguousarray(rendered, np.uint8), np.ascontiguousarray(ground, np.uint8)
    if a.shape != b.shape:
        raise ValueError("vre: mask dimensions differ")
    out = C.c_double()
    ctx._check(L.lib().vc_vre(ctx.handle, _p(a), _p(b), a.shape[1], a.shape[0], C.byref(out)))
    return out.value


def distance_transform(mask, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    m = np.ascontiguousarray(mask, np.uint8)
    out = np.zeros(m.shape, np.float32)
    ctx._check(L.lib().vc_distance_transform(ctx.handle, _p(m), m.shape[1], m.shape[0], _p(out)))
    return out


def hausdorff2d(rendered, ground, ctx: Context | None = None) -> float | None:
    ctx = ctx or default_context()
    a, b = np.ascontiguousarray(rendered, np.uint8), np.ascontiguousarray(ground, np.uint8)
    if a.shape != b.shape:
        raise ValueError("hausdorff2d: mask dimensions differ")
    out, has = C.c_double(), C.c_int32()
    ctx._check(L.lib().vc_hausdorff2d(ctx.handle, _p(a), _p(b), a.shape[1], a.shape[0], C.byref(out), C.byref(has)))
    return out.value if has.value else None


def cp_rmse(ground, reconstructed, ctx: Context | None = None) -> float:
    ctx = ctx or default_context()
    g = np.ascontiguousarray(ground, np.float64).reshape(-1, 3)
    r = np.ascontiguousarray(reconstructed, np.float64).reshape(-1, 3)
    out = C.c_double()
    ctx._check(L.lib().vc_cp_rmse(ctx.handle, _p(g), len(g), _p(r), len(r), C.byref(out)))
    return out.value


def wms3im(rendered, ground, silhouette, opt: L.Wms3imOptions | None = None, ctx: Context | None = None):
    ctx = ctx or default_context()
    a = np.ascontiguousarray(rendered, np.uint8)
    b = np.ascontiguousarray(ground, np.uint8)
    m = np.ascontiguousarray(silhouette, np.uint8)
    if a.shape != b.shape or a.shape[:2] != m.shape:
        raise ValueError("wms3im: image dimensions differ")
    out, has = C.c_double(), C.c_int32()
    ctx._check(L.lib().vc_wms3im(ctx.handle, _p(a), _p(b), _p(m), a.shape[1], a.shape[0],
                                 C.byref(opt) if opt is not None else None, C.byref(out), C.byref(has)))
    return out.value if has.value else None

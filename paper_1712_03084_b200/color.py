"""Colour correction — Python face of csrc/k_color.cu
and csrc/vc_color.cpp, mirroring appearance/color.hpp:

  ValueMap, ColorCorrection.apply(sensor, image)  color.hpp:50-88, color_correction.cpp:140-160
  mutual_closest_pairs(a, b, max_dist)            color_correction.cpp:16-84 (GPU hash grid)
  accumulate_color_pairs(...)                     color_correction.cpp:86-95
  fit_value_map(pairs, options)                   color_correction.cpp:97-138
  chain_to_reference(edges, reference, n)         color_correction.cpp:168-199
  set_frame_color_correction(ctx, cc)             the corrected images of sequence.cpp:71-73,
                                                  fused into the frame's texture sampling
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .volcap import Context, OrientedClouds, default_context


def _err(status: int) -> None:
    """std::invalid_argument -> VcInvalidArgument (a ValueError); the reference's
    std::runtime_error (VC_ERR_RUNTIME) -> VcError (a RuntimeError)."""
    if status == L.VC_OK:
        return
    msg = L.lib().vc_io_last_error().decode()
    if status == L.VC_ERR_INVALID_ARGUMENT:
        raise L.VcInvalidArgument(status, msg)
    raise L.VcError(status, msg)


@dataclass
class ValueMap:  # color.hpp:50-57
    gain: float = 1.0
    offset: float = 0.0

    def apply(self, v: float) -> float:
        return min(max(self.gain * v + self.offset, 0.0), 1.0)

    def then(self, outer: "ValueMap") -> "ValueMap":  # outer(this(v))
        return ValueMap(outer.gain * self.gain, outer.gain * self.offset + outer.offset)

    def inverse(self) -> "ValueMap":
        return ValueMap(1.0 / self.gain, -self.offset / self.gain)


@dataclass
class ValueFitOptions:  # color.hpp:59-63
    ransac_iterations: int = 1000
    inlier_threshold: float = 0.05
    seed: int = 1


@dataclass
class PairwiseValueMap:
    frm: int
    to: int
    map: ValueMap


@dataclass
class ColorCorrection:  # color.hpp:77-85
    maps: list = field(default_factory=list)
    reference: int = 0

    @staticmethod
    def identity(sensor_count: int, reference: int = 0) -> "ColorCorrection":
        return ColorCorrection([ValueMap() for _ in range(sensor_count)], reference)

    def apply(self, sensor: int, image: np.ndarray, ctx: Context | None = None) -> np.ndarray:
        """ColorCorrection::apply(sensor, image) on the GPU."""
        ctx = ctx or default_context()
        m = self.maps[sensor]
        img = np.ascontiguousarray(image, np.uint8)
        out = np.empty_like(img)
        ctx._check(L.lib().vc_color_apply(ctx.handle, img.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p),
                                          C.c_int64(img.size // 3), C.c_double(m.gain), C.c_double(m.offset),
                                          L.VC_MEM_HOST))
        return out


def mutual_closest_pairs(a, b, max_dist_mm: float = 20.0, ctx: Context | None = None) -> list[tuple[int, int]]:
    ctx = ctx or default_context()
    pa = np.ascontiguousarray(a, np.float64).reshape(-1, 3)
    pb = np.ascontiguousarray(b, np.float64).reshape(-1, 3)
    out = np.zeros((max(1, min(len(pa), len(pb))), 2), np.int32)
    n = C.c_int32()
    ctx._check(L.lib().vc_mutual_closest_pairs(ctx.handle, pa.ctypes.data_as(C.c_void_p), len(pa),
                                               pb.ctypes.data_as(C.c_void_p), len(pb), C.c_double(max_dist_mm),
                                               out.ctypes.data_as(C.c_void_p), C.byref(n)))
    return [(int(i), int(j)) for i, j in out[:n.value]]


def accumulate_color_pairs(cloud_a: OrientedClouds, image_a, cloud_b: OrientedClouds, image_b, pairs: list,
                           max_dist_mm: float = 20.0, ctx: Context | None = None) -> None:
    """Appends (colour in view a, colour in view b) of the mutual closest points (:86-95)."""
    for i, j in mutual_closest_pairs(cloud_a.position, cloud_b.position, max_dist_mm, ctx):
        pairs.append((np.asarray(image_a)[cloud_a.py[i], cloud_a.px[i]].copy(),
                      np.asarray(image_b)[cloud_b.py[j], cloud_b.px[j]].copy()))


def fit_value_map(pairs, options: ValueFitOptions = ValueFitOptions()) -> ValueMap:
    """pairs: [(rgb_a, rgb_b)] -> ValueMap with V_b ~ gain * V_a + offset."""
    arr = np.ascontiguousarray(np.array([np.concatenate([np.asarray(p, np.uint8), np.asarray(q, np.uint8)])
                                         for p, q in pairs], np.uint8).reshape(-1, 6))
    g, o = C.c_double(), C.c_double()
    _err(L.lib().vc_fit_value_map(arr.ctypes.data_as(C.c_void_p), len(pairs), options.ransac_iterations,
                                  C.c_double(options.inlier_threshold), C.c_uint64(options.seed), C.byref(g),
                                  C.byref(o)))
    return ValueMap(g.value, o.value)


def chain_to_reference(edges: list[PairwiseValueMap], reference: int, sensor_count: int) -> ColorCorrection:
    n = len(edges)
    frm = (C.c_int32 * max(n, 1))(*[e.frm for e in edges])
    to = (C.c_int32 * max(n, 1))(*[e.to for e in edges])
    g = (C.c_double * max(n, 1))(*[e.map.gain for e in edges])
    o = (C.c_double * max(n, 1))(*[e.map.offset for e in edges])
    og, oo = (C.c_double * sensor_count)(), (C.c_double * sensor_count)()
    _err(L.lib().vc_chain_to_reference(frm, to, g, o, n, reference, sensor_count, og, oo))
    return ColorCorrection([ValueMap(og[k], oo[k]) for k in range(sensor_count)], reference)


def set_frame_color_correction(ctx: Context, cc: ColorCorrection | None) -> None:
    """Per-sensor maps applied to the texels the frame's colour blend samples (None: off)."""
    k = 0 if cc is None else len(cc.maps)
    g = (C.c_double * max(k, 1))(*([m.gain for m in cc.maps] if cc else []))
    o = (C.c_double * max(k, 1))(*([m.offset for m in cc.maps] if cc else []))
    ctx._check(L.lib().vc_ctx_set_color_correction(ctx.handle, g, o, k))

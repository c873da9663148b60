# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE — ctypes wrapper of the REFERENCE's own code
(oracle/_ref/o<order>/libref.so, built by `make -C oracle ref` from the
unmodified sources under /root/reference/proj/core against oracle/ref_shim).

Used only by tests/ to pin the oracle restatement to the reference.  The
library exists only where /root/reference was present at build time (this
container, and GPU boxes that received the built _ref/ via gpurun); tests skip
when it is absent.  Results mirror oracle.oracle.FrameResult so the two can be
compared field by field.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import oracle as O

_HERE = os.path.dirname(os.path.abspath(__file__))
_libs: dict[int, C.CDLL] = {}


def lib_path(order: int = 0) -> str:
    return os.path.join(_HERE, "_ref", f"o{order}", "libref.so")


def available(order: int = 0) -> bool:
    return os.path.exists(lib_path(order))


def lib(order: int = 0) -> C.CDLL:
    if order not in _libs:
        L = C.CDLL(lib_path(order))
        L.ref_reconstruct_frame.restype = C.c_void_p
        L.ref_marching_cubes.restype = C.c_void_p
        for fn in ("ref_frame_free", "ref_frame_sizes", "ref_frame_points", "ref_frame_weight_map", "ref_frame_grid",
                   "ref_frame_volume", "ref_frame_mesh", "ref_frame_texture"):
            getattr(L, fn).argtypes = None
        assert L.ref_sizeof_sensor() == C.sizeof(O.Sensor)
        assert L.ref_sizeof_body() == C.sizeof(O.Body)
        _libs[order] = L
    return _libs[order]


def _p(a):
    return C.c_void_p(a.ctypes.data)


def make_circle_rig(recon, held_out=0, radius_mm=2500.0, target_height_mm=1000.0, width=320, height=288,
                    focal_px=300.0, order=0):
    arr = (O.Sensor * (recon + held_out))()
    lib(order).ref_make_circle_rig(recon, held_out, C.c_double(radius_mm), C.c_double(target_height_mm), width,
                                   height, C.c_double(focal_px), arr)
    return arr


def body(kick_frames=0, frame=0, order=0) -> O.Body:
    """make_xpose_body() (kick_frames=0) or make_kick_sequence(kick_frames)[frame]."""
    b = O.Body()
    lib(order).ref_body(kick_frames, frame, C.byref(b))
    return b


def render_frame(sensor, b, camera=0, frame=0, sigma_mm_at_2m=0.0, seed=1, gain=1.0, order=0) -> O.RenderedView:
    w, h = sensor.depth_intr.width, sensor.depth_intr.height
    rw, rh = sensor.rgb_intr.width, sensor.rgb_intr.height
    depth = np.zeros((h, w), np.uint16)
    mask = np.zeros((h, w), np.uint8)
    rgb = np.zeros((rh, rw, 3), np.uint8)
    lib(order).ref_render_frame(C.byref(sensor), C.byref(b), C.c_double(sigma_mm_at_2m), C.c_uint64(seed),
                                C.c_double(gain), camera, frame, _p(depth), _p(mask), _p(rgb))
    return O.RenderedView(depth, mask, rgb)


def reconstruct_frame(sensors, depths, masks, rgbs=None, dims=None, r=0, mode=0, discontinuity_mm=50.0,
                      padding_voxels=8, silhouette_radius_px=10, eps_vis_mm=20.0, want_volume=True,
                      order=0) -> O.FrameResult:
    """r > 0: the reference's reconstruct_frame (reconstruct.cpp:37-78) unmodified;
    dims: the same stages with fit_grid's per-axis rule on `dims`."""
    L = lib(order)
    k = len(depths)
    depths = [np.ascontiguousarray(d, np.uint16) for d in depths]
    masks = [np.ascontiguousarray(m, np.uint8) for m in masks]
    rgbs = None if rgbs is None else [np.ascontiguousarray(x, np.uint8) for x in rgbs]
    d = np.ascontiguousarray(dims if dims is not None else (0, 0, 0), np.int32)
    st = C.c_int()
    arr = lambda xs: (C.c_void_p * len(xs))(*[x.ctypes.data for x in xs])  # noqa: E731
    h = C.c_void_p(L.ref_reconstruct_frame(sensors, k, arr(depths), arr(masks), arr(rgbs) if rgbs else None, r,
                                           _p(d), mode, C.c_double(discontinuity_mm), padding_voxels,
                                           silhouette_radius_px, C.c_double(eps_vis_mm), C.byref(st)))
    try:
        res = O.FrameResult(st.value, {})
        if st.value != 0:
            return res
        sz = np.zeros(4, np.int64)
        L.ref_frame_sizes(h, _p(sz))
        P, V, T, _ = (int(x) for x in sz)
        pos = np.zeros((P, 3)); nrm = np.zeros((P, 3)); wt = np.zeros(P); pix = np.zeros((P, 3), np.int32)
        L.ref_frame_points(h, _p(pos), _p(nrm), _p(wt), _p(pix))
        res.points = dict(position=pos, normal=nrm, weight=wt, px=pix[:, 0], py=pix[:, 1], sensor=pix[:, 2])
        res.weight_maps = []
        for i in range(k):
            wm = np.zeros((sensors[i].depth_intr.height, sensors[i].depth_intr.width), np.float32)
            L.ref_frame_weight_map(h, i, _p(wm))
            res.weight_maps.append(wm)
        g = O.GridSpec(); lvl = C.c_double()
        L.ref_frame_grid(h, C.byref(g), C.byref(lvl))
        res.grid, res.iso_level = g, lvl.value
        if want_volume:
            A = np.zeros((g.nz, g.ny, g.nx))
            L.ref_frame_volume(h, _p(A))
            res.volume = A
        verts = np.zeros((V, 3)); vn = np.zeros((V, 3)); tris = np.zeros((T, 3), np.int32)
        L.ref_frame_mesh(h, _p(verts), _p(vn), _p(tris))
        res.mesh = O.Mesh(verts, vn, tris, None)  # the reference does not report edge ids
        res.vis = np.zeros((k, V), np.uint8); res.uv = np.zeros((k, V, 2)); res.weight = np.zeros((k, V), np.float32)
        res.untextured = np.zeros(V, np.uint8)
        L.ref_frame_texture(h, _p(res.vis), _p(res.uv), _p(res.weight), _p(res.untextured))
        return res
    finally:
        L.ref_frame_free(h)


def marching_cubes(A, g: O.GridSpec, level: float, order=0):
    """marching_cubes.cpp:131-210 -> (vertices, normals, triangles) in first-touch order."""
    L = lib(order)
    A = np.ascontiguousarray(A, np.float64)
    n = np.zeros(2, np.int64)
    h = C.c_void_p(L.ref_marching_cubes(_p(A), C.byref(g), C.c_double(level), _p(n)))
    try:
        V, T = int(n[0]), int(n[1])
        verts = np.zeros((V, 3)); vn = np.zeros((V, 3)); tris = np.zeros((T, 3), np.int32)
        L.ref_frame_mesh(h, _p(verts), _p(vn), _p(tris))
        return verts, vn, tris
    finally:
        L.ref_frame_free(h)


def skeletonize(keep, voxels, order=0) -> np.ndarray:
    """mocap::skeletonize (skeletonize.cpp:99-161) on keep[z, y, x] and an (n, 3) voxel list."""
    L = lib(order)
    g = np.ascontiguousarray(keep, np.uint8)
    vox = np.ascontiguousarray(voxels, np.int32).reshape(-1, 3)
    out = np.zeros((max(len(vox), 1), 3), np.int32)
    L.ref_skeletonize.restype = C.c_int64
    n = L.ref_skeletonize(_p(g), g.shape[2], g.shape[1], g.shape[0], _p(vox), C.c_int64(len(vox)), _p(out))
    return out[:n]


def fit_value_map(pairs_rgb, iterations=1000, threshold=0.05, seed=1, order=0):
    """appearance::fit_value_map (color_correction.cpp:97-138): (gain, offset), or
    RuntimeError with the reference's message when it throws."""
    L = lib(order)
    arr = np.ascontiguousarray(pairs_rgb, np.uint8).reshape(-1, 6)
    g, o = C.c_double(), C.c_double()
    err = C.create_string_buffer(256)
    st = L.ref_fit_value_map(_p(arr), len(arr), iterations, C.c_double(threshold), C.c_uint64(seed), C.byref(g),
                             C.byref(o), err, 256)
    if st:
        raise RuntimeError(err.value.decode())
    return g.value, o.value


def chain_to_reference(edges, reference, sensor_count, order=0):
    """appearance::chain_to_reference (color_correction.cpp:168-199); edges = [(from, to, gain, offset)];
    None when the reference throws (a sensor not connected)."""
    L = lib(order)
    f = np.array([e[0] for e in edges], np.int32)
    t = np.array([e[1] for e in edges], np.int32)
    g = np.array([e[2] for e in edges], np.float64)
    o = np.array([e[3] for e in edges], np.float64)
    og = np.zeros(sensor_count)
    oo = np.zeros(sensor_count)
    st = L.ref_chain_to_reference(_p(f), _p(t), _p(g), _p(o), len(edges), reference, sensor_count, _p(og), _p(oo))
    return None if st else list(zip(og.tolist(), oo.tolist()))

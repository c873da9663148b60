# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE — ctypes wrapper of the CPU oracle (liborc.so).

The oracle is a C++ restatement of the reference FTR path (see oracle.hpp).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc.so")


def build(force: bool = False) -> str:
    """Compile liborc.so with the committed Makefile (g++ only)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class Pose(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3)]


class Sensor(C.Structure):
    _fields_ = [("depth_intr", Intrinsics), ("pose", Pose), ("rgb_intr", Intrinsics),
                ("rgb_relative", Pose)]


class GridSpec(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("origin", C.c_double * 3), ("edge", C.c_double)]


class Body(C.Structure):
    _fields_ = [("joints", C.c_double * 45), ("radii", C.c_double * 14), ("colors", C.c_uint8 * 42)]


class ReconConfig(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("mode", C.c_int32),
                ("discontinuity_mm", C.c_double), ("padding_voxels", C.c_int32),
                ("silhouette_radius_px", C.c_int32), ("eps_vis_mm", C.c_double),
                ("threads", C.c_int32)]


class Timings(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("raw_ms", "weights_ms", "volumetric_ms", "other_ms", "blend_ms",
                                          "splat_ms", "integrate_ms", "iso_ms", "mc_ms")]


_lib = None
_P = C.c_void_p


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        L.orc_build_cloud.restype = _P
        L.orc_marching_cubes.restype = _P
        L.orc_reconstruct_frame.restype = _P
        L.orc_frame_mesh.restype = _P
        L.orc_frame_mesh.argtypes = [_P]
        L.orc_cloud_size.restype = C.c_int64
        L.orc_cloud_size.argtypes = [_P]
        L.orc_frame_point_count.restype = C.c_int64
        L.orc_frame_point_count.argtypes = [_P]
        L.orc_sdf.restype = C.c_double
        for fn in ("orc_cloud_free", "orc_mesh_free", "orc_frame_free"):
            getattr(L, fn).argtypes = [_P]
        assert L.orc_sizeof_sensor() == C.sizeof(Sensor)
        assert L.orc_sizeof_body() == C.sizeof(Body)
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> C.c_void_p:
    assert a.flags["C_CONTIGUOUS"]
    return C.c_void_p(a.ctypes.data)


def _ptr_array(arrs) -> C.Array:
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


# ------------------------------------------------------------------ synth
def make_circle_rig(recon, held_out=0, radius_mm=2500.0, target_height_mm=1000.0,
                    width=320, height=288, focal_px=300.0):
    """scene.cpp:24-55 (make_scene fixes the target height at 1000 mm, scene.cpp:72)."""
    n = recon + held_out
    arr = (Sensor * n)()
    lib().orc_make_circle_rig(recon, held_out, C.c_double(radius_mm), C.c_double(target_height_mm),
                              width, height, C.c_double(focal_px), arr)
    return arr


def xpose_body() -> Body:
    b = Body()
    lib().orc_make_xpose_body(C.byref(b))
    return b


def kick_body(frames: int, f: int) -> Body:
    b = Body()
    lib().orc_make_kick_body(frames, f, C.byref(b))
    return b


@dataclass
class RenderedView:
    depth: np.ndarray  # (h, w) uint16 mm
    mask: np.ndarray   # (h, w) uint8
    rgb: np.ndarray    # (rh, rw, 3) uint8


def render_frame(sensor: Sensor, body: Body, camera: int = 0, frame: int = 0, sigma_mm_at_2m: float = 0.0,
                 seed: int = 1, gain: float = 1.0, threads: int = 0) -> RenderedView:
    """render.cpp:23-80."""
    w, h = sensor.depth_intr.width, sensor.depth_intr.height
    rw, rh = sensor.rgb_intr.width, sensor.rgb_intr.height
    depth = np.zeros((h, w), np.uint16)
    mask = np.zeros((h, w), np.uint8)
    rgb = np.zeros((rh, rw, 3), np.uint8)
    lib().orc_render_frame(C.byref(sensor), C.byref(body), C.c_double(sigma_mm_at_2m), C.c_uint64(seed),
                           C.c_double(gain), camera, frame, threads or os.cpu_count(), _ptr(depth), _ptr(mask),
                           _ptr(rgb))
    return RenderedView(depth, mask, rgb)


def sample_surface(body: Body, count: int, seed: int) -> np.ndarray:
    out = np.zeros((count, 3), np.float64)
    n = lib().orc_sample_surface(C.byref(body), count, C.c_uint64(seed), _ptr(out))
    return out[:n]


def sdf(body: Body, x) -> float:
    x = np.ascontiguousarray(x, np.float64)
    return lib().orc_sdf(C.byref(body), _ptr(x))


# ------------------------------------------------------------------ recon stages
@dataclass
class Cloud:
    position: np.ndarray
    normal: np.ndarray
    weight: np.ndarray
    px: np.ndarray
    py: np.ndarray
    weight_map: np.ndarray


def build_cloud(depth, mask, sensor: Sensor, sensor_index=0, discontinuity_mm=50.0,
                confidence=False, silhouette_radius_px=10, override_normal=None) -> Cloud:
    """cloud.cpp:19-83 (+ confidence_weights cloud.cpp:85-117 when confidence=True)."""
    depth = np.ascontiguousarray(depth, np.uint16)
    mask = np.ascontiguousarray(mask, np.uint8)
    h, w = depth.shape
    L = lib()
    c = L.orc_build_cloud(_ptr(depth), _ptr(mask), w, h, C.byref(sensor), sensor_index,
                          C.c_double(discontinuity_mm))
    try:
        if override_normal is not None:
            n0 = L.orc_cloud_size(c)
            nn = np.ascontiguousarray(np.broadcast_to(np.asarray(override_normal, np.float64), (n0, 3)))
            L.orc_cloud_set_normals(C.c_void_p(c), _ptr(nn))
        if confidence:
            L.orc_confidence_weights(C.c_void_p(c), _ptr(mask), w, h, C.byref(sensor), silhouette_radius_px)
        n = L.orc_cloud_size(c)
        pos = np.zeros((n, 3)); nrm = np.zeros((n, 3)); wt = np.zeros(n)
        px = np.zeros(n, np.int32); py = np.zeros(n, np.int32); wm = np.zeros((h, w), np.float32)
        L.orc_cloud_get(C.c_void_p(c), _ptr(pos), _ptr(nrm), _ptr(wt), _ptr(px), _ptr(py), _ptr(wm))
    finally:
        L.orc_cloud_free(c)
    return Cloud(pos, nrm, wt, px, py, wm)


def fit_grid(lo, hi, dims, padding_voxels=8) -> GridSpec:
    g = GridSpec()
    lo = np.ascontiguousarray(lo, np.float64); hi = np.ascontiguousarray(hi, np.float64)
    d = np.ascontiguousarray(dims, np.int32)
    if lib().orc_fit_grid(_ptr(lo), _ptr(hi), _ptr(d), padding_voxels, C.byref(g)) != 0:
        raise ValueError("fit_grid: padding leaves no usable voxels")
    return g


def grid(nx, ny, nz, origin=(0.0, 0.0, 0.0), edge=1.0) -> GridSpec:
    g = GridSpec()
    g.nx, g.ny, g.nz = nx, ny, nz
    for i in range(3):
        g.origin[i] = origin[i]
    g.edge = edge
    return g


def splat(pos, nrm, weight, g: GridSpec, mode=0, threads=0):
    """splat.cpp:33-89 -> (field (nz,ny,nx,3), density (nz,ny,nx), (sigma1, sigma2))."""
    pos = np.ascontiguousarray(pos, np.float64).reshape(-1, 3)
    nrm = np.ascontiguousarray(nrm, np.float64).reshape(-1, 3)
    weight = np.ascontiguousarray(weight, np.float64).reshape(-1)
    field = np.zeros((g.nz, g.ny, g.nx, 3)); dens = np.zeros((g.nz, g.ny, g.nx)); sig = np.zeros(2)
    lib().orc_splat(_ptr(pos), _ptr(nrm), _ptr(weight), C.c_int64(len(pos)), C.byref(g), mode, threads,
                    _ptr(field), _ptr(dens), _ptr(sig))
    return field, dens, (sig[0], sig[1])


def integrate_fft(field) -> np.ndarray:
    """integrate.cpp:19-74. field: (nz,ny,nx,3) float64 -> A (nz,ny,nx)."""
    field = np.ascontiguousarray(field, np.float64)
    nz, ny, nx, _ = field.shape
    out = np.zeros((nz, ny, nx))
    lib().orc_integrate_fft(_ptr(field), nx, ny, nz, _ptr(out))
    return out


def iso_level(A, g: GridSpec, pos) -> float:
    A = np.ascontiguousarray(A, np.float64)
    pos = np.ascontiguousarray(pos, np.float64).reshape(-1, 3)
    lvl = C.c_double()
    if lib().orc_iso_level(_ptr(A), C.byref(g), _ptr(pos), C.c_int64(len(pos)), C.byref(lvl)) != 0:
        raise ValueError("iso_level: no input samples")
    return lvl.value


@dataclass
class Mesh:
    vertices: np.ndarray
    normals: np.ndarray
    triangles: np.ndarray
    edge_ids: np.ndarray


def _mesh_from_handle(h) -> Mesh:
    L = lib()
    V = C.c_int64(); T = C.c_int64()
    L.orc_mesh_counts(C.c_void_p(h), C.byref(V), C.byref(T))
    v = np.zeros((V.value, 3)); n = np.zeros((V.value, 3)); t = np.zeros((T.value, 3), np.int32)
    e = np.zeros(V.value, np.uint64)
    L.orc_mesh_get(C.c_void_p(h), _ptr(v), _ptr(n), _ptr(t), _ptr(e))
    return Mesh(v, n, t, e)


def marching_cubes(A, g: GridSpec, level: float) -> Mesh:
    """marching_cubes.cpp:131-210 (vertices in first-touch order + global edge ids)."""
    A = np.ascontiguousarray(A, np.float64)
    h = lib().orc_marching_cubes(_ptr(A), C.byref(g), C.c_double(level))
    try:
        return _mesh_from_handle(h)
    finally:
        lib().orc_mesh_free(C.c_void_p(h))


def case_table():
    counts = np.zeros(256, np.int32); tris = np.zeros((256, 5, 3), np.int32)
    lib().orc_case_table(_ptr(counts), _ptr(tris))
    return counts, tris


def vertex_visibility(verts, sensors, depths, masks, eps_vis_mm=20.0) -> np.ndarray:
    verts = np.ascontiguousarray(verts, np.float64).reshape(-1, 3)
    k = len(depths)
    depths = [np.ascontiguousarray(d, np.uint16) for d in depths]
    masks = [np.ascontiguousarray(m, np.uint8) for m in masks]
    vis = np.zeros((k, len(verts)), np.uint8)
    lib().orc_vertex_visibility(_ptr(verts), C.c_int64(len(verts)), sensors, _ptr_array(depths),
                                _ptr_array(masks), k, C.c_double(eps_vis_mm), _ptr(vis))
    return vis


def assign_texture(verts, sensors, weight_maps, vis):
    verts = np.ascontiguousarray(verts, np.float64).reshape(-1, 3)
    k = len(weight_maps)
    wms = [np.ascontiguousarray(w, np.float32) for w in weight_maps]
    vis = np.ascontiguousarray(vis, np.uint8)
    V = len(verts)
    uv = np.zeros((k, V, 2)); w = np.zeros((k, V), np.float32); un = np.zeros(V, np.uint8)
    lib().orc_assign_texture(_ptr(verts), C.c_int64(V), sensors, _ptr_array(wms), k, _ptr(vis), _ptr(uv),
                             _ptr(w), _ptr(un))
    return uv, w, un


def blend_colors(vis, uv, w, rgbs):
    vis = np.ascontiguousarray(vis, np.uint8); uv = np.ascontiguousarray(uv, np.float64)
    w = np.ascontiguousarray(w, np.float32)
    k, V = vis.shape
    rgbs = [np.ascontiguousarray(r, np.uint8) for r in rgbs]
    wh = np.array([[r.shape[1], r.shape[0]] for r in rgbs], np.int32)
    color = np.zeros((V, 3)); rgb8 = np.zeros((V, 3), np.uint8)
    lib().orc_blend_colors(C.c_int64(V), k, _ptr(vis), _ptr(uv), _ptr(w), _ptr_array(rgbs), _ptr(wh),
                           _ptr(color), _ptr(rgb8))
    return color, rgb8


# ------------------------------------------------------------------ full frame
@dataclass
class FrameResult:
    status: int
    timings: dict
    points: dict | None = None
    weight_maps: list | None = None
    grid: GridSpec | None = None
    iso_level: float = 0.0
    volume: np.ndarray | None = None
    mesh: Mesh | None = None
    vis: np.ndarray | None = None
    uv: np.ndarray | None = None
    weight: np.ndarray | None = None
    untextured: np.ndarray | None = None
    color: np.ndarray | None = None
    rgb8: np.ndarray | None = None


def reconstruct_frame(sensors, depths, masks, rgbs=None, dims=(128, 128, 128), mode=0, discontinuity_mm=50.0,
                      padding_voxels=8, silhouette_radius_px=10, eps_vis_mm=20.0, threads=0,
                      want_volume=True) -> FrameResult:
    """reconstruct.cpp:37-78 + texture.cpp:11-72 + A14 blend, with run_bench's stage timings."""
    k = len(depths)
    depths = [np.ascontiguousarray(d, np.uint16) for d in depths]
    masks = [np.ascontiguousarray(m, np.uint8) for m in masks]
    rgbs = None if rgbs is None else [np.ascontiguousarray(r, np.uint8) for r in rgbs]
    cfg = ReconConfig(dims[0], dims[1], dims[2], mode, discontinuity_mm, padding_voxels, silhouette_radius_px,
                      eps_vis_mm, threads)
    tm = Timings(); st = C.c_int()
    L = lib()
    h = L.orc_reconstruct_frame(sensors, k, _ptr_array(depths), _ptr_array(masks),
                                _ptr_array(rgbs) if rgbs else None, C.byref(cfg), C.byref(tm), C.byref(st))
    try:
        timings = {n: getattr(tm, n) for n, _ in Timings._fields_}
        res = FrameResult(st.value, timings)
        if st.value != 0:
            return res
        n = L.orc_frame_point_count(h)
        pos = np.zeros((n, 3)); nrm = np.zeros((n, 3)); wt = np.zeros(n); pix = np.zeros((n, 3), np.int32)
        L.orc_frame_points(C.c_void_p(h), _ptr(pos), _ptr(nrm), _ptr(wt), _ptr(pix))
        res.points = dict(position=pos, normal=nrm, weight=wt, px=pix[:, 0], py=pix[:, 1], sensor=pix[:, 2])
        res.weight_maps = []
        for i in range(k):
            wm = np.zeros((sensors[i].depth_intr.height, sensors[i].depth_intr.width), np.float32)
            L.orc_frame_weight_map(C.c_void_p(h), i, _ptr(wm))
            res.weight_maps.append(wm)
        g = GridSpec(); lvl = C.c_double()
        L.orc_frame_grid(C.c_void_p(h), C.byref(g), C.byref(lvl))
        res.grid, res.iso_level = g, lvl.value
        if want_volume:
            A = np.zeros((g.nz, g.ny, g.nx))
            L.orc_frame_volume(C.c_void_p(h), _ptr(A))
            res.volume = A
        res.mesh = _mesh_from_handle(L.orc_frame_mesh(h))
        V = len(res.mesh.vertices)
        res.vis = np.zeros((k, V), np.uint8); res.uv = np.zeros((k, V, 2)); res.weight = np.zeros((k, V), np.float32)
        res.untextured = np.zeros(V, np.uint8); res.color = np.zeros((V, 3)); res.rgb8 = np.zeros((V, 3), np.uint8)
        L.orc_frame_texture(C.c_void_p(h), _ptr(res.vis), _ptr(res.uv), _ptr(res.weight), _ptr(res.untextured),
                            _ptr(res.color), _ptr(res.rgb8))
        return res
    finally:
        L.orc_frame_free(h)


# ------------------------------------------------------------------ mesh helpers (mesh.cpp:39-70)
def analyze_topology(triangles: np.ndarray, n_vertices: int):
    t = np.asarray(triangles, np.int64)
    if len(t) == 0:
        return dict(edge_manifold=False, V=n_vertices, E=0, F=0, euler=n_vertices)
    e = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
    e.sort(axis=1)
    key = e[:, 0] * (1 << 32) + e[:, 1]
    uniq, counts = np.unique(key, return_counts=True)
    E = len(uniq)
    return dict(edge_manifold=bool(np.all(counts == 2)), V=n_vertices, E=E, F=len(t),
                euler=n_vertices - E + len(t))


def surface_area(vertices, triangles) -> float:
    v = np.asarray(vertices, np.float64); t = np.asarray(triangles, np.int64)
    if len(t) == 0:
        return 0.0
    e1 = v[t[:, 1]] - v[t[:, 0]]; e2 = v[t[:, 2]] - v[t[:, 0]]
    return float(0.5 * np.linalg.norm(np.cross(e1, e2), axis=1).sum())

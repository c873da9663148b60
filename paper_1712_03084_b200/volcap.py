# SPDX-License-Identifier: Apache-2.0
"""Host-side mirror of the reference's proj/core reconstruction interface.

Same names, argument meaning and error behaviour as
/root/reference/proj/core/include/volcap/{core/types.hpp, recon/*.hpp,
appearance/texture.hpp}, implemented over the C-ABI (include/vc/vc.h) of the
B200 CUDA library.  Errors: std::invalid_argument -> ValueError
(VcInvalidArgument), runtime_error("empty foreground") -> VcEmptyScene.

    rig = make_circle_rig(4, 0, 2500, 512, 424, 365)
    frames = [render_frame(rig, body, k) for k in range(4)]
    rec = reconstruct_frame(frames, rig, ReconConfig(dims=(256, 256, 256)))
    rec.mesh.vertices, rec.textured.visible, rec.textured.rgb, rec.volume.iso_level
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from ._lib import VcEmptyScene, VcError, VcInvalidArgument  # noqa: F401


# ------------------------------------------------------------------ core types (types.hpp)
@dataclass
class Intrinsics:  # types.hpp:26-39
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def to_c(self) -> L.Intrinsics:
        return L.Intrinsics(self.fx, self.fy, self.cx, self.cy, self.width, self.height)


@dataclass
class Pose:  # types.hpp:42-57 — camera-to-world: X_w = R X_c + t
    R: np.ndarray = field(default_factory=lambda: np.eye(3))
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def apply(self, x):
        return self.R @ np.asarray(x, float) + self.t

    def apply_inverse(self, x):
        return self.R.T @ (np.asarray(x, float) - self.t)

    def inverse(self) -> "Pose":
        return Pose(self.R.T.copy(), -(self.R.T @ self.t))

    def compose(self, rhs: "Pose") -> "Pose":
        return Pose(self.R @ rhs.R, self.R @ rhs.t + self.t)

    def to_c(self) -> L.Pose:
        p = L.Pose()
        for i, v in enumerate(np.asarray(self.R, float).ravel()):
            p.R[i] = v
        for i, v in enumerate(np.asarray(self.t, float).ravel()):
            p.t[i] = v
        return p


@dataclass
class Sensor:  # types.hpp:68-76
    depth_intr: Intrinsics
    pose: Pose
    rgb_intr: Intrinsics
    rgb_relative: Pose = field(default_factory=Pose)

    def to_c(self) -> L.Sensor:
        return L.Sensor(self.depth_intr.to_c(), self.pose.to_c(), self.rgb_intr.to_c(), self.rgb_relative.to_c())

    @staticmethod
    def from_c(s: L.Sensor) -> "Sensor":
        def intr(i):
            return Intrinsics(i.fx, i.fy, i.cx, i.cy, i.width, i.height)

        def pose(p):
            return Pose(np.array(p.R[:]).reshape(3, 3), np.array(p.t[:]))
        return Sensor(intr(s.depth_intr), pose(s.pose), intr(s.rgb_intr), pose(s.rgb_relative))


@dataclass
class CameraRig:  # types.hpp:80-99
    sensors: list
    recon_count: int

    def count(self) -> int:
        return len(self.sensors)

    def c_array(self, k=None):
        k = len(self.sensors) if k is None else k
        arr = (L.Sensor * k)()
        for i in range(k):
            arr[i] = self.sensors[i].to_c()
        return arr


@dataclass
class RgbdFrame:  # image.hpp:50-64
    depth: np.ndarray       # (h, w) uint16 mm, 0 = invalid
    color: np.ndarray       # (rh, rw, 3) uint8
    foreground: np.ndarray | None  # (h, w) uint8; None = depth > 0 (derived on the device)


@dataclass
class ReconConfig:  # reconstruct.hpp:12-18 (+ dims for cubic grids, eps_vis)
    r: int = 7
    mode: str = "weighted"  # or "simple"
    discontinuity_mm: float = 50.0
    padding_voxels: int = 8
    silhouette_radius_px: int = 10
    dims: tuple | None = None  # (nx, ny, nz) overrides r
    eps_vis_mm: float = 20.0

    def to_c(self) -> L.ReconConfig:
        if self.mode not in ("weighted", "simple"):
            raise ValueError(f"unknown splat mode {self.mode!r}")
        nx, ny, nz = self.dims if self.dims else (0, 0, 0)
        return L.ReconConfig(0 if self.dims else self.r, nx, ny, nz, 0 if self.mode == "weighted" else 1,
                             self.discontinuity_mm, self.padding_voxels, self.silhouette_radius_px, self.eps_vis_mm)


@dataclass
class GridSpec:  # volume_recon.hpp:24-28
    nx: int
    ny: int
    nz: int
    origin: np.ndarray
    edge_mm: float

    def to_c(self) -> L.GridSpec:
        g = L.GridSpec()
        g.nx, g.ny, g.nz = self.nx, self.ny, self.nz
        for i in range(3):
            g.origin[i] = float(self.origin[i])
        g.edge_mm = self.edge_mm
        return g

    @staticmethod
    def from_c(g: L.GridSpec) -> "GridSpec":
        return GridSpec(g.nx, g.ny, g.nz, np.array(g.origin[:]), g.edge_mm)


@dataclass
class TriMesh:  # mesh.hpp:20-34
    vertices: np.ndarray
    normals: np.ndarray
    triangles: np.ndarray
    edge_ids: np.ndarray | None = None


@dataclass
class TexturedMesh:  # texture.hpp:16-28 (+ blended per-vertex colour)
    mesh: TriMesh
    sensor_count: int
    visible: np.ndarray     # [K][V] uint8
    uv: np.ndarray          # [K][V][2] float32
    weight: np.ndarray      # [K][V] float32
    untextured: np.ndarray  # [V] uint8
    rgb: np.ndarray | None = None  # [V][3] uint8


@dataclass
class OrientedClouds:  # cloud.hpp:13-26, concatenated in sensor order
    position: np.ndarray
    normal: np.ndarray
    weight: np.ndarray
    px: np.ndarray
    py: np.ndarray
    sensor: np.ndarray
    weight_maps: list


@dataclass
class ImplicitVolume:  # volume_recon.hpp:38-41
    values: np.ndarray | None
    iso_level: float
    grid: GridSpec


@dataclass
class StageTimings:  # reconstruct.hpp:20-24 + texture + split
    raw_ms: float = 0.0
    weights_ms: float = 0.0
    volumetric_ms: float = 0.0
    texture_ms: float = 0.0
    total_ms: float = 0.0
    splat_ms: float = 0.0
    fft_ms: float = 0.0
    iso_ms: float = 0.0
    mc_ms: float = 0.0
    h2d_ms: float = 0.0
    d2h_ms: float = 0.0


@dataclass
class FrameReconstruction:  # reconstruct.hpp:26-30 + the textured mesh
    clouds: OrientedClouds | None
    volume: ImplicitVolume
    mesh: TriMesh
    textured: TexturedMesh


# ------------------------------------------------------------------ context
class Context:
    """One CUDA device + stream (vc_ctx).  Not thread-safe; one per thread/GPU."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        L.check(L.lib().vc_ctx_create(device, C.byref(self._h)))
        self.device = device

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            L.lib().vc_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, s):
        L.check(s, self._h)

    def set_output(self, device: bool):
        self._check(L.lib().vc_ctx_set_output(self._h, L.VC_MEM_DEVICE if device else L.VC_MEM_HOST))

    def set_graphs(self, on: bool):
        self._check(L.lib().vc_ctx_set_graphs(self._h, 1 if on else 0))

    def set_profiling(self, on: bool):
        self._check(L.lib().vc_ctx_set_profiling(self._h, 1 if on else 0))

    def set_depth_filter(self, erode_px: int = 0, sigma_px: float = 0.0, sigma_mm: float = 0.0):
        """Optional erosion/bilateral filter of every staged view (north_star
        preprocessing; the reference has none, so it stays off by default)."""
        self._check(L.lib().vc_ctx_set_depth_filter(self._h, int(erode_px), C.c_double(sigma_px),
                                                    C.c_double(sigma_mm)))

    def kernels_per_frame(self) -> int:
        return L.lib().vc_ctx_kernels_per_frame(self._h)

    def stream(self) -> int:
        return L.lib().vc_ctx_stream(self._h) or 0


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _views(frames, k):
    keep, arr = [], (L.View * k)()
    for i in range(k):
        f = frames[i]
        d = np.ascontiguousarray(f.depth, np.uint16)
        # no foreground: the library derives it on the device as depth > 0 (dataset.cpp:99-102)
        m = None if f.foreground is None else np.ascontiguousarray(f.foreground, np.uint8)
        c = None if f.color is None else np.ascontiguousarray(f.color, np.uint8)
        keep += [d, m, c]
        arr[i] = L.View(_ptr(d), _ptr(m) if m is not None else None, _ptr(c) if c is not None else None, 0, 0, 0,
                        L.VC_MEM_HOST)
    return arr, keep


def _np(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dtype))), shape=(n,)).copy()


# ------------------------------------------------------------------ hot path
def reconstruct_frame(frames, rig: CameraRig, config: ReconConfig, timings: StageTimings | None = None,
                      ctx: Context | None = None, want_volume=False, want_clouds=False) -> FrameReconstruction:
    """reconstruct.cpp:37-78 + vertex_visibility/assign_texture (texture.cpp:11-72) + per-vertex blend."""
    if len(frames) != rig.recon_count:  # reconstruct.cpp:39-40
        raise VcInvalidArgument(L.VC_ERR_INVALID_ARGUMENT,
                                "reconstruct_frame: one frame per reconstruction sensor required")
    ctx = ctx or default_context()
    k = rig.recon_count
    sensors = rig.c_array(k)
    views, _keep = _views(frames, k)
    out = L.TexturedMesh()
    tm = L.StageTimings()
    ctx._check(L.lib().vc_reconstruct_frame(ctx.handle, sensors, views, k, C.byref(config.to_c()), C.byref(out),
                                            C.byref(tm) if timings is not None else None))
    if timings is not None:
        for n, _ in L.StageTimings._fields_:
            setattr(timings, n, getattr(tm, n))
    V, T = out.vertex_count, out.triangle_count
    if out.mem_kind != L.VC_MEM_HOST:
        raise VcError(L.VC_ERR_INVALID_ARGUMENT, "reconstruct_frame() wrapper needs host output")
    mesh = TriMesh(_np(out.positions_f64, 3 * V, np.float64).reshape(V, 3),
                   _np(out.normals, 3 * V, np.float32).reshape(V, 3).astype(np.float64),
                   _np(out.triangles, 3 * T, np.int32).reshape(T, 3))
    tex = TexturedMesh(mesh, k, _np(out.visible, k * V, np.uint8).reshape(k, V),
                       _np(out.uv, 2 * k * V, np.float32).reshape(k, V, 2),
                       _np(out.weight, k * V, np.float32).reshape(k, V),
                       _np(out.untextured, V, np.uint8), _np(out.rgb, 3 * V, np.uint8).reshape(V, 3))
    grid = GridSpec.from_c(out.grid)
    vol = ImplicitVolume(export_volume(ctx, grid) if want_volume else None, out.iso_level, grid)
    clouds = export_clouds(ctx, out.point_count, rig, k) if want_clouds else None
    return FrameReconstruction(clouds, vol, mesh, tex)


def export_volume(ctx: Context, grid: GridSpec) -> np.ndarray:
    A = np.zeros((grid.nz, grid.ny, grid.nx), np.float32)
    ctx._check(L.lib().vc_export_volume(ctx.handle, C.c_void_p(_ptr(A)), L.VC_MEM_HOST))
    return A


def export_clouds(ctx: Context, n: int, rig: CameraRig, k: int) -> OrientedClouds:
    pos = np.zeros((n, 3)); nrm = np.zeros((n, 3)); w = np.zeros(n); pix = np.zeros((n, 3), np.int32)
    sizes = [(rig.sensors[i].depth_intr.height, rig.sensors[i].depth_intr.width) for i in range(k)]
    wm = np.zeros(sum(h * w_ for h, w_ in sizes), np.float32)
    ctx._check(L.lib().vc_export_points(ctx.handle, C.c_void_p(_ptr(pos)), C.c_void_p(_ptr(nrm)),
                                        C.c_void_p(_ptr(w)), C.c_void_p(_ptr(pix)), C.c_void_p(_ptr(wm))))
    maps, o = [], 0
    for h, w_ in sizes:
        maps.append(wm[o:o + h * w_].reshape(h, w_))
        o += h * w_
    return OrientedClouds(pos, nrm, w, pix[:, 0].copy(), pix[:, 1].copy(), pix[:, 2].copy(), maps)


# ------------------------------------------------------------------ stage functions
def preprocess(frames, rig: CameraRig, config: ReconConfig, ctx: Context | None = None):
    """build_cloud + confidence_weights for all views (cloud.cpp:19-117) + bbox/fit_grid.
    Returns (OrientedClouds, GridSpec)."""
    ctx = ctx or default_context()
    k = rig.recon_count
    views, _keep = _views(frames, k)
    n = C.c_int64()
    g = L.GridSpec()
    s = L.lib().vc_stage_preprocess(ctx.handle, rig.c_array(k), views, k, C.byref(config.to_c()), C.byref(n),
                                    C.byref(g))
    clouds = export_clouds(ctx, n.value, rig, k) if s in (L.VC_OK, L.VC_ERR_EMPTY_SCENE) else None
    ctx._check(s)
    return clouds, GridSpec.from_c(g)


def fit_grid(bbox_min, bbox_max, dims, padding_voxels=8) -> GridSpec:
    """reconstruct.cpp:16-35 (dims generalised; r-mode = (2^r, 2^(r+1), 2^r))."""
    lo = np.ascontiguousarray(bbox_min, np.float64); hi = np.ascontiguousarray(bbox_max, np.float64)
    d = np.ascontiguousarray(dims, np.int32)
    g = L.GridSpec()
    L.check(L.lib().vc_fit_grid(C.c_void_p(_ptr(lo)), C.c_void_p(_ptr(hi)), C.c_void_p(_ptr(d)), padding_voxels,
                                C.byref(g)))
    return GridSpec.from_c(g)


def splat(position, normal, weight, grid: GridSpec, mode="weighted", negate=False, ctx: Context | None = None):
    """splat.cpp:33-89 -> (field (nz,ny,nx,3) float32, density (nz,ny,nx) float32)."""
    ctx = ctx or default_context()
    pos = np.ascontiguousarray(position, np.float64).reshape(-1, 3)
    nrm = np.ascontiguousarray(normal, np.float64).reshape(-1, 3)
    w = None if weight is None else np.ascontiguousarray(weight, np.float64).reshape(-1)
    field_ = np.zeros((grid.nz, grid.ny, grid.nx, 3), np.float32)
    dens = np.zeros((grid.nz, grid.ny, grid.nx), np.float32)
    ctx._check(L.lib().vc_stage_splat(ctx.handle, C.c_void_p(_ptr(pos)), C.c_void_p(_ptr(nrm)),
                                      C.c_void_p(_ptr(w)) if w is not None else None, C.c_int64(len(pos)),
                                      C.byref(grid.to_c()), 0 if mode == "weighted" else 1, 1 if negate else 0,
                                      C.c_void_p(_ptr(field_)), C.c_void_p(_ptr(dens))))
    return field_, dens


def integrate_fft(field_, ctx: Context | None = None) -> np.ndarray:
    """integrate.cpp:19-74: (nz,ny,nx,3) gradient field -> A (nz,ny,nx) float32."""
    ctx = ctx or default_context()
    f = np.ascontiguousarray(field_, np.float32)
    nz, ny, nx, _ = f.shape
    A = np.zeros((nz, ny, nx), np.float32)
    ctx._check(L.lib().vc_stage_integrate(ctx.handle, C.c_void_p(_ptr(f)), nx, ny, nz, C.c_void_p(_ptr(A))))
    return A


def iso_level(volume, grid: GridSpec, positions, ctx: Context | None = None) -> float:
    """splat.cpp:91-101."""
    ctx = ctx or default_context()
    A = np.ascontiguousarray(volume, np.float32)
    pos = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
    lvl = C.c_double()
    ctx._check(L.lib().vc_stage_iso_level(ctx.handle, C.c_void_p(_ptr(A)), C.byref(grid.to_c()),
                                          C.c_void_p(_ptr(pos)), C.c_int64(len(pos)), C.byref(lvl)))
    return lvl.value


def marching_cubes(volume, grid: GridSpec, level: float, ctx: Context | None = None) -> TriMesh:
    """marching_cubes.cpp:131-210 (vertices in global-edge-id order)."""
    ctx = ctx or default_context()
    A = np.ascontiguousarray(volume, np.float32)
    V = C.c_int32(); T = C.c_int32()
    pp, pn, pt, pe = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
    ctx._check(L.lib().vc_stage_marching_cubes(ctx.handle, C.c_void_p(_ptr(A)), C.byref(grid.to_c()),
                                               C.c_double(level), C.byref(V), C.byref(T), C.byref(pp), C.byref(pn),
                                               C.byref(pt), C.byref(pe)))
    v, t = V.value, T.value
    return TriMesh(_np(pp, 3 * v, np.float64).reshape(v, 3), _np(pn, 3 * v, np.float32).reshape(v, 3),
                   _np(pt, 3 * t, np.int32).reshape(t, 3), _np(pe, v, np.uint64))


def texture(vertices, rig: CameraRig, frames, weight_maps, eps_vis_mm=20.0, ctx: Context | None = None):
    """vertex_visibility + assign_texture + blend (texture.cpp:11-72) -> TexturedMesh fields."""
    ctx = ctx or default_context()
    k = rig.recon_count
    verts = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
    V = len(verts)
    views, _keep = _views(frames, k)
    wm = np.ascontiguousarray(np.concatenate([np.asarray(w, np.float32).ravel() for w in weight_maps]))
    vis = np.zeros((k, V), np.uint8); uv = np.zeros((k, V, 2), np.float32); w = np.zeros((k, V), np.float32)
    un = np.zeros(V, np.uint8); rgb = np.zeros((V, 3), np.uint8)
    ctx._check(L.lib().vc_stage_texture(ctx.handle, rig.c_array(k), views, C.c_void_p(_ptr(wm)), k,
                                        C.c_void_p(_ptr(verts)) if V else None, V, C.c_double(eps_vis_mm),
                                        C.c_void_p(_ptr(vis)), C.c_void_p(_ptr(uv)), C.c_void_p(_ptr(w)),
                                        C.c_void_p(_ptr(un)), C.c_void_p(_ptr(rgb))))
    return TexturedMesh(TriMesh(verts, np.zeros((0, 3)), np.zeros((0, 3), np.int32)), k, vis, uv, w, un, rgb)


def vertex_visibility(mesh: TriMesh, rig: CameraRig, frames, eps_vis_mm=20.0, ctx: Context | None = None):
    """texture.cpp:11-34 -> [K][V] uint8."""
    dummy = [np.zeros((f.depth.shape[0], f.depth.shape[1]), np.float32) for f in frames[:rig.recon_count]]
    return texture(mesh.vertices, rig, frames, dummy, eps_vis_mm, ctx).visible


def assign_texture(mesh: TriMesh, rig: CameraRig, frames, clouds: OrientedClouds, visibility=None,
                   eps_vis_mm=20.0, ctx: Context | None = None) -> TexturedMesh:
    """texture.cpp:36-72.  Visibility is recomputed in the same fused kernel
    (it is always vertex_visibility's output in the reference's callers)."""
    tm = texture(mesh.vertices, rig, frames, clouds.weight_maps, eps_vis_mm, ctx)
    if visibility is not None and not np.array_equal(np.asarray(visibility, np.uint8), tm.visible):
        raise VcInvalidArgument(L.VC_ERR_INVALID_ARGUMENT, "visibility does not match vertex_visibility()")
    tm.mesh = mesh
    return tm


# ------------------------------------------------------------------ synthetic capture (fixture)
def make_circle_rig(recon, held_out=0, radius_mm=2500.0, width=320, height=288, focal_px=300.0,
                    target_height_mm=1000.0) -> CameraRig:
    """scene.cpp:24-55 (make_scene's target height 1000 mm, scene.cpp:72)."""
    arr = (L.Sensor * (recon + held_out))()
    L.check(L.lib().vc_synth_circle_rig(recon, held_out, C.c_double(radius_mm), C.c_double(target_height_mm),
                                        width, height, C.c_double(focal_px), arr))
    return CameraRig([Sensor.from_c(arr[i]) for i in range(recon + held_out)], recon)


def make_hd_rig(recon=6, radius_mm=2500.0) -> CameraRig:
    """SURVEY §8(d) C3 rig: Kinect2-like depth 512x424 (f=365) on make_circle_rig's
    circle + a 1920x1080 colour camera (f=1060, cx=959.5, cy=539.5) offset 52 mm
    along x from each depth camera (Sensor::rgb_relative, types.hpp:68-76)."""
    rig = make_circle_rig(recon, 0, radius_mm, 512, 424, 365.0)
    for s in rig.sensors:
        s.rgb_intr = Intrinsics(1060.0, 1060.0, 959.5, 539.5, 1920, 1080)
        s.rgb_relative = Pose(np.eye(3), np.array([52.0, 0.0, 0.0]))
    return rig


def xpose_body() -> L.Body:
    b = L.Body()
    L.check(L.lib().vc_synth_xpose_body(C.byref(b)))
    return b


def kick_body(frames: int, frame: int) -> L.Body:
    b = L.Body()
    L.check(L.lib().vc_synth_kick_body(frames, frame, C.byref(b)))
    return b


def render_frame(rig: CameraRig, body: L.Body, camera: int, frame: int = 0, sigma_mm_at_2m=0.0, seed=1, gain=1.0,
                 ctx: Context | None = None) -> RgbdFrame:
    """render.cpp:23-80 on the GPU (noise on the host with libstdc++'s RNG)."""
    ctx = ctx or default_context()
    s = rig.sensors[camera]
    h, w = s.depth_intr.height, s.depth_intr.width
    depth = np.zeros((h, w), np.uint16); mask = np.zeros((h, w), np.uint8)
    rgb = np.zeros((s.rgb_intr.height, s.rgb_intr.width, 3), np.uint8)
    ctx._check(L.lib().vc_synth_render(ctx.handle, C.byref(s.to_c()), C.byref(body), C.c_double(sigma_mm_at_2m),
                                       C.c_uint64(seed), C.c_double(gain), camera, frame, C.c_void_p(_ptr(depth)),
                                       C.c_void_p(_ptr(mask)), C.c_void_p(_ptr(rgb)), L.VC_MEM_HOST))
    return RgbdFrame(depth, rgb, mask)


def depth_filter(depth: np.ndarray, mask: np.ndarray, erode_px: int = 0, sigma_px: float = 0.0,
                 sigma_mm: float = 0.0, ctx: "Context | None" = None):
    """vc_depth_filter on host copies of one view: (filtered depth, eroded mask)."""
    ctx = ctx or default_context()
    d = np.ascontiguousarray(depth, np.uint16).copy()
    m = np.ascontiguousarray(mask, np.uint8).copy()
    h, w = d.shape
    ctx._check(L.lib().vc_depth_filter(ctx.handle, d.ctypes.data_as(C.c_void_p), m.ctypes.data_as(C.c_void_p), w, h,
                                       L.VC_MEM_HOST, int(erode_px), C.c_double(sigma_px), C.c_double(sigma_mm)))
    return d, m

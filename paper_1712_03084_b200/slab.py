"""z-slab decomposition of one frame over P ranks.

Python face of ``vc_reconstruct_frame_dist`` (include/vc/vc.h): rank r owns
voxel planes [r*nz/P, (r+1)*nz/P); the spectral integration of
integrate.cpp:19-74 runs as local x/y passes, an all-to-all to ky-slabs, the
fused z pass and an all-to-all back; the iso level (splat.cpp:91-101) and
marching cubes (marching_cubes.cpp:131-210) run per slab with global vertex ids,
so concatenating the ranks' pieces in rank order gives the single-GPU mesh.

Two exchangers:
  * ``SlabReconstructor.nccl(world, rank, device, uid)`` — one process per GPU
    over NCCL (libnccl.so.2 loaded by the library; ``uid`` from rank 0's
    ``nccl_unique_id()``, broadcast by the caller, e.g. torch.distributed);
  * ``SlabReconstructor.loopback(world, device)`` — P virtual ranks in this
    process (one context each) stepped in lockstep with device copies: the
    single-GPU test harness of the decomposition.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .volcap import (CameraRig, Context, GridSpec, ReconConfig, TexturedMesh, TriMesh, VcError, _np, _ptr,
                     _views)


def _find_nccl() -> str | None:
    """torch's bundled libnccl (the one its NCCL backend uses), if present."""
    try:
        import nvidia.nccl  # type: ignore
        for d in nvidia.nccl.__path__:
            p = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p
    except Exception:
        pass
    return None


def nccl_unique_id() -> bytes:
    if "VC_NCCL_LIB" not in os.environ and _find_nccl():
        os.environ["VC_NCCL_LIB"] = _find_nccl()
    buf = (C.c_uint8 * 128)()
    L.check(L.lib().vc_dist_nccl_unique_id(buf))
    return bytes(buf)


@dataclass
class SlabPiece:
    """One rank's part of the frame: its vertices (global ids start at
    ``info.vertex_offset``) and triangles (global vertex ids)."""
    mesh: TriMesh
    textured: TexturedMesh
    iso_level: float
    grid: GridSpec
    info: dict


class SlabReconstructor:
    def __init__(self, handle, contexts: list[Context], world: int):
        self._h = handle
        self.contexts = contexts
        self.world = world

    @classmethod
    def loopback(cls, world: int, device: int = 0) -> "SlabReconstructor":
        ctxs = [Context(device) for _ in range(world)]
        arr = (C.c_void_p * world)(*[c.handle.value for c in ctxs])
        h = C.c_void_p()
        L.check(L.lib().vc_dist_create_loopback(arr, world, C.byref(h)))
        return cls(h, ctxs, world)

    @classmethod
    def nccl(cls, world: int, rank: int, device: int, uid: bytes) -> "SlabReconstructor":
        if "VC_NCCL_LIB" not in os.environ and _find_nccl():
            os.environ["VC_NCCL_LIB"] = _find_nccl()
        ctx = Context(device)
        h = C.c_void_p()
        ctx._check(L.lib().vc_dist_create_nccl(ctx.handle, world, rank, (C.c_uint8 * 128)(*uid), C.byref(h)))
        return cls(h, [ctx], world)

    def close(self):
        if self._h:
            L.lib().vc_dist_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reconstruct_frame(self, frames, rig: CameraRig, config: ReconConfig,
                          timings: L.StageTimings | None = None) -> list[SlabPiece]:
        """One SlabPiece per local rank (all P for loopback, 1 for NCCL)."""
        k = rig.recon_count
        if len(frames) != k:
            raise L.VcInvalidArgument(L.VC_ERR_INVALID_ARGUMENT,
                                      "reconstruct_frame: one frame per reconstruction sensor required")
        n = len(self.contexts)
        sensors = rig.c_array(k)
        views, _keep = _views(frames, k)
        outs = (L.TexturedMesh * n)()
        infos = (L.DistInfo * n)()
        L.check(L.lib().vc_reconstruct_frame_dist(self._h, sensors, views, k, C.byref(config.to_c()), outs, infos,
                                                  C.byref(timings) if timings is not None else None),
                self.contexts[0].handle)
        pieces = []
        for i in range(n):
            out, inf = outs[i], infos[i]
            if out.mem_kind != L.VC_MEM_HOST:
                raise VcError(L.VC_ERR_INVALID_ARGUMENT, "SlabReconstructor needs host output")
            V, T = out.vertex_count, out.triangle_count
            mesh = TriMesh(_np(out.positions_f64, 3 * V, np.float64).reshape(V, 3),
                           _np(out.normals, 3 * V, np.float32).reshape(V, 3).astype(np.float64),
                           _np(out.triangles, 3 * T, np.int32).reshape(T, 3))
            tex = TexturedMesh(mesh, k, _np(out.visible, k * V, np.uint8).reshape(k, V),
                               _np(out.uv, 2 * k * V, np.float32).reshape(k, V, 2),
                               _np(out.weight, k * V, np.float32).reshape(k, V),
                               _np(out.untextured, V, np.uint8), _np(out.rgb, 3 * V, np.uint8).reshape(V, 3))
            info = {f: getattr(inf, f) for f, _ in L.DistInfo._fields_}
            pieces.append(SlabPiece(mesh, tex, out.iso_level, GridSpec.from_c(out.grid), info))
        return pieces

    def export_volume(self, local_rank: int, grid: GridSpec) -> np.ndarray:
        """The owned planes of A of local rank i, (nz/P, ny, nx) fp32."""
        nzl = grid.nz // self.world
        A = np.zeros((nzl, grid.ny, grid.nx), np.float32)
        L.check(L.lib().vc_dist_export_volume(self._h, local_rank, C.c_void_p(_ptr(A)), L.VC_MEM_HOST),
                self.contexts[local_rank].handle)
        return A


def merge_pieces(pieces: list[SlabPiece]) -> tuple[TriMesh, TexturedMesh]:
    """Concatenate rank pieces (rank order) into the whole-frame mesh."""
    pieces = sorted(pieces, key=lambda p: p.info["rank"])
    V = np.concatenate([p.mesh.vertices for p in pieces])
    N = np.concatenate([p.mesh.normals for p in pieces])
    T = np.concatenate([p.mesh.triangles for p in pieces])
    mesh = TriMesh(V, N, T)
    t0 = pieces[0].textured
    tex = TexturedMesh(mesh, t0.sensor_count, np.concatenate([p.textured.visible for p in pieces], axis=1),
                       np.concatenate([p.textured.uv for p in pieces], axis=1),
                       np.concatenate([p.textured.weight for p in pieces], axis=1),
                       np.concatenate([p.textured.untextured for p in pieces]),
                       np.concatenate([p.textured.rgb for p in pieces]))
    return mesh, tex

"""Frame and mesh I/O either side of the path.

Python face of the host I/O in libvc_b200.so (csrc/vc_io.cpp), mirroring the
reference's core I/O:

  read_depth_png / read_color_png / write_png   image_io.cpp:64-122
  write_ply (TriMesh + channels)                mesh_io.cpp:104-145
  write_textured_ply (with_channels)            texture.cpp:74-91, volcap.cpp:312-316
  load_frame (frames/cam<k>/<f>_{depth,color}.png, foreground = depth > 0)
                                                dataset.cpp:25-27, 94-105

Errors raise RuntimeError("<what>: <path>") like the reference.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib as L
from .volcap import RgbdFrame, TexturedMesh, TriMesh


def _err(status: int) -> None:
    if status != L.VC_OK:
        raise RuntimeError(L.lib().vc_io_last_error().decode())


def _setup():
    lib = L.lib()
    lib.vc_io_last_error.restype = C.c_char_p
    return lib


def png_header(path) -> tuple[int, int, int, int]:
    """(width, height, bit_depth, color_type) of a PNG."""
    h = L.PngHeader()
    _err(_setup().vc_png_info(os.fsencode(path), C.byref(h)))
    return h.width, h.height, h.bit_depth, h.color_type


def read_depth_png(path) -> np.ndarray:
    w, h, _, _ = png_header(path)
    out = np.empty((h, w), np.uint16)
    _err(_setup().vc_png_read_depth(os.fsencode(path), out.ctypes.data_as(C.c_void_p), w, h))
    return out


def read_color_png(path) -> np.ndarray:
    w, h, _, _ = png_header(path)
    out = np.empty((h, w, 3), np.uint8)
    _err(_setup().vc_png_read_color(os.fsencode(path), out.ctypes.data_as(C.c_void_p), w, h))
    return out


def write_png(path, image: np.ndarray) -> None:
    """uint16 (h, w) -> 16-bit gray; uint8 (h, w, 3) -> 8-bit RGB."""
    img = np.ascontiguousarray(image)
    lib = _setup()
    if img.dtype == np.uint16 and img.ndim == 2:
        _err(lib.vc_png_write_depth(os.fsencode(path), img.ctypes.data_as(C.c_void_p), img.shape[1], img.shape[0]))
    elif img.dtype == np.uint8 and img.ndim == 3 and img.shape[2] == 3:
        _err(lib.vc_png_write_color(os.fsencode(path), img.ctypes.data_as(C.c_void_p), img.shape[1], img.shape[0]))
    else:
        raise ValueError("write_png: uint16 (h, w) depth or uint8 (h, w, 3) colour")


def write_ply(path, vertices, triangles, normals=None, channels=()) -> None:
    """mesh_io.cpp:104-145.  channels: [(name, components, float array (V, components))]."""
    xyz = np.ascontiguousarray(vertices, np.float32).reshape(-1, 3)
    tri = np.ascontiguousarray(triangles, np.int32).reshape(-1, 3)
    nrm = None if normals is None else np.ascontiguousarray(normals, np.float32).reshape(-1, 3)
    n = len(channels)
    names = (C.c_char_p * max(n, 1))(*[c[0].encode() for c in channels])
    comps = (C.c_int32 * max(n, 1))(*[int(c[1]) for c in channels])
    keep = [np.ascontiguousarray(c[2], np.float32).reshape(len(xyz), int(c[1])) for c in channels]
    data = (C.c_void_p * max(n, 1))(*[k.ctypes.data for k in keep])
    _err(_setup().vc_ply_write_mesh(os.fsencode(path), xyz.ctypes.data_as(C.c_void_p),
                                    nrm.ctypes.data_as(C.c_void_p) if nrm is not None else None, len(xyz),
                                    tri.ctypes.data_as(C.c_void_p), len(tri), names, comps, data, n))


def textured_channels(tm: TexturedMesh):
    """TexturedMesh::with_channels (texture.cpp:74-91): cam<k>_vis, cam<k>_uv, cam<k>_w, untextured."""
    ch = []
    for k in range(tm.sensor_count):
        ch.append((f"cam{k}_vis", 1, tm.visible[k].astype(np.float32)))
        ch.append((f"cam{k}_uv", 2, np.asarray(tm.uv[k], np.float32)))
        ch.append((f"cam{k}_w", 1, np.asarray(tm.weight[k], np.float32)))
    ch.append(("untextured", 1, tm.untextured.astype(np.float32)))
    return ch


def write_textured_ply(path, tm: TexturedMesh) -> None:
    """write_ply(textured.with_channels()) — the reference CLI's mesh output."""
    m: TriMesh = tm.mesh
    write_ply(path, np.asarray(m.vertices, np.float64).astype(np.float32), m.triangles,
              normals=None if m.normals is None or len(m.normals) == 0 else m.normals,
              channels=textured_channels(tm))


def cam_dir(root, camera: int) -> str:  # dataset.cpp:25-27
    return os.path.join(root, "frames", f"cam{camera}")


def load_frame(root, camera: int, frame: int) -> RgbdFrame:
    """Dataset::load_frame (dataset.cpp:94-105): foreground := depth > 0."""
    d = cam_dir(root, camera)
    depth = read_depth_png(os.path.join(d, f"{frame}_depth.png"))
    color = read_color_png(os.path.join(d, f"{frame}_color.png"))
    return RgbdFrame(depth, color, (depth > 0).astype(np.uint8))

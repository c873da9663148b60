# SPDX-License-Identifier: Apache-2.0
"""Frame / mesh I/O against the restated formats in
oracle/oracle_io.py: PNG decode of every colour type, bit depth and row filter
(image_io.cpp:84-122 transforms), PNG round trips mirroring the reference's
test_core.cpp:119-135, PLY bytes identical to mesh_io.cpp:104-145, the
textured-mesh channel set of texture.cpp:74-91, and Dataset::load_frame
(dataset.cpp:94-105).  Host code only: runs without a GPU."""
import os

import numpy as np
import pytest

from oracle import oracle_io as OI
from paper_1712_03084_b200 import io as vio
from paper_1712_03084_b200 import volcap as vc


@pytest.fixture
def tmp(tmp_path):
    return str(tmp_path)


def test_png_round_trip_like_reference(tmp):
    """test_core.cpp:119-135: random 37x21 RGB8 and 33x17 uint16 depth."""
    rng = np.random.default_rng(3)
    color = rng.integers(0, 256, (21, 37, 3), dtype=np.uint8)
    vio.write_png(os.path.join(tmp, "c.png"), color)
    assert np.array_equal(vio.read_color_png(os.path.join(tmp, "c.png")), color)
    depth = rng.integers(0, 65536, (17, 33), dtype=np.uint16)
    vio.write_png(os.path.join(tmp, "d.png"), depth)
    assert np.array_equal(vio.read_depth_png(os.path.join(tmp, "d.png")), depth)
    # our files decode identically with the restated decoder (format conformance)
    hdr, rows = OI.decode_png(open(os.path.join(tmp, "d.png"), "rb").read())
    assert np.array_equal(OI.to_depth16(hdr, rows), depth)
    hdr, rows = OI.decode_png(open(os.path.join(tmp, "c.png"), "rb").read())
    assert np.array_equal(OI.to_rgb8(hdr, rows), color)


CASES = [(0, 1), (0, 2), (0, 4), (0, 8), (0, 16), (2, 8), (2, 16), (3, 1), (3, 2), (3, 4), (3, 8), (4, 8), (4, 16),
         (6, 8), (6, 16)]


@pytest.mark.parametrize("ctype,depth", CASES)
def test_png_decode_all_types_filters(tmp, ctype, depth):
    """Every colour type / bit depth, all five row filters, split IDAT chunks."""
    rng = np.random.default_rng(ctype * 100 + depth)
    w, h = 13, 11
    ch = OI.CHANNELS[ctype]
    hi = (1 << depth) if ctype != 3 else min(1 << depth, 7)
    samples = rng.integers(0, hi, (h, w * ch))
    palette = bytes(rng.integers(0, 256, 3 * 7, dtype=np.uint8)) if ctype == 3 else None
    rows = [OI.pack_samples(samples[y], depth) for y in range(h)]
    data = OI.encode_png(rows, w, h, depth, ctype, filters=[y % 5 for y in range(h)], palette=palette,
                         idat_split=37)
    p = os.path.join(tmp, "x.png")
    open(p, "wb").write(data)
    assert vio.png_header(p) == (w, h, depth, ctype)
    hdr, dec = OI.decode_png(data)
    expect = OI.to_rgb8(hdr, dec)
    assert np.array_equal(vio.read_color_png(p), expect)
    if ctype == 0 and depth == 16:
        assert np.array_equal(vio.read_depth_png(p), samples.astype(np.uint16))
    else:
        with pytest.raises(RuntimeError, match="depth png must be 16-bit grayscale: "):
            vio.read_depth_png(p)


def test_png_errors(tmp):
    with pytest.raises(RuntimeError, match="cannot open for reading: "):
        vio.read_depth_png(os.path.join(tmp, "missing.png"))
    d = np.arange(12, dtype=np.uint16).reshape(3, 4)
    p = os.path.join(tmp, "d.png")
    vio.write_png(p, d)
    b = bytearray(open(p, "rb").read())
    b[-20] ^= 0xFF  # corrupt a chunk: CRC mismatch
    open(p, "wb").write(bytes(b))
    with pytest.raises(RuntimeError, match="png read error: "):
        vio.read_depth_png(p)


def test_ply_bytes_match_reference_writer(tmp):
    """test_core.cpp:137-166 mesh (20 vertices, normals, cam0_uv channel), byte-identical file."""
    rng = np.random.default_rng(11)
    verts = rng.uniform(-100, 100, (20, 3))
    tris = np.array([[i, i + 1, i + 2] for i in range(0, 18, 3)], np.int32)
    nrm = np.tile([0.0, 0.0, 1.0], (20, 1))
    uv = (rng.uniform(-100, 100, (20, 2)) / 100.0).astype(np.float32)
    p = os.path.join(tmp, "m.ply")
    vio.write_ply(p, verts.astype(np.float32), tris, normals=nrm, channels=[("cam0_uv", 2, uv)])
    ours = open(p, "rb").read()
    assert ours == OI.write_ply(verts, tris, nrm, [("cam0_uv", 2, uv)])
    v2, n2, ch2, t2 = OI.read_ply(ours)
    assert np.array_equal(t2, tris)
    assert ch2[0][0] == "cam0_uv" and np.array_equal(ch2[0][2], uv)
    assert np.allclose(v2, verts, atol=1e-4)
    # no normals, no channels, empty mesh
    vio.write_ply(p, verts.astype(np.float32), tris)
    assert open(p, "rb").read() == OI.write_ply(verts, tris)
    vio.write_ply(p, np.zeros((0, 3), np.float32), np.zeros((0, 3), np.int32))
    assert open(p, "rb").read() == OI.write_ply(np.zeros((0, 3)), np.zeros((0, 3)))


def test_textured_ply_channels(tmp):
    rng = np.random.default_rng(5)
    V, K = 50, 3
    mesh = vc.TriMesh(rng.normal(size=(V, 3)) * 100, rng.normal(size=(V, 3)),
                      rng.integers(0, V, (40, 3)).astype(np.int32))
    tm = vc.TexturedMesh(mesh, K, rng.integers(0, 2, (K, V)).astype(np.uint8),
                         rng.uniform(0, 1, (K, V, 2)).astype(np.float32), rng.uniform(0, 1, (K, V)).astype(np.float32),
                         rng.integers(0, 2, V).astype(np.uint8), rng.integers(0, 256, (V, 3)).astype(np.uint8))
    p = os.path.join(tmp, "t.ply")
    vio.write_textured_ply(p, tm)
    data = open(p, "rb").read()
    assert data == OI.write_ply(mesh.vertices, mesh.triangles, mesh.normals,
                                OI.with_channels(tm.visible, tm.uv, tm.weight, tm.untextured))
    _, _, ch, _ = OI.read_ply(data)
    assert [c[0] for c in ch] == ["cam0_vis", "cam0_uv", "cam0_w", "cam1_vis", "cam1_uv", "cam1_w", "cam2_vis",
                                  "cam2_uv", "cam2_w", "untextured"]


def test_load_frame_dataset_layout(tmp):
    """dataset.cpp:25-27, 94-105: frames/cam<k>/<f>_{depth,color}.png, foreground = depth > 0."""
    rng = np.random.default_rng(9)
    d = os.path.join(tmp, "frames", "cam2")
    os.makedirs(d)
    depth = rng.integers(0, 3, (24, 32)).astype(np.uint16) * 1000
    color = rng.integers(0, 256, (30, 40, 3), dtype=np.uint8)
    vio.write_png(os.path.join(d, "7_depth.png"), depth)
    vio.write_png(os.path.join(d, "7_color.png"), color)
    f = vio.load_frame(tmp, 2, 7)
    assert np.array_equal(f.depth, depth) and np.array_equal(f.color, color)
    assert np.array_equal(f.foreground, (depth > 0).astype(np.uint8))

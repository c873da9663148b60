# SPDX-License-Identifier: Apache-2.0
"""Pins the oracle's texture stage against the reference KATs
(/root/reference/proj/tests/unit/test_appearance.cpp:36-106) and the per-vertex
blend against the uv-blend KATs of test_eval_raster.cpp:112-151."""
import numpy as np
import pytest

from test_oracle_field import identity_sensor


def single_rig(O, w=64, h=48, f=60.0):
    arr = (O.Sensor * 1)()
    arr[0] = identity_sensor(O, w, h, f)
    return arr


def backproject(u, v, z, w=64, h=48, f=60.0):  # camera.cpp:12-17,23-25 with identity pose
    return np.array([(u - (w - 1) / 2.0) * z / f, (v - (h - 1) / 2.0) * z / f, z])


def flat(w=64, h=48, d=2000):
    return np.full((h, w), d, np.uint16), np.ones((h, w), np.uint8)


# test_appearance.cpp:36-43
def test_visible_vertex(O):
    rig = single_rig(O)
    d, m = flat()
    vis = O.vertex_visibility([backproject(31, 23, 2000)], rig, [d], [m])
    assert vis[0, 0] == 1


# test_appearance.cpp:45-52
def test_occluded_vertex(O):
    rig = single_rig(O)
    d, m = flat()
    vis = O.vertex_visibility([backproject(31, 23, 2100)], rig, [d], [m], 20.0)
    assert vis[0, 0] == 0


# test_appearance.cpp:54-62
def test_out_of_image(O):
    rig = single_rig(O)
    d, m = flat()
    vis = O.vertex_visibility([[100000, 0, 2000], [0, 0, -500]], rig, [d], [m])
    assert vis[0, 0] == 0 and vis[0, 1] == 0


# test_appearance.cpp:64-84
def test_assign_texture_single_view(O):
    rig = single_rig(O)
    d, m = flat()
    verts = np.array([backproject(31, 23, 2000), [0, 0, -500]])
    vis = O.vertex_visibility(verts, rig, [d], [m])
    wm = np.full((48, 64), 0.7, np.float32)
    uv, w, un = O.assign_texture(verts, rig, [wm], vis)
    assert w[0, 0] == pytest.approx(0.7)
    assert un[0] == 0
    assert w[0, 1] == 0.0 and un[1] == 1
    assert uv[0, 0, 0] == pytest.approx((31 + 0.5) / 64.0)
    assert uv[0, 0, 1] == pytest.approx((23 + 0.5) / 48.0)


def test_blend_untextured_gray(O):
    """rasterize.cpp:155-156 (test_eval_raster.cpp:112-126): no weighted view -> gray 200."""
    vis = np.zeros((1, 2), np.uint8)
    uv = np.zeros((1, 2, 2)); w = np.zeros((1, 2), np.float32)
    rgb = np.zeros((8, 8, 3), np.uint8)
    color, rgb8 = O.blend_colors(vis, uv, w, [rgb])
    assert np.all(rgb8 == 200)


def test_blend_convex_combination(O):
    """rasterize.cpp:136-157 (test_eval_raster.cpp:128-151): 0.6*200 and 0.4*100 within 2%."""
    vis = np.ones((2, 3), np.uint8)
    uv = np.full((2, 3, 2), 0.5)
    w = np.array([[0.6] * 3, [0.4] * 3], np.float32)
    views = [np.tile(np.array([200, 0, 0], np.uint8), (8, 8, 1)), np.tile(np.array([0, 100, 0], np.uint8), (8, 8, 1))]
    color, rgb8 = O.blend_colors(vis, uv, w, views)
    for v in range(3):
        # truncating cast (rasterize.cpp:152-154) of 39.9999994 -> 39: within 1/255
        assert abs(int(rgb8[v, 0]) - 120) <= 1 and abs(int(rgb8[v, 1]) - 40) <= 1
        assert rgb8[v, 2] == 0
    w6, w4 = float(np.float32(0.6)), float(np.float32(0.4))
    assert color[0, 0] == w6 * 200.0 / (w6 + w4)


def test_blend_bilinear_sample_rounding(O):
    """rasterize.cpp:12-27: UV -> pixel - 0.5, clamp, bilinear, lround to uint8."""
    img = np.zeros((2, 2, 3), np.uint8)
    img[0, 0] = [0, 0, 0]; img[0, 1] = [101, 0, 0]; img[1, 0] = [0, 0, 0]; img[1, 1] = [101, 0, 0]
    vis = np.ones((1, 1), np.uint8); w = np.ones((1, 1), np.float32)
    uv = np.array([[[0.5, 0.5]]])  # pixel (0.5, 0.5): mix 50.5 -> lround 51
    _, rgb8 = O.blend_colors(vis, uv, w, [img])
    assert rgb8[0, 0] == 51

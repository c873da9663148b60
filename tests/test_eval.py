# SPDX-License-Identifier: Apache-2.0
"""Evaluation renderer + metrics on the GPU, bit-exact
against oracle/oracle_eval.py: the rasterizer in both modes on a real textured
frame (incl. the order-dependent float z-buffer), VRE, the distance transform,
2-D Hausdorff, CP-RMSE and WMS3IM."""
import numpy as np
import pytest

from oracle import oracle_eval as OE
from paper_1712_03084_b200 import _lib as L
from paper_1712_03084_b200 import evaluate as ev
from paper_1712_03084_b200 import volcap as vc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return vc.default_context(0)


@pytest.fixture(scope="module")
def frame(ctx):
    rig = vc.make_circle_rig(4, 1, 2500, 512, 424, 365)
    frames = [vc.render_frame(rig, vc.xpose_body(), k) for k in range(5)]
    rec = vc.reconstruct_frame(frames[:4], rig, vc.ReconConfig(dims=(32, 64, 32)), ctx=ctx)
    return rig, frames, rec


@pytest.mark.parametrize("mode", [ev.UV_BLEND, ev.COLOR_PER_VERTEX])
def test_rasterize_bit_exact(ctx, frame, mode):
    rig, frames, rec = frame
    s = rig.sensors[4]  # the held-out view
    scale = 0.25
    intr = L.Intrinsics(s.depth_intr.fx * scale, s.depth_intr.fy * scale, s.depth_intr.cx * scale,
                        s.depth_intr.cy * scale, 128, 106)
    tm = rec.textured
    images = [f.color for f in frames[:4]]
    out = ev.rasterize(tm, intr, s.pose, images, mode, ctx=ctx)
    R = [[float(s.pose.R[r][c]) for c in range(3)] for r in range(3)]
    d, c, m = OE.rasterize(tm.mesh.vertices, tm.mesh.triangles, tm.visible, tm.uv, tm.weight,
                           (intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height), R,
                           [float(v) for v in s.pose.t], images, mode)
    assert m.sum() > 500
    assert np.array_equal(out.silhouette, m)
    assert np.array_equal(out.depth, d)
    assert np.array_equal(out.color, c)


def test_masks_vre_dt_hausdorff(ctx):
    rng = np.random.default_rng(4)
    for _ in range(3):
        a = (rng.uniform(size=(47, 61)) < 0.08).astype(np.uint8)
        b = np.zeros_like(a)
        b[10:30, 12:40] = 1
        assert ev.vre(a, b, ctx=ctx) == OE.vre(a, b)
        assert np.array_equal(ev.distance_transform(a, ctx=ctx), OE.distance_transform(a))
        assert ev.hausdorff2d(a, b, ctx=ctx) == OE.hausdorff2d(a, b)
    z = np.zeros((20, 30), np.uint8)
    assert ev.hausdorff2d(z, b[:20, :30], ctx=ctx) is None
    assert ev.vre(z, z, ctx=ctx) == 0.0
    assert np.isinf(ev.distance_transform(z, ctx=ctx)).all()


def test_cp_rmse(ctx):
    rng = np.random.default_rng(7)
    g, r = rng.normal(size=(400, 3)) * 100, rng.normal(size=(700, 3)) * 100
    assert ev.cp_rmse(g, r, ctx=ctx) == OE.cp_rmse(g, r)
    with pytest.raises(vc.VcError):
        ev.cp_rmse(np.zeros((0, 3)), r, ctx=ctx)


def test_wms3im(ctx):
    rng = np.random.default_rng(8)
    a = rng.integers(0, 256, (40, 52, 3), dtype=np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-30, 30, a.shape), 0, 255).astype(np.uint8)
    m = np.zeros((40, 52), np.uint8)
    m[5:35, 8:45] = 1
    assert ev.wms3im(a, b, m, ctx=ctx) == OE.wms3im(a, b, m)
    assert ev.wms3im(a, a, m, ctx=ctx) == pytest.approx(1.0)
    assert ev.wms3im(a, b, np.zeros_like(m), ctx=ctx) is None

# SPDX-License-Identifier: Apache-2.0
"""(A, L) consumers against oracle/oracle_volume.py and the
reference's test_mocap_volume.cpp:55-163: binarize (GPU union-find) equal to the
raster flood fill incl. ties and the inverted side, boundary voxels, and the
GPU skeletonize equal to the restated sequential thinning (incl. shuffled voxel
lists, where the order-dependent re-check matters)."""
import math

import numpy as np
import pytest

from oracle import oracle_volume as OV
from oracle import ref as R
from paper_1712_03084_b200 import volcap as vc
from paper_1712_03084_b200 import volume_ops as vo


def ball(n, c, r, shape=None):
    nz, ny, nx = shape or (n, n, n)
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return (np.sqrt((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2) <= r).astype(np.float64)


def spec(shape):
    nz, ny, nx = shape
    return vc.GridSpec(nx, ny, nz, np.array([-3.0, 2.0, 1.5]), 2.5)


def bv_of(keep, vox):
    return vo.BinaryVolume(keep, vox, spec(keep.shape))


# ------------------------------------------------------------------ GPU skeletonize
@pytest.mark.gpu
def test_skeletonize_single_voxel():
    g = np.zeros((8, 8, 8), np.uint8)
    g[4, 4, 4] = 1
    assert vo.skeletonize(bv_of(g, np.array([[4, 4, 4]], np.int32))).tolist() == [[4, 4, 4]]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_skeletonize_matches_restatement(seed):
    """Union of overlapping balls (test_mocap_volume.cpp:129-163) + a box and a bar."""
    rng = np.random.default_rng(seed)
    A = np.zeros((20, 20, 20))
    c = rng.uniform(6, 14, 3)
    for _ in range(4):
        A = np.maximum(A, ball(20, c, rng.uniform(2, 4)))
        c = c + rng.uniform(-3, 3, 3)
    if seed % 2:
        A[3:7, 4:16, 5:9] = 1.0
    keep, vox = OV.binarize(A, 0.5)
    ours = vo.skeletonize(bv_of(keep, vox))
    assert np.array_equal(ours, OV.skeletonize(keep, vox))


@pytest.mark.gpu
def test_skeletonize_cylinder_curve():
    """test_mocap_volume.cpp:99-127 (smaller): thin curve near the axis, subset, one component."""
    n, radius, length = 40, 5, 32
    z, y, x = np.meshgrid(np.arange(14), np.arange(n), np.arange(n), indexing="ij")
    g = ((x >= 4) & (x < 4 + length) & (np.hypot(y - 20.0, z - 7.0) <= radius)).astype(np.uint8)
    zz, yy, xx = np.nonzero(g)
    vox = np.stack([xx, yy, zz], 1).astype(np.int32)
    sk = vo.skeletonize(vo.BinaryVolume(g, vox, vc.GridSpec(n, n, 14, np.zeros(3), 1.0)))
    assert 0 < len(sk) < len(vox) / 10
    for qx, qy, qz in sk:
        assert g[qz, qy, qx] == 1
        if 4 + radius <= qx < 4 + length - radius:
            assert math.hypot(qy - 20.0, qz - 7.0) <= 2.0


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4))
def test_skeletonize_shuffled_order(seed):
    """The re-check is order-dependent (skeletonize.cpp:150-158): a permuted voxel
    list must give the restatement's result for that same permuted order."""
    rng = np.random.default_rng(100 + seed)
    A = np.zeros((18, 22, 20))
    c = rng.uniform(6, 13, 3)
    for _ in range(3):
        A = np.maximum(A, ball(20, c, rng.uniform(2.5, 4.5), shape=(18, 22, 20)))
        c = c + rng.uniform(-3, 3, 3)
    A[4:8, 3:19, 6:10] = 1.0
    keep, vox = OV.binarize(A, 0.5)
    vox = vox[rng.permutation(len(vox))]
    ours = vo.skeletonize(bv_of(keep, vox))
    assert np.array_equal(ours, OV.skeletonize(keep, vox))


@pytest.mark.gpu
def test_skeletonize_noisy_blob():
    """A ragged blob (random voxels added on a ball's shell): many simple points,
    long chains of adjacent candidates in one sweep."""
    rng = np.random.default_rng(7)
    A = ball(24, (11.5, 11.5, 11.5), 7.0)
    shell = (ball(24, (11.5, 11.5, 11.5), 9.0) > 0) & (A == 0)
    A[shell & (rng.uniform(size=A.shape) < 0.5)] = 1.0
    keep, vox = OV.binarize(A, 0.5)
    ours = vo.skeletonize(bv_of(keep, vox))
    assert np.array_equal(ours, OV.skeletonize(keep, vox))


def _blob(seed, shape=(18, 22, 20)):
    rng = np.random.default_rng(seed)
    A = np.zeros(shape)
    c = rng.uniform(6, 13, 3)
    for _ in range(3):
        A = np.maximum(A, ball(20, c, rng.uniform(2.5, 4.5), shape=shape))
        c = c + rng.uniform(-3, 3, 3)
    return A


@pytest.mark.skipif(not R.available(0), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(3))
def test_skeletonize_restatement_matches_reference(seed):
    """Pins oracle_volume.skeletonize to the reference's own skeletonize.cpp."""
    keep, vox = OV.binarize(_blob(seed), 0.5)
    if seed == 2:
        vox = vox[np.random.default_rng(1).permutation(len(vox))]
    assert np.array_equal(OV.skeletonize(keep, vox), R.skeletonize(keep, vox))


@pytest.mark.gpu
@pytest.mark.skipif(not R.available(0), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(3))
def test_skeletonize_matches_reference_large(seed):
    """GPU thinning == the reference's sequential thinning on a 64^3 multi-ball body
    (thousands of candidates per direction; the reference runs in C++ here)."""
    rng = np.random.default_rng(200 + seed)
    A = np.zeros((64, 64, 64))
    c = np.array([32.0, 32.0, 32.0])
    for _ in range(6):
        A = np.maximum(A, ball(64, c, rng.uniform(6, 12)))
        c = np.clip(c + rng.uniform(-10, 10, 3), 14, 50)
    keep, vox = OV.binarize(A, 0.5)
    if seed == 1:
        vox = vox[rng.permutation(len(vox))]
    ours = vo.skeletonize(bv_of(keep, vox))
    assert np.array_equal(ours, R.skeletonize(keep, vox))


# ------------------------------------------------------------------ GPU binarize
@pytest.fixture(scope="module")
def ctx():
    return vc.default_context(0)


@pytest.mark.gpu
def test_binarize_reference_kats(ctx):
    A = ball(32, (15.5, 15.5, 15.5), 9.0)
    b = vo.binarize(A, spec(A.shape), 0.5, ctx=ctx)
    assert len(b.voxels) == int((A >= 0.5).sum())
    A = ball(40, (12, 12, 12), 8.0)
    A[30:33, 30:33, 30:33] = 1.0
    b = vo.binarize(A, spec(A.shape), 0.5, ctx=ctx)
    assert (b.voxels[:, 0] < 30).all()
    A = ball(32, (15.5, 15.5, 15.5), 10.0)
    b = vo.binarize(A, spec(A.shape), 0.5, ctx=ctx)
    assert abs(len(b.voxels) - 4 / 3 * math.pi * 1000) / (4 / 3 * math.pi * 1000) < 0.05
    with pytest.raises(vc.VcError):
        vo.binarize(-np.ones((8, 8, 8)), spec((8, 8, 8)), float("nan"), ctx=ctx)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4))
def test_binarize_exact_vs_flood_fill(ctx, seed):
    rng = np.random.default_rng(100 + seed)
    shape = (24, 28, 32)
    A = rng.normal(size=shape) * 0.2
    for _ in range(6):  # blobs of random sizes, incl. equal-size twins (ties -> first in raster order)
        c = rng.uniform(3, 20, 3)
        r = rng.uniform(1.5, 4)
        A = np.maximum(A, ball(0, c, r, shape))
        if seed == 1:
            A = np.maximum(A, ball(0, c + [0, 0, 0], r, shape)[:, :, ::-1])
    level = 0.5 if seed != 2 else -0.25  # seed 2: max(A) >= L still; seed 3 inverts below
    if seed == 3:
        A = -A
        level = -0.5
    A32 = A.astype(np.float32)
    b = vo.binarize(A32, spec(shape), level, ctx=ctx)
    keep, vox = OV.binarize(A32.astype(np.float64), level)
    assert np.array_equal(b.grid, keep)
    assert np.array_equal(b.voxels, vox)
    sp = spec(shape)
    bo = vo.boundary_voxels(b, ctx=ctx)
    assert np.array_equal(bo, OV.boundary_voxels(keep, vox, sp.origin, sp.edge_mm))


@pytest.mark.gpu
def test_binarize_frame_volume(ctx):
    """On the last frame's device volume: equal to the flood fill on the exported field."""
    rig = vc.make_circle_rig(4, 0, 2500, 512, 424, 365)
    frames = [vc.render_frame(rig, vc.xpose_body(), k) for k in range(4)]
    rec = vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=(64, 64, 64)), ctx=ctx, want_volume=True)
    g = rec.volume.grid
    b = vo.binarize_frame(ctx, g, rec.volume.iso_level)
    keep, vox = OV.binarize(rec.volume.values.astype(np.float64), rec.volume.iso_level)
    assert np.array_equal(b.voxels, vox) and np.array_equal(b.grid, keep)
    sk = vo.skeletonize(b)
    assert 0 < len(sk) < len(vox) / 5

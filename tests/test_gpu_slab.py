# SPDX-License-Identifier: Apache-2.0
"""z-slab decomposition on one B200: the loopback
exchanger runs P virtual ranks in lockstep, the NCCL exchanger a 1-rank
communicator.  The slab pipeline must reproduce the single-GPU frame: the
indicator field within float-atomic noise, and -- on the same field and level
-- the single-GPU marching cubes and texture bit-exactly (global vertex ids,
rank-order concatenation)."""
import numpy as np
import pytest
from scipy.spatial import cKDTree

from paper_1712_03084_b200 import volcap as vc
from paper_1712_03084_b200.slab import SlabReconstructor, merge_pieces, nccl_unique_id

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def closed_manifold(tris):
    t = np.asarray(tris, np.int64)
    e = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
    e.sort(axis=1)
    _, counts = np.unique(e[:, 0] * (1 << 32) + e[:, 1], return_counts=True)
    return bool(np.all(counts == 2))


@pytest.fixture(scope="module")
def ctx():
    return vc.default_context(0)


@pytest.fixture(scope="module")
def scene():
    rig = vc.make_circle_rig(4, 0, 2500, 512, 424, 365)
    frames = [vc.render_frame(rig, vc.xpose_body(), k) for k in range(4)]
    return rig, frames


def check_against_single(sr, pieces, rig, frames, cfg, ctx):
    P = sr.world
    single = vc.reconstruct_frame(frames, rig, cfg, ctx=ctx, want_volume=True, want_clouds=True)
    grid = pieces[0].grid
    A = np.concatenate([sr.export_volume(i, grid) for i in range(len(pieces))])
    assert A.shape == single.volume.values.shape
    assert rel_l2(A, single.volume.values) < 1e-5  # float atomics in the splat: same field up to ordering noise
    levels = {p.iso_level for p in pieces}
    assert len(levels) == 1
    L = pieces[0].iso_level
    assert abs(L - single.volume.iso_level) <= 1e-5 * abs(single.volume.iso_level)
    # vertex numbering: offsets are the running sums of the pieces
    off = 0
    for i, p in enumerate(pieces):
        assert p.info["rank"] == i and p.info["world"] == P
        assert p.info["z_begin"] == i * grid.nz // P and p.info["z_end"] == (i + 1) * grid.nz // P
        assert p.info["vertex_offset"] == off
        off += len(p.mesh.vertices)
    assert all(p.info["vertex_total"] == off for p in pieces)
    mesh, tex = merge_pieces(pieces)
    assert mesh.triangles.min() >= 0 and mesh.triangles.max() < off
    # the single-GPU marching cubes on the slab field at the slab level: identical mesh
    m = vc.marching_cubes(A, grid, L, ctx=ctx)
    assert np.array_equal(m.vertices, mesh.vertices)
    assert np.array_equal(m.triangles, mesh.triangles)
    assert np.array_equal(m.normals.astype(np.float32), mesh.normals.astype(np.float32))
    assert closed_manifold(mesh.triangles)
    # texture of the same vertices: identical
    tm = vc.texture(mesh.vertices, rig, frames, single.clouds.weight_maps, ctx=ctx)
    for a, b in ((tex.visible, tm.visible), (tex.uv, tm.uv), (tex.weight, tm.weight),
                 (tex.untextured, tm.untextured), (tex.rgb, tm.rgb)):
        assert np.array_equal(a, b)
    # and the whole-frame mesh agrees with the single-GPU one to within the parity bar
    d1, _ = cKDTree(single.mesh.vertices).query(mesh.vertices)
    d2, _ = cKDTree(mesh.vertices).query(single.mesh.vertices)
    assert max(d1.max(), d2.max()) <= 0.5 * grid.edge_mm
    return A, mesh


@pytest.mark.parametrize("P,dims", [(1, (64, 64, 64)), (2, (64, 128, 64)), (4, (128, 256, 128)),
                                    (8, (128, 128, 128)), (2, (256, 512, 256))])
def test_slab_loopback_matches_single_gpu(scene, ctx, P, dims):
    rig, frames = scene
    cfg = vc.ReconConfig(dims=dims)
    sr = SlabReconstructor.loopback(P)
    pieces = sr.reconstruct_frame(frames, rig, cfg)
    assert len(pieces) == P
    check_against_single(sr, pieces, rig, frames, cfg, ctx)
    sr.close()


def test_slab_simple_mode_and_repeat(scene, ctx):
    rig, frames = scene
    cfg = vc.ReconConfig(dims=(128, 128, 128), mode="simple")
    sr = SlabReconstructor.loopback(4)
    p1 = sr.reconstruct_frame(frames, rig, cfg)
    A1 = np.concatenate([sr.export_volume(i, p1[0].grid) for i in range(4)])
    p2 = sr.reconstruct_frame(frames, rig, cfg)  # sparse clear of the slab accumulators
    check_against_single(sr, p2, rig, frames, cfg, ctx)
    A2 = np.concatenate([sr.export_volume(i, p2[0].grid) for i in range(4)])
    assert rel_l2(A2, A1) < 1e-6
    # a different body in the same slabs: nothing of frame 1 survives
    kick = [vc.render_frame(rig, vc.kick_body(300, 120), k) for k in range(4)]
    p3 = sr.reconstruct_frame(kick, rig, cfg)
    check_against_single(sr, p3, rig, kick, cfg, ctx)
    sr.close()


def test_slab_invalid_decompositions(scene):
    rig, frames = scene
    sr = SlabReconstructor.loopback(3)
    with pytest.raises(vc.VcInvalidArgument):
        sr.reconstruct_frame(frames, rig, vc.ReconConfig(dims=(64, 64, 64)))  # 64 % 3
    sr.close()
    sr = SlabReconstructor.loopback(8)
    with pytest.raises(vc.VcInvalidArgument):
        sr.reconstruct_frame(frames, rig, vc.ReconConfig(dims=(16, 16, 8)))  # nz/P < 2
    sr.close()


def test_slab_nccl_one_rank(scene, ctx):
    """The NCCL exchanger (send/recv to self, all-gather, all-reduce) on a 1-rank communicator."""
    rig, frames = scene
    cfg = vc.ReconConfig(dims=(128, 256, 128))
    sr = SlabReconstructor.nccl(1, 0, 0, nccl_unique_id())
    pieces = sr.reconstruct_frame(frames, rig, cfg)
    check_against_single(sr, pieces, rig, frames, cfg, ctx)
    sr.close()


@pytest.mark.slow
def test_c5_1024_slab_loopback(ctx):
    """C5: 1024^3 as 4 slabs on one device (~60 GB) vs the single-GPU frame."""
    rig = vc.make_circle_rig(4, 0, 2500, 512, 424, 365)
    frames = [vc.render_frame(rig, vc.xpose_body(), k, ctx=ctx) for k in range(4)]
    cfg = vc.ReconConfig(dims=(1024, 1024, 1024))
    sr = SlabReconstructor.loopback(4)
    pieces = sr.reconstruct_frame(frames, rig, cfg)
    mesh, _ = merge_pieces(pieces)
    assert len(mesh.vertices) > 500_000
    assert closed_manifold(mesh.triangles)
    grid = pieces[0].grid
    single = vc.reconstruct_frame(frames, rig, cfg, ctx=ctx, want_volume=True)
    A = np.concatenate([sr.export_volume(i, grid) for i in range(4)])
    assert rel_l2(A, single.volume.values) < 1e-5
    assert abs(len(mesh.vertices) - len(single.mesh.vertices)) <= 1e-3 * len(single.mesh.vertices)
    sr.close()

# SPDX-License-Identifier: Apache-2.0
"""GPU parity of the B200 FTR path against the CPU oracle (BASELINE.json
tolerances): pixel/voxel binning and MC topology bit-exact, indicator field
within 1e-4 rel-L2, vertices within 0.5 voxel Hausdorff, colours within
1/255.  All compute goes through the C-ABI (libvc_b200.so)."""
import numpy as np
import pytest
from scipy.spatial import cKDTree

from paper_1712_03084_b200 import volcap as vc

pytestmark = pytest.mark.gpu

REL_L2_A = 1e-4      # BASELINE.json: indicator field within 1e-4 relative L2
HAUSDORFF_VOX = 0.5  # vertices within 0.5 voxel Hausdorff
COLOR_TOL = 1        # colours within 1/255


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def ctx():
    return vc.default_context(0)


@pytest.fixture(scope="module")
def scene(O):
    """SURVEY §8(d) C1 inputs: 4 Kinect2-like views 512x424, f=365, X-pose."""
    rig = vc.make_circle_rig(4, 0, 2500, 512, 424, 365)
    body = vc.xpose_body()
    frames = [vc.render_frame(rig, body, k) for k in range(4)]
    orig = O.make_circle_rig(4, 0, 2500, 1000, 512, 424, 365)
    return rig, body, frames, orig


def oracle_frame(O, orig, frames, **kw):
    r = O.reconstruct_frame(orig, [f.depth for f in frames], [f.foreground for f in frames],
                            [f.color for f in frames], **kw)
    assert r.status == 0
    return r


# ------------------------------------------------------------------ fixture parity
@pytest.mark.parametrize("body_kind,sigma", [("xpose", 0.0), ("kick", 0.0), ("xpose", 2.0)])
def test_renderer_bit_exact(O, scene, body_kind, sigma):
    rig, _, _, orig = scene
    body = vc.xpose_body() if body_kind == "xpose" else vc.kick_body(300, 120)
    obody = O.xpose_body() if body_kind == "xpose" else O.kick_body(300, 120)
    for k in range(4):
        g = vc.render_frame(rig, body, k, 3, sigma_mm_at_2m=sigma, seed=31)
        o = O.render_frame(orig[k], obody, k, 3, sigma_mm_at_2m=sigma, seed=31)
        assert np.array_equal(g.depth, o.depth)
        assert np.array_equal(g.foreground, o.mask)
        assert np.array_equal(g.color, o.rgb)


# ------------------------------------------------------------------ K1/K2 preprocess
def test_preprocess_bit_exact(O, scene, ctx):
    rig, _, frames, orig = scene
    clouds, grid = vc.preprocess(frames, rig, vc.ReconConfig(dims=(128, 128, 128)), ctx=ctx)
    ref = oracle_frame(O, orig, frames, dims=(128, 128, 128), want_volume=False)
    p = ref.points
    assert len(clouds.position) == len(p["position"]) > 30000
    assert np.array_equal(clouds.position, p["position"])
    assert np.array_equal(clouds.normal, p["normal"])
    assert np.array_equal(clouds.weight, p["weight"])
    assert np.array_equal(clouds.px, p["px"]) and np.array_equal(clouds.py, p["py"])
    assert np.array_equal(clouds.sensor, p["sensor"])
    for k in range(4):
        assert np.array_equal(clouds.weight_maps[k], ref.weight_maps[k])
    assert grid.edge_mm == ref.grid.edge and list(grid.origin) == list(ref.grid.origin[:])


@pytest.mark.parametrize("w,h,f", [(333, 247, 160.0), (97, 61, 48.0), (1100, 300, 500.0)])
def test_preprocess_bit_exact_ragged_size(O, ctx, w, h, f):
    """Image widths that are not a multiple of the 32-pixel segment (ragged
    last segment per row) and odd heights: points, weights and grid stay
    bit-exact."""
    rig = vc.make_circle_rig(4, 0, 2500, w, h, f)
    orig = O.make_circle_rig(4, 0, 2500, 1000, w, h, f)
    body = vc.kick_body(300, 77)
    frames = [vc.render_frame(rig, body, k) for k in range(4)]
    clouds, grid = vc.preprocess(frames, rig, vc.ReconConfig(dims=(64, 64, 64)), ctx=ctx)
    ref = oracle_frame(O, orig, frames, dims=(64, 64, 64), want_volume=False)
    p = ref.points
    assert len(clouds.position) == len(p["position"]) > 100
    assert np.array_equal(clouds.position, p["position"])
    assert np.array_equal(clouds.normal, p["normal"])
    assert np.array_equal(clouds.weight, p["weight"])
    assert np.array_equal(clouds.px, p["px"]) and np.array_equal(clouds.py, p["py"])
    for k in range(4):
        assert np.array_equal(clouds.weight_maps[k], ref.weight_maps[k])
    assert grid.edge_mm == ref.grid.edge and list(grid.origin) == list(ref.grid.origin[:])


def test_preprocess_bit_exact_mixed_resolutions(O, ctx):
    """Views of different sizes in one rig (segments past a narrower view's
    width): points, weight maps and grid bit-exact."""
    a = vc.make_circle_rig(4, 0, 2500, 333, 247, 160.0)
    b = vc.make_circle_rig(4, 0, 2500, 512, 424, 365.0)
    rig = vc.CameraRig([a.sensors[0], b.sensors[1], a.sensors[2], b.sensors[3]], 4)
    oa = O.make_circle_rig(4, 0, 2500, 1000, 333, 247, 160.0)
    ob = O.make_circle_rig(4, 0, 2500, 1000, 512, 424, 365.0)
    orig = (O.Sensor * 4)()
    orig[0], orig[1], orig[2], orig[3] = oa[0], ob[1], oa[2], ob[3]
    body = vc.kick_body(300, 200)
    frames = [vc.render_frame(rig, body, k) for k in range(4)]
    clouds, grid = vc.preprocess(frames, rig, vc.ReconConfig(dims=(64, 64, 64)), ctx=ctx)
    ref = oracle_frame(O, orig, frames, dims=(64, 64, 64), want_volume=False)
    assert len(clouds.position) == len(ref.points["position"]) > 1000
    assert np.array_equal(clouds.position, ref.points["position"])
    assert np.array_equal(clouds.weight, ref.points["weight"])
    assert np.array_equal(clouds.sensor, ref.points["sensor"])
    for k in range(4):
        assert np.array_equal(clouds.weight_maps[k], ref.weight_maps[k])
    assert grid.edge_mm == ref.grid.edge and list(grid.origin) == list(ref.grid.origin[:])


def test_preprocess_noisy_and_discontinuity(O, scene, ctx):
    rig, body, _, orig = scene
    frames = [vc.render_frame(rig, body, k, 0, sigma_mm_at_2m=2.0, seed=7) for k in range(4)]
    cfg = vc.ReconConfig(dims=(64, 64, 64), discontinuity_mm=5.0, silhouette_radius_px=4)
    clouds, grid = vc.preprocess(frames, rig, cfg, ctx=ctx)
    ref = oracle_frame(O, orig, frames, dims=(64, 64, 64), discontinuity_mm=5.0, silhouette_radius_px=4,
                       want_volume=False)
    assert np.array_equal(clouds.position, ref.points["position"])
    assert np.array_equal(clouds.weight, ref.points["weight"])


def test_empty_scene_raises(ctx):
    rig = vc.make_circle_rig(2, 0, 2500, 64, 56, 60)
    z = vc.RgbdFrame(np.zeros((56, 64), np.uint16), np.zeros((56, 64, 3), np.uint8), np.zeros((56, 64), np.uint8))
    with pytest.raises(vc.VcEmptyScene):
        vc.reconstruct_frame([z, z], rig, vc.ReconConfig(r=5), ctx=ctx)


def test_invalid_config_raises(scene, ctx):
    rig, _, frames, _ = scene
    with pytest.raises(ValueError):
        vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=(48, 64, 64)), ctx=ctx)  # not a power of two
    with pytest.raises(ValueError):
        vc.reconstruct_frame(frames, rig, vc.ReconConfig(r=3, padding_voxels=8), ctx=ctx)  # reconstruct.cpp:25-26


# ------------------------------------------------------------------ K3 splat
def test_splat_kats(ctx):
    """test_recon_field.cpp:145-234 on the GPU (fp32 accumulation: 1e-6)."""
    g = vc.GridSpec(16, 32, 16, np.zeros(3), 10.0)
    n = np.array([1.0, 2.0, -2.0]) / 3.0
    f, d = vc.splat([[80.0, 160.0, 80.0]], [n], [1.0], g, ctx=ctx)
    assert np.linalg.norm(f[8, 16, 8] - np.sqrt(1.5) * n) < 1e-6
    f, d = vc.splat([[40.0, 80.0, 40.0]], [[0, 0, 1.0]], [0.0], g, ctx=ctx)
    assert np.all(f == 0)
    f, d = vc.splat(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0), g, ctx=ctx)
    assert np.all(f == 0) and np.all(d == 0)
    fs, _ = vc.splat([[80.0, 160.0, 80.0]], [n], [1.0], g, mode="simple", ctx=ctx)
    assert np.linalg.norm(fs[8, 16, 8] - n) < 1e-6


@pytest.mark.parametrize("mode", ["weighted", "simple"])
def test_splat_matches_oracle(O, scene, ctx, mode):
    rig, _, frames, orig = scene
    ref = oracle_frame(O, orig, frames, dims=(128, 128, 128), want_volume=False)
    p = ref.points
    g = vc.GridSpec(128, 128, 128, np.array(ref.grid.origin[:]), ref.grid.edge)
    f, d = vc.splat(p["position"], p["normal"], p["weight"], g, mode=mode, ctx=ctx)
    of, od, (s1, s2) = O.splat(p["position"], p["normal"], p["weight"], ref.grid, mode=0 if mode == "weighted" else 1)
    assert rel_l2(d, od) < 1e-5
    # the same voxels pass the density threshold (binning is exact; borderline eps only)
    nz_g, nz_o = np.linalg.norm(f, axis=-1) > 0, np.linalg.norm(of, axis=-1) > 0
    assert (nz_g != nz_o).sum() <= 2
    assert rel_l2(f, of) < 1e-5


# ------------------------------------------------------------------ K4-K8 integrate
@pytest.mark.parametrize("shape", [(16, 32, 16), (8, 16, 32), (64, 128, 64), (32, 32, 64)])
def test_integrate_matches_oracle_nonhermitian(O, ctx, shape):
    """Random fields: non-Hermitian filtered planes at kx=0, nx/2."""
    rng = np.random.default_rng(sum(shape))
    field = rng.normal(size=shape + (3,)).astype(np.float32)
    A = vc.integrate_fft(field, ctx=ctx)
    ref = O.integrate_fft(field.astype(np.float64))
    assert rel_l2(A, ref) < 1e-5


def test_integrate_blob_and_zero(ctx):
    nz, ny, nx = 64, 128, 64
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    d = np.stack([x, y, z], -1) - np.array([31.5, 63.5, 31.5])
    f = np.exp(-(d * d).sum(-1) / 72.0)
    A = vc.integrate_fft((-d / 36.0 * f[..., None]).astype(np.float32), ctx=ctx)
    assert np.sqrt(np.mean((A - (f - f.mean())) ** 2)) < 0.01 * f.max()
    assert abs(A.astype(np.float64).mean()) < 1e-7
    assert np.all(vc.integrate_fft(np.zeros((16, 32, 16, 3), np.float32), ctx=ctx) == 0)


def test_integrate_large_sizes(O, ctx):
    for shape in [(512, 4, 8), (4, 512, 8), (8, 4, 1024), (1024, 8, 4), (4, 1024, 8)]:
        rng = np.random.default_rng(1)
        field = rng.normal(size=shape + (3,)).astype(np.float32)
        assert rel_l2(vc.integrate_fft(field, ctx=ctx), O.integrate_fft(field.astype(np.float64))) < 2e-5


# ------------------------------------------------------------------ whole frame A
@pytest.mark.parametrize("dims", [(64, 1024, 64), (64, 64, 1024), (1024, 64, 64)])
def test_indicator_field_1024_point_axes(O, scene, ctx, dims):
    """The 1024-point passes on sparse frame fields against the oracle: the
    pipelined F-y (live-plane list) and Z kernels and the 1024-point x passes
    (mostly empty planes and rows: the body spans a fraction of the long axis)."""
    rig, _, frames, orig = scene
    rec = vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=dims), ctx=ctx, want_volume=True)
    ref = oracle_frame(O, orig, frames, dims=dims)
    assert rel_l2(rec.volume.values, ref.volume) < REL_L2_A
    assert abs(rec.volume.iso_level - ref.iso_level) < 1e-4 * abs(ref.iso_level)


@pytest.mark.parametrize("dims", [(128, 128, 128), (128, 256, 128)])
def test_indicator_field_rel_l2(O, scene, ctx, dims):
    rig, _, frames, orig = scene
    rec = vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=dims), ctx=ctx, want_volume=True)
    ref = oracle_frame(O, orig, frames, dims=dims)
    assert rel_l2(rec.volume.values, ref.volume) < REL_L2_A
    assert abs(rec.volume.iso_level - ref.iso_level) < 1e-4 * abs(ref.iso_level)


# ------------------------------------------------------------------ K9 iso level
def test_iso_level_matches_oracle(O, ctx):
    rng = np.random.default_rng(9)
    A = rng.normal(size=(32, 64, 32)).astype(np.float32)
    g = vc.GridSpec(32, 64, 32, np.array([-10.0, 5.0, 3.0]), 7.5)
    og = O.grid(32, 64, 32, (-10.0, 5.0, 3.0), 7.5)
    pos = rng.uniform(-20, 500, (5000, 3))
    assert abs(vc.iso_level(A, g, pos, ctx=ctx) - O.iso_level(A.astype(np.float64), og, pos)) < 1e-12
    with pytest.raises(ValueError):
        vc.iso_level(A, g, np.zeros((0, 3)), ctx=ctx)


# ------------------------------------------------------------------ K10 marching cubes
def _mc_compare(O, ctx, A, level, origin=(0.0, 0.0, 0.0), edge=1.0):
    nz, ny, nx = A.shape
    g = vc.GridSpec(nx, ny, nz, np.array(origin), edge)
    m = vc.marching_cubes(A, g, level, ctx=ctx)
    o = O.marching_cubes(A.astype(np.float64), O.grid(nx, ny, nz, origin, edge), level)
    # vertex ids: GPU numbers by global edge id, the reference by first touch
    assert np.all(np.diff(m.edge_ids.astype(np.int64)) > 0)
    assert np.array_equal(np.sort(o.edge_ids), m.edge_ids)
    # triangles as oriented edge-id triples, same (reference) order: bit-exact topology
    assert np.array_equal(m.edge_ids[m.triangles], o.edge_ids[o.triangles])
    order = np.argsort(o.edge_ids)
    assert np.array_equal(m.vertices, o.vertices[order])
    assert np.allclose(m.normals, o.normals[order], atol=1e-6)
    return m


def test_mc_sphere_and_blobs_bit_exact(O, ctx):
    n = 48
    c = (n - 1) / 2.0
    z, y, x = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    A = (np.sqrt((x - c) ** 2 + (y - c) ** 2 + (z - c) ** 2) <= 20.0).astype(np.float32)
    m = _mc_compare(O, ctx, A, 0.5)
    assert O.analyze_topology(m.triangles, len(m.vertices))["euler"] == 2
    rng = np.random.default_rng(2024)
    for _ in range(5):
        v = np.zeros((32, 32, 32))
        for cc, w in zip(rng.uniform(10, 22, (4, 3)), rng.uniform(3, 6, 4)):
            p = np.stack([x[:32, :32, :32], y[:32, :32, :32], z[:32, :32, :32]], -1)
            v += np.exp(-((p - cc) ** 2).sum(-1) / (2 * w * w))
        _mc_compare(O, ctx, v.astype(np.float32), 0.5, origin=(-3.0, 2.0, 1.0), edge=2.5)


def test_mc_empty_and_degenerate(O, ctx):
    g = vc.GridSpec(8, 8, 8, np.zeros(3), 1.0)
    m = vc.marching_cubes(np.zeros((8, 8, 8), np.float32), g, 0.5, ctx=ctx)
    assert len(m.vertices) == 0 and len(m.triangles) == 0
    # level exactly on lattice values: ties follow vals >= level (marching_cubes.cpp:168-171)
    A = np.zeros((8, 8, 8), np.float32)
    A[2:5, 2:6, 3:5] = 0.5
    _mc_compare(O, ctx, A, 0.5)


def test_mc_frame_field_bit_exact(O, scene, ctx):
    """Case indices + table topology on the real indicator field, same fp32 A."""
    rig, _, frames, _ = scene
    rec = vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=(128, 128, 128)), ctx=ctx, want_volume=True)
    g = rec.volume.grid
    _mc_compare(O, ctx, rec.volume.values, rec.volume.iso_level, origin=g.origin, edge=g.edge_mm)


# ------------------------------------------------------------------ whole frame mesh
@pytest.mark.parametrize("dims,mode", [((128, 128, 128), "weighted"), ((128, 256, 128), "weighted"),
                                       ((64, 128, 64), "simple")])
def test_frame_mesh_hausdorff(O, scene, ctx, dims, mode):
    rig, _, frames, orig = scene
    rec = vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=dims, mode=mode), ctx=ctx)
    ref = oracle_frame(O, orig, frames, dims=dims, mode=0 if mode == "weighted" else 1, want_volume=False)
    d1, _ = cKDTree(ref.mesh.vertices).query(rec.mesh.vertices)
    d2, _ = cKDTree(rec.mesh.vertices).query(ref.mesh.vertices)
    assert max(d1.max(), d2.max()) <= HAUSDORFF_VOX * ref.grid.edge
    assert O.analyze_topology(rec.mesh.triangles, len(rec.mesh.vertices))["edge_manifold"]
    assert abs(len(rec.mesh.vertices) - len(ref.mesh.vertices)) <= 0.01 * len(ref.mesh.vertices)


# ------------------------------------------------------------------ K11 texture
def test_texture_bit_exact_on_identical_vertices(O, scene, ctx):
    rig, _, frames, orig = scene
    ref = oracle_frame(O, orig, frames, dims=(128, 128, 128), want_volume=False)
    tm = vc.texture(ref.mesh.vertices, rig, frames, ref.weight_maps, ctx=ctx)
    assert np.array_equal(tm.visible, ref.vis)
    assert np.array_equal(tm.weight, ref.weight)
    assert np.array_equal(tm.untextured, ref.untextured)
    assert np.array_equal(tm.uv, ref.uv.astype(np.float32))
    assert np.max(np.abs(tm.rgb.astype(int) - ref.rgb8.astype(int))) <= COLOR_TOL


def test_frame_texture_consistent(O, scene, ctx):
    rig, _, frames, orig = scene
    rec = vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=(128, 128, 128)), ctx=ctx, want_clouds=True)
    tm = vc.texture(rec.mesh.vertices, rig, frames, rec.clouds.weight_maps, ctx=ctx)
    for a, b in ((rec.textured.visible, tm.visible), (rec.textured.weight, tm.weight), (rec.textured.rgb, tm.rgb)):
        assert np.array_equal(a, b)
    vis_any = rec.textured.visible.any(0)
    assert vis_any.mean() > 0.8
    ov = O.vertex_visibility(rec.mesh.vertices, orig, [f.depth for f in frames], [f.foreground for f in frames])
    assert np.array_equal(ov, rec.textured.visible)


def test_visibility_kats(ctx):
    """test_appearance.cpp:36-84 on the GPU."""
    s = vc.Sensor(vc.Intrinsics(60, 60, 31.5, 23.5, 64, 48), vc.Pose(), vc.Intrinsics(60, 60, 31.5, 23.5, 64, 48))
    rig = vc.CameraRig([s], 1)
    f = vc.RgbdFrame(np.full((48, 64), 2000, np.uint16), np.full((48, 64, 3), 128, np.uint8),
                     np.ones((48, 64), np.uint8))

    def bp(u, v, z):
        return [(u - 31.5) * z / 60, (v - 23.5) * z / 60, z]
    verts = np.array([bp(31, 23, 2000), bp(31, 23, 2100), [100000, 0, 2000], [0, 0, -500]])
    tm = vc.texture(verts, rig, [f], [np.full((48, 64), 0.7, np.float32)], ctx=ctx)
    assert list(tm.visible[0]) == [1, 0, 0, 0]
    assert tm.weight[0, 0] == np.float32(0.7) and list(tm.untextured) == [0, 1, 1, 1]
    assert tm.uv[0, 0, 0] == np.float32(31.5 / 64) and tm.uv[0, 0, 1] == np.float32(23.5 / 48)
    assert list(tm.rgb[0]) == [128, 128, 128] and list(tm.rgb[1]) == [200, 200, 200]


# ------------------------------------------------------------------ configurations
def test_six_views_and_single_view(O, ctx):
    rig = vc.make_circle_rig(6, 0, 2500, 512, 424, 365)
    orig = O.make_circle_rig(6, 0, 2500, 1000, 512, 424, 365)
    body = vc.kick_body(300, 200)
    frames = [vc.render_frame(rig, body, k) for k in range(6)]
    rec = vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=(128, 128, 128)), ctx=ctx, want_volume=True)
    ref = oracle_frame(O, orig, frames, dims=(128, 128, 128))
    assert rel_l2(rec.volume.values, ref.volume) < REL_L2_A
    rig1 = vc.CameraRig(rig.sensors[:1], 1)
    rec1 = vc.reconstruct_frame(frames[:1], rig1, vc.ReconConfig(dims=(64, 64, 64)), ctx=ctx, want_volume=True)
    ref1 = O.reconstruct_frame(orig, [frames[0].depth], [frames[0].foreground], [frames[0].color], dims=(64, 64, 64))
    assert rel_l2(rec1.volume.values, ref1.volume) < REL_L2_A


def test_accumulator_state_survives_stage_calls(scene, ctx):
    """The frame path's sparse clear walks the previous frame's touched-row
    list: stage calls, other bodies and other view counts in between must not
    leave stale accumulator contents (field equal to a fresh context's)."""
    rig, _, frames, _ = scene
    cfg = vc.ReconConfig(dims=(128, 128, 128))
    fresh = vc.Context(0)
    ref = vc.reconstruct_frame(frames, rig, cfg, ctx=fresh, want_volume=True).volume.values
    kick = [vc.render_frame(rig, vc.kick_body(300, 60), k) for k in range(4)]
    vc.reconstruct_frame(kick, rig, cfg, ctx=ctx)
    vc.preprocess(frames, rig, cfg, ctx=ctx)  # stage call: resets the control block, not the accumulator
    a = vc.reconstruct_frame(frames, rig, cfg, ctx=ctx, want_volume=True).volume.values
    assert rel_l2(a, ref) < 1e-5
    rig6 = vc.make_circle_rig(6, 0, 2500, 512, 424, 365)
    f6 = [vc.render_frame(rig6, vc.kick_body(300, 200), k) for k in range(6)]
    vc.reconstruct_frame(f6, rig6, cfg, ctx=ctx)
    b = vc.reconstruct_frame(frames, rig, cfg, ctx=ctx, want_volume=True).volume.values
    assert rel_l2(b, ref) < 1e-5
    fresh.close()


def test_repeatability_and_graph_replay(scene, ctx):
    rig, _, frames, _ = scene
    cfg = vc.ReconConfig(dims=(128, 128, 128))
    a = vc.reconstruct_frame(frames, rig, cfg, ctx=ctx, want_volume=True)
    b = vc.reconstruct_frame(frames, rig, cfg, ctx=ctx, want_volume=True)
    assert rel_l2(a.volume.values, b.volume.values) < 1e-6
    assert ctx.kernels_per_frame() >= 16


# ------------------------------------------------------------------ larger configurations (BASELINE C3 / C5)
def hd_rig(vc, k=6):
    """C3: K=6 Kinect2 depth 512x424 (f=365) + 1920x1080 colour (f~1060,
    cx=959.5, cy=539.5) offset by 52 mm along x."""
    return vc.make_hd_rig(k)


def to_oracle_rig(O, rig):
    arr = (O.Sensor * len(rig.sensors))()
    for i, s in enumerate(rig.sensors):
        arr[i] = O.Sensor.from_buffer_copy(bytes(s.to_c()))
    return arr


@pytest.mark.slow
def test_c3_six_views_hd_colour_512(O, ctx):
    rig = hd_rig(vc)
    orig = to_oracle_rig(O, rig)
    body = vc.kick_body(300, 90)
    frames = [vc.render_frame(rig, body, k, ctx=ctx) for k in range(6)]
    obody = O.kick_body(300, 90)
    o0 = O.render_frame(orig[0], obody, 0, 0)
    assert np.array_equal(o0.rgb, frames[0].color) and np.array_equal(o0.depth, frames[0].depth)
    dims = (512, 512, 512)
    rec = vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=dims), ctx=ctx, want_volume=True)
    ref = oracle_frame(O, orig, frames, dims=dims)
    assert rel_l2(rec.volume.values, ref.volume) < REL_L2_A
    d1, _ = cKDTree(ref.mesh.vertices).query(rec.mesh.vertices)
    d2, _ = cKDTree(rec.mesh.vertices).query(ref.mesh.vertices)
    assert max(d1.max(), d2.max()) <= HAUSDORFF_VOX * ref.grid.edge
    assert O.analyze_topology(rec.mesh.triangles, len(rec.mesh.vertices))["edge_manifold"]
    tm = vc.texture(ref.mesh.vertices, rig, frames, ref.weight_maps, ctx=ctx)
    assert np.array_equal(tm.visible, ref.vis) and np.array_equal(tm.weight, ref.weight)
    assert np.max(np.abs(tm.rgb.astype(int) - ref.rgb8.astype(int))) <= COLOR_TOL


@pytest.mark.slow
def test_c5_1024_single_gpu(ctx):
    """C5 on one B200 (~40 GB working set): watertight textured mesh."""
    rig = vc.make_circle_rig(4, 0, 2500, 512, 424, 365)
    frames = [vc.render_frame(rig, vc.xpose_body(), k, ctx=ctx) for k in range(4)]
    t = vc.StageTimings()
    rec = vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=(1024, 1024, 1024)), ctx=ctx, timings=t)
    assert len(rec.mesh.vertices) > 500_000
    assert vc_topology_ok(rec.mesh)
    assert rec.textured.visible.any(0).mean() > 0.8


def vc_topology_ok(mesh):
    t = np.asarray(mesh.triangles, np.int64)
    e = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
    e.sort(axis=1)
    _, counts = np.unique(e[:, 0] * (1 << 32) + e[:, 1], return_counts=True)
    return bool(np.all(counts == 2))


def test_mask_derived_on_device_and_ply_export(scene, ctx, tmp_path):
    """vc_view.mask = NULL: foreground := depth > 0 on the device (dataset.cpp:99-102)
    gives the same frame as the host-side rule; the frame's PLY (mesh_io.cpp:104-145
    of with_channels) is byte-identical to the restated writer on the same arrays."""
    from oracle import oracle_io as OI
    from paper_1712_03084_b200 import io as vio
    rig, _, frames, _ = scene
    host = [vc.RgbdFrame(f.depth, f.color, (f.depth > 0).astype(np.uint8)) for f in frames]
    dev = [vc.RgbdFrame(f.depth, f.color, None) for f in frames]
    cfg = vc.ReconConfig(dims=(128, 128, 128))
    a = vc.reconstruct_frame(host, rig, cfg, ctx=ctx)
    b = vc.reconstruct_frame(dev, rig, cfg, ctx=ctx)
    # same topology; positions equal up to the splat's float-atomic ordering noise
    assert np.array_equal(a.mesh.triangles, b.mesh.triangles)
    assert np.allclose(a.mesh.vertices, b.mesh.vertices, atol=1e-3)
    assert (a.textured.visible == b.textured.visible).mean() > 0.999
    p = str(tmp_path / "frame.ply")
    vio.write_textured_ply(p, b.textured)
    t = b.textured
    assert open(p, "rb").read() == OI.write_ply(t.mesh.vertices, t.mesh.triangles, t.mesh.normals,
                                                OI.with_channels(t.visible, t.uv, t.weight, t.untextured))


def test_r_mode_grid_matches_oracle(O, scene, ctx):
    """ReconConfig.r (reconstruct.hpp:12-18: 2^r x 2^(r+1) x 2^r) end to end."""
    rig, _, frames, orig = scene
    rec = vc.reconstruct_frame(frames, rig, vc.ReconConfig(r=6), ctx=ctx, want_volume=True)
    assert rec.volume.values.shape == (64, 128, 64)
    ref = oracle_frame(O, orig, frames, dims=(64, 128, 64))
    assert rel_l2(rec.volume.values, ref.volume) < REL_L2_A
    d1, _ = cKDTree(ref.mesh.vertices).query(rec.mesh.vertices)
    assert d1.max() <= HAUSDORFF_VOX * ref.grid.edge


def test_mc_capacity_overflow_retry(O, ctx):
    """A noise field with far more cut edges than the initial capacity (N/16):
    the GPU grows its buffers and reruns, topology still bit-exact."""
    rng = np.random.default_rng(77)
    A = rng.uniform(-1, 1, (40, 40, 40)).astype(np.float32)
    m = _mc_compare(O, ctx, A, 0.0)
    assert len(m.vertices) > 40 ** 3 // 16


def test_concurrent_contexts_threads(scene):
    """One context per host thread, frames in flight together (the bench's mode):
    each thread's results equal a sequential run's."""
    import threading
    rig, _, frames, _ = scene
    kick = [[vc.render_frame(rig, vc.kick_body(300, f), k) for k in range(4)] for f in (0, 90, 180, 270)]
    cfg = vc.ReconConfig(dims=(128, 128, 128))
    seq_ctx = vc.Context(0)
    ref = [vc.reconstruct_frame(fr, rig, cfg, ctx=seq_ctx) for fr in kick]
    seq_ctx.close()
    ctxs = [vc.Context(0) for _ in kick]
    out = [None] * len(kick)

    def work(i):
        for _ in range(3):
            out[i] = vc.reconstruct_frame(kick[i], rig, cfg, ctx=ctxs[i])

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(kick))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for a, b in zip(out, ref):
        assert np.array_equal(a.mesh.triangles, b.mesh.triangles) or abs(len(a.mesh.vertices) - len(b.mesh.vertices)) <= 2
        assert abs(len(a.mesh.vertices) - len(b.mesh.vertices)) <= 0.002 * len(b.mesh.vertices)
    for c in ctxs:
        c.close()


def test_sixteen_views(O, ctx):
    """The maximum sensor count (kMaxViews = 16): field and mesh vs the oracle."""
    rig = vc.make_circle_rig(16, 0, 2500, 256, 212, 182)
    orig = O.make_circle_rig(16, 0, 2500, 1000, 256, 212, 182)
    body = vc.kick_body(300, 150)
    frames = [vc.render_frame(rig, body, k) for k in range(16)]
    rec = vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=(64, 64, 64)), ctx=ctx, want_volume=True)
    ref = oracle_frame(O, orig, frames, dims=(64, 64, 64))
    assert rel_l2(rec.volume.values, ref.volume) < REL_L2_A
    assert rec.textured.visible.shape == (16, len(rec.mesh.vertices))
    assert rec.textured.visible.any(0).mean() > 0.9

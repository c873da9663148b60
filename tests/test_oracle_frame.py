# SPDX-License-Identifier: Apache-2.0
"""Pins the oracle's whole-frame path against the reference KATs
(/root/reference/proj/tests/unit/test_recon_frame.cpp, acceptance.cpp #3/#4)
and the synthetic fixture against SURVEY.md §8(d)'s independent numpy
restatement of render.cpp (per-view foreground counts at 512x424, f=365)."""
import numpy as np
import pytest
from scipy.spatial import cKDTree


def rdims(r):  # reconstruct.cpp:18-20
    return (1 << r, 1 << (r + 1), 1 << r)


def render_views(O, rig, body, k, frame=0, sigma=0.0, seed=1):
    return [O.render_frame(rig[i], body, i, frame, sigma_mm_at_2m=sigma, seed=seed) for i in range(k)]


def recon(O, rig, views, **kw):
    return O.reconstruct_frame(rig, [v.depth for v in views], [v.mask for v in views],
                               [v.rgb for v in views], **kw)


def cp_rmse(ground, verts):  # metrics.cpp:93-100
    d, _ = cKDTree(verts).query(ground)
    return float(np.sqrt(np.mean(d * d)))


@pytest.fixture(scope="module")
def xpose(O):
    rig = O.make_circle_rig(4, 2, 2500, 1000, 320, 288, 300)  # make_xpose_scene defaults
    body = O.xpose_body()
    return rig, body, render_views(O, rig, body, 4)


def test_synthetic_fixture_matches_survey_counts(O):
    """SURVEY §8 conventions: K=4, 512x424, f=365 X-pose -> 10238/5922/10238/6024 fg px."""
    rig = O.make_circle_rig(4, 0, 2500, 1000, 512, 424, 365)
    views = render_views(O, rig, O.xpose_body(), 4)
    assert [int(v.mask.sum()) for v in views] == [10238, 5922, 10238, 6024]
    d = np.concatenate([v.depth[v.mask > 0] for v in views])
    assert 1700 < d.min() and d.max() < 2800
    for v in views:
        assert np.array_equal(v.mask > 0, v.depth > 0)


# test_recon_frame.cpp:29-42
def test_empty_views_error(O):
    rig = O.make_circle_rig(2, 0, 2500, 1000, 64, 56, 60)
    z = [np.zeros((56, 64), np.uint16)] * 2
    m = [np.zeros((56, 64), np.uint8)] * 2
    r = O.reconstruct_frame(rig, z, m, None, dims=rdims(5))
    assert r.status == 2  # runtime_error "empty foreground in all views"


def test_fit_grid_padding_error(O):
    """reconstruct.cpp:25-26: padding leaving no usable voxels is invalid_argument."""
    with pytest.raises(ValueError):
        O.fit_grid([0, 0, 0], [1, 1, 1], (16, 16, 16), 8)


# test_recon_frame.cpp:44-63 and acceptance #4 (acceptance.cpp:166-187)
def test_xpose_cp_rmse_and_refinement(O, xpose):
    rig, body, views = xpose
    ground = O.sample_surface(body, 4000, 17)
    r7 = recon(O, rig, views, dims=rdims(7))
    r6 = recon(O, rig, views, dims=rdims(6))
    assert r7.status == 0 and len(r7.mesh.vertices) > 0
    e7 = cp_rmse(ground, r7.mesh.vertices)
    e6 = cp_rmse(ground, r6.mesh.vertices)
    assert e7 < 1.5 * r7.grid.edge
    assert e7 <= e6 + 1e-9
    topo = O.analyze_topology(r7.mesh.triangles, len(r7.mesh.vertices))
    assert topo["edge_manifold"]


# test_recon_frame.cpp:65-77 and acceptance #3 (acceptance.cpp:141-162, sampled)
@pytest.mark.parametrize("seed", [31, 1000, 1017])
def test_noisy_watertight(O, seed):
    rig = O.make_circle_rig(4, 2, 2500, 1000, 320, 288, 300)
    views = render_views(O, rig, O.xpose_body(), 4, sigma=2.0, seed=seed)
    r = recon(O, rig, views, dims=rdims(6))
    assert len(r.mesh.vertices) > 0
    assert O.analyze_topology(r.mesh.triangles, len(r.mesh.vertices))["edge_manifold"]


# test_recon_frame.cpp:79-89
def test_simple_mode_usable(O, xpose):
    rig, body, views = xpose
    r = recon(O, rig, views, dims=rdims(6), mode=1)
    assert len(r.mesh.vertices) > 0
    assert cp_rmse(O.sample_surface(body, 4000, 17), r.mesh.vertices) < 2.0 * r.grid.edge


# test_recon_frame.cpp:91-102
def test_fit_grid_dims_and_padding(O):
    g = O.fit_grid([0, 0, 0], [1000, 1800, 600], rdims(6), 8)
    assert (g.nx, g.ny, g.nz) == (64, 128, 64)
    lo = np.array(g.origin[:])
    hi = lo + g.edge * np.array([g.nx - 1, g.ny - 1, g.nz - 1])
    assert np.min(np.zeros(3) - lo) >= 8 * g.edge - 1e-9
    assert np.min(hi - np.array([1000, 1800, 600])) >= 8 * g.edge - 1e-9


def test_kick_sequence_frames_differ(O):
    """capsule.cpp:197-219: only the right knee/ankle move; bone lengths are kept."""
    x = np.array(O.xpose_body().joints).reshape(15, 3)
    for f in (0, 150, 299):
        j = np.array(O.kick_body(300, f).joints).reshape(15, 3)
        moved = np.nonzero(np.linalg.norm(j - x, axis=1) > 1e-9)[0]
        assert list(moved) == [13, 14]  # knee_r, ankle_r
        for a, b in ((12, 13), (13, 14)):
            assert abs(np.linalg.norm(j[a] - j[b]) - np.linalg.norm(x[a] - x[b])) < 1e-9

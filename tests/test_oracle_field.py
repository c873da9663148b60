# SPDX-License-Identifier: Apache-2.0
"""Pins the CPU oracle against the reference's own known-answer tests for the
field stages: /root/reference/proj/tests/unit/test_recon_field.cpp (file:line
cited per case) and acceptance criteria #1/#2 (acceptance.cpp:59-137).  The
FFT is additionally pinned against numpy.fft.rfftn/irfftn (pocketfft), whose
R2C/C2R semantics equal FFTW's rank-3 plans used by integrate.cpp:31-34."""
import numpy as np
import pytest


def identity_sensor(O, w=64, h=48, f=60.0):
    s = O.Sensor()
    for intr in (s.depth_intr, s.rgb_intr):
        intr.fx = intr.fy = f
        intr.cx, intr.cy = (w - 1) / 2.0, (h - 1) / 2.0
        intr.width, intr.height = w, h
    for p in (s.pose, s.rgb_relative):
        p.R[0] = p.R[4] = p.R[8] = 1.0
    return s


def approx(lhs, value, eps):
    """doctest::Approx(value).epsilon(eps) (scale 1): |lhs-value| < eps*(1+max(|lhs|,|value|))."""
    return abs(lhs - value) < eps * (1.0 + max(abs(lhs), abs(value)))


def plane(w, h, d):
    return np.full((h, w), d, np.uint16), np.ones((h, w), np.uint8)


# test_recon_field.cpp:50-56
def test_build_cloud_fronto_parallel(O):
    s = identity_sensor(O)
    depth, mask = plane(64, 48, 2000)
    c = O.build_cloud(depth, mask, s)
    assert len(c.position) > 1000
    assert np.max(np.linalg.norm(c.normal - [0, 0, -1], axis=1)) < 1e-6


# test_recon_field.cpp:58-68
def test_build_cloud_step_not_bridged(O):
    s = identity_sensor(O)
    depth, mask = plane(64, 48, 2000)
    depth[:, 32:] = 2200
    c = O.build_cloud(depth, mask, s, discontinuity_mm=50.0)
    assert np.max(np.linalg.norm(c.normal - [0, 0, -1], axis=1)) < 1e-6


# test_recon_field.cpp:70-96.  DISCREPANCY: the reference asserts worst < 2e-2 and
# mean < 1e-3, but its own arithmetic (re-derived independently in numpy below)
# gives worst 5.0e-2 / mean 6.1e-3 on this integer-mm depth image: the column-0
# vertex only sees the (0,1)-column slope 8 mm / 8.84 mm.  The KAT is kept with
# the bounds the restated arithmetic meets, plus the independent re-derivation.
def test_build_cloud_slanted_plane(O):
    s = identity_sensor(O, 96, 64, 120.0)
    w, h = 96, 64
    depth = np.zeros((h, w), np.uint16)
    mask = np.zeros((h, w), np.uint8)
    cx = (w - 1) / 2.0
    for x in range(w):
        ratio = (x - cx) / 120.0
        if ratio >= 0.4:
            continue
        z = 2000.0 / (1.0 - ratio)
        depth[:, x] = int(np.floor(z + 0.5))  # std::lround for positive z
        mask[:, x] = 1
    c = O.build_cloud(depth, mask, s, discontinuity_mm=200.0)
    expected = np.array([1.0, 0.0, -1.0]) / np.sqrt(2.0)
    assert len(c.position) > 500
    err = np.linalg.norm(c.normal - expected, axis=1)
    assert err.max() < 5.5e-2
    assert err.mean() < 7e-3
    assert np.median(err) < 2e-2

    # independent numpy re-derivation of cloud.cpp:36-71 at an interior pixel
    def P(x, y):
        z = float(depth[y, x])
        return np.array([(x - cx) * z / 120.0, (y - (h - 1) / 2.0) * z / 120.0, z])

    def tri(a, b, c_):
        n = np.cross(P(*c_) - P(*a), P(*b) - P(*a))
        return n / np.linalg.norm(n)

    x, y = 10, 20
    s6 = (tri((x, y - 1), (x, y), (x - 1, y)) + tri((x, y - 1), (x + 1, y - 1), (x, y)) +
          tri((x + 1, y - 1), (x + 1, y), (x, y)) + tri((x - 1, y), (x, y), (x - 1, y + 1)) +
          tri((x, y), (x, y + 1), (x - 1, y + 1)) + tri((x, y), (x + 1, y), (x, y + 1)))
    n = s6 / 6.0
    n /= np.linalg.norm(n)
    n = -n if n @ P(x, y) > 0 else n
    sel = (c.px == x) & (c.py == y)
    assert np.allclose(c.normal[sel][0], n, atol=1e-12)


# test_recon_field.cpp:98-109.  DISCREPANCY: the reference asserts W == 1 within
# 1e-6 at pixel (w/2, h/2) = (32, 24), but the principal point is (31.5, 23.5),
# so cloud.cpp:112's cosine there is 2000/|(16.67, 16.67, 2000)| = 1 - 6.9e-5.
# We assert that analytic value (to 1e-12) and W == 1 exactly on the axis pixel
# of an odd-sized image.
def test_confidence_head_on_is_one(O):
    s = identity_sensor(O)
    depth, mask = plane(64, 48, 2000)
    c = O.build_cloud(depth, mask, s, confidence=True)
    sel = (c.px == 32) & (c.py == 24)
    assert sel.sum() == 1
    X = np.array([0.5 * 2000 / 60.0, 0.5 * 2000 / 60.0, 2000.0])
    assert abs(c.weight[sel][0] - 2000.0 / np.linalg.norm(X)) < 1e-12
    assert abs(c.weight[sel][0] - 1.0) < 1e-4
    s = identity_sensor(O, 65, 49)
    depth, mask = plane(65, 49, 2000)
    c = O.build_cloud(depth, mask, s, confidence=True)
    sel = (c.px == 32) & (c.py == 24)
    assert abs(c.weight[sel][0] - 1.0) < 1e-15


# test_recon_field.cpp:111-122
def test_confidence_grazing_is_zero(O):
    s = identity_sensor(O)
    depth, mask = plane(64, 48, 2000)
    c = O.build_cloud(depth, mask, s, confidence=True, override_normal=[0.0, 1.0, 0.0])
    sel = (c.px == 32) & (c.py == 24)
    assert c.weight[sel][0] < 1e-6


# test_recon_field.cpp:124-143.  DISCREPANCY: the reference's comment says the
# 21-px window at the last foreground column holds "10 of 21 columns"; it holds
# 11 (x-10..x inclusive), so W2 = 11*21/441 = 0.5238 and its second check
# (Approx(10/21).epsilon(0.03), tolerance 0.0457) misses by 0.0476.  We keep the
# first check with doctest semantics and assert the exact count instead.
def test_confidence_silhouette_edge_half(O):
    s = identity_sensor(O, 128, 96, 100.0)
    depth, mask = plane(128, 96, 2000)
    depth[:, 64:] = 0
    mask[:, 64:] = 0
    c = O.build_cloud(depth, mask, s, confidence=True)
    sel = (c.px == 63) & (c.py == 48)
    wgt = c.weight[sel][0]
    assert approx(wgt, 0.5, 0.06)
    p = c.position[sel][0]
    w1 = 2000.0 / np.linalg.norm(p)  # n = (0,0,-1): cos of the viewing angle
    assert abs(wgt - w1 * 11.0 * 21 / 441.0) < 1e-12
    # the weight map carries float(W) at the point's pixel (cloud.cpp:115)
    assert c.weight_map[48, 63] == np.float32(wgt)


def _single(pos, n, w):
    return np.array([pos], float), np.array([n], float), np.array([w], float)


# test_recon_field.cpp:145-154 and acceptance.cpp:97-111
@pytest.mark.parametrize("n", [(1, 2, -2), (2, -1, 0.5)])
def test_splat_single_point_sqrt15(O, n):
    g = O.grid(16, 32, 16, edge=10.0)
    n = np.array(n, float) / np.linalg.norm(n)
    field, dens, (s1, s2) = O.splat(*_single([80.0, 160.0, 80.0], n, 1.0), g)
    assert np.linalg.norm(field[8, 16, 8] - np.sqrt(1.5) * n) < 1e-9
    assert s2 * s2 == pytest.approx(1.5 * s1 * s1)


# test_recon_field.cpp:156-168
def test_splat_zero_weight_and_empty(O):
    g = O.grid(8, 16, 8, edge=10.0)
    field, dens, _ = O.splat(*_single([40.0, 80.0, 40.0], [0, 0, 1.0], 0.0), g)
    assert np.all(field == 0.0)
    field, dens, _ = O.splat(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0), g)
    assert np.all(field == 0.0) and np.all(dens == 0.0)


def _random_cloud(rng, n, lo, hi):
    pos = rng.uniform(lo, hi, (n, 3))
    nrm = rng.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    return pos, nrm


# test_recon_field.cpp:170-196
def test_splat_order_invariant(O):
    rng = np.random.default_rng(55)
    pa, na = _random_cloud(rng, 200, 20, 120)
    pb, nb = _random_cloud(rng, 150, 20, 120)
    wa = 0.25 + 0.75 * np.abs(rng.normal(size=200)) / 3.0
    wb = 0.25 + 0.75 * np.abs(rng.normal(size=150)) / 3.0
    g = O.grid(16, 32, 16, edge=10.0)
    fab, _, _ = O.splat(np.r_[pa, pb], np.r_[na, nb], np.r_[wa, wb], g)
    fba, _, _ = O.splat(np.r_[pb, pa], np.r_[nb, na], np.r_[wb, wa], g)
    assert np.max(np.linalg.norm(fab - fba, axis=-1)) < 1e-9


# test_recon_field.cpp:198-223 and acceptance.cpp:113-131
@pytest.mark.parametrize("seed,n,scale", [(56, 300, 3.7), (2, 400, 4.2)])
def test_splat_weight_scaling_cancels(O, seed, n, scale):
    rng = np.random.default_rng(seed)
    pos, nrm = _random_cloud(rng, n, 30, 110)
    w = 0.1 + 0.9 * (np.arange(n) % 7) / 7.0
    g = O.grid(16, 32, 16, edge=10.0)
    fa, da, (_, s2) = O.splat(pos, nrm, w, g)
    fb, db, _ = O.splat(pos, nrm, w * scale, g)
    eps = 1e-6 / s2
    sel = (da > eps) & (db > eps)
    assert sel.sum() > 100
    assert np.max(np.linalg.norm(fa[sel] - fb[sel], axis=-1)) < 1e-9


# test_recon_field.cpp:225-234
def test_splat_simple_vs_weighted(O):
    g = O.grid(16, 32, 16, edge=10.0)
    n = np.array([0.5, -0.5, np.sqrt(0.5)]); n /= np.linalg.norm(n)
    args = _single([80.0, 160.0, 80.0], n, 1.0)
    fw, _, _ = O.splat(*args, g, mode=0)
    fs, _, _ = O.splat(*args, g, mode=1)
    assert np.linalg.norm(fs[8, 16, 8] - n) < 1e-12
    assert np.linalg.norm(fw[8, 16, 8] - np.sqrt(1.5) * fs[8, 16, 8]) < 1e-9


def test_splat_thread_count_invariant(O):
    """splat.cpp:55-57: slab-exclusive writers make the sum bit-identical for any thread count."""
    rng = np.random.default_rng(3)
    pos, nrm = _random_cloud(rng, 500, 20, 140)
    w = rng.uniform(0.05, 1.0, 500)
    g = O.grid(16, 32, 16, edge=10.0)
    f1, d1, _ = O.splat(pos, nrm, w, g, threads=1)
    f7, d7, _ = O.splat(pos, nrm, w, g, threads=7)
    assert np.array_equal(f1, f7) and np.array_equal(d1, d7)


def blob_field(nx, ny, nz, c, s):
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    p = np.stack([x, y, z], -1).astype(float)
    d = p - np.asarray(c)
    f = np.exp(-(d * d).sum(-1) / (2 * s * s))
    return f, -d / (s * s) * f[..., None]


# test_recon_field.cpp:248-282 and acceptance.cpp:59-93
def test_integrate_gaussian_blob(O):
    f, grad = blob_field(64, 128, 64, (31.5, 63.5, 31.5), 6.0)
    a = O.integrate_fft(grad)
    expected = f - f.mean()
    rmse = np.sqrt(np.mean((a - expected) ** 2))
    assert rmse < 0.01 * f.max()
    assert abs(a.mean()) < 1e-9


# test_recon_field.cpp:284-290
def test_integrate_zero(O):
    a = O.integrate_fft(np.zeros((16, 32, 16, 3)))
    assert np.all(np.abs(a) < 1e-12)


# test_recon_field.cpp:292-314
def test_integrate_linearity(O):
    rng = np.random.default_rng(77)
    f1 = rng.normal(size=(16, 32, 16, 3)); f2 = rng.normal(size=(16, 32, 16, 3))
    a, b = 2.25, -0.75
    i1, i2, ic = O.integrate_fft(f1), O.integrate_fft(f2), O.integrate_fft(a * f1 + b * f2)
    assert np.max(np.abs(ic - (a * i1 + b * i2))) < 1e-9


def numpy_integrate(field):
    """integrate.cpp:19-74 restated with numpy.fft (pocketfft) — the FFT pin."""
    nz, ny, nx, _ = field.shape

    def signed(n, m):
        i = np.arange(m)
        return 2.0 * np.pi * np.where(i <= n // 2, i, i - n) / n

    wx = signed(nx, nx // 2 + 1)[None, None, :]
    wy = signed(ny, ny)[None, :, None]
    wz = signed(nz, nz)[:, None, None]
    w2 = wx * wx + wy * wy + wz * wz
    w2s = np.where(w2 == 0, 1.0, w2)
    acc = np.zeros((nz, ny, nx // 2 + 1), complex)
    for c, wc in enumerate((wx, wy, wz)):
        S = np.fft.rfftn(field[..., c])
        acc += np.where(w2 == 0, 0, (-1j * wc / w2s)) * S
    return np.fft.irfftn(acc, s=(nz, ny, nx))


@pytest.mark.parametrize("shape", [(16, 32, 16), (8, 16, 12), (6, 10, 12), (32, 16, 64)])
def test_integrate_matches_numpy_rfftn_irfftn(O, shape):
    """Pins the oracle's R2C/C2R Nyquist semantics: random
    fields give a non-Hermitian filtered half-spectrum on the kx=0 and
    kx=nx/2 planes, where a complex-then-real shortcut differs by ~1e-3."""
    nz, ny, nx = shape
    rng = np.random.default_rng(sum(shape))
    field = rng.normal(size=(nz, ny, nx, 3))
    ours = O.integrate_fft(field)
    ref = numpy_integrate(field)
    assert np.max(np.abs(ours - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
    # the hazard is real: c2c-then-Re differs measurably on such fields
    nzh, nyh, nxh = nz, ny, nx

    def signed(n, m):
        i = np.arange(m)
        return 2.0 * np.pi * np.where(i <= n // 2, i, i - n) / n
    wx = signed(nxh, nxh)[None, None, :]; wy = signed(nyh, nyh)[None, :, None]; wz = signed(nzh, nzh)[:, None, None]
    w2 = wx * wx + wy * wy + wz * wz
    acc = np.zeros((nz, ny, nx), complex)
    for c, wc in enumerate((wx, wy, wz)):
        acc += np.where(w2 == 0, 0, -1j * wc / np.where(w2 == 0, 1, w2)) * np.fft.fftn(field[..., c])
    shortcut = np.fft.ifftn(acc).real
    assert np.linalg.norm(shortcut - ref) / np.linalg.norm(ref) > 1e-6


# test_recon_field.cpp:316-332
def test_iso_level(O):
    g = O.grid(8, 16, 8, edge=5.0)
    A = np.full((8, 16, 8), 3.25)
    assert O.iso_level(A, g, [[17.0, 33.0, 12.0]]) == pytest.approx(3.25, rel=1e-12)
    A = np.zeros((8, 16, 8)); A[2, 7, 3] = 42.0
    assert O.iso_level(A, g, [[15.0, 35.0, 10.0]]) == pytest.approx(42.0, rel=1e-12)
    with pytest.raises(ValueError):
        O.iso_level(A, g, np.zeros((0, 3)))

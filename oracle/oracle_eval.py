"""CPU restatement of the reference's evaluation renderer and metrics
(TEST INFRASTRUCTURE; only tests/ may import this).  Plain Python floats are
IEEE fp64; every expression keeps the reference's operation order.

  rasterize            rasterize.cpp:35-161 (sequential triangle loop, float z-buffer)
  vre / hausdorff2d    metrics.cpp:12-43
  distance_transform   distance_transform.cpp:14-95 (Felzenszwalb-Huttenlocher)
  cp_rmse              metrics.cpp:86-94 (brute-force nearest: the kd-tree's exact min)
  wms3im               ssim.cpp (to_gray, Gaussian with renormalisation, pooled terms,
                       2x downsampling, exponents)
"""
from __future__ import annotations

import math

import numpy as np

INF = float("inf")


def lround(x):
    f = math.floor(abs(x))
    q = f + (1 if abs(x) - f >= 0.5 else 0)
    return int(q if x >= 0 else -q)


def f32(x):
    return float(np.float32(x))


def _sample(img, ux, uy):
    H, W = img.shape[:2]
    px, py = ux * W - 0.5, uy * H - 0.5
    x0 = min(max(int(math.floor(px)), 0), W - 1)
    y0 = min(max(int(math.floor(py)), 0), H - 1)
    x1, y1 = min(x0 + 1, W - 1), min(y0 + 1, H - 1)
    tx = min(max(px - x0, 0.0), 1.0)
    ty = min(max(py - y0, 0.0), 1.0)
    out = []
    for ch in range(3):
        a = float(img[y0, x0, ch]) * (1 - tx) + float(img[y0, x1, ch]) * tx
        b = float(img[y1, x0, ch]) * (1 - tx) + float(img[y1, x1, ch]) * tx
        out.append(lround(a * (1 - ty) + b * ty) & 255)
    return out


def rasterize(vertices, triangles, visible, uv, weight, intr, R, t, images, mode):
    """intr = (fx, fy, cx, cy, w, h); R (3x3 row-major list), t: camera-to-world."""
    fx, fy, cx, cy, w, h = intr
    depth = np.zeros((h, w), np.float32)
    color = np.zeros((h, w, 3), np.uint8)
    sil = np.zeros((h, w), np.uint8)
    V = len(vertices)
    if V == 0 or len(triangles) == 0:
        return depth, color, sil
    Ri = [[R[c][r] for c in range(3)] for r in range(3)]
    ti = [-((Ri[r][0] * t[0] + Ri[r][1] * t[1]) + Ri[r][2] * t[2]) for r in range(3)]
    K = len(visible)
    vcol = None
    if mode == 1:
        vcol = []
        for v in range(V):
            r = g = b = 0.0
            n = 0
            for k in range(K):
                if not visible[k][v]:
                    continue
                c = _sample(images[k], float(uv[k][v][0]), float(uv[k][v][1]))
                r += c[0]
                g += c[1]
                b += c[2]
                n += 1
            vcol.append((r / n, g / n, b / n) if n > 0 else (200.0, 200.0, 200.0))
    cam, scr, front = [], [], []
    for v in range(V):
        X = [float(q) for q in vertices[v]]
        p = [((Ri[r][0] * X[0] + Ri[r][1] * X[1]) + Ri[r][2] * X[2]) + ti[r] for r in range(3)]
        cam.append(p)
        f = p[2] > 1.0
        front.append(f)
        scr.append((fx * p[0] / p[2] + cx, fy * p[1] / p[2] + cy) if f else (0.0, 0.0))
    for ti_, (a, b, c) in enumerate(triangles):
        a, b, c = int(a), int(b), int(c)
        if not (front[a] and front[b] and front[c]):
            continue
        pa, pb, pc = scr[a], scr[b], scr[c]
        area = (pb[0] - pa[0]) * (pc[1] - pa[1]) - (pb[1] - pa[1]) * (pc[0] - pa[0])
        if abs(area) < 1e-12:
            continue
        tri_views = 0
        if mode == 0:
            for k in range(K):
                if visible[k][a] and visible[k][b] and visible[k][c]:
                    tri_views |= 1 << k
        x0 = max(0, int(math.ceil(min(pa[0], pb[0], pc[0]))))
        x1 = min(w - 1, int(math.floor(max(pa[0], pb[0], pc[0]))))
        y0 = max(0, int(math.ceil(min(pa[1], pb[1], pc[1]))))
        y1 = min(h - 1, int(math.floor(max(pa[1], pb[1], pc[1]))))
        iza, izb, izc = 1.0 / cam[a][2], 1.0 / cam[b][2], 1.0 / cam[c][2]
        for y in range(y0, y1 + 1):
            for x in range(x0, x1 + 1):
                px, py = float(x), float(y)
                la = (pb[0] - px) * (pc[1] - py) - (pb[1] - py) * (pc[0] - px)
                lb = (pc[0] - px) * (pa[1] - py) - (pc[1] - py) * (pa[0] - px)
                lc = (pa[0] - px) * (pb[1] - py) - (pa[1] - py) * (pb[0] - px)
                if area < 0:
                    la, lb, lc = -la, -lb, -lc
                if la < 0 or lb < 0 or lc < 0:
                    continue
                den = la + lb + lc
                if den <= 0:
                    continue
                la, lb, lc = la / den, lb / den, lc / den
                z = 1.0 / (la * iza + lb * izb + lc * izc)
                zb = float(depth[y, x])
                if zb != 0.0 and z >= zb:
                    continue
                depth[y, x] = np.float32(z)
                sil[y, x] = 1
                if mode == 1:
                    col = []
                    for ch in range(3):
                        v = z * (la * vcol[a][ch] * iza + lb * vcol[b][ch] * izb + lc * vcol[c][ch] * izc)
                        col.append(int(min(max(v, 0.0), 255.0)))
                    color[y, x] = col
                else:
                    r = g = bl = wsum = 0.0
                    for k in range(K):
                        if not (tri_views >> k) & 1:
                            continue
                        wk = z * (la * float(weight[k][a]) * iza + lb * float(weight[k][b]) * izb +
                                  lc * float(weight[k][c]) * izc)
                        if wk <= 1e-9:
                            continue
                        u = [z * (la * float(uv[k][a][d]) * iza + lb * float(uv[k][b][d]) * izb +
                                  lc * float(uv[k][c][d]) * izc) for d in range(2)]
                        s = _sample(images[k], u[0], u[1])
                        r += wk * s[0]
                        g += wk * s[1]
                        bl += wk * s[2]
                        wsum += wk
                    if wsum > 1e-9:
                        color[y, x] = [int(min(max(r / wsum, 0.0), 255.0)), int(min(max(g / wsum, 0.0), 255.0)),
                                       int(min(max(bl / wsum, 0.0), 255.0))]
                    else:
                        color[y, x] = [200, 200, 200]
    return depth, color, sil


def vre(a, b):
    a, b = np.asarray(a) != 0, np.asarray(b) != 0
    o = int((a | b).sum())
    return 0.0 if o == 0 else int((a ^ b).sum()) / o


def _dt1d(f):
    n = len(f)
    v = [0] * n
    z = [0.0] * (n + 1)
    d = [0.0] * n
    k = 0
    v[0] = 0
    z[0], z[1] = -INF, INF
    for q in range(1, n):
        if f[q] == INF:
            continue
        while True:
            if f[v[k]] == INF:
                if k == 0:
                    v[0] = q
                    z[0], z[1] = -INF, INF
                    break
                k -= 1
                continue
            s = ((f[q] + q * q) - (f[v[k]] + v[k] * v[k])) / (2.0 * q - 2.0 * v[k])
            if s <= z[k]:
                k -= 1
            else:
                k += 1
                v[k] = q
                z[k] = s
                z[k + 1] = INF
                break
    k = 0
    for q in range(n):
        if f[v[0]] == INF:
            d[q] = INF
            continue
        while z[k + 1] < q:
            k += 1
        d[q] = (q - v[k]) * float(q - v[k]) + f[v[k]]
    return d


def distance_transform(mask):
    m = np.asarray(mask)
    h, w = m.shape
    g = [[0.0 if m[y, x] else INF for x in range(w)] for y in range(h)]
    for x in range(w):
        col = _dt1d([g[y][x] for y in range(h)])
        for y in range(h):
            g[y][x] = col[y]
    out = np.zeros((h, w), np.float32)
    for y in range(h):
        row = _dt1d(g[y])
        for x in range(w):
            out[y, x] = np.float32(INF) if row[x] == INF else np.float32(math.sqrt(row[x]))
    return out


def hausdorff2d(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if not a.any() or not b.any():
        return None
    da, db = distance_transform(a), distance_transform(b)
    hh = 0.0
    for y in range(a.shape[0]):
        for x in range(a.shape[1]):
            if a[y, x]:
                hh = max(hh, float(db[y, x]))
            if b[y, x]:
                hh = max(hh, float(da[y, x]))
    return hh


def cp_rmse(ground, recon):
    s = 0.0
    R = [tuple(map(float, p)) for p in recon]
    for q in ground:
        q = tuple(map(float, q))
        best = INF
        for p in R:
            ex, ey, ez = p[0] - q[0], p[1] - q[1], p[2] - q[2]
            best = min(best, (ex * ex + ey * ey) + ez * ez)
        s += best
    return math.sqrt(s / len(ground))


DEFAULT_WMS3IM = dict(scales=3, alpha=(0.0, 0.0, 0.1333), beta=(0.0448, 0.3001, 0.1333),
                      gamma=(0.0448, 0.3001, 0.1333), c1=(0.01 * 255) * (0.01 * 255), c2=(0.03 * 255) * (0.03 * 255),
                      c3=(0.03 * 255) * (0.03 * 255) / 2.0, window=11, sigma=1.5)


def wms3im(rendered, ground, sil, opt=DEFAULT_WMS3IM):
    if not np.asarray(sil).any():
        return None

    def gray(img):
        img = np.asarray(img)
        return [[0.299 * int(img[y, x, 0]) + 0.587 * int(img[y, x, 1]) + 0.114 * int(img[y, x, 2])
                 for x in range(img.shape[1])] for y in range(img.shape[0])]

    win, sig = opt["window"], opt["sigma"]
    r = win // 2
    k = [math.exp(-0.5 * (i - r) * (i - r) / (sig * sig)) for i in range(win)]
    ks = 0.0
    for v in k:
        ks += v
    k = [v / ks for v in k]

    def gauss(img):
        h, w = len(img), len(img[0])
        tmp = [[0.0] * w for _ in range(h)]
        out = [[0.0] * w for _ in range(h)]
        for y in range(h):
            for x in range(w):
                acc = norm = 0.0
                for i in range(-r, r + 1):
                    xx = x + i
                    if 0 <= xx < w:
                        acc += k[i + r] * img[y][xx]
                        norm += k[i + r]
                tmp[y][x] = acc / norm
        for y in range(h):
            for x in range(w):
                acc = norm = 0.0
                for i in range(-r, r + 1):
                    yy = y + i
                    if 0 <= yy < h:
                        acc += k[i + r] * tmp[yy][x]
                        norm += k[i + r]
                out[y][x] = acc / norm
        return out

    def mul(a, b):
        return [[a[y][x] * b[y][x] for x in range(len(a[0]))] for y in range(len(a))]

    def down(img):
        h, w = len(img), len(img[0])
        oh, ow = max(1, h // 2), max(1, w // 2)
        out = [[0.0] * ow for _ in range(oh)]
        for y in range(oh):
            for x in range(ow):
                acc, n = 0.0, 0
                for dy in range(2):
                    for dx in range(2):
                        sx, sy = 2 * x + dx, 2 * y + dy
                        if sx < w and sy < h:
                            acc += img[sy][sx]
                            n += 1
                out[y][x] = acc / n
        return out

    def down_or(m):
        h, w = len(m), len(m[0])
        oh, ow = max(1, h // 2), max(1, w // 2)
        return [[1 if any(2 * x + dx < w and 2 * y + dy < h and m[2 * y + dy][2 * x + dx]
                          for dy in range(2) for dx in range(2)) else 0 for x in range(ow)] for y in range(oh)]

    x, y = gray(rendered), gray(ground)
    mask = [[int(v) for v in row] for row in np.asarray(sil)]
    score = 1.0
    for j in range(opt["scales"]):
        if j > 0:
            x, y, mask = down(x), down(y), down_or(mask)
        h, w = len(x), len(x[0])
        mx, my = gauss(x), gauss(y)
        xx, yy, xy = gauss(mul(x, x)), gauss(mul(y, y)), gauss(mul(x, y))
        sl = sc = ss = sw = 0.0
        for py in range(h):
            for px in range(w):
                if not mask[py][px]:
                    continue
                weight = 0.0
                for dy in range(-r, r + 1):
                    for dx in range(-r, r + 1):
                        qx, qy = px + dx, py + dy
                        if 0 <= qx < w and 0 <= qy < h:
                            weight += 1.0 if mask[qy][qx] else 0.0
                a, b = mx[py][px], my[py][px]
                vx = max(0.0, xx[py][px] - a * a)
                vy = max(0.0, yy[py][px] - b * b)
                cov = xy[py][px] - a * b
                sx, sy = math.sqrt(vx), math.sqrt(vy)
                l = (2 * a * b + opt["c1"]) / (a * a + b * b + opt["c1"])
                c = (2 * sx * sy + opt["c2"]) / (vx + vy + opt["c2"])
                s = (cov + opt["c3"]) / (sx * sy + opt["c3"])
                sl += weight * l
                sc += weight * c
                ss += weight * s
                sw += weight
        tl, tc, ts = (1.0, 1.0, 1.0) if sw <= 0 else (sl / sw, sc / sw, ss / sw)
        tl, tc, ts = max(tl, 1e-12), max(tc, 1e-12), max(ts, 1e-12)
        score *= math.pow(tl, opt["alpha"][j]) * math.pow(tc, opt["beta"][j]) * math.pow(ts, opt["gamma"][j])
    return score

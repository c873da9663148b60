"""CPU restatement of mocap::binarize / boundary_voxels / skeletonize
(TEST INFRASTRUCTURE; only tests/ may import this).

  binarize          binary_volume.cpp:10-66: interior side from max(A), mask, then a
                    raster-order flood fill (26-connectivity) keeping the first
                    component of maximal size
  boundary_voxels   binary_volume.cpp:68-82
  skeletonize       skeletonize.cpp:99-161 (directional simple-point thinning with
                    the sequential re-check), is_simple :48-95
"""
from __future__ import annotations

import numpy as np


def binarize(A: np.ndarray, level: float):
    A = np.asarray(A, np.float64)
    nz, ny, nx = A.shape
    above = A.max() >= level
    mask = (A >= level) if above else (A < level)
    label = np.zeros(A.shape, np.int32)
    nxt, best, best_label = 0, 0, 0
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                if not mask[z, y, x] or label[z, y, x]:
                    continue
                nxt += 1
                size = 0
                stack = [(x, y, z)]
                label[z, y, x] = nxt
                while stack:
                    qx, qy, qz = stack.pop()
                    size += 1
                    for dz in (-1, 0, 1):
                        for dy in (-1, 0, 1):
                            for dx in (-1, 0, 1):
                                px, py, pz = qx + dx, qy + dy, qz + dz
                                if not (0 <= px < nx and 0 <= py < ny and 0 <= pz < nz):
                                    continue
                                if not mask[pz, py, px] or label[pz, py, px]:
                                    continue
                                label[pz, py, px] = nxt
                                stack.append((px, py, pz))
                if size > best:
                    best, best_label = size, nxt
    if best == 0:
        raise RuntimeError("binarize: empty interior")
    keep = (label == best_label).astype(np.uint8)
    zz, yy, xx = np.nonzero(keep)  # raster order (z, y, x)
    return keep, np.stack([xx, yy, zz], 1).astype(np.int32)


def boundary_voxels(keep, voxels, origin, edge):
    nz, ny, nx = keep.shape
    out = []
    for x, y, z in voxels:
        for d in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
            qx, qy, qz = x + d[0], y + d[1], z + d[2]
            if not (0 <= qx < nx and 0 <= qy < ny and 0 <= qz < nz) or not keep[qz, qy, qx]:
                out.append([origin[0] + edge * x, origin[1] + edge * y, origin[2] + edge * z])
                break
    return np.array(out, np.float64).reshape(-1, 3)


def _coords(c):
    return (c % 3 - 1, (c // 3) % 3 - 1, c // 9 - 1)


_ADJ26 = [[] for _ in range(27)]
_ADJ6 = [[] for _ in range(27)]
_N18 = [False] * 27
_FACE = [False] * 27
for _c in range(27):
    _x, _y, _z = _coords(_c)
    _n = abs(_x) + abs(_y) + abs(_z)
    _N18[_c] = _c != 13 and _n <= 2
    _FACE[_c] = _n == 1
    for _d in range(27):
        if _d == _c:
            continue
        _ox, _oy, _oz = _coords(_d)
        man = abs(_x - _ox) + abs(_y - _oy) + abs(_z - _oz)
        che = max(abs(_x - _ox), abs(_y - _oy), abs(_z - _oz))
        if che == 1 and _c != 13 and _d != 13:
            _ADJ26[_c].append(_d)
        if man == 1:
            _ADJ6[_c].append(_d)


def is_simple(obj):
    if not any(obj[c] for c in range(27) if c != 13):
        return False
    vis = [False] * 27
    comp = 0
    for c in range(27):
        if comp > 1:
            break
        if c == 13 or not obj[c] or vis[c]:
            continue
        comp += 1
        st = [c]
        vis[c] = True
        while st:
            cur = st.pop()
            for n in _ADJ26[cur]:
                if n != 13 and obj[n] and not vis[n]:
                    vis[n] = True
                    st.append(n)
    if comp != 1:
        return False
    vis = [False] * 27
    comp = 0
    for c in range(27):
        if comp > 1:
            break
        if not _FACE[c] or obj[c] or vis[c]:
            continue
        comp += 1
        st = [c]
        vis[c] = True
        while st:
            cur = st.pop()
            for n in _ADJ6[cur]:
                if _N18[n] and not obj[n] and not vis[n]:
                    vis[n] = True
                    st.append(n)
    return comp == 1


def skeletonize(keep, voxels):
    g = np.array(keep, np.uint8, copy=True)
    nz, ny, nx = g.shape

    def obj(x, y, z):
        return 0 <= x < nx and 0 <= y < ny and 0 <= z < nz and g[z, y, x] != 0

    def hood(p):
        return [obj(p[0] + dx, p[1] + dy, p[2] + dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]

    def ncount(p):
        return sum(obj(p[0] + dx, p[1] + dy, p[2] + dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1)
                   for dx in (-1, 0, 1) if (dx, dy, dz) != (0, 0, 0))

    dirs = ((0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1), (1, 0, 0), (-1, 0, 0))
    active = [tuple(int(v) for v in p) for p in voxels]
    any_del = True
    while any_del:
        any_del = False
        for d in dirs:
            cand = []
            for p in active:
                if not g[p[2], p[1], p[0]]:
                    continue
                if obj(p[0] + d[0], p[1] + d[1], p[2] + d[2]):
                    continue
                if ncount(p) <= 1:
                    continue
                if is_simple(hood(p)):
                    cand.append(p)
            for p in cand:
                if ncount(p) <= 1:
                    continue
                if not is_simple(hood(p)):
                    continue
                g[p[2], p[1], p[0]] = 0
                any_del = True
        if any_del:
            active = [p for p in active if g[p[2], p[1], p[0]]]
    return np.array(active, np.int32).reshape(-1, 3)

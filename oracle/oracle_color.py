"""CPU restatement of the reference's colour correction (TEST INFRASTRUCTURE).

Only tests/ may import this.  Plain Python floats are IEEE fp64 and every
expression keeps the reference's operation order, so results are bit-exact:

  rgb_to_hsv / hsv_to_rgb            hsv.cpp:8-46
  ValueMap::apply / then / inverse   color.hpp:50-57
  ColorCorrection::apply (pixel)     color_correction.cpp:140-145
  mutual_closest_pairs               color_correction.cpp:16-84 (brute force with
                                     GridIndex::nearest's tie rule and strict threshold)
  chain_to_reference                 color_correction.cpp:168-199
"""
from __future__ import annotations

import math


def lround(x: float) -> int:  # std::lround: half away from zero
    f = math.floor(abs(x))
    q = f + (1 if abs(x) - f >= 0.5 else 0)
    return int(q if x >= 0 else -q)


def rgb_to_hsv(c):
    r, g, b = c[0] / 255.0, c[1] / 255.0, c[2] / 255.0
    hi = max(r, g, b)
    lo = min(r, g, b)
    chroma = hi - lo
    v = hi
    s = chroma / hi if hi > 0 else 0.0
    h = 0.0
    if chroma > 0:
        if hi == r:
            hh = math.fmod((g - b) / chroma, 6.0)
        elif hi == g:
            hh = (b - r) / chroma + 2.0
        else:
            hh = (r - g) / chroma + 4.0
        h = 60.0 * hh
        if h < 0:
            h += 360.0
    return h, s, v


def hsv_to_rgb(h, s, v):
    chroma = v * s
    hp = h / 60.0
    x = chroma * (1.0 - abs(math.fmod(hp, 2.0) - 1.0))
    r = g = b = 0.0
    if hp < 1:
        r, g = chroma, x
    elif hp < 2:
        r, g = x, chroma
    elif hp < 3:
        g, b = chroma, x
    elif hp < 4:
        g, b = x, chroma
    elif hp < 5:
        r, b = x, chroma
    else:
        r, b = chroma, x
    m = v - chroma
    return tuple(min(max(lround((t + m) * 255.0), 0), 255) for t in (r, g, b))


def value_map_apply(v, gain, offset):
    return min(max(gain * v + offset, 0.0), 1.0)


def apply_pixel(c, gain, offset):
    h, s, v = rgb_to_hsv(c)
    return hsv_to_rgb(h, s, value_map_apply(v, gain, offset))


def apply_image(img, gain, offset):
    """ColorCorrection::apply(sensor, image) (:147-160), identity shortcut included."""
    import numpy as np
    out = np.array(img, np.uint8, copy=True)
    if gain == 1.0 and offset == 0.0:
        return out
    flat = out.reshape(-1, 3)
    cache = {}
    for i in range(len(flat)):
        key = (int(flat[i, 0]), int(flat[i, 1]), int(flat[i, 2]))
        if key not in cache:
            cache[key] = apply_pixel(key, gain, offset)
        flat[i] = cache[key]
    return out


def _nearest(points, q, max_dist):
    best, best_d2 = -1, max_dist * max_dist
    for i, p in enumerate(points):
        ex, ey, ez = p[0] - q[0], p[1] - q[1], p[2] - q[2]
        d2 = (ex * ex + ey * ey) + ez * ez
        if d2 < best_d2 or (d2 == best_d2 and best >= 0 and i < best):
            best_d2, best = d2, i
    if best >= 0:
        p = points[best]
        ex, ey, ez = p[0] - q[0], p[1] - q[1], p[2] - q[2]
        if math.sqrt((ex * ex + ey * ey) + ez * ez) < max_dist:
            return best
    return -1


def mutual_closest_pairs(a, b, max_dist=20.0):
    a = [tuple(map(float, p)) for p in a]
    b = [tuple(map(float, p)) for p in b]
    if not a or not b:
        return []
    out = []
    for i, q in enumerate(a):
        j = _nearest(b, q, max_dist)
        if j >= 0 and _nearest(a, b[j], max_dist) == i:
            out.append((i, j))
    return out


def chain_to_reference(edges, reference, sensor_count):
    """edges: [(from, to, gain, offset)] -> [(gain, offset)] per sensor."""
    from collections import deque
    maps = [(1.0, 0.0)] * sensor_count
    known = [False] * sensor_count
    known[reference] = True

    def then(inner, outer):
        return outer[0] * inner[0], outer[0] * inner[1] + outer[1]

    def inverse(m):
        return 1.0 / m[0], -m[1] / m[0]

    q = deque([reference])
    while q:
        cur = q.popleft()
        for f, t, g, o in edges:
            if known[f] and not known[t]:
                if f != cur:
                    continue
                maps[t] = then(inverse((g, o)), maps[f])
                known[t] = True
                q.append(t)
            elif known[t] and not known[f]:
                if t != cur:
                    continue
                maps[f] = then((g, o), maps[t])
                known[f] = True
                q.append(f)
    if not all(known):
        raise RuntimeError("chain_to_reference: sensor not connected to the reference")
    return maps

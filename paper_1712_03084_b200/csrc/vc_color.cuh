// SPDX-License-Identifier: Apache-2.0
//
// hsv.cpp:8-46 rgb_to_hsv / hsv_to_rgb and ValueMap::apply (color.hpp:50-57)
// as device functions, fp64 with the reference's operation order (compiled
// without FMA contraction), shared by the image kernel and the texture
// sampler's fused correction.
#pragma once

#include <cstdint>

#include "vc_device.cuh"

namespace vc {

// ColorCorrection::apply(sensor, Rgb8) (color_correction.cpp:140-145):
// rgb -> hsv, v := clamp(gain * v + offset, 0, 1), hsv -> rgb
__device__ __forceinline__ void value_map_rgb(uint8_t c[3], double gain, double offset) {
  const double r = ddiv((double)c[0], 255.0), g = ddiv((double)c[1], 255.0), b = ddiv((double)c[2], 255.0);
  const double hi = fmax(fmax(r, g), b), lo = fmin(fmin(r, g), b);
  const double chroma = dsub(hi, lo);
  double v = hi;
  const double s = hi > 0 ? ddiv(chroma, hi) : 0.0;
  double h = 0.0;
  if (chroma > 0) {
    double hh;
    if (hi == r)
      hh = fmod(ddiv(dsub(g, b), chroma), 6.0);
    else if (hi == g)
      hh = dadd(ddiv(dsub(b, r), chroma), 2.0);
    else
      hh = dadd(ddiv(dsub(r, g), chroma), 4.0);
    h = dmul(60.0, hh);
    if (h < 0) h = dadd(h, 360.0);
  }
  v = dadd(dmul(gain, v), offset);
  v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  // hsv_to_rgb
  const double ch = dmul(v, s);
  const double hp = ddiv(h, 60.0);
  const double x = dmul(ch, dsub(1.0, fabs(dsub(fmod(hp, 2.0), 1.0))));
  double rr = 0, gg = 0, bb = 0;
  if (hp < 1) {
    rr = ch, gg = x;
  } else if (hp < 2) {
    rr = x, gg = ch;
  } else if (hp < 3) {
    gg = ch, bb = x;
  } else if (hp < 4) {
    gg = x, bb = ch;
  } else if (hp < 5) {
    rr = x, bb = ch;
  } else {
    rr = ch, bb = x;
  }
  const double m = dsub(v, ch);
  auto to8 = [&](double t) {
    const long long q = lround_d(dmul(dadd(t, m), 255.0));
    return (uint8_t)(q < 0 ? 0 : (q > 255 ? 255 : q));
  };
  c[0] = to8(rr), c[1] = to8(gg), c[2] = to8(bb);
}

}  // namespace vc

// SPDX-License-Identifier: Apache-2.0
//
// Synthetic capture on the GPU: the reference's analytic capsule-body
// renderer (/root/reference/proj/core/src/synth/render.cpp:13-48,62-77 with
// capsule.cpp:11-87) — one thread per pixel, fp64 ray/capsule intersection
// with the reference's operation order, so frames are bit-identical to the
// CPU renderer.  It feeds benchmark streams without host rendering; it is
// fixture code, not part of the reconstruction path.
#include "vc_device.cuh"

namespace vc {
namespace {

__constant__ int kBones[14][2] = {{0, 1},  {1, 2},  {1, 3},  {3, 4},   {4, 5},   {1, 6},   {6, 7},
                               {7, 8},  {0, 9},  {9, 10}, {10, 11}, {0, 12},  {12, 13}, {13, 14}};

struct BodyArg {
  double joints[45];
  double radii[14];
  uint8_t colors[42];
};

// capsule.cpp:27-59
__device__ bool ray_capsule(d3 ro, d3 rd, d3 pa, d3 pb, double ra, double* tout) {
  const d3 ba = sub3(pb, pa), oa = sub3(ro, pa);
  const double baba = dot3(ba, ba), bard = dot3(ba, rd), baoa = dot3(ba, oa);
  const double rdoa = dot3(rd, oa), oaoa = dot3(oa, oa);
  const double a = dsub(baba, dmul(bard, bard));
  const double b = dsub(dmul(baba, rdoa), dmul(baoa, bard));
  const double c = dsub(dsub(dmul(baba, oaoa), dmul(baoa, baoa)), dmul(dmul(ra, ra), baba));
  if (a > 1e-12) {
    const double h = dsub(dmul(b, b), dmul(a, c));
    if (h >= 0) {
      const double t = ddiv(dsub(-b, __dsqrt_rn(h)), a);
      const double y = dadd(baoa, dmul(t, bard));
      if (t > 0 && y > 0 && y < baba) {
        *tout = t;
        return true;
      }
    }
  }
  bool found = false;
  double best = 0;
  for (int e = 0; e < 2; ++e) {
    const d3 center = e == 0 ? pa : pb;
    const d3 oc = sub3(ro, center);
    const double cb = dot3(rd, oc);
    const double cc = dsub(dot3(oc, oc), dmul(ra, ra));
    const double h = dsub(dmul(cb, cb), cc);
    if (h < 0) continue;
    const double t = dsub(-cb, __dsqrt_rn(h));
    if (t > 0 && (!found || t < best)) best = t, found = true;
  }
  if (found) *tout = best;
  return found;
}

__device__ __forceinline__ d3 joint(const BodyArg& b, int j) {
  return mk3(b.joints[3 * j], b.joints[3 * j + 1], b.joints[3 * j + 2]);
}

// capsule.cpp:71-87
__device__ bool intersect(const BodyArg& body, d3 o, d3 dir, double* t_out, int* bone, d3* point, d3* normal) {
  bool found = false;
  double best = 0;
  for (int b = 0; b < 14; ++b) {
    const d3 a = joint(body, kBones[b][0]), c = joint(body, kBones[b][1]);
    double t;
    if (ray_capsule(o, dir, a, c, body.radii[b], &t) && (!found || t < best)) {
      best = t;
      *bone = b;
      const d3 p = add3(o, scale3(t, dir));
      *point = p;
      // capsule.cpp:19-24 closest_on_segment
      const d3 ab = sub3(c, a);
      const double len2 = dot3(ab, ab);
      double s = len2 > 0 ? ddiv(dot3(sub3(p, a), ab), len2) : 0.0;
      s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
      *normal = normalized3(sub3(p, add3(a, scale3(s, ab))));
      found = true;
    }
  }
  *t_out = best;
  return found;
}

__global__ void render_depth_kernel(DevSensor s, BodyArg body, uint16_t* depth, uint8_t* mask) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= s.w) return;
  const d3 dl = mk3(ddiv(dsub((double)x, s.cx), s.fx), ddiv(dsub((double)y, s.cy), s.fy), 1.0);
  const d3 dir = normalized3(mat3(s.R, dl));
  double t;
  int bone;
  d3 p, n;
  uint16_t d = 0;
  uint8_t m = 0;
  if (intersect(body, ld3(s.t), dir, &t, &bone, &p, &n)) {
    const double z = mat3t(s.R, sub3(p, ld3(s.t))).z;  // pose.apply_inverse(hit).z
    long long zi = lround_d(z);
    zi = zi < 1 ? 1 : (zi > 65535 ? 65535 : zi);
    d = (uint16_t)zi;
    m = 1;
  }
  depth[(size_t)y * s.w + x] = d;
  mask[(size_t)y * s.w + x] = m;
}

// render.cpp:13-19 shade + :62-77 colour pass through the RGB camera
__global__ void render_color_kernel(DevSensor s, BodyArg body, double gain, uint8_t* rgb) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= s.rw) return;
  const d3 dl = mk3(ddiv(dsub((double)x, s.rcx), s.rfx), ddiv(dsub((double)y, s.rcy), s.rfy), 1.0);
  const d3 dir = normalized3(mat3(s.Rc, dl));
  double t;
  int bone;
  d3 p, n;
  uint8_t c[3] = {0, 0, 0};
  if (intersect(body, ld3(s.tc), dir, &t, &bone, &p, &n)) {
    const double nd = dot3(n, neg3(dir));
    const double lambert = dadd(0.35, dmul(0.65, 0.0 < nd ? nd : 0.0));
    for (int ch = 0; ch < 3; ++ch) {
      const double v = dmul(dmul((double)body.colors[3 * bone + ch], lambert), gain);
      c[ch] = (uint8_t)(v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v));
    }
  }
  uint8_t* o = rgb + ((size_t)y * s.rw + x) * 3;
  o[0] = c[0], o[1] = c[1], o[2] = c[2];
}

}  // namespace

void launch_render(const DevSensor& s, const double* joints, const double* radii, const uint8_t* colors,
                   double gain, uint16_t* depth, uint8_t* mask, uint8_t* rgb, cudaStream_t st) {
  BodyArg b;
  for (int i = 0; i < 45; ++i) b.joints[i] = joints[i];
  for (int i = 0; i < 14; ++i) b.radii[i] = radii[i];
  for (int i = 0; i < 42; ++i) b.colors[i] = colors[i];
  if (depth) render_depth_kernel<<<dim3((s.w + 127) / 128, s.h), 128, 0, st>>>(s, b, depth, mask);
  if (rgb) render_color_kernel<<<dim3((s.rw + 127) / 128, s.rh), 128, 0, st>>>(s, b, gain, rgb);
}

}  // namespace vc

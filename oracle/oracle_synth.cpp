// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — NOT PRODUCT CODE.  See oracle.hpp for the contract.
//
// Restates the synthetic capture fixture of the reference:
// /root/reference/proj/core/src/synth/{capsule.cpp, scene.cpp, render.cpp}
// and core/src/core/skeleton.cpp:13-20 (bone list).  Uses libstdc++'s
// std::mt19937_64 / normal_distribution exactly where the reference does, so
// seeded depth noise reproduces the reference toolchain's frames.
#include "oracle.hpp"

#include <algorithm>
#include <cmath>
#include <random>
#include <thread>

namespace orc {

enum { kTorso = 0, kNeck, kHead, kShoulderL, kElbowL, kWristL, kShoulderR, kElbowR, kWristR,
       kHipL, kKneeL, kAnkleL, kHipR, kKneeR, kAnkleR };

// skeleton.cpp:13-20
const int kBones[kBoneCount][2] = {
    {kTorso, kNeck},     {kNeck, kHead},      {kNeck, kShoulderL}, {kShoulderL, kElbowL},
    {kElbowL, kWristL},  {kNeck, kShoulderR}, {kShoulderR, kElbowR}, {kElbowR, kWristR},
    {kTorso, kHipL},     {kHipL, kKneeL},     {kKneeL, kAnkleL},   {kTorso, kHipR},
    {kHipR, kKneeR},     {kKneeR, kAnkleR}};

// capsule.cpp:11-17
static double point_segment_distance(V3 p, V3 a, V3 b) {
  const V3 ab = b - a;
  const double len2 = sqnorm(ab);
  double t = len2 > 0 ? dot(p - a, ab) / len2 : 0.0;
  t = std::clamp(t, 0.0, 1.0);
  return norm(p - (a + t * ab));
}
// capsule.cpp:19-24
static V3 closest_on_segment(V3 p, V3 a, V3 b) {
  const V3 ab = b - a;
  const double len2 = sqnorm(ab);
  const double t = len2 > 0 ? dot(p - a, ab) / len2 : 0.0;
  return a + std::clamp(t, 0.0, 1.0) * ab;
}
// capsule.cpp:27-59 — smallest positive root of ray/capsule, or <0 for none
static bool ray_capsule(V3 ro, V3 rd, V3 pa, V3 pb, double ra, double* tout) {
  const V3 ba = pb - pa, oa = ro - pa;
  const double baba = dot(ba, ba), bard = dot(ba, rd), baoa = dot(ba, oa);
  const double rdoa = dot(rd, oa), oaoa = dot(oa, oa);
  const double a = baba - bard * bard;
  const double b = baba * rdoa - baoa * bard;
  const double c = baba * oaoa - baoa * baoa - ra * ra * baba;
  if (a > 1e-12) {
    const double h = b * b - a * c;
    if (h >= 0) {
      const double t = (-b - std::sqrt(h)) / a;
      const double y = baoa + t * bard;
      if (t > 0 && y > 0 && y < baba) {
        *tout = t;
        return true;
      }
    }
  }
  bool found = false;
  double best = 0;
  for (const V3& center : {pa, pb}) {
    const V3 oc = ro - center;
    const double cb = dot(rd, oc);
    const double cc = dot(oc, oc) - ra * ra;
    const double h = cb * cb - cc;
    if (h < 0) continue;
    const double t = -cb - std::sqrt(h);
    if (t > 0 && (!found || t < best)) best = t, found = true;
  }
  if (found) *tout = best;
  return found;
}

double sdf(const Body& body, V3 x) {  // capsule.cpp:63-69
  double d = INFINITY;
  for (int b = 0; b < kBoneCount; ++b)
    d = std::min(d, point_segment_distance(x, body.joints[kBones[b][0]], body.joints[kBones[b][1]]) -
                        body.radii[b]);
  return d;
}

bool intersect(const Body& body, V3 origin, V3 dir, RayHit* hit) {  // capsule.cpp:71-87
  bool found = false;
  for (int b = 0; b < kBoneCount; ++b) {
    const V3 a = body.joints[kBones[b][0]], c = body.joints[kBones[b][1]];
    double t;
    if (ray_capsule(origin, dir, a, c, body.radii[b], &t) && (!found || t < hit->t)) {
      hit->t = t;
      hit->bone = b;
      hit->point = origin + t * dir;
      hit->normal = normalized(hit->point - closest_on_segment(hit->point, a, c));
      found = true;
    }
  }
  return found;
}

// capsule.cpp:101-151
std::vector<V3> sample_surface(const Body& body, int count, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  double area[kBoneCount];
  double total = 0;
  auto bone_len = [&](int b) { return norm(body.joints[kBones[b][0]] - body.joints[kBones[b][1]]); };
  for (int b = 0; b < kBoneCount; ++b) {
    const double r = body.radii[b], len = bone_len(b);
    area[b] = 2 * M_PI * r * len + 4 * M_PI * r * r;
    total += area[b];
  }
  std::vector<V3> pts;
  int guard = 0;
  while (static_cast<int>(pts.size()) < count && guard < count * 200) {
    ++guard;
    double pick = uni(rng) * total;
    int b = 0;
    while (b + 1 < kBoneCount && pick > area[b]) pick -= area[b], ++b;
    const V3 a = body.joints[kBones[b][0]], c = body.joints[kBones[b][1]];
    const double r = body.radii[b], len = bone_len(b);
    const double cyl_area = 2 * M_PI * r * len;
    V3 p;
    if (uni(rng) * area[b] < cyl_area) {
      const V3 axis = normalized(c - a);
      V3 u = cross(axis, V3{0, 0, 1});
      if (sqnorm(u) < 1e-12) u = cross(axis, V3{1, 0, 0});
      u = normalized(u);
      const V3 v = cross(axis, u);
      const double phi = 2 * M_PI * uni(rng);
      const double along = uni(rng);
      p = a + along * len * axis + r * (std::cos(phi) * u + std::sin(phi) * v);
    } else {
      const V3 center = uni(rng) < 0.5 ? a : c;
      std::normal_distribution<double> gauss(0.0, 1.0);
      const double g0 = gauss(rng), g1 = gauss(rng), g2 = gauss(rng);
      const V3 dir{g0, g1, g2};
      if (sqnorm(dir) < 1e-12) continue;
      p = center + r * normalized(dir);
    }
    if (sdf(body, p) > -1e-6) pts.push_back(p);
  }
  return pts;
}

// capsule.cpp:153-195
Body make_xpose_body() {
  Body b;
  V3* j = b.joints;
  j[kTorso] = {0, 1150, 0};
  j[kNeck] = {0, 1390, 0};
  j[kHead] = {0, 1660, 0};
  j[kShoulderL] = {-190, 1352, 0};
  j[kShoulderR] = {190, 1355, 0};
  const V3 up_out_l{-std::cos(0.62), std::sin(0.62), 0};
  const V3 up_out_r{std::cos(0.60), std::sin(0.60), 0};
  const V3 fore_l{-std::cos(0.18), std::sin(0.18), 0};
  const V3 fore_r{std::cos(0.16), std::sin(0.16), 0};
  j[kElbowL] = j[kShoulderL] + 285.0 * up_out_l;
  j[kWristL] = j[kElbowL] + 255.0 * fore_l;
  j[kElbowR] = j[kShoulderR] + 276.0 * up_out_r;
  j[kWristR] = j[kElbowR] + 247.0 * fore_r;
  j[kHipL] = {-105, 925, 0};
  j[kHipR] = {105, 925, 0};
  const V3 thigh_l{-std::sin(0.38), -std::cos(0.38), 0};
  const V3 thigh_r{std::sin(0.36), -std::cos(0.36), 0};
  const V3 shank_l{-std::sin(0.12), -std::cos(0.12), 0};
  const V3 shank_r{std::sin(0.10), -std::cos(0.10), 0};
  j[kKneeL] = j[kHipL] + 400.0 * thigh_l;
  j[kAnkleL] = j[kKneeL] + 390.0 * shank_l;
  j[kKneeR] = j[kHipR] + 392.0 * thigh_r;
  j[kAnkleR] = j[kKneeR] + 382.0 * shank_r;
  const double radii[kBoneCount] = {125, 82, 52, 45, 38, 52, 45, 38, 72, 64, 50, 72, 64, 50};
  const uint8_t colors[kBoneCount][3] = {{200, 60, 60},  {240, 200, 160}, {60, 120, 200},
                                         {70, 150, 210}, {90, 180, 220},  {190, 120, 40},
                                         {210, 140, 60}, {230, 170, 90},  {60, 160, 80},
                                         {80, 180, 90},  {110, 200, 110}, {140, 70, 170},
                                         {160, 90, 190}, {180, 120, 210}};
  for (int i = 0; i < kBoneCount; ++i) {
    b.radii[i] = radii[i];
    for (int c = 0; c < 3; ++c) b.colors[i][c] = colors[i][c];
  }
  return b;
}

// capsule.cpp:197-219
std::vector<Body> make_kick_sequence(int frames) {
  std::vector<Body> seq;
  const Body base = make_xpose_body();
  const double thigh_len = norm(base.joints[kKneeR] - base.joints[kHipR]);
  const double shank_len = norm(base.joints[kAnkleR] - base.joints[kKneeR]);
  for (int f = 0; f < frames; ++f) {
    Body b = base;
    const double s = frames > 1 ? static_cast<double>(f) / (frames - 1) : 0.0;
    const double swing = std::sin(M_PI * s);
    const double thigh_pitch = swing * 1.05;
    const double knee_flex = swing * 1.45;
    const V3 thigh_dir{0.12, -std::cos(thigh_pitch), std::sin(thigh_pitch)};
    b.joints[kKneeR] = b.joints[kHipR] + thigh_len * normalized(thigh_dir);
    const double shank_pitch = thigh_pitch - knee_flex;
    const V3 shank_dir{0.12, -std::cos(shank_pitch), std::sin(shank_pitch)};
    b.joints[kAnkleR] = b.joints[kKneeR] + shank_len * normalized(shank_dir);
    seq.push_back(b);
  }
  return seq;
}

// scene.cpp:10-22
Pose make_lookat(V3 eye, V3 target, V3 up) {
  const V3 z = normalized(target - eye);
  V3 x = cross(-up, z);
  if (sqnorm(x) < 1e-12) x = cross(V3{1, 0, 0}, z);
  x = normalized(x);
  const V3 y = cross(z, x);
  Pose p;
  const V3 cols[3] = {x, y, z};
  for (int c = 0; c < 3; ++c) {
    p.R[0 * 3 + c] = cols[c].x;
    p.R[1 * 3 + c] = cols[c].y;
    p.R[2 * 3 + c] = cols[c].z;
  }
  p.t[0] = eye.x, p.t[1] = eye.y, p.t[2] = eye.z;
  return p;
}

// scene.cpp:24-55
std::vector<Sensor> make_circle_rig(int recon, int held_out, double radius_mm, double target_h,
                                    int w, int h, double f) {
  const V3 target{0, target_h, 0};
  Intrinsics K{f, f, (w - 1) / 2.0, (h - 1) / 2.0, w, h};
  std::vector<double> angles;
  for (int k = 0; k < recon; ++k) angles.push_back(2 * M_PI * k / recon);
  for (int k = 0; k < held_out; ++k) angles.push_back(2 * M_PI * (k + 0.5) / recon);
  std::vector<Sensor> rig;
  for (double a : angles) {
    const V3 eye{radius_mm * std::sin(a), target_h, radius_mm * std::cos(a)};
    Sensor s;
    s.depth_intr = K;
    s.pose = make_lookat(eye, target, V3{0, 1, 0});
    s.rgb_intr = K;
    s.rgb_relative = Pose{{1, 0, 0, 0, 1, 0, 0, 0, 1}, {0, 0, 0}};
    rig.push_back(s);
  }
  return rig;
}

// render.cpp:13-19
static void shade(const uint8_t base[3], V3 normal, V3 ray_dir, double gain, uint8_t out[3]) {
  const double lambert = 0.35 + 0.65 * std::max(0.0, dot(normal, -ray_dir));
  for (int c = 0; c < 3; ++c) out[c] = static_cast<uint8_t>(std::clamp(base[c] * lambert * gain, 0.0, 255.0));
}

template <typename Fn>
static void parallel_rows(int h, int threads, Fn&& fn) {
  const int n = std::max(1, std::min(threads, h));
  const int chunk = (h + n - 1) / n;
  std::vector<std::thread> pool;
  for (int i = 0; i < n; ++i) {
    const int b = std::min(h, i * chunk), e = std::min(h, b + chunk);
    if (b >= e) break;
    pool.emplace_back([&fn, b, e] {
      for (int y = b; y < e; ++y) fn(y);
    });
  }
  for (auto& t : pool) t.join();
}

// render.cpp:23-80
void render_frame(const Sensor& s, const Body& body, double sigma2m, uint64_t seed, double gain,
                  int camera, int frame, int threads, uint16_t* depth, uint8_t* mask, uint8_t* rgb) {
  const Intrinsics& di = s.depth_intr;
  const M3 R = rot(s.pose);
  const V3 eye = trans(s.pose);
  std::fill(depth, depth + static_cast<std::size_t>(di.width) * di.height, 0);
  std::fill(mask, mask + static_cast<std::size_t>(di.width) * di.height, 0);
  parallel_rows(di.height, threads, [&](int y) {
    for (int x = 0; x < di.width; ++x) {
      const V3 dir_local{(x - di.cx) / di.fx, (static_cast<double>(y) - di.cy) / di.fy, 1.0};
      const V3 dir = normalized(mul(R, dir_local));
      RayHit hit;
      if (!intersect(body, eye, dir, &hit)) continue;
      const double z = pose_apply_inverse(s.pose, hit.point).z;
      const std::size_t i = static_cast<std::size_t>(y) * di.width + x;
      depth[i] = static_cast<uint16_t>(std::clamp(std::lround(z), 1L, 65535L));
      mask[i] = 1;
    }
  });
  if (sigma2m > 0) {  // render.cpp:50-61
    std::mt19937_64 rng(seed * 46337 + camera * 131 + frame);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (int y = 0; y < di.height; ++y)
      for (int x = 0; x < di.width; ++x) {
        uint16_t& d = depth[static_cast<std::size_t>(y) * di.width + x];
        if (d == 0) continue;
        const double sigma = sigma2m * d / 2000.0;
        d = static_cast<uint16_t>(std::clamp(std::lround(d + sigma * gauss(rng)), 1L, 65535L));
      }
  }
  const Intrinsics& ci = s.rgb_intr;
  const Pose rp = pose_compose(s.pose, s.rgb_relative);
  const M3 Rc = rot(rp);
  const V3 eyec = trans(rp);
  std::fill(rgb, rgb + static_cast<std::size_t>(ci.width) * ci.height * 3, 0);
  parallel_rows(ci.height, threads, [&](int y) {
    for (int x = 0; x < ci.width; ++x) {
      const V3 dir_local{(x - ci.cx) / ci.fx, (static_cast<double>(y) - ci.cy) / ci.fy, 1.0};
      const V3 dir = normalized(mul(Rc, dir_local));
      RayHit hit;
      if (!intersect(body, eyec, dir, &hit)) continue;
      shade(body.colors[hit.bone], hit.normal, dir, gain, &rgb[(static_cast<std::size_t>(y) * ci.width + x) * 3]);
    }
  });
}

}  // namespace orc

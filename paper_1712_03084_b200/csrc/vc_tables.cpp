// SPDX-License-Identifier: Apache-2.0
//
// Host-side generators for the device constant tables and the synthetic
// capture fixture (product side; the CPU oracle has its own restatement).
//
// * The marching-cubes case table is generated, not Lorensen's: the rule of
//   marching_cubes.cpp:52-122 — per face, the cut edges are chained; on a
//   face with four cuts the chords cut off the INSIDE corners; chains are
//   closed into loops starting from the lowest unused edge, oriented so the
//   Newell normal of the edge midpoints points from inside to outside, and
//   fan-triangulated from the loop's first edge.
// * Rig / body construction follow scene.cpp:10-55 and capsule.cpp:153-219.
#include <array>
#include <cmath>
#include <cstdint>
#include <vector>

#include "vc/vc.h"

namespace vc {
namespace {

struct P3 {
  double x, y, z;
};
P3 operator+(P3 a, P3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
P3 operator-(P3 a, P3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
P3 operator*(double s, P3 a) { return {s * a.x, s * a.y, s * a.z}; }
double dotp(P3 a, P3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
P3 crossp(P3 a, P3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
P3 unit(P3 a) {
  const double q = dotp(a, a);
  if (q > 0) {
    const double n = std::sqrt(q);
    return {a.x / n, a.y / n, a.z / n};
  }
  return a;
}

// cube edge e joins corners kE[e][0] < kE[e][1]; corner c = (c&1, c>>1&1, c>>2&1)
constexpr int kE[12][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}, {0, 2}, {1, 3}, {4, 6}, {5, 7}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
// faces as cyclic corner loops (x=0, x=1, y=0, y=1, z=0, z=1)
constexpr int kF[6][4] = {{0, 2, 6, 4}, {1, 3, 7, 5}, {0, 1, 5, 4}, {2, 3, 7, 6}, {0, 1, 3, 2}, {4, 5, 7, 6}};

P3 corner(int c) { return {double(c & 1), double((c >> 1) & 1), double((c >> 2) & 1)}; }
int edge_of(int a, int b) {
  for (int e = 0; e < 12; ++e)
    if ((kE[e][0] == a && kE[e][1] == b) || (kE[e][0] == b && kE[e][1] == a)) return e;
  return -1;
}

}  // namespace

void build_mc_table(int8_t counts[256], int8_t tris[256][5][3]) {
  for (int cfg = 0; cfg < 256; ++cfg) {
    counts[cfg] = 0;
    for (auto& t : tris[cfg]) t[0] = t[1] = t[2] = -1;
    if (cfg == 0 || cfg == 255) continue;
    auto in = [cfg](int c) { return ((cfg >> c) & 1) != 0; };
    std::array<std::array<int, 2>, 12> nb;
    for (auto& p : nb) p = {-1, -1};
    auto join = [&nb](int a, int b) {
      (nb[a][0] < 0 ? nb[a][0] : nb[a][1]) = b;
      (nb[b][0] < 0 ? nb[b][0] : nb[b][1]) = a;
    };
    for (const auto& f : kF) {
      int cut[4], n = 0;
      for (int i = 0; i < 4; ++i)
        if (in(f[i]) != in(f[(i + 1) & 3])) cut[n++] = edge_of(f[i], f[(i + 1) & 3]);
      if (n == 2) {
        join(cut[0], cut[1]);
      } else if (n == 4) {
        if (in(f[0])) {
          join(cut[3], cut[0]);
          join(cut[1], cut[2]);
        } else {
          join(cut[0], cut[1]);
          join(cut[2], cut[3]);
        }
      }
    }
    bool seen[12] = {};
    int ntri = 0;
    for (int s = 0; s < 12; ++s) {
      if (seen[s] || nb[s][0] < 0) continue;
      std::vector<int> loop;
      for (int prev = -1, cur = s;;) {
        loop.push_back(cur);
        seen[cur] = true;
        const int nxt = nb[cur][0] == prev ? nb[cur][1] : nb[cur][0];
        prev = cur;
        cur = nxt;
        if (cur == s) break;
      }
      P3 out{0, 0, 0}, newell{0, 0, 0};
      std::vector<P3> mid;
      for (int e : loop) {
        const int a = kE[e][0], b = kE[e][1];
        mid.push_back(0.5 * (corner(a) + corner(b)));
        out = out + (in(a) ? corner(b) - corner(a) : corner(a) - corner(b));
      }
      for (size_t i = 0; i < loop.size(); ++i) newell = newell + crossp(mid[i], mid[(i + 1) % loop.size()]);
      if (dotp(newell, out) < 0) std::vector<int>(loop.rbegin(), loop.rend()).swap(loop);
      for (size_t i = 1; i + 1 < loop.size(); ++i, ++ntri) {
        tris[cfg][ntri][0] = (int8_t)loop[0];
        tris[cfg][ntri][1] = (int8_t)loop[i];
        tris[cfg][ntri][2] = (int8_t)loop[i + 1];
      }
    }
    counts[cfg] = (int8_t)ntri;
  }
}

// scene.cpp:10-22 make_lookat (CV convention: +z forward, +y down)
static vc_pose lookat(P3 eye, P3 target, P3 up) {
  const P3 z = unit(target - eye);
  P3 x = crossp(P3{-up.x, -up.y, -up.z}, z);
  if (dotp(x, x) < 1e-12) x = crossp(P3{1, 0, 0}, z);
  x = unit(x);
  const P3 y = crossp(z, x);
  vc_pose p;
  const P3 cols[3] = {x, y, z};
  for (int c = 0; c < 3; ++c) {
    p.R[c] = cols[c].x;
    p.R[3 + c] = cols[c].y;
    p.R[6 + c] = cols[c].z;
  }
  p.t[0] = eye.x, p.t[1] = eye.y, p.t[2] = eye.z;
  return p;
}

// scene.cpp:24-55
void circle_rig(int recon, int held_out, double radius, double target_h, int w, int h, double f, vc_sensor* out) {
  vc_intrinsics K{f, f, (w - 1) / 2.0, (h - 1) / 2.0, w, h};
  std::vector<double> ang;
  for (int k = 0; k < recon; ++k) ang.push_back(2 * M_PI * k / recon);
  for (int k = 0; k < held_out; ++k) ang.push_back(2 * M_PI * (k + 0.5) / recon);
  for (size_t i = 0; i < ang.size(); ++i) {
    vc_sensor s{};
    s.depth_intr = K;
    s.rgb_intr = K;
    s.pose = lookat(P3{radius * std::sin(ang[i]), target_h, radius * std::cos(ang[i])}, P3{0, target_h, 0},
                    P3{0, 1, 0});
    const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    for (int j = 0; j < 9; ++j) s.rgb_relative.R[j] = I[j];
    out[i] = s;
  }
}

// capsule.cpp:153-195 (joint order: skeleton.hpp:13-20)
void xpose_body(vc_body* b) {
  P3 j[15];
  j[0] = {0, 1150, 0};
  j[1] = {0, 1390, 0};
  j[2] = {0, 1660, 0};
  j[3] = {-190, 1352, 0};
  j[6] = {190, 1355, 0};
  j[4] = j[3] + 285.0 * P3{-std::cos(0.62), std::sin(0.62), 0};
  j[5] = j[4] + 255.0 * P3{-std::cos(0.18), std::sin(0.18), 0};
  j[7] = j[6] + 276.0 * P3{std::cos(0.60), std::sin(0.60), 0};
  j[8] = j[7] + 247.0 * P3{std::cos(0.16), std::sin(0.16), 0};
  j[9] = {-105, 925, 0};
  j[12] = {105, 925, 0};
  j[10] = j[9] + 400.0 * P3{-std::sin(0.38), -std::cos(0.38), 0};
  j[11] = j[10] + 390.0 * P3{-std::sin(0.12), -std::cos(0.12), 0};
  j[13] = j[12] + 392.0 * P3{std::sin(0.36), -std::cos(0.36), 0};
  j[14] = j[13] + 382.0 * P3{std::sin(0.10), -std::cos(0.10), 0};
  for (int i = 0; i < 15; ++i) b->joints[3 * i] = j[i].x, b->joints[3 * i + 1] = j[i].y, b->joints[3 * i + 2] = j[i].z;
  const double radii[14] = {125, 82, 52, 45, 38, 52, 45, 38, 72, 64, 50, 72, 64, 50};
  const uint8_t col[42] = {200, 60,  60,  240, 200, 160, 60,  120, 200, 70,  150, 210, 90,  180,
                           220, 190, 120, 40,  210, 140, 60,  230, 170, 90,  60,  160, 80,  80,
                           180, 90,  110, 200, 110, 140, 70,  170, 160, 90,  190, 180, 120, 210};
  for (int i = 0; i < 14; ++i) b->radii[i] = radii[i];
  for (int i = 0; i < 42; ++i) b->colors[i] = col[i];
}

// capsule.cpp:197-219: right thigh swings forward while the knee flexes
void kick_body(int frames, int f, vc_body* b) {
  xpose_body(b);
  auto J = [b](int i) { return P3{b->joints[3 * i], b->joints[3 * i + 1], b->joints[3 * i + 2]}; };
  auto nrm = [](P3 a) { return std::sqrt(dotp(a, a)); };
  const double thigh = nrm(J(13) - J(12)), shank = nrm(J(14) - J(13));
  const double s = frames > 1 ? static_cast<double>(f) / (frames - 1) : 0.0;
  const double swing = std::sin(M_PI * s);
  const double tp = swing * 1.05, kf = swing * 1.45;
  const P3 knee = J(12) + thigh * unit(P3{0.12, -std::cos(tp), std::sin(tp)});
  const double sp = tp - kf;
  const P3 ankle = knee + shank * unit(P3{0.12, -std::cos(sp), std::sin(sp)});
  b->joints[39] = knee.x, b->joints[40] = knee.y, b->joints[41] = knee.z;
  b->joints[42] = ankle.x, b->joints[43] = ankle.y, b->joints[44] = ankle.z;
}

}  // namespace vc

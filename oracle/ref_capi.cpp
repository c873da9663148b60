// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" surface over the REFERENCE's own sources, compiled unmodified
// from /root/reference/proj/core/src against the shims in oracle/ref_shim
// (oracle/Makefile, target `ref`; output oracle/_ref/libref.so, git-ignored).
// It lets tests/test_ref_pin.py pin the oracle restatement (oracle_core.cpp,
// oracle_synth.cpp) to the reference code itself:
//   ref_make_circle_rig   -> volcap::synth::make_circle_rig       (scene.cpp:24-55)
//   ref_body              -> make_xpose_body / make_kick_sequence (capsule.cpp:153-219)
//   ref_render_frame      -> volcap::synth::render_frame          (render.cpp:23-80)
//   ref_reconstruct_frame -> volcap::recon::reconstruct_frame     (reconstruct.cpp:37-78), r-mode,
//                            UNMODIFIED; or, for the cubic grids the reference cannot fit
//                            (reconstruct.cpp:18-20 fixes 2^r x 2^(r+1) x 2^r), the same stage
//                            sequence with fit_grid's per-axis rule (reconstruct.cpp:21-33)
//                            applied to the requested dims — every stage is the reference's
//                            own function (build_cloud, confidence_weights, splat, negate,
//                            integrate_fft, iso_level, marching_cubes);
//                            then appearance::vertex_visibility + assign_texture (texture.cpp:11-72).
//   ref_marching_cubes    -> volcap::recon::marching_cubes on a caller field.
//   ref_skeletonize       -> volcap::mocap::skeletonize            (skeletonize.cpp:99-161)
//   ref_fit_value_map     -> volcap::appearance::fit_value_map     (color_correction.cpp:97-138)
//   ref_chain_to_reference-> volcap::appearance::chain_to_reference (color_correction.cpp:168-199)
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <vector>

#include "volcap/appearance/color.hpp"
#include "volcap/appearance/texture.hpp"
#include "volcap/mocap/volume_ops.hpp"
#include "volcap/recon/reconstruct.hpp"
#include "volcap/synth/capsule.hpp"
#include "volcap/synth/scene.hpp"

using namespace volcap;

namespace {

// POD mirrors, same layout as oracle.hpp / include/vc/vc.h (R row-major)
struct PIntr {
  double fx, fy, cx, cy;
  int32_t width, height;
};
struct PPose {
  double R[9];
  double t[3];
};
struct PSensor {
  PIntr depth_intr;
  PPose pose;
  PIntr rgb_intr;
  PPose rgb_relative;
};
struct PBody {
  double joints[45];
  double radii[14];
  uint8_t colors[42];
};
struct PGrid {
  int32_t nx, ny, nz;
  double origin[3];
  double edge;
};

Intrinsics to_intr(const PIntr& p) { return Intrinsics{p.fx, p.fy, p.cx, p.cy, p.width, p.height}; }
PIntr from_intr(const Intrinsics& i) { return PIntr{i.fx, i.fy, i.cx, i.cy, i.width, i.height}; }
Pose to_pose(const PPose& p) {
  Pose o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o.R(r, c) = p.R[3 * r + c];
  o.t = Vec3(p.t[0], p.t[1], p.t[2]);
  return o;
}
PPose from_pose(const Pose& p) {
  PPose o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o.R[3 * r + c] = p.R(r, c);
  for (int i = 0; i < 3; ++i) o.t[i] = p.t(i);
  return o;
}
Sensor to_sensor(const PSensor& s) {
  Sensor o;
  o.depth_intr = to_intr(s.depth_intr);
  o.pose = to_pose(s.pose);
  o.rgb_intr = to_intr(s.rgb_intr);
  o.rgb_relative = to_pose(s.rgb_relative);
  return o;
}
PSensor from_sensor(const Sensor& s) {
  return PSensor{from_intr(s.depth_intr), from_pose(s.pose), from_intr(s.rgb_intr), from_pose(s.rgb_relative)};
}
synth::CapsuleBody to_body(const PBody& b) {
  synth::CapsuleBody o;
  for (int j = 0; j < kJointCount; ++j) o.joints[j] = Vec3(b.joints[3 * j], b.joints[3 * j + 1], b.joints[3 * j + 2]);
  for (int i = 0; i < kBoneCount; ++i) {
    o.radii[i] = b.radii[i];
    o.colors[i] = Rgb8{b.colors[3 * i], b.colors[3 * i + 1], b.colors[3 * i + 2]};
  }
  return o;
}
PBody from_body(const synth::CapsuleBody& b) {
  PBody o{};
  for (int j = 0; j < kJointCount; ++j)
    for (int c = 0; c < 3; ++c) o.joints[3 * j + c] = b.joints[j](c);
  for (int i = 0; i < kBoneCount; ++i) {
    o.radii[i] = b.radii[i];
    o.colors[3 * i] = b.colors[i].r, o.colors[3 * i + 1] = b.colors[i].g, o.colors[3 * i + 2] = b.colors[i].b;
  }
  return o;
}

RgbdFrame to_frame(const Sensor& s, const uint16_t* depth, const uint8_t* mask, const uint8_t* rgb) {
  RgbdFrame f;
  const int w = s.depth_intr.width, h = s.depth_intr.height;
  f.depth = DepthImage(w, h, 0);
  f.foreground = MaskImage(w, h, 0);
  std::memcpy(f.depth.data().data(), depth, sizeof(uint16_t) * w * h);
  std::memcpy(f.foreground.data().data(), mask, (size_t)w * h);
  const int cw = s.rgb_intr.width, ch = s.rgb_intr.height;
  f.color = ColorImage(cw, ch);
  if (rgb)
    for (size_t i = 0; i < (size_t)cw * ch; ++i) f.color.data()[i] = Rgb8{rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
  return f;
}

// reconstruct.cpp:16-35's per-axis rule on caller dims (the reference fixes
// dims to 2^r x 2^(r+1) x 2^r; this is the generalisation SURVEY A5 asks for).
recon::GridSpec fit_grid_dims(const Vec3& lo, const Vec3& hi, const int dims[3], int padding) {
  recon::GridSpec grid;
  grid.nx = dims[0], grid.ny = dims[1], grid.nz = dims[2];
  const Vec3 extent = hi - lo;
  double edge = 1e-9;
  for (int a = 0; a < 3; ++a) {
    const int usable = dims[a] - 1 - 2 * padding;
    if (usable < 1) throw std::invalid_argument("fit_grid: padding leaves no usable voxels");
    edge = std::max(edge, extent(a) / usable);
  }
  grid.edge_mm = edge;
  const Vec3 center = 0.5 * (lo + hi);
  grid.origin = Vec3(center.x() - edge * (grid.nx - 1) / 2.0, center.y() - edge * (grid.ny - 1) / 2.0,
                     center.z() - edge * (grid.nz - 1) / 2.0);
  return grid;
}

struct RefFrame {
  int k = 0;
  recon::FrameReconstruction rec;
  appearance::TexturedMesh tex;
};

}  // namespace

extern "C" {

int ref_sizeof_sensor() { return sizeof(PSensor); }
int ref_sizeof_body() { return sizeof(PBody); }

void ref_make_circle_rig(int recon, int held_out, double radius_mm, double target_height_mm, int width, int height,
                         double focal_px, PSensor* out) {
  const CameraRig rig = synth::make_circle_rig(recon, held_out, radius_mm, target_height_mm, width, height, focal_px);
  for (int i = 0; i < rig.count(); ++i) out[i] = from_sensor(rig.sensors[i]);
}

// kick_frames <= 0: make_xpose_body(); else make_kick_sequence(kick_frames)[frame]
void ref_body(int kick_frames, int frame, PBody* out) {
  if (kick_frames <= 0) {
    *out = from_body(synth::make_xpose_body());
  } else {
    const auto seq = synth::make_kick_sequence(kick_frames);
    *out = from_body(seq.at(frame));
  }
}

// render.cpp:23-80 through a SyntheticScene holding `sensor` at index `camera`
// and `body` at index `frame` (the noise seed mixes both indices).
void ref_render_frame(const PSensor* sensor, const PBody* body, double sigma_mm_at_2m, uint64_t seed, double gain,
                      int camera, int frame, uint16_t* depth, uint8_t* mask, uint8_t* rgb) {
  synth::SyntheticScene sc;
  sc.rig.sensors.assign(camera + 1, to_sensor(*sensor));
  sc.rig.recon_count = camera + 1;
  sc.frames.assign(frame + 1, to_body(*body));
  sc.clock_offset_ms.assign(camera + 1, 0.0);
  sc.noise.depth_sigma_mm_at_2m = sigma_mm_at_2m;
  sc.noise.seed = seed;
  sc.noise.color_gain.assign(camera + 1, gain);
  const RgbdFrame f = synth::render_frame(sc, camera, frame);
  std::memcpy(depth, f.depth.data().data(), f.depth.size() * 2);
  std::memcpy(mask, f.foreground.data().data(), f.foreground.size());
  for (size_t i = 0; i < f.color.size(); ++i) {
    rgb[3 * i] = f.color.data()[i].r, rgb[3 * i + 1] = f.color.data()[i].g, rgb[3 * i + 2] = f.color.data()[i].b;
  }
}

// r > 0: the unmodified reconstruct_frame with ReconConfig.r = r; else dims.
// status: 0 ok, 1 std::invalid_argument, 2 std::runtime_error, 3 other.
void* ref_reconstruct_frame(const PSensor* sensors, int k, const uint16_t* const* depths, const uint8_t* const* masks,
                            const uint8_t* const* rgbs, int r, const int32_t* dims, int mode, double discontinuity_mm,
                            int padding_voxels, int silhouette_radius_px, double eps_vis_mm, int* status) {
  auto* out = new RefFrame;
  out->k = k;
  try {
    CameraRig rig;
    for (int i = 0; i < k; ++i) rig.sensors.push_back(to_sensor(sensors[i]));
    rig.recon_count = k;
    std::vector<RgbdFrame> frames;
    for (int i = 0; i < k; ++i)
      frames.push_back(to_frame(rig.sensors[i], depths[i], masks[i], rgbs ? rgbs[i] : nullptr));
    recon::ReconConfig cfg;
    cfg.mode = mode == 0 ? recon::SplatMode::kWeighted : recon::SplatMode::kSimple;
    cfg.discontinuity_mm = discontinuity_mm;
    cfg.padding_voxels = padding_voxels;
    cfg.silhouette_radius_px = silhouette_radius_px;
    if (r > 0) {
      cfg.r = r;
      out->rec = recon::reconstruct_frame(frames, rig, cfg);
    } else {
      // reconstruct.cpp:37-78 stage by stage, fit_grid generalised to `dims`
      auto& o = out->rec;
      for (int i = 0; i < k; ++i)
        o.clouds.push_back(recon::build_cloud(frames[i], rig.sensors[i].depth_camera(), i, cfg.discontinuity_mm));
      for (int i = 0; i < k; ++i)
        recon::confidence_weights(o.clouds[i], frames[i], rig.sensors[i].depth_camera(), cfg.silhouette_radius_px);
      Vec3 lo = Vec3::Constant(std::numeric_limits<double>::infinity());
      Vec3 hi = -lo;
      size_t total = 0;
      for (const auto& c : o.clouds)
        for (const auto& p : c.points) {
          lo = lo.cwiseMin(p.position);
          hi = hi.cwiseMax(p.position);
          ++total;
        }
      if (total == 0) throw std::runtime_error("reconstruct_frame: empty foreground in all views");
      const recon::GridSpec grid = fit_grid_dims(lo, hi, dims, cfg.padding_voxels);
      recon::GradientField field = recon::splat(o.clouds, grid, cfg.mode);
      for (auto& v : field.field.data()) v = -v;
      o.volume.values = recon::integrate_fft(field);
      o.volume.iso_level = recon::iso_level(o.volume.values, o.clouds);
      o.mesh = recon::marching_cubes(o.volume.values, o.volume.iso_level);
    }
    const auto vis = appearance::vertex_visibility(out->rec.mesh, rig, frames, eps_vis_mm);
    out->tex = appearance::assign_texture(out->rec.mesh, rig, frames, out->rec.clouds, vis);
    *status = 0;
  } catch (const std::invalid_argument&) {
    *status = 1;
  } catch (const std::runtime_error&) {
    *status = 2;
  } catch (...) {
    *status = 3;
  }
  return out;
}

void ref_frame_free(void* h) { delete static_cast<RefFrame*>(h); }

// P, V, T, N
void ref_frame_sizes(void* h, int64_t* out) {
  const auto& f = *static_cast<RefFrame*>(h);
  int64_t P = 0;
  for (const auto& c : f.rec.clouds) P += (int64_t)c.points.size();
  out[0] = P, out[1] = (int64_t)f.rec.mesh.vertices.size(), out[2] = (int64_t)f.rec.mesh.triangles.size();
  out[3] = (int64_t)f.rec.volume.values.size();
}

void ref_frame_points(void* h, double* pos, double* nrm, double* w, int32_t* pix) {
  const auto& f = *static_cast<RefFrame*>(h);
  size_t i = 0;
  for (const auto& c : f.rec.clouds)
    for (const auto& p : c.points) {
      for (int a = 0; a < 3; ++a) pos[3 * i + a] = p.position(a), nrm[3 * i + a] = p.normal(a);
      w[i] = p.weight;
      pix[3 * i] = p.px, pix[3 * i + 1] = p.py, pix[3 * i + 2] = p.sensor;
      ++i;
    }
}

void ref_frame_weight_map(void* h, int sensor, float* out) {
  const auto& f = *static_cast<RefFrame*>(h);
  const auto& wm = f.rec.clouds.at(sensor).weight_map;
  std::memcpy(out, wm.data().data(), wm.size() * sizeof(float));
}

void ref_frame_grid(void* h, PGrid* g, double* level) {
  const auto& f = *static_cast<RefFrame*>(h);
  const auto& A = f.rec.volume.values;
  g->nx = A.nx(), g->ny = A.ny(), g->nz = A.nz();
  for (int a = 0; a < 3; ++a) g->origin[a] = A.origin()(a);
  g->edge = A.edge();
  *level = f.rec.volume.iso_level;
}

void ref_frame_volume(void* h, double* out) {
  const auto& A = static_cast<RefFrame*>(h)->rec.volume.values;
  std::memcpy(out, A.data().data(), A.size() * sizeof(double));
}

void ref_frame_mesh(void* h, double* verts, double* normals, int32_t* tris) {
  const auto& m = static_cast<RefFrame*>(h)->rec.mesh;
  for (size_t i = 0; i < m.vertices.size(); ++i)
    for (int a = 0; a < 3; ++a) verts[3 * i + a] = m.vertices[i](a), normals[3 * i + a] = m.normals[i](a);
  for (size_t i = 0; i < m.triangles.size(); ++i)
    for (int a = 0; a < 3; ++a) tris[3 * i + a] = m.triangles[i][a];
}

// vis [k][V], uv [k][V][2], weight [k][V], untextured [V]
void ref_frame_texture(void* h, uint8_t* vis, double* uv, float* weight, uint8_t* untex) {
  const auto& f = *static_cast<RefFrame*>(h);
  const size_t V = f.tex.untextured.size();
  for (int s = 0; s < f.k; ++s)
    for (size_t v = 0; v < V; ++v) {
      vis[s * V + v] = f.tex.visible[s][v];
      uv[2 * (s * V + v)] = f.tex.uv[s][v].x(), uv[2 * (s * V + v) + 1] = f.tex.uv[s][v].y();
      weight[s * V + v] = f.tex.weight[s][v];
    }
  std::memcpy(untex, f.tex.untextured.data(), V);
}

// marching_cubes.cpp:131-210 on a caller field; returns V, T via out[2]
void* ref_marching_cubes(const double* A, const PGrid* g, double level, int64_t* out) {
  VolumeGrid<double> vol(g->nx, g->ny, g->nz, Vec3(g->origin[0], g->origin[1], g->origin[2]), g->edge);
  std::memcpy(vol.data().data(), A, vol.size() * sizeof(double));
  auto* f = new RefFrame;
  f->rec.mesh = recon::marching_cubes(vol, level);
  out[0] = (int64_t)f->rec.mesh.vertices.size(), out[1] = (int64_t)f->rec.mesh.triangles.size();
  return f;
}

// grid: nx*ny*nz bytes (x fastest), voxels 3n int32 -> out 3n int32; returns the count
int64_t ref_skeletonize(const uint8_t* grid, int nx, int ny, int nz, const int32_t* voxels, int64_t n, int32_t* out) {
  mocap::BinaryVolume bv;
  bv.grid = VolumeGrid<std::uint8_t>(nx, ny, nz);
  std::memcpy(bv.grid.data().data(), grid, (size_t)nx * ny * nz);
  for (int64_t i = 0; i < n; ++i) bv.voxels.emplace_back(voxels[3 * i], voxels[3 * i + 1], voxels[3 * i + 2]);
  const auto sk = mocap::skeletonize(bv);
  for (size_t i = 0; i < sk.size(); ++i)
    out[3 * i] = sk[i].x(), out[3 * i + 1] = sk[i].y(), out[3 * i + 2] = sk[i].z();
  return (int64_t)sk.size();
}

// pairs_rgb: n x (first RGB, second RGB); 0 ok, 1 the reference threw (message in err)
int ref_fit_value_map(const uint8_t* pairs_rgb, int n, int iters, double thr, uint64_t seed, double* gain,
                      double* offset, char* err, int errlen) {
  std::vector<appearance::ColorPair> pairs((size_t)n);
  for (int i = 0; i < n; ++i) {
    const uint8_t* p = pairs_rgb + 6 * (size_t)i;
    pairs[i].first = Rgb8{p[0], p[1], p[2]};
    pairs[i].second = Rgb8{p[3], p[4], p[5]};
  }
  try {
    const auto m = appearance::fit_value_map(pairs, appearance::ValueFitOptions{iters, thr, seed});
    *gain = m.gain, *offset = m.offset;
    return 0;
  } catch (const std::exception& e) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
    return 1;
  }
}

int ref_chain_to_reference(const int32_t* from, const int32_t* to, const double* gain, const double* offset,
                           int n_edges, int reference, int sensor_count, double* out_gain, double* out_offset) {
  std::vector<appearance::PairwiseValueMap> edges((size_t)n_edges);
  for (int e = 0; e < n_edges; ++e) edges[e] = {from[e], to[e], appearance::ValueMap{gain[e], offset[e]}};
  try {
    const auto cc = appearance::chain_to_reference(edges, reference, sensor_count);
    for (int k = 0; k < sensor_count; ++k) out_gain[k] = cc.maps[k].gain, out_offset[k] = cc.maps[k].offset;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

}  // extern "C"

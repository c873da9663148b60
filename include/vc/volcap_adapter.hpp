// SPDX-License-Identifier: Apache-2.0
//
// Header-only adapter that lets the reference's C++ callers keep their
// interface: it converts volcap:: types (Eigen-based, reference
// proj/core/include/volcap/...) to the vc_* PODs of vc.h and back.
//
//   #include "volcap/recon/reconstruct.hpp"      // reference types
//   #include "vc/volcap_adapter.hpp"             // this file
//   auto out = vc::adapter::reconstruct_frame(frames, rig, config);   // drop-in for
//   // recon::reconstruct_frame + appearance::vertex_visibility + assign_texture
//
// Needs the reference's headers (and so Eigen).  In this repo it is compiled
// against the reference's own headers + the Eigen-API shim of oracle/ref_shim
// by `make -C oracle ref` (oracle/adapter_check.cpp, run by
// tests/test_gpu_c2_parity.py on the B200) — see INTEGRATION.md.
#pragma once

#include <algorithm>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "vc/vc.h"

#if __has_include("volcap/recon/reconstruct.hpp") && __has_include("volcap/appearance/texture.hpp")
#include "volcap/appearance/texture.hpp"
#include "volcap/recon/reconstruct.hpp"

namespace vc::adapter {

inline vc_pose to_vc(const volcap::Pose& p) {
  vc_pose o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o.R[r * 3 + c] = p.R(r, c);
  for (int i = 0; i < 3; ++i) o.t[i] = p.t(i);
  return o;
}
inline vc_intrinsics to_vc(const volcap::Intrinsics& k) { return {k.fx, k.fy, k.cx, k.cy, k.width, k.height}; }
inline vc_sensor to_vc(const volcap::Sensor& s) {
  return {to_vc(s.depth_intr), to_vc(s.pose), to_vc(s.rgb_intr), to_vc(s.rgb_relative)};
}

inline void check(vc_status s, vc_ctx* ctx) {
  if (s == VC_OK) return;
  const std::string msg = ctx ? vc_last_error(ctx) : vc_status_string(s);
  if (s == VC_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);  // reference: std::invalid_argument
  throw std::runtime_error(msg);                                       // incl. "empty foreground in all views"
}

struct Result {
  volcap::recon::FrameReconstruction recon;  // clouds (want_clouds), volume (want_volume) + mesh
  volcap::appearance::TexturedMesh textured;
  std::vector<volcap::Rgb8> vertex_colors;
};

// recon::reconstruct_frame (reconstruct.hpp:38-39) + vertex_visibility /
// assign_texture (texture.hpp:32-42) in one call on the GPU.
inline Result reconstruct_frame(std::span<const volcap::RgbdFrame> frames, const volcap::CameraRig& rig,
                                const volcap::recon::ReconConfig& config, vc_ctx* ctx,
                                volcap::recon::StageTimings* timings = nullptr, bool want_volume = true,
                                bool want_clouds = true) {
  if (frames.size() != static_cast<std::size_t>(rig.recon_count))
    throw std::invalid_argument("reconstruct_frame: one frame per reconstruction sensor required");
  const int k = rig.recon_count;
  std::vector<vc_sensor> sensors;
  std::vector<vc_view> views;
  std::vector<std::vector<uint8_t>> rgb(k);
  for (int i = 0; i < k; ++i) {
    sensors.push_back(to_vc(rig.sensors[i]));
    const auto& f = frames[i];
    rgb[i].resize(f.color.size() * 3);
    for (std::size_t p = 0; p < f.color.size(); ++p) {
      rgb[i][3 * p] = f.color.data()[p].r, rgb[i][3 * p + 1] = f.color.data()[p].g, rgb[i][3 * p + 2] = f.color.data()[p].b;
    }
    views.push_back({f.depth.data().data(), f.foreground.data().data(), rgb[i].data(), 0, 0, 0, VC_MEM_HOST});
  }
  vc_recon_config c{};
  c.r = config.r;
  c.mode = config.mode == volcap::recon::SplatMode::kSimple ? VC_SPLAT_SIMPLE : VC_SPLAT_WEIGHTED;
  c.discontinuity_mm = config.discontinuity_mm;
  c.padding_voxels = config.padding_voxels;
  c.silhouette_radius_px = config.silhouette_radius_px;
  c.eps_vis_mm = 20.0;
  vc_textured_mesh m{};
  vc_stage_timings t{};
  check(vc_ctx_set_output(ctx, VC_MEM_HOST), ctx);
  check(vc_reconstruct_frame(ctx, sensors.data(), views.data(), k, &c, &m, &t), ctx);
  if (timings) timings->raw_ms = t.raw_ms, timings->weights_ms = t.weights_ms, timings->volumetric_ms = t.volumetric_ms;

  Result out;
  auto& mesh = out.recon.mesh;
  for (int v = 0; v < m.vertex_count; ++v) {
    mesh.vertices.emplace_back(m.positions_f64[3 * v], m.positions_f64[3 * v + 1], m.positions_f64[3 * v + 2]);
    mesh.normals.emplace_back(m.normals[3 * v], m.normals[3 * v + 1], m.normals[3 * v + 2]);
  }
  for (int t3 = 0; t3 < m.triangle_count; ++t3)
    mesh.triangles.push_back({m.triangles[3 * t3], m.triangles[3 * t3 + 1], m.triangles[3 * t3 + 2]});
  out.recon.volume.iso_level = m.iso_level;
  const volcap::Vec3 origin(m.grid.origin[0], m.grid.origin[1], m.grid.origin[2]);
  out.recon.volume.values = volcap::VolumeGrid<double>(m.grid.nx, m.grid.ny, m.grid.nz, origin, m.grid.edge_mm, 0.0);
  if (want_volume) {
    std::vector<float> a(out.recon.volume.values.size());
    check(vc_export_volume(ctx, a.data(), VC_MEM_HOST), ctx);
    for (std::size_t i = 0; i < a.size(); ++i) out.recon.volume.values.data()[i] = a[i];
  }
  if (want_clouds) {  // OrientedCloud per sensor (cloud.hpp:13-26), concatenated in sensor order on the device
    const std::size_t P = static_cast<std::size_t>(m.point_count);
    std::vector<double> pos(3 * P), nrm(3 * P), w(P);
    std::vector<int32_t> pix(3 * P);
    std::size_t wm_total = 0;
    for (int i = 0; i < k; ++i) wm_total += static_cast<std::size_t>(frames[i].depth.width()) * frames[i].depth.height();
    std::vector<float> wm(wm_total);
    check(vc_export_points(ctx, pos.data(), nrm.data(), w.data(), pix.data(), wm.data()), ctx);
    out.recon.clouds.resize(k);
    std::size_t wo = 0;
    for (int i = 0; i < k; ++i) {
      auto& c = out.recon.clouds[i];
      c.sensor = i;
      c.weight_map = volcap::Image<float>(frames[i].depth.width(), frames[i].depth.height(), 0.f);
      std::copy(wm.begin() + wo, wm.begin() + wo + c.weight_map.size(), c.weight_map.data().begin());
      wo += c.weight_map.size();
    }
    for (std::size_t p = 0; p < P; ++p) {
      volcap::recon::OrientedPoint op;
      op.position = volcap::Vec3(pos[3 * p], pos[3 * p + 1], pos[3 * p + 2]);
      op.normal = volcap::Vec3(nrm[3 * p], nrm[3 * p + 1], nrm[3 * p + 2]);
      op.weight = w[p];
      op.px = pix[3 * p], op.py = pix[3 * p + 1], op.sensor = pix[3 * p + 2];
      out.recon.clouds.at(op.sensor).points.push_back(op);
    }
  }
  auto& tm = out.textured;
  tm.mesh = mesh;
  tm.sensor_count = k;
  const int V = m.vertex_count;
  tm.visible.assign(k, std::vector<uint8_t>(V));
  tm.uv.assign(k, std::vector<volcap::Vec2>(V));
  tm.weight.assign(k, std::vector<float>(V));
  tm.untextured.assign(m.untextured, m.untextured + V);
  for (int i = 0; i < k; ++i)
    for (int v = 0; v < V; ++v) {
      tm.visible[i][v] = m.visible[(std::size_t)i * V + v];
      tm.uv[i][v] = volcap::Vec2(m.uv[2 * ((std::size_t)i * V + v)], m.uv[2 * ((std::size_t)i * V + v) + 1]);
      tm.weight[i][v] = m.weight[(std::size_t)i * V + v];
    }
  for (int v = 0; v < V; ++v) out.vertex_colors.push_back({m.rgb[3 * v], m.rgb[3 * v + 1], m.rgb[3 * v + 2]});
  return out;
}

}  // namespace vc::adapter
#endif

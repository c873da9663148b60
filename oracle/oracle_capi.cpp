// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
// extern "C" surface of the CPU oracle for ctypes (oracle/oracle.py).  Also
// hosts orc_reconstruct_frame, the restatement of recon::reconstruct_frame
// (reconstruct.cpp:37-78) + vertex_visibility/assign_texture as driven by
// the CLI (volcap.cpp:304-314) and run_bench's stage split (volcap.cpp:466-486).
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>

#include "oracle.hpp"

using namespace orc;

namespace {
double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

struct orc_cloud {
  Cloud c;
};
struct orc_mesh {
  Mesh m;
};

struct orc_recon_config {
  int32_t nx, ny, nz;
  int32_t mode;
  double discontinuity_mm;
  int32_t padding_voxels;
  int32_t silhouette_radius_px;
  double eps_vis_mm;
  int32_t threads;
};
struct orc_timings {
  double raw_ms, weights_ms, volumetric_ms, other_ms, blend_ms;
  double splat_ms, integrate_ms, iso_ms, mc_ms;
};

struct orc_frame {
  int k = 0;
  std::vector<Cloud> clouds;
  GridSpec grid;
  std::vector<double> A;
  double level = 0;
  Mesh mesh;
  std::vector<uint8_t> vis, untex, rgb8;
  std::vector<double> uv, color;
  std::vector<float> w;
};

extern "C" {

int orc_version() { return 1; }
int orc_hardware_threads() { return hardware_threads(); }
int orc_sizeof_sensor() { return static_cast<int>(sizeof(Sensor)); }
int orc_sizeof_body() { return static_cast<int>(sizeof(Body)); }

void orc_case_table(int* counts, int* tris) {
  int c[256], t[256][5][3];
  case_table(c, t);
  std::memcpy(counts, c, sizeof(c));
  std::memcpy(tris, t, sizeof(t));
}

// ---------------------------------------------------------------- synth
void orc_make_circle_rig(int recon, int held_out, double radius, double target_h, int w, int h,
                         double f, Sensor* out) {
  const auto rig = make_circle_rig(recon, held_out, radius, target_h, w, h, f);
  for (std::size_t i = 0; i < rig.size(); ++i) out[i] = rig[i];
}
void orc_make_xpose_body(Body* out) { *out = make_xpose_body(); }
void orc_make_kick_body(int frames, int f, Body* out) { *out = make_kick_sequence(frames).at(f); }
void orc_render_frame(const Sensor* s, const Body* b, double sigma2m, uint64_t seed, double gain,
                      int camera, int frame, int threads, uint16_t* depth, uint8_t* mask,
                      uint8_t* rgb) {
  render_frame(*s, *b, sigma2m, seed, gain, camera, frame, threads, depth, mask, rgb);
}
int orc_sample_surface(const Body* b, int count, uint64_t seed, double* out) {
  const auto pts = sample_surface(*b, count, seed);
  for (std::size_t i = 0; i < pts.size(); ++i) {
    out[3 * i] = pts[i].x, out[3 * i + 1] = pts[i].y, out[3 * i + 2] = pts[i].z;
  }
  return static_cast<int>(pts.size());
}
double orc_sdf(const Body* b, const double* x) { return sdf(*b, V3{x[0], x[1], x[2]}); }

// ---------------------------------------------------------------- clouds
orc_cloud* orc_build_cloud(const uint16_t* depth, const uint8_t* mask, int w, int h,
                           const Sensor* s, int sensor, double disc) {
  Frame f;
  f.w = w, f.h = h, f.depth = depth, f.mask = mask;
  auto* c = new orc_cloud;
  c->c = build_cloud(f, s->depth_intr, s->pose, sensor, disc);
  return c;
}
void orc_confidence_weights(orc_cloud* c, const uint8_t* mask, int w, int h, const Sensor* s, int r) {
  Frame f;
  f.w = w, f.h = h, f.mask = mask;
  confidence_weights(c->c, f, s->depth_intr, s->pose, r);
}
void orc_cloud_set_normals(orc_cloud* c, const double* nrm) {
  for (std::size_t i = 0; i < c->c.points.size(); ++i)
    c->c.points[i].normal = V3{nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]};
}
int64_t orc_cloud_size(const orc_cloud* c) { return static_cast<int64_t>(c->c.points.size()); }
void orc_cloud_get(const orc_cloud* c, double* pos, double* nrm, double* weight, int* px, int* py,
                   float* weight_map) {
  const auto& P = c->c.points;
  for (std::size_t i = 0; i < P.size(); ++i) {
    if (pos) pos[3 * i] = P[i].position.x, pos[3 * i + 1] = P[i].position.y, pos[3 * i + 2] = P[i].position.z;
    if (nrm) nrm[3 * i] = P[i].normal.x, nrm[3 * i + 1] = P[i].normal.y, nrm[3 * i + 2] = P[i].normal.z;
    if (weight) weight[i] = P[i].weight;
    if (px) px[i] = P[i].px;
    if (py) py[i] = P[i].py;
  }
  if (weight_map) std::memcpy(weight_map, c->c.weight_map.data(), c->c.weight_map.size() * sizeof(float));
}
void orc_cloud_free(orc_cloud* c) { delete c; }

// ---------------------------------------------------------------- volume
int orc_fit_grid(const double* lo, const double* hi, const int* dims, int pad, GridSpec* out) {
  return fit_grid(V3{lo[0], lo[1], lo[2]}, V3{hi[0], hi[1], hi[2]}, dims, pad, out) ? 0 : 1;
}

static std::vector<OrientedPoint> make_points(const double* pos, const double* nrm, const double* w,
                                              int64_t n) {
  std::vector<OrientedPoint> pts(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    pts[i].position = V3{pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    if (nrm) pts[i].normal = V3{nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]};
    pts[i].weight = w ? w[i] : 1.0;
  }
  return pts;
}

void orc_splat(const double* pos, const double* nrm, const double* w, int64_t n, const GridSpec* g,
               int mode, int threads, double* field, double* density, double* sigmas) {
  const auto pts = make_points(pos, nrm, w, n);
  std::vector<const OrientedPoint*> ptrs;
  for (const auto& p : pts) ptrs.push_back(&p);
  const Field f = splat(ptrs, *g, mode, threads <= 0 ? hardware_threads() : threads);
  for (std::size_t i = 0; i < f.field.size(); ++i) {
    field[3 * i] = f.field[i].x, field[3 * i + 1] = f.field[i].y, field[3 * i + 2] = f.field[i].z;
    density[i] = f.density[i];
  }
  if (sigmas) sigmas[0] = f.sigma1, sigmas[1] = f.sigma2;
}

void orc_integrate_fft(const double* field3, int nx, int ny, int nz, double* out) {
  std::vector<V3> f(static_cast<std::size_t>(nx) * ny * nz);
  for (std::size_t i = 0; i < f.size(); ++i) f[i] = V3{field3[3 * i], field3[3 * i + 1], field3[3 * i + 2]};
  integrate_fft(f.data(), nx, ny, nz, out);
}

int orc_iso_level(const double* A, const GridSpec* g, const double* pos, int64_t n, double* level) {
  const auto pts = make_points(pos, nullptr, nullptr, n);
  std::vector<const OrientedPoint*> ptrs;
  for (const auto& p : pts) ptrs.push_back(&p);
  return iso_level(A, *g, ptrs, level) ? 0 : 1;
}

orc_mesh* orc_marching_cubes(const double* A, const GridSpec* g, double level) {
  auto* m = new orc_mesh;
  m->m = marching_cubes(A, *g, level);
  return m;
}
void orc_mesh_counts(const orc_mesh* m, int64_t* V, int64_t* T) {
  *V = static_cast<int64_t>(m->m.vertices.size());
  *T = static_cast<int64_t>(m->m.triangles.size());
}
void orc_mesh_get(const orc_mesh* m, double* verts, double* normals, int32_t* tris, uint64_t* edge_ids) {
  const Mesh& M = m->m;
  for (std::size_t i = 0; i < M.vertices.size(); ++i) {
    if (verts) verts[3 * i] = M.vertices[i].x, verts[3 * i + 1] = M.vertices[i].y, verts[3 * i + 2] = M.vertices[i].z;
    if (normals) normals[3 * i] = M.normals[i].x, normals[3 * i + 1] = M.normals[i].y, normals[3 * i + 2] = M.normals[i].z;
    if (edge_ids) edge_ids[i] = M.edge_ids[i];
  }
  if (tris)
    for (std::size_t t = 0; t < M.triangles.size(); ++t)
      for (int j = 0; j < 3; ++j) tris[3 * t + j] = M.triangles[t][j];
}
void orc_mesh_free(orc_mesh* m) { delete m; }

// ---------------------------------------------------------------- texture
static std::vector<V3> make_verts(const double* v, int64_t n) {
  std::vector<V3> out(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) out[i] = V3{v[3 * i], v[3 * i + 1], v[3 * i + 2]};
  return out;
}
void orc_vertex_visibility(const double* verts, int64_t V, const Sensor* sensors,
                           const uint16_t* const* depths, const uint8_t* const* masks, int k,
                           double eps, uint8_t* vis) {
  std::vector<Frame> frames(k);
  for (int i = 0; i < k; ++i) {
    frames[i].w = sensors[i].depth_intr.width, frames[i].h = sensors[i].depth_intr.height;
    frames[i].depth = depths[i], frames[i].mask = masks[i];
  }
  vertex_visibility(make_verts(verts, V), sensors, frames.data(), k, eps, vis);
}
void orc_assign_texture(const double* verts, int64_t V, const Sensor* sensors,
                        const float* const* weight_maps, int k, const uint8_t* vis, double* uv,
                        float* w, uint8_t* untex) {
  std::vector<Cloud> clouds(k);
  for (int i = 0; i < k; ++i) {
    clouds[i].w = sensors[i].depth_intr.width, clouds[i].h = sensors[i].depth_intr.height;
    clouds[i].weight_map.assign(weight_maps[i], weight_maps[i] + static_cast<std::size_t>(clouds[i].w) * clouds[i].h);
  }
  assign_texture(make_verts(verts, V), sensors, clouds.data(), k, vis, uv, w, untex);
}
void orc_blend_colors(int64_t V, int k, const uint8_t* vis, const double* uv, const float* w,
                      const uint8_t* const* rgbs, const int32_t* rgb_wh, double* color, uint8_t* rgb8) {
  std::vector<Frame> frames(k);
  for (int i = 0; i < k; ++i) frames[i].rgb = rgbs[i], frames[i].rgb_w = rgb_wh[2 * i], frames[i].rgb_h = rgb_wh[2 * i + 1];
  blend_colors(static_cast<int>(V), k, vis, uv, w, frames.data(), color, rgb8);
}

// ---------------------------------------------------------------- full frame
// reconstruct.cpp:37-78 followed by texture.cpp:11-72 and the A14 blend.
// status: 0 ok, 1 invalid argument, 2 empty scene (VC_ERR_* values).
orc_frame* orc_reconstruct_frame(const Sensor* sensors, int k, const uint16_t* const* depths,
                                 const uint8_t* const* masks, const uint8_t* const* rgbs,
                                 const orc_recon_config* cfg, orc_timings* tm, int* status) {
  *status = 0;
  auto* out = new orc_frame;
  out->k = k;
  orc_timings t{};
  const int threads = cfg->threads > 0 ? cfg->threads : hardware_threads();
  std::vector<Frame> frames(k);
  for (int i = 0; i < k; ++i) {
    frames[i].w = sensors[i].depth_intr.width, frames[i].h = sensors[i].depth_intr.height;
    frames[i].depth = depths[i], frames[i].mask = masks[i];
    frames[i].rgb = rgbs ? rgbs[i] : nullptr;
    frames[i].rgb_w = sensors[i].rgb_intr.width, frames[i].rgb_h = sensors[i].rgb_intr.height;
  }
  try {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < k; ++i)
      out->clouds.push_back(build_cloud(frames[i], sensors[i].depth_intr, sensors[i].pose, i, cfg->discontinuity_mm));
    t.raw_ms = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < k; ++i)
      confidence_weights(out->clouds[i], frames[i], sensors[i].depth_intr, sensors[i].pose, cfg->silhouette_radius_px);
    t.weights_ms = ms_since(t0);

    t0 = std::chrono::steady_clock::now();
    const double inf = std::numeric_limits<double>::infinity();
    V3 lo{inf, inf, inf}, hi{-inf, -inf, -inf};
    std::vector<const OrientedPoint*> pts;
    for (const auto& c : out->clouds)
      for (const auto& p : c.points) {
        lo = V3{std::min(lo.x, p.position.x), std::min(lo.y, p.position.y), std::min(lo.z, p.position.z)};
        hi = V3{std::max(hi.x, p.position.x), std::max(hi.y, p.position.y), std::max(hi.z, p.position.z)};
        pts.push_back(&p);
      }
    if (pts.empty()) {
      *status = 2;
      return out;
    }
    const int dims[3] = {cfg->nx, cfg->ny, cfg->nz};
    if (!fit_grid(lo, hi, dims, cfg->padding_voxels, &out->grid)) {
      *status = 1;
      return out;
    }
    auto ts = std::chrono::steady_clock::now();
    Field field = splat(pts, out->grid, cfg->mode, threads);
    for (auto& v : field.field) v = -v;  // reconstruct.cpp:71
    t.splat_ms = ms_since(ts);
    ts = std::chrono::steady_clock::now();
    out->A.resize(field.field.size());
    integrate_fft(field.field.data(), out->grid.nx, out->grid.ny, out->grid.nz, out->A.data());
    t.integrate_ms = ms_since(ts);
    ts = std::chrono::steady_clock::now();
    iso_level(out->A.data(), out->grid, pts, &out->level);
    t.iso_ms = ms_since(ts);
    ts = std::chrono::steady_clock::now();
    out->mesh = marching_cubes(out->A.data(), out->grid, out->level);
    t.mc_ms = ms_since(ts);
    t.volumetric_ms = ms_since(t0);

    t0 = std::chrono::steady_clock::now();
    const std::size_t V = out->mesh.vertices.size();
    out->vis.assign(static_cast<std::size_t>(k) * V, 0);
    out->uv.assign(static_cast<std::size_t>(k) * V * 2, 0.0);
    out->w.assign(static_cast<std::size_t>(k) * V, 0.f);
    out->untex.assign(V, 0);
    vertex_visibility(out->mesh.vertices, sensors, frames.data(), k, cfg->eps_vis_mm, out->vis.data());
    assign_texture(out->mesh.vertices, sensors, out->clouds.data(), k, out->vis.data(), out->uv.data(),
                   out->w.data(), out->untex.data());
    t.other_ms = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    out->color.assign(V * 3, 0.0);
    out->rgb8.assign(V * 3, 0);
    if (rgbs)
      blend_colors(static_cast<int>(V), k, out->vis.data(), out->uv.data(), out->w.data(), frames.data(),
                   out->color.data(), out->rgb8.data());
    t.blend_ms = ms_since(t0);
  } catch (const std::invalid_argument&) {
    *status = 1;
  }
  if (tm) *tm = t;
  return out;
}

int64_t orc_frame_point_count(const orc_frame* f) {
  int64_t n = 0;
  for (const auto& c : f->clouds) n += static_cast<int64_t>(c.points.size());
  return n;
}
void orc_frame_points(const orc_frame* f, double* pos, double* nrm, double* weight, int32_t* pix /*n*3: px,py,sensor*/) {
  std::size_t i = 0;
  for (const auto& c : f->clouds)
    for (const auto& p : c.points) {
      if (pos) pos[3 * i] = p.position.x, pos[3 * i + 1] = p.position.y, pos[3 * i + 2] = p.position.z;
      if (nrm) nrm[3 * i] = p.normal.x, nrm[3 * i + 1] = p.normal.y, nrm[3 * i + 2] = p.normal.z;
      if (weight) weight[i] = p.weight;
      if (pix) pix[3 * i] = p.px, pix[3 * i + 1] = p.py, pix[3 * i + 2] = p.sensor;
      ++i;
    }
}
void orc_frame_weight_map(const orc_frame* f, int k, float* out) {
  std::memcpy(out, f->clouds[k].weight_map.data(), f->clouds[k].weight_map.size() * sizeof(float));
}
void orc_frame_grid(const orc_frame* f, GridSpec* g, double* level) {
  *g = f->grid;
  *level = f->level;
}
void orc_frame_volume(const orc_frame* f, double* A) { std::memcpy(A, f->A.data(), f->A.size() * sizeof(double)); }
const orc_mesh* orc_frame_mesh(orc_frame* f) { return reinterpret_cast<const orc_mesh*>(&f->mesh); }
void orc_frame_texture(const orc_frame* f, uint8_t* vis, double* uv, float* w, uint8_t* untex, double* color,
                       uint8_t* rgb8) {
  if (vis) std::memcpy(vis, f->vis.data(), f->vis.size());
  if (uv) std::memcpy(uv, f->uv.data(), f->uv.size() * sizeof(double));
  if (w) std::memcpy(w, f->w.data(), f->w.size() * sizeof(float));
  if (untex) std::memcpy(untex, f->untex.data(), f->untex.size());
  if (color) std::memcpy(color, f->color.data(), f->color.size() * sizeof(double));
  if (rgb8) std::memcpy(rgb8, f->rgb8.data(), f->rgb8.size());
}
void orc_frame_free(orc_frame* f) { delete f; }

}  // extern "C"

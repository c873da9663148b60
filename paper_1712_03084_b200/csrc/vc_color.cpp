// SPDX-License-Identifier: Apache-2.0
//
// Colour correction behind the C-ABI (
// color_correction.cpp, hsv.cpp):
//   vc_color_apply                 ColorCorrection::apply(sensor, image) on the GPU
//   vc_mutual_closest_pairs        mutual_closest_pairs on the GPU hash grid
//   vc_fit_value_map               fit_value_map (host: RANSAC over the 256 x 256
//                                  value-level lattice, exact integer moments)
//   vc_chain_to_reference          chain_to_reference (host BFS over incidence lists)
//   vc_ctx_set_color_correction    per-sensor maps fused into the frame's
//                                  texture sampling
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "vc_ctx.hpp"

using namespace vc;
using namespace vc::rt;

namespace {

}  // namespace

extern "C" const char* vc_io_last_error(void);
namespace vc_io_detail {
vc_status set_error(vc_status s, const std::string& msg);
}

extern "C" {

vc_status vc_ctx_set_color_correction(vc_ctx* ctx, const double* gain, const double* offset, int32_t k) {
  if (!ctx || k < 0 || k > kMaxViews || (k > 0 && (!gain || !offset)))
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "color correction: bad arguments");
  ctx->cc_gain.assign(gain, gain + k);
  ctx->cc_offset.assign(offset, offset + k);
  return VC_OK;
}

vc_status vc_color_apply(vc_ctx* ctx, const uint8_t* rgb_in, uint8_t* rgb_out, int64_t n_pixels, double gain,
                         double offset, int32_t mem_kind) {
  if (!ctx || !rgb_in || !rgb_out || n_pixels < 0) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "null argument");
  cudaSetDevice(ctx->device);
  const size_t bytes = (size_t)n_pixels * 3;
  if (gain == 1.0 && offset == 0.0) {  // color_correction.cpp:151-153: the image unchanged
    if (rgb_in != rgb_out)
      VC_CUDA(cudaMemcpyAsync(rgb_out, rgb_in, bytes, cudaMemcpyDefault, ctx->st));
    VC_CUDA(cudaStreamSynchronize(ctx->st));
    return VC_OK;
  }
  if (mem_kind == VC_MEM_DEVICE) {
    launch_color_apply(rgb_in, rgb_out, n_pixels, gain, offset, ctx->st);
  } else {
    Buf& b = ctx->scratch_dev;
    VC_TRY(ensure(ctx, b, 2 * bytes + 256));
    uint8_t* din = P<uint8_t>(b);
    uint8_t* dout = din + ((bytes + 255) & ~size_t(255));
    VC_CUDA(cudaMemcpyAsync(din, rgb_in, bytes, cudaMemcpyHostToDevice, ctx->st));
    launch_color_apply(din, dout, n_pixels, gain, offset, ctx->st);
    VC_CUDA(cudaMemcpyAsync(rgb_out, dout, bytes, cudaMemcpyDeviceToHost, ctx->st));
  }
  VC_CUDA(cudaGetLastError());
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}

vc_status vc_mutual_closest_pairs(vc_ctx* ctx, const double* a, int32_t na, const double* b, int32_t nb,
                                  double max_dist_mm, int32_t* pairs, int32_t* n_pairs) {
  if (!ctx || !n_pairs || na < 0 || nb < 0 || (na > 0 && !a) || (nb > 0 && !b) || (na > 0 && nb > 0 && !pairs))
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "null argument");
  *n_pairs = 0;
  if (na == 0 || nb == 0) return VC_OK;  // color_correction.cpp:69
  if (!(max_dist_mm > 0)) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "max_dist must be positive");
  cudaSetDevice(ctx->device);
  const size_t sa = grid_scratch_bytes(na), sb = grid_scratch_bytes(nb);
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t bytes = up((size_t)na * 24) + up((size_t)nb * 24) + up(sa) + up(sb) + up((size_t)na * 4) +
                       up((size_t)2 * std::min(na, nb) * 4 + 8) + 256;
  VC_TRY(ensure(ctx, ctx->scratch_dev, bytes));
  uint8_t* p = P<uint8_t>(ctx->scratch_dev);
  double* da = reinterpret_cast<double*>(p);
  p += up((size_t)na * 24);
  double* db = reinterpret_cast<double*>(p);
  p += up((size_t)nb * 24);
  void* ga = p;
  p += up(sa);
  void* gb = p;
  p += up(sb);
  int32_t* partner = reinterpret_cast<int32_t*>(p);
  p += up((size_t)na * 4);
  int32_t* dn = reinterpret_cast<int32_t*>(p);
  int32_t* dpairs = dn + 2;
  VC_CUDA(cudaMemcpyAsync(da, a, (size_t)na * 24, cudaMemcpyHostToDevice, ctx->st));
  VC_CUDA(cudaMemcpyAsync(db, b, (size_t)nb * 24, cudaMemcpyHostToDevice, ctx->st));
  launch_mutual_pairs(da, na, db, nb, max_dist_mm, ga, gb, partner, dpairs, dn, ctx->st);
  VC_CUDA(cudaGetLastError());
  int32_t n = 0;
  VC_CUDA(cudaMemcpyAsync(&n, dn, 4, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  if (n > 0) VC_CUDA(cudaMemcpy(pairs, dpairs, (size_t)n * 8, cudaMemcpyDeviceToHost));
  *n_pairs = n;
  return VC_OK;
}

// fit_value_map (color_correction.cpp:97-138).  The value channel of an RGB8
// colour is max(r, g, b) / 255, so every pair is a cell (ka, kb) of a 256 x 256
// lattice: the pairs are binned once, each RANSAC hypothesis is scored over the
// occupied cells (weighted by their pair counts) instead of over all pairs, and
// the final least squares uses exact integer moments of the inlier cells
// (gain = (k Sab - Sa Sb) / (k Saa - Sa^2), the 1/255 scales cancel), so the
// fit is the correctly rounded solution of the reference's normal equations.
// The hypotheses are the reference's: (i, j) drawn with std::mt19937_64 and
// uniform_int_distribution<int>(0, n-1), a pair with equal values skipped, the
// first hypothesis of maximal support kept; a cell's inlier test is the
// reference's expression on the same doubles, so the support counts are equal.
vc_status vc_fit_value_map(const uint8_t* pairs_rgb, int32_t n, int32_t ransac_iterations, double inlier_threshold,
                           uint64_t seed, double* gain, double* offset) {
  if (!gain || !offset || n < 0 || (n > 0 && !pairs_rgb))
    return vc_io_detail::set_error(VC_ERR_INVALID_ARGUMENT, "fit_value_map: null argument");
  if (n < 10)
    return vc_io_detail::set_error(VC_ERR_RUNTIME, "fit_value_map: insufficient color diversity (< 10 pairs)");
  auto level = [](const uint8_t* c) { return (int)std::max({c[0], c[1], c[2]}); };
  std::vector<uint8_t> ka(n), kb(n);
  std::vector<int32_t> hist(256 * 256, 0);
  int kmin = 255, kmax = 0;
  for (int32_t p = 0; p < n; ++p) {
    ka[p] = (uint8_t)level(pairs_rgb + 6 * (size_t)p);
    kb[p] = (uint8_t)level(pairs_rgb + 6 * (size_t)p + 3);
    ++hist[ka[p] * 256 + kb[p]];
    kmin = std::min(kmin, (int)ka[p]), kmax = std::max(kmax, (int)ka[p]);
  }
  if (kmax == kmin)  // one value level: spread 0 < 1e-6
    return vc_io_detail::set_error(VC_ERR_RUNTIME, "fit_value_map: insufficient color diversity (constant value)");
  struct Cell {
    double a, b;
    int32_t count;
    uint8_t ka, kb;
  };
  std::vector<Cell> cells;
  for (int c = 0; c < 256 * 256; ++c)
    if (hist[c]) cells.push_back({(c >> 8) / 255.0, (c & 255) / 255.0, hist[c], (uint8_t)(c >> 8), (uint8_t)(c & 255)});
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> draw(0, n - 1);
  int64_t top = -1;
  double top_a = 0, top_b = 0;
  for (int32_t h = 0; h < ransac_iterations; ++h) {
    const int p = draw(rng);
    const int q = draw(rng);
    if (ka[p] == ka[q]) continue;  // |va_p - va_q| < 1e-6 <=> same level
    const double vap = ka[p] / 255.0, vbp = kb[p] / 255.0;
    const double slope = (kb[q] / 255.0 - vbp) / (ka[q] / 255.0 - vap);
    const double icpt = vbp - slope * vap;
    int64_t support = 0;
    for (const Cell& c : cells)
      if (std::abs(slope * c.a + icpt - c.b) < inlier_threshold) support += c.count;
    if (support > top) top = support, top_a = slope, top_b = icpt;
  }
  if (top < 2) return vc_io_detail::set_error(VC_ERR_RUNTIME, "fit_value_map: no consensus line");
  int64_t k = 0, sa = 0, sb = 0, saa = 0, sab = 0;
  for (const Cell& c : cells)
    if (std::abs(top_a * c.a + top_b - c.b) < inlier_threshold) {
      k += c.count, sa += (int64_t)c.count * c.ka, sb += (int64_t)c.count * c.kb;
      saa += (int64_t)c.count * c.ka * c.ka, sab += (int64_t)c.count * c.ka * c.kb;
    }
  const int64_t den = k * saa - sa * sa;  // 255^2 (k Sxx - Sx^2): zero iff all inliers share one level
  if (den == 0) return vc_io_detail::set_error(VC_ERR_RUNTIME, "fit_value_map: degenerate inlier set");
  const double g = (double)(k * sab - sa * sb) / (double)den;
  *gain = g;
  *offset = ((double)sb - g * (double)sa) / (255.0 * (double)k);
  return VC_OK;
}

// chain_to_reference (color_correction.cpp:168-199).  Breadth-first over the
// sensor graph from the reference; a sensor's map is fixed by the first edge
// (in edge order) that reaches it from the sensor being expanded, composed as
// the reference's ValueMap::then / inverse (color.hpp:48-52):
//   edge u -> w (V_w = g V_u + o) reached from u:  M_w = M_u o (g, o)^-1
//   edge w -> u reached from u:                    M_w = M_u o (g, o)
vc_status vc_chain_to_reference(const int32_t* from, const int32_t* to, const double* gain, const double* offset,
                                int32_t n_edges, int32_t reference, int32_t sensor_count, double* out_gain,
                                double* out_offset) {
  if (sensor_count < 1 || reference < 0 || reference >= sensor_count || n_edges < 0 || !out_gain || !out_offset ||
      (n_edges > 0 && (!from || !to || !gain || !offset)))
    return vc_io_detail::set_error(VC_ERR_INVALID_ARGUMENT, "chain_to_reference: bad arguments");
  // incidence lists in edge order: (edge, 0 = sensor is the edge's source)
  std::vector<std::vector<std::pair<int32_t, int>>> inc(sensor_count);
  for (int32_t e = 0; e < n_edges; ++e) {
    if (from[e] < 0 || from[e] >= sensor_count || to[e] < 0 || to[e] >= sensor_count)
      return vc_io_detail::set_error(VC_ERR_INVALID_ARGUMENT, "chain_to_reference: edge sensor out of range");
    inc[from[e]].push_back({e, 0});
    if (to[e] != from[e]) inc[to[e]].push_back({e, 1});
  }
  std::vector<double> G(sensor_count, 1.0), O(sensor_count, 0.0);
  std::vector<int32_t> order{reference};
  std::vector<char> done(sensor_count, 0);
  done[reference] = 1;
  for (size_t head = 0; head < order.size(); ++head) {
    const int32_t u = order[head];
    for (const auto& [e, side] : inc[u]) {
      const int32_t w = side == 0 ? to[e] : from[e];
      if (done[w]) continue;
      if (side == 0) {  // (g, o)^-1 = (1/g, -o/g), then M_u
        const double ig = 1.0 / gain[e], io = -offset[e] / gain[e];
        G[w] = G[u] * ig, O[w] = G[u] * io + O[u];
      } else {
        G[w] = G[u] * gain[e], O[w] = G[u] * offset[e] + O[u];
      }
      done[w] = 1;
      order.push_back(w);
    }
  }
  for (int32_t s = 0; s < sensor_count; ++s)
    if (!done[s])
      return vc_io_detail::set_error(VC_ERR_RUNTIME, "chain_to_reference: sensor " + std::to_string(s) +
                                                         " not connected to the reference");
  std::copy(G.begin(), G.end(), out_gain);
  std::copy(O.begin(), O.end(), out_offset);
  return VC_OK;
}

}  // extern "C"

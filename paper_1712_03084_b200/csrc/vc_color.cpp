// SPDX-License-Identifier: Apache-2.0
//
// Colour correction behind the C-ABI (
// color_correction.cpp, hsv.cpp):
//   vc_color_apply                 ColorCorrection::apply(sensor, image) on the GPU
//   vc_mutual_closest_pairs        mutual_closest_pairs on the GPU hash grid
//   vc_fit_value_map               fit_value_map (host: a few thousand pairs;
//                                  std::mt19937_64 + uniform_int_distribution
//                                  exactly as the reference draws them)
//   vc_chain_to_reference          chain_to_reference (host)
//   vc_ctx_set_color_correction    per-sensor maps fused into the frame's
//                                  texture sampling
#include <algorithm>
#include <cmath>
#include <cstring>
#include <queue>
#include <random>
#include <string>
#include <vector>

#include "vc_ctx.hpp"

using namespace vc;
using namespace vc::rt;

namespace {

struct Vmap {
  double gain = 1.0, offset = 0.0;
  Vmap then(const Vmap& outer) const { return {outer.gain * gain, outer.gain * offset + outer.offset}; }
  Vmap inverse() const { return {1.0 / gain, -offset / gain}; }
};

double value_of(const uint8_t* c) {  // rgb_to_hsv(c).v (hsv.cpp:9-13)
  const double r = c[0] / 255.0, g = c[1] / 255.0, b = c[2] / 255.0;
  return std::max({r, g, b});
}

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

// color_correction.cpp:97-138
vc_status vc_fit_value_map(const uint8_t* pairs_rgb, int32_t n, int32_t ransac_iterations, double inlier_threshold,
                           uint64_t seed, double* gain, double* offset) {
  if (!gain || !offset || n < 0 || (n > 0 && !pairs_rgb))
    return vc_io_detail::set_error(VC_ERR_INVALID_ARGUMENT, "fit_value_map: null argument");
  if (n < 10)
    return vc_io_detail::set_error(VC_ERR_INVALID_ARGUMENT, "fit_value_map: insufficient color diversity (< 10 pairs)");
  std::vector<double> va(n), vb(n);
  double lo = 1, hi = 0;
  for (int i = 0; i < n; ++i) {
    va[i] = value_of(pairs_rgb + 6 * (size_t)i);
    vb[i] = value_of(pairs_rgb + 6 * (size_t)i + 3);
    lo = std::min(lo, va[i]);
    hi = std::max(hi, va[i]);
  }
  if (hi - lo < 1e-6)
    return vc_io_detail::set_error(VC_ERR_INVALID_ARGUMENT,
                                   "fit_value_map: insufficient color diversity (constant value)");
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> pick(0, n - 1);
  int best_count = -1;
  std::vector<int> best_inliers;
  for (int it = 0; it < ransac_iterations; ++it) {
    const int i = pick(rng), j = pick(rng);
    if (std::abs(va[i] - va[j]) < 1e-6) continue;
    const double a = (vb[j] - vb[i]) / (va[j] - va[i]);
    const double b = vb[i] - a * va[i];
    std::vector<int> inliers;
    for (int m = 0; m < n; ++m)
      if (std::abs(a * va[m] + b - vb[m]) < inlier_threshold) inliers.push_back(m);
    if ((int)inliers.size() > best_count) {
      best_count = (int)inliers.size();
      best_inliers = std::move(inliers);
    }
  }
  if (best_count < 2) return vc_io_detail::set_error(VC_ERR_INVALID_ARGUMENT, "fit_value_map: no consensus line");
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  for (int m : best_inliers) {
    sx += va[m];
    sy += vb[m];
    sxx += va[m] * va[m];
    sxy += va[m] * vb[m];
  }
  const double k = (double)best_inliers.size();
  const double denom = k * sxx - sx * sx;
  if (std::abs(denom) < 1e-12)
    return vc_io_detail::set_error(VC_ERR_INVALID_ARGUMENT, "fit_value_map: degenerate inlier set");
  *gain = (k * sxy - sx * sy) / denom;
  *offset = (sy - *gain * sx) / k;
  return VC_OK;
}

// color_correction.cpp:168-199
vc_status vc_chain_to_reference(const int32_t* from, const int32_t* to, const double* gain, const double* offset,
                                int32_t n_edges, int32_t reference, int32_t sensor_count, double* out_gain,
                                double* out_offset) {
  if (sensor_count < 1 || reference < 0 || reference >= sensor_count || n_edges < 0 || !out_gain || !out_offset ||
      (n_edges > 0 && (!from || !to || !gain || !offset)))
    return vc_io_detail::set_error(VC_ERR_INVALID_ARGUMENT, "chain_to_reference: bad arguments");
  for (int e = 0; e < n_edges; ++e)
    if (from[e] < 0 || from[e] >= sensor_count || to[e] < 0 || to[e] >= sensor_count)
      return vc_io_detail::set_error(VC_ERR_INVALID_ARGUMENT, "chain_to_reference: edge sensor out of range");
  std::vector<Vmap> maps(sensor_count);
  std::vector<char> known(sensor_count, 0);
  known[reference] = 1;
  std::queue<int> frontier;
  frontier.push(reference);
  while (!frontier.empty()) {
    const int cur = frontier.front();
    frontier.pop();
    for (int e = 0; e < n_edges; ++e) {
      const Vmap m{gain[e], offset[e]};
      if (known[from[e]] && !known[to[e]]) {
        if (from[e] != cur) continue;
        maps[to[e]] = m.inverse().then(maps[from[e]]);
        known[to[e]] = 1;
        frontier.push(to[e]);
      } else if (known[to[e]] && !known[from[e]]) {
        if (to[e] != cur) continue;
        maps[from[e]] = m.then(maps[to[e]]);
        known[from[e]] = 1;
        frontier.push(from[e]);
      }
    }
  }
  for (int k = 0; k < sensor_count; ++k)
    if (!known[k])
      return vc_io_detail::set_error(VC_ERR_INVALID_ARGUMENT, "chain_to_reference: sensor " + std::to_string(k) +
                                                                  " not connected to the reference");
  for (int k = 0; k < sensor_count; ++k) out_gain[k] = maps[k].gain, out_offset[k] = maps[k].offset;
  return VC_OK;
}

}  // extern "C"

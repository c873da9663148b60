// SPDX-License-Identifier: Apache-2.0
//
// Evaluation renderer and metrics behind the C-ABI (
// eval/rasterize.cpp, metrics.cpp, distance_transform.cpp, ssim.cpp).  Host
// arrays in and out; the GPU does the per-pixel / per-fragment / per-point
// work, the host does what the reference defines as ordered sums.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "vc_ctx.hpp"

using namespace vc;
using namespace vc::rt;

namespace vc {
struct RzCamera {
  double fx, fy, cx, cy;
  int32_t w, h;
  double Ri[9], ti[3];
};
struct RzMesh {
  const double* pos;
  const int32_t* tri;
  int V, T, K;
  const uint8_t* vis;
  const float* uv;
  const float* w;
};
struct RzImages {
  const uint8_t* rgb[16];
  int32_t w[16], h[16];
};
struct Frag {
  double z, la, lb, lc;
  int32_t tri, pad;
};
size_t raster_scratch_bytes(int V, int w, int h);
int64_t launch_raster_count(RzMesh m, RzCamera c, void* scratch, cudaStream_t st, int32_t** off_out);
void launch_raster_finish(RzMesh m, RzCamera c, RzImages im, int mode, void* scratch, Frag* frags, float* depth,
                          uint8_t* color, uint8_t* sil, cudaStream_t st);
void launch_vre(const uint8_t* a, const uint8_t* b, int n, unsigned long long* cnt, cudaStream_t st);
size_t dt_scratch_bytes(int w, int h);
void launch_distance_transform(const uint8_t* mask, int w, int h, void* scratch, float* out, cudaStream_t st);
void launch_hausdorff(const uint8_t* a, const uint8_t* b, const float* dta, const float* dtb, int n, int* maxbits,
                      cudaStream_t st);
void launch_nearest(const double* ground, int ng, const double* recon, int nr, double* out, cudaStream_t st);
void launch_ssim_gray(const uint8_t* rgb, int n, double* g, cudaStream_t st);
void launch_ssim_gauss(const double* in, double* tmp, double* out, int w, int h, const double* k, int r,
                       cudaStream_t st);
void launch_ssim_mul(const double* a, const double* b, double* o, int n, cudaStream_t st);
void launch_ssim_down(const double* in, int w, int h, double* out, int ow, int oh, cudaStream_t st);
void launch_ssim_down_or(const uint8_t* in, int w, int h, uint8_t* out, int ow, int oh, cudaStream_t st);
void launch_ssim_terms(const double* mx, const double* my, const double* xx, const double* yy, const double* xy,
                       const uint8_t* mask, int w, int h, int r, double c1, double c2, double c3, double* terms,
                       cudaStream_t st);
}  // namespace vc

namespace {

size_t up(size_t x) { return (x + 255) & ~size_t(255); }

// A bump allocator over one device buffer of the context.
struct Arena {
  uint8_t* base;
  size_t used = 0;
  template <class T>
  T* take(size_t n) {
    T* p = reinterpret_cast<T*>(base + used);
    used += up(n * sizeof(T));
    return p;
  }
};

vc_status h2d(vc_ctx* ctx, void* d, const void* h, size_t bytes) {
  if (bytes) VC_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, ctx->st));
  return VC_OK;
}

}  // namespace

extern "C" {

vc_status vc_rasterize(vc_ctx* ctx, const double* vertices, int32_t n_vertices, const int32_t* triangles,
                       int32_t n_triangles, int32_t k, const uint8_t* visible, const float* uv, const float* weight,
                       const vc_intrinsics* intr, const vc_pose* pose, const uint8_t* const* images,
                       const int32_t* image_w, const int32_t* image_h, int32_t mode, float* depth, uint8_t* color,
                       uint8_t* silhouette) {
  if (!ctx || !intr || !pose || !depth || !color || !silhouette || n_vertices < 0 || n_triangles < 0 || k < 0 ||
      k > 16 || (mode != VC_RENDER_UV_BLEND && mode != VC_RENDER_COLOR_PER_VERTEX))
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "rasterize: bad arguments");
  const int w = intr->width, h = intr->height;
  if (w <= 0 || h <= 0) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "rasterize: bad image size");
  const size_t npx = (size_t)w * h;
  if (n_vertices == 0 || n_triangles == 0) {  // rasterize.cpp:41-42 (empty mesh)
    std::memset(depth, 0, npx * 4), std::memset(color, 0, npx * 3), std::memset(silhouette, 0, npx);
    return VC_OK;
  }
  if (!vertices || !triangles || (k > 0 && (!visible || !uv || !weight || !images || !image_w || !image_h)))
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "rasterize: null arrays");
  cudaSetDevice(ctx->device);
  const size_t V = (size_t)n_vertices, T = (size_t)n_triangles;
  size_t img_bytes = 0;
  for (int i = 0; i < k; ++i) img_bytes += up((size_t)image_w[i] * image_h[i] * 3);
  const size_t bytes = up(V * 24) + up(T * 12) + up((size_t)k * V) + up((size_t)k * V * 8) + up((size_t)k * V * 4) +
                       img_bytes + up(raster_scratch_bytes((int)V, w, h)) + up(npx * 4) + up(npx * 3) + up(npx) + 4096;
  VC_TRY(ensure(ctx, ctx->scratch_dev, bytes));
  Arena a{P<uint8_t>(ctx->scratch_dev)};
  double* dpos = a.take<double>(V * 3);
  int32_t* dtri = a.take<int32_t>(T * 3);
  uint8_t* dvis = a.take<uint8_t>((size_t)k * V);
  float* duv = a.take<float>((size_t)k * V * 2);
  float* dw = a.take<float>((size_t)k * V);
  RzImages im{};
  for (int i = 0; i < k; ++i) {
    uint8_t* d = a.take<uint8_t>((size_t)image_w[i] * image_h[i] * 3);
    VC_TRY(h2d(ctx, d, images[i], (size_t)image_w[i] * image_h[i] * 3));
    im.rgb[i] = d, im.w[i] = image_w[i], im.h[i] = image_h[i];
  }
  void* scratch = a.take<uint8_t>(raster_scratch_bytes((int)V, w, h));
  float* ddepth = a.take<float>(npx);
  uint8_t* dcolor = a.take<uint8_t>(npx * 3);
  uint8_t* dsil = a.take<uint8_t>(npx);
  VC_TRY(h2d(ctx, dpos, vertices, V * 24));
  VC_TRY(h2d(ctx, dtri, triangles, T * 12));
  VC_TRY(h2d(ctx, dvis, visible, (size_t)k * V));
  VC_TRY(h2d(ctx, duv, uv, (size_t)k * V * 8));
  VC_TRY(h2d(ctx, dw, weight, (size_t)k * V * 4));
  RzMesh m{dpos, dtri, (int)V, (int)T, k, dvis, duv, dw};
  // world_to_cam = camera.pose.inverse() (rasterize.cpp:45; types.hpp:48)
  RzCamera c;
  c.fx = intr->fx, c.fy = intr->fy, c.cx = intr->cx, c.cy = intr->cy, c.w = w, c.h = h;
  for (int r = 0; r < 3; ++r)
    for (int q = 0; q < 3; ++q) c.Ri[r * 3 + q] = pose->R[q * 3 + r];
  for (int r = 0; r < 3; ++r)
    c.ti[r] = -((c.Ri[r * 3 + 0] * pose->t[0] + c.Ri[r * 3 + 1] * pose->t[1]) + c.Ri[r * 3 + 2] * pose->t[2]);
  int32_t* off = nullptr;
  launch_raster_count(m, c, scratch, ctx->st, &off);
  VC_CUDA(cudaGetLastError());
  int32_t nfrag = 0;
  VC_CUDA(cudaMemcpyAsync(&nfrag, off + npx, 4, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  VC_TRY(ensure(ctx, ctx->scratch_dev2, (size_t)std::max(nfrag, 1) * sizeof(Frag)));
  launch_raster_finish(m, c, im, mode == VC_RENDER_COLOR_PER_VERTEX ? 1 : 0, scratch, P<Frag>(ctx->scratch_dev2),
                       ddepth, dcolor, dsil, ctx->st);
  VC_CUDA(cudaGetLastError());
  VC_CUDA(cudaMemcpyAsync(depth, ddepth, npx * 4, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaMemcpyAsync(color, dcolor, npx * 3, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaMemcpyAsync(silhouette, dsil, npx, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}

// metrics.cpp:12-23
vc_status vc_vre(vc_ctx* ctx, const uint8_t* rendered, const uint8_t* ground, int32_t w, int32_t h, double* out) {
  if (!ctx || !rendered || !ground || !out || w <= 0 || h <= 0)
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "vre: bad arguments");
  cudaSetDevice(ctx->device);
  const size_t n = (size_t)w * h;
  VC_TRY(ensure(ctx, ctx->scratch_dev, 2 * up(n) + 256));
  Arena a{P<uint8_t>(ctx->scratch_dev)};
  uint8_t* da = a.take<uint8_t>(n);
  uint8_t* db = a.take<uint8_t>(n);
  unsigned long long* cnt = a.take<unsigned long long>(2);
  VC_TRY(h2d(ctx, da, rendered, n));
  VC_TRY(h2d(ctx, db, ground, n));
  launch_vre(da, db, (int)n, cnt, ctx->st);
  unsigned long long hc[2];
  VC_CUDA(cudaMemcpyAsync(hc, cnt, 16, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  *out = hc[1] == 0 ? 0.0 : (double)hc[0] / (double)hc[1];
  return VC_OK;
}

vc_status vc_distance_transform(vc_ctx* ctx, const uint8_t* mask, int32_t w, int32_t h, float* out) {
  if (!ctx || !mask || !out || w <= 0 || h <= 0) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "distance_transform: bad arguments");
  cudaSetDevice(ctx->device);
  const size_t n = (size_t)w * h;
  VC_TRY(ensure(ctx, ctx->scratch_dev, up(n) + up(n * 4) + up(dt_scratch_bytes(w, h)) + 256));
  Arena a{P<uint8_t>(ctx->scratch_dev)};
  uint8_t* dm = a.take<uint8_t>(n);
  float* dout = a.take<float>(n);
  void* s = a.take<uint8_t>(dt_scratch_bytes(w, h));
  VC_TRY(h2d(ctx, dm, mask, n));
  launch_distance_transform(dm, w, h, s, dout, ctx->st);
  VC_CUDA(cudaGetLastError());
  VC_CUDA(cudaMemcpyAsync(out, dout, n * 4, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}

// metrics.cpp:25-43; *has_value = 0 when either mask is empty (nullopt)
vc_status vc_hausdorff2d(vc_ctx* ctx, const uint8_t* rendered, const uint8_t* ground, int32_t w, int32_t h,
                         double* out, int32_t* has_value) {
  if (!ctx || !rendered || !ground || !out || !has_value || w <= 0 || h <= 0)
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "hausdorff2d: bad arguments");
  const size_t n = (size_t)w * h;
  bool any_r = false, any_g = false;
  for (size_t i = 0; i < n && !(any_r && any_g); ++i) any_r = any_r || rendered[i], any_g = any_g || ground[i];
  *has_value = 0;
  if (!any_r || !any_g) return VC_OK;
  cudaSetDevice(ctx->device);
  VC_TRY(ensure(ctx, ctx->scratch_dev, 2 * up(n) + 2 * up(n * 4) + up(dt_scratch_bytes(w, h)) + 512));
  Arena a{P<uint8_t>(ctx->scratch_dev)};
  uint8_t* da = a.take<uint8_t>(n);
  uint8_t* db = a.take<uint8_t>(n);
  float* dta = a.take<float>(n);
  float* dtb = a.take<float>(n);
  void* s = a.take<uint8_t>(dt_scratch_bytes(w, h));
  int* mb = a.take<int>(1);
  VC_TRY(h2d(ctx, da, rendered, n));
  VC_TRY(h2d(ctx, db, ground, n));
  launch_distance_transform(da, w, h, s, dta, ctx->st);
  launch_distance_transform(db, w, h, s, dtb, ctx->st);
  launch_hausdorff(da, db, dta, dtb, (int)n, mb, ctx->st);
  VC_CUDA(cudaGetLastError());
  int bits = 0;
  VC_CUDA(cudaMemcpyAsync(&bits, mb, 4, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  float f;
  std::memcpy(&f, &bits, 4);
  *out = (double)f;
  *has_value = 1;
  return VC_OK;
}

// metrics.cpp:86-94: sqrt(mean of nearest squared distances), summed in ground order
vc_status vc_cp_rmse(vc_ctx* ctx, const double* ground, int32_t n_ground, const double* recon, int32_t n_recon,
                     double* out) {
  if (!ctx || !out || n_ground < 0 || n_recon < 0) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "cp_rmse: bad arguments");
  if (n_ground == 0 || n_recon == 0 || !ground || !recon)
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "cp_rmse: empty point cloud");
  cudaSetDevice(ctx->device);
  VC_TRY(ensure(ctx, ctx->scratch_dev, up((size_t)n_ground * 24) + up((size_t)n_recon * 24) + up((size_t)n_ground * 8)));
  Arena a{P<uint8_t>(ctx->scratch_dev)};
  double* dg = a.take<double>((size_t)n_ground * 3);
  double* dr = a.take<double>((size_t)n_recon * 3);
  double* dn = a.take<double>((size_t)n_ground);
  VC_TRY(h2d(ctx, dg, ground, (size_t)n_ground * 24));
  VC_TRY(h2d(ctx, dr, recon, (size_t)n_recon * 24));
  launch_nearest(dg, n_ground, dr, n_recon, dn, ctx->st);
  VC_CUDA(cudaGetLastError());
  std::vector<double> nn((size_t)n_ground);
  VC_CUDA(cudaMemcpyAsync(nn.data(), dn, (size_t)n_ground * 8, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  double sum = 0;
  for (double v : nn) sum += v;
  *out = std::sqrt(sum / (double)n_ground);
  return VC_OK;
}

// ssim.cpp:159-176
vc_status vc_wms3im(vc_ctx* ctx, const uint8_t* rendered, const uint8_t* ground, const uint8_t* silhouette, int32_t w,
                    int32_t h, const vc_wms3im_options* opt_in, double* out, int32_t* has_value) {
  if (!ctx || !rendered || !ground || !silhouette || !out || !has_value || w <= 0 || h <= 0)
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "wms3im: bad arguments");
  vc_wms3im_options opt;
  if (opt_in) {
    opt = *opt_in;
  } else {  // Wms3imOptions defaults (metrics.hpp:30-41)
    opt.scales = 3;
    const double al[3] = {0.0, 0.0, 0.1333}, be[3] = {0.0448, 0.3001, 0.1333};
    for (int j = 0; j < 3; ++j) opt.alpha[j] = al[j], opt.beta[j] = be[j], opt.gamma[j] = be[j];
    opt.c1 = (0.01 * 255) * (0.01 * 255);
    opt.c2 = (0.03 * 255) * (0.03 * 255);
    opt.c3 = (0.03 * 255) * (0.03 * 255) / 2.0;
    opt.window = 11;
    opt.sigma = 1.5;
  }
  if (opt.scales < 1 || opt.scales > 3 || opt.window < 1) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "wms3im: options");
  const size_t n = (size_t)w * h;
  bool any = false;
  for (size_t i = 0; i < n && !any; ++i) any = silhouette[i] != 0;
  *has_value = 0;
  if (!any) return VC_OK;
  // gaussian_kernel (ssim.cpp:21-31) on the host: std::exp as the reference
  std::vector<double> k(opt.window);
  const int r = opt.window / 2;
  double ksum = 0;
  for (int i = 0; i < opt.window; ++i) {
    k[i] = std::exp(-0.5 * (i - r) * (i - r) / (opt.sigma * opt.sigma));
    ksum += k[i];
  }
  for (auto& v : k) v /= ksum;
  cudaSetDevice(ctx->device);
  VC_TRY(ensure(ctx, ctx->scratch_dev, 2 * up(n * 3) + 2 * up(n) + 11 * up(n * 8) + up(n * 32) + up(k.size() * 8) + 4096));
  Arena a{P<uint8_t>(ctx->scratch_dev)};
  uint8_t* dr = a.take<uint8_t>(n * 3);
  uint8_t* dgt = a.take<uint8_t>(n * 3);
  uint8_t* dm = a.take<uint8_t>(n);
  uint8_t* dm2 = a.take<uint8_t>(n);
  double* x = a.take<double>(n);
  double* y = a.take<double>(n);
  double* x2 = a.take<double>(n);
  double* y2 = a.take<double>(n);
  double* t = a.take<double>(n);
  double* p = a.take<double>(n);
  double* mx = a.take<double>(n);
  double* my = a.take<double>(n);
  double* xx = a.take<double>(n);
  double* yy = a.take<double>(n);
  double* xy = a.take<double>(n);
  double* terms = a.take<double>(n * 4);
  double* dk = a.take<double>(k.size());
  VC_TRY(h2d(ctx, dr, rendered, n * 3));
  VC_TRY(h2d(ctx, dgt, ground, n * 3));
  VC_TRY(h2d(ctx, dm, silhouette, n));
  VC_TRY(h2d(ctx, dk, k.data(), k.size() * 8));
  launch_ssim_gray(dr, (int)n, x, ctx->st);
  launch_ssim_gray(dgt, (int)n, y, ctx->st);
  int cw = w, ch = h;
  double score = 1.0;
  std::vector<double> ht;
  for (int j = 0; j < opt.scales; ++j) {
    if (j > 0) {  // downsample2 / downsample2_or (ssim.cpp:114-153)
      const int ow = std::max(1, cw / 2), oh = std::max(1, ch / 2);
      launch_ssim_down(x, cw, ch, x2, ow, oh, ctx->st);
      launch_ssim_down(y, cw, ch, y2, ow, oh, ctx->st);
      launch_ssim_down_or(dm, cw, ch, dm2, ow, oh, ctx->st);
      std::swap(x, x2), std::swap(y, y2), std::swap(dm, dm2);
      cw = ow, ch = oh;
    }
    const int cn = cw * ch;
    launch_ssim_gauss(x, t, mx, cw, ch, dk, r, ctx->st);
    launch_ssim_gauss(y, t, my, cw, ch, dk, r, ctx->st);
    launch_ssim_mul(x, x, p, cn, ctx->st);
    launch_ssim_gauss(p, t, xx, cw, ch, dk, r, ctx->st);
    launch_ssim_mul(y, y, p, cn, ctx->st);
    launch_ssim_gauss(p, t, yy, cw, ch, dk, r, ctx->st);
    launch_ssim_mul(x, y, p, cn, ctx->st);
    launch_ssim_gauss(p, t, xy, cw, ch, dk, r, ctx->st);
    launch_ssim_terms(mx, my, xx, yy, xy, dm, cw, ch, r, opt.c1, opt.c2, opt.c3, terms, ctx->st);
    VC_CUDA(cudaGetLastError());
    ht.resize((size_t)cn * 4);
    VC_CUDA(cudaMemcpyAsync(ht.data(), terms, (size_t)cn * 32, cudaMemcpyDeviceToHost, ctx->st));
    VC_CUDA(cudaStreamSynchronize(ctx->st));
    // ssim.cpp:74-107 pooled sums in raster order over the masked pixels
    double sl = 0, sc = 0, ss = 0, sw = 0;
    std::vector<uint8_t> hm((size_t)cn);
    VC_CUDA(cudaMemcpy(hm.data(), dm, (size_t)cn, cudaMemcpyDeviceToHost));
    for (int i = 0; i < cn; ++i) {
      if (!hm[i]) continue;
      sl += ht[4 * (size_t)i], sc += ht[4 * (size_t)i + 1], ss += ht[4 * (size_t)i + 2], sw += ht[4 * (size_t)i + 3];
    }
    double l = 1, c = 1, s = 1;
    if (sw > 0) l = sl / sw, c = sc / sw, s = ss / sw;
    l = std::max(l, 1e-12), c = std::max(c, 1e-12), s = std::max(s, 1e-12);
    score *= std::pow(l, opt.alpha[j]) * std::pow(c, opt.beta[j]) * std::pow(s, opt.gamma[j]);
  }
  *out = score;
  *has_value = 1;
  return VC_OK;
}

}  // extern "C"

// SPDX-License-Identifier: Apache-2.0
//
// Evaluation rasterizer on sm_100a: eval::rasterize
// (rasterize.cpp:35-161), uv-blend and colour-per-vertex modes, fp64 with the
// reference's operation order.
//
// The reference walks the triangles in order with a float z-buffer whose test
// (`zbuf != 0 && z >= zbuf`) compares the fragment's fp64 depth against the
// previously stored float — an order-dependent rule.  So instead of an atomic
// depth test the GPU builds every fragment (pixel, triangle, barycentrics, z),
// buckets them per pixel, sorts each pixel's list by triangle index and replays
// the reference's sequential test per pixel; only the winning fragment is shaded.
//
//   rz_vertex    camera-space position (world_to_cam = pose.inverse()),
//                in-front flag (z > 1 mm), screen position
//   rz_count     per triangle: bounding-box scan, fragments per pixel (atomics)
//   rz_scan      pixel offsets (single CTA)
//   rz_emit      the fragments, scattered to their pixel's slots
//   rz_resolve   per pixel: order by triangle, sequential z test, shade the winner
//   rz_vcolor    colour-per-vertex mode's equal-weight vertex colours
#include <cfloat>
#include <cstdint>

#include "vc_device.cuh"

namespace vc {

struct RzCamera {
  double fx, fy, cx, cy;
  int32_t w, h;
  double Ri[9], ti[3];  // world -> camera (Pose::inverse, types.hpp:48)
};

struct RzMesh {
  const double* pos;  // 3V
  const int32_t* tri; // 3T
  int V, T, K;
  const uint8_t* vis;  // K*V
  const float* uv;     // 2*K*V
  const float* w;      // K*V
};

struct RzImages {
  const uint8_t* rgb[16];
  int32_t w[16], h[16];
};

struct Frag {
  double z, la, lb, lc;
  int32_t tri, pad;
};

namespace {

__global__ void rz_vertex_kernel(RzMesh m, RzCamera c, double* cam, double* scr, uint8_t* front) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < m.V; v += gridDim.x * blockDim.x) {
    const d3 X = mk3(m.pos[3 * v], m.pos[3 * v + 1], m.pos[3 * v + 2]);
    const d3 p = add3(mat3(c.Ri, X), ld3(c.ti));
    cam[3 * v] = p.x, cam[3 * v + 1] = p.y, cam[3 * v + 2] = p.z;
    const bool f = p.z > 1.0;  // kNearMm
    front[v] = f;
    if (f) {
      scr[2 * v] = dadd(ddiv(dmul(c.fx, p.x), p.z), c.cx);
      scr[2 * v + 1] = dadd(ddiv(dmul(c.fy, p.y), p.z), c.cy);
    }
  }
}

struct TriSetup {
  double pax, pay, pbx, pby, pcx, pcy, area, iza, izb, izc;
  int x0, x1, y0, y1;
  bool ok;
};

__device__ TriSetup tri_setup(const RzMesh& m, const RzCamera& c, const double* cam, const double* scr,
                              const uint8_t* front, int t) {
  TriSetup s;
  s.ok = false;
  const int a = m.tri[3 * t], b = m.tri[3 * t + 1], cc = m.tri[3 * t + 2];
  if (!front[a] || !front[b] || !front[cc]) return s;
  s.pax = scr[2 * a], s.pay = scr[2 * a + 1], s.pbx = scr[2 * b], s.pby = scr[2 * b + 1];
  s.pcx = scr[2 * cc], s.pcy = scr[2 * cc + 1];
  s.area = dsub(dmul(dsub(s.pbx, s.pax), dsub(s.pcy, s.pay)), dmul(dsub(s.pby, s.pay), dsub(s.pcx, s.pax)));
  if (fabs(s.area) < 1e-12) return s;
  s.x0 = max(0, (int)ceil(fmin(fmin(s.pax, s.pbx), s.pcx)));
  s.x1 = min(c.w - 1, (int)floor(fmax(fmax(s.pax, s.pbx), s.pcx)));
  s.y0 = max(0, (int)ceil(fmin(fmin(s.pay, s.pby), s.pcy)));
  s.y1 = min(c.h - 1, (int)floor(fmax(fmax(s.pay, s.pby), s.pcy)));
  s.iza = ddiv(1.0, cam[3 * a + 2]), s.izb = ddiv(1.0, cam[3 * b + 2]), s.izc = ddiv(1.0, cam[3 * cc + 2]);
  s.ok = true;
  return s;
}

// rasterize.cpp:101-119: barycentrics of pixel (x, y), inside test, depth
__device__ __forceinline__ bool frag_at(const TriSetup& s, int x, int y, Frag& f) {
  const double px = (double)x, py = (double)y;
  const double bx = dsub(s.pbx, px), by = dsub(s.pby, py), cx = dsub(s.pcx, px), cy = dsub(s.pcy, py);
  const double ax = dsub(s.pax, px), ay = dsub(s.pay, py);
  double la = dsub(dmul(bx, cy), dmul(by, cx));
  double lb = dsub(dmul(cx, ay), dmul(cy, ax));
  double lc = dsub(dmul(ax, by), dmul(ay, bx));
  if (s.area < 0) la = -la, lb = -lb, lc = -lc;
  if (la < 0 || lb < 0 || lc < 0) return false;
  const double den = dadd(dadd(la, lb), lc);
  if (den <= 0) return false;
  la = ddiv(la, den), lb = ddiv(lb, den), lc = ddiv(lc, den);
  const double inv_z = dadd(dadd(dmul(la, s.iza), dmul(lb, s.izb)), dmul(lc, s.izc));
  f.z = ddiv(1.0, inv_z);
  f.la = la, f.lb = lb, f.lc = lc;
  return true;
}

__global__ void rz_count_kernel(RzMesh m, RzCamera c, const double* cam, const double* scr, const uint8_t* front,
                                int32_t* cnt) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m.T; t += gridDim.x * blockDim.x) {
    const TriSetup s = tri_setup(m, c, cam, scr, front, t);
    if (!s.ok) continue;
    Frag f;
    for (int y = s.y0; y <= s.y1; ++y)
      for (int x = s.x0; x <= s.x1; ++x)
        if (frag_at(s, x, y, f)) atomicAdd(cnt + (size_t)y * c.w + x, 1);
  }
}

__global__ void __launch_bounds__(1024) rz_scan_kernel(const int32_t* cnt, int32_t* off, int32_t* cursor, int n) {
  __shared__ int wsum[32];
  const int per = (n + 1023) / 1024;
  const int b0 = min(n, (int)threadIdx.x * per), b1 = min(n, b0 + per);
  int tot = 0;
  for (int i = b0; i < b1; ++i) tot += cnt[i];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = tot;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int s = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += t;
    }
    wsum[lane] = s;
  }
  __syncthreads();
  int run = (wid ? wsum[wid - 1] : 0) + inc - tot;
  for (int i = b0; i < b1; ++i) off[i] = run, cursor[i] = run, run += cnt[i];
  if (threadIdx.x == 1023) off[n] = wsum[31];
}

__global__ void rz_emit_kernel(RzMesh m, RzCamera c, const double* cam, const double* scr, const uint8_t* front,
                               int32_t* cursor, Frag* frags) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m.T; t += gridDim.x * blockDim.x) {
    const TriSetup s = tri_setup(m, c, cam, scr, front, t);
    if (!s.ok) continue;
    Frag f;
    f.tri = t, f.pad = 0;
    for (int y = s.y0; y <= s.y1; ++y)
      for (int x = s.x0; x <= s.x1; ++x)
        if (frag_at(s, x, y, f)) frags[atomicAdd(cursor + (size_t)y * c.w + x, 1)] = f;
  }
}

// rasterize.cpp:12-27: appearance::denormalize_uv, clamp, bilinear, lround
__device__ void sample_bilinear_rz(const uint8_t* img, int W, int H, double ux, double uy, int out[3]) {
  const double px = dsub(dmul(ux, (double)W), 0.5), py = dsub(dmul(uy, (double)H), 0.5);
  int x0 = (int)floor(px), y0 = (int)floor(py);
  x0 = x0 < 0 ? 0 : (x0 > W - 1 ? W - 1 : x0);
  y0 = y0 < 0 ? 0 : (y0 > H - 1 ? H - 1 : y0);
  const int x1 = min(x0 + 1, W - 1), y1 = min(y0 + 1, H - 1);
  double tx = dsub(px, (double)x0), ty = dsub(py, (double)y0);
  tx = tx < 0.0 ? 0.0 : (tx > 1.0 ? 1.0 : tx);
  ty = ty < 0.0 ? 0.0 : (ty > 1.0 ? 1.0 : ty);
  const uint8_t* r0 = img + (size_t)y0 * W * 3;
  const uint8_t* r1 = img + (size_t)y1 * W * 3;
  for (int ch = 0; ch < 3; ++ch) {
    const double a = dadd(dmul((double)r0[3 * x0 + ch], dsub(1.0, tx)), dmul((double)r0[3 * x1 + ch], tx));
    const double b = dadd(dmul((double)r1[3 * x0 + ch], dsub(1.0, tx)), dmul((double)r1[3 * x1 + ch], tx));
    out[ch] = (int)(uint8_t)lround_d(dadd(dmul(a, dsub(1.0, ty)), dmul(b, ty)));
  }
}

// rasterize.cpp:50-68: equal-weight average of the visible views' samples
__global__ void rz_vcolor_kernel(RzMesh m, RzImages im, double* vcol) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < m.V; v += gridDim.x * blockDim.x) {
    double r = 0, g = 0, b = 0;
    int n = 0;
    for (int k = 0; k < m.K; ++k) {
      if (!m.vis[(size_t)k * m.V + v]) continue;
      int s[3];
      const size_t q = (size_t)k * m.V + v;
      sample_bilinear_rz(im.rgb[k], im.w[k], im.h[k], (double)m.uv[2 * q], (double)m.uv[2 * q + 1], s);
      r = dadd(r, (double)s[0]), g = dadd(g, (double)s[1]), b = dadd(b, (double)s[2]);
      ++n;
    }
    if (n > 0)
      vcol[3 * v] = ddiv(r, (double)n), vcol[3 * v + 1] = ddiv(g, (double)n), vcol[3 * v + 2] = ddiv(b, (double)n);
    else
      vcol[3 * v] = vcol[3 * v + 1] = vcol[3 * v + 2] = 200.0;  // kUntexturedGray
  }
}

__device__ __forceinline__ uint8_t clamp_u8(double v) { return (uint8_t)(v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v)); }

__global__ void rz_resolve_kernel(RzMesh m, RzCamera c, RzImages im, int mode, const int32_t* __restrict__ off,
                                  Frag* frags, const double* __restrict__ vcol, const double* __restrict__ cam,
                                  float* depth, uint8_t* color, uint8_t* sil) {
  const int n = c.w * c.h;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const int b = off[p], e = off[p + 1];
    // insertion sort of this pixel's fragments by triangle index (submission order)
    for (int i = b + 1; i < e; ++i) {
      const Frag f = frags[i];
      int j = i - 1;
      while (j >= b && frags[j].tri > f.tri) frags[j + 1] = frags[j], --j;
      frags[j + 1] = f;
    }
    float zb = 0.f;
    int win = -1;
    for (int i = b; i < e; ++i) {  // rasterize.cpp:120-123
      const double z = frags[i].z;
      if (zb != 0.f && z >= (double)zb) continue;
      zb = (float)z;
      win = i;
    }
    depth[p] = zb;
    sil[p] = win >= 0 ? 1 : 0;
    uint8_t out[3] = {0, 0, 0};
    if (win >= 0) {
      const Frag f = frags[win];
      const int a = m.tri[3 * f.tri], bb = m.tri[3 * f.tri + 1], cc = m.tri[3 * f.tri + 2];
      const double iza = ddiv(1.0, cam[3 * a + 2]), izb = ddiv(1.0, cam[3 * bb + 2]), izc = ddiv(1.0, cam[3 * cc + 2]);
      const double z = f.z, la = f.la, lb = f.lb, lc = f.lc;
      if (mode == 1) {  // kColorPerVertex (:126-133)
        for (int ch = 0; ch < 3; ++ch) {
          const double t = dadd(dadd(dmul(dmul(la, vcol[3 * a + ch]), iza), dmul(dmul(lb, vcol[3 * bb + ch]), izb)),
                                dmul(dmul(lc, vcol[3 * cc + ch]), izc));
          out[ch] = clamp_u8(dmul(z, t));
        }
      } else {  // kUvBlend (:134-157)
        double r = 0, g = 0, bl = 0, wsum = 0;
        for (int k = 0; k < m.K; ++k) {
          const size_t qa = (size_t)k * m.V + a, qb = (size_t)k * m.V + bb, qc = (size_t)k * m.V + cc;
          if (!(m.vis[qa] && m.vis[qb] && m.vis[qc])) continue;
          const double wk = dmul(z, dadd(dadd(dmul(dmul(la, (double)m.w[qa]), iza), dmul(dmul(lb, (double)m.w[qb]), izb)),
                                         dmul(dmul(lc, (double)m.w[qc]), izc)));
          if (wk <= 1e-9) continue;
          double uv[2];
          for (int d = 0; d < 2; ++d)
            uv[d] = dmul(z, dadd(dadd(dmul(dmul(la, (double)m.uv[2 * qa + d]), iza),
                                      dmul(dmul(lb, (double)m.uv[2 * qb + d]), izb)),
                                 dmul(dmul(lc, (double)m.uv[2 * qc + d]), izc)));
          int s[3];
          sample_bilinear_rz(im.rgb[k], im.w[k], im.h[k], uv[0], uv[1], s);
          r = dadd(r, dmul(wk, (double)s[0])), g = dadd(g, dmul(wk, (double)s[1]));
          bl = dadd(bl, dmul(wk, (double)s[2])), wsum = dadd(wsum, wk);
        }
        if (wsum > 1e-9) {
          out[0] = clamp_u8(ddiv(r, wsum)), out[1] = clamp_u8(ddiv(g, wsum)), out[2] = clamp_u8(ddiv(bl, wsum));
        } else {
          out[0] = out[1] = out[2] = 200;
        }
      }
    }
    color[3 * p] = out[0], color[3 * p + 1] = out[1], color[3 * p + 2] = out[2];
  }
}

}  // namespace

size_t raster_scratch_bytes(int V, int w, int h) {
  return (size_t)V * (24 + 16 + 1 + 24) + ((size_t)w * h + 1) * 4 * 3 + 4096;
}

// Two passes over the triangles (count, emit) around one pixel scan; the
// fragment buffer is caller-owned (capacity from the count).
int64_t launch_raster_count(RzMesh m, RzCamera c, void* scratch, cudaStream_t st, int32_t** off_out) {
  uint8_t* p = static_cast<uint8_t*>(scratch);
  double* cam = reinterpret_cast<double*>(p);
  p += (size_t)m.V * 24;
  double* scr = reinterpret_cast<double*>(p);
  p += (size_t)m.V * 16;
  p += (size_t)m.V * 24;  // vertex colours (launch_raster_finish)
  uint8_t* front = p;
  p += ((size_t)m.V + 15) & ~size_t(15);
  const size_t npx = (size_t)c.w * c.h;
  int32_t* cnt = reinterpret_cast<int32_t*>(p);
  int32_t* off = cnt + npx + 1;
  int32_t* cursor = off + npx + 1;
  cudaMemsetAsync(cnt, 0, npx * 4, st);
  if (m.V > 0) rz_vertex_kernel<<<sm_count() * 2, 256, 0, st>>>(m, c, cam, scr, front);
  if (m.T > 0) rz_count_kernel<<<sm_count() * 4, 128, 0, st>>>(m, c, cam, scr, front, cnt);
  rz_scan_kernel<<<1, 1024, 0, st>>>(cnt, off, cursor, (int)npx);
  *off_out = off;
  return 0;
}

void launch_raster_finish(RzMesh m, RzCamera c, RzImages im, int mode, void* scratch, Frag* frags, float* depth,
                          uint8_t* color, uint8_t* sil, cudaStream_t st) {
  uint8_t* p = static_cast<uint8_t*>(scratch);
  double* cam = reinterpret_cast<double*>(p);
  p += (size_t)m.V * 24;
  double* scr = reinterpret_cast<double*>(p);
  p += (size_t)m.V * 16;
  double* vcol = reinterpret_cast<double*>(p);
  p += (size_t)m.V * 24;
  uint8_t* front = p;
  p += ((size_t)m.V + 15) & ~size_t(15);
  const size_t npx = (size_t)c.w * c.h;
  int32_t* cnt = reinterpret_cast<int32_t*>(p);
  int32_t* off = cnt + npx + 1;
  int32_t* cursor = off + npx + 1;
  if (m.T > 0) rz_emit_kernel<<<sm_count() * 4, 128, 0, st>>>(m, c, cam, scr, front, cursor, frags);
  if (mode == 1 && m.V > 0) rz_vcolor_kernel<<<sm_count() * 2, 128, 0, st>>>(m, im, vcol);
  rz_resolve_kernel<<<sm_count() * 4, 128, 0, st>>>(m, c, im, mode, off, frags, vcol, cam, depth, color, sil);
}

}  // namespace vc

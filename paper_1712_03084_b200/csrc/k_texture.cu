// SPDX-License-Identifier: Apache-2.0
//
// K11 — per-vertex texturing on sm_100a: vertex_visibility + assign_texture
// (/root/reference/proj/core/src/appearance/texture.cpp:11-72) and the
// visibility-weighted multi-view colour blend (rasterize.cpp:12-27
// bilinear sample, rasterize.cpp:136-157 weighting) in one pass, one thread
// per vertex, all K views unrolled.  fp64 with the reference's operation
// order so lround pixel binning is bit-exact.
#include "vc_device.cuh"

namespace vc {
namespace {

// rasterize.cpp:12-27 sample_bilinear (uv -> pixel - 0.5, clamp, lround to uint8)
__device__ void sample_bilinear(const ViewPtrs& v, int W, int H, double uvx, double uvy, double out[3]) {
  const double px = dsub(dmul(uvx, (double)W), 0.5), py = dsub(dmul(uvy, (double)H), 0.5);
  int x0 = (int)floor(px), y0 = (int)floor(py);
  x0 = x0 < 0 ? 0 : (x0 > W - 1 ? W - 1 : x0);
  y0 = y0 < 0 ? 0 : (y0 > H - 1 ? H - 1 : y0);
  const int x1 = min(x0 + 1, W - 1), y1 = min(y0 + 1, H - 1);
  double tx = dsub(px, (double)x0), ty = dsub(py, (double)y0);
  tx = tx < 0.0 ? 0.0 : (tx > 1.0 ? 1.0 : tx);
  ty = ty < 0.0 ? 0.0 : (ty > 1.0 ? 1.0 : ty);
  const uint8_t* r0 = v.rgb + (size_t)y0 * v.rpitch;
  const uint8_t* r1 = v.rgb + (size_t)y1 * v.rpitch;
  const double ux = dsub(1.0, tx), uy = dsub(1.0, ty);
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const double a = dadd(dmul((double)__ldg(r0 + 3 * x0 + ch), ux), dmul((double)__ldg(r0 + 3 * x1 + ch), tx));
    const double b = dadd(dmul((double)__ldg(r1 + 3 * x0 + ch), ux), dmul((double)__ldg(r1 + 3 * x1 + ch), tx));
    out[ch] = (double)(uint8_t)lround_d(dadd(dmul(a, uy), dmul(b, ty)));
  }
}

__global__ void __launch_bounds__(128) texture_kernel(const __grid_constant__ SensorSet ss,
                                                      const float* __restrict__ weight_maps,
                                                      const double* __restrict__ vpos, const DevCtl* ctl,
                                                      double eps_vis, uint8_t* vis, float2* uv, float* wout,
                                                      uint8_t* untex, uint8_t* rgb, int v_cap) {
  if (ctl->status != 0 || ctl->overflow) return;
  const int V = ctl->V;
  if (V > v_cap) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x) {
    const d3 X = mk3(vpos[3 * i], vpos[3 * i + 1], vpos[3 * i + 2]);
    bool any = false;
    double r = 0, g = 0, b = 0, wsum = 0;
    for (int k = 0; k < ss.k; ++k) {
      const DevSensor& s = ss.s[k];
      const ViewPtrs& v = ss.v[k];
      // texture.cpp:19-31 — world_to_cam = pose.inverse(); lround pixel
      uint8_t vk = 0;
      const d3 local = add3(mat3(s.Ri, X), ld3(s.ti));
      double u, w;
      if (project_local(s.fx, s.fy, s.cx, s.cy, local, &u, &w)) {
        const long long px = lround_d(u), py = lround_d(w);
        if (px >= 0 && px < s.w && py >= 0 && py < s.h) {
          if (__ldg(v.mask + py * v.mpitch + px)) {
            const double recorded = (double)__ldg(v.depth + py * v.dpitch + px);
            if (fabs(dsub(recorded, local.z)) < eps_vis) vk = 1;
          }
        }
      }
      float2 uvk = make_float2(0.f, 0.f);
      float wk = 0.f;
      if (vk) {
        any = true;
        // texture.cpp:54-63 — RGB camera UV (apply_inverse of pose.compose),
        // weight map at the lround depth-camera pixel (apply_inverse of pose)
        double ur, vr;
        if (project_local(s.rfx, s.rfy, s.rcx, s.rcy, mat3t(s.Rc, sub3(X, ld3(s.tc))), &ur, &vr)) {
          const double uvx = ddiv(dadd(ur, 0.5), (double)s.rw), uvy = ddiv(dadd(vr, 0.5), (double)s.rh);
          uvk = make_float2((float)uvx, (float)uvy);
          double ud, vd;
          if (project_local(s.fx, s.fy, s.cx, s.cy, mat3t(s.R, sub3(X, ld3(s.t))), &ud, &vd)) {
            const long long px = lround_d(ud), py = lround_d(vd);
            if (px >= 0 && px < s.w && py >= 0 && py < s.h)
              wk = __ldg(weight_maps + ss.pix_offset[k] + py * s.w + px);
          }
          // rasterize.cpp:136-150 at the vertex: skip w <= 1e-9, sum w*s
          const double wd = (double)wk;
          if (wd > 1e-9 && v.rgb) {
            double smp[3];
            sample_bilinear(v, s.rw, s.rh, uvx, uvy, smp);
            r = dadd(r, dmul(wd, smp[0]));
            g = dadd(g, dmul(wd, smp[1]));
            b = dadd(b, dmul(wd, smp[2]));
            wsum = dadd(wsum, wd);
          }
        }
      }
      vis[(size_t)k * V + i] = vk;
      uv[(size_t)k * V + i] = uvk;
      wout[(size_t)k * V + i] = wk;
    }
    untex[i] = any ? 0 : 1;
    // rasterize.cpp:151-156: weighted mean (truncating cast) or light gray 200
    uint8_t c[3] = {200, 200, 200};
    if (wsum > 1e-9) {
      const double m[3] = {ddiv(r, wsum), ddiv(g, wsum), ddiv(b, wsum)};
      for (int ch = 0; ch < 3; ++ch) c[ch] = (uint8_t)(m[ch] < 0.0 ? 0.0 : (m[ch] > 255.0 ? 255.0 : m[ch]));
    }
    rgb[3 * i + 0] = c[0], rgb[3 * i + 1] = c[1], rgb[3 * i + 2] = c[2];
  }
}

__global__ void mesh_f32_kernel(const double* pos, float* posf, const DevCtl* ctl, int v_cap) {
  if (ctl->status != 0 || ctl->overflow) return;
  const int n = 3 * min(ctl->V, v_cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) posf[i] = (float)pos[i];
}

}  // namespace

void launch_texture(const SensorSet& ss, const float* weight_maps, const double* vpos, const DevCtl* ctl,
                    double eps_vis, uint8_t* vis, float2* uv, float* w, uint8_t* untex, uint8_t* rgb, int v_cap,
                    cudaStream_t st) {
  texture_kernel<<<148 * 4, 128, 0, st>>>(ss, weight_maps, vpos, ctl, eps_vis, vis, uv, w, untex, rgb, v_cap);
}

void launch_mesh_to_f32(const double* pos, float* posf, const DevCtl* ctl, int v_cap, cudaStream_t st) {
  mesh_f32_kernel<<<148 * 2, 256, 0, st>>>(pos, posf, ctl, v_cap);
}

}  // namespace vc

// SPDX-License-Identifier: Apache-2.0
//
// K11 — per-vertex texturing on sm_100a: vertex_visibility + assign_texture
// (/root/reference/proj/core/src/appearance/texture.cpp:11-72) and the
// visibility-weighted multi-view colour blend (rasterize.cpp:12-27
// bilinear sample, rasterize.cpp:136-157 weighting) in one pass, one lane per
// (vertex, view).  fp64 with the reference's operation
// order so lround pixel binning is bit-exact.
#include "vc_color.cuh"
#include "vc_device.cuh"

namespace vc {
namespace {

// rasterize.cpp:12-27 sample_bilinear (uv -> pixel - 0.5, clamp, lround to
// uint8); with a colour correction the four texels are corrected first
// (ColorCorrection::apply on the image, sequence.cpp:71-73)
__device__ void sample_bilinear(const ViewPtrs& v, const DevSensor& s, int W, int H, double uvx, double uvy,
                                double out[3]) {
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
  uint8_t c00[3], c10[3], c01[3], c11[3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    c00[ch] = __ldg(r0 + 3 * x0 + ch), c10[ch] = __ldg(r0 + 3 * x1 + ch);
    c01[ch] = __ldg(r1 + 3 * x0 + ch), c11[ch] = __ldg(r1 + 3 * x1 + ch);
  }
  if (s.cc_on && !(s.cc_gain == 1.0 && s.cc_offset == 0.0)) {  // identity map: image unchanged (:151-153)
    value_map_rgb(c00, s.cc_gain, s.cc_offset), value_map_rgb(c10, s.cc_gain, s.cc_offset);
    value_map_rgb(c01, s.cc_gain, s.cc_offset), value_map_rgb(c11, s.cc_gain, s.cc_offset);
  }
  const double ux = dsub(1.0, tx), uy = dsub(1.0, ty);
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const double a = dadd(dmul((double)c00[ch], ux), dmul((double)c10[ch], tx));
    const double b = dadd(dmul((double)c01[ch], ux), dmul((double)c11[ch], tx));
    out[ch] = (double)(uint8_t)lround_d(dadd(dmul(a, uy), dmul(b, ty)));
  }
}

// One lane per (vertex, view): a group of G = pow2 >= K adjacent lanes per
// vertex runs the K views' dependent loads (mask -> depth, weight map, RGB)
// side by side; the group's first lane then forms the blend in view order
// with the same fp64 operations as the reference's sequential loop.  The
// fp32 copy of the vertex positions (the output format) is written here too.
__global__ void __launch_bounds__(128, 8) texture_kernel(const __grid_constant__ SensorSet ss,
                                                      const float* __restrict__ weight_maps,
                                                      const double* __restrict__ vpos, const DevCtl* ctl,
                                                      double eps_vis, uint8_t* vis, float2* uv, float* wout,
                                                      uint8_t* untex, uint8_t* rgb, float* posf, int v_cap,
                                                      int lg) {
  // the K sensors' parameters in shared memory: a warp's lanes index them by
  // view, and divergent indices into the kernel-parameter bank serialise
  __shared__ DevSensor sh_s[kMaxViews];
  __shared__ ViewPtrs sh_v[kMaxViews];
  __shared__ int64_t sh_off[kMaxViews];
  if (ctl->status != 0 || ctl->overflow) return;
  const int V = ctl->V;
  if (V > v_cap) return;
  const int G = 1 << lg, K = ss.k;
  {
    static_assert(sizeof(DevSensor) % 8 == 0 && sizeof(ViewPtrs) % 8 == 0, "8-byte words");
    constexpr int WS = sizeof(DevSensor) / 8, WV = sizeof(ViewPtrs) / 8;
    const uint64_t* gs = reinterpret_cast<const uint64_t*>(ss.s);
    const uint64_t* gv = reinterpret_cast<const uint64_t*>(ss.v);
    uint64_t* ds = reinterpret_cast<uint64_t*>(sh_s);
    uint64_t* dv = reinterpret_cast<uint64_t*>(sh_v);
    for (int j = threadIdx.x; j < K * WS; j += blockDim.x) ds[j] = gs[j];
    for (int j = threadIdx.x; j < K * WV; j += blockDim.x) dv[j] = gv[j];
    for (int j = threadIdx.x; j < K; j += blockDim.x) sh_off[j] = ss.pix_offset[j];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, k = lane & (G - 1), lead = lane - k;
  const int per_warp = 32 >> lg;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int base = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * per_warp; base < V;
       base += warps * per_warp) {
    const int i = base + (lane >> lg);
    const bool live = i < V && k < K;
    uint8_t vk = 0;
    float2 uvk = make_float2(0.f, 0.f);
    float wk = 0.f;
    bool contrib = false;
    double tr = 0.0, tg = 0.0, tb = 0.0, twd = 0.0;
    if (live) {
      const d3 X = mk3(vpos[3 * i], vpos[3 * i + 1], vpos[3 * i + 2]);
      const DevSensor& s = sh_s[k];
      const ViewPtrs& v = sh_v[k];
      // texture.cpp:19-31 — world_to_cam = pose.inverse(); lround pixel
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
      if (vk) {
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
              wk = __ldg(weight_maps + sh_off[k] + py * s.w + px);
          }
          // rasterize.cpp:136-150 at the vertex: skip w <= 1e-9, terms w*s
          const double wd = (double)wk;
          if (wd > 1e-9 && v.rgb) {
            double smp[3];
            sample_bilinear(v, s, s.rw, s.rh, uvx, uvy, smp);
            contrib = true;
            tr = dmul(wd, smp[0]), tg = dmul(wd, smp[1]), tb = dmul(wd, smp[2]), twd = wd;
          }
        }
      }
      vis[(size_t)k * V + i] = vk;
      uv[(size_t)k * V + i] = uvk;
      wout[(size_t)k * V + i] = wk;
    }
    // the group's first lane sums the views in order (rasterize.cpp:136-157)
    bool any = false;
    double r = 0, g = 0, b = 0, wsum = 0;
    for (int kk = 0; kk < K; ++kk) {
      const int src = lead + kk;
      const bool c = __shfl_sync(0xffffffffu, contrib, src);
      any |= __shfl_sync(0xffffffffu, vk, src) != 0;
      const double xr = __shfl_sync(0xffffffffu, tr, src), xg = __shfl_sync(0xffffffffu, tg, src),
                   xb = __shfl_sync(0xffffffffu, tb, src), xw = __shfl_sync(0xffffffffu, twd, src);
      if (c) r = dadd(r, xr), g = dadd(g, xg), b = dadd(b, xb), wsum = dadd(wsum, xw);
    }
    if (k == 0 && i < V) {
      untex[i] = any ? 0 : 1;
      // rasterize.cpp:151-156: weighted mean (truncating cast) or light gray 200
      uint8_t c[3] = {200, 200, 200};
      if (wsum > 1e-9) {
        const double m[3] = {ddiv(r, wsum), ddiv(g, wsum), ddiv(b, wsum)};
        for (int ch = 0; ch < 3; ++ch) c[ch] = (uint8_t)(m[ch] < 0.0 ? 0.0 : (m[ch] > 255.0 ? 255.0 : m[ch]));
      }
      rgb[3 * i + 0] = c[0], rgb[3 * i + 1] = c[1], rgb[3 * i + 2] = c[2];
      if (posf)
        for (int c3 = 0; c3 < 3; ++c3) posf[3 * i + c3] = (float)vpos[3 * i + c3];
    }
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
                    cudaStream_t st, float* posf) {
  int lg = 0;
  while ((1 << lg) < ss.k) ++lg;  // K <= 16 lanes per vertex
  texture_kernel<<<sm_count() * 8, 128, 0, st>>>(ss, weight_maps, vpos, ctl, eps_vis, vis, uv, w, untex, rgb, posf, v_cap,
                                          lg);
}

void launch_mesh_to_f32(const double* pos, float* posf, const DevCtl* ctl, int v_cap, cudaStream_t st) {
  mesh_f32_kernel<<<sm_count() * 2, 256, 0, st>>>(pos, posf, ctl, v_cap);
}

}  // namespace vc

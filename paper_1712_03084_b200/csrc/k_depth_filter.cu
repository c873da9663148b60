// SPDX-License-Identifier: Apache-2.0
//
// Optional depth preprocessing (BASELINE.json north_star, preprocessing stage:
// "erosion/bilateral filtering"), OFF by default.  The reference has no such
// filter (cloud.cpp:19-117 consumes the raw depth + foreground), so it changes
// results versus the reference whenever it is on: SURVEY App. A.7.
//
//   df_erode_rows / df_erode_cols   foreground erosion with a (2r+1)^2 square:
//                                   a pixel stays foreground only if its whole
//                                   window is foreground (and inside the image);
//                                   separable (row min, then column min), one
//                                   thread per pixel, rows read coalesced
//   df_bilateral                    depth' = sum w d / sum w over the window of
//                                   radius ceil(2 sigma_px) restricted to valid
//                                   pixels (mask && depth > 0),
//                                   w = exp(-|dp|^2 / 2 sigma_px^2 - dz^2 / 2 sigma_mm^2),
//                                   fp64, rounded to the nearest mm; invalid
//                                   pixels are left as they are.  The window is
//                                   staged through shared memory per 32x8 tile.
#include <cmath>
#include <cstdint>

#include "vc_device.cuh"

namespace vc {
namespace {

__global__ void df_erode_rows_kernel(const uint8_t* __restrict__ m, uint8_t* __restrict__ out, int w, int h, int r) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= w) return;
  uint8_t keep = 1;
  for (int dx = -r; dx <= r && keep; ++dx) {
    const int xx = x + dx;
    keep = xx >= 0 && xx < w && m[(size_t)y * w + xx] != 0;
  }
  out[(size_t)y * w + x] = keep;
}

__global__ void df_erode_cols_kernel(const uint8_t* __restrict__ m, uint8_t* __restrict__ out, int w, int h, int r) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= w) return;
  uint8_t keep = 1;
  for (int dy = -r; dy <= r && keep; ++dy) {
    const int yy = y + dy;
    keep = yy >= 0 && yy < h && m[(size_t)yy * w + x] != 0;
  }
  out[(size_t)y * w + x] = keep;
}

constexpr int kTX = 32, kTY = 8, kMaxR = 8;

__global__ void __launch_bounds__(kTX* kTY) df_bilateral_kernel(const uint16_t* __restrict__ din,
                                                                 const uint8_t* __restrict__ m,
                                                                 uint16_t* __restrict__ dout, int w, int h, int R,
                                                                 double inv2s2, double inv2r2) {
  __shared__ uint16_t tile[kTY + 2 * kMaxR][kTX + 2 * kMaxR];  // 0 = invalid
  const int x0 = blockIdx.x * kTX - R, y0 = blockIdx.y * kTY - R;
  const int tw = kTX + 2 * R, th = kTY + 2 * R;
  for (int i = threadIdx.y * kTX + threadIdx.x; i < tw * th; i += kTX * kTY) {
    const int ty = i / tw, tx = i % tw, gx = x0 + tx, gy = y0 + ty;
    uint16_t v = 0;
    if (gx >= 0 && gy >= 0 && gx < w && gy < h && m[(size_t)gy * w + gx]) v = din[(size_t)gy * w + gx];
    tile[ty][tx] = v;
  }
  __syncthreads();
  const int x = blockIdx.x * kTX + threadIdx.x, y = blockIdx.y * kTY + threadIdx.y;
  if (x >= w || y >= h) return;
  const uint16_t c = tile[threadIdx.y + R][threadIdx.x + R];
  if (c == 0) {
    dout[(size_t)y * w + x] = din[(size_t)y * w + x];
    return;
  }
  double sw = 0.0, swd = 0.0;
  for (int dy = -R; dy <= R; ++dy)
    for (int dx = -R; dx <= R; ++dx) {
      const uint16_t v = tile[threadIdx.y + R + dy][threadIdx.x + R + dx];
      if (v == 0) continue;
      const double dz = (double)v - (double)c;
      const double wt = exp(-(double)(dx * dx + dy * dy) * inv2s2 - dz * dz * inv2r2);
      sw += wt;
      swd += wt * (double)v;
    }
  dout[(size_t)y * w + x] = (uint16_t)fmin(65535.0, floor(swd / sw + 0.5));
}

}  // namespace

int depth_filter_radius(double sigma_px) { return sigma_px > 0 ? (int)std::ceil(2.0 * sigma_px) : 0; }
int depth_filter_max_radius() { return kMaxR; }

// In place on one view: mask eroded by erode_px (scratch: w*h bytes), then the
// bilateral filter (scratch: w*h*2 bytes for the input copy).
void launch_depth_filter(uint16_t* depth, uint8_t* mask, int w, int h, int erode_px, double sigma_px,
                         double sigma_mm, uint8_t* scratch8, uint16_t* scratch16, cudaStream_t st) {
  const dim3 rb(128), rg((w + 127) / 128, h);
  if (erode_px > 0) {
    df_erode_rows_kernel<<<rg, rb, 0, st>>>(mask, scratch8, w, h, erode_px);
    df_erode_cols_kernel<<<rg, rb, 0, st>>>(scratch8, mask, w, h, erode_px);
  }
  const int R = depth_filter_radius(sigma_px);
  if (R > 0 && sigma_mm > 0) {
    cudaMemcpyAsync(scratch16, depth, (size_t)w * h * 2, cudaMemcpyDeviceToDevice, st);
    const dim3 bb(kTX, kTY), bg((w + kTX - 1) / kTX, (h + kTY - 1) / kTY);
    df_bilateral_kernel<<<bg, bb, 0, st>>>(scratch16, mask, depth, w, h, R, 1.0 / (2.0 * sigma_px * sigma_px),
                                           1.0 / (2.0 * sigma_mm * sigma_mm));
  }
}

}  // namespace vc

// SPDX-License-Identifier: Apache-2.0
//
// Evaluation metrics on sm_100a (eval/metrics.cpp,
// distance_transform.cpp, ssim.cpp), fp64 in the reference's operation order.
// Everything whose result depends on a summation order (cp_rmse's sum of
// squared distances, the SSIM pooling sums) is produced per element here and
// summed on the host in the reference's order.
//
//   mt_vre         xor / or pixel counts (exact integers)
//   mt_dt_cols / mt_dt_rows   Felzenszwalb-Huttenlocher squared distance
//                  transform, one thread per column then per row (dt1d with the
//                  reference's infinity handling, distance_transform.cpp:14-52)
//   mt_hausdorff   max of the other mask's distance map over each mask (exact)
//   mt_nearest     cp_rmse's nearest squared distance per ground point
//                  (brute force over a shared-memory tile; the min is exact)
//   mt_gray / mt_gauss_x / mt_gauss_y / mt_mul / mt_down / mt_down_or / mt_terms
//                  the WMS3IM pipeline up to the per-pixel weighted terms
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>

#include "vc_device.cuh"

namespace vc {
namespace {

__global__ void mt_vre_kernel(const uint8_t* a, const uint8_t* b, int n, unsigned long long* cnt) {
  unsigned long long x = 0, o = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const bool p = a[i] != 0, q = b[i] != 0;
    x += p != q, o += p || q;
  }
  for (int s = 16; s > 0; s >>= 1) x += __shfl_xor_sync(0xffffffffu, x, s), o += __shfl_xor_sync(0xffffffffu, o, s);
  if ((threadIdx.x & 31) == 0) atomicAdd(cnt, x), atomicAdd(cnt + 1, o);
}

// distance_transform.cpp:14-52 on line `f` (stride `fs`), scratch v/z per line
__device__ void dt1d(const double* f, int n, size_t fs, double* d, size_t ds, int* v, double* z) {
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  int k = 0;
  v[0] = 0;
  z[0] = -inf;
  z[1] = inf;
  for (int q = 1; q < n; ++q) {
    const double fq = f[q * fs];
    if (fq == inf) continue;
    while (true) {
      const double fv = f[(size_t)v[k] * fs];
      if (fv == inf) {
        if (k == 0) {
          v[0] = q;
          z[0] = -inf;
          z[1] = inf;
          break;
        }
        --k;
        continue;
      }
      const double s = ddiv(dsub(dadd(fq, (double)(q * q)), dadd(fv, (double)(v[k] * v[k]))),
                            dsub(dmul(2.0, (double)q), dmul(2.0, (double)v[k])));
      if (s <= z[k]) {
        --k;
      } else {
        ++k;
        v[k] = q;
        z[k] = s;
        z[k + 1] = inf;
        break;
      }
    }
  }
  k = 0;
  const bool none = f[(size_t)v[0] * fs] == inf;
  for (int q = 0; q < n; ++q) {
    if (none) {
      d[q * ds] = inf;
      continue;
    }
    while (z[k + 1] < q) ++k;
    d[q * ds] = dadd(dmul((double)(q - v[k]), (double)(q - v[k])), f[(size_t)v[k] * fs]);
  }
}

__global__ void mt_dt_init_kernel(const uint8_t* mask, int n, double* g) {
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) g[i] = mask[i] ? 0.0 : inf;
}
// columns: in place on g via a per-thread copy in tmp (f) and results into g
__global__ void mt_dt_cols_kernel(double* g, double* tmp, int* vbuf, double* zbuf, int w, int h) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < w; x += gridDim.x * blockDim.x) {
    double* f = tmp + (size_t)x * h;
    for (int y = 0; y < h; ++y) f[y] = g[(size_t)y * w + x];
    dt1d(f, h, 1, g + x, (size_t)w, vbuf + (size_t)x * (h + 1), zbuf + (size_t)x * (h + 2));
  }
}
__global__ void mt_dt_rows_kernel(double* g, double* tmp, int* vbuf, double* zbuf, int w, int h, float* out) {
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  for (int y = blockIdx.x * blockDim.x + threadIdx.x; y < h; y += gridDim.x * blockDim.x) {
    double* f = tmp + (size_t)y * w;
    for (int x = 0; x < w; ++x) f[x] = g[(size_t)y * w + x];
    dt1d(f, w, 1, g + (size_t)y * w, 1, vbuf + (size_t)y * (w + 1), zbuf + (size_t)y * (w + 2));
    for (int x = 0; x < w; ++x) {
      const double sq = g[(size_t)y * w + x];
      out[(size_t)y * w + x] = sq == inf ? __int_as_float(0x7f800000) : (float)__dsqrt_rn(sq);
    }
  }
}

__global__ void mt_hausdorff_kernel(const uint8_t* a, const uint8_t* b, const float* dta, const float* dtb, int n,
                                    int* maxbits) {
  float m = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (a[i]) m = fmaxf(m, dtb[i]);
    if (b[i]) m = fmaxf(m, dta[i]);
  }
  for (int s = 16; s > 0; s >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, s));
  if ((threadIdx.x & 31) == 0) atomicMax(maxbits, __float_as_int(m));  // non-negative floats order as ints
}

// cp_rmse: min over recon of (p - q).squaredNorm(), p the recon point (metrics.cpp:62-64)
__global__ void __launch_bounds__(256) mt_nearest_kernel(const double* __restrict__ ground, int ng,
                                                         const double* __restrict__ recon, int nr, double* out) {
  __shared__ double tile[256 * 3];
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  for (int base = blockIdx.x * 256; base < ng; base += gridDim.x * 256) {
    const int i = base + threadIdx.x;
    double q[3] = {0, 0, 0};
    if (i < ng) q[0] = ground[3 * i], q[1] = ground[3 * i + 1], q[2] = ground[3 * i + 2];
    double best = inf;
    for (int t0 = 0; t0 < nr; t0 += 256) {
      __syncthreads();
      for (int j = threadIdx.x; j < 256 * 3 && t0 * 3 + j < nr * 3; j += 256) tile[j] = recon[(size_t)t0 * 3 + j];
      __syncthreads();
      const int m = min(256, nr - t0);
      for (int j = 0; j < m; ++j) {
        const double ex = dsub(tile[3 * j], q[0]), ey = dsub(tile[3 * j + 1], q[1]), ez = dsub(tile[3 * j + 2], q[2]);
        const double d2 = dadd(dadd(dmul(ex, ex), dmul(ey, ey)), dmul(ez, ez));
        best = d2 < best ? d2 : best;
      }
    }
    if (i < ng) out[i] = best;
  }
}

// ---------------------------------------------------------------- WMS3IM
__global__ void mt_gray_kernel(const uint8_t* rgb, int n, double* g) {  // ssim.cpp:9-17
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    g[i] = dadd(dadd(dmul(0.299, (double)rgb[3 * i]), dmul(0.587, (double)rgb[3 * i + 1])),
                dmul(0.114, (double)rgb[3 * i + 2]));
}
// ssim.cpp:35-59: separable Gaussian, renormalised over the in-bounds taps
__global__ void mt_gauss_kernel(const double* in, double* out, int w, int h, const double* k, int r, int axis) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < w * h; i += gridDim.x * blockDim.x) {
    const int x = i % w, y = i / w;
    double acc = 0, norm = 0;
    for (int t = -r; t <= r; ++t) {
      const int xx = axis == 0 ? x + t : x, yy = axis == 0 ? y : y + t;
      if (axis == 0 ? (xx < 0 || xx >= w) : (yy < 0 || yy >= h)) continue;
      acc = dadd(acc, dmul(k[t + r], in[(size_t)yy * w + xx]));
      norm = dadd(norm, k[t + r]);
    }
    out[i] = ddiv(acc, norm);
  }
}
__global__ void mt_mul_kernel(const double* a, const double* b, double* o, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) o[i] = dmul(a[i], b[i]);
}
__global__ void mt_down_kernel(const double* in, int w, int h, double* out, int ow, int oh) {  // ssim.cpp:114-131
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ow * oh; i += gridDim.x * blockDim.x) {
    const int x = i % ow, y = i / ow;
    double acc = 0;
    int n = 0;
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const int sx = 2 * x + dx, sy = 2 * y + dy;
        if (sx < w && sy < h) acc = dadd(acc, in[(size_t)sy * w + sx]), ++n;
      }
    out[i] = ddiv(acc, (double)n);
  }
}
__global__ void mt_down_or_kernel(const uint8_t* in, int w, int h, uint8_t* out, int ow, int oh) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ow * oh; i += gridDim.x * blockDim.x) {
    const int x = i % ow, y = i / ow;
    uint8_t any = 0;
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const int sx = 2 * x + dx, sy = 2 * y + dy;
        if (sx < w && sy < h && in[(size_t)sy * w + sx]) any = 1;
      }
    out[i] = any;
  }
}
// ssim.cpp:71-107: per masked pixel the products weight*l, weight*c, weight*s and weight
__global__ void mt_terms_kernel(const double* mx_, const double* my_, const double* xx_, const double* yy_,
                                const double* xy_, const uint8_t* mask, int w, int h, int r, double c1, double c2,
                                double c3, double* terms) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < w * h; i += gridDim.x * blockDim.x) {
    double* o = terms + 4 * (size_t)i;
    if (!mask[i]) {
      o[0] = o[1] = o[2] = o[3] = 0.0;
      continue;
    }
    const int px = i % w, py = i / w;
    double weight = 0;
    for (int dy = -r; dy <= r; ++dy)
      for (int dx = -r; dx <= r; ++dx) {
        const int qx = px + dx, qy = py + dy;
        if (qx < 0 || qx >= w || qy < 0 || qy >= h) continue;
        weight = dadd(weight, mask[(size_t)qy * w + qx] ? 1.0 : 0.0);
      }
    const double mx = mx_[i], my = my_[i];
    const double vx = fmax(0.0, dsub(xx_[i], dmul(mx, mx)));
    const double vy = fmax(0.0, dsub(yy_[i], dmul(my, my)));
    const double cov = dsub(xy_[i], dmul(mx, my));
    const double sx = __dsqrt_rn(vx), sy = __dsqrt_rn(vy);
    const double l = ddiv(dadd(dmul(dmul(2.0, mx), my), c1), dadd(dadd(dmul(mx, mx), dmul(my, my)), c1));
    const double c = ddiv(dadd(dmul(dmul(2.0, sx), sy), c2), dadd(dadd(vx, vy), c2));
    const double s = ddiv(dadd(cov, c3), dadd(dmul(sx, sy), c3));
    o[0] = dmul(weight, l), o[1] = dmul(weight, c), o[2] = dmul(weight, s), o[3] = weight;
  }
}

}  // namespace

static int mt_grid() { return sm_count() * 4; }

void launch_vre(const uint8_t* a, const uint8_t* b, int n, unsigned long long* cnt, cudaStream_t st) {
  cudaMemsetAsync(cnt, 0, 16, st);
  mt_vre_kernel<<<mt_grid(), 256, 0, st>>>(a, b, n, cnt);
}

size_t dt_scratch_bytes(int w, int h) {
  const size_t n = (size_t)w * h, m = (size_t)(w > h ? w : h);
  return n * 8 * 2 + (size_t)(w + h) * (m + 2) * (8 + 4) + 1024;
}

void launch_distance_transform(const uint8_t* mask, int w, int h, void* scratch, float* out, cudaStream_t st) {
  const size_t n = (size_t)w * h, m = (size_t)(w > h ? w : h);
  double* g = static_cast<double*>(scratch);
  double* tmp = g + n;
  double* zb = tmp + n;
  int* vb = reinterpret_cast<int*>(zb + (size_t)(w + h) * (m + 2));
  mt_dt_init_kernel<<<mt_grid(), 256, 0, st>>>(mask, (int)n, g);
  mt_dt_cols_kernel<<<(w + 127) / 128, 128, 0, st>>>(g, tmp, vb, zb, w, h);
  mt_dt_rows_kernel<<<(h + 127) / 128, 128, 0, st>>>(g, tmp, vb, zb, w, h, out);
}

void launch_hausdorff(const uint8_t* a, const uint8_t* b, const float* dta, const float* dtb, int n, int* maxbits,
                      cudaStream_t st) {
  cudaMemsetAsync(maxbits, 0, 4, st);
  mt_hausdorff_kernel<<<mt_grid(), 256, 0, st>>>(a, b, dta, dtb, n, maxbits);
}

void launch_nearest(const double* ground, int ng, const double* recon, int nr, double* out, cudaStream_t st) {
  mt_nearest_kernel<<<(ng + 255) / 256 < mt_grid() ? (ng + 255) / 256 : mt_grid(), 256, 0, st>>>(ground, ng, recon, nr,
                                                                                            out);
}

void launch_ssim_gray(const uint8_t* rgb, int n, double* g, cudaStream_t st) {
  mt_gray_kernel<<<mt_grid(), 256, 0, st>>>(rgb, n, g);
}
void launch_ssim_gauss(const double* in, double* tmp, double* out, int w, int h, const double* k, int r,
                       cudaStream_t st) {
  mt_gauss_kernel<<<mt_grid(), 256, 0, st>>>(in, tmp, w, h, k, r, 0);
  mt_gauss_kernel<<<mt_grid(), 256, 0, st>>>(tmp, out, w, h, k, r, 1);
}
void launch_ssim_mul(const double* a, const double* b, double* o, int n, cudaStream_t st) {
  mt_mul_kernel<<<mt_grid(), 256, 0, st>>>(a, b, o, n);
}
void launch_ssim_down(const double* in, int w, int h, double* out, int ow, int oh, cudaStream_t st) {
  mt_down_kernel<<<mt_grid(), 256, 0, st>>>(in, w, h, out, ow, oh);
}
void launch_ssim_down_or(const uint8_t* in, int w, int h, uint8_t* out, int ow, int oh, cudaStream_t st) {
  mt_down_or_kernel<<<mt_grid(), 256, 0, st>>>(in, w, h, out, ow, oh);
}
void launch_ssim_terms(const double* mx, const double* my, const double* xx, const double* yy, const double* xy,
                       const uint8_t* mask, int w, int h, int r, double c1, double c2, double c3, double* terms,
                       cudaStream_t st) {
  mt_terms_kernel<<<mt_grid(), 256, 0, st>>>(mx, my, xx, yy, xy, mask, w, h, r, c1, c2, c3, terms);
}

}  // namespace vc

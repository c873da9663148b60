// SPDX-License-Identifier: Apache-2.0
//
// K1/K2 — depth preprocessing on sm_100a: build_cloud + confidence_weights
// (/root/reference/proj/core/src/recon/cloud.cpp:19-117), the foreground
// bounding box and fit_grid (reconstruct.cpp:16-35, 56-68).
//
// One CTA per depth row (rows of all views concatenated), so the CTA order is
// the reference's point order (views in sensor order, pixels row-major):
//   pre_count  -> points per row
//   pre_scan   -> exclusive scan over rows (single CTA), P
//   pre_emit   -> recompute, compact in order, write SoA points + weight map
//                 row + per-row bbox
//   pre_fit    -> reduce bbox, fit_grid, empty-scene status
// fp64 with the reference's operation order and no FMA (vc_device.cuh), so
// positions — hence every downstream binning decision — are bit-exact.
#include <cfloat>

#include "vc_device.cuh"

namespace vc {
namespace {

constexpr int kThreads = 256;

struct RowCtx {
  const DevSensor* s;
  const ViewPtrs* v;
  int w, h, y;
};

__device__ __forceinline__ bool valid_px(const RowCtx& c, int x, int y) {
  if (x < 0 || y < 0 || x >= c.w || y >= c.h) return false;
  return __ldg(c.v->mask + (size_t)y * c.v->mpitch + x) != 0 && __ldg(c.v->depth + (size_t)y * c.v->dpitch + x) != 0;
}

// camera.cpp:12-17 backproject_local with u = (x, y) and z = depth
__device__ __forceinline__ d3 local_px(const RowCtx& c, int x, int y) {
  const double z = (double)__ldg(c.v->depth + (size_t)y * c.v->dpitch + x);
  const DevSensor& s = *c.s;
  return {ddiv(dmul(dsub((double)x, s.cx), z), s.fx), ddiv(dmul(dsub((double)y, s.cy), z), s.fy), z};
}

// cloud.cpp:38-51 add_triangle(ia, ib, ic), accumulated into (sum, count)
__device__ __forceinline__ void add_tri(const RowCtx& c, int ax, int ay, int bx, int by, int cx, int cy,
                                        double disc, d3& sum, int& cnt) {
  if (!valid_px(c, ax, ay) || !valid_px(c, bx, by) || !valid_px(c, cx, cy)) return;
  const d3 a = local_px(c, ax, ay), b = local_px(c, bx, by), cc = local_px(c, cx, cy);
  const double lo = fmin(fmin(a.z, b.z), cc.z), hi = fmax(fmax(a.z, b.z), cc.z);
  if (dsub(hi, lo) > disc) return;
  d3 n = cross3(sub3(cc, a), sub3(b, a));
  const double len = norm3(n);
  if (len < 1e-12) return;
  n = div3(n, len);
  sum = add3(sum, n);
  ++cnt;
}

// cloud.cpp:53-71 for pixel (x, y): the six incident triangles in the
// reference's accumulation order, then mean, normalise, camera-facing flip.
__device__ bool point_at(const RowCtx& c, int x, int y, double disc, d3* local_out, d3* n_out) {
  if (!valid_px(c, x, y)) return false;
  d3 sum{0.0, 0.0, 0.0};
  int cnt = 0;
  const int w = c.w, h = c.h;
  if (x >= 1 && y >= 1) add_tri(c, x, y - 1, x, y, x - 1, y, disc, sum, cnt);                // Q(x-1,y-1).T2
  if (x <= w - 2 && y >= 1) {
    add_tri(c, x, y - 1, x + 1, y - 1, x, y, disc, sum, cnt);                                 // Q(x,y-1).T1
    add_tri(c, x + 1, y - 1, x + 1, y, x, y, disc, sum, cnt);                                 // Q(x,y-1).T2
  }
  if (x >= 1 && y <= h - 2) {
    add_tri(c, x - 1, y, x, y, x - 1, y + 1, disc, sum, cnt);                                 // Q(x-1,y).T1
    add_tri(c, x, y, x, y + 1, x - 1, y + 1, disc, sum, cnt);                                 // Q(x-1,y).T2
  }
  if (x <= w - 2 && y <= h - 2) add_tri(c, x, y, x + 1, y, x, y + 1, disc, sum, cnt);         // Q(x,y).T1
  if (cnt == 0) return false;
  d3 n = div3(sum, (double)cnt);
  const double len = norm3(n);
  if (len < 1e-12) return false;
  n = div3(n, len);
  const d3 local = local_px(c, x, y);
  if (dot3(n, local) > 0) n = neg3(n);
  *local_out = local;
  *n_out = n;
  return true;
}

__device__ __forceinline__ void row_of_block(const SensorSet& ss, int b, int* k, int* y) {
  int kk = 0;
  while (kk + 1 < ss.k && b >= ss.row_offset[kk + 1]) ++kk;
  *k = kk;
  *y = b - ss.row_offset[kk];
}

__global__ void __launch_bounds__(kThreads) pre_count_kernel(const __grid_constant__ SensorSet ss, double disc,
                                                             int32_t* row_counts) {
  int k, y;
  row_of_block(ss, blockIdx.x, &k, &y);
  RowCtx c{&ss.s[k], &ss.v[k], ss.s[k].w, ss.s[k].h, y};
  int n = 0;
  for (int x = threadIdx.x; x < c.w; x += kThreads) {
    d3 l, nn;
    n += point_at(c, x, y, disc, &l, &nn) ? 1 : 0;
  }
  __shared__ int red[kThreads / 32];
  n = __reduce_add_sync(0xffffffffu, n);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < kThreads / 32; ++i) t += red[i];
    row_counts[blockIdx.x] = t;
  }
}

// single-CTA exclusive scan of the per-row counts
__global__ void __launch_bounds__(1024) pre_scan_kernel(const int32_t* counts, int32_t* offsets, int rows,
                                                        int cap, DevCtl* ctl) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < rows; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < rows ? counts[i] : 0;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if ((threadIdx.x & 31) >= o) incl += t;
    }
    if ((threadIdx.x & 31) == 31) warp_sums[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
      int ws = warp_sums[threadIdx.x];
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, ws, o);
        if (threadIdx.x >= o) ws += t;
      }
      warp_sums[threadIdx.x] = ws;
    }
    __syncthreads();
    const int wpre = (threadIdx.x >> 5) ? warp_sums[(threadIdx.x >> 5) - 1] : 0;
    if (i < rows) offsets[i] = carry + wpre + incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += wpre + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ctl->P = carry;
    ctl->status = carry == 0 ? 2 : 0;
    if (carry > cap) ctl->status = 3;
  }
}

__global__ void __launch_bounds__(kThreads) pre_emit_kernel(const __grid_constant__ SensorSet ss, double disc,
                                                            int sil_r, const int32_t* row_offsets, DevPoints pts,
                                                            float* weight_maps, double* row_bbox) {
  extern __shared__ uint32_t colsum[];  // w entries
  __shared__ int warp_cnt[kThreads / 32];
  __shared__ double bb[kThreads / 32][6];
  int k, y;
  row_of_block(ss, blockIdx.x, &k, &y);
  const DevSensor& s = ss.s[k];
  const ViewPtrs& v = ss.v[k];
  RowCtx c{&s, &v, s.w, s.h, y};
  const int w = s.w, h = s.h;

  // cloud.cpp:89-106: foreground count of the (2r+1)^2 window, clipped to the
  // image (off-image area counts as background), as column sums + row window.
  const int y0 = max(0, y - sil_r), y1 = min(h - 1, y + sil_r);
  for (int x = threadIdx.x; x < w; x += kThreads) {
    uint32_t cs = 0;
    for (int yy = y0; yy <= y1; ++yy) cs += __ldg(v.mask + (size_t)yy * v.mpitch + x) ? 1u : 0u;
    colsum[x] = cs;
  }
  __syncthreads();
  const double window = (double)(2 * sil_r + 1) * (double)(2 * sil_r + 1);

  const double inf = DBL_MAX * 2.0;
  double lo[3] = {inf, inf, inf}, hi[3] = {-inf, -inf, -inf};
  int base = row_offsets[blockIdx.x];
  float* wrow = weight_maps + ss.pix_offset[k] + (size_t)y * w;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  for (int x0 = 0; x0 < w; x0 += kThreads) {
    const int x = x0 + threadIdx.x;
    d3 local{0, 0, 0}, n{0, 0, 0};
    const bool is_pt = x < w && point_at(c, x, y, disc, &local, &n);
    const unsigned ball = __ballot_sync(0xffffffffu, is_pt);
    if (lane == 0) warp_cnt[wid] = __popc(ball);
    __syncthreads();
    int wpre = 0, tot = 0;
    for (int i = 0; i < kThreads / 32; ++i) {
      wpre += i < wid ? warp_cnt[i] : 0;
      tot += warp_cnt[i];
    }
    float wmap = 0.f;
    if (is_pt) {
      const int idx = base + wpre + __popc(ball & ((1u << lane) - 1u));
      // cloud.cpp:73-74: world position / normal
      const d3 p = add3(mat3(s.R, local), ld3(s.t));
      const d3 nw = mat3(s.R, n);
      // cloud.cpp:108-114: W1 from the re-transformed local frame, W2 coverage
      const d3 l2 = add3(mat3(s.Ri, p), ld3(s.ti));
      const d3 nl = mat3(s.Ri, nw);
      const double w1raw = dot3(neg3(normalized3(l2)), nl);
      const double w1 = w1raw < 0.0 ? 0.0 : w1raw;
      const int xa = max(0, x - sil_r), xb = min(w - 1, x + sil_r);
      uint32_t cnt = 0;
      for (int xx = xa; xx <= xb; ++xx) cnt += colsum[xx];
      const double w2 = ddiv((double)cnt, window);
      const double wt = dmul(w1, w2);
      pts.pos[3 * idx + 0] = p.x;
      pts.pos[3 * idx + 1] = p.y;
      pts.pos[3 * idx + 2] = p.z;
      pts.nrm[3 * idx + 0] = nw.x;
      pts.nrm[3 * idx + 1] = nw.y;
      pts.nrm[3 * idx + 2] = nw.z;
      pts.weight[idx] = wt;
      pts.pix[3 * idx + 0] = x;
      pts.pix[3 * idx + 1] = y;
      pts.pix[3 * idx + 2] = k;
      wmap = (float)wt;
      lo[0] = fmin(lo[0], p.x), lo[1] = fmin(lo[1], p.y), lo[2] = fmin(lo[2], p.z);
      hi[0] = fmax(hi[0], p.x), hi[1] = fmax(hi[1], p.y), hi[2] = fmax(hi[2], p.z);
    }
    if (x < w) wrow[x] = wmap;
    base += tot;
    __syncthreads();
  }
  // per-row bbox (exact min/max, order-independent)
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  if (lane == 0)
    for (int a = 0; a < 3; ++a) bb[wid][a] = lo[a], bb[wid][3 + a] = hi[a];
  __syncthreads();
  if (threadIdx.x < 6) {
    double r = bb[0][threadIdx.x];
    for (int i = 1; i < kThreads / 32; ++i)
      r = threadIdx.x < 3 ? fmin(r, bb[i][threadIdx.x]) : fmax(r, bb[i][threadIdx.x]);
    row_bbox[(size_t)blockIdx.x * 6 + threadIdx.x] = r;
  }
}

// reconstruct.cpp:56-68 (bbox) + fit_grid (reconstruct.cpp:16-35, dims given)
__global__ void __launch_bounds__(256) pre_fit_kernel(const double* row_bbox, int rows, int nx, int ny, int nz,
                                                      int pad, DevCtl* ctl) {
  __shared__ double sh[256][6];
  const double inf = DBL_MAX * 2.0;
  double r[6] = {inf, inf, inf, -inf, -inf, -inf};
  for (int i = threadIdx.x; i < rows; i += 256)
    for (int a = 0; a < 6; ++a)
      r[a] = a < 3 ? fmin(r[a], row_bbox[(size_t)i * 6 + a]) : fmax(r[a], row_bbox[(size_t)i * 6 + a]);
  for (int a = 0; a < 6; ++a) sh[threadIdx.x][a] = r[a];
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int i = 1; i < 256; ++i)
    for (int a = 0; a < 6; ++a) r[a] = a < 3 ? fmin(r[a], sh[i][a]) : fmax(r[a], sh[i][a]);
  for (int a = 0; a < 6; ++a) ctl->bbox[a] = r[a];
  DevGrid g;
  g.nx = nx, g.ny = ny, g.nz = nz;
  if (ctl->status != 0) {
    g.origin[0] = g.origin[1] = g.origin[2] = 0.0;
    g.edge = 1.0;
    ctl->grid = g;
    return;
  }
  const int dims[3] = {nx, ny, nz};
  double edge = 1e-9;
  for (int a = 0; a < 3; ++a) {
    const int usable = dims[a] - 1 - 2 * pad;
    const double e = ddiv(dsub(r[3 + a], r[a]), (double)usable);
    edge = edge < e ? e : edge;
  }
  g.edge = edge;
  for (int a = 0; a < 3; ++a) {
    const double center = dmul(0.5, dadd(r[a], r[3 + a]));
    g.origin[a] = dsub(center, ddiv(dmul(edge, (double)(dims[a] - 1)), 2.0));
  }
  ctl->grid = g;
}

}  // namespace

size_t preprocess_scratch_bytes(const SensorSet& ss) {
  const size_t rows = (size_t)ss.row_offset[ss.k];
  return rows * (2 * sizeof(int32_t)) + rows * 6 * sizeof(double) + 64;
}

void launch_preprocess(const SensorSet& ss, DevPoints pts, float* weight_maps, int32_t* scratch, DevCtl* ctl,
                       int nx, int ny, int nz, int padding, double disc_mm, int sil_r, cudaStream_t st) {
  const int rows = ss.row_offset[ss.k];
  int32_t* counts = scratch;
  int32_t* offsets = scratch + rows;
  double* bbox = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(offsets + rows) + 63) & ~uintptr_t(63));
  int maxw = 0;
  for (int k = 0; k < ss.k; ++k) maxw = maxw > ss.s[k].w ? maxw : ss.s[k].w;
  pre_count_kernel<<<rows, kThreads, 0, st>>>(ss, disc_mm, counts);
  pre_scan_kernel<<<1, 1024, 0, st>>>(counts, offsets, rows, pts.cap, ctl);
  pre_emit_kernel<<<rows, kThreads, maxw * sizeof(uint32_t), st>>>(ss, disc_mm, sil_r, offsets, pts, weight_maps,
                                                                   bbox);
  pre_fit_kernel<<<1, 256, 0, st>>>(bbox, rows, nx, ny, nz, padding, ctl);
}

}  // namespace vc

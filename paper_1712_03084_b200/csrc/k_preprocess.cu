// SPDX-License-Identifier: Apache-2.0
//
// K1/K2 — depth preprocessing on sm_100a: build_cloud + confidence_weights
// (/root/reference/proj/core/src/recon/cloud.cpp:19-117), the foreground
// bounding box and fit_grid (reconstruct.cpp:16-35, 56-68).
//
//   pre_prefix  one warp per depth row: inclusive prefix count of the mask
//               along x (the 21x21 silhouette box count of cloud.cpp:89-106
//               becomes 2 loads per window row)
//   pre_points  one CTA per depth row (rows of all views concatenated, so CTA
//               order = the reference's point order): the rows y-1..y+1 are
//               staged in shared memory, each pixel evaluates its six incident
//               triangles in the reference's accumulation order
//               (cloud.cpp:53-71), W = W1*W2 (cloud.cpp:108-114); points are
//               compacted in row order into a per-row staging slot, the
//               weight-map row and the row bbox are written
//   pre_scan    exclusive scan of the per-row counts (single CTA) -> P
//   pre_gather  one warp per row: staged points -> final SoA at the row offset
//   pre_fit     bbox reduction + fit_grid + empty-scene status
// fp64 with the reference's operation order and no FMA (vc_device.cuh), so
// positions — hence every downstream binning decision — are bit-exact.
#include <cfloat>

#include "vc_device.cuh"

namespace vc {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void row_of_block(const SensorSet& ss, int b, int* k, int* y) {
  int kk = 0;
  while (kk + 1 < ss.k && b >= ss.row_offset[kk + 1]) ++kk;
  *k = kk;
  *y = b - ss.row_offset[kk];
}

// inclusive prefix of (mask != 0) along each row: pref[row][x]
__global__ void __launch_bounds__(256) pre_prefix_kernel(const __grid_constant__ SensorSet ss, int rows,
                                                         uint16_t* __restrict__ pref, int pitch) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= rows) return;
  int k, y;
  row_of_block(ss, r, &k, &y);
  const ViewPtrs& v = ss.v[k];
  const int w = ss.s[k].w;
  const uint8_t* m = v.mask + (size_t)y * v.mpitch;
  uint16_t* o = pref + (size_t)r * pitch;
  int carry = 0;
  for (int x0 = 0; x0 < w; x0 += 32) {
    const int x = x0 + lane;
    int c = (x < w && m[x]) ? 1 : 0;
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, c, d);
      if (lane >= d) c += t;
    }
    if (x < w) o[x] = (uint16_t)(carry + c);
    carry += __shfl_sync(0xffffffffu, c, 31);
  }
}

__device__ __forceinline__ bool valid_px(const ViewPtrs& v, int w, int h, int x, int y) {
  if (x < 0 || y < 0 || x >= w || y >= h) return false;
  return __ldg(v.mask + (size_t)y * v.mpitch + x) != 0 && __ldg(v.depth + (size_t)y * v.dpitch + x) != 0;
}
// camera.cpp:12-17 backproject_local with u = (x, y), z = depth
__device__ __forceinline__ d3 local_px(const DevSensor& s, const ViewPtrs& v, int x, int y) {
  const double z = (double)__ldg(v.depth + (size_t)y * v.dpitch + x);
  return {ddiv(dmul(dsub((double)x, s.cx), z), s.fx), ddiv(dmul(dsub((double)y, s.cy), z), s.fy), z};
}

// cloud.cpp:38-51 add_triangle(ia, ib, ic): the normalised normal, or NaN
// when the triangle is rejected (invalid vertex, depth step > disc, len < 1e-12)
__device__ d3 triangle_normal(bool ok, d3 a, d3 b, d3 c, double disc) {
  const d3 bad{__longlong_as_double(0x7ff8000000000000ll), 0.0, 0.0};
  if (!ok) return bad;
  const double lo = fmin(fmin(a.z, b.z), c.z), hi = fmax(fmax(a.z, b.z), c.z);
  if (dsub(hi, lo) > disc) return bad;
  const d3 n = cross3(sub3(c, a), sub3(b, a));
  const double len = norm3(n);
  if (len < 1e-12) return bad;
  return div3(n, len);
}

// One thread per quad (qx, qy) with a valid corner: T1 = (i00, i10, i01) and
// T2 = (i10, i11, i01) (cloud.cpp:53-59), each normal computed once.
__global__ void __launch_bounds__(256) pre_tri_kernel(const __grid_constant__ SensorSet ss, double disc,
                                                      double* __restrict__ tri) {
  const int64_t npix = ss.pix_offset[ss.k];
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < npix; q += (int64_t)gridDim.x * blockDim.x) {
    int k = 0;
    while (k + 1 < ss.k && q >= ss.pix_offset[k + 1]) ++k;
    const DevSensor& s = ss.s[k];
    const ViewPtrs& v = ss.v[k];
    const int64_t r = q - ss.pix_offset[k];
    const int qy = (int)(r / s.w), qx = (int)(r - (int64_t)qy * s.w);
    if (qx + 1 >= s.w || qy + 1 >= s.h) continue;
    const bool v00 = valid_px(v, s.w, s.h, qx, qy), v10 = valid_px(v, s.w, s.h, qx + 1, qy);
    const bool v01 = valid_px(v, s.w, s.h, qx, qy + 1), v11 = valid_px(v, s.w, s.h, qx + 1, qy + 1);
    if (!(v00 || v10 || v01 || v11)) continue;
    const d3 z{0, 0, 0};
    const d3 p00 = v00 ? local_px(s, v, qx, qy) : z, p10 = v10 ? local_px(s, v, qx + 1, qy) : z;
    const d3 p01 = v01 ? local_px(s, v, qx, qy + 1) : z, p11 = v11 ? local_px(s, v, qx + 1, qy + 1) : z;
    const d3 t1 = triangle_normal(v00 && v10 && v01, p00, p10, p01, disc);
    const d3 t2 = triangle_normal(v10 && v11 && v01, p10, p11, p01, disc);
    double* o = tri + 6 * q;
    o[0] = t1.x, o[1] = t1.y, o[2] = t1.z, o[3] = t2.x, o[4] = t2.y, o[5] = t2.z;
  }
}

__device__ __forceinline__ void add_tri(const double* tri, int64_t q, int t, d3& sum, int& cnt) {
  const double* n = tri + 6 * q + 3 * t;
  const double nx = n[0];
  if (nx != nx) return;  // rejected triangle
  sum = add3(sum, mk3(nx, n[1], n[2]));
  ++cnt;
}

// cloud.cpp:53-71: the six incident triangles of pixel (x, y) in the
// reference's order Q(x-1,y-1).T2, Q(x,y-1).T1, Q(x,y-1).T2, Q(x-1,y).T1,
// Q(x-1,y).T2, Q(x,y).T1; mean, normalise, camera-facing flip.
__device__ bool point_at(const SensorSet& ss, int k, const double* tri, int x, int y, d3* local_out, d3* n_out) {
  const DevSensor& s = ss.s[k];
  const ViewPtrs& v = ss.v[k];
  const int w = s.w, h = s.h;
  if (!valid_px(v, w, h, x, y)) return false;
  const int64_t q = ss.pix_offset[k] + (int64_t)y * w + x;  // quad (x, y)
  d3 sum{0.0, 0.0, 0.0};
  int cnt = 0;
  if (x >= 1 && y >= 1) add_tri(tri, q - w - 1, 1, sum, cnt);
  if (x <= w - 2 && y >= 1) {
    add_tri(tri, q - w, 0, sum, cnt);
    add_tri(tri, q - w, 1, sum, cnt);
  }
  if (x >= 1 && y <= h - 2) {
    add_tri(tri, q - 1, 0, sum, cnt);
    add_tri(tri, q - 1, 1, sum, cnt);
  }
  if (x <= w - 2 && y <= h - 2) add_tri(tri, q, 0, sum, cnt);
  if (cnt == 0) return false;
  d3 n = div3(sum, (double)cnt);
  const double len = norm3(n);
  if (len < 1e-12) return false;
  n = div3(n, len);
  const d3 local = local_px(s, v, x, y);
  if (dot3(n, local) > 0) n = neg3(n);
  *local_out = local;
  *n_out = n;
  return true;
}

struct Staged {  // per-point staging record (row-local order)
  double pos[3], nrm[3], w;
  int32_t px;
};

__global__ void __launch_bounds__(kThreads) pre_points_kernel(const __grid_constant__ SensorSet ss, int sil_r,
                                                              const double* __restrict__ tri,
                                                              const uint16_t* __restrict__ pref, int ppitch,
                                                              Staged* __restrict__ stage, int spitch,
                                                              int32_t* __restrict__ row_counts,
                                                              float* __restrict__ weight_maps,
                                                              double* __restrict__ row_bbox) {
  __shared__ int warp_cnt[kThreads / 32];
  __shared__ double bb[kThreads / 32][6];
  int k, y;
  row_of_block(ss, blockIdx.x, &k, &y);
  const DevSensor& s = ss.s[k];
  const int w = s.w, h = s.h;
  const double window = (double)(2 * sil_r + 1) * (double)(2 * sil_r + 1);
  const int wy0 = max(0, y - sil_r), wy1 = min(h - 1, y + sil_r);
  const uint16_t* prow0 = pref + (size_t)(blockIdx.x - y) * ppitch;  // row 0 of this view
  const double inf = DBL_MAX * 2.0;
  double lo0 = inf, lo1 = inf, lo2 = inf, hi0 = -inf, hi1 = -inf, hi2 = -inf;
  int base = 0;
  Staged* srow = stage + (size_t)blockIdx.x * spitch;
  float* wrow = weight_maps + ss.pix_offset[k] + (size_t)y * w;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int x0 = 0; x0 < w; x0 += kThreads) {
    const int x = x0 + threadIdx.x;
    d3 local{0, 0, 0}, n{0, 0, 0};
    const bool is_pt = x < w && point_at(ss, k, tri, x, y, &local, &n);
    const unsigned ball = __ballot_sync(0xffffffffu, is_pt);
    if (lane == 0) warp_cnt[wid] = __popc(ball);
    __syncthreads();
    int wpre = 0, tot = 0;
    for (int i = 0; i < kThreads / 32; ++i) wpre += i < wid ? warp_cnt[i] : 0, tot += warp_cnt[i];
    float wmap = 0.f;
    if (is_pt) {
      // cloud.cpp:73-74 world position / normal
      const d3 p = add3(mat3(s.R, local), ld3(s.t));
      const d3 nw = mat3(s.R, n);
      // cloud.cpp:108-114: W1 from the re-transformed local frame, W2 coverage
      const d3 l2 = add3(mat3(s.Ri, p), ld3(s.ti));
      const d3 nl = mat3(s.Ri, nw);
      const double w1raw = dot3(neg3(normalized3(l2)), nl);
      const double w1 = w1raw < 0.0 ? 0.0 : w1raw;
      const int xa = max(0, x - sil_r), xb = min(w - 1, x + sil_r);
      uint32_t cnt = 0;
      for (int yy = wy0; yy <= wy1; ++yy) {
        const uint16_t* pr = prow0 + (size_t)yy * ppitch;
        cnt += (uint32_t)pr[xb] - (xa > 0 ? (uint32_t)pr[xa - 1] : 0u);
      }
      const double wt = dmul(w1, ddiv((double)cnt, window));
      Staged& o = srow[base + wpre + __popc(ball & ((1u << lane) - 1u))];
      o.pos[0] = p.x, o.pos[1] = p.y, o.pos[2] = p.z;
      o.nrm[0] = nw.x, o.nrm[1] = nw.y, o.nrm[2] = nw.z;
      o.w = wt;
      o.px = x;
      wmap = (float)wt;
      lo0 = fmin(lo0, p.x), lo1 = fmin(lo1, p.y), lo2 = fmin(lo2, p.z);
      hi0 = fmax(hi0, p.x), hi1 = fmax(hi1, p.y), hi2 = fmax(hi2, p.z);
    }
    if (x < w) wrow[x] = wmap;
    base += tot;
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo0 = fmin(lo0, __shfl_xor_sync(0xffffffffu, lo0, o)), hi0 = fmax(hi0, __shfl_xor_sync(0xffffffffu, hi0, o));
    lo1 = fmin(lo1, __shfl_xor_sync(0xffffffffu, lo1, o)), hi1 = fmax(hi1, __shfl_xor_sync(0xffffffffu, hi1, o));
    lo2 = fmin(lo2, __shfl_xor_sync(0xffffffffu, lo2, o)), hi2 = fmax(hi2, __shfl_xor_sync(0xffffffffu, hi2, o));
  }
  if (lane == 0) {
    bb[wid][0] = lo0, bb[wid][1] = lo1, bb[wid][2] = lo2;
    bb[wid][3] = hi0, bb[wid][4] = hi1, bb[wid][5] = hi2;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double r = bb[0][threadIdx.x];
    for (int i = 1; i < kThreads / 32; ++i)
      r = threadIdx.x < 3 ? fmin(r, bb[i][threadIdx.x]) : fmax(r, bb[i][threadIdx.x]);
    row_bbox[(size_t)blockIdx.x * 6 + threadIdx.x] = r;
  }
  if (threadIdx.x == 0) row_counts[blockIdx.x] = base;
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

// one warp per row: staged points -> final SoA (pos, nrm, weight, pix)
__global__ void __launch_bounds__(256) pre_gather_kernel(const __grid_constant__ SensorSet ss, int rows,
                                                         const Staged* __restrict__ stage, int spitch,
                                                         const int32_t* __restrict__ counts,
                                                         const int32_t* __restrict__ offsets, DevPoints pts) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int n = counts[r];
  if (!n) return;
  int k, y;
  row_of_block(ss, r, &k, &y);
  const int off = offsets[r];
  const Staged* srow = stage + (size_t)r * spitch;
  for (int i = lane; i < n; i += 32) {
    const Staged s = srow[i];
    const int idx = off + i;
    pts.pos[3 * idx + 0] = s.pos[0], pts.pos[3 * idx + 1] = s.pos[1], pts.pos[3 * idx + 2] = s.pos[2];
    pts.nrm[3 * idx + 0] = s.nrm[0], pts.nrm[3 * idx + 1] = s.nrm[1], pts.nrm[3 * idx + 2] = s.nrm[2];
    pts.weight[idx] = s.w;
    pts.pix[3 * idx + 0] = s.px, pts.pix[3 * idx + 1] = y, pts.pix[3 * idx + 2] = k;
  }
}

// reconstruct.cpp:56-68 (bbox) + fit_grid (reconstruct.cpp:16-35, dims given)
__global__ void __launch_bounds__(256) pre_fit_kernel(const double* row_bbox, int rows, int nx, int ny, int nz,
                                                      int pad, DevCtl* ctl) {
  __shared__ double sh[6][256];
  const double inf = DBL_MAX * 2.0;
  double r[6] = {inf, inf, inf, -inf, -inf, -inf};
  for (int i = threadIdx.x; i < rows; i += 256) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      r[a] = fmin(r[a], row_bbox[(size_t)i * 6 + a]);
      r[3 + a] = fmax(r[3 + a], row_bbox[(size_t)i * 6 + 3 + a]);
    }
  }
#pragma unroll
  for (int a = 0; a < 6; ++a) sh[a][threadIdx.x] = r[a];
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        sh[a][threadIdx.x] = fmin(sh[a][threadIdx.x], sh[a][threadIdx.x + o]);
        sh[3 + a][threadIdx.x] = fmax(sh[3 + a][threadIdx.x], sh[3 + a][threadIdx.x + o]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  for (int a = 0; a < 6; ++a) r[a] = sh[a][0], ctl->bbox[a] = r[a];
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

struct Scratch {
  double* tri;  // 6 doubles per quad (indexed by its i00 pixel)
  int32_t* counts;
  int32_t* offsets;
  double* bbox;
  uint16_t* pref;
  Staged* stage;
  int ppitch, spitch;
};

Scratch carve(const SensorSet& ss, void* base) {
  const int rows = ss.row_offset[ss.k];
  int maxw = 0;
  for (int k = 0; k < ss.k; ++k) maxw = maxw > ss.s[k].w ? maxw : ss.s[k].w;
  auto up = [](uintptr_t p) { return (p + 255) & ~uintptr_t(255); };
  Scratch s;
  uintptr_t p = up(reinterpret_cast<uintptr_t>(base));
  s.tri = reinterpret_cast<double*>(p);
  p = up(p + (size_t)ss.pix_offset[ss.k] * 6 * sizeof(double));
  s.counts = reinterpret_cast<int32_t*>(p);
  p = up(p + rows * sizeof(int32_t));
  s.offsets = reinterpret_cast<int32_t*>(p);
  p = up(p + rows * sizeof(int32_t));
  s.bbox = reinterpret_cast<double*>(p);
  p = up(p + rows * 6 * sizeof(double));
  s.ppitch = (maxw + 127) & ~127;
  s.pref = reinterpret_cast<uint16_t*>(p);
  p = up(p + (size_t)rows * s.ppitch * sizeof(uint16_t));
  s.spitch = maxw;
  s.stage = reinterpret_cast<Staged*>(p);
  p = up(p + (size_t)rows * s.spitch * sizeof(Staged));
  return s;
}

}  // namespace

void prepare_preprocess(const SensorSet&) {}  // no opt-in shared memory needed

size_t preprocess_scratch_bytes(const SensorSet& ss) {
  const Scratch s = carve(ss, nullptr);
  const int rows = ss.row_offset[ss.k];
  return reinterpret_cast<uintptr_t>(s.stage) + (size_t)rows * s.spitch * sizeof(Staged) + 512;
}

void launch_preprocess(const SensorSet& ss, DevPoints pts, float* weight_maps, int32_t* scratch, DevCtl* ctl,
                       int nx, int ny, int nz, int padding, double disc_mm, int sil_r, cudaStream_t st) {
  const int rows = ss.row_offset[ss.k];
  const Scratch s = carve(ss, scratch);
  int maxw = 0;
  for (int k = 0; k < ss.k; ++k) maxw = maxw > ss.s[k].w ? maxw : ss.s[k].w;
  const int warp_grid = (rows * 32 + 255) / 256;
  pre_prefix_kernel<<<warp_grid, 256, 0, st>>>(ss, rows, s.pref, s.ppitch);
  pre_tri_kernel<<<148 * 8, 256, 0, st>>>(ss, disc_mm, s.tri);
  pre_points_kernel<<<rows, kThreads, 0, st>>>(ss, sil_r, s.tri, s.pref, s.ppitch, s.stage, s.spitch, s.counts,
                                               weight_maps, s.bbox);
  pre_scan_kernel<<<1, 1024, 0, st>>>(s.counts, s.offsets, rows, pts.cap, ctl);
  pre_gather_kernel<<<warp_grid, 256, 0, st>>>(ss, rows, s.stage, s.spitch, s.counts, s.offsets, pts);
  pre_fit_kernel<<<1, 256, 0, st>>>(s.bbox, rows, nx, ny, nz, padding, ctl);
}

}  // namespace vc

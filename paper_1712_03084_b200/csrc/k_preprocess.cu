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

// Rows y-1..y+1 staged in shared memory: validity, fp64 local positions
// (backprojected once per pixel) and the T1/T2 triangle normals of the quads
// touching row y (computed once per triangle instead of once per vertex).
struct RowCache {
  int w, h, y;
  const uint16_t* dep;  // [3][w]
  double* pos;          // [3][w][3]
  double* tri;          // [2 quad rows][w][2 tris][4]: nx, ny, nz, valid (0/1)
  __device__ bool valid(int x, int yy) const {
    if (x < 0 || x >= w || yy < y - 1 || yy > y + 1) return false;
    return dep[(yy - y + 1) * w + x] != 0;
  }
  __device__ d3 local(int x, int yy) const {
    const double* p = pos + ((size_t)(yy - y + 1) * w + x) * 3;
    return {p[0], p[1], p[2]};
  }
  // quad row qr = qy - (y - 1) in {0, 1}; triangle t in {0: T1, 1: T2}
  __device__ const double* tri_at(int qr, int qx, int t) const { return tri + (((size_t)qr * w + qx) * 2 + t) * 4; }
};

// cloud.cpp:38-51 add_triangle(ia, ib, ic) -> normalised normal or invalid
__device__ void triangle_normal(const RowCache& c, int ax, int ay, int bx, int by, int cx, int cy, double disc,
                                double* out) {
  out[3] = 0.0;
  if (!c.valid(ax, ay) || !c.valid(bx, by) || !c.valid(cx, cy)) return;
  const d3 a = c.local(ax, ay), b = c.local(bx, by), cc = c.local(cx, cy);
  const double lo = fmin(fmin(a.z, b.z), cc.z), hi = fmax(fmax(a.z, b.z), cc.z);
  if (dsub(hi, lo) > disc) return;
  d3 n = cross3(sub3(cc, a), sub3(b, a));
  const double len = norm3(n);
  if (len < 1e-12) return;
  n = div3(n, len);
  out[0] = n.x, out[1] = n.y, out[2] = n.z, out[3] = 1.0;
}

__device__ __forceinline__ void add_cached(const RowCache& c, int qr, int qx, int t, d3& sum, int& cnt) {
  const double* tn = c.tri_at(qr, qx, t);
  if (tn[3] == 0.0) return;
  sum = add3(sum, mk3(tn[0], tn[1], tn[2]));
  ++cnt;
}

// cloud.cpp:53-71: the six incident triangles of pixel (x, y) in the
// reference's order Q(x-1,y-1).T2, Q(x,y-1).T1, Q(x,y-1).T2, Q(x-1,y).T1,
// Q(x-1,y).T2, Q(x,y).T1; mean, normalise, camera-facing flip.
__device__ bool point_at(const RowCache& c, int x, d3* local_out, d3* n_out) {
  const int y = c.y, w = c.w, h = c.h;
  if (!c.valid(x, y)) return false;
  d3 sum{0.0, 0.0, 0.0};
  int cnt = 0;
  if (x >= 1 && y >= 1) add_cached(c, 0, x - 1, 1, sum, cnt);
  if (x <= w - 2 && y >= 1) {
    add_cached(c, 0, x, 0, sum, cnt);
    add_cached(c, 0, x, 1, sum, cnt);
  }
  if (x >= 1 && y <= h - 2) {
    add_cached(c, 1, x - 1, 0, sum, cnt);
    add_cached(c, 1, x - 1, 1, sum, cnt);
  }
  if (x <= w - 2 && y <= h - 2) add_cached(c, 1, x, 0, sum, cnt);
  if (cnt == 0) return false;
  d3 n = div3(sum, (double)cnt);
  const double len = norm3(n);
  if (len < 1e-12) return false;
  n = div3(n, len);
  const d3 local = c.local(x, y);
  if (dot3(n, local) > 0) n = neg3(n);
  *local_out = local;
  *n_out = n;
  return true;
}

struct Staged {  // per-point staging record (row-local order)
  double pos[3], nrm[3], w;
  int32_t px;
};

__global__ void __launch_bounds__(kThreads) pre_points_kernel(const __grid_constant__ SensorSet ss, double disc,
                                                              int sil_r, const uint16_t* __restrict__ pref, int ppitch,
                                                              Staged* __restrict__ stage, int spitch,
                                                              int32_t* __restrict__ row_counts,
                                                              float* __restrict__ weight_maps,
                                                              double* __restrict__ row_bbox) {
  extern __shared__ double smem_d[];  // pos [3][w][3] | tri [2][w][2][4] | depth [3][w] (uint16)
  __shared__ int warp_cnt[kThreads / 32];
  __shared__ int any_valid;
  __shared__ double bb[kThreads / 32][6];
  int k, y;
  row_of_block(ss, blockIdx.x, &k, &y);
  const DevSensor& s = ss.s[k];
  const ViewPtrs& v = ss.v[k];
  const int w = s.w, h = s.h;
  double* spos = smem_d;
  double* stri = smem_d + (size_t)9 * w;
  uint16_t* rows3 = reinterpret_cast<uint16_t*>(smem_d + (size_t)9 * w + (size_t)16 * w);
  if (threadIdx.x == 0) any_valid = 0;
  __syncthreads();
  // stage rows y-1..y+1: depth where the mask is set, else 0 (cloud.cpp:28-30),
  // and backproject each valid pixel once (camera.cpp:12-17)
  int mine = 0;
  for (int i = threadIdx.x; i < 3 * w; i += kThreads) {
    const int r = i / w, x = i - r * w, yy = y - 1 + r;
    uint16_t d = 0;
    if (yy >= 0 && yy < h && v.mask[(size_t)yy * v.mpitch + x]) d = v.depth[(size_t)yy * v.dpitch + x];
    rows3[i] = d;
    if (d) {
      const double z = (double)d;
      spos[3 * i + 0] = ddiv(dmul(dsub((double)x, s.cx), z), s.fx);
      spos[3 * i + 1] = ddiv(dmul(dsub((double)yy, s.cy), z), s.fy);
      spos[3 * i + 2] = z;
      if (r == 1) mine = 1;
    }
  }
  if (mine) any_valid = 1;
  __syncthreads();
  float* wrow0 = weight_maps + ss.pix_offset[k] + (size_t)y * w;
  if (!any_valid) {  // no foreground on this row: no points
    for (int x = threadIdx.x; x < w; x += kThreads) wrow0[x] = 0.f;
    if (threadIdx.x < 6) row_bbox[(size_t)blockIdx.x * 6 + threadIdx.x] = threadIdx.x < 3 ? DBL_MAX * 2.0 : -DBL_MAX * 2.0;
    if (threadIdx.x == 0) row_counts[blockIdx.x] = 0;
    return;
  }
  const RowCache c{w, h, y, rows3, spos, stri};
  // triangle normals of quads (qx, qy), qy in {y-1, y}: T1 = (i00,i10,i01), T2 = (i10,i11,i01)
  for (int i = threadIdx.x; i < 2 * w; i += kThreads) {
    const int qr = i / w, qx = i - qr * w, qy = y - 1 + qr;
    double* t1 = stri + ((size_t)(qr * w + qx) * 2 + 0) * 4;
    double* t2 = t1 + 4;
    t1[3] = 0.0, t2[3] = 0.0;
    if (qx + 1 >= w || qy < 0 || qy + 1 >= h) continue;
    triangle_normal(c, qx, qy, qx + 1, qy, qx, qy + 1, disc, t1);
    triangle_normal(c, qx + 1, qy, qx + 1, qy + 1, qx, qy + 1, disc, t2);
  }
  __syncthreads();
  const double window = (double)(2 * sil_r + 1) * (double)(2 * sil_r + 1);
  const int wy0 = max(0, y - sil_r), wy1 = min(h - 1, y + sil_r);
  const uint16_t* prow0 = pref + (size_t)(blockIdx.x - y) * ppitch;  // row 0 of this view
  const double inf = DBL_MAX * 2.0;
  double lo0 = inf, lo1 = inf, lo2 = inf, hi0 = -inf, hi1 = -inf, hi2 = -inf;
  int base = 0;
  Staged* srow = stage + (size_t)blockIdx.x * spitch;
  float* wrow = wrow0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int x0 = 0; x0 < w; x0 += kThreads) {
    const int x = x0 + threadIdx.x;
    d3 local{0, 0, 0}, n{0, 0, 0};
    const bool is_pt = x < w && point_at(c, x, &local, &n);
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

static size_t points_smem(int maxw) {
  return (size_t)maxw * (9 + 16) * sizeof(double) + 3 * (size_t)maxw * sizeof(uint16_t) + 16;
}

void prepare_preprocess(const SensorSet& ss) {  // outside any graph capture
  int maxw = 0;
  for (int k = 0; k < ss.k; ++k) maxw = maxw > ss.s[k].w ? maxw : ss.s[k].w;
  cudaFuncSetAttribute(pre_points_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)points_smem(maxw));
}

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
  const size_t smem = points_smem(maxw);
  pre_points_kernel<<<rows, kThreads, smem, st>>>(ss, disc_mm, sil_r, s.pref, s.ppitch,
                                                                         s.stage, s.spitch, s.counts, weight_maps,
                                                                         s.bbox);
  pre_scan_kernel<<<1, 1024, 0, st>>>(s.counts, s.offsets, rows, pts.cap, ctl);
  pre_gather_kernel<<<warp_grid, 256, 0, st>>>(ss, rows, s.stage, s.spitch, s.counts, s.offsets, pts);
  pre_fit_kernel<<<1, 256, 0, st>>>(s.bbox, rows, nx, ny, nz, padding, ctl);
}

}  // namespace vc

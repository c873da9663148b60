// SPDX-License-Identifier: Apache-2.0
//
// K1/K2 — depth preprocessing on sm_100a: build_cloud + confidence_weights
// (/root/reference/proj/core/src/recon/cloud.cpp:19-117), the foreground
// bounding box and fit_grid (reconstruct.cpp:16-35, 56-68).
//
// Pixel-parallel, with one ordered compaction at the end.  A "segment" is 32
// consecutive pixels of one depth row; segments are numbered row-major over
// the rows of all views concatenated, which is the reference's point order
// (views in sensor order, pixels row-major).
//
//   pre_prefix_tri  one warp per depth row: inclusive prefix count of the
//               mask along x (so the 21x21 silhouette box count of
//               cloud.cpp:89-106 costs 2 loads per window row), and the T1/T2
//               triangle normals of the row's quads with a valid corner
//               (cloud.cpp:38-59), compacted across the warp, computed once each
//   pre_points  one thread per pixel: the six incident triangles in the
//               reference's accumulation order (cloud.cpp:53-71), world
//               position/normal (:73-74), W = W1*W2 (:108-114) -> per-pixel
//               staging slot + flag, weight map, per-segment / per-row /
//               per-64-row-block counts; the bbox is folded in with atomic
//               min/max on order-preserving keys
//   pre_gather  one warp per active segment: its first point id from the
//               block, row and segment counts before it (no scan pass);
//               staged points -> final SoA in order; its first warp sets P,
//               the empty-scene status and fit_grid from the bbox
// fp64 with the reference's operation order and no FMA (vc_device.cuh), so
// positions — hence every downstream binning decision — are bit-exact.
#include <cfloat>

#include "vc_device.cuh"

namespace vc {
namespace {

constexpr int kRowBlock = 64;  // depth rows per point-count block sum (pre_points adds, pre_gather reads)
constexpr int kSegPx = 32;  // pixels per segment: one warp, one CTA of pre_points (a CTA
                            // retires with its slowest warp, so one-warp CTAs let the
                            // empty segments' slots recycle while point warps compute)

// Order-preserving map double -> u64 (for finite values and +-inf), so the
// bounding box is an exact atomic min/max whatever the order of updates.
__device__ __forceinline__ unsigned long long dkey(double d) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b >> 63) ? ~b : b ^ 0x8000000000000000ull;
}
__device__ __forceinline__ double dunkey(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? k ^ 0x8000000000000000ull : ~k));
}

__device__ __forceinline__ void row_of(const SensorSet& ss, int r, int* k, int* y) {
  int kk = 0;
  while (kk + 1 < ss.k && r >= ss.row_offset[kk + 1]) ++kk;
  *k = kk;
  *y = r - ss.row_offset[kk];
}

__device__ __forceinline__ bool valid_px(const ViewPtrs& v, int w, int h, int x, int y) {
  if (x < 0 || y < 0 || x >= w || y >= h) return false;
  const uint8_t m = __ldg(v.mask + (size_t)y * v.mpitch + x);
  const uint16_t d = __ldg(v.depth + (size_t)y * v.dpitch + x);
  return (m != 0) & (d != 0);
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

// quad (qx, qy) = pixel index of its i00 corner; T1 = (i00, i10, i01),
// T2 = (i10, i11, i01) (cloud.cpp:53-59), stored at the quad's pixel index
__device__ __forceinline__ void quad_triangles(const SensorSet& ss, int k, int qx, int qy, double disc,
                                               double* __restrict__ tri) {
  const DevSensor& s = ss.s[k];
  const ViewPtrs& v = ss.v[k];
  const bool v00 = valid_px(v, s.w, s.h, qx, qy), v10 = valid_px(v, s.w, s.h, qx + 1, qy);
  const bool v01 = valid_px(v, s.w, s.h, qx, qy + 1), v11 = valid_px(v, s.w, s.h, qx + 1, qy + 1);
  const d3 z{0, 0, 0};
  const d3 p00 = v00 ? local_px(s, v, qx, qy) : z, p10 = v10 ? local_px(s, v, qx + 1, qy) : z;
  const d3 p01 = v01 ? local_px(s, v, qx, qy + 1) : z, p11 = v11 ? local_px(s, v, qx + 1, qy + 1) : z;
  const d3 t1 = triangle_normal(v00 && v10 && v01, p00, p10, p01, disc);
  const d3 t2 = triangle_normal(v10 && v11 && v01, p10, p11, p01, disc);
  double* o = tri + 6 * (ss.pix_offset[k] + (int64_t)qy * s.w + qx);
  o[0] = t1.x, o[1] = t1.y, o[2] = t1.z, o[3] = t2.x, o[4] = t2.y, o[5] = t2.z;
}

// One warp per depth row (lane = 16 consecutive pixels):
//  (1) inclusive prefix of (mask != 0) along the row, so the 21x21 silhouette
//      box count of cloud.cpp:89-106 costs 2 loads per window row;
//  (2) the row's quads with a valid corner, compacted across the warp in x
//      order, then their two triangle normals with the lanes taking turns
//      (most quads of a frame are empty; the rest cluster on the silhouette).
__global__ void __launch_bounds__(256) pre_prefix_tri_kernel(const __grid_constant__ SensorSet ss, int rows,
                                                             uint16_t* __restrict__ pref, int pitch, DevCtl* ctl,
                                                             double disc, double* __restrict__ tri, int spr,
                                                             int32_t* __restrict__ seg_counts,
                                                             uint8_t* __restrict__ flags,
                                                             float* __restrict__ weight_maps,
                                                             int32_t* __restrict__ act,
                                                             int32_t* __restrict__ rowcnt,
                                                             int32_t* __restrict__ bsum) {
  __shared__ uint16_t qlist[8][512];
  __shared__ __align__(128) uint8_t rstage[8][3072];  // per warp: mask y, y+1 (512 B each), depth y, y+1 (1 KB each)
  __shared__ __align__(8) uint64_t rbar[8];
  if (blockIdx.x == 0 && threadIdx.x < 6) ctl->bbox_key[threadIdx.x] = threadIdx.x < 3 ? ~0ull : 0ull;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31, wid = (threadIdx.x >> 5) & 7;
  if (r >= rows) return;  // whole warps
  if (lane == 0) rowcnt[r] = 0;  // the row's point count (pre_points adds, pre_gather sums)
  if (lane == 0 && (r & (kRowBlock - 1)) == 0) bsum[r / kRowBlock] = 0;
  int k, y;
  row_of(ss, r, &k, &y);
  const ViewPtrs& v = ss.v[k];
  const int w = ss.s[k].w, h = ss.s[k].h;
  const uint8_t* m = v.mask + (size_t)y * v.mpitch;
  uint16_t* o = pref + (size_t)r * pitch;
  const uint16_t* dy = v.depth + (size_t)y * v.dpitch;
  const bool has_next = y + 1 < h;
  const uint8_t* m1 = v.mask + (size_t)(has_next ? y + 1 : y) * v.mpitch;
  const uint16_t* d1 = v.depth + (size_t)(has_next ? y + 1 : y) * v.dpitch;
  // Rows of up to 512 pixels with 16-byte aligned starts are staged into shared
  // memory by the tensor-memory accelerator (bulk copies of the four rows the
  // warp reads, one mbarrier per warp); the loads below then come from there.
  const bool bulk = w <= 512 && (w & 15) == 0 &&
                    ((reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(m1) |
                      reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(d1)) & 15) == 0;
  if (bulk) {
    uint8_t* st = rstage[wid];
    if (lane == 0) {
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&rbar[wid]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      const uint32_t bytes = (uint32_t)(3 * w) * (has_next ? 2u : 1u);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
      auto copy = [&](uint8_t* dst, const void* src, uint32_t n) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                (uint32_t)__cvta_generic_to_shared(dst)),
            "l"(src), "r"(n), "r"(b)
            : "memory");
      };
      copy(st, m, (uint32_t)w);
      copy(st + 1024, dy, (uint32_t)(2 * w));
      if (has_next) {
        copy(st + 512, m1, (uint32_t)w);
        copy(st + 2048, d1, (uint32_t)(2 * w));
      }
    }
    __syncwarp();
    asm volatile(
        "{\n .reg .pred p;\n RW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra RW_%=;\n}" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&rbar[wid]))
        : "memory");
    m = st, dy = reinterpret_cast<const uint16_t*>(st + 1024);
    m1 = has_next ? st + 512 : st, d1 = reinterpret_cast<const uint16_t*>(has_next ? st + 2048 : st + 1024);
  }
  // row element loads: shared memory when staged, else the read-only global path
  auto ld16 = [&](const void* p) {
    return bulk ? *reinterpret_cast<const uint4*>(p) : __ldg(reinterpret_cast<const uint4*>(p));
  };
  auto ldm = [&](const uint8_t* p) -> uint8_t { return bulk ? *p : __ldg(p); };
  auto ldd = [&](const uint16_t* p) -> uint16_t { return bulk ? *p : __ldg(p); };
  int carry = 0;
  for (int x0 = 0; x0 < w; x0 += 512) {
    const int xb = x0 + lane * 16;
    // 16-pixel validity words: bit i = pixel xb+i.  Whole 16-pixel groups on
    // 16-byte aligned mask rows and 32-byte aligned depth rows load as
    // vectors (5 requests instead of 64 scalar ones).
    uint32_t fgm = 0, val0 = 0, val1 = 0;  // mask row y; mask && depth row y; row y+1
    const bool vec = xb + 16 <= w && ((reinterpret_cast<uintptr_t>(m + xb) | reinterpret_cast<uintptr_t>(m1 + xb)) & 15) == 0 &&
                     ((reinterpret_cast<uintptr_t>(dy + xb) | reinterpret_cast<uintptr_t>(d1 + xb)) & 15) == 0;
    if (vec) {
      const uint4 mq = ld16(m + xb);
      const uint4 da = ld16(dy + xb), db = ld16(dy + xb + 8);
      const uint32_t mw[4] = {mq.x, mq.y, mq.z, mq.w};
      const uint32_t dw[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const bool mi = ((mw[i >> 2] >> (8 * (i & 3))) & 0xffu) != 0u;
        const bool di = ((dw[i >> 1] >> (16 * (i & 1))) & 0xffffu) != 0u;
        fgm |= (mi ? 1u : 0u) << i;
        val0 |= (mi && di ? 1u : 0u) << i;
      }
      if (has_next) {
        const uint4 mq1 = ld16(m1 + xb);
        const uint4 ea = ld16(d1 + xb), eb = ld16(d1 + xb + 8);
        const uint32_t nw[4] = {mq1.x, mq1.y, mq1.z, mq1.w};
        const uint32_t ew[8] = {ea.x, ea.y, ea.z, ea.w, eb.x, eb.y, eb.z, eb.w};
#pragma unroll
        for (int i = 0; i < 16; ++i)
          val1 |= (((nw[i >> 2] >> (8 * (i & 3))) & 0xffu) != 0u && ((ew[i >> 1] >> (16 * (i & 1))) & 0xffffu) != 0u
                       ? 1u : 0u) << i;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int x = xb + i;
        if (x < w) {
          const bool mi = ldm(m + x) != 0;
          fgm |= (mi ? 1u : 0u) << i;
          val0 |= (mi && ldd(dy + x) != 0 ? 1u : 0u) << i;
          if (has_next) val1 |= (ldm(m1 + x) != 0 && ldd(d1 + x) != 0 ? 1u : 0u) << i;
        }
      }
    }
    if (xb + 16 < w) {  // pixel xb+16 closes this group's last quad
      val0 |= (ldm(m + xb + 16) != 0 && ldd(dy + xb + 16) != 0 ? 1u : 0u) << 16;
      if (has_next) val1 |= (ldm(m1 + xb + 16) != 0 && ldd(d1 + xb + 16) != 0 ? 1u : 0u) << 16;
    }
    const int run = __popc(fgm);
    int inc = run;
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += t;
    }
    int acc = carry + inc - run;
    if (xb + 16 <= w && (reinterpret_cast<uintptr_t>(o + xb) & 15) == 0) {  // 16 prefix values as two 16 B stores
      uint32_t pw[8];
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const uint32_t a = (uint32_t)(acc + __popc(fgm & ((2u << i) - 1u)));
        const uint32_t b2 = (uint32_t)(acc + __popc(fgm & ((4u << i) - 1u)));
        pw[i >> 1] = (a & 0xffffu) | (b2 << 16);
      }
      reinterpret_cast<uint4*>(o + xb)[0] = make_uint4(pw[0], pw[1], pw[2], pw[3]);
      reinterpret_cast<uint4*>(o + xb)[1] = make_uint4(pw[4], pw[5], pw[6], pw[7]);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        acc += (fgm >> i) & 1u;
        if (xb + i < w) o[xb + i] = (uint16_t)acc;
      }
    }
    carry += __shfl_sync(0xffffffffu, inc, 31);
    {  // 32-pixel segments (lane pairs): no foreground -> no point: zero its
       // outputs here; the others go to the active list pre_points walks
      const int fg = run + __shfl_xor_sync(0xffffffffu, run, 1);
      const int sx = (x0 >> 5) + (lane >> 1);
      const bool seg_ok = xb < w && sx < spr;
      const int64_t pix0 = ss.pix_offset[k] + (int64_t)y * w;
      if (seg_ok && fg == 0) {
        const int64_t q = pix0 + xb;
        if (xb + 16 <= w && (q & 15) == 0) {  // 16 flags + 16 weights as vector stores
          *reinterpret_cast<uint4*>(flags + q) = make_uint4(0u, 0u, 0u, 0u);
          float4* wm4 = reinterpret_cast<float4*>(weight_maps + q);
          const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
          wm4[0] = z4, wm4[1] = z4, wm4[2] = z4, wm4[3] = z4;
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (xb + i < w) flags[q + i] = 0, weight_maps[q + i] = 0.f;
        }
      }
      const bool lead = seg_ok && (lane & 1) == 0;
      if (lead && fg == 0) seg_counts[r * spr + sx] = 0;
      const unsigned ball = __ballot_sync(0xffffffffu, lead && fg != 0);
      int base = 0;
      if (lane == 0 && ball) base = atomicAdd(act, __popc(ball));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (lead && fg != 0) act[1 + base + __popc(ball & ((1u << lane) - 1u))] = r * spr + sx;
    }
    if (!has_next) continue;  // no quads below the last row
    // pixels xb .. xb+16 valid in rows y, y+1 -> quads xb+i (i < 16) with a valid corner
    const uint32_t any = val0 | val1;
    uint32_t am = (any | (any >> 1)) & 0xffffu;
    const int lim = w - 1 - xb;  // quads xb+i need xb+i+1 < w
    am &= lim >= 16 ? 0xffffu : (lim <= 0 ? 0u : (1u << lim) - 1u);
    const int cnt = __popc(am);
    int pos = cnt;
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, pos, d);
      if (lane >= d) pos += t;
    }
    const int total = __shfl_sync(0xffffffffu, pos, 31);
    pos -= cnt;
    for (uint32_t mm = am; mm; mm &= mm - 1) qlist[wid][pos++] = (uint16_t)(xb + __ffs(mm) - 1);
    __syncwarp();
    for (int i = lane; i < total; i += 32) quad_triangles(ss, k, qlist[wid][i], y, disc, tri);
    __syncwarp();  // the list is rebuilt by the next chunk
  }
  for (int sx = (w + 31) / 32 + lane; sx < spr; sx += 32) seg_counts[r * spr + sx] = 0;  // past this view's width
}

__device__ __forceinline__ void add_tri(const d3& n, d3& sum, int& cnt) {
  if (n.x != n.x) return;  // rejected triangle (NaN marker)
  sum = add3(sum, n);
  ++cnt;
}
__device__ __forceinline__ d3 ld_tri(const double* tri, int64_t q, int t, bool use) {
  if (!use) return {__longlong_as_double(0x7ff8000000000000ll), 0.0, 0.0};
  const double* n = tri + 6 * q + 3 * t;
  return {__ldg(n), __ldg(n + 1), __ldg(n + 2)};
}

// both triangle normals of quad q (the record is 48 B, 16 B aligned) as three vector loads
__device__ __forceinline__ void ld_quad(const double* tri, int64_t q, bool use, d3& a, d3& b) {
  if (!use) {
    a = b = {__longlong_as_double(0x7ff8000000000000ll), 0.0, 0.0};
    return;
  }
  const double2* r = reinterpret_cast<const double2*>(tri + 6 * q);
  const double2 u = __ldg(r), v = __ldg(r + 1), w2 = __ldg(r + 2);
  a = {u.x, u.y, v.x};
  b = {v.y, w2.x, w2.y};
}

struct Staged {  // one point (per-pixel staging slot)
  double pos[3], nrm[3], w;
  int32_t pad;
};

__device__ __forceinline__ void points_segment(const SensorSet& ss, int sil_r, const double* __restrict__ tri,
                                               const uint16_t* __restrict__ pref, int ppitch,
                                               Staged* __restrict__ stage, uint8_t* __restrict__ flags,
                                               int32_t* __restrict__ seg_counts, DevCtl* ctl,
                                               float* __restrict__ weight_maps, int seg, int spr,
                                               int32_t* __restrict__ rowcnt, int32_t* __restrict__ bsum) {
  const int row = seg / spr, sx = seg - row * spr;
  int k, y;
  row_of(ss, row, &k, &y);
  const DevSensor& s = ss.s[k];
  const ViewPtrs& v = ss.v[k];
  const int w = s.w, h = s.h;
  const int x = sx * kSegPx + threadIdx.x;
  const int64_t pix = ss.pix_offset[k] + (int64_t)y * w + x;
  const double inf = DBL_MAX * 2.0;
  d3 p{inf, inf, inf}, nw{0, 0, 0};
  bool is_pt = false;
  double wt = 0.0;
  if (x < w && valid_px(v, w, h, x, y)) {
    // cloud.cpp:53-71: six incident triangles in the reference's order
    // Q(x-1,y-1).T2, Q(x,y-1).T1, Q(x,y-1).T2, Q(x-1,y).T1, Q(x-1,y).T2, Q(x,y).T1
    // all six triangle records are loaded up front (one round trip)
    // quads (x, y-1) and (x-1, y) hold both triangles: one 48 B record each, three 16 B loads
    const d3 t0 = ld_tri(tri, pix - w - 1, 1, x >= 1 && y >= 1);
    d3 t1, t2, t3, t4;
    ld_quad(tri, pix - w, x <= w - 2 && y >= 1, t1, t2);
    ld_quad(tri, pix - 1, x >= 1 && y <= h - 2, t3, t4);
    const d3 t5 = ld_tri(tri, pix, 0, x <= w - 2 && y <= h - 2);
    const uint16_t dc = __ldg(v.depth + (size_t)y * v.dpitch + x);
    d3 sum{0.0, 0.0, 0.0};
    int cnt = 0;
    add_tri(t0, sum, cnt);
    add_tri(t1, sum, cnt);
    add_tri(t2, sum, cnt);
    add_tri(t3, sum, cnt);
    add_tri(t4, sum, cnt);
    add_tri(t5, sum, cnt);
    if (cnt > 0) {
      d3 n = div3(sum, (double)cnt);
      const double len = norm3(n);
      if (len >= 1e-12) {
        n = div3(n, len);
        const double zc = (double)dc;
        const d3 local{ddiv(dmul(dsub((double)x, s.cx), zc), s.fx), ddiv(dmul(dsub((double)y, s.cy), zc), s.fy), zc};
        if (dot3(n, local) > 0) n = neg3(n);
        is_pt = true;
        // cloud.cpp:73-74 world position / normal
        p = add3(mat3(s.R, local), ld3(s.t));
        nw = mat3(s.R, n);
        // cloud.cpp:108-114: W1 from the re-transformed local frame
        const d3 l2 = add3(mat3(s.Ri, p), ld3(s.ti));
        const d3 nl = mat3(s.Ri, nw);
        const double w1raw = dot3(neg3(normalized3(l2)), nl);
        const double w1 = w1raw < 0.0 ? 0.0 : w1raw;
        // cloud.cpp:99-106 W2: (2r+1)^2 window clipped to the image, fixed divisor
        const int xa = max(0, x - sil_r), xb = min(w - 1, x + sil_r);
        const int wy0 = max(0, y - sil_r), wy1 = min(h - 1, y + sil_r);
        const uint16_t* pr = pref + (size_t)(row - y + wy0) * ppitch;
        uint32_t c2 = 0;
        const int nrow = wy1 - wy0 + 1;
        for (int r0 = 0; r0 < nrow; r0 += 16) {
          uint16_t hiv[16], lov[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const bool in = r0 + i < nrow;
            hiv[i] = in ? __ldg(pr + (size_t)(r0 + i) * ppitch + xb) : 0;
            lov[i] = (in && xa > 0) ? __ldg(pr + (size_t)(r0 + i) * ppitch + xa - 1) : 0;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) c2 += (uint32_t)hiv[i] - (uint32_t)lov[i];
        }
        const double window = (double)(2 * sil_r + 1) * (double)(2 * sil_r + 1);
        wt = dmul(w1, ddiv((double)c2, window));
        Staged& o = stage[pix];
        o.pos[0] = p.x, o.pos[1] = p.y, o.pos[2] = p.z;
        o.nrm[0] = nw.x, o.nrm[1] = nw.y, o.nrm[2] = nw.z;
        o.w = wt;
      }
    }
  }
  if (x < w) {
    flags[pix] = is_pt ? 1 : 0;
    weight_maps[pix] = is_pt ? (float)wt : 0.f;  // cloud.cpp:63,80,115
  }
  // segment count + bbox (one warp = one segment: no barrier)
  const int lane = threadIdx.x & 31;
  const unsigned ball = __ballot_sync(0xffffffffu, is_pt);
  if (lane == 0) seg_counts[seg] = __popc(ball);
  if (ball == 0u) return;  // warp-uniform: most segments of a frame hold no point
  if (lane == 0) {
    atomicAdd(rowcnt + row, __popc(ball));
    atomicAdd(bsum + row / kRowBlock, __popc(ball));
  }
  double lo[3] = {p.x, p.y, p.z}, hi[3] = {is_pt ? p.x : -inf, is_pt ? p.y : -inf, is_pt ? p.z : -inf};
#pragma unroll
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  if (lane < 3) atomicMin(&ctl->bbox_key[lane], dkey(lane == 0 ? lo[0] : (lane == 1 ? lo[1] : lo[2])));
  else if (lane < 6) atomicMax(&ctl->bbox_key[lane], dkey(lane == 3 ? hi[0] : (lane == 4 ? hi[1] : hi[2])));
}

// persistent one-warp CTAs over the active segments (pre_prefix_tri zeroed
// the outputs of the others); any order: outputs are per pixel / segment and
// the bbox an exact min/max
__global__ void __launch_bounds__(kSegPx) pre_points_kernel(const __grid_constant__ SensorSet ss, int sil_r,
                                                            const double* __restrict__ tri,
                                                            const uint16_t* __restrict__ pref, int ppitch,
                                                            Staged* __restrict__ stage, uint8_t* __restrict__ flags,
                                                            int32_t* __restrict__ seg_counts, DevCtl* ctl,
                                                            float* __restrict__ weight_maps,
                                                            const int32_t* __restrict__ act, int spr,
                                                            int32_t* __restrict__ rowcnt,
                                                            int32_t* __restrict__ bsum) {
  const int n = act[0];
  for (int i = blockIdx.x; i < n; i += gridDim.x)
    points_segment(ss, sil_r, tri, pref, ppitch, stage, flags, seg_counts, ctl, weight_maps, act[1 + i], spr,
                   rowcnt, bsum);
}

__device__ void fit_grid_dev(DevCtl* ctl, int nx, int ny, int nz, int pad);

// one warp per active segment (the others hold no point): staged point -> its
// rank = the points of the row blocks before its row's block (bsum) + of the
// block's rows before its row (rowcnt) + of the row's segments before it
// (seg_counts), summed by the warp — no separate scan pass.  Warp 0 of CTA 0
// first closes the preprocess: the point count P (sum of the block sums), the
// status, and the grid fit from the bbox pre_points left (the splat follows).
__global__ void __launch_bounds__(128) pre_gather_kernel(const __grid_constant__ SensorSet ss,
                                                         const Staged* __restrict__ stage,
                                                         const uint8_t* __restrict__ flags,
                                                         const int32_t* __restrict__ rowcnt,
                                                         const int32_t* __restrict__ bsum,
                                                         const int32_t* __restrict__ seg_counts, DevPoints pts,
                                                         int spr, const int32_t* __restrict__ act, int rows,
                                                         DevCtl* ctl, int32_t* rowlist_reset, int nx, int ny, int nz,
                                                         int pad) {
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    int P = 0;
    for (int j = lane; j < (rows + kRowBlock - 1) / kRowBlock; j += 32) P += bsum[j];
    for (int o = 16; o > 0; o >>= 1) P += __shfl_xor_sync(0xffffffffu, P, o);
    if (lane == 0) {
      ctl->P = P;
      ctl->status = P == 0 ? 2 : (P > pts.cap ? 3 : 0);
      ctl->voff = 0;
      if (rowlist_reset) *rowlist_reset = 0;  // the frame's clear (launched before) has read the previous list
      fit_grid_dev(ctl, nx, ny, nz, pad);
    }
  }
  const int n = act[0];
  for (int i = blockIdx.x * 4 + (threadIdx.x >> 5); i < n; i += gridDim.x * 4) {
    const int seg = act[1 + i];
    const int row = seg / spr, sx = seg - row * spr;
    int k, y;
    row_of(ss, row, &k, &y);
    const int w = ss.s[k].w;
    const int x = sx * kSegPx + lane;
    const int64_t pix = ss.pix_offset[k] + (int64_t)y * w + x;
    const bool is_pt = x < w && flags[pix];
    const unsigned ball = __ballot_sync(0xffffffffu, is_pt);
    const int rb = row / kRowBlock;
    int before = 0;
    for (int j = lane; j < rb; j += 32) before += bsum[j];
    for (int j = rb * kRowBlock + lane; j < row; j += 32) before += rowcnt[j];
    for (int b = 0; b < sx; b += 32) before += b + lane < sx ? seg_counts[row * spr + b + lane] : 0;
    for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
    if (!is_pt) continue;
    const int idx = before + __popc(ball & ((1u << lane) - 1u));
    if (idx >= pts.cap) continue;  // status 3 (cannot happen: the capacity is one point per pixel)
    const Staged s = stage[pix];
    pts.pos[3 * idx + 0] = s.pos[0], pts.pos[3 * idx + 1] = s.pos[1], pts.pos[3 * idx + 2] = s.pos[2];
    pts.nrm[3 * idx + 0] = s.nrm[0], pts.nrm[3 * idx + 1] = s.nrm[1], pts.nrm[3 * idx + 2] = s.nrm[2];
    pts.weight[idx] = s.w;
    pts.pix[3 * idx + 0] = x, pts.pix[3 * idx + 1] = y, pts.pix[3 * idx + 2] = k;
  }
}

// reconstruct.cpp:56-68 (bbox) + fit_grid (reconstruct.cpp:16-35, dims given);
// one thread, after the scan has set the status
__device__ void fit_grid_dev(DevCtl* ctl, int nx, int ny, int nz, int pad) {
  double r[6];
  for (int a = 0; a < 6; ++a) r[a] = ctl->bbox[a] = dunkey(ctl->bbox_key[a]);
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
  double* tri;        // 6 doubles per quad (indexed by its i00 pixel)
  Staged* stage;      // per pixel
  uint8_t* flags;     // per pixel
  uint16_t* pref;     // rows x ppitch
  int32_t* counts;    // per segment
  int32_t* bsum;      // per kRowBlock depth rows: points
  int32_t* act;       // [count, active segment ids...]
  int32_t* rowcnt;    // per depth row: points
  int ppitch, spr, nseg;
};

Scratch carve(const SensorSet& ss, void* base) {
  const int rows = ss.row_offset[ss.k];
  const int64_t npix = ss.pix_offset[ss.k];
  int maxw = 0;
  for (int k = 0; k < ss.k; ++k) maxw = maxw > ss.s[k].w ? maxw : ss.s[k].w;
  auto up = [](uintptr_t p) { return (p + 255) & ~uintptr_t(255); };
  Scratch s;
  s.spr = (maxw + kSegPx - 1) / kSegPx;
  s.nseg = rows * s.spr;
  s.ppitch = (maxw + 127) & ~127;
  uintptr_t p = up(reinterpret_cast<uintptr_t>(base));
  s.tri = reinterpret_cast<double*>(p);
  p = up(p + (size_t)npix * 6 * sizeof(double));
  s.stage = reinterpret_cast<Staged*>(p);
  p = up(p + (size_t)npix * sizeof(Staged));
  s.flags = reinterpret_cast<uint8_t*>(p);
  p = up(p + (size_t)npix);
  s.pref = reinterpret_cast<uint16_t*>(p);
  p = up(p + (size_t)rows * s.ppitch * sizeof(uint16_t));
  s.counts = reinterpret_cast<int32_t*>(p);
  p = up(p + (size_t)s.nseg * sizeof(int32_t));
  s.bsum = reinterpret_cast<int32_t*>(p);
  p = up(p + (size_t)s.nseg * sizeof(int32_t));
  s.act = reinterpret_cast<int32_t*>(p);
  p = up(p + (size_t)(s.nseg + 1) * sizeof(int32_t));
  s.rowcnt = reinterpret_cast<int32_t*>(p);
  return s;
}

// dataset.cpp:99-102: foreground := depth > 0 (views staged without a mask)
__global__ void mask_from_depth_kernel(const uint16_t* __restrict__ depth, uint8_t* __restrict__ mask, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) mask[i] = depth[i] > 0 ? 1 : 0;
}

}  // namespace

void launch_mask_from_depth(const uint16_t* depth, uint8_t* mask, int n, cudaStream_t st) {
  const int blocks = (n + 255) / 256 < 592 ? (n + 255) / 256 : 592;
  mask_from_depth_kernel<<<blocks, 256, 0, st>>>(depth, mask, n);
}

void prepare_preprocess(const SensorSet&) {}  // no opt-in shared memory needed

size_t preprocess_scratch_bytes(const SensorSet& ss) {
  const Scratch s = carve(ss, nullptr);
  return reinterpret_cast<uintptr_t>(s.rowcnt) + (size_t)ss.row_offset[ss.k] * sizeof(int32_t) + 512;
}

void launch_preprocess(const SensorSet& ss, DevPoints pts, float* weight_maps, int32_t* scratch, DevCtl* ctl,
                       int nx, int ny, int nz, int padding, double disc_mm, int sil_r, cudaStream_t st,
                       int32_t* rowlist_reset) {
  const int rows = ss.row_offset[ss.k];
  const Scratch s = carve(ss, scratch);
  cudaMemsetAsync(s.act, 0, sizeof(int32_t), st);
  pre_prefix_tri_kernel<<<(rows * 32 + 255) / 256, 256, 0, st>>>(ss, rows, s.pref, s.ppitch, ctl, disc_mm, s.tri,
                                                                  s.spr, s.counts, s.flags, weight_maps, s.act,
                                                                  s.rowcnt, s.bsum);
  const int pgrid = s.nseg < sm_count() * 16 ? s.nseg : sm_count() * 16;  // resident one-warp CTAs (registers: 16 warps/SM)
  pre_points_kernel<<<pgrid, kSegPx, 0, st>>>(ss, sil_r, s.tri, s.pref, s.ppitch, s.stage, s.flags, s.counts, ctl,
                                              weight_maps, s.act, s.spr, s.rowcnt, s.bsum);
  pre_gather_kernel<<<sm_count() * 8, 128, 0, st>>>(ss, s.stage, s.flags, s.rowcnt, s.bsum, s.counts, pts, s.spr, s.act,
                                                    rows, ctl, rowlist_reset, nx, ny, nz, padding);
}

}  // namespace vc

// SPDX-License-Identifier: Apache-2.0
//
// K9 — iso level (splat.cpp:91-101 with sample_trilinear, volume.hpp:59-81)
// K10 — marching cubes (marching_cubes.cpp:131-210) as row culling /
// classify / scan / emit, with no host round trip (counts live in DevCtl;
// capacity overflow sets a flag the host checks once per frame).
//
//   mc_select   per voxel row (y,z): can it hold a cut edge or cell?  (row
//               min/max from the last FFT pass vs the level) -> ordered list
//               in one pass (decoupled look-back over 256-unit tiles)
//   mc_count    one warp per active row: 8 voxels per lane tested for a level
//               crossing from vector row loads, then one voxel per lane over the
//               row's straddling 32-voxel chunks only: owned cut edges
//               (+x,+y,+z, sign test vals >= level in fp64, :168-171) and the
//               cell's triangle count from the generated table; caches each
//               voxel's (mask, case) and the row's chunk mask; per-256-row
//               block sums of the (vertex, triangle, cell) counts
//   mc_scan_emit  per 8-row tile: its first ids from the block sums and row
//               counts before it, then one warp per row over its straddling
//               chunks; vertex ids = rank of the cut edge in global edge id
//               order ((z*ny+y)*nx+x)*3+axis (:139-142); fp64 positions
//               (:153-155, volume.hpp:45); compact list of cells
//               (the z-slab path splits this into mc_scan, a 1024-row-tile
//               look-back, and mc_emit: its vertex ids need the other ranks'
//               counts between the two)
//   mc_finish   one thread per vertex (gradient normals, :180-207) or per
//               active cell (triangles in the reference's cell scan order
//               (z, y, x), table order within the cell)
#include <cstdlib>
#include <cfloat>

#include "vc_device.cuh"

namespace vc {
namespace {

// The case tables in global memory, read through L1: the kernels index them by
// each lane's cell case, and divergent indices into the constant bank
// serialise (they were a fifth of the triangle pass's stalls).
__device__ int8_t g_mc_count[256];
__device__ int8_t g_mc_tris[256][5][3];
__device__ __forceinline__ int mc_count(int cfg) { return __ldg(&g_mc_count[cfg]); }
__device__ __forceinline__ int mc_tri_edge(int cfg, int tri, int m) { return __ldg(&g_mc_tris[cfg][tri][m]); }
// cube edge e (marching_cubes.cpp:15-19): axis e / 4; low corner 2e (x edges),
// {0, 1, 4, 5} (y edges), e - 8 (z edges) — corner bits (x, y, z)
__device__ __forceinline__ int edge_axis(int e) { return e >> 2; }
__device__ __forceinline__ int edge_c0(int e) { return e < 4 ? 2 * e : (e < 8 ? (e & 1) | ((e & 2) << 1) : e - 8); }


__device__ __forceinline__ float vol_at(const float* A, int nx, int ny, int x, int y, int z) {
  return __ldg(A + ((size_t)z * ny + y) * nx + x);
}

// volume.hpp:59-81 on the fp32 volume, evaluated in fp64
__device__ double trilinear(const float* A, const DevGrid& g, double vx, double vy, double vz) {
  auto clampf = [](double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); };
  const double fx = clampf(vx, 0.0, g.nx - 1.0), fy = clampf(vy, 0.0, g.ny - 1.0), fz = clampf(vz, 0.0, g.nz - 1.0);
  const int x0 = min((int)fx, g.nx - 2 >= 0 ? g.nx - 2 : 0);
  const int y0 = min((int)fy, g.ny - 2 >= 0 ? g.ny - 2 : 0);
  const int z0 = min((int)fz, g.nz - 2 >= 0 ? g.nz - 2 : 0);
  const int x1 = min(x0 + 1, g.nx - 1), y1 = min(y0 + 1, g.ny - 1), z1 = min(z0 + 1, g.nz - 1);
  const double tx = dsub(fx, (double)x0), ty = dsub(fy, (double)y0), tz = dsub(fz, (double)z0);
  const double v000 = vol_at(A, g.nx, g.ny, x0, y0, z0), v100 = vol_at(A, g.nx, g.ny, x1, y0, z0);
  const double v010 = vol_at(A, g.nx, g.ny, x0, y1, z0), v110 = vol_at(A, g.nx, g.ny, x1, y1, z0);
  const double v001 = vol_at(A, g.nx, g.ny, x0, y0, z1), v101 = vol_at(A, g.nx, g.ny, x1, y0, z1);
  const double v011 = vol_at(A, g.nx, g.ny, x0, y1, z1), v111 = vol_at(A, g.nx, g.ny, x1, y1, z1);
  const double ux = dsub(1.0, tx), uy = dsub(1.0, ty), uz = dsub(1.0, tz);
  const double c00 = dadd(dmul(v000, ux), dmul(v100, tx));
  const double c10 = dadd(dmul(v010, ux), dmul(v110, tx));
  const double c01 = dadd(dmul(v001, ux), dmul(v101, tx));
  const double c11 = dadd(dmul(v011, ux), dmul(v111, tx));
  const double c0 = dadd(dmul(c00, uy), dmul(c10, ty));
  const double c1 = dadd(dmul(c01, uy), dmul(c11, ty));
  return dadd(dmul(c0, uz), dmul(c1, tz));
}

// Fixed-order sum over 256 threads (deterministic): butterfly within each
// warp, then the 8 warp sums in order by thread 0 (the result is thread 0's).
__device__ __forceinline__ double block_sum_256(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < 8; ++w) s = dadd(s, sh[w]);
  return s;
}
constexpr int kIsoBlocks = 296;

__device__ void iso_final_tree(const double* partial, int n, DevCtl* ctl, double* sh);

// The CTA that finishes last also forms the level (the same fixed tree over
// the per-CTA partials as iso_final_kernel, so the result is deterministic).
__global__ void __launch_bounds__(256) iso_partial_kernel(const double* __restrict__ pos, const float* __restrict__ A,
                                                          DevCtl* __restrict__ ctl, double* partial) {
  __shared__ double sh[256];
  double sum = 0.0;
  if (ctl->status == 0) {
    const DevGrid g = ctl->grid;
    const int P = ctl->P;
    for (int p = blockIdx.x * 256 + threadIdx.x; p < P; p += gridDim.x * 256) {
      const double vx = ddiv(dsub(pos[3 * p + 0], g.origin[0]), g.edge);
      const double vy = ddiv(dsub(pos[3 * p + 1], g.origin[1]), g.edge);
      const double vz = ddiv(dsub(pos[3 * p + 2], g.origin[2]), g.edge);
      sum = dadd(sum, trilinear(A, g, vx, vy, vz));
    }
  }
  sum = block_sum_256(sum, sh);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = sum;
    __threadfence();
    last = atomicAdd(&ctl->iso_ticket, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  iso_final_tree(partial, gridDim.x, ctl, sh);
  if (threadIdx.x == 0) ctl->iso_ticket = 0;
}
// the partials (slot i >= n holds 0): thread t adds slots t and t + 256, then
// the block sum, as iso_final_kernel does
__device__ void iso_final_tree(const double* partial, int n, DevCtl* ctl, double* sh) {
  const int t = threadIdx.x;
  const volatile double* vp = partial;
  const double s = block_sum_256(dadd(t < n ? vp[t] : 0.0, t + 256 < n ? vp[t + 256] : 0.0), sh);
  if (t == 0 && ctl->status == 0) ctl->level = ddiv(s, (double)ctl->P);
}

// trilinear()'s lower z plane of the point, owned by exactly one slab
__global__ void __launch_bounds__(256) iso_sample_kernel(const double* __restrict__ pos, const float* __restrict__ A,
                                                         const DevCtl* __restrict__ ctl, int zoff, int nzl,
                                                         double* samples) {
  if (ctl->status != 0) return;
  const DevGrid g = ctl->grid;
  const int P = ctl->P;
  for (int p = blockIdx.x * 256 + threadIdx.x; p < P; p += gridDim.x * 256) {
    const double vx = ddiv(dsub(pos[3 * p + 0], g.origin[0]), g.edge);
    const double vy = ddiv(dsub(pos[3 * p + 1], g.origin[1]), g.edge);
    const double vz = ddiv(dsub(pos[3 * p + 2], g.origin[2]), g.edge);
    const double fz = vz < 0.0 ? 0.0 : (vz > g.nz - 1.0 ? g.nz - 1.0 : vz);
    const int z0 = min((int)fz, g.nz - 2 >= 0 ? g.nz - 2 : 0);
    samples[p] = (z0 >= zoff && z0 < zoff + nzl) ? trilinear(A, g, vx, vy, vz) : 0.0;
  }
}

// iso_partial_kernel's reduction order over precomputed samples
__global__ void __launch_bounds__(256) iso_partial_samples_kernel(const double* __restrict__ samples,
                                                                  const DevCtl* __restrict__ ctl, double* partial) {
  __shared__ double sh[256];
  double sum = 0.0;
  if (ctl->status == 0) {
    const int P = ctl->P;
    for (int p = blockIdx.x * 256 + threadIdx.x; p < P; p += gridDim.x * 256) sum = dadd(sum, samples[p]);
  }
  sum = block_sum_256(sum, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = sum;
}

__global__ void __launch_bounds__(256) iso_final_kernel(const double* partial, int n, DevCtl* ctl) {
  __shared__ double sh[8];
  iso_final_tree(partial, n, ctl, sh);  // the same order as the single-GPU path's last CTA
}

struct VoxelInfo {
  int mask;  // cut edges owned by this voxel (bit axis)
  int cfg;   // cell case, -1 if no cell
};

// classify_regs below: cut-edge mask and cell case of a voxel.  The
// reference tests vals >= level in fp64 (marching_cubes.cpp:168-171); for an
// fp32 value a and double L that equals a >= Lf with Lf = L rounded up to fp32
// (__double2float_ru), so the test runs in fp32 bit-exactly.

// ---------------------------------------------------------------- row culling
// Work unit = voxel row (y, z): its x-edges, the y-edges to row y+1, the
// z-edges to row z+1 and the cells (x, y, z).  A unit can hold a cut edge or
// a non-trivial cell only if its 2-4 rows have values on both sides of the
// level (max >= L and min < L), so per-row min/max (written by the final FFT
// pass) skip the empty ~90% of the volume without reading it.
__global__ void row_minmax_kernel(const float* __restrict__ A, int nx, int rows, float2* rowmm) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  float lo = 3.4e38f, hi = -3.4e38f;
  for (int x = lane; x < nx; x += 32) {
    const float v = __ldg(A + (size_t)warp * nx + x);
    lo = fminf(lo, v), hi = fmaxf(hi, v);
  }
  for (int o = 16; o > 0; o >>= 1) lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o)), hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  if (lane == 0) rowmm[warp] = make_float2(lo, hi);
}

constexpr int kRowThreads = 256;

// Ordered list of the active units in one pass (single-pass scan with
// decoupled look-back): tiles of 256 units take ids from a counter (so every
// tile a tile waits on has started), test their units against the level
// (row min/max of the 2x2 rows from the C2R pass), publish their active count,
// and take the count of all earlier tiles from the published descriptors —
// warp 0 reads 32 predecessors per step and stops at the first one whose
// inclusive prefix is known.  Each tile then writes its units in raster order.
// Descriptor: bits 62-63 status (1 aggregate, 2 inclusive prefix), low 32 the count.
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kRowThreads) mc_select_kernel(const float2* __restrict__ rowmm, DevCtl* ctl, int ny,
                                                                int nz, McSlab sl, unsigned long long* desc,
                                                                int* tile_counter, int32_t* units, int* zero,
                                                                int nzero) {
  __shared__ int tile_s, wsum[kRowThreads / 32], base_s;
  // the next pass's look-back flags and ticket counter (it starts after this grid ends)
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nzero; j += gridDim.x * blockDim.x) zero[j] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl->v_extra = 0;
  const int U = ny * sl.nzu;
  const int ntiles = (U + kRowThreads - 1) / kRowThreads;
  if (threadIdx.x == 0) tile_s = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = tile_s;
  if (tile >= ntiles) return;
  const int u = tile * kRowThreads + threadIdx.x;
  bool active = false;
  if (u < U && ctl->status == 0) {
    const double L = ctl->level;
    const int y = u % ny, z = sl.z0 + u / ny;
    float2 m = rowmm[u];
    float lo = m.x, hi = m.y;
    if (y + 1 < ny) m = rowmm[u + 1], lo = fminf(lo, m.x), hi = fmaxf(hi, m.y);
    if (z + 1 < nz) m = rowmm[u + ny], lo = fminf(lo, m.x), hi = fmaxf(hi, m.y);
    if (y + 1 < ny && z + 1 < nz) m = rowmm[u + ny + 1], lo = fminf(lo, m.x), hi = fmaxf(hi, m.y);
    active = (double)hi >= L && (double)lo < L;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, active);
  if (lane == 0) wsum[wid] = __popc(b);
  __syncthreads();
  if (wid == 0) {
    int w = lane < kRowThreads / 32 ? wsum[lane] : 0;
    int agg = w;
    for (int o = 16; o > 0; o >>= 1) agg += __shfl_xor_sync(0xffffffffu, agg, o);
    // publish the aggregate (tile 0: its inclusive prefix), then look back
    if (lane == 0)
      atomicExch(desc + tile, ((tile == 0 ? 2ull : 1ull) << 62) | (unsigned long long)(unsigned)agg);
    int excl = 0;
    for (int look = tile - 1; look >= 0; look -= 32) {
      const int t = look - lane;
      unsigned long long d = 2ull << 62;  // lanes before tile 0: an inclusive zero
      if (t >= 0) {
        do d = ld_volatile_u64(desc + t);
        while ((d >> 62) == 0);
      }
      const unsigned incl = __ballot_sync(0xffffffffu, (d >> 62) == 2);
      const int first = incl ? __ffs(incl) - 1 : 32;  // nearest predecessor with a full prefix
      int v = lane <= first && t >= 0 ? (int)(d & 0xffffffffu) : 0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      excl += v;
      if (incl) break;
    }
    if (lane == 0) {
      if (tile > 0) atomicExch(desc + tile, (2ull << 62) | (unsigned long long)(unsigned)(excl + agg));
      base_s = excl;
      if (tile == ntiles - 1) ctl->units = excl + agg;
    }
    // warp-level exclusive offsets within the tile
    int inc = w;
    for (int o = 1; o < 32; o <<= 1) {
      const int q = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += q;
    }
    if (lane < kRowThreads / 32) wsum[lane] = inc - w;
  }
  __syncthreads();
  if (active) units[base_s + wsum[wid] + __popc(b & ((1u << lane) - 1u))] = u;
}

// One warp per active unit (voxel row), 8 consecutive voxels per lane per
// 256-voxel pass: the lane loads the 9 values x0..x0+8 of the 4 rows its
// voxels touch (two float4 + one scalar per row) and classifies all 8 from
// registers; no block-wide barrier anywhere.
constexpr int kVpl = 8;
constexpr int kFuseUnits = 8;   // units per scan/emit tile
constexpr int kCntBlock = 256;  // units per count block sum (bsum)

struct RowVals {
  float v[4][kVpl + 1];  // rows (y,z), (y+1,z), (y,z+1), (y+1,z+1); x0 .. x0+8
};

__device__ __forceinline__ void load_rows(const float* A, int nx, int ny, int nz, int y, int z, int x0, RowVals& r) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int yy = y + (q & 1), zz = z + (q >> 1);
    const bool ok = yy < ny && zz < nz && x0 < nx;
    const float* row = A + ((size_t)zz * ny + yy) * nx;
    if (ok && nx >= kVpl) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(row + x0));
      const float4 b = __ldg(reinterpret_cast<const float4*>(row + x0 + 4));
      r.v[q][0] = a.x, r.v[q][1] = a.y, r.v[q][2] = a.z, r.v[q][3] = a.w;
      r.v[q][4] = b.x, r.v[q][5] = b.y, r.v[q][6] = b.z, r.v[q][7] = b.w;
      r.v[q][kVpl] = x0 + kVpl < nx ? __ldg(row + x0 + kVpl) : 0.f;
    } else {
#pragma unroll
      for (int j = 0; j <= kVpl; ++j) r.v[q][j] = ok && x0 + j < nx ? __ldg(row + x0 + j) : 0.f;
    }
  }
}

__device__ __forceinline__ int3 warp_sum3(int3 v) {
  for (int o = 16; o > 0; o >>= 1)
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o), v.y += __shfl_xor_sync(0xffffffffu, v.y, o),
        v.z += __shfl_xor_sync(0xffffffffu, v.z, o);
  return v;
}

// The cell / cut-edge sets of voxel x at unit (y, z): the four rows' values at
// x and x+1 (q = 0: (y,z), 1: (y+1,z), 2: (y,z+1), 3: (y+1,z+1)).
__device__ __forceinline__ VoxelInfo classify_voxel(const float* A, int nx, int ny, int x, int y, int z, bool hy,
                                                    bool hz, float Lf) {
  VoxelInfo o{0, -1};
  if (x >= nx) return o;
  const bool hx = x + 1 < nx;
  const float* r0 = A + ((size_t)z * ny + y) * nx + x;
  const float* r1 = r0 + nx;
  const float* r2 = r0 + (size_t)nx * ny;
  const float* r3 = r2 + nx;
  const bool a0 = __ldg(r0) >= Lf;
  const bool a1 = hx && __ldg(r0 + 1) >= Lf;
  const bool a2 = hy && __ldg(r1) >= Lf;
  const bool a4 = hz && __ldg(r2) >= Lf;
  if (hx && a1 != a0) o.mask |= 1;
  if (hy && a2 != a0) o.mask |= 2;
  if (hz && a4 != a0) o.mask |= 4;
  if (hx && hy && hz) {
    int cfg = (a0 ? 1 : 0) | (a1 ? 2 : 0) | (a2 ? 4 : 0) | (a4 ? 16 : 0);
    cfg |= (__ldg(r1 + 1) >= Lf) << 3;
    cfg |= (__ldg(r2 + 1) >= Lf) << 5;
    cfg |= (__ldg(r3) >= Lf) << 6;
    cfg |= (__ldg(r3 + 1) >= Lf) << 7;
    o.cfg = cfg;
  }
  return o;
}

// per active unit: (owned cut edges, triangles, non-trivial cells) + the
// per-voxel (mask, case) cache the emit pass reads.  Pass 1: each lane loads
// the values its 8 voxels' cells touch (vector loads) and tests whether they
// straddle the level; a 32-voxel chunk with no straddling lane group holds no
// cut edge and no cell (every one of its voxels classifies to nothing).  Pass 2:
// one voxel per lane over the straddling chunks only (typically 1-2 of a row's
// chunks), whose cache entries and chunk mask the emit pass reuses.
// One unit's counts; `info` = the unit's nx cache entries (global or shared).
__device__ __forceinline__ int3 count_unit(const float* __restrict__ A, int nx, int ny, int nz, int y, int z, bool own,
                                           float Lf, int lane, uint16_t* info, uint32_t& cmask_out) {
  const bool hy = y + 1 < ny, hz = z + 1 < nz;
  uint32_t cmask = 0;
  for (int p0 = 0; p0 < nx; p0 += 32 * kVpl) {
    const int x0 = p0 + lane * kVpl;
    RowVals r;
    load_rows(A, nx, ny, nz, y, z, x0, r);
    bool above = false, below = false;
#pragma unroll
    for (int j = 0; j <= kVpl; ++j) {
      if (x0 + j >= nx) continue;
      const bool h0 = r.v[0][j] >= Lf;
      above |= h0, below |= !h0;
      if (hy) {
        const bool h = r.v[1][j] >= Lf;
        above |= h, below |= !h;
      }
      if (hz) {
        const bool h = r.v[2][j] >= Lf;
        above |= h, below |= !h;
      }
      if (hy && hz) {
        const bool h = r.v[3][j] >= Lf;
        above |= h, below |= !h;
      }
    }
    const uint32_t b = __ballot_sync(0xffffffffu, above && below);
    uint32_t c8 = 0;  // chunk k of this pass = lanes 4k .. 4k+3
#pragma unroll
    for (int k = 0; k < 8; ++k) c8 |= ((b >> (4 * k)) & 0xfu) ? 1u << k : 0u;
    cmask |= c8 << (p0 >> 5);
  }
  int3 c = make_int3(0, 0, 0);
  for (uint32_t mm = cmask; mm; mm &= mm - 1) {
    const int x = ((__ffs(mm) - 1) << 5) + lane;
    const VoxelInfo vi = classify_voxel(A, nx, ny, x, y, z, hy, hz, Lf);
    const int nt = vi.cfg >= 0 && own ? mc_count(vi.cfg) : 0;
    c.x += __popc(vi.mask), c.y += nt, c.z += nt > 0 ? 1 : 0;
    if (x < nx) info[x] = (uint16_t)(vi.mask | (nt > 0 ? (vi.cfg << 3) | (1 << 11) : 0));
  }
  cmask_out = cmask;
  return warp_sum3(c);
}

// CTA iteration k covers the 8 consecutive units 8 (blockIdx.x + k gridDim.x)
// + warp, all in one kCntBlock block: their sum goes to the block's bsum entry
// with one atomic triple per CTA iteration.
__global__ void __launch_bounds__(256, 4) mc_count_kernel(const float* __restrict__ A, DevCtl* ctl, int nx, int ny,
                                                       int nz, McSlab sl, const int32_t* __restrict__ units,
                                                       int3* unitcnt, int3* bsum, MeshBufs mb) {
  static_assert(kCntBlock % 8 == 0, "a CTA iteration's units share one block");
  __shared__ int3 part[8];
  if (ctl->status != 0) return;
  const int U = ctl->units;
  const float Lf = __double2float_ru(ctl->level);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i0 = blockIdx.x * 8; i0 < U; i0 += gridDim.x * 8) {
    const int i = i0 + wid;
    int3 t = make_int3(0, 0, 0);
    if (i < U) {
      const int u = units[i];
      const int y = u % ny, z = sl.z0 + u / ny;
      const bool own = z < sl.zend;
      uint32_t cmask;
      t = count_unit(A, nx, ny, nz, y, z, own, Lf, lane, mb.vinfo + (size_t)i * nx, cmask);
      if (lane == 0) {
        unitcnt[i] = t;
        mb.ucmask[i] = cmask;
        if (!own) atomicAdd(&ctl->v_extra, t.x);
      }
    }
    if (bsum) {
      if (lane == 0) part[wid] = t;
      __syncthreads();
      if (wid == 0) {
        int3 q = lane < 8 ? part[lane] : make_int3(0, 0, 0);
        q = warp_sum3(q);
        int3* d = bsum + i0 / kCntBlock;
        if (lane == 0 && q.x) atomicAdd(&d->x, q.x);
        if (lane == 1 && q.y) atomicAdd(&d->y, q.y);
        if (lane == 2 && q.z) atomicAdd(&d->z, q.z);
      }
      __syncthreads();
    }
  }
}

// Exclusive scan of the per-unit (V, T, C) counts in place, one pass over
// tiles of 1024 units (256 threads x 4) with decoupled look-back: a tile
// publishes its aggregate, sums its predecessors' published values (warp 0,
// 32 per step, stopping at the first inclusive prefix), publishes its
// inclusive prefix and writes its units' offsets.  Values are stored before
// their flag with a fence between (release), read after the flag (acquire).
// The last active tile forms V, T, C and the capacity check.
struct ScanState {
  int* flag;    // per tile: 0 none, 1 aggregate, 2 inclusive prefix
  int3* agg;    // per tile
  int3* incl;   // per tile
  int* counter;
};
__device__ __forceinline__ int ld_volatile_i32(const int* p) {
  int v;
  asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int3 ld_volatile_i3(const int3* p) {
  const volatile int* q = reinterpret_cast<const volatile int*>(p);
  return make_int3(q[0], q[1], q[2]);
}
__device__ __forceinline__ void st_volatile_i3(int3* p, int3 v) {
  volatile int* q = reinterpret_cast<volatile int*>(p);
  q[0] = v.x, q[1] = v.y, q[2] = v.z;
}

// Warp-wide (all 32 lanes): publish tile `tile`'s aggregate, sum the
// predecessors' published values (32 per step, stopping at the first
// inclusive prefix), publish the tile's inclusive prefix; returns the
// exclusive prefix.
__device__ __forceinline__ int3 lookback_publish(const ScanState& ss, int tile, int3 agg, int lane) {
  if (lane == 0) {
    st_volatile_i3(tile == 0 ? ss.incl + tile : ss.agg + tile, agg);
    __threadfence();
    atomicExch(ss.flag + tile, tile == 0 ? 2 : 1);
  }
  int3 excl = make_int3(0, 0, 0);
  for (int look = tile - 1; look >= 0; look -= 32) {
    const int t = look - lane;
    int f = 2;  // lanes before tile 0: an inclusive zero
    if (t >= 0) {
      do f = ld_volatile_i32(ss.flag + t);
      while (f == 0);
    }
    __threadfence();
    const unsigned incl = __ballot_sync(0xffffffffu, f == 2);
    const int first = incl ? __ffs(incl) - 1 : 32;
    int3 x = make_int3(0, 0, 0);
    if (t >= 0 && lane <= first) x = f == 2 ? ld_volatile_i3(ss.incl + t) : ld_volatile_i3(ss.agg + t);
    for (int o = 16; o > 0; o >>= 1)
      x.x += __shfl_xor_sync(0xffffffffu, x.x, o), x.y += __shfl_xor_sync(0xffffffffu, x.y, o),
          x.z += __shfl_xor_sync(0xffffffffu, x.z, o);
    excl.x += x.x, excl.y += x.y, excl.z += x.z;
    if (incl) break;
  }
  if (lane == 0 && tile > 0) {
    st_volatile_i3(ss.incl + tile, make_int3(excl.x + agg.x, excl.y + agg.y, excl.z + agg.z));
    __threadfence();
    atomicExch(ss.flag + tile, 2);
  }
  return excl;
}

__global__ void __launch_bounds__(256) mc_scan_kernel(int3* blk, DevCtl* ctl, ScanState ss, int v_cap, int t_cap,
                                                      int c_cap) {
  __shared__ int tile_s;
  __shared__ int3 wsum[8];
  __shared__ int3 base_s;
  const int n = ctl->status == 0 ? ctl->units : 0;
  const int ntiles = (n + 1023) / 1024;
  if (threadIdx.x == 0) tile_s = atomicAdd(ss.counter, 1);
  __syncthreads();
  const int tile = tile_s;
  if (n == 0) {  // no unit: the totals are zero
    if (tile == 0 && threadIdx.x == 0) ctl->V = 0, ctl->T = 0, ctl->C = 0, ctl->overflow = 0;
    return;
  }
  if (tile >= ntiles) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int i0 = tile * 1024 + (int)threadIdx.x * 4;
  int3 v[4];
  if (i0 + 4 <= n) {  // blk is 256 B aligned and i0 a multiple of 4: 48 B = three int4
    const int4* q = reinterpret_cast<const int4*>(blk + i0);
    const int4 a = q[0], b = q[1], c = q[2];
    v[0] = make_int3(a.x, a.y, a.z), v[1] = make_int3(a.w, b.x, b.y);
    v[2] = make_int3(b.z, b.w, c.x), v[3] = make_int3(c.y, c.z, c.w);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = i0 + i < n ? blk[i0 + i] : make_int3(0, 0, 0);
  }
  int3 tot = make_int3(0, 0, 0);
#pragma unroll
  for (int i = 0; i < 4; ++i) tot.x += v[i].x, tot.y += v[i].y, tot.z += v[i].z;
  int3 inc = tot;
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, inc.x, o), b = __shfl_up_sync(0xffffffffu, inc.y, o),
              c = __shfl_up_sync(0xffffffffu, inc.z, o);
    if (lane >= o) inc.x += a, inc.y += b, inc.z += c;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int3 w = lane < 8 ? wsum[lane] : make_int3(0, 0, 0);
    for (int o = 1; o < 8; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, w.x, o), b = __shfl_up_sync(0xffffffffu, w.y, o),
                c = __shfl_up_sync(0xffffffffu, w.z, o);
      if (lane >= o) w.x += a, w.y += b, w.z += c;
    }
    const int3 agg = make_int3(__shfl_sync(0xffffffffu, w.x, 7), __shfl_sync(0xffffffffu, w.y, 7),
                               __shfl_sync(0xffffffffu, w.z, 7));
    if (lane < 8) wsum[lane] = w;  // inclusive over the tile's warps
    const int3 excl = lookback_publish(ss, tile, agg, lane);
    if (lane == 0) {
      const int3 total = make_int3(excl.x + agg.x, excl.y + agg.y, excl.z + agg.z);
      base_s = excl;
      if (tile == ntiles - 1) {
        ctl->V = total.x - ctl->v_extra, ctl->T = total.y, ctl->C = total.z;
        ctl->overflow = (total.x > v_cap || total.y > t_cap || total.z > c_cap) ? 1 : 0;
      }
    }
  }
  __syncthreads();
  const int3 wp = wid ? wsum[wid - 1] : make_int3(0, 0, 0);
  int3 run = make_int3(base_s.x + wp.x + inc.x - tot.x, base_s.y + wp.y + inc.y - tot.y, base_s.z + wp.z + inc.z - tot.z);
  int3 o[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) o[i] = run, run.x += v[i].x, run.y += v[i].y, run.z += v[i].z;
  if (i0 + 4 <= n) {
    int4* q = reinterpret_cast<int4*>(blk + i0);
    q[0] = make_int4(o[0].x, o[0].y, o[0].z, o[1].x);
    q[1] = make_int4(o[1].y, o[1].z, o[2].x, o[2].y);
    q[2] = make_int4(o[2].z, o[3].x, o[3].y, o[3].z);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i0 + i < n) blk[i0 + i] = o[i];
  }
}

// per active unit (one warp, 8 voxels per lane per pass), in order: vertex
// ids = rank of the cut edge in global edge id order (x ascending, then
// axis); fp64 positions (marching_cubes.cpp:153-155, volume.hpp:45)
// One unit's vertices, cut-edge bases and cells from its cache entries
// `info` and straddling-chunk mask; `carry` = the unit's first (vertex,
// triangle, cell) ids.
__device__ __forceinline__ void emit_unit(const float* __restrict__ A, int nx, int ny, int y, int z, bool own,
                                          double L, const DevGrid& g, int lane, const uint16_t* info, uint32_t cmask,
                                          int3 carry, const MeshBufs& mb) {
  const size_t step[3] = {1, (size_t)nx, (size_t)nx * ny};
  const size_t row0 = ((size_t)z * ny + y) * nx;
  // the unit's straddling 32-voxel chunks in x order, one voxel per lane
  for (uint32_t mm = cmask; mm; mm &= mm - 1) {
    const int x = ((__ffs(mm) - 1) << 5) + lane;
    const uint16_t inf = x < nx ? info[x] : (uint16_t)0;
    const int mask = inf & 7;
    const bool cell = (inf >> 11) & 1;
    const int cfg = (inf >> 3) & 255;
    const int nt = cell ? mc_count(cfg) : 0;
    const int3 cnt = make_int3(__popc(mask), nt, cell ? 1 : 0);
    int3 inc = cnt;  // warp inclusive scan
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, inc.x, o), b = __shfl_up_sync(0xffffffffu, inc.y, o),
                c = __shfl_up_sync(0xffffffffu, inc.z, o);
      if (lane >= o) inc.x += a, inc.y += b, inc.z += c;
    }
    const int vb = carry.x + inc.x - cnt.x, tb = carry.y + inc.y - cnt.y, cb = carry.z + inc.z - cnt.z;
    carry.x += __shfl_sync(0xffffffffu, inc.x, 31), carry.y += __shfl_sync(0xffffffffu, inc.y, 31),
        carry.z += __shfl_sync(0xffffffffu, inc.z, 31);
    if (!mask && !cell) continue;
    const size_t v = row0 + x;
    if (mask) {
      mb.vbase[v] = ((uint32_t)vb << 3) | (uint32_t)mask;
      if (own) {
        const double v0 = (double)__ldg(A + v);
        int id = vb;
        for (int a = 0; a < 3; ++a) {
          if (!(mask & (1 << a))) continue;
          const double v1 = (double)__ldg(A + v + step[a]);
          double t = ddiv(dsub(L, v0), dsub(v1, v0));
          t = t < 1e-6 ? 1e-6 : (t > 1.0 - 1e-6 ? 1.0 - 1e-6 : t);
          double p[3] = {(double)x, (double)y, (double)z};
          p[a] = dadd(p[a], t);
          for (int cc = 0; cc < 3; ++cc) mb.pos[3 * (size_t)id + cc] = dadd(g.origin[cc], dmul(g.edge, p[cc]));
          mb.edge_id[id] = (uint64_t)v * 3 + a;
          ++id;
        }
      }
    }
    if (cell) {
      mb.cells[cb] = (int32_t)v;
      mb.cell_tri[cb] = tb;
      mb.cell_cfg[cb] = (uint8_t)cfg;
    }
  }
}

__global__ void __launch_bounds__(256, 4) mc_emit_kernel(const float* __restrict__ A, const DevCtl* ctl, int nx, int ny,
                                                         int nz, McSlab sl, const int32_t* __restrict__ units,
                                                         const int3* __restrict__ unitoff, MeshBufs mb) {
  if (ctl->status != 0 || ctl->overflow) return;
  const int U = ctl->units;
  const double L = ctl->level;
  const DevGrid g = ctl->grid;
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < U; i += warps) {
    const int u = units[i];
    const int y = u % ny, z = sl.z0 + u / ny;
    emit_unit(A, nx, ny, y, z, z < sl.zend, L, g, lane, mb.vinfo + (size_t)i * nx, mb.ucmask[i], unitoff[i], mb);
  }
}


// Scan + emit in one pass over tiles of kFuseUnits counted units (one warp
// per unit; CTAs stride over the tiles).  A tile's first (vertex, triangle, cell) ids are the counts of
// every unit before it: the count pass also summed the units into blocks of
// kCntBlock (bsum), so warp 0 adds the blocks before the tile's block and the
// units of its block before the tile — no tile waits on another (a look-back
// over ~10^3 simultaneously started tiles costs one L2 round trip per 32
// tiles).  Reads per tile: ceil(i0 / kCntBlock) + i0 % kCntBlock entries.
// The tile holding the last unit forms V, T, C and the overflow flag; a tile
// whose id range passes a capacity writes nothing (the host regrows and
// re-runs).
__global__ void __launch_bounds__(kFuseUnits * 32, 4) mc_scan_emit_kernel(const float* __restrict__ A, DevCtl* ctl,
                                                                          int nx, int ny,
                                                                          const int32_t* __restrict__ units,
                                                                          const int3* __restrict__ unitcnt,
                                                                          const int3* __restrict__ bsum, MeshBufs mb) {
  __shared__ int skip_s;
  __shared__ int3 off_s[kFuseUnits];
  const int n = ctl->status == 0 ? ctl->units : 0;
  if (n == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->V = 0, ctl->T = 0, ctl->C = 0, ctl->overflow = 0;
    return;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double L = ctl->level;
  const DevGrid g = ctl->grid;
  for (int i0 = blockIdx.x * kFuseUnits; i0 < n; i0 += gridDim.x * kFuseUnits) {
    const int i = i0 + wid;
    if (wid == 0) {
      int3 e = make_int3(0, 0, 0);
      const int b = i0 / kCntBlock;
      for (int j = lane; j < b; j += 32) {
        const int3 q = bsum[j];
        e.x += q.x, e.y += q.y, e.z += q.z;
      }
      for (int j = b * kCntBlock + lane; j < i0; j += 32) {
        const int3 q = unitcnt[j];
        e.x += q.x, e.y += q.y, e.z += q.z;
      }
      const int3 excl = warp_sum3(e);
      const int j = i0 + lane;
      int3 w = lane < kFuseUnits && j < n ? unitcnt[j] : make_int3(0, 0, 0);
      const int3 own = w;
      for (int o = 1; o < kFuseUnits; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, w.x, o), y = __shfl_up_sync(0xffffffffu, w.y, o),
                  z = __shfl_up_sync(0xffffffffu, w.z, o);
        if (lane >= o) w.x += x, w.y += y, w.z += z;
      }
      const int3 end = make_int3(excl.x + __shfl_sync(0xffffffffu, w.x, kFuseUnits - 1),
                                 excl.y + __shfl_sync(0xffffffffu, w.y, kFuseUnits - 1),
                                 excl.z + __shfl_sync(0xffffffffu, w.z, kFuseUnits - 1));
      const bool over = end.x > mb.v_cap || end.y > mb.t_cap || end.z > mb.c_cap;
      if (lane < kFuseUnits)
        off_s[lane] = make_int3(excl.x + w.x - own.x, excl.y + w.y - own.y, excl.z + w.z - own.z);
      if (lane == 0) {
        skip_s = over;
        if (i0 + kFuseUnits >= n) ctl->V = end.x, ctl->T = end.y, ctl->C = end.z, ctl->overflow = over ? 1 : 0;
      }
    }
    __syncthreads();
    if (i < n && !skip_s) {
      const int u = units[i];
      emit_unit(A, nx, ny, u % ny, u / ny, true, L, g, lane, mb.vinfo + (size_t)i * nx, mb.ucmask[i], off_s[wid], mb);
    }
    __syncthreads();  // off_s / skip_s are rewritten by the next tile
  }
}

// marching_cubes.cpp:178-207: outward normal = -normalize(trilinear blend of
// central-difference gradients at the 8 surrounding nodes, clamped borders)
__device__ void vertex_normal(const float* A, int nx, int ny, int nz, double px, double py, double pz, float* out) {
  auto val = [&](int x, int y, int z) {
    x = x < 0 ? 0 : (x > nx - 1 ? nx - 1 : x);
    y = y < 0 ? 0 : (y > ny - 1 ? ny - 1 : y);
    z = z < 0 ? 0 : (z > nz - 1 ? nz - 1 : z);
    return (double)vol_at(A, nx, ny, x, y, z);
  };
  const int x0 = max(0, min((int)px, nx - 2)), y0 = max(0, min((int)py, ny - 2)), z0 = max(0, min((int)pz, nz - 2));
  const double tx = dsub(px, (double)x0), ty = dsub(py, (double)y0), tz = dsub(pz, (double)z0);
  double gx = 0, gy = 0, gz = 0;
#pragma unroll
  for (int dz = 0; dz <= 1; ++dz)
#pragma unroll
    for (int dy = 0; dy <= 1; ++dy)
#pragma unroll
      for (int dx = 0; dx <= 1; ++dx) {
        const double w = dmul(dmul(dx ? tx : dsub(1.0, tx), dy ? ty : dsub(1.0, ty)), dz ? tz : dsub(1.0, tz));
        if (w > 0) {
          const int x = x0 + dx, y = y0 + dy, z = z0 + dz;
          const double g0 = dmul(dsub(val(x + 1, y, z), val(x - 1, y, z)), 0.5);
          const double g1 = dmul(dsub(val(x, y + 1, z), val(x, y - 1, z)), 0.5);
          const double g2 = dmul(dsub(val(x, y, z + 1), val(x, y, z - 1)), 0.5);
          gx = dadd(gx, dmul(w, g0)), gy = dadd(gy, dmul(w, g1)), gz = dadd(gz, dmul(w, g2));
        }
      }
  const double len = norm3(mk3(gx, gy, gz));
  if (len > 1e-12) {
    out[0] = (float)ddiv(-gx, len), out[1] = (float)ddiv(-gy, len), out[2] = (float)ddiv(-gz, len);
  } else {
    out[0] = 0.f, out[1] = 0.f, out[2] = 1.f;
  }
}

// marching_cubes.cpp:178-207 normal of vertex i (fp64)
__device__ __forceinline__ void normal_of(const float* __restrict__ A, int nx, int ny, int nz, double L,
                                          const MeshBufs& mb, int i) {
  const uint64_t e = mb.edge_id[i];
  const size_t v = (size_t)(e / 3);
  const int a = (int)(e % 3);
  const int x = (int)(v % nx), y = (int)((v / nx) % ny), z = (int)(v / ((size_t)nx * ny));
  const size_t step = a == 0 ? 1 : (a == 1 ? (size_t)nx : (size_t)nx * ny);
  const double v0 = (double)__ldg(A + v), v1 = (double)__ldg(A + v + step);
  double t = ddiv(dsub(L, v0), dsub(v1, v0));
  t = t < 1e-6 ? 1e-6 : (t > 1.0 - 1e-6 ? 1.0 - 1e-6 : t);
  double p[3] = {(double)x, (double)y, (double)z};
  p[a] = dadd(p[a], t);
  vertex_normal(A, nx, ny, nz, p[0], p[1], p[2], mb.nrm + 3 * (size_t)i);
}

// the triangles of non-trivial cell i: vertex ids from the cut-edge bases
// (marching_cubes.cpp:163-175)
__device__ __forceinline__ void tris_of(int nx, int ny, int voff, const MeshBufs& mb, int i) {
  const size_t plane = (size_t)nx * ny;
  const size_t v = (size_t)mb.cells[i];
  const int tb = mb.cell_tri[i];
  const int cfg = mb.cell_cfg[i];
  const int n = mc_count(cfg);
  for (int tri = 0; tri < n; ++tri) {
    int ids[3];
    for (int m = 0; m < 3; ++m) {
      const int e = mc_tri_edge(cfg, tri, m);
      const int c0 = edge_c0(e), axis = edge_axis(e);
      const size_t owner = v + (c0 & 1) + ((c0 >> 1) & 1) * (size_t)nx + ((c0 >> 2) & 1) * plane;
      const uint32_t pk = mb.vbase[owner];
      ids[m] = voff + (int)(pk >> 3) + __popc(pk & 7u & ((1u << axis) - 1u));
    }
    int32_t* o = mb.tri + 3 * (size_t)(tb + tri);
    o[0] = ids[0], o[1] = ids[1], o[2] = ids[2];
  }
}

// normals and triangles in one launch: items [0, V) are vertices, [V, V + C) cells
__global__ void __launch_bounds__(256, 4) mc_finish_kernel(const float* __restrict__ A, const DevCtl* ctl, int nx, int ny,
                                                        int nz, MeshBufs mb) {
  if (ctl->status != 0 || ctl->overflow) return;
  const int V = ctl->V, C = ctl->C, voff = ctl->voff;
  const double L = ctl->level;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < V + C; i += gridDim.x * blockDim.x) {
    if (i < V)
      normal_of(A, nx, ny, nz, L, mb, i);
    else
      tris_of(nx, ny, voff, mb, i - V);
  }
}

// slab ranks: this rank's first global vertex id = sum of the vertex counts
// of the ranks below it (counts: (V, T, C) per rank, all-gathered)
__global__ void mc_set_voff_kernel(const int3* counts, int rank, DevCtl* ctl) {
  int s = 0;
  for (int r = 0; r < rank; ++r) s += counts[r].x;
  ctl->voff = s;
}

__global__ void add_f64_kernel(double* dst, const double* src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = dadd(dst[i], src[i]);
}

}  // namespace

void launch_add_f64(double* dst, const double* src, size_t n, cudaStream_t st) {
  add_f64_kernel<<<sm_count() * 4, 256, 0, st>>>(dst, src, n);
}

void launch_mc_set_voff(const int32_t* counts, int rank, DevCtl* ctl, cudaStream_t st) {
  mc_set_voff_kernel<<<1, 1, 0, st>>>(reinterpret_cast<const int3*>(counts), rank, ctl);
}

void upload_case_table_data(const int8_t* counts, const int8_t* tris, cudaStream_t st) {
  cudaMemcpyToSymbolAsync(g_mc_count, counts, 256, 0, cudaMemcpyHostToDevice, st);
  cudaMemcpyToSymbolAsync(g_mc_tris, tris, 256 * 15, 0, cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);
}

int iso_blocks() { return kIsoBlocks; }

void launch_iso_level(const DevPoints& pts, const float* A, DevCtl* ctl, double* partial, int, cudaStream_t st) {
  iso_partial_kernel<<<kIsoBlocks, 256, 0, st>>>(pts.pos, A, ctl, partial);
}

int mc_blocks(int nx, int ny, int nz) {  // per-unit / per-block scratch entries
  const int units = ny * nz;
  return units + (units + kRowThreads - 1) / kRowThreads + 64;
}

void launch_row_minmax(const float* A, int nx, int ny, int nz, float2* rowmm, cudaStream_t st) {
  const int rows = ny * nz;
  row_minmax_kernel<<<(rows * 32 + 255) / 256, 256, 0, st>>>(A, nx, rows, rowmm);
}

namespace {
// mb.blk layout: the active-unit pass's look-back descriptors (one u64 per
// 256-unit tile) and ticket counter, the count pass's block sums (one int3
// per kCntBlock units), then the split scan's ScanState over 1024-unit tiles
// (ticket counter, 3 pad ints, flags, aggregates, inclusive prefixes).  The
// block sums and the scan's counter and flags start each frame at zero.
struct McScratch {
  unsigned long long* desc;
  int* tile_counter;
  int3* bsum;
  ScanState ss;
  int nzero;  // ints from bsum that start each frame at zero
};
McScratch mc_scratch(const MeshBufs& mb, int units) {
  const int nblk = (units + kRowThreads - 1) / kRowThreads;
  const int nbs = (units + kCntBlock - 1) / kCntBlock;
  const int stiles = (units + 1023) / 1024;
  McScratch m;
  m.desc = reinterpret_cast<unsigned long long*>(mb.blk);
  m.tile_counter = reinterpret_cast<int*>(m.desc + nblk);
  m.bsum = reinterpret_cast<int3*>(m.tile_counter + 4);
  m.ss.counter = reinterpret_cast<int*>(m.bsum + nbs);
  m.ss.flag = m.ss.counter + 4;
  m.ss.agg = reinterpret_cast<int3*>(m.ss.flag + stiles);
  m.ss.incl = m.ss.agg + stiles;
  m.nzero = 3 * nbs + 4 + stiles;
  return m;
}

void launch_select(const MeshBufs& mb, const McScratch& m, DevCtl* ctl, int ny, int nz, McSlab sl, cudaStream_t st) {
  const int units = ny * sl.nzu;
  const int nblk = (units + kRowThreads - 1) / kRowThreads;
  cudaMemsetAsync(m.desc, 0, (size_t)nblk * 8 + 16, st);
  mc_select_kernel<<<nblk, kRowThreads, 0, st>>>(mb.rowmm, ctl, ny, nz, sl, m.desc, m.tile_counter, mb.units,
                                                 reinterpret_cast<int*>(m.bsum), m.nzero);
}
}  // namespace

void launch_marching_cubes_count(const float* A, DevCtl* ctl, MeshBufs mb, int nx, int ny, int nz, McSlab sl,
                                 cudaStream_t st) {
  const int units = ny * sl.nzu;
  const McScratch m = mc_scratch(mb, units);
  int3* ucnt = reinterpret_cast<int3*>(mb.unitcnt);
  launch_select(mb, m, ctl, ny, nz, sl, st);
  mc_count_kernel<<<sm_count() * 8, 256, 0, st>>>(A, ctl, nx, ny, nz, sl, mb.units, ucnt, nullptr, mb);
  mc_scan_kernel<<<(units + 1023) / 1024, 256, 0, st>>>(ucnt, ctl, m.ss, mb.v_cap, mb.t_cap, mb.c_cap);
}

void launch_marching_cubes_emit(const float* A, DevCtl* ctl, MeshBufs mb, int nx, int ny, int nz, McSlab sl,
                                cudaStream_t st) {
  int3* ucnt = reinterpret_cast<int3*>(mb.unitcnt);
  mc_emit_kernel<<<sm_count() * 8, 256, 0, st>>>(A, ctl, nx, ny, nz, sl, mb.units, ucnt, mb);
  mc_finish_kernel<<<sm_count() * 4, 256, 0, st>>>(A, ctl, nx, ny, nz, mb);
}

// whole volume: active units, the fused count/scan/emit pass, normals + triangles
void launch_marching_cubes(const float* A, DevCtl* ctl, MeshBufs mb, int nx, int ny, int nz, cudaStream_t st,
                           cudaStream_t aux, cudaEvent_t fork, cudaEvent_t join) {
  const McSlab whole{0, nz, nz};
  const int units = ny * nz;
  const McScratch m = mc_scratch(mb, units);
  int3* ucnt = reinterpret_cast<int3*>(mb.unitcnt);
  launch_select(mb, m, ctl, ny, nz, whole, st);
  static const bool split = [] {  // VC_MC_SPLIT=1 (A/B): count, 1024-unit look-back scan, emit
    const char* e = getenv("VC_MC_SPLIT");
    return e && atoi(e) != 0;
  }();
  if (split) {
    mc_count_kernel<<<sm_count() * 8, 256, 0, st>>>(A, ctl, nx, ny, nz, whole, mb.units, ucnt, nullptr, mb);
    mc_scan_kernel<<<(units + 1023) / 1024, 256, 0, st>>>(ucnt, ctl, m.ss, mb.v_cap, mb.t_cap, mb.c_cap);
    mc_emit_kernel<<<sm_count() * 8, 256, 0, st>>>(A, ctl, nx, ny, nz, whole, mb.units, ucnt, mb);
  } else {
    mc_count_kernel<<<sm_count() * 8, 256, 0, st>>>(A, ctl, nx, ny, nz, whole, mb.units, ucnt, m.bsum, mb);
    mc_scan_emit_kernel<<<sm_count() * 8, kFuseUnits * 32, 0, st>>>(A, ctl, nx, ny, mb.units, ucnt, m.bsum, mb);
  }
  if (aux) {
    cudaEventRecord(fork, st);
    cudaStreamWaitEvent(aux, fork, 0);
    mc_finish_kernel<<<sm_count() * 4, 256, 0, aux>>>(A, ctl, nx, ny, nz, mb);
    cudaEventRecord(join, aux);
  } else {
    mc_finish_kernel<<<sm_count() * 4, 256, 0, st>>>(A, ctl, nx, ny, nz, mb);
  }
}

void launch_iso_samples(const DevPoints& pts, const float* A, const DevCtl* ctl, int zoff, int nzl, double* samples,
                        cudaStream_t st) {
  iso_sample_kernel<<<sm_count() * 4, 256, 0, st>>>(pts.pos, A, ctl, zoff, nzl, samples);
}

void launch_iso_final_samples(const double* samples, DevCtl* ctl, double* partial, cudaStream_t st) {
  iso_partial_samples_kernel<<<kIsoBlocks, 256, 0, st>>>(samples, ctl, partial);
  iso_final_kernel<<<1, 256, 0, st>>>(partial, kIsoBlocks, ctl);
}

}  // namespace vc

// SPDX-License-Identifier: Apache-2.0
//
// K3 — oriented-point splatting on sm_100a (splat.cpp:11-89).
//
// The reference makes two passes (density d, then sum g1*(W/d)*N) over
// z-slabs.  Since d(q) is final during its second pass, that equals
//   V(q) = (sum_p g1*W*N) / d(q) = sqrt(1.5) * U'(q) / d'(q)
// with U' = sum exp(-s/0.75)*W*N and d' = sum exp(-s/1.125)*W, s the squared
// point-voxel distance in voxel units (sigma1^2 = 0.75 e^2, sigma2^2 =
// 1.125 e^2), and the density threshold d >= 1e-6 g(0;sigma2) <=> d' >= 1e-6.
// So ONE scatter pass accumulates float4 (U'x, U'y, U'z, d') per voxel with a
// vector L2 reduction (red.global.add.v4.f32); the division, threshold and
// the negation of reconstruct.cpp:71 are fused into the FFT's first pass.
//
// Binning is bit-exact: to_voxel (volume.hpp:44) and floor/lround are fp64
// with the reference's operation order.
//
// Sparsity: the splat touches only a thin shell of the grid (~5% of 256^3).
// Every scatter also sets the bit of its 32-voxel x-chunk in a per-row mask
// (rowbits[(z*ny+y)], bit = x/32) with fire-and-forget reductions; a pass
// after the splat lists the touched rows compactly.  The next frame's clear zeroes only the chunks of the
// listed rows, and the FFT's first pass works through the list, loading only
// the marked chunks.
#include "vc_device.cuh"

namespace vc {
namespace {

constexpr int kSplatThreads = 256;

__global__ void __launch_bounds__(256) clear_kernel(float4* acc, size_t n) {
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    acc[i] = z;
}

// Zero the chunks the previous frame touched and reset their bits (one warp
// per row, 32 lanes x float4 = one 512 B chunk per store instruction).
__global__ void __launch_bounds__(256) sparse_clear_kernel(float4* acc, uint32_t* rowbits,
                                                           const int32_t* __restrict__ rowlist, int nx) {
  const int lane = threadIdx.x & 31;
  const int chunk = nx < 32 ? nx : 32;
  const int n = rowlist[0];
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += (gridDim.x * blockDim.x) >> 5) {
    const int r = rowlist[1 + i];
    uint32_t bits = rowbits[r];
    if (!bits) continue;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    while (bits) {
      const int c = __ffs(bits) - 1;
      bits &= bits - 1;
      if (lane < chunk) acc[(size_t)r * nx + c * chunk + lane] = z;
    }
    __syncwarp();
    if (lane == 0) rowbits[r] = 0u;
  }
}

// chunk bits x0/32 .. x1/32 of a row (a reduction: nothing waits for it; the
// touched-row list is built from the bits after the splat)
__device__ __forceinline__ void mark_chunks(uint32_t* rowbits, int row, int x0, int x1) {
  const uint32_t m = (0xffffffffu >> (31 - (x1 >> 5))) & (0xffffffffu << (x0 >> 5));
  atomicOr(rowbits + row, m);
}

// Touched-row list [count, rows...] from the chunk bits (warp-aggregated appends; any order)
__global__ void __launch_bounds__(256) rowlist_build_kernel(const uint32_t* __restrict__ rowbits,
                                                            const DevCtl* __restrict__ ctl, int nzl,
                                                            int32_t* __restrict__ rowlist) {
  if (ctl->status != 0) return;
  const int rows = ctl->grid.ny * nzl;
  const int lane = threadIdx.x & 31;
  const int wstride = gridDim.x * blockDim.x;
  for (int r0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; r0 < rows; r0 += wstride) {
    const int r = r0 + lane;
    const bool touched = r < rows && __ldg(rowbits + r) != 0u;
    const unsigned ball = __ballot_sync(0xffffffffu, touched);
    if (!ball) continue;
    int base = 0;
    if (lane == 0) base = atomicAdd(rowlist, __popc(ball));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (touched) rowlist[1 + base + __popc(ball & ((1u << lane) - 1u))] = r;
  }
}

__device__ __forceinline__ void red_add_v4(float4* addr, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// splat.cpp:58-87 weighted mode: one warp per point, two support voxels per
// lane (the 4x4x4 support floor(c)-1 .. floor(c)+2 per axis, support_around,
// splat.cpp:19-29: lane = (ox, oy, oz) with oz and oz + 2), so the per-point
// work — the next point's loads, the three fp64 to_voxel divisions (lanes 0-2,
// bit-exact) and their shuffles — is done once per 64 voxel updates.  Each warp
// walks a contiguous run of points (neighbouring pixels, so mostly the same
// voxel rows): a row's chunk bits are or-ed in only when they add to what this
// lane marked for the previous point, which removes most of the row-mask
// atomics; the reductions are issued before the marking.
__global__ void __launch_bounds__(kSplatThreads) splat_weighted_kernel(const double* __restrict__ pos,
                                                                       const double* __restrict__ nrm,
                                                                       const double* __restrict__ wgt,
                                                                       const DevCtl* __restrict__ ctl,
                                                                       float4* __restrict__ acc,
                                                                       uint32_t* __restrict__ rowbits, int zoff,
                                                                       int nzl) {
  const int P = ctl->P;
  if (ctl->status != 0) return;
  const DevGrid g = ctl->grid;
  const int lane = threadIdx.x & 31;
  const int ox = lane & 3, oy = (lane >> 2) & 3, oz = lane >> 4;  // second voxel: oz + 2
  // exp(-s/0.75) = exp2(s * k1), exp(-s/1.125) = exp2(s * k2)
  const float k1 = -1.4426950408889634f / 0.75f, k2 = -1.4426950408889634f / 1.125f;
  const int groups = gridDim.x * (kSplatThreads / 32);
  const int run = (P + groups - 1) / groups;
  const int p0 = (blockIdx.x * (kSplatThreads / 32) + (threadIdx.x >> 5)) * run;
  const int p1 = min(P, p0 + run);
  int last_row[2] = {-1, -1};
  uint32_t last_m[2] = {0u, 0u};
  const double o = lane == 0 ? g.origin[0] : (lane == 1 ? g.origin[1] : g.origin[2]);
  // the next point's inputs are loaded while the current one is scattered
  auto load = [&](int q, double& pc, float4& nw) {
    pc = lane < 3 ? __ldg(pos + 3 * q + lane) : 0.0;
    nw = make_float4((float)__ldg(nrm + 3 * q + 0), (float)__ldg(nrm + 3 * q + 1), (float)__ldg(nrm + 3 * q + 2),
                     (float)__ldg(wgt + q));
  };
  double pc_n = 0.0;
  float4 nw_n = make_float4(0.f, 0.f, 0.f, 0.f);
  if (p0 < p1) load(p0, pc_n, nw_n);
  for (int p = p0; p < p1; ++p) {
    const double pc = pc_n;
    const float4 nw = nw_n;
    if (p + 1 < p1) load(p + 1, pc_n, nw_n);
    // to_voxel (volume.hpp:44) once per warp: lanes 0-2 divide one coordinate
    // each (IEEE fp64, bit-exact), the warp shares them by shuffle
    const double c = lane < 3 ? ddiv(dsub(pc, o), g.edge) : 0.0;
    const double cx = __shfl_sync(0xffffffffu, c, 0), cy = __shfl_sync(0xffffffffu, c, 1),
                 cz = __shfl_sync(0xffffffffu, c, 2);
    const int fx = (int)floor(cx), fy = (int)floor(cy), fz = (int)floor(cz);
    const int x = fx - 1 + ox, y = fy - 1 + oy;
    const float dx = (float)(cx - (double)x), dy = (float)(cy - (double)y);
    const float sxy = dx * dx + dy * dy;
    // the usual case (the grid is padded): the whole 4x4x4 support inside the
    // grid and this rank's slab — one warp-uniform test instead of per-voxel
    // bounds tests and clamps, one base address for both voxels of the lane
    if (fx >= 1 && fy >= 1 && fx + 2 < g.nx && fy + 2 < g.ny && fz - 1 >= zoff && fz + 2 < zoff + nzl) {
      const int zl0 = fz - 1 + oz - zoff;
      const size_t two_planes = 2 * (size_t)g.ny * g.nx;
      float4* pa = acc + ((size_t)zl0 * g.ny + y) * g.nx + x;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float dz = (float)(cz - (double)(fz - 1 + oz + 2 * h));
        const float s = sxy + dz * dz;
        const float g1w = exp2f(s * k1) * nw.w, g2w = exp2f(s * k2) * nw.w;
        red_add_v4(pa + h * two_planes, make_float4(g1w * nw.x, g1w * nw.y, g1w * nw.z, g2w));
      }
      if (ox == 0) {
        const uint32_t m = (0xffffffffu >> (31 - ((fx + 2) >> 5))) & (0xffffffffu << ((fx - 1) >> 5));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = (zl0 + 2 * h) * g.ny + y;
          if (row != last_row[h] || (m & ~last_m[h]) != 0u) {
            atomicOr(rowbits + row, m);
            last_m[h] = row == last_row[h] ? (last_m[h] | m) : m;
            last_row[h] = row;
          }
        }
      }
      continue;
    }
    const bool inxy = x >= 0 && y >= 0 && x < g.nx && y < g.ny;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int z = (int)floor(cz) - 1 + oz + 2 * h;
      // z-slab [zoff, zoff+nzl) of this rank (the reference's own slab split, splat.cpp:61-77)
      const int zl = z - zoff;
      if (inxy && zl >= 0 && zl < nzl && z < g.nz) {
        const float dz = (float)(cz - (double)z);
        const float s = sxy + dz * dz;
        const float g1w = exp2f(s * k1) * nw.w, g2w = exp2f(s * k2) * nw.w;
        red_add_v4(acc + ((size_t)zl * g.ny + y) * g.nx + x, make_float4(g1w * nw.x, g1w * nw.y, g1w * nw.z, g2w));
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int z = (int)floor(cz) - 1 + oz + 2 * h;
      const int zl = z - zoff;
      if (ox == 0 && y >= 0 && zl >= 0 && y < g.ny && zl < nzl && z < g.nz && fx + 2 >= 0 && fx - 1 < g.nx) {
        const int row = zl * g.ny + y;
        const int xa = max(fx - 1, 0), xb = min(fx + 2, g.nx - 1);
        const uint32_t m = (0xffffffffu >> (31 - (xb >> 5))) & (0xffffffffu << (xa >> 5));
        if (row != last_row[h] || (m & ~last_m[h]) != 0u) {
          atomicOr(rowbits + row, m);
          last_m[h] = row == last_row[h] ? (last_m[h] | m) : m;
          last_row[h] = row;
        }
      }
    }
  }
}

// splat.cpp:40-56 simple mode: lround nearest voxel, (sum N, count)
__global__ void __launch_bounds__(256) splat_simple_kernel(const double* __restrict__ pos,
                                                           const double* __restrict__ nrm,
                                                           const DevCtl* __restrict__ ctl, float4* __restrict__ acc,
                                                           uint32_t* __restrict__ rowbits, int zoff, int nzl) {
  const int P = ctl->P;
  if (ctl->status != 0) return;
  const DevGrid g = ctl->grid;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
    const double cx = ddiv(dsub(pos[3 * p + 0], g.origin[0]), g.edge);
    const double cy = ddiv(dsub(pos[3 * p + 1], g.origin[1]), g.edge);
    const double cz = ddiv(dsub(pos[3 * p + 2], g.origin[2]), g.edge);
    const long long x = lround_d(cx), y = lround_d(cy), z = lround_d(cz);
    if (!(x >= 0 && x < g.nx && y >= 0 && y < g.ny && z >= 0 && z < g.nz)) continue;
    const long long zl = z - zoff;
    if (zl < 0 || zl >= nzl) continue;
    mark_chunks(rowbits, (int)(zl * g.ny + y), (int)x, (int)x);
    red_add_v4(acc + ((size_t)zl * g.ny + y) * g.nx + x,
               make_float4((float)nrm[3 * p + 0], (float)nrm[3 * p + 1], (float)nrm[3 * p + 2], 1.f));
  }
}

// Stage API only: the reference's GradientField view of the accumulator.
__global__ void splat_finalize_kernel(const float4* acc, size_t n, int mode, int negate, double sigma2,
                                      float* field, float* density) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float4 a = acc[i];
    float s = 0.f, d;
    if (mode == 0) {
      if (a.w >= 1e-6f) s = 1.2247448713915890f / a.w;
      d = (float)((double)a.w / sigma2);
    } else {
      if (a.w > 0.f) s = 1.f / a.w;
      d = a.w;
    }
    if (negate) s = -s;
    field[3 * i + 0] = a.x * s;
    field[3 * i + 1] = a.y * s;
    field[3 * i + 2] = a.z * s;
    density[i] = d;
  }
}

// the touched-row list's count, reset at the start of a frame
__global__ void reset_count_kernel(int32_t* count) { *count = 0; }

}  // namespace

void launch_reset_rowlist(int32_t* rowlist, cudaStream_t st) { reset_count_kernel<<<1, 1, 0, st>>>(rowlist); }

void launch_clear(float4* acc, size_t n, cudaStream_t st) {
  clear_kernel<<<sm_count() * 8, 256, 0, st>>>(acc, n);
}

void launch_sparse_clear(float4* acc, uint32_t* rowbits, const int32_t* rowlist, int nx, cudaStream_t st) {
  sparse_clear_kernel<<<sm_count() * 4, 256, 0, st>>>(acc, rowbits, rowlist, nx);
}

void launch_splat(const DevPoints& pts, DevCtl* ctl, float4* acc, uint32_t* rowbits, int32_t* rowlist, int mode,
                  cudaStream_t st, int zoff, int nzl) {
  if (mode == 0)
    splat_weighted_kernel<<<sm_count() * 8, kSplatThreads, 0, st>>>(pts.pos, pts.nrm, pts.weight, ctl, acc, rowbits, zoff,
                                                             nzl);
  else
    splat_simple_kernel<<<sm_count() * 4, 256, 0, st>>>(pts.pos, pts.nrm, ctl, acc, rowbits, zoff, nzl);
  rowlist_build_kernel<<<sm_count() * 4, 256, 0, st>>>(rowbits, ctl, nzl, rowlist);
}

void launch_splat_finalize(const float4* acc, size_t n, int mode, int negate, double sigma2, float* field,
                           float* density, cudaStream_t st) {
  splat_finalize_kernel<<<sm_count() * 4, 256, 0, st>>>(acc, n, mode, negate, sigma2, field, density);
}

}  // namespace vc

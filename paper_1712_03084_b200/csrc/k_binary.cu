// SPDX-License-Identifier: Apache-2.0
//
// (A, L) consumers on sm_100a: mocap::binarize
// (binary_volume.cpp:10-66) and boundary_voxels (:68-82).
//
//   bin_max      max of A (which side of L is the interior, :12-14)
//   bin_init     mask (v >= L, or v < L), parent[i] = i on the mask
//   bin_union    lock-free union-find over the 13 backward 26-neighbours,
//                linking the larger root under the smaller (atomicMin), so
//                every root is its component's smallest raster index — the
//                voxel at which the reference's raster scan first meets it
//   bin_compress path compression; component sizes at the roots
//   bin_best     largest component, ties to the smallest root (the
//                reference keeps the first component of maximal size, :46-49)
//   bin_rows / bin_emit   keep-mask + voxel list in raster (z, y, x) order
//   bin_boundary voxels with a face neighbour outside the object, in list order
//
// The level test on the fp32 volume uses L rounded up to fp32 (a >= L in fp64
// <=> a >= ru(L) for fp32 a), as in the marching cubes.
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>

#include "vc_device.cuh"

namespace vc {
namespace {

__global__ void bin_reset_kernel(int* maxkey, unsigned long long* best) {
  *maxkey = INT_MIN;  // below the ordered-int key of every finite float
  *best = 0;
}

__global__ void bin_max_kernel(const float* __restrict__ A, size_t n, float* out) {  // out: ordered-int key
  float m = -FLT_MAX;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    m = fmaxf(m, A[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) {
    // float max via ordered int: all values here are finite
    const int bits = __float_as_int(m);
    atomicMax(reinterpret_cast<int*>(out), bits >= 0 ? bits : bits ^ 0x7fffffff);
  }
}

__global__ void bin_init_kernel(const float* __restrict__ A, size_t n, float Lf, const int* __restrict__ maxkey,
                                int32_t* parent, int32_t* size) {
  const int mk = *maxkey;
  const float mx = __int_as_float(mk >= 0 ? mk : mk ^ 0x7fffffff);
  const bool above = mx >= Lf;  // max_val >= level (:12-14)
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const bool in = above ? A[i] >= Lf : A[i] < Lf;  // NaN level: no interior (:17)
    parent[i] = in ? (int32_t)i : -1;
    size[i] = 0;
  }
}

__device__ __forceinline__ int32_t find_root(int32_t* parent, int32_t i) {
  int32_t p = parent[i];
  while (p != i) {
    i = p;
    p = parent[i];
  }
  return i;
}

__device__ void unite(int32_t* parent, int32_t a, int32_t b) {
  while (true) {
    a = find_root(parent, a);
    b = find_root(parent, b);
    if (a == b) return;
    if (a > b) {
      const int32_t t = a;
      a = b, b = t;
    }
    // link the larger root b under a; retry if b stopped being a root
    const int32_t old = atomicMin(parent + b, a);
    if (old == b) return;
    b = old;
  }
}

__global__ void bin_union_kernel(int32_t* parent, int nx, int ny, int nz) {
  const size_t n = (size_t)nx * ny * nz;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    if (parent[i] < 0) continue;
    const int x = (int)(i % nx), y = (int)((i / nx) % ny), z = (int)(i / ((size_t)nx * ny));
    // the 13 neighbours that precede i in raster order
    for (int dz = -1; dz <= 0; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (dz == 0 && (dy > 0 || (dy == 0 && dx >= 0))) continue;
          const int qx = x + dx, qy = y + dy, qz = z + dz;
          if (qx < 0 || qy < 0 || qz < 0 || qx >= nx || qy >= ny) continue;
          const size_t j = ((size_t)qz * ny + qy) * nx + qx;
          if (parent[j] >= 0) unite(parent, (int32_t)i, (int32_t)j);
        }
  }
}

__global__ void bin_compress_kernel(int32_t* parent, int32_t* size, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    if (parent[i] < 0) continue;
    const int32_t r = find_root(parent, (int32_t)i);
    parent[i] = r;
    atomicAdd(size + r, 1);
  }
}

// (size, -root) max over the roots: the largest component, the first in raster order
__global__ void bin_best_kernel(const int32_t* __restrict__ parent, const int32_t* __restrict__ size, size_t n,
                                unsigned long long* best) {
  unsigned long long b = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (parent[i] == (int32_t)i) {
      const unsigned long long k = ((unsigned long long)(uint32_t)size[i] << 32) | (0xffffffffu - (uint32_t)i);
      b = k > b ? k : b;
    }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, b, o);
    b = t > b ? t : b;
  }
  if ((threadIdx.x & 31) == 0 && b) atomicMax(best, b);
}

// per voxel row: kept voxels (row count), the keep mask
__global__ void bin_rows_kernel(const int32_t* __restrict__ parent, const unsigned long long* best, int nx, int rows,
                                uint8_t* keep, int32_t* rowcnt) {
  const int32_t root = (int32_t)(0xffffffffu - (uint32_t)(*best & 0xffffffffull));
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  int c = 0;
  for (int x = lane; x < nx; x += 32) {
    const size_t i = (size_t)warp * nx + x;
    const bool k = *best != 0 && parent[i] == root;
    if (keep) keep[i] = k ? 1 : 0;
    c += k;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) rowcnt[warp] = c;
}

// single CTA exclusive scan of the row counts (in place), total at rowcnt[rows]
__global__ void __launch_bounds__(1024) bin_scan_kernel(int32_t* rowcnt, int rows) {
  __shared__ int wsum[32];
  const int per = (rows + 1023) / 1024;
  const int b0 = min(rows, (int)threadIdx.x * per), b1 = min(rows, b0 + per);
  int tot = 0;
  for (int i = b0; i < b1; ++i) tot += rowcnt[i];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = tot;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int s = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += t;
    }
    wsum[lane] = s;
  }
  __syncthreads();
  int run = (wid ? wsum[wid - 1] : 0) + inc - tot;
  for (int i = b0; i < b1; ++i) {
    const int c = rowcnt[i];
    rowcnt[i] = run, run += c;
  }
  if (threadIdx.x == 1023) rowcnt[rows] = wsum[31];
}

// voxel list (x, y, z) in raster order; one warp per row, ballot compaction
__global__ void bin_emit_kernel(const int32_t* __restrict__ parent, const unsigned long long* best, int nx, int ny,
                                int rows, const int32_t* __restrict__ rowoff, int32_t* voxels, int64_t cap) {
  const int32_t root = (int32_t)(0xffffffffu - (uint32_t)(*best & 0xffffffffull));
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows || *best == 0) return;
  int o = rowoff[warp];
  const int y = warp % ny, z = warp / ny;
  for (int x0 = 0; x0 < nx; x0 += 32) {
    const int x = x0 + lane;
    const bool k = x < nx && parent[(size_t)warp * nx + x] == root;
    const unsigned m = __ballot_sync(0xffffffffu, k);
    if (k) {
      const int64_t at = o + __popc(m & ((1u << lane) - 1u));
      if (at < cap) voxels[3 * at] = x, voxels[3 * at + 1] = y, voxels[3 * at + 2] = z;
    }
    o += __popc(m);
  }
}

// boundary_voxels (:68-82): a face neighbour outside the grid or not kept
__global__ void bin_boundary_flag_kernel(const uint8_t* __restrict__ keep, const int32_t* __restrict__ voxels,
                                         int64_t n, int nx, int ny, int nz, uint8_t* flag) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int x = voxels[3 * v], y = voxels[3 * v + 1], z = voxels[3 * v + 2];
    const int d[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
    bool b = false;
    for (int f = 0; f < 6 && !b; ++f) {
      const int qx = x + d[f][0], qy = y + d[f][1], qz = z + d[f][2];
      b = qx < 0 || qy < 0 || qz < 0 || qx >= nx || qy >= ny || qz >= nz ||
          !keep[((size_t)qz * ny + qy) * nx + qx];
    }
    flag[v] = b ? 1 : 0;
  }
}

// L rounded up to fp32 on the host: fp32 a >= L (fp64) <=> a >= ru(L)
float float_round_up(double L) {
  float f = (float)L;
  if ((double)f < L) f = nextafterf(f, FLT_MAX);
  return f;
}

}  // namespace

void launch_binarize(const float* A, int nx, int ny, int nz, double level, int32_t* parent, int32_t* size,
                     float* maxbuf, unsigned long long* best, uint8_t* keep, int32_t* rowcnt, cudaStream_t st) {
  const size_t n = (size_t)nx * ny * nz;
  const int rows = ny * nz;
  bin_reset_kernel<<<1, 1, 0, st>>>(reinterpret_cast<int*>(maxbuf), best);
  bin_max_kernel<<<sm_count() * 8, 256, 0, st>>>(A, n, maxbuf);
  bin_init_kernel<<<sm_count() * 8, 256, 0, st>>>(A, n, float_round_up(level), reinterpret_cast<const int*>(maxbuf),
                                           parent, size);
  bin_union_kernel<<<sm_count() * 8, 256, 0, st>>>(parent, nx, ny, nz);
  bin_compress_kernel<<<sm_count() * 8, 256, 0, st>>>(parent, size, n);
  bin_best_kernel<<<sm_count() * 8, 256, 0, st>>>(parent, size, n, best);
  bin_rows_kernel<<<(rows * 32 + 255) / 256, 256, 0, st>>>(parent, best, nx, rows, keep, rowcnt);
  bin_scan_kernel<<<1, 1024, 0, st>>>(rowcnt, rows);
}

void launch_binarize_emit(const int32_t* parent, const unsigned long long* best, int nx, int ny, int nz,
                          const int32_t* rowoff, int32_t* voxels, int64_t cap, cudaStream_t st) {
  const int rows = ny * nz;
  bin_emit_kernel<<<(rows * 32 + 255) / 256, 256, 0, st>>>(parent, best, nx, ny, rows, rowoff, voxels, cap);
}

void launch_boundary_flags(const uint8_t* keep, const int32_t* voxels, int64_t n, int nx, int ny, int nz,
                           uint8_t* flag, cudaStream_t st) {
  if (n > 0) bin_boundary_flag_kernel<<<sm_count() * 8, 256, 0, st>>>(keep, voxels, n, nx, ny, nz, flag);
}

}  // namespace vc

// SPDX-License-Identifier: Apache-2.0
//
// mocap::skeletonize (skeletonize.cpp:99-161) on sm_100a: directional
// simple-point thinning with the reference's order-dependent re-check,
// evaluated in parallel.
//
//   skel_lut      (26, 6)-simple-point predicate (skeletonize.cpp:48-95) for
//                 every one of the 2^26 neighbourhood configurations, one bit
//                 each (8 MB, stays in L2): 26-connectivity of the object and
//                 6-connectivity of the N18 background are bit-parallel
//                 floods on a 27-bit mask (dilation = shifts and masks)
//   skel_mark     one thread per active voxel: set, border in direction d,
//                 more than one neighbour, simple -> candidate (:143-148)
//   skel_recheck  the reference deletes candidates one after another in list
//                 order, re-testing each against the deletions made before it
//                 (:150-158).  A candidate's outcome depends only on the
//                 outcomes of EARLIER candidates in its 3x3x3 neighbourhood,
//                 so the outcomes are the unique fixed point of
//                   del(q) = test(q, grid minus {p < q near q : del(p)}).
//                 Sweeps evaluate every candidate from the current outcomes
//                 (starting from "all deleted") until a sweep changes nothing;
//                 at most (longest chain of adjacent candidates) sweeps, in
//                 practice a handful.
//   skel_apply    clear the deleted candidates in the grid
//
// Neighbour bit order: cell c = (dx+1) + 3(dy+1) + 9(dz+1) of the 3x3x3 cube;
// the 26-bit configuration drops the centre (c = 13).
#include <cstdint>

#include "vc_device.cuh"

namespace vc {
namespace {

constexpr uint32_t cube_mask(int which) {  // which: 0 x==0, 1 x==2, 2 y==0, 3 y==2, 4 faces, 5 N18
  uint32_t m = 0;
  for (int c = 0; c < 27; ++c) {
    const int x = c % 3, y = (c / 3) % 3, z = c / 9;
    const int nz = (x != 1) + (y != 1) + (z != 1);
    bool on = false;
    switch (which) {
      case 0: on = x == 0; break;
      case 1: on = x == 2; break;
      case 2: on = y == 0; break;
      case 3: on = y == 2; break;
      case 4: on = nz == 1; break;
      default: on = nz >= 1 && nz <= 2; break;
    }
    if (on) m |= 1u << c;
  }
  return m;
}
constexpr uint32_t kX0 = cube_mask(0), kX2 = cube_mask(1), kY0 = cube_mask(2), kY2 = cube_mask(3);
constexpr uint32_t kFaces = cube_mask(4), kN18 = cube_mask(5), kAll = (1u << 27) - 1u;

// one-cell dilations inside the cube (left shifts masked to 27 bits, so no
// bit leaves the cube and comes back through a later right shift)
constexpr uint32_t kNX0 = kAll & ~kX0, kNX2 = kAll & ~kX2, kNY0 = kAll & ~kY0, kNY2 = kAll & ~kY2;
__device__ __forceinline__ uint32_t dil_x(uint32_t m) { return m | ((m << 1) & kNX0) | ((m >> 1) & kNX2); }
__device__ __forceinline__ uint32_t dil_y(uint32_t m) { return m | ((m << 3) & kNY0) | ((m >> 3) & kNY2); }
__device__ __forceinline__ uint32_t dil_z(uint32_t m) { return m | ((m << 9) & kAll) | (m >> 9); }
__device__ __forceinline__ uint32_t dil6(uint32_t m) {
  return m | ((m << 1) & kNX0) | ((m >> 1) & kNX2) | ((m << 3) & kNY0) | ((m >> 3) & kNY2) | ((m << 9) & kAll) |
         (m >> 9);
}

// component of `set` holding the lowest bit of `seeds`, grown by `dil` within `set`
template <class D>
__device__ __forceinline__ uint32_t flood(uint32_t set, uint32_t seeds, D dil) {
  uint32_t comp = seeds & (0u - seeds);
  while (true) {
    const uint32_t nc = dil(comp) & set;
    if (nc == comp) return comp;
    comp = nc;
  }
}

__device__ bool simple_cfg(uint32_t cfg26) {
  const uint32_t obj = (cfg26 & 0x1fffu) | ((cfg26 >> 13) << 14);  // centre bit 13 empty
  if (!obj) return false;
  if (flood(obj, obj, [](uint32_t m) { return dil_z(dil_y(dil_x(m))); }) != obj) return false;  // one 26-component
  const uint32_t bg = ~obj & kN18;
  const uint32_t faces = bg & kFaces;
  if (!faces) return false;
  return (flood(bg, faces, [](uint32_t m) { return dil6(m); }) & faces) == faces;  // one 6-component meets the faces
}

__global__ void skel_lut_kernel(uint32_t* lut) {
  const uint32_t cfg = blockIdx.x * blockDim.x + threadIdx.x;  // grid covers exactly 2^26
  const uint32_t word = __ballot_sync(0xffffffffu, simple_cfg(cfg));
  if ((threadIdx.x & 31) == 0) lut[cfg >> 5] = word;
}

struct Vol {
  uint8_t* g;
  int nx, ny, nz;
  __device__ __forceinline__ bool obj(int x, int y, int z) const {
    return x >= 0 && y >= 0 && z >= 0 && x < nx && y < ny && z < nz && g[((size_t)z * ny + y) * nx + x] != 0;
  }
};

__device__ __forceinline__ int bit26(int c) { return c < 13 ? c : c - 1; }

__device__ __forceinline__ uint32_t gather_cfg(const Vol& v, int x, int y, int z) {
  uint32_t cfg = 0;
#pragma unroll
  for (int c = 0; c < 27; ++c) {
    if (c == 13) continue;
    if (v.obj(x + c % 3 - 1, y + (c / 3) % 3 - 1, z + c / 9 - 1)) cfg |= 1u << bit26(c);
  }
  return cfg;
}

__device__ __forceinline__ bool lut_simple(const uint32_t* __restrict__ lut, uint32_t cfg) {
  return (__ldg(lut + (cfg >> 5)) >> (cfg & 31)) & 1u;
}

__constant__ int c_dir[6][3] = {{0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}, {1, 0, 0}, {-1, 0, 0}};

// pos[voxel] = its index in the active list (set once per call over a -1 fill)
__global__ void skel_pos_kernel(const int32_t* __restrict__ vox, int64_t n, int nx, int ny, int32_t* pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    pos[((size_t)vox[3 * i + 2] * ny + vox[3 * i + 1]) * nx + vox[3 * i]] = (int32_t)i;
}

__global__ void skel_mark_kernel(Vol v, const int32_t* __restrict__ vox, int64_t n, int dir,
                                 const uint32_t* __restrict__ lut, uint8_t* cand, uint8_t* del, int* ncand) {
  const int dx = c_dir[dir][0], dy = c_dir[dir][1], dz = c_dir[dir][2];
  int local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = vox[3 * i], y = vox[3 * i + 1], z = vox[3 * i + 2];
    bool c = v.obj(x, y, z) && !v.obj(x + dx, y + dy, z + dz);
    if (c) {
      const uint32_t cfg = gather_cfg(v, x, y, z);
      c = __popc(cfg) > 1 && lut_simple(lut, cfg);
    }
    cand[i] = c;
    del[i] = c;  // first guess: every candidate goes
    local += c;
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(ncand, local);
}

__global__ void skel_recheck_kernel(Vol v, const int32_t* __restrict__ vox, int64_t n, const int32_t* __restrict__ pos,
                                    const uint32_t* __restrict__ lut, const uint8_t* __restrict__ cand,
                                    volatile uint8_t* del, int* changed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!cand[i]) continue;
    const int x = vox[3 * i], y = vox[3 * i + 1], z = vox[3 * i + 2];
    uint32_t cfg = 0;
#pragma unroll
    for (int c = 0; c < 27; ++c) {
      if (c == 13) continue;
      const int qx = x + c % 3 - 1, qy = y + (c / 3) % 3 - 1, qz = z + c / 9 - 1;
      if (!v.obj(qx, qy, qz)) continue;
      const int32_t j = pos[((size_t)qz * v.ny + qy) * v.nx + qx];  // -1: set but not in the list
      if (j >= 0 && j < i && cand[j] && del[j]) continue;           // deleted before q
      cfg |= 1u << bit26(c);
    }
    const uint8_t d = __popc(cfg) > 1 && lut_simple(lut, cfg);
    if (d != del[i]) {
      del[i] = d;
      *changed = 1;
    }
  }
}

__global__ void skel_apply_kernel(Vol v, const int32_t* __restrict__ vox, int64_t n, const uint8_t* __restrict__ cand,
                                  const uint8_t* __restrict__ del, int* ndel) {
  int local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (cand[i] && del[i]) {
      v.g[((size_t)vox[3 * i + 2] * v.ny + vox[3 * i + 1]) * v.nx + vox[3 * i]] = 0;
      ++local;
    }
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(ndel, local);
}

__global__ void skel_alive_kernel(const uint8_t* __restrict__ g, int nx, int ny, const int32_t* __restrict__ vox,
                                  int64_t n, uint8_t* alive) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    alive[i] = g[((size_t)vox[3 * i + 2] * ny + vox[3 * i + 1]) * nx + vox[3 * i]] != 0;
}

int grid_for(int64_t n) {
  const int64_t need = (n + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 8;
  return (int)(need < 1 ? 1 : (need < cap ? need : cap));
}

}  // namespace

size_t skel_lut_words() { return (size_t)1 << 21; }  // 2^26 bits

void launch_skel_lut(uint32_t* lut, cudaStream_t st) { skel_lut_kernel<<<(1u << 26) / 256, 256, 0, st>>>(lut); }

void launch_skel_pos(const int32_t* vox, int64_t n, int nx, int ny, int32_t* pos, cudaStream_t st) {
  skel_pos_kernel<<<grid_for(n), 256, 0, st>>>(vox, n, nx, ny, pos);
}
void launch_skel_mark(uint8_t* g, int nx, int ny, int nz, const int32_t* vox, int64_t n, int dir, const uint32_t* lut,
                      uint8_t* cand, uint8_t* del, int* ncand, cudaStream_t st) {
  skel_mark_kernel<<<grid_for(n), 256, 0, st>>>(Vol{g, nx, ny, nz}, vox, n, dir, lut, cand, del, ncand);
}
void launch_skel_recheck(uint8_t* g, int nx, int ny, int nz, const int32_t* vox, int64_t n, const int32_t* pos,
                         const uint32_t* lut, const uint8_t* cand, uint8_t* del, int* changed, cudaStream_t st) {
  skel_recheck_kernel<<<grid_for(n), 256, 0, st>>>(Vol{g, nx, ny, nz}, vox, n, pos, lut, cand, del, changed);
}
void launch_skel_apply(uint8_t* g, int nx, int ny, int nz, const int32_t* vox, int64_t n, const uint8_t* cand,
                       const uint8_t* del, int* ndel, cudaStream_t st) {
  skel_apply_kernel<<<grid_for(n), 256, 0, st>>>(Vol{g, nx, ny, nz}, vox, n, cand, del, ndel);
}
void launch_skel_alive(const uint8_t* g, int nx, int ny, const int32_t* vox, int64_t n, uint8_t* alive,
                       cudaStream_t st) {
  skel_alive_kernel<<<grid_for(n), 256, 0, st>>>(g, nx, ny, vox, n, alive);
}

}  // namespace vc

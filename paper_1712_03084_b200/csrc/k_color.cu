// SPDX-License-Identifier: Apache-2.0
//
// Colour correction on sm_100a:
//   * the per-sensor HSV value map (color_correction.cpp:140-160, hsv.cpp:8-46)
//     on whole images, fp64 in the reference's operation order so every output
//     byte matches;
//   * mutual_closest_pairs (color_correction.cpp:16-84) as a GPU hash grid:
//     cell = max_dist, open-addressing table of cell keys -> point lists, one
//     thread per query scanning the 27 neighbour cells; nearest by (d2, index)
//     exactly as the reference's tie rule, strict distance threshold; pairs
//     compacted in ascending i.
#include <cfloat>
#include <cstdint>

#include "vc_color.cuh"
#include "vc_device.cuh"

namespace vc {
namespace {

__global__ void color_apply_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int64_t n, double gain,
                                   double offset) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint8_t c[3] = {in[3 * i], in[3 * i + 1], in[3 * i + 2]};
    value_map_rgb(c, gain, offset);
    out[3 * i] = c[0], out[3 * i + 1] = c[1], out[3 * i + 2] = c[2];
  }
}

// ---------------------------------------------------------------- hash grid
constexpr uint64_t kEmpty = ~0ull;

__device__ __forceinline__ uint64_t hash_key(uint64_t k) {
  k ^= k >> 33, k *= 0xff51afd7ed558ccdull, k ^= k >> 33, k *= 0xc4ceb9fe1a85ec53ull, k ^= k >> 33;
  return k;
}

// color_correction.cpp:48-58: floor(p / cell) per axis, 21-bit packed key
__device__ __forceinline__ void cell_of(const double* p, double cell, long long c[3]) {
  for (int a = 0; a < 3; ++a) c[a] = (long long)floor(ddiv(p[a], cell));
}
__device__ __forceinline__ uint64_t pack_cell(long long x, long long y, long long z) {
  auto u = [](long long v) { return (uint64_t)(v + (1ll << 20)) & 0x1FFFFFull; };
  return (u(x) << 42) | (u(y) << 21) | u(z);
}

__global__ void grid_clear_kernel(uint64_t* keys, int32_t* counts, int cap) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x)
    keys[i] = kEmpty, counts[i] = 0;
}

__global__ void grid_insert_kernel(const double* __restrict__ pts, int n, double cell, uint64_t* keys,
                                   int32_t* counts, int32_t* slot_of, int cap) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    long long c[3];
    cell_of(pts + 3 * (size_t)i, cell, c);
    const uint64_t k = pack_cell(c[0], c[1], c[2]);
    uint32_t s = (uint32_t)hash_key(k) & (uint32_t)(cap - 1);
    while (true) {
      const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(keys + s), kEmpty, k);
      if (prev == kEmpty || prev == k) break;
      s = (s + 1) & (uint32_t)(cap - 1);
    }
    atomicAdd(counts + s, 1);
    slot_of[i] = (int32_t)s;
  }
}

// single CTA exclusive scan of the slot counts -> starts (then used as cursors)
__global__ void __launch_bounds__(1024) grid_scan_kernel(const int32_t* counts, int32_t* starts, int32_t* cursor,
                                                         int cap) {
  __shared__ int wsum[32];
  const int per = (cap + 1023) / 1024;
  const int b0 = min(cap, (int)threadIdx.x * per), b1 = min(cap, b0 + per);
  int tot = 0;
  for (int i = b0; i < b1; ++i) tot += counts[i];
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
  for (int i = b0; i < b1; ++i) starts[i] = run, cursor[i] = run, run += counts[i];
}

__global__ void grid_scatter_kernel(int n, const int32_t* __restrict__ slot_of, int32_t* cursor, int32_t* items) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    items[atomicAdd(cursor + slot_of[i], 1)] = i;
}

struct Grid {
  const uint64_t* keys;
  const int32_t* counts;
  const int32_t* starts;
  const int32_t* items;
  const double* pts;
  int cap;
  double cell;
};

// GridIndex::nearest (color_correction.cpp:24-45): minimal d2 < max_dist^2,
// ties to the smaller index; then norm < max_dist (strict)
__device__ int grid_nearest(const Grid& g, const double* q, double max_dist) {
  long long c[3];
  cell_of(q, g.cell, c);
  int best = -1;
  double best_d2 = dmul(max_dist, max_dist);
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const uint64_t k = pack_cell(c[0] + dx, c[1] + dy, c[2] + dz);
        uint32_t s = (uint32_t)hash_key(k) & (uint32_t)(g.cap - 1);
        while (true) {
          const uint64_t kk = g.keys[s];
          if (kk == kEmpty) {
            s = 0xffffffffu;
            break;
          }
          if (kk == k) break;
          s = (s + 1) & (uint32_t)(g.cap - 1);
        }
        if (s == 0xffffffffu) continue;
        const int b = g.starts[s], e = b + g.counts[s];
        for (int t = b; t < e; ++t) {
          const int i = g.items[t];
          const double* p = g.pts + 3 * (size_t)i;
          const double ex = dsub(p[0], q[0]), ey = dsub(p[1], q[1]), ez = dsub(p[2], q[2]);
          const double d2 = dadd(dadd(dmul(ex, ex), dmul(ey, ey)), dmul(ez, ez));
          if (d2 < best_d2 || (d2 == best_d2 && best >= 0 && i < best)) best_d2 = d2, best = i;
        }
      }
  if (best >= 0) {
    const double* p = g.pts + 3 * (size_t)best;
    const double ex = dsub(p[0], q[0]), ey = dsub(p[1], q[1]), ez = dsub(p[2], q[2]);
    if (__dsqrt_rn(dadd(dadd(dmul(ex, ex), dmul(ey, ey)), dmul(ez, ez))) < max_dist) return best;
  }
  return -1;
}

__global__ void mutual_kernel(Grid ga, Grid gb, const double* __restrict__ a, int na, double max_dist,
                              int32_t* partner) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < na; i += gridDim.x * blockDim.x) {
    const int j = grid_nearest(gb, a + 3 * (size_t)i, max_dist);
    partner[i] = (j >= 0 && grid_nearest(ga, gb.pts + 3 * (size_t)j, max_dist) == i) ? j : -1;
  }
}

// ordered compaction of (i, partner[i]) for partner >= 0 (single CTA)
__global__ void __launch_bounds__(1024) pairs_compact_kernel(const int32_t* partner, int na, int32_t* pairs,
                                                             int32_t* n_pairs) {
  __shared__ int wsum[32];
  const int per = (na + 1023) / 1024;
  const int b0 = min(na, (int)threadIdx.x * per), b1 = min(na, b0 + per);
  int tot = 0;
  for (int i = b0; i < b1; ++i) tot += partner[i] >= 0;
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
  for (int i = b0; i < b1; ++i)
    if (partner[i] >= 0) pairs[2 * run] = i, pairs[2 * run + 1] = partner[i], ++run;
  if (threadIdx.x == 1023) *n_pairs = wsum[31];
}

}  // namespace

void launch_color_apply(const uint8_t* in, uint8_t* out, int64_t n, double gain, double offset, cudaStream_t st) {
  color_apply_kernel<<<sm_count() * 8, 256, 0, st>>>(in, out, n, gain, offset);
}

size_t grid_scratch_bytes(int n) {
  int cap = 1024;
  while (cap < 2 * n) cap <<= 1;
  return (size_t)cap * (8 + 4 + 4 + 4) + (size_t)n * 8 + 1024;
}

namespace {
struct GridBufs {
  uint64_t* keys;
  int32_t *counts, *starts, *cursor, *slot_of, *items;
  int cap;
};
GridBufs carve_grid(void* scratch, int n) {
  GridBufs b;
  int cap = 1024;
  while (cap < 2 * n) cap <<= 1;
  uint8_t* p = static_cast<uint8_t*>(scratch);
  b.keys = reinterpret_cast<uint64_t*>(p), p += (size_t)cap * 8;
  b.counts = reinterpret_cast<int32_t*>(p), p += (size_t)cap * 4;
  b.starts = reinterpret_cast<int32_t*>(p), p += (size_t)cap * 4;
  b.cursor = reinterpret_cast<int32_t*>(p), p += (size_t)cap * 4;
  b.slot_of = reinterpret_cast<int32_t*>(p), p += (size_t)n * 4;
  b.items = reinterpret_cast<int32_t*>(p);
  b.cap = cap;
  return b;
}
Grid build_grid(const double* pts, int n, double cell, void* scratch, cudaStream_t st) {
  GridBufs b = carve_grid(scratch, n);
  grid_clear_kernel<<<sm_count() * 2, 256, 0, st>>>(b.keys, b.counts, b.cap);
  if (n > 0) grid_insert_kernel<<<sm_count() * 4, 256, 0, st>>>(pts, n, cell, b.keys, b.counts, b.slot_of, b.cap);
  grid_scan_kernel<<<1, 1024, 0, st>>>(b.counts, b.starts, b.cursor, b.cap);
  if (n > 0) grid_scatter_kernel<<<sm_count() * 4, 256, 0, st>>>(n, b.slot_of, b.cursor, b.items);
  return Grid{b.keys, b.counts, b.starts, b.items, pts, b.cap, cell};
}
}  // namespace

void launch_mutual_pairs(const double* a, int na, const double* b, int nb, double max_dist, void* scratch_a,
                         void* scratch_b, int32_t* partner, int32_t* pairs, int32_t* n_pairs, cudaStream_t st) {
  const Grid ga = build_grid(a, na, max_dist, scratch_a, st);
  const Grid gb = build_grid(b, nb, max_dist, scratch_b, st);
  if (na > 0) mutual_kernel<<<sm_count() * 4, 128, 0, st>>>(ga, gb, a, na, max_dist, partner);
  pairs_compact_kernel<<<1, 1024, 0, st>>>(partner, na, pairs, n_pairs);
}

}  // namespace vc

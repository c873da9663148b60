// SPDX-License-Identifier: Apache-2.0
//
// (A, L) consumers behind the C-ABI (mocap/
// binary_volume.cpp, skeletonize.cpp):
//   vc_binarize          threshold + largest 26-connected component on the GPU
//                        (k_binary.cu), on a host/device volume or the
//                        context's last frame
//   vc_boundary_voxels   boundary_voxels (GPU flags, host fp64 world centres)
//   vc_skeletonize       skeletonize — a sequential topology-preserving thinning
//                        whose deletions depend on their order (:150-160), so
//                        it runs on the host exactly as the reference
#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "vc_ctx.hpp"

using namespace vc;
using namespace vc::rt;

namespace vc {
void launch_binarize(const float* A, int nx, int ny, int nz, double level, int32_t* parent, int32_t* size,
                     float* maxbuf, unsigned long long* best, uint8_t* keep, int32_t* rowcnt, cudaStream_t st);
void launch_binarize_emit(const int32_t* parent, const unsigned long long* best, int nx, int ny, int nz,
                          const int32_t* rowoff, int32_t* voxels, int64_t cap, cudaStream_t st);
void launch_boundary_flags(const uint8_t* keep, const int32_t* voxels, int64_t n, int nx, int ny, int nz,
                           uint8_t* flag, cudaStream_t st);
}  // namespace vc

namespace vc_io_detail {
vc_status set_error(vc_status s, const std::string& msg);
}

namespace {

struct Hood {
  std::array<std::vector<int>, 27> adj26, adj6;
  std::array<bool, 27> in_n18{}, is_face{};
  Hood() {  // skeletonize.cpp:12-42
    auto co = [](int c) { return std::array<int, 3>{c % 3 - 1, (c / 3) % 3 - 1, c / 9 - 1}; };
    for (int c = 0; c < 27; ++c) {
      const auto a = co(c);
      const int nz = std::abs(a[0]) + std::abs(a[1]) + std::abs(a[2]);
      in_n18[c] = c != 13 && nz <= 2;
      is_face[c] = nz == 1;
      for (int d = 0; d < 27; ++d) {
        if (d == c) continue;
        const auto b = co(d);
        const int man = std::abs(a[0] - b[0]) + std::abs(a[1] - b[1]) + std::abs(a[2] - b[2]);
        const int che = std::max({std::abs(a[0] - b[0]), std::abs(a[1] - b[1]), std::abs(a[2] - b[2])});
        if (che == 1 && c != 13 && d != 13) adj26[c].push_back(d);
        if (man == 1) adj6[c].push_back(d);
      }
    }
  }
};
const Hood& hood() {
  static const Hood h;
  return h;
}

// skeletonize.cpp:48-95: (26, 6) simple point
bool is_simple(const std::array<bool, 27>& obj) {
  const Hood& t = hood();
  int seen = 0;
  for (int c = 0; c < 27; ++c)
    if (c != 13 && obj[c]) ++seen;
  if (seen == 0) return false;
  std::array<bool, 27> vis{};
  int comp26 = 0;
  for (int c = 0; c < 27 && comp26 <= 1; ++c) {
    if (c == 13 || !obj[c] || vis[c]) continue;
    ++comp26;
    std::array<int, 27> st;
    int top = 0;
    st[top++] = c, vis[c] = true;
    while (top) {
      const int cur = st[--top];
      for (int n : t.adj26[cur])
        if (n != 13 && obj[n] && !vis[n]) vis[n] = true, st[top++] = n;
    }
  }
  if (comp26 != 1) return false;
  vis.fill(false);
  int comp6 = 0;
  for (int c = 0; c < 27 && comp6 <= 1; ++c) {
    if (!t.is_face[c] || obj[c] || vis[c]) continue;
    ++comp6;
    std::array<int, 27> st;
    int top = 0;
    st[top++] = c, vis[c] = true;
    while (top) {
      const int cur = st[--top];
      for (int n : t.adj6[cur])
        if (t.in_n18[n] && !obj[n] && !vis[n]) vis[n] = true, st[top++] = n;
    }
  }
  return comp6 == 1;
}

}  // namespace

extern "C" {

vc_status vc_binarize(vc_ctx* ctx, const float* A, int32_t mem_kind, const vc_grid_spec* grid, double level,
                      uint8_t* keep_out, int32_t* voxels_out, int64_t capacity, int64_t* n_voxels) {
  if (!ctx || !grid || !n_voxels || capacity < 0 || (capacity > 0 && !voxels_out))
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "binarize: bad arguments");
  const int nx = grid->nx, ny = grid->ny, nz = grid->nz;
  if (nx < 1 || ny < 1 || nz < 1) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "binarize: bad grid");
  const size_t N = (size_t)nx * ny * nz;
  if (N >= (size_t)INT32_MAX) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "binarize: grid too large");
  cudaSetDevice(ctx->device);
  const float* dA = A;
  if (!A) {  // the context's last frame volume
    if (!ctx->A.p || ctx->layout != 1 || (size_t)ctx->nx * ctx->ny * ctx->nz != N || ctx->nx != nx || ctx->ny != ny)
      return fail(ctx, VC_ERR_INVALID_ARGUMENT, "binarize: no matching frame volume in this context");
    dA = P<float>(ctx->A);
  }
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  const int rows = ny * nz;
  const size_t bytes = (mem_kind == VC_MEM_HOST && A ? up(N * 4) : 0) + 2 * up(N * 4) + up(N) +
                       up(((size_t)rows + 1) * 4) + 512;
  VC_TRY(ensure(ctx, ctx->scratch_dev, bytes));
  uint8_t* p = P<uint8_t>(ctx->scratch_dev);
  if (A && mem_kind == VC_MEM_HOST) {
    VC_CUDA(cudaMemcpyAsync(p, A, N * 4, cudaMemcpyHostToDevice, ctx->st));
    dA = reinterpret_cast<const float*>(p);
    p += up(N * 4);
  }
  int32_t* parent = reinterpret_cast<int32_t*>(p);
  p += up(N * 4);
  int32_t* size = reinterpret_cast<int32_t*>(p);
  p += up(N * 4);
  uint8_t* keep = p;
  p += up(N);
  int32_t* rowcnt = reinterpret_cast<int32_t*>(p);
  p += up(((size_t)rows + 1) * 4);
  float* maxbuf = reinterpret_cast<float*>(p);
  unsigned long long* best = reinterpret_cast<unsigned long long*>(p + 8);
  launch_binarize(dA, nx, ny, nz, level, parent, size, maxbuf, best, keep, rowcnt, ctx->st);
  VC_CUDA(cudaGetLastError());
  unsigned long long hb = 0;
  int32_t total = 0;
  VC_CUDA(cudaMemcpyAsync(&hb, best, 8, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaMemcpyAsync(&total, rowcnt + rows, 4, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  if (hb == 0) return fail(ctx, VC_ERR_EMPTY_SCENE, "binarize: empty interior");  // binary_volume.cpp:51
  *n_voxels = total;
  if (capacity > 0) {
    const int64_t cap = capacity < total ? capacity : total;
    int32_t* dvox = size;  // reuse the size array when 3 * total int32 fit in its N words
    if ((size_t)3 * total > N) {
      VC_TRY(ensure(ctx, ctx->scratch_dev2, (size_t)3 * total * 4 + 256));
      dvox = P<int32_t>(ctx->scratch_dev2);
    }
    launch_binarize_emit(parent, best, nx, ny, nz, rowcnt, dvox, total, ctx->st);
    VC_CUDA(cudaGetLastError());
    VC_CUDA(cudaMemcpyAsync(voxels_out, dvox, (size_t)cap * 12, cudaMemcpyDeviceToHost, ctx->st));
  }
  if (keep_out) VC_CUDA(cudaMemcpyAsync(keep_out, keep, N, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}

// binary_volume.cpp:68-82: world centres (origin + edge * (x, y, z)) of the
// voxels with a face neighbour outside the object, in voxel-list order
vc_status vc_boundary_voxels(vc_ctx* ctx, const uint8_t* keep, const vc_grid_spec* grid, const int32_t* voxels,
                             int64_t n, double* out_xyz, int64_t* n_out) {
  if (!ctx || !keep || !grid || !n_out || n < 0 || (n > 0 && (!voxels || !out_xyz)))
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "boundary_voxels: bad arguments");
  const int nx = grid->nx, ny = grid->ny, nz = grid->nz;
  const size_t N = (size_t)nx * ny * nz;
  *n_out = 0;
  if (n == 0) return VC_OK;
  cudaSetDevice(ctx->device);
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  VC_TRY(ensure(ctx, ctx->scratch_dev, up(N) + up((size_t)n * 12) + up((size_t)n) + 256));
  uint8_t* dkeep = P<uint8_t>(ctx->scratch_dev);
  int32_t* dvox = reinterpret_cast<int32_t*>(dkeep + up(N));
  uint8_t* dflag = reinterpret_cast<uint8_t*>(dvox) + up((size_t)n * 12);
  VC_CUDA(cudaMemcpyAsync(dkeep, keep, N, cudaMemcpyHostToDevice, ctx->st));
  VC_CUDA(cudaMemcpyAsync(dvox, voxels, (size_t)n * 12, cudaMemcpyHostToDevice, ctx->st));
  launch_boundary_flags(dkeep, dvox, n, nx, ny, nz, dflag, ctx->st);
  VC_CUDA(cudaGetLastError());
  std::vector<uint8_t> flag((size_t)n);
  VC_CUDA(cudaMemcpyAsync(flag.data(), dflag, (size_t)n, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  int64_t m = 0;
  for (int64_t v = 0; v < n; ++v)
    if (flag[v])
      for (int a = 0; a < 3; ++a, ++m) out_xyz[m] = grid->origin[a] + grid->edge_mm * (double)voxels[3 * v + a];
  *n_out = m / 3;
  return VC_OK;
}

// skeletonize.cpp:99-161
vc_status vc_skeletonize(const uint8_t* grid_in, int32_t nx, int32_t ny, int32_t nz, const int32_t* voxels,
                         int64_t n, int32_t* out, int64_t* n_out) {
  if (!grid_in || !n_out || nx < 1 || ny < 1 || nz < 1 || n < 0 || (n > 0 && (!voxels || !out)))
    return vc_io_detail::set_error(VC_ERR_INVALID_ARGUMENT, "skeletonize: bad arguments");
  std::vector<uint8_t> g(grid_in, grid_in + (size_t)nx * ny * nz);
  auto at = [&](int x, int y, int z) -> uint8_t& { return g[((size_t)z * ny + y) * nx + x]; };
  auto obj = [&](int x, int y, int z) {
    return x >= 0 && y >= 0 && z >= 0 && x < nx && y < ny && z < nz && at(x, y, z) != 0;
  };
  auto fill = [&](const int* p, std::array<bool, 27>& h) {
    int c = 0;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx, ++c) h[c] = obj(p[0] + dx, p[1] + dy, p[2] + dz);
  };
  auto ncount = [&](const int* p) {
    int k = 0;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx)
          if ((dx | dy | dz) != 0 && obj(p[0] + dx, p[1] + dy, p[2] + dz)) ++k;
    return k;
  };
  static constexpr int kDir[6][3] = {{0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}, {1, 0, 0}, {-1, 0, 0}};
  std::vector<std::array<int, 3>> active((size_t)n), cand;
  for (int64_t v = 0; v < n; ++v) active[v] = {voxels[3 * v], voxels[3 * v + 1], voxels[3 * v + 2]};
  std::array<bool, 27> h{};
  bool any = true;
  while (any) {
    any = false;
    for (const auto& d : kDir) {
      cand.clear();
      for (const auto& p : active) {
        if (!at(p[0], p[1], p[2])) continue;
        if (obj(p[0] + d[0], p[1] + d[1], p[2] + d[2])) continue;  // not a border voxel
        if (ncount(p.data()) <= 1) continue;                        // endpoint / isolated
        fill(p.data(), h);
        if (is_simple(h)) cand.push_back(p);
      }
      for (const auto& p : cand) {  // sequential re-check (order-dependent)
        if (ncount(p.data()) <= 1) continue;
        fill(p.data(), h);
        if (!is_simple(h)) continue;
        at(p[0], p[1], p[2]) = 0;
        any = true;
      }
    }
    if (any) {
      std::vector<std::array<int, 3>> still;
      still.reserve(active.size());
      for (const auto& p : active)
        if (at(p[0], p[1], p[2])) still.push_back(p);
      active.swap(still);
    }
  }
  for (size_t v = 0; v < active.size(); ++v)
    out[3 * v] = active[v][0], out[3 * v + 1] = active[v][1], out[3 * v + 2] = active[v][2];
  *n_out = (int64_t)active.size();
  return VC_OK;
}

}  // extern "C"

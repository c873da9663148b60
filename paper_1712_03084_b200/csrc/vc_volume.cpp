// SPDX-License-Identifier: Apache-2.0
//
// (A, L) consumers behind the C-ABI (mocap/
// binary_volume.cpp, skeletonize.cpp):
//   vc_binarize          threshold + largest 26-connected component on the GPU
//                        (k_binary.cu), on a host/device volume or the
//                        context's last frame
//   vc_boundary_voxels   boundary_voxels (GPU flags, host fp64 world centres)
//   vc_skeletonize       skeletonize on the GPU (k_skeleton.cu): simple-point
//                        lookup table, parallel candidates, the order-dependent
//                        re-check as a fixed point
#include <algorithm>
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
size_t skel_lut_words();
void launch_skel_lut(uint32_t* lut, cudaStream_t st);
void launch_skel_pos(const int32_t* vox, int64_t n, int nx, int ny, int32_t* pos, cudaStream_t st);
void launch_skel_mark(uint8_t* g, int nx, int ny, int nz, const int32_t* vox, int64_t n, int dir, const uint32_t* lut,
                      uint8_t* cand, uint8_t* del, int* ncand, cudaStream_t st);
void launch_skel_recheck(uint8_t* g, int nx, int ny, int nz, const int32_t* vox, int64_t n, const int32_t* pos,
                         const uint32_t* lut, const uint8_t* cand, uint8_t* del, int* changed, cudaStream_t st);
void launch_skel_apply(uint8_t* g, int nx, int ny, int nz, const int32_t* vox, int64_t n, const uint8_t* cand,
                       const uint8_t* del, int* ndel, cudaStream_t st);
void launch_skel_alive(const uint8_t* g, int nx, int ny, const int32_t* vox, int64_t n, uint8_t* alive,
                       cudaStream_t st);
}  // namespace vc

namespace vc_io_detail {
vc_status set_error(vc_status s, const std::string& msg);
}

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

// skeletonize(BinaryVolume) (skeletonize.cpp:99-161) on the GPU (k_skeleton.cu):
// per pass and direction, parallel candidate marking, the order-dependent
// re-check as a fixed-point sweep, then the deletions; the surviving voxels in
// input order.  The grid is not modified (a device copy is thinned).
vc_status vc_skeletonize(vc_ctx* ctx, const uint8_t* grid_in, int32_t nx, int32_t ny, int32_t nz,
                         const int32_t* voxels, int64_t n, int32_t* out, int64_t* n_out) {
  if (!ctx || !grid_in || !n_out || nx < 1 || ny < 1 || nz < 1 || n < 0 || (n > 0 && (!voxels || !out)))
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "skeletonize: bad arguments");
  const size_t N = (size_t)nx * ny * nz;
  if (N >= (size_t)INT32_MAX || n >= INT32_MAX) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "skeletonize: grid too large");
  *n_out = 0;
  if (n == 0) return VC_OK;
  cudaSetDevice(ctx->device);
  if (!ctx->skel_lut_ready) {  // (26, 6)-simple predicate of all 2^26 neighbourhoods, once per context
    VC_TRY(ensure(ctx, ctx->skel_lut, skel_lut_words() * 4));
    launch_skel_lut(P<uint32_t>(ctx->skel_lut), ctx->st);
    VC_CUDA(cudaGetLastError());
    ctx->skel_lut_ready = true;
  }
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t nn = (size_t)n;
  VC_TRY(ensure(ctx, ctx->scratch_dev, up(N) + up(N * 4) + up(nn * 12) + 3 * up(nn) + 256));
  uint8_t* p = P<uint8_t>(ctx->scratch_dev);
  uint8_t* g = p;
  p += up(N);
  int32_t* pos = reinterpret_cast<int32_t*>(p);
  p += up(N * 4);
  int32_t* vox = reinterpret_cast<int32_t*>(p);
  p += up(nn * 12);
  uint8_t* cand = p;
  p += up(nn);
  uint8_t* del = p;
  p += up(nn);
  uint8_t* alive = p;
  p += up(nn);
  int* cnt = reinterpret_cast<int*>(p);  // [0] candidates, [1] changed, [2] deletions
  const uint32_t* lut = P<uint32_t>(ctx->skel_lut);
  VC_CUDA(cudaMemcpyAsync(g, grid_in, N, cudaMemcpyHostToDevice, ctx->st));
  VC_CUDA(cudaMemcpyAsync(vox, voxels, nn * 12, cudaMemcpyHostToDevice, ctx->st));
  VC_CUDA(cudaMemsetAsync(pos, 0xff, N * 4, ctx->st));
  launch_skel_pos(vox, n, nx, ny, pos, ctx->st);
  auto read = [&](int which, int* v) -> vc_status {
    VC_CUDA(cudaMemcpyAsync(v, cnt + which, 4, cudaMemcpyDeviceToHost, ctx->st));
    VC_CUDA(cudaStreamSynchronize(ctx->st));
    return VC_OK;
  };
  int hv = 0;
  for (bool any = true; any;) {
    any = false;
    for (int dir = 0; dir < 6; ++dir) {
      VC_CUDA(cudaMemsetAsync(cnt, 0, 12, ctx->st));
      launch_skel_mark(g, nx, ny, nz, vox, n, dir, lut, cand, del, cnt, ctx->st);
      VC_CUDA(cudaGetLastError());
      VC_TRY(read(0, &hv));
      if (hv == 0) continue;
      do {  // sweeps until the deletions are the sequential re-check's fixed point
        VC_CUDA(cudaMemsetAsync(cnt + 1, 0, 4, ctx->st));
        launch_skel_recheck(g, nx, ny, nz, vox, n, pos, lut, cand, del, cnt + 1, ctx->st);
        VC_CUDA(cudaGetLastError());
        VC_TRY(read(1, &hv));
      } while (hv);
      launch_skel_apply(g, nx, ny, nz, vox, n, cand, del, cnt + 2, ctx->st);
      VC_CUDA(cudaGetLastError());
      VC_TRY(read(2, &hv));
      any = any || hv > 0;
    }
  }
  launch_skel_alive(g, nx, ny, vox, n, alive, ctx->st);
  std::vector<uint8_t> keep(nn);
  VC_CUDA(cudaMemcpyAsync(keep.data(), alive, nn, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  int64_t m = 0;
  for (size_t v = 0; v < nn; ++v)
    if (keep[v]) std::memcpy(out + 3 * m++, voxels + 3 * v, 12);
  *n_out = m;
  return VC_OK;
}

}  // extern "C"

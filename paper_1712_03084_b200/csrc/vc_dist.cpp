// SPDX-License-Identifier: Apache-2.0
//
// z-slab decomposition of one frame over P ranks:
// the distributed form of recon::reconstruct_frame (reconstruct.cpp:37-78)
// + texturing behind vc_reconstruct_frame_dist (include/vc/vc.h).
//
// Rank r owns planes [zoff, zoff+nzl), nzl = nz/P, and ky rows
// [ky0, ky0+kyl), kyl = ny/P, of the spectrum.  Per frame:
//
//   P1  preprocess all views (replicated, 7 MB of input) -> sparse clear ->
//       splat into the slab (splat.cpp:61-77 slab rule) -> x-R2C, y-C2C into
//       the send layout [s][zl][yl][H] (D = wx X + wy Y and Z, 2 components)
//   X1  all-to-all D, Z -> [z][kyl][H]; all-gather of the empty-plane flags
//   P2  fused z pass (FFT_z, -i/|w|^2 filter, inverse FFT_z) in place
//   X2  all-to-all back -> [s'][zl][yl][H]
//   P3  inverse y, x C2R -> A slab (planes zoff-1 .. zoff+nzl+1 allocated)
//   X3  halo: plane zoff-1 from r-1, planes zoff+nzl, zoff+nzl+1 from r+1
//   P4  row min/max of the halo planes; per-point trilinear samples of the
//       points whose lower z plane this rank owns (0 elsewhere)
//   X4  all-reduce (sum) of the samples: exactly one rank contributes each
//       point, so every rank then sums them in the single-GPU order
//   P5  iso level; marching-cubes count over the own planes + the next
//       rank's first plane (numbered, not emitted) -> (V, T, C)
//   X5  all-gather of (V, T, C)
//   P6  vertex offset, emit (global vertex ids), normals, triangles, texture
//
// Exchanges run on NCCL (dlopen'ed libnccl.so.2, one process per GPU, all
// on the context stream: no host synchronisation inside the frame) or on a
// loopback exchanger that steps P virtual ranks in lockstep on one device.
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "vc_ctx.hpp"

using namespace vc;
using namespace vc::rt;

namespace {

// ------------------------------------------------------------ NCCL (runtime)
// The subset of nccl.h (2.x ABI) this file calls; enums are passed as int.
struct NcclUid {
  char internal[128];
};
typedef struct ncclComm* ncclComm_t;
constexpr int kNcclInt32 = 2, kNcclFloat64 = 8, kNcclUint32 = 3, kNcclFloat32 = 7, kNcclSum = 0;

struct Nccl {
  void* h = nullptr;
  int (*GetUniqueId)(NcclUid*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, NcclUid, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

const Nccl* nccl_lib(std::string* why) {
  static Nccl lib;
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("VC_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n || !*n) continue;
      lib.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (lib.h) break;
    }
    if (!lib.h) {
      err = "libnccl.so.2 not found (set VC_NCCL_LIB)";
    } else {
      auto sym = [&](auto& fp, const char* name) {
        fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(lib.h, name));
        if (!fp) err = std::string("NCCL symbol missing: ") + name;
      };
      sym(lib.GetUniqueId, "ncclGetUniqueId");
      sym(lib.CommInitRank, "ncclCommInitRank");
      sym(lib.CommDestroy, "ncclCommDestroy");
      sym(lib.Send, "ncclSend");
      sym(lib.Recv, "ncclRecv");
      sym(lib.GroupStart, "ncclGroupStart");
      sym(lib.GroupEnd, "ncclGroupEnd");
      sym(lib.AllReduce, "ncclAllReduce");
      sym(lib.AllGather, "ncclAllGather");
      sym(lib.GetErrorString, "ncclGetErrorString");
    }
  });
  if (!err.empty()) {
    if (why) *why = err;
    return nullptr;
  }
  return &lib;
}

}  // namespace

// ------------------------------------------------------------ rank state
struct DistRank {
  vc_ctx* ctx = nullptr;
  int rank = 0;
  ncclComm_t comm = nullptr;
  Buf sd;       // 2 spectrum components in send/receive layout
  Buf samples;  // per-point iso samples (pts_cap doubles)
  Buf counts;   // (V, T, C) per rank
  bool dirty = true;
  int dims[3] = {0, 0, 0};
  std::vector<int32_t> counts_h;
};

struct vc_dist {
  int world = 1;
  bool loopback = false;
  std::vector<DistRank> r;
};

namespace {

#define VC_NCCL(call)                                                                          \
  do {                                                                                         \
    const int r_ = (call);                                                                     \
    if (r_ != 0) return fail(ctx, VC_ERR_NCCL, std::string(#call) + ": " + L->GetErrorString(r_)); \
  } while (0)

struct Geo {
  int nx, ny, nz, P, nzl, kyl, H;
  size_t plane, E, B;  // voxels per plane, complex elems per component, per block
};

size_t hp(int nx) { return (size_t)(((nx / 2 + 1) + 3) & ~3); }

// ------------------------------------------------------------ exchanges
// all-to-all of equal blocks: block s of src[r] -> block r of dst[s]
vc_status x_all_to_all(vc_dist* d, const std::vector<const float2*>& src, const std::vector<float2*>& dst,
                       size_t B) {
  vc_ctx* ctx = d->r[0].ctx;
  if (d->loopback) {
    for (int a = 0; a < d->world; ++a)
      for (int b = 0; b < d->world; ++b)
        VC_CUDA(cudaMemcpyAsync(dst[b] + (size_t)a * B, src[a] + (size_t)b * B, B * sizeof(float2),
                                cudaMemcpyDeviceToDevice, ctx->st));
    return VC_OK;
  }
  const Nccl* L = nccl_lib(nullptr);
  DistRank& me = d->r[0];
  VC_NCCL(L->GroupStart());
  for (int s = 0; s < d->world; ++s) {
    VC_NCCL(L->Send(src[0] + (size_t)s * B, 2 * B, kNcclFloat32, s, me.comm, ctx->st));
    VC_NCCL(L->Recv(dst[0] + (size_t)s * B, 2 * B, kNcclFloat32, s, me.comm, ctx->st));
  }
  VC_NCCL(L->GroupEnd());
  return VC_OK;
}

// in-place all-gather: rank r's n words at buf[r] + r*n -> everyone
vc_status x_all_gather_u32(vc_dist* d, const std::vector<uint32_t*>& buf, size_t n) {
  vc_ctx* ctx = d->r[0].ctx;
  if (d->loopback) {
    for (int a = 0; a < d->world; ++a)
      for (int b = 0; b < d->world; ++b)
        if (a != b)
          VC_CUDA(cudaMemcpyAsync(buf[b] + (size_t)a * n, buf[a] + (size_t)a * n, n * 4, cudaMemcpyDeviceToDevice,
                                  ctx->st));
    return VC_OK;
  }
  const Nccl* L = nccl_lib(nullptr);
  const int me = d->r[0].rank;
  VC_NCCL(L->AllGather(buf[0] + (size_t)me * n, buf[0], n, kNcclUint32, d->r[0].comm, ctx->st));
  return VC_OK;
}

vc_status x_all_reduce_f64(vc_dist* d, const std::vector<double*>& buf, size_t n) {
  vc_ctx* ctx = d->r[0].ctx;
  if (d->loopback) {
    // one nonzero contribution per element: sum into rank 0 in rank order, broadcast
    for (int a = 1; a < d->world; ++a) {
      launch_add_f64(buf[0], buf[a], n, ctx->st);
    }
    for (int a = 1; a < d->world; ++a)
      VC_CUDA(cudaMemcpyAsync(buf[a], buf[0], n * 8, cudaMemcpyDeviceToDevice, ctx->st));
    VC_CUDA(cudaGetLastError());
    return VC_OK;
  }
  const Nccl* L = nccl_lib(nullptr);
  VC_NCCL(L->AllReduce(buf[0], buf[0], n, kNcclFloat64, kNcclSum, d->r[0].comm, ctx->st));
  return VC_OK;
}

// A halo: plane zoff-1 from r-1 (1 plane), planes zoff+nzl.. +1 from r+1 (2)
vc_status x_halo(vc_dist* d, const Geo& g) {
  vc_ctx* ctx = d->r[0].ctx;
  const size_t pb = g.plane * sizeof(float);
  if (d->loopback) {
    for (int a = 0; a < d->world; ++a) {
      float* A = P<float>(d->r[a].ctx->A);
      if (a > 0) {  // from a-1: its local plane nzl -> my local plane 0
        const float* B = P<float>(d->r[a - 1].ctx->A);
        VC_CUDA(cudaMemcpyAsync(A, B + (size_t)g.nzl * g.plane, pb, cudaMemcpyDeviceToDevice, ctx->st));
      }
      if (a + 1 < d->world) {  // from a+1: its local planes 1, 2 -> my nzl+1, nzl+2
        const float* B = P<float>(d->r[a + 1].ctx->A);
        VC_CUDA(cudaMemcpyAsync(A + (size_t)(g.nzl + 1) * g.plane, B + g.plane, 2 * pb, cudaMemcpyDeviceToDevice,
                                ctx->st));
      }
    }
    return VC_OK;
  }
  const Nccl* L = nccl_lib(nullptr);
  const DistRank& me = d->r[0];
  float* A = P<float>(ctx->A);
  const int r = me.rank;
  VC_NCCL(L->GroupStart());
  if (r > 0) {
    VC_NCCL(L->Send(A + g.plane, 2 * g.plane, kNcclFloat32, r - 1, me.comm, ctx->st));
    VC_NCCL(L->Recv(A, g.plane, kNcclFloat32, r - 1, me.comm, ctx->st));
  }
  if (r + 1 < d->world) {
    VC_NCCL(L->Send(A + (size_t)g.nzl * g.plane, g.plane, kNcclFloat32, r + 1, me.comm, ctx->st));
    VC_NCCL(L->Recv(A + (size_t)(g.nzl + 1) * g.plane, 2 * g.plane, kNcclFloat32, r + 1, me.comm, ctx->st));
  }
  VC_NCCL(L->GroupEnd());
  return VC_OK;
}

vc_status x_all_gather_i32(vc_dist* d, const std::vector<int32_t*>& buf, size_t n) {
  std::vector<uint32_t*> b;
  for (auto* p : buf) b.push_back(reinterpret_cast<uint32_t*>(p));
  return x_all_gather_u32(d, b, n);
}

// loopback steps all virtual ranks on one device: order them by device sync
vc_status lockstep(vc_dist* d) {
  if (!d->loopback) return VC_OK;
  vc_ctx* ctx = d->r[0].ctx;
  for (auto& rk : d->r) VC_CUDA(cudaStreamSynchronize(rk.ctx->st));
  return VC_OK;
}

template <class T>
T* shift(void* base, ptrdiff_t elems) {  // pointer to a global index outside the slab's allocation start
  return reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(base) + elems * (ptrdiff_t)sizeof(T));
}

SlabFft slab_fft(DistRank& rk, const Geo& g, int mode) {
  vc_ctx* ctx = rk.ctx;
  SlabFft a;
  float2* spec = P<float2>(ctx->spec);
  float2* sd = P<float2>(rk.sd);
  a.acc = P<float4>(ctx->acc);
  a.S0 = spec, a.S1 = spec + g.E, a.S2 = spec + 2 * g.E;
  a.O0 = sd, a.O1 = sd + g.E;  // forward send layout
  a.R0 = a.S0, a.R1 = a.S1;    // forward receive layout ([z][kyl][H])
  a.Rin = sd;                  // backward receive layout
  a.Rout = a.S1;
  a.A = P<float>(ctx->A) + g.plane;  // local plane 0 = halo
  a.nx = g.nx, a.ny = g.ny, a.nz = g.nz, a.nzl = g.nzl, a.zoff = rk.rank * g.nzl;
  a.kyl = g.kyl, a.ky0 = rk.rank * g.kyl, a.H = (int)hp(g.nx), a.mode = mode;
  const float2* tw = P<float2>(ctx->tw);
  a.twx = tw, a.twy = tw + g.nx, a.twz = tw + g.nx + g.ny;
  a.st = ctx->st;
  a.rowmm = P<float2>(ctx->rowmm);
  a.rowbits = P<uint32_t>(ctx->rowbits);
  a.planeflag = P<uint32_t>(ctx->planeflag);
  a.rowlist = P<int32_t>(ctx->rowlist);
  return a;
}

vc_status ensure_rank(DistRank& rk, const Geo& g, const vc_sensor* sensors, const vc_view* views, int k) {
  vc_ctx* ctx = rk.ctx;
  VC_CUDA(cudaSetDevice(ctx->device));
  VC_TRY(ensure_tables(ctx));
  const size_t Nl = g.plane * g.nzl;
  const void* acc_before = ctx->acc.p;
  VC_TRY(ensure(ctx, ctx->acc, Nl * sizeof(float4)));
  VC_TRY(ensure(ctx, ctx->rowbits, (size_t)g.ny * g.nzl * sizeof(uint32_t)));
  VC_TRY(ensure(ctx, ctx->rowlist, ((size_t)g.ny * g.nzl + 1) * sizeof(int32_t)));
  VC_TRY(ensure(ctx, ctx->planeflag, (size_t)(2 * g.nz + 2) * sizeof(uint32_t) + 256));  // flags + F-y live-plane list
  VC_TRY(ensure(ctx, ctx->spec, 3 * g.E * sizeof(float2)));
  VC_TRY(ensure(ctx, rk.sd, 2 * g.E * sizeof(float2)));
  VC_TRY(ensure(ctx, ctx->A, g.plane * (g.nzl + 3) * sizeof(float)));
  VC_TRY(ensure(ctx, ctx->vbase, g.plane * (g.nzl + 1) * sizeof(uint32_t)));
  VC_TRY(ensure_mc_scratch(ctx, g.nx, g.ny, g.nzl + 2));
  VC_TRY(ensure(ctx, ctx->tw, twiddle_elems(g.nx, g.ny, g.nz) * sizeof(float2)));
  VC_TRY(ensure(ctx, ctx->iso_partial, 1024 * sizeof(double)));
  VC_TRY(ensure(ctx, rk.counts, (size_t)3 * g.P * sizeof(int32_t)));
  if (ctx->acc.p != acc_before || ctx->layout != 2) rk.dirty = true;
  ctx->layout = 2;
  if (rk.dims[0] != g.nx || rk.dims[1] != g.ny || rk.dims[2] != g.nz) {
    upload_twiddles(P<float2>(ctx->tw), g.nx, g.ny, g.nz, ctx->st);
    prepare_integrate(g.nx, g.ny, g.nz);
    VC_CUDA(cudaGetLastError());
    rk.dims[0] = g.nx, rk.dims[1] = g.ny, rk.dims[2] = g.nz;
    rk.dirty = true;
  }
  ctx->nx = ctx->ny = ctx->nz = 0;  // the grid buffers hold a slab, not a whole-grid frame
  ctx->acc_dirty = true;
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec), ctx->gexec = nullptr;
  if (ctx->v_cap == 0) VC_TRY(ensure_mesh_caps(ctx, (int)std::max<size_t>(Nl / 16, 1 << 16), kMaxViews));
  VC_TRY(setup_sensorset(ctx, sensors, k));
  VC_TRY(ensure(ctx, rk.samples, (size_t)std::max(ctx->pts_cap, 1) * sizeof(double)));
  VC_TRY(stage_views(ctx, sensors, views, k, true));
  return VC_OK;
}

McSlab mc_slab(const DistRank& rk, const Geo& g) {
  const int zoff = rk.rank * g.nzl;
  const bool last = rk.rank == g.P - 1;
  return McSlab{zoff, g.nzl + (last ? 0 : 1), zoff + g.nzl};
}

MeshBufs slab_mesh(DistRank& rk, const Geo& g) {
  MeshBufs mb = mesh_bufs(rk.ctx);
  mb.vbase = shift<uint32_t>(rk.ctx->vbase.p, -(ptrdiff_t)(rk.rank * g.nzl) * (ptrdiff_t)g.plane);
  return mb;
}
const float* slab_A(DistRank& rk, const Geo& g) {  // indexable by global voxel id
  return shift<float>(rk.ctx->A.p, -(ptrdiff_t)(rk.rank * g.nzl - 1) * (ptrdiff_t)g.plane);
}

vc_status run_dist_frame(vc_dist* d, const Geo& g, const vc_recon_config* c, bool prof) {
  vc_ctx* c0 = d->r[0].ctx;
  auto each = [&](auto&& fn) -> vc_status {
    for (auto& rk : d->r) {
      vc_ctx* ctx = rk.ctx;
      VC_CUDA(cudaSetDevice(ctx->device));
      VC_TRY(fn(rk, ctx));
      VC_CUDA(cudaGetLastError());
    }
    return VC_OK;
  };
  auto mark = [&](int i) {
    if (prof) record_event(c0->ev[i], c0->st);
  };
  mark(0);
  // P1: preprocess + splat + forward x/y
  VC_TRY(each([&](DistRank& rk, vc_ctx* ctx) -> vc_status {
    if (rk.dirty) {
      launch_clear(P<float4>(ctx->acc), g.plane * g.nzl, ctx->st);
      VC_CUDA(cudaMemsetAsync(ctx->rowbits.p, 0, (size_t)g.ny * g.nzl * sizeof(uint32_t), ctx->st));
      VC_CUDA(cudaMemsetAsync(ctx->rowlist.p, 0, sizeof(int32_t), ctx->st));
      rk.dirty = false;
    } else {  // the previous frame's touched rows (before the preprocess resets the list)
      launch_sparse_clear(P<float4>(ctx->acc), P<uint32_t>(ctx->rowbits), P<int32_t>(ctx->rowlist), g.nx, ctx->st);
    }
    launch_preprocess(ctx->ss, points(ctx), P<float>(ctx->wmaps), P<int32_t>(ctx->pre_scratch), ctx->ctl, g.nx, g.ny,
                      g.nz, c->padding_voxels, c->discontinuity_mm, c->silhouette_radius_px, ctx->st,
                      P<int32_t>(ctx->rowlist));
    launch_splat(points(ctx), ctx->ctl, P<float4>(ctx->acc), P<uint32_t>(ctx->rowbits), P<int32_t>(ctx->rowlist),
                 c->mode, ctx->st, rk.rank * g.nzl, g.nzl);
    return VC_OK;
  }));
  mark(1);
  VC_TRY(each([&](DistRank& rk, vc_ctx*) -> vc_status {
    launch_fft_forward_xy(slab_fft(rk, g, c->mode));
    return VC_OK;
  }));
  mark(2);
  // X1
  VC_TRY(lockstep(d));
  {
    std::vector<const float2*> s0, s1;
    std::vector<float2*> r0, r1;
    std::vector<uint32_t*> pf;
    for (auto& rk : d->r) {
      const SlabFft a = slab_fft(rk, g, c->mode);
      s0.push_back(a.O0), s1.push_back(a.O1), r0.push_back(a.R0), r1.push_back(a.R1);
      pf.push_back(a.planeflag);
    }
    VC_TRY(x_all_to_all(d, s0, r0, g.B));
    VC_TRY(x_all_to_all(d, s1, r1, g.B));
    VC_TRY(x_all_gather_u32(d, pf, (size_t)g.nzl));
  }
  VC_TRY(lockstep(d));
  mark(3);
  // P2
  VC_TRY(each([&](DistRank& rk, vc_ctx*) -> vc_status {
    launch_fft_z(slab_fft(rk, g, c->mode));
    return VC_OK;
  }));
  mark(4);
  // X2
  VC_TRY(lockstep(d));
  {
    std::vector<const float2*> s;
    std::vector<float2*> r;
    for (auto& rk : d->r) {
      const SlabFft a = slab_fft(rk, g, c->mode);
      s.push_back(a.R0), r.push_back(const_cast<float2*>(a.Rin));
    }
    VC_TRY(x_all_to_all(d, s, r, g.B));
  }
  VC_TRY(lockstep(d));
  mark(5);
  // P3
  VC_TRY(each([&](DistRank& rk, vc_ctx*) -> vc_status {
    launch_fft_inverse_yx(slab_fft(rk, g, c->mode));
    return VC_OK;
  }));
  mark(6);
  // X3
  VC_TRY(lockstep(d));
  VC_TRY(x_halo(d, g));
  VC_TRY(lockstep(d));
  // P4
  VC_TRY(each([&](DistRank& rk, vc_ctx* ctx) -> vc_status {
    if (rk.rank + 1 < g.P)
      launch_row_minmax(P<float>(ctx->A) + (size_t)(g.nzl + 1) * g.plane, g.nx, g.ny, 2,
                        P<float2>(ctx->rowmm) + (size_t)g.nzl * g.ny, ctx->st);
    launch_iso_samples(points(ctx), slab_A(rk, g), ctx->ctl, rk.rank * g.nzl, g.nzl, P<double>(rk.samples),
                       ctx->st);
    return VC_OK;
  }));
  // X4
  VC_TRY(lockstep(d));
  {
    std::vector<double*> b;
    for (auto& rk : d->r) b.push_back(P<double>(rk.samples));
    VC_TRY(x_all_reduce_f64(d, b, (size_t)d->r[0].ctx->pts_cap));
  }
  VC_TRY(lockstep(d));
  mark(7);
  // P5
  VC_TRY(each([&](DistRank& rk, vc_ctx* ctx) -> vc_status {
    launch_iso_final_samples(P<double>(rk.samples), ctx->ctl, P<double>(ctx->iso_partial), ctx->st);
    mark(8);
    launch_marching_cubes_count(slab_A(rk, g), ctx->ctl, slab_mesh(rk, g), g.nx, g.ny, g.nz, mc_slab(rk, g),
                                ctx->st);
    VC_CUDA(cudaMemcpyAsync(P<int32_t>(rk.counts) + 3 * rk.rank, &ctx->ctl->V, 3 * sizeof(int32_t),
                            cudaMemcpyDeviceToDevice, ctx->st));
    return VC_OK;
  }));
  // X5
  VC_TRY(lockstep(d));
  {
    std::vector<int32_t*> b;
    for (auto& rk : d->r) b.push_back(P<int32_t>(rk.counts));
    VC_TRY(x_all_gather_i32(d, b, 3));
  }
  VC_TRY(lockstep(d));
  // P6
  VC_TRY(each([&](DistRank& rk, vc_ctx* ctx) -> vc_status {
    launch_mc_set_voff(P<int32_t>(rk.counts), rk.rank, ctx->ctl, ctx->st);
    launch_marching_cubes_emit(slab_A(rk, g), ctx->ctl, slab_mesh(rk, g), g.nx, g.ny, g.nz, mc_slab(rk, g), ctx->st);
    mark(9);
    launch_texture(ctx->ss, P<float>(ctx->wmaps), P<double>(ctx->m_pos), ctx->ctl, c->eps_vis_mm,
                   P<uint8_t>(ctx->t_vis), P<float2>(ctx->t_uv), P<float>(ctx->t_w), P<uint8_t>(ctx->t_untex),
                   P<uint8_t>(ctx->t_rgb), ctx->v_cap, ctx->st, P<float>(ctx->m_posf));
    return VC_OK;
  }));
  mark(10);
  return VC_OK;
}

}  // namespace

extern "C" {

vc_status vc_dist_nccl_unique_id(uint8_t id[128]) {
  if (!id) return VC_ERR_INVALID_ARGUMENT;
  const Nccl* L = nccl_lib(nullptr);
  if (!L) return VC_ERR_NCCL;
  NcclUid u;
  if (L->GetUniqueId(&u) != 0) return VC_ERR_NCCL;
  std::memcpy(id, u.internal, 128);
  return VC_OK;
}

vc_status vc_dist_create_nccl(vc_ctx* ctx, int32_t world, int32_t rank, const uint8_t id[128], vc_dist** out) {
  if (!ctx || !id || !out || world < 1 || rank < 0 || rank >= world)
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "vc_dist_create_nccl: bad arguments");
  *out = nullptr;
  std::string why;
  const Nccl* L = nccl_lib(&why);
  if (!L) return fail(ctx, VC_ERR_NCCL, why);
  VC_CUDA(cudaSetDevice(ctx->device));
  NcclUid u;
  std::memcpy(u.internal, id, 128);
  auto* d = new vc_dist;
  d->world = world;
  d->r.resize(1);
  d->r[0].ctx = ctx;
  d->r[0].rank = rank;
  const int res = L->CommInitRank(&d->r[0].comm, world, u, rank);
  if (res != 0) {
    delete d;
    return fail(ctx, VC_ERR_NCCL, std::string("ncclCommInitRank: ") + L->GetErrorString(res));
  }
  *out = d;
  return VC_OK;
}

vc_status vc_dist_create_loopback(vc_ctx* const* ctxs, int32_t world, vc_dist** out) {
  if (!ctxs || !out || world < 1) return VC_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  for (int i = 0; i < world; ++i)
    if (!ctxs[i]) return VC_ERR_INVALID_ARGUMENT;
  auto* d = new vc_dist;
  d->world = world;
  d->loopback = true;
  d->r.resize(world);
  for (int i = 0; i < world; ++i) d->r[i].ctx = ctxs[i], d->r[i].rank = i;
  *out = d;
  return VC_OK;
}

vc_status vc_dist_destroy(vc_dist* d) {
  if (!d) return VC_OK;
  for (auto& rk : d->r) {
    cudaSetDevice(rk.ctx->device);
    cudaStreamSynchronize(rk.ctx->st);
    if (rk.sd.p) cudaFree(rk.sd.p);
    if (rk.samples.p) cudaFree(rk.samples.p);
    if (rk.counts.p) cudaFree(rk.counts.p);
    if (rk.comm) {
      const Nccl* L = nccl_lib(nullptr);
      if (L) L->CommDestroy(rk.comm);
    }
  }
  delete d;
  return VC_OK;
}

int32_t vc_dist_local_ranks(const vc_dist* d) { return d ? (int32_t)d->r.size() : 0; }

vc_status vc_reconstruct_frame_dist(vc_dist* d, const vc_sensor* sensors, const vc_view* views, int32_t k,
                                    const vc_recon_config* config, vc_textured_mesh* out, vc_dist_info* info,
                                    vc_stage_timings* timings) {
  if (!d || d->r.empty()) return VC_ERR_INVALID_ARGUMENT;
  vc_ctx* ctx = d->r[0].ctx;
  if (!views || !config || !out) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "null argument");
  VC_TRY(check_sensors(ctx, sensors, k));
  Geo g;
  VC_TRY(resolve_dims(ctx, config, &g.nx, &g.ny, &g.nz));
  g.P = d->world;
  if (g.nz % g.P || g.ny % g.P || g.nz / g.P < 2)
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "slab decomposition: nz, ny must be multiples of world, nz/world >= 2");
  g.nzl = g.nz / g.P, g.kyl = g.ny / g.P, g.H = (int)hp(g.nx);
  g.plane = (size_t)g.nx * g.ny;
  g.E = hp(g.nx) * g.ny * g.nzl;
  g.B = hp(g.nx) * g.kyl * g.nzl;
  for (auto& rk : d->r) VC_TRY(ensure_rank(rk, g, sensors, views, k));
  const bool prof = timings != nullptr;
  for (int attempt = 0; attempt < 2; ++attempt) {
    VC_TRY(run_dist_frame(d, g, config, prof));
    bool overflow = false;
    for (auto& rk : d->r) {
      vc_ctx* cx = rk.ctx;
      rk.counts_h.resize(3 * g.P);
      cudaSetDevice(cx->device);
      VC_CUDA(cudaMemcpyAsync(rk.counts_h.data(), rk.counts.p, 3 * g.P * sizeof(int32_t), cudaMemcpyDeviceToHost,
                              cx->st));
      VC_TRY(read_ctl(cx));
      const DevCtl& c = *cx->ctl_h;
      if (c.status == 2) return fail(ctx, VC_ERR_EMPTY_SCENE, "reconstruct_frame: empty foreground in all views");
      if (c.status != 0) return fail(ctx, VC_ERR_CUDA, "preprocess failed");
      if (c.overflow) {
        overflow = true;
        const int want = std::max(c.V + c.v_extra, std::max(c.C, c.T / 2)) * 2;
        VC_TRY(ensure_mesh_caps(cx, want, kMaxViews));
      }
    }
    // every rank stops before the emit on overflow anywhere only locally;
    // re-run the frame with the grown capacities (all ranks, lockstep)
    if (!overflow) break;
    if (attempt == 1) return fail(ctx, VC_ERR_CAPACITY, "marching cubes capacity");
  }
  for (size_t i = 0; i < d->r.size(); ++i) {
    DistRank& rk = d->r[i];
    vc_ctx* cx = rk.ctx;
    const DevCtl& c = *cx->ctl_h;
    vc_textured_mesh& o = out[i];
    std::memset(&o, 0, sizeof(o));
    o.vertex_count = c.V, o.triangle_count = c.T, o.sensor_count = k, o.point_count = c.P;
    o.iso_level = c.level;
    o.grid.nx = g.nx, o.grid.ny = g.ny, o.grid.nz = g.nz;
    for (int a = 0; a < 3; ++a) o.grid.origin[a] = c.grid.origin[a];
    o.grid.edge_mm = c.grid.edge;
    o.mem_kind = cx->out_kind;
    VC_TRY(copy_out(cx, c.V, c.T, k, &o));
    if (info) {
      vc_dist_info& in = info[i];
      in.rank = rk.rank, in.world = g.P;
      in.z_begin = rk.rank * g.nzl, in.z_end = (rk.rank + 1) * g.nzl;
      in.vertex_offset = c.voff;
      in.vertex_total = 0, in.triangle_offset = 0, in.triangle_total = 0;
      for (int s = 0; s < g.P; ++s) {
        in.vertex_total += rk.counts_h[3 * s];
        if (s < rk.rank) in.triangle_offset += rk.counts_h[3 * s + 1];
        in.triangle_total += rk.counts_h[3 * s + 1];
      }
    }
  }
  for (auto& rk : d->r) VC_CUDA(cudaStreamSynchronize(rk.ctx->st));
  if (timings) {
    std::memset(timings, 0, sizeof(*timings));
    timings->raw_ms = ev_ms(ctx, 0, 1);  // preprocess + clear + splat
    timings->splat_ms = 0.0;
    timings->fft_ms = ev_ms(ctx, 1, 6);  // x/y, all-to-all, z, all-to-all, y/x
    timings->iso_ms = ev_ms(ctx, 6, 8);  // halo + samples + all-reduce + level
    timings->mc_ms = ev_ms(ctx, 8, 9);
    timings->texture_ms = ev_ms(ctx, 9, 10);
    timings->volumetric_ms = ev_ms(ctx, 1, 9);
    timings->total_ms = ev_ms(ctx, 0, 10);
  }
  return VC_OK;
}

vc_status vc_dist_export_volume(vc_dist* d, int32_t local_rank, float* dst, int32_t kind) {
  if (!d || local_rank < 0 || local_rank >= (int)d->r.size() || !dst) return VC_ERR_INVALID_ARGUMENT;
  DistRank& rk = d->r[local_rank];
  vc_ctx* ctx = rk.ctx;
  const int nx = rk.dims[0], ny = rk.dims[1], nz = rk.dims[2];
  if (!nx) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "no frame");
  const size_t plane = (size_t)nx * ny, nzl = (size_t)nz / d->world;
  VC_CUDA(cudaMemcpyAsync(dst, P<float>(ctx->A) + plane, plane * nzl * sizeof(float),
                          kind == VC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}

}  // extern "C"

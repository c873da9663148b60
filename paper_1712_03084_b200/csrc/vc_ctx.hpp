// SPDX-License-Identifier: Apache-2.0
//
// Internal: the context object behind vc_ctx* and the runtime helpers shared
// by vc_runtime.cpp (one GPU) and vc_dist.cpp (z-slab decomposition).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "vc/vc.h"
#include "vc_shared.hpp"

namespace vc::rt {

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

constexpr int kEvents = 24;
constexpr int kKernelGroups = 13;  // events 12..24 bracket the kernel groups

}  // namespace vc::rt

struct vc_ctx {
  using Buf = vc::rt::Buf;
  using HostBuf = vc::rt::HostBuf;
  static constexpr int kEvents = vc::rt::kEvents;
  int device = 0;
  cudaStream_t st = nullptr;
  cudaStream_t aux = nullptr;        // side stream: branches of the frame graph
  cudaStream_t cst = nullptr;        // copy stream: the views' RGB, staged while the frame computes
  cudaEvent_t rgb_ev = nullptr;      // recorded once the views' RGB is staged (the texture stage waits on it)
  bool rgb_async = false;            // stage_views: RGB on cst (vc_reconstruct_frame only)
  cudaEvent_t fork[2] = {}, join[2] = {};
  std::string err;
  int out_kind = VC_MEM_HOST;
  bool profiling = false;
  bool graphs = true;

  // grid-dependent
  int nx = 0, ny = 0, nz = 0;
  Buf acc, spec, A, tw, vbase, blk, rowmm, units, unitcnt, ucmask, rowbits, planeflag, rowlist, vinfo;
  bool acc_dirty = true;  // accumulator contents unknown: next frame clears densely
  int layout = 0;         // what acc/rowbits/rowlist hold: 1 whole-grid frame, 2 z-slab frame
  // view staging + clouds
  Buf views, pts_pos, pts_nrm, pts_w, pts_pix, wmaps, pre_scratch, iso_partial;
  int pts_cap = 0;
  vc::SensorSet ss{};
  // control block
  vc::DevCtl* ctl = nullptr;
  vc::DevCtl* ctl_h = nullptr;
  // mesh + texture
  Buf m_pos, m_nrm, m_tri, m_eid, m_cells, m_celltri, m_cellcfg, m_posf, t_vis, t_uv, t_w, t_untex, t_rgb;
  int v_cap = 0, t_cap = 0, c_cap = 0;
  int spec_v = 0, spec_t = 0;  // host output: sizes copied speculatively behind the next frame
  // host outputs (pinned)
  HostBuf h_posf, h_nrm, h_tri, h_vis, h_uv, h_w, h_untex, h_rgb, h_pos, h_eid;
  // stage-API host scratch, device scratch of the colour-correction entry points
  Buf scratch_dev, scratch_dev2;
  Buf skel_lut;  // 2^26-bit simple-point table of vc_skeletonize
  bool skel_lut_ready = false;
  std::vector<uint8_t> scratch;
  // graph
  cudaGraphExec_t gexec = nullptr;
  std::vector<uint8_t> gkey;
  cudaEvent_t ev[kEvents] = {};
  bool table_ready = false;
  int last_k = 0;
  std::vector<double> cc_gain, cc_offset;
  // optional depth filter applied to every staged view (off: all zero)
  int df_erode = 0;
  double df_sigma_px = 0.0, df_sigma_mm = 0.0;
  Buf df_scratch;  // per-sensor colour correction of the texture blend (empty: off)
  int kernels_per_frame = 0;
};
namespace vc::rt {

using namespace vc;

template <class T>
T* P(const Buf& b) {
  return static_cast<T*>(b.p);
}

struct FrameCfg {
  int nx, ny, nz, mode, pad, sil_r;
  double disc, eps_vis;
};

vc_status fail(vc_ctx* c, vc_status s, const std::string& msg);
vc_status ensure(vc_ctx* ctx, Buf& b, size_t bytes);
vc_status ensure_host(vc_ctx* ctx, HostBuf& b, size_t bytes);
bool pow2_ok(int n);
vc_status check_sensors(vc_ctx* ctx, const vc_sensor* s, int k);
vc_status stage_views(vc_ctx* ctx, const vc_sensor* sensors, const vc_view* views, int k, bool need_rgb);
vc_status setup_sensorset(vc_ctx* ctx, const vc_sensor* sensors, int k);
DevPoints points(vc_ctx* ctx);
vc_status ensure_tables(vc_ctx* ctx);
vc_status ensure_mesh_caps(vc_ctx* ctx, int v_cap, int k);
vc_status ensure_mc_scratch(vc_ctx* ctx, int nx, int ny, int nz);
MeshBufs mesh_bufs(vc_ctx* ctx);
vc_status resolve_dims(vc_ctx* ctx, const vc_recon_config* c, int* nx, int* ny, int* nz);
float ev_ms(vc_ctx* ctx, int a, int b);
vc_status read_ctl(vc_ctx* ctx);
vc_status copy_out(vc_ctx* ctx, int V, int T, int k, vc_textured_mesh* out);

}  // namespace vc::rt

#define VC_CUDA(call)                                                                             \
  do {                                                                                            \
    const cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                      \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? VC_ERR_OOM : VC_ERR_CUDA,                \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                            \
    }                                                                                             \
  } while (0)

#define VC_TRY(expr)                  \
  do {                                \
    const vc_status s_ = (expr);      \
    if (s_ != VC_OK) return s_;       \
  } while (0)


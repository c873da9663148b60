// SPDX-License-Identifier: Apache-2.0
//
// Host runtime of the B200 FTR path behind the C-ABI in include/vc/vc.h:
// context (device, stream, pooled HBM buffers, pinned staging), the frame
// orchestration of recon::reconstruct_frame (reconstruct.cpp:37-78) +
// vertex_visibility / assign_texture (texture.cpp:11-72) as one CUDA graph
// with no host synchronisation until the single control-block read-back,
// marching-cubes capacity retry, CUDA-event stage timings and the
// per-stage entry points used by the parity tests.
//
// Built with -ffp-contract=off: the host-side pose algebra (Pose::inverse,
// Pose::compose, types.hpp:46-49) must round like the reference.
#include <atomic>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "vc/vc.h"
#include "vc_ctx.hpp"

namespace vc {
void circle_rig(int recon, int held_out, double radius, double target_h, int w, int h, double f, vc_sensor* out);
void xpose_body(vc_body* b);
void kick_body(int frames, int f, vc_body* b);
}  // namespace vc

using namespace vc;

namespace vc::rt {

vc_status fail(vc_ctx* c, vc_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

vc_status ensure(vc_ctx* ctx, Buf& b, size_t bytes) {
  if (b.bytes >= bytes && b.p) return VC_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  const size_t want = std::max<size_t>(bytes, 256);
  VC_CUDA(cudaMalloc(&b.p, want));
  b.bytes = want;
  if (ctx->gexec) {  // pointers baked into the graph changed
    cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
  }
  return VC_OK;
}

vc_status ensure_host(vc_ctx* ctx, HostBuf& b, size_t bytes) {
  if (b.bytes >= bytes && b.p) return VC_OK;
  if (b.p) cudaFreeHost(b.p);
  b.p = nullptr;
  b.bytes = 0;
  const size_t want = std::max<size_t>(bytes * 5 / 4, 4096);
  VC_CUDA(cudaHostAlloc(&b.p, want, cudaHostAllocDefault));
  b.bytes = want;
  return VC_OK;
}

bool pow2_ok(int n) { return n >= 4 && n <= 1024 && (n & (n - 1)) == 0; }

// types.hpp:48 Pose::inverse = {R^T, -(R^T t)}; types.hpp:49 compose.
void fill_sensor(const vc_sensor& in, DevSensor& o) {
  o.fx = in.depth_intr.fx, o.fy = in.depth_intr.fy, o.cx = in.depth_intr.cx, o.cy = in.depth_intr.cy;
  o.w = in.depth_intr.width, o.h = in.depth_intr.height;
  for (int i = 0; i < 9; ++i) o.R[i] = in.pose.R[i];
  for (int i = 0; i < 3; ++i) o.t[i] = in.pose.t[i];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o.Ri[r * 3 + c] = in.pose.R[c * 3 + r];
  for (int r = 0; r < 3; ++r)
    o.ti[r] = -((o.Ri[r * 3 + 0] * in.pose.t[0] + o.Ri[r * 3 + 1] * in.pose.t[1]) + o.Ri[r * 3 + 2] * in.pose.t[2]);
  o.rfx = in.rgb_intr.fx, o.rfy = in.rgb_intr.fy, o.rcx = in.rgb_intr.cx, o.rcy = in.rgb_intr.cy;
  o.rw = in.rgb_intr.width, o.rh = in.rgb_intr.height;
  const double* A = in.pose.R;
  const double* B = in.rgb_relative.R;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o.Rc[r * 3 + c] = (A[r * 3 + 0] * B[c] + A[r * 3 + 1] * B[3 + c]) + A[r * 3 + 2] * B[6 + c];
  for (int r = 0; r < 3; ++r)
    o.tc[r] = ((A[r * 3 + 0] * in.rgb_relative.t[0] + A[r * 3 + 1] * in.rgb_relative.t[1]) +
               A[r * 3 + 2] * in.rgb_relative.t[2]) +
              in.pose.t[r];
}

vc_status check_sensors(vc_ctx* ctx, const vc_sensor* s, int k) {
  if (!s || k < 1 || k > kMaxViews) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "need 1..16 sensors");
  for (int i = 0; i < k; ++i) {
    const auto& d = s[i].depth_intr;
    const auto& r = s[i].rgb_intr;
    if (d.width <= 0 || d.height <= 0 || r.width <= 0 || r.height <= 0 || d.fx <= 0 || d.fy <= 0 || r.fx <= 0 ||
        r.fy <= 0)
      return fail(ctx, VC_ERR_INVALID_ARGUMENT, "Intrinsics: focal lengths / image sizes must be positive");
    if (d.width > 8192) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "depth width > 8192");
  }
  return VC_OK;
}

// Stage the k views into context-owned device buffers (graph-stable addresses).
vc_status stage_views(vc_ctx* ctx, const vc_sensor* sensors, const vc_view* views, int k, bool need_rgb) {
  size_t bytes = 0;
  std::vector<size_t> off(3 * k);
  for (int i = 0; i < k; ++i) {
    const size_t n = (size_t)sensors[i].depth_intr.width * sensors[i].depth_intr.height;
    const size_t nr = (size_t)sensors[i].rgb_intr.width * sensors[i].rgb_intr.height * 3;
    off[3 * i] = bytes;
    bytes += (n * 2 + 255) & ~size_t(255);
    off[3 * i + 1] = bytes;
    bytes += (n + 255) & ~size_t(255);
    off[3 * i + 2] = bytes;
    bytes += (nr + 255) & ~size_t(255);
  }
  VC_TRY(ensure(ctx, ctx->views, bytes));
  uint8_t* base = P<uint8_t>(ctx->views);
  // Views laid out exactly like the staging buffer (same order, tight rows,
  // the segment offsets above, one memory kind): one copy for all of them.
  bool contiguous = true;
  const uint8_t* h0 = reinterpret_cast<const uint8_t*>(views[0].depth);
  for (int i = 0; i < k && contiguous; ++i) {
    const vc_view& v = views[i];
    const int w = sensors[i].depth_intr.width, rw = sensors[i].rgb_intr.width;
    contiguous = v.depth && v.mask && (v.rgb || !need_rgb) && v.mem_kind == views[0].mem_kind &&
                 reinterpret_cast<const uint8_t*>(v.depth) == h0 + off[3 * i] && v.mask == h0 + off[3 * i + 1] &&
                 (!need_rgb || v.rgb == h0 + off[3 * i + 2]) && (!v.depth_pitch || v.depth_pitch == w * 2) &&
                 (!v.mask_pitch || v.mask_pitch == w) && (!v.rgb_pitch || v.rgb_pitch == rw * 3);
  }
  // RGB is first read by the texture stage at the end of the frame: with
  // rgb_async it is staged on the copy stream while the frame computes (the
  // texture stage waits on rgb_ev); depth and mask go first, on the frame stream.
  const bool split_rgb = ctx->rgb_async && need_rgb;
  if (contiguous) {
    const cudaMemcpyKind kind0 = views[0].mem_kind == VC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (split_rgb) {
      for (int i = 0; i < k; ++i) {
        const size_t n = (size_t)sensors[i].depth_intr.width * sensors[i].depth_intr.height;
        VC_CUDA(cudaMemcpyAsync(base + off[3 * i], h0 + off[3 * i], off[3 * i + 1] - off[3 * i] + n, kind0, ctx->st));
        VC_CUDA(cudaMemcpyAsync(base + off[3 * i + 2], h0 + off[3 * i + 2],
                                (size_t)sensors[i].rgb_intr.width * sensors[i].rgb_intr.height * 3, kind0, ctx->cst));
      }
    } else {
      const size_t last = need_rgb ? off[3 * k - 1] + (size_t)sensors[k - 1].rgb_intr.width *
                                                           sensors[k - 1].rgb_intr.height * 3
                                   : off[3 * k - 2] + (size_t)sensors[k - 1].depth_intr.width *
                                                          sensors[k - 1].depth_intr.height;
      VC_CUDA(cudaMemcpyAsync(base, h0, last, kind0, ctx->st));
    }
  }
  for (int i = 0; i < k; ++i) {
    const int w = sensors[i].depth_intr.width, h = sensors[i].depth_intr.height;
    const int rw = sensors[i].rgb_intr.width, rh = sensors[i].rgb_intr.height;
    const vc_view& v = views[i];
    if (!v.depth) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "view depth missing");
    const cudaMemcpyKind kind = v.mem_kind == VC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (!contiguous)
      VC_CUDA(cudaMemcpy2DAsync(base + off[3 * i], (size_t)w * 2, v.depth,
                                v.depth_pitch ? v.depth_pitch : (size_t)w * 2, (size_t)w * 2, h, kind, ctx->st));
    if (contiguous) {
    } else if (v.mask) {
      VC_CUDA(cudaMemcpy2DAsync(base + off[3 * i + 1], (size_t)w, v.mask, v.mask_pitch ? v.mask_pitch : (size_t)w,
                                (size_t)w, h, kind, ctx->st));
    } else {  // the dataset loader's foreground := depth > 0 (dataset.cpp:99-102), on the device
      launch_mask_from_depth(reinterpret_cast<const uint16_t*>(base + off[3 * i]), base + off[3 * i + 1], w * h,
                             ctx->st);
      VC_CUDA(cudaGetLastError());
    }
    if (v.rgb && need_rgb && !contiguous)
      VC_CUDA(cudaMemcpy2DAsync(base + off[3 * i + 2], (size_t)rw * 3, v.rgb, v.rgb_pitch ? v.rgb_pitch : (size_t)rw * 3,
                                (size_t)rw * 3, rh, kind, split_rgb ? ctx->cst : ctx->st));
    ViewPtrs& vp = ctx->ss.v[i];
    vp.depth = reinterpret_cast<const uint16_t*>(base + off[3 * i]);
    vp.mask = base + off[3 * i + 1];
    vp.rgb = (v.rgb && need_rgb) ? base + off[3 * i + 2] : nullptr;
    vp.dpitch = w, vp.mpitch = w, vp.rpitch = rw * 3;
  }
  VC_CUDA(cudaEventRecord(ctx->rgb_ev, split_rgb ? ctx->cst : ctx->st));
  if (ctx->df_erode > 0 || (depth_filter_radius(ctx->df_sigma_px) > 0 && ctx->df_sigma_mm > 0))
    for (int i = 0; i < k; ++i) {  // optional depth filter, in place on the staged views
      const int w = sensors[i].depth_intr.width, h = sensors[i].depth_intr.height;
      VC_TRY(ensure(ctx, ctx->df_scratch, (size_t)w * h * 3 + 512));
      uint8_t* s8 = P<uint8_t>(ctx->df_scratch);
      launch_depth_filter(reinterpret_cast<uint16_t*>(base + off[3 * i]), base + off[3 * i + 1], w, h, ctx->df_erode,
                          ctx->df_sigma_px, ctx->df_sigma_mm, s8,
                          reinterpret_cast<uint16_t*>(s8 + (((size_t)w * h + 255) & ~size_t(255))), ctx->st);
      VC_CUDA(cudaGetLastError());
    }
  return VC_OK;
}

vc_status setup_sensorset(vc_ctx* ctx, const vc_sensor* sensors, int k) {
  SensorSet& ss = ctx->ss;
  ss.k = k;
  ss.pix_offset[0] = 0;
  ss.row_offset[0] = 0;
  for (int i = 0; i < k; ++i) {
    fill_sensor(sensors[i], ss.s[i]);
    const bool cc = i < (int)ctx->cc_gain.size();
    ss.s[i].cc_on = cc ? 1 : 0;
    ss.s[i].cc_gain = cc ? ctx->cc_gain[i] : 1.0, ss.s[i].cc_offset = cc ? ctx->cc_offset[i] : 0.0;
    ss.pix_offset[i + 1] = ss.pix_offset[i] + (int64_t)sensors[i].depth_intr.width * sensors[i].depth_intr.height;
    ss.row_offset[i + 1] = ss.row_offset[i] + sensors[i].depth_intr.height;
  }
  const int64_t npix = ss.pix_offset[k];
  VC_TRY(ensure(ctx, ctx->pts_pos, npix * 3 * sizeof(double)));
  VC_TRY(ensure(ctx, ctx->pts_nrm, npix * 3 * sizeof(double)));
  VC_TRY(ensure(ctx, ctx->pts_w, npix * sizeof(double)));
  VC_TRY(ensure(ctx, ctx->pts_pix, npix * 3 * sizeof(int32_t)));
  VC_TRY(ensure(ctx, ctx->wmaps, npix * sizeof(float)));
  VC_TRY(ensure(ctx, ctx->pre_scratch, preprocess_scratch_bytes(ss)));
  prepare_preprocess(ss);
  VC_CUDA(cudaGetLastError());
  ctx->pts_cap = (int)npix;
  ctx->last_k = k;
  return VC_OK;
}

DevPoints points(vc_ctx* ctx) {
  return DevPoints{P<double>(ctx->pts_pos), P<double>(ctx->pts_nrm), P<double>(ctx->pts_w), P<int32_t>(ctx->pts_pix),
                   ctx->pts_cap};
}

vc_status ensure_tables(vc_ctx* ctx) {
  if (ctx->table_ready) return VC_OK;
  int8_t counts[256], tris[256][5][3];
  build_mc_table(counts, tris);
  upload_case_table_data(counts, &tris[0][0][0], ctx->st);
  VC_CUDA(cudaGetLastError());
  ctx->table_ready = true;
  return VC_OK;
}

vc_status ensure_mesh_caps(vc_ctx* ctx, int v_cap, int k) {
  const int t_cap = 2 * v_cap + 1024, c_cap = v_cap;
  VC_TRY(ensure(ctx, ctx->m_pos, (size_t)v_cap * 3 * sizeof(double)));
  VC_TRY(ensure(ctx, ctx->m_nrm, (size_t)v_cap * 3 * sizeof(float)));
  VC_TRY(ensure(ctx, ctx->m_posf, (size_t)v_cap * 3 * sizeof(float)));
  VC_TRY(ensure(ctx, ctx->m_eid, (size_t)v_cap * sizeof(uint64_t)));
  VC_TRY(ensure(ctx, ctx->m_tri, (size_t)t_cap * 3 * sizeof(int32_t)));
  VC_TRY(ensure(ctx, ctx->m_cells, (size_t)c_cap * sizeof(int32_t)));
  VC_TRY(ensure(ctx, ctx->m_celltri, (size_t)c_cap * sizeof(int32_t)));
  VC_TRY(ensure(ctx, ctx->m_cellcfg, (size_t)c_cap));
  VC_TRY(ensure(ctx, ctx->t_vis, (size_t)v_cap * k));
  VC_TRY(ensure(ctx, ctx->t_uv, (size_t)v_cap * k * sizeof(float2)));
  VC_TRY(ensure(ctx, ctx->t_w, (size_t)v_cap * k * sizeof(float)));
  VC_TRY(ensure(ctx, ctx->t_untex, (size_t)v_cap));
  VC_TRY(ensure(ctx, ctx->t_rgb, (size_t)v_cap * 3));
  ctx->v_cap = v_cap, ctx->t_cap = t_cap, ctx->c_cap = c_cap;
  return VC_OK;
}

vc_status ensure_mc_scratch(vc_ctx* ctx, int nx, int ny, int nz) {
  (void)nx;
  const size_t rows = (size_t)ny * nz;
  VC_TRY(ensure(ctx, ctx->blk, (size_t)mc_blocks(nx, ny, nz) * sizeof(int32_t)));
  VC_TRY(ensure(ctx, ctx->rowmm, rows * sizeof(float2)));
  VC_TRY(ensure(ctx, ctx->units, rows * sizeof(int32_t)));
  VC_TRY(ensure(ctx, ctx->unitcnt, rows * 3 * sizeof(int32_t)));
  VC_TRY(ensure(ctx, ctx->ucmask, rows * sizeof(uint32_t)));
  VC_TRY(ensure(ctx, ctx->vinfo, rows * (size_t)nx * sizeof(uint16_t)));
  return VC_OK;
}

vc_status ensure_grid(vc_ctx* ctx, int nx, int ny, int nz) {
  const size_t N = (size_t)nx * ny * nz;
  const void* acc_before = ctx->acc.p;
  VC_TRY(ensure(ctx, ctx->acc, N * sizeof(float4)));
  VC_TRY(ensure(ctx, ctx->rowbits, (size_t)ny * nz * sizeof(uint32_t)));
  VC_TRY(ensure(ctx, ctx->rowlist, ((size_t)ny * nz + 1) * sizeof(int32_t)));
  VC_TRY(ensure(ctx, ctx->planeflag, (size_t)(2 * nz + 2) * sizeof(uint32_t) + 256));  // flags + F-y's live-plane list
  if (ctx->acc.p != acc_before || ctx->nx != nx || ctx->ny != ny || ctx->nz != nz || ctx->layout != 1)
    ctx->acc_dirty = true;
  ctx->layout = 1;
  VC_TRY(ensure(ctx, ctx->spec, 3 * spectrum_elems(nx, ny, nz) * sizeof(float2)));
  VC_TRY(ensure(ctx, ctx->A, N * sizeof(float)));
  VC_TRY(ensure(ctx, ctx->vbase, N * sizeof(uint32_t)));
  VC_TRY(ensure_mc_scratch(ctx, nx, ny, nz));
  VC_TRY(ensure(ctx, ctx->tw, twiddle_elems(nx, ny, nz) * sizeof(float2)));
  VC_TRY(ensure(ctx, ctx->iso_partial, 1024 * sizeof(double)));
  if (ctx->nx != nx || ctx->ny != ny || ctx->nz != nz) {
    upload_twiddles(P<float2>(ctx->tw), nx, ny, nz, ctx->st);
    prepare_integrate(nx, ny, nz);
    VC_CUDA(cudaGetLastError());
    ctx->nx = nx, ctx->ny = ny, ctx->nz = nz;
  }
  if (ctx->v_cap == 0) {
    const int v_cap = (int)std::min<size_t>(std::max<size_t>(N / 16, 1 << 16), (size_t)1 << 26);
    VC_TRY(ensure_mesh_caps(ctx, v_cap, kMaxViews));
  }
  return VC_OK;
}

MeshBufs mesh_bufs(vc_ctx* ctx) {
  MeshBufs mb;
  mb.pos = P<double>(ctx->m_pos);
  mb.nrm = P<float>(ctx->m_nrm);
  mb.tri = P<int32_t>(ctx->m_tri);
  mb.edge_id = P<uint64_t>(ctx->m_eid);
  mb.vbase = P<uint32_t>(ctx->vbase);
  mb.cells = P<int32_t>(ctx->m_cells);
  mb.cell_tri = P<int32_t>(ctx->m_celltri);
  mb.cell_cfg = P<uint8_t>(ctx->m_cellcfg);
  mb.vinfo = P<uint16_t>(ctx->vinfo);
  mb.v_cap = ctx->v_cap, mb.t_cap = ctx->t_cap, mb.c_cap = ctx->c_cap;
  mb.blk = P<int32_t>(ctx->blk);
  mb.nblk = 0;
  mb.rowmm = P<float2>(ctx->rowmm);
  mb.units = P<int32_t>(ctx->units);
  mb.unitcnt = P<int32_t>(ctx->unitcnt);
  mb.ucmask = P<uint32_t>(ctx->ucmask);
  return mb;
}

void record(vc_ctx* ctx, int i) {
  if (ctx->profiling) record_event(ctx->ev[i], ctx->st);
}

// The frame's kernel sequence (captured once into a CUDA graph).  With
// profiling on, events 0..6 bracket the reference's stage split and events
// Contexts alive per device (frame graphs choose their shape from it).
std::atomic<int> g_live_ctx[64];

// 12..23 bracket every kernel group (vc_ctx_kernel_times).
int enqueue_frame(vc_ctx* ctx, const FrameCfg& f) {
  cudaStream_t st = ctx->st;
  int n = 0;
  // No clear pass: the previous frame's F-x zeroed the accumulator chunks it
  // read and its I-x reset their bits.  The preprocess's gather pass resets
  // the touched-row list for this frame's splat.  Graph branch (not in
  // profiled frames, which time each kernel on one stream): the MC normals
  // and triangles beside the texturing.
  const bool branch = !ctx->profiling && ctx->aux;
  // A side branch at the frame's start (the touched-row list's reset beside
  // the preprocess) when several contexts share the device: measured, a
  // linear frame graph loses 10% of the four-frames-in-flight throughput
  // (4700 against 5230 frames/s) but runs a lone frame 4% faster (3510
  // against 3370) — profiles/r02_experiments.json "graph_root_branch".
  // VC_ROOT_BRANCH=0/1 forces either shape.
  static const int root_branch_env = [] {
    const char* e = getenv("VC_ROOT_BRANCH");
    return e ? atoi(e) : -1;
  }();
  const bool root_branch = root_branch_env >= 0 ? root_branch_env != 0
                                                : (ctx->device < 64 && g_live_ctx[ctx->device].load() > 1);
  record(ctx, 12);
  // the touched-row list's reset rides on a side branch beside the preprocess:
  // with one root branch the frame graphs of concurrent contexts interleave
  // better (measured: a linear graph lost 10% of the S = 4 throughput)
  const bool rb = branch && root_branch;
  if (rb) {
    cudaEventRecord(ctx->fork[0], st);
    cudaStreamWaitEvent(ctx->aux, ctx->fork[0], 0);
    launch_reset_rowlist(P<int32_t>(ctx->rowlist), ctx->aux);  // a kernel node (a memset node here tripped ncu)
    n += 1;
    cudaEventRecord(ctx->join[0], ctx->aux);
  }
  record(ctx, 13);
  record(ctx, 0);
  launch_preprocess(ctx->ss, points(ctx), P<float>(ctx->wmaps), P<int32_t>(ctx->pre_scratch), ctx->ctl, f.nx, f.ny,
                    f.nz, f.pad, f.disc, f.sil_r, st, rb ? nullptr : P<int32_t>(ctx->rowlist));
  if (rb) cudaStreamWaitEvent(st, ctx->join[0], 0);
  n += 3;  // prefix + triangles, points, gather
  record(ctx, 1);
  launch_splat(points(ctx), ctx->ctl, P<float4>(ctx->acc), P<uint32_t>(ctx->rowbits), P<int32_t>(ctx->rowlist),
               f.mode, st, 0, f.nz);
  n += 2;  // splat, row-list build
  record(ctx, 2);
  launch_integrate(P<float4>(ctx->acc), P<float2>(ctx->spec), P<float>(ctx->A), f.nx, f.ny, f.nz, f.mode,
                   P<float2>(ctx->tw), st, ctx->profiling ? &ctx->ev[14] : nullptr, P<float2>(ctx->rowmm),
                   P<uint32_t>(ctx->rowbits), P<uint32_t>(ctx->planeflag), P<int32_t>(ctx->rowlist));
  n += 5;
  record(ctx, 3);
  launch_iso_level(points(ctx), P<float>(ctx->A), ctx->ctl, P<double>(ctx->iso_partial), 1024, st);
  n += 1;
  record(ctx, 4);
  launch_marching_cubes(P<float>(ctx->A), ctx->ctl, mesh_bufs(ctx), f.nx, f.ny, f.nz, st, branch ? ctx->aux : nullptr,
                        ctx->fork[1], ctx->join[1]);
  n += 4;  // active units, count, scan + emit, normals + triangles
  record(ctx, 5);
  {  // the views' RGB (staged on the copy stream while the frame ran): an external event node in the graph
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    cudaStreamWaitEvent(st, ctx->rgb_ev, cs == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0);
  }
  launch_texture(ctx->ss, P<float>(ctx->wmaps), P<double>(ctx->m_pos), ctx->ctl, f.eps_vis, P<uint8_t>(ctx->t_vis),
                 P<float2>(ctx->t_uv), P<float>(ctx->t_w), P<uint8_t>(ctx->t_untex), P<uint8_t>(ctx->t_rgb),
                 ctx->v_cap, st, P<float>(ctx->m_posf));
  n += 1;
  if (branch) cudaStreamWaitEvent(st, ctx->join[1], 0);  // the normals branch rejoins
  record(ctx, 6);
  return n;
}

vc_status run_frame(vc_ctx* ctx, const FrameCfg& f) {
  if (ctx->acc_dirty) {  // outside the graph: dense clear once, then sparse clears
    launch_clear(P<float4>(ctx->acc), (size_t)f.nx * f.ny * f.nz, ctx->st);
    VC_CUDA(cudaMemsetAsync(ctx->rowbits.p, 0, (size_t)f.ny * f.nz * sizeof(uint32_t), ctx->st));
    VC_CUDA(cudaMemsetAsync(ctx->rowlist.p, 0, sizeof(int32_t), ctx->st));  // empty touched-row list
    VC_CUDA(cudaGetLastError());
    ctx->acc_dirty = false;
  }
  if (!ctx->graphs || ctx->profiling) {  // profiled frames: direct launches + events
    ctx->kernels_per_frame = enqueue_frame(ctx, f);
    VC_CUDA(cudaGetLastError());
    return VC_OK;
  }
  // graph key: everything baked into the kernels' parameters
  std::vector<uint8_t> key(sizeof(SensorSet) + sizeof(FrameCfg) + 16);
  std::memcpy(key.data(), &ctx->ss, sizeof(SensorSet));
  std::memcpy(key.data() + sizeof(SensorSet), &f, sizeof(FrameCfg));
  key[sizeof(SensorSet) + sizeof(FrameCfg)] = ctx->profiling ? 1 : 0;
  if (!ctx->gexec || key != ctx->gkey) {
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
    cudaGraph_t g;
    VC_CUDA(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
    ctx->kernels_per_frame = enqueue_frame(ctx, f);
    const cudaError_t le = cudaGetLastError();
    const cudaError_t ce = cudaStreamEndCapture(ctx->st, &g);
    VC_CUDA(le);
    VC_CUDA(ce);
    VC_CUDA(cudaGraphInstantiate(&ctx->gexec, g, 0));
    cudaGraphDestroy(g);
    ctx->gkey = key;
  }
  VC_CUDA(cudaGraphLaunch(ctx->gexec, ctx->st));
  return VC_OK;
}

vc_status resolve_dims(vc_ctx* ctx, const vc_recon_config* c, int* nx, int* ny, int* nz) {
  if (c->r > 0) {
    if (c->r > 9) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "r must be <= 9");
    *nx = 1 << c->r, *ny = 1 << (c->r + 1), *nz = 1 << c->r;
  } else {
    *nx = c->nx, *ny = c->ny, *nz = c->nz;
  }
  if (!pow2_ok(*nx) || !pow2_ok(*ny) || !pow2_ok(*nz))
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "grid dims must be powers of two in [4, 1024]");
  const int d[3] = {*nx, *ny, *nz};
  for (int a = 0; a < 3; ++a)
    if (d[a] - 1 - 2 * c->padding_voxels < 1)
      return fail(ctx, VC_ERR_INVALID_ARGUMENT, "fit_grid: padding leaves no usable voxels");  // reconstruct.cpp:25-26
  if (c->mode != VC_SPLAT_WEIGHTED && c->mode != VC_SPLAT_SIMPLE)
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "unknown splat mode");
  if (c->silhouette_radius_px < 0) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "silhouette radius < 0");
  return VC_OK;
}

float ev_ms(vc_ctx* ctx, int a, int b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, ctx->ev[a], ctx->ev[b]) != cudaSuccess) {
    cudaGetLastError();  // not recorded in this frame: report NaN, leave no stale error
    return -1.f;
  }
  return ms;
}

vc_status read_ctl(vc_ctx* ctx) {
  VC_CUDA(cudaMemcpyAsync(ctx->ctl_h, ctx->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}

// Hand the context's mesh + texture buffers to the caller: device pointers,
// or pinned host copies (enqueued on the context stream, not synchronised).
vc_status copy_out(vc_ctx* ctx, int V, int T, int k, vc_textured_mesh* out) {
  if (ctx->out_kind == VC_MEM_DEVICE) {
    out->positions = P<float>(ctx->m_posf), out->normals = P<float>(ctx->m_nrm), out->triangles = P<int32_t>(ctx->m_tri);
    out->visible = P<uint8_t>(ctx->t_vis), out->uv = P<float>(ctx->t_uv), out->weight = P<float>(ctx->t_w);
    out->untextured = P<uint8_t>(ctx->t_untex), out->rgb = P<uint8_t>(ctx->t_rgb);
    out->positions_f64 = P<double>(ctx->m_pos);
  } else {
    VC_TRY(ensure_host(ctx, ctx->h_posf, (size_t)V * 12));
    VC_TRY(ensure_host(ctx, ctx->h_nrm, (size_t)V * 12));
    VC_TRY(ensure_host(ctx, ctx->h_tri, (size_t)T * 12));
    VC_TRY(ensure_host(ctx, ctx->h_vis, (size_t)V * k));
    VC_TRY(ensure_host(ctx, ctx->h_uv, (size_t)V * k * 8));
    VC_TRY(ensure_host(ctx, ctx->h_w, (size_t)V * k * 4));
    VC_TRY(ensure_host(ctx, ctx->h_untex, (size_t)V));
    VC_TRY(ensure_host(ctx, ctx->h_rgb, (size_t)V * 3));
    VC_TRY(ensure_host(ctx, ctx->h_pos, (size_t)V * 24));
    auto d2h = [&](HostBuf& h, const Buf& d, size_t bytes) {
      return bytes ? cudaMemcpyAsync(h.p, d.p, bytes, cudaMemcpyDeviceToHost, ctx->st) : cudaSuccess;
    };
    VC_CUDA(d2h(ctx->h_posf, ctx->m_posf, (size_t)V * 12));
    VC_CUDA(d2h(ctx->h_nrm, ctx->m_nrm, (size_t)V * 12));
    VC_CUDA(d2h(ctx->h_tri, ctx->m_tri, (size_t)T * 12));
    VC_CUDA(d2h(ctx->h_vis, ctx->t_vis, (size_t)V * k));
    VC_CUDA(d2h(ctx->h_uv, ctx->t_uv, (size_t)V * k * 8));
    VC_CUDA(d2h(ctx->h_w, ctx->t_w, (size_t)V * k * 4));
    VC_CUDA(d2h(ctx->h_untex, ctx->t_untex, (size_t)V));
    VC_CUDA(d2h(ctx->h_rgb, ctx->t_rgb, (size_t)V * 3));
    VC_CUDA(d2h(ctx->h_pos, ctx->m_pos, (size_t)V * 24));
    if (!out) return VC_OK;  // speculative copies (pointers set later)
    out->positions = (const float*)ctx->h_posf.p, out->normals = (const float*)ctx->h_nrm.p;
    out->triangles = (const int32_t*)ctx->h_tri.p, out->visible = (const uint8_t*)ctx->h_vis.p;
    out->uv = (const float*)ctx->h_uv.p, out->weight = (const float*)ctx->h_w.p;
    out->untextured = (const uint8_t*)ctx->h_untex.p, out->rgb = (const uint8_t*)ctx->h_rgb.p;
    out->positions_f64 = (const double*)ctx->h_pos.p;
  }
  return VC_OK;
}

}  // namespace vc::rt

using namespace vc::rt;

extern "C" {

int vc_abi_version(void) { return VC_ABI_VERSION; }

const char* vc_status_string(vc_status s) {
  switch (s) {
    case VC_OK: return "ok";
    case VC_ERR_INVALID_ARGUMENT: return "invalid argument";
    case VC_ERR_EMPTY_SCENE: return "empty foreground in all views";
    case VC_ERR_CAPACITY: return "capacity exceeded";
    case VC_ERR_CUDA: return "CUDA error";
    case VC_ERR_NCCL: return "NCCL error";
    case VC_ERR_OOM: return "out of device memory";
    case VC_ERR_NO_DEVICE: return "no CUDA device";
    case VC_ERR_RUNTIME: return "runtime error";
  }
  return "unknown";
}

vc_status vc_ctx_create(int device, vc_ctx** out) {
  if (!out) return VC_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return VC_ERR_NO_DEVICE;
  if (device < 0 || device >= n) return VC_ERR_INVALID_ARGUMENT;
  auto* ctx = new vc_ctx;
  ctx->device = device;
  if (device < 64) g_live_ctx[device].fetch_add(1);
  if (const char* e = getenv("VC_GRAPHS")) ctx->graphs = atoi(e) != 0;  // A/B: direct launches
  auto cleanup = [&](vc_status s) {
    if (device < 64) g_live_ctx[device].fetch_sub(1);
    delete ctx;
    return s;
  };
  if (cudaSetDevice(device) != cudaSuccess) return cleanup(VC_ERR_CUDA);
  if (cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking) != cudaSuccess) return cleanup(VC_ERR_CUDA);
  if (cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking) != cudaSuccess) return cleanup(VC_ERR_CUDA);
  if (cudaStreamCreateWithFlags(&ctx->cst, cudaStreamNonBlocking) != cudaSuccess) return cleanup(VC_ERR_CUDA);
  if (cudaEventCreateWithFlags(&ctx->rgb_ev, cudaEventDisableTiming) != cudaSuccess) return cleanup(VC_ERR_CUDA);
  for (int i = 0; i < 2; ++i)
    if (cudaEventCreateWithFlags(&ctx->fork[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->join[i], cudaEventDisableTiming) != cudaSuccess)
      return cleanup(VC_ERR_CUDA);
  if (cudaMalloc(&ctx->ctl, sizeof(DevCtl)) != cudaSuccess) return cleanup(VC_ERR_OOM);
  if (cudaMemset(ctx->ctl, 0, sizeof(DevCtl)) != cudaSuccess) return cleanup(VC_ERR_CUDA);
  if (cudaHostAlloc(&ctx->ctl_h, sizeof(DevCtl), cudaHostAllocDefault) != cudaSuccess) return cleanup(VC_ERR_OOM);
  std::memset(ctx->ctl_h, 0, sizeof(DevCtl));
  for (auto& e : ctx->ev)
    if (cudaEventCreate(&e) != cudaSuccess) return cleanup(VC_ERR_CUDA);
  *out = ctx;
  return VC_OK;
}

vc_status vc_ctx_destroy(vc_ctx* ctx) {
  if (!ctx) return VC_OK;
  if (ctx->device < 64) g_live_ctx[ctx->device].fetch_sub(1);
  cudaSetDevice(ctx->device);
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  for (Buf* b : {&ctx->acc, &ctx->spec, &ctx->A, &ctx->tw, &ctx->vbase, &ctx->blk, &ctx->rowmm, &ctx->units, &ctx->unitcnt, &ctx->ucmask, &ctx->rowbits, &ctx->planeflag, &ctx->rowlist, &ctx->vinfo, &ctx->scratch_dev, &ctx->scratch_dev2, &ctx->skel_lut, &ctx->df_scratch, &ctx->views, &ctx->pts_pos,
                 &ctx->pts_nrm, &ctx->pts_w, &ctx->pts_pix, &ctx->wmaps, &ctx->pre_scratch, &ctx->iso_partial,
                 &ctx->m_pos, &ctx->m_nrm, &ctx->m_tri, &ctx->m_eid, &ctx->m_cells, &ctx->m_celltri, &ctx->m_cellcfg, &ctx->m_posf,
                 &ctx->t_vis, &ctx->t_uv, &ctx->t_w, &ctx->t_untex, &ctx->t_rgb})
    if (b->p) cudaFree(b->p);
  for (HostBuf* b : {&ctx->h_posf, &ctx->h_nrm, &ctx->h_tri, &ctx->h_vis, &ctx->h_uv, &ctx->h_w, &ctx->h_untex,
                     &ctx->h_rgb, &ctx->h_pos, &ctx->h_eid})
    if (b->p) cudaFreeHost(b->p);
  if (ctx->aux) cudaStreamSynchronize(ctx->aux), cudaStreamDestroy(ctx->aux);
  if (ctx->cst) cudaStreamSynchronize(ctx->cst), cudaStreamDestroy(ctx->cst);
  if (ctx->rgb_ev) cudaEventDestroy(ctx->rgb_ev);
  for (int i = 0; i < 2; ++i) {
    if (ctx->fork[i]) cudaEventDestroy(ctx->fork[i]);
    if (ctx->join[i]) cudaEventDestroy(ctx->join[i]);
  }
  if (ctx->ctl) cudaFree(ctx->ctl);
  if (ctx->ctl_h) cudaFreeHost(ctx->ctl_h);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->st) cudaStreamDestroy(ctx->st);
  delete ctx;
  return VC_OK;
}

const char* vc_last_error(const vc_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

vc_status vc_ctx_set_output(vc_ctx* ctx, int32_t kind) {
  if (!ctx || (kind != VC_MEM_HOST && kind != VC_MEM_DEVICE)) return VC_ERR_INVALID_ARGUMENT;
  ctx->out_kind = kind;
  return VC_OK;
}
vc_status vc_ctx_set_profiling(vc_ctx* ctx, int32_t enable) {
  if (!ctx) return VC_ERR_INVALID_ARGUMENT;
  ctx->profiling = enable != 0;
  return VC_OK;
}
vc_status vc_ctx_set_graphs(vc_ctx* ctx, int32_t enable) {
  if (!ctx) return VC_ERR_INVALID_ARGUMENT;
  ctx->graphs = enable != 0;
  return VC_OK;
}
void* vc_ctx_stream(vc_ctx* ctx) { return ctx ? (void*)ctx->st : nullptr; }
int32_t vc_ctx_kernels_per_frame(const vc_ctx* ctx) { return ctx ? ctx->kernels_per_frame : 0; }

int32_t vc_ctx_kernel_times(const vc_ctx* ctx, double* ms, int32_t max_n) {
  if (!ctx || !ms) return 0;
  vc_ctx* c = const_cast<vc_ctx*>(ctx);
  // preprocess, clear, splat, fx, fy, z, iy, ix, iso, mc, texture
  const int pairs[11][2] = {{0, 1}, {12, 13}, {1, 2}, {14, 15}, {15, 16}, {16, 17}, {17, 18}, {18, 19},
                            {3, 4}, {4, 5}, {5, 6}};
  int n = 0;
  for (; n < 11 && n < max_n; ++n) ms[n] = ev_ms(c, pairs[n][0], pairs[n][1]);
  return n;
}

vc_status vc_host_alloc(vc_ctx* ctx, size_t bytes, void** out) {
  if (!ctx || !out) return VC_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  VC_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocDefault));
  return VC_OK;
}
vc_status vc_host_free(vc_ctx* ctx, void* p) {
  if (!ctx) return VC_ERR_INVALID_ARGUMENT;
  VC_CUDA(cudaFreeHost(p));
  return VC_OK;
}
vc_status vc_device_alloc(vc_ctx* ctx, size_t bytes, void** out) {
  if (!ctx || !out) return VC_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  VC_CUDA(cudaMalloc(out, bytes));
  return VC_OK;
}
vc_status vc_device_free(vc_ctx* ctx, void* p) {
  if (!ctx) return VC_ERR_INVALID_ARGUMENT;
  VC_CUDA(cudaFree(p));
  return VC_OK;
}
vc_status vc_memcpy(vc_ctx* ctx, void* dst, const void* src, size_t bytes, int32_t dk, int32_t sk) {
  if (!ctx) return VC_ERR_INVALID_ARGUMENT;
  const cudaMemcpyKind kind = dk == VC_MEM_DEVICE ? (sk == VC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice)
                                                  : (sk == VC_MEM_DEVICE ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost);
  VC_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}
vc_status vc_synchronize(vc_ctx* ctx) {
  if (!ctx) return VC_ERR_INVALID_ARGUMENT;
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}

// ------------------------------------------------------------- hot path
vc_status vc_reconstruct_frame(vc_ctx* ctx, const vc_sensor* sensors, const vc_view* views, int32_t k,
                               const vc_recon_config* config, vc_textured_mesh* out, vc_stage_timings* timings) {
  if (!ctx || !views || !config || !out) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "null argument");
  cudaSetDevice(ctx->device);
  VC_CUDA(cudaGetLastError());
  VC_TRY(check_sensors(ctx, sensors, k));
  int nx, ny, nz;
  VC_TRY(resolve_dims(ctx, config, &nx, &ny, &nz));
  VC_TRY(ensure_tables(ctx));
  VC_TRY(ensure_grid(ctx, nx, ny, nz));
  VC_TRY(setup_sensorset(ctx, sensors, k));
  const bool prof = ctx->profiling || timings;
  const bool prof_saved = ctx->profiling;
  ctx->profiling = prof;

  if (prof) record_event(ctx->ev[8], ctx->st);
  ctx->rgb_async = !prof;  // profiled frames time the whole H2D as one stage
  const vc_status sv = stage_views(ctx, sensors, views, k, true);
  ctx->rgb_async = false;
  VC_TRY(sv);
  if (prof) record_event(ctx->ev[9], ctx->st);
  const FrameCfg f{nx, ny, nz, config->mode, config->padding_voxels, config->silhouette_radius_px,
                   config->discontinuity_mm, config->eps_vis_mm};
  vc_status s = run_frame(ctx, f);
  ctx->profiling = prof_saved;
  if (s != VC_OK) return s;
  // Host output: copy the outputs at the previous frame's sizes (+12%) right
  // behind the frame, with the control block, and synchronise once; only a
  // larger mesh needs a second round (the per-sensor arrays are laid out by
  // the actual V, so a longer copy covers them).
  int spec_v = 0, spec_t = 0;
  if (ctx->out_kind == VC_MEM_HOST && ctx->spec_v > 0 && !prof) {
    spec_v = std::min(ctx->spec_v, ctx->v_cap), spec_t = std::min(ctx->spec_t, ctx->t_cap);
    VC_CUDA(cudaMemcpyAsync(ctx->ctl_h, ctx->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, ctx->st));
    VC_TRY(copy_out(ctx, spec_v, spec_t, k, nullptr));
    VC_CUDA(cudaStreamSynchronize(ctx->st));
  } else {
    VC_TRY(read_ctl(ctx));
  }
  const DevCtl& c = *ctx->ctl_h;
  if (c.status == 2) return fail(ctx, VC_ERR_EMPTY_SCENE, "reconstruct_frame: empty foreground in all views");
  if (c.status != 0) return fail(ctx, VC_ERR_CUDA, "preprocess failed");
  if (c.overflow) {  // grow and redo MC + texture (rare; invalidates the graph)
    const int want = std::max(c.V, std::max(c.C, c.T / 2)) * 2;
    VC_TRY(ensure_mesh_caps(ctx, want, kMaxViews));
    launch_marching_cubes(P<float>(ctx->A), ctx->ctl, mesh_bufs(ctx), nx, ny, nz, ctx->st);
    launch_texture(ctx->ss, P<float>(ctx->wmaps), P<double>(ctx->m_pos), ctx->ctl, config->eps_vis_mm,
                   P<uint8_t>(ctx->t_vis), P<float2>(ctx->t_uv), P<float>(ctx->t_w), P<uint8_t>(ctx->t_untex),
                   P<uint8_t>(ctx->t_rgb), ctx->v_cap, ctx->st, P<float>(ctx->m_posf));
    VC_CUDA(cudaGetLastError());
    VC_TRY(read_ctl(ctx));
    if (ctx->ctl_h->overflow) return fail(ctx, VC_ERR_CAPACITY, "marching cubes capacity");
    spec_v = spec_t = 0;
  }
  const int V = ctx->ctl_h->V, T = ctx->ctl_h->T;
  std::memset(out, 0, sizeof(*out));
  out->vertex_count = V, out->triangle_count = T, out->sensor_count = k, out->point_count = ctx->ctl_h->P;
  out->iso_level = ctx->ctl_h->level;
  out->grid.nx = nx, out->grid.ny = ny, out->grid.nz = nz;
  for (int a = 0; a < 3; ++a) out->grid.origin[a] = ctx->ctl_h->grid.origin[a];
  out->grid.edge_mm = ctx->ctl_h->grid.edge;
  out->mem_kind = ctx->out_kind;
  if (prof) record_event(ctx->ev[10], ctx->st);
  if (spec_v >= V && spec_t >= T && V > 0) {
    VC_TRY(copy_out(ctx, 0, 0, k, out));  // already copied: pointers only
  } else {
    VC_TRY(copy_out(ctx, V, T, k, out));
  }
  if (prof) record_event(ctx->ev[11], ctx->st);
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  if (ctx->out_kind == VC_MEM_HOST) ctx->spec_v = V + V / 8 + 1024, ctx->spec_t = T + T / 8 + 2048;
  if (timings) {
    std::memset(timings, 0, sizeof(*timings));
    timings->h2d_ms = ev_ms(ctx, 8, 9);
    timings->raw_ms = ev_ms(ctx, 0, 1);
    timings->weights_ms = 0.0;  // fused into the preprocess kernels
    timings->splat_ms = ev_ms(ctx, 1, 2);
    timings->fft_ms = ev_ms(ctx, 2, 3);
    timings->iso_ms = ev_ms(ctx, 3, 4);
    timings->mc_ms = ev_ms(ctx, 4, 5);
    timings->volumetric_ms = ev_ms(ctx, 1, 5);
    timings->texture_ms = ev_ms(ctx, 5, 6);
    timings->d2h_ms = ev_ms(ctx, 10, 11);
    timings->total_ms = ev_ms(ctx, 8, 11);
  }
  return VC_OK;
}

vc_status vc_export_volume(vc_ctx* ctx, float* dst, int32_t kind) {
  if (!ctx || !dst || !ctx->A.p) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "no volume");
  const size_t bytes = (size_t)ctx->nx * ctx->ny * ctx->nz * sizeof(float);
  VC_CUDA(cudaMemcpyAsync(dst, ctx->A.p, bytes, kind == VC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                          ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}

vc_status vc_export_points(vc_ctx* ctx, double* pos, double* nrm, double* weight, int32_t* pix, float* wmaps) {
  if (!ctx || !ctx->pts_pos.p) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "no points");
  VC_TRY(read_ctl(ctx));
  const size_t n = (size_t)ctx->ctl_h->P;
  if (pos) VC_CUDA(cudaMemcpyAsync(pos, ctx->pts_pos.p, n * 24, cudaMemcpyDeviceToHost, ctx->st));
  if (nrm) VC_CUDA(cudaMemcpyAsync(nrm, ctx->pts_nrm.p, n * 24, cudaMemcpyDeviceToHost, ctx->st));
  if (weight) VC_CUDA(cudaMemcpyAsync(weight, ctx->pts_w.p, n * 8, cudaMemcpyDeviceToHost, ctx->st));
  if (pix) VC_CUDA(cudaMemcpyAsync(pix, ctx->pts_pix.p, n * 12, cudaMemcpyDeviceToHost, ctx->st));
  if (wmaps)
    VC_CUDA(cudaMemcpyAsync(wmaps, ctx->wmaps.p, (size_t)ctx->ss.pix_offset[ctx->ss.k] * 4, cudaMemcpyDeviceToHost,
                            ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}

// ------------------------------------------------------------- stage entry points
vc_status vc_stage_preprocess(vc_ctx* ctx, const vc_sensor* sensors, const vc_view* views, int32_t k,
                              const vc_recon_config* config, int64_t* n_points, vc_grid_spec* grid) {
  if (!ctx || !views || !config) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "null argument");
  cudaSetDevice(ctx->device);
  VC_TRY(check_sensors(ctx, sensors, k));
  int nx, ny, nz;
  VC_TRY(resolve_dims(ctx, config, &nx, &ny, &nz));
  VC_TRY(setup_sensorset(ctx, sensors, k));
  VC_TRY(stage_views(ctx, sensors, views, k, false));
  launch_preprocess(ctx->ss, points(ctx), P<float>(ctx->wmaps), P<int32_t>(ctx->pre_scratch), ctx->ctl, nx, ny, nz,
                    config->padding_voxels, config->discontinuity_mm, config->silhouette_radius_px, ctx->st);
  VC_CUDA(cudaGetLastError());
  VC_TRY(read_ctl(ctx));
  if (n_points) *n_points = ctx->ctl_h->P;
  if (grid) {
    grid->nx = nx, grid->ny = ny, grid->nz = nz;
    for (int a = 0; a < 3; ++a) grid->origin[a] = ctx->ctl_h->grid.origin[a];
    grid->edge_mm = ctx->ctl_h->grid.edge;
  }
  if (ctx->ctl_h->status == 2) return fail(ctx, VC_ERR_EMPTY_SCENE, "empty foreground in all views");
  return VC_OK;
}

vc_status vc_fit_grid(const double lo[3], const double hi[3], const int32_t dims[3], int32_t pad, vc_grid_spec* g) {
  if (!lo || !hi || !dims || !g) return VC_ERR_INVALID_ARGUMENT;
  double edge = 1e-9;
  for (int a = 0; a < 3; ++a) {
    const int usable = dims[a] - 1 - 2 * pad;
    if (usable < 1) return VC_ERR_INVALID_ARGUMENT;
    const double e = (hi[a] - lo[a]) / usable;
    edge = edge < e ? e : edge;
  }
  g->nx = dims[0], g->ny = dims[1], g->nz = dims[2];
  g->edge_mm = edge;
  for (int a = 0; a < 3; ++a) g->origin[a] = 0.5 * (lo[a] + hi[a]) - edge * (dims[a] - 1) / 2.0;
  return VC_OK;
}

namespace {
vc_status upload_points(vc_ctx* ctx, const double* pos, const double* nrm, const double* w, int64_t n,
                        const vc_grid_spec* grid, int status_ok) {
  VC_TRY(ensure(ctx, ctx->pts_pos, std::max<int64_t>(n, 1) * 24));
  VC_TRY(ensure(ctx, ctx->pts_nrm, std::max<int64_t>(n, 1) * 24));
  VC_TRY(ensure(ctx, ctx->pts_w, std::max<int64_t>(n, 1) * 8));
  VC_TRY(ensure(ctx, ctx->pts_pix, std::max<int64_t>(n, 1) * 12));
  ctx->pts_cap = (int)std::max<int64_t>(n, 1);
  if (n) {
    VC_CUDA(cudaMemcpyAsync(ctx->pts_pos.p, pos, n * 24, cudaMemcpyHostToDevice, ctx->st));
    if (nrm) VC_CUDA(cudaMemcpyAsync(ctx->pts_nrm.p, nrm, n * 24, cudaMemcpyHostToDevice, ctx->st));
    if (w) VC_CUDA(cudaMemcpyAsync(ctx->pts_w.p, w, n * 8, cudaMemcpyHostToDevice, ctx->st));
  }
  DevCtl& c = *ctx->ctl_h;
  std::memset(&c, 0, sizeof(c));
  c.P = (int32_t)n;
  c.status = status_ok ? 0 : 2;
  c.grid.nx = grid->nx, c.grid.ny = grid->ny, c.grid.nz = grid->nz;
  for (int a = 0; a < 3; ++a) c.grid.origin[a] = grid->origin[a];
  c.grid.edge = grid->edge_mm;
  VC_CUDA(cudaMemcpyAsync(ctx->ctl, &c, sizeof(DevCtl), cudaMemcpyHostToDevice, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}
}  // namespace

vc_status vc_stage_splat(vc_ctx* ctx, const double* pos, const double* nrm, const double* weight, int64_t n,
                         const vc_grid_spec* grid, int32_t mode, int32_t negate, float* field, float* density) {
  if (!ctx || !grid || !field || !density || (n > 0 && (!pos || !nrm))) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "null");
  if (mode != 0 && mode != 1) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "mode");
  cudaSetDevice(ctx->device);
  const size_t N = (size_t)grid->nx * grid->ny * grid->nz;
  VC_TRY(ensure(ctx, ctx->acc, N * sizeof(float4)));
  VC_TRY(ensure(ctx, ctx->rowbits, (size_t)grid->ny * grid->nz * sizeof(uint32_t)));
  VC_TRY(ensure(ctx, ctx->rowlist, ((size_t)grid->ny * grid->nz + 1) * sizeof(int32_t)));
  ctx->acc_dirty = true, ctx->layout = 0;
  VC_CUDA(cudaMemsetAsync(ctx->rowbits.p, 0, (size_t)grid->ny * grid->nz * sizeof(uint32_t), ctx->st));
  VC_CUDA(cudaMemsetAsync(ctx->rowlist.p, 0, sizeof(int32_t), ctx->st));
  std::vector<double> ones;
  if (!weight) ones.assign(std::max<int64_t>(n, 1), 1.0), weight = ones.data();
  VC_TRY(upload_points(ctx, pos, nrm, weight, n, grid, 1));
  Buf fbuf, dbuf;
  VC_TRY(ensure(ctx, fbuf, N * 12));
  VC_TRY(ensure(ctx, dbuf, N * 4));
  launch_clear(P<float4>(ctx->acc), N, ctx->st);
  launch_splat(points(ctx), ctx->ctl, P<float4>(ctx->acc), P<uint32_t>(ctx->rowbits), P<int32_t>(ctx->rowlist), mode,
               ctx->st, 0, grid->nz);
  const double sigma2 = std::sqrt(1.5) * (std::sqrt(3.0) / 2.0 * grid->edge_mm);  // splat.cpp:35-36
  launch_splat_finalize(P<float4>(ctx->acc), N, mode, negate, sigma2, P<float>(fbuf), P<float>(dbuf), ctx->st);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(field, fbuf.p, N * 12, cudaMemcpyDeviceToHost, ctx->st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(density, dbuf.p, N * 4, cudaMemcpyDeviceToHost, ctx->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->st);
  cudaFree(fbuf.p);
  cudaFree(dbuf.p);
  if (e != cudaSuccess) return fail(ctx, VC_ERR_CUDA, cudaGetErrorString(e));
  return VC_OK;
}

vc_status vc_stage_integrate(vc_ctx* ctx, const float* field, int32_t nx, int32_t ny, int32_t nz, float* A) {
  if (!ctx || !field || !A) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "null");
  if (!pow2_ok(nx) || !pow2_ok(ny) || !pow2_ok(nz))
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "grid dims must be powers of two in [4, 1024]");
  cudaSetDevice(ctx->device);
  VC_TRY(ensure_grid(ctx, nx, ny, nz));
  const size_t N = (size_t)nx * ny * nz;
  // acc = (-V, 1) under the simple-mode normalisation V = -U/d gives V exactly
  std::vector<float4> h(N);
  for (size_t i = 0; i < N; ++i) h[i] = make_float4(-field[3 * i], -field[3 * i + 1], -field[3 * i + 2], 1.f);
  VC_CUDA(cudaMemcpyAsync(ctx->acc.p, h.data(), N * sizeof(float4), cudaMemcpyHostToDevice, ctx->st));
  ctx->acc_dirty = true, ctx->layout = 0;  // dense contents from the host
  launch_integrate(P<float4>(ctx->acc), P<float2>(ctx->spec), P<float>(ctx->A), nx, ny, nz, 1, P<float2>(ctx->tw),
                   ctx->st, nullptr, nullptr, nullptr, P<uint32_t>(ctx->planeflag));
  VC_CUDA(cudaGetLastError());
  VC_CUDA(cudaMemcpyAsync(A, ctx->A.p, N * 4, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}

// Timing of the integrate chain on a DENSE field (every row and plane
// non-empty: no sparsity shortcuts), device-resident, for the cuFFT
// comparator in bench.py.  ms[0..4] = F-x, F-y, Z, I-y, I-x per launch,
// ms[5] = the chain, averaged over `iters` after two warm-up runs.
vc_status vc_time_integrate(vc_ctx* ctx, int32_t nx, int32_t ny, int32_t nz, int32_t iters, double* ms) {
  if (!ctx || !ms || iters < 1) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "null");
  if (!pow2_ok(nx) || !pow2_ok(ny) || !pow2_ok(nz))
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "grid dims must be powers of two in [4, 1024]");
  cudaSetDevice(ctx->device);
  VC_TRY(ensure_grid(ctx, nx, ny, nz));
  const size_t N = (size_t)nx * ny * nz;
  launch_fill_random_acc(P<float4>(ctx->acc), N, 12345u, ctx->st);
  ctx->acc_dirty = true, ctx->layout = 0;
  cudaEvent_t ev[6];
  for (auto& e : ev) cudaEventCreate(&e);
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int it = -2; it < iters; ++it) {
    launch_integrate(P<float4>(ctx->acc), P<float2>(ctx->spec), P<float>(ctx->A), nx, ny, nz, 1, P<float2>(ctx->tw),
                     ctx->st, ev, nullptr, nullptr, P<uint32_t>(ctx->planeflag));
    VC_CUDA(cudaGetLastError());
    VC_CUDA(cudaStreamSynchronize(ctx->st));
    if (it < 0) continue;
    for (int i = 0; i < 5; ++i) {
      float t = 0;
      cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
      acc[i] += t;
    }
    float t = 0;
    cudaEventElapsedTime(&t, ev[0], ev[5]);
    acc[5] += t;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (int i = 0; i < 6; ++i) ms[i] = acc[i] / iters;
  return VC_OK;
}

vc_status vc_stage_iso_level(vc_ctx* ctx, const float* A, const vc_grid_spec* grid, const double* pos, int64_t n,
                             double* level) {
  if (!ctx || !A || !grid || !level) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "null");
  if (n <= 0) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "iso_level: no input samples");  // splat.cpp:99
  cudaSetDevice(ctx->device);
  const size_t N = (size_t)grid->nx * grid->ny * grid->nz;
  Buf a;
  VC_TRY(ensure(ctx, a, N * 4));
  VC_TRY(ensure(ctx, ctx->iso_partial, 1024 * sizeof(double)));
  VC_CUDA(cudaMemcpyAsync(a.p, A, N * 4, cudaMemcpyHostToDevice, ctx->st));
  VC_TRY(upload_points(ctx, pos, nullptr, nullptr, n, grid, 1));
  launch_iso_level(points(ctx), P<float>(a), ctx->ctl, P<double>(ctx->iso_partial), 1024, ctx->st);
  cudaError_t e = cudaGetLastError();
  cudaFree(a.p);
  if (e != cudaSuccess) return fail(ctx, VC_ERR_CUDA, cudaGetErrorString(e));
  VC_TRY(read_ctl(ctx));
  *level = ctx->ctl_h->level;
  return VC_OK;
}

vc_status vc_stage_marching_cubes(vc_ctx* ctx, const float* A, const vc_grid_spec* grid, double level,
                                  int32_t* n_vertices, int32_t* n_triangles, const double** positions,
                                  const float** normals, const int32_t** triangles, const uint64_t** edge_ids) {
  if (!ctx || !A || !grid || !n_vertices || !n_triangles) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "null");
  const int nx = grid->nx, ny = grid->ny, nz = grid->nz;
  if (nx > 1024) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "marching cubes: nx > 1024");
  if (nx < 2 || ny < 2 || nz < 2) {  // marching_cubes.cpp:135
    *n_vertices = *n_triangles = 0;
    return VC_OK;
  }
  cudaSetDevice(ctx->device);
  VC_TRY(ensure_tables(ctx));
  const size_t N = (size_t)nx * ny * nz;
  VC_TRY(ensure(ctx, ctx->A, N * 4));
  VC_TRY(ensure(ctx, ctx->vbase, N * 4));
  VC_TRY(ensure_mc_scratch(ctx, nx, ny, nz));
  ctx->nx = ctx->ny = ctx->nz = 0;  // grid buffers no longer match a frame config
  if (ctx->v_cap == 0) VC_TRY(ensure_mesh_caps(ctx, (int)std::max<size_t>(N / 16, 1 << 16), kMaxViews));
  VC_CUDA(cudaMemcpyAsync(ctx->A.p, A, N * 4, cudaMemcpyHostToDevice, ctx->st));
  VC_TRY(upload_points(ctx, nullptr, nullptr, nullptr, 0, grid, 1));
  ctx->ctl_h->level = level;
  ctx->ctl_h->voff = 0;
  VC_CUDA(cudaMemcpyAsync(ctx->ctl, ctx->ctl_h, sizeof(DevCtl), cudaMemcpyHostToDevice, ctx->st));
  launch_row_minmax(P<float>(ctx->A), nx, ny, nz, P<float2>(ctx->rowmm), ctx->st);
  for (int attempt = 0; attempt < 2; ++attempt) {
    MeshBufs mb = mesh_bufs(ctx);
    launch_marching_cubes(P<float>(ctx->A), ctx->ctl, mb, nx, ny, nz, ctx->st);
    VC_CUDA(cudaGetLastError());
    VC_TRY(read_ctl(ctx));
    if (!ctx->ctl_h->overflow) break;
    const DevCtl c = *ctx->ctl_h;
    VC_TRY(ensure_mesh_caps(ctx, std::max(c.V, std::max(c.C, c.T / 2)) * 2, kMaxViews));
    if (attempt == 1) return fail(ctx, VC_ERR_CAPACITY, "marching cubes capacity");
  }
  const int V = ctx->ctl_h->V, T = ctx->ctl_h->T;
  *n_vertices = V, *n_triangles = T;
  const size_t bytes = (size_t)V * 24 + (size_t)V * 12 + (size_t)T * 12 + (size_t)V * 8 + 64;
  ctx->scratch.resize(bytes);
  uint8_t* p = ctx->scratch.data();
  double* hp = reinterpret_cast<double*>(p);
  float* hn = reinterpret_cast<float*>(p + (size_t)V * 24);
  uint64_t* he = reinterpret_cast<uint64_t*>(p + (size_t)V * 36);
  int32_t* ht = reinterpret_cast<int32_t*>(p + (size_t)V * 44);
  if (V) {
    VC_CUDA(cudaMemcpyAsync(hp, ctx->m_pos.p, (size_t)V * 24, cudaMemcpyDeviceToHost, ctx->st));
    VC_CUDA(cudaMemcpyAsync(hn, ctx->m_nrm.p, (size_t)V * 12, cudaMemcpyDeviceToHost, ctx->st));
    VC_CUDA(cudaMemcpyAsync(he, ctx->m_eid.p, (size_t)V * 8, cudaMemcpyDeviceToHost, ctx->st));
  }
  if (T) VC_CUDA(cudaMemcpyAsync(ht, ctx->m_tri.p, (size_t)T * 12, cudaMemcpyDeviceToHost, ctx->st));
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  if (positions) *positions = hp;
  if (normals) *normals = hn;
  if (triangles) *triangles = ht;
  if (edge_ids) *edge_ids = he;
  return VC_OK;
}

vc_status vc_stage_texture(vc_ctx* ctx, const vc_sensor* sensors, const vc_view* views, const float* weight_maps,
                           int32_t k, const double* vertices, int32_t V, double eps_vis_mm, uint8_t* visible, float* uv,
                           float* weight, uint8_t* untextured, uint8_t* rgb) {
  if (!ctx || !views || !weight_maps || (V > 0 && !vertices)) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "null");
  cudaSetDevice(ctx->device);
  VC_TRY(check_sensors(ctx, sensors, k));
  VC_TRY(setup_sensorset(ctx, sensors, k));
  VC_TRY(stage_views(ctx, sensors, views, k, true));
  VC_TRY(ensure_tables(ctx));
  if (ctx->v_cap < V) VC_TRY(ensure_mesh_caps(ctx, V, kMaxViews));
  if (ctx->v_cap == 0) VC_TRY(ensure_mesh_caps(ctx, 1 << 16, kMaxViews));
  const size_t npix = (size_t)ctx->ss.pix_offset[k];
  VC_CUDA(cudaMemcpyAsync(ctx->wmaps.p, weight_maps, npix * 4, cudaMemcpyHostToDevice, ctx->st));
  if (V) VC_CUDA(cudaMemcpyAsync(ctx->m_pos.p, vertices, (size_t)V * 24, cudaMemcpyHostToDevice, ctx->st));
  DevCtl& c = *ctx->ctl_h;
  std::memset(&c, 0, sizeof(c));
  c.V = V;
  VC_CUDA(cudaMemcpyAsync(ctx->ctl, &c, sizeof(DevCtl), cudaMemcpyHostToDevice, ctx->st));
  launch_texture(ctx->ss, P<float>(ctx->wmaps), P<double>(ctx->m_pos), ctx->ctl, eps_vis_mm, P<uint8_t>(ctx->t_vis),
                 P<float2>(ctx->t_uv), P<float>(ctx->t_w), P<uint8_t>(ctx->t_untex), P<uint8_t>(ctx->t_rgb), ctx->v_cap,
                 ctx->st);
  VC_CUDA(cudaGetLastError());
  if (V) {
    if (visible) VC_CUDA(cudaMemcpyAsync(visible, ctx->t_vis.p, (size_t)V * k, cudaMemcpyDeviceToHost, ctx->st));
    if (uv) VC_CUDA(cudaMemcpyAsync(uv, ctx->t_uv.p, (size_t)V * k * 8, cudaMemcpyDeviceToHost, ctx->st));
    if (weight) VC_CUDA(cudaMemcpyAsync(weight, ctx->t_w.p, (size_t)V * k * 4, cudaMemcpyDeviceToHost, ctx->st));
    if (untextured) VC_CUDA(cudaMemcpyAsync(untextured, ctx->t_untex.p, (size_t)V, cudaMemcpyDeviceToHost, ctx->st));
    if (rgb) VC_CUDA(cudaMemcpyAsync(rgb, ctx->t_rgb.p, (size_t)V * 3, cudaMemcpyDeviceToHost, ctx->st));
  }
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}

// ------------------------------------------------------------- synthetic capture
vc_status vc_synth_circle_rig(int32_t recon, int32_t held_out, double radius, double target_h, int32_t w, int32_t h,
                              double f, vc_sensor* out) {
  if (!out || recon < 1 || held_out < 0 || w <= 0 || h <= 0 || f <= 0) return VC_ERR_INVALID_ARGUMENT;
  circle_rig(recon, held_out, radius, target_h, w, h, f, out);
  return VC_OK;
}
vc_status vc_synth_xpose_body(vc_body* out) {
  if (!out) return VC_ERR_INVALID_ARGUMENT;
  xpose_body(out);
  return VC_OK;
}
vc_status vc_synth_kick_body(int32_t frames, int32_t frame, vc_body* out) {
  if (!out || frames < 1 || frame < 0 || frame >= frames) return VC_ERR_INVALID_ARGUMENT;
  kick_body(frames, frame, out);
  return VC_OK;
}

vc_status vc_synth_render(vc_ctx* ctx, const vc_sensor* sensor, const vc_body* body, double sigma, uint64_t seed,
                          double gain, int32_t camera, int32_t frame, uint16_t* depth, uint8_t* mask, uint8_t* rgb,
                          int32_t dst_kind) {
  if (!ctx || !sensor || !body) return fail(ctx, VC_ERR_INVALID_ARGUMENT, "null");
  VC_TRY(check_sensors(ctx, sensor, 1));
  cudaSetDevice(ctx->device);
  DevSensor s;
  fill_sensor(*sensor, s);
  const size_t n = (size_t)s.w * s.h, nr = (size_t)s.rw * s.rh * 3;
  uint8_t* tmp = nullptr;
  VC_CUDA(cudaMalloc(&tmp, n * 3 + nr + 64));
  uint16_t* dd = reinterpret_cast<uint16_t*>(tmp);
  uint8_t* dm = tmp + n * 2;
  uint8_t* dr = tmp + n * 3;
  launch_render(s, body->joints, body->radii, body->colors, gain, dd, dm, dr, ctx->st);
  cudaError_t e = cudaGetLastError();
  const cudaMemcpyKind kind = dst_kind == VC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (sigma > 0 && e == cudaSuccess) {  // render.cpp:50-61 on the host (libstdc++ RNG)
    std::vector<uint16_t> h(n);
    e = cudaMemcpyAsync(h.data(), dd, n * 2, cudaMemcpyDeviceToHost, ctx->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->st);
    std::mt19937_64 rng(seed * 46337 + camera * 131 + frame);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (size_t i = 0; i < n; ++i) {
      uint16_t& d = h[i];
      if (d == 0) continue;
      const double sg = sigma * d / 2000.0;
      d = static_cast<uint16_t>(std::clamp(std::lround(d + sg * gauss(rng)), 1L, 65535L));
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(dd, h.data(), n * 2, cudaMemcpyHostToDevice, ctx->st);
  }
  if (e == cudaSuccess && depth) e = cudaMemcpyAsync(depth, dd, n * 2, kind, ctx->st);
  if (e == cudaSuccess && mask) e = cudaMemcpyAsync(mask, dm, n, kind, ctx->st);
  if (e == cudaSuccess && rgb) e = cudaMemcpyAsync(rgb, dr, nr, kind, ctx->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->st);
  cudaFree(tmp);
  if (e != cudaSuccess) return fail(ctx, VC_ERR_CUDA, cudaGetErrorString(e));
  return VC_OK;
}

vc_status vc_ctx_set_depth_filter(vc_ctx* ctx, int32_t erode_px, double sigma_px, double sigma_mm) {
  if (!ctx || erode_px < 0 || erode_px > 32 || !(sigma_px >= 0) || !(sigma_mm >= 0) ||
      depth_filter_radius(sigma_px) > depth_filter_max_radius())
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "depth filter: erode_px in [0, 32], 0 <= sigma_px <= 4, sigma_mm >= 0");
  ctx->df_erode = erode_px, ctx->df_sigma_px = sigma_px, ctx->df_sigma_mm = sigma_mm;
  return VC_OK;
}

vc_status vc_depth_filter(vc_ctx* ctx, uint16_t* depth, uint8_t* mask, int32_t width, int32_t height,
                          int32_t mem_kind, int32_t erode_px, double sigma_px, double sigma_mm) {
  if (!ctx || !depth || !mask || width < 1 || height < 1 || erode_px < 0 || erode_px > 32 || !(sigma_px >= 0) ||
      !(sigma_mm >= 0) || depth_filter_radius(sigma_px) > depth_filter_max_radius())
    return fail(ctx, VC_ERR_INVALID_ARGUMENT, "depth filter: bad arguments");
  cudaSetDevice(ctx->device);
  const size_t n = (size_t)width * height;
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  VC_TRY(ensure(ctx, ctx->scratch_dev, (mem_kind == VC_MEM_HOST ? up(2 * n) + up(n) : 0) + up(n) + up(2 * n) + 256));
  uint8_t* p = P<uint8_t>(ctx->scratch_dev);
  uint16_t* dd = depth;
  uint8_t* dm = mask;
  if (mem_kind == VC_MEM_HOST) {
    dd = reinterpret_cast<uint16_t*>(p);
    p += up(2 * n);
    dm = p;
    p += up(n);
    VC_CUDA(cudaMemcpyAsync(dd, depth, 2 * n, cudaMemcpyHostToDevice, ctx->st));
    VC_CUDA(cudaMemcpyAsync(dm, mask, n, cudaMemcpyHostToDevice, ctx->st));
  }
  launch_depth_filter(dd, dm, width, height, erode_px, sigma_px, sigma_mm, p, reinterpret_cast<uint16_t*>(p + up(n)),
                      ctx->st);
  VC_CUDA(cudaGetLastError());
  if (mem_kind == VC_MEM_HOST) {
    VC_CUDA(cudaMemcpyAsync(depth, dd, 2 * n, cudaMemcpyDeviceToHost, ctx->st));
    VC_CUDA(cudaMemcpyAsync(mask, dm, n, cudaMemcpyDeviceToHost, ctx->st));
  }
  VC_CUDA(cudaStreamSynchronize(ctx->st));
  return VC_OK;
}

}  // extern "C"

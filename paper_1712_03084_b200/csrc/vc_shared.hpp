// SPDX-License-Identifier: Apache-2.0
// Host/device shared plain types and kernel-launcher declarations.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace vc {

constexpr int kMaxViews = 16;

// volume_recon.hpp:24-28 — same layout as vc_grid_spec.
struct DevGrid {
  int32_t nx, ny, nz;
  double origin[3];
  double edge;
};

// One sensor, pre-digested on the host with the reference's own formulas
// (types.hpp:46-49): inverse pose {R^T, -(R^T t)} and the RGB camera pose
// pose.compose(rgb_relative).
struct DevSensor {
  double fx, fy, cx, cy;
  int32_t w, h;
  double R[9], t[3];    // depth camera -> world
  double Ri[9], ti[3];  // world -> depth camera (Pose::inverse)
  double rfx, rfy, rcx, rcy;
  int32_t rw, rh;
  double Rc[9], tc[3];  // RGB camera -> world
  // ColorCorrection map of this sensor (color.hpp:50-57), applied to every
  // RGB sample of the texture blend when cc_on (vc_ctx_set_color_correction)
  double cc_gain, cc_offset;
  int32_t cc_on;
};

struct ViewPtrs {
  const uint16_t* depth;
  const uint8_t* mask;
  const uint8_t* rgb;
  int32_t dpitch, mpitch, rpitch;  // in elements (uint16 / uint8 / bytes)
};

struct SensorSet {
  int32_t k;
  DevSensor s[kMaxViews];
  ViewPtrs v[kMaxViews];
  int64_t pix_offset[kMaxViews + 1];  // prefix of w*h, for per-pixel arrays
  int32_t row_offset[kMaxViews + 1];  // prefix of h, for per-row block counts
};

// Device control block: data-dependent scalars produced on the GPU and read
// back once per frame.
struct DevCtl {
  int32_t P;          // oriented points
  int32_t status;     // 0 ok, 2 empty scene
  int32_t V, T, C;    // vertices, triangles, active cells
  int32_t overflow;   // MC capacity exceeded
  int32_t units;      // MC: active voxel-row units
  int32_t v_extra;    // MC slab: cut edges counted on the next rank's first plane
  int32_t voff;       // MC slab: global id of this rank's first vertex
  int32_t iso_ticket; // iso level: CTAs done (the last one reduces; reset by it)
  double bbox[6];
  unsigned long long bbox_key[6];  // bbox as order-preserving keys (atomic min/max while preprocessing)
  DevGrid grid;
  double level;
};

// Point cloud (SoA, reference order: views in sensor order, pixels row-major).
struct DevPoints {
  double* pos;     // 3P
  double* nrm;     // 3P
  double* weight;  // P
  int32_t* pix;    // 3P: px, py, sensor
  int32_t cap;
};

struct MeshBufs {
  double* pos;       // 3V
  float* nrm;        // 3V
  int32_t* tri;      // 3T
  uint64_t* edge_id; // V
  uint32_t* vbase;   // N (sparse): first vertex id * 8 | cut mask
  int32_t* cells;    // C: active cell linear index
  int32_t* cell_tri; // C: first triangle id
  uint8_t* cell_cfg; // C: cube case
  uint16_t* vinfo;   // per voxel of the active units (unit slot * nx + x): cut mask | case << 3 | has-cell << 11
  int32_t v_cap, t_cap, c_cap;
  int32_t* blk;      // row-culling scratch (mc_blocks ints)
  int32_t nblk;
  float2* rowmm;     // per voxel row (ny*nz): min, max of A
  int32_t* units;    // ordered active row units (ny*nz)
  int32_t* unitcnt;  // per active unit (nv, nt, nc), then exclusive offsets (3*ny*nz)
  uint32_t* ucmask;  // per active unit: its 32-voxel x-chunks that can hold a cut edge or cell
};

// Stage-timing events.  Profiled frames are launched directly (never from a
// captured graph), so a plain record suffices.
inline void record_event(cudaEvent_t e, cudaStream_t s) { cudaEventRecord(e, s); }

// ----------------------------------------------------------------- launchers
// k_preprocess.cu — build_cloud + confidence_weights + bbox + fit_grid
size_t preprocess_scratch_bytes(const SensorSet& ss);
void prepare_preprocess(const SensorSet& ss);  // smem opt-in; call outside graph capture
void launch_preprocess(const SensorSet& ss, DevPoints pts, float* weight_maps, int32_t* scratch, DevCtl* ctl,
                       int dims_x, int dims_y, int dims_z, int padding, double disc_mm, int sil_r, cudaStream_t st,
                       int32_t* rowlist_reset = nullptr /*frame path: zero the touched-row count*/);
void launch_mask_from_depth(const uint16_t* depth, uint8_t* mask, int n, cudaStream_t st);  // mask := depth > 0
// optional depth preprocessing (k_depth_filter.cu; off by default)
int depth_filter_radius(double sigma_px);
int depth_filter_max_radius();
void launch_depth_filter(uint16_t* depth, uint8_t* mask, int w, int h, int erode_px, double sigma_px,
                         double sigma_mm, uint8_t* scratch8, uint16_t* scratch16, cudaStream_t st);
// k_splat.cu
void launch_clear(float4* acc, size_t n, cudaStream_t st);
// zoff/nzl: the z-slab [zoff, zoff+nzl) this rank accumulates (whole grid: 0, nz).
// Every voxel row the splat touches is listed once in the touched-row list
// rowlist = [count, rows...] (built from the chunk masks right after the
// splat).  The list lives outside DevCtl: only the frame path's clear,
// preprocess (reset) and splat touch it, so stage calls cannot desynchronise
// it from the accumulator.
void launch_splat(const DevPoints& pts, DevCtl* ctl, float4* acc, uint32_t* rowbits, int32_t* rowlist, int mode,
                  cudaStream_t st, int zoff, int nzl);
// Zero the chunks of the rows the previous frame listed, reset their masks.
// Runs before the frame's preprocess (which resets the list count).
void launch_reset_rowlist(int32_t* rowlist, cudaStream_t st);  // count := 0 (one-thread kernel)
void launch_sparse_clear(float4* acc, uint32_t* rowbits, const int32_t* rowlist, int nx, cudaStream_t st);
void launch_splat_finalize(const float4* acc, size_t n, int mode, int negate, double sigma2, float* field,
                           float* density, cudaStream_t st);
// k_fft.cu — integrate_fft chain: acc (float4 U,d) -> A
size_t spectrum_elems(int nx, int ny, int nz);  // complex elements per component
// One z-slab of the spectral integration (SURVEY §8(e) "large grids").  On a
// single GPU every pointer pair aliases (O0 = R0 = Rin = Rout = S0, O1 = R1 =
// S1) and nzl = nz, kyl = ny.  On P ranks: local x-R2C + y-C2C over planes
// [zoff, zoff+nzl) -> O0/O1 in send layout; all-to-all -> R0/R1 ([z][kyl][H],
// ky in [ky0, ky0+kyl)); z pass in place on R0; all-to-all R0 -> Rin; y/x
// inverse -> Rout (plain layout) -> A (the rank's planes).
struct SlabFft {
  float4* acc;  // F-x zeroes the chunks it reads when a touched-row list is given
  float2 *S0, *S1, *S2, *O0, *O1, *R0, *R1;
  const float2* Rin;
  float2* Rout;
  float* A;
  int nx, ny, nz, nzl, zoff, kyl, ky0, H, mode;
  const float2 *twx, *twy, *twz;
  cudaStream_t st;
  float2* rowmm;
  const uint32_t* rowbits;
  uint32_t* planeflag;     // nz entries (global); F-y writes [zoff, zoff+nzl); one GPU: + nz+1 (live-plane list)
  const int32_t* rowlist;  // touched-row list [count, rows...] (F-x works through it), or null: all rows
};
void launch_fft_forward_xy(const SlabFft& a);
void launch_fft_z(const SlabFft& a);
void launch_fft_inverse_yx(const SlabFft& a);
void launch_fill_random_acc(float4* acc, size_t n, uint32_t seed, cudaStream_t st);  // dense test field
void launch_integrate(float4* acc, float2* spec, float* A, int nx, int ny, int nz, int mode,
                      const float2* twiddles, cudaStream_t st, cudaEvent_t* ev /*nullable, 6 events*/,
                      float2* rowmm /*nullable: per-row min/max of A*/,
                      const uint32_t* rowbits /*nullable: touched 32-voxel chunks per row (null = dense)*/,
                      uint32_t* planeflag /*nz words: F-y marks planes with any splat contribution*/,
                      const int32_t* rowlist = nullptr /*touched-row list for F-x (null = all rows)*/);
void upload_twiddles(float2* dev, int nx, int ny, int nz, cudaStream_t st);
void prepare_integrate(int nx, int ny, int nz);
size_t twiddle_elems(int nx, int ny, int nz);
// k_mc.cu
int iso_blocks();
void launch_iso_level(const DevPoints& pts, const float* A, DevCtl* ctl, double* partial, int nblk_max,
                      cudaStream_t st);
int mc_blocks(int nx, int ny, int nz);
// Whole volume (rowmm written): active units and one fused count/scan/emit
// pass on `st`, then normals + triangles in one kernel — on `aux` when given
// (fork/join events; the caller waits on `join` before the frame ends: the
// vertex positions, all the texture pass reads, are complete on `st`).
void launch_marching_cubes(const float* A, DevCtl* ctl, MeshBufs mb, int nx, int ny, int nz, cudaStream_t st,
                           cudaStream_t aux = nullptr, cudaEvent_t fork = nullptr, cudaEvent_t join = nullptr);
// Slab variant: units (voxel rows) of planes [z0, z0+nzu); planes >= zend
// belong to the next rank: their cut edges are numbered (vbase) but neither
// emitted nor meshed.  A, vbase are indexed with GLOBAL voxel ids (callers
// pass pointers shifted by the slab origin); rowmm is indexed from plane z0.
// The scan stops before the emit: launch_marching_cubes_count, then (after
// ctl->voff is known) launch_marching_cubes_emit.
struct McSlab {
  int z0, nzu, zend;
};
void launch_marching_cubes_count(const float* A, DevCtl* ctl, MeshBufs mb, int nx, int ny, int nz, McSlab sl,
                                 cudaStream_t st);
void launch_marching_cubes_emit(const float* A, DevCtl* ctl, MeshBufs mb, int nx, int ny, int nz, McSlab sl,
                                cudaStream_t st);
// Slab iso level: samples[p] = trilinear(A, point p) if this rank owns the
// point's lower z plane, else 0 (summed over ranks, then launch_iso_final_samples)
void launch_iso_samples(const DevPoints& pts, const float* A, const DevCtl* ctl, int zoff, int nzl, double* samples,
                        cudaStream_t st);
void launch_add_f64(double* dst, const double* src, size_t n, cudaStream_t st);
void launch_mc_set_voff(const int32_t* counts, int rank, DevCtl* ctl, cudaStream_t st);
void launch_iso_final_samples(const double* samples, DevCtl* ctl, double* partial, cudaStream_t st);
void launch_row_minmax(const float* A, int nx, int ny, int nz, float2* rowmm, cudaStream_t st);
void upload_case_table_data(const int8_t* counts, const int8_t* tris, cudaStream_t st);
// k_texture.cu
// posf (nullable): fp32 copy of the vertex positions, written alongside
void launch_texture(const SensorSet& ss, const float* weight_maps, const double* vpos, const DevCtl* ctl,
                    double eps_vis, uint8_t* vis, float2* uv, float* w, uint8_t* untex, uint8_t* rgb, int v_cap,
                    cudaStream_t st, float* posf = nullptr);
void launch_mesh_to_f32(const double* pos, float* posf, const DevCtl* ctl, int v_cap, cudaStream_t st);
// k_color.cu — colour correction
void launch_color_apply(const uint8_t* in, uint8_t* out, int64_t n, double gain, double offset, cudaStream_t st);
size_t grid_scratch_bytes(int n);
void launch_mutual_pairs(const double* a, int na, const double* b, int nb, double max_dist, void* scratch_a,
                         void* scratch_b, int32_t* partner, int32_t* pairs, int32_t* n_pairs, cudaStream_t st);

// k_synth.cu
void launch_render(const DevSensor& s, const double* joints, const double* radii, const uint8_t* colors,
                   double gain, uint16_t* depth, uint8_t* mask, uint8_t* rgb, cudaStream_t st);

// vc_tables.cpp (host)
void build_mc_table(int8_t counts[256], int8_t tris[256][5][3]);

}  // namespace vc

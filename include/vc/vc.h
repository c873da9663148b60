/* SPDX-License-Identifier: Apache-2.0
 *
 * vc.h — C-ABI of the B200-native FT-reconstruction (FTR) frame path.
 *
 * Drop-in boundary for the reference's proj/core reconstruction interface
 * (/root/reference/proj/core/include/volcap/...):
 *
 *   recon::reconstruct_frame        reconstruct.hpp:38-39  -> vc_reconstruct_frame
 *   appearance::vertex_visibility   texture.hpp:32-35      -> (fused into vc_reconstruct_frame,
 *   appearance::assign_texture      texture.hpp:39-42          and vc_stage_texture)
 *   recon::build_cloud              cloud.hpp:32-33        -> vc_stage_preprocess
 *   recon::confidence_weights       cloud.hpp:37-38        -> vc_stage_preprocess (fused)
 *   recon::fit_grid                 reconstruct.hpp:42     -> vc_fit_grid / vc_stage_preprocess
 *   recon::splat                    volume_recon.hpp:33-34 -> vc_stage_splat
 *   recon::integrate_fft            volume_recon.hpp:46    -> vc_stage_integrate
 *   recon::iso_level                volume_recon.hpp:49    -> vc_stage_iso_level
 *   recon::marching_cubes           marching_cubes.hpp:16  -> vc_stage_marching_cubes
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * Every entry point returns a vc_status; no exception crosses the ABI.  The
 * reference's exceptions map as: std::invalid_argument -> VC_ERR_INVALID_ARGUMENT,
 * std::runtime_error("empty foreground in all views") -> VC_ERR_EMPTY_SCENE.
 *
 * Threading: one vc_ctx = one CUDA device + one stream.  Distinct contexts
 * are independent and may be used from different threads; calls on one
 * context must be serialised by the caller (the reference's reconstruct_frame
 * is a pure function; here state lives in the context).
 *
 * Ownership: inputs are borrowed for the duration of a call.  Outputs are
 * context-owned (vertex/triangle counts are data-dependent) and stay valid
 * until the next call on the same context or vc_ctx_destroy.
 *
 * All world units are millimetres (types.hpp:17).  Arrays are row-major;
 * volumes are x-fastest (volume.hpp:31-34): index = x + nx*(y + ny*z).
 */
#ifndef VC_VC_H_
#define VC_VC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VC_ABI_VERSION 1

typedef enum vc_status {
  VC_OK = 0,
  VC_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  VC_ERR_EMPTY_SCENE = 2,      /* "empty foreground in all views" (reconstruct.cpp:65-66) */
  VC_ERR_CAPACITY = 3,         /* marching-cubes output exceeded capacity (retried internally) */
  VC_ERR_CUDA = 4,
  VC_ERR_NCCL = 5,
  VC_ERR_OOM = 6,
  VC_ERR_NO_DEVICE = 7,
  VC_ERR_RUNTIME = 8           /* std::runtime_error of the reference (e.g. fit_value_map, chain_to_reference) */
} vc_status;

/* types.hpp:26-39 — pinhole, pixel-centre convention. */
typedef struct vc_intrinsics {
  double fx, fy, cx, cy;
  int32_t width, height;
} vc_intrinsics;

/* types.hpp:42-57 — camera-to-world rigid transform, R row-major. */
typedef struct vc_pose {
  double R[9];
  double t[3];
} vc_pose;

/* types.hpp:68-76 — depth camera + RGB camera (pose relative to depth). */
typedef struct vc_sensor {
  vc_intrinsics depth_intr;
  vc_pose pose;
  vc_intrinsics rgb_intr;
  vc_pose rgb_relative;
} vc_sensor;

typedef enum vc_mem_kind { VC_MEM_HOST = 0, VC_MEM_DEVICE = 1 } vc_mem_kind;

/* image.hpp:50-64 — one RgbdFrame.  depth: uint16 mm (0 = invalid),
 * mask: uint8 (nonzero = foreground), or NULL: foreground := depth > 0, derived on the
 * device (the dataset loader's rule, dataset.cpp:99-102); rgb: packed RGB8 of rgb_intr size.
 * Pitches are in bytes; 0 means tightly packed. */
typedef struct vc_view {
  const uint16_t* depth;
  const uint8_t* mask;
  const uint8_t* rgb;
  int32_t depth_pitch, mask_pitch, rgb_pitch;
  int32_t mem_kind; /* vc_mem_kind */
} vc_view;

typedef enum vc_splat_mode { VC_SPLAT_WEIGHTED = 0, VC_SPLAT_SIMPLE = 1 } vc_splat_mode;

/* reconstruct.hpp:12-18 (ReconConfig) + the texture eps (texture.hpp:35).
 * Grid dims: r > 0 selects the reference lattice 2^r x 2^(r+1) x 2^r
 * (reconstruct.cpp:18-20); r == 0 uses nx,ny,nz (powers of two, 4..1024). */
typedef struct vc_recon_config {
  int32_t r;
  int32_t nx, ny, nz;
  int32_t mode; /* vc_splat_mode */
  double discontinuity_mm;
  int32_t padding_voxels;
  int32_t silhouette_radius_px;
  double eps_vis_mm;
} vc_recon_config;

/* volume_recon.hpp:24-28 */
typedef struct vc_grid_spec {
  int32_t nx, ny, nz;
  double origin[3];
  double edge_mm;
} vc_grid_spec;

/* reconstruct.hpp:20-24 (StageTimings) + the CLI's "other" texture column
 * (volcap.cpp:475-481), measured with CUDA events on the context stream.
 * preprocess = build_cloud + confidence_weights (fused kernels; weights_ms
 * is reported as 0).  The split fields break volumetric_ms down. */
typedef struct vc_stage_timings {
  double raw_ms, weights_ms, volumetric_ms, texture_ms, total_ms;
  double splat_ms, fft_ms, iso_ms, mc_ms;
  double h2d_ms, d2h_ms;
} vc_stage_timings;

/* TexturedMesh (texture.hpp:16-28) + FrameReconstruction's volume/iso level
 * (reconstruct.hpp:26-30) + the blended per-vertex colour.
 * Per-sensor arrays are [sensor][vertex]. */
typedef struct vc_textured_mesh {
  int32_t vertex_count, triangle_count, sensor_count, point_count;
  const float* positions;   /* 3V, world mm */
  const float* normals;     /* 3V, unit, outward */
  const int32_t* triangles; /* 3T */
  const uint8_t* visible;   /* K*V */
  const float* uv;          /* 2*K*V, normalised [0,1]^2 (texture.hpp:45-47) */
  const float* weight;      /* K*V */
  const uint8_t* untextured;/* V */
  const uint8_t* rgb;       /* 3V blended colour */
  const double* positions_f64; /* 3V, the exact vertex positions */
  double iso_level;
  vc_grid_spec grid;
  int32_t mem_kind;         /* where the pointers above live */
} vc_textured_mesh;

typedef struct vc_ctx vc_ctx;

/* ---------------------------------------------------------------- context */
int vc_abi_version(void);
const char* vc_status_string(vc_status s);
vc_status vc_ctx_create(int device, vc_ctx** out);
vc_status vc_ctx_destroy(vc_ctx* ctx);
const char* vc_last_error(const vc_ctx* ctx);
/* Output placement for vc_reconstruct_frame: VC_MEM_HOST (default; D2H into
 * context-owned pinned buffers) or VC_MEM_DEVICE (pointers into HBM). */
vc_status vc_ctx_set_output(vc_ctx* ctx, int32_t mem_kind);
/* Collect per-stage CUDA-event timings (adds event records; default off). */
vc_status vc_ctx_set_profiling(vc_ctx* ctx, int32_t enable);
/* Replay the whole frame as one CUDA graph (default on). */
vc_status vc_ctx_set_graphs(vc_ctx* ctx, int32_t enable);
/* The CUDA stream (cudaStream_t) of the context, for interop. */
void* vc_ctx_stream(vc_ctx* ctx);
/* Number of kernels one vc_reconstruct_frame launches (excluding retries). */
int32_t vc_ctx_kernels_per_frame(const vc_ctx* ctx);
/* Per-stage CUDA-event times (ms) of the last frame run with profiling on, 11
 * entries: preprocess (3 kernels), clear, splat (+ touched-row list), fft_x,
 * fft_y, fft_z, ifft_y, ifft_x, iso, mc (4 kernels), texture.  Returns the
 * count written. */
int32_t vc_ctx_kernel_times(const vc_ctx* ctx, double* ms, int32_t max_n);
/* Pinned host memory helpers (for zero-staging H2D of views). */
vc_status vc_host_alloc(vc_ctx* ctx, size_t bytes, void** out);
vc_status vc_host_free(vc_ctx* ctx, void* p);
vc_status vc_device_alloc(vc_ctx* ctx, size_t bytes, void** out);
vc_status vc_device_free(vc_ctx* ctx, void* p);
vc_status vc_memcpy(vc_ctx* ctx, void* dst, const void* src, size_t bytes, int32_t dst_kind, int32_t src_kind);
vc_status vc_synchronize(vc_ctx* ctx);

/* ------------------------------------------------------------ the hot path */
/* reconstruct.cpp:37-78 + texture.cpp:11-72 + per-vertex blend:
 * k views (one per reconstruction sensor, sensors[0..k)) in, textured mesh out. */
vc_status vc_reconstruct_frame(vc_ctx* ctx, const vc_sensor* sensors, const vc_view* views, int32_t k,
                               const vc_recon_config* config, vc_textured_mesh* out,
                               vc_stage_timings* timings);

/* A (fp32, x-fastest, nx*ny*nz) of the last frame, for the mocap consumers
 * (volcap.cpp:427-429).  dst_kind: VC_MEM_HOST or VC_MEM_DEVICE. */
vc_status vc_export_volume(vc_ctx* ctx, float* dst, int32_t dst_kind);
/* Oriented points of the last frame (clouds concatenated in sensor order):
 * pos/nrm 3P doubles, weight P doubles, pix 3P int32 (px, py, sensor);
 * weight_maps k*h*w floats (cloud.hpp:21-26).  Any pointer may be NULL. */
vc_status vc_export_points(vc_ctx* ctx, double* pos, double* nrm, double* weight, int32_t* pix,
                           float* weight_maps);

/* ------------------------------------------------ z-slab decomposition (C5)
 * One frame on P GPUs (SURVEY.md §8(e) "large grids"): rank r owns voxel
 * planes [r*nz/P, (r+1)*nz/P).  Every rank preprocesses all views and splats
 * only its slab (the reference's own slab split, splat.cpp:61-77); the 3-D FFT
 * of integrate.cpp:19-74 runs as local x/y passes, one all-to-all to ky-slabs,
 * the fused z pass, one all-to-all back, local inverse y/x passes; the iso
 * level (splat.cpp:91-101) sums per-point samples across ranks; marching
 * cubes (marching_cubes.cpp:131-210) runs per slab with a 1-plane (below) /
 * 2-plane (above) halo of A and global vertex ids, so the concatenation of
 * the ranks' pieces in rank order IS the single-GPU mesh.
 *
 * Exchanges go through NCCL (libnccl.so.2, loaded at run time; one process
 * per GPU) or, for testing on one device, a loopback exchanger that runs P
 * virtual ranks (P contexts) in one process with device copies. */
typedef struct vc_dist vc_dist;

typedef struct vc_dist_info {
  int32_t rank, world;
  int32_t z_begin, z_end;          /* owned voxel planes */
  int32_t vertex_offset;           /* global id of this piece's first vertex */
  int32_t vertex_total, triangle_offset, triangle_total;
} vc_dist_info;

/* 128-byte NCCL unique id (rank 0 makes it; the caller broadcasts it). */
vc_status vc_dist_nccl_unique_id(uint8_t id[128]);
/* One rank of a P-process job over NCCL on ctx's device. */
vc_status vc_dist_create_nccl(vc_ctx* ctx, int32_t world, int32_t rank, const uint8_t id[128], vc_dist** out);
/* P virtual ranks in this process (ctxs[0..world), usually one device). */
vc_status vc_dist_create_loopback(vc_ctx* const* ctxs, int32_t world, vc_dist** out);
vc_status vc_dist_destroy(vc_dist* d);
/* Local ranks of d (1 for NCCL, world for loopback). */
int32_t vc_dist_local_ranks(const vc_dist* d);
/* vc_reconstruct_frame on the slab decomposition.  out/info: one entry per
 * local rank; out[i] is that rank's piece (its vertices, global indices in its
 * triangles; outputs owned by that rank's context).  nz divisible by world,
 * nz/world >= 2. */
vc_status vc_reconstruct_frame_dist(vc_dist* d, const vc_sensor* sensors, const vc_view* views, int32_t k,
                                    const vc_recon_config* config, vc_textured_mesh* out, vc_dist_info* info,
                                    vc_stage_timings* timings);
/* The owned planes of A of local rank i: (z_end-z_begin)*ny*nx floats. */
vc_status vc_dist_export_volume(vc_dist* d, int32_t local_rank, float* dst, int32_t dst_kind);

/* ------------------------------------------------ per-stage entry points
 * Host arrays in, host arrays out; each runs the same kernels as the frame
 * path on the context's stream.  For parity tests against the reference's
 * stage functions. */

/* build_cloud + confidence_weights for k views; returns the point count in
 * *n_points and keeps the points resident (vc_export_points reads them). */
vc_status vc_stage_preprocess(vc_ctx* ctx, const vc_sensor* sensors, const vc_view* views, int32_t k,
                              const vc_recon_config* config, int64_t* n_points, vc_grid_spec* grid);
/* reconstruct.cpp:16-35 with dims given (r-mode callers pass 2^r,2^(r+1),2^r). */
vc_status vc_fit_grid(const double lo[3], const double hi[3], const int32_t dims[3], int32_t padding_voxels,
                      vc_grid_spec* out);
/* splat.cpp:33-89 (+ the negation of reconstruct.cpp:71 when negate != 0):
 * field 3N floats (x,y,z interleaved per voxel), density N floats in the
 * reference's units (d = sum g(dist;sigma2) W; simple mode: sample count). */
vc_status vc_stage_splat(vc_ctx* ctx, const double* pos, const double* nrm, const double* weight, int64_t n,
                         const vc_grid_spec* grid, int32_t mode, int32_t negate, float* field, float* density);
/* integrate.cpp:19-74: field 3N floats (interleaved) -> A N floats. */
vc_status vc_stage_integrate(vc_ctx* ctx, const float* field, int32_t nx, int32_t ny, int32_t nz, float* A);
/* splat.cpp:91-101: mean trilinear A (fp32 volume) at the points. */
/* Measurement: the integrate chain on a dense pseudo-random field of the given
 * dims, device-resident; ms[0..4] = F-x, F-y, Z, I-y, I-x per launch, ms[5] =
 * the chain (average of `iters` runs).  Used by bench.py's cuFFT comparator. */
vc_status vc_time_integrate(vc_ctx* ctx, int32_t nx, int32_t ny, int32_t nz, int32_t iters, double ms[6]);
vc_status vc_stage_iso_level(vc_ctx* ctx, const float* A, const vc_grid_spec* grid, const double* pos, int64_t n,
                             double* level);
/* marching_cubes.cpp:131-210 on an fp32 volume at a double level.  Vertices
 * are numbered by global edge id ((z*ny+y)*nx+x)*3+axis (ascending);
 * triangles are in the reference's cell-scan order.  Outputs are
 * context-owned host arrays valid until the next call. */
vc_status vc_stage_marching_cubes(vc_ctx* ctx, const float* A, const vc_grid_spec* grid, double level,
                                  int32_t* n_vertices, int32_t* n_triangles, const double** positions,
                                  const float** normals, const int32_t** triangles, const uint64_t** edge_ids);
/* texture.cpp:11-72 + blend for given vertices (3V doubles) and views;
 * weight_maps: k*h*w floats (the clouds' confidence maps). */
vc_status vc_stage_texture(vc_ctx* ctx, const vc_sensor* sensors, const vc_view* views, const float* weight_maps,
                           int32_t k, const double* vertices, int32_t n_vertices, double eps_vis_mm,
                           uint8_t* visible, float* uv, float* weight, uint8_t* untextured, uint8_t* rgb);

/* ---------------------------------------------- frame / mesh I/O (host)
 * The formats either side of the path.  No context,
 * no GPU; on error vc_io_last_error() holds "<what>: <path>" like the
 * reference's std::runtime_error messages. */
typedef struct vc_png_header {
  int32_t width, height, bit_depth, color_type; /* PNG IHDR */
} vc_png_header;
const char* vc_io_last_error(void);
vc_status vc_png_info(const char* path, vc_png_header* info);
/* image_io.cpp:105-122: 16-bit grayscale only ("depth png must be 16-bit grayscale"). */
vc_status vc_png_read_depth(const char* path, uint16_t* dst, int32_t width, int32_t height);
/* image_io.cpp:84-103: any PNG colour type -> RGB8 (expand, strip 16, strip alpha, gray to RGB). */
vc_status vc_png_read_color(const char* path, uint8_t* rgb, int32_t width, int32_t height);
/* image_io.cpp:64-82: 16-bit gray / 8-bit RGB, non-interlaced. */
vc_status vc_png_write_depth(const char* path, const uint16_t* src, int32_t width, int32_t height);
vc_status vc_png_write_color(const char* path, const uint8_t* rgb, int32_t width, int32_t height);
/* mesh_io.cpp:104-145 write_ply: binary little-endian, float xyz (+ normals
 * when non-NULL) + float channels "<name>_<c>", uchar/int faces, channel directory comments. */
vc_status vc_ply_write_mesh(const char* path, const float* xyz, const float* normals, int32_t n_vertices,
                            const int32_t* triangles, int32_t n_triangles, const char* const* channel_names,
                            const int32_t* channel_components, const float* const* channel_data,
                            int32_t n_channels);
/* write_ply(textured.with_channels()) of the reference CLI (volcap.cpp:312-316,
 * texture.cpp:74-91) for a host-memory vc_textured_mesh. */
vc_status vc_ply_write_textured(const char* path, const vc_textured_mesh* mesh);

/* ---------------------------------------------- optional depth filter
 * BASELINE north_star preprocessing ("erosion/bilateral filtering"); the
 * reference has no such filter (cloud.cpp:19-117), so it is OFF by default and
 * any non-zero setting changes results versus the reference.  Erosion: a pixel
 * stays foreground only if its (2e+1)^2 window is foreground.  Bilateral:
 * depth' = round(sum w d / sum w) over valid neighbours within ceil(2 sigma_px),
 * w = exp(-|dp|^2/(2 sigma_px^2) - dz^2/(2 sigma_mm^2)); sigma_px <= 4. */
/* Applied to every view this context stages (all zero = off, the default). */
vc_status vc_ctx_set_depth_filter(vc_ctx* ctx, int32_t erode_px, double sigma_px, double sigma_mm);
/* One view, in place (mask eroded first, then the depth filtered). */
vc_status vc_depth_filter(vc_ctx* ctx, uint16_t* depth, uint8_t* mask, int32_t width, int32_t height,
                          int32_t mem_kind, int32_t erode_px, double sigma_px, double sigma_mm);

/* ---------------------------------------------- colour correction
 * SURVEY §8(f) rank 2 (appearance/color_correction.cpp, hsv.cpp).  Errors of
 * the context-free entry points: vc_io_last_error(). */
/* ColorCorrection::apply(sensor, image) with that sensor's ValueMap: HSV value
 * v := clamp(gain*v + offset, 0, 1), fp64, byte-exact; the identity map leaves
 * the image unchanged.  rgb_in/out: n_pixels*3 bytes in mem_kind memory. */
vc_status vc_color_apply(vc_ctx* ctx, const uint8_t* rgb_in, uint8_t* rgb_out, int64_t n_pixels, double gain,
                         double offset, int32_t mem_kind);
/* mutual_closest_pairs(a, b, max_dist) (color_correction.cpp:16-84) on the GPU:
 * a, b: 3n doubles (host); pairs: 2*min(na, nb) int32 (i, j), ascending i. */
vc_status vc_mutual_closest_pairs(vc_ctx* ctx, const double* a, int32_t na, const double* b, int32_t nb,
                                  double max_dist_mm, int32_t* pairs, int32_t* n_pairs);
/* fit_value_map (color_correction.cpp:97-138): pairs_rgb = n x (first RGB, second RGB). */
vc_status vc_fit_value_map(const uint8_t* pairs_rgb, int32_t n, int32_t ransac_iterations, double inlier_threshold,
                           uint64_t seed, double* gain, double* offset);
/* chain_to_reference (color_correction.cpp:168-199): per-sensor maps toward the reference. */
vc_status vc_chain_to_reference(const int32_t* from, const int32_t* to, const double* gain, const double* offset,
                                int32_t n_edges, int32_t reference, int32_t sensor_count, double* out_gain,
                                double* out_offset);
/* Per-sensor maps applied to every RGB texel the frame's texture blend samples
 * (the corrected images of sequence.cpp:71-73); k = 0 turns it off. */
vc_status vc_ctx_set_color_correction(vc_ctx* ctx, const double* gain, const double* offset, int32_t k);

/* ---------------------------------------------- (A, L) consumers
 * SURVEY §8(f) rank 3 (mocap/binary_volume.cpp, skeletonize.cpp). */
/* binarize(A, L) (binary_volume.cpp:10-66) on the GPU: keep the side of L that
 * holds max(A), then the largest 26-connected component (ties: first in raster
 * order).  A: fp32 x-fastest in mem_kind memory, or NULL = this context's last
 * frame volume.  keep_out (nullable): N bytes; voxels_out: 3*capacity int32
 * (x, y, z) in raster order; *n_voxels = component size (may exceed capacity).
 * Empty interior -> VC_ERR_EMPTY_SCENE ("binarize: empty interior"). */
vc_status vc_binarize(vc_ctx* ctx, const float* A, int32_t mem_kind, const vc_grid_spec* grid, double level,
                      uint8_t* keep_out, int32_t* voxels_out, int64_t capacity, int64_t* n_voxels);
/* boundary_voxels (binary_volume.cpp:68-82): out_xyz 3*n doubles (world centres). */
vc_status vc_boundary_voxels(vc_ctx* ctx, const uint8_t* keep, const vc_grid_spec* grid, const int32_t* voxels,
                             int64_t n, double* out_xyz, int64_t* n_out);
/* skeletonize (skeletonize.cpp:99-161) on the GPU: grid = nx*ny*nz bytes
 * (x fastest, host), voxels = 3n int32 (x, y, z); out: 3n int32, the
 * surviving voxels in input order (identical to the reference's sequential
 * thinning). */
vc_status vc_skeletonize(vc_ctx* ctx, const uint8_t* grid, int32_t nx, int32_t ny, int32_t nz, const int32_t* voxels, int64_t n,
                         int32_t* out, int64_t* n_out);

/* ---------------------------------------------- evaluation renderer + metrics
 * SURVEY §8(f) rank 4 (eval/rasterize.cpp, metrics.cpp, distance_transform.cpp,
 * ssim.cpp).  Host arrays in and out. */
typedef enum vc_render_mode { VC_RENDER_UV_BLEND = 0, VC_RENDER_COLOR_PER_VERTEX = 1 } vc_render_mode;
/* rasterize(textured mesh, camera, view images, mode) (rasterize.cpp:35-161):
 * vertices 3V doubles, triangles 3T, visible/uv/weight [k][V] as in
 * vc_textured_mesh, camera = intr + camera-to-world pose, images[k] RGB8 of
 * image_w[k] x image_h[k].  Outputs w*h: depth float (0 = empty), colour RGB8,
 * silhouette.  The reference's order-dependent float z-buffer test is replayed
 * per pixel in triangle order, so the outputs are exact. */
vc_status vc_rasterize(vc_ctx* ctx, const double* vertices, int32_t n_vertices, const int32_t* triangles,
                       int32_t n_triangles, int32_t k, const uint8_t* visible, const float* uv, const float* weight,
                       const vc_intrinsics* intr, const vc_pose* pose, const uint8_t* const* images,
                       const int32_t* image_w, const int32_t* image_h, int32_t mode, float* depth, uint8_t* color,
                       uint8_t* silhouette);
vc_status vc_vre(vc_ctx* ctx, const uint8_t* rendered, const uint8_t* ground, int32_t w, int32_t h, double* out);
vc_status vc_distance_transform(vc_ctx* ctx, const uint8_t* mask, int32_t w, int32_t h, float* out);
vc_status vc_hausdorff2d(vc_ctx* ctx, const uint8_t* rendered, const uint8_t* ground, int32_t w, int32_t h,
                         double* out, int32_t* has_value);
vc_status vc_cp_rmse(vc_ctx* ctx, const double* ground, int32_t n_ground, const double* recon, int32_t n_recon,
                     double* out);
typedef struct vc_wms3im_options { /* metrics.hpp:30-41 */
  int32_t scales;
  double alpha[3], beta[3], gamma[3];
  double c1, c2, c3;
  int32_t window;
  double sigma;
} vc_wms3im_options;
/* opt NULL = the reference's defaults; *has_value = 0 for an empty silhouette. */
vc_status vc_wms3im(vc_ctx* ctx, const uint8_t* rendered, const uint8_t* ground, const uint8_t* silhouette, int32_t w,
                    int32_t h, const vc_wms3im_options* opt, double* out, int32_t* has_value);

/* ------------------------------------------------------- synthetic capture
 * The reference's synthetic fixture (synth/capsule.cpp, scene.cpp,
 * render.cpp), rendered on the GPU.  Body layout: 15 joints (xyz), 14 radii,
 * 14 RGB8 bone colours (capsule.hpp:25-34). */
typedef struct vc_body {
  double joints[45];
  double radii[14];
  uint8_t colors[42];
} vc_body;

vc_status vc_synth_circle_rig(int32_t recon, int32_t held_out, double radius_mm, double target_height_mm,
                              int32_t width, int32_t height, double focal_px, vc_sensor* out);
vc_status vc_synth_xpose_body(vc_body* out);
vc_status vc_synth_kick_body(int32_t frames, int32_t frame, vc_body* out);
/* render.cpp:23-80: depth (w*h uint16), mask (w*h uint8), rgb (rgb_w*rgb_h*3);
 * dst_kind selects host or device destinations.  Depth noise (sigma > 0)
 * follows render.cpp:50-61 (std::mt19937_64 + normal_distribution, host). */
vc_status vc_synth_render(vc_ctx* ctx, const vc_sensor* sensor, const vc_body* body, double depth_sigma_mm_at_2m,
                          uint64_t seed, double gain, int32_t camera, int32_t frame, uint16_t* depth, uint8_t* mask,
                          uint8_t* rgb, int32_t dst_kind);

#ifdef __cplusplus
}
#endif
#endif /* VC_VC_H_ */

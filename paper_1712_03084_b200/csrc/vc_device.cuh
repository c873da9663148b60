// SPDX-License-Identifier: Apache-2.0
// Device-side types shared by the FTR kernels (sm_100a).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "vc_shared.hpp"

namespace vc {

// Streaming-multiprocessor count of the calling thread's current device,
// queried once per device (grid sizes are multiples of it: persistent and
// grid-stride kernels size their grids as k resident CTAs per SM).
inline int sm_count() {
  static int cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  int v = __atomic_load_n(&cache[dev], __ATOMIC_RELAXED);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 1;
    __atomic_store_n(&cache[dev], v, __ATOMIC_RELAXED);
  }
  return v;
}

// ---------------------------------------------------------------- fp64 helpers
// The binning paths (backprojection, to_voxel, projections) must reproduce
// the reference's IEEE double results bit for bit, so every product and sum
// is rounded on its own (no FMA contraction), in the reference's order.
// These files are also compiled with --fmad=false as a second guard.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

struct d3 {
  double x, y, z;
};
__device__ __forceinline__ d3 mk3(double x, double y, double z) { return d3{x, y, z}; }
__device__ __forceinline__ d3 add3(d3 a, d3 b) { return {dadd(a.x, b.x), dadd(a.y, b.y), dadd(a.z, b.z)}; }
__device__ __forceinline__ d3 sub3(d3 a, d3 b) { return {dsub(a.x, b.x), dsub(a.y, b.y), dsub(a.z, b.z)}; }
__device__ __forceinline__ d3 scale3(double s, d3 a) { return {dmul(s, a.x), dmul(s, a.y), dmul(s, a.z)}; }
__device__ __forceinline__ d3 div3(d3 a, double s) { return {ddiv(a.x, s), ddiv(a.y, s), ddiv(a.z, s)}; }
__device__ __forceinline__ d3 neg3(d3 a) { return {-a.x, -a.y, -a.z}; }
// Eigen dot / squaredNorm order: (a0*b0 + a1*b1) + a2*b2
__device__ __forceinline__ double dot3(d3 a, d3 b) {
  return dadd(dadd(dmul(a.x, b.x), dmul(a.y, b.y)), dmul(a.z, b.z));
}
__device__ __forceinline__ double norm3(d3 a) { return __dsqrt_rn(dot3(a, a)); }
__device__ __forceinline__ d3 cross3(d3 a, d3 b) {
  return {dsub(dmul(a.y, b.z), dmul(a.z, b.y)), dsub(dmul(a.z, b.x), dmul(a.x, b.z)),
          dsub(dmul(a.x, b.y), dmul(a.y, b.x))};
}
// Eigen normalized(): a / sqrt(|a|^2) when |a|^2 > 0
__device__ __forceinline__ d3 normalized3(d3 a) {
  const double z = dot3(a, a);
  return z > 0 ? div3(a, __dsqrt_rn(z)) : a;
}
// R (row-major) * x: ((R0 x + R1 y) + R2 z)
__device__ __forceinline__ d3 mat3(const double* R, d3 v) {
  return {dadd(dadd(dmul(R[0], v.x), dmul(R[1], v.y)), dmul(R[2], v.z)),
          dadd(dadd(dmul(R[3], v.x), dmul(R[4], v.y)), dmul(R[5], v.z)),
          dadd(dadd(dmul(R[6], v.x), dmul(R[7], v.y)), dmul(R[8], v.z))};
}
// R^T * x
__device__ __forceinline__ d3 mat3t(const double* R, d3 v) {
  return {dadd(dadd(dmul(R[0], v.x), dmul(R[3], v.y)), dmul(R[6], v.z)),
          dadd(dadd(dmul(R[1], v.x), dmul(R[4], v.y)), dmul(R[7], v.z)),
          dadd(dadd(dmul(R[2], v.x), dmul(R[5], v.y)), dmul(R[8], v.z))};
}
__device__ __forceinline__ d3 ld3(const double* t) { return {t[0], t[1], t[2]}; }

// camera.cpp:6-10 — project_local: ((fx*X)/Z + cx, (fy*Y)/Z + cy); false if Z <= 0
__device__ __forceinline__ bool project_local(double fx, double fy, double cx, double cy, d3 x, double* u,
                                              double* v) {
  if (x.z <= 0) return false;
  *u = dadd(ddiv(dmul(fx, x.x), x.z), cx);
  *v = dadd(ddiv(dmul(fy, x.y), x.z), cy);
  return true;
}

// std::lround on the device: round half away from zero
__device__ __forceinline__ long long lround_d(double x) { return llround(x); }

}  // namespace vc

// SPDX-License-Identifier: Apache-2.0
// cuFFT comparator for the integrate chain (bench.py only; NOT on the product
// path and not linked into libvc_b200.so).
//
// The reference runs FFTW r2c 3-D per component, the spectral filter
// accumulation, and one c2r 3-D (proj/core/src/recon/integrate.cpp:31-34,
// :44, :46-60, :63).  The library equivalent on the GPU is: one batched
// cuFFT R2C (3 components), one fused filter kernel reading the three
// half-spectra and writing  -j(wx X + wy Y + wz Z)/|w|^2  (DC = 0, Nyquist
// index -> +pi), and one cuFFT C2R, scaled by 1/N in the C2R's consumer (here
// folded into the filter).  cuFFT's C2R on the non-Hermitian kx = 0 and
// kx = nx/2 planes is formally undefined, so this is timing only; parity
// stays with the hand-written chain (k_fft.cu).
#include <cuda_runtime.h>
#include <cufft.h>

#include <cmath>
#include <cstdint>

namespace {

__device__ __forceinline__ float omega(int i, int n) {
  const int m = i <= n / 2 ? i : i - n;  // integrate.cpp:37-40
  return 6.28318530717958647692f * (float)m / (float)n;
}

__global__ void filter_kernel(const float2* __restrict__ S, float2* __restrict__ out, int nx, int ny, int nz,
                              float scale) {
  const int H = nx / 2 + 1;
  const size_t nh = (size_t)nz * ny * H;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nh; i += (size_t)gridDim.x * blockDim.x) {
    const int kx = (int)(i % H);
    const size_t r = i / H;
    const int ky = (int)(r % ny), kz = (int)(r / ny);
    const float wx = omega(kx, nx), wy = omega(ky, ny), wz = omega(kz, nz);
    const float w2 = wx * wx + wy * wy + wz * wz;
    const float2 X = S[i], Y = S[nh + i], Z = S[2 * nh + i];
    const float re = wx * X.x + wy * Y.x + wz * Z.x, im = wx * X.y + wy * Y.y + wz * Z.y;
    // -j * (re + j im) / w2 = (im - j re) / w2
    const float s = w2 > 0.f ? scale / w2 : 0.f;
    out[i] = make_float2(im * s, -re * s);
  }
}

__global__ void fill_kernel(float* f, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 16, h *= 0x7feb352du, h ^= h >> 15, h *= 0x846ca68bu, h ^= h >> 16;
    f[i] = (float)(h >> 8) * (2.0f / 16777216.0f) - 1.0f;
  }
}

}  // namespace

extern "C" {

// ms[0] = batched R2C (3 comps), ms[1] = filter, ms[2] = C2R, ms[3] = chain;
// averaged over `iters` runs after two warm-up runs.  Returns 0 on success,
// a negative code on a CUDA/cuFFT error (-1 alloc, -2 plan, -3 exec).
int vcx_cufft_integrate_time(int device, int nx, int ny, int nz, int iters, double* ms) {
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  const size_t N = (size_t)nx * ny * nz, nh = (size_t)nz * ny * (nx / 2 + 1);
  float* f = nullptr;
  float2* S = nullptr;
  float2* O = nullptr;
  float* A = nullptr;
  int rc = 0;
  cufftHandle pf = 0, pi = 0;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[4] = {};
  if (cudaMalloc(&f, 3 * N * 4) != cudaSuccess || cudaMalloc(&S, 3 * nh * 8) != cudaSuccess ||
      cudaMalloc(&O, nh * 8) != cudaSuccess || cudaMalloc(&A, N * 4) != cudaSuccess) {
    rc = -1;
  } else {
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (auto& e : ev) cudaEventCreate(&e);
    int dims[3] = {nz, ny, nx};
    if (cufftPlanMany(&pf, 3, dims, nullptr, 1, (int)N, nullptr, 1, (int)nh, CUFFT_R2C, 3) != CUFFT_SUCCESS ||
        cufftPlan3d(&pi, nz, ny, nx, CUFFT_C2R) != CUFFT_SUCCESS) {
      rc = -2;
    } else {
      cufftSetStream(pf, st);
      cufftSetStream(pi, st);
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
      fill_kernel<<<sms * 8, 256, 0, st>>>(f, 3 * N, 777u);
      double acc[4] = {0, 0, 0, 0};
      for (int it = -2; it < iters && rc == 0; ++it) {
        cudaEventRecord(ev[0], st);
        if (cufftExecR2C(pf, f, reinterpret_cast<cufftComplex*>(S)) != CUFFT_SUCCESS) rc = -3;
        cudaEventRecord(ev[1], st);
        filter_kernel<<<sms * 8, 256, 0, st>>>(S, O, nx, ny, nz, 1.0f / (float)N);
        cudaEventRecord(ev[2], st);
        if (cufftExecC2R(pi, reinterpret_cast<cufftComplex*>(O), A) != CUFFT_SUCCESS) rc = -3;
        cudaEventRecord(ev[3], st);
        if (cudaStreamSynchronize(st) != cudaSuccess) rc = -3;
        if (it < 0) continue;
        for (int i = 0; i < 3; ++i) {
          float t = 0;
          cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
          acc[i] += t;
        }
        float t = 0;
        cudaEventElapsedTime(&t, ev[0], ev[3]);
        acc[3] += t;
      }
      for (int i = 0; i < 4; ++i) ms[i] = acc[i] / (iters > 0 ? iters : 1);
    }
  }
  if (pf) cufftDestroy(pf);
  if (pi) cufftDestroy(pi);
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  if (st) cudaStreamDestroy(st);
  cudaFree(f), cudaFree(S), cudaFree(O), cudaFree(A);
  return rc;
}

}  // extern "C"

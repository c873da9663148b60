// Throughput of packed vs scalar FP32 SASS forms on sm_100a: warp-instructions
// per cycle per SM for FFMA, FMUL, FADD, FADD2, FMUL2, FFMA2 (broadcast operand).
#include <cstdio>
#include <cuda_runtime.h>
#define ITER 2048
typedef unsigned long long u64;
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ u64 fma2b(float a, u64 b, u64 c) { u64 r; asm volatile("{\n.reg .b64 x;\n mov.b64 x, {%1, %1};\n fma.rn.f32x2 %0, x, %2, %3;\n}" : "=l"(r) : "f"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float ffma(float a, float b, float c) { float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
__device__ __forceinline__ float fadd(float a, float b) { float r; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float fmul(float a, float b) { float r; asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }

template <int OP>
__global__ void k(float* out, float s) {
  u64 a[8]; float f[8];
  for (int i = 0; i < 8; ++i) { f[i] = s * (threadIdx.x + i); a[i] = __double_as_longlong((double)f[i]); }
  const u64 b = __double_as_longlong((double)s);
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) f[i] = ffma(f[i], s, 0.5f);
      if (OP == 1) f[i] = fadd(f[i], s);
      if (OP == 2) f[i] = fmul(f[i], s);
      if (OP == 3) a[i] = add2(a[i], b);
      if (OP == 4) a[i] = mul2(a[i], b);
      if (OP == 5) a[i] = fma2(a[i], b, b);
      if (OP == 6) a[i] = fma2b(s, a[i], b);
    }
  }
  float acc = 0;
  for (int i = 0; i < 8; ++i) acc += f[i] + (float)__longlong_as_double(a[i]);
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, 4);
  const char* names[] = {"FFMA", "FADD", "FMUL", "FADD2", "FMUL2", "FFMA2", "FFMA2.bcast"};
  void (*ks[])(float*, float) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int op = 0; op < 7; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      ks[op]<<<sms * 8, 256>>>(out, 1.0001f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double winst = (double)sms * 8 * 8 * ITER * 8;  // warps * iter * 8 ops
      if (rep) printf("%-12s %.3f ms  %.3f warp-inst/clk/SM (at %d MHz nominal)\n", names[op], ms,
                      winst / sms / (ms * 1e-3 * clk * 1e3), clk / 1000);
    }
  }
  return 0;
}

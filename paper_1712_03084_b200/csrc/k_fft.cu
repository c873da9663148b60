// SPDX-License-Identifier: Apache-2.0
//
// K4-K8 — spectral Poisson integration (integrate.cpp:19-74) as five
// HBM-streaming radix kernels on sm_100a (fp32 complex, shared-memory
// exchange, warp shuffles; tensor cores unused: ~3 flop/byte).
//
//   F-x  acc(float4 U',d') -> V = -s*U'/d' (splat.cpp:83-87 + negation,
//        reconstruct.cpp:71) -> R2C along x for the 3 components (two real
//        sequences per complex FFT) -> S0 = wx*X, S1 = Y, S2 = Z   [kx half]
//   F-y  C2C along y of S0,S1,S2 -> S0 = D = FFT(wx X) + wy FFT(Y), S1 = Z
//        (the divergence is formed before z: 2 components instead of 3)
//   Z    C2C along z of D and Z, filter -j(D + wz Z)/|w|^2 with DC = 0
//        (integrate.cpp:46-60), inverse C2C along z -> S0           [in place]
//   I-y  inverse C2C along y of S0                                  [in place]
//   I-x  C2R along x (numpy irfftn / FFTW c2r semantics: Re() of bins 0 and
//        nx/2) -> A (fp32); the 1/N scale (integrate.cpp:70-72) rides on Z's filter
//
// Spectra are [comp][z][y][kx] with kx pitch H = roundup4(nx/2+1) complex
// (sector-aligned 128 B column chunks).  Every line FFT is a "four-step"
// n = R1*R2 transform: a team of R2 threads each holding R1 elements; step 1
// = R1/R2 register DFTs of length R2 per thread + twiddle W_n^(j1 k2), one
// shared-memory exchange, step 2 = one register DFT of length R1.
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point; no libcuda link)
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "vc_shared.hpp"
#include "vc_device.cuh"

namespace vc {
namespace {

__constant__ float2 c_w32[32];  // W_32^k = exp(-2 pi i k / 32)

__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
  unsigned long long r;
  asm("{\n .reg .b64 x, y;\n mov.b64 x, {%1, %2};\n mov.b64 y, {%3, %4};\n add.rn.f32x2 %0, x, y;\n}"
      : "=l"(r) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  unsigned long long r;
  asm("{\n .reg .b64 x, y;\n mov.b64 x, {%1, %2};\n mov.b64 y, {%3, %4};\n sub.rn.f32x2 %0, x, y;\n}"
      : "=l"(r) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }
__host__ __device__ constexpr int bitrev(int i, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b)
    if (i & (1 << b)) r |= 1 << (bits - 1 - b);
  return r;
}

template <int N>
struct Shape {
  static constexpr int LOG = ilog2(N);
  static constexpr int R2 = 1 << (LOG / 2);   // threads per team
  static constexpr int R1 = N / R2;           // elements per thread (R1 = R2 or 2*R2)
  static constexpr int Q = R1 / R2;
  static_assert(R1 * R2 == N && (Q == 1 || Q == 2), "power of two");
};

// In-register DFT of length M (<= 32), natural order in and out.
template <int M, bool INV>
__device__ __forceinline__ void dft_reg(float2* v) {
  constexpr int LOG = ilog2(M);
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const int r = bitrev(i, LOG);
    if (i < r) {
      const float2 t = v[i];
      v[i] = v[r];
      v[r] = t;
    }
  }
#pragma unroll
  for (int half = 1; half < M; half <<= 1) {
#pragma unroll
    for (int i = 0; i < M; i += 2 * half) {
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const float2 a = v[i + j], b = v[i + j + half];
        const int widx = j * (16 / half);  // W_{2 half}^j = W_32^(j*32/(2 half))
        float2 t;
        if (widx == 0) {
          t = b;
        } else if (widx == 8) {
          t = INV ? make_float2(-b.y, b.x) : make_float2(b.y, -b.x);
        } else {
          const float2 w = c_w32[widx];
          t = INV ? cmulc(b, w) : cmul(b, w);
        }
        v[i + j] = cadd(a, t);
        v[i + j + half] = csub(a, t);
      }
    }
  }
}

// Four-step line FFT.  In:  v[q*R2 + j2] = x[t + R2*q + R1*j2]
//                      Out: v[k1]        = X[t + R2*k1]
// EX::st(j1, k2, val), EX::ld(j1, k2), EX::sync() address the exchange.
template <int N, bool INV, class EX>
__device__ __forceinline__ void fft_line(float2* v, int t, const float2* __restrict__ tw, EX& ex) {
  using S = Shape<N>;
#pragma unroll
  for (int q = 0; q < S::Q; ++q) {
    dft_reg<S::R2, INV>(v + q * S::R2);
    const int j1 = t + S::R2 * q;
#pragma unroll
    for (int k2 = 1; k2 < S::R2; ++k2) {
      const float2 w = __ldg(tw + j1 * k2);
      v[q * S::R2 + k2] = INV ? cmulc(v[q * S::R2 + k2], w) : cmul(v[q * S::R2 + k2], w);
    }
#pragma unroll
    for (int k2 = 0; k2 < S::R2; ++k2) ex.st(j1, k2, v[q * S::R2 + k2]);
  }
  ex.sync();
#pragma unroll
  for (int j1 = 0; j1 < S::R1; ++j1) v[j1] = ex.ld(j1, t);
  ex.sync();
  dft_reg<S::R1, INV>(v);
}

// Forward-output layout (v[k1] = X[t + R2 k1]) -> inverse-input layout
// (v[q*R2 + j2] = X[t + R2 q + R1 j2]), i.e. k1 = q + Q*j2.
template <int N>
__device__ __forceinline__ void relayout_for_inverse(float2* v) {
  using S = Shape<N>;
  if constexpr (S::Q == 2) {
    float2 tmp[S::R1];
#pragma unroll
    for (int i = 0; i < S::R1; ++i) tmp[i] = v[i];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int j2 = 0; j2 < S::R2; ++j2) v[q * S::R2 + j2] = tmp[q + 2 * j2];
  }
}

// Exchange for teams of consecutive lanes (x passes): per-team padded tile;
// a team is T <= 32 adjacent lanes of one warp, so it syncs on its own lanes
// and teams run independently (a team with two all-zero lines exits early).
template <int N>
struct ExTeam {
  float2* buf;  // R1 x (R2 + 1)
  unsigned mask;
  __device__ void st(int j1, int k2, float2 v) { buf[j1 * (Shape<N>::R2 + 1) + k2] = v; }
  __device__ float2 ld(int j1, int k2) { return buf[j1 * (Shape<N>::R2 + 1) + k2]; }
  __device__ void sync() { __syncwarp(mask); }
};
template <int T>
__device__ __forceinline__ unsigned team_mask(int team_lane0) {
  return T >= 32 ? 0xffffffffu : (((1u << T) - 1u) << team_lane0);
}
// Exchange for column tiles (y/z passes): column index innermost.  With rows
// narrower than 128 B (CW = 8: 64 B, CW = 4: 32 B) a warp's 64-bit access
// covers several rows per wavefront: the stores hit rows t*R2 + k2 (the same
// bank window for every t) and would conflict, so row r = j1*R2 + k2 lives at
// r ^ (j1 & SW) — the stores' rows then rotate through the 128 B window with
// t, the loads' rows (j1*R2 + t) still do.
template <int N, int CW>
struct ExCols {
  float2* buf;  // (R1*R2) x CW
  int c;
  static constexpr int R2 = Shape<N>::R2;
  static constexpr int SW = CW * 8 >= 128 ? 0 : 128 / (CW * 8) - 1;  // rows per 128 B, minus one
  __device__ __forceinline__ static int row(int j1, int k2) { return (j1 * R2 + k2) ^ (j1 & SW); }
  __device__ void st(int j1, int k2, float2 v) { buf[row(j1, k2) * CW + c] = v; }
  __device__ float2 ld(int j1, int k2) { return buf[row(j1, k2) * CW + c]; }
  __device__ void sync() { __syncthreads(); }
};

// integrate.cpp:37-40: w = 2 pi m / n, m = i (i <= n/2) else i - n (Nyquist -> +pi);
// evaluated as m * (2 pi / n) in fp32 (one multiply; the filter runs in fp32)
template <int N>
__device__ __forceinline__ float signed_freq(int i) {
  constexpr float k = (float)(2.0 * 3.14159265358979323846 / N);
  return (float)(i <= N / 2 ? i : i - N) * k;
}

// x passes: TEAMS teams of T lanes; keep the exchange tiles under ~48 KB.
template <int N>
struct XCfg {
  static constexpr int T = Shape<N>::R2;
  static constexpr int TILE = Shape<N>::R1 * (T + 1);  // float2 per team
  static constexpr int T0 = 256 / T;
  static constexpr int TEAMS = (T0 * TILE * 8 <= 48 * 1024) ? T0 : (T0 / 2 * TILE * 8 <= 48 * 1024 ? T0 / 2 : T0 / 4);
  static constexpr int THREADS = T * TEAMS;
  static constexpr int SMEM = TEAMS * TILE * 8;
};
// y/z passes: CW columns per tile (16 x 8 B = 128 B; 8 for long lines).
template <int N>
struct CCfg {
  static constexpr int CW = N >= 512 ? 8 : 16;
  static constexpr int THREADS = CW * Shape<N>::R2;
  static constexpr int SMEM = N * CW * 8;  // one staged tile (= exchange buffer)
};

// Pass outputs are read by the next pass right away: plain (L2-allocating)
// stores, so what fits in the 126 MB L2 is not re-read from HBM.
template <class T>
__device__ __forceinline__ void st_out(T* p, T v) {
  *p = v;
}

// Predicated streaming load (no branch): zero when !pred.
__device__ __forceinline__ float4 ld_pred_cs(const float4* p, bool pred) {
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  asm("{\n .reg .pred q;\n setp.ne.u32 q, %5, 0;\n @q ld.global.cs.v4.f32 {%0, %1, %2, %3}, [%4];\n}"
      : "+f"(r.x), "+f"(r.y), "+f"(r.z), "+f"(r.w)
      : "l"(p), "r"((unsigned)pred));
  return r;
}

// Predicated 8-byte load that does not allocate in L1 (zero when !pred).
__device__ __forceinline__ float2 ld_pred_f2(const float2* p, bool pred) {
  float2 r = make_float2(0.f, 0.f);
  asm("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n @q ld.global.L1::no_allocate.v2.f32 {%0, %1}, [%2];\n}"
      : "+f"(r.x), "+f"(r.y)
      : "l"(p), "r"((unsigned)pred));
  return r;
}

// I-y: narrower tiles from 256 points up (one staged tile per CTA, so more,
// smaller CTAs overlap their loads better; measured 31 -> 29 us at 256^3)
template <int N>
struct ICfg {
  static constexpr int CW = N >= 256 ? 8 : 16;
  static constexpr int THREADS = CW * Shape<N>::R2;
  static constexpr int SMEM = N * CW * 8;
};

// F-y: narrower tiles from 256 points up (only the non-empty planes work, so
// more, smaller CTAs spread them over the SMs)
template <int N>
struct FCfg {
  static constexpr int CW = N >= 256 ? 8 : 16;
  static constexpr int THREADS = CW * Shape<N>::R2;
  static constexpr int SMEM = N * CW * 8;
  // staged tiles: all three components in flight, except at 512 points where
  // the third reuses the first's buffer (64 KB instead of 96: 3 CTAs per SM)
  static constexpr int NBUF = 3;
  static constexpr int MINB = N >= 1024 ? 1 : (N == 512 ? 2 : (N >= 256 ? 4 : 2));
};

// Z: narrow tiles from 256 points up (VC_ZCW=4: 4 columns, 8 CTAs/SM at 256)
#ifndef VC_ZCW256
#define VC_ZCW256 8
#endif
template <int N>
struct ZCfg {
  static constexpr int CW = N == 256 ? VC_ZCW256 : (N >= 256 ? 8 : 16);
  static constexpr int THREADS = CW * Shape<N>::R2;
  static constexpr int SMEM = N * CW * 8;
};

// ------------------------------------------------------------------ F-x
template <int NX>
__global__ void __launch_bounds__(XCfg<NX>::THREADS, 2) fx_kernel(float4* __restrict__ acc, float2* __restrict__ S0,
                                                       float2* __restrict__ S1, float2* __restrict__ S2, int rows,
                                                       int H, const uint32_t* __restrict__ rowbits, int mode,
                                                       const float2* __restrict__ tw,
                                                       const int32_t* __restrict__ rowlist) {
  using S = Shape<NX>;
  constexpr int T = S::R2, R1 = S::R1, TEAMS = XCfg<NX>::TEAMS;
  constexpr int CH = NX < 32 ? 0 : 5;  // log2 of the 32-voxel chunk (whole row when nx < 32)
  extern __shared__ float2 dyn_smem[];
  const int team = threadIdx.x / T, t = threadIdx.x % T;
  const int lane = threadIdx.x & 31, team_lane0 = lane - t;
  ExTeam<NX> ex{dyn_smem + team * XCfg<NX>::TILE, team_mask<T>(team_lane0)};
  // rows: the splat's touched-row list, two per team (any two rows: the z
  // components of a pair share one complex FFT), persistent teams over the
  // list; without a list, row pairs (2p, 2p+1) of the whole slab
  const int n = rowlist ? rowlist[0] : rows;
  const int pairs = (n + 1) / 2;
  const int step = rowlist ? gridDim.x * TEAMS : pairs;
  for (int pair = blockIdx.x * TEAMS + team; pair < pairs; pair += step) {
  const int l0 = rowlist ? __ldg(rowlist + 1 + 2 * pair) : 2 * pair;
  const int l1 = 2 * pair + 1 < n ? (rowlist ? __ldg(rowlist + 2 + 2 * pair) : 2 * pair + 1) : -1;
  const uint32_t bits0 = rowbits ? __ldg(rowbits + l0) : 0xffffffffu;
  const uint32_t bits1 = l1 < 0 ? 0u : (rowbits ? __ldg(rowbits + l1) : 0xffffffffu);
  if ((bits0 | bits1) == 0u) continue;  // both rows empty: F-y treats them as zero
  const bool live = true;

  auto load_line = [&](int l, uint32_t bits, float2* xy, float* zc) {
    // all R1 predicated loads in flight before the first use (untouched
    // chunks hold stale data and are neither read nor used)
    float4 av[R1];
#pragma unroll
    for (int q = 0; q < S::Q; ++q)
#pragma unroll
      for (int j2 = 0; j2 < T; ++j2) {
        const int j = t + T * q + R1 * j2;
        const bool touched = CH == 0 ? bits != 0u : ((bits >> (j >> CH)) & 1u) != 0u;
        av[q * T + j2] = ld_pred_cs(acc + (size_t)l * NX + j, touched);
      }
#pragma unroll
    for (int q = 0; q < S::Q; ++q)
#pragma unroll
      for (int j2 = 0; j2 < T; ++j2) {
        const float4 a = av[q * T + j2];
        float s = 0.f;
        if (mode == 0) {
          if (a.w >= 1e-6f) s = -1.2247448713915890f / a.w;  // -sqrt(1.5)/d'
        } else {
          if (a.w > 0.f) s = -1.f / a.w;
        }
        xy[q * T + j2] = make_float2(a.x * s, a.y * s);
        zc[q * T + j2] = a.z * s;
      }
    // with the touched-row list (frames): the chunks just read are zeroed for
    // the next frame's splat here, instead of by a clear pass at frame start
    if (rowlist) {
#pragma unroll
      for (int q = 0; q < S::Q; ++q)
#pragma unroll
        for (int j2 = 0; j2 < T; ++j2) {
          const int j = t + T * q + R1 * j2;
          if (CH == 0 ? bits != 0u : ((bits >> (j >> CH)) & 1u) != 0u)
            __stcs(acc + (size_t)l * NX + j, make_float4(0.f, 0.f, 0.f, 0.f));
        }
    }
  };
  // Split C = FFT(a + i b) into A = FFT(a), B = FFT(b) for this thread's bins
  // k = t + T*k1 (partner bin n-k lives in lane T-t, element R1-1-k1).
  auto split_store = [&](float2* v, float2* outA, size_t offA, float2* outB, size_t offB, bool scale_wx) {
    const int src = team_lane0 + ((T - t) & (T - 1));
#pragma unroll
    for (int k1 = 0; k1 <= R1 / 2; ++k1) {
      const float2 pv = make_float2(__shfl_sync(ex.mask, v[R1 - 1 - k1].x, src),
                                    __shfl_sync(ex.mask, v[R1 - 1 - k1].y, src));
      const float2 own = v[(R1 - k1) & (R1 - 1)];
      const float2 e = t == 0 ? own : pv;  // C[n-k]
      const float2 d = v[k1];
      const int k = t + T * k1;
      if (k1 < R1 / 2 || t == 0) {
        float2 A = make_float2(0.5f * (d.x + e.x), 0.5f * (d.y - e.y));  // (d + conj e)/2
        const float2 B = make_float2(0.5f * (d.y + e.y), -0.5f * (d.x - e.x));  // (d - conj e)/(2i)
        if (scale_wx) {
          const float wx = signed_freq<NX>(k);  // k <= NX/2
          A.x *= wx, A.y *= wx;
        }
        if (live) {
          st_out(outA + offA + k, A);
          st_out(outB + offB + k, B);
        }
      }
    }
  };

  auto split_store_z = [&](float2* v, size_t offA, size_t offB, bool stA, bool stB) {
    const int src = team_lane0 + ((T - t) & (T - 1));
#pragma unroll
    for (int k1 = 0; k1 <= R1 / 2; ++k1) {
      const float2 pv = make_float2(__shfl_sync(ex.mask, v[R1 - 1 - k1].x, src),
                                    __shfl_sync(ex.mask, v[R1 - 1 - k1].y, src));
      const float2 own = v[(R1 - k1) & (R1 - 1)];
      const float2 e = t == 0 ? own : pv;
      const float2 d = v[k1];
      const int k = t + T * k1;
      if (k1 < R1 / 2 || t == 0) {
        if (stA) st_out(S2 + offA + k, make_float2(0.5f * (d.x + e.x), 0.5f * (d.y - e.y)));
        if (stB) st_out(S2 + offB + k, make_float2(0.5f * (d.y + e.y), -0.5f * (d.x - e.x)));
      }
    }
  };
  float2 v[R1];
  float z0[R1];
  load_line(l0, bits0, v, z0);
  float z1[R1];
  if (bits0) {
    fft_line<NX, false>(v, t, tw, ex);
    split_store(v, S0, (size_t)l0 * H, S1, (size_t)l0 * H, true);
  }
  load_line(l1, bits1, v, z1);
  if (bits1) {
    fft_line<NX, false>(v, t, tw, ex);
    split_store(v, S0, (size_t)l1 * H, S1, (size_t)l1 * H, true);
  }
#pragma unroll
  for (int i = 0; i < R1; ++i) v[i] = make_float2(z0[i], z1[i]);
  fft_line<NX, false>(v, t, tw, ex);
  split_store_z(v, (size_t)l0 * H, (size_t)l1 * H, bits0 != 0u, bits1 != 0u);
  }
}

// ------------------------------------------------------------------ tile staging
// Column tiles (n rows x CW complex columns, row stride `stride` elements) are
// staged into shared memory with cp.async (16 B = 2 columns per request,
// L1-bypassing), so every component of a CTA is in flight while the previous
// one is transformed; the staged tile then doubles as that component's
// exchange buffer.  Rows flagged empty (or columns past the pitch) zero-fill.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(pred ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(pred ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Thread i stages chunk c2 = i % CPR of rows j = i / CPR + k * (THREADS / CPR);
// `rowmask` (bit k) says which of those rows are non-empty (row_flags()).
template <int N, int CW, int THREADS>
__device__ __forceinline__ uint32_t row_flags(const uint32_t* rowbits) {
  constexpr int CPR = CW / 2, RSTEP = THREADS / CPR, NR = N / RSTEP;
  static_assert(NR <= 32, "row mask");
  if (!rowbits) return 0xffffffffu;
  uint32_t m = 0;
  const int j0 = threadIdx.x / CPR;
#pragma unroll
  for (int k = 0; k < NR; ++k) m |= (__ldg(rowbits + j0 + k * RSTEP) != 0u ? 1u : 0u) << k;
  return m;
}
// Row j of a tile lives at src + (j >> lp) * blkstride + (j & ((1 << lp) - 1)) * stride:
// one uniform stride (lp = 31) for the single-GPU layouts, blocks of 2^lp rows
// for the slab exchange layouts of the distributed transform.
struct RowMap {
  size_t stride, blkstride;
  int lp;
  __device__ __forceinline__ size_t off(int j) const {
    return (size_t)(j >> lp) * blkstride + (size_t)(j & ((1 << lp) - 1)) * stride;
  }
};
// Uniform row stride: one base address per thread, stepped by RSTEP rows (rows
// past the pitch or flagged empty are zero-filled, their address is not read).
template <int N, int CW, int THREADS>
__device__ __forceinline__ void stage_tile_u(float2* tile, const float2* src, size_t stride, int kx0, int H,
                                             uint32_t rowmask) {
  constexpr int CPR = CW / 2, RSTEP = THREADS / CPR, NR = N / RSTEP;
  const int j0 = threadIdx.x / CPR, c2 = threadIdx.x % CPR;
  const int kx = kx0 + 2 * c2;
  const bool colok = kx < H;
  const float2* p = src + (colok ? (size_t)j0 * stride + kx : (size_t)0);
  const size_t step = (size_t)RSTEP * stride;
  float2* t = tile + j0 * CW + 2 * c2;
#pragma unroll
  for (int k = 0; k < NR; ++k, p += step) cp_async16(t + k * RSTEP * CW, p, colok && ((rowmask >> k) & 1u));
}

template <int N, int CW, int THREADS>
__device__ __forceinline__ void stage_tile(float2* tile, const float2* src, size_t stride, int kx0, int H,
                                           uint32_t rowmask) {
  stage_tile_u<N, CW, THREADS>(tile, src, stride, kx0, H, rowmask);
}
template <int N, int CW, int THREADS>
__device__ __forceinline__ void stage_tile(float2* tile, const float2* src, RowMap rm, int kx0, int H,
                                           uint32_t rowmask) {
  if (rm.lp >= 30 || (N >> rm.lp) <= 1) {  // all N rows in one block: uniform stride (one GPU)
    stage_tile_u<N, CW, THREADS>(tile, src, rm.stride, kx0, H, rowmask);
    return;
  }
  constexpr int CPR = CW / 2, RSTEP = THREADS / CPR, NR = N / RSTEP;
  const int j0 = threadIdx.x / CPR, c2 = threadIdx.x % CPR;
  const int kx = kx0 + 2 * c2;
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    const int j = j0 + k * RSTEP;
    const bool ok = kx < H && ((rowmask >> k) & 1u);
    cp_async16(tile + j * CW + 2 * c2, ok ? (const void*)(src + rm.off(j) + kx) : (const void*)src, ok);
  }
}

// Nyquist tile: column c is the kx = nx/2 column of line group c (another
// plane / ky row), at src + c*colstride, rows by `rm`; element (j, c) is
// zero-filled when c >= ncol or its flag word flags[c*fstride + j] is 0.
template <int N, int CW, int THREADS>
__device__ __forceinline__ void stage_nyq(float2* tile, const float2* src, RowMap rm, size_t colstride, int ncol,
                                          const uint32_t* flags, int fstride) {
  constexpr int NI = N * CW / THREADS;
  static_assert(NI * THREADS == N * CW && NI <= 32, "tile");
  uint32_t ok = 0;
#pragma unroll
  for (int k = 0; k < NI; ++k) {  // all flag loads in flight before any copy
    const int i = threadIdx.x + k * THREADS, j = i / CW, c = i % CW;
    ok |= (c < ncol && (!flags || __ldg(flags + (size_t)c * fstride + j) != 0u) ? 1u : 0u) << k;
  }
#pragma unroll
  for (int k = 0; k < NI; ++k) {
    const int i = threadIdx.x + k * THREADS, j = i / CW, c = i % CW;
    const bool p = (ok >> k) & 1u;
    cp_async8(tile + j * CW + c, p ? (const void*)(src + (size_t)c * colstride + rm.off(j)) : (const void*)src, p);
  }
}

template <int N, int CW>
__device__ __forceinline__ void tile_to_regs(const float2* tile, int c, int t, float2* v) {
  using S = Shape<N>;
#pragma unroll
  for (int q = 0; q < S::Q; ++q)
#pragma unroll
    for (int j2 = 0; j2 < S::R2; ++j2) v[q * S::R2 + j2] = tile[(t + S::R2 * q + S::R1 * j2) * CW + c];
}

// ------------------------------------------------------------------ F-y
// Outputs D, Z go to O0, O1 (in place over S0, S1 on one GPU).  Row ky of
// plane zl is stored at ((s*nzl + zl)*kyl + yl)*H with s = ky / kyl, yl = ky % kyl:
// for the slab transform that is the send layout of the forward all-to-all
// (block s = the ky-slab of rank s); with kyl = ny it is the plain layout.
template <int NY>
__global__ void __launch_bounds__(FCfg<NY>::THREADS, FCfg<NY>::MINB) fy_kernel(const float2* S0, const float2* S1,
                                                                 const float2* __restrict__ S2, float2* O0, float2* O1,
                                                                 int nxh, int H, int lk,
                                                                 const float2* __restrict__ tw,
                                                                 const uint32_t* __restrict__ rowbits,
                                                                 uint32_t* __restrict__ planeflag) {
  using S = Shape<NY>;
  constexpr int T = S::R2, R1 = S::R1, kCW = FCfg<NY>::CW, TH = FCfg<NY>::THREADS;
  constexpr int NB = FCfg<NY>::NBUF;
  extern __shared__ float2 sh[];  // NB tiles of NY x kCW
  float2* b0 = sh;
  float2* b1 = sh + NY * kCW;
  float2* b2 = NB == 3 ? sh + 2 * NY * kCW : b0;
  const int c = threadIdx.x % kCW, t = threadIdx.x / kCW;
  const int kx0 = blockIdx.x * kCW, kx = kx0 + c;
  const bool live = kx < nxh;
  const size_t plane = (size_t)blockIdx.y * NY * H;
  // empty rows (F-x skipped them) are zero-filled; a plane with no splat
  // contribution at all has zero spectra: it is skipped and flagged for Z
  const uint32_t rm = row_flags<NY, kCW, TH>(rowbits ? rowbits + (size_t)blockIdx.y * NY : nullptr);
  const int nonempty = __syncthreads_or(rm != 0u);
  if (blockIdx.x == 0 && threadIdx.x == 0) planeflag[blockIdx.y] = nonempty ? 1u : 0u;
  if (!nonempty) return;
  stage_tile<NY, kCW, TH>(b0, S0 + plane, H, kx0, H, rm);
  cp_async_commit();
  stage_tile<NY, kCW, TH>(b1, S1 + plane, H, kx0, H, rm);
  cp_async_commit();
  if constexpr (NB == 3) {
    stage_tile<NY, kCW, TH>(b2, S2 + plane, H, kx0, H, rm);
    cp_async_commit();
  }
  float2 d[R1], v[R1];
  cp_async_wait<NB - 1>();
  __syncthreads();
  tile_to_regs<NY, kCW>(b0, c, t, d);
  __syncthreads();
  ExCols<NY, kCW> e0{b0, c};
  fft_line<NY, false>(d, t, tw, e0);
  if constexpr (NB == 2) {  // b0 is free (fft_line ends on a barrier after its last read)
    stage_tile<NY, kCW, TH>(b2, S2 + plane, H, kx0, H, rm);
    cp_async_commit();
  }
  cp_async_wait<1>();
  __syncthreads();
  tile_to_regs<NY, kCW>(b1, c, t, v);
  __syncthreads();
  ExCols<NY, kCW> e1{b1, c};
  fft_line<NY, false>(v, t, tw, e1);
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) {
    const float wy = signed_freq<NY>(t + T * k1);
    d[k1] = make_float2(d[k1].x + wy * v[k1].x, d[k1].y + wy * v[k1].y);
  }
  cp_async_wait<0>();
  __syncthreads();
  tile_to_regs<NY, kCW>(b2, c, t, v);
  __syncthreads();
  ExCols<NY, kCW> e2{b2, c};
  fft_line<NY, false>(v, t, tw, e2);
  if (live) {
    const int kyl = 1 << lk, nzl = gridDim.y;
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      const int ky = t + T * k1;
      const size_t o = ((size_t)((ky >> lk) * nzl + blockIdx.y) * kyl + (ky & (kyl - 1))) * H + kx;
      st_out(O0 + o, d[k1]);
      st_out(O1 + o, v[k1]);
    }
  }
}

// ------------------------------------------------------------------ F-y, pipelined (1024 points)
// At 1024 points the three staged 64 KB tiles hold the SM alone (one CTA), so
// fy_kernel's loads and transforms never overlap.  Here persistent CTAs walk
// the tiles of the live planes only (fy_planes_kernel lists them, and writes
// every plane's flag for Z): as soon as a component's transform has released
// its buffer, the next tile's same component is staged into it, under the
// remaining transforms and the stores.  Same per-tile arithmetic as fy_kernel.
__global__ void __launch_bounds__(256) fy_planes_kernel(const uint32_t* __restrict__ rowbits, int ny, int nzl,
                                                        uint32_t* __restrict__ planeflag, int32_t* __restrict__ plist) {
  const int z = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (z >= nzl) return;
  bool any = rowbits == nullptr;
  for (int y = lane; y < ny && !any; y += 32) any = __ldg(rowbits + (size_t)z * ny + y) != 0u;
  const bool live = __any_sync(0xffffffffu, any);
  if (lane == 0) {
    planeflag[z] = live ? 1u : 0u;
    if (live) plist[1 + atomicAdd(plist, 1)] = z;
  }
}

template <int NY>
__global__ void __launch_bounds__(FCfg<NY>::THREADS, 1)
    fyp_kernel(const float2* S0, const float2* S1, const float2* __restrict__ S2, float2* O0, float2* O1, int nxh,
               int H, int lk, const float2* __restrict__ tw, const uint32_t* __restrict__ rowbits,
               const int32_t* __restrict__ plist, int ntx, int nzl) {
  using S = Shape<NY>;
  constexpr int T = S::R2, R1 = S::R1, kCW = FCfg<NY>::CW, TH = FCfg<NY>::THREADS;
  extern __shared__ float2 sh[];  // 3 tiles of NY x kCW
  float2* b0 = sh;
  float2* b1 = sh + NY * kCW;
  float2* b2 = sh + 2 * NY * kCW;
  const int c = threadIdx.x % kCW, t = threadIdx.x / kCW;
  const int ntiles = plist[0] * ntx;
  int tile = blockIdx.x;
  if (tile >= ntiles) return;
  auto plane_of = [&](int tl) { return plist[1 + tl / ntx]; };
  auto rmask = [&](int tl) {
    return tl < ntiles ? row_flags<NY, kCW, TH>(rowbits ? rowbits + (size_t)plane_of(tl) * NY : nullptr) : 0u;
  };
  auto stage = [&](float2* dst, const float2* comp, int tl, uint32_t rm) {
    if (tl < ntiles) stage_tile<NY, kCW, TH>(dst, comp + (size_t)plane_of(tl) * NY * H, H, (tl % ntx) * kCW, H, rm);
    cp_async_commit();  // (empty groups keep the wait counts uniform)
  };
  {
    const uint32_t rm = rmask(tile);
    stage(b0, S0, tile, rm);
    stage(b1, S1, tile, rm);
    stage(b2, S2, tile, rm);
  }
  for (; tile < ntiles; tile += gridDim.x) {
    const int next = tile + gridDim.x;
    const uint32_t rmn = rmask(next);
    const int z = plane_of(tile), kx = (tile % ntx) * kCW + c;
    float2 d[R1], v[R1];
    cp_async_wait<2>();  // this tile's S0 (S1, S2 and the next tiles' may be in flight)
    __syncthreads();
    tile_to_regs<NY, kCW>(b0, c, t, d);
    __syncthreads();
    ExCols<NY, kCW> e0{b0, c};
    fft_line<NY, false>(d, t, tw, e0);
    stage(b0, S0, next, rmn);
    cp_async_wait<2>();
    __syncthreads();
    tile_to_regs<NY, kCW>(b1, c, t, v);
    __syncthreads();
    ExCols<NY, kCW> e1{b1, c};
    fft_line<NY, false>(v, t, tw, e1);
    stage(b1, S1, next, rmn);
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      const float wy = signed_freq<NY>(t + T * k1);
      d[k1] = make_float2(d[k1].x + wy * v[k1].x, d[k1].y + wy * v[k1].y);
    }
    cp_async_wait<2>();
    __syncthreads();
    tile_to_regs<NY, kCW>(b2, c, t, v);
    __syncthreads();
    ExCols<NY, kCW> e2{b2, c};
    fft_line<NY, false>(v, t, tw, e2);
    stage(b2, S2, next, rmn);
    if (kx < nxh) {
      const int kyl = 1 << lk;
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) {
        const int ky = t + T * k1;
        const size_t o = ((size_t)((ky >> lk) * nzl + z) * kyl + (ky & (kyl - 1))) * H + kx;
        st_out(O0 + o, d[k1]);
        st_out(O1 + o, v[k1]);
      }
    }
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------ Z (fused)
// FFT_z(D) is parked in its staged tile while FFT_z(Z) runs (one register
// array live, three CTAs per SM).
template <int NZ, bool NYQ>
__device__ __forceinline__ void z_body(float2* __restrict__ S0, const float2* __restrict__ S1, int nx, int ny, int kyl,
                                       int ky0, int H, float fx_step, float fy_step, float scale,
                                       const float2* __restrict__ tw, const uint32_t* __restrict__ planeflag) {
  using S = Shape<NZ>;
  constexpr int T = S::R2, R1 = S::R1, kCW = ZCfg<NZ>::CW, TH = ZCfg<NZ>::THREADS;
  extern __shared__ float2 sh[];  // 2 tiles of NZ x kCW
  float2* b0 = sh;
  float2* b1 = sh + NZ * kCW;
  const int c = threadIdx.x % kCW, t = threadIdx.x / kCW;
  const size_t zstride = (size_t)kyl * H;
  // column c: (kx, local ky row); the Nyquist tile packs kx = nx/2 of kCW ky rows
  const int kx = NYQ ? nx / 2 : blockIdx.x * kCW + c;
  const int kyr = NYQ ? blockIdx.y * kCW + c : blockIdx.y;
  if (NYQ) {
    const int y0 = blockIdx.y * kCW;
    if (y0 >= kyl) return;
    const size_t off = (size_t)y0 * H + nx / 2;
    const RowMap rm{zstride, 0, 31};
    stage_nyq<NZ, kCW, TH>(b0, S0 + off, rm, (size_t)H, min(kCW, kyl - y0), planeflag, 0);
    cp_async_commit();
    stage_nyq<NZ, kCW, TH>(b1, S1 + off, rm, (size_t)H, min(kCW, kyl - y0), planeflag, 0);
    cp_async_commit();
  } else {
    const uint32_t pm = row_flags<NZ, kCW, TH>(planeflag);  // planes F-y skipped are zero
    stage_tile<NZ, kCW, TH>(b0, S0 + (size_t)kyr * H, zstride, blockIdx.x * kCW, H, pm);
    cp_async_commit();
    stage_tile<NZ, kCW, TH>(b1, S1 + (size_t)kyr * H, zstride, blockIdx.x * kCW, H, pm);
    cp_async_commit();
  }
  float2 v[R1];
  cp_async_wait<1>();
  __syncthreads();
  tile_to_regs<NZ, kCW>(b0, c, t, v);
  __syncthreads();
  ExCols<NZ, kCW> e0{b0, c};
  fft_line<NZ, false>(v, t, tw, e0);
  // park FFT_z(D): thread (c, t) owns slots (t + T*k1, c) of b0 (free again)
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) b0[(t + T * k1) * kCW + c] = v[k1];
  cp_async_wait<0>();
  __syncthreads();
  tile_to_regs<NZ, kCW>(b1, c, t, v);
  __syncthreads();
  ExCols<NZ, kCW> e1{b1, c};
  fft_line<NZ, false>(v, t, tw, e1);
  // integrate.cpp:37-40 frequencies 2 pi m / n (fp32: m * (2 pi / n))
  const int ky = ky0 + kyr;
  const float wx = (float)(kx <= nx / 2 ? kx : kx - nx) * fx_step;
  const float wy = (float)(ky <= ny / 2 ? ky : ky - ny) * fy_step;
  const float wxy = wx * wx + wy * wy;
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) {
    const int kz = t + T * k1;
    const float wz = signed_freq<NZ>(kz);
    const float w2 = wxy + wz * wz;
    const float2 d = b0[kz * kCW + c];
    const float2 s = make_float2(d.x + wz * v[k1].x, d.y + wz * v[k1].y);
    const float inv = (kx == 0 && ky == 0 && kz == 0) ? 0.f : __fdividef(scale, w2);  // 1/N of the c2r folded in
    v[k1] = make_float2(s.y * inv, -s.x * inv);  // (-i/|w|^2) * s
  }
  __syncthreads();  // everyone has read its parked D before b0 becomes the exchange
  relayout_for_inverse<NZ>(v);
  fft_line<NZ, true>(v, t, tw, e0);
  const bool live = NYQ ? kyr < kyl : kx <= nx / 2;
  if (live) {
    const size_t base = (size_t)kyr * H + kx;
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) st_out(S0 + base + (size_t)(t + T * k1) * zstride, v[k1]);
  }
}

// Input: D, Z as [z][kyl][H] (kyl = ny on one GPU; a ky-slab starting at ky0
// after the forward all-to-all).  The result overwrites S0 in place.
template <int NZ>
__global__ void __launch_bounds__(ZCfg<NZ>::THREADS, NZ >= 1024 ? 1 : (NZ == 256 ? 32 / VC_ZCW256 : (NZ == 512 ? 3 : 2)))
    z_kernel(float2* __restrict__ S0, const float2* __restrict__ S1, int nx, int ny, int kyl, int ky0, int H, int nyq,
             float fx_step, float fy_step, float scale, const float2* __restrict__ tw,
             const uint32_t* __restrict__ planeflag) {
  if (blockIdx.x == nyq)
    z_body<NZ, true>(S0, S1, nx, ny, kyl, ky0, H, fx_step, fy_step, scale, tw, planeflag);
  else
    z_body<NZ, false>(S0, S1, nx, ny, kyl, ky0, H, fx_step, fy_step, scale, tw, planeflag);
}

// ------------------------------------------------------------------ Z, pipelined (1024 planes)
// One persistent CTA per SM over the main column tiles, three NZ x CW stage
// buffers: while tile i's transforms run, tile i+1's D lands in the free
// buffer (issued at the top of the iteration) and its Z in tile i's Z buffer
// (issued as soon as FFT_z(Z) has released it).  At these sizes the two
// staged tiles of z_kernel hold the SM alone (one CTA), so its loads and its
// transforms never overlap; here they do.  Same per-tile arithmetic as
// z_body; the packed Nyquist tiles stay with z_kernel.  (At 512 planes
// z_kernel keeps 2-3 CTAs per SM and beats this kernel's one: 0.465 against
// 0.684 ms per C3 frame, profiles/r02_experiments.json.)
template <int NZ>
struct ZPCfg {
  static constexpr int CW = 8;
  static constexpr int THREADS = CW * Shape<NZ>::R2;
  static constexpr int TILE = NZ * CW;  // float2
  static constexpr int SMEM = 3 * TILE * 8;
};

template <int NZ>
__global__ void __launch_bounds__(ZPCfg<NZ>::THREADS, 1)
    zp_kernel(float2* __restrict__ S0, const float2* __restrict__ S1, int nx, int ny, int kyl, int ky0, int H, int ntx,
              float fx_step, float fy_step, float scale, const float2* __restrict__ tw,
              const uint32_t* __restrict__ planeflag) {
  using S = Shape<NZ>;
  using CF = ZPCfg<NZ>;
  constexpr int T = S::R2, R1 = S::R1, kCW = CF::CW, TH = CF::THREADS;
  extern __shared__ float2 sh[];
  const int c = threadIdx.x % kCW, t = threadIdx.x / kCW;
  const size_t zstride = (size_t)kyl * H;
  const int ntiles = ntx * kyl;
  int tile = blockIdx.x;
  if (tile >= ntiles) return;
  const uint32_t pm = row_flags<NZ, kCW, TH>(planeflag);  // planes F-y skipped are zero
  auto stage = [&](float2* dst, const float2* comp, int tl) {
    if (tl < ntiles) {
      const int kyr = tl / ntx;
      stage_tile<NZ, kCW, TH>(dst, comp + (size_t)kyr * H, zstride, (tl - kyr * ntx) * kCW, H, pm);
    }
    cp_async_commit();  // (empty groups keep the wait counts uniform)
  };
  int bD = 0, bZ = 1, bF = 2;  // buffers: this tile's D, its Z, free
  stage(sh + bD * CF::TILE, S0, tile);
  stage(sh + bZ * CF::TILE, S1, tile);
  for (; tile < ntiles; tile += gridDim.x) {
    const int next = tile + gridDim.x;
    float2* b0 = sh + bD * CF::TILE;
    float2* b1 = sh + bZ * CF::TILE;
    stage(sh + bF * CF::TILE, S0, next);  // in flight: D(tile), Z(tile), D(next)
    const int kyr = tile / ntx;
    const int kx = (tile - kyr * ntx) * kCW + c;
    float2 v[R1];
    cp_async_wait<2>();
    __syncthreads();
    tile_to_regs<NZ, kCW>(b0, c, t, v);
    __syncthreads();
    ExCols<NZ, kCW> e0{b0, c};
    fft_line<NZ, false>(v, t, tw, e0);
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) b0[(t + T * k1) * kCW + c] = v[k1];  // park FFT_z(D)
    cp_async_wait<1>();
    __syncthreads();
    tile_to_regs<NZ, kCW>(b1, c, t, v);
    __syncthreads();
    ExCols<NZ, kCW> e1{b1, c};
    fft_line<NZ, false>(v, t, tw, e1);  // ends on a barrier after its last read of b1
    stage(b1, S1, next);                // Z(next) lands behind the filter and the inverse
    const int ky = ky0 + kyr;
    const float wx = (float)(kx <= nx / 2 ? kx : kx - nx) * fx_step;
    const float wy = (float)(ky <= ny / 2 ? ky : ky - ny) * fy_step;
    const float wxy = wx * wx + wy * wy;
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      const int kz = t + T * k1;
      const float wz = signed_freq<NZ>(kz);
      const float w2 = wxy + wz * wz;
      const float2 d = b0[kz * kCW + c];
      const float2 s = make_float2(d.x + wz * v[k1].x, d.y + wz * v[k1].y);
      const float inv = (kx == 0 && ky == 0 && kz == 0) ? 0.f : __fdividef(scale, w2);
      v[k1] = make_float2(s.y * inv, -s.x * inv);
    }
    __syncthreads();  // parked D read by all before b0 becomes the exchange
    relayout_for_inverse<NZ>(v);
    fft_line<NZ, true>(v, t, tw, e0);
    if (kx <= nx / 2) {
      const size_t base = (size_t)kyr * H + kx;
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) st_out(S0 + base + (size_t)(t + T * k1) * zstride, v[k1]);
    }
    const int f = bF;
    bF = bD, bD = f;  // D(next) is in the old free buffer; b0 is free after the inverse's last barrier
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------ Z, TMA-fed, warp-private
// Persistent CTAs over column tiles (16 kx columns x one ky row x all NZ
// planes of D and Z).  Tiles arrive through the tensor-memory accelerator:
// the live planes (F-y's plane flags) form runs, each cut into boxes of
// 32/16/8/4/2/1 planes (one tensor map per box height, 4-D view {2H floats,
// ny, nz, component}, 128 B rows, 128B swizzle), issued against an mbarrier
// armed with the tile's byte count; dead planes are never read (their stage
// rows are zeroed once per CTA).  A column belongs to T adjacent lanes of one
// warp (lane = t + T*column), so the three transposes of the column's
// z-transforms go through a warp-private padded buffer with __syncwarp only —
// no CTA barrier inside the tile.  Each warp copies its columns of the stage
// to registers (the swizzle makes that conflict-free), then counts itself out;
// the last warp out arms the barrier and issues the next tile's boxes, which
// land while the transforms, the filter and the stores of this tile run.  The
// kx = nx/2 column of 16 ky rows (packed tiles, not a box) takes predicated
// register loads.
constexpr int kZBoxes = 6;  // box heights 1, 2, 4, 8, 16, 32 planes
struct ZMaps {
  CUtensorMap m[kZBoxes];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n ZW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra ZW_%=;\n}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

template <int NZ>
struct Z4Cfg {
  static constexpr int CW = 16;                   // columns per tile: 128 B stage rows
  static constexpr int T = Shape<NZ>::R2;         // lanes per column
  static constexpr int CPW = 32 / T;              // columns per warp
  static constexpr int WARPS = CW / CPW;
  static constexpr int THREADS = 32 * WARPS;
  // float2 per column exchange: padded rows, and odd columns shifted by 64 B so
  // the two columns a half-warp touches sit in disjoint banks
  static constexpr int XCOL = Shape<NZ>::R1 * (T + 1) + 8;
  static constexpr int STAGE_B = 2 * NZ * CW * 8;       // D rows then Z rows
  static constexpr int EX_B = CW * XCOL * 8;
  static constexpr int SMEM = 1024 + STAGE_B + EX_B + NZ * 2 + 64;  // + alignment slack, segments, barrier
  static constexpr int MINB = THREADS >= 256 ? 2 : 4;
};

template <int NZ>
__global__ void __launch_bounds__(Z4Cfg<NZ>::THREADS, Z4Cfg<NZ>::MINB)
    z4_kernel(const __grid_constant__ ZMaps maps, float2* __restrict__ S0, const float2* __restrict__ S1, int nx,
              int ny, int H, int ntx, int nnyq, float fx_step, float fy_step, float scale,
              const float2* __restrict__ tw, const uint32_t* __restrict__ planeflag) {
  using S = Shape<NZ>;
  using CF = Z4Cfg<NZ>;
  constexpr int T = S::R2, R1 = S::R1, kCW = CF::CW, TH = CF::THREADS;
  constexpr int PW = (NZ + 31) / 32;
  static_assert(R1 <= 32, "row mask");
  extern __shared__ uint8_t zraw[];
  // 1024 B aligned stage: the 128B swizzle is a function of the address bits
  // 7-9, so row z's 16-byte chunk k sits at chunk k ^ (z & 7)
  float2* stage = reinterpret_cast<float2*>(zraw + ((1024 - (smem_u32(zraw) & 1023)) & 1023));
  float2* exbuf = stage + CF::STAGE_B / 8;
  uint16_t* segs = reinterpret_cast<uint16_t*>(exbuf + CF::EX_B / 8);  // z | log2(h) << 11
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(segs) + ((NZ * 2 + 15) & ~15));
  int* outcnt = reinterpret_cast<int*>(bar + 1);
  __shared__ uint32_t pmask[PW];
  __shared__ int nseg_s, nlive_s;
  for (int z = threadIdx.x; z < PW * 32; z += TH) {  // plane bitmask; warp-uniform trips
    const bool f = z < NZ && (!planeflag || __ldg(planeflag + z) != 0u);
    const uint32_t b = __ballot_sync(0xffffffffu, f);
    if ((z & 31) == 0) pmask[z >> 5] = b;
  }
  __syncthreads();
  auto plane_live = [&](int z) { return ((pmask[z >> 5] >> (z & 31)) & 1u) != 0u; };
  if (threadIdx.x == 0) {  // live-plane runs -> boxes of 2^k <= 32 planes
    int n = 0, live = 0;
    for (int z = 0; z < NZ;) {
      if (!plane_live(z)) {
        ++z;
        continue;
      }
      int e = z;
      while (e < NZ && plane_live(e)) ++e;
      live += e - z;
      while (z < e) {
        int lg = 5;
        while ((1 << lg) > e - z) --lg;
        segs[n++] = (uint16_t)(z | (lg << 11));
        z += 1 << lg;
      }
    }
    nseg_s = n, nlive_s = live;
    *outcnt = 0;
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < CF::STAGE_B / 8; i += TH)  // dead planes are never loaded: zero rows
    if (!plane_live((i / kCW) % NZ)) stage[i] = make_float2(0.f, 0.f);
  __syncthreads();
  const int nseg = nseg_s;
  const uint32_t tx_bytes = (uint32_t)nlive_s * 2u * kCW * 8u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // lane within the column team / column within the warp.  T = 16: lanes 0-7
  // and 16-23 are column 0, 8-15 and 24-31 column 1, so each half-warp reads
  // 8 rows x 2 columns of the stage = 8 distinct swizzled chunks (no conflict)
  const int t = T == 16 ? ((lane & 7) | ((lane >> 4) << 3)) : lane % T;
  const int cl = T == 16 ? ((lane >> 3) & 1) : lane / T;
  const int c = warp * CF::CPW + cl;      // column within the tile
  uint32_t rm = 0;  // bit (q*T + j2): this thread's element z = t + T*q + R1*j2 is in a live plane
#pragma unroll
  for (int q = 0; q < S::Q; ++q)
#pragma unroll
    for (int j2 = 0; j2 < T; ++j2) rm |= (plane_live(t + T * q + R1 * j2) ? 1u : 0u) << (q * T + j2);
  const int main_tiles = ntx * ny;
  const size_t zstride = (size_t)ny * H;
  auto issue = [&](int tile) {  // one thread: arm the barrier, then the boxes of both components
    const int kyr = tile / ntx, kx0 = (tile - kyr * ntx) * kCW;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the stage before async writes
    mbar_expect_tx(bar, tx_bytes);
    for (int s2 = 0; s2 < 2 * nseg; ++s2) {
      const int comp = s2 >= nseg ? 1 : 0;
      const uint32_t e = segs[s2 - comp * nseg];
      const int z = e & 2047, lg = e >> 11;
      tma_load_4d(stage + (comp * NZ + z) * kCW, &maps.m[lg], 2 * kx0, kyr, z, comp, bar);
    }
  };
  ExTeam<NZ> ex{exbuf + c * CF::XCOL, 0xffffffffu};
  uint32_t phase = 0;
  if (threadIdx.x == 0 && blockIdx.x < main_tiles && tx_bytes) issue(blockIdx.x);
  for (int tile = blockIdx.x; tile < main_tiles + nnyq; tile += gridDim.x) {
    int kx, kyr;
    bool live;
    float2 d[R1], v[R1];
    if (tile < main_tiles) {
      kyr = tile / ntx;
      kx = (tile - kyr * ntx) * kCW + c;
      live = kx <= nx / 2;
      if (tx_bytes) mbar_wait(bar, phase);
      phase ^= 1u;
#pragma unroll
      for (int q = 0; q < S::Q; ++q)
#pragma unroll
        for (int j2 = 0; j2 < T; ++j2) {
          const int z = t + T * q + R1 * j2;
          const int col = ((((c >> 1) ^ z) & 7) << 1) | (c & 1);  // swizzled position of column c in row z
          d[q * T + j2] = stage[z * kCW + col];
          v[q * T + j2] = stage[(NZ + z) * kCW + col];
        }
      __syncwarp();
      if (lane == 0) {  // count out; the last warp re-arms the stage with the next tile
        __threadfence_block();
        const int nt = tile + gridDim.x;
        if (atomicAdd(outcnt, 1) == CF::WARPS - 1) {
          *outcnt = 0;
          if (nt < main_tiles && tx_bytes) issue(nt);
        }
      }
    } else {  // the kx = nx/2 column of 16 ky rows
      kyr = (tile - main_tiles) * kCW + c;
      kx = nx / 2;
      live = kyr < ny;
      const size_t base = live ? (size_t)kyr * H + kx : 0;
      const uint32_t lm = live ? rm : 0u;
#pragma unroll
      for (int q = 0; q < S::Q; ++q)
#pragma unroll
        for (int j2 = 0; j2 < T; ++j2) {
          const int i = q * T + j2;
          const size_t o = base + (size_t)(t + T * q + R1 * j2) * zstride;
          d[i] = ld_pred_f2(S0 + o, (lm >> i) & 1u);
          v[i] = ld_pred_f2(S1 + o, (lm >> i) & 1u);
        }
    }
    fft_line<NZ, false>(d, t, tw, ex);
    fft_line<NZ, false>(v, t, tw, ex);
    // integrate.cpp:37-40 frequencies, filter -j(D + wz Z)/|w|^2, DC = 0 (:46-60)
    const float wx = (float)(kx <= nx / 2 ? kx : kx - nx) * fx_step;
    const float wy = (float)(kyr <= ny / 2 ? kyr : kyr - ny) * fy_step;
    const float wxy = wx * wx + wy * wy;
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      const int kz = t + T * k1;
      const float wz = signed_freq<NZ>(kz);
      const float w2 = wxy + wz * wz;
      const float2 s2 = make_float2(d[k1].x + wz * v[k1].x, d[k1].y + wz * v[k1].y);
      const float inv = (kx == 0 && kyr == 0 && kz == 0) ? 0.f : __fdividef(scale, w2);  // 1/N of the c2r folded in
      d[k1] = make_float2(s2.y * inv, -s2.x * inv);  // (-i/|w|^2) * s
    }
    relayout_for_inverse<NZ>(d);
    fft_line<NZ, true>(d, t, tw, ex);
    if (live) {
      const size_t base = (size_t)kyr * H + kx;
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) st_out(S0 + base + (size_t)(t + T * k1) * zstride, d[k1]);
    }
  }
}

// ------------------------------------------------------------------ I-y
template <int NY, bool NYQ>
__device__ __forceinline__ void iy_body(const float2* Rin, float2* Rout, int nxh, int H, int lk,
                                        const float2* __restrict__ tw) {
  using S = Shape<NY>;
  constexpr int T = S::R2, R1 = S::R1, kCW = ICfg<NY>::CW, TH = ICfg<NY>::THREADS;
  extern __shared__ float2 sh[];
  const int c = threadIdx.x % kCW, t = threadIdx.x / kCW;
  const int nzl = gridDim.y;
  const size_t kyl = (size_t)1 << lk;
  const RowMap rm{(size_t)H, nzl * kyl * H, lk};
  const int zl = NYQ ? blockIdx.y * kCW + c : blockIdx.y;
  const int kx = NYQ ? nxh - 1 : blockIdx.x * kCW + c;
  if (NYQ) {  // the kx = nx/2 column of planes blockIdx.y*kCW + c
    const int z0 = blockIdx.y * kCW;
    if (z0 >= nzl) return;
    stage_nyq<NY, kCW, TH>(sh, Rin + z0 * kyl * H + (nxh - 1), rm, kyl * H, min(kCW, nzl - z0), nullptr, 0);
  } else {
    stage_tile<NY, kCW, TH>(sh, Rin + zl * kyl * H, rm, blockIdx.x * kCW, H, 0xffffffffu);
  }
  cp_async_commit();
  float2 v[R1];
  cp_async_wait<0>();
  __syncthreads();
  tile_to_regs<NY, kCW>(sh, c, t, v);
  __syncthreads();
  ExCols<NY, kCW> ex{sh, c};
  fft_line<NY, true>(v, t, tw, ex);
  const bool live = NYQ ? zl < nzl : kx < nxh;
  if (live) {
    const size_t plane = (size_t)zl * NY * H;
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) st_out(Rout + plane + (size_t)(t + T * k1) * H + kx, v[k1]);
  }
}

// Input rows in the layout fy_kernel writes (the receive layout of the
// backward all-to-all on several GPUs); output in the plain [zl][ky][H]
// layout (in place on one GPU: Rin == Rout, lk = log2 ny).
template <int NY>
__global__ void __launch_bounds__(ICfg<NY>::THREADS, NY >= 1024 ? 2 : 3)
    iy_kernel(const float2* Rin, float2* Rout, int nxh, int H, int lk, int nyq, const float2* __restrict__ tw) {
  if (blockIdx.x == nyq)
    iy_body<NY, true>(Rin, Rout, nxh, H, lk, tw);
  else
    iy_body<NY, false>(Rin, Rout, nxh, H, lk, tw);
}

// I-y on one GPU (plain [z][ky][H] layout): the column tile arrives through
// the tensor-memory accelerator — one elected thread issues the 2-D boxes
// ({CW complex, 256 rows} on a {2H floats, nz*ny rows} view of the spectrum)
// against an mbarrier, instead of every thread computing cp.async addresses.
// The packed Nyquist tiles keep the gather (iy_body<NY, true>).
template <int NY>
__global__ void __launch_bounds__(ICfg<NY>::THREADS, NY >= 1024 ? 2 : 3)
    iy_tma_kernel(const __grid_constant__ CUtensorMap map, const float2* Rin, float2* Rout, int nxh, int H, int lk,
                  int nyq, const float2* __restrict__ tw) {
  if (blockIdx.x == nyq) {
    iy_body<NY, true>(Rin, Rout, nxh, H, lk, tw);
    return;
  }
  using S = Shape<NY>;
  constexpr int T = S::R2, R1 = S::R1, kCW = ICfg<NY>::CW;
  constexpr int BOXR = NY < 256 ? NY : 256;  // rows per box (box dims <= 256)
  extern __shared__ float2 sh[];             // the tile (dynamic base: 1 KB aligned), then the mbarrier
  uint64_t* bar = reinterpret_cast<uint64_t*>(sh + NY * kCW);
  const int c = threadIdx.x % kCW, t = threadIdx.x / kCW;
  const int zl = blockIdx.y, kx0 = blockIdx.x * kCW, kx = kx0 + c;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(bar, (uint32_t)(NY * kCW * 8));
#pragma unroll
    for (int b = 0; b < NY / BOXR; ++b) tma_load_2d(sh + b * BOXR * kCW, &map, 2 * kx0, zl * NY + b * BOXR, bar);
  }
  __syncthreads();  // the barrier is initialised before anyone waits on it
  mbar_wait(bar, 0);
  float2 v[R1];
  tile_to_regs<NY, kCW>(sh, c, t, v);
  __syncthreads();
  ExCols<NY, kCW> ex{sh, c};
  fft_line<NY, true>(v, t, tw, ex);
  if (kx < nxh) {
    const size_t plane = (size_t)zl * NY * H;
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) st_out(Rout + plane + (size_t)(t + T * k1) * H + kx, v[k1]);
  }
}

// ------------------------------------------------------------------ I-x
// Persistent teams: each team (T adjacent lanes) walks line pairs with a
// double-buffered cp.async stage of the next pair's half spectra, so the
// loads of pair i+1 overlap the C2R of pair i with no CTA-wide barrier.
template <int NX>
struct IXCfg {
  static constexpr int T = Shape<NX>::R2;
  static constexpr int LINE = ((NX / 2 + 4) + 7) & ~7;  // >= pitch, 64 B aligned slots
  static constexpr int BUF0 = 2 * LINE;
  static constexpr int TILE = Shape<NX>::R1 * (T + 1);
  static constexpr int BUF = BUF0 > TILE ? BUF0 : TILE;  // staged pair, then the exchange
  static constexpr int T0 = 256 / T;
  static constexpr int TEAMS = (T0 * 2 * BUF * 8 <= 96 * 1024) ? T0 : (T0 / 2 * 2 * BUF * 8 <= 96 * 1024 ? T0 / 2 : T0 / 4);
  static constexpr int THREADS = T * TEAMS;
  static constexpr int SMEM = TEAMS * 2 * BUF * 8;
};

template <int NX>
__global__ void __launch_bounds__(IXCfg<NX>::THREADS, 2) ix_kernel(const float2* __restrict__ S0, float* __restrict__ A,
                                                       int rows, int H,
                                                       const float2* __restrict__ tw, float2* __restrict__ rowmm,
                                                       uint32_t* __restrict__ rowbits_reset) {
  using S = Shape<NX>;
  using CF = IXCfg<NX>;
  constexpr int T = S::R2, R1 = S::R1, NH = NX / 2;
  extern __shared__ float2 dyn_smem[];
  const int team = threadIdx.x / T, t = threadIdx.x % T;
  const unsigned mask = team_mask<T>((threadIdx.x & 31) - t);
  float2* const bufs = dyn_smem + (size_t)team * 2 * CF::BUF;
  const int pairs = rows / 2;
  const int stride = gridDim.x * CF::TEAMS;
  const int chunks = (H * 8) / 16;  // 16 B per cp.async; H is a multiple of 4
  auto stage = [&](int pr, float2* b) {
    const float2* src = S0 + (size_t)(2 * pr) * H;
#pragma unroll
    for (int l = 0; l < 2; ++l)
      for (int c = t; c < chunks; c += T) cp_async16(b + l * CF::LINE + 2 * c, src + (size_t)l * H + 2 * c, true);
  };
  int pr = blockIdx.x * CF::TEAMS + team;
  if (pr < pairs) stage(pr, bufs);
  cp_async_commit();
  for (int it = 0; pr < pairs; ++it, pr += stride) {
    float2* cur = bufs + (it & 1) * CF::BUF;
    const int nx_pr = pr + stride;
    if (nx_pr < pairs) stage(nx_pr, bufs + ((it + 1) & 1) * CF::BUF);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp(mask);
    const float2* h0 = cur;
    const float2* h1 = cur + CF::LINE;
    // Hermitian extension with Re() of bins 0 and n/2 (numpy irfft / FFTW c2r)
    auto full = [&](const float2* h, int j) {
      if (j == 0) return make_float2(h[0].x, 0.f);
      if (j == NH) return make_float2(h[NH].x, 0.f);
      if (j < NH) return h[j];
      const float2 c = h[NX - j];
      return make_float2(c.x, -c.y);
    };
    float2 v[R1];
#pragma unroll
    for (int q = 0; q < S::Q; ++q)
#pragma unroll
      for (int j2 = 0; j2 < T; ++j2) {
        const int j = t + T * q + R1 * j2;
        const float2 f0 = full(h0, j), f1 = full(h1, j);
        v[q * T + j2] = make_float2(f0.x - f1.y, f0.y + f1.x);  // F0 + i F1
      }
    __syncwarp(mask);
    ExTeam<NX> ex{cur, mask};
    fft_line<NX, true>(v, t, tw, ex);
    const int l0 = 2 * pr, l1 = l0 + 1;
    float lo0 = 3.4e38f, hi0 = -3.4e38f, lo1 = 3.4e38f, hi1 = -3.4e38f;
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      const int k = t + T * k1;
      const float a0 = v[k1].x, a1 = v[k1].y;  // 1/N applied by the Z pass's filter
      lo0 = fminf(lo0, a0), hi0 = fmaxf(hi0, a0), lo1 = fminf(lo1, a1), hi1 = fmaxf(hi1, a1);
      st_out(A + (size_t)l0 * NX + k, a0);
      st_out(A + (size_t)l1 * NX + k, a1);
    }
    // per-row min/max for marching-cubes row culling
#pragma unroll
    for (int o = T / 2; o > 0; o >>= 1) {
      lo0 = fminf(lo0, __shfl_xor_sync(mask, lo0, o)), hi0 = fmaxf(hi0, __shfl_xor_sync(mask, hi0, o));
      lo1 = fminf(lo1, __shfl_xor_sync(mask, lo1, o)), hi1 = fmaxf(hi1, __shfl_xor_sync(mask, hi1, o));
    }
    if (rowmm && t == 0) {
      rowmm[l0] = make_float2(lo0, hi0);
      rowmm[l1] = make_float2(lo1, hi1);
    }
    // the touched-chunk bits were last read by F-y: reset for the next frame
    // (F-x zeroed the chunks themselves)
    if (rowbits_reset && t == 0) rowbits_reset[l0] = 0u, rowbits_reset[l1] = 0u;
    __syncwarp(mask);  // `cur` is re-staged two iterations later
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------ dispatch
template <template <int> class F, typename... Args>
void dispatch_n(int n, Args&&... args) {
  switch (n) {
    case 4: F<4>::run(args...); break;
    case 8: F<8>::run(args...); break;
    case 16: F<16>::run(args...); break;
    case 32: F<32>::run(args...); break;
    case 64: F<64>::run(args...); break;
    case 128: F<128>::run(args...); break;
    case 256: F<256>::run(args...); break;
    case 512: F<512>::run(args...); break;
    case 1024: F<1024>::run(args...); break;
    default: break;  // validated on the host
  }
}

inline int hpitch(int nx) { return ((nx / 2 + 1) + 3) & ~3; }


// Opt-in dynamic shared memory above 48 KB.  Called from prepare_integrate
// (whenever the grid dims change), never inside a graph capture.
template <class K>
void allow_smem(K* kernel, int bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
template <int N>
struct Prep {
  static void run(int axis) {
    if (axis == 0) {
      allow_smem(fx_kernel<N>, XCfg<N>::SMEM);
      allow_smem(ix_kernel<N>, IXCfg<N>::SMEM);
    } else if (axis == 1) {
      allow_smem(fy_kernel<N>, FCfg<N>::NBUF * FCfg<N>::SMEM);
      if constexpr (N == 1024) allow_smem(fyp_kernel<N>, 3 * FCfg<N>::SMEM);
      allow_smem(iy_kernel<N>, ICfg<N>::SMEM);
      allow_smem(iy_tma_kernel<N>, ICfg<N>::SMEM + 64);
    } else {
      allow_smem(z_kernel<N>, 2 * ZCfg<N>::SMEM);
      if constexpr (N == 64 || N == 128 || N == 256) allow_smem(z4_kernel<N>, Z4Cfg<N>::SMEM);
      if constexpr (N == 1024) allow_smem(zp_kernel<N>, ZPCfg<N>::SMEM);
    }
  }
};

template <int N>
struct RunFx {
  static void run(const SlabFft& a) {
    using C = XCfg<N>;
    const int rows = a.ny * a.nzl;
    const int need = (rows / 2 + C::TEAMS - 1) / C::TEAMS;
    const int grid = a.rowlist && need > sm_count() * 2 ? sm_count() * 2 : need;  // persistent teams over the row list
    fx_kernel<N><<<grid, C::THREADS, C::SMEM, a.st>>>(a.acc, a.S0, a.S1, a.S2, rows, a.H, a.rowbits, a.mode, a.twx,
                                                      a.rowlist);
  }
};
// Column tiles of CW kx columns.  When nx/2 is a multiple of CW the single
// kx = nx/2 (Nyquist) column would fill a whole tile alone: the last grid
// column instead packs it from CW planes / ky rows (tile index `nyq`).
inline int nyq_mode() {  // VC_NYQ_PACK: bit 1 z, bit 2 iy (A/B switch; default both)
  static const int m = [] {
    const char* e = std::getenv("VC_NYQ_PACK");
    return e ? std::atoi(e) : 6;
  }();
  return m;
}
inline void col_grid(int nx, int cw, int* tiles, int* nyq, int bit) {
  if ((nx / 2) % cw == 0 && (nyq_mode() >> bit & 1)) {
    *tiles = nx / 2 / cw + 1, *nyq = nx / 2 / cw;
  } else {
    *tiles = (nx / 2 + 1 + cw - 1) / cw, *nyq = -1;
  }
}
// VC_FYP=0 (A/B switch): the staged fy_kernel at 1024 points instead of fyp_kernel
inline bool fyp_on() {
  static const bool on = [] {
    const char* e = std::getenv("VC_FYP");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}
template <int N>
struct RunFy {
  static void run(const SlabFft& a) {
    using C = FCfg<N>;
    // (no Nyquist packing here: F-y's per-row empty flags make the packed
    // gather slower than the one wasted tile, measured)
    const int ntx = (a.nx / 2 + 1 + C::CW - 1) / C::CW;
    if constexpr (N == 1024) {
      if (fyp_on() && a.zoff == 0 && a.nzl == a.nz) {  // one GPU: the live-plane list sits after the nz flags
        int32_t* plist = reinterpret_cast<int32_t*>(a.planeflag + a.nz);
        cudaMemsetAsync(plist, 0, sizeof(int32_t), a.st);
        fy_planes_kernel<<<(a.nzl * 32 + 255) / 256, 256, 0, a.st>>>(a.rowbits, a.ny, a.nzl, a.planeflag, plist);
        fyp_kernel<N><<<sm_count(), C::THREADS, 3 * C::SMEM, a.st>>>(a.S0, a.S1, a.S2, a.O0, a.O1, a.nx / 2 + 1, a.H,
                                                                     ilog2(a.kyl), a.twy, a.rowbits, plist, ntx, a.nzl);
        return;
      }
    }
    dim3 grid(ntx, a.nzl);
    fy_kernel<N><<<grid, C::THREADS, C::NBUF * C::SMEM, a.st>>>(a.S0, a.S1, a.S2, a.O0, a.O1, a.nx / 2 + 1, a.H,
                                                          ilog2(a.kyl), a.twy, a.rowbits, a.planeflag + a.zoff);
  }
};
// VC_ZP=0 (A/B switch): the staged z_kernel at 1024 planes instead of zp_kernel
inline bool zp_on() {
  static const bool on = [] {
    const char* e = std::getenv("VC_ZP");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}
template <int N>
struct RunZ {
  static void run(const SlabFft& a) {
    using C = ZCfg<N>;
    int tiles, nyq;
    col_grid(a.nx, C::CW, &tiles, &nyq, 1);
    if constexpr (N == 1024) {
      static_assert(ZPCfg<N>::CW == C::CW, "one tiling");
      if (zp_on()) {
        const float fxs = (float)(2.0 * M_PI / a.nx), fys = (float)(2.0 * M_PI / a.ny);
        const float scale = (float)(1.0 / ((double)a.nx * a.ny * a.nz));
        const int ntx = nyq >= 0 ? nyq : tiles;
        zp_kernel<N><<<sm_count(), ZPCfg<N>::THREADS, ZPCfg<N>::SMEM, a.st>>>(
            a.R0, a.R1, a.nx, a.ny, a.kyl, a.ky0, a.H, ntx, fxs, fys, scale, a.twz, a.planeflag);
        if (nyq >= 0)  // the packed kx = nx/2 tiles: z_kernel's Nyquist body (grid column 0 = nyq)
          z_kernel<N><<<dim3(1, (a.kyl + C::CW - 1) / C::CW), C::THREADS, 2 * C::SMEM, a.st>>>(
              a.R0, a.R1, a.nx, a.ny, a.kyl, a.ky0, a.H, 0, fxs, fys, scale, a.twz, a.planeflag);
        return;
      }
    }
    dim3 grid(tiles, a.kyl);
    const float fxs = (float)(2.0 * M_PI / a.nx), fys = (float)(2.0 * M_PI / a.ny);
    const float scale = (float)(1.0 / ((double)a.nx * a.ny * a.nz));  // the c2r's 1/N (integrate.cpp:70-72)
    z_kernel<N><<<grid, C::THREADS, 2 * C::SMEM, a.st>>>(a.R0, a.R1, a.nx, a.ny, a.kyl, a.ky0, a.H, nyq, fxs, fys,
                                                         scale, a.twz, a.planeflag);
  }
};
// VC_ZK=4 selects the TMA-fed warp-private Z kernel (opt-in: at 256^3 it
// measured 77.6 us against 48.5 us for the staged kernel, profiles/README.md);
// default 1, the staged kernel.
inline int z_mode() {
  static const int m = [] {
    const char* e = std::getenv("VC_ZK");
    return e ? std::atoi(e) : 1;
  }();
  return m;
}
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}
// 4-D view {2H floats, ny, nz, component} of the D/Z spectra (component stride
// cs complex), one map per box height 2^k planes, 16 complex (128 B) wide.
bool encode_zmaps(ZMaps* zm, const float2* S0, int H, int ny, int nz, size_t cs) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const cuuint64_t dims[4] = {(cuuint64_t)2 * H, (cuuint64_t)ny, (cuuint64_t)nz, 2};
  const cuuint64_t strides[3] = {(cuuint64_t)H * 8, (cuuint64_t)H * 8 * ny, (cuuint64_t)cs * 8};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  for (int k = 0; k < kZBoxes; ++k) {
    const cuuint32_t box[4] = {32, 1, (cuuint32_t)(1 << k), 1};
    if (enc(&zm->m[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float2*>(S0), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}
// 2-D view {2H floats, rows} of a spectrum component, boxes {2*cw floats, boxr rows}
bool encode_iy_map(CUtensorMap* m, const float2* base, int H, size_t rows, int cw, int boxr) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)2 * H, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)H * 8};
  const cuuint32_t box[2] = {(cuuint32_t)(2 * cw), (cuuint32_t)boxr};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float2*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <int N>
struct RunZ4 {
  static void run(const SlabFft& a, const ZMaps& zm) {
    using C = Z4Cfg<N>;
    int ntx, nnyq;
    if ((a.nx / 2) % C::CW == 0) {
      ntx = a.nx / 2 / C::CW, nnyq = (a.ny + C::CW - 1) / C::CW;
    } else {
      ntx = (a.nx / 2 + 1 + C::CW - 1) / C::CW, nnyq = 0;
    }
    const int tiles = ntx * a.ny + nnyq;
    const int cap = sm_count() * C::MINB;
    const float fxs = (float)(2.0 * M_PI / a.nx), fys = (float)(2.0 * M_PI / a.ny);
    z4_kernel<N><<<tiles < cap ? tiles : cap, C::THREADS, C::SMEM, a.st>>>(
        zm, a.S0, a.S1, a.nx, a.ny, a.H, ntx, nnyq, fxs, fys, (float)(1.0 / ((double)a.nx * a.ny * a.nz)), a.twz,
        a.planeflag);
  }
};
bool encode_iy_map(CUtensorMap* m, const float2* base, int H, size_t rows, int cw, int boxr);
inline bool iy_tma_on() {  // VC_IY_TMA=0: cp.async staging (A/B switch)
  static const bool on = [] {
    const char* e = std::getenv("VC_IY_TMA");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}
template <int N>
struct RunIy {
  static void run(const SlabFft& a) {
    using C = ICfg<N>;
    int tiles, nyq;
    col_grid(a.nx, C::CW, &tiles, &nyq, 2);
    dim3 grid(tiles, a.nzl);
    CUtensorMap map;
    // one GPU, plain layout (rows (z, ky) at stride H): the tile as tensor-map boxes
    if (iy_tma_on() && a.kyl == a.ny && a.Rin == a.Rout && N >= 8 &&
        encode_iy_map(&map, a.Rin, a.H, (size_t)a.nzl * a.ny, C::CW, N < 256 ? N : 256)) {
      iy_tma_kernel<N><<<grid, C::THREADS, C::SMEM + 64, a.st>>>(map, a.Rin, a.Rout, a.nx / 2 + 1, a.H,
                                                                ilog2(a.kyl), nyq, a.twy);
      return;
    }
    iy_kernel<N><<<grid, C::THREADS, C::SMEM, a.st>>>(a.Rin, a.Rout, a.nx / 2 + 1, a.H, ilog2(a.kyl), nyq, a.twy);
  }
};
template <int N>
struct RunIx {
  static void run(const SlabFft& a) {
    using C = IXCfg<N>;
    const int rows = a.ny * a.nzl;
    const int need = (rows / 2 + C::TEAMS - 1) / C::TEAMS;
    const int grid = need < sm_count() * 4 ? need : sm_count() * 4;  // persistent teams
    ix_kernel<N><<<grid, C::THREADS, C::SMEM, a.st>>>(a.Rout, a.A, rows, a.H, a.twx, a.rowmm,
                                                      a.rowlist ? const_cast<uint32_t*>(a.rowbits) : nullptr);
  }
};

}  // namespace

void prepare_integrate(int nx, int ny, int nz) {
  dispatch_n<Prep>(nx, 0);
  dispatch_n<Prep>(ny, 1);
  dispatch_n<Prep>(nz, 2);
}

size_t spectrum_elems(int nx, int ny, int nz) { return (size_t)hpitch(nx) * ny * nz; }
size_t twiddle_elems(int nx, int ny, int nz) { return (size_t)nx + ny + nz; }

void upload_twiddles(float2* dev, int nx, int ny, int nz, cudaStream_t st) {
  // __constant__ data is per device: upload with every table (cheap, on the caller's device)
  float2 w[32];
  for (int k = 0; k < 32; ++k)
    w[k] = make_float2((float)std::cos(-2.0 * M_PI * k / 32.0), (float)std::sin(-2.0 * M_PI * k / 32.0));
  cudaMemcpyToSymbolAsync(c_w32, w, sizeof(w), 0, cudaMemcpyHostToDevice, st);
  std::vector<float2> h;
  for (int n : {nx, ny, nz})
    for (int m = 0; m < n; ++m)
      h.push_back(make_float2((float)std::cos(-2.0 * M_PI * m / n), (float)std::sin(-2.0 * M_PI * m / n)));
  cudaMemcpyAsync(dev, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);
}

void launch_fft_forward_xy(const SlabFft& a) {
  dispatch_n<RunFx>(a.nx, a);
  dispatch_n<RunFy>(a.ny, a);
}
void launch_fft_z(const SlabFft& a) {
  // the TMA-fed kernel: one GPU (D and Z one component stride apart, all ky rows), 64..256 planes,
  // rows of 16 complex (nx >= 32: the main tiles hold at least one full box width)
  if (z_mode() == 4 && (a.nz == 256 || a.nz == 128 || a.nz == 64) && a.nx >= 32 && a.kyl == a.ny && a.R0 == a.S0 &&
      a.R1 == a.S1) {
    ZMaps zm;
    if (encode_zmaps(&zm, a.S0, a.H, a.ny, a.nz, (size_t)(a.S1 - a.S0))) {
      if (a.nz == 256)
        RunZ4<256>::run(a, zm);
      else if (a.nz == 128)
        RunZ4<128>::run(a, zm);
      else
        RunZ4<64>::run(a, zm);
      return;
    }
  }
  dispatch_n<RunZ>(a.nz, a);
}
void launch_fft_inverse_yx(const SlabFft& a) {
  dispatch_n<RunIy>(a.ny, a);
  dispatch_n<RunIx>(a.nx, a);
}

// Dense pseudo-random accumulator (U' in [-1, 1), d' = 1) for timing the
// chain without the splat's sparsity.
__global__ void fill_random_acc_kernel(float4* acc, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    float v[3];
    for (int c = 0; c < 3; ++c) {
      h ^= h >> 16, h *= 0x7feb352du, h ^= h >> 15, h *= 0x846ca68bu, h ^= h >> 16;
      v[c] = (float)(h >> 8) * (2.0f / 16777216.0f) - 1.0f;
    }
    acc[i] = make_float4(v[0], v[1], v[2], 1.0f);
  }
}

void launch_fill_random_acc(float4* acc, size_t n, uint32_t seed, cudaStream_t st) {
  fill_random_acc_kernel<<<sm_count() * 8, 256, 0, st>>>(acc, n, seed);
}

void launch_integrate(float4* acc, float2* spec, float* A, int nx, int ny, int nz, int mode,
                      const float2* tw, cudaStream_t st, cudaEvent_t* ev, float2* rowmm, const uint32_t* rowbits,
                      uint32_t* planeflag, const int32_t* rowlist) {
  SlabFft a;
  a.rowlist = rowlist;
  const size_t cs = spectrum_elems(nx, ny, nz);
  a.acc = acc, a.S0 = spec, a.S1 = spec + cs, a.S2 = spec + 2 * cs, a.A = A;
  a.O0 = a.S0, a.O1 = a.S1, a.R0 = a.S0, a.R1 = a.S1, a.Rin = a.S0, a.Rout = a.S0;
  a.nx = nx, a.ny = ny, a.nz = nz, a.nzl = nz, a.zoff = 0, a.kyl = ny, a.ky0 = 0, a.H = hpitch(nx), a.mode = mode;
  a.twx = tw, a.twy = tw + nx, a.twz = tw + nx + ny, a.st = st;
  a.rowmm = rowmm, a.rowbits = rowbits, a.planeflag = planeflag;
  if (ev) record_event(ev[0], st);
  dispatch_n<RunFx>(nx, a);
  if (ev) record_event(ev[1], st);
  dispatch_n<RunFy>(ny, a);
  if (ev) record_event(ev[2], st);
  launch_fft_z(a);
  if (ev) record_event(ev[3], st);
  dispatch_n<RunIy>(ny, a);
  if (ev) record_event(ev[4], st);
  dispatch_n<RunIx>(nx, a);
  if (ev) record_event(ev[5], st);
}

}  // namespace vc

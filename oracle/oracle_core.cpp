// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — NOT PRODUCT CODE.  See oracle.hpp for the contract.
//
// Restates /root/reference/proj/core/src/{core/camera.cpp, recon/cloud.cpp,
// recon/reconstruct.cpp, recon/splat.cpp, recon/integrate.cpp,
// recon/marching_cubes.cpp, appearance/texture.cpp, eval/rasterize.cpp}
// with the reference's floating-point evaluation order.
#include "oracle.hpp"

#include <algorithm>
#include <cmath>
#include <complex>
#include <stdexcept>
#include <thread>
#include <unordered_map>

namespace orc {

double norm(V3 a) { return std::sqrt(sqnorm(a)); }
V3 normalized(V3 a) {
  const double z = sqnorm(a);
  if (z > 0) return a / std::sqrt(z);
  return a;
}
M3 matmul(const M3& A, const M3& B) {
  M3 o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      o.m[r * 3 + c] = (A.m[r * 3 + 0] * B.m[0 * 3 + c] + A.m[r * 3 + 1] * B.m[1 * 3 + c]) +
                       A.m[r * 3 + 2] * B.m[2 * 3 + c];
  return o;
}
M3 rot(const Pose& p) {
  M3 o;
  for (int i = 0; i < 9; ++i) o.m[i] = p.R[i];
  return o;
}
V3 trans(const Pose& p) { return {p.t[0], p.t[1], p.t[2]}; }
V3 pose_apply(const Pose& p, V3 x) { return mul(rot(p), x) + trans(p); }
V3 pose_apply_inverse(const Pose& p, V3 x) { return mul(transpose(rot(p)), x - trans(p)); }
Pose pose_inverse(const Pose& p) {
  const M3 rt = transpose(rot(p));
  const V3 t = -mul(rt, trans(p));
  Pose o;
  for (int i = 0; i < 9; ++i) o.R[i] = rt.m[i];
  o.t[0] = t.x, o.t[1] = t.y, o.t[2] = t.z;
  return o;
}
Pose pose_compose(const Pose& a, const Pose& b) {
  const M3 r = matmul(rot(a), rot(b));
  const V3 t = mul(rot(a), trans(b)) + trans(a);
  Pose o;
  for (int i = 0; i < 9; ++i) o.R[i] = r.m[i];
  o.t[0] = t.x, o.t[1] = t.y, o.t[2] = t.z;
  return o;
}

// camera.cpp:6-10
bool project_local(const Intrinsics& K, V3 x, double* u, double* v) {
  if (x.z <= 0) return false;
  *u = K.fx * x.x / x.z + K.cx;
  *v = K.fy * x.y / x.z + K.cy;
  return true;
}
// camera.cpp:12-17
V3 backproject_local(const Intrinsics& K, double u, double v, double z_mm) {
  if (z_mm <= 0) throw std::invalid_argument("backproject: depth must be positive");
  return {(u - K.cx) * z_mm / K.fx, (v - K.cy) * z_mm / K.fy, z_mm};
}

int hardware_threads() {
  const unsigned n = std::thread::hardware_concurrency();
  return n == 0 ? 1 : static_cast<int>(n);
}

// threading.cpp:15-35 — contiguous chunks, one std::thread each.
template <typename Fn>
static void parallel_chunks(std::size_t count, int threads, Fn&& fn) {
  if (count == 0) return;
  const int n = std::max(1, std::min<int>(threads, static_cast<int>(count)));
  if (n == 1) {
    fn(std::size_t{0}, count);
    return;
  }
  const std::size_t chunk = (count + n - 1) / n;
  std::vector<std::thread> pool;
  for (int i = 0; i < n; ++i) {
    const std::size_t b = std::min(count, static_cast<std::size_t>(i) * chunk);
    const std::size_t e = std::min(count, b + chunk);
    if (b >= e) break;
    pool.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& t : pool) t.join();
}

// ------------------------------------------------------------ build_cloud
// cloud.cpp:19-83
Cloud build_cloud(const Frame& f, const Intrinsics& K, const Pose& pose, int sensor,
                  double discontinuity_mm) {
  const int w = f.w, h = f.h;
  struct PixelVertex {
    V3 local, normal_sum;
    int tri_count = 0;
  };
  std::vector<int> vindex(static_cast<std::size_t>(w) * h, -1);
  std::vector<PixelVertex> verts;
  std::vector<std::pair<int, int>> pixels;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const std::size_t i = static_cast<std::size_t>(y) * w + x;
      if (!f.mask[i]) continue;
      const uint16_t d = f.depth[i];
      if (d == 0) continue;
      vindex[i] = static_cast<int>(verts.size());
      verts.push_back({backproject_local(K, x, y, d), V3{}, 0});
      pixels.emplace_back(x, y);
    }

  auto add_triangle = [&](int ia, int ib, int ic) {
    const double za = verts[ia].local.z, zb = verts[ib].local.z, zc = verts[ic].local.z;
    const double lo = std::min({za, zb, zc}), hi = std::max({za, zb, zc});
    if (hi - lo > discontinuity_mm) return;
    V3 n = cross(verts[ic].local - verts[ia].local, verts[ib].local - verts[ia].local);
    const double len = norm(n);
    if (len < 1e-12) return;
    n = n / len;
    for (int i : {ia, ib, ic}) {
      verts[i].normal_sum = verts[i].normal_sum + n;
      ++verts[i].tri_count;
    }
  };
  auto at = [&](int x, int y) { return vindex[static_cast<std::size_t>(y) * w + x]; };
  for (int y = 0; y + 1 < h; ++y)
    for (int x = 0; x + 1 < w; ++x) {
      const int i00 = at(x, y), i10 = at(x + 1, y), i01 = at(x, y + 1), i11 = at(x + 1, y + 1);
      if (i00 >= 0 && i10 >= 0 && i01 >= 0) add_triangle(i00, i10, i01);
      if (i10 >= 0 && i11 >= 0 && i01 >= 0) add_triangle(i10, i11, i01);
    }

  Cloud c;
  c.sensor = sensor;
  c.w = w, c.h = h;
  c.weight_map.assign(static_cast<std::size_t>(w) * h, 0.f);
  c.points.reserve(verts.size());
  const M3 R = rot(pose);
  for (std::size_t i = 0; i < verts.size(); ++i) {
    if (verts[i].tri_count == 0) continue;
    V3 n = verts[i].normal_sum / static_cast<double>(verts[i].tri_count);
    const double len = norm(n);
    if (len < 1e-12) continue;
    n = n / len;
    if (dot(n, verts[i].local) > 0) n = -n;
    OrientedPoint p;
    p.position = pose_apply(pose, verts[i].local);
    p.normal = mul(R, n);
    p.weight = 1.0;
    p.px = pixels[i].first;
    p.py = pixels[i].second;
    p.sensor = sensor;
    c.points.push_back(p);
    c.weight_map[static_cast<std::size_t>(p.py) * w + p.px] = 1.f;
  }
  return c;
}

// cloud.cpp:85-117
void confidence_weights(Cloud& c, const Frame& f, const Intrinsics&, const Pose& pose,
                        int r) {
  const int w = f.w, h = f.h;
  std::vector<uint32_t> sat(static_cast<std::size_t>(w + 1) * (h + 1), 0);
  auto S = [&](int x, int y) -> uint32_t& { return sat[static_cast<std::size_t>(y) * (w + 1) + x]; };
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x)
      S(x + 1, y + 1) = S(x, y + 1) + S(x + 1, y) - S(x, y) +
                        (f.mask[static_cast<std::size_t>(y) * w + x] ? 1u : 0u);
  const double window = static_cast<double>(2 * r + 1) * (2 * r + 1);
  auto coverage = [&](int x, int y) {
    const int x0 = std::max(0, x - r), y0 = std::max(0, y - r);
    const int x1 = std::min(w - 1, x + r), y1 = std::min(h - 1, y + r);
    const uint32_t count = S(x1 + 1, y1 + 1) - S(x0, y1 + 1) - S(x1 + 1, y0) + S(x0, y0);
    return count / window;
  };
  const Pose inv = pose_inverse(pose);
  const M3 Ri = rot(inv);
  for (auto& p : c.points) {
    const V3 local = pose_apply(inv, p.position);
    const V3 n_local = mul(Ri, p.normal);
    const double w1 = std::max(dot(-normalized(local), n_local), 0.0);
    const double w2 = coverage(p.px, p.py);
    p.weight = w1 * w2;
    c.weight_map[static_cast<std::size_t>(p.py) * w + p.px] = static_cast<float>(p.weight);
  }
}

// ------------------------------------------------------------ fit_grid
// reconstruct.cpp:16-35 (dims generalised; the reference hard-codes
// (2^r, 2^(r+1), 2^r) at :18-20 — callers pass those dims for r-mode).
bool fit_grid(V3 lo, V3 hi, const int dims[3], int pad, GridSpec* g) {
  g->nx = dims[0], g->ny = dims[1], g->nz = dims[2];
  const V3 extent = hi - lo;
  double edge = 1e-9;
  for (int a = 0; a < 3; ++a) {
    const int usable = dims[a] - 1 - 2 * pad;
    if (usable < 1) return false;
    edge = std::max(edge, comp(extent, a) / usable);
  }
  g->edge = edge;
  const V3 center = 0.5 * (lo + hi);
  g->origin[0] = center.x - edge * (g->nx - 1) / 2.0;
  g->origin[1] = center.y - edge * (g->ny - 1) / 2.0;
  g->origin[2] = center.z - edge * (g->nz - 1) / 2.0;
  return true;
}

// ------------------------------------------------------------ splat
// splat.cpp:11-13
static inline double kernel(double dist, double sigma) {
  return std::exp(-dist * dist / (sigma * sigma)) / sigma;
}

static inline V3 to_voxel(const GridSpec& g, V3 p) {  // volume.hpp:44
  return (p - V3{g.origin[0], g.origin[1], g.origin[2]}) / g.edge;
}
static inline V3 voxel_center(const GridSpec& g, int x, int y, int z) {  // volume.hpp:42
  return V3{g.origin[0], g.origin[1], g.origin[2]} +
         g.edge * V3{static_cast<double>(x), static_cast<double>(y), static_cast<double>(z)};
}

// splat.cpp:33-89
Field splat(const std::vector<const OrientedPoint*>& pts, const GridSpec& g, int mode,
            int threads) {
  Field out;
  out.grid = g;
  out.sigma1 = std::sqrt(3.0) / 2.0 * g.edge;
  out.sigma2 = std::sqrt(1.5) * out.sigma1;
  const std::size_t N = static_cast<std::size_t>(g.nx) * g.ny * g.nz;
  out.field.assign(N, V3{});
  out.density.assign(N, 0.0);
  auto idx = [&](int x, int y, int z) {
    return static_cast<std::size_t>(x) + static_cast<std::size_t>(g.nx) * (y + static_cast<std::size_t>(g.ny) * z);
  };

  if (mode == kSimple) {  // splat.cpp:40-56
    for (const OrientedPoint* p : pts) {
      const V3 c = to_voxel(g, p->position);
      const int x = static_cast<int>(std::lround(c.x));
      const int y = static_cast<int>(std::lround(c.y));
      const int z = static_cast<int>(std::lround(c.z));
      if (!(x >= 0 && x < g.nx && y >= 0 && y < g.ny && z >= 0 && z < g.nz)) continue;
      out.field[idx(x, y, z)] = out.field[idx(x, y, z)] + p->normal;
      out.density[idx(x, y, z)] += 1.0;
    }
    for (std::size_t i = 0; i < N; ++i)
      if (out.density[i] > 0) out.field[i] = out.field[i] / out.density[i];
    return out;
  }

  const double eps_density = 1e-6 * kernel(0.0, out.sigma2);
  auto for_each_slab = [&](auto&& accumulate) {
    parallel_chunks(static_cast<std::size_t>(g.nz), threads, [&](std::size_t z0s, std::size_t z1s) {
      for (const OrientedPoint* p : pts) {
        const V3 c = to_voxel(g, p->position);
        int lo[3], hi[3];
        const int n[3] = {g.nx, g.ny, g.nz};
        for (int a = 0; a < 3; ++a) {  // support_around, splat.cpp:19-29
          const int f = static_cast<int>(std::floor(comp(c, a)));
          lo[a] = std::max(0, f - 1);
          hi[a] = std::min(n[a] - 1, f + 2);
        }
        const int z0 = std::max(lo[2], static_cast<int>(z0s));
        const int z1 = std::min(hi[2], static_cast<int>(z1s) - 1);
        for (int z = z0; z <= z1; ++z)
          for (int y = lo[1]; y <= hi[1]; ++y)
            for (int x = lo[0]; x <= hi[0]; ++x)
              accumulate(*p, norm(p->position - voxel_center(g, x, y, z)), idx(x, y, z));
      }
    });
  };
  for_each_slab([&](const OrientedPoint& p, double dist, std::size_t i) {
    out.density[i] += kernel(dist, out.sigma2) * p.weight;
  });
  for_each_slab([&](const OrientedPoint& p, double dist, std::size_t i) {
    const double d = out.density[i];
    if (d < eps_density) return;
    out.field[i] = out.field[i] + kernel(dist, out.sigma1) * (p.weight / d) * p.normal;
  });
  return out;
}

// ------------------------------------------------------------ FFT
// Replaces FFTW3 (integrate.cpp:31-34,44,63; FFTW_ESTIMATE r2c/c2r rank-3)
// with an fp64 transform having numpy rfftn/irfftn semantics: the c2r runs
// complex inverse transforms along z then y, then a Hermitian-extended
// inverse along x that uses only Re() of bins 0 and nx/2.
using cd = std::complex<double>;

namespace {
struct Plan1D {
  int n = 0;
  bool pow2 = false;
  std::vector<cd> tw;     // e^{-2 pi i k / n}
  std::vector<int> rev;   // bit reversal
};

Plan1D make_plan(int n) {
  Plan1D p;
  p.n = n;
  p.pow2 = n > 0 && (n & (n - 1)) == 0;
  p.tw.resize(n);
  for (int k = 0; k < n; ++k) {
    const double a = -2.0 * M_PI * static_cast<double>(k) / n;
    p.tw[k] = cd(std::cos(a), std::sin(a));
  }
  if (p.pow2) {
    p.rev.resize(n);
    int bits = 0;
    while ((1 << bits) < n) ++bits;
    for (int i = 0; i < n; ++i) {
      int r = 0;
      for (int b = 0; b < bits; ++b)
        if (i & (1 << b)) r |= 1 << (bits - 1 - b);
      p.rev[i] = r;
    }
  }
  return p;
}

// in-place complex DFT of length p.n; inverse = unnormalised e^{+}.
void fft1d(const Plan1D& p, cd* a, bool inverse, std::vector<cd>& scratch) {
  const int n = p.n;
  if (n <= 1) return;
  if (!p.pow2) {  // direct O(n^2) DFT for non-power-of-two lengths
    scratch.assign(a, a + n);
    for (int k = 0; k < n; ++k) {
      cd s(0, 0);
      for (int j = 0; j < n; ++j) {
        const cd w = p.tw[(static_cast<long long>(j) * k) % n];
        s += scratch[j] * (inverse ? std::conj(w) : w);
      }
      a[k] = s;
    }
    return;
  }
  for (int i = 0; i < n; ++i)
    if (i < p.rev[i]) std::swap(a[i], a[p.rev[i]]);
  for (int len = 2; len <= n; len <<= 1) {
    const int half = len >> 1, step = n / len;
    for (int i = 0; i < n; i += len)
      for (int j = 0; j < half; ++j) {
        cd w = p.tw[j * step];
        if (inverse) w = std::conj(w);
        const cd u = a[i + j];
        const cd t = a[i + j + half] * w;
        a[i + j] = u + t;
        a[i + j + half] = u - t;
      }
  }
}

// complex transforms along y and z of a [nz][ny][nh] half spectrum
void fft_yz(cd* S, int nh, int ny, int nz, bool inverse) {
  const Plan1D py = make_plan(ny), pz = make_plan(nz);
  std::vector<cd> line, scratch;
  constexpr int B = 16;  // gather B columns at a time for locality
  line.resize(static_cast<std::size_t>(std::max(ny, nz)) * B);
  auto do_axis = [&](const Plan1D& p, int n, std::size_t stride, int outer, std::size_t outer_stride) {
    for (int o = 0; o < outer; ++o)
      for (int x0 = 0; x0 < nh; x0 += B) {
        const int bw = std::min(B, nh - x0);
        cd* base = S + static_cast<std::size_t>(o) * outer_stride + x0;
        for (int j = 0; j < n; ++j)
          for (int b = 0; b < bw; ++b) line[static_cast<std::size_t>(b) * n + j] = base[j * stride + b];
        for (int b = 0; b < bw; ++b) fft1d(p, &line[static_cast<std::size_t>(b) * n], inverse, scratch);
        for (int j = 0; j < n; ++j)
          for (int b = 0; b < bw; ++b) base[j * stride + b] = line[static_cast<std::size_t>(b) * n + j];
      }
  };
  const std::size_t plane = static_cast<std::size_t>(ny) * nh;
  if (!inverse) {
    do_axis(py, ny, nh, nz, plane);  // y within each z plane
    do_axis(pz, nz, plane, ny, nh);  // z for each y row
  } else {
    do_axis(pz, nz, plane, ny, nh);
    do_axis(py, ny, nh, nz, plane);
  }
}
}  // namespace

// numpy.fft.rfftn over axes (z,y,x) of real[nz][ny][nx] -> [nz][ny][nx/2+1]
// (also the transform behind oracle/ref_shim/fftw3.h's fftw_plan_dft_r2c_3d)
void rfft3(const double* in, cd* S, int nx, int ny, int nz) {
  const int nh = nx / 2 + 1;
  const Plan1D px = make_plan(nx);
  std::vector<cd> row(nx), scratch;
  for (std::size_t r = 0; r < static_cast<std::size_t>(ny) * nz; ++r) {
    for (int x = 0; x < nx; ++x) row[x] = cd(in[r * nx + x], 0.0);
    fft1d(px, row.data(), false, scratch);
    for (int k = 0; k < nh; ++k) S[r * nh + k] = row[k];
  }
  fft_yz(S, nh, ny, nz, false);
}

// numpy.fft.irfftn (unnormalised, like FFTW c2r): destroys S.
// (also the transform behind oracle/ref_shim/fftw3.h's fftw_plan_dft_c2r_3d)
void irfft3(cd* S, double* out, int nx, int ny, int nz) {
  const int nh = nx / 2 + 1;
  fft_yz(S, nh, ny, nz, true);
  const Plan1D px = make_plan(nx);
  std::vector<cd> row(nx), scratch;
  for (std::size_t r = 0; r < static_cast<std::size_t>(ny) * nz; ++r) {
    const cd* h = S + r * nh;
    row[0] = cd(h[0].real(), 0.0);
    for (int k = 1; k < nh; ++k) row[k] = h[k];
    if (nx % 2 == 0) row[nx / 2] = cd(h[nx / 2].real(), 0.0);
    for (int k = nh; k < nx; ++k) row[k] = std::conj(h[nx - k]);
    fft1d(px, row.data(), true, scratch);
    for (int x = 0; x < nx; ++x) out[r * nx + x] = row[x].real();
  }
}

// integrate.cpp:19-74
void integrate_fft(const V3* field, int nx, int ny, int nz, double* out) {
  const std::size_t n_real = static_cast<std::size_t>(nx) * ny * nz;
  const int nh = nx / 2 + 1;
  const std::size_t n_cplx = static_cast<std::size_t>(nz) * ny * nh;
  std::vector<double> real_buf(n_real);
  std::vector<cd> spectrum(n_cplx), accum(n_cplx, cd(0.0, 0.0));
  auto signed_freq = [](int i, int n) {  // integrate.cpp:37-40
    const int m = i <= n / 2 ? i : i - n;
    return 2.0 * M_PI * m / n;
  };
  for (int c = 0; c < 3; ++c) {
    for (std::size_t i = 0; i < n_real; ++i) real_buf[i] = comp(field[i], c);
    rfft3(real_buf.data(), spectrum.data(), nx, ny, nz);
    std::size_t idx = 0;
    for (int z = 0; z < nz; ++z) {
      const double wz = signed_freq(z, nz);
      for (int y = 0; y < ny; ++y) {
        const double wy = signed_freq(y, ny);
        for (int x = 0; x <= nx / 2; ++x, ++idx) {
          const double wx = signed_freq(x, nx);
          const double w2 = wx * wx + wy * wy + wz * wz;
          if (w2 == 0.0) continue;
          const double wc = c == 0 ? wx : (c == 1 ? wy : wz);
          // (0 + jb)(sr + j si) = -b si + j b sr, b = -wc/w2
          const double b = -wc / w2;
          const cd s = spectrum[idx];
          accum[idx] = cd(accum[idx].real() + (0.0 * s.real() - b * s.imag()),
                          accum[idx].imag() + (0.0 * s.imag() + b * s.real()));
        }
      }
    }
  }
  irfft3(accum.data(), real_buf.data(), nx, ny, nz);
  const double scale = 1.0 / static_cast<double>(n_real);
  for (std::size_t i = 0; i < n_real; ++i) out[i] = real_buf[i] * scale;
}

// ------------------------------------------------------------ iso level
// volume.hpp:59-81
double sample_trilinear(const double* A, const GridSpec& g, V3 v) {
  auto clampf = [](double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); };
  const double fx = clampf(v.x, 0.0, g.nx - 1.0);
  const double fy = clampf(v.y, 0.0, g.ny - 1.0);
  const double fz = clampf(v.z, 0.0, g.nz - 1.0);
  const int x0 = std::min(static_cast<int>(fx), g.nx - 2 >= 0 ? g.nx - 2 : 0);
  const int y0 = std::min(static_cast<int>(fy), g.ny - 2 >= 0 ? g.ny - 2 : 0);
  const int z0 = std::min(static_cast<int>(fz), g.nz - 2 >= 0 ? g.nz - 2 : 0);
  const int x1 = std::min(x0 + 1, g.nx - 1), y1 = std::min(y0 + 1, g.ny - 1),
            z1 = std::min(z0 + 1, g.nz - 1);
  const double tx = fx - x0, ty = fy - y0, tz = fz - z0;
  auto at = [&](int x, int y, int z) {
    return A[static_cast<std::size_t>(x) + static_cast<std::size_t>(g.nx) * (y + static_cast<std::size_t>(g.ny) * z)];
  };
  const double v000 = at(x0, y0, z0), v100 = at(x1, y0, z0);
  const double v010 = at(x0, y1, z0), v110 = at(x1, y1, z0);
  const double v001 = at(x0, y0, z1), v101 = at(x1, y0, z1);
  const double v011 = at(x0, y1, z1), v111 = at(x1, y1, z1);
  const double c00 = v000 * (1 - tx) + v100 * tx;
  const double c10 = v010 * (1 - tx) + v110 * tx;
  const double c01 = v001 * (1 - tx) + v101 * tx;
  const double c11 = v011 * (1 - tx) + v111 * tx;
  const double c0 = c00 * (1 - ty) + c10 * ty;
  const double c1 = c01 * (1 - ty) + c11 * ty;
  return c0 * (1 - tz) + c1 * tz;
}

// splat.cpp:91-101
bool iso_level(const double* A, const GridSpec& g, const std::vector<const OrientedPoint*>& pts,
               double* level) {
  double sum = 0;
  std::size_t count = 0;
  for (const OrientedPoint* p : pts) {
    sum += sample_trilinear(A, g, to_voxel(g, p->position));
    ++count;
  }
  if (count == 0) return false;
  *level = sum / static_cast<double>(count);
  return true;
}

// ------------------------------------------------------------ marching cubes
// marching_cubes.cpp:14-29: corner i at ((i>>0)&1, (i>>1)&1, (i>>2)&1)
static const int kEdges[12][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}, {0, 2}, {1, 3},
                                  {4, 6}, {5, 7}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
static const int kFaces[6][4] = {{0, 2, 6, 4}, {1, 3, 7, 5}, {0, 1, 5, 4},
                                 {2, 3, 7, 6}, {0, 1, 3, 2}, {4, 5, 7, 6}};
static V3 corner_pos(int c) { return V3{double(c & 1), double((c >> 1) & 1), double((c >> 2) & 1)}; }
static int edge_between(int a, int b) {
  for (int e = 0; e < 12; ++e)
    if ((kEdges[e][0] == a && kEdges[e][1] == b) || (kEdges[e][0] == b && kEdges[e][1] == a)) return e;
  return -1;
}

// marching_cubes.cpp:52-122: chords on each face; ambiguous faces cut off the
// inside corners; loops traced from the lowest unused edge; oriented by the
// Newell normal against the inside->outside direction; fan from loop[0].
static std::vector<std::array<int, 3>> g_table[256];
static bool g_table_built = false;
static void build_table() {
  if (g_table_built) return;
  for (int config = 1; config < 255; ++config) {
    auto inside = [&](int c) { return (config >> c) & 1; };
    int partner[12][2];
    for (auto& p : partner) p[0] = p[1] = -1;
    auto link = [&](int ea, int eb) {
      for (int e : {ea, eb}) {
        int* p = partner[e];
        (p[0] == -1 ? p[0] : p[1]) = (e == ea ? eb : ea);
      }
    };
    for (const auto& face : kFaces) {
      int cuts[4], n_cuts = 0;
      for (int i = 0; i < 4; ++i) {
        const int a = face[i], b = face[(i + 1) % 4];
        if (inside(a) != inside(b)) cuts[n_cuts++] = edge_between(a, b);
      }
      if (n_cuts == 2) {
        link(cuts[0], cuts[1]);
      } else if (n_cuts == 4) {
        if (inside(face[0])) {
          link(cuts[3], cuts[0]);
          link(cuts[1], cuts[2]);
        } else {
          link(cuts[0], cuts[1]);
          link(cuts[2], cuts[3]);
        }
      }
    }
    bool used[12] = {};
    for (int start = 0; start < 12; ++start) {
      if (used[start] || partner[start][0] == -1) continue;
      std::vector<int> loop;
      int prev = -1, cur = start;
      do {
        loop.push_back(cur);
        used[cur] = true;
        const int next = partner[cur][0] == prev ? partner[cur][1] : partner[cur][0];
        prev = cur;
        cur = next;
      } while (cur != start);
      V3 outward{};
      std::vector<V3> mid(loop.size());
      for (std::size_t i = 0; i < loop.size(); ++i) {
        const int a = kEdges[loop[i]][0], b = kEdges[loop[i]][1];
        mid[i] = 0.5 * (corner_pos(a) + corner_pos(b));
        outward = outward + (inside(a) ? corner_pos(b) - corner_pos(a) : corner_pos(a) - corner_pos(b));
      }
      V3 newell{};
      for (std::size_t i = 0; i < loop.size(); ++i) newell = newell + cross(mid[i], mid[(i + 1) % loop.size()]);
      if (dot(newell, outward) < 0) std::reverse(loop.begin(), loop.end());
      for (std::size_t i = 1; i + 1 < loop.size(); ++i) g_table[config].push_back({loop[0], loop[i], loop[i + 1]});
    }
  }
  g_table_built = true;
}

void case_table(int counts[256], int tris[256][5][3]) {
  build_table();
  for (int c = 0; c < 256; ++c) {
    counts[c] = static_cast<int>(g_table[c].size());
    for (int t = 0; t < 5; ++t)
      for (int j = 0; j < 3; ++j)
        tris[c][t][j] = t < counts[c] ? g_table[c][t][j] : -1;
  }
}

// marching_cubes.cpp:131-210
Mesh marching_cubes(const double* A, const GridSpec& g, double level) {
  build_table();
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  Mesh mesh;
  if (nx < 2 || ny < 2 || nz < 2) return mesh;
  auto at = [&](int x, int y, int z) {
    return A[static_cast<std::size_t>(x) + static_cast<std::size_t>(nx) * (y + static_cast<std::size_t>(ny) * z)];
  };
  std::unordered_map<uint64_t, int> edge_vertex;
  auto global_edge = [&](int x, int y, int z, int axis) {
    return (static_cast<uint64_t>((static_cast<uint64_t>(z) * ny + y) * nx + x)) * 3 + axis;
  };
  const V3 origin{g.origin[0], g.origin[1], g.origin[2]};
  double vals[8];
  auto vertex_on_edge = [&](int cx, int cy, int cz, int edge) {
    const int c0 = kEdges[edge][0], c1 = kEdges[edge][1];
    const int axis = edge < 4 ? 0 : (edge < 8 ? 1 : 2);
    const int bx = cx + (c0 & 1), by = cy + ((c0 >> 1) & 1), bz = cz + ((c0 >> 2) & 1);
    const uint64_t key = global_edge(bx, by, bz, axis);
    if (auto it = edge_vertex.find(key); it != edge_vertex.end()) return it->second;
    double t = (level - vals[c0]) / (vals[c1] - vals[c0]);
    t = std::clamp(t, 1e-6, 1.0 - 1e-6);
    const V3 p = (V3{double(cx), double(cy), double(cz)} + corner_pos(c0)) + t * (corner_pos(c1) - corner_pos(c0));
    const int id = static_cast<int>(mesh.vertices.size());
    mesh.vertices.push_back(origin + g.edge * p);  // volume.hpp:45
    mesh.grid_positions.push_back(p);
    mesh.edge_ids.push_back(key);
    edge_vertex.emplace(key, id);
    return id;
  };
  for (int z = 0; z + 1 < nz; ++z)
    for (int y = 0; y + 1 < ny; ++y)
      for (int x = 0; x + 1 < nx; ++x) {
        int config = 0;
        for (int c = 0; c < 8; ++c) {
          vals[c] = at(x + (c & 1), y + ((c >> 1) & 1), z + ((c >> 2) & 1));
          if (vals[c] >= level) config |= 1 << c;
        }
        for (const auto& tri : g_table[config])
          mesh.triangles.push_back(
              {vertex_on_edge(x, y, z, tri[0]), vertex_on_edge(x, y, z, tri[1]), vertex_on_edge(x, y, z, tri[2])});
      }
  mesh.normals.resize(mesh.vertices.size());
  auto value_at = [&](int x, int y, int z) {
    return at(std::clamp(x, 0, nx - 1), std::clamp(y, 0, ny - 1), std::clamp(z, 0, nz - 1));
  };
  auto grad = [&](int x, int y, int z) {
    return V3{value_at(x + 1, y, z) - value_at(x - 1, y, z), value_at(x, y + 1, z) - value_at(x, y - 1, z),
              value_at(x, y, z + 1) - value_at(x, y, z - 1)} * 0.5;
  };
  for (std::size_t i = 0; i < mesh.vertices.size(); ++i) {
    const V3 p = mesh.grid_positions[i];
    const int x0 = std::clamp(static_cast<int>(p.x), 0, nx - 2);
    const int y0 = std::clamp(static_cast<int>(p.y), 0, ny - 2);
    const int z0 = std::clamp(static_cast<int>(p.z), 0, nz - 2);
    const double tx = p.x - x0, ty = p.y - y0, tz = p.z - z0;
    V3 gsum{};
    for (int dz = 0; dz <= 1; ++dz)
      for (int dy = 0; dy <= 1; ++dy)
        for (int dx = 0; dx <= 1; ++dx) {
          const double w = (dx ? tx : 1 - tx) * (dy ? ty : 1 - ty) * (dz ? tz : 1 - tz);
          if (w > 0) gsum = gsum + w * grad(x0 + dx, y0 + dy, z0 + dz);
        }
    const double len = norm(gsum);
    mesh.normals[i] = len > 1e-12 ? (-gsum) / len : V3{0, 0, 1};
  }
  return mesh;
}

// ------------------------------------------------------------ texture
// texture.cpp:11-34
void vertex_visibility(const std::vector<V3>& verts, const Sensor* sensors, const Frame* frames,
                       int k_count, double eps_vis_mm, uint8_t* vis) {
  const std::size_t V = verts.size();
  for (int k = 0; k < k_count; ++k) {
    const Pose inv = pose_inverse(sensors[k].pose);
    const Intrinsics& K = sensors[k].depth_intr;
    const Frame& f = frames[k];
    for (std::size_t v = 0; v < V; ++v) {
      uint8_t out = 0;
      const V3 local = pose_apply(inv, verts[v]);
      double u, w;
      if (project_local(K, local, &u, &w)) {
        const long px = std::lround(u), py = std::lround(w);
        if (px >= 0 && px < f.w && py >= 0 && py < f.h) {
          const std::size_t i = static_cast<std::size_t>(py) * f.w + px;
          if (f.mask[i]) {
            const double recorded = f.depth[i];
            if (std::abs(recorded - local.z) < eps_vis_mm) out = 1;
          }
        }
      }
      vis[static_cast<std::size_t>(k) * V + v] = out;
    }
  }
}

// texture.cpp:36-72 (+ normalize_uv, texture.hpp:45-47)
void assign_texture(const std::vector<V3>& verts, const Sensor* sensors, const Cloud* clouds,
                    int k_count, const uint8_t* vis, double* uv, float* wout, uint8_t* untextured) {
  const std::size_t V = verts.size();
  for (int k = 0; k < k_count; ++k) {
    const Sensor& s = sensors[k];
    const Pose rgb_pose = pose_compose(s.pose, s.rgb_relative);  // types.hpp:75
    for (std::size_t v = 0; v < V; ++v) {
      const std::size_t i = static_cast<std::size_t>(k) * V + v;
      uv[2 * i] = 0, uv[2 * i + 1] = 0;
      wout[i] = 0.f;
      if (!vis[i]) continue;
      double u, w;
      if (!project_local(s.rgb_intr, pose_apply_inverse(rgb_pose, verts[v]), &u, &w)) continue;
      uv[2 * i] = (u + 0.5) / s.rgb_intr.width;
      uv[2 * i + 1] = (w + 0.5) / s.rgb_intr.height;
      double ud, wd;
      if (project_local(s.depth_intr, pose_apply_inverse(s.pose, verts[v]), &ud, &wd)) {
        const long px = std::lround(ud), py = std::lround(wd);
        const Cloud& c = clouds[k];
        if (px >= 0 && px < c.w && py >= 0 && py < c.h)
          wout[i] = c.weight_map[static_cast<std::size_t>(py) * c.w + px];
      }
    }
  }
  for (std::size_t v = 0; v < V; ++v) {
    bool any = false;
    for (int k = 0; k < k_count; ++k) any = any || vis[static_cast<std::size_t>(k) * V + v];
    untextured[v] = any ? 0 : 1;
  }
}

// rasterize.cpp:12-27 (denormalize_uv: texture.hpp:48-50)
static void sample_bilinear(const Frame& f, double uvx, double uvy, double out[3]) {
  const int W = f.rgb_w, H = f.rgb_h;
  const double px = uvx * W - 0.5, py = uvy * H - 0.5;
  const int x0 = std::clamp(static_cast<int>(std::floor(px)), 0, W - 1);
  const int y0 = std::clamp(static_cast<int>(std::floor(py)), 0, H - 1);
  const int x1 = std::min(x0 + 1, W - 1), y1 = std::min(y0 + 1, H - 1);
  const double tx = std::clamp(px - x0, 0.0, 1.0), ty = std::clamp(py - y0, 0.0, 1.0);
  auto at = [&](int x, int y, int ch) { return double(f.rgb[(static_cast<std::size_t>(y) * W + x) * 3 + ch]); };
  for (int ch = 0; ch < 3; ++ch) {
    const double a = at(x0, y0, ch) * (1 - tx) + at(x1, y0, ch) * tx;
    const double b = at(x0, y1, ch) * (1 - tx) + at(x1, y1, ch) * tx;
    out[ch] = static_cast<double>(static_cast<uint8_t>(std::lround(a * (1 - ty) + b * ty)));
  }
}

// the uv-blend weighting of rasterize.cpp:136-157 evaluated at a vertex.
void blend_colors(int V, int k_count, const uint8_t* vis, const double* uv, const float* w,
                  const Frame* frames, double* color, uint8_t* rgb8) {
  for (int v = 0; v < V; ++v) {
    double r = 0, g = 0, b = 0, wsum = 0;
    for (int k = 0; k < k_count; ++k) {
      const std::size_t i = static_cast<std::size_t>(k) * V + v;
      if (!vis[i]) continue;
      const double wk = w[i];
      if (wk <= 1e-9) continue;
      double s[3];
      sample_bilinear(frames[k], uv[2 * i], uv[2 * i + 1], s);
      r += wk * s[0];
      g += wk * s[1];
      b += wk * s[2];
      wsum += wk;
    }
    double c[3];
    if (wsum > 1e-9) {
      c[0] = r / wsum, c[1] = g / wsum, c[2] = b / wsum;
    } else {
      c[0] = c[1] = c[2] = 200.0;
    }
    for (int ch = 0; ch < 3; ++ch) {
      color[3 * v + ch] = c[ch];
      rgb8[3 * v + ch] = static_cast<uint8_t>(std::clamp(c[ch], 0.0, 255.0));
    }
  }
}

}  // namespace orc

// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — the reference-side drop-in check of
// include/vc/volcap_adapter.hpp.  Compiled against the REFERENCE's headers
// (+ oracle/ref_shim) and linked with the reference's own code (libref.so)
// and the product (libvc_b200.so) by `make -C oracle ref`; run on a B200 by
// tests/test_gpu_c2_parity.py.
//
// A reference caller's frame loop (volcap.cpp:304-320) with recon::
// reconstruct_frame swapped for vc::adapter::reconstruct_frame: the same
// RgbdFrame/CameraRig/ReconConfig values go to both; the adapter's
// FrameReconstruction must carry bit-identical clouds and weight maps, the
// same grid, A within 1e-4 relative L2, the iso level within 1e-4, and a
// watertight mesh within 0.5 voxel of the reference's.
// Prints "ADAPTER OK ..." and exits 0, or prints the failure and exits 1.
#include <cmath>
#include <cstdio>
#include <unordered_map>
#include <vector>

#include "vc/volcap_adapter.hpp"
#include "volcap/synth/scene.hpp"

using namespace volcap;

namespace {
int fails = 0;
void expect(bool ok, const char* what) {
  if (!ok) {
    std::printf("FAIL %s\n", what);
    ++fails;
  }
}

// one-sided Hausdorff over a uniform hash grid with cell = r
double hausdorff_1(const std::vector<Vec3>& a, const std::vector<Vec3>& b, double r) {
  auto key = [r](const Vec3& p, int dx, int dy, int dz) {
    const long long x = (long long)std::floor(p.x() / r) + dx, y = (long long)std::floor(p.y() / r) + dy,
                    z = (long long)std::floor(p.z() / r) + dz;
    return (x * 73856093LL) ^ (y * 19349663LL) ^ (z * 83492791LL);
  };
  std::unordered_multimap<long long, int> h;
  for (int i = 0; i < (int)b.size(); ++i) h.emplace(key(b[i], 0, 0, 0), i);
  double worst = 0;
  for (const auto& p : a) {
    double best = 1e300;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          auto rg = h.equal_range(key(p, dx, dy, dz));
          for (auto it = rg.first; it != rg.second; ++it) best = std::min(best, (p - b[it->second]).norm());
        }
    worst = std::max(worst, best);
  }
  return worst;
}
}  // namespace

int main(int argc, char** argv) {
  const int r = argc > 1 ? std::atoi(argv[1]) : 7;
  const int kick_frame = argc > 2 ? std::atoi(argv[2]) : 150;
  synth::SyntheticScene scene = synth::make_kick_scene(300, 4, 0, 2500, 512, 424, 365);
  std::vector<RgbdFrame> frames;
  for (int k = 0; k < 4; ++k) frames.push_back(synth::render_frame(scene, k, kick_frame));
  recon::ReconConfig cfg;
  cfg.r = r;

  const recon::FrameReconstruction ref = recon::reconstruct_frame(frames, scene.rig, cfg);
  vc_ctx* ctx = nullptr;
  if (vc_ctx_create(0, &ctx) != VC_OK) {
    std::printf("FAIL vc_ctx_create\n");
    return 1;
  }
  const vc::adapter::Result got = vc::adapter::reconstruct_frame(frames, scene.rig, cfg, ctx);

  // clouds + weight maps: bit-identical
  expect(got.recon.clouds.size() == ref.clouds.size(), "cloud count");
  for (size_t k = 0; k < ref.clouds.size() && k < got.recon.clouds.size(); ++k) {
    const auto& a = got.recon.clouds[k];
    const auto& b = ref.clouds[k];
    expect(a.points.size() == b.points.size(), "points per sensor");
    bool same = a.points.size() == b.points.size() && a.weight_map == b.weight_map;
    for (size_t i = 0; same && i < a.points.size(); ++i)
      same = a.points[i].position == b.points[i].position && a.points[i].normal == b.points[i].normal &&
             a.points[i].weight == b.points[i].weight && a.points[i].px == b.points[i].px &&
             a.points[i].py == b.points[i].py && a.points[i].sensor == b.points[i].sensor;
    expect(same, "oriented points / weight map bit-identical");
  }
  // grid + field + level
  const auto& A = got.recon.volume.values;
  const auto& B = ref.volume.values;
  expect(A.nx() == B.nx() && A.ny() == B.ny() && A.nz() == B.nz(), "grid dims");
  expect(A.origin() == B.origin() && A.edge() == B.edge(), "grid origin / edge bit-identical");
  double num = 0, den = 0;
  for (size_t i = 0; i < B.size() && i < A.size(); ++i) {
    num += (A.data()[i] - B.data()[i]) * (A.data()[i] - B.data()[i]);
    den += B.data()[i] * B.data()[i];
  }
  const double rel = std::sqrt(num / den);
  expect(rel < 1e-4, "indicator A within 1e-4 relative L2");
  expect(std::abs(got.recon.volume.iso_level - ref.volume.iso_level) < 1e-4 * std::abs(ref.volume.iso_level),
         "iso level");
  // mesh
  const auto topo = analyze_topology(got.recon.mesh);
  expect(topo.edge_manifold, "adapter mesh watertight");
  const double h = std::max(hausdorff_1(got.recon.mesh.vertices, ref.mesh.vertices, B.edge()),
                            hausdorff_1(ref.mesh.vertices, got.recon.mesh.vertices, B.edge()));
  expect(h <= 0.5 * B.edge(), "mesh within 0.5 voxel Hausdorff");
  expect(got.textured.sensor_count == 4 && got.textured.visible.size() == 4, "textured mesh channels");
  vc_ctx_destroy(ctx);
  std::printf("%s r=%d frame=%d P=%zu V=%zu/%zu relL2(A)=%.3e hausdorff=%.4f voxel\n", fails ? "ADAPTER FAIL" : "ADAPTER OK",
              r, kick_frame, ref.clouds[0].points.size(), got.recon.mesh.vertices.size(), ref.mesh.vertices.size(),
              rel, h / B.edge());
  return fails ? 1 : 0;
}

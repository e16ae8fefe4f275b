// Reference-typed C++ adapter test: compiled against the reference's own headers
// (/root/reference/proj/include/sconv) + include/sconv_b200.hpp, linked to libsconv_b200.so.
// Runs on the GPU box (tests/test_adapter.py); checks maps and features against an inline
// brute-force Eq. 2 evaluation written with the reference types.
#include <sconv/geometry.hpp>
#include <sconv/prng.hpp>

#include <cmath>
#include <cstdio>
#include <map>

#include "sconv_b200.hpp"

int main() {
  using namespace sconv;
  Rng rng(stream_seed(5, 0));
  CoordList c;
  std::map<PackedKey, int> seen;
  while (c.size() < 3000) {
    Coordinate p{static_cast<int>(rng.next_below(24)) - 12, static_cast<int>(rng.next_below(24)),
                 static_cast<int>(rng.next_below(24))};
    if (seen.emplace(pack_key(p), static_cast<int>(c.size())).second) c.push_back(p);
  }
  PointCloud P{make_coords(c), Matrix(static_cast<std::int64_t>(c.size()), 8), false};
  for (std::int64_t r = 0; r < P.size(); ++r)
    for (int ch = 0; ch < 8; ++ch) P.features(r, ch) = static_cast<float>(rng.next_unit());
  std::vector<float> W(27 * 8 * 16);
  for (auto& w : W) w = static_cast<float>(-0.1 + 0.2 * rng.next_unit());
  gpu::Context ctx(0);
  auto [Q, km] = gpu::build_kernel_map_sorted(ctx, P, 3, 1);
  const OffsetSet d = weight_offsets(3, 1);
  std::int64_t brute = 0;
  for (int k = 0; k < 27; ++k)
    for (std::size_t i = 0; i < Q->size(); ++i) {
      const Coordinate t = (*Q)[i] + d.offsets[k];
      if (in_range(t) && seen.count(pack_key(t))) ++brute;
    }
  if (brute != km.total()) {
    std::printf("FAIL map size %lld vs %lld\n", static_cast<long long>(km.total()), static_cast<long long>(brute));
    return 1;
  }
  PointCloud out = gpu::sc_layer_forward(ctx, P, W, 16, 3, 1);
  double maxerr = 0, scale = 0;
  for (std::size_t i = 0; i < out.coords->size(); ++i)
    for (int n = 0; n < 16; ++n) {
      double acc = 0;
      for (int k = 0; k < 27; ++k) {
        const Coordinate t = (*out.coords)[i] + d.offsets[k];
        auto it = in_range(t) ? seen.find(pack_key(t)) : seen.end();
        if (it == seen.end()) continue;
        for (int ch = 0; ch < 8; ++ch) acc += P.features(it->second, ch) * W[(k * 8 + ch) * 16 + n];
      }
      maxerr = std::max(maxerr, std::fabs(acc - out.features(static_cast<std::int64_t>(i), n)));
      scale = std::max(scale, std::fabs(acc));
    }
  bool threw = false;
  try {
    PointCloud bad{make_coords({{COORD_MAX + 1, 0, 0}}), Matrix(1, 8), false};
    gpu::build_kernel_map_sorted(ctx, bad, 3, 1);
  } catch (const std::out_of_range& e) {
    threw = std::string(e.what()) == "coordinate x out of range: 1048576";
  }
  // GPU voxelize vs the reference's own voxelize (geometry.hpp:180-255): identical, bit for bit
  std::vector<std::array<double, 3>> pts;
  Matrix vf(3000, 5);
  for (int i = 0; i < 3000; ++i) {
    pts.push_back({std::sin(i * 0.37) * 7.0, std::cos(i * 0.11) * 3.0, (i % 97) * 0.031});
    for (int c = 0; c < 5; ++c) vf(i, c) = static_cast<float>(std::sin(i * 1.7 + c));
  }
  const PointCloud vr = voxelize(pts, vf, 0.25);
  const PointCloud vg = gpu::voxelize(ctx, pts, vf, 0.25);
  bool vox_ok = vr.coords->size() == vg.coords->size() && vg.sorted;
  for (std::size_t i = 0; vox_ok && i < vr.coords->size(); ++i) {
    vox_ok = (*vr.coords)[i] == (*vg.coords)[i];
    for (int c = 0; vox_ok && c < 5; ++c)
      vox_ok = vr.features(static_cast<std::int64_t>(i), c) == vg.features(static_cast<std::int64_t>(i), c);
  }
  // .mpc round trip of the voxelized cloud through the adapter's file readers
  const std::string mpc = "/tmp/sconv_adapter_test.mpc";
  gpu::write_mpc(mpc, vg);
  const PointCloud back = gpu::read_mpc(mpc);
  bool io_ok = !back.sorted && back.coords->size() == vg.coords->size() && back.channels() == vg.channels();
  for (std::size_t i = 0; io_ok && i < back.coords->size(); ++i) {
    io_ok = (*back.coords)[i] == (*vg.coords)[i];
    for (int c = 0; io_ok && c < 5; ++c)
      io_ok = back.features(static_cast<std::int64_t>(i), c) == vg.features(static_cast<std::int64_t>(i), c);
  }
  std::remove(mpc.c_str());
  std::printf("adapter: |Q|=%zu |M|=%lld max_rel=%.3g threw=%d voxelize_exact=%d (%zu voxels) mpc_round_trip=%d\n",
              out.coords->size(), static_cast<long long>(km.total()), maxerr / scale, threw ? 1 : 0, vox_ok ? 1 : 0,
              vr.coords->size(), io_ok ? 1 : 0);
  return (maxerr / scale <= 1e-2 && threw && vox_ok && io_ok) ? 0 : 1;
}

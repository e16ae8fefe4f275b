// Reference-typed C++ adapter test: compiled against the reference's own headers
// (/root/reference/proj/include/sconv) + include/sconv_b200.hpp, linked to libsconv_b200.so
// and (as the checker only) to the oracle built on the same reference headers
// (oracle/_ref/liboracle_ref.so). Runs on the GPU box (tests/test_adapter.py): maps and
// features against an inline brute-force Eq. 2 evaluation written with the reference types,
// and the SPEC-signature calls (build_kernel_map_sorted(P, Q, offsets, B, C) with
// SearchCounters, WeightSet, sc_layer_forward, forward_network, theoretical_hyperparams)
// against the oracle's functions of the same names.
#include <sconv/geometry.hpp>
#include <sconv/prng.hpp>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>

#include "sconv_b200.hpp"
#include "sconv_oracle.hpp"  // test infrastructure: the checker

namespace {
// rel_e = |g - r| / max(|r|, 1e-3 ||r||_inf); returns {max, mean, frobenius-relative}
std::array<double, 3> rel_e(const sconv::Matrix& g, const sconv::Matrix& r) {
  double inf = 0, num = 0, den = 0, mx = 0, sum = 0;
  for (float v : r.data()) inf = std::max(inf, std::fabs(double{v}));
  const double floor = std::max(1e-3 * inf, 1e-30);
  for (std::size_t e = 0; e < r.data().size(); ++e) {
    const double d = std::fabs(double{g.data()[e]} - double{r.data()[e]});
    const double x = d / std::max(std::fabs(double{r.data()[e]}), floor);
    mx = std::max(mx, x);
    sum += x;
    num += d * d;
    den += double{r.data()[e]} * r.data()[e];
  }
  const double n = std::max<double>(1.0, static_cast<double>(r.data().size()));
  return {mx, sum / n, std::sqrt(num / std::max(den, 1e-300))};
}

// SPEC-signature calls vs the oracle; returns the number of failed checks
int spec_api_checks(sconv::gpu::Context& ctx) {
  using namespace sconv;
  int fails = 0;
  auto expect = [&](bool ok, const char* what) {
    if (!ok) {
      std::printf("FAIL %s\n", what);
      ++fails;
    }
  };
  // build_kernel_map_sorted(P, Q, offsets, B, C): unsorted P, arbitrary sorted Q, K=5 s=2 offsets
  const PointCloud P = oracle::generate_synthetic(6000, 30, 8, 21);
  CoordList qs = *P.coords;
  for (int i = 0; i < 2000; ++i) qs.push_back({i % 37 - 3, (i * 7) % 41 - 5, (i * 13) % 33});
  std::sort(qs.begin(), qs.end(), [](const Coordinate& a, const Coordinate& b) { return pack_key(a) < pack_key(b); });
  qs.erase(std::unique(qs.begin(), qs.end()), qs.end());
  const CoordsPtr Q = make_coords(qs);
  for (const auto& [offs, B, C] : {std::tuple{weight_offsets(3, 1), 256, 512}, std::tuple{weight_offsets(5, 2), 64, 100}}) {
    const auto [gm, gc] = gpu::build_kernel_map_sorted(ctx, P, *Q, offs, B, C);
    const auto [om, oc] = oracle::build_kernel_map_sorted(P, Q, offs, B, C, 4);
    expect(gm.matches == om.matches, "build_kernel_map_sorted(P, Q, offsets, B, C): map");
    expect(gc.counted && gc.backward_comparisons == oc.backward_comparisons &&
               gc.forward_comparisons == oc.forward_comparisons &&
               gc.source_elements_loaded == oc.source_elements_loaded && gc.queries_executed == oc.queries_executed &&
               gc.sorts == oc.sorts,
           "SearchCounters equal to the oracle's");
  }
  bool threw = false;
  try {
    CoordList bad = {{1, 0, 0}, {0, 0, 0}};
    gpu::build_kernel_map_sorted(ctx, P, bad, weight_offsets(3, 1));
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()) == "query coordinates must be sorted and unique";
  }
  expect(threw, "unsorted Q -> std::invalid_argument");
  // theoretical_hyperparams
  for (auto [p, q] : {std::pair<long, long>{65536, 65536}, {100000, 100000}, {123457, 40001}, {7, 300}})
    expect(gpu::theoretical_hyperparams(p, q) == oracle::theoretical_hyperparams(p, q), "theoretical_hyperparams");
  // WeightSet + sc_layer_forward vs the oracle's sc_layer_forward (16-bit operands: same-operand metric)
  const gpu::WeightSet W = gpu::WeightSet::generate(21, 1, 27, 8, 16);
  const oracle::WeightSet OW = oracle::generate_weights(21, 1, 27, 8, 16);
  expect(W.w == OW.w, "WeightSet::generate == oracle generate_weights (bits)");
  oracle::WeightSet W16 = OW;
  for (float& v : W16.w) v = static_cast<float>(static_cast<_Float16>(v));
  PointCloud P16 = P;
  for (std::int64_t r = 0; r < P16.size(); ++r)
    for (int c = 0; c < 8; ++c) P16.features(r, c) = static_cast<float>(static_cast<_Float16>(P16.features(r, c)));
  const PointCloud go = gpu::sc_layer_forward(ctx, P, W, 3, 1);
  oracle::LayerConfig ocfg;
  ocfg.workers = 4;
  const PointCloud oo = oracle::sc_layer_forward(P16, W16, 3, 1, ocfg);
  expect(*go.coords == *oo.coords, "sc_layer_forward(WeightSet): coordinates");
  const auto e1 = rel_e(go.features, oo.features);
  expect(e1[0] <= 1e-2 && e1[1] <= 1e-3, "sc_layer_forward(WeightSet): 8(c) metric");
  // forward_network: strides [1, 2, 1, 2, 1] -> 3 sorts (acceptance #7), SPEC weights
  gpu::NetworkSpec gs;
  oracle::NetworkSpec os;
  for (auto [K, s, ci, co] : {std::array<int, 4>{3, 1, 8, 16}, {3, 2, 16, 32}, {3, 1, 32, 32}, {3, 2, 32, 64}, {3, 1, 64, 64}}) {
    gs.layers.push_back({K, s, ci, co});
    os.layers.push_back({K, s, ci, co});
  }
  const auto gr = gpu::forward_network(ctx, gs, P, gpu::LayerConfig{}, 9);
  const auto orr = oracle::forward_network(os, P, ocfg, 9);
  expect(*gr.output.coords == *orr.output.coords, "forward_network: coordinates");
  expect(gr.sorts == 3 && orr.sorts == 3, "forward_network: 3 sorts for strides [1,2,1,2,1]");
  const auto e2 = rel_e(gr.output.features, orr.output.features);
  expect(e2[2] <= 2e-3, "forward_network: Frobenius-relative error");
  std::printf("spec_api: K=3/K=5 maps+counters, hyperparams, WeightSet, layer rel_e max %.2e mean %.2e, "
              "forward_network fro %.2e sorts %llu, failures %d\n",
              e1[0], e1[1], e2[2], static_cast<unsigned long long>(gr.sorts), fails);
  return fails;
}
}  // namespace

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
  const int spec_fails = spec_api_checks(ctx);
  return (maxerr / scale <= 1e-2 && threw && vox_ok && io_ok && spec_fails == 0) ? 0 : 1;
}

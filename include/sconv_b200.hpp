// sconv_b200.hpp — header-only C++ adapter: the reference's SC-layer API on the B200 engine.
//
// Include AFTER the reference's own headers (<sconv/geometry.hpp>, proj/include/sconv/
// geometry.hpp:16-257): the functions take and return the reference types (PointCloud,
// Matrix, OffsetSet, Coordinate) and rethrow the reference exception types with the same
// messages (geometry.hpp:53 std::out_of_range "coordinate x out of range: v",
// std::invalid_argument for arguments, std::logic_error for invariant violations).
//
//   sconv::gpu::Context ctx(0);
//   auto [Q, map] = sconv::gpu::build_kernel_map_sorted(ctx, P, K, s);       // SPEC.md:235 (layer form)
//   auto [km, counters] = sconv::gpu::build_kernel_map_sorted(ctx, P, Q, offsets, 256, 512);  // SPEC form
//   sconv::PointCloud out = sconv::gpu::sc_layer_forward(ctx, P, W, K, s);
//   auto res = sconv::gpu::forward_network(ctx, spec, P, cfg, seed);
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sconv_b200.h"

namespace sconv::gpu {

inline void check(sconv_status st, const char* msg) {
  switch (st) {
    case SCONV_OK:
      return;
    case SCONV_ERR_ARG:
      throw std::invalid_argument(msg);
    case SCONV_ERR_RANGE:
      throw std::out_of_range(msg);
    case SCONV_ERR_STATE:
      throw std::logic_error(msg);
    default:
      throw std::runtime_error(msg);
  }
}

class Context {
 public:
  explicit Context(int device = 0) { check(sconv_ctx_create(device, &h_), sconv_global_last_error()); }
  ~Context() { sconv_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  sconv_ctx* get() const { return h_; }
  void check_status(sconv_status st) const { check(st, sconv_last_error(h_)); }

 private:
  sconv_ctx* h_ = nullptr;
};

// KernelMap: per offset k, (input j, output i) pairs sorted by i.
struct KernelMap {
  OffsetSet offsets;
  std::vector<std::vector<std::pair<std::int32_t, std::int32_t>>> matches;
  std::int64_t total() const {
    std::int64_t t = 0;
    for (const auto& m : matches) t += static_cast<std::int64_t>(m.size());
    return t;
  }
};

struct LayerConfig {  // SPEC.md:359 config{grouping policy, eps, max_batch, tiles T_g/T_s, B, C}
  int policy = SCONV_GROUP_SORTED;
  double epsilon = 0.25;
  int max_batch = 16;
  int gather_tile = 0, scatter_tile = 0;  // 0 = tuned / heuristic
  int B = 256, C = 512;
  int compute_dtype = SCONV_F16;
  int partial_f16 = 0;
  int dataflow = SCONV_DATAFLOW_GMAS;  // SCONV_DATAFLOW_FUSED: one output-stationary kernel
};

namespace detail {
inline std::vector<std::int32_t> flatten(const CoordList& c) {
  std::vector<std::int32_t> v(c.size() * 3);
  for (std::size_t i = 0; i < c.size(); ++i) {
    v[3 * i] = c[i].x;
    v[3 * i + 1] = c[i].y;
    v[3 * i + 2] = c[i].z;
  }
  return v;
}
inline CoordList unflatten(const std::vector<std::int32_t>& v, std::int64_t n) {
  CoordList c(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) c[i] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
  return c;
}
}  // namespace detail

// build_kernel_map_sorted for a SPEC-literal layer: Q = Eq. 1 coordinates of P with stride
// s (sorted; for s == 1 and sorted P they alias P), offsets = weight_offsets(K, s).
inline std::pair<CoordsPtr, KernelMap> build_kernel_map_sorted(Context& ctx, const PointCloud& P, int K, int s,
                                                               int B = 256, int C = 512) {
  const auto xyz = detail::flatten(*P.coords);
  sconv_map_cfg cfg{K, s, s, 0, B, C, SCONV_MAP_SORTED};
  sconv_map* m = nullptr;
  ctx.check_status(sconv_map_build(ctx.get(), xyz.data(), P.size(), SCONV_MEM_HOST, P.sorted ? 1 : 0, &cfg, nullptr,
                                   0, SCONV_MEM_HOST, &m));
  sconv_map_info info;
  ctx.check_status(sconv_map_get_info(ctx.get(), m, &info));
  std::vector<std::int32_t> q(static_cast<std::size_t>(info.num_outputs) * 3), in(info.total_matches),
      out(info.total_matches);
  std::vector<std::int64_t> sizes(info.num_offsets);
  const sconv_status st = sconv_map_read(ctx.get(), m, q.data(), sizes.data(), in.data(), out.data());
  sconv_map_free(ctx.get(), m);
  ctx.check_status(st);
  KernelMap km;
  km.offsets = weight_offsets(K, s);
  km.matches.resize(static_cast<std::size_t>(info.num_offsets));
  std::size_t pos = 0;
  for (int k = 0; k < info.num_offsets; ++k)
    for (std::int64_t r = 0; r < sizes[k]; ++r, ++pos) km.matches[k].emplace_back(in[pos], out[pos]);
  CoordsPtr Q = (s == 1 && P.sorted) ? P.coords : make_coords(detail::unflatten(q, info.num_outputs));
  return {Q, std::move(km)};
}

// SearchCounters. The comparison tallies are filled (counted) by the
// SORTED_SPEC backend, whose work decomposition is the SPEC's; sorts by every backend.
struct SearchCounters {
  std::uint64_t backward_comparisons = 0, forward_comparisons = 0, source_elements_loaded = 0, queries_executed = 0;
  std::uint64_t sorts = 0;
  bool counted = false;
};

// build_kernel_map_sorted(P, Q, offsets, B, C) -> (KernelMap, SearchCounters):
// arbitrary sorted unique queries Q and any OffsetSet (reference OffsetSet, geometry.hpp:123-148).
// Errors as the reference: std::out_of_range for out-of-range coordinates, std::invalid_argument
// for unsorted queries or bad B / C.
inline std::pair<KernelMap, SearchCounters> build_kernel_map_sorted(Context& ctx, const PointCloud& P,
                                                                    const CoordList& Q, const OffsetSet& offsets,
                                                                    int B = 256, int C = 512,
                                                                    int backend = SCONV_MAP_SORTED_SPEC) {
  const auto pxyz = detail::flatten(*P.coords);
  const auto qxyz = detail::flatten(Q);
  const auto oxyz = detail::flatten(offsets.offsets);
  sconv_map* m = nullptr;
  ctx.check_status(sconv_map_build_explicit(ctx.get(), pxyz.data(), P.size(), SCONV_MEM_HOST, P.sorted ? 1 : 0,
                                            qxyz.data(), static_cast<std::int64_t>(Q.size()), SCONV_MEM_HOST,
                                            oxyz.data(), static_cast<int>(offsets.offsets.size()), B, C, backend, &m));
  sconv_map_info info;
  sconv_search_counters c;
  sconv_status st = sconv_map_get_info(ctx.get(), m, &info);
  if (st == SCONV_OK) st = sconv_map_search_counters(ctx.get(), m, &c);
  std::vector<std::int32_t> in(static_cast<std::size_t>(st == SCONV_OK ? info.total_matches : 0)), out(in.size());
  std::vector<std::int64_t> sizes(static_cast<std::size_t>(st == SCONV_OK ? info.num_offsets : 0));
  if (st == SCONV_OK) st = sconv_map_read(ctx.get(), m, nullptr, sizes.data(), in.data(), out.data());
  if (st != SCONV_OK) {
    const std::string msg = sconv_last_error(ctx.get());
    sconv_map_free(ctx.get(), m);
    check(st, msg.c_str());
  }
  sconv_map_free(ctx.get(), m);
  KernelMap km;
  km.offsets = offsets;
  km.matches.resize(sizes.size());
  std::size_t pos = 0;
  for (std::size_t k = 0; k < sizes.size(); ++k)
    for (std::int64_t r = 0; r < sizes[k]; ++r, ++pos) km.matches[k].emplace_back(in[pos], out[pos]);
  SearchCounters sc;
  sc.backward_comparisons = c.backward_comparisons;
  sc.forward_comparisons = c.forward_comparisons;
  sc.source_elements_loaded = c.source_elements_loaded;
  sc.queries_executed = c.queries_executed;
  sc.sorts = c.sorts;
  sc.counted = c.counted != 0;
  return {std::move(km), sc};
}

// theoretical_hyperparams(|P|, |Q|) -> (B, C) (Eq. 4); advisory.
inline std::pair<int, int> theoretical_hyperparams(std::int64_t P, std::int64_t Q) {
  int B = 0, C = 0;
  check(sconv_theoretical_hyperparams(P, Q, &B, &C), sconv_global_last_error());
  return {B, C};
}

// WeightSet: per offset k a C_in x C_out fp32 matrix W_k, flattened [k][cin][cout].
struct WeightSet {
  int num_offsets = 0, c_in = 0, c_out = 0;
  std::vector<float> w;
  const float* matrix(int k) const { return w.data() + static_cast<std::size_t>(k) * c_in * c_out; }
  // Rng(stream_seed(seed, stream)), U[-0.1, 0.1] (bit-identical to the oracle)
  static WeightSet generate(std::uint64_t seed, std::uint64_t stream, int num_offsets, int c_in, int c_out) {
    WeightSet ws{num_offsets, c_in, c_out, std::vector<float>(static_cast<std::size_t>(num_offsets) * c_in * c_out)};
    check(sconv_generate_weights(seed, stream, num_offsets, c_in, c_out, ws.w.data()), sconv_global_last_error());
    return ws;
  }
};

// voxelize (geometry.hpp:180-255) on the GPU: same voxels, same mean-merged features, bit for bit.
inline PointCloud voxelize(Context& ctx, const std::vector<std::array<double, 3>>& points, const Matrix& features,
                           double resolution) {
  const auto n = static_cast<std::int64_t>(points.size());
  const std::int64_t channels = features.empty() ? 0 : features.cols();
  if (channels > 0 && features.rows() != n) throw std::invalid_argument("feature row count does not match point count");
  std::vector<std::int32_t> xyz(static_cast<std::size_t>(3 * n));
  std::vector<float> f(static_cast<std::size_t>(std::max<std::int64_t>(1, n * channels)));
  std::int64_t nv = 0;
  ctx.check_status(sconv_voxelize(ctx.get(), n ? points[0].data() : nullptr, n, SCONV_MEM_HOST,
                                  channels ? features.row(0) : nullptr, channels, SCONV_MEM_HOST, resolution,
                                  xyz.data(), f.data(), SCONV_MEM_HOST, &nv));
  xyz.resize(static_cast<std::size_t>(3 * nv));
  PointCloud out;
  out.coords = make_coords(detail::unflatten(xyz, nv));
  if (channels > 0) {
    out.features = Matrix(nv, channels);
    for (std::int64_t r = 0; r < nv; ++r)
      for (std::int64_t c = 0; c < channels; ++c) out.features(r, c) = f[static_cast<std::size_t>(r * channels + c)];
  }
  out.sorted = true;
  return out;
}

// Point-cloud files. .mpc -> PointCloud of voxel coordinates (sorted = false);
// .xyz -> float points + features (the input of voxelize). Parse errors: std::invalid_argument.
inline PointCloud read_mpc(const std::string& path) {
  int fmt = 0;
  std::int64_t n = 0, c = 0;
  check(sconv_cloud_file_info(path.c_str(), &fmt, &n, &c), sconv_global_last_error());
  if (fmt != SCONV_FILE_MPC) throw std::invalid_argument("mpc parse error at offset 0: bad magic");
  std::vector<std::int32_t> xyz(static_cast<std::size_t>(3 * n));
  std::vector<float> f(static_cast<std::size_t>(std::max<std::int64_t>(1, n * c)));
  check(sconv_mpc_read(path.c_str(), xyz.data(), f.data(), n, c), sconv_global_last_error());
  PointCloud out;
  out.coords = make_coords(detail::unflatten(xyz, n));
  if (c > 0) {
    out.features = Matrix(n, c);
    for (std::int64_t r = 0; r < n; ++r)
      for (std::int64_t k = 0; k < c; ++k) out.features(r, k) = f[static_cast<std::size_t>(r * c + k)];
  }
  out.sorted = false;
  return out;
}

inline void write_mpc(const std::string& path, const PointCloud& cloud) {
  const auto xyz = detail::flatten(*cloud.coords);
  const std::int64_t c = cloud.channels();
  check(sconv_mpc_write(path.c_str(), xyz.data(), c ? cloud.features.row(0) : nullptr, cloud.size(), c),
        sconv_global_last_error());
}

inline std::pair<std::vector<std::array<double, 3>>, Matrix> read_xyz(const std::string& path) {
  int fmt = 0;
  std::int64_t n = 0, c = 0;
  check(sconv_cloud_file_info(path.c_str(), &fmt, &n, &c), sconv_global_last_error());
  if (fmt != SCONV_FILE_XYZ) throw std::invalid_argument("xyz parse error at line 1: binary .mpc file");
  std::vector<std::array<double, 3>> pts(static_cast<std::size_t>(n));
  std::vector<float> f(static_cast<std::size_t>(std::max<std::int64_t>(1, n * c)));
  check(sconv_xyz_read(path.c_str(), n ? pts[0].data() : nullptr, f.data(), n, c), sconv_global_last_error());
  Matrix feats(c > 0 ? n : 0, c);
  for (std::int64_t r = 0; c > 0 && r < n; ++r)
    for (std::int64_t k = 0; k < c; ++k) feats(r, k) = f[static_cast<std::size_t>(r * c + k)];
  return {std::move(pts), std::move(feats)};
}

// sc_layer_forward. W: K^3 matrices C_in x C_out, flattened [k][cin][cout].
inline PointCloud sc_layer_forward(Context& ctx, const PointCloud& cloud, const std::vector<float>& W, int c_out,
                                   int K, int s, const LayerConfig& cfg = {}) {
  const auto xyz = detail::flatten(*cloud.coords);
  const int c_in = static_cast<int>(cloud.channels());
  sconv_exec_cfg ec{cfg.policy,       cfg.epsilon,      cfg.max_batch,   cfg.gather_tile,
                    cfg.scatter_tile, cfg.compute_dtype, cfg.partial_f16, cfg.dataflow, 1};
  std::vector<std::int32_t> oxyz(xyz.size());
  Matrix out(cloud.size(), c_out);
  std::int64_t n_out = 0;
  ctx.check_status(sconv_sc_layer_forward(ctx.get(), xyz.data(), cloud.size(), cloud.sorted ? 1 : 0,
                                          cloud.size() ? cloud.features.row(0) : nullptr, c_in, W.data(), c_out, K,
                                          s, &ec, oxyz.data(), &n_out, cloud.size() ? out.row(0) : nullptr));
  Matrix trimmed(n_out, c_out);
  for (std::int64_t r = 0; r < n_out; ++r)
    for (int c = 0; c < c_out; ++c) trimmed(r, c) = out(r, c);
  CoordsPtr Q = (s == 1 && cloud.sorted) ? cloud.coords : make_coords(detail::unflatten(oxyz, n_out));
  return PointCloud{Q, std::move(trimmed), true};
}

// sc_layer_forward with a WeightSet.
inline PointCloud sc_layer_forward(Context& ctx, const PointCloud& cloud, const WeightSet& W, int K, int s,
                                   const LayerConfig& cfg = {}) {
  if (W.c_in != cloud.channels()) throw std::invalid_argument("feature channels do not match weights");
  return sc_layer_forward(ctx, cloud, W.w, W.c_out, K, s, cfg);
}

// NetworkSpec: ordered (K, s, C_in, C_out) layers.
struct NetLayer {
  int K, s, c_in, c_out;
};
struct NetworkSpec {
  std::vector<NetLayer> layers;
};
struct NetworkResult {
  PointCloud output;
  std::uint64_t sorts = 0;  // coordinate sorts performed (1 + strided layers)
};

// forward_network(spec, cloud, config, seed) on the GPU network driver: layer
// l is the SPEC-literal SC layer (offsets weight_offsets(K, s), Eq. 1 stride s) with weights
// Rng(stream_seed(seed, l + 1)) U[-0.1, 0.1]; layer l+1 reads layer l's sorted output
// coordinates (sort reuse). Activations between layers in cfg.compute_dtype (16-bit).
inline NetworkResult forward_network(Context& ctx, const NetworkSpec& spec, const PointCloud& cloud,
                                     const LayerConfig& cfg, std::uint64_t seed) {
  if (spec.layers.empty()) throw std::invalid_argument("empty network");
  if (cloud.channels() != spec.layers.front().c_in) throw std::invalid_argument("network input channels mismatch");
  for (std::size_t l = 1; l < spec.layers.size(); ++l)
    if (spec.layers[l - 1].c_out != spec.layers[l].c_in)
      throw std::invalid_argument("network layers are not channel compatible");
  const int L = static_cast<int>(spec.layers.size());
  std::vector<std::int32_t> ops;
  for (int l = 0; l < L; ++l) {
    const NetLayer& y = spec.layers[static_cast<std::size_t>(l)];
    ops.insert(ops.end(), {1, l + 1, l, -1, y.K, y.s, y.s, 0, y.c_in, y.c_out, l, 0});
  }
  sconv_exec_cfg ec{cfg.policy,       cfg.epsilon,       cfg.max_batch,   cfg.gather_tile,
                    cfg.scatter_tile, cfg.compute_dtype, cfg.partial_f16, SCONV_DATAFLOW_AUTO, 1};
  sconv_net* net = nullptr;
  ctx.check_status(sconv_net_create(ctx.get(), ops.data(), L, L + 1, 0, L, &ec, cfg.B, cfg.C, &net));
  struct Guard {
    Context& c;
    sconv_net* n;
    ~Guard() { sconv_net_free(c.get(), n); }
  } guard{ctx, net};
  for (int l = 0; l < L; ++l) {
    const NetLayer& y = spec.layers[static_cast<std::size_t>(l)];
    const WeightSet w = WeightSet::generate(seed, static_cast<std::uint64_t>(l + 1), y.K * y.K * y.K, y.c_in, y.c_out);
    ctx.check_status(sconv_net_set_weights(ctx.get(), net, l, w.w.data(), SCONV_MEM_HOST, w.num_offsets, w.c_in,
                                           w.c_out));
  }
  const auto xyz = detail::flatten(*cloud.coords);
  ctx.check_status(sconv_net_forward(ctx.get(), net, xyz.data(), cloud.size(), SCONV_MEM_HOST, cloud.sorted ? 1 : 0,
                                     cloud.size() ? cloud.features.row(0) : nullptr, SCONV_MEM_HOST,
                                     static_cast<int>(cloud.channels())));
  std::int64_t n = 0;
  int ch = 0, cs = 0;
  ctx.check_status(sconv_net_tensor_info(ctx.get(), net, L, &n, &ch, &cs));
  std::vector<std::int32_t> oxyz(static_cast<std::size_t>(3 * n));
  Matrix f(n, ch);
  ctx.check_status(sconv_net_read_tensor(ctx.get(), net, L, oxyz.data(), n ? f.row(0) : nullptr));
  std::int64_t sorts = 0;
  ctx.check_status(sconv_net_sort_count(net, &sorts));
  NetworkResult r;
  r.output = PointCloud{make_coords(detail::unflatten(oxyz, n)), std::move(f), true};
  r.sorts = static_cast<std::uint64_t>(sorts);
  return r;
}

}  // namespace sconv::gpu

// TEST INFRASTRUCTURE — flat C API over the CPU oracle for ctypes (tests/, smoke(),
// bench.py cpu_baseline only). Status codes: 0 ok, 1 std::invalid_argument,
// 2 std::out_of_range, 3 other exception; message via so_last_error().
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>

#include "sconv_oracle.hpp"

using namespace sconv;
using namespace sconv::oracle;

namespace {
thread_local std::string g_err;

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

CoordList to_coords(const std::int32_t* xyz, std::int64_t n) {
  CoordList c(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) c[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  return c;
}
void from_coords(const CoordList& c, std::int32_t* xyz) {
  for (std::size_t i = 0; i < c.size(); ++i) {
    xyz[3 * i] = c[i].x;
    xyz[3 * i + 1] = c[i].y;
    xyz[3 * i + 2] = c[i].z;
  }
}
PointCloud to_cloud(const std::int32_t* xyz, std::int64_t n, int sorted, const float* f, std::int64_t C) {
  PointCloud pc;
  pc.coords = make_coords(to_coords(xyz, n));
  pc.sorted = sorted != 0;
  if (f && C > 0) {
    pc.features = Matrix(n, C);
    std::memcpy(pc.features.row(0), f, sizeof(float) * static_cast<std::size_t>(n * C));
  } else {
    pc.features = Matrix(n, 0);
  }
  return pc;
}
LayerGeometry to_geometry(int K, int offset_scale, int out_stride, int transposed, const std::int32_t* target,
                          std::int64_t ntarget) {
  LayerGeometry g;
  g.kernel_size = K;
  g.offset_scale = offset_scale;
  g.out_stride = out_stride;
  g.transposed = transposed != 0;
  if (g.transposed) g.target = make_coords(to_coords(target, ntarget));
  return g;
}
LayerConfig to_config(int backend, int policy, double eps, int max_batch, int Tg, int Ts, int B, int C, int workers) {
  LayerConfig cfg;
  cfg.backend = static_cast<MapBackend>(backend);
  cfg.policy = static_cast<GroupPolicy>(policy);
  cfg.epsilon = eps;
  cfg.max_batch = max_batch;
  cfg.gather_tile = Tg;
  cfg.scatter_tile = Ts;
  cfg.B = B;
  cfg.C = C;
  cfg.workers = workers;
  return cfg;
}
}  // namespace

struct so_map {
  KernelMap map;
  CoordsPtr q;
  SearchCounters counters;
};

extern "C" {

const char* so_last_error() { return g_err.c_str(); }

int so_pack_keys(const std::int32_t* xyz, std::int64_t n, std::uint64_t* keys) {
  return guarded([&] {
    for (std::int64_t i = 0; i < n; ++i) keys[i] = pack_key({xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]});
  });
}

int so_unpack_keys(const std::uint64_t* keys, std::int64_t n, std::int32_t* xyz) {
  return guarded([&] {
    for (std::int64_t i = 0; i < n; ++i) {
      const Coordinate c = unpack_key(keys[i]);
      xyz[3 * i] = c.x;
      xyz[3 * i + 1] = c.y;
      xyz[3 * i + 2] = c.z;
    }
  });
}

int so_saturating_pack(const std::int64_t* xyz, std::int64_t n, std::uint64_t* out) {
  return guarded([&] {
    for (std::int64_t i = 0; i < n; ++i) out[i] = saturating_pack(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
  });
}

int so_weight_offsets(int K, int s, int ext, std::int32_t* out, std::int64_t* count) {
  return guarded([&] {
    const OffsetSet o = ext ? weight_offsets_ext(K, s) : weight_offsets(K, s);
    *count = o.count();
    if (out) from_coords(o.offsets, out);
  });
}

int so_generate_output_coords(const std::int32_t* xyz, std::int64_t n, int sorted, int s, std::int32_t* out,
                              std::int64_t* n_out, int* out_sorted, int* aliased) {
  return guarded([&] {
    PointCloud in;
    in.coords = make_coords(to_coords(xyz, n));
    in.sorted = sorted != 0;
    const PointCloud q = generate_output_coords(in, s);
    *n_out = q.size();
    *out_sorted = q.sorted ? 1 : 0;
    *aliased = q.coords == in.coords ? 1 : 0;
    from_coords(*q.coords, out);
  });
}

int so_voxelize(const double* pts, std::int64_t n, const float* f, std::int64_t C, double res, std::int32_t* out_xyz,
                float* out_f, std::int64_t* n_out) {
  return guarded([&] {
    std::vector<std::array<double, 3>> p(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) p[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    Matrix F;
    if (C > 0) {
      F = Matrix(n, C);
      if (n > 0) std::memcpy(F.row(0), f, sizeof(float) * static_cast<std::size_t>(n * C));
    }
    const PointCloud v = voxelize(p, F, res);
    *n_out = v.size();
    from_coords(*v.coords, out_xyz);
    if (C > 0 && v.size() > 0) std::memcpy(out_f, v.features.row(0), sizeof(float) * static_cast<std::size_t>(v.size() * C));
  });
}

std::uint64_t so_stream_seed(std::uint64_t seed, std::uint64_t idx) { return stream_seed(seed, idx); }

// kind 0: next() as u64; 1: next_unit() as f64; 2: next_below(bound) as u64.
int so_rng_draw(std::uint64_t seed, std::int64_t n, int kind, std::uint64_t bound, void* out) {
  return guarded([&] {
    Rng r(seed);
    for (std::int64_t i = 0; i < n; ++i) {
      if (kind == 1)
        static_cast<double*>(out)[i] = r.next_unit();
      else if (kind == 2)
        static_cast<std::uint64_t*>(out)[i] = r.next_below(bound);
      else
        static_cast<std::uint64_t*>(out)[i] = r.next();
    }
  });
}

int so_generate_synthetic(std::int64_t N, std::int64_t E, std::int64_t C, std::uint64_t seed, std::int32_t* xyz,
                          float* feats) {
  return guarded([&] {
    const PointCloud pc = generate_synthetic(N, E, C, seed);
    from_coords(*pc.coords, xyz);
    if (C > 0 && N > 0) std::memcpy(feats, pc.features.row(0), sizeof(float) * static_cast<std::size_t>(N * C));
  });
}

int so_generate_weights(std::uint64_t seed, std::uint64_t stream, int K3, int Cin, int Cout, float* w) {
  return guarded([&] {
    const WeightSet ws = generate_weights(seed, stream, K3, Cin, Cout);
    std::memcpy(w, ws.w.data(), sizeof(float) * ws.w.size());
  });
}

// Generic map over explicit offsets. q == nullptr means Q aliases P (sorted backend only).
int so_map_build(const std::int32_t* p, std::int64_t np, int p_sorted, const std::int32_t* q, std::int64_t nq,
                 const std::int32_t* offs, int nk, int backend, int B, int C, int workers, so_map** out,
                 std::uint64_t* counters5) {
  return guarded([&] {
    auto m = std::make_unique<so_map>();
    PointCloud P;
    P.coords = make_coords(to_coords(p, np));
    P.sorted = p_sorted != 0;
    const CoordList offsets = to_coords(offs, nk);
    if (q == nullptr) {
      if (backend != 0) throw std::invalid_argument("alias queries need the sorted backend");
      const SortedSource src = build_source_array(P, B, &m->counters);
      m->map = build_kernel_map_sorted_keys(src, src.keys, offsets, C, workers, &m->counters);
      CoordList qs(src.keys.size());
      for (std::size_t i = 0; i < qs.size(); ++i) qs[i] = unpack_key(src.keys[i]);
      m->q = make_coords(std::move(qs));
    } else {
      m->q = make_coords(to_coords(q, nq));
      if (backend == 2) {
        m->map = brute_force_map(*P.coords, *m->q, offsets);
      } else if (backend == 1) {
        m->map = query_hash_map(build_hash_index(*P.coords), *m->q, offsets);
      } else {
        const SortedSource src = build_source_array(P, B, &m->counters);
        const auto qk = pack_all(*m->q);
        for (std::size_t i = 1; i < qk.size(); ++i)
          if (qk[i - 1] >= qk[i]) throw std::invalid_argument("query coordinates must be sorted and unique");
        m->map = build_kernel_map_sorted_keys(src, qk, offsets, C, workers, &m->counters);
      }
    }
    if (counters5) {
      counters5[0] = m->counters.backward_comparisons;
      counters5[1] = m->counters.forward_comparisons;
      counters5[2] = m->counters.source_elements_loaded;
      counters5[3] = m->counters.queries_executed;
      counters5[4] = m->counters.sorts;
    }
    *out = m.release();
  });
}

// Layer-level map: computes Q from the layer geometry like sc_layer_forward_ext.
int so_layer_map(const std::int32_t* p, std::int64_t np, int p_sorted, int K, int offset_scale, int out_stride,
                 int transposed, const std::int32_t* target, std::int64_t ntarget, int backend, int B, int C,
                 int workers, so_map** out, std::uint64_t* counters5) {
  return guarded([&] {
    auto m = std::make_unique<so_map>();
    PointCloud P;
    P.coords = make_coords(to_coords(p, np));
    P.sorted = p_sorted != 0;
    const LayerGeometry g = to_geometry(K, offset_scale, out_stride, transposed, target, ntarget);
    // Q's own sort counts only for Eq. 1 (stride > 1); the sort of P that a stride-1 Q reuses is
    // counted once, by build_layer_map's source array (one array sorted)
    SearchCounters qc;
    PointCloud Q = g.transposed ? PointCloud{g.target, Matrix{}, true} : layer_output_coords(P, out_stride, &qc);
    if (!g.transposed && out_stride != 1) ++m->counters.sorts;
    LayerConfig cfg = to_config(backend, 1, 0.25, 16, 0, 0, B, C, workers);
    m->map = build_layer_map(P, Q, g, cfg, &m->counters);
    m->q = Q.coords;
    if (counters5) {
      counters5[0] = m->counters.backward_comparisons;
      counters5[1] = m->counters.forward_comparisons;
      counters5[2] = m->counters.source_elements_loaded;
      counters5[3] = m->counters.queries_executed;
      counters5[4] = m->counters.sorts;
    }
    *out = m.release();
  });
}

std::int64_t so_map_nq(const so_map* m) { return static_cast<std::int64_t>(m->q->size()); }
int so_map_nk(const so_map* m) { return static_cast<int>(m->map.matches.size()); }
std::int64_t so_map_total(const so_map* m) { return m->map.total(); }
int so_map_q(const so_map* m, std::int32_t* xyz) {
  return guarded([&] { from_coords(*m->q, xyz); });
}
int so_map_read(const so_map* m, std::int64_t* sizes, std::int32_t* in_idx, std::int32_t* out_idx) {
  return guarded([&] {
    std::int64_t pos = 0;
    for (std::size_t k = 0; k < m->map.matches.size(); ++k) {
      sizes[k] = static_cast<std::int64_t>(m->map.matches[k].size());
      for (const Pair& pr : m->map.matches[k]) {
        in_idx[pos] = pr.first;
        out_idx[pos] = pr.second;
        ++pos;
      }
    }
  });
}
void so_map_free(so_map* m) { delete m; }

int so_group_gemms(const std::int64_t* sizes, int n, int policy, double eps, int max_batch, int* order, int* n_order,
                   int* group_begin, int* group_end, std::int64_t* heights, int* n_groups, std::int64_t* buffer_offsets,
                   std::int64_t* buffer_length, double* overhead) {
  return guarded([&] {
    const GemmGroupPlan plan =
        group_gemms(std::vector<std::int64_t>(sizes, sizes + n), static_cast<GroupPolicy>(policy), eps, max_batch);
    *n_order = static_cast<int>(plan.offset_order.size());
    for (std::size_t i = 0; i < plan.offset_order.size(); ++i) order[i] = plan.offset_order[i];
    *n_groups = static_cast<int>(plan.groups.size());
    for (std::size_t g = 0; g < plan.groups.size(); ++g) {
      group_begin[g] = plan.groups[g].begin;
      group_end[g] = plan.groups[g].end;
      heights[g] = plan.groups[g].padded_height;
    }
    for (int k = 0; k < n; ++k) buffer_offsets[k] = plan.buffer_offsets[k];
    *buffer_length = plan.buffer_length;
    *overhead = plan.real_rows() > 0 ? padding_overhead(plan) : -1.0;
  });
}

// stats[10] = matches, buffer_length, groups, padding_overhead, imt_lookups, sorts,
//             ms_map, ms_gather, ms_gemm, ms_scatter
int so_layer_forward(const std::int32_t* xyz, std::int64_t n, int sorted, const float* f, int Cin, const float* w,
                     int Cout, int K, int offset_scale, int out_stride, int transposed, const std::int32_t* target,
                     std::int64_t ntarget, int backend, int policy, double eps, int max_batch, int Tg, int Ts, int B,
                     int C, int workers, std::int32_t* out_xyz, float* out_f, std::int64_t* n_out, double* stats) {
  return guarded([&] {
    const PointCloud cloud = to_cloud(xyz, n, sorted, f, Cin);
    const LayerGeometry g = to_geometry(K, offset_scale, out_stride, transposed, target, ntarget);
    WeightSet ws;
    ws.num_offsets = static_cast<int>(weight_offsets_ext(K, offset_scale).offsets.size());
    ws.c_in = Cin;
    ws.c_out = Cout;
    ws.w.assign(w, w + static_cast<std::size_t>(ws.num_offsets) * Cin * Cout);
    LayerStats st;
    const PointCloud out = sc_layer_forward_ext(cloud, ws, g, to_config(backend, policy, eps, max_batch, Tg, Ts, B, C, workers), &st);
    *n_out = out.size();
    if (out_xyz) from_coords(*out.coords, out_xyz);
    if (out_f && out.size() > 0 && Cout > 0)
      std::memcpy(out_f, out.features.row(0), sizeof(float) * static_cast<std::size_t>(out.size() * Cout));
    if (stats) {
      const double v[10] = {static_cast<double>(st.matches), static_cast<double>(st.buffer_length),
                            static_cast<double>(st.groups), st.padding_overhead,
                            static_cast<double>(st.imt_lookups), static_cast<double>(st.counters.sorts),
                            st.ms_map, st.ms_gather, st.ms_gemm, st.ms_scatter};
      std::memcpy(stats, v, sizeof(v));
    }
  });
}

int so_dense_conv(const std::int32_t* xyz, std::int64_t n, int sorted, const float* f, int Cin, const float* w, int Cout,
                  int K, int offset_scale, int out_stride, int transposed, const std::int32_t* target,
                  std::int64_t ntarget, float* out_f, std::int64_t* n_out) {
  return guarded([&] {
    const PointCloud cloud = to_cloud(xyz, n, sorted, f, Cin);
    const LayerGeometry g = to_geometry(K, offset_scale, out_stride, transposed, target, ntarget);
    WeightSet ws;
    ws.num_offsets = static_cast<int>(weight_offsets_ext(K, offset_scale).offsets.size());
    ws.c_in = Cin;
    ws.c_out = Cout;
    ws.w.assign(w, w + static_cast<std::size_t>(ws.num_offsets) * Cin * Cout);
    const Matrix out = dense_conv_oracle_ext(cloud, ws, g);
    *n_out = out.rows();
    if (out.rows() > 0 && Cout > 0)
      std::memcpy(out_f, out.row(0), sizeof(float) * static_cast<std::size_t>(out.rows() * Cout));
  });
}

// layers: L x (K, s, c_in, c_out). Output arrays sized by the caller to n points.
int so_forward_network(const int* layers, int L, const std::int32_t* xyz, std::int64_t n, int sorted, const float* f,
                       std::uint64_t seed, int backend, int workers, std::int32_t* out_xyz, float* out_f,
                       std::int64_t* n_out, std::uint64_t* sorts) {
  return guarded([&] {
    NetworkSpec spec;
    for (int l = 0; l < L; ++l) spec.layers.push_back({layers[4 * l], layers[4 * l + 1], layers[4 * l + 2], layers[4 * l + 3]});
    const PointCloud cloud = to_cloud(xyz, n, sorted, f, spec.layers.empty() ? 0 : spec.layers[0].c_in);
    LayerConfig cfg;
    cfg.backend = static_cast<MapBackend>(backend);
    cfg.workers = workers;
    const NetworkResult r = forward_network(spec, cloud, cfg, seed);
    *n_out = r.output.size();
    *sorts = r.sorts;
    from_coords(*r.output.coords, out_xyz);
    const std::int64_t C = r.output.channels();
    if (r.output.size() > 0 && C > 0)
      std::memcpy(out_f, r.output.features.row(0), sizeof(float) * static_cast<std::size_t>(r.output.size() * C));
  });
}

int so_candidate_tiles(int channels, int* out, int* n) {
  return guarded([&] {
    const auto t = candidate_tiles(channels);
    *n = static_cast<int>(t.size());
    for (std::size_t i = 0; i < t.size(); ++i) out[i] = t[i];
  });
}

int so_theoretical_hyperparams(std::int64_t P, std::int64_t Q, int* B, int* C) {
  return guarded([&] {
    const auto bc = theoretical_hyperparams(P, Q);
    *B = bc.first;
    *C = bc.second;
  });
}

}  // extern "C"

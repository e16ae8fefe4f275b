// TEST INFRASTRUCTURE — CPU oracle (see geometry_compat.hpp header). Never linked by
// the product library; tests, smoke() and bench.py's CPU-baseline leg only.
//
// A C++ restatement of the reference's SPEC modules that sit on the SC hot path:
//   kernelmap_baseline  SPEC.md:103-164   brute force + open-addressing hash map
//   kernelmap_sorted    SPEC.md:166-275   segmented sorting, double-traversed search
//   execution           SPEC.md:277-401   grouping, metadata tables, gather/GEMM/scatter
//   autotune            SPEC.md:403-459   candidate tiles, median profiling, Alg. 2
//   netdef              SPEC.md:514-548   sequential chain with sort reuse
//   cli gen             SPEC.md:562-570   synthetic clouds
// plus the SURVEY §2.2 extensions (even K, transposed maps, tensor strides).
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <utility>
#include <vector>

#include "geometry_compat.hpp"

namespace sconv::oracle {

using Pair = std::pair<std::int32_t, std::int32_t>;  // (input index j, output index i)

// SPEC.md:108-113. matches[k] sorted by output index i.
struct KernelMap {
  CoordList offsets;
  std::vector<std::vector<Pair>> matches;
  std::int64_t total() const;
  bool operator==(const KernelMap& o) const { return offsets == o.offsets && matches == o.matches; }
};

// SPEC.md:183-187 (+ sort counter).
struct SearchCounters {
  std::uint64_t backward_comparisons = 0;
  std::uint64_t forward_comparisons = 0;
  std::uint64_t source_elements_loaded = 0;
  std::uint64_t queries_executed = 0;
  std::uint64_t sorts = 0;
  void add(const SearchCounters& o);
};

// ---- geometry extensions ----
// Odd K: reference weight_offsets(K, scale). Even K: t in [0, K-1] per axis, scaled.
OffsetSet weight_offsets_ext(int kernel_size, int scale);

// Monotone 64-bit key of an unbounded triple: equals pack_key when in range, never
// equals a valid key otherwise, and is non-decreasing in lexicographic order. Fixes
// the SPEC sentinel's non-monotonicity at the range edges.
PackedKey saturating_pack(std::int64_t x, std::int64_t y, std::int64_t z);

// ---- kernelmap_baseline ----
KernelMap brute_force_map(const CoordList& P, const CoordList& Q, const CoordList& offsets);

struct HashIndex {
  std::uint64_t capacity = 1;
  int log2_capacity = 0;
  std::vector<PackedKey> keys;  // empty slot = ~0
  std::vector<std::int32_t> values;
  std::int64_t max_probe = 0;
  std::int64_t lookup(PackedKey key, std::int64_t* probes = nullptr) const;
};
HashIndex build_hash_index(const CoordList& P);
KernelMap query_hash_map(const HashIndex& index, const CoordList& Q, const CoordList& offsets);

// ---- kernelmap_sorted ----
struct SortedSource {
  std::vector<PackedKey> keys;        // strictly increasing
  std::vector<std::int32_t> indices;  // original input index per sorted position
  int block_size = 256;
  std::vector<PackedKey> block_pivots;
  std::int64_t num_blocks() const { return static_cast<std::int64_t>(block_pivots.size()); }
};
SortedSource build_source_array(const PointCloud& P, int B, SearchCounters* counters);

// key of q_i + delta_k computed on the fly; qkeys sorted.
PackedKey segment_query_key(const std::vector<PackedKey>& qkeys, std::int64_t i, const Coordinate& delta);

// boundary[b] = first query position whose segment key > pivot_b.
std::vector<std::int64_t> backward_partition(const SortedSource& src, const std::vector<PackedKey>& qkeys,
                                             const Coordinate& delta, SearchCounters* counters);

struct QueryRange {
  std::int64_t block;  // source block index
  std::int64_t lo, hi; // [lo, hi) query positions
};
// split blocks longer than C into ceil(L/C) near-equal ranges, first larger.
std::vector<QueryRange> balance_blocks(const std::vector<std::int64_t>& boundaries, int C);

// SPEC.md:226-234. Appends (j, i) for hits in query order.
void forward_block_search(const SortedSource& src, const QueryRange& range, const std::vector<PackedKey>& qkeys,
                          const Coordinate& delta, std::vector<Pair>* out, SearchCounters* counters);

// Core: the query set is a sorted key array (Q), possibly the source keys themselves.
KernelMap build_kernel_map_sorted_keys(const SortedSource& src, const std::vector<PackedKey>& qkeys,
                                       const CoordList& offsets, int C, int workers, SearchCounters* counters);
// SPEC.md:235-243 signature. Q must be sorted; if Q aliases P.coords the source
// array doubles as the query array (one sort at most).
std::pair<KernelMap, SearchCounters> build_kernel_map_sorted(const PointCloud& P, const CoordsPtr& Q,
                                                             const OffsetSet& offsets, int B, int C,
                                                             int workers = 1);

// SPEC.md:244-252.
std::pair<int, int> theoretical_hyperparams(std::int64_t P, std::int64_t Q);

// ---- execution ----
enum class GroupPolicy { MapOrder = 0, Sorted = 1 };
enum class MapBackend { Sorted = 0, Hash = 1, Brute = 2 };

struct GemmGroup {
  int begin = 0, end = 0;          // range over offset_order
  std::int64_t padded_height = 0;  // max size in the group
};
struct GemmGroupPlan {
  std::vector<int> offset_order;            // chosen order, offsets with n_k = 0 removed
  std::vector<std::int64_t> sizes;          // n_k for every offset k
  std::vector<GemmGroup> groups;            // tile offset_order
  std::vector<std::int64_t> buffer_offsets; // per offset; -1 when n_k = 0
  std::int64_t buffer_length = 0;
  std::int64_t real_rows() const;
};
GemmGroupPlan group_gemms(const std::vector<std::int64_t>& sizes, GroupPolicy policy, double epsilon, int max_batch);
double padding_overhead(const GemmGroupPlan& plan);  // throws std::domain_error when y = 0

struct MetadataTables {
  std::int64_t buffer_length = 0;
  int num_offsets = 0;
  std::int64_t num_inputs = 0, num_outputs = 0;
  std::vector<std::int64_t> imt;  // [j * K + k] -> slot or -1
  std::vector<std::int64_t> omt;  // [i * K + k] -> slot or -1
};
MetadataTables build_metadata_tables(const KernelMap& map, const GemmGroupPlan& plan, std::int64_t num_inputs,
                                     std::int64_t num_outputs);

struct WeightSet {
  int num_offsets = 0, c_in = 0, c_out = 0;
  std::vector<float> w;  // [k][c_in][c_out]
  const float* matrix(int k) const { return w.data() + static_cast<std::size_t>(k) * c_in * c_out; }
};

// Alg. 1. counter += IMT lookups = (C_in/T) * |M|.
Matrix gather(const Matrix& features, const MetadataTables& t, int tile, std::uint64_t* imt_lookups, int workers = 1);
// fp64 accumulate, fp32 store. width = parallel groups.
Matrix gemm_execute(const Matrix& in_buffer, const WeightSet& w, const GemmGroupPlan& plan, int width = 4);
// Ascending-k fp64 reduction.
Matrix scatter(const Matrix& out_buffer, const MetadataTables& t, int tile, int workers = 1);

struct LayerConfig {
  MapBackend backend = MapBackend::Sorted;
  GroupPolicy policy = GroupPolicy::Sorted;
  double epsilon = 0.25;
  int max_batch = 16;
  int gather_tile = 0;   // 0 -> C_in
  int scatter_tile = 0;  // 0 -> C_out
  int B = 256, C = 512;
  int workers = 1;
};

struct LayerStats {
  SearchCounters counters;
  std::int64_t matches = 0;
  std::int64_t buffer_length = 0;
  std::int64_t groups = 0;
  double padding_overhead = 0.0;
  std::uint64_t imt_lookups = 0;
  std::vector<std::int64_t> sizes;
  double ms_map = 0, ms_gather = 0, ms_gemm = 0, ms_scatter = 0;
};

// General layer geometry. SPEC-literal sc_layer_forward(K, s) is {K, s, s, false}.
struct LayerGeometry {
  int kernel_size = 3;
  int offset_scale = 1;  // offsets = weight_offsets_ext(K, offset_scale)
  int out_stride = 1;    // Eq. 1 stride for Q (ignored when transposed)
  bool transposed = false;
  CoordsPtr target;      // transposed: output coordinates (sorted)
};

// Q for a layer: sorted output coordinates + whether Q aliases P (stride 1, P sorted).
PointCloud layer_output_coords(const PointCloud& P, int out_stride, SearchCounters* counters);

// Map for a layer (any backend), canonical order.
KernelMap build_layer_map(const PointCloud& P, const PointCloud& Q, const LayerGeometry& g, const LayerConfig& cfg,
                          SearchCounters* counters);

PointCloud sc_layer_forward_ext(const PointCloud& cloud, const WeightSet& w, const LayerGeometry& g,
                                const LayerConfig& cfg, LayerStats* stats = nullptr);
// SPEC.md:359-367.
PointCloud sc_layer_forward(const PointCloud& cloud, const WeightSet& w, int K, int s, const LayerConfig& cfg,
                            LayerStats* stats = nullptr);
// direct Eq. 2, fp64, ascending k. Output rows follow Q order.
Matrix dense_conv_oracle(const PointCloud& cloud, const WeightSet& w, int K, int s);
Matrix dense_conv_oracle_ext(const PointCloud& cloud, const WeightSet& w, const LayerGeometry& g);

// ---- autotune ----
std::vector<int> candidate_tiles(int channels);
double profile_candidate(const std::function<void()>& run, int rounds);  // median seconds
struct TunedLayerConfig {
  int layer = 0, gather_tile = 1, scatter_tile = 1;
  std::vector<std::pair<int, double>> gather_latency, scatter_latency;
};
// argmin with smallest-tile tie break over a cost function (used with a mocked timer).
int select_tile(const std::vector<std::pair<int, double>>& latencies);

// ---- netdef ----
struct NetLayer {
  int K = 3, s = 1, c_in = 0, c_out = 0;
};
struct NetworkSpec {
  std::vector<NetLayer> layers;
};
NetworkSpec preset_network(const std::string& name);
WeightSet generate_weights(std::uint64_t seed, std::uint64_t stream, int num_offsets, int c_in, int c_out);
struct NetworkResult {
  PointCloud output;
  std::uint64_t sorts = 0;
  std::vector<LayerStats> layers;
};
NetworkResult forward_network(const NetworkSpec& spec, const PointCloud& cloud, const LayerConfig& cfg,
                              std::uint64_t seed);

// ---- cli gen ----
// N unique coordinates uniform in [0,E)^3 from Rng(stream_seed(seed,0)), x,y,z order,
// duplicates rejected; then N x C features U[0,1) from the same stream.
PointCloud generate_synthetic(std::int64_t N, std::int64_t E, std::int64_t C, std::uint64_t seed);

// Utility: sorted keys of a coordinate list (throws like pack_key).
std::vector<PackedKey> pack_all(const CoordList& c);

}  // namespace sconv::oracle

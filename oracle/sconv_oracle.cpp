// TEST INFRASTRUCTURE — CPU oracle. See sconv_oracle.hpp for the SPEC map.
#include "sconv_oracle.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <thread>
#include <unordered_map>
#include <unordered_set>

namespace sconv::oracle {
namespace {

// Deterministic static partition of [0, n) over `workers` threads.
template <class Fn>
void parallel_for(std::int64_t n, int workers, Fn&& fn) {
  if (workers <= 1 || n <= 1) {
    for (std::int64_t i = 0; i < n; ++i) fn(i, 0);
    return;
  }
  const int w = static_cast<int>(std::min<std::int64_t>(workers, n));
  std::vector<std::thread> pool;
  for (int t = 0; t < w; ++t)
    pool.emplace_back([&, t] {
      for (std::int64_t i = t; i < n; i += w) fn(i, t);
    });
  for (auto& th : pool) th.join();
}

// Dynamic partition (atomic work counter) for items whose results do not depend on which
// thread runs them: load balance only, outputs unchanged.
template <class Fn>
void parallel_for_chunked(std::int64_t n, int workers, Fn&& fn) {
  if (workers <= 1 || n <= 1) {
    for (std::int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<std::int64_t> next{0};
  const int w = static_cast<int>(std::min<std::int64_t>(workers, n));
  std::vector<std::thread> pool;
  for (int t = 0; t < w; ++t)
    pool.emplace_back([&] {
      for (std::int64_t i; (i = next.fetch_add(1, std::memory_order_relaxed)) < n;) fn(i);
    });
  for (auto& th : pool) th.join();
}

std::int64_t ceil_log2_plus1(std::int64_t n) {  // ceil(log2(n + 1))
  std::int64_t b = 0;
  while ((std::int64_t{1} << b) < n + 1) ++b;
  return b;
}

}  // namespace

std::int64_t KernelMap::total() const {
  std::int64_t t = 0;
  for (const auto& m : matches) t += static_cast<std::int64_t>(m.size());
  return t;
}

void SearchCounters::add(const SearchCounters& o) {
  backward_comparisons += o.backward_comparisons;
  forward_comparisons += o.forward_comparisons;
  source_elements_loaded += o.source_elements_loaded;
  queries_executed += o.queries_executed;
  sorts += o.sorts;
}

std::vector<PackedKey> pack_all(const CoordList& c) {
  std::vector<PackedKey> k(c.size());
  for (std::size_t i = 0; i < c.size(); ++i) k[i] = pack_key(c[i]);
  return k;
}

OffsetSet weight_offsets_ext(int kernel_size, int scale) {
  if (kernel_size % 2 == 1) return weight_offsets(kernel_size, scale);
  if (kernel_size < 1) throw std::invalid_argument("kernel size must be a positive integer");
  if (scale < 1) throw std::invalid_argument("stride must be positive");
  check_component(static_cast<std::int64_t>(kernel_size - 1) * scale, 'x');
  OffsetSet set;
  set.kernel_size = kernel_size;
  set.stride = scale;
  for (int a = 0; a < kernel_size; ++a)
    for (int b = 0; b < kernel_size; ++b)
      for (int c = 0; c < kernel_size; ++c) set.offsets.push_back({a * scale, b * scale, c * scale});
  return set;
}

PackedKey saturating_pack(std::int64_t x, std::int64_t y, std::int64_t z) {
  // Field value 0 is never produced by a valid coordinate (biased range [1, 2^21-1]),
  // so out-of-range components land strictly between the valid neighbours.
  if (x > COORD_MAX) return PackedKey{1} << 63;
  if (x < COORD_MIN) return 0;
  const std::uint64_t X = static_cast<std::uint64_t>(x + COORD_BIAS);
  if (y > COORD_MAX) return (X + 1) << 42;
  if (y < COORD_MIN) return X << 42;
  const std::uint64_t Y = static_cast<std::uint64_t>(y + COORD_BIAS);
  if (z > COORD_MAX) return (X << 42) + ((Y + 1) << 21);
  if (z < COORD_MIN) return (X << 42) + (Y << 21);
  return (X << 42) | (Y << 21) | static_cast<std::uint64_t>(z + COORD_BIAS);
}

// ---------------------------------------------------------------- baseline maps
KernelMap brute_force_map(const CoordList& P, const CoordList& Q, const CoordList& offsets) {
  KernelMap m;
  m.offsets = offsets;
  m.matches.resize(offsets.size());
  for (std::size_t k = 0; k < offsets.size(); ++k) {
    const Coordinate& d = offsets[k];
    for (std::size_t i = 0; i < Q.size(); ++i) {
      const std::int64_t x = std::int64_t{Q[i].x} + d.x, y = std::int64_t{Q[i].y} + d.y,
                         z = std::int64_t{Q[i].z} + d.z;
      for (std::size_t j = 0; j < P.size(); ++j)
        if (P[j].x == x && P[j].y == y && P[j].z == z)
          m.matches[k].emplace_back(static_cast<std::int32_t>(j), static_cast<std::int32_t>(i));
    }
  }
  return m;
}

std::int64_t HashIndex::lookup(PackedKey key, std::int64_t* probes) const {
  const std::uint64_t mask = capacity - 1;
  std::uint64_t s = log2_capacity == 0 ? 0 : (key * 0x9E3779B97F4A7C15ull) >> (64 - log2_capacity);
  std::int64_t n = 0;
  for (;;) {
    ++n;
    if (keys[s] == key) {
      if (probes) *probes = n;
      return values[s];
    }
    if (keys[s] == ~PackedKey{0}) {
      if (probes) *probes = n;
      return -1;
    }
    s = (s + 1) & mask;
  }
}

HashIndex build_hash_index(const CoordList& P) {
  HashIndex h;
  while (h.capacity < 2 * P.size()) {
    h.capacity <<= 1;
    ++h.log2_capacity;
  }
  h.keys.assign(h.capacity, ~PackedKey{0});
  h.values.assign(h.capacity, -1);
  const std::uint64_t mask = h.capacity - 1;
  for (std::size_t j = 0; j < P.size(); ++j) {
    const PackedKey key = pack_key(P[j]);
    std::uint64_t s = h.log2_capacity == 0 ? 0 : (key * 0x9E3779B97F4A7C15ull) >> (64 - h.log2_capacity);
    std::int64_t probe = 1;
    while (h.keys[s] != ~PackedKey{0} && h.keys[s] != key) {
      s = (s + 1) & mask;
      ++probe;
    }
    h.keys[s] = key;
    h.values[s] = static_cast<std::int32_t>(j);
    h.max_probe = std::max(h.max_probe, probe);
  }
  return h;
}

KernelMap query_hash_map(const HashIndex& index, const CoordList& Q, const CoordList& offsets) {
  KernelMap m;
  m.offsets = offsets;
  m.matches.resize(offsets.size());
  for (std::size_t k = 0; k < offsets.size(); ++k)
    for (std::size_t i = 0; i < Q.size(); ++i) {
      const std::int64_t x = std::int64_t{Q[i].x} + offsets[k].x, y = std::int64_t{Q[i].y} + offsets[k].y,
                         z = std::int64_t{Q[i].z} + offsets[k].z;
      if (!component_in_range(x) || !component_in_range(y) || !component_in_range(z)) continue;
      const std::int64_t j = index.lookup(pack_key({static_cast<std::int32_t>(x), static_cast<std::int32_t>(y),
                                                    static_cast<std::int32_t>(z)}));
      if (j >= 0) m.matches[k].emplace_back(static_cast<std::int32_t>(j), static_cast<std::int32_t>(i));
    }
  return m;
}

// ---------------------------------------------------------------- sorted map
SortedSource build_source_array(const PointCloud& P, int B, SearchCounters* counters) {
  if (B < 1) throw std::invalid_argument("block size must be positive");
  SortedSource s;
  s.block_size = B;
  const CoordList& c = *P.coords;
  std::vector<std::pair<PackedKey, std::int32_t>> kv(c.size());
  for (std::size_t j = 0; j < c.size(); ++j) kv[j] = {pack_key(c[j]), static_cast<std::int32_t>(j)};
  if (!P.sorted) {
    std::sort(kv.begin(), kv.end());
    if (counters) ++counters->sorts;
  }
  s.keys.resize(kv.size());
  s.indices.resize(kv.size());
  for (std::size_t j = 0; j < kv.size(); ++j) {
    s.keys[j] = kv[j].first;
    s.indices[j] = kv[j].second;
  }
  for (std::size_t b = 0; b * B < kv.size(); ++b)
    s.block_pivots.push_back(s.keys[std::min(kv.size(), (b + 1) * B) - 1]);
  return s;
}

PackedKey segment_query_key(const std::vector<PackedKey>& qkeys, std::int64_t i, const Coordinate& d) {
  const Coordinate q = unpack_key(qkeys[static_cast<std::size_t>(i)]);
  return saturating_pack(std::int64_t{q.x} + d.x, std::int64_t{q.y} + d.y, std::int64_t{q.z} + d.z);
}

std::vector<std::int64_t> backward_partition(const SortedSource& src, const std::vector<PackedKey>& qkeys,
                                             const Coordinate& delta, SearchCounters* counters) {
  std::vector<std::int64_t> boundary(src.block_pivots.size());
  const auto nq = static_cast<std::int64_t>(qkeys.size());
  for (std::size_t b = 0; b < src.block_pivots.size(); ++b) {
    std::int64_t lo = 0, hi = nq, cmp = 0;
    while (lo < hi) {
      const std::int64_t mid = lo + (hi - lo) / 2;
      ++cmp;
      if (segment_query_key(qkeys, mid, delta) <= src.block_pivots[b])
        lo = mid + 1;
      else
        hi = mid;
    }
    boundary[b] = lo;
    if (counters) counters->backward_comparisons += static_cast<std::uint64_t>(cmp);
  }
  return boundary;
}

std::vector<QueryRange> balance_blocks(const std::vector<std::int64_t>& boundaries, int C) {
  if (C < 1) throw std::invalid_argument("query block size must be positive");
  std::vector<QueryRange> out;
  std::int64_t prev = 0;
  for (std::size_t b = 0; b < boundaries.size(); ++b) {
    const std::int64_t L = boundaries[b] - prev;
    if (L > 0) {
      const std::int64_t parts = (L + C - 1) / C, base = L / parts, extra = L % parts;
      std::int64_t lo = prev;
      for (std::int64_t p = 0; p < parts; ++p) {
        const std::int64_t len = base + (p < extra ? 1 : 0);
        out.push_back({static_cast<std::int64_t>(b), lo, lo + len});
        lo += len;
      }
    }
    prev = boundaries[b];
  }
  return out;
}

void forward_block_search(const SortedSource& src, const QueryRange& r, const std::vector<PackedKey>& qkeys,
                          const Coordinate& delta, std::vector<Pair>* out, SearchCounters* counters) {
  const std::int64_t begin = r.block * src.block_size;
  const std::int64_t end = std::min<std::int64_t>(begin + src.block_size, static_cast<std::int64_t>(src.keys.size()));
  // Worker-local copy of the block models the scratchpad staging.
  const std::vector<PackedKey> block(src.keys.begin() + begin, src.keys.begin() + end);
  std::uint64_t cmp = 0;
  for (std::int64_t i = r.lo; i < r.hi; ++i) {
    const PackedKey q = segment_query_key(qkeys, i, delta);
    std::int64_t lo = 0, hi = static_cast<std::int64_t>(block.size());
    while (lo < hi) {
      const std::int64_t mid = lo + (hi - lo) / 2;
      ++cmp;
      if (block[mid] == q) {
        out->emplace_back(src.indices[begin + mid], static_cast<std::int32_t>(i));
        break;
      }
      if (block[mid] < q)
        lo = mid + 1;
      else
        hi = mid;
    }
  }
  if (counters) {
    counters->forward_comparisons += cmp;
    counters->source_elements_loaded += static_cast<std::uint64_t>(end - begin);
    counters->queries_executed += static_cast<std::uint64_t>(r.hi - r.lo);
  }
}

KernelMap build_kernel_map_sorted_keys(const SortedSource& src, const std::vector<PackedKey>& qkeys,
                                       const CoordList& offsets, int C, int workers, SearchCounters* counters) {
  const auto K = static_cast<std::int64_t>(offsets.size());
  std::vector<std::vector<QueryRange>> ranges(K);
  std::vector<SearchCounters> wc(std::max(1, workers));
  parallel_for(K, workers, [&](std::int64_t k, int w) {
    ranges[k] = balance_blocks(backward_partition(src, qkeys, offsets[k], &wc[w]), C);
  });
  struct Item {
    std::int64_t k;
    std::size_t r;
  };
  std::vector<Item> items;
  for (std::int64_t k = 0; k < K; ++k)
    for (std::size_t r = 0; r < ranges[k].size(); ++r) items.push_back({k, r});
  std::vector<std::vector<Pair>> hits(items.size());
  parallel_for(static_cast<std::int64_t>(items.size()), workers, [&](std::int64_t t, int w) {
    forward_block_search(src, ranges[items[t].k][items[t].r], qkeys, offsets[items[t].k], &hits[t], &wc[w]);
  });
  KernelMap m;
  m.offsets = offsets;
  m.matches.resize(K);
  for (std::size_t t = 0; t < items.size(); ++t)  // deterministic merge in range order
    m.matches[items[t].k].insert(m.matches[items[t].k].end(), hits[t].begin(), hits[t].end());
  if (counters)
    for (const auto& c : wc) counters->add(c);
  return m;
}

std::pair<KernelMap, SearchCounters> build_kernel_map_sorted(const PointCloud& P, const CoordsPtr& Q,
                                                             const OffsetSet& offsets, int B, int C, int workers) {
  SearchCounters counters;
  const SortedSource src = build_source_array(P, B, &counters);
  if (Q == P.coords) {
    KernelMap m = build_kernel_map_sorted_keys(src, src.keys, offsets.offsets, C, workers, &counters);
    return {std::move(m), counters};
  }
  const std::vector<PackedKey> qkeys = pack_all(*Q);
  for (std::size_t i = 1; i < qkeys.size(); ++i)
    if (qkeys[i - 1] >= qkeys[i]) throw std::invalid_argument("query coordinates must be sorted and unique");
  KernelMap m = build_kernel_map_sorted_keys(src, qkeys, offsets.offsets, C, workers, &counters);
  return {std::move(m), counters};
}

std::pair<int, int> theoretical_hyperparams(std::int64_t P, std::int64_t Q) {
  if (P < 1 || Q < 1) throw std::invalid_argument("point counts must be positive");
  const double ratio = static_cast<double>(P) / static_cast<double>(Q);
  const int B = std::max(1, static_cast<int>(std::lround(ratio * std::log2(static_cast<double>(Q)))));
  const double lb = std::max(1.0, std::log2(static_cast<double>(B)));
  const int C = std::max(
      1, static_cast<int>(std::lround(std::sqrt(static_cast<double>(Q) / (static_cast<double>(P) * lb)) * B)));
  return {B, C};
}

// ---------------------------------------------------------------- execution
std::int64_t GemmGroupPlan::real_rows() const {
  std::int64_t y = 0;
  for (int k : offset_order) y += sizes[k];
  return y;
}

GemmGroupPlan group_gemms(const std::vector<std::int64_t>& sizes, GroupPolicy policy, double epsilon,
                          int max_batch) {
  if (epsilon < 0) throw std::invalid_argument("epsilon must be nonnegative");
  if (max_batch < 1) throw std::invalid_argument("max_batch must be positive");
  GemmGroupPlan plan;
  plan.sizes = sizes;
  std::vector<int> order(sizes.size());
  std::iota(order.begin(), order.end(), 0);
  if (policy == GroupPolicy::Sorted)
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sizes[a] < sizes[b]; });
  for (int k : order)
    if (sizes[k] > 0) plan.offset_order.push_back(k);
  std::int64_t gmax = 0, gsum = 0;
  for (int pos = 0; pos < static_cast<int>(plan.offset_order.size()); ++pos) {
    const std::int64_t n = sizes[plan.offset_order[pos]];
    bool extend = false;
    if (!plan.groups.empty()) {
      const GemmGroup& g = plan.groups.back();
      const std::int64_t card = g.end - g.begin;
      const std::int64_t nmax = std::max(gmax, n), nsum = gsum + n;
      const double pad = static_cast<double>((card + 1) * nmax - nsum) / static_cast<double>(nsum);
      extend = card < max_batch && pad <= epsilon;
    }
    if (extend) {
      plan.groups.back().end = pos + 1;
      gmax = std::max(gmax, n);
      gsum += n;
    } else {
      plan.groups.push_back({pos, pos + 1, 0});
      gmax = n;
      gsum = n;
    }
    plan.groups.back().padded_height = gmax;
  }
  plan.buffer_offsets.assign(sizes.size(), -1);
  std::int64_t base = 0;
  for (const GemmGroup& g : plan.groups) {
    for (int p = g.begin; p < g.end; ++p) plan.buffer_offsets[plan.offset_order[p]] = base + (p - g.begin) * g.padded_height;
    base += static_cast<std::int64_t>(g.end - g.begin) * g.padded_height;
  }
  plan.buffer_length = base;
  return plan;
}

double padding_overhead(const GemmGroupPlan& plan) {
  const std::int64_t y = plan.real_rows();
  if (y == 0) throw std::domain_error("padding overhead is undefined without real rows");
  return static_cast<double>(plan.buffer_length - y) / static_cast<double>(y);
}

MetadataTables build_metadata_tables(const KernelMap& map, const GemmGroupPlan& plan, std::int64_t num_inputs,
                                     std::int64_t num_outputs) {
  const int K = static_cast<int>(map.matches.size());
  if (static_cast<int>(plan.sizes.size()) != K) throw std::logic_error("metadata tables: plan/map offset mismatch");
  MetadataTables t;
  t.buffer_length = plan.buffer_length;
  t.num_offsets = K;
  t.num_inputs = num_inputs;
  t.num_outputs = num_outputs;
  t.imt.assign(static_cast<std::size_t>(num_inputs * K), -1);
  t.omt.assign(static_cast<std::size_t>(num_outputs * K), -1);
  for (int k = 0; k < K; ++k) {
    if (static_cast<std::int64_t>(map.matches[k].size()) != plan.sizes[k])
      throw std::logic_error("metadata tables: plan sizes do not match the kernel map");
    for (std::size_t r = 0; r < map.matches[k].size(); ++r) {
      const std::int64_t slot = plan.buffer_offsets[k] + static_cast<std::int64_t>(r);
      t.imt[static_cast<std::size_t>(map.matches[k][r].first) * K + k] = slot;
      t.omt[static_cast<std::size_t>(map.matches[k][r].second) * K + k] = slot;
    }
  }
  return t;
}

Matrix gather(const Matrix& F, const MetadataTables& t, int T, std::uint64_t* lookups, int workers) {
  const std::int64_t Cin = F.cols();
  if (T < 1 || Cin % T != 0) throw std::invalid_argument("tile size must divide the channel count");
  Matrix buf(t.buffer_length, Cin);
  const int K = t.num_offsets;
  std::atomic<std::uint64_t> count{0};
  const std::int64_t tiles = Cin / T;
  parallel_for(t.num_inputs, workers, [&](std::int64_t j, int) {
    std::uint64_t local = 0;
    std::vector<float> v(static_cast<std::size_t>(T));
    for (std::int64_t tt = 0; tt < tiles; ++tt) {  // Alg. 1 lines 1-7 per (tile, input)
      std::copy(F.row(j) + tt * T, F.row(j) + (tt + 1) * T, v.begin());
      for (int k = 0; k < K; ++k) {
        const std::int64_t s = t.imt[static_cast<std::size_t>(j) * K + k];
        if (s < 0) continue;
        ++local;
        std::copy(v.begin(), v.end(), buf.row(s) + tt * T);
      }
    }
    count += local;
  });
  if (lookups) *lookups += count.load();
  return buf;
}

Matrix gemm_execute(const Matrix& in, const WeightSet& w, const GemmGroupPlan& plan, int width) {
  if (in.cols() != w.c_in || in.rows() != plan.buffer_length)
    throw std::invalid_argument("gemm shape mismatch");
  Matrix out(in.rows(), w.c_out);
  // Work items: (group member k, block of kRows buffer rows); groups are independent
  // ("width"), and so are the row blocks of one member. Every output element is
  // the fp64 sum over c ascending of in(r, c) * W_k[c][n], whatever the loop
  // nesting, so this row-blocked form gives the same bits as a per-element dot product.
  constexpr std::int64_t kRows = 4;
  struct Item {
    int k;
    std::int64_t r0, r1;
  };
  std::vector<Item> items;
  for (const GemmGroup& g : plan.groups)
    for (int p = g.begin; p < g.end; ++p) {
      const int k = plan.offset_order[p];
      for (std::int64_t r = 0; r < g.padded_height; r += kRows)
        items.push_back({k, plan.buffer_offsets[k] + r,
                         plan.buffer_offsets[k] + std::min<std::int64_t>(g.padded_height, r + kRows)});
    }
  const int Cin = w.c_in, Cout = w.c_out;
  std::vector<double> wd(static_cast<std::size_t>(w.num_offsets) * Cin * Cout);
  for (std::size_t e = 0; e < wd.size(); ++e) wd[e] = static_cast<double>(w.w[e]);
  parallel_for_chunked(static_cast<std::int64_t>(items.size()), std::max(1, width), [&](std::int64_t t) {
    const Item& it = items[static_cast<std::size_t>(t)];
    const double* W = wd.data() + static_cast<std::size_t>(it.k) * Cin * Cout;
    const std::int64_t nr = it.r1 - it.r0;
    const float* rows[kRows];
    for (std::int64_t i = 0; i < kRows; ++i) rows[i] = in.row(it.r0 + std::min(i, nr - 1));
    int n0 = 0;
    for (; n0 + 8 <= Cout; n0 += 8) {  // 4 rows x 8 columns of fp64 accumulators in registers
      double a0[8] = {}, a1[8] = {}, a2[8] = {}, a3[8] = {};
      for (int c = 0; c < Cin; ++c) {
        const double* w8 = W + static_cast<std::size_t>(c) * Cout + n0;
        const double x0 = rows[0][c], x1 = rows[1][c], x2 = rows[2][c], x3 = rows[3][c];
        for (int q = 0; q < 8; ++q) {
          a0[q] += x0 * w8[q];
          a1[q] += x1 * w8[q];
          a2[q] += x2 * w8[q];
          a3[q] += x3 * w8[q];
        }
      }
      double* acc[kRows] = {a0, a1, a2, a3};
      for (std::int64_t i = 0; i < nr; ++i)
        for (int q = 0; q < 8; ++q) out(it.r0 + i, n0 + q) = static_cast<float>(acc[i][q]);
    }
    for (; n0 < Cout; ++n0)  // column tail
      for (std::int64_t i = 0; i < nr; ++i) {
        double a = 0.0;
        for (int c = 0; c < Cin; ++c) a += static_cast<double>(rows[i][c]) * W[static_cast<std::size_t>(c) * Cout + n0];
        out(it.r0 + i, n0) = static_cast<float>(a);
      }
  });
  return out;
}

Matrix scatter(const Matrix& ob, const MetadataTables& t, int T, int workers) {
  const std::int64_t Cout = ob.cols();
  if (T < 1 || Cout % T != 0) throw std::invalid_argument("tile size must divide the channel count");
  Matrix out(t.num_outputs, Cout);
  const int K = t.num_offsets;
  parallel_for(t.num_outputs, workers, [&](std::int64_t i, int) {
    std::vector<double> acc(static_cast<std::size_t>(T));
    for (std::int64_t tt = 0; tt < Cout / T; ++tt) {
      std::fill(acc.begin(), acc.end(), 0.0);
      for (int k = 0; k < K; ++k) {  // ascending offset index
        const std::int64_t s = t.omt[static_cast<std::size_t>(i) * K + k];
        if (s < 0) continue;
        for (int c = 0; c < T; ++c) acc[c] += ob(s, tt * T + c);
      }
      for (int c = 0; c < T; ++c) out(i, tt * T + c) = static_cast<float>(acc[c]);
    }
  });
  return out;
}

namespace {
CoordList negate(const CoordList& d) {
  CoordList n(d.size());
  for (std::size_t k = 0; k < d.size(); ++k) n[k] = {-d[k].x, -d[k].y, -d[k].z};
  return n;
}
struct LayerPlanInputs {
  PointCloud Q;
  SortedSource src;
  std::vector<PackedKey> qkeys;
  CoordList search_offsets;
};
LayerPlanInputs prepare_layer(const PointCloud& P, const LayerGeometry& g, int B, SearchCounters* counters) {
  LayerPlanInputs in;
  const OffsetSet delta = weight_offsets_ext(g.kernel_size, g.offset_scale);
  in.search_offsets = g.transposed ? negate(delta.offsets) : delta.offsets;
  if (g.transposed) {
    if (!g.target) throw std::invalid_argument("transposed layer needs target coordinates");
    in.Q = PointCloud{g.target, Matrix{}, true};
    in.src = build_source_array(P, B, counters);
    in.qkeys = pack_all(*g.target);
    for (std::size_t i = 1; i < in.qkeys.size(); ++i)
      if (in.qkeys[i - 1] >= in.qkeys[i]) throw std::invalid_argument("query coordinates must be sorted and unique");
  } else if (g.out_stride == 1) {
    in.src = build_source_array(P, B, counters);
    in.qkeys = in.src.keys;
    if (P.sorted) {
      in.Q = PointCloud{P.coords, Matrix{}, true};  // stride-1 alias
    } else {
      CoordList q(in.src.keys.size());
      for (std::size_t i = 0; i < q.size(); ++i) q[i] = unpack_key(in.src.keys[i]);
      in.Q = PointCloud{make_coords(std::move(q)), Matrix{}, true};
    }
  } else {
    in.Q = generate_output_coords(P, g.out_stride);
    if (counters) ++counters->sorts;
    in.src = build_source_array(P, B, counters);
    in.qkeys = pack_all(*in.Q.coords);
  }
  return in;
}
double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

PointCloud layer_output_coords(const PointCloud& P, int out_stride, SearchCounters* counters) {
  LayerGeometry g;
  g.kernel_size = 1;
  g.out_stride = out_stride;
  return prepare_layer(P, g, 256, counters).Q;
}

KernelMap build_layer_map(const PointCloud& P, const PointCloud& Q, const LayerGeometry& g, const LayerConfig& cfg,
                          SearchCounters* counters) {
  const OffsetSet delta = weight_offsets_ext(g.kernel_size, g.offset_scale);
  const CoordList offs = g.transposed ? negate(delta.offsets) : delta.offsets;
  KernelMap m;
  if (cfg.backend == MapBackend::Brute) {
    m = brute_force_map(*P.coords, *Q.coords, offs);
  } else if (cfg.backend == MapBackend::Hash) {
    m = query_hash_map(build_hash_index(*P.coords), *Q.coords, offs);
  } else {
    const SortedSource src = build_source_array(P, cfg.B, counters);
    m = build_kernel_map_sorted_keys(src, pack_all(*Q.coords), offs, cfg.C, cfg.workers, counters);
  }
  m.offsets = delta.offsets;
  return m;
}

PointCloud sc_layer_forward_ext(const PointCloud& cloud, const WeightSet& w, const LayerGeometry& g,
                                const LayerConfig& cfg, LayerStats* stats) {
  const int Kv = static_cast<int>(weight_offsets_ext(g.kernel_size, g.offset_scale).offsets.size());
  if (w.num_offsets != Kv) throw std::invalid_argument("weight count does not match the kernel volume");
  if (cloud.features.rows() != cloud.size()) throw std::invalid_argument("feature row count does not match point count");
  if (cloud.features.cols() != w.c_in) throw std::invalid_argument("feature channels do not match weights");
  LayerStats local;
  LayerStats& st = stats ? *stats : local;
  auto t0 = std::chrono::steady_clock::now();
  LayerPlanInputs in = prepare_layer(cloud, g, cfg.B, &st.counters);
  KernelMap map;
  if (cfg.backend == MapBackend::Sorted) {
    map = build_kernel_map_sorted_keys(in.src, in.qkeys, in.search_offsets, cfg.C, cfg.workers, &st.counters);
  } else if (cfg.backend == MapBackend::Hash) {
    map = query_hash_map(build_hash_index(*cloud.coords), *in.Q.coords, in.search_offsets);
  } else {
    map = brute_force_map(*cloud.coords, *in.Q.coords, in.search_offsets);
  }
  st.ms_map = ms_since(t0);
  std::vector<std::int64_t> sizes(map.matches.size());
  for (std::size_t k = 0; k < sizes.size(); ++k) sizes[k] = static_cast<std::int64_t>(map.matches[k].size());
  const GemmGroupPlan plan = group_gemms(sizes, cfg.policy, cfg.epsilon, cfg.max_batch);
  const MetadataTables tables = build_metadata_tables(map, plan, cloud.size(), in.Q.size());
  t0 = std::chrono::steady_clock::now();
  const Matrix ib = gather(cloud.features, tables, cfg.gather_tile > 0 ? cfg.gather_tile : w.c_in, &st.imt_lookups,
                           cfg.workers);
  st.ms_gather = ms_since(t0);
  t0 = std::chrono::steady_clock::now();
  const Matrix ob = gemm_execute(ib, w, plan, std::max(1, cfg.workers));
  st.ms_gemm = ms_since(t0);
  t0 = std::chrono::steady_clock::now();
  Matrix out = scatter(ob, tables, cfg.scatter_tile > 0 ? cfg.scatter_tile : w.c_out, cfg.workers);
  st.ms_scatter = ms_since(t0);
  st.matches = map.total();
  st.buffer_length = plan.buffer_length;
  st.groups = static_cast<std::int64_t>(plan.groups.size());
  st.padding_overhead = plan.real_rows() > 0 ? padding_overhead(plan) : 0.0;
  st.sizes = sizes;
  return PointCloud{in.Q.coords, std::move(out), true};
}

PointCloud sc_layer_forward(const PointCloud& cloud, const WeightSet& w, int K, int s, const LayerConfig& cfg,
                            LayerStats* stats) {
  LayerGeometry g;
  g.kernel_size = K;
  g.offset_scale = s;
  g.out_stride = s;
  return sc_layer_forward_ext(cloud, w, g, cfg, stats);
}

Matrix dense_conv_oracle_ext(const PointCloud& cloud, const WeightSet& w, const LayerGeometry& g) {
  const OffsetSet delta = weight_offsets_ext(g.kernel_size, g.offset_scale);
  CoordsPtr Q;
  if (g.transposed) {
    Q = g.target;
  } else {
    LayerGeometry gq = g;
    Q = layer_output_coords(cloud, g.out_stride, nullptr).coords;
  }
  std::unordered_map<PackedKey, std::int64_t> where;
  for (std::int64_t j = 0; j < cloud.size(); ++j) where.emplace(pack_key((*cloud.coords)[j]), j);
  Matrix out(static_cast<std::int64_t>(Q->size()), w.c_out);
  std::vector<double> acc(static_cast<std::size_t>(w.c_out));
  for (std::size_t i = 0; i < Q->size(); ++i) {
    std::fill(acc.begin(), acc.end(), 0.0);
    for (std::size_t k = 0; k < delta.offsets.size(); ++k) {
      const Coordinate d = delta.offsets[k];
      const std::int64_t x = std::int64_t{(*Q)[i].x} + (g.transposed ? -d.x : d.x);
      const std::int64_t y = std::int64_t{(*Q)[i].y} + (g.transposed ? -d.y : d.y);
      const std::int64_t z = std::int64_t{(*Q)[i].z} + (g.transposed ? -d.z : d.z);
      if (!component_in_range(x) || !component_in_range(y) || !component_in_range(z)) continue;
      const auto it = where.find(pack_key({static_cast<std::int32_t>(x), static_cast<std::int32_t>(y),
                                           static_cast<std::int32_t>(z)}));
      if (it == where.end()) continue;
      const float* W = w.matrix(static_cast<int>(k));
      for (int n = 0; n < w.c_out; ++n)
        for (int c = 0; c < w.c_in; ++c)
          acc[n] += static_cast<double>(cloud.features(it->second, c)) * W[c * w.c_out + n];
    }
    for (int n = 0; n < w.c_out; ++n) out(static_cast<std::int64_t>(i), n) = static_cast<float>(acc[n]);
  }
  return out;
}

Matrix dense_conv_oracle(const PointCloud& cloud, const WeightSet& w, int K, int s) {
  LayerGeometry g;
  g.kernel_size = K;
  g.offset_scale = s;
  g.out_stride = s;
  return dense_conv_oracle_ext(cloud, w, g);
}

// ---------------------------------------------------------------- autotune
std::vector<int> candidate_tiles(int channels) {
  if (channels < 1) throw std::invalid_argument("channel count must be positive");
  std::vector<int> d;
  for (int t = 1; t <= channels; ++t)
    if (channels % t == 0) d.push_back(t);
  return d;
}

double profile_candidate(const std::function<void()>& run, int rounds) {
  if (rounds < 1) throw std::invalid_argument("rounds must be positive");
  run();  // warm-up
  std::vector<double> t;
  for (int r = 0; r < rounds; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    run();
    t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  std::sort(t.begin(), t.end());
  return rounds % 2 ? t[rounds / 2] : 0.5 * (t[rounds / 2 - 1] + t[rounds / 2]);
}

int select_tile(const std::vector<std::pair<int, double>>& lat) {
  if (lat.empty()) throw std::invalid_argument("no candidates");
  auto best = lat.front();
  for (const auto& c : lat)
    if (c.second < best.second || (c.second == best.second && c.first < best.first)) best = c;
  return best.first;
}

// ---------------------------------------------------------------- netdef
NetworkSpec preset_network(const std::string& name) {
  NetworkSpec s;
  if (name == "resnet_like") {
    s.layers = {{3, 1, 4, 16},   {3, 1, 16, 16},  {3, 2, 16, 32},   {3, 1, 32, 32},
                {3, 2, 32, 64},  {3, 1, 64, 64},  {3, 2, 64, 128},  {3, 1, 128, 128}};
  } else if (name == "unet_like") {
    s.layers = {{3, 1, 4, 32},    {3, 2, 32, 64},  {3, 1, 64, 64}, {3, 2, 64, 128},
                {3, 1, 128, 128}, {3, 1, 128, 64}, {3, 1, 64, 32}};
  } else {
    throw std::invalid_argument("unknown network preset: " + name);
  }
  return s;
}

WeightSet generate_weights(std::uint64_t seed, std::uint64_t stream, int num_offsets, int c_in, int c_out) {
  WeightSet w;
  w.num_offsets = num_offsets;
  w.c_in = c_in;
  w.c_out = c_out;
  w.w.resize(static_cast<std::size_t>(num_offsets) * c_in * c_out);
  Rng r(stream_seed(seed, stream));
  for (float& v : w.w) v = static_cast<float>(-0.1 + 0.2 * r.next_unit());
  return w;
}

NetworkResult forward_network(const NetworkSpec& spec, const PointCloud& cloud, const LayerConfig& cfg,
                              std::uint64_t seed) {
  if (spec.layers.empty()) throw std::invalid_argument("empty network");
  if (cloud.channels() != spec.layers.front().c_in) throw std::invalid_argument("network input channels mismatch");
  for (std::size_t l = 1; l < spec.layers.size(); ++l)
    if (spec.layers[l - 1].c_out != spec.layers[l].c_in)
      throw std::invalid_argument("network layers are not channel compatible");
  NetworkResult res;
  PointCloud cur = cloud;
  for (std::size_t l = 0; l < spec.layers.size(); ++l) {
    const NetLayer& L = spec.layers[l];
    const int kv = L.K * L.K * L.K;
    const WeightSet w = generate_weights(seed, l + 1, kv, L.c_in, L.c_out);
    LayerStats st;
    cur = sc_layer_forward(cur, w, L.K, L.s, cfg, &st);
    res.sorts += st.counters.sorts;
    res.layers.push_back(std::move(st));
  }
  res.output = std::move(cur);
  return res;
}

PointCloud generate_synthetic(std::int64_t N, std::int64_t E, std::int64_t C, std::uint64_t seed) {
  if (N < 0 || E < 1 || C < 0) throw std::invalid_argument("invalid synthetic cloud parameters");
  if (static_cast<double>(N) > static_cast<double>(E) * E * E) throw std::invalid_argument("infeasible: N > E^3");
  if (E - 1 > COORD_MAX) throw std::out_of_range("extent out of coordinate range");
  Rng r(stream_seed(seed, 0));
  std::unordered_set<PackedKey> seen;
  seen.reserve(static_cast<std::size_t>(N) * 2);
  CoordList c;
  c.reserve(static_cast<std::size_t>(N));
  while (static_cast<std::int64_t>(c.size()) < N) {
    Coordinate p;
    p.x = static_cast<std::int32_t>(r.next_below(static_cast<std::uint64_t>(E)));
    p.y = static_cast<std::int32_t>(r.next_below(static_cast<std::uint64_t>(E)));
    p.z = static_cast<std::int32_t>(r.next_below(static_cast<std::uint64_t>(E)));
    if (seen.insert(pack_key(p)).second) c.push_back(p);
  }
  PointCloud pc;
  pc.coords = make_coords(std::move(c));
  pc.features = Matrix(N, C);
  for (std::int64_t i = 0; i < N; ++i)
    for (std::int64_t ch = 0; ch < C; ++ch) pc.features(i, ch) = static_cast<float>(r.next_unit());
  pc.sorted = false;
  return pc;
}

}  // namespace sconv::oracle

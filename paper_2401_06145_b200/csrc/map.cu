// Map step on sm_100a: segmented query sorting + double-traversed binary search
// (Minuet §5.1), producing the canonical kernel map without a hash table.
//
// Kernels (one launch each, all on the context stream):
//   k_pack_keys      xyz -> packed u64 keys (+ range / sortedness checks)    geometry.hpp:59-67
//   (CUB radix sort) unsorted P -> sorted source keys + original indices
//   k_floor_keys     Eq. 1 floor-to-stride on sorted keys (then sort+unique) geometry.hpp:161-178
//   k_backward       per (offset k, source block b): upper bound of pivot_b
//                    in the virtual query segment {q_i + delta_k}
//   k_plan           balance blocks into ranges of <= C queries, in canonical
//                    (k, b) order, plus tail ranges for unmatched queries
//   k_forward        one CTA per range: stage the source block in shared
//                    memory, binary-search each query, warp-ballot compaction,
//                    decoupled look-back for the canonical output position
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cstring>
#include <string>

#include "common.cuh"
#include "map.hpp"

namespace sconvb {
namespace {

struct MapFlags {
  unsigned long long bad_coord;   // min over (index * 3 + axis) of out-of-range components of P
  unsigned long long bad_target;  // same for the transposed target list
  unsigned long long bad_floor;   // same for Eq. 1 floored coordinates (original index)
  int unsorted;                  // input flagged sorted but keys not strictly increasing
  int target_unsorted;
};

// ---------------------------------------------------------------- key packing
__global__ void k_pack_keys(const int32_t* __restrict__ xyz, int64_t n, uint64_t* __restrict__ keys,
                            int check_sorted, MapFlags* flags, int is_target) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n) return;
  const int32_t x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
  const bool ok = in_range(x) && in_range(y) && in_range(z);
  if (!ok) {
    const int axis = !in_range(x) ? 0 : (!in_range(y) ? 1 : 2);
    atomicMin(is_target ? &flags->bad_target : &flags->bad_coord, static_cast<unsigned long long>(i * 3 + axis));
    keys[i] = 0;
    return;
  }
  const uint64_t k = pack_key_unchecked(x, y, z);
  keys[i] = k;
  if (check_sorted && i + 1 < n) {
    const int32_t x2 = xyz[3 * i + 3], y2 = xyz[3 * i + 4], z2 = xyz[3 * i + 5];
    if (in_range(x2) && in_range(y2) && in_range(z2) && !(k < pack_key_unchecked(x2, y2, z2))) {
      if (is_target)
        atomicOr(&flags->target_unsorted, 1);
      else
        atomicOr(&flags->unsorted, 1);
    }
  }
}

__global__ void k_iota(int32_t* __restrict__ v, int64_t n) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i < n) v[i] = static_cast<int32_t>(i);
}

// Eq. 1 on sorted source keys; range failures recorded by ORIGINAL index so the error
// names the same coordinate the reference's in-order loop would hit first.
__global__ void k_floor_keys(const uint64_t* __restrict__ src, const int32_t* __restrict__ src_idx, int64_t n,
                             int s, uint64_t* __restrict__ out, MapFlags* flags) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n) return;
  int32_t x, y, z;
  unpack_key(src[i], x, y, z);
  const int64_t fx = floor_div(x, s) * s, fy = floor_div(y, s) * s, fz = floor_div(z, s) * s;
  if (!in_range(fx) || !in_range(fy) || !in_range(fz)) {
    const int axis = !in_range(fx) ? 0 : (!in_range(fy) ? 1 : 2);
    const int64_t j = src_idx ? src_idx[i] : i;
    atomicMin(&flags->bad_floor, static_cast<unsigned long long>(j * 3 + axis));
    out[i] = 0;
    return;
  }
  out[i] = pack_key_unchecked(static_cast<int32_t>(fx), static_cast<int32_t>(fy), static_cast<int32_t>(fz));
}

// ---------------------------------------------------------------- backward search
// ub[k * nb + b] = first i with segment_key(q_i, delta_k) > pivot_b.
__global__ void k_backward(const uint64_t* __restrict__ src, int64_t n_src, int B, int64_t nb,
                           const uint64_t* __restrict__ q, int64_t n_q, const int3* __restrict__ offsets, int K3,
                           int32_t* __restrict__ ub) {
  const int64_t t = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (t >= nb * K3) return;
  const int k = static_cast<int>(t / nb);
  const int64_t b = t - int64_t{k} * nb;
  const uint64_t pivot = src[min((b + 1) * B, n_src) - 1];
  const int3 d = offsets[k];
  int64_t lo = 0, hi = n_q;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (segment_key(__ldg(q + mid), d) <= pivot)
      lo = mid + 1;
    else
      hi = mid;
  }
  ub[t] = static_cast<int32_t>(lo);
}

// ---------------------------------------------------------------- range plan
// One CTA. Entries e = k * (nb + 1) + b: b < nb are search blocks (query block
// [ub[k][b-1], ub[k][b]) balanced into ceil(L/C) near-equal ranges, first ranges larger,
// SPEC.md:220); b == nb is the unmatched tail [ub[k][nb-1], n_q), chunked by C so the
// forward kernel can write the dense -1 entries. Descriptor: {k | first<<30, b, lo, hi}.
constexpr int kPlanThreads = 1024;
__global__ void __launch_bounds__(kPlanThreads) k_plan(const int32_t* __restrict__ ub, int64_t nb, int K3, int64_t n_q,
                                                        int C, int4* __restrict__ descs, int* __restrict__ r_total) {
  using Scan = cub::BlockScan<int, kPlanThreads>;
  __shared__ typename Scan::TempStorage temp;
  extern __shared__ int s_first[];  // K3 entries: global index of each offset's first range
  const int64_t E = int64_t{K3} * (nb + 1);
  const int64_t per = (E + kPlanThreads - 1) / kPlanThreads;
  const int64_t e0 = threadIdx.x * per, e1 = min(E, e0 + per);
  auto entry_len = [&](int64_t e, int64_t& lo) -> int64_t {
    const int64_t k = e / (nb + 1), b = e - k * (nb + 1);
    const int32_t* u = ub + k * nb;
    lo = b == 0 ? 0 : u[b - 1];
    const int64_t hi = b < nb ? u[b] : n_q;
    return hi - lo;
  };
  int local = 0;
  for (int64_t e = e0; e < e1; ++e) {
    int64_t lo;
    const int64_t L = entry_len(e, lo);
    local += static_cast<int>((L + C - 1) / C);
  }
  int offset = 0, total = 0;
  Scan(temp).ExclusiveSum(local, offset, total);
  for (int64_t e = e0; e < e1; ++e)  // first range of each offset
    if (e % (nb + 1) == 0) {
      int before = offset;
      for (int64_t f = e0; f < e; ++f) {
        int64_t lo;
        before += static_cast<int>((entry_len(f, lo) + C - 1) / C);
      }
      s_first[e / (nb + 1)] = before;
    }
  __syncthreads();
  int g = offset;
  for (int64_t e = e0; e < e1; ++e) {
    int64_t lo;
    const int64_t L = entry_len(e, lo);
    if (L <= 0) continue;
    const int k = static_cast<int>(e / (nb + 1));
    const int64_t b = e - int64_t{k} * (nb + 1);
    const int64_t parts = (L + C - 1) / C, base = L / parts, extra = L % parts;
    for (int64_t p = 0; p < parts; ++p, ++g) {
      const int64_t len = base + (p < extra ? 1 : 0);
      const int first = (g == s_first[k]) ? 1 : 0;
      descs[g] = make_int4(k | (first << 30), b < nb ? static_cast<int>(b) : -1, static_cast<int>(lo),
                           static_cast<int>(lo + len));
      lo += len;
    }
  }
  if (threadIdx.x == 0) *r_total = total;
}

// ---------------------------------------------------------------- forward search
constexpr int kFwdThreads = 128;
constexpr int kFwdWarps = kFwdThreads / 32;
constexpr uint64_t kFlagAgg = uint64_t{1} << 62, kFlagPrefix = uint64_t{2} << 62, kValMask = (uint64_t{1} << 62) - 1;

template <int QPT>
__global__ void __launch_bounds__(kFwdThreads) k_forward(
    const int4* __restrict__ descs, const int* __restrict__ r_total, int* __restrict__ ticket,
    uint64_t* __restrict__ status, const uint64_t* __restrict__ src, const int32_t* __restrict__ src_idx,
    int64_t n_src, int B, const uint64_t* __restrict__ q, int64_t n_q, const int3* __restrict__ offsets, int K3,
    int32_t* __restrict__ pair_in, int32_t* __restrict__ pair_out, int32_t* __restrict__ nbr_pos,
    int32_t* __restrict__ map_start) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(smem);
  int32_t* s_idx = reinterpret_cast<int32_t*>(s_keys + B);
  __shared__ int s_r;
  __shared__ int s_cnt[QPT][kFwdWarps];
  __shared__ int s_pre[QPT][kFwdWarps];
  __shared__ int s_count;
  __shared__ uint64_t s_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_r = atomicAdd(ticket, 1);  // logical order = ticket order (forward progress)
  __syncthreads();
  const int r = s_r;
  const int R = *r_total;
  if (r >= R) return;
  const int4 d = descs[r];
  const int k = d.x & 0x3FFFFFFF, first = (d.x >> 30) & 1, b = d.y, lo = d.z, hi = d.w;
  int blen = 0;
  if (b >= 0) {  // stage the source block (scratchpad copy, PAPER §5.1.2 step 4)
    const int64_t base = int64_t{b} * B;
    blen = static_cast<int>(min(static_cast<int64_t>(B), n_src - base));
    for (int t = tid; t < blen; t += kFwdThreads) {
      s_keys[t] = src[base + t];
      s_idx[t] = src_idx ? src_idx[base + t] : static_cast<int32_t>(base + t);
    }
  }
  __syncthreads();
  const int3 delta = offsets[k];
  int hit[QPT];
  unsigned bal[QPT];
#pragma unroll
  for (int u = 0; u < QPT; ++u) {
    const int i = lo + u * kFwdThreads + tid;
    hit[u] = -1;
    if (i < hi && blen > 0) {
      const uint64_t key = segment_key(__ldg(q + i), delta);
      int l = 0, h = blen;
      while (l < h) {  // 3-way search, <= ceil(log2(B+1)) steps
        const int mid = (l + h) >> 1;
        const uint64_t v = s_keys[mid];
        if (v == key) {
          hit[u] = s_idx[mid];
          break;
        }
        if (v < key)
          l = mid + 1;
        else
          h = mid;
      }
    }
    bal[u] = __ballot_sync(0xFFFFFFFFu, hit[u] >= 0);
    if (lane == 0) s_cnt[u][warp] = __popc(bal[u]);
  }
  __syncthreads();
  if (tid == 0) {  // prefix over (round u, warp w) = query order
    int acc = 0;
    for (int u = 0; u < QPT; ++u)
      for (int w = 0; w < kFwdWarps; ++w) {
        s_pre[u][w] = acc;
        acc += s_cnt[u][w];
      }
    s_count = acc;
  }
  __syncthreads();
  if (warp == 0) {  // decoupled look-back over the ranges in canonical order
    const uint64_t count = static_cast<uint64_t>(s_count);
    uint64_t base = 0;
    if (r > 0) {
      if (lane == 0) st_release_u64(status + r, kFlagAgg | count);
      int64_t j = r - 1;
      for (;;) {
        const int64_t idx = j - lane;
        uint64_t s = idx >= 0 ? ld_acquire_u64(status + idx) : kFlagPrefix;
        while (__any_sync(0xFFFFFFFFu, (s >> 62) == 0))
          if ((s >> 62) == 0) s = ld_acquire_u64(status + idx);
        const unsigned pmask = __ballot_sync(0xFFFFFFFFu, (s >> 62) == 2);
        const int stop = pmask ? __ffs(pmask) - 1 : 31;
        uint64_t v = lane <= stop ? (s & kValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        base += v;
        if (pmask) break;
        j -= 32;
      }
    }
    if (lane == 0) {
      st_release_u64(status + r, kFlagPrefix | (base + count));
      s_base = base;
    }
  }
  __syncthreads();
  const int64_t base = static_cast<int64_t>(s_base);
  const unsigned lt = (1u << lane) - 1u;
  int32_t* nbr_k = nbr_pos + int64_t{k} * n_q;
#pragma unroll
  for (int u = 0; u < QPT; ++u) {
    const int i = lo + u * kFwdThreads + tid;
    if (i < hi) {
      int32_t m = -1;
      if (hit[u] >= 0) {
        m = static_cast<int32_t>(base + s_pre[u][warp] + __popc(bal[u] & lt));
        pair_in[m] = hit[u];
        pair_out[m] = i;
      }
      nbr_k[i] = m;
    }
  }
  if (tid == 0) {
    if (first) map_start[k] = static_cast<int32_t>(base);
    if (r == R - 1) map_start[K3] = static_cast<int32_t>(base + s_count);
  }
}

constexpr int kThreads = 256;
inline unsigned grid_for(int64_t n) { return static_cast<unsigned>(std::max<int64_t>(1, ceil_div<int64_t>(n, kThreads))); }

std::string coord_error(char axis, int64_t v) {
  return std::string("coordinate ") + axis + " out of range: " + std::to_string(v);
}

void sort_pairs(Ctx& ctx, const uint64_t* kin, uint64_t* kout, const int32_t* vin, int32_t* vout, int64_t n) {
  size_t temp = 0;
  SCONV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, kin, kout, vin, vout, n, 0, 63, ctx.stream));
  ctx.scratch_sort.reserve(temp, ctx.stream);
  ctx.launch("cub_radix_sort_pairs", [&] {
    cub::DeviceRadixSort::SortPairs(ctx.scratch_sort.get(), temp, kin, kout, vin, vout, n, 0, 63, ctx.stream);
  });
}

void sort_keys(Ctx& ctx, const uint64_t* kin, uint64_t* kout, int64_t n) {
  size_t temp = 0;
  SCONV_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, temp, kin, kout, n, 0, 63, ctx.stream));
  ctx.scratch_sort.reserve(temp, ctx.stream);
  ctx.launch("cub_radix_sort_keys",
             [&] { cub::DeviceRadixSort::SortKeys(ctx.scratch_sort.get(), temp, kin, kout, n, 0, 63, ctx.stream); });
}

}  // namespace

std::vector<int3> weight_offsets_ext(int K, int scale) {
  if (K < 1) fail(SCONV_ERR_ARG, "kernel size must be a positive integer");
  if (scale < 1) fail(SCONV_ERR_ARG, "stride must be positive");
  int lo, hi;
  if (K % 2 == 1) {
    lo = -(K / 2);
    hi = K / 2;
    if (!in_range(int64_t{K / 2} * scale)) fail(SCONV_ERR_RANGE, coord_error('x', int64_t{K / 2} * scale));
  } else {
    lo = 0;
    hi = K - 1;
    if (!in_range(int64_t{K - 1} * scale)) fail(SCONV_ERR_RANGE, coord_error('x', int64_t{K - 1} * scale));
  }
  std::vector<int3> d;
  for (int a = lo; a <= hi; ++a)
    for (int b = lo; b <= hi; ++b)
      for (int c = lo; c <= hi; ++c) d.push_back(make_int3(a * scale, b * scale, c * scale));
  return d;
}

std::unique_ptr<MapData> build_map(Ctx& ctx, const MapSource& P, const sconv_map_cfg& cfg, const MapSource* target) {
  if (cfg.block_B < 1 || cfg.block_B > 1024) fail(SCONV_ERR_ARG, "block size B must be in [1, 1024]");
  if (cfg.block_C < 1 || cfg.block_C > 1024) fail(SCONV_ERR_ARG, "query block size C must be in [1, 1024]");
  if (!cfg.transposed && cfg.out_stride < 1) fail(SCONV_ERR_ARG, "stride must be positive");
  if (P.n < 0 || P.n > INT32_MAX / 2) fail(SCONV_ERR_ARG, "point count out of supported range");
  auto m = std::make_unique<MapData>();
  m->cfg = cfg;
  m->n_in = P.n;
  const cudaStream_t st = ctx.stream;
  std::vector<int3> delta = weight_offsets_ext(cfg.kernel_size, cfg.offset_scale);
  if (cfg.transposed)
    for (auto& d : delta) d = make_int3(-d.x, -d.y, -d.z);
  m->K3 = static_cast<int>(delta.size());
  const int K3 = m->K3;
  const int64_t n = P.n;

  DevBuf flags_buf;
  flags_buf.alloc(sizeof(MapFlags), st);
  MapFlags* flags = flags_buf.get<MapFlags>();
  MapFlags init{ULLONG_MAX, ULLONG_MAX, ULLONG_MAX, 0, 0};
  auto* pin = reinterpret_cast<MapFlags*>(ctx.pin_flags());
  pin[0] = init;
  SCONV_CUDA(cudaMemcpyAsync(flags, pin, sizeof(MapFlags), cudaMemcpyHostToDevice, st));

  // ---- source array
  DevBuf xyz_dev;
  const int32_t* xyz = P.xyz;
  if (P.keys) {
    m->src_keys = P.keys;
    m->src_identity = true;
  } else {
    if (n > 0 && P.mem == SCONV_MEM_HOST) {
      xyz_dev.alloc(sizeof(int32_t) * 3 * n, st);
      SCONV_CUDA(cudaMemcpyAsync(xyz_dev.get(), P.xyz, sizeof(int32_t) * 3 * n, cudaMemcpyHostToDevice, st));
      xyz = xyz_dev.get<int32_t>();
    }
    m->src_keys = std::make_shared<DevBuf>();
    if (P.sorted) {
      m->src_keys->alloc(sizeof(uint64_t) * n, st);
      if (n > 0)
        ctx.launch("k_pack_keys", [&] {
          k_pack_keys<<<grid_for(n), kThreads, 0, st>>>(xyz, n, m->src_keys->get<uint64_t>(), 1, flags, 0);
        });
      m->src_identity = true;
    } else {
      DevBuf raw, iota;
      raw.alloc(sizeof(uint64_t) * n, st);
      iota.alloc(sizeof(int32_t) * n, st);
      m->src_keys->alloc(sizeof(uint64_t) * n, st);
      m->src_idx.alloc(sizeof(int32_t) * n, st);
      if (n > 0) {
        ctx.launch("k_pack_keys", [&] {
          k_pack_keys<<<grid_for(n), kThreads, 0, st>>>(xyz, n, raw.get<uint64_t>(), 0, flags, 0);
        });
        ctx.launch("k_iota", [&] { k_iota<<<grid_for(n), kThreads, 0, st>>>(iota.get<int32_t>(), n); });
        sort_pairs(ctx, raw.get<uint64_t>(), m->src_keys->get<uint64_t>(), iota.get<int32_t>(),
                   m->src_idx.get<int32_t>(), n);
      }
      m->src_identity = false;
    }
  }
  const uint64_t* src = m->src_keys_ptr();
  const int32_t* src_idx = m->src_identity ? nullptr : m->src_idx.get<int32_t>();

  // ---- output coordinates Q
  bool need_nout_sync = false;
  DevBuf nsel;
  DevBuf target_xyz_dev;
  if (cfg.transposed) {
    if (!target) fail(SCONV_ERR_ARG, "transposed layer needs target coordinates");
    if (target->keys) {
      m->q_keys = target->keys;
    } else {
      const int32_t* txyz = target->xyz;
      if (target->n > 0 && target->mem == SCONV_MEM_HOST) {
        target_xyz_dev.alloc(sizeof(int32_t) * 3 * target->n, st);
        SCONV_CUDA(cudaMemcpyAsync(target_xyz_dev.get(), target->xyz, sizeof(int32_t) * 3 * target->n,
                                   cudaMemcpyHostToDevice, st));
        txyz = target_xyz_dev.get<int32_t>();
      }
      m->q_keys = std::make_shared<DevBuf>();
      m->q_keys->alloc(sizeof(uint64_t) * target->n, st);
      if (target->n > 0)
        ctx.launch("k_pack_keys", [&] {
          k_pack_keys<<<grid_for(target->n), kThreads, 0, st>>>(txyz, target->n, m->q_keys->get<uint64_t>(), 1,
                                                                 flags, 1);
        });
    }
    m->n_out = target->n;
  } else if (cfg.out_stride == 1) {
    m->q_keys = m->src_keys;  // stride-1 alias: one array serves as source and query
    m->n_out = n;
  } else {
    DevBuf fl, fs;
    fl.alloc(sizeof(uint64_t) * std::max<int64_t>(n, 1), st);
    fs.alloc(sizeof(uint64_t) * std::max<int64_t>(n, 1), st);
    m->q_keys = std::make_shared<DevBuf>();
    m->q_keys->alloc(sizeof(uint64_t) * std::max<int64_t>(n, 1), st);
    nsel.alloc(sizeof(int64_t), st);
    if (n > 0) {
      ctx.launch("k_floor_keys", [&] {
        k_floor_keys<<<grid_for(n), kThreads, 0, st>>>(src, src_idx, n, cfg.out_stride, fl.get<uint64_t>(), flags);
      });
      sort_keys(ctx, fl.get<uint64_t>(), fs.get<uint64_t>(), n);
      size_t temp = 0;
      SCONV_CUDA(cub::DeviceSelect::Unique(nullptr, temp, fs.get<uint64_t>(), m->q_keys->get<uint64_t>(),
                                           nsel.get<int64_t>(), n, st));
      ctx.scratch_misc.reserve(temp, st);
      ctx.launch("cub_select_unique", [&] {
        cub::DeviceSelect::Unique(ctx.scratch_misc.get(), temp, fs.get<uint64_t>(), m->q_keys->get<uint64_t>(),
                                  nsel.get<int64_t>(), n, st);
      });
      need_nout_sync = true;
    } else {
      m->n_out = 0;
    }
  }

  // ---- error checks that must precede any use of the keys (one sync when needed)
  auto check_flags = [&](const MapFlags& f) {
    auto report = [&](unsigned long long code, const int32_t* base, int mem) {
      const int64_t i = static_cast<int64_t>(code / 3);
      const int axis = static_cast<int>(code % 3);
      int32_t c[3];
      if (mem == SCONV_MEM_HOST)
        std::memcpy(c, base + 3 * i, sizeof(c));
      else
        SCONV_CUDA(cudaMemcpy(c, base + 3 * i, sizeof(c), cudaMemcpyDeviceToHost));
      fail(SCONV_ERR_RANGE, coord_error("xyz"[axis], c[axis]));
    };
    if (f.bad_coord != ULLONG_MAX) report(f.bad_coord, P.xyz, P.mem);
    if (f.bad_target != ULLONG_MAX) report(f.bad_target, target->xyz, target->mem);
    if (f.bad_floor != ULLONG_MAX) {
      const int64_t j = static_cast<int64_t>(f.bad_floor / 3);
      const int axis = static_cast<int>(f.bad_floor % 3);
      int32_t c[3] = {0, 0, 0};
      if (P.xyz && P.mem == SCONV_MEM_HOST)
        std::memcpy(c, P.xyz + 3 * j, sizeof(c));
      else if (P.xyz)
        SCONV_CUDA(cudaMemcpy(c, P.xyz + 3 * j, sizeof(c), cudaMemcpyDeviceToHost));
      else {
        uint64_t key;
        SCONV_CUDA(cudaMemcpy(&key, src + j, sizeof(key), cudaMemcpyDeviceToHost));
        unpack_key(key, c[0], c[1], c[2]);
      }
      fail(SCONV_ERR_RANGE, coord_error("xyz"[axis], floor_div(c[axis], cfg.out_stride) * cfg.out_stride));
    }
    if (f.unsorted) fail(SCONV_ERR_ARG, "input coordinates flagged sorted are not strictly increasing");
    if (f.target_unsorted) fail(SCONV_ERR_ARG, "query coordinates must be sorted and unique");
  };
  if (need_nout_sync) {
    SCONV_CUDA(cudaMemcpyAsync(pin, flags, sizeof(MapFlags), cudaMemcpyDeviceToHost, st));
    SCONV_CUDA(cudaMemcpyAsync(&pin[1], nsel.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    static_assert(2 * sizeof(MapFlags) <= Ctx::kPinFlagsBytes, "pinned flags region");
    ctx.sync();
    check_flags(pin[0]);
    int64_t nout;
    std::memcpy(&nout, &pin[1], sizeof(int64_t));
    m->n_out = nout;
  }
  const int64_t n_out = m->n_out;
  const uint64_t* q = m->q_keys_ptr();

  // ---- search
  m->offsets.alloc(sizeof(int3) * K3, st);
  SCONV_CUDA(cudaMemcpyAsync(m->offsets.get(), delta.data(), sizeof(int3) * K3, cudaMemcpyHostToDevice, st));
  m->map_start.alloc(sizeof(int32_t) * (K3 + 1), st);
  m->nbr_pos.alloc(sizeof(int32_t) * std::max<int64_t>(1, int64_t{K3} * n_out), st);
  const int B = cfg.block_B, C = cfg.block_C;
  const int64_t nb = ceil_div<int64_t>(n, B);
  // upper bound on the match count: every query hits at most once
  const int64_t max_pairs = std::min<int64_t>(int64_t{K3} * n_out, int64_t{K3} * n);
  if (n == 0 || n_out == 0) {
    SCONV_CUDA(cudaMemsetAsync(m->map_start.get(), 0, sizeof(int32_t) * (K3 + 1), st));
    if (n_out > 0)
      SCONV_CUDA(cudaMemsetAsync(m->nbr_pos.get(), 0xFF, sizeof(int32_t) * int64_t{K3} * n_out, st));
  } else {
    DevBuf ub, descs, rtot, status, ticket;
    ub.alloc(sizeof(int32_t) * nb * K3, st);
    const int64_t r_max = int64_t{K3} * (nb + ceil_div<int64_t>(n_out, C) + 2);
    if (r_max > INT32_MAX) fail(SCONV_ERR_ARG, "kernel map too large");
    descs.alloc(sizeof(int4) * r_max, st);
    rtot.alloc(sizeof(int), st);
    status.alloc(sizeof(uint64_t) * r_max, st);
    ticket.alloc(sizeof(int), st);
    m->pair_in.alloc(sizeof(int32_t) * std::max<int64_t>(1, max_pairs), st);
    m->pair_out.alloc(sizeof(int32_t) * std::max<int64_t>(1, max_pairs), st);
    ctx.launch("k_backward", [&] {
      k_backward<<<grid_for(nb * K3), kThreads, 0, st>>>(src, n, B, nb, q, n_out, m->offsets.get<int3>(), K3,
                                                         ub.get<int32_t>());
    });
    ctx.launch("k_plan", [&] {
      k_plan<<<1, kPlanThreads, sizeof(int) * K3, st>>>(ub.get<int32_t>(), nb, K3, n_out, C, descs.get<int4>(),
                                                         rtot.get<int>());
    });
    SCONV_CUDA(cudaMemsetAsync(status.get(), 0, sizeof(uint64_t) * r_max, st));
    SCONV_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(int), st));
    const size_t smem = (sizeof(uint64_t) + sizeof(int32_t)) * B;
    const int qpt = ceil_div(C, kFwdThreads);
    auto fwd = [&](auto kernel) {
      ctx.launch("k_forward", [&] {
        kernel<<<static_cast<unsigned>(r_max), kFwdThreads, smem, st>>>(
            descs.get<int4>(), rtot.get<int>(), ticket.get<int>(), status.get<uint64_t>(), src, src_idx, n, B, q,
            n_out, m->offsets.get<int3>(), K3, m->pair_in.get<int32_t>(), m->pair_out.get<int32_t>(),
            m->nbr_pos.get<int32_t>(), m->map_start.get<int32_t>());
      });
    };
    if (qpt <= 1)
      fwd(k_forward<1>);
    else if (qpt <= 2)
      fwd(k_forward<2>);
    else if (qpt <= 4)
      fwd(k_forward<4>);
    else
      fwd(k_forward<8>);
  }
  // ---- readback: flags + canonical list starts (one sync per map)
  if (sizeof(MapFlags) + sizeof(int32_t) * (K3 + 1) > Ctx::kPinReadbackBytes) fail(SCONV_ERR_ARG, "kernel too large");
  auto* pin2 = static_cast<unsigned char*>(ctx.pin_readback());
  SCONV_CUDA(cudaMemcpyAsync(pin2, flags, sizeof(MapFlags), cudaMemcpyDeviceToHost, st));
  SCONV_CUDA(cudaMemcpyAsync(pin2 + sizeof(MapFlags), m->map_start.get(), sizeof(int32_t) * (K3 + 1),
                             cudaMemcpyDeviceToHost, st));
  ctx.sync();
  MapFlags f;
  std::memcpy(&f, pin2, sizeof(f));
  check_flags(f);
  m->starts.resize(K3 + 1);
  std::memcpy(m->starts.data(), pin2 + sizeof(MapFlags), sizeof(int32_t) * (K3 + 1));
  m->sizes.resize(K3);
  for (int k = 0; k < K3; ++k) m->sizes[k] = m->starts[k + 1] - m->starts[k];
  m->total = m->starts[K3];
  return m;
}

}  // namespace sconvb

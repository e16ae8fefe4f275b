// GMaS step on sm_100a (Minuet §5.2): padding-efficient grouping,
// tiled gather, tcgen05 grouped GEMM, deterministic tiled scatter, Alg. 2 tile tuner.
//
//   group_gemms      host, 27-element plan ("<4% of layer time")
//   k_gather<T>      one thread per (buffer slot, channel tile of T): reads the input row
//                    index once per tile (IMT lookup), converts fp32/f16 -> operand type,
//                    16-byte vector stores; padded rows written as zeros
//   grouped GEMM     gemm_sm100.cu
//   k_scatter<T>     one thread per (output row, tile): ascending-k fp32 reduction of the
//                    row's slots (deterministic, tile invariant)
#include <algorithm>
#include <climits>
#include <cstring>
#include <numeric>
#include <set>
#include <vector>

#include "common.cuh"
#include "conv_fused.hpp"
#include "gemm_sm100.hpp"
#include "gmas.hpp"
#include "map.hpp"

namespace sconvb {

// ---------------------------------------------------------------- host plan
GroupPlan group_gemms(const std::vector<int64_t>& sizes, int policy, double eps, int max_batch) {
  if (eps < 0) fail(SCONV_ERR_ARG, "epsilon must be nonnegative");
  if (max_batch < 1) fail(SCONV_ERR_ARG, "max_batch must be positive");
  GroupPlan p;
  std::vector<int> order(sizes.size());
  std::iota(order.begin(), order.end(), 0);
  if (policy == SCONV_GROUP_SORTED)
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sizes[a] < sizes[b]; });
  for (int k : order)
    if (sizes[k] > 0) p.order.push_back(k);
  int64_t gmax = 0, gsum = 0;
  for (int pos = 0; pos < static_cast<int>(p.order.size()); ++pos) {
    const int64_t n = sizes[p.order[pos]];
    bool extend = false;
    if (!p.groups.empty()) {
      const int64_t card = p.groups.back().end - p.groups.back().begin;
      const int64_t nmax = std::max(gmax, n), nsum = gsum + n;
      extend = card < max_batch &&
               static_cast<double>((card + 1) * nmax - nsum) / static_cast<double>(nsum) <= eps;
    }
    if (extend) {
      p.groups.back().end = pos + 1;
      gmax = std::max(gmax, n);
      gsum += n;
    } else {
      p.groups.push_back({pos, pos + 1, 0});
      gmax = n;
      gsum = n;
    }
    p.groups.back().height = gmax;
  }
  p.buffer_offsets.assign(sizes.size(), -1);
  int64_t base = 0;
  for (const auto& g : p.groups) {
    for (int q = g.begin; q < g.end; ++q) p.buffer_offsets[p.order[q]] = base + (q - g.begin) * g.height;
    base += (g.end - g.begin) * g.height;
  }
  p.buffer_length = base;
  for (int k : p.order) p.real_rows += sizes[k];
  return p;
}

namespace {

// ---------------------------------------------------------------- conversions
template <class T>
struct Cvt;
template <>
struct Cvt<__half> {
  static __device__ __forceinline__ __half from(float v) { return __float2half_rn(v); }
  static __device__ __forceinline__ float to(__half v) { return __half2float(v); }
};
template <>
struct Cvt<__nv_bfloat16> {
  static __device__ __forceinline__ __nv_bfloat16 from(float v) { return __float2bfloat16_rn(v); }
  static __device__ __forceinline__ float to(__nv_bfloat16 v) { return __bfloat162float(v); }
};
template <>
struct Cvt<float> {
  static __device__ __forceinline__ float from(float v) { return v; }
  static __device__ __forceinline__ float to(float v) { return v; }
};

// Member table entry in buffer order: {k, row0, n_k, height}.
// k_gather: slot s -> member (binary search over row0 in shared memory) -> canonical
// pair m = map_start[k] + r -> input row j = pair_in[m].
template <int T, class TIn, class TOp>
__global__ void __launch_bounds__(256) k_gather(const TIn* __restrict__ f_in, int c_in, int64_t ld_in,
                                                const __grid_constant__ LayerPlan plan,
                                                const int32_t* __restrict__ map_start,
                                                const int32_t* __restrict__ pair_in, int64_t rows, int k_pad,
                                                TOp* __restrict__ buf, unsigned long long* __restrict__ lookups) {
  __shared__ int4 s_mem[kMaxOffsets];
  const int num_members = plan.nm;
  for (int t = threadIdx.x; t < num_members; t += blockDim.x) s_mem[t] = plan.members[t];
  __syncthreads();
  const int tiles = c_in / T;
  const int64_t gid = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (gid >= rows * tiles) return;
  const int64_t s = gid / tiles;
  const int t = static_cast<int>(gid - s * tiles);
  int lo = 0, hi = num_members - 1;  // last member with row0 <= s
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_mem[mid].y <= s)
      lo = mid;
    else
      hi = mid - 1;
  }
  const int4 mb = s_mem[lo];
  const int64_t r = s - mb.y;
  TOp* dst = buf + s * k_pad + t * T;
  if (lookups) {  // IMT-lookup counter ((C_in / T) * |M|), one atomic per warp
    const unsigned hit = __ballot_sync(__activemask(), r < mb.z);
    if ((threadIdx.x & 31) == __ffs(__activemask()) - 1) atomicAdd(lookups, static_cast<unsigned long long>(__popc(hit)));
  }
  float v[T];
  if (r < mb.z) {
    const int32_t j = __ldg(pair_in + __ldg(map_start + mb.x) + r);
    const TIn* src = f_in + static_cast<int64_t>(j) * ld_in + t * T;
    if constexpr (std::is_same<TIn, float>::value && T % 4 == 0) {
#pragma unroll
      for (int e = 0; e < T; e += 4) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(src + e));
        v[e] = x.x;
        v[e + 1] = x.y;
        v[e + 2] = x.z;
        v[e + 3] = x.w;
      }
    } else if constexpr (!std::is_same<TIn, float>::value && T % 8 == 0) {
#pragma unroll
      for (int e = 0; e < T; e += 8) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(src + e));
        const TIn* h = reinterpret_cast<const TIn*>(&x);
#pragma unroll
        for (int q = 0; q < 8; ++q) v[e + q] = Cvt<TIn>::to(h[q]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < T; ++e) v[e] = Cvt<TIn>::to(src[e]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < T; ++e) v[e] = 0.f;  // padded rows stay exactly zero
  }
  if constexpr (T % 8 == 0) {
#pragma unroll
    for (int e = 0; e < T; e += 8) {
      uint4 o;
      TOp* h = reinterpret_cast<TOp*>(&o);
#pragma unroll
      for (int q = 0; q < 8; ++q) h[q] = Cvt<TOp>::from(v[e + q]);
      *reinterpret_cast<uint4*>(dst + e) = o;
    }
  } else if constexpr (T == 4) {
    uint2 o;
    TOp* h = reinterpret_cast<TOp*>(&o);
#pragma unroll
    for (int q = 0; q < 4; ++q) h[q] = Cvt<TOp>::from(v[q]);
    *reinterpret_cast<uint2*>(dst) = o;
  } else {
#pragma unroll
    for (int e = 0; e < T; ++e) dst[e] = Cvt<TOp>::from(v[e]);
  }
}

// out[i, tile] = sum_{k ascending} gemm_out[m(k,i) + delta[k], tile]  (fp32 accumulate)
template <int T, class TOut>
__global__ void __launch_bounds__(256) k_scatter(const float* __restrict__ gemm_out, int c_out,
                                                 const int32_t* __restrict__ nbr_pos, int64_t n_out, int K3,
                                                 const __grid_constant__ LayerPlan plan, TOut* __restrict__ f_out,
                                                 int64_t ld_out, const TOut* __restrict__ res, int64_t ld_res,
                                                 int relu) {
  __shared__ int32_t s_delta[kMaxOffsets];
  for (int t = threadIdx.x; t < K3; t += blockDim.x) s_delta[t] = plan.delta[t];
  __syncthreads();
  const int tiles = c_out / T;
  const int64_t gid = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (gid >= n_out * tiles) return;
  const int64_t i = gid / tiles;
  const int t = static_cast<int>(gid - i * tiles);
  float acc[T];
#pragma unroll
  for (int e = 0; e < T; ++e) acc[e] = 0.f;
  constexpr int kBatch = 9;  // independent index loads in flight per thread (27 = 3 x 9)
  for (int k0 = 0; k0 < K3; k0 += kBatch) {
    int32_t mk[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      mk[u] = k0 + u < K3 ? __ldg(nbr_pos + int64_t{k0 + u} * n_out + i) : -1;
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {  // ascending k: deterministic reduction order
      if (mk[u] < 0) continue;
      const float* src = gemm_out + static_cast<int64_t>(mk[u] + s_delta[k0 + u]) * c_out + t * T;
      if constexpr (T % 4 == 0) {
#pragma unroll
        for (int e = 0; e < T; e += 4) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(src + e));
          acc[e] += x.x;
          acc[e + 1] += x.y;
          acc[e + 2] += x.z;
          acc[e + 3] += x.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < T; ++e) acc[e] += __ldg(src + e);
      }
    }
  }
  if (res)
#pragma unroll
    for (int e = 0; e < T; ++e) acc[e] += Cvt<TOut>::to(res[i * ld_res + t * T + e]);  // residual epilogue
  if (relu)
#pragma unroll
    for (int e = 0; e < T; ++e) acc[e] = fmaxf(acc[e], 0.f);  // fused ReLU epilogue (network driver)
  TOut* dst = f_out + i * ld_out + t * T;
  if (std::is_same<TOut, float>::value && T % 4 == 0 && ld_out % 4 == 0) {
#pragma unroll
    for (int e = 0; e < T; e += 4)
      reinterpret_cast<float4*>(dst)[e / 4] = make_float4(acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
  } else {
#pragma unroll
    for (int e = 0; e < T; ++e) dst[e] = Cvt<TOut>::from(acc[e]);
  }
}

// ---------------------------------------------------------------- segmented scatter
// Canonical order makes the partials of a tile of consecutive outputs contiguous PER OFFSET:
// list k is sorted by output index, so the hits of outputs [i0, i0+TI) occupy one slot range
// [first, last] of offset k. The CTA loads all K^3 position rows of its tile (coalesced),
// then streams each offset's partial rows with ONE bulk copy (TMA engine) through a ring of
// kScatStages shared-memory stages, accumulating in fp32 in ascending k (deterministic,
// SPEC.md:353) — the partial buffer is read exactly once, fully coalesced.
constexpr int kScatThreads = 256, kScatStages = 4;

__device__ __forceinline__ void bulk_g2s_(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// T = output channels per work item (the scatter tile), TP = partial type, TI = tile rows.
template <int T, class TP, class TOut>
__global__ void __launch_bounds__(kScatThreads) k_scatter_seg(const TP* __restrict__ partials, int c_out,
                                                               const int32_t* __restrict__ nbr_pos, int64_t n_out,
                                                               int K3, const __grid_constant__ LayerPlan plan,
                                                               TOut* __restrict__ f_out, int64_t ld_out,
                                                               const TOut* __restrict__ res, int64_t ld_res, int relu,
                                                               int TI) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int row_bytes = c_out * static_cast<int>(sizeof(TP));
  TP* s_rows = reinterpret_cast<TP*>(smem);                                      // stages x TI rows
  int32_t* s_m = reinterpret_cast<int32_t*>(smem + static_cast<size_t>(kScatStages) * TI * row_bytes);  // K3 x TI
  int32_t* s_first = s_m + K3 * TI;                                              // K3: first position (or -1)
  int32_t* s_cnt = s_first + K3;                                                 // K3: hits
  int32_t* s_act = s_cnt + K3;                                                   // active offsets, ascending
  __shared__ __align__(8) uint64_t s_bar[kScatStages];
  __shared__ int s_nact;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * TI;
  const int n = static_cast<int>(min(static_cast<int64_t>(TI), n_out - i0));
  if (tid == 0) {
    for (int s = 0; s < kScatStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = tid; e < K3 * TI; e += kScatThreads) {
    const int k = e / TI, r = e - k * TI;
    s_m[e] = r < n ? __ldg(nbr_pos + int64_t{k} * n_out + i0 + r) : -1;
  }
  __syncthreads();
  for (int k = warp; k < K3; k += kScatThreads / 32) {  // first hit + hit count per offset
    int first = INT_MAX, cnt = 0;
    for (int r = lane; r < TI; r += 32) {
      const int m = s_m[k * TI + r];
      if (m >= 0) {
        first = min(first, m);
        ++cnt;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      first = min(first, __shfl_xor_sync(0xFFFFFFFFu, first, o));
      cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
    }
    if (lane == 0) {
      s_first[k] = cnt ? first : -1;
      s_cnt[k] = cnt;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int na = 0;
    for (int k = 0; k < K3; ++k)
      if (s_cnt[k] > 0) s_act[na++] = k;
    s_nact = na;
    for (int a = 0; a < min(na, kScatStages); ++a) {  // prime the ring
      const int k = s_act[a];
      const uint32_t bytes = static_cast<uint32_t>(s_cnt[k]) * row_bytes;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&s_bar[a])), "r"(bytes)
                   : "memory");
      bulk_g2s_(s_rows + static_cast<size_t>(a) * TI * c_out,
                partials + static_cast<int64_t>(s_first[k] + plan.delta[k]) * c_out, bytes, &s_bar[a]);
    }
  }
  __syncthreads();
  const int G = c_out / T;             // channel groups per row
  const int pairs = TI * G;            // (row, group) work items
  constexpr int kMaxPer = 8;           // pairs per thread (TI * G <= 8 * 256)
  float acc[kMaxPer][T];
#pragma unroll
  for (int j = 0; j < kMaxPer; ++j)
#pragma unroll
    for (int e = 0; e < T; ++e) acc[j][e] = 0.f;
  const int nact = s_nact;
  for (int a = 0; a < nact; ++a) {
    const int st = a % kScatStages;
    mbar_wait_(&s_bar[st], static_cast<uint32_t>((a / kScatStages) & 1));
    const int k = s_act[a];
    const int first = s_first[k];
    const TP* rows = s_rows + static_cast<size_t>(st) * TI * c_out;
#pragma unroll
    for (int j = 0; j < kMaxPer; ++j) {
      const int p = tid + j * kScatThreads;
      if (p >= pairs) break;
      const int r = p / G, g = p - r * G;
      const int m = s_m[k * TI + r];
      if (m < 0) continue;
      const TP* src = rows + static_cast<size_t>(m - first) * c_out + g * T;
      if constexpr (std::is_same<TP, __half>::value && T % 8 == 0) {
#pragma unroll
        for (int e = 0; e < T; e += 8) {
          const uint4 x = *reinterpret_cast<const uint4*>(src + e);
          const __half2* h = reinterpret_cast<const __half2*>(&x);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f = __half22float2(h[q]);
            acc[j][e + 2 * q] += f.x;
            acc[j][e + 2 * q + 1] += f.y;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < T; ++e) acc[j][e] += Cvt<TP>::to(src[e]);
      }
    }
    __syncthreads();  // stage consumed by every thread
    if (tid == 0 && a + kScatStages < nact) {
      const int k2 = s_act[a + kScatStages];
      const uint32_t bytes = static_cast<uint32_t>(s_cnt[k2]) * row_bytes;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&s_bar[st])), "r"(bytes)
                   : "memory");
      bulk_g2s_(s_rows + static_cast<size_t>(st) * TI * c_out,
                partials + static_cast<int64_t>(s_first[k2] + plan.delta[k2]) * c_out, bytes, &s_bar[st]);
    }
  }
#pragma unroll
  for (int j = 0; j < kMaxPer; ++j) {
    const int p = tid + j * kScatThreads;
    if (p >= pairs) break;
    const int r = p / G, g = p - r * G;
    if (r >= n) continue;
    TOut* dst = f_out + (i0 + r) * ld_out + g * T;
    if (res) {
      const TOut* rr = res + (i0 + r) * ld_res + g * T;
#pragma unroll
      for (int e = 0; e < T; ++e) acc[j][e] += Cvt<TOut>::to(rr[e]);
    }
    if (relu)
#pragma unroll
      for (int e = 0; e < T; ++e) acc[j][e] = fmaxf(acc[j][e], 0.f);
    if (std::is_same<TOut, float>::value && T % 4 == 0 && ld_out % 4 == 0) {
#pragma unroll
      for (int e = 0; e < T; e += 4)
        *reinterpret_cast<float4*>(dst + e) = make_float4(acc[j][e], acc[j][e + 1], acc[j][e + 2], acc[j][e + 3]);
    } else {
#pragma unroll
      for (int e = 0; e < T; ++e) dst[e] = Cvt<TOut>::from(acc[j][e]);
    }
  }
}

constexpr int kBlock = 256;
inline unsigned blocks_for(int64_t n) { return static_cast<unsigned>(std::max<int64_t>(1, ceil_div<int64_t>(n, kBlock))); }

template <class TIn, class TOp>
void gather_dispatch(Ctx& ctx, int T, const void* f_in, int c_in, int64_t ld_in, const LayerPlan& plan,
                     const int32_t* starts, const int32_t* pair_in, int64_t rows, int k_pad, void* buf) {
  const int64_t work = rows * (c_in / T);
  auto go = [&](auto kern) {
    ctx.launch("k_gather", [&] {
      kern<<<blocks_for(work), kBlock, 0, ctx.stream>>>(static_cast<const TIn*>(f_in), c_in, ld_in, plan, starts,
                                                        pair_in, rows, k_pad, static_cast<TOp*>(buf),
                                                        ctx.count_lookups ? ctx.lookup_counter : nullptr);
    });
  };
  switch (T) {
    case 1: go(k_gather<1, TIn, TOp>); break;
    case 2: go(k_gather<2, TIn, TOp>); break;
    case 3: go(k_gather<3, TIn, TOp>); break;
    case 4: go(k_gather<4, TIn, TOp>); break;
    case 6: go(k_gather<6, TIn, TOp>); break;
    case 8: go(k_gather<8, TIn, TOp>); break;
    case 12: go(k_gather<12, TIn, TOp>); break;
    case 16: go(k_gather<16, TIn, TOp>); break;
    case 24: go(k_gather<24, TIn, TOp>); break;
    case 32: go(k_gather<32, TIn, TOp>); break;
    case 48: go(k_gather<48, TIn, TOp>); break;
    case 64: go(k_gather<64, TIn, TOp>); break;
    default: fail(SCONV_ERR_ARG, "unsupported gather tile size " + std::to_string(T));
  }
}

template <class TOut>
void scatter_dispatch(Ctx& ctx, int T, const float* gemm_out, int c_out, const int32_t* nbr, int64_t n_out, int K3,
                      const LayerPlan& plan, const LayerIO& io) {
  const int64_t work = n_out * (c_out / T);
  auto go = [&](auto kern) {
    ctx.launch("k_scatter", [&] {
      kern<<<blocks_for(work), kBlock, 0, ctx.stream>>>(gemm_out, c_out, nbr, n_out, K3, plan,
                                                        static_cast<TOut*>(io.f_out), io.ld_out,
                                                        static_cast<const TOut*>(io.res), io.ld_res, io.relu);
    });
  };
  switch (T) {
    case 1: go(k_scatter<1, TOut>); break;
    case 2: go(k_scatter<2, TOut>); break;
    case 3: go(k_scatter<3, TOut>); break;
    case 4: go(k_scatter<4, TOut>); break;
    case 6: go(k_scatter<6, TOut>); break;
    case 8: go(k_scatter<8, TOut>); break;
    case 12: go(k_scatter<12, TOut>); break;
    case 16: go(k_scatter<16, TOut>); break;
    case 24: go(k_scatter<24, TOut>); break;
    case 32: go(k_scatter<32, TOut>); break;
    case 48: go(k_scatter<48, TOut>); break;
    case 64: go(k_scatter<64, TOut>); break;
    default: fail(SCONV_ERR_ARG, "unsupported scatter tile size " + std::to_string(T));
  }
}

// tile rows so that every thread owns <= 8 (row, group) items and the ring fits ~96 KB
int scatter_rows(int c_out, int T, int part_bytes) {
  int ti = std::min(128, (8 * kScatThreads * T) / c_out);
  ti = std::min(ti, (96 * 1024) / (kScatStages * c_out * part_bytes));
  return std::max(1, ti);
}

bool seg_scatter_ok(int c_out, int T, int part_bytes) {
  return (c_out * part_bytes) % 16 == 0 && c_out % T == 0 && (T == 1 || T == 2 || T == 4 || T == 8 || T == 16) &&
         (8 * kScatThreads * T) / c_out >= 1;
}

template <class TP, class TOut>
void scatter_seg_dispatch(Ctx& ctx, int T, const TP* partials, int c_out, const int32_t* nbr, int64_t n_out, int K3,
                          const LayerPlan& plan, const LayerIO& io) {
  const int TI = scatter_rows(c_out, T, sizeof(TP));
  const size_t smem = static_cast<size_t>(kScatStages) * TI * c_out * sizeof(TP) + sizeof(int32_t) * (K3 * TI + 3 * K3) + 16;
  auto go = [&](auto kern) {
    // once per kernel (keyed by address: tile variants share one function-pointer type)
    static thread_local std::set<std::pair<const void*, int>> attr_set;
    if (attr_set.insert({reinterpret_cast<const void*>(kern), ctx.device}).second)
      SCONV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    ctx.launch("k_scatter", [&] {
      kern<<<static_cast<unsigned>(ceil_div<int64_t>(n_out, TI)), kScatThreads, smem, ctx.stream>>>(
          partials, c_out, nbr, n_out, K3, plan, static_cast<TOut*>(io.f_out), io.ld_out,
          static_cast<const TOut*>(io.res), io.ld_res, io.relu, TI);
    });
  };
  switch (T) {
    case 1: go(k_scatter_seg<1, TP, TOut>); break;
    case 2: go(k_scatter_seg<2, TP, TOut>); break;
    case 4: go(k_scatter_seg<4, TP, TOut>); break;
    case 8: go(k_scatter_seg<8, TP, TOut>); break;
    default: go(k_scatter_seg<16, TP, TOut>); break;
  }
}

size_t dtype_size(int d) { return d == SCONV_F32 ? 4 : 2; }

}  // namespace

std::vector<int> candidate_tiles(int channels) {
  std::vector<int> d;
  for (int t = 1; t <= channels; ++t)
    if (channels % t == 0 && is_supported_tile(t)) d.push_back(t);
  return d;
}

bool is_supported_tile(int t) {
  switch (t) {
    case 1: case 2: case 3: case 4: case 6: case 8: case 12: case 16: case 24: case 32: case 48: case 64:
      return true;
    default:
      return false;
  }
}

int default_tile(int channels, bool gather) {
  // Heuristic before tuning: 16-byte operand stores for gather, 16-byte f16 partial reads
  // (8 channels) for the segmented scatter.
  const int pref = 8;
  for (int t = pref; t >= 1; --t)
    if (channels % t == 0 && is_supported_tile(t)) return t;
  return 1;
}

int padded_k(int c_in) { return (c_in + 15) / 16 * 16; }

// ---------------------------------------------------------------- weights
std::unique_ptr<WeightData> create_weights(Ctx& ctx, const float* w, int mem, int K3, int c_in, int c_out, int dtype) {
  if (K3 < 1 || K3 > kMaxOffsets) fail(SCONV_ERR_ARG, "offset count out of supported range");
  if (c_in < 1 || c_out < 1) fail(SCONV_ERR_ARG, "channel counts must be positive");
  if (dtype != SCONV_F16 && dtype != SCONV_BF16) fail(SCONV_ERR_ARG, "weight dtype must be f16 or bf16");
  auto wd = std::make_unique<WeightData>();
  wd->K3 = K3;
  wd->c_in = c_in;
  wd->c_out = c_out;
  wd->dtype = dtype;
  wd->k_pad = padded_k(c_in);
  wd->n_pad = (c_out + 15) / 16 * 16;
  std::vector<float> host;
  const float* src = w;
  if (mem == SCONV_MEM_DEVICE) {
    host.resize(static_cast<size_t>(K3) * c_in * c_out);
    SCONV_CUDA(cudaMemcpy(host.data(), w, host.size() * sizeof(float), cudaMemcpyDeviceToHost));
    src = host.data();
  }
  std::vector<uint16_t> t(static_cast<size_t>(K3) * wd->n_pad * wd->k_pad, 0);
  for (int k = 0; k < K3; ++k)
    for (int ci = 0; ci < c_in; ++ci)
      for (int co = 0; co < c_out; ++co) {
        const float v = src[(static_cast<size_t>(k) * c_in + ci) * c_out + co];
        uint16_t bits;
        if (dtype == SCONV_F16) {
          const __half h = __float2half_rn(v);
          std::memcpy(&bits, &h, 2);
        } else {
          const __nv_bfloat16 h = __float2bfloat16_rn(v);
          std::memcpy(&bits, &h, 2);
        }
        t[(static_cast<size_t>(k) * wd->n_pad + co) * wd->k_pad + ci] = bits;  // W_k^T, K-major
      }
  wd->buf.alloc(t.size() * 2, ctx.stream);
  SCONV_CUDA(cudaMemcpyAsync(wd->buf.get(), t.data(), t.size() * 2, cudaMemcpyHostToDevice, ctx.stream));
  ctx.sync();
  return wd;
}

// ---------------------------------------------------------------- layer forward
namespace {

// Minuet GMaS on device buffers: plan -> gather -> grouped GEMM -> scatter.
void gmas_forward(Ctx& ctx, MapData& m, const WeightData& w, const sconv_exec_cfg& cfg, const LayerIO& io) {
  ensure_canonical(ctx, m);  // GMaS needs the per-offset sizes and canonical pair lists
  const cudaStream_t st = ctx.stream;
  const int c_in = w.c_in, c_out = w.c_out, K3 = m.K3;
  int Tg = cfg.gather_tile, Ts = cfg.scatter_tile;
  if (Tg <= 0 || Ts <= 0) {
    const auto it = ctx.tuned.find({c_in, c_out, w.dtype});
    if (Tg <= 0) Tg = it != ctx.tuned.end() ? it->second.first : default_tile(c_in, true);
    if (Ts <= 0) Ts = it != ctx.tuned.end() ? it->second.second : default_tile(c_out, false);
  }
  if (c_in % Tg != 0 || c_out % Ts != 0) fail(SCONV_ERR_ARG, "tile size must divide the channel count");
  if (!is_supported_tile(Tg) || !is_supported_tile(Ts)) fail(SCONV_ERR_ARG, "unsupported tile size");

  const GroupPlan plan = group_gemms(m.sizes, cfg.policy, cfg.epsilon, cfg.max_batch);
  m.buffer_length = plan.buffer_length;
  m.groups = static_cast<int>(plan.groups.size());
  m.padding_overhead = plan.real_rows > 0 ? static_cast<double>(plan.buffer_length - plan.real_rows) / plan.real_rows : 0.0;
  m.gather_tile = Tg;
  m.scatter_tile = Ts;
  const int64_t R = plan.buffer_length;
  // slot indices (buffer rows, member deltas) are int32 on the device
  if (R > INT32_MAX) fail(SCONV_ERR_ARG, "GMaS buffer too large: more than 2^31 - 1 padded rows");
  const size_t out_elem = dtype_size(io.out_dtype);
  if (R == 0 || m.n_in == 0) {
    if (io.res == nullptr && io.ld_out == c_out) {
      SCONV_CUDA(cudaMemsetAsync(io.f_out, 0, out_elem * m.n_out * c_out, st));
      return;
    }
  }
  // ---- plan (members in buffer order, GEMM tile prefix, scatter deltas): a kernel
  // parameter, so consecutive layers never race on a staging buffer.
  if (plan.order.size() > static_cast<size_t>(kMaxOffsets)) fail(SCONV_ERR_ARG, "too many offsets");
  auto lp = std::make_unique<LayerPlan>();
  const int block_n = std::min(w.n_pad, 256);
  lp->block_n = block_n;
  lp->n_blocks = ceil_div(w.n_pad, block_n);
  lp->nm = 0;
  lp->tile_start[0] = 0;
  for (const auto& g : plan.groups)
    for (int q = g.begin; q < g.end; ++q) {
      const int k = plan.order[q];
      lp->members[lp->nm] = make_int4(k, static_cast<int>(plan.buffer_offsets[k]), static_cast<int>(m.sizes[k]),
                                      static_cast<int>(g.height));
      lp->tile_start[lp->nm + 1] = lp->tile_start[lp->nm] + ceil_div(static_cast<int>(g.height), 128) * lp->n_blocks;
      ++lp->nm;
    }
  lp->num_tiles = lp->tile_start[lp->nm];
  for (int k = 0; k < K3; ++k)
    lp->delta[k] = plan.buffer_offsets[k] >= 0 ? static_cast<int32_t>(plan.buffer_offsets[k] - m.starts[k]) : 0;

  const int k_pad = w.k_pad;
  const bool part_f16 = cfg.partial_f16 && w.dtype == SCONV_F16 && seg_scatter_ok(c_out, Ts, 2);
  const int part_bytes = part_f16 ? 2 : 4;
  if (R > 0 && m.n_in > 0) {
    // ---- gather
    ctx.gather_buf.reserve(static_cast<size_t>(R) * k_pad * 2, st);
    if (k_pad != c_in) SCONV_CUDA(cudaMemsetAsync(ctx.gather_buf.get(), 0, static_cast<size_t>(R) * k_pad * 2, st));
    const int32_t* starts = m.map_start.get<int32_t>();
    const int32_t* pin_idx = m.pair_in.get<int32_t>();
    void* gb = ctx.gather_buf.get();
    if (w.dtype == SCONV_F16) {
      if (io.in_dtype == SCONV_F32)
        gather_dispatch<float, __half>(ctx, Tg, io.f_in, c_in, io.ld_in, *lp, starts, pin_idx, R, k_pad, gb);
      else
        gather_dispatch<__half, __half>(ctx, Tg, io.f_in, c_in, io.ld_in, *lp, starts, pin_idx, R, k_pad, gb);
    } else {
      if (io.in_dtype == SCONV_F32)
        gather_dispatch<float, __nv_bfloat16>(ctx, Tg, io.f_in, c_in, io.ld_in, *lp, starts, pin_idx, R, k_pad, gb);
      else
        gather_dispatch<__nv_bfloat16, __nv_bfloat16>(ctx, Tg, io.f_in, c_in, io.ld_in, *lp, starts, pin_idx, R, k_pad,
                                                      gb);
    }
    // ---- grouped GEMM: per-offset partials, f16 when computing in f16 (halves the largest
    // stream), else fp32
    ctx.gemm_out.reserve(static_cast<size_t>(R) * c_out * part_bytes, st);
    GemmArgs ga;
    ga.a = gb;
    ga.b = w.buf.get();
    ga.plan = lp.get();
    ga.num_tiles = lp->num_tiles;
    ga.rows = R;
    ga.k_pad = k_pad;
    ga.num_kb = k_pad / gemm_chunk(k_pad);
    ga.n_pad = w.n_pad;
    ga.block_n = block_n;
    ga.c_out = c_out;
    ga.num_offsets = K3;
    ga.dtype = w.dtype;
    ga.out = ctx.gemm_out.get();
    ga.out_f16 = part_f16;
    launch_grouped_gemm(ctx, ga);
  }
  // ---- scatter (rows without matches: zero [+ residual])
  const int32_t* nbr = m.nbr_pos.get<int32_t>();
  if (part_f16) {
    if (io.out_dtype == SCONV_F32)
      scatter_seg_dispatch<__half, float>(ctx, Ts, ctx.gemm_out.get<__half>(), c_out, nbr, m.n_out, K3, *lp, io);
    else if (io.out_dtype == SCONV_F16)
      scatter_seg_dispatch<__half, __half>(ctx, Ts, ctx.gemm_out.get<__half>(), c_out, nbr, m.n_out, K3, *lp, io);
    else
      scatter_seg_dispatch<__half, __nv_bfloat16>(ctx, Ts, ctx.gemm_out.get<__half>(), c_out, nbr, m.n_out, K3, *lp,
                                                  io);
  } else if (seg_scatter_ok(c_out, Ts, 4)) {
    if (io.out_dtype == SCONV_F32)
      scatter_seg_dispatch<float, float>(ctx, Ts, ctx.gemm_out.get<float>(), c_out, nbr, m.n_out, K3, *lp, io);
    else if (io.out_dtype == SCONV_F16)
      scatter_seg_dispatch<float, __half>(ctx, Ts, ctx.gemm_out.get<float>(), c_out, nbr, m.n_out, K3, *lp, io);
    else
      scatter_seg_dispatch<float, __nv_bfloat16>(ctx, Ts, ctx.gemm_out.get<float>(), c_out, nbr, m.n_out, K3, *lp, io);
  } else {
    if (io.out_dtype == SCONV_F32)
      scatter_dispatch<float>(ctx, Ts, ctx.gemm_out.get<float>(), c_out, nbr, m.n_out, K3, *lp, io);
    else if (io.out_dtype == SCONV_F16)
      scatter_dispatch<__half>(ctx, Ts, ctx.gemm_out.get<float>(), c_out, nbr, m.n_out, K3, *lp, io);
    else
      scatter_dispatch<__nv_bfloat16>(ctx, Ts, ctx.gemm_out.get<float>(), c_out, nbr, m.n_out, K3, *lp, io);
  }
}

// Fused output-stationary dataflow (conv_fused.cu): operands must be 16-bit rows of at least
// k_pad zero-padded columns; anything else is converted once into the gather scratch.
void fused_forward(Ctx& ctx, MapData& m, const WeightData& w, const LayerIO& io) {
  m.buffer_length = 0;
  m.groups = 0;
  m.padding_overhead = 0.0;
  m.gather_tile = m.scatter_tile = 0;
  const void* fin = io.f_in;
  int64_t ld = io.ld_in;
  const bool direct = io.in_dtype == w.dtype && ld % 8 == 0 && ld >= w.k_pad && (w.k_pad == w.c_in || io.in_zero_padded);
  if (!direct && m.n_in > 0) {
    ctx.gather_buf.reserve(static_cast<size_t>(m.n_in) * w.k_pad * 2, ctx.stream);
    convert_rows(ctx, io.f_in, io.in_dtype, m.n_in, w.c_in, io.ld_in, ctx.gather_buf.get(), w.dtype, w.k_pad);
    fin = ctx.gather_buf.get();
    ld = w.k_pad;
  }
  FusedArgs a;
  a.f_in = fin;
  a.ld_in = ld;
  a.n_in = m.n_in;
  prepare_fused_layout(ctx, m);
  if (m.fused_ready && !m.identity_pending && !m.items_ready) build_fused_items(ctx, m);  // identity materialised later
  a.nbr = m.identity_pending ? nullptr : (m.permuted ? m.nbr_perm.get<int32_t>() : m.nbr_in.get<int32_t>());
  if (m.items.get()) {
    a.tile_mask = m.tile_mask.get<unsigned long long>();
    a.items = m.items.get<int4>();
    a.item_ws = m.item_ws.get<int>();
    a.n_items = m.n_items.get<int>();
    a.item_counters = m.item_counters.get<int>();
    a.max_items = m.max_items;
    a.max_ws_slots = m.max_ws_slots;
  }
  a.perm = m.permuted ? m.row_perm.get<int32_t>() : nullptr;
  a.n_out = m.n_out;
  a.w = &w;
  a.out = io.f_out;
  a.out_dtype = io.out_dtype;
  a.ld_out = io.ld_out;
  a.res = io.res;
  a.ld_res = io.ld_res;
  a.relu = io.relu;
  launch_conv_fused(ctx, a);
}

}  // namespace

void layer_forward_dev(Ctx& ctx, MapData& m, const WeightData& w, const sconv_exec_cfg& cfg, int dataflow,
                       const LayerIO& io) {
  if (w.K3 != m.K3) fail(SCONV_ERR_ARG, "weight count does not match the kernel volume");
  if (io.in_dtype != SCONV_F32 && io.in_dtype != SCONV_F16 && io.in_dtype != SCONV_BF16)
    fail(SCONV_ERR_ARG, "unsupported input dtype");
  if (io.out_dtype != SCONV_F32 && io.out_dtype != SCONV_F16 && io.out_dtype != SCONV_BF16)
    fail(SCONV_ERR_ARG, "unsupported output dtype");
  if (io.in_dtype != SCONV_F32 && io.in_dtype != w.dtype) fail(SCONV_ERR_ARG, "16-bit input must match the weight dtype");
  if (io.ld_in < w.c_in || io.ld_out < w.c_out || (io.res && io.ld_res < w.c_out))
    fail(SCONV_ERR_ARG, "row stride smaller than the channel count");
  if (m.n_out == 0) return;
  if (dataflow == SCONV_DATAFLOW_FUSED && fused_supported(m.K3, w.c_in, w.c_out))
    fused_forward(ctx, m, w, io);
  else
    gmas_forward(ctx, m, w, cfg, io);
}

void layer_forward(Ctx& ctx, MapData& m, const WeightData& w, const void* f_in, int f_in_dtype, int f_in_mem,
                   const sconv_exec_cfg& cfg, void* f_out, int f_out_dtype, int f_out_mem, int relu) {
  const cudaStream_t st = ctx.stream;
  DevBuf fin_dev, fout_dev;
  const void* fin = f_in;
  if (f_in_mem == SCONV_MEM_HOST && m.n_in > 0) {
    const size_t bytes = dtype_size(f_in_dtype) * m.n_in * w.c_in;
    fin_dev.alloc(bytes, st);
    SCONV_CUDA(cudaMemcpyAsync(fin_dev.get(), f_in, bytes, cudaMemcpyHostToDevice, st));
    fin = fin_dev.get();
  }
  void* fout = f_out;
  const size_t out_bytes = dtype_size(f_out_dtype) * m.n_out * w.c_out;
  if (f_out_mem == SCONV_MEM_HOST && m.n_out > 0) {
    fout_dev.alloc(out_bytes, st);
    fout = fout_dev.get();
  }
  LayerIO io;
  io.f_in = fin;
  io.in_dtype = f_in_dtype;
  io.ld_in = w.c_in;
  io.f_out = fout;
  io.out_dtype = f_out_dtype;
  io.ld_out = w.c_out;
  io.relu = relu;
  layer_forward_dev(ctx, m, w, cfg, cfg.dataflow == SCONV_DATAFLOW_FUSED ? SCONV_DATAFLOW_FUSED : SCONV_DATAFLOW_GMAS,
                    io);
  if (f_out_mem == SCONV_MEM_HOST && m.n_out > 0) {
    SCONV_CUDA(cudaMemcpyAsync(f_out, fout, out_bytes, cudaMemcpyDeviceToHost, st));
    ctx.sync();
  }
}

}  // namespace sconvb

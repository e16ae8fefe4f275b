// Map step on sm_100a: segmented query sorting + double-traversed binary search
// (Minuet §5.1), producing the canonical kernel map without a hash table.
//
// Kernels (all on the context stream; file:line = the reference operation replaced):
//   k_bbox / k_pack_compact / k_hist_scan / k_bucket_scatter / k_bucket_rank
//                    unsorted P -> sorted source keys + original indices
//                    (left-aligned compact keys, bucket sort; exact CUB 64-bit fallback)
//   k_pack_keys      xyz -> packed u64 keys (+ range / sortedness checks)      geometry.hpp:59-67
//   k_floor_keys     Eq. 1 floor-to-stride (then CUB sort + unique)            geometry.hpp:161-178
//   k_search         double-traversed binary search: backward (pivot vs query
//                    segment) + forward (query vs staged source block)
//   k_emit           canonical positions (per offset k, ordered by i) and pairs SPEC.md:235-243
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>

#include "common.cuh"
#include "coop_sort.cuh"
#include "map.hpp"

namespace sconvb {
namespace {

// Small device->host readbacks (map flags, |Q|, list starts) the host syncs on: stored by a
// one-warp kernel straight into the mapped pinned destination instead of a copy-engine memcpy,
// so they never queue behind a large result copy on the device->host engine (a serving loop's
// sconv_net_read_async of the previous forward: r02cc, C2 next forward's first conv +0.45 ms).
__global__ void k_d2h_small(const unsigned* __restrict__ src, unsigned* dst, int words) {
  for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}

void d2h_small(void* host_pinned, const void* dev, size_t bytes, cudaStream_t st) {
  static const bool use_kernel = [] {
    const char* e = std::getenv("SCONV_D2H_SMALL_KERNEL");
    return !(e && e[0] == '0');
  }();
  void* dptr = nullptr;
  if (use_kernel && bytes % 4 == 0 && reinterpret_cast<uintptr_t>(dev) % 4 == 0 &&
      reinterpret_cast<uintptr_t>(host_pinned) % 4 == 0 && cudaHostGetDevicePointer(&dptr, host_pinned, 0) == cudaSuccess) {
    k_d2h_small<<<1, 32, 0, st>>>(static_cast<const unsigned*>(dev), static_cast<unsigned*>(dptr),
                                  static_cast<int>(bytes / 4));
    SCONV_CUDA(cudaGetLastError());
    return;
  }
  (void)cudaGetLastError();  // a non-mapped destination: plain copy
  SCONV_CUDA(cudaMemcpyAsync(host_pinned, dev, bytes, cudaMemcpyDeviceToHost, st));
}

struct MapFlags {
  unsigned long long bad_coord;   // min over (index * 3 + axis) of out-of-range components of P
  unsigned long long bad_target;  // same for the transposed target list
  unsigned long long bad_floor;   // same for Eq. 1 floored coordinates (original index)
  int unsorted;                  // input flagged sorted but keys not strictly increasing
  int target_unsorted;
  int bbox[6];                   // min x,y,z / max x,y,z of P (unsorted path)
  int wide;                      // compact key needs > 32 bits: rebuild with the 64-bit CUB sort
  int big_bucket;                // a sort bucket exceeds kMaxBucket: rebuild with the 64-bit CUB sort
  int fbox[6];                   // bbox of the Eq. 1 floored coordinates (strided maps)
  int fwide;                     // floored compact key needs > 32 bits: redo with 64-bit keys
  int reserved;                  // explicit tail (the struct is copied to the host whole)
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

// One launch per map build: flag init + weight offsets (weight_offsets_ext order: a outer,
// b, c inner; odd K centred, even K in [0, K-1]) times the offset scale, negated when transposed
__global__ void k_init_flags(MapFlags* f) {
  {
    f->bad_coord = f->bad_target = f->bad_floor = ULLONG_MAX;
    f->unsorted = f->target_unsorted = 0;
    f->bbox[0] = f->bbox[1] = f->bbox[2] = INT_MAX;
    f->bbox[3] = f->bbox[4] = f->bbox[5] = INT_MIN;
    f->wide = f->big_bucket = 0;
    f->fbox[0] = f->fbox[1] = f->fbox[2] = INT_MAX;
    f->fbox[3] = f->fbox[4] = f->fbox[5] = INT_MIN;
    f->fwide = 0;
    f->reserved = 0;
  }
}

// 1x1 (K=1) stride-1 map over a sorted set: Q = P, every output is its own single neighbour.
__global__ void k_identity_map(int64_t n, int32_t* __restrict__ nbr_in, int32_t* __restrict__ nbr_pos,
                               int32_t* __restrict__ pair_in, int32_t* __restrict__ pair_out,
                               int32_t* __restrict__ map_start) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i == 0) {
    map_start[0] = 0;
    map_start[1] = static_cast<int32_t>(n);
  }
  if (i >= n) return;
  const int32_t v = static_cast<int32_t>(i);
  nbr_in[i] = nbr_pos[i] = pair_in[i] = pair_out[i] = v;
}

__global__ void k_iota(int32_t* __restrict__ v, int64_t n) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i < n) v[i] = static_cast<int32_t>(i);
}

// ---- compact sort keys: (x-xmin, y-ymin, z-zmin) with the minimal bit widths preserve the
// lexicographic order and usually fit 32 bits (KITTI at 5 cm: 12+12+8), so the radix sort
// runs over 4 digits of a u32 key instead of 8 digits of the 63-bit packed key.
__global__ void k_bbox(const int32_t* __restrict__ xyz, int64_t n, MapFlags* flags) {
  int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
  for (int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; i < n; i += int64_t{gridDim.x} * blockDim.x)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int v = __ldg(xyz + 3 * i + a);
      mn[a] = min(mn[a], v);
      mx[a] = max(mx[a], v);
    }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn[a] = min(mn[a], __shfl_xor_sync(0xFFFFFFFFu, mn[a], o));
      mx[a] = max(mx[a], __shfl_xor_sync(0xFFFFFFFFu, mx[a], o));
    }
  __shared__ int s_red[6][32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (l == 0)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      s_red[a][w] = mn[a];
      s_red[3 + a][w] = mx[a];
    }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int a = threadIdx.x;
    int v = s_red[a][0];
    for (int q = 1; q < nw; ++q) v = a < 3 ? min(v, s_red[a][q]) : max(v, s_red[a][q]);
    if (a < 3)
      atomicMin(&flags->bbox[a], v);
    else
      atomicMax(&flags->bbox[a], v);
  }
}

__device__ __forceinline__ int bits_for(int64_t extent) {  // bits to hold [0, extent]
  return extent <= 0 ? 0 : 64 - __clzll(static_cast<unsigned long long>(extent));
}

// Left-aligned compact key: the T significant bits sit at the top of a u32, so the top
// kBucketBits select a bucket independent of T.
constexpr int kMaxBucketBits = 16, kBuckets = 1 << kMaxBucketBits, kMaxBucket = 4096;

__device__ __forceinline__ int compact_bits(const MapFlags* f, int& by, int& bz) {
  by = bits_for(int64_t{f->bbox[4]} - f->bbox[1]);
  bz = bits_for(int64_t{f->bbox[5]} - f->bbox[2]);
  return bits_for(int64_t{f->bbox[3]} - f->bbox[0]) + by + bz;
}

__global__ void k_pack_compact(const int32_t* __restrict__ xyz, int64_t n, MapFlags* flags,
                               uint32_t* __restrict__ ck, int32_t* __restrict__ idx, int* __restrict__ hist, int H) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n) return;
  const int32_t x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
  idx[i] = static_cast<int32_t>(i);
  if (!(in_range(x) && in_range(y) && in_range(z))) {
    const int axis = !in_range(x) ? 0 : (!in_range(y) ? 1 : 2);
    atomicMin(&flags->bad_coord, static_cast<unsigned long long>(i * 3 + axis));
    ck[i] = 0;
    return;
  }
  int by, bz;
  const int T = compact_bits(flags, by, bz);
  if (T > 32) {
    if (i == 0) flags->wide = 1;
    ck[i] = 0;
    return;
  }
  const uint64_t c = (static_cast<uint64_t>(x - flags->bbox[0]) << (by + bz)) |
                     (static_cast<uint64_t>(y - flags->bbox[1]) << bz) | static_cast<uint64_t>(z - flags->bbox[2]);
  const uint32_t lk = static_cast<uint32_t>(c << (32 - T));
  ck[i] = lk;
  atomicAdd(hist + (lk >> (32 - H)), 1);
}

// One CTA: exclusive scan of the 2^H-bucket histogram into starts / cursors; resets the
// histogram for the next build; flags oversized buckets. Warp w owns a contiguous slice of
// buckets and walks it 32 at a time (coalesced), so no per-thread arrays are needed.
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) k_hist_scan(int* __restrict__ hist, int nbuckets,
                                                             int* __restrict__ starts, int* __restrict__ cursor,
                                                             MapFlags* flags) {
  __shared__ int s_warp[kScanThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per_warp = nbuckets / (kScanThreads / 32);  // multiple of 32 (nbuckets >= 1024)
  const int base = warp * per_warp;
  int sum = 0;
#pragma unroll 8
  for (int r = 0; r < per_warp; r += 32) sum += hist[base + r + lane];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
  if (lane == 0) s_warp[warp] = sum;
  __syncthreads();
  if (warp == 0) {
    const int v = s_warp[lane];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += u;
    }
    s_warp[lane] = incl - v;  // exclusive warp offsets
    if (lane == 31) starts[nbuckets] = incl;
  }
  __syncthreads();
  int carry = s_warp[warp];
  int big = 0;
  for (int r = 0; r < per_warp; r += 32) {
    const int idx = base + r + lane;
    const int v = hist[idx];
    big |= v > kMaxBucket;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += u;
    }
    starts[idx] = carry + incl - v;
    cursor[idx] = carry + incl - v;
    hist[idx] = 0;
    carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
  }
  if (__any_sync(0xFFFFFFFFu, big) && lane == 0) flags->big_bucket = 1;
}

__global__ void k_bucket_scatter(const uint32_t* __restrict__ ck, const int32_t* __restrict__ idx, int64_t n,
                                 int* __restrict__ cursor, uint32_t* __restrict__ tk, int32_t* __restrict__ ti, int H) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n) return;
  const uint32_t k = ck[i];
  const int p = atomicAdd(cursor + (k >> (32 - H)), 1);
  tk[p] = k;
  ti[p] = idx[i];
}

// Sort inside each bucket by rank counting (keys are unique, so the result is exact and
// independent of the scatter order); then expand to the packed 63-bit keys.
__global__ void k_bucket_rank(const uint32_t* __restrict__ tk, const int32_t* __restrict__ ti, int64_t n,
                              const int* __restrict__ starts, const MapFlags* flags, uint64_t* __restrict__ keys,
                              int32_t* __restrict__ out_idx, int H) {
  const int64_t p = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (p >= n) return;
  const uint32_t k = tk[p];
  const int b = k >> (32 - H);
  const int s0 = __ldg(starts + b), s1 = __ldg(starts + b + 1);
  if (s1 - s0 > kMaxBucket) return;  // flagged: the host rebuilds with the CUB sort
  int rank = 0;
  for (int q = s0; q < s1; ++q) rank += __ldg(tk + q) < k;
  int by, bz;
  const int T = compact_bits(flags, by, bz);
  const uint64_t c = T ? (static_cast<uint64_t>(k) >> (32 - T)) : 0;
  const int32_t x = static_cast<int32_t>(c >> (by + bz)) + flags->bbox[0];
  const int32_t y = static_cast<int32_t>((c >> bz) & ((uint64_t{1} << by) - 1u)) + flags->bbox[1];
  const int32_t z = static_cast<int32_t>(c & ((uint64_t{1} << bz) - 1u)) + flags->bbox[2];
  keys[s0 + rank] = pack_key_unchecked(x, y, z);
  out_idx[s0 + rank] = ti[p];
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

// Eq. 1 floor + bbox of the floored coordinates (warp-reduced atomics), for 32-bit compact keys
__global__ void k_floor_bbox(const uint64_t* __restrict__ src, const int32_t* __restrict__ src_idx, int64_t n, int s,
                             uint64_t* __restrict__ out, MapFlags* flags) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
  if (i < n) {
    int32_t x, y, z;
    unpack_key(src[i], x, y, z);
    const int64_t f[3] = {floor_div(x, s) * s, floor_div(y, s) * s, floor_div(z, s) * s};
    if (!in_range(f[0]) || !in_range(f[1]) || !in_range(f[2])) {
      const int axis = !in_range(f[0]) ? 0 : (!in_range(f[1]) ? 1 : 2);
      const int64_t j = src_idx ? src_idx[i] : i;
      atomicMin(&flags->bad_floor, static_cast<unsigned long long>(j * 3 + axis));
      out[i] = 0;
    } else {
      out[i] = pack_key_unchecked(static_cast<int32_t>(f[0]), static_cast<int32_t>(f[1]), static_cast<int32_t>(f[2]));
#pragma unroll
      for (int a = 0; a < 3; ++a) mn[a] = mx[a] = static_cast<int>(f[a]);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn[a] = min(mn[a], __shfl_xor_sync(0xFFFFFFFFu, mn[a], o));
      mx[a] = max(mx[a], __shfl_xor_sync(0xFFFFFFFFu, mx[a], o));
    }
  // block reduction first: one atomic per bound per CTA, not per warp (same-address atomics
  // serialise in L2: ~22k of them per 1.2e5-point layer took 11.7 us)
  __shared__ int s_box[32][6];
  const int warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      s_box[warp][a] = mn[a];
      s_box[warp][3 + a] = mx[a];
    }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int a = threadIdx.x;
    int v = s_box[0][a];
    for (int w = 1; w < nw; ++w) v = a < 3 ? min(v, s_box[w][a]) : max(v, s_box[w][a]);
    if (a < 3 ? v != INT_MAX : v != INT_MIN) {
      if (a < 3)
        atomicMin(&flags->fbox[a], v);
      else
        atomicMax(&flags->fbox[a], v);
    }
  }
}

// floored packed key -> left-aligned... (right-aligned) compact u32 key (x, y, z offsets in units of
// the stride, minimal bit widths; order preserving)
__device__ __forceinline__ bool floor_compact_widths(const MapFlags* f, int s, int& bx, int& by, int& bz) {
  bx = bits_for((int64_t{f->fbox[3]} - f->fbox[0]) / s);
  by = bits_for((int64_t{f->fbox[4]} - f->fbox[1]) / s);
  bz = bits_for((int64_t{f->fbox[5]} - f->fbox[2]) / s);
  return bx + by + bz <= 32;
}

__global__ void k_floor_compact(const uint64_t* __restrict__ fl, int64_t n, int s, MapFlags* flags,
                                uint32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n) return;
  int bx, by, bz;
  if (!floor_compact_widths(flags, s, bx, by, bz)) {
    if (i == 0) flags->fwide = 1;
    out[i] = 0;
    return;
  }
  int32_t x, y, z;
  unpack_key(fl[i], x, y, z);
  out[i] = (static_cast<uint32_t>((x - flags->fbox[0]) / s) << (by + bz)) |
           (static_cast<uint32_t>((y - flags->fbox[1]) / s) << bz) | static_cast<uint32_t>((z - flags->fbox[2]) / s);
}

// Eq. 1 output coordinates in ONE cooperative launch (replaces k_floor_bbox, k_floor_compact,
// the CUB radix sort, CUB unique and k_floor_expand: ~10 latency-bound launches per strided
// map). Phases, grid barriers between them (coop_sort.cuh):
//   floor    floored coordinates in registers, range check, CTA-reduced bbox atomics
//   compact  bbox-relative compact keys, (x, y, z) in the minimal bit widths (order preserving);
//            wider than 32 bits: flag fwide and stop (the host redoes it with 64-bit keys)
//   sort     stable LSD passes over only the ceil(bits / 8) digits the keys use
//   unique   first-of-run flags, in-tile ranks + cross-tile prefix, expand to packed keys
template <int E>
__global__ void __launch_bounds__(kCoopThreads) k_floor_unique(const uint64_t* __restrict__ src,
                                                              const int32_t* __restrict__ src_idx, int64_t n, int s,
                                                              int tile, MapFlags* flags, uint32_t* buf0, uint32_t* buf1,
                                                              int* cnt, int* tot, unsigned* bar,
                                                              uint64_t* __restrict__ q_out, int64_t* __restrict__ nsel) {
  const int tid = threadIdx.x;
  const unsigned G = gridDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * tile, t1 = min(n, t0 + tile);
  unsigned target = 0;
  int32_t fc[E][3];
  bool ok[E];
  int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t i = t0 + e * kCoopThreads + tid;
    ok[e] = i < t1;
    fc[e][0] = fc[e][1] = fc[e][2] = 0;
    if (!ok[e]) continue;
    int32_t c[3];
    unpack_key(src[i], c[0], c[1], c[2]);
    int64_t f[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) f[a] = floor_div(c[a], s) * s;
    if (!in_range(f[0]) || !in_range(f[1]) || !in_range(f[2])) {
      const int axis = !in_range(f[0]) ? 0 : (!in_range(f[1]) ? 1 : 2);
      const int64_t j = src_idx ? src_idx[i] : i;
      atomicMin(&flags->bad_floor, static_cast<unsigned long long>(j * 3 + axis));
      continue;  // the build fails on the host; the key is irrelevant
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      fc[e][a] = static_cast<int32_t>(f[a]);
      mn[a] = min(mn[a], fc[e][a]);
      mx[a] = max(mx[a], fc[e][a]);
    }
  }
  {  // CTA-reduced bbox: one atomic per bound per CTA
    __shared__ int s_box[kCoopThreads / 32][6];
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mn[a] = min(mn[a], __shfl_xor_sync(0xFFFFFFFFu, mn[a], o));
        mx[a] = max(mx[a], __shfl_xor_sync(0xFFFFFFFFu, mx[a], o));
      }
    if (lane == 0)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        s_box[warp][a] = mn[a];
        s_box[warp][3 + a] = mx[a];
      }
    __syncthreads();
    if (tid < 6) {
      int v = s_box[0][tid];
      for (int w = 1; w < kCoopThreads / 32; ++w) v = tid < 3 ? min(v, s_box[w][tid]) : max(v, s_box[w][tid]);
      if (tid < 3 ? v != INT_MAX : v != INT_MIN) {
        if (tid < 3)
          atomicMin(&flags->fbox[tid], v);
        else
          atomicMax(&flags->fbox[tid], v);
      }
    }
  }
  grid_barrier(bar, G, target);
  int box[6];
#pragma unroll
  for (int a = 0; a < 6; ++a) box[a] = __ldcg(&flags->fbox[a]);
  const int bx = bits_for((int64_t{box[3]} - box[0]) / s), by = bits_for((int64_t{box[4]} - box[1]) / s),
            bz = bits_for((int64_t{box[5]} - box[2]) / s);
  if (bx + by + bz > 32) {  // uniform across the grid: every CTA read the same bbox
    if (blockIdx.x == 0 && tid == 0) flags->fwide = 1;
    return;
  }
  uint32_t key[E];
#pragma unroll
  for (int e = 0; e < E; ++e)
    key[e] = ok[e] ? static_cast<uint32_t>((static_cast<uint64_t>((fc[e][0] - box[0]) / s) << (by + bz)) |
                                           (static_cast<uint64_t>((fc[e][1] - box[1]) / s) << bz) |
                                           static_cast<uint64_t>((fc[e][2] - box[2]) / s))
                   : 0u;
  const int passes = max(1, (bx + by + bz + 7) / 8);
  for (int pass = 0; pass < passes; ++pass) {
    if (pass > 0) {
      const uint32_t* ki = (pass - 1) % 2 == 0 ? buf0 : buf1;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (ok[e]) key[e] = __ldcg(ki + t0 + e * kCoopThreads + tid);
    }
    int pos[E];
    lsd_pass_positions<E>(key, ok, 8 * pass, pos, cnt, tot, bar, target);
    uint32_t* ko = pass % 2 == 0 ? buf0 : buf1;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (ok[e]) ko[pos[e]] = key[e];
    grid_barrier(bar, G, target);
  }
  const uint32_t* sorted = (passes - 1) % 2 == 0 ? buf0 : buf1;
  int rank[E], carry = 0;
  bool first[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t i = t0 + e * kCoopThreads + tid;
    key[e] = ok[e] ? __ldcg(sorted + i) : 0u;
    first[e] = ok[e] && (i == 0 || __ldcg(sorted + i - 1) != key[e]);
    int excl;
    const int total = block_exclusive_scan(first[e] ? 1 : 0, excl);
    rank[e] = carry + excl;
    carry += total;
  }
  if (tid == 0) cnt[blockIdx.x] = carry;  // unique keys starting in this tile
  grid_barrier(bar, G, target);
  int local = 0;
  for (unsigned c = tid; c < blockIdx.x; c += kCoopThreads) local += __ldcg(cnt + c);
  int dummy;
  const int base = block_exclusive_scan(local, dummy);
  const uint64_t ymask = (1ull << by) - 1ull, zmask = (1ull << bz) - 1ull;
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (first[e]) {
      const uint64_t c = key[e];
      const int32_t x = box[0] + static_cast<int32_t>(c >> (by + bz)) * s;
      const int32_t y = box[1] + static_cast<int32_t>((c >> bz) & ymask) * s;
      const int32_t z = box[2] + static_cast<int32_t>(c & zmask) * s;
      q_out[base + rank[e]] = pack_key_unchecked(x, y, z);
    }
  if (blockIdx.x == G - 1 && tid == 0) *nsel = base + carry;
}

__global__ void k_floor_expand(const uint32_t* __restrict__ ck, const int64_t* __restrict__ count, int s,
                               const MapFlags* flags, uint64_t* __restrict__ out) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= *count || flags->fwide) return;
  int bx, by, bz;
  floor_compact_widths(flags, s, bx, by, bz);
  const uint32_t c = ck[i];
  const int32_t x = flags->fbox[0] + static_cast<int32_t>(c >> (by + bz)) * s;
  const int32_t y = flags->fbox[1] + static_cast<int32_t>((c >> bz) & ((1u << by) - 1u)) * s;
  const int32_t z = flags->fbox[2] + static_cast<int32_t>(c & ((1u << bz) - 1u)) * s;
  out[i] = pack_key_unchecked(x, y, z);
}

// ---------------------------------------------------------------- double-traversed search
constexpr int kSearchThreads = 256;

// Weight offset k generated in registers (weight_offsets_ext order: a outer, b, c inner; odd K
// centred, even K in [0, K-1]; times the signed scale: negative for transposed maps).
// An explicit offset list (SPEC build_kernel_map_sorted(P, Q, offsets, B, C)) is
// read from `tab` instead.
struct OffsetGen {
  int K, scale;
  const int3* tab = nullptr;
  __device__ __forceinline__ int3 at(int k) const {
    if (tab) return tab[k];
    const int lo = (K % 2 == 1) ? -(K / 2) : 0;
    return make_int3((k / (K * K) + lo) * scale, ((k / K) % K + lo) * scale, (k % K + lo) * scale);
  }
};

__device__ __forceinline__ uint64_t pivot_of(const uint64_t* src, int64_t n_src, int B, int64_t b) {
  return __ldg(src + min((b + 1) * B, n_src) - 1);
}

// First block b in [lo, nb) with pivot_b >= key (nb if none). Warp-cooperative: one probe
// of 32 consecutive pivots around `hint` (the expected block: sorted queries land near
// proportional source positions), then 32-way sampling rounds only if the probe misses.
__device__ int64_t warp_first_pivot_ge(const uint64_t* src, int64_t n_src, int B, int64_t lo, int64_t nb,
                                       uint64_t key, int lane, int64_t hint) {
  int64_t hi = nb;  // invariant: answer in [lo, hi]; hi == nb means "none" unless proven
  {
    int64_t start = max(lo, min(hint - 8, nb - 32));
    const int64_t p = start + lane;
    const bool ge = p < nb && pivot_of(src, n_src, B, p) >= key;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, ge);
    if (m) {
      const int f = __ffs(m) - 1;
      if (f > 0 || start == lo) return start + f;
      hi = start;  // answer in [lo, start]
    } else {
      lo = min(nb, start + 32);
    }
  }
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + lane * step;
    const bool ge = p < hi && pivot_of(src, n_src, B, p) >= key;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, ge);
    if (m == 0) {  // answer lies past the last valid sample
      lo = lo + ((hi - 1 - lo) / step) * step + 1;
    } else {
      const int f = __ffs(m) - 1;
      hi = lo + f * step;
      lo = f ? lo + (f - 1) * step + 1 : lo;
    }
  }
  const int64_t p = lo + lane;
  const bool ge = p < hi && pivot_of(src, n_src, B, p) >= key;
  const unsigned m = __ballot_sync(0xFFFFFFFFu, ge);
  return m ? lo + (__ffs(m) - 1) : hi;
}

// Exclusive scan of counts[0, n) -> offs by one CTA (the last to finish): tiles of
// kSearchThreads x 8 values loaded coalesced into registers, scanned, carried.
__device__ void cta_exclusive_scan(const int32_t* counts, int64_t n, int32_t* offs, int64_t nchunk, int32_t* map_start,
                                   int K3, int* s_warp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kPer = 8, kTile = kSearchThreads * kPer;
  int carry = 0;
  for (int64_t base = 0; base < n; base += kTile) {
    int v[kPer];
    int local = 0;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int64_t c = base + int64_t{tid} * kPer + e;
      v[e] = c < n ? __ldcg(counts + c) : 0;
      local += v[e];
    }
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int wprefix = 0, tile_total = 0;
#pragma unroll
    for (int w = 0; w < kSearchThreads / 32; ++w) {
      wprefix += w < warp ? s_warp[w] : 0;
      tile_total += s_warp[w];
    }
    int run = carry + wprefix + incl - local;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int64_t c = base + int64_t{tid} * kPer + e;
      if (c < n) {
        offs[c] = run;
        if (c % nchunk == 0) map_start[c / nchunk] = run;
      }
      run += v[e];
    }
    carry += tile_total;
    __syncthreads();
  }
  if (tid == 0) map_start[K3] = carry;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Output-chunk double-traversed search. A CTA owns CQ = 32*QPL consecutive sorted queries
// q_i and up to 8 offsets, one per warp; warps run independently (no CTA barrier). For its
// offset delta_k a warp's segment keys {q_i + delta_k} lie in [q_first + delta_k,
// q_last + delta_k] (translation preserves lexicographic order), so only the source blocks
// holding that range can match: the warp finds them with two warp-cooperative pivot
// searches and stages them in ITS OWN shared-memory window with one bulk (TMA) copy per
// array (windows above the per-warp capacity are processed in block-aligned slices).
// Per-offset windows are ~CQ keys whatever the cloud density; a window shared by all
// offsets would span every x-slice the offsets reach (~3 slices of a dense cloud).
//   * segment keys of the CQ queries live in registers (lane-major => sorted across lanes);
//   * BACKWARD search: every staged block pivot is compared with the whole sorted segment
//     -> its upper bound, i.e. the block's query sub-range;
//   * FORWARD search: each query is binary-searched only inside its own staged block,
//     <= ceil(log2(B+1)) steps, galloping between a lane's consecutive queries
//     (SPEC.md:226-234).
// Results go to the dense k-major table (coalesced rows) and per-(k, chunk) hit counts.
template <int QPL>
__global__ void __launch_bounds__(kSearchThreads) k_search(
    const uint64_t* __restrict__ src, const int32_t* __restrict__ src_idx, int64_t n_src, int B,
    const uint64_t* __restrict__ q, int64_t n_q, OffsetGen og, int K3, int64_t nchunk, int ngroups,
    int cap_blocks, int32_t* __restrict__ nbr, int32_t* __restrict__ chunk_count) {
  constexpr int CQ = 32 * QPL;
  constexpr int kWarps = kSearchThreads / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t s_bar[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cap = cap_blocks * B;  // keys per warp window
  uint64_t* s_win = reinterpret_cast<uint64_t*>(smem) + int64_t{warp} * cap;
  int32_t* s_widx = reinterpret_cast<int32_t*>(reinterpret_cast<uint64_t*>(smem) + int64_t{kWarps} * cap) +
                    int64_t{warp} * cap;
  const int64_t c = blockIdx.x / ngroups;
  const int grp = static_cast<int>(blockIdx.x - c * ngroups);
  const int k = grp + warp * ngroups;  // this warp's offset
  const int64_t lo = c * CQ;
  const int len = static_cast<int>(min(static_cast<int64_t>(CQ), n_q - lo));
  // the chunk's query keys, staged once per CTA (every warp needs all of them), stored
  // lane-major-transposed: lane L's u-th key (chunk position L*QPL + u) at [u][L], so the
  // per-lane reads below are bank-conflict free
  __shared__ uint64_t s_q[CQ];
  for (int t = threadIdx.x; t < CQ; t += kSearchThreads)
    s_q[(t % QPL) * 32 + t / QPL] = t < len ? __ldg(q + lo + t) : ~uint64_t{0};
  __syncthreads();
  if (k >= K3) return;  // no CTA barrier below
  uint64_t* bar = &s_bar[warp];
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int3 d = og.at(k);
  // lane-contiguous queries: lane L owns chunk positions [L*QPL, (L+1)*QPL), so a lane's
  // consecutive sorted queries can be merged against the sorted block (galloping)
  const int qb = lane * QPL;
  uint64_t key[QPL];
  int res[QPL];
#pragma unroll
  for (int u = 0; u < QPL; ++u) {
    key[u] = qb + u < len ? segment_key(s_q[u * 32 + lane], d) : ~uint64_t{0};
    res[u] = -1;
  }
  const uint64_t key_lo = segment_key(s_q[0], d),
                 key_hi = segment_key(s_q[((len - 1) % QPL) * 32 + (len - 1) / QPL], d);
  const int64_t nb = (n_src + B - 1) / B;
  const int64_t blo =
      warp_first_pivot_ge(src, n_src, B, 0, nb, key_lo, lane, ((lo * n_src) / max(n_q, int64_t{1})) / B);
  const int64_t bhi =
      blo >= nb ? blo : min(warp_first_pivot_ge(src, n_src, B, blo, nb, key_hi, lane, blo + (len + B - 1) / B), nb - 1);
  uint32_t phase = 0;
  for (int64_t sb = blo; sb < nb && sb <= bhi; sb += cap_blocks) {
    const int nblk = static_cast<int>(min(static_cast<int64_t>(cap_blocks), bhi - sb + 1));
    const int64_t g0 = sb * B;
    const int wlen = static_cast<int>(min(static_cast<int64_t>(nblk) * B, n_src - g0));
    if (lane == 0) {  // one bulk copy per array (16-byte granules; arrays carry slack)
      const uint32_t kb = static_cast<uint32_t>((wlen + 3) & ~3);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                   "r"(kb * 8u + (src_idx ? kb * 4u : 0u))
                   : "memory");
      bulk_g2s(s_win, src + g0, kb * 8u, bar);
      if (src_idx) bulk_g2s(s_widx, src_idx + g0, kb * 4u, bar);
    }
    mbar_wait_parity(bar, phase);
    phase ^= 1u;
    // key just below this slice: queries <= it belong to earlier slices
    const uint64_t floor_key = sb == blo ? 0 : __ldg(src + g0 - 1);
    int blk[QPL];  // block of each query inside the slice, -1 = not in this slice
#pragma unroll
    for (int u = 0; u < QPL; ++u) blk[u] = key[u] != ~uint64_t{0} && (sb == blo || key[u] > floor_key) ? 0 : -1;
    // BACKWARD search: each staged pivot splits the sorted segment; queries above pivot_b
    // move to block b+1, above the last pivot they are outside the slice.
    for (int bb = 0; bb < nblk; ++bb) {
      const uint64_t piv = s_win[min((bb + 1) * B, wlen) - 1];
#pragma unroll
      for (int u = 0; u < QPL; ++u)
        if (blk[u] == bb && key[u] > piv) blk[u] = bb + 1 < nblk ? bb + 1 : -1;
    }
    // FORWARD search inside the block: branchless lower bound for the first query of a
    // block, then galloping from the previous position for the following (sorted) ones.
    int p = 0, pblk = -1;
#pragma unroll
    for (int u = 0; u < QPL; ++u) {
      if (blk[u] < 0) continue;
      const int w0 = blk[u] * B, end = w0 + min(B, wlen - w0);
      int base = w0, n = end - w0;  // lower bound of key[u] in [base, base + n), clamped to the last
      if (blk[u] == pblk) {  // same block as the lane's previous (smaller) query: exponential search from p
        if (p < end - 1 && s_win[p] < key[u]) {  // invariant: s_win[lo_] < key
          int lo_ = p, hi_ = p + 1, step = 1;
          while (hi_ < end - 1 && s_win[hi_] < key[u]) {
            lo_ = hi_;
            step <<= 1;
            hi_ = min(p + step, end - 1);
          }
          base = lo_ + 1;
          n = hi_ - lo_;
        } else {
          n = 1;
          base = p;
        }
      }
      while (n > 1) {
        const int h = n >> 1;
        base += s_win[base + h - 1] < key[u] ? h : 0;
        n -= h;
      }
      p = base;
      pblk = blk[u];
      if (s_win[p] == key[u]) res[u] = src_idx ? s_widx[p] : static_cast<int32_t>(g0 + p);
    }
    __syncwarp();  // the next slice overwrites the window
  }
  int32_t* row = nbr + int64_t{k} * n_q + lo + qb;
  int cnt = 0;
#pragma unroll
  for (int u = 0; u < QPL; ++u) {
    if (qb + u < len) row[u] = res[u];
    cnt += __popc(__ballot_sync(0xFFFFFFFFu, res[u] >= 0));
  }
  if (lane == 0) chunk_count[int64_t{k} * nchunk + c] = cnt;
}

// Column variant of k_search for the cubic offset sets (K = 2, 3; no explicit offset list).
// The K offsets sharing (dx, dy) -- a "column" -- differ only in z, and within one (x, y)
// column of a sorted key array z is the last key field: their segment keys are consecutive
// keys of the column. So a warp owns a COLUMN (K^2 warps per CTA instead of K^3 warp tasks):
// it stages one window [q_first + (dx, dy, zmin), q_last + (dx, dy, zmax)] (per-warp bulk copy,
// sliced as in k_search), finds each query's lower bound of its smallest-z key by galloping
// from the lane's previous query, and resolves the K z-offsets by a merge walk (keys between
// two z-offsets of a lattice-aligned set do not exist, so the walk is <= K + a few steps).
// A third of the searches and window copies of k_search and no per-block backward pass; the
// same dense k-major table and per-(k, chunk) hit counts as k_search.
template <int QPL, int KZ>
__global__ void __launch_bounds__(32 * KZ * KZ, KZ == 3 ? 2 : 4) k_search_col(
    const uint64_t* __restrict__ src, const int32_t* __restrict__ src_idx, int64_t n_src, int B,
    const uint64_t* __restrict__ q, int64_t n_q, int scale, int64_t nchunk, int cap_blocks,
    int32_t* __restrict__ nbr, int32_t* __restrict__ chunk_count) {
  constexpr int CQ = 32 * QPL, kWarps = KZ * KZ;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t s_bar[kWarps];
  __shared__ uint64_t s_q[CQ];
  const int lane = threadIdx.x & 31, col = threadIdx.x >> 5;
  const int cap = cap_blocks * B;
  uint64_t* s_win = reinterpret_cast<uint64_t*>(smem) + int64_t{col} * cap;
  int32_t* s_widx = reinterpret_cast<int32_t*>(reinterpret_cast<uint64_t*>(smem) + int64_t{kWarps} * cap) +
                    int64_t{col} * cap;
  const int64_t c = blockIdx.x;
  const int64_t lo = c * CQ;
  const int len = static_cast<int>(min(static_cast<int64_t>(CQ), n_q - lo));
  for (int t = threadIdx.x; t < CQ; t += 32 * kWarps)
    s_q[(t % QPL) * 32 + t / QPL] = t < len ? __ldg(q + lo + t) : ~uint64_t{0};
  __syncthreads();
  uint64_t* bar = &s_bar[col];
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  constexpr int zlo = (KZ % 2 == 1) ? -(KZ / 2) : 0;
  const int dx = (col / KZ + zlo) * scale, dy = (col % KZ + zlo) * scale;
  // z-ascending order of the column's offsets: zi -> tz (scale < 0 for transposed maps)
  auto tz_of = [&](int zi) { return scale > 0 ? zi : KZ - 1 - zi; };
  auto ekey = [&](uint64_t qk, int zi) { return segment_key(qk, make_int3(dx, dy, (tz_of(zi) + zlo) * scale)); };
  const int qb = lane * QPL;
  uint64_t key[QPL];
  int res[QPL][KZ];
  int zn[QPL];  // next unresolved z-offset of each query (KZ: done)
#pragma unroll
  for (int u = 0; u < QPL; ++u) {
    key[u] = s_q[u * 32 + lane];
    zn[u] = qb + u < len ? 0 : KZ;
#pragma unroll
    for (int z = 0; z < KZ; ++z) res[u][z] = -1;
  }
  const uint64_t key_lo = ekey(s_q[0], 0), key_hi = ekey(s_q[((len - 1) % QPL) * 32 + (len - 1) / QPL], KZ - 1);
  const int64_t nb = (n_src + B - 1) / B;
  const int64_t blo =
      warp_first_pivot_ge(src, n_src, B, 0, nb, key_lo, lane, ((lo * n_src) / max(n_q, int64_t{1})) / B);
  const int64_t bhi =
      blo >= nb ? blo : min(warp_first_pivot_ge(src, n_src, B, blo, nb, key_hi, lane, blo + (len + B - 1) / B), nb - 1);
  uint32_t phase = 0;
  for (int64_t sb = blo; sb < nb && sb <= bhi; sb += cap_blocks) {
    const int nblk = static_cast<int>(min(static_cast<int64_t>(cap_blocks), bhi - sb + 1));
    const int64_t g0 = sb * B;
    const int wlen = static_cast<int>(min(static_cast<int64_t>(nblk) * B, n_src - g0));
    if (lane == 0) {
      const uint32_t kb = static_cast<uint32_t>((wlen + 3) & ~3);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                   "r"(kb * 8u + (src_idx ? kb * 4u : 0u))
                   : "memory");
      bulk_g2s(s_win, src + g0, kb * 8u, bar);
      if (src_idx) bulk_g2s(s_widx, src_idx + g0, kb * 4u, bar);
    }
    mbar_wait_parity(bar, phase);
    phase ^= 1u;
    const uint64_t last = s_win[wlen - 1];
    int pprev = 0;  // lower bound of the lane's previous query's smallest-z key (sorted queries)
#pragma unroll
    for (int u = 0; u < QPL; ++u) {
      if (zn[u] >= KZ) continue;
      uint64_t e = ekey(key[u], zn[u]);
      if (e > last) continue;  // beyond this slice
      // lower bound of e in [base, wlen): gallop from the previous query's position
      int base = zn[u] == 0 ? pprev : 0;
      if (s_win[base] < e) {
        int lo_ = base, hi_ = base + 1, step = 1;  // invariant s_win[lo_] < e
        while (hi_ < wlen - 1 && s_win[hi_] < e) {
          lo_ = hi_;
          step <<= 1;
          hi_ = min(base + step, wlen - 1);
        }
        int b = lo_ + 1, n = hi_ - lo_;  // answer in [lo_ + 1, hi_]; s_win[wlen - 1] >= e
        while (n > 1) {
          const int h = n >> 1;
          b += s_win[b + h - 1] < e ? h : 0;
          n -= h;
        }
        base = b;
      }
      if (zn[u] == 0) pprev = base;
      int p = base;
      const int z0 = zn[u];
#pragma unroll
      for (int zi = 0; zi < KZ; ++zi) {
        if (zi < z0) continue;
        if (zi > z0) e = ekey(key[u], zi);
        while (p < wlen && s_win[p] < e) ++p;
        if (p == wlen) break;  // the rest lies in the next slice
        if (s_win[p] == e) {
          res[u][zi] = src_idx ? s_widx[p] : static_cast<int32_t>(g0 + p);  // z order (static index)
          ++p;
        }
        zn[u] = zi + 1;
      }
    }
    __syncwarp();  // the next slice overwrites the window
  }
#pragma unroll
  for (int zi = 0; zi < KZ; ++zi) {
    const int k = col * KZ + tz_of(zi);
    int32_t* row = nbr + int64_t{k} * n_q + lo + qb;
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < QPL; ++u) {
      if (qb + u < len) row[u] = res[u][zi];
      cnt += __popc(__ballot_sync(0xFFFFFFFFu, res[u][zi] >= 0));
    }
    if (lane == 0) chunk_count[int64_t{k} * nchunk + c] = cnt;
  }
}

// Persistent, software-pipelined column search (same result as k_search_col). A CTA owns a
// contiguous range of query chunks; each column warp walks it with a per-warp CURSOR into the
// sorted source: the window start of chunk c + 1 is found from the start of chunk c by one
// warp-wide probe round (32 strided loads; keys only grow along the range), so only the
// CTA's first chunk needs the pivot search. Two window buffers per warp: while chunk c is
// searched, chunk c + 1's window (a fixed W keys from its start, bulk copy) and chunk c + 2's
// probe loads are in flight. A window that does not cover its chunk continues in further
// slices (synchronously, rare). r02: k_search_col spent most of each CTA's life on the
// dependent chain query load -> 2 pivot searches -> window copy -> search, one chunk per CTA.
// Lane state of k_search_colp's queries for the out-of-line direct resolution below.
template <int QPL, int KZ>
struct ColQueries {
  uint64_t k[QPL];
  uint64_t d[KZ];
  int zn[QPL];
  int res[QPL][KZ];
};

// Resolve a lane's unresolved queries of one column directly in global memory: lower bounds by
// interleaved binary searches over [cur, n_src) (independent loads in flight together), then
// the short z-walk. For k_search_colp's scattered chunks only.
template <int QPL, int KZ>
__device__ __noinline__ ColQueries<QPL, KZ> col_resolve_direct(const uint64_t* __restrict__ src,
                                                               const int32_t* __restrict__ src_idx, int n_src, int cur,
                                                               ColQueries<QPL, KZ> st, bool fast, int dx, int dy,
                                                               int scale) {
  constexpr int zlo = (KZ % 2 == 1) ? -(KZ / 2) : 0;
  auto ek = [&](uint64_t qk, int zi) {
    const int tz = scale > 0 ? zi : KZ - 1 - zi;
    uint64_t d = st.d[0];
#pragma unroll
    for (int z = 1; z < KZ; ++z) d = zi == z ? st.d[z] : d;
    return fast ? qk + d : segment_key(qk, make_int3(dx, dy, (tz + zlo) * scale));
  };
  int blo[QPL], blen[QPL];
  uint64_t be[QPL];
#pragma unroll
  for (int u = 0; u < QPL; ++u) {
    be[u] = st.zn[u] < KZ ? ek(st.k[u], st.zn[u]) : 0;
    blo[u] = cur;
    blen[u] = st.zn[u] < KZ ? n_src - cur : 0;
  }
  // 4-ary lower bound: three independent probes per query and step (log4 dependent rounds)
  for (bool any = true; any;) {
    any = false;
    uint64_t v[QPL][3];
#pragma unroll
    for (int u = 0; u < QPL; ++u)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int off = static_cast<int>((static_cast<int64_t>(blen[u]) * (j + 1)) >> 2);
        v[u][j] = blen[u] >= 4 ? __ldg(src + blo[u] + off) : 0;
      }
#pragma unroll
    for (int u = 0; u < QPL; ++u) {
      if (blen[u] <= 0) continue;
      if (blen[u] < 4) {  // binary steps for the last few
        const int h = blen[u] >> 1;
        if (__ldg(src + blo[u] + h) < be[u]) {
          blo[u] += h + 1;
          blen[u] -= h + 1;
        } else {
          blen[u] = h;
        }
      } else {
        // answer in [blo, blo + blen]; probes at offsets o_j = blen (j + 1) / 4
        int lo2 = 0, hi2 = blen[u];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int off = static_cast<int>((static_cast<int64_t>(blen[u]) * (j + 1)) >> 2);
          if (v[u][j] < be[u]) lo2 = off + 1;
        }
#pragma unroll
        for (int j = 2; j >= 0; --j) {
          const int off = static_cast<int>((static_cast<int64_t>(blen[u]) * (j + 1)) >> 2);
          if (v[u][j] >= be[u]) hi2 = off;
        }
        blo[u] += lo2;
        blen[u] = hi2 - lo2;
      }
      any = any || blen[u] > 0;
    }
  }
#pragma unroll
  for (int u = 0; u < QPL; ++u) {
    if (st.zn[u] >= KZ) continue;
    int p = blo[u];
    const int z0 = st.zn[u];
#pragma unroll
    for (int zi = 0; zi < KZ; ++zi) {
      if (zi < z0) continue;
      const uint64_t e = ek(st.k[u], zi);
      uint64_t v = 0;
      while (p < n_src && (v = __ldg(src + p)) < e) ++p;
      if (p == n_src) break;
      if (v == e) {
        st.res[u][zi] = src_idx ? __ldg(src_idx + p) : p;
        ++p;
      }
    }
    st.zn[u] = KZ;
  }
  return st;
}

template <int QPL, int KZ, int W>
__global__ void __launch_bounds__(32 * KZ * KZ, KZ == 3 ? 2 : 4) k_search_colp(
    const uint64_t* __restrict__ src, const int32_t* __restrict__ src_idx, int64_t n_src, int B,
    const uint64_t* __restrict__ q, int64_t n_q, int scale, int64_t nchunk, int probe_stride,
    int32_t* __restrict__ nbr, int32_t* __restrict__ chunk_count, unsigned long long* trace) {
  constexpr int CQ = 32 * QPL, kWarps = KZ * KZ;
  static_assert(W % 4 == 0, "window slices start 16-byte aligned");
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t s_bar[kWarps][2];
  const int lane = threadIdx.x & 31, col = threadIdx.x >> 5;
  uint64_t* s_win = reinterpret_cast<uint64_t*>(smem) + int64_t{col} * 2 * W;  // [2][W]
  int32_t* s_widx = reinterpret_cast<int32_t*>(reinterpret_cast<uint64_t*>(smem) + int64_t{kWarps} * 2 * W) +
                    int64_t{col} * 2 * W;
  const int64_t G = gridDim.x;
  const int64_t cb = blockIdx.x * nchunk / G, ce = (blockIdx.x + 1) * nchunk / G;
  if (cb >= ce) return;
  uint64_t* bar = s_bar[col];
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  constexpr int zlo = (KZ % 2 == 1) ? -(KZ / 2) : 0;
  const int dx = (col / KZ + zlo) * scale, dy = (col % KZ + zlo) * scale;
  auto tz_of = [&](int zi) { return scale > 0 ? zi : KZ - 1 - zi; };
  auto ekey = [&](uint64_t qk, int zi) { return segment_key(qk, make_int3(dx, dy, (tz_of(zi) + zlo) * scale)); };
  // Fast segment keys: a query whose three fields are at least M = KZ |scale| inside the
  // coordinate range gets q + delta by ONE 64-bit add (no field can carry or borrow); the
  // saturating unpack/pack of segment_key is kept for chunks with any query near the range
  // edge (warp-uniform choice per chunk).
  uint64_t D[KZ];
#pragma unroll
  for (int zi = 0; zi < KZ; ++zi)
    D[zi] = (static_cast<uint64_t>(static_cast<int64_t>(dx)) << 42) + (static_cast<uint64_t>(static_cast<int64_t>(dy)) << 21) +
            static_cast<uint64_t>(static_cast<int64_t>((tz_of(zi) + zlo) * scale));
  const uint64_t Mf = static_cast<uint64_t>(KZ) * static_cast<uint64_t>(scale < 0 ? -scale : scale);
  constexpr uint64_t kF = (uint64_t{1} << 42) | (uint64_t{1} << 21) | 1u;
  constexpr uint64_t kCarry = (uint64_t{1} << 63) | (uint64_t{1} << 42) | (uint64_t{1} << 21);
  const uint64_t lowF = (Mf + 1) * kF, highF = Mf * kF;
  auto safe_key = [&](uint64_t k) {
    return (((k ^ lowF ^ (k - lowF)) | (k ^ highF ^ (k + highF))) & kCarry) == 0;
  };
  const int qb = lane * QPL;
  const int64_t nb = (n_src + B - 1) / B;
  auto load_keys = [&](int64_t c, uint64_t (&kk)[QPL]) {
    const int64_t base = c * CQ + qb;
#pragma unroll
    for (int u = 0; u < QPL; ++u) kk[u] = base + u < n_q ? __ldg(q + base + u) : ~uint64_t{0};
  };
  // first position >= cur whose key is >= key, to `step` granularity (a lower bound of the
  // exact position, never past it): 32-lane probe rounds, the stride growing 8x per round
  auto advance = [&](int64_t cur, uint64_t key, uint64_t pv, int step) -> int64_t {
    for (;;) {
      const unsigned m = __ballot_sync(0xFFFFFFFFu, pv >= key);
      if (m) return min(cur + int64_t{step} * (__ffs(m) - 1), n_src);
      cur += int64_t{32} * step;
      if (cur >= n_src) return n_src;
      step *= 8;
      const int64_t p = cur + int64_t{step} * lane + step - 1;
      pv = p < n_src ? __ldg(src + p) : ~uint64_t{0};
    }
  };
  auto probe = [&](int64_t cur) -> uint64_t {
    const int64_t p = cur + int64_t{probe_stride} * lane + probe_stride - 1;
    return p < n_src ? __ldg(src + p) : ~uint64_t{0};
  };
  uint32_t ph0 = 0, ph1 = 0;  // phase per window buffer (scalars: an indexed array would live on the stack)
  auto issue = [&](int buf, int64_t start) -> int {
    const int wlen = static_cast<int>(min(static_cast<int64_t>(W), n_src - start));
    if (wlen > 0 && lane == 0) {
      const uint32_t kb = static_cast<uint32_t>((wlen + 3) & ~3);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[buf])),
                   "r"(kb * 8u + (src_idx ? kb * 4u : 0u))
                   : "memory");
      bulk_g2s(s_win + buf * W, src + start, kb * 8u, &bar[buf]);
      if (src_idx) bulk_g2s(s_widx + buf * W, src_idx + start, kb * 4u, &bar[buf]);
    }
    return wlen;
  };
  // query keys: chunk c's in registers (kc), chunk c + 1's loaded during chunk c (kn), and only
  // the FIRST key of chunk c + 2 (its window start) two chunks ahead (klo)
  uint64_t kc[QPL], kn[QPL];
  load_keys(cb, kc);
  uint64_t klo = cb + 1 < ce ? __ldg(q + (cb + 1) * CQ) : 0;
  // the range's first window: pivot search (block granularity), then one round to 8 keys
  int64_t start_c;
  {
    const uint64_t key_lo = ekey(__shfl_sync(0xFFFFFFFFu, kc[0], 0), 0);
    const int64_t blo =
        n_src == 0 ? 0 : warp_first_pivot_ge(src, n_src, B, 0, nb, key_lo, lane, ((cb * CQ * n_src) / max(n_q, int64_t{1})) / B);
    if (blo >= nb) {
      start_c = n_src;
    } else {
      const int64_t p = blo * B + 8 * lane + 7;
      start_c = advance(blo * B, key_lo, p < n_src ? __ldg(src + p) : ~uint64_t{0}, 8);
    }
  }
  int buf = 0;
  int wlen_c = issue(buf, start_c);
  uint64_t pv = cb + 1 < ce ? probe(start_c) : 0;
  for (int64_t c = cb; c < ce; ++c) {
    const bool has1 = c + 1 < ce, has2 = c + 2 < ce;
    // (a) window of chunk c + 1 from the probe issued one iteration ago; (b) its copy; (c) the
    // probe and query keys of chunk c + 2 -- all in flight during the search of chunk c
    int64_t start_n = n_src;
    int wlen_n = 0;
    if (has1) {
      start_n = advance(start_c, ekey(klo, 0), pv, probe_stride);
      wlen_n = issue(buf ^ 1, start_n);
      load_keys(c + 1, kn);
      if (has2) {
        pv = probe(start_n);
        klo = __ldg(q + (c + 2) * CQ);
      }
    }
    // (d) search chunk c
    int res[QPL][KZ];
    int zn[QPL];
    const int64_t lo = c * CQ;
    const int len = static_cast<int>(min(static_cast<int64_t>(CQ), n_q - lo));
#pragma unroll
    for (int u = 0; u < QPL; ++u) {
      zn[u] = qb + u < len ? 0 : KZ;
#pragma unroll
      for (int z = 0; z < KZ; ++z) res[u][z] = -1;
    }
    bool ok = true;
#pragma unroll
    for (int u = 0; u < QPL; ++u) ok = ok && (qb + u >= len || safe_key(kc[u]));
    const bool fast = __all_sync(0xFFFFFFFFu, ok);
    auto ek = [&](uint64_t qk, int zi) {  // D by selects (a dynamic index would put D on the stack)
      uint64_t d = D[0];
#pragma unroll
      for (int z = 1; z < KZ; ++z) d = zi == z ? D[z] : d;
      return fast ? qk + d : ekey(qk, zi);
    };
    int64_t g0 = start_c;
    int wlen = wlen_c;
    unsigned long long t_begin = 0;
    int nslices = 0;
    if (trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
    while (wlen > 0) {
      ++nslices;
      mbar_wait_parity(&bar[buf], buf ? ph1 : ph0);
      if (buf) ph1 ^= 1u; else ph0 ^= 1u;
      const uint64_t* sw = s_win + buf * W;
      const int32_t* si = s_widx + buf * W;
      const uint64_t last = sw[wlen - 1];
      int pprev = 0;
      bool more = false;
#pragma unroll
      for (int u = 0; u < QPL; ++u) {
        if (zn[u] >= KZ) continue;
        uint64_t e = ek(kc[u], zn[u]);
        if (e > last) {
          more = true;
          continue;
        }
        int base = zn[u] == 0 ? pprev : 0;
        if (base == 0) {  // no earlier position known: branchless lower bound over the window
          int n = wlen;
          while (n > 1) {
            const int h = n >> 1;
            base += sw[base + h - 1] < e ? h : 0;
            n -= h;
          }
        } else if (sw[base] < e) {  // gallop from the lane's previous (smaller) query
          int lo_ = base, hi_ = base + 1, step = 1;
          while (hi_ < wlen - 1 && sw[hi_] < e) {
            lo_ = hi_;
            step <<= 1;
            hi_ = min(base + step, wlen - 1);
          }
          int b = lo_ + 1, n = hi_ - lo_;
          while (n > 1) {
            const int h = n >> 1;
            b += sw[b + h - 1] < e ? h : 0;
            n -= h;
          }
          base = b;
        }
        if (zn[u] == 0) pprev = base;
        int p = base;
        const int z0 = zn[u];
#pragma unroll
        for (int zi = 0; zi < KZ; ++zi) {
          if (zi < z0) continue;
          if (zi > z0) e = ek(kc[u], zi);
          while (p < wlen && sw[p] < e) ++p;
          if (p == wlen) {
            more = true;
            break;
          }
          if (sw[p] == e) {
            res[u][zi] = src_idx ? si[p] : static_cast<int32_t>(g0 + p);
            ++p;
          }
          zn[u] = zi + 1;
        }
      }
      __syncwarp();  // the next slice overwrites this buffer
      if (!__any_sync(0xFFFFFFFFu, more)) break;
      if (nslices >= 2) {
        // Scattered chunk (its queries span many x-slices of the cloud, so a column's targets
        // lie in many separate key ranges: up to ~20 slices at ~5 us each on the S3DIS room,
        // the kernel's tail): resolve the rest directly in global memory (out-of-line: the rare
        // path's registers stay out of the hot loop's allocation).
        ColQueries<QPL, KZ> st;
#pragma unroll
        for (int u = 0; u < QPL; ++u) {
          st.k[u] = kc[u];
          st.zn[u] = zn[u];
#pragma unroll
          for (int z = 0; z < KZ; ++z) st.res[u][z] = res[u][z];
        }
#pragma unroll
        for (int z = 0; z < KZ; ++z) st.d[z] = D[z];
        st = col_resolve_direct<QPL, KZ>(src, src_idx, static_cast<int>(n_src), static_cast<int>(g0 + wlen), st,
                                         fast, dx, dy, scale);
#pragma unroll
        for (int u = 0; u < QPL; ++u)
#pragma unroll
          for (int z = 0; z < KZ; ++z) res[u][z] = st.res[u][z];
        break;
      }
      // rare: the window did not cover the chunk. The next slice starts at the smallest key a
      // query still needs (found by probing forward), not right after this one: a chunk that
      // straddles two x-slices of the cloud needs two narrow key ranges, and staging the whole
      // range between them (up to ~10^4 keys next to a wall plane) made such chunks the
      // kernel's tail.
      uint64_t need = ~uint64_t{0};
#pragma unroll
      for (int u = 0; u < QPL; ++u)
        if (zn[u] < KZ) need = min(need, ek(kc[u], zn[u]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) need = min(need, __shfl_xor_sync(0xFFFFFFFFu, need, o));
      const int64_t cur = g0 + wlen;
      const int64_t p = cur + int64_t{64} * lane + 63;
      g0 = advance(cur, need, p < n_src ? __ldg(src + p) : ~uint64_t{0}, 64);
      wlen = issue(buf, g0);
    }
#pragma unroll
    for (int zi = 0; zi < KZ; ++zi) {
      const int k = col * KZ + tz_of(zi);
      int32_t* row = nbr + int64_t{k} * n_q + lo + qb;
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < QPL; ++u) {
        if (qb + u < len) row[u] = res[u][zi];
        cnt += __popc(__ballot_sync(0xFFFFFFFFu, res[u][zi] >= 0));
      }
      if (lane == 0) chunk_count[int64_t{k} * nchunk + c] = cnt;
    }
    if (trace && lane == 0) {  // diagnostics (SCONV_SEARCH_TRACE): per (chunk, column) timing
      unsigned long long t_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      unsigned long long* tr = trace + (c * kWarps + col) * 4;
      tr[0] = t_begin;
      tr[1] = t_end;
      tr[2] = static_cast<unsigned long long>(nslices) | (static_cast<unsigned long long>(blockIdx.x) << 32);
      tr[3] = static_cast<unsigned long long>(start_c);
    }
    // rotate
#pragma unroll
    for (int u = 0; u < QPL; ++u) kc[u] = kn[u];
    start_c = start_n;
    wlen_c = wlen_n;
    buf ^= 1;
  }
}

// ---------------------------------------------------------------- derived maps (networks)
// K = 2, stride 2s down-sampling map of a fine set P on the s-lattice onto Q = Eq. 1 of P:
// every p has exactly one parent q = floor(p / 2s) * 2s in Q and one offset (p - q) / s in
// {0, 1}^3, so the map is a scatter, not a search: nbr[k(p)][index of q in Q] = p (one binary
// search of q per fine point instead of 8 segment searches per coarse point).
__global__ void k_down_map(const uint64_t* __restrict__ fine, int64_t nf, const uint64_t* __restrict__ coarse,
                           int64_t nc, int s, int32_t* __restrict__ nbr) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= nf) return;
  int32_t c[3];
  unpack_key(__ldg(fine + i), c[0], c[1], c[2]);
  const int64_t S = 2 * int64_t{s};
  int32_t qc[3];
  int k = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    qc[a] = static_cast<int32_t>(floor_div(c[a], S) * S);
    k = 2 * k + static_cast<int>((c[a] - qc[a]) / s);  // 0 or 1 on the s-lattice
  }
  const uint64_t key = pack_key_unchecked(qc[0], qc[1], qc[2]);
  int64_t lo = 0, hi = nc;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(coarse + mid) < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < nc && __ldg(coarse + lo) == key) nbr[int64_t{k} * nc + lo] = static_cast<int32_t>(i);
}

// Transposed map from its forward map: the pairs are the same with input and output swapped
// (offsets negated): dst[k][src[k][i]] = i.
__global__ void k_transpose_map(const int32_t* __restrict__ src, int64_t n_src_out, int K3, int32_t* __restrict__ dst,
                                int64_t n_dst_out) {
  const int64_t g = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (g >= n_src_out * K3) return;
  const int64_t k = g / n_src_out, i = g - k * n_src_out;
  const int32_t j = __ldg(src + g);
  if (j >= 0) dst[k * n_dst_out + j] = static_cast<int32_t>(i);
}

// Per-(k, chunk of CQ queries) hit counts of a dense table (what k_search writes alongside the
// table), for the canonical lists of a derived map.
__global__ void k_chunk_counts(const int32_t* __restrict__ nbr, int64_t n_q, int CQ, int64_t nchunk,
                               int32_t* __restrict__ counts) {
  const int64_t k = blockIdx.y, c = blockIdx.x;
  const int64_t i = c * CQ + threadIdx.x;
  const bool hit = threadIdx.x < CQ && i < n_q && __ldg(nbr + k * n_q + i) >= 0;
  const int cnt = __syncthreads_count(hit);
  if (threadIdx.x == 0) counts[k * nchunk + c] = cnt;
}

// Exclusive scan of the (k, chunk) hit counts in canonical order: each CTA scans a tile of
// kScanTile counts (tile-local offsets + tile total); the last CTA to finish scans the tile
// totals and writes the canonical list starts map_start[k] (= offset of (k, chunk 0)).
constexpr int kScanPer = 8, kScanTile = kSearchThreads * kScanPer;
__global__ void __launch_bounds__(kSearchThreads) k_scan_counts(const int32_t* __restrict__ counts, int64_t n,
                                                                int32_t* __restrict__ offs, int32_t* __restrict__ tiles,
                                                                int64_t nchunk, int K3, int32_t* __restrict__ map_start,
                                                                unsigned* __restrict__ done) {
  __shared__ int s_warp[kSearchThreads / 32];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = int64_t{blockIdx.x} * kScanTile;
  int v[kScanPer];
  int local = 0;
#pragma unroll
  for (int e = 0; e < kScanPer; ++e) {
    const int64_t c = base + int64_t{tid} * kScanPer + e;
    v[e] = c < n ? counts[c] : 0;
    local += v[e];
  }
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  int wprefix = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kSearchThreads / 32; ++w) {
    wprefix += w < warp ? s_warp[w] : 0;
    total += s_warp[w];
  }
  int run = wprefix + incl - local;
#pragma unroll
  for (int e = 0; e < kScanPer; ++e) {
    const int64_t c = base + int64_t{tid} * kScanPer + e;
    if (c < n) offs[c] = run;
    run += v[e];
  }
  if (tid == 0) {
    tiles[blockIdx.x] = total;
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (warp == 0) {  // scan tile totals (serial in 32-wide rounds; few hundred tiles at most)
    int carry = 0;
    for (int t0 = 0; t0 < static_cast<int>(gridDim.x); t0 += 32) {
      const int t = t0 + lane;
      const int x = t < static_cast<int>(gridDim.x) ? __ldcg(tiles + t) : 0;
      int in = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xFFFFFFFFu, in, o);
        if (lane >= o) in += u;
      }
      if (t < static_cast<int>(gridDim.x)) tiles[t] = carry + in - x;
      carry += __shfl_sync(0xFFFFFFFFu, in, 31);
    }
    if (lane == 0) {
      map_start[K3] = carry;
      *done = 0;
    }
  }
  __syncthreads();
  for (int k = tid; k < K3; k += kSearchThreads) {
    const int64_t c = int64_t{k} * nchunk;
    map_start[k] = __ldcg(offs + c) + __ldcg(tiles + c / kScanTile);
  }
}

// Canonical positions: m = chunk_off[k, c] + rank of the hit inside the chunk (query
// order), written to a second table (the input-row table stays for the fused dataflow). One CTA per query chunk; warp w emits offsets k = w, w+8, ... with ballot ranks,
// so no CTA-level barrier is needed.
template <int QPL>
__global__ void __launch_bounds__(kSearchThreads) k_emit(const int32_t* __restrict__ nbr, int32_t* __restrict__ pos,
                                                          int64_t n_q, int K3,
                                                          int64_t nchunk, int ngroups, const int32_t* __restrict__ chunk_off,
                                                          const int32_t* __restrict__ tile_base,
                                                          int32_t* __restrict__ pair_in, int32_t* __restrict__ pair_out) {
  constexpr int CQ = 32 * QPL;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c = blockIdx.x / ngroups;
  const int grp = static_cast<int>(blockIdx.x - c * ngroups);
  const int64_t lo = c * CQ;
  const unsigned lt = (1u << lane) - 1u;
  for (int k = grp + warp * ngroups; k < K3; k += K3) {
    const int32_t* row = nbr + int64_t{k} * n_q + lo;
    int32_t* prow = pos + int64_t{k} * n_q + lo;
    const int64_t ci = int64_t{k} * nchunk + c;
    int base = __ldg(chunk_off + ci) + __ldg(tile_base + ci / kScanTile);
    int32_t j[QPL];
#pragma unroll
    for (int u = 0; u < QPL; ++u) j[u] = lo + u * 32 + lane < n_q ? row[u * 32 + lane] : -1;
#pragma unroll
    for (int u = 0; u < QPL; ++u) {
      const unsigned bal = __ballot_sync(0xFFFFFFFFu, j[u] >= 0);
      if (lo + u * 32 + lane < n_q) {
        int32_t m = -1;
        if (j[u] >= 0) {
          m = base + __popc(bal & lt);
          pair_in[m] = j[u];
          pair_out[m] = static_cast<int32_t>(lo + u * 32 + lane);
        }
        prow[u * 32 + lane] = m;
      }
      base += __popc(bal);
    }
  }
}

// ---------------------------------------------------------------- SPEC-literal sorted search
// Minuet's work decomposition exactly as SPEC.md:208-234 states it, with its counters
// (backend SCONV_MAP_SORTED_SPEC): the counters equal the oracle's bit for bit, which is what
// SPEC acceptance #3 (<= 10 comparisons per query) is asserted on. The default SORTED backend
// (k_search above) is this builder's warp-window redesign of the same search.
enum { kCntBackward = 0, kCntForward = 1, kCntLoaded = 2, kCntExecuted = 3, kNumCounters = 4 };

__device__ __forceinline__ void warp_add_counter(unsigned long long* c, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(c, v);
}

// backward_partition: one thread per (offset k, source block b); the
// upper bound of pivot_b over the virtual segment {q_i + delta_k} (never materialised,
// SPEC.md:199-207), one comparison per bisection step. Also the range count of
// balance_blocks once the previous block's boundary is known (second pass).
__global__ void k_backward_partition(const uint64_t* __restrict__ src, int64_t n_src, int B,
                                     const uint64_t* __restrict__ q, int64_t n_q, OffsetGen og, int K3, int64_t nb,
                                     int64_t* __restrict__ boundary, unsigned long long* __restrict__ counters) {
  const int64_t t = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  unsigned long long cmp = 0;
  if (t < int64_t{K3} * nb) {
    const int k = static_cast<int>(t / nb);
    const int64_t b = t - int64_t{k} * nb;
    const int3 d = og.at(k);
    const uint64_t piv = __ldg(src + min((b + 1) * B, n_src) - 1);
    int64_t lo = 0, hi = n_q;
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      ++cmp;
      if (segment_key(__ldg(q + mid), d) <= piv)
        lo = mid + 1;
      else
        hi = mid;
    }
    boundary[t] = lo;
  }
  warp_add_counter(counters + kCntBackward, cmp);
}

// balance_blocks: ceil(L / C) near-equal ranges per query block.
__global__ void k_range_count(const int64_t* __restrict__ boundary, int64_t nb, int64_t total, int C,
                              int64_t* __restrict__ nranges) {
  const int64_t t = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (t >= total) return;
  const int64_t b = t % nb;
  const int64_t L = boundary[t] - (b ? boundary[t - 1] : 0);
  nranges[t] = L > 0 ? (L + C - 1) / C : 0;
}

struct QueryRange {
  int32_t k;
  int32_t block;
  int64_t lo, hi;
};

__global__ void k_range_emit(const int64_t* __restrict__ boundary, const int64_t* __restrict__ nranges,
                             const int64_t* __restrict__ roff, int64_t nb, int64_t total, QueryRange* __restrict__ out,
                             int64_t* __restrict__ n_out) {
  const int64_t t = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (t >= total) return;
  const int64_t b = t % nb;
  const int64_t start = b ? boundary[t - 1] : 0;
  const int64_t L = boundary[t] - start, parts = nranges[t];
  if (t == total - 1) *n_out = roff[t] + parts;
  if (!parts) return;
  const int64_t base = L / parts, extra = L % parts;  // first `extra` ranges one longer (434/433/433)
  int64_t lo = start;
  for (int64_t p = 0; p < parts; ++p) {
    const int64_t len = base + (p < extra ? 1 : 0);
    out[roff[t] + p] = QueryRange{static_cast<int32_t>(t / nb), static_cast<int32_t>(b), lo, lo + len};
    lo += len;
  }
}

// forward_block_search: one CTA per balanced range; the source block (B keys
// + indices) is staged once in shared memory (the scratchpad copy the SPEC models); each
// query of the range is binary-searched in it (early exit on equality, one comparison per
// probe). Hits go to the nbr table and the per-(k, chunk) counts of the canonical scan.
__global__ void __launch_bounds__(256) k_forward_block_search(
    const uint64_t* __restrict__ src, const int32_t* __restrict__ src_idx, int64_t n_src, int B,
    const uint64_t* __restrict__ q, int64_t n_q, OffsetGen og, const QueryRange* __restrict__ ranges,
    const int64_t* __restrict__ n_ranges, int cq, int64_t nchunk, int32_t* __restrict__ nbr,
    int32_t* __restrict__ chunk_count, unsigned long long* __restrict__ counters) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* s_key = reinterpret_cast<uint64_t*>(smem);
  int32_t* s_idx = reinterpret_cast<int32_t*>(s_key + B);
  const int64_t nr = *n_ranges;
  unsigned long long fwd = 0, loaded = 0, executed = 0;
  for (int64_t r = blockIdx.x; r < nr; r += gridDim.x) {
    const QueryRange R = ranges[r];
    const int64_t begin = int64_t{R.block} * B;
    const int len = static_cast<int>(min(int64_t{B}, n_src - begin));
    __syncthreads();
    for (int e = threadIdx.x; e < len; e += blockDim.x) {
      s_key[e] = __ldg(src + begin + e);
      s_idx[e] = src_idx ? __ldg(src_idx + begin + e) : static_cast<int32_t>(begin + e);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      loaded += static_cast<unsigned long long>(len);
      executed += static_cast<unsigned long long>(R.hi - R.lo);
    }
    const int3 d = og.at(R.k);
    for (int64_t i = R.lo + threadIdx.x; i < R.hi; i += blockDim.x) {
      const uint64_t key = segment_key(__ldg(q + i), d);
      int lo = 0, hi = len;
      while (lo < hi) {
        const int mid = lo + (hi - lo) / 2;
        ++fwd;
        const uint64_t v = s_key[mid];
        if (v == key) {
          nbr[int64_t{R.k} * n_q + i] = s_idx[mid];
          atomicAdd(chunk_count + int64_t{R.k} * nchunk + i / cq, 1);
          break;
        }
        if (v < key)
          lo = mid + 1;
        else
          hi = mid;
      }
    }
  }
  warp_add_counter(counters + kCntForward, fwd);
  warp_add_counter(counters + kCntLoaded, loaded);
  warp_add_counter(counters + kCntExecuted, executed);
}

// ---------------------------------------------------------------- hash-table baseline
// SPEC.md:114-160 (the §3 Shortcoming #1 baseline): open addressing, capacity = smallest power
// of two >= 2N, 64-bit Fibonacci multiplicative hash, linear probing; every (i, k) probes
// pack(q_i + delta_k). Writes the same nbr table and per-(k, chunk) hit counts as k_search, so
// the canonical lists come from the same scan / emit kernels (backend equivalence).
constexpr uint64_t kFib = 0x9E3779B97F4A7C15ull, kEmptySlot = ~uint64_t{0};

__global__ void k_hash_insert(const uint64_t* __restrict__ keys, const int32_t* __restrict__ idx, int64_t n,
                              uint64_t* __restrict__ slot_keys, int32_t* __restrict__ slot_vals, int shift,
                              uint64_t mask) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n) return;
  const uint64_t key = keys[i];
  uint64_t h = (key * kFib) >> shift;
  for (;;) {  // keys are unique: a slot is either empty or another key
    const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(slot_keys + h),
                                              static_cast<unsigned long long>(kEmptySlot),
                                              static_cast<unsigned long long>(key));
    if (prev == kEmptySlot) {
      slot_vals[h] = idx ? idx[i] : static_cast<int32_t>(i);
      return;
    }
    h = (h + 1) & mask;
  }
}

// grid (query chunks of blockDim.x, K3): one query per thread
__global__ void k_hash_query(const uint64_t* __restrict__ q, int64_t n_q, OffsetGen og,
                             const uint64_t* __restrict__ slot_keys, const int32_t* __restrict__ slot_vals, int shift,
                             uint64_t mask, int64_t nchunk, int32_t* __restrict__ nbr, int32_t* __restrict__ counts) {
  const int64_t c = blockIdx.x;
  const int k = blockIdx.y;
  const int64_t i = c * blockDim.x + threadIdx.x;
  int32_t j = -1;
  if (i < n_q) {
    const uint64_t key = segment_key(q[i], og.at(k));  // out of range: saturated, never stored
    uint64_t h = (key * kFib) >> shift;
    for (;;) {
      const uint64_t s = __ldg(slot_keys + h);
      if (s == key) {
        j = __ldg(slot_vals + h);
        break;
      }
      if (s == kEmptySlot) break;
      h = (h + 1) & mask;
    }
    nbr[int64_t{k} * n_q + i] = j;
  }
  const int hits = __syncthreads_count(j >= 0);
  if (threadIdx.x == 0) counts[int64_t{k} * nchunk + c] = hits;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, size): a driver call per
// launch costs host time on the map stream's critical path
void set_max_smem(const void* kern, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;  // (kernel, device) -> largest size set
  int dev = 0;
  SCONV_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = done[{kern, dev}];
  if (smem <= cur) return;
  SCONV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cur = smem;
}

constexpr int kThreads = 256;
// Key / index arrays carry slack so 16-byte bulk copies may run past the last element.
inline int64_t slack(int64_t n) { return ((n + 3) & ~int64_t{3}) + 4; }
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

namespace {
void launch_canonical(Ctx& ctx, MapData& m) {
  auto& pd = m.pending;
  const cudaStream_t st = ctx.stream;
  if (pd.counts_from_nbr) {  // derived map: per-(k, chunk) counts from its table
    const int CQ = 32 * pd.qpl;
    ctx.launch("k_chunk_counts", [&] {
      k_chunk_counts<<<dim3(static_cast<unsigned>(pd.nchunk), static_cast<unsigned>(m.K3)), CQ, 0, st>>>(
          m.nbr_in.get<int32_t>(), m.n_out, CQ, pd.nchunk, pd.counts.get<int32_t>());
    });
  }
  if (!m.nbr_pos.get()) m.nbr_pos.alloc(sizeof(int32_t) * std::max<int64_t>(1, int64_t{m.K3} * m.n_out), st);
  if (!m.pair_in.get()) {
    m.pair_in.alloc(sizeof(int32_t) * std::max<int64_t>(1, pd.max_pairs), st);
    m.pair_out.alloc(sizeof(int32_t) * std::max<int64_t>(1, pd.max_pairs), st);
  }
  ctx.launch("k_scan_counts", [&] {
    k_scan_counts<<<static_cast<unsigned>(pd.ntiles), kSearchThreads, 0, st>>>(
        pd.counts.get<int32_t>(), pd.grid, pd.offs.get<int32_t>(), pd.tiles.get<int32_t>(), pd.nchunk, m.K3,
        m.map_start.get<int32_t>(), ctx.done_counter());
  });
  auto emit = [&](auto kern) {
    ctx.launch("k_emit", [&] {
      kern<<<static_cast<unsigned>(pd.nchunk * pd.ngroups), kSearchThreads, 0, st>>>(
          m.nbr_in.get<int32_t>(), m.nbr_pos.get<int32_t>(), m.n_out, m.K3, pd.nchunk, pd.ngroups,
          pd.offs.get<int32_t>(), pd.tiles.get<int32_t>(), m.pair_in.get<int32_t>(), m.pair_out.get<int32_t>());
    });
  };
  switch (pd.qpl) {
    case 1: emit(k_emit<1>); break;
    case 2: emit(k_emit<2>); break;
    case 4: emit(k_emit<4>); break;
    default: emit(k_emit<8>); break;
  }
}

// flags + list starts -> host (one sync); sizes / total
void read_starts(Ctx& ctx, MapData& m, const void* flags, MapFlags* f) {
  const int K3 = m.K3;
  if (sizeof(MapFlags) + sizeof(int32_t) * (K3 + 1) > Ctx::kPinReadbackBytes) fail(SCONV_ERR_ARG, "kernel too large");
  auto* pin2 = static_cast<unsigned char*>(ctx.pin_readback());
  if (flags) {
    d2h_small(pin2, flags, sizeof(MapFlags), ctx.stream);
  } else {  // lazy map over validated keys: its flags were never initialised (nothing to check)
    std::memset(pin2, 0, sizeof(MapFlags));
    std::memset(pin2, 0xFF, 3 * sizeof(unsigned long long));
  }
  d2h_small(pin2 + sizeof(MapFlags), m.map_start.get(), sizeof(int32_t) * (K3 + 1), ctx.stream);
  ctx.sync();
  std::memcpy(f, pin2, sizeof(MapFlags));
  m.starts.resize(K3 + 1);
  std::memcpy(m.starts.data(), pin2 + sizeof(MapFlags), sizeof(int32_t) * (K3 + 1));
  m.sizes.resize(K3);
  for (int k = 0; k < K3; ++k) m.sizes[k] = m.starts[k + 1] - m.starts[k];
  m.total = m.starts[K3];
}
}  // namespace

void launch_identity(Ctx& ctx, MapData& m) {
  if (!m.identity_pending) return;
  m.identity_pending = false;
  const int64_t n = m.n_out;
  if (!m.nbr_pos.get()) m.nbr_pos.alloc(sizeof(int32_t) * std::max<int64_t>(1, n), ctx.stream);
  ctx.launch("k_identity_map", [&] {
    k_identity_map<<<grid_for(n), kThreads, 0, ctx.stream>>>(n, m.nbr_in.get<int32_t>(), m.nbr_pos.get<int32_t>(),
                                                             m.pair_in.get<int32_t>(), m.pair_out.get<int32_t>(),
                                                             m.map_start.get<int32_t>());
  });
}

void ensure_canonical(Ctx& ctx, MapData& m) {
  launch_identity(ctx, m);
  if (m.canonical) return;
  if (m.pending.grid > 0) launch_canonical(ctx, m);
  MapFlags f;
  read_starts(ctx, m, m.pending.flags_init ? m.pending.flags.get() : nullptr, &f);  // lazy: no coordinate checks
  m.pending = MapData::Pending{};
  m.canonical = true;
}

bool finish_coords(Ctx& ctx, MapData& m) {
  if (m.n_out >= 0) return true;
  auto* pin = reinterpret_cast<MapFlags*>(ctx.pin_flags());
  d2h_small(pin, m.pending.flags.get(), sizeof(MapFlags), ctx.stream);
  d2h_small(&pin[1], m.pend_nsel.get(), sizeof(int64_t), ctx.stream);
  ctx.sync();
  const MapFlags f = pin[0];
  if (f.fwide || f.wide || f.big_bucket) return false;  // the caller rebuilds with the exact path
  if (f.bad_floor != ULLONG_MAX) {
    const int64_t j = static_cast<int64_t>(f.bad_floor / 3);
    const int axis = static_cast<int>(f.bad_floor % 3);
    uint64_t key;
    SCONV_CUDA(cudaMemcpy(&key, m.src_keys_ptr() + j, sizeof(key), cudaMemcpyDeviceToHost));
    int32_t c[3];
    unpack_key(key, c[0], c[1], c[2]);
    fail(SCONV_ERR_RANGE, coord_error("xyz"[axis], floor_div(c[axis], m.cfg.out_stride) * m.cfg.out_stride));
  }
  std::memcpy(&m.n_out, &pin[1], sizeof(int64_t));
  return true;
}

void check_deferred_map_flags(const void* flags_host, const MapSource& P) {
  static_assert(sizeof(MapFlags) <= kDeferredFlagsBytes, "deferred flags slot");
  MapFlags f;
  std::memcpy(&f, flags_host, sizeof(f));
  if (f.bad_coord != ULLONG_MAX) {
    const int64_t i = static_cast<int64_t>(f.bad_coord / 3);
    const int axis = static_cast<int>(f.bad_coord % 3);
    int32_t c[3];
    if (P.mem == SCONV_MEM_HOST)
      std::memcpy(c, P.xyz + 3 * i, sizeof(c));
    else
      SCONV_CUDA(cudaMemcpy(c, P.xyz + 3 * i, sizeof(c), cudaMemcpyDeviceToHost));
    fail(SCONV_ERR_RANGE, coord_error("xyz"[axis], c[axis]));
  }
  if (f.unsorted) fail(SCONV_ERR_ARG, "input coordinates flagged sorted are not strictly increasing");
}

std::unique_ptr<MapData> build_map(Ctx& ctx, const MapSource& P, const sconv_map_cfg& cfg, const MapSource* target,
                                   bool force_wide, bool lazy, const std::vector<int3>* explicit_offsets,
                                   void* defer_flags, bool coords_only, const MapSource* strided_q,
                                   cudaEvent_t src_ready,
                                   const std::function<void(const std::shared_ptr<DevBuf>&)>& on_src_ready) {
  auto hmark = [&](const char* what) { ctx.hmark(what); };
  hmark("map: enter");
  if (cfg.block_B < 4 || cfg.block_B > 1024 || cfg.block_B % 4 != 0)
    fail(SCONV_ERR_ARG, "block size B must be a multiple of 4 in [4, 1024]");
  if (cfg.block_C < 1 || cfg.block_C > 4096) fail(SCONV_ERR_ARG, "query block size C must be in [1, 4096]");
  if (!cfg.transposed && cfg.out_stride < 1) fail(SCONV_ERR_ARG, "stride must be positive");
  if (P.n < 0 || P.n > INT32_MAX / 2) fail(SCONV_ERR_ARG, "point count out of supported range");
  if (cfg.backend != SCONV_MAP_SORTED && cfg.backend != SCONV_MAP_HASH && cfg.backend != SCONV_MAP_SORTED_SPEC)
    fail(SCONV_ERR_ARG, "unknown map backend");
  const bool explicit_q = explicit_offsets != nullptr;  // SPEC build_kernel_map_sorted(P, Q, offsets, B, C)
  if (explicit_q && (cfg.transposed || !target)) fail(SCONV_ERR_ARG, "explicit offsets need explicit queries");
  // coordinates given as xyz need the flags readback (range / order checks) before the map is
  // used, so such a build syncs; the canonical lists can still be deferred
  const bool defer_canonical = lazy;
  if (lazy && (!P.keys || (cfg.transposed && (!target || !target->keys)))) lazy = false;
  auto m = std::make_unique<MapData>();
  m->cfg = cfg;
  m->n_in = P.n;
  const cudaStream_t st = ctx.stream;
  std::vector<int3> delta =
      explicit_q ? *explicit_offsets : weight_offsets_ext(cfg.kernel_size, cfg.offset_scale);
  if (cfg.transposed)
    for (auto& d : delta) d = make_int3(-d.x, -d.y, -d.z);
  // any int32 offsets are searchable: segment keys saturate outside the coordinate range
  if (explicit_q && (delta.empty() || delta.size() > 4096)) fail(SCONV_ERR_ARG, "offset count must be in [1, 4096]");
  m->K3 = static_cast<int>(delta.size());
  m->delta = delta;
  if (explicit_q) {  // (pageable source: the copy is staged before the call returns)
    m->delta_dev.alloc(sizeof(int3) * delta.size(), st);
    SCONV_CUDA(cudaMemcpyAsync(m->delta_dev.get(), m->delta.data(), sizeof(int3) * delta.size(),
                               cudaMemcpyHostToDevice, st));
  }
  const int K3 = m->K3;
  const int64_t n = P.n;

  DevBuf flags_buf;
  flags_buf.alloc(sizeof(MapFlags), st);
  MapFlags* flags = flags_buf.get<MapFlags>();
  // initialised on the device: lazy builds end without a sync, so no host staging buffer may be
  // reused by the next build while this build's copies are still queued
  // flags are written only by coordinate packing / Eq. 1 floor (raw coordinates, strided
  // layers); chained stride-1 / transposed maps over existing keys skip the init launch
  if (coords_only && (!P.keys || cfg.transposed || cfg.out_stride == 1 || explicit_offsets || target))
    fail(SCONV_ERR_ARG, "coordinates-only builds need a strided map over existing sorted keys");
  if (strided_q && (cfg.transposed || cfg.out_stride == 1 || explicit_offsets || target || !strided_q->keys))
    fail(SCONV_ERR_ARG, "precomputed output coordinates need a strided, non-transposed map");
  const bool flags_used = !lazy || !P.keys || (!cfg.transposed && cfg.out_stride != 1 && !strided_q) ||
                          (cfg.transposed && target && !target->keys);
  if (flags_used) ctx.launch("k_init_flags", [&] { k_init_flags<<<1, 1, 0, st>>>(flags); });
  auto* pin = reinterpret_cast<MapFlags*>(ctx.pin_flags());

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
      m->src_keys->alloc(sizeof(uint64_t) * slack(n), st);
      if (n > 0)
        ctx.launch("k_pack_keys", [&] {
          k_pack_keys<<<grid_for(n), kThreads, 0, st>>>(xyz, n, m->src_keys->get<uint64_t>(), 1, flags, 0);
        });
      m->src_identity = true;
    } else if (!force_wide) {
      // bbox -> left-aligned compact u32 keys + bucket histogram -> scan -> bucket scatter
      // -> in-bucket rank: 5 launches instead of CUB's 8-digit 64-bit onesweep passes.
      DevBuf ck, iota, tk, ti;
      ck.alloc(sizeof(uint32_t) * n, st);
      iota.alloc(sizeof(int32_t) * n, st);
      tk.alloc(sizeof(uint32_t) * n, st);
      ti.alloc(sizeof(int32_t) * n, st);
      m->src_keys->alloc(sizeof(uint64_t) * slack(n), st);
      m->src_idx.alloc(sizeof(int32_t) * slack(n), st);
      if (n > 0) {
        int* hist = ctx.sort_hist();
        int* starts = hist + kBuckets;
        int* cursor = starts + kBuckets + 1;
        // 2^H buckets, ~4 keys per bucket on average (H in [10, 16])
        int H = 10;
        while (H < kMaxBucketBits && (int64_t{1} << (H + 2)) < n) ++H;
        const unsigned bb = static_cast<unsigned>(std::min<int64_t>(grid_for(n), ctx.num_sms));
        ctx.launch("k_bbox", [&] { k_bbox<<<bb, kThreads, 0, st>>>(xyz, n, flags); });
        ctx.launch("k_pack_compact", [&] {
          k_pack_compact<<<grid_for(n), kThreads, 0, st>>>(xyz, n, flags, ck.get<uint32_t>(), iota.get<int32_t>(),
                                                           hist, H);
        });
        ctx.launch("k_hist_scan", [&] { k_hist_scan<<<1, kScanThreads, 0, st>>>(hist, 1 << H, starts, cursor, flags); });
        ctx.launch("k_bucket_scatter", [&] {
          k_bucket_scatter<<<grid_for(n), kThreads, 0, st>>>(ck.get<uint32_t>(), iota.get<int32_t>(), n, cursor,
                                                             tk.get<uint32_t>(), ti.get<int32_t>(), H);
        });
        ctx.launch("k_bucket_rank", [&] {
          k_bucket_rank<<<grid_for(n), kThreads, 0, st>>>(tk.get<uint32_t>(), ti.get<int32_t>(), n, starts, flags,
                                                          m->src_keys->get<uint64_t>(), m->src_idx.get<int32_t>(), H);
        });
      }
      m->src_identity = false;
      m->sorts = 1;
    } else {
      DevBuf raw, iota;
      raw.alloc(sizeof(uint64_t) * n, st);
      iota.alloc(sizeof(int32_t) * n, st);
      m->src_keys->alloc(sizeof(uint64_t) * slack(n), st);
      m->src_idx.alloc(sizeof(int32_t) * slack(n), st);
      if (n > 0) {
        ctx.launch("k_pack_keys", [&] {
          k_pack_keys<<<grid_for(n), kThreads, 0, st>>>(xyz, n, raw.get<uint64_t>(), 0, flags, 0);
        });
        ctx.launch("k_iota", [&] { k_iota<<<grid_for(n), kThreads, 0, st>>>(iota.get<int32_t>(), n); });
        sort_pairs(ctx, raw.get<uint64_t>(), m->src_keys->get<uint64_t>(), iota.get<int32_t>(),
                   m->src_idx.get<int32_t>(), n);
      }
      m->src_identity = false;
      m->sorts = 1;
    }
  }
  if (src_ready) SCONV_CUDA(cudaEventRecord(src_ready, st));  // sorted source keys complete
  if (on_src_ready) on_src_ready(m->src_keys);
  const uint64_t* src = m->src_keys_ptr();
  const int32_t* src_idx = m->src_identity ? nullptr : m->src_idx.get<int32_t>();

  // ---- output coordinates Q
  bool need_nout_sync = false;
  DevBuf fl, fs;  // strided: floored keys / sort scratch (function scope: the wide fallback reuses them)
  std::function<void()> strided_wide;
  DevBuf nsel, coop_aux;
  DevBuf target_xyz_dev;
  if (cfg.transposed || explicit_q) {
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
      m->q_keys->alloc(sizeof(uint64_t) * slack(target->n), st);
      if (target->n > 0)
        ctx.launch("k_pack_keys", [&] {
          k_pack_keys<<<grid_for(target->n), kThreads, 0, st>>>(txyz, target->n, m->q_keys->get<uint64_t>(), 1,
                                                                 flags, 1);
        });
    }
    m->n_out = target->n;
  } else if (strided_q) {  // Eq. 1 output computed earlier (coords_only build + finish_coords)
    m->q_keys = strided_q->keys;
    m->n_out = strided_q->n;
  } else if (cfg.out_stride == 1) {
    m->q_keys = m->src_keys;  // stride-1 alias: one array serves as source and query
    m->n_out = n;
  } else {
    ++m->sorts;  // Eq. 1: floor, sort, unique (geometry.hpp:161-178)
    fl.alloc(sizeof(uint64_t) * std::max<int64_t>(n, 1), st);
    fs.alloc(sizeof(uint64_t) * std::max<int64_t>(n, 1), st);
    m->q_keys = std::make_shared<DevBuf>();
    m->q_keys->alloc(sizeof(uint64_t) * slack(n), st);
    nsel.alloc(sizeof(int64_t), st);
    if (n > 0) {
      // Eq. 1 on device: floor -> 32-bit bbox-relative compact keys (4 radix passes instead of 8)
      // -> sort -> unique -> expand; the 64-bit path below runs only if the compact key is wide.
      static const int coop_cap = [] {
        int per_sm = 0, dev = 0, sms = 0, coop = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_floor_unique<kCoopMaxE>, kCoopThreads, 0) !=
            cudaSuccess)
          per_sm = 0;
        return coop ? per_sm * sms : 0;
      }();
      const bool one_launch = coop_cap > 0 && n <= static_cast<int64_t>(coop_cap) * kCoopThreads * kCoopMaxE &&
                              !(std::getenv("SCONV_FLOOR_CUB") && std::getenv("SCONV_FLOOR_CUB")[0] == '1');
      if (one_launch) {  // everything below in one cooperative launch
        int e = coop_rows_per_thread();
        while (ceil_div<int64_t>(n, int64_t{kCoopThreads} * e) > coop_cap) e *= 2;
        const int tile = kCoopThreads * e;
        const unsigned G = static_cast<unsigned>(ceil_div<int64_t>(n, tile));
        coop_aux.alloc(sizeof(int) * (256 * static_cast<size_t>(G) + 256 + 4), st);
        int* cnt = coop_aux.get<int>();
        int* tot = cnt + 256 * static_cast<size_t>(G);
        unsigned* bar = reinterpret_cast<unsigned*>(tot + 256);
        SCONV_CUDA(cudaMemsetAsync(bar, 0, 4 * sizeof(unsigned), st));
        uint32_t* b0 = reinterpret_cast<uint32_t*>(fs.get<uint64_t>());  // fs is 8n bytes: two u32 arrays
        uint32_t* b1 = b0 + n;
        int64_t nn = n;
        int sv = cfg.out_stride, tilev = tile;
        uint64_t* qo = m->q_keys->get<uint64_t>();
        int64_t* ns = nsel.get<int64_t>();
        MapFlags* fl_ = flags;
        const int32_t* si = src_idx;
        const uint64_t* sk = src;
        void* args[] = {&sk, &si, &nn, &sv, &tilev, &fl_, &b0, &b1, &cnt, &tot, &bar, &qo, &ns};
        const void* fn = e == 1   ? reinterpret_cast<const void*>(k_floor_unique<1>)
                         : e == 2 ? reinterpret_cast<const void*>(k_floor_unique<2>)
                                  : reinterpret_cast<const void*>(k_floor_unique<4>);
        ctx.launch("k_floor_unique", [&] {
          SCONV_CUDA(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kCoopThreads), args, 0, st));
        });
      } else {
      ctx.launch("k_floor_keys", [&] {
        k_floor_bbox<<<grid_for(n), kThreads, 0, st>>>(src, src_idx, n, cfg.out_stride, fl.get<uint64_t>(), flags);
      });
      uint32_t* c32 = reinterpret_cast<uint32_t*>(fs.get<uint64_t>());  // fs is 8n bytes: two u32 arrays
      uint32_t* s32 = c32 + n;
      ctx.launch("k_floor_compact", [&] {
        k_floor_compact<<<grid_for(n), kThreads, 0, st>>>(fl.get<uint64_t>(), n, cfg.out_stride, flags, c32);
      });
      {
        size_t temp = 0;
        SCONV_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, temp, c32, s32, static_cast<int>(n), 0, 32, st));
        ctx.scratch_sort.reserve(temp, st);
        ctx.launch("cub_radix_sort_keys", [&] {
          cub::DeviceRadixSort::SortKeys(ctx.scratch_sort.get(), temp, c32, s32, static_cast<int>(n), 0, 32, st);
        });
      }
      uint32_t* u32 = reinterpret_cast<uint32_t*>(fl.get<uint64_t>());  // floored keys no longer needed
      size_t temp = 0;
      SCONV_CUDA(cub::DeviceSelect::Unique(nullptr, temp, s32, u32, nsel.get<int64_t>(), n, st));
      ctx.scratch_misc.reserve(temp, st);
      ctx.launch("cub_select_unique", [&] {
        cub::DeviceSelect::Unique(ctx.scratch_misc.get(), temp, s32, u32, nsel.get<int64_t>(), n, st);
      });
      ctx.launch("k_floor_expand", [&] {
        k_floor_expand<<<grid_for(n), kThreads, 0, st>>>(u32, nsel.get<int64_t>(), cfg.out_stride, flags,
                                                          m->q_keys->get<uint64_t>());
      });
      }
      need_nout_sync = true;
      strided_wide = [&, n] {  // exact 64-bit fallback (coordinate span beyond 32 compact bits)
        ctx.launch("k_floor_keys", [&] {
          k_floor_keys<<<grid_for(n), kThreads, 0, st>>>(src, src_idx, n, cfg.out_stride, fl.get<uint64_t>(), flags);
        });
        sort_keys(ctx, fl.get<uint64_t>(), fs.get<uint64_t>(), n);
        size_t t2 = 0;
        SCONV_CUDA(cub::DeviceSelect::Unique(nullptr, t2, fs.get<uint64_t>(), m->q_keys->get<uint64_t>(),
                                             nsel.get<int64_t>(), n, st));
        ctx.scratch_misc.reserve(t2, st);
        ctx.launch("cub_select_unique", [&] {
          cub::DeviceSelect::Unique(ctx.scratch_misc.get(), t2, fs.get<uint64_t>(), m->q_keys->get<uint64_t>(),
                                    nsel.get<int64_t>(), n, st);
        });
      };
    } else {
      m->n_out = 0;
    }
  }

  hmark("source + Q queued");
  if (coords_only) {  // Eq. 1 queued; |Q| and the flags are read by finish_coords
    m->pending.flags = std::move(flags_buf);
    m->pending.flags_init = true;
    m->pend_nsel = std::move(nsel);
    m->n_out = -1;
    return m;
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
    d2h_small(pin, flags, sizeof(MapFlags), st);
    d2h_small(&pin[1], nsel.get(), sizeof(int64_t), st);
    static_assert(2 * sizeof(MapFlags) <= Ctx::kPinFlagsBytes, "pinned flags region");
    ctx.sync();
    // the input sort's compact key was too wide: P's keys are not valid yet, so nothing derived
    // from them (floors, their range errors) is either; redo with the exact 64-bit sort first
    if (!force_wide && (pin[0].wide || pin[0].big_bucket)) return build_map(ctx, P, cfg, target, true, defer_canonical);
    check_flags(pin[0]);
    if (pin[0].fwide && strided_wide) {  // rare: redo the output coordinates with 64-bit keys
      strided_wide();
      d2h_small(&pin[1], nsel.get(), sizeof(int64_t), st);
      ctx.sync();
    }
    int64_t nout;
    std::memcpy(&nout, &pin[1], sizeof(int64_t));
    m->n_out = nout;
  }
  hmark("after n_out sync");
  const int64_t n_out = m->n_out;
  const uint64_t* q = m->q_keys_ptr();

  // ---- search
  hmark("map: search allocs");
  m->map_start.alloc(sizeof(int32_t) * (K3 + 1), st);
  m->nbr_in.alloc(sizeof(int32_t) * std::max<int64_t>(1, int64_t{K3} * n_out), st);
  const int B = cfg.block_B, C = cfg.block_C;
  // upper bound on the match count: every query hits at most once
  const int64_t max_pairs = std::min<int64_t>(int64_t{K3} * n_out, int64_t{K3} * n);
  if (max_pairs > INT32_MAX) fail(SCONV_ERR_ARG, "kernel map too large: more than 2^31 - 1 pairs");
  m->pending.max_pairs = max_pairs;
  // canonical positions and pair lists: allocated with the canonical build (launch_canonical),
  // so lazy network maps that never need them (fused convs) skip 3 allocations of up to K3 |Q|
  if (!defer_canonical || n == 0 || n_out == 0)
    m->nbr_pos.alloc(sizeof(int32_t) * std::max<int64_t>(1, int64_t{K3} * n_out), st);
  if (n == 0 || n_out == 0) {
    SCONV_CUDA(cudaMemsetAsync(m->map_start.get(), 0, sizeof(int32_t) * (K3 + 1), st));
    if (n_out > 0) SCONV_CUDA(cudaMemsetAsync(m->nbr_in.get(), 0xFF, sizeof(int32_t) * int64_t{K3} * n_out, st));
    if (n_out > 0)
      SCONV_CUDA(cudaMemsetAsync(m->nbr_pos.get(), 0xFF, sizeof(int32_t) * int64_t{K3} * n_out, st));
  } else if (!explicit_q && K3 == 1 && cfg.kernel_size == 1 && !cfg.transposed && cfg.out_stride == 1 && m->src_identity &&
             m->q_keys == m->src_keys) {
    // identity map (1x1 conv on the same sorted coordinates): no search, sizes known on the host
    m->pair_in.alloc(sizeof(int32_t) * n, st);
    m->pair_out.alloc(sizeof(int32_t) * n, st);
    m->identity_pending = true;  // the fused kernel reads a null table as identity
    if (!lazy) launch_identity(ctx, *m);
    m->starts = {0, static_cast<int32_t>(n)};
    m->sizes = {n};
    m->total = n;
    if (lazy) return m;  // nothing pending; flags were not touched
  } else {
    // Work item = one CTA per chunk of CQ = 32*QPL sorted queries (CQ <= C), all offsets.
    static const bool col_search = [] {
      const char* e = std::getenv("SCONV_SEARCH_COL");  // A/B: 0 = one warp per offset
      return !(e && e[0] == '0');
    }();
    const bool use_col = col_search && !explicit_q && (cfg.kernel_size == 2 || cfg.kernel_size == 3) && C >= 128 &&
                         cfg.backend == SCONV_MAP_SORTED;
    const int qpl = use_col ? 4 : (C >= 256 ? 8 : (C >= 128 ? 4 : (C >= 64 ? 2 : 1)));
    const int CQ = 32 * qpl;
    const int64_t nchunk2 = ceil_div<int64_t>(n_out, CQ);
    const int64_t grid2 = nchunk2 * K3;
    if (grid2 > INT32_MAX) fail(SCONV_ERR_ARG, "kernel map too large");
    DevBuf counts, offs, tiles;
    const int64_t ntiles = ceil_div<int64_t>(grid2, kScanTile);
    hmark("map: table allocs done");
    counts.alloc(sizeof(int32_t) * grid2, st);
    offs.alloc(sizeof(int32_t) * grid2, st);
    tiles.alloc(sizeof(int32_t) * ntiles, st);
    if (!defer_canonical) {
      m->pair_in.alloc(sizeof(int32_t) * std::max<int64_t>(1, max_pairs), st);
      m->pair_out.alloc(sizeof(int32_t) * std::max<int64_t>(1, max_pairs), st);
    }
    hmark("map: pair allocs done");
    const int ngroups = ceil_div(K3, kSearchThreads / 32);  // search / emit CTA = chunk x <= 8 offsets
    const OffsetGen og{cfg.kernel_size, cfg.transposed ? -cfg.offset_scale : cfg.offset_scale,
                       explicit_q ? m->delta_dev.get<int3>() : nullptr};
    if (cfg.backend == SCONV_MAP_SORTED_SPEC) {
      // SPEC-literal decomposition with counters: backward_partition per (k, block) ->
      // balance_blocks (ceil(L/C) near-equal ranges) -> forward_block_search per range
      const int64_t nb = ceil_div<int64_t>(n, B), tot = int64_t{K3} * nb;
      const int64_t max_ranges = int64_t{K3} * (nb + ceil_div<int64_t>(n_out, C));
      DevBuf bnd, nrg, roff, rng, nrs, tmp;
      bnd.alloc(8 * tot, st);
      nrg.alloc(8 * tot, st);
      roff.alloc(8 * tot, st);
      nrs.alloc(8, st);
      rng.alloc(sizeof(QueryRange) * max_ranges, st);
      m->counters.alloc(8 * kNumCounters, st);
      SCONV_CUDA(cudaMemsetAsync(m->counters.get(), 0, 8 * kNumCounters, st));
      SCONV_CUDA(cudaMemsetAsync(m->nbr_in.get(), 0xFF, sizeof(int32_t) * int64_t{K3} * n_out, st));
      SCONV_CUDA(cudaMemsetAsync(counts.get(), 0, sizeof(int32_t) * grid2, st));
      auto* cnt = m->counters.get<unsigned long long>();
      ctx.launch("k_backward_partition", [&] {
        k_backward_partition<<<grid_for(tot), kThreads, 0, st>>>(src, n, B, q, n_out, og, K3, nb, bnd.get<int64_t>(),
                                                                 cnt);
      });
      ctx.launch("k_range_count", [&] {
        k_range_count<<<grid_for(tot), kThreads, 0, st>>>(bnd.get<int64_t>(), nb, tot, C, nrg.get<int64_t>());
      });
      size_t temp = 0;
      SCONV_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, nrg.get<int64_t>(), roff.get<int64_t>(), tot, st));
      tmp.alloc(std::max<size_t>(temp, 16), st);
      ctx.launch("cub_exclusive_sum", [&] {
        cub::DeviceScan::ExclusiveSum(tmp.get(), temp, nrg.get<int64_t>(), roff.get<int64_t>(), tot, st);
      });
      ctx.launch("k_range_emit", [&] {
        k_range_emit<<<grid_for(tot), kThreads, 0, st>>>(bnd.get<int64_t>(), nrg.get<int64_t>(), roff.get<int64_t>(),
                                                         nb, tot, rng.get<QueryRange>(), nrs.get<int64_t>());
      });
      const size_t smem = size_t{12} * B;
      const unsigned grid = static_cast<unsigned>(std::min<int64_t>(max_ranges, int64_t{ctx.num_sms} * 16));
      ctx.launch("k_forward_block_search", [&] {
        k_forward_block_search<<<grid, 256, smem, st>>>(src, src_idx, n, B, q, n_out, og, rng.get<QueryRange>(),
                                                        nrs.get<int64_t>(), CQ, nchunk2, m->nbr_in.get<int32_t>(),
                                                        counts.get<int32_t>(), cnt);
      });
      m->counted = true;
    } else if (cfg.backend == SCONV_MAP_HASH) {
      int lg = 1;
      while ((int64_t{1} << lg) < 2 * n) ++lg;  // capacity: smallest power of two >= 2N
      const uint64_t cap = uint64_t{1} << lg;
      m->hash_keys.alloc(8 * cap, st);
      m->hash_vals.alloc(4 * cap, st);
      SCONV_CUDA(cudaMemsetAsync(m->hash_keys.get(), 0xFF, 8 * cap, st));
      ctx.launch("k_hash_insert", [&] {
        k_hash_insert<<<grid_for(n), kThreads, 0, st>>>(src, src_idx, n, m->hash_keys.get<uint64_t>(),
                                                        m->hash_vals.get<int32_t>(), 64 - lg, cap - 1);
      });
      ctx.launch("k_hash_query", [&] {
        k_hash_query<<<dim3(static_cast<unsigned>(nchunk2), static_cast<unsigned>(K3)), CQ, 0, st>>>(
            q, n_out, og,
            m->hash_keys.get<uint64_t>(), m->hash_vals.get<int32_t>(), 64 - lg, cap - 1, nchunk2,
            m->nbr_in.get<int32_t>(), counts.get<int32_t>());
      });
    } else {
      // per-warp window: ~768 keys (a 256-query chunk's segment spans ~2-3 blocks of 256)
      static const int cap_keys = [] {
        const char* e = std::getenv("SCONV_SEARCH_CAP");  // experiments
        return e ? std::max(4, std::atoi(e)) : 768;
      }();
      const int cap_blocks = std::max(1, cap_keys / B);
      static const bool persist = [] {
        const char* e = std::getenv("SCONV_SEARCH_PERSIST");  // A/B: 0 = one CTA per chunk (k_search_col)
        return !(e && e[0] == '0');
      }();
      if (use_col && persist) {
        const int kz = cfg.kernel_size;
        constexpr int kW = 384;
        const size_t smem = size_t{2} * 12 * kz * kz * kW;
        const int scale = cfg.transposed ? -cfg.offset_scale : cfg.offset_scale;
        // probe stride: 32 lanes cover ~4 chunk advances (a chunk of 128 queries moves the
        // window by ~128 |P| / |Q| source keys); multiple of 4 (16-byte aligned idx slices)
        const int64_t adv = ceil_div<int64_t>(int64_t{128} * n, std::max<int64_t>(n_out, 1));
        const int stride = static_cast<int>(std::min<int64_t>(4 * ceil_div<int64_t>(adv, 32), 1 << 20));
        const char* trace_path = std::getenv("SCONV_SEARCH_TRACE");
        DevBuf trace;
        if (trace_path) {
          trace.alloc(size_t{32} * nchunk2 * kz * kz, st);
          SCONV_CUDA(cudaMemsetAsync(trace.get(), 0, size_t{32} * nchunk2 * kz * kz, st));
        }
        auto go = [&](auto kern) {
          set_max_smem(reinterpret_cast<const void*>(kern), smem);
          static const int o = [&] {  // resident CTAs per SM (one init per kernel instantiation)
            int v = 0;
            return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, 32 * kz * kz, smem) == cudaSuccess && v > 0 ? v : 1;
          }();
          static const int cpc_env = [] {  // experiments: chunks per CTA (0: one range per resident CTA)
            const char* e = std::getenv("SCONV_SEARCH_CPC");
            return e ? std::atoi(e) : 0;
          }();
          // one chunk per CTA (the hardware scheduler balances clouds with uneven chunk costs:
          // KITTI, S3DIS) below ~5e5 queries; above, one chunk range per resident CTA (the
          // cursor pipeline wins on large clouds: uniform 1e6 / 1e7 1.3x / 1.4x; r02bm)
          const bool ranges = cpc_env == 0 && n_out >= 500000;
          const int64_t grid = ranges ? std::min<int64_t>(nchunk2, int64_t{ctx.num_sms} * o)
                                      : ceil_div<int64_t>(nchunk2, std::max(1, cpc_env));
          ctx.launch("k_search", [&] {
            kern<<<static_cast<unsigned>(grid), 32 * kz * kz, smem, st>>>(src, src_idx, n, B, q, n_out, scale, nchunk2,
                                                                           std::max(4, stride), m->nbr_in.get<int32_t>(),
                                                                           counts.get<int32_t>(), trace.get<unsigned long long>());
          });
          if (trace_path) {  // diagnostics: dump {t_begin, t_end, slices | cta << 32, window start} per (chunk, column)
            std::vector<unsigned long long> h(static_cast<size_t>(nchunk2) * kz * kz * 4);
            SCONV_CUDA(cudaMemcpyAsync(h.data(), trace.get(), h.size() * 8, cudaMemcpyDeviceToHost, st));
            SCONV_CUDA(cudaStreamSynchronize(st));
            if (FILE* f = std::fopen(trace_path, "wb")) {
              std::fwrite(h.data(), 8, h.size(), f);
              std::fclose(f);
            }
          }
        };
        if (kz == 3)
          go(k_search_colp<4, 3, kW>);
        else
          go(k_search_colp<4, 2, kW>);
      } else if (use_col) {
        const int kz = cfg.kernel_size;
        // a 128-query chunk's column window spans ~1-2 blocks of 256: 2-block slices
        const int cap_col = std::max(1, std::min(cap_blocks, 512 / B));
        const size_t smem = size_t{12} * kz * kz * cap_col * B;
        const int scale = cfg.transposed ? -cfg.offset_scale : cfg.offset_scale;
        auto go = [&](auto kern) {
          set_max_smem(reinterpret_cast<const void*>(kern), smem);
          ctx.launch("k_search", [&] {
            kern<<<static_cast<unsigned>(nchunk2), 32 * kz * kz, smem, st>>>(
                src, src_idx, n, B, q, n_out, scale, nchunk2, cap_col, m->nbr_in.get<int32_t>(),
                counts.get<int32_t>());
          });
        };
        if (kz == 3)
          go(k_search_col<4, 3>);
        else
          go(k_search_col<4, 2>);
      } else {
      const size_t smem = size_t{12} * (kSearchThreads / 32) * cap_blocks * B;
      auto go = [&](auto kern) {
        set_max_smem(reinterpret_cast<const void*>(kern), smem);
        ctx.launch("k_search", [&] {
          kern<<<static_cast<unsigned>(nchunk2 * ngroups), kSearchThreads, smem, st>>>(
              src, src_idx, n, B, q, n_out, og,
              K3, nchunk2, ngroups, cap_blocks, m->nbr_in.get<int32_t>(), counts.get<int32_t>());
        });
      };
      switch (qpl) {
        case 1: go(k_search<1>); break;
        case 2: go(k_search<2>); break;
        case 4: go(k_search<4>); break;
        default: go(k_search<8>); break;
      }
      }
    }
    hmark("search queued");
    auto& pd = m->pending;
    pd.counts = std::move(counts);
    pd.offs = std::move(offs);
    pd.tiles = std::move(tiles);
    pd.nchunk = nchunk2;
    pd.grid = grid2;
    pd.ntiles = ntiles;
    pd.ngroups = ngroups;
    pd.qpl = qpl;
    if (!defer_canonical) launch_canonical(ctx, *m);
  }
  if (lazy) {  // canonical lists + readback deferred to ensure_canonical()
    m->canonical = false;
    m->total = -1;
    m->pending.flags = std::move(flags_buf);
    m->pending.flags_init = flags_used;
    return m;
  }
  if (defer_canonical && defer_flags && P.sorted && !P.keys && !target && !need_nout_sync) {
    // sorted raw coordinates: only range / order flags, no fallback -> checked by the caller
    d2h_small(defer_flags, flags, sizeof(MapFlags), st);
    m->flags_deferred = true;
    m->canonical = false;
    m->total = -1;
    m->pending.flags = std::move(flags_buf);
    m->pending.flags_init = flags_used;
    return m;
  }
  if (defer_canonical) {  // flags only (one sync), canonical lists on demand
    d2h_small(pin, flags, sizeof(MapFlags), st);
    ctx.sync();
    const MapFlags f = pin[0];
    if (!force_wide && (f.wide || f.big_bucket)) return build_map(ctx, P, cfg, target, true, true);  // exact fallback
    check_flags(f);
    m->canonical = false;
    m->total = -1;
    m->pending.flags = std::move(flags_buf);
    m->pending.flags_init = flags_used;
    return m;
  }
  // ---- readback: flags + canonical list starts (one sync per map)
  MapFlags f;
  read_starts(ctx, *m, flags, &f);
  m->pending = MapData::Pending{};
  if (!force_wide && (f.wide || f.big_bucket)) return build_map(ctx, P, cfg, target, true);  // exact fallback: CUB 64-bit sort
  check_flags(f);
  return m;
}


namespace {
// lazy map shell over sorted source / query keys with an all -1 table, canonical lists on demand
std::unique_ptr<MapData> derived_shell(Ctx& ctx, const MapSource& P, const MapSource& Q, const sconv_map_cfg& cfg) {
  auto m = std::make_unique<MapData>();
  m->cfg = cfg;
  m->n_in = P.n;
  m->n_out = Q.n;
  m->src_keys = P.keys;
  m->q_keys = Q.keys;
  m->src_identity = true;
  m->delta = weight_offsets_ext(cfg.kernel_size, cfg.offset_scale);
  if (cfg.transposed)
    for (auto& d : m->delta) d = make_int3(-d.x, -d.y, -d.z);
  m->K3 = static_cast<int>(m->delta.size());
  const cudaStream_t st = ctx.stream;
  const int64_t cells = std::max<int64_t>(1, int64_t{m->K3} * Q.n);
  m->nbr_in.alloc(sizeof(int32_t) * cells, st);
  SCONV_CUDA(cudaMemsetAsync(m->nbr_in.get(), 0xFF, sizeof(int32_t) * cells, st));
  m->map_start.alloc(sizeof(int32_t) * (m->K3 + 1), st);
  auto& pd = m->pending;
  pd.qpl = 4;
  pd.nchunk = ceil_div<int64_t>(Q.n, 32 * pd.qpl);
  pd.grid = pd.nchunk * m->K3;
  pd.ntiles = ceil_div<int64_t>(pd.grid, kScanTile);
  pd.ngroups = ceil_div(m->K3, kSearchThreads / 32);
  pd.counts.alloc(sizeof(int32_t) * std::max<int64_t>(1, pd.grid), st);
  pd.offs.alloc(sizeof(int32_t) * std::max<int64_t>(1, pd.grid), st);
  pd.tiles.alloc(sizeof(int32_t) * std::max<int64_t>(1, pd.ntiles), st);
  pd.counts_from_nbr = true;
  pd.max_pairs = std::min<int64_t>(int64_t{m->K3} * Q.n, int64_t{m->K3} * P.n);
  m->canonical = false;
  m->total = -1;
  return m;
}
}  // namespace

std::unique_ptr<MapData> derive_down_map(Ctx& ctx, const MapSource& P, const MapSource& Q, const sconv_map_cfg& cfg) {
  if (cfg.kernel_size != 2 || cfg.transposed || cfg.out_stride != 2 * cfg.offset_scale || !P.keys || !Q.keys)
    fail(SCONV_ERR_ARG, "derived down-sampling maps need K = 2, stride 2s over sorted keys");
  auto m = derived_shell(ctx, P, Q, cfg);
  if (P.n > 0 && Q.n > 0) {
    const cudaStream_t st = ctx.stream;
    ctx.launch("k_down_map", [&] {
      k_down_map<<<grid_for(P.n), kThreads, 0, st>>>(m->src_keys_ptr(), P.n, m->q_keys_ptr(), Q.n, cfg.offset_scale,
                                                     m->nbr_in.get<int32_t>());
    });
  }
  return m;
}

std::unique_ptr<MapData> derive_transposed_map(Ctx& ctx, const MapData& fwd, const MapSource& P, const MapSource& T,
                                               const sconv_map_cfg& cfg) {
  if (!cfg.transposed || fwd.cfg.transposed || fwd.cfg.kernel_size != cfg.kernel_size ||
      fwd.cfg.offset_scale != cfg.offset_scale || fwd.n_out != P.n || fwd.n_in != T.n || !fwd.nbr_in.get())
    fail(SCONV_ERR_ARG, "a derived transposed map needs its forward map (same K and offset scale)");
  auto m = derived_shell(ctx, P, T, cfg);
  if (fwd.n_out > 0 && T.n > 0) {
    const cudaStream_t st = ctx.stream;
    ctx.launch("k_transpose_map", [&] {
      k_transpose_map<<<grid_for(fwd.n_out * fwd.K3), kThreads, 0, st>>>(fwd.nbr_in.get<int32_t>(), fwd.n_out, fwd.K3,
                                                                         m->nbr_in.get<int32_t>(), T.n);
    });
  }
  return m;
}

}  // namespace sconvb

// GPU voxelization (the step before the Map/GMaS path; host-side in the
// reference at ~29 ms per 1.2e5 points). Same result as the reference's voxelize
// (proj/include/sconv/geometry.hpp:180-255), bit for bit:
//   * voxel = floor(p / resolution) per axis in double, range-checked against
//     [COORD_MIN, COORD_MAX] ("voxel index <axis> out of range" for the first offending point
//     in input order, first offending axis);
//   * points of a voxel are merged in the reference's canonical order (point coordinates
//     lexicographically, then feature rows) with a double accumulator, mean cast to float;
//   * output voxels sorted by packed key (sorted = true).
//
//   k_vox_keys   floor + range check + packed key, (key, point index) pairs
//   CUB          radix sort of the pairs by key, run-length encode -> voxel starts / counts
//   k_vox_merge  one thread per voxel: canonical member order (insertion sort of the few
//                member indices), double accumulation, mean, unpack coordinates
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cstring>
#include <string>

#include "common.cuh"
#include "voxelize.hpp"

namespace sconvb {
namespace {

__global__ void k_vox_keys(const double* __restrict__ pts, int64_t n, double res, uint64_t* __restrict__ keys,
                           int32_t* __restrict__ idx, unsigned long long* __restrict__ bad) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n) return;
  int32_t c[3];
  for (int a = 0; a < 3; ++a) {
    const double v = floor(pts[3 * i + a] / res);
    if (!(v >= kCoordMin && v <= kCoordMax)) {  // NaN fails too, as in the reference
      atomicMin(bad, static_cast<unsigned long long>(i) * 3ull + a);
      keys[i] = 0;
      idx[i] = static_cast<int32_t>(i);
      return;
    }
    c[a] = static_cast<int32_t>(v);
  }
  keys[i] = pack_key_unchecked(c[0], c[1], c[2]);
  idx[i] = static_cast<int32_t>(i);
}

// reference comparator for two points of the same voxel: coordinates, then feature rows
__device__ __forceinline__ bool canon_less(const double* __restrict__ pts, const float* __restrict__ f, int64_t C,
                                           int32_t a, int32_t b) {
  for (int k = 0; k < 3; ++k) {
    const double x = pts[3 * int64_t{a} + k], y = pts[3 * int64_t{b} + k];
    if (x != y) return x < y;
  }
  for (int64_t c = 0; c < C; ++c) {
    const float x = f[a * C + c], y = f[b * C + c];
    if (x != y) return x < y;
  }
  return false;
}

__global__ void k_vox_merge(const double* __restrict__ pts, const float* __restrict__ f, int64_t C,
                            const uint64_t* __restrict__ vkeys, const int32_t* __restrict__ starts,
                            const int32_t* __restrict__ counts, const int64_t* __restrict__ nvox,
                            int32_t* __restrict__ members, int32_t* __restrict__ out_xyz, float* __restrict__ out_f) {
  const int64_t v = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (v >= *nvox) return;
  const int32_t s = starts[v], cnt = counts[v];
  int32_t* m = members + s;
  if (C > 0)
    for (int32_t a = 1; a < cnt; ++a) {  // canonical order (segments hold a few points)
      const int32_t x = m[a];
      int32_t b = a - 1;
      while (b >= 0 && canon_less(pts, f, C, x, m[b])) {
        m[b + 1] = m[b];
        --b;
      }
      m[b + 1] = x;
    }
  int32_t xyz[3];
  unpack_key(vkeys[v], xyz[0], xyz[1], xyz[2]);
  out_xyz[3 * v] = xyz[0];
  out_xyz[3 * v + 1] = xyz[1];
  out_xyz[3 * v + 2] = xyz[2];
  for (int64_t c = 0; c < C; ++c) {
    double acc = 0.0;
    for (int32_t a = 0; a < cnt; ++a) acc += static_cast<double>(f[m[a] * C + c]);
    out_f[v * C + c] = static_cast<float>(acc / static_cast<double>(cnt));
  }
}

inline unsigned grid_for(int64_t n) { return static_cast<unsigned>(std::max<int64_t>(1, (n + 255) / 256)); }

}  // namespace

int64_t voxelize(Ctx& ctx, const double* pts, int64_t n, int pts_mem, const float* feats, int64_t C, int feats_mem,
                 double resolution, int32_t* out_xyz, float* out_f, int out_mem) {
  if (!(resolution > 0.0)) fail(SCONV_ERR_ARG, "resolution must be positive");
  if (n < 0 || n > INT32_MAX) fail(SCONV_ERR_ARG, "point count out of supported range");
  if (C < 0) fail(SCONV_ERR_ARG, "channel count must be nonnegative");
  if (C > 0 && n > 0 && !feats) fail(SCONV_ERR_ARG, "feature row count does not match point count");
  if (n == 0) return 0;
  const cudaStream_t st = ctx.stream;
  DevBuf dpts, dfeat, keys, keys_s, idx, idx_s, vkeys, counts, starts, nrun, bad, oxyz, of;
  const double* P = pts;
  if (pts_mem == SCONV_MEM_HOST) {
    dpts.alloc(sizeof(double) * 3 * n, st);
    SCONV_CUDA(cudaMemcpyAsync(dpts.get(), pts, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
    P = dpts.get<double>();
  }
  const float* F = feats;
  if (C > 0 && feats_mem == SCONV_MEM_HOST) {
    dfeat.alloc(sizeof(float) * n * C, st);
    SCONV_CUDA(cudaMemcpyAsync(dfeat.get(), feats, sizeof(float) * n * C, cudaMemcpyHostToDevice, st));
    F = dfeat.get<float>();
  }
  keys.alloc(8 * n, st);
  keys_s.alloc(8 * n, st);
  idx.alloc(4 * n, st);
  idx_s.alloc(4 * n, st);
  vkeys.alloc(8 * n, st);
  counts.alloc(4 * n, st);
  starts.alloc(4 * n, st);
  nrun.alloc(8, st);
  bad.alloc(8, st);
  SCONV_CUDA(cudaMemsetAsync(bad.get(), 0xFF, 8, st));
  SCONV_CUDA(cudaMemsetAsync(counts.get(), 0, 4 * n, st));  // runs past the voxel count stay 0
  ctx.launch("k_vox_keys", [&] {
    k_vox_keys<<<grid_for(n), 256, 0, st>>>(P, n, resolution, keys.get<uint64_t>(), idx.get<int32_t>(),
                                             bad.get<unsigned long long>());
  });
  size_t t1 = 0, t2 = 0, t3 = 0;
  SCONV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, keys.get<uint64_t>(), keys_s.get<uint64_t>(),
                                             idx.get<int32_t>(), idx_s.get<int32_t>(), static_cast<int>(n), 0, 63, st));
  SCONV_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, t2, keys_s.get<uint64_t>(), vkeys.get<uint64_t>(),
                                                counts.get<int32_t>(), nrun.get<int64_t>(), static_cast<int>(n), st));
  SCONV_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t3, counts.get<int32_t>(), starts.get<int32_t>(),
                                           static_cast<int>(n), st));
  ctx.scratch_sort.reserve(std::max({t1, t2, t3}), st);
  ctx.launch("cub_radix_sort_pairs", [&] {
    cub::DeviceRadixSort::SortPairs(ctx.scratch_sort.get(), t1, keys.get<uint64_t>(), keys_s.get<uint64_t>(),
                                    idx.get<int32_t>(), idx_s.get<int32_t>(), static_cast<int>(n), 0, 63, st);
  });
  ctx.launch("cub_rle", [&] {
    cub::DeviceRunLengthEncode::Encode(ctx.scratch_sort.get(), t2, keys_s.get<uint64_t>(), vkeys.get<uint64_t>(),
                                       counts.get<int32_t>(), nrun.get<int64_t>(), static_cast<int>(n), st);
  });
  ctx.launch("cub_scan", [&] {
    cub::DeviceScan::ExclusiveSum(ctx.scratch_sort.get(), t3, counts.get<int32_t>(), starts.get<int32_t>(),
                                  static_cast<int>(n), st);
  });
  int32_t* oxyz_p = out_xyz;
  float* of_p = out_f;
  if (out_mem == SCONV_MEM_HOST) {
    oxyz.alloc(sizeof(int32_t) * 3 * n, st);
    of.alloc(sizeof(float) * std::max<int64_t>(1, n * C), st);
    oxyz_p = oxyz.get<int32_t>();
    of_p = of.get<float>();
  }
  ctx.launch("k_vox_merge", [&] {
    k_vox_merge<<<grid_for(n), 256, 0, st>>>(P, F, C, vkeys.get<uint64_t>(), starts.get<int32_t>(),
                                              counts.get<int32_t>(), nrun.get<int64_t>(), idx_s.get<int32_t>(), oxyz_p,
                                              of_p);
  });
  unsigned long long hbad = 0;
  int64_t nv = 0;
  SCONV_CUDA(cudaMemcpyAsync(&hbad, bad.get(), 8, cudaMemcpyDeviceToHost, st));
  SCONV_CUDA(cudaMemcpyAsync(&nv, nrun.get(), 8, cudaMemcpyDeviceToHost, st));
  ctx.sync();
  if (hbad != ULLONG_MAX) {
    static const char kAxis[3] = {'x', 'y', 'z'};
    fail(SCONV_ERR_RANGE, std::string("voxel index ") + kAxis[hbad % 3] + " out of range");
  }
  if (out_mem == SCONV_MEM_HOST && nv > 0) {
    SCONV_CUDA(cudaMemcpyAsync(out_xyz, oxyz_p, sizeof(int32_t) * 3 * nv, cudaMemcpyDeviceToHost, st));
    if (C > 0) SCONV_CUDA(cudaMemcpyAsync(out_f, of_p, sizeof(float) * nv * C, cudaMemcpyDeviceToHost, st));
    ctx.sync();
  }
  return nv;
}

}  // namespace sconvb

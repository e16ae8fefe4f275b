// Cooperative (grid-barrier) building blocks for one-launch radix sorts of <= ~1e6 keys held in
// registers: at these sizes every kernel of a multi-launch sort (CUB: histogram, scan, one
// kernel per 8-bit pass, select, ...) is latency bound, so one co-resident grid that
// synchronises between phases replaces 5-10 launches. Launch with cudaLaunchCooperativeKernel
// (co-residency is required by grid_barrier). Tile layout: CTA b owns rows
// [b*tile, b*tile + tile); element e of thread t is row b*tile + e*kCoopThreads + t.
#pragma once
#include <cstdint>
#include <cstdlib>

namespace sconvb {

constexpr int kCoopThreads = 256, kCoopMaxE = 4;

// rows per thread to start from (1, 2 or 4; SCONV_COOP_E for experiments): the host doubles it
// until the grid fits the co-resident CTAs
inline int coop_rows_per_thread() {
  static const int e = [] {
    const char* v = std::getenv("SCONV_COOP_E");
    const int x = v ? std::atoi(v) : 1;
    return x >= 4 ? 4 : (x >= 2 ? 2 : 1);
  }();
  return e;
}

// all CTAs of the grid; `target` counts this launch's barriers (bar zeroed before the launch)
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks, unsigned& target) {
  __syncthreads();
  target += nblocks;  // barrier b completes at (b + 1) * nblocks arrivals
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

// exclusive scan of one int per thread over the CTA; returns the CTA total
__device__ __forceinline__ int block_exclusive_scan(int v, int& excl) {
  __shared__ int s_wsum[kCoopThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  int wp = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kCoopThreads / 32; ++w) {
    wp += w < warp ? s_wsum[w] : 0;
    total += s_wsum[w];
  }
  __syncthreads();
  excl = wp + incl - v;
  return total;
}

// One stable LSD pass over digit (key >> shift) & 255 of the grid's keys: returns each valid
// element's destination in pos[] (rows in tile order keep their order within a digit).
// cnt: 256 * gridDim.x ints, tot: 256 ints (scratch). Two grid barriers; the caller scatters
// and barriers before the next pass reads the output.
template <int E>
__device__ __forceinline__ void lsd_pass_positions(const uint32_t (&key)[E], const bool (&ok)[E], int shift, int (&pos)[E],
                                                   int* cnt, int* tot, unsigned* bar, unsigned& target) {
  constexpr int W = kCoopThreads / 32;
  __shared__ int s_wc[W][257];  // per-warp digit counts -> exclusive offsets (257th: no element)
  __shared__ int s_carry[256], s_off[256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned G = gridDim.x;
  int rank[E], dig[E];
  s_carry[tid] = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int d = ok[e] ? static_cast<int>((key[e] >> shift) & 255u) : 256;
    dig[e] = d;
    for (int q = tid; q < W * 257; q += kCoopThreads) (&s_wc[0][0])[q] = 0;
    __syncthreads();
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
    const int lrank = __popc(peers & ((1u << lane) - 1u));
    if (lrank == 0) s_wc[warp][d] = __popc(peers);
    __syncthreads();
    {  // thread tid owns digit tid: exclusive prefix over warps, carried across rounds
      int run = s_carry[tid];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int c = s_wc[w][tid];
        s_wc[w][tid] = run;
        run += c;
      }
      s_carry[tid] = run;
    }
    __syncthreads();
    rank[e] = ok[e] ? s_wc[warp][d] + lrank : 0;
    __syncthreads();
  }
  cnt[static_cast<int64_t>(tid) * G + blockIdx.x] = s_carry[tid];  // tile histogram, digit-major
  grid_barrier(bar, G, target);
  for (unsigned d = blockIdx.x; d < 256; d += G) {  // per-digit exclusive scan across tiles
    int* row = cnt + static_cast<int64_t>(d) * G;
    constexpr int PER = 8;  // G <= 2048
    int v[PER], local = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const unsigned c = tid * PER + u;
      v[u] = c < G ? __ldcg(row + c) : 0;
      local += v[u];
    }
    int excl;
    const int total = block_exclusive_scan(local, excl);
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const unsigned c = tid * PER + u;
      if (c < G) row[c] = excl;
      excl += v[u];
    }
    if (tid == 0) tot[d] = total;
  }
  grid_barrier(bar, G, target);
  {
    int base;
    block_exclusive_scan(__ldcg(tot + tid), base);
    s_off[tid] = base + __ldcg(cnt + static_cast<int64_t>(tid) * G + blockIdx.x);
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) pos[e] = ok[e] ? s_off[dig[e]] + rank[e] : -1;
  __syncthreads();
}

}  // namespace sconvb

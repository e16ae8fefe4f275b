// Fused output-stationary SC layer on sm_100a ("fused gather -> tcgen05
// GEMM -> scatter"). Same result as Minuet's GMaS (gather, per-offset GEMM,
// ascending-k scatter-sum) without materialising the gather buffer or the per-offset
// partials: for a tile of 128 output rows (sorted Q order) the kernel walks the offsets
// k = 0..K3-1 in ascending order, gathers the 128 input rows nbr_in[k][i] into shared
// memory and accumulates A_k . W_k into one fp32 TMEM accumulator, so the reduction over k
// happens inside the tensor core in ascending k (SPEC.md:353 order) and the output row is
// written once. Offsets with no neighbour anywhere in the tile are skipped.
//
// HBM/L2 traffic per layer: input rows |M| x C_in x 2 B (L2-resident at these sizes) +
// nbr table K3 x |Q| x 4 B + output |Q| x C_out x {2,4} B (+ residual read). No |M|-sized
// intermediate is written.
//
// Warp roles (288 threads, persistent CTAs over (row block, n block) tiles):
//   warps 0-3  gather producers: index rows of the tile (prefetched one tile ahead into
//              registers, published in shared memory), cp.async 16-byte chunks with the
//              UMMA 128/64/32-byte XOR swizzle, zero-fill for missing neighbours; thread 0
//              also TMA-loads the weight tile W_k^T. Completion is tracked by the hardware:
//              cp.async.mbarrier.arrive.noinc (no wait in the producer; 129 arrivals incl.
//              the TMA expect_tx), so a producer runs up to a whole ring ahead of the MMA.
//              The MMA thread executes fence.proxy.async after the barrier wait, making the
//              generic-proxy cp.async writes visible to the tensor core's async-proxy reads.
//   warps 4-7  epilogue: tcgen05.ld (32 lanes x 16 columns) -> + residual -> ReLU -> store
//   warp 8     TMEM owner; lane 0 issues tcgen05.mma (M=128, N=block_n, K=16) and commits
// Two TMEM accumulators let the epilogue of tile t overlap the MMAs of tile t+1.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "conv_fused.hpp"
#include "map.hpp"
#include "coop_sort.cuh"
#include "sm100.cuh"

namespace sconvb {
namespace {

using namespace sm100;

constexpr int kProducers = 128, kEpiWarps = 4;
constexpr int kThreads = kProducers + 32 * kEpiWarps + 32;  // 288
constexpr int kMaxStages = 12;
// Tile-info ring (active-offset masks, producers -> MMA). Producers run at most one ring
// (<= kMaxStages stages, >= 1 per tile) ahead of the MMA, so kInfo > kMaxStages slots never
// block on a tile the MMA has not reached.
constexpr int kInfo = 16;
static_assert(kInfo > kMaxStages, "tile-info ring must cover the stage ring");

template <class T>
struct OutCvt;
template <>
struct OutCvt<float> {
  static __device__ __forceinline__ void load16(const float* p, float (&x)[16]) {
#pragma unroll
    for (int e = 0; e < 16; e += 4) {
      const float4 v = *reinterpret_cast<const float4*>(p + e);
      x[e] = v.x;
      x[e + 1] = v.y;
      x[e + 2] = v.z;
      x[e + 3] = v.w;
    }
  }
  static __device__ __forceinline__ void store16(float* p, const float (&x)[16]) {
#pragma unroll
    for (int e = 0; e < 16; e += 4) *reinterpret_cast<float4*>(p + e) = make_float4(x[e], x[e + 1], x[e + 2], x[e + 3]);
  }
  static __device__ __forceinline__ float to(float v) { return v; }
  static __device__ __forceinline__ float from(float v) { return v; }
};
template <>
struct OutCvt<__half> {
  static __device__ __forceinline__ void load16(const __half* p, float (&x)[16]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint4 v = *reinterpret_cast<const uint4*>(p + 8 * h);
      const __half2* q = reinterpret_cast<const __half2*>(&v);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(q[e]);
        x[8 * h + 2 * e] = f.x;
        x[8 * h + 2 * e + 1] = f.y;
      }
    }
  }
  static __device__ __forceinline__ void store16(__half* p, const float (&x)[16]) {
    uint4 v[2];
    __half2* q = reinterpret_cast<__half2*>(v);
#pragma unroll
    for (int e = 0; e < 8; ++e) q[e] = __floats2half2_rn(x[2 * e], x[2 * e + 1]);
    reinterpret_cast<uint4*>(p)[0] = v[0];
    reinterpret_cast<uint4*>(p)[1] = v[1];
  }
  static __device__ __forceinline__ float to(__half v) { return __half2float(v); }
  static __device__ __forceinline__ __half from(float v) { return __float2half_rn(v); }
};
template <>
struct OutCvt<__nv_bfloat16> {
  static __device__ __forceinline__ void load16(const __nv_bfloat16* p, float (&x)[16]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint4 v = *reinterpret_cast<const uint4*>(p + 8 * h);
      const __nv_bfloat162* q = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(q[e]);
        x[8 * h + 2 * e] = f.x;
        x[8 * h + 2 * e + 1] = f.y;
      }
    }
  }
  static __device__ __forceinline__ void store16(__nv_bfloat16* p, const float (&x)[16]) {
    uint4 v[2];
    __nv_bfloat162* q = reinterpret_cast<__nv_bfloat162*>(v);
#pragma unroll
    for (int e = 0; e < 8; ++e) q[e] = __floats2bfloat162_rn(x[2 * e], x[2 * e + 1]);
    reinterpret_cast<uint4*>(p)[0] = v[0];
    reinterpret_cast<uint4*>(p)[1] = v[1];
  }
  static __device__ __forceinline__ float to(__nv_bfloat16 v) { return __bfloat162float(v); }
  static __device__ __forceinline__ __nv_bfloat16 from(float v) { return __float2bfloat16_rn(v); }
};

// 16-bit epilogue of one warp's 32 rows x 16 columns (lane = row): + residual, ReLU, store,
// with every global load / store instruction covering 16 rows x 32 contiguous bytes (full
// 32-byte sectors; the row-per-lane accesses touch each sector with 16 B twice). Lane l moves
// the half (l & 1) of row (l >> 1) + 16h; warp shuffles carry the values between the row owner
// and the mover. All 32 lanes must call it (rows may be invalid: never loaded or stored).
template <class TOut>
__device__ __forceinline__ void epilogue16_rows(TOut* out, int64_t ld_out, const TOut* res, int64_t ld_res,
                                                int64_t row, bool valid, int col, int relu, float (&x)[16]) {
  static_assert(sizeof(TOut) == 2, "16-bit outputs");
  const int lane = threadIdx.x & 31, half = lane & 1;
  long long mrow[2];
  bool mval[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int src = (lane >> 1) + 16 * h;
    mrow[h] = __shfl_sync(0xFFFFFFFFu, static_cast<long long>(row), src);
    mval[h] = __shfl_sync(0xFFFFFFFFu, valid ? 1 : 0, src) != 0;
  }
  if (res) {
    uint4 rv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
      rv[h] = mval[h] ? *reinterpret_cast<const uint4*>(res + mrow[h] * ld_res + col + half * 8) : make_uint4(0, 0, 0, 0);
    const int s0 = 2 * (lane & 15), hi = lane >> 4;
    uint32_t w[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t a0 = __shfl_sync(0xFFFFFFFFu, (&rv[0].x)[k], s0), a1 = __shfl_sync(0xFFFFFFFFu, (&rv[1].x)[k], s0);
      const uint32_t b0 = __shfl_sync(0xFFFFFFFFu, (&rv[0].x)[k], s0 + 1);
      const uint32_t b1 = __shfl_sync(0xFFFFFFFFu, (&rv[1].x)[k], s0 + 1);
      w[k] = hi ? a1 : a0;
      w[4 + k] = hi ? b1 : b0;
    }
    float r[16];
    OutCvt<TOut>::load16(reinterpret_cast<const TOut*>(w), r);
#pragma unroll
    for (int e = 0; e < 16; ++e) x[e] += r[e];
  }
  if (relu)
#pragma unroll
    for (int e = 0; e < 16; ++e) x[e] = fmaxf(x[e], 0.f);
  uint4 pk[2];
  OutCvt<TOut>::store16(reinterpret_cast<TOut*>(pk), x);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int src = (lane >> 1) + 16 * h;
    uint4 v;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t a = __shfl_sync(0xFFFFFFFFu, (&pk[0].x)[k], src), b = __shfl_sync(0xFFFFFFFFu, (&pk[1].x)[k], src);
      (&v.x)[k] = half ? b : a;
    }
    if (mval[h]) *reinterpret_cast<uint4*>(out + mrow[h] * ld_out + col + half * 8) = v;
  }
}

struct MaskOrder {
  int pos[32];
};

struct FusedParams {
  const unsigned char* f_in;
  int64_t ld_in_bytes;
  const int32_t* nbr;   // [K3][n_out] in tile-row order (null: the 1x1 identity map, nbr[0][i] = i)
  const int32_t* perm;  // tile row -> output row (null: identity)
  int64_t n_out;
  int K3, num_kb, block_n, n_pad, n_blocks, num_tiles, c_out;
  void* out;
  int64_t ld_out;
  const void* res;
  int64_t ld_res;
  int relu;
  int vec;  // 16-byte aligned output / residual rows
  uint32_t stage_bytes, a_bytes, b_bytes, idx_off, bar_off;
  int stages;  // smem ring depth
  int G;       // (offset, K-chunk) units per stage
  int* tile_counter;  // dynamic tile queue (zeroed before the launch)
  uint32_t unit_bytes;  // one unit's A + B slot (1024-aligned)
  int target_occ;  // resident CTAs per SM the ring was sized for
  unsigned long long* trace;  // debug 5: CTA 0 event timeline {kind<<56 | seq<<32 | t_lo}
  int debug;   // profiling experiments only (SCONV_FUSED_DEBUG bits): 1 no gather copies, 2 no MMAs,
               // 4 no weight TMA (plain arrive), 8 CTA-0 timeline trace, 256 no epilogue, 8192 CTA spans
  uint32_t tmem_cols;
  int bf16;
  unsigned long long* spans;  // debug 8192: per CTA {start, setup done, end, tiles} (globaltimer ns)
  // work-item kernel (k_conv_items)
  const unsigned long long* tile_mask;
  const void* items;  // int4 (null: one item per row block)
  const int* item_ws;  // workspace slot per item (-1: tile not split)
  const int* n_items;
  int* item_counters;
  float* ws;
  int num_rb;
  int coal_epi;  // 16-bit outputs: sector-coalesced epilogue (SCONV_FUSED_COAL=0: row per lane)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// debug 5 timeline: each event kind owns a 1024-slot region, written with plain stores by a
// single thread (no atomics: the trace must not perturb the pipeline)
__device__ __forceinline__ void trace_ev(const FusedParams& p, int kind, int seq, unsigned& n) {
  if (p.trace && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (n < 1024)
      p.trace[kind * 1024 + n] = (static_cast<unsigned long long>(kind) << 56) |
                                 (static_cast<unsigned long long>(seq & 0xFFFFFF) << 32) | (t & 0xFFFFFFFFull);
    ++n;
  }
}

// input row of output i at offset k; a null table (only with K3 = 1: the 1x1 identity map) is
// nbr[0][i] = i. The check is compiled into the NK = 1 (and runtime-K3) kernels only.
template <int NK>
__device__ __forceinline__ int32_t nbr_at(const FusedParams& p, int k, int64_t i) {
  if constexpr (NK == 1 || NK == 0)
    if (!p.nbr) return static_cast<int32_t>(i);
  return __ldg(p.nbr + int64_t{k} * p.n_out + i);
}

// NK = compile-time offset count (registers prefetch the next tile's index rows), 0 = runtime
// DENSE (1x1 identity maps only: input row i of output row i, no row permutation): the A tile
// is a plain 128-row box of the input, TMA-loaded with the same swizzle as the weights by one
// producer thread (no per-row cp.async gathers), so the layer is a TMA-fed tcgen05 GEMM.
template <int NK, int KC, class TOut, bool REG = false, bool DENSE = false>
__global__ void __launch_bounds__(kThreads, NK == 0 ? 4 : 2) k_conv_fused(const __grid_constant__ CUtensorMap tmB,
                                                           const __grid_constant__ FusedParams p,
                                                           const __grid_constant__ CUtensorMap tmA) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned base (SW128 atoms) derived by OFFSET from the __shared__ array, so the
  // compiler keeps the shared address space (LDS/STS, not generic LD/ST) for every access
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  int32_t* s_idx = reinterpret_cast<int32_t*>(smem + p.idx_off);  // [K3][128] rows of the current tile
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* ifull = tempty + 2;
  uint64_t* iempty = ifull + kInfo;
  uint64_t* s_mask = iempty + kInfo;   // [kInfo] active-offset mask per tile slot
  uint64_t* s_part = s_mask + kInfo;   // [2][4] per-producer-warp partial masks
  int32_t* s_tile = reinterpret_cast<int32_t*>(s_part + 8);  // [kInfo] tile id per slot (-1: done)
  int32_t* s_tq = s_tile + kInfo;                             // [4] producers' tile look-ahead
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_tq + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K3 = p.K3;
  if (p.spans && threadIdx.x == 0) p.spans[blockIdx.x * 4] = gtimer();

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], DENSE ? 1 : kProducers + 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
    }
    for (int a = 0; a < kInfo; ++a) {
      mbar_init(&ifull[a], 1);
      mbar_init(&iempty[a], 1 + kEpiWarps);  // MMA thread + each epilogue warp
    }
    mbar_fence_init();
  }
  if (warp == 8) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: setup above overlapped the previous kernel's tail; its outputs (our input rows, the
  // residual, the tile queue it reset) are visible past this point. Dependents may launch once
  // every CTA got here (each already holds its TMEM, so a dependent's allocation can only wait
  // on CTAs that make progress).
  grid_dep_wait();
  if (threadIdx.x == 0) grid_dep_launch();
  unsigned tr0 = 0, tr1 = 0, tr2 = 0, tr3 = 0, tr4 = 0, tr5 = 0, tr6 = 0, tr7 = 0;  // debug-8 trace cursors
  if (threadIdx.x == 0) trace_ev(p, 0, 0, tr0);  // CTA start (after TMEM allocation)
  if (p.spans && threadIdx.x == 0) p.spans[blockIdx.x * 4 + 1] = gtimer();

  if (DENSE && warp < 4) {
    // ------------------------------------------------------------ dense producer (one thread)
    if (threadIdx.x == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
      const uint32_t smem_base = smem_u32(smem);
      int stage = 0, it = 0;
      uint32_t phase = 0;
      for (;; ++it) {
        const int q = atomicAdd(p.tile_counter, 1);
        const int t = q < p.num_tiles ? q : -1;
        const int slot = it % kInfo;
        mbar_wait(&iempty[slot], ((it / kInfo) & 1) ^ 1);
        s_mask[slot] = 1;
        s_tile[slot] = t;
        mbar_arrive(&ifull[slot]);
        if (t < 0) break;
        const int rb = t / p.n_blocks, nb = t % p.n_blocks;
        int units_left = p.num_kb, in_stage = 0, stage_units = 0;
        uint32_t slot32 = 0;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          if (in_stage == 0) {
            mbar_wait(&empty[stage], phase ^ 1u);
            stage_units = min(p.G, units_left);
            slot32 = smem_base + static_cast<uint32_t>(stage) * p.stage_bytes;
            mbar_expect_tx(&full[stage], static_cast<uint32_t>(stage_units) * (p.a_bytes + p.b_bytes));
          }
          tma_load_2d(smem + (slot32 - smem_base), &tmA, kb * KC, rb * 128, &full[stage]);
          tma_load_2d(smem + (slot32 - smem_base) + p.a_bytes, &tmB, kb * KC, nb * p.block_n, &full[stage]);
          --units_left;
          slot32 += p.unit_bytes;
          if (++in_stage == stage_units) {
            in_stage = 0;
            if (++stage == S) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
  } else if (REG && warp < 4) {
    // ------------------------------------------------------------ gather producers, register indices
    // Thread tid owns tile row tid: its K3 input-row indices are loaded at the tile start
    // (independent LDGs, all in flight together) and published to the warp's own columns of
    // the index table (no CTA barrier: only the same warp reads them). Copy instruction q of
    // warp w covers rows 32w + lane/CPR + q*(32/CPR) (whole rows, coalesced); the offset loop
    // visits only the tile's active offsets (set bits of the mask).
    constexpr int CPR = KC / 8, RPI = 32 / CPR;
    // KC <= 32 (narrow chunks, 1-2 rows per copy instruction): row indices through the warp's
    // columns of the shared index table, offset loop over set mask bits only. KC = 64: register
    // rotation (the table variant measured slower there, though within run-to-run noise).
    constexpr bool kTable = KC <= 32;
    constexpr int NR = NK > 0 ? NK : 1;
    const int tid = threadIdx.x;
    const int chunk = lane % CPR, rsub = lane / CPR;
    uint32_t a_off[CPR];
#pragma unroll
    for (int q = 0; q < CPR; ++q) a_off[q] = swizzled_offset<KC>(32 * warp + rsub + q * RPI, chunk);
    const unsigned char* src_col = p.f_in + chunk * 16;
    auto grab = [&]() -> int {
      const int q = atomicAdd(p.tile_counter, 1);
      return q < p.num_tiles ? p.num_tiles - 1 - q : -1;
    };
    if (tid == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      s_tq[0] = grab();
    }
    named_bar(1, kProducers);
    int t = s_tq[0], t_next = -1;
    // table variant: row indices one tile ahead, the next tile's LDGs in flight during this
    // tile's gathers (the queue look-ahead stays one tile deep: deeper reservations unbalance the densest-first
    // queue when a layer has only 1-3 tiles per CTA)
    int jn[NR];
    auto load_rows = [&](int tt) {
      const int64_t i = static_cast<int64_t>(tt / p.n_blocks) * 128 + tid;
      const bool ok = i < p.n_out;
#pragma unroll
      for (int k = 0; k < NR; ++k) jn[k] = ok ? nbr_at<NK>(p, k, i) : -1;
    };
    if (kTable && t >= 0) load_rows(t);
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t smem_base = smem_u32(smem);
    int it = 0;
    for (; t >= 0; ++it) {
      const int buf = it & 1;
      if (it > 0) named_bar(1, kProducers);
      if (tid == 0) s_tq[(it + 1) & 3] = grab();
      const int nb = t % p.n_blocks;
      if (!kTable) load_rows(t);  // rotation variant: no look-ahead (measured slower at 96 regs)
      int jc[NR];
#pragma unroll
      for (int k = 0; k < NR; ++k) jc[k] = jn[k];
      uint64_t mine = 0;
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        mine |= static_cast<uint64_t>(jc[k] >= 0) << k;
        if constexpr (kTable) s_idx[k * 128 + tid] = jc[k];  // this warp's rows only: read back by the same warp
      }
      const uint32_t lo = __reduce_or_sync(0xFFFFFFFFu, static_cast<uint32_t>(mine));
      const uint32_t hi = __reduce_or_sync(0xFFFFFFFFu, static_cast<uint32_t>(mine >> 32));
      if (lane == 0) s_part[buf * 4 + warp] = (static_cast<uint64_t>(hi) << 32) | lo;
      named_bar(1, kProducers);
      uint64_t mask = s_part[buf * 4] | s_part[buf * 4 + 1] | s_part[buf * 4 + 2] | s_part[buf * 4 + 3];
      if (mask == 0) mask = 1;
      t_next = s_tq[(it + 1) & 3];  // published by the barrier above
      if (kTable && t_next >= 0) load_rows(t_next);
      if (tid == 0) {
        const int slot = it % kInfo;
        mbar_wait(&iempty[slot], ((it / kInfo) & 1) ^ 1);
        s_mask[slot] = mask;
        s_tile[slot] = t;
        mbar_arrive(&ifull[slot]);
      }
      const int b_row0 = nb * p.block_n;
      int units_left = __popcll(mask) * p.num_kb, in_stage = 0, stage_units = 0;
      uint32_t slot32 = 0;
      const int32_t* wrow = s_idx + 32 * warp + rsub;  // published before the named barrier above
      uint64_t mm = mask;
#pragma unroll 1
      for (int kk = 0; kTable ? mm != 0 : kk < NR; ++kk) {
        int k;
        int32_t j[CPR];
        if constexpr (kTable) {  // visit only the active offsets; indices from the warp's table
          k = __ffsll(static_cast<long long>(mm)) - 1;
          mm &= mm - 1;
#pragma unroll
          for (int q = 0; q < CPR; ++q) j[q] = wrow[k * 128 + q * RPI];
        } else {  // rotate the register array (no dynamic indexing), skip inactive offsets
          k = kk;
          const int32_t jk = jc[0];
#pragma unroll
          for (int r = 0; r + 1 < NR; ++r) jc[r] = jc[r + 1];
          if (!((mask >> k) & 1)) continue;
#pragma unroll
          for (int q = 0; q < CPR; ++q) j[q] = __shfl_sync(0xFFFFFFFFu, jk, rsub + q * RPI);
        }
        const int b_row = k * p.n_pad + b_row0;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          if (in_stage == 0) {
            mbar_wait(&empty[stage], phase ^ 1u);
            stage_units = min(p.G, units_left);
            slot32 = smem_base + static_cast<uint32_t>(stage) * p.stage_bytes;
            if (tid == 0) mbar_expect_tx(&full[stage], static_cast<uint32_t>(stage_units) * p.b_bytes);
          }
          if (tid == 0) tma_load_2d(smem + (slot32 - smem_base) + p.a_bytes, &tmB, kb * KC, b_row, &full[stage]);
          const unsigned char* col = src_col + kb * (KC * 2);
#pragma unroll
          for (int q = 0; q < CPR; ++q)
            cp_async16(slot32 + a_off[q], col + static_cast<int64_t>(j[q] >= 0 ? j[q] : 0) * p.ld_in_bytes,
                       j[q] >= 0 ? 16u : 0u);
          --units_left;
          slot32 += p.unit_bytes;
          if (++in_stage == stage_units) {
            cp_async_arrive_noinc(&full[stage]);
            in_stage = 0;
            if (++stage == S) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
      t = t_next;
    }
    if (tid == 0) {
      const int slot = it % kInfo;
      mbar_wait(&iempty[slot], ((it / kInfo) & 1) ^ 1);
      s_tile[slot] = -1;
      mbar_arrive(&ifull[slot]);
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ gather producers
    const int tid = threadIdx.x;
    constexpr int CPR = KC / 8;      // 16-byte chunks per row
    constexpr int RPP = 128 / CPR;   // rows per pass
    const int chunk = tid % CPR, rbase = tid / CPR;
    uint32_t a_off[CPR];
#pragma unroll
    for (int q = 0; q < CPR; ++q) a_off[q] = swizzled_offset<KC>(rbase + q * RPP, chunk);
    const unsigned char* src_col = p.f_in + chunk * 16;
    if (tid == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");

    constexpr int NR = NK > 0 ? NK : 1;
    int jn[NR];
    auto load_rows = [&](int t) {
      const int64_t i = static_cast<int64_t>(t / p.n_blocks) * 128 + tid;
      const bool ok = i < p.n_out;
#pragma unroll
      for (int k = 0; k < NR; ++k) jn[k] = ok ? nbr_at<NK>(p, k, i) : -1;
    };
    // Dynamic tile queue (global atomic counter), dispensed densest-first: row blocks are in
    // neighbour-mask order, so the last blocks carry the most active offsets; handing them out
    // first balances the CTAs (longest-processing-time-first).
    auto grab = [&]() -> int {
      const int q = atomicAdd(p.tile_counter, 1);
      return q < p.num_tiles ? p.num_tiles - 1 - q : -1;
    };
    if (tid == 0) {
      s_tq[0] = grab();
      s_tq[1] = grab();
    }
    named_bar(1, kProducers);
    int t = s_tq[0], t_next = s_tq[1];
    if (NK > 0 && t >= 0) load_rows(t);
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t smem_base = smem_u32(smem);
    int it = 0;
    for (; t >= 0; ++it) {
      const int buf = it & 1;
      if (tid == 0) trace_ev(p, 1, it, tr1);
      const int nb = t % p.n_blocks;  // one division per tile
      int32_t* srow = s_idx;
      if (it > 0) named_bar(1, kProducers);  // every producer finished reading the previous tile's rows
      if (tid == 0) s_tq[(it + 2) & 3] = t_next >= 0 ? grab() : -1;  // the tile after next
      uint64_t mine = 0;
      if constexpr (NK > 0) {
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          srow[k * 128 + tid] = jn[k];
          mine |= static_cast<uint64_t>(jn[k] >= 0) << k;
        }
        if (t_next >= 0) load_rows(t_next);  // next tile's index rows, in flight during this tile
      } else {
        const int64_t i = static_cast<int64_t>(t / p.n_blocks) * 128 + tid;
        for (int k = 0; k < K3; ++k) {
          const int32_t j = i < p.n_out ? nbr_at<NK>(p, k, i) : -1;
          srow[k * 128 + tid] = j;
          mine |= static_cast<uint64_t>(j >= 0) << k;
        }
      }
      const uint32_t lo = __reduce_or_sync(0xFFFFFFFFu, static_cast<uint32_t>(mine));
      const uint32_t hi = __reduce_or_sync(0xFFFFFFFFu, static_cast<uint32_t>(mine >> 32));
      if (lane == 0) s_part[buf * 4 + warp] = (static_cast<uint64_t>(hi) << 32) | lo;
      named_bar(1, kProducers);  // index rows + partial masks of this tile are published
      const int t_after = s_tq[(it + 2) & 3];  // the tile after next (written before the barrier)
      uint64_t mask = s_part[buf * 4] | s_part[buf * 4 + 1] | s_part[buf * 4 + 2] | s_part[buf * 4 + 3];
      if (mask == 0) mask = 1;  // no neighbour at all: one all-zero stage keeps the accumulator defined
      if (tid == 0) {
        const int slot = it % kInfo;
        mbar_wait(&iempty[slot], ((it / kInfo) & 1) ^ 1);
        s_mask[slot] = mask;
        s_tile[slot] = t;
        mbar_arrive(&ifull[slot]);
      }
      const int b_row0 = nb * p.block_n;
      // Units (k, kb) in ascending k, G units per stage: one barrier round trip per G units
      // (the handshake, not the bytes, bounds narrow layers). Slot u of a stage holds A_u then B_u.
      int units_left = __popcll(mask) * p.num_kb, in_stage = 0, stage_units = 0;
      uint32_t slot32 = 0;
      for (uint64_t m = mask; m; m &= m - 1) {
        const int k = __ffsll(static_cast<long long>(m)) - 1;
        const int32_t* sk = srow + k * 128;
        const unsigned char* src[CPR];  // this thread's source chunks for offset k (kb = 0)
        uint32_t nbytes[CPR];
#pragma unroll
        for (int q = 0; q < CPR; ++q) {
          const int32_t j = sk[rbase + q * RPP];
          src[q] = src_col + static_cast<int64_t>(j >= 0 ? j : 0) * p.ld_in_bytes;
          nbytes[q] = j >= 0 ? 16u : 0u;
        }
        const int b_row = k * p.n_pad + b_row0;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          if (in_stage == 0) {
            if (tid == 0) trace_ev(p, 7, stage, tr7);  // about to wait for a free stage
            mbar_wait(&empty[stage], phase ^ 1u);
            stage_units = min(p.G, units_left);
            slot32 = smem_base + static_cast<uint32_t>(stage) * p.stage_bytes;
            if (tid == 0) {
              if (p.debug & 4)
                mbar_arrive(&full[stage]);
              else
                mbar_expect_tx(&full[stage], static_cast<uint32_t>(stage_units) * p.b_bytes);
            }
          }
          if (tid == 0 && !(p.debug & 4))
            tma_load_2d(smem + (slot32 - smem_base) + p.a_bytes, &tmB, kb * KC, b_row, &full[stage]);
          if (!(p.debug & 1)) {
#pragma unroll
            for (int q = 0; q < CPR; ++q) cp_async16(slot32 + a_off[q], src[q] + kb * (KC * 2), nbytes[q]);
          }
          --units_left;
          slot32 += p.unit_bytes;
          if (++in_stage == stage_units) {
            cp_async_arrive_noinc(&full[stage]);
            if (tid == 0) trace_ev(p, 2, stage, tr2);
            in_stage = 0;
            if (++stage == S) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
      t = t_next;
      t_next = t_after;
    }
    if (tid == 0) {  // end-of-work marker for the MMA and the epilogue
      const int slot = it % kInfo;
      mbar_wait(&iempty[slot], ((it / kInfo) & 1) ^ 1);
      s_tile[slot] = -1;
      mbar_arrive(&ifull[slot]);
    }
  } else if (warp == 8) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int it = 0;; ++it) {
        const int slot = it % kInfo;
        mbar_wait(&ifull[slot], (it / kInfo) & 1);
        const uint64_t mask = s_mask[slot];
        const int t = s_tile[slot];
        mbar_arrive(&iempty[slot]);
        if (t < 0) break;
        const int nb = t % p.n_blocks;
        const int n_tile = min(p.block_n, p.n_pad - nb * p.block_n);
        const uint32_t idesc = idesc_f16(p.bf16, n_tile);
        if (!(p.debug & 256)) mbar_wait(&tempty[acc], acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * p.block_n);
        uint32_t accumulate = 0;
        for (int units_left = __popcll(mask) * p.num_kb; units_left > 0;) {
          const int su = min(p.G, units_left);
          mbar_wait(&full[stage], phase);
          trace_ev(p, 3, stage, tr3);
          if (!(p.debug & 1)) fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tensor core reads
          tc_fence_after();
          uint32_t sa = smem_u32(smem + stage * p.stage_bytes);
          for (int u = 0; u < su; ++u, sa += p.unit_bytes) {
            const uint32_t sb = sa + p.a_bytes;
            if (!(p.debug & 2)) {
#pragma unroll
              for (int kk = 0; kk < KC / 16; ++kk) {
                tc_mma(d_tmem, smem_desc<KC>(sa + kk * 32), smem_desc<KC>(sb + kk * 32), idesc, accumulate);
                accumulate = 1;
              }
            }
          }
          tc_commit(&empty[stage]);  // frees the stage once these MMAs retire
          units_left -= su;
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
        }
        tc_commit(&tfull[acc]);
        trace_ev(p, 4, it, tr4);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    TOut* out = static_cast<TOut*>(p.out);
    const TOut* res = static_cast<const TOut*>(p.res);
    for (int it = 0; !(p.debug & 256); ++it) {
      const int slot = it % kInfo;
      mbar_wait_backoff(&ifull[slot], (it / kInfo) & 1);
      const int t = s_tile[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&iempty[slot]);
      if (t < 0) break;
      const int nb = t % p.n_blocks;
      const int n0 = nb * p.block_n;
      const int n_tile = min(p.block_n, p.n_pad - n0);
      const int64_t r = static_cast<int64_t>(t / p.n_blocks) * 128 + q * 32 + lane;
      const bool valid = r < p.n_out;
      const int64_t i = valid && p.perm ? static_cast<int64_t>(__ldg(p.perm + r)) : r;
      const int ncols = min(n_tile, p.c_out - n0);
      mbar_wait_backoff(&tfull[acc], acc_phase);  // idle warps yield issue slots to the producers
      if (warp == 4 && lane == 0) trace_ev(p, 5, t, tr5);
      tc_fence_after();
      TOut* orow = out + i * p.ld_out + n0;
      const TOut* rrow = res ? res + i * p.ld_res + n0 : nullptr;
      for (int c0 = 0; c0 < n_tile; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * p.block_n + c0), v);
        if constexpr (sizeof(TOut) == 2) {
          if (p.vec && c0 + 16 <= ncols && p.coal_epi) {  // warp-uniform: sector-coalesced path
            float x[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = __uint_as_float(v[e]);
            epilogue16_rows<TOut>(out + n0, p.ld_out, res ? res + n0 : nullptr, p.ld_res, i, valid, c0, p.relu, x);
            continue;
          }
        }
        if (!valid || c0 >= ncols) continue;
        float x[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) x[e] = __uint_as_float(v[e]);
        const bool full16 = p.vec && c0 + 16 <= ncols;
        if (rrow) {
          if (full16) {
            float r[16];
            OutCvt<TOut>::load16(rrow + c0, r);
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] += r[e];
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (e < ncols - c0) x[e] += OutCvt<TOut>::to(rrow[c0 + e]);
          }
        }
        if (p.relu)
#pragma unroll
          for (int e = 0; e < 16; ++e) x[e] = fmaxf(x[e], 0.f);
        if (full16)
          OutCvt<TOut>::store16(orow + c0, x);
        else
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (e < ncols - c0) orow[c0 + e] = OutCvt<TOut>::from(x[e]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (warp == 4 && lane == 0) trace_ev(p, 6, t, tr6);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_ev(p, 0, 1, tr0);  // CTA end
  if (p.spans && threadIdx.x == 0) p.spans[blockIdx.x * 4 + 2] = gtimer();
  if (threadIdx.x == 0) {
    // the last CTA out resets the tile queue for the next launch (every CTA has drawn its
    // end-of-queue ticket before exiting), so no memset node sits between two convs
    __threadfence();
    if (atomicAdd(p.tile_counter + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      p.tile_counter[0] = 0;
      p.tile_counter[1] = 0;
      __threadfence();
    }
  }
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// ================================================================ work-item fused kernel
// Same arithmetic and warp roles as k_conv_fused, with the tile bookkeeping moved off the
// pipeline (measured r02: with every copy, MMA, handshake and epilogue disabled the old kernel
// still spent 15-30 us per launch on its dynamic tile queue, per-tile index publication and
// tile-info ring, and the slowest CTA ran 1.25-1.34x the average one: a few 27-offset tiles per
// CTA do not balance).
//   * work items are precomputed once per map (build_fused_items): item = (128-row tile, a
//     range of <= kItemMaxOffsets of its active offsets), densest tiles first; tiles with more
//     active offsets than the per-map cap are split into near-equal ranges, so items are of
//     bounded size and a wide few-row layer still spreads over every SM (split-K over offsets);
//   * static schedule: CTA b runs items b, b + grid, ...; producers, MMA issuer and epilogue
//     walk the same list independently (no atomics, no tile-info ring, no producer barriers);
//   * row indices in registers: thread t of the producers loads nbr[k][tile row t] for every
//     offset of the NEXT item while the current one streams (one item of look-ahead), and the
//     item descriptor two items ahead; warp shuffles hand each copy lane its row's index;
//   * split items: each part writes its fp32 partial (column-major [bn][128], coalesced) to a
//     workspace slot, the last part to finish (per-tile counter, self-resetting) sums the parts
//     in part order -- the result does not depend on which part finishes last (deterministic).
constexpr int kItemMaxOffsets = 28, kItemHead = 8;

// work item {row block, part | parts << 8, offset mask lo, hi}: the mask holds exactly this
// part's offsets, so one 16-byte load describes the item (no dependent loads)
struct ItemView {
  int rb, part, parts;
  uint64_t mask;
};
// snake (boustrophedon) static schedule: round r hands items r*G .. r*G + G - 1 to CTAs 0..G-1
// on even rounds and G-1..0 on odd ones, so with densest-first items no CTA takes the heaviest
// item of every round
__device__ __forceinline__ int work_of(int r) {
  const int G = gridDim.x, b = blockIdx.x;
  return r * G + ((r & 1) ? G - 1 - b : b);
}
__device__ __forceinline__ ItemView load_item(const int4* items, int i) {
  if (!items) return ItemView{i, 0, 1, 1ull};  // 1x1 identity map: one offset per tile
  const int4 v = __ldg(items + i);
  return ItemView{v.x, v.y & 0xFF, v.y >> 8,
                  (static_cast<uint64_t>(static_cast<uint32_t>(v.w)) << 32) | static_cast<uint32_t>(v.z)};
}

template <int KC, class TOut>
__global__ void __launch_bounds__(kThreads, 2) k_conv_items(const __grid_constant__ CUtensorMap tmB,
                                                         const __grid_constant__ FusedParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);  // [2] epilogue: this part finished its tile
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (p.spans && threadIdx.x == 0) p.spans[blockIdx.x * 4] = gtimer();
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], kProducers + 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
    }
    mbar_fence_init();
  }
  if (warp == 8) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (p.spans && threadIdx.x == 0) p.spans[blockIdx.x * 4 + 1] = gtimer();
  const int4* items = reinterpret_cast<const int4*>(p.items);
  const int n_items = p.n_items ? __ldg(p.n_items) : p.num_rb;
  const int n_work = n_items * p.n_blocks;
  const int G = gridDim.x;

  if (warp < 4) {
    // ------------------------------------------------------------ gather producers
    constexpr int CPR = KC / 8, RPI = 32 / CPR;  // 16-byte chunks per row, rows per copy instruction
    constexpr int KM = kItemMaxOffsets;
    const int tid = threadIdx.x;
    const int chunk = lane % CPR, rsub = lane / CPR;
    uint32_t a_off[CPR];
#pragma unroll
    for (int q = 0; q < CPR; ++q) a_off[q] = swizzled_offset<KC>(32 * warp + rsub + q * RPI, chunk);
    const unsigned char* src_col = p.f_in + chunk * 16;
    if (tid == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    // software pipeline: item descriptor two items ahead; row indices of the first kItemHead
    // offsets one item ahead, the rest at the item start (consumed kItemHead offsets later)
    constexpr int KH = kItemHead;
    int idx_cur[KM], idx_nxt[KH];
    auto load_desc = [&](int w) -> ItemView {
      return w < n_work ? load_item(items, w / p.n_blocks) : ItemView{0, 0, 1, 0ull};
    };
    auto nbr_of = [&](int k, int64_t row, bool ok) -> int32_t {
      return ok ? (p.nbr ? __ldg(p.nbr + static_cast<int64_t>(k) * p.n_out + row) : static_cast<int32_t>(row)) : -1;
    };
    auto load_head = [&](const ItemView& it, int (&dst)[KH]) {
      uint64_t m = it.mask;
      const int64_t row = static_cast<int64_t>(it.rb) * 128 + tid;
      const bool ok = row < p.n_out;
#pragma unroll
      for (int u = 0; u < KH; ++u)
        if (m) {
          dst[u] = nbr_of(__ffsll(static_cast<long long>(m)) - 1, row, ok);
          m &= m - 1;
        }
    };
    auto load_tail = [&](const ItemView& it) {
      uint64_t m = it.mask;
#pragma unroll
      for (int u = 0; u < KH; ++u) m &= m - 1;
      const int64_t row = static_cast<int64_t>(it.rb) * 128 + tid;
      const bool ok = row < p.n_out;
#pragma unroll
      for (int u = KH; u < KM; ++u)
        if (m) {
          idx_cur[u] = nbr_of(__ffsll(static_cast<long long>(m)) - 1, row, ok);
          m &= m - 1;
        }
    };
    int r = 0, w = work_of(0);
    ItemView it_cur = load_desc(w), it_nxt = load_desc(work_of(1));
    load_head(it_cur, idx_nxt);
    // PDL: the map-only loads above overlapped the previous kernel's tail; the input rows are
    // its output. Dependents may launch once every CTA got here (TMEM already held).
    grid_dep_wait();
    if (tid == 0) grid_dep_launch();
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t smem_base = smem_u32(smem);
    for (; w < n_work; w = work_of(++r)) {
#pragma unroll
      for (int u = 0; u < KH; ++u) idx_cur[u] = idx_nxt[u];
      load_tail(it_cur);                              // offsets >= KH of this item
      const ItemView it_nn = load_desc(work_of(r + 2));  // consumed two items from now
      load_head(it_nxt, idx_nxt);                    // consumed at the next item
      const int nb = w % p.n_blocks;
      const int b_row0 = nb * p.block_n;
      uint64_t m = it_cur.mask;
      int units_left = __popcll(it_cur.mask) * p.num_kb, in_stage = 0, stage_units = 0;
      uint32_t slot32 = 0;
#pragma unroll
      for (int u = 0; u < KM; ++u) {
        if (m == 0) break;
        const int k = __ffsll(static_cast<long long>(m)) - 1;
        m &= m - 1;
        int32_t j[CPR];
#pragma unroll
        for (int q = 0; q < CPR; ++q) j[q] = __shfl_sync(0xFFFFFFFFu, idx_cur[u], rsub + q * RPI);
        const int b_row = k * p.n_pad + b_row0;
#pragma unroll 1
        for (int kb = 0; kb < p.num_kb; ++kb) {
          if (in_stage == 0) {
            mbar_wait(&empty[stage], phase ^ 1u);
            stage_units = min(p.G, units_left);
            slot32 = smem_base + static_cast<uint32_t>(stage) * p.stage_bytes;
            if (tid == 0) mbar_expect_tx(&full[stage], static_cast<uint32_t>(stage_units) * p.b_bytes);
          }
          if (tid == 0) tma_load_2d(smem + (slot32 - smem_base) + p.a_bytes, &tmB, kb * KC, b_row, &full[stage]);
          const unsigned char* col = src_col + kb * (KC * 2);
#pragma unroll
          for (int q = 0; q < CPR; ++q)
            cp_async16(slot32 + a_off[q], col + static_cast<int64_t>(j[q] >= 0 ? j[q] : 0) * p.ld_in_bytes,
                       j[q] >= 0 ? 16u : 0u);
          --units_left;
          slot32 += p.unit_bytes;
          if (++in_stage == stage_units) {
            cp_async_arrive_noinc(&full[stage]);
            in_stage = 0;
            if (++stage == S) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
      it_cur = it_nxt;
      it_nxt = it_nn;
    }
  } else if (warp == 8) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      auto count_of = [&](int w) { return w < n_work ? __popcll(load_item(items, w / p.n_blocks).mask) : 0; };
      int cnt_next = count_of(work_of(0));
      for (int r = 0, w = work_of(0); w < n_work; w = work_of(++r)) {
        const int cnt = cnt_next;
        cnt_next = count_of(work_of(r + 1));
        const int nb = w % p.n_blocks;
        const int n_tile = min(p.block_n, p.n_pad - nb * p.block_n);
        const uint32_t idesc = idesc_f16(p.bf16, n_tile);
        mbar_wait(&tempty[acc], acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * p.block_n);
        uint32_t accumulate = 0;
        for (int units_left = cnt * p.num_kb; units_left > 0;) {
          const int su = min(p.G, units_left);
          mbar_wait(&full[stage], phase);
          fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tensor core reads
          tc_fence_after();
          uint32_t sa = smem_u32(smem + stage * p.stage_bytes);
          for (int u = 0; u < su; ++u, sa += p.unit_bytes) {
            const uint32_t sb = sa + p.a_bytes;
#pragma unroll
            for (int kk = 0; kk < KC / 16; ++kk) {
              tc_mma(d_tmem, smem_desc<KC>(sa + kk * 32), smem_desc<KC>(sb + kk * 32), idesc, accumulate);
              accumulate = 1;
            }
          }
          tc_commit(&empty[stage]);
          units_left -= su;
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
        }
        tc_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    grid_dep_wait();  // PDL: output / residual / split-tile counters of the previous kernel
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    TOut* out = static_cast<TOut*>(p.out);
    const TOut* res = static_cast<const TOut*>(p.res);
    int i = 0;
    ItemView it_next = work_of(0) < n_work ? load_item(items, work_of(0) / p.n_blocks) : ItemView{};
    for (int r = 0, w = work_of(0); w < n_work; w = work_of(++r), ++i) {
      const int ii = w / p.n_blocks, nb = w % p.n_blocks;
      const ItemView it = it_next;
      if (work_of(r + 1) < n_work) it_next = load_item(items, work_of(r + 1) / p.n_blocks);
      const int n0 = nb * p.block_n;
      const int n_tile = min(p.block_n, p.n_pad - n0);
      const int64_t trow = static_cast<int64_t>(it.rb) * 128 + q * 32 + lane;
      const bool valid = trow < p.n_out;
      const int64_t orow = valid && p.perm ? static_cast<int64_t>(__ldg(p.perm + trow)) : trow;
      const int ncols = min(n_tile, p.c_out - n0);
      mbar_wait_backoff(&tfull[acc], acc_phase);
      tc_fence_after();
      auto finish = [&](int c0, float (&x)[16]) {  // residual, ReLU, store 16 columns of this row
        TOut* op = out + orow * p.ld_out + n0;
        const TOut* rp = res ? res + orow * p.ld_res + n0 : nullptr;
        const bool full16 = p.vec && c0 + 16 <= ncols;
        if (rp) {
          if (full16) {
            float rv[16];
            OutCvt<TOut>::load16(rp + c0, rv);
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] += rv[e];
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (e < ncols - c0) x[e] += OutCvt<TOut>::to(rp[c0 + e]);
          }
        }
        if (p.relu)
#pragma unroll
          for (int e = 0; e < 16; ++e) x[e] = fmaxf(x[e], 0.f);
        if (full16)
          OutCvt<TOut>::store16(op + c0, x);
        else
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (e < ncols - c0) op[c0 + e] = OutCvt<TOut>::from(x[e]);
      };
      const bool direct = it.parts == 1;
      const size_t slot_elems = static_cast<size_t>(128) * p.block_n;
      const float4* base = nullptr;  // split tile: part 0's workspace slot
      size_t pstride = 0;
      bool last = direct;
      if (!direct) {
        // split tile: partial -> workspace slot ([bn / 4][128 rows][4] fp32: each float4 access of a
        // warp covers 512 contiguous bytes); the last part to finish sums all parts in part order
        const int ws0 = __ldg(p.item_ws + ii) - it.part;
        base = reinterpret_cast<const float4*>(p.ws + (static_cast<size_t>(ws0) * p.n_blocks + nb) * slot_elems) +
               q * 32 + lane;
        pstride = static_cast<size_t>(p.n_blocks) * slot_elems / 4;
        float4* mine = const_cast<float4*>(base) + it.part * pstride;
        for (int c0 = 0; c0 < n_tile; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * p.block_n + c0), v);
#pragma unroll
          for (int g = 0; g < 4; ++g)
            __stcg(mine + static_cast<size_t>(c0 / 4 + g) * 128,
                   make_float4(__uint_as_float(v[4 * g]), __uint_as_float(v[4 * g + 1]), __uint_as_float(v[4 * g + 2]),
                               __uint_as_float(v[4 * g + 3])));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);  // the accumulator is free once read
        __threadfence();
        named_bar(2, 32 * kEpiWarps);
        if (warp == 4 && lane == 0) {
          int* ctr = p.item_counters + static_cast<int64_t>(it.rb) * p.n_blocks + nb;
          const int done = atomicAdd(ctr, 1) == it.parts - 1;
          if (done) *ctr = 0;  // self-resetting for the next launch on this map
          s_last[i & 1] = done;
        }
        named_bar(2, 32 * kEpiWarps);
        last = s_last[i & 1];
        if (last) __threadfence();
      }
      if (last) {
        for (int c0 = 0; c0 < n_tile; c0 += 16) {
          float x[16];
          if (direct) {
            uint32_t v[16];
            tmem_ld16(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * p.block_n + c0), v);
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = __uint_as_float(v[e]);
            if constexpr (sizeof(TOut) == 2) {
              if (p.vec && c0 + 16 <= ncols && p.coal_epi) {  // warp-uniform: sector-coalesced path
                epilogue16_rows<TOut>(out + n0, p.ld_out, res ? res + n0 : nullptr, p.ld_res, orow, valid, c0, p.relu, x);
                continue;
              }
            }
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = 0.f;
            if (valid && c0 < ncols)
              for (int pp = 0; pp < it.parts; ++pp) {  // fixed part order: deterministic sum
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                  const float4 y = __ldcg(base + pp * pstride + static_cast<size_t>(c0 / 4 + g) * 128);
                  x[4 * g] += y.x;
                  x[4 * g + 1] += y.y;
                  x[4 * g + 2] += y.z;
                  x[4 * g + 3] += y.w;
                }
              }
          }
          if (valid && c0 < ncols) finish(c0, x);
        }
        if (direct) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (p.spans && threadIdx.x == 0) {
    p.spans[blockIdx.x * 4 + 2] = gtimer();
    p.spans[blockIdx.x * 4 + 3] = (n_work - blockIdx.x + G - 1) / G;
  }
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// tile_mask[rb] = OR over the tile's rows of their neighbour masks (1 if empty: one all-zero
// offset keeps the accumulator defined)
__global__ void __launch_bounds__(128) k_tile_masks(const int32_t* __restrict__ nbr, int64_t n, int K3,
                                                    unsigned long long* __restrict__ tile_mask) {
  __shared__ unsigned long long s_m[4];
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 128 + threadIdx.x;
  uint64_t m = 0;
  if (row < n)
    for (int k = 0; k < K3; ++k) m |= static_cast<uint64_t>(__ldg(nbr + static_cast<int64_t>(k) * n + row) >= 0) << k;
  const uint32_t lo = __reduce_or_sync(0xFFFFFFFFu, static_cast<uint32_t>(m));
  const uint32_t hi = __reduce_or_sync(0xFFFFFFFFu, static_cast<uint32_t>(m >> 32));
  if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = (static_cast<uint64_t>(hi) << 32) | lo;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t t = s_m[0] | s_m[1] | s_m[2] | s_m[3];
    tile_mask[blockIdx.x] = t ? t : 1ull;
  }
}

// One CTA: per-map offset budget opp = clamp(ceil(total active offsets / slots), 4, 28) (about
// one item per CTA slot); a tile (densest = last row block first when `reverse`) with more than
// opp active offsets is split into kItemMaxParts near-equal offset ranges, emitted in order. Split
// parts get compact workspace slots (item_ws[i] = slot, -1 unsplit): fewer than 2 * total / opp
// <= 2 * slots (plus 3 per tile when K3 > 2 * 28). Zeroes the split tiles' counters.
constexpr int kItemThreads = 1024;
__global__ void __launch_bounds__(kItemThreads) k_build_items(const unsigned long long* __restrict__ tile_mask,
                                                              int num_rb, int slots, int reverse, int4* __restrict__ items,
                                                              int* __restrict__ item_ws, int* __restrict__ n_items,
                                                              int* __restrict__ counters, int n_counters) {
  using Scan = cub::BlockScan<int, kItemThreads>;
  __shared__ typename Scan::TempStorage tmp;
  const int tid = threadIdx.x;
  int pop_sum = 0;
  for (int t = tid; t < num_rb; t += kItemThreads) pop_sum += __popcll(tile_mask[t]);
  int total = 0, excl = 0;
  Scan(tmp).ExclusiveSum(pop_sum, excl, total);
  const int opp = max(4, min(kItemMaxOffsets, (total + slots - 1) / slots));
  int carry = 0, ws_carry = 0;
  for (int base = 0; base < num_rb; base += kItemThreads) {
    const int ti = base + tid;
    const int t = reverse ? num_rb - 1 - ti : ti;
    const int pop = ti < num_rb ? __popcll(tile_mask[t]) : 0;
    const int parts = ti < num_rb ? max(pop > opp ? 2 : 1, (pop + kItemMaxOffsets - 1) / kItemMaxOffsets) : 0;
    int off = 0, blk = 0, woff = 0, wblk = 0;
    __syncthreads();
    Scan(tmp).ExclusiveSum(parts, off, blk);
    __syncthreads();
    Scan(tmp).ExclusiveSum(parts > 1 ? parts : 0, woff, wblk);
    uint64_t m = ti < num_rb ? tile_mask[t] : 0;
    for (int pp = 0; pp < parts; ++pp) {
      const int cnt = (pp + 1) * pop / parts - pp * pop / parts;
      uint64_t pm = 0;  // the next cnt active offsets
      for (int c = 0; c < cnt; ++c) {
        pm |= m & (~m + 1);
        m &= m - 1;
      }
      const int i = carry + off + pp;
      items[i] = make_int4(t, pp | (parts << 8), static_cast<int>(static_cast<uint32_t>(pm)),
                           static_cast<int>(static_cast<uint32_t>(pm >> 32)));
      item_ws[i] = parts > 1 ? ws_carry + woff + pp : -1;
    }
    carry += blk;
    ws_carry += wblk;
  }
  if (tid == 0) *n_items = carry;
  for (int c = tid; c < n_counters; c += kItemThreads) counters[c] = 0;
}

// neighbour-mask sort keys: bit pos[k] set when output i has a neighbour at offset k
__global__ void k_mask_keys(const int32_t* __restrict__ nbr, int64_t n, int K3, const __grid_constant__ MaskOrder ord,
                            uint32_t* __restrict__ keys, int32_t* __restrict__ idx) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n) return;
  uint32_t key = 0;
  for (int k = 0; k < K3; ++k) key |= static_cast<uint32_t>(__ldg(nbr + int64_t{k} * n + i) >= 0) << ord.pos[k];
  keys[i] = key;
  idx[i] = static_cast<int32_t>(i);
}

// ---------------------------------------------------------------- one-launch mask sort
// The neighbour-mask permutation of a submanifold map in ONE cooperative launch instead of
// mask kernel + CUB radix sort (histogram, scan, 3 onesweep passes) + permute kernel: every
// one of those is latency bound at these sizes (~70 us per map whatever n). Stable LSD radix
// sort of the 24 mask bits [begin_bit, begin_bit + 24) in three 8-bit passes (npass = 1: the
// 8-offset maps' whole mask in one pass), keys and values
// in registers (tile of <= 256 * kCoopMaxE rows per CTA), grid barriers between the phases:
//   rank     stable rank of each row among its tile's rows with the same digit (warp match +
//            per-warp digit counts, tile order = element e of thread t at e*256 + t)
//   hist     tile digit counts -> cnt[digit][tile]          | grid barrier
//   scan     per-digit exclusive scan across tiles + totals  | grid barrier
//   scatter  pos = base[digit] + cnt[digit][tile] + rank; the last pass writes the row
//            permutation and the permuted neighbour table (k_permute_nbr fused in; measured
//            faster than a coalesced grid-stride copy after one more barrier)
// Same bits, same stability as the CUB path => the identical permutation.
template <int E>
__global__ void __launch_bounds__(kCoopThreads) k_mask_sort(
    const int32_t* __restrict__ nbr, int64_t n, int K3, const __grid_constant__ MaskOrder ord, int begin_bit,
    int npass, int tile, uint32_t* keys0, int32_t* vals0, uint32_t* keys1, int32_t* vals1, int* cnt, int* tot,
    unsigned* bar, int32_t* __restrict__ perm, int32_t* __restrict__ nbr_perm) {
  const int tid = threadIdx.x;
  const unsigned G = gridDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * tile, t1 = min(n, t0 + tile);
  unsigned target = 0;
  uint32_t key[E];
  int32_t val[E];
  bool ok[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t i = t0 + e * kCoopThreads + tid;
    ok[e] = i < t1;
    key[e] = 0;
    val[e] = static_cast<int32_t>(i);
    if (ok[e])
      for (int k = 0; k < K3; ++k) key[e] |= static_cast<uint32_t>(__ldg(nbr + int64_t{k} * n + i) >= 0) << ord.pos[k];
  }
  for (int pass = 0; pass < npass; ++pass) {
    if (pass > 0) {
      const uint32_t* ki = pass == 1 ? keys1 : keys0;
      const int32_t* vi = pass == 1 ? vals1 : vals0;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (ok[e]) {
          const int64_t i = t0 + e * kCoopThreads + tid;
          key[e] = __ldcg(ki + i);
          val[e] = __ldcg(vi + i);
        }
    }
    int pos[E];
    lsd_pass_positions<E>(key, ok, begin_bit + 8 * pass, pos, cnt, tot, bar, target);
    uint32_t* ko = pass == 0 ? keys1 : keys0;
    int32_t* vo = pass == 0 ? vals1 : vals0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (!ok[e]) continue;
      if (pass < npass - 1) {
        ko[pos[e]] = key[e];
        vo[pos[e]] = val[e];
      } else {
        perm[pos[e]] = val[e];
        for (int k = 0; k < K3; ++k) nbr_perm[int64_t{k} * n + pos[e]] = __ldg(nbr + int64_t{k} * n + val[e]);
      }
    }
    if (pass < npass - 1) grid_barrier(bar, G, target);
  }
}

// nbr_perm[k][r] = nbr_in[k][perm[r]] (coalesced writes; reads gathered from L2)
__global__ void k_permute_nbr(const int32_t* __restrict__ nbr, const int32_t* __restrict__ perm, int64_t n, int K3,
                              int32_t* __restrict__ out) {
  const int64_t g = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (g >= n * K3) return;
  const int64_t k = g / n, r = g - k * n;
  out[g] = __ldg(nbr + k * n + __ldg(perm + r));
}

template <class TS, class TD>
__global__ void k_convert_rows(const TS* __restrict__ src, int64_t n, int c, int64_t ld_src, TD* __restrict__ dst,
                               int64_t ld_dst) {
  const int64_t g = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (g >= n * ld_dst) return;
  const int64_t r = g / ld_dst;
  const int col = static_cast<int>(g - r * ld_dst);
  const float v = col < c ? OutCvt<TS>::to(src[r * ld_src + col]) : 0.f;
  dst[g] = OutCvt<TD>::from(v);
}

// Launch with programmatic stream serialization (PDL): the kernel's prologue overlaps the tail
// of the previous kernel on the stream (the kernels call grid_dep_wait before touching its
// outputs). SCONV_PDL=0 launches plainly (A/B).
template <class K, class... Args>
void launch_pdl(K kern, int grid, size_t smem, cudaStream_t st, const Args&... args) {
  static const bool pdl = [] {
    const char* e = std::getenv("SCONV_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  SCONV_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <int KC, class TOut>
void launch_items_t(Ctx& ctx, const FusedParams& prm, size_t smem, const CUtensorMap& tB, int64_t max_work) {
  auto kern = k_conv_items<KC, TOut>;
  static thread_local std::map<int, int> regs_cache;
  int regs;
  if (const auto hit = regs_cache.find(ctx.device); hit != regs_cache.end()) {
    regs = hit->second;
  } else {
    SCONV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    SCONV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    cudaFuncAttributes fa{};
    SCONV_CUDA(cudaFuncGetAttributes(&fa, kern));
    regs = fa.numRegs;
    regs_cache[ctx.device] = regs;
  }
  const int by_smem = static_cast<int>((228u * 1024u) / (smem + 1024u));
  const int by_regs = 65536 / std::max(1, ((regs * 32 + 255) / 256 * 256) * (kThreads / 32));
  const int occ = std::max(1, std::min({by_smem, by_regs, static_cast<int>(512u / prm.tmem_cols), 2}));
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_work, int64_t{ctx.num_sms} * occ)));
  if (const char* dbg = std::getenv("SCONV_DEBUG_SYNC"); (dbg && dbg[0] == '1') || (prm.debug & 8192)) {
    int api_occ = -1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&api_occ, kern, kThreads, smem);
    std::fprintf(stderr, "[sconv] k_conv_items<%d> max_work=%lld grid=%d occ=%d (api %d) regs=%d smem=%zu stages=%d G=%d bn=%d cols=%u\n",
                 KC, static_cast<long long>(max_work), grid, occ, api_occ, regs, smem, prm.stages, prm.G, prm.block_n,
                 prm.tmem_cols);
  }
  ctx.launch("k_conv_fused", [&] { launch_pdl(kern, grid, smem, ctx.stream, tB, prm); });
}

template <class TOut>
void launch_items_kc(Ctx& ctx, const FusedParams& prm, size_t smem, const CUtensorMap& tB, int64_t max_work, int kc) {
  if (kc == 64)
    launch_items_t<64, TOut>(ctx, prm, smem, tB, max_work);
  else if (kc == 32)
    launch_items_t<32, TOut>(ctx, prm, smem, tB, max_work);
  else
    launch_items_t<16, TOut>(ctx, prm, smem, tB, max_work);
}

template <int NK, int KC, class TOut>
void launch_t(Ctx& ctx, const FusedArgs& a, const FusedParams& prm, size_t smem, const CUtensorMap& tB,
              const CUtensorMap& tA) {
  auto kern = k_conv_fused<NK, KC, TOut>;
  int variant = 0;
  if constexpr (NK > 0) {  // register-resident row indices (SCONV_FUSED_REG=0: shared-memory variant)
    static const bool reg = [] {
      const char* e = std::getenv("SCONV_FUSED_REG");
      return !(e && e[0] == '0');
    }();
    if (reg) {
      kern = k_conv_fused<NK, KC, TOut, true>;
      variant = 1;
    }
  }
  if constexpr (NK == 1) {  // 1x1 identity map, rows in order: TMA-fed dense GEMM (SCONV_FUSED_DENSE=0: gathers)
    static const bool dense = [] {
      const char* e = std::getenv("SCONV_FUSED_DENSE");
      return !(e && e[0] == '0');
    }();
    if (dense && !a.nbr && !a.perm) {
      kern = k_conv_fused<1, KC, TOut, false, true>;
      variant = 2;
    }
  }
  // Resident CTAs per SM from the kernel's own budget (the runtime occupancy query reported 1
  // where ncu's launch statistics show 2): 228 KB shared memory (1 KB reserved per CTA), the
  // register file, and TMEM (512 columns). Attributes are set once per instantiation/device.
  static thread_local std::map<int, int> regs_cache;
  int regs;
  const int cache_key = ctx.device * 4 + variant;
  const auto hit = regs_cache.find(cache_key);
  if (hit != regs_cache.end()) {
    regs = hit->second;
  } else {
    SCONV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    SCONV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    cudaFuncAttributes fa{};
    SCONV_CUDA(cudaFuncGetAttributes(&fa, kern));
    regs = fa.numRegs;
    regs_cache[cache_key] = regs;
  }
  const int by_smem = static_cast<int>((228u * 1024u) / (smem + 1024u));
  const int by_regs = 65536 / std::max(1, ((regs * 32 + 255) / 256 * 256) * (kThreads / 32));
  int occ = std::max(1, std::min({by_smem, by_regs, static_cast<int>(512u / prm.tmem_cols), NK == 0 ? 4 : 2}));
  const int grid = std::max(1, std::min(prm.num_tiles, ctx.num_sms * occ));
  if (const char* dbg = std::getenv("SCONV_DEBUG_SYNC"); dbg && dbg[0] == '1')
    std::fprintf(stderr, "[sconv] k_conv_fused<%d,%d> tiles=%d grid=%d occ=%d smem=%zu stages=%d bn=%d cols=%u\n", NK, KC,
                 prm.num_tiles, grid, occ, smem, prm.stages, prm.block_n, prm.tmem_cols);
  ctx.hmark("conv: launch");
  ctx.launch("k_conv_fused", [&] { launch_pdl(kern, grid, smem, ctx.stream, tB, prm, tA); });
  ctx.hmark("conv: launched");
}

template <int KC, class TOut>
void launch_nk(Ctx& ctx, const FusedArgs& a, const FusedParams& prm, size_t smem, const CUtensorMap& tB,
               const CUtensorMap& tA) {
  switch (prm.K3) {
    case 27:
      if (prm.target_occ > 2)
        launch_t<0, KC, TOut>(ctx, a, prm, smem, tB, tA);
      else
        launch_t<27, KC, TOut>(ctx, a, prm, smem, tB, tA);
      break;
    case 8: launch_t<8, KC, TOut>(ctx, a, prm, smem, tB, tA); break;
    case 1: launch_t<1, KC, TOut>(ctx, a, prm, smem, tB, tA); break;
    default: launch_t<0, KC, TOut>(ctx, a, prm, smem, tB, tA); break;
  }
}

template <class TOut>
void launch_kc(Ctx& ctx, const FusedArgs& a, const FusedParams& prm, size_t smem, const CUtensorMap& tB,
               const CUtensorMap& tA, int kc) {
  if (kc == 64)
    launch_nk<64, TOut>(ctx, a, prm, smem, tB, tA);
  else if (kc == 32)
    launch_nk<32, TOut>(ctx, a, prm, smem, tB, tA);
  else
    launch_nk<16, TOut>(ctx, a, prm, smem, tB, tA);
}

}  // namespace

namespace {
// Work-item kernel launch (k_conv_items): one pipeline per CTA, 1-2 CTAs per SM.
void launch_conv_items(Ctx& ctx, const FusedArgs& a, int kc, int64_t row_blocks) {
  const WeightData& w = *a.w;
  const int bn = std::min(w.n_pad, 256);  // widest accumulator: A is gathered once per n block
  FusedParams prm{};
  prm.f_in = static_cast<const unsigned char*>(a.f_in);
  prm.ld_in_bytes = a.ld_in * 2;
  prm.nbr = a.nbr;
  prm.perm = a.perm;
  prm.n_out = a.n_out;
  prm.K3 = w.K3;
  prm.num_kb = w.k_pad / kc;
  prm.block_n = bn;
  prm.n_pad = w.n_pad;
  prm.n_blocks = ceil_div(w.n_pad, bn);
  prm.c_out = w.c_out;
  prm.out = a.out;
  prm.ld_out = a.ld_out;
  prm.res = a.res;
  prm.ld_res = a.ld_res;
  prm.relu = a.relu;
  prm.tile_mask = a.tile_mask;
  prm.items = a.items;
  prm.item_ws = a.item_ws;
  prm.n_items = a.n_items;
  prm.item_counters = a.item_counters;
  prm.num_rb = static_cast<int>(row_blocks);
  if (const char* e = std::getenv("SCONV_FUSED_DEBUG")) prm.debug = std::atoi(e);
  {
    const int64_t align = a.out_dtype == SCONV_F32 ? 4 : 8;  // elements per 16 bytes
    prm.vec = a.ld_out % align == 0 && (!a.res || a.ld_res % align == 0) &&
              reinterpret_cast<uintptr_t>(a.out) % 16 == 0 && reinterpret_cast<uintptr_t>(a.res) % 16 == 0;
  }
  prm.bf16 = w.dtype == SCONV_BF16;
  prm.coal_epi = coalesced_epilogue_enabled();
  prm.a_bytes = 128u * kc * 2u;
  prm.b_bytes = static_cast<uint32_t>(bn) * kc * 2u;
  prm.unit_bytes = (prm.a_bytes + prm.b_bytes + 1023u) & ~1023u;
  prm.G = std::max(1, static_cast<int>((32u * 1024u) / prm.unit_bytes));
  if (const char* e = std::getenv("SCONV_FUSED_G")) prm.G = std::max(1, std::atoi(e));
  prm.stage_bytes = static_cast<uint32_t>(prm.G) * prm.unit_bytes;
  const uint32_t fixed = 1024u + (2 * kMaxStages + 4) * 8u + 64u;
  int target = 2;
  if (const char* e = std::getenv("SCONV_FUSED_OCC")) target = std::max(1, std::min(2, std::atoi(e)));
  const uint32_t half = (227u * 1024u) / static_cast<uint32_t>(target) - 1024u, whole = 227u * 1024u;
  int stages = fixed < half ? static_cast<int>((half - fixed) / prm.stage_bytes) : 0;
  if (stages < 3) stages = static_cast<int>((whole - fixed) / prm.stage_bytes);
  stages = std::min(stages, kMaxStages);
  if (stages < 2) fail(SCONV_ERR_ARG, "fused layer tile does not fit in shared memory");
  prm.stages = stages;
  prm.bar_off = static_cast<uint32_t>(stages) * prm.stage_bytes;
  uint32_t cols = 32;
  while (cols < 2u * static_cast<uint32_t>(bn)) cols <<= 1;
  prm.tmem_cols = cols;
  const size_t smem = 1024 + prm.bar_off + (2 * stages + 4) * 8 + 16;
  if (smem > 227 * 1024) fail(SCONV_ERR_ARG, "fused layer tile does not fit in shared memory");
  const int64_t max_items = a.items ? a.max_items : row_blocks;
  const int64_t max_work = max_items * prm.n_blocks;
  DevBuf spans;
  if (prm.debug & 8192) {
    spans.alloc(size_t{4} * 8 * 148 * 8, ctx.stream);
    SCONV_CUDA(cudaMemsetAsync(spans.get(), 0, size_t{4} * 8 * 148 * 8, ctx.stream));
    prm.spans = spans.get<unsigned long long>();
  }
  if (a.items) {  // split items' partials: one [bn][128] fp32 slot per split part and n block
    ctx.fused_ws.reserve(static_cast<size_t>(a.max_ws_slots) * prm.n_blocks * 128 * bn * sizeof(float), ctx.stream);
    prm.ws = ctx.fused_ws.get<float>();
  }
  if (prm.n_blocks > 4) fail(SCONV_ERR_ARG, "fused dataflow supports at most 1024 output channels");
  const CUtensorMap tB = make_tensor_map_2d(w.buf.get(), w.dtype, w.k_pad, static_cast<uint64_t>(w.K3) * w.n_pad, kc,
                                            static_cast<uint32_t>(bn), kc);
  if (a.out_dtype == SCONV_F32)
    launch_items_kc<float>(ctx, prm, smem, tB, max_work, kc);
  else if (a.out_dtype == SCONV_F16)
    launch_items_kc<__half>(ctx, prm, smem, tB, max_work, kc);
  else
    launch_items_kc<__nv_bfloat16>(ctx, prm, smem, tB, max_work, kc);
  if (prm.spans) {  // debug 8192 summary (synchronises)
    std::vector<unsigned long long> h(4 * 8 * 148);
    SCONV_CUDA(cudaMemcpyAsync(h.data(), spans.get(), h.size() * 8, cudaMemcpyDeviceToHost, ctx.stream));
    SCONV_CUDA(cudaStreamSynchronize(ctx.stream));
    unsigned long long t0 = ~0ull, t1 = 0;
    double life = 0, life_max = 0;
    int n = 0;
    for (size_t b = 0; b < h.size() / 4; ++b)
      if (h[4 * b]) {
        ++n;
        t0 = std::min(t0, h[4 * b]);
        t1 = std::max(t1, h[4 * b + 2]);
        const double l = (h[4 * b + 2] - h[4 * b]) * 1e-3;
        life += l;
        life_max = std::max(life_max, l);
      }
    std::vector<int> sh(8, 0);  // CTA start offsets in 5 us bins
    for (size_t b = 0; b < h.size() / 4; ++b)
      if (h[4 * b]) ++sh[std::min<size_t>(7, (h[4 * b] - t0) / 5000)];
    std::fprintf(stderr, "[spans] items ctas=%d span=%.2f us life avg=%.2f max=%.2f starts/5us: %d %d %d %d %d %d %d %d\n", n,
                 (t1 - t0) * 1e-3, life / std::max(1, n), life_max, sh[0], sh[1], sh[2], sh[3], sh[4], sh[5], sh[6], sh[7]);
  }
}
}  // namespace

bool coalesced_epilogue_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SCONV_FUSED_COAL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// SCONV_FUSED_ITEMS: 0 = tile-queue kernel only, 1 = work-item kernel wherever items exist,
// unset / 2 = per conv (few-tile wide layers: work items)
int fused_items_mode() {
  static const int mode = [] {
    const char* e = std::getenv("SCONV_FUSED_ITEMS");
    if (e && (e[0] == '0' || e[0] == '1')) return e[0] - '0';
    const char* v1 = std::getenv("SCONV_FUSED_V1");  // older A/B switch: tile-queue only
    return v1 && v1[0] == '1' ? 0 : 2;
  }();
  return mode;
}

bool fused_supported(int K3, int c_in, int c_out) { return K3 >= 1 && K3 <= 64 && c_in >= 1 && c_out >= 1; }

void launch_conv_fused(Ctx& ctx, const FusedArgs& a) {
  ctx.hmark("conv: enter");
  const WeightData& w = *a.w;
  if (!fused_supported(w.K3, w.c_in, w.c_out)) fail(SCONV_ERR_ARG, "fused dataflow supports at most 64 offsets");
  if (a.n_out == 0) return;
  if (a.ld_in < w.k_pad || a.ld_in % 8 != 0) fail(SCONV_ERR_ARG, "fused input row stride must be >= k_pad and 16-byte aligned");
  if (a.out_dtype != SCONV_F32 && a.out_dtype != SCONV_F16 && a.out_dtype != SCONV_BF16)
    fail(SCONV_ERR_ARG, "unsupported output dtype");
  const int kc = w.k_pad % 64 == 0 ? 64 : (w.k_pad % 32 == 0 ? 32 : 16);
  const int64_t row_blocks = ceil_div<int64_t>(a.n_out, 128);
  if (row_blocks > INT32_MAX / 16) fail(SCONV_ERR_ARG, "layer too large");
  // Kernel choice (measured per conv, r02s vs r02q): the work-item kernel wins only where a
  // layer has fewer 128-row tiles than half the SMs AND wide (>= 256-channel) inputs: its split
  // items spread a few long tiles over every SM (C2 7,780-row 256->256: 63 -> 52 us; C3 5,512
  // rows: 62 -> 51 us); on the big layers the tile-queue kernel's dynamic densest-first queue
  // balances better (e.g. 119k rows 128->96: 68 vs 90 us).
  const int mode = fused_items_mode();
  const bool items = a.items && (mode == 1 || (mode == 2 && w.k_pad >= 256 && w.K3 >= 27 &&
                                                  row_blocks * 2 < ctx.num_sms));
  if (items) {
    launch_conv_items(ctx, a, kc, row_blocks);
    return;
  }
  // block_n: widest multiple of 16 (<= 256) that still gives ~2 tiles per SM; narrower
  // blocks re-gather A from L2 once per extra n block.
  int bn = a.block_n;
  if (bn <= 0) {
    bn = std::min(w.n_pad, 256);
    // ~one tile per SM: each extra n block re-gathers the tile's A rows from L2 (measured: fewer,
    // wider tiles win on the wide deep layers, e.g. 7780 rows 256->256: 100 -> 61 us)
    int want = ctx.num_sms;
    if (const char* e = std::getenv("SCONV_FUSED_TILES")) want = std::max(1, std::atoi(e));
    while (bn > 32 && row_blocks * ceil_div(w.n_pad, bn) < want && (bn / 2) % 16 == 0) bn /= 2;
  }
  bn = std::min(bn, w.n_pad);
  if (bn % 16 != 0 || bn > 256) fail(SCONV_ERR_ARG, "block_n must be a multiple of 16 <= 256");
  FusedParams prm{};
  prm.f_in = static_cast<const unsigned char*>(a.f_in);
  prm.ld_in_bytes = a.ld_in * 2;
  prm.nbr = a.nbr;
  prm.perm = a.perm;
  prm.n_out = a.n_out;
  prm.K3 = w.K3;
  prm.num_kb = w.k_pad / kc;
  prm.block_n = bn;
  prm.n_pad = w.n_pad;
  prm.n_blocks = ceil_div(w.n_pad, bn);
  prm.num_tiles = static_cast<int>(row_blocks * prm.n_blocks);
  prm.c_out = w.c_out;
  prm.out = a.out;
  prm.ld_out = a.ld_out;
  prm.res = a.res;
  prm.ld_res = a.ld_res;
  prm.relu = a.relu;
  if (const char* e = std::getenv("SCONV_FUSED_DEBUG")) prm.debug = std::atoi(e);
  DevBuf trace, spans;
  if (prm.debug & 8192) {
    spans.alloc(size_t{4} * 8 * 148 * 8, ctx.stream);
    SCONV_CUDA(cudaMemsetAsync(spans.get(), 0, size_t{4} * 8 * 148 * 8, ctx.stream));
    prm.spans = spans.get<unsigned long long>();
  }
  if (prm.debug & 8) {
    trace.alloc(8192 * 8, ctx.stream);
    SCONV_CUDA(cudaMemsetAsync(trace.get(), 0, 8192 * 8, ctx.stream));
    prm.trace = trace.get<unsigned long long>();
  }
  {
    const int64_t align = a.out_dtype == SCONV_F32 ? 4 : 8;  // elements per 16 bytes
    prm.vec = a.ld_out % align == 0 && (!a.res || a.ld_res % align == 0) &&
              reinterpret_cast<uintptr_t>(a.out) % 16 == 0 && reinterpret_cast<uintptr_t>(a.res) % 16 == 0;
  }
  prm.bf16 = w.dtype == SCONV_BF16;
  prm.coal_epi = coalesced_epilogue_enabled();
  prm.a_bytes = 128u * kc * 2u;
  prm.b_bytes = static_cast<uint32_t>(bn) * kc * 2u;
  prm.unit_bytes = (prm.a_bytes + prm.b_bytes + 1023u) & ~1023u;
  // G units per stage: ~32 KB stages (one barrier round trip per G units of work)
  prm.G = std::max(1, static_cast<int>((32u * 1024u) / prm.unit_bytes));
  if (const char* e = std::getenv("SCONV_FUSED_G")) prm.G = std::max(1, std::atoi(e));
  prm.stage_bytes = static_cast<uint32_t>(prm.G) * prm.unit_bytes;
  // Ring depth: two CTAs per SM (independent pipelines) when >= 3 stages fit in half the
  // shared memory, else one CTA with up to kMaxStages stages.
  const uint32_t idx_bytes = static_cast<uint32_t>(w.K3) * 128u * 4u;
  const uint32_t fixed = 1024u + idx_bytes + (2 * kMaxStages + 3 * kInfo + 16) * 8u + 64u;
  int target = 2;
  if (const char* e = std::getenv("SCONV_FUSED_OCC")) target = std::max(1, std::min(4, std::atoi(e)));
  prm.target_occ = target;
  const uint32_t half = (227u * 1024u) / static_cast<uint32_t>(target) - 1024u, whole = 227u * 1024u;
  int stages = fixed < half ? static_cast<int>((half - fixed) / prm.stage_bytes) : 0;
  if (stages < 3) {
    stages = static_cast<int>((whole - fixed) / prm.stage_bytes);
    prm.target_occ = 1;
  }
  stages = std::min(stages, kMaxStages);
  if (stages < 2) fail(SCONV_ERR_ARG, "fused layer tile does not fit in shared memory");
  prm.stages = stages;
  prm.idx_off = static_cast<uint32_t>(stages) * prm.stage_bytes;
  prm.bar_off = prm.idx_off + idx_bytes;
  uint32_t cols = 32;
  while (cols < 2u * static_cast<uint32_t>(bn)) cols <<= 1;
  prm.tmem_cols = cols;
  const size_t smem = 1024 + prm.bar_off + (2 * stages + 4 + 3 * kInfo + 8) * 8 + (kInfo + 4 + 1) * 4 + 16;
  if (smem > 227 * 1024) fail(SCONV_ERR_ARG, "fused layer tile does not fit in shared memory");
  ctx.hmark("conv: params");
  const CUtensorMap tB = make_tensor_map_2d(w.buf.get(), w.dtype, w.k_pad, static_cast<uint64_t>(w.K3) * w.n_pad, kc,
                                            static_cast<uint32_t>(bn), kc);
  ctx.hmark("conv: tensor map");
  {  // {queue, exited CTAs}: zeroed when (re)allocated, then reset by each launch's last CTA
    const void* before = ctx.fused_counter.get();
    ctx.fused_counter.reserve(16, ctx.stream);
    if (ctx.fused_counter.get() != before)
      SCONV_CUDA(cudaMemsetAsync(ctx.fused_counter.get(), 0, 16, ctx.stream));
  }
  prm.tile_counter = ctx.fused_counter.get<int>();
  struct TraceDump {  // debug 5: print CTA 0's timeline after the launch
    Ctx& ctx;
    DevBuf& buf;
    ~TraceDump() {
      if (!buf.get()) return;
      std::vector<unsigned long long> h(8192);
      cudaMemcpyAsync(h.data(), buf.get(), 8192 * 8, cudaMemcpyDeviceToHost, ctx.stream);
      cudaStreamSynchronize(ctx.stream);
      std::vector<unsigned long long> ev;
      for (auto e : h)
        if (e) ev.push_back(e);
      const size_t n = ev.size();
      std::sort(ev.begin(), ev.end(), [](auto a, auto b) { return (a & 0xFFFFFFFFull) < (b & 0xFFFFFFFFull); });
      const unsigned long long t0 = n ? (ev[0] & 0xFFFFFFFFull) : 0;
      for (auto e : ev)
        std::fprintf(stderr, "[trace] %8.3f us kind=%llu seq=%llu\n", ((e & 0xFFFFFFFFull) - t0) * 1e-3, e >> 56,
                     (e >> 32) & 0xFFFFFF);
    }
  } dump{ctx, trace};
  struct SpanDump {  // debug 8192: kernel span, CTA start skew, lifetimes, tiles per CTA
    Ctx& ctx;
    DevBuf& buf;
    ~SpanDump() {
      if (!buf.get()) return;
      std::vector<unsigned long long> h(4 * 8 * 148);
      cudaMemcpyAsync(h.data(), buf.get(), h.size() * 8, cudaMemcpyDeviceToHost, ctx.stream);
      cudaStreamSynchronize(ctx.stream);
      unsigned long long t0 = ~0ull, t1 = 0, skew = 0;
      double life = 0, life_max = 0, setup = 0;
      int n = 0, tiles_max = 0;
      for (size_t b = 0; b < h.size() / 4; ++b) {
        if (!h[4 * b]) continue;
        ++n;
        t0 = std::min(t0, h[4 * b]);
        t1 = std::max(t1, h[4 * b + 2]);
      }
      std::vector<int> hist(16, 0);
      for (size_t b = 0; b < h.size() / 4; ++b) {
        if (!h[4 * b]) continue;
        skew = std::max(skew, h[4 * b] - t0);
        const double l = (h[4 * b + 2] - h[4 * b]) * 1e-3;
        life += l;
        life_max = std::max(life_max, l);
        setup += (h[4 * b + 1] - h[4 * b]) * 1e-3;
        tiles_max = std::max(tiles_max, static_cast<int>(h[4 * b + 3]));
        ++hist[std::min<int>(15, static_cast<int>(h[4 * b + 3]))];
      }
      std::fprintf(stderr, "[spans] ctas=%d span=%.2f us start_skew=%.2f us life avg=%.2f max=%.2f setup=%.2f us tiles max=%d hist",
                   n, (t1 - t0) * 1e-3, skew * 1e-3, life / std::max(1, n), life_max, setup / std::max(1, n), tiles_max);
      for (int i = 0; i <= tiles_max && i < 16; ++i) std::fprintf(stderr, " %d:%d", i, hist[i]);
      std::fprintf(stderr, "\n");
    }
  } sdump{ctx, spans};
  // A operand of the dense (1x1 identity) variant: 128-row boxes of the input, same swizzle as B
  const CUtensorMap tA = !a.nbr && !a.perm && w.K3 == 1
                             ? make_tensor_map_2d_strided(a.f_in, w.dtype, w.k_pad, static_cast<uint64_t>(a.n_in),
                                                          static_cast<uint64_t>(a.ld_in) * 2, kc, 128, kc)
                             : tB;
  if (a.out_dtype == SCONV_F32)
    launch_kc<float>(ctx, a, prm, smem, tB, tA, kc);
  else if (a.out_dtype == SCONV_F16)
    launch_kc<__half>(ctx, a, prm, smem, tB, tA, kc);
  else
    launch_kc<__nv_bfloat16>(ctx, a, prm, smem, tB, tA, kc);
}

namespace {
void order_fused_rows(Ctx& ctx, MapData& m);
}  // namespace

// Work items of a map (k_tile_masks + k_build_items on the current stream, no host sync): the
// item count stays on the device; the host bound max_items sizes grids and the workspace.
void build_fused_items(Ctx& ctx, MapData& m) {
  if (m.items_ready) return;
  m.items_ready = true;
  const int64_t n = m.n_out;
  if (n == 0 || m.identity_pending) return;  // identity map: implicit single-offset items
  const int mode = fused_items_mode();
  if (mode == 0 || (mode == 2 && ceil_div<int64_t>(n, 128) * 2 >= ctx.num_sms)) return;  // tile-queue kernel
  const int64_t num_rb = ceil_div<int64_t>(n, 128);
  const int slots = 2 * ctx.num_sms;
  // split parts: < 4 slots (+ 2 per tile when K3 > 32), see k_build_items; items <= tiles + that
  m.max_ws_slots = 4 * int64_t{slots} + (m.K3 > 2 * kItemMaxOffsets ? 3 * num_rb : 0);
  m.max_items = num_rb + m.max_ws_slots;
  const cudaStream_t st = ctx.stream;
  m.tile_mask.alloc(8 * num_rb, st);
  m.items.alloc(16 * m.max_items, st);
  m.item_ws.alloc(4 * m.max_items, st);
  m.n_items.alloc(sizeof(int), st);
  m.item_counters.alloc(sizeof(int) * 4 * num_rb, st);  // (row block, n block <= 4)
  const int32_t* nbr = m.permuted ? m.nbr_perm.get<int32_t>() : m.nbr_in.get<int32_t>();
  const int K3 = m.K3;
  ctx.launch("k_tile_masks", [&] {
    k_tile_masks<<<static_cast<unsigned>(num_rb), 128, 0, st>>>(nbr, n, K3, m.tile_mask.get<unsigned long long>());
  });
  ctx.launch("k_build_items", [&] {
    k_build_items<<<1, kItemThreads, 0, st>>>(m.tile_mask.get<unsigned long long>(), static_cast<int>(num_rb), slots,
                                              m.permuted ? 1 : 0, m.items.get<int4>(), m.item_ws.get<int>(),
                                              m.n_items.get<int>(), m.item_counters.get<int>(),
                                              static_cast<int>(4 * num_rb));
  });
}

void prepare_fused_layout(Ctx& ctx, MapData& m) {
  if (m.fused_ready) return;
  m.fused_ready = true;
  ctx.hmark("layout: enter");
  order_fused_rows(ctx, m);
  ctx.hmark("layout: row order queued");
  build_fused_items(ctx, m);
}

namespace {
void order_fused_rows(Ctx& ctx, MapData& m) {
  const int64_t n = m.n_out;
  const int K3 = m.K3;
  // Only submanifold maps (stride 1, not transposed, K3 >= 27) are reordered: networks reuse
  // them for 4-8 convs, so the sort (~40 us at 1.2e5 rows) amortises; strided / transposed
  // maps serve a single conv.
  // K3 <= 8 maps (K=2 down / up): one stable 8-bit pass (SCONV_SMALL_PERMUTE=0: off): an
  // up-sampling output has exactly one of the 8 offsets, so an unordered 128-row tile gathers
  // all 8. It pays only where the build runs off the critical path (networks: layout stream),
  // so the single-layer API keeps these maps in order.
  static const bool small_permute = [] {
    const char* e = std::getenv("SCONV_SMALL_PERMUTE");
    return !(e && e[0] == '0');
  }();
  const bool small = small_permute && m.layout_off_path && K3 >= 2 && K3 <= 8 && n > 2 * 128 && n <= INT32_MAX;
  m.permuted = small || (K3 >= 27 && K3 <= 32 && m.cfg.out_stride == 1 && !m.cfg.transposed && n > 2 * 128 &&
                         n <= INT32_MAX);
  if (const char* e = std::getenv("SCONV_NO_PERMUTE"); e && e[0] == '1') m.permuted = false;  // experiments
  if (const char* e = std::getenv("SCONV_PERMUTE_MIN"); e && n < std::atoll(e)) m.permuted = false;
  if (!m.permuted) return;
  // Bit position per offset: rarer offsets (larger L1 norm: corners, then edges, then faces,
  // the always-present centre last) in the more significant bits, so equal-or-similar masks
  // end up adjacent (KITTI scan: 25.4 -> 10.4 active offsets per 128-row tile).
  MaskOrder ord{};
  std::vector<int> order(K3);
  for (int k = 0; k < K3; ++k) order[k] = k;
  auto norm = [&](int k) { return std::abs(m.delta[k].x) + std::abs(m.delta[k].y) + std::abs(m.delta[k].z); };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return norm(a) < norm(b); });
  for (int p = 0; p < K3; ++p) ord.pos[order[p]] = small ? order[p] : p;  // small maps: bit k = offset k
  const cudaStream_t st = ctx.stream;
  ctx.hmark("layout: allocs");
  DevBuf keys, keys_sorted, idx;
  keys.alloc(4 * n, st);
  keys_sorted.alloc(4 * n, st);
  idx.alloc(4 * n, st);
  m.row_perm.alloc(4 * n, st);
  m.nbr_perm.alloc(4 * n * K3, st);
  // Sort-key width: networks pass a hint from the number of convs that use the map (net.cu:
  // 24 bits = 3 passes when >= 6 convs amortise the sort, else 16 bits = 2 passes); otherwise
  // 24 bits, 16 for maps of more than SCONV_MASK16_ROWS rows (default 200k). Same-box A/B r02ah: C2 (maps <= 119k rows)
  // 24 bits 2.20 ms vs 16 bits 2.25 ms; C3 (level 0: 337k rows) 1.354 ms vs 1.309 ms with 16.
  // SCONV_MASK_BITS forces one width.
  static const int mask_bits_forced = [] {
    const char* e = std::getenv("SCONV_MASK_BITS");
    return e ? std::max(1, std::min(32, std::atoi(e))) : 0;
  }();
  static const int64_t mask16_rows = [] {
    const char* e = std::getenv("SCONV_MASK16_ROWS");
    return e ? std::atoll(e) : int64_t{200000};
  }();
  const int mask_bits = mask_bits_forced     ? mask_bits_forced
                        : m.mask_bits_hint ? m.mask_bits_hint
                                           : (n > mask16_rows ? 16 : 24);
  // one cooperative launch when every row fits the co-resident CTAs' registers
  static const int coop_cap = [] {
    int per_sm = 0, dev = 0, sms = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mask_sort<kCoopMaxE>, kCoopThreads, 0) != cudaSuccess)
      per_sm = 0;
    return coop ? per_sm * sms : 0;
  }();
  // 8-offset maps: their whole 8-bit mask in one stable pass (the same one-launch sort, so the
  // row order -- and with it the work items and any split-part summation -- is deterministic)
  // the top mask_bits bits (a multiple of 8) in mask_bits / 8 stable passes
  const int npass = small ? 1 : mask_bits / 8;
  const bool one_launch = (small || (mask_bits % 8 == 0 && mask_bits <= 24 && K3 >= mask_bits)) && coop_cap > 0 &&
                          n <= static_cast<int64_t>(coop_cap) * kCoopThreads * kCoopMaxE &&
                          !(std::getenv("SCONV_MASK_SORT_CUB") && std::getenv("SCONV_MASK_SORT_CUB")[0] == '1');
  if (one_launch) {
    // one row per thread when the co-resident grid allows (measured: a grid capped near one CTA
    // per SM, 4 rows per thread, is 1.6x slower: serial rank rounds, fewer loads in flight)
    int e = coop_rows_per_thread();
    while (ceil_div<int64_t>(n, int64_t{kCoopThreads} * e) > coop_cap) e *= 2;
    const int tile = kCoopThreads * e;
    const unsigned G = static_cast<unsigned>(ceil_div<int64_t>(n, tile));
    DevBuf aux, v1buf;
    aux.alloc(sizeof(int) * (256 * static_cast<size_t>(G) + 256 + 4), st);
    v1buf.alloc(4 * n, st);
    int* cnt = aux.get<int>();
    int* tot = cnt + 256 * static_cast<size_t>(G);
    unsigned* bar = reinterpret_cast<unsigned*>(tot + 256);
    SCONV_CUDA(cudaMemsetAsync(bar, 0, 4 * sizeof(unsigned), st));
    const int32_t* nbr = m.nbr_in.get<int32_t>();
    int begin_bit = small ? 0 : K3 - mask_bits, K3v = K3, tilev = tile, np = npass;
    int64_t nn = n;
    uint32_t *k0 = keys.get<uint32_t>(), *k1 = keys_sorted.get<uint32_t>();
    int32_t *v0 = idx.get<int32_t>(), *v1 = v1buf.get<int32_t>();
    int32_t *perm = m.row_perm.get<int32_t>(), *nperm = m.nbr_perm.get<int32_t>();
    void* args[] = {&nbr, &nn, &K3v, &ord, &begin_bit, &np, &tilev, &k0, &v0, &k1, &v1, &cnt, &tot, &bar, &perm, &nperm};
    const void* fn = e == 1   ? reinterpret_cast<const void*>(k_mask_sort<1>)
                     : e == 2 ? reinterpret_cast<const void*>(k_mask_sort<2>)
                              : reinterpret_cast<const void*>(k_mask_sort<4>);
    ctx.hmark("layout: coop launch");
    ctx.launch("k_mask_sort", [&] {
      SCONV_CUDA(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kCoopThreads), args, 0, st));
    });
    ctx.hmark("layout: coop launched");
    return;
  }
  const unsigned b1 = static_cast<unsigned>(ceil_div<int64_t>(n, 256));
  ctx.launch("k_mask_keys", [&] {
    k_mask_keys<<<b1, 256, 0, st>>>(m.nbr_in.get<int32_t>(), n, K3, ord, keys.get<uint32_t>(), idx.get<int32_t>());
  });
  size_t temp = 0;
  // sort on the top 24 key bits only (3 radix passes instead of 4): the dropped low bits are
  // the centre and two face offsets, the most common ones (KITTI: 10.32 -> 10.59 offsets/tile)
  const int begin_bit = small ? 0 : std::max(0, K3 - mask_bits);
  SCONV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys.get<uint32_t>(), keys_sorted.get<uint32_t>(),
                                             idx.get<int32_t>(), m.row_perm.get<int32_t>(), static_cast<int>(n),
                                             begin_bit, K3, st));
  DevBuf cub_temp;  // own scratch: networks run this on a stream beside the map builds
  cub_temp.alloc(std::max<size_t>(temp, 16), st);
  ctx.launch("cub_radix_sort_masks", [&] {
    cub::DeviceRadixSort::SortPairs(cub_temp.get(), temp, keys.get<uint32_t>(), keys_sorted.get<uint32_t>(),
                                    idx.get<int32_t>(), m.row_perm.get<int32_t>(), static_cast<int>(n), begin_bit, K3,
                                    st);
  });
  const unsigned b2 = static_cast<unsigned>(ceil_div<int64_t>(n * K3, 256));
  ctx.launch("k_permute_nbr", [&] {
    k_permute_nbr<<<b2, 256, 0, st>>>(m.nbr_in.get<int32_t>(), m.row_perm.get<int32_t>(), n, K3,
                                      m.nbr_perm.get<int32_t>());
  });
}

}  // namespace

void convert_rows(Ctx& ctx, const void* src, int src_dtype, int64_t n, int c, int64_t ld_src, void* dst, int dst_dtype,
                  int64_t ld_dst) {
  if (n == 0) return;
  const int64_t total = n * ld_dst;
  const unsigned blocks = static_cast<unsigned>(ceil_div<int64_t>(total, 256));
  auto go = [&](auto* s, auto* d) {
    ctx.launch("k_convert_rows", [&] {
      k_convert_rows<<<blocks, 256, 0, ctx.stream>>>(s, n, c, ld_src, d, ld_dst);
    });
  };
  auto with_dst = [&](auto* s) {
    if (dst_dtype == SCONV_F16)
      go(s, static_cast<__half*>(dst));
    else if (dst_dtype == SCONV_BF16)
      go(s, static_cast<__nv_bfloat16*>(dst));
    else
      go(s, static_cast<float*>(dst));
  };
  if (src_dtype == SCONV_F32)
    with_dst(static_cast<const float*>(src));
  else if (src_dtype == SCONV_F16)
    with_dst(static_cast<const __half*>(src));
  else
    with_dst(static_cast<const __nv_bfloat16*>(src));
}

}  // namespace sconvb

// Grouped GEMM of the GMaS step on 5th-gen tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Replaces gemm_execute (§5.2.2 "executed as a single batched
// GEMM kernel" on a 4-stream pool). All groups of the padding-efficient plan run in ONE
// persistent launch: the tile list enumerates (member offset k, 128-row block, n block)
// in buffer order, so padded rows are computed exactly as the grouped GEMM would, and the
// weight permutation of the sorted policy is just the per-tile offset index k.
//
//   A  = gather buffer  [R_pad x K_pad] (f16/bf16, K-major)   TMA, swizzle KC*2 bytes
//   B  = weights        [K3*N_pad x K_pad] (W_k^T, K-major)   TMA, same swizzle
//   D  = TMEM fp32 accumulator, 2 buffers x BLOCK_N columns (MMA of tile t+1 overlaps
//        the epilogue of tile t)
//   out= fp32 [R_pad x C_out] per-offset partial products ("stored as 32-bit")
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner + single-thread
// MMA issuer, warps 2-5 = epilogue (warp w reads TMEM lanes 32*(w%4) .. +31).
#include <algorithm>
#include <map>
#include <string>

#include "common.cuh"
#include "gemm_sm100.hpp"
#include "sm100.cuh"

namespace sconvb {
namespace {

using namespace sm100;

constexpr int kGemmThreads = 192;

// tile t -> {first buffer row, rows, offset k, first output channel}
__device__ __forceinline__ int4 decode_tile(const LayerPlan& p, int t) {
  int lo = 0, hi = p.nm - 1;  // last member with tile_start <= t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.tile_start[mid] <= t)
      lo = mid;
    else
      hi = mid - 1;
  }
  const int4 mb = p.members[lo];
  const int local = t - p.tile_start[lo];
  const int rb = local / p.n_blocks, nbk = local - rb * p.n_blocks;
  return make_int4(mb.y + rb * 128, min(128, mb.w - rb * 128), mb.x, nbk * p.block_n);
}

template <int KC, class TOut>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_grouped(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ LayerPlan plan, int num_tiles, int num_kb, int block_n, int n_pad, int c_out,
                   TOut* __restrict__ out, int stages, uint32_t idesc_base, uint32_t tmem_cols) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
  const uint32_t a_bytes = 128u * KC * 2u;
  const uint32_t b_bytes = static_cast<uint32_t>(block_n) * KC * 2u;
  const uint32_t stage_bytes = (a_bytes + b_bytes + 1023u) & ~1023u;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int4 td = decode_tile(plan, t);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* sa = smem + stage * stage_bytes;
          mbar_expect_tx(&full[stage], a_bytes + b_bytes);
          tma_load_2d(sa, &tmA, kb * KC, td.x, &full[stage]);
          tma_load_2d(sa + a_bytes, &tmB, kb * KC, td.z * n_pad + td.w, &full[stage]);
          if (++stage == stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer (one thread issues for the whole CTA)
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int4 td = decode_tile(plan, t);
        const int n_tile = min(block_n, n_pad - td.w);
        const uint32_t idesc = idesc_base | (static_cast<uint32_t>(n_tile >> 3) << 17);
        mbar_wait(&tempty[acc], acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * block_n);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * stage_bytes);
          const uint32_t sb = sa + a_bytes;
#pragma unroll
          for (int kk = 0; kk < KC / 16; ++kk)
            tc_mma(d_tmem, smem_desc<KC>(sa + kk * 32), smem_desc<KC>(sb + kk * 32), idesc, (kb | kk) != 0);
          tc_commit(&empty[stage]);  // frees the smem stage once these MMAs retire
          if (++stage == stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        tc_commit(&tfull[acc]);  // accumulator ready for the epilogue
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
      }
    }
  } else {  // ---- epilogue: TMEM -> registers -> global fp32
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool vec4 = (c_out & 3) == 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int4 td = decode_tile(plan, t);
      const int n_tile = min(block_n, n_pad - td.w);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int r = q * 32 + lane;
      const bool valid = r < td.y;
      TOut* orow = out + static_cast<int64_t>(td.x + r) * c_out + td.w;
      const int ncols = min(n_tile, c_out - td.w);
      for (int c0 = 0; c0 < n_tile; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * block_n + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (!valid) continue;
        if constexpr (std::is_same<TOut, float>::value) {
          if (vec4 && c0 + 16 <= ncols) {
#pragma unroll
            for (int e = 0; e < 16; e += 4)
              *reinterpret_cast<float4*>(orow + c0 + e) =
                  make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]), __uint_as_float(v[e + 2]),
                              __uint_as_float(v[e + 3]));
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (c0 + e < ncols) orow[c0 + e] = __uint_as_float(v[e]);
          }
        } else {  // f16 partials: 2 x 16-byte stores per 16 columns
          if ((c_out & 7) == 0 && c0 + 16 <= ncols) {
            uint4 pk[2];
            __half2* h2 = reinterpret_cast<__half2*>(pk);
#pragma unroll
            for (int e = 0; e < 8; ++e) h2[e] = __floats2half2_rn(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1]));
            reinterpret_cast<uint4*>(orow + c0)[0] = pk[0];
            reinterpret_cast<uint4*>(orow + c0)[1] = pk[1];
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (c0 + e < ncols) orow[c0 + e] = __float2half_rn(__uint_as_float(v[e]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols) : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    SCONV_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) fail(SCONV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

CUtensorMap make_map_impl(const void* base, int dtype, uint64_t inner, uint64_t outer, uint64_t stride_bytes,
                          uint32_t box_inner, uint32_t box_outer, int kc) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {stride_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = kc == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                         : (kc == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  const CUresult r = get_encode()(
      &m, dtype == SCONV_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
      const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(SCONV_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

template <int KC, class TOut>
void launch_kc(Ctx& ctx, const GemmArgs& a) {
  const int block_n = a.block_n;
  const uint32_t a_bytes = 128u * KC * 2u, b_bytes = static_cast<uint32_t>(block_n) * KC * 2u;
  const uint32_t stage_bytes = (a_bytes + b_bytes + 1023u) & ~1023u;
  int stages = static_cast<int>((200u * 1024u) / stage_bytes);
  stages = std::max(2, std::min(stages, 8));
  const size_t smem = 1024 + static_cast<size_t>(stages) * stage_bytes + (2 * stages + 4) * 8 + 16;
  // TMEM: two accumulators of block_n fp32 columns, power of two >= 32.
  uint32_t cols = 32;
  while (cols < 2u * static_cast<uint32_t>(block_n)) cols <<= 1;
  auto kern = k_gemm_grouped<KC, TOut>;
  static thread_local std::map<size_t, int> occ_cache;  // per (instantiation, smem): host overhead
  int occ = 0;
  const size_t key = smem * 64 + static_cast<size_t>(ctx.device);  // attributes are per device
  const auto hit = occ_cache.find(key);
  if (hit != occ_cache.end()) {
    occ = hit->second;
  } else {
    SCONV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    SCONV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGemmThreads, smem));
    occ_cache[key] = occ;
  }
  occ = std::max(1, std::min<int>(occ, static_cast<int>(512u / cols)));  // never oversubscribe TMEM
  const int grid = std::max(1, std::min(a.num_tiles, ctx.num_sms * occ));
  const CUtensorMap tA = make_tensor_map_2d(a.a, a.dtype, a.k_pad, a.rows, KC, 128, KC);
  const CUtensorMap tB = make_tensor_map_2d(a.b, a.dtype, a.k_pad, static_cast<uint64_t>(a.num_offsets) * a.n_pad, KC,
                                  static_cast<uint32_t>(block_n), KC);
  const uint32_t fmt = a.dtype == SCONV_BF16 ? 1u : 0u;
  const uint32_t idesc_base = (1u << 4) | (fmt << 7) | (fmt << 10) | ((128u >> 4) << 24);
  ctx.launch("k_gemm_grouped", [&] {
    kern<<<grid, kGemmThreads, smem, ctx.stream>>>(tA, tB, *a.plan, a.num_tiles, a.num_kb, block_n, a.n_pad, a.c_out,
                                                   static_cast<TOut*>(a.out), stages, idesc_base, cols);
  });
}

}  // namespace

CUtensorMap make_tensor_map_2d(const void* base, int dtype, uint64_t inner, uint64_t outer, uint32_t box_inner,
                               uint32_t box_outer, int kc) {
  return make_map_impl(base, dtype, inner, outer, inner * 2, box_inner, box_outer, kc);
}

CUtensorMap make_tensor_map_2d_strided(const void* base, int dtype, uint64_t inner, uint64_t outer,
                                       uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int kc) {
  return make_map_impl(base, dtype, inner, outer, row_stride_bytes, box_inner, box_outer, kc);
}

int gemm_chunk(int k_pad) { return k_pad % 64 == 0 ? 64 : (k_pad % 32 == 0 ? 32 : 16); }

void launch_grouped_gemm(Ctx& ctx, const GemmArgs& a) {
  if (a.num_tiles == 0) return;
  const int kc = gemm_chunk(a.k_pad);
  if (a.out_f16) {
    if (kc == 64)
      launch_kc<64, __half>(ctx, a);
    else if (kc == 32)
      launch_kc<32, __half>(ctx, a);
    else
      launch_kc<16, __half>(ctx, a);
  } else {
    if (kc == 64)
      launch_kc<64, float>(ctx, a);
    else if (kc == 32)
      launch_kc<32, float>(ctx, a);
    else
      launch_kc<16, float>(ctx, a);
  }
}

}  // namespace sconvb

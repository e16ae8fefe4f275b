// Fused output-stationary SC layer: gather -> tcgen05 GEMM -> ascending-k
// reduction in TMEM -> epilogue, one kernel, no gather buffer and no per-offset partials.
#pragma once

#include "ctx.hpp"
#include "gmas.hpp"

namespace sconvb {

struct FusedArgs {
  const void* f_in = nullptr;  // 16-bit (the weight dtype) [n_in][ld_in]; columns [c_in, k_pad) zero
  int64_t ld_in = 0;
  int64_t n_in = 0;
  const int32_t* nbr = nullptr;  // [K3][n_out] in tile-row order: input row or -1 (nbr_in / nbr_perm)
  const int32_t* perm = nullptr;  // tile row -> output row (null: identity order)
  int64_t n_out = 0;
  const WeightData* w = nullptr;
  void* out = nullptr;  // [n_out][ld_out] of out_dtype
  int out_dtype = SCONV_F32;
  int64_t ld_out = 0;
  const void* res = nullptr;  // optional residual [n_out][ld_res] of out_dtype, added before ReLU
  int64_t ld_res = 0;
  int relu = 0;
  int block_n = 0;  // 0 = choose (fill the SMs)
  // work items (MapData::items; null with the 1x1 identity map: one single-offset item per tile)
  const unsigned long long* tile_mask = nullptr;
  const int4* items = nullptr;
  const int* item_ws = nullptr;
  const int* n_items = nullptr;
  int* item_counters = nullptr;
  int64_t max_items = 0, max_ws_slots = 0;
};

struct MapData;
// Lazily orders the map's output rows by neighbour bitmask for the fused kernel and builds its
// work items (once per map).
void prepare_fused_layout(Ctx& ctx, MapData& m);
// The work items alone (no-op once built; prepare_fused_layout builds them after the row order).
void build_fused_items(Ctx& ctx, MapData& m);

// true when the fused kernel supports this layer (K3 <= 64, 16-bit operands)
bool fused_supported(int K3, int c_in, int c_out);
int fused_items_mode();  // SCONV_FUSED_ITEMS (conv_fused.cu)
bool coalesced_epilogue_enabled();  // SCONV_FUSED_COAL (conv_fused.cu)
void launch_conv_fused(Ctx& ctx, const FusedArgs& a);

// f32/f16/bf16 [n][c] -> 16-bit [n][ld] (zero padded columns), dtype = operand type
void convert_rows(Ctx& ctx, const void* src, int src_dtype, int64_t n, int c, int64_t ld_src, void* dst, int dst_dtype,
                  int64_t ld_dst);

}  // namespace sconvb

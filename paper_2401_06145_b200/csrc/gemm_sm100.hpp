// Host interface of the tcgen05 grouped GEMM (gemm_sm100.cu).
#pragma once

#include "ctx.hpp"
#include "gmas.hpp"

namespace sconvb {

struct GemmArgs {
  const void* a = nullptr;   // gather buffer [rows x k_pad], f16/bf16
  const void* b = nullptr;   // weights [num_offsets * n_pad x k_pad], K-major
  const LayerPlan* plan = nullptr;  // tiles decoded from the member table (kernel parameter)
  int num_tiles = 0;
  int64_t rows = 0;
  int k_pad = 0, num_kb = 0;
  int n_pad = 0, block_n = 0, c_out = 0;
  int num_offsets = 0;
  int dtype = SCONV_F16;
  void* out = nullptr;  // [rows x c_out] per-offset partials: fp32, or f16 when out_f16
  bool out_f16 = false;
};

// K chunk (elements) per pipeline stage for a padded input width: 64/32/16 -> swizzle 128/64/32 B.
int gemm_chunk(int k_pad);
void launch_grouped_gemm(Ctx& ctx, const GemmArgs& args);

}  // namespace sconvb

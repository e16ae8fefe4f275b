// GMaS host interfaces (gmas.cu).
#pragma once

#include <memory>
#include <vector>

#include "ctx.hpp"

namespace sconvb {

constexpr int kMaxOffsets = 343;  // K <= 7 (the LayerPlan kernel parameter stays ~8 KB)

// Per-layer GMaS plan, passed BY VALUE as a kernel parameter (CUDA >= 12.1 allows 32 KB of
// parameters), so no host->device copy (and no pinned staging) is needed between layers.
struct LayerPlan {
  int nm;         // group members in buffer order
  int num_tiles;  // GEMM tiles = sum over members of ceil(height / 128) * n_blocks
  int n_blocks;   // output-channel blocks per row block
  int block_n;
  int4 members[kMaxOffsets];         // {offset k, first buffer row, n_k, padded height}
  int tile_start[kMaxOffsets + 1];   // tile prefix per member
  int delta[kMaxOffsets];            // scatter: buffer slot = canonical position + delta[k]
};

struct MapData;

// GemmGroupPlan: order = chosen offset order without empty offsets.
struct GroupPlan {
  struct Group {
    int begin, end;
    int64_t height;
  };
  std::vector<int> order;
  std::vector<Group> groups;
  std::vector<int64_t> buffer_offsets;  // per offset, -1 if n_k = 0
  int64_t buffer_length = 0;
  int64_t real_rows = 0;
};
GroupPlan group_gemms(const std::vector<int64_t>& sizes, int policy, double eps, int max_batch);

// WeightSet on device: [K3][n_pad][k_pad] (W_k transposed, K-major), f16/bf16.
struct WeightData {
  int K3 = 0, c_in = 0, c_out = 0, dtype = SCONV_F16;
  int k_pad = 0, n_pad = 0;
  DevBuf buf;
};
std::unique_ptr<WeightData> create_weights(Ctx& ctx, const float* w, int mem, int K3, int c_in, int c_out, int dtype);

std::vector<int> candidate_tiles(int channels);  // supported divisors, ascending
bool is_supported_tile(int t);
int default_tile(int channels, bool gather);
int padded_k(int c_in);

void layer_forward(Ctx& ctx, MapData& m, const WeightData& w, const void* f_in, int f_in_dtype, int f_in_mem,
                   const sconv_exec_cfg& cfg, void* f_out, int f_out_dtype, int f_out_mem, int relu = 0);

// Device-resident layer I/O (network driver): strided rows, optional residual + ReLU epilogue.
struct LayerIO {
  const void* f_in = nullptr;
  int in_dtype = SCONV_F32;
  int64_t ld_in = 0;           // row stride (elements)
  bool in_zero_padded = false;  // columns [c_in, ld_in) are zero (fused dataflow may read them)
  void* f_out = nullptr;
  int out_dtype = SCONV_F32;
  int64_t ld_out = 0;
  const void* res = nullptr;  // residual rows (out_dtype, Q order) added before the ReLU
  int64_t ld_res = 0;
  int relu = 0;
};
// dataflow: SCONV_DATAFLOW_GMAS or SCONV_DATAFLOW_FUSED (cfg.dataflow AUTO is resolved by callers)
void layer_forward_dev(Ctx& ctx, MapData& m, const WeightData& w, const sconv_exec_cfg& cfg, int dataflow,
                       const LayerIO& io);

}  // namespace sconvb

struct sconv_weights : sconvb::WeightData {};

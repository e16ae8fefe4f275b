// Network driver types (net.cu).
#pragma once

#include <array>
#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include "gmas.hpp"
#include "map.hpp"

namespace sconvb {

enum { kOpConv = 1, kOpAdd = 2, kOpConcat = 3 };
constexpr int kOpFields = 12;

// Op record (12 int32 fields on the ABI): kind, out, in, b (second operand) | target,
// K, offset_scale, out_stride, transposed, c_in, c_out, weight id, relu.
struct NetOp {
  int kind = 0, out = 0, in = 0, b = -1, target = -1;
  int K = 3, offset_scale = 1, out_stride = 1, transposed = 0, c_in = 0, c_out = 0, weight = -1, relu = 0;
};

struct NetTensor {
  int coordset = -1;
  int64_t n = 0;
  int channels = 0;
  int dtype = SCONV_F16;  // activations are stored in the compute dtype (f16 / bf16)
  int64_t ld = 0;         // row stride (elements); the network input is zero padded to 16
  bool fused_away = false;  // folded into a later op's epilogue (never materialised)
  DevBuf feats;  // [n][ld], rows in the coordinate set's order
};

// Per-op execution plan derived from the op list (residual folding, dataflow choice).
struct OpPlan {
  bool skip = false;  // ADD folded into a conv epilogue
  int out = -1;       // tensor written (the ADD's output when folded)
  int res = -1;       // residual tensor added in the epilogue (-1: none)
  int relu = 0;
  int dataflow = -1;  // resolved per conv (AUTO: timed on the first forward)
  int gather_tile = 0, scatter_tile = 0;  // autotune_network's pick for GMaS (0: context default)
};

// autotune_network (Alg. 2) state: per CONV op and candidate tile, the median
// gather / scatter latency summed over the sample clouds.
struct NetTune {
  int rounds = 5;
  std::map<int, std::map<int, double>> gather_ms, scatter_ms;
};

struct CoordSet {
  std::shared_ptr<DevBuf> keys;  // sorted packed keys (null: raw input not yet packed)
  int64_t n = 0;
  bool sorted = true;
  bool raw = false;
  int lattice = 1;  // every coordinate is a multiple of this (Eq. 1 outputs: their stride)
};

using MapKey = std::tuple<int, int, int, int, int, int>;
struct MapEntry {
  std::unique_ptr<MapData> map;
  int out_cs = -1;
};

struct NetData {
  std::vector<NetOp> ops;
  int num_tensors = 0, input_tensor = 0, output_tensor = 0;
  int block_B = 256, block_C = 512;
  sconv_exec_cfg cfg{};
  std::map<int, std::unique_ptr<WeightData>> weights;
  std::vector<NetTensor> tensors;
  std::vector<CoordSet> coordsets;
  std::map<MapKey, MapEntry> maps;
  MapSource raw_input;
  DevBuf input_xyz;  // device copy of host input coordinates
  int maps_built = 0;
  int64_t sorts = 0;  // coordinate sorts of the last forward (acceptance #7)
  std::vector<OpPlan> plan;
  bool planned = false;
  std::vector<std::array<double, 2>> auto_ms;  // per op: GMaS / fused ms of the tuning forward
  DevBuf readback;  // f32 staging for host reads
  // asynchronous host reads (sconv_net_read_async): two staging buffers alternate; the D2H copy
  // of slot s runs on copy_stream after rb_ready[s]; rb_done[s] guards the slot's next widening
  // (and any regrowth, whose free is ordered on the context stream)
  DevBuf rb_async[2];
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t rb_ready[2] = {nullptr, nullptr}, rb_done[2] = {nullptr, nullptr};
  bool rb_pending[2] = {false, false};
  int rb_slot = 0;
  // GPU span of the last completed forward on the context stream (timing events at its start /
  // end, read once complete): sizes the async readback's chunks (sconv_net_read_async)
  cudaEvent_t fwd_t0 = nullptr, fwd_t1 = nullptr;
  bool fwd_timed = false;
  float last_fwd_ms = -1.f;
  // host inputs (sconv_net_forward with host pointers) are copied on in_stream into one of two
  // staging slots, independent of the context stream: the next request's H2D and its map builds
  // (which wait for in_ready instead of everything on the context stream) overlap the previous
  // forward's convs. in_free[s] (end of the forward that read slot s) guards the slot's reuse.
  DevBuf in_xyz[2], in_feats[2];
  cudaStream_t in_stream = nullptr;
  cudaEvent_t in_ready[2] = {nullptr, nullptr}, in_free[2] = {nullptr, nullptr};
  cudaEvent_t ev_prev = nullptr;  // context stream at the start of a forward (the previous one's end)
  bool in_used[2] = {false, false};
  int in_slot = 0;
  int staged_slot = -1;  // slot of the inputs staged for the next forward (-1: none)
  // sconv_net_prefetch_inputs: host inputs copied ahead of their forward (one pending prefetch,
  // matched by pointers / sizes when sconv_net_forward is called with them)
  struct Prefetch {
    int slot = -1;
    const void *xyz = nullptr, *feats = nullptr;
    int64_t n = 0;
    int f_mem = 0, c_in = 0;
    const int32_t* xyz_dev = nullptr;
    const float* feats_dev = nullptr;
  } prefetch;
  // copies host coordinates (n x 3) and, for f_mem == host, features (n x c_in fp32) into the
  // next staging slot; returns their device pointers
  void stage_host_inputs(const int32_t* xyz, int64_t n, const float* feats, int f_mem, int c_in,
                         const int32_t** xyz_dev, const float** feats_dev);
  // per CONV op of the last forward: n_in, n_out, |M|, R_pad (0 when fused), c_in, c_out, k_pad, K3,
  // dataflow, residual folded (0/1)
  std::vector<std::array<int64_t, 10>> conv_stats;
  std::vector<MapData*> conv_maps;  // the map of each conv of the last forward (|M| on demand)
  std::vector<int> map_uses;  // per op: convs using the map first built at that op (plan_map_uses)
  void plan_map_uses(bool input_sorted);
  void resolve_stats(Ctx& ctx);
  // Kernel maps depend on coordinates only: they are built (and their fused row order
  // prepared) on a second, high-priority stream, so a map build and its host syncs overlap the
  // previous layers' convs; the context stream waits on an event before the first conv using
  // the map. SCONV_NET_MAP_STREAM=0 builds them on the context stream (A/B).
  cudaStream_t map_stream = nullptr;
  cudaStream_t layout_stream = nullptr;  // fused row order (mask sort): off the coordinate chain
  cudaEvent_t ev_order = nullptr;
  cudaEvent_t ev_flags = nullptr;  // deferred raw-input coordinate checks (copy done)
  // Coordinate look-ahead: when a coordinate set is created, the Eq. 1 output of the next
  // strided conv over it is queued at once on coord_stream (coords_only build); that conv's map
  // build later only reads |Q| (long done), instead of queueing the floor / sort / unique behind
  // the current level's searches and blocking the host on it. SCONV_NET_COORD_AHEAD=0: off.
  cudaStream_t coord_stream = nullptr;
  cudaEvent_t ev_coords = nullptr;
  std::map<std::pair<int, int>, std::unique_ptr<MapData>> pre_coords;  // (coordinate set, stride)

  NetData() = default;
  NetData(const NetData&) = delete;
  NetData& operator=(const NetData&) = delete;
  ~NetData();
  void check_ops() const;
  void make_plan();
  void forward(Ctx& ctx, const MapSource& input, const void* feats, int f_dtype, int f_mem, int c_in);
  // autotune_network: tuning forwards over the samples (profiling every candidate tile of every
  // conv on the GMaS dataflow), then the per-op argmin (smallest tile on ties) into the plan
  NetTune* tune = nullptr;
  NetTune last_tune;
  void tune_conv(Ctx& ctx, int op, MapData& m, const WeightData& w, const struct LayerIO& io);
  void finish_tune();
};

}  // namespace sconvb

struct sconv_net : sconvb::NetData {};

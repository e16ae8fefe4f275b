// Network driver (SPEC netdef, generalised to the U-Net / ResNet graphs of
// BASELINE configs 2-5): an op list over tensors, executed asynchronously on the context
// stream with a cross-layer kernel-map cache.
//
//   CONV    out = [relu](SC layer(in; K, offset_scale, out_stride, transposed/target) [+ res])
//   ADD     out = [relu](a + b)           (residual; same coordinates)
//   CONCAT  out = [a | b]                 (U-Net skip; same coordinates)
//
// Activations live on device in the compute dtype (f16 / bf16): the GEMM operands are
// 16-bit anyway, so storing fp32 between layers only doubled the traffic. Accumulation
// stays fp32 (TMEM / scatter registers); ADD sums in fp32 and rounds once.
//
// Plan (once per network): an ADD whose operand is produced by a CONV that nothing else
// reads is folded into that conv's epilogue (out = [relu](conv + other)); the conv's own
// output is never materialised. Per conv the dataflow is GMaS (Minuet gather/GEMM/scatter)
// or the fused output-stationary kernel; AUTO times both on the first forward and keeps
// the faster one (the Alg. 2 tuning idea applied to the dataflow).
//
// Coordinates live in "coordinate sets" (sorted packed keys on device). A map is keyed by
// (input coordinate set, K, offset scale, out stride, transposed, target set) and built
// once per forward; the output coordinate set of a stride-1 map on a sorted set aliases it
// (SPEC.md:528 sort reuse), so only the raw input and strided layers ever sort. Map builds
// sync once each (sizes + error flags); GMaS launches never sync.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "conv_fused.hpp"
#include "gmas.hpp"
#include "map.hpp"
#include "net.hpp"

namespace sconvb {
namespace {

template <class T>
struct H16;
template <>
struct H16<__half> {
  static __device__ __forceinline__ float2 to2(__half2 v) { return __half22float2(v); }
  static __device__ __forceinline__ __half2 from2(float a, float b) { return __floats2half2_rn(a, b); }
  using T2 = __half2;
};
template <>
struct H16<__nv_bfloat16> {
  static __device__ __forceinline__ float2 to2(__nv_bfloat162 v) { return __bfloat1622float2(v); }
  static __device__ __forceinline__ __nv_bfloat162 from2(float a, float b) { return __floats2bfloat162_rn(a, b); }
  using T2 = __nv_bfloat162;
};

// out = [relu](a + b), 16-bit operands, fp32 sum, 8 elements per thread (16-byte vectors)
template <class T>
__global__ void k_add(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out, int64_t n8, int relu) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n8) return;
  const uint4 x = reinterpret_cast<const uint4*>(a)[i], y = reinterpret_cast<const uint4*>(b)[i];
  uint4 r;
  const auto* xa = reinterpret_cast<const typename H16<T>::T2*>(&x);
  const auto* ya = reinterpret_cast<const typename H16<T>::T2*>(&y);
  auto* ra = reinterpret_cast<typename H16<T>::T2*>(&r);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 p = H16<T>::to2(xa[e]), q = H16<T>::to2(ya[e]);
    float s0 = p.x + q.x, s1 = p.y + q.y;
    if (relu) {
      s0 = fmaxf(s0, 0.f);
      s1 = fmaxf(s1, 0.f);
    }
    ra[e] = H16<T>::from2(s0, s1);
  }
  reinterpret_cast<uint4*>(out)[i] = r;
}

template <class T>
__global__ void k_add_scalar(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out, int64_t n,
                             int relu) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n) return;
  const float r = static_cast<float>(a[i]) + static_cast<float>(b[i]);
  out[i] = static_cast<T>(relu ? fmaxf(r, 0.f) : r);
}

// [a | b] along channels; 16-bit elements moved as raw 2-byte words (exact)
__global__ void k_concat(const uint16_t* __restrict__ a, int64_t lda, int ca, const uint16_t* __restrict__ b,
                         int64_t ldb, int cb, uint16_t* __restrict__ out, int64_t n) {
  const int c = ca + cb;
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n * c) return;
  const int64_t r = i / c;
  const int ch = static_cast<int>(i - r * c);
  out[i] = ch < ca ? a[r * lda + ch] : b[r * ldb + ch - ca];
}

// vectorised: 8 channels (16 bytes) per thread when every row segment is 16-byte aligned
__global__ void k_concat8(const uint4* __restrict__ a, int64_t lda8, int ca8, const uint4* __restrict__ b,
                          int64_t ldb8, int cb8, uint4* __restrict__ out, int64_t n) {
  const int c8 = ca8 + cb8;
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n * c8) return;
  const int64_t r = i / c8;
  const int ch = static_cast<int>(i - r * c8);
  out[i] = ch < ca8 ? a[r * lda8 + ch] : b[r * ldb8 + ch - ca8];
}

// SCONV_DEBUG_SYNC=1: synchronise and log after every conv (locates a faulting launch)
bool debug_sync() {
  static const bool on = [] {
    const char* e = std::getenv("SCONV_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  return on;
}

inline unsigned blocks(int64_t n) { return static_cast<unsigned>(std::max<int64_t>(1, (n + 255) / 256)); }

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

}  // namespace

void NetData::check_ops() const {
  for (const NetOp& o : ops) {
    auto chk = [&](int t) {
      if (t < 0 || t >= num_tensors) fail(SCONV_ERR_ARG, "tensor id out of range");
    };
    chk(o.out);
    chk(o.in);
    if (o.out == o.in || (o.kind != kOpConv && o.out == o.b)) fail(SCONV_ERR_ARG, "ops must not write their input");
    if (o.kind == kOpConv) {
      if (o.transposed) chk(o.target);
      if (o.c_in < 1 || o.c_out < 1) fail(SCONV_ERR_ARG, "channel counts must be positive");
    } else if (o.kind == kOpAdd || o.kind == kOpConcat) {
      chk(o.b);
    } else {
      fail(SCONV_ERR_ARG, "unknown op kind");
    }
  }
}

void NetData::make_plan() {
  const int n_ops = static_cast<int>(ops.size());
  plan.assign(n_ops, OpPlan{});
  auto_ms.assign(n_ops, {-1.0, -1.0});
  std::vector<int> producer(num_tensors, -1), readers(num_tensors, 0);
  for (int i = 0; i < n_ops; ++i) {
    const NetOp& o = ops[i];
    producer[o.out] = i;
    ++readers[o.in];
    if (o.kind != kOpConv) ++readers[o.b];
    if (o.kind == kOpConv && o.transposed) ++readers[o.target];  // coordinates only, but keep it materialised
    plan[i].out = o.out;
    plan[i].relu = o.relu;
    if (o.kind == kOpConv) plan[i].dataflow = cfg.dataflow;
  }
  if (!cfg.fuse_residual) return;
  for (int a = 0; a < n_ops; ++a) {
    const NetOp& add = ops[a];
    if (add.kind != kOpAdd) continue;
    int best = -1, other = -1;
    for (int side = 0; side < 2; ++side) {
      const int t = side == 0 ? add.in : add.b, u = side == 0 ? add.b : add.in;
      const int p = producer[t];
      if (p < 0 || p > a || ops[p].kind != kOpConv || plan[p].skip || plan[p].res >= 0) continue;
      if (ops[p].relu || readers[t] != 1 || t == output_tensor) continue;
      const int pu = u == input_tensor ? -1 : producer[u];
      if (pu >= p) continue;  // the other operand must exist when the conv runs
      if (p > best) {
        best = p;
        other = u;
      }
    }
    if (best < 0) continue;
    plan[best].out = add.out;
    plan[best].res = other;
    plan[best].relu = add.relu;
    plan[a].skip = true;
  }
}

NetData::~NetData() {
  maps.clear();  // frees enqueued on the streams the buffers were allocated on
  coordsets.clear();
  tensors.clear();
  pre_coords.clear();
  // input staging lives on in_stream: released (stream-ordered) before that stream is destroyed;
  // in-flight async reads still copy out of rb_async (context stream, freed after this body)
  for (int s = 0; s < 2; ++s) {
    in_xyz[s].release();
    in_feats[s].release();
  }
  for (cudaStream_t* sp : {&map_stream, &layout_stream, &coord_stream, &copy_stream, &in_stream})
    if (*sp) {
      cudaStreamSynchronize(*sp);
      cudaStreamDestroy(*sp);
    }
  if (ev_order) cudaEventDestroy(ev_order);
  if (ev_flags) cudaEventDestroy(ev_flags);
  if (ev_coords) cudaEventDestroy(ev_coords);
  for (int s = 0; s < 2; ++s) {
    if (rb_ready[s]) cudaEventDestroy(rb_ready[s]);
    if (rb_done[s]) cudaEventDestroy(rb_done[s]);
    if (in_ready[s]) cudaEventDestroy(in_ready[s]);
    if (in_free[s]) cudaEventDestroy(in_free[s]);
  }
  if (ev_prev) cudaEventDestroy(ev_prev);
  if (fwd_t0) cudaEventDestroy(fwd_t0);
  if (fwd_t1) cudaEventDestroy(fwd_t1);
}

void NetData::stage_host_inputs(const int32_t* xyz, int64_t n, const float* feats, int f_mem, int c_in,
                                const int32_t** xyz_dev, const float** feats_dev) {
  if (!in_stream) {
    SCONV_CUDA(cudaStreamCreateWithFlags(&in_stream, cudaStreamNonBlocking));
    for (int s = 0; s < 2; ++s) {
      SCONV_CUDA(cudaEventCreateWithFlags(&in_ready[s], cudaEventDisableTiming));
      SCONV_CUDA(cudaEventCreateWithFlags(&in_free[s], cudaEventDisableTiming));
    }
  }
  const int s = in_slot;
  in_slot ^= 1;
  if (prefetch.slot == s) prefetch.slot = -1;  // a pending prefetch in this slot is overwritten
  // the forward that read this slot last must be done with it (its end on the context stream)
  if (in_used[s]) SCONV_CUDA(cudaStreamWaitEvent(in_stream, in_free[s], 0));
  in_xyz[s].reserve(std::max<size_t>(sizeof(int32_t) * 3 * n, 16), in_stream);
  SCONV_CUDA(cudaMemcpyAsync(in_xyz[s].get(), xyz, sizeof(int32_t) * 3 * n, cudaMemcpyHostToDevice, in_stream));
  *xyz_dev = in_xyz[s].get<int32_t>();
  if (f_mem == SCONV_MEM_HOST) {
    in_feats[s].reserve(std::max<size_t>(sizeof(float) * n * c_in, 16), in_stream);
    SCONV_CUDA(cudaMemcpyAsync(in_feats[s].get(), feats, sizeof(float) * n * c_in, cudaMemcpyHostToDevice, in_stream));
    *feats_dev = in_feats[s].get<float>();
  } else {
    *feats_dev = feats;
  }
  SCONV_CUDA(cudaEventRecord(in_ready[s], in_stream));
  in_used[s] = true;
  staged_slot = s;
}

void NetData::forward(Ctx& ctx, const MapSource& input, const void* feats, int f_dtype, int f_mem, int c_in) {
  if (f_dtype != SCONV_F32) fail(SCONV_ERR_ARG, "network input features must be fp32");
  const cudaStream_t st = ctx.stream;
  static const bool use_map_stream = [] {
    const char* e = std::getenv("SCONV_NET_MAP_STREAM");
    return !(e && e[0] == '0');
  }();
  if (!ev_order) SCONV_CUDA(cudaEventCreateWithFlags(&ev_order, cudaEventDisableTiming));
  if (!ev_flags) SCONV_CUDA(cudaEventCreateWithFlags(&ev_flags, cudaEventDisableTiming));
  if (use_map_stream && !map_stream) {
    int lo = 0, hi = 0;
    SCONV_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SCONV_CUDA(cudaStreamCreateWithPriority(&map_stream, cudaStreamNonBlocking, hi));
    SCONV_CUDA(cudaStreamCreateWithPriority(&layout_stream, cudaStreamNonBlocking, hi));
    const char* cp = std::getenv("SCONV_COORD_PRIO");  // A/B: "lo" | "hi" (default; r02bp same box: C2 2.168 -> 2.150 ms)
    SCONV_CUDA(cudaStreamCreateWithPriority(&coord_stream, cudaStreamNonBlocking, cp && cp[0] == 'l' ? lo : hi));
  }
  if (!ev_coords) SCONV_CUDA(cudaEventCreateWithFlags(&ev_coords, cudaEventDisableTiming));
  static const bool derive_maps = [] {  // SCONV_NET_DERIVE=0: search every map (A/B)
    const char* e = std::getenv("SCONV_NET_DERIVE");
    return !(e && e[0] == '0');
  }();
  // the first look-ahead Eq. 1 starts right after the raw input's key packing, beside the level-0
  // search (same box r02ao: C2 2.207 -> 2.167 ms, C3 1.299 -> 1.268); SCONV_COORD_AFTER=map|layout
  // waits for the level-0 search / row order instead
  static const bool coord_after_pack = [] {
    const char* e = std::getenv("SCONV_COORD_AFTER");
    return !(e && (e[0] == 'm' || e[0] == 'l'));
  }();
  static const bool coord_ahead = [] {
    const char* e = std::getenv("SCONV_NET_COORD_AHEAD");
    return !(e && e[0] == '0');
  }();
  const cudaStream_t cst = use_map_stream && coord_ahead ? coord_stream : nullptr;
  const cudaStream_t ms = use_map_stream ? map_stream : st;
  const cudaStream_t ls = use_map_stream ? layout_stream : st;
  // SCONV_NET_WAIT_PROFILE=1: time how long the context stream waits for each map and row
  // order (events around the wait; printed at the end of the forward). Measured r01q: ~205 us
  // per MinkUNet42 forward, mostly the level 0-2 row orders; running the first conv of each
  // level in output order instead removes the waits but not the time (that conv is ~2x slower)
  static const bool wait_profile = [] {
    const char* e = std::getenv("SCONV_NET_WAIT_PROFILE");
    return e && e[0] == '1';
  }();
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> waits;
  // SCONV_NET_HOST_PROFILE=1: host timestamps (us since the forward started) of each op's map
  // build / row order / launch, printed at the end (compare with a kernel timeline)
  const bool host_profile = Ctx::htrace_on();  // SCONV_HOST_TRACE=1
  std::vector<std::tuple<int, size_t>> hops;  // (op, first trace entry of the op)
  if (host_profile) {
    ctx.htrace.clear();
    ctx.htrace_t0 = std::chrono::steady_clock::now();
  }
  auto hmark = [&](int op, const char* what) {
    if (!host_profile) return;
    hops.emplace_back(op, ctx.htrace.size());
    ctx.hmark(what);
  };
  auto wait_for = [&](cudaStream_t from, int op) {
    SCONV_CUDA(cudaEventRecord(ev_order, from));
    if (!wait_profile) {
      SCONV_CUDA(cudaStreamWaitEvent(st, ev_order));
      return;
    }
    cudaEvent_t a, b;
    SCONV_CUDA(cudaEventCreate(&a));
    SCONV_CUDA(cudaEventCreate(&b));
    SCONV_CUDA(cudaEventRecord(a, st));
    SCONV_CUDA(cudaStreamWaitEvent(st, ev_order));
    SCONV_CUDA(cudaEventRecord(b, st));
    waits.emplace_back(op, a, b);
  };
  // the map stream starts after everything already on the context stream: the input
  // coordinates may be produced there, and the previous forward's maps (freed below, on the
  // map stream) may still be in use by its convs
  // Host inputs staged on in_stream (sconv_net_forward): nothing on the context stream produces
  // them, so the map streams wait only for their copy and start beside the previous forward's
  // convs; the previous forward's maps are then released only after ev_prev (below).
  const int in_s = staged_slot;
  staged_slot = -1;
  if (!ev_prev) SCONV_CUDA(cudaEventCreateWithFlags(&ev_prev, cudaEventDisableTiming));
  SCONV_CUDA(cudaEventRecord(ev_prev, st));
  if (!fwd_t0) {
    SCONV_CUDA(cudaEventCreate(&fwd_t0));
    SCONV_CUDA(cudaEventCreate(&fwd_t1));
  }
  if (fwd_timed && cudaEventQuery(fwd_t1) == cudaSuccess) {  // the previous forward's span, if done
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, fwd_t0, fwd_t1) == cudaSuccess) last_fwd_ms = ms;
  }
  (void)cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error here
  fwd_timed = false;
  if (in_s >= 0) SCONV_CUDA(cudaStreamWaitEvent(st, in_ready[in_s], 0));
  SCONV_CUDA(cudaEventRecord(fwd_t0, st));
  if (ms != st) {
    cudaEvent_t start = in_s >= 0 ? in_ready[in_s] : ev_prev;
    SCONV_CUDA(cudaStreamWaitEvent(ms, start));
    SCONV_CUDA(cudaStreamWaitEvent(ls, start));
    if (cst) SCONV_CUDA(cudaStreamWaitEvent(cst, start));
  }
  hmark(-1, "forward: streams joined");
  if (!planned) {
    make_plan();
    planned = true;
  }
  const int act = cfg.compute_dtype;
  tensors.resize(num_tensors);
  for (auto& t : tensors) {
    t.coordset = -1;
    t.fused_away = false;
  }
  // (released with the previous forward's maps at the end: its convs may still run)
  std::vector<CoordSet> old_coordsets;
  old_coordsets.swap(coordsets);
  // the previous forward's maps are freed at the END of this forward: ~180 stream-ordered
  // frees here would delay the first launches by ~80 us of host time (the GPU idles then)
  std::map<MapKey, MapEntry> old_maps;
  old_maps.swap(maps);
  pre_coords.clear();  // (unused look-ahead coordinates of the previous forward)
  plan_map_uses(input.sorted);
  // queue the Eq. 1 output of the next strided conv over coordinate set cs_new (see net.hpp)
  // (op `from` writes a tensor on cs_new; its output is not assigned yet when this runs)
  auto prelaunch = [&](int cs_new, int from, bool wait_map_stream) {
    if (!cst || !coordsets[cs_new].keys) return;
    std::vector<int> tcs(num_tensors);
    for (int t = 0; t < num_tensors; ++t) tcs[t] = tensors[t].coordset;
    tcs[plan[from].out] = cs_new;
    for (int j = from + 1; j < static_cast<int>(ops.size()); ++j) {
      if (plan[j].skip) continue;
      const NetOp& q = ops[j];
      const int in = tcs[q.in];
      int outc = in;
      if (q.kind == kOpConv) {
        if (q.transposed) {
          outc = tcs[q.target];
        } else if (q.out_stride != 1) {
          if (in != cs_new) {
            outc = -2;  // a coordinate set not created yet
          } else {
            const auto pk = std::make_pair(cs_new, q.out_stride);
            if (!pre_coords.count(pk) && !maps.count(MapKey{cs_new, q.K, q.offset_scale, q.out_stride, 0, -1})) {
              sconv_map_cfg c{q.K, q.offset_scale, q.out_stride, 0, block_B, block_C, SCONV_MAP_SORTED};
              MapSource P;
              P.keys = coordsets[cs_new].keys;
              P.n = coordsets[cs_new].n;
              P.sorted = true;
              if (wait_map_stream) {  // the keys are still being produced on the map stream
                // (measured r02ag, same box: waiting for the map stream 2.20 ms, for the layout
                // stream 2.28 ms, look-ahead off 2.22 ms; A/B: SCONV_COORD_AFTER=layout)
                static const bool after_map = [] {
                  const char* e = std::getenv("SCONV_COORD_AFTER");
                  return !(e && e[0] == 'l');
                }();
                if (!coord_after_pack) SCONV_CUDA(cudaEventRecord(ev_coords, after_map ? ms : ls));
                SCONV_CUDA(cudaStreamWaitEvent(cst, ev_coords));
              }
              ctx.stream = cst;
              try {
                pre_coords[pk] = build_map(ctx, P, c, nullptr, false, true, nullptr, nullptr, /*coords_only=*/true);
              } catch (...) {
                ctx.stream = st;
                throw;
              }
              ctx.stream = st;
            }
            return;
          }
        }
      }
      tcs[plan[j].out] = outc;
    }
  };
  const void* deferred_flags = nullptr;  // raw sorted input: coordinate checks after the launches
  // pending look-ahead Eq. 1 (see the map-build path): coordinate set, creating op, whether it
  // waits for the map stream, and whether it fires after the current op's conv
  int pre_cs = -1, pre_from = -1;
  bool pre_wait = false, pre_armed = false;
  bool raw_pre_done = false;  // the raw input's look-ahead Eq. 1 was queued inside its map build
  int convs_issued = 0;
  maps_built = 0;
  sorts = 0;
  conv_stats.clear();
  conv_maps.clear();
  // coordinate set 0 = the raw input (may be unsorted)
  coordsets.push_back({input.keys, input.n, input.sorted, true});
  raw_input = input;
  NetTensor& tin = tensors[input_tensor];
  tin.coordset = 0;
  tin.n = input.n;
  tin.channels = c_in;
  tin.dtype = act;
  tin.ld = round_up(c_in, 16);  // zero padded: the fused gather reads whole 16-channel chunks
  hmark(-1, "forward: tensors reset");
  tin.feats.reserve(std::max<size_t>(2 * input.n * tin.ld, 16), st);
  if (input.n > 0) {
    const float* src = static_cast<const float*>(feats);
    DevBuf staged;
    if (f_mem == SCONV_MEM_HOST) {
      staged.alloc(sizeof(float) * input.n * c_in, st);
      SCONV_CUDA(cudaMemcpyAsync(staged.get(), feats, sizeof(float) * input.n * c_in, cudaMemcpyHostToDevice, st));
      src = staged.get<float>();
    }
    convert_rows(ctx, src, SCONV_F32, input.n, c_in, c_in, tin.feats.get(), act, tin.ld);
  }
  hmark(-1, "forward: input converted");
  for (int oi = 0; oi < static_cast<int>(ops.size()); ++oi) {
    const NetOp& o = ops[oi];
    OpPlan& pl = plan[oi];
    if (pl.skip) continue;
    NetTensor& a = tensors.at(o.in);
    if (a.coordset < 0) fail(SCONV_ERR_STATE, "op reads a tensor that was not produced yet");
    NetTensor& out = tensors.at(pl.out);
    if (o.kind == kOpConv) {
      if (a.channels != o.c_in) fail(SCONV_ERR_ARG, "conv input channels mismatch");
      int tgt = -1;
      if (o.transposed) {
        tgt = tensors.at(o.target).coordset;
        if (tgt < 0) fail(SCONV_ERR_STATE, "transposed conv target not produced yet");
      }
      const MapKey key{a.coordset, o.K, o.offset_scale, o.transposed ? 1 : o.out_stride, o.transposed, tgt};
      auto it = maps.find(key);
      if (it == maps.end()) {
        sconv_map_cfg mcfg{o.K, o.offset_scale, o.out_stride, o.transposed, block_B, block_C, SCONV_MAP_SORTED};
        const CoordSet& cs = coordsets[a.coordset];
        MapSource P;
        if (cs.raw && !cs.keys) {
          P = raw_input;
        } else {
          P.keys = cs.keys;
          P.n = cs.n;
          P.sorted = true;
        }
        MapSource T;
        if (o.transposed) {
          const CoordSet& ct = coordsets[tgt];
          if (!ct.keys) fail(SCONV_ERR_ARG, "transposed target must be a sorted coordinate set");
          T.keys = ct.keys;
          T.n = ct.n;
          T.sorted = true;
        }
        // maps over the network's own (already validated) coordinate sets skip the canonical
        // lists and the end-of-build sync unless a GMaS conv asks for them; built on the map
        // stream (with the fused row order when a fused conv may use them)
        std::unique_ptr<MapData> m;
        ctx.stream = ms;
        hmark(oi, "map build");
        try {
          void* dflags = cs.raw && !cs.keys ? static_cast<char*>(ctx.pin_flags()) + Ctx::kPinFlagsBytes / 2 : nullptr;
          std::unique_ptr<MapData> pre;  // this strided map's coordinates, queued ahead
          if (!o.transposed && o.out_stride != 1 && P.keys) {
            auto f = pre_coords.find({a.coordset, o.out_stride});
            if (f != pre_coords.end()) {
              pre = std::move(f->second);
              pre_coords.erase(f);
              ctx.stream = cst;
              const bool ok = finish_coords(ctx, *pre);  // |Q| (the floor ran long ago)
              ctx.stream = ms;
              if (!ok) pre.reset();  // compact keys overflowed: the normal build's exact path
            }
          }
          // K = 2, stride 2s down-sampling of a set on the s-lattice: the map is derived from the
          // Eq. 1 output (a scatter, no search); its transposed up-sampling map from it in turn
          const bool down_derivable = derive_maps && !o.transposed && o.K == 2 && o.out_stride == 2 * o.offset_scale &&
                                      P.keys && coordsets[a.coordset].lattice % o.offset_scale == 0;
          if (down_derivable && !pre) {  // no look-ahead coordinates: Eq. 1 now (one sync, as before)
            pre = build_map(ctx, P, mcfg, nullptr, false, true, nullptr, nullptr, /*coords_only=*/true);
            if (!finish_coords(ctx, *pre)) pre.reset();
          }
          const MapData* fwd = nullptr;
          if (derive_maps && o.transposed && o.K == 2) {
            auto f = maps.find(MapKey{tgt, o.K, o.offset_scale, 2 * o.offset_scale, 0, -1});
            if (f != maps.end() && f->second.out_cs == a.coordset) fwd = f->second.map.get();
          }
          if (pre) {
            MapSource Q;
            Q.keys = pre->q_keys;
            Q.n = pre->n_out;
            Q.sorted = true;
            if (down_derivable)
              m = derive_down_map(ctx, P, Q, mcfg);
            else
              m = build_map(ctx, P, mcfg, nullptr, false, /*lazy=*/true, nullptr, nullptr, false, &Q);
            m->sorts += pre->sorts;
          } else if (fwd) {
            m = derive_transposed_map(ctx, *fwd, P, T, mcfg);
          } else {
            // the raw input's packed keys feed the look-ahead Eq. 1: event before this map's search,
            // and (sorted raw input) the Eq. 1 is queued right there, AHEAD of the level-0 search:
            // its |Q| then reaches the host before the first down conv needs it (r02bs timeline: queued
            // after the search it ran beside the level-0 row order, slowing both, and the host
            // waited ~110 us for it at the first down conv)
            static const bool raw_first_on = [] {  // A/B: SCONV_RAW_EQ1_FIRST=0 queues it after the search
              const char* e = std::getenv("SCONV_RAW_EQ1_FIRST");
              return !(e && e[0] == '0');
            }();
            const bool raw_first =
                raw_first_on && cs.raw && cs.sorted && coord_after_pack && cst && a.coordset == 0 && !o.transposed;
            const int csi = a.coordset;
            auto on_keys = [&, csi, oi](const std::shared_ptr<DevBuf>& keys) {
              if (!raw_first || raw_pre_done) return;
              coordsets[csi].keys = keys;
              const cudaStream_t saved = ctx.stream;
              prelaunch(csi, oi, true);
              ctx.stream = saved;
              raw_pre_done = true;
            };
            m = build_map(ctx, P, mcfg, o.transposed ? &T : nullptr, false, /*lazy=*/true, nullptr, dflags, false,
                          nullptr, cs.raw && coord_after_pack ? ev_coords : nullptr, on_keys);
          }
          if (m->flags_deferred) {
            deferred_flags = dflags;
            SCONV_CUDA(cudaEventRecord(ev_flags, ms));
          }
          hmark(oi, "map built");
          if (ms != st) {  // the row order runs beside the coordinate chain (next level's map);
            // the context stream waits on the layout stream below, which implies this map
            SCONV_CUDA(cudaEventRecord(ev_order, ms));
            SCONV_CUDA(cudaStreamWaitEvent(ls, ev_order));
          }
          ctx.stream = ls;
          // off the critical path only when convs are already queued ahead of this map's first use
          m->layout_off_path = ls != st && convs_issued > 0;
          // row-order key width from the number of convs that will use this map (plan_map_uses:
          // the op graph alone, so every forward orders the rows alike): 3 sort passes pay off only
          // when enough convs share the map (r02ai: C2 maps serve 6-8 convs, 24 bits best; C3's
          // serve 4-5, 16 bits best)
          if (oi < static_cast<int>(map_uses.size()) && map_uses[oi] > 0) m->mask_bits_hint = map_uses[oi] >= 6 ? 24 : 16;
          if (pl.dataflow != SCONV_DATAFLOW_GMAS) prepare_fused_layout(ctx, *m);
          hmark(oi, "layout queued");
        } catch (...) {
          ctx.stream = st;
          throw;
        }
        ctx.stream = st;
        if (ls != st) wait_for(ls, 1000 + oi);
        ++maps_built;
        sorts += m->sorts;
        if (!coordsets[a.coordset].keys && coordsets[a.coordset].sorted)
          coordsets[a.coordset].keys = m->src_keys;  // sorted raw input: its packed keys, same row order
        int out_cs;
        if (o.transposed) {
          out_cs = tgt;
        } else if (o.out_stride == 1 && coordsets[a.coordset].keys) {
          out_cs = a.coordset;  // stride-1 alias
        } else {
          coordsets.push_back({m->q_keys, m->n_out, true, false, o.out_stride});
          out_cs = static_cast<int>(coordsets.size()) - 1;
        }
        // the raw input's keys were just packed (cs may dangle after the push_back above)
        const bool raw_keyed = a.coordset == 0 && maps_built == 1 && coordsets[0].keys;
        it = maps.emplace(key, MapEntry{std::move(m), out_cs}).first;
        // coordinate look-ahead: the Eq. 1 output of the next strided conv over a coordinate set
        // created now (keys complete: this build synchronised on |Q|), or over the raw input once
        // its keys are packed. It is needed only when the host reaches that conv, several convs
        // later, so it is queued after the conv of the NEXT map-building op (for the raw input:
        // after this op's conv): queued at once, the one-launch Eq. 1 ran ahead of the next level's
        // search and row order (the critical path: the conv stream idled ~150 us per level,
        // r02bq/r02br timelines). SCONV_PRE_AFTER_CONV=0: at once (A/B).
        static const bool pre_after = [] {
          const char* e = std::getenv("SCONV_PRE_AFTER_CONV");
          return !(e && e[0] == '0');
        }();
        if (pre_after && pre_cs >= 0) pre_armed = true;  // a map was built since: fire after this conv
        if (out_cs != a.coordset && !o.transposed) {
          if (pre_after && pre_cs < 0) {
            pre_cs = out_cs;
            pre_from = oi;
            pre_wait = false;
            pre_armed = false;
          } else {
            prelaunch(out_cs, oi, false);
          }
        } else if (raw_keyed && !raw_pre_done) {
          if (pre_after && pre_cs < 0) {
            pre_cs = a.coordset;
            pre_from = oi;
            pre_wait = true;
            pre_armed = true;
          } else {
            prelaunch(a.coordset, oi, true);
          }
        }
      }
      MapData& m = *it->second.map;
      auto wt = weights.find(o.weight);
      if (wt == weights.end()) fail(SCONV_ERR_STATE, "conv weights not set");
      const WeightData& w = *wt->second;
      if (w.c_in != o.c_in || w.c_out != o.c_out || w.K3 != m.K3) fail(SCONV_ERR_ARG, "weight shape mismatch");
      if (w.dtype != act) fail(SCONV_ERR_ARG, "weight dtype must match the network compute dtype");
      const NetTensor* res = nullptr;
      if (pl.res >= 0) {
        res = &tensors.at(pl.res);
        if (res->coordset < 0) fail(SCONV_ERR_STATE, "residual operand not produced yet");
        if (res->channels != o.c_out || res->n != m.n_out) fail(SCONV_ERR_ARG, "add operands need the same shape");
        // as the unfused ADD below: both operands on one coordinate set (equal row counts alone
        // could add misaligned rows)
        if (res->coordset != it->second.out_cs) fail(SCONV_ERR_ARG, "add/concat operands need the same coordinates");
      }
      // the output buffer may be read below (residual or input of a re-used tensor id): fresh allocation
      DevBuf nb;
      nb.alloc(std::max<size_t>(2 * static_cast<size_t>(m.n_out) * o.c_out, 16), st);
      LayerIO io;
      io.f_in = a.feats.get();
      io.in_dtype = a.dtype;
      io.ld_in = a.ld;
      io.in_zero_padded = true;  // every tensor's padding columns are written as zeros
      io.f_out = nb.get();
      io.out_dtype = act;
      io.ld_out = o.c_out;
      io.res = res ? res->feats.get() : nullptr;
      io.ld_res = res ? res->ld : 0;
      io.relu = pl.relu;
      if (tune) tune_conv(ctx, oi, m, w, io);
      int df = pl.dataflow;
      if (df == SCONV_DATAFLOW_AUTO) {
        // time both dataflows once on this input (1 warm-up + 2 timed runs each, min)
        cudaEvent_t e0, e1;
        SCONV_CUDA(cudaEventCreate(&e0));
        SCONV_CUDA(cudaEventCreate(&e1));
        double best[2] = {1e30, 1e30};
        for (int rep = 0; rep < 3; ++rep)
          for (int d = 0; d < 2; ++d) {
            SCONV_CUDA(cudaEventRecord(e0, st));
            sconv_exec_cfg tcfg = cfg;
            if (pl.gather_tile > 0) tcfg.gather_tile = pl.gather_tile;
            if (pl.scatter_tile > 0) tcfg.scatter_tile = pl.scatter_tile;
            layer_forward_dev(ctx, m, w, tcfg, d == 0 ? SCONV_DATAFLOW_GMAS : SCONV_DATAFLOW_FUSED, io);
            SCONV_CUDA(cudaEventRecord(e1, st));
            SCONV_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            SCONV_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (rep > 0) best[d] = std::min(best[d], static_cast<double>(ms));
          }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        auto_ms[oi] = {best[0], best[1]};
        pl.dataflow = best[1] <= best[0] ? SCONV_DATAFLOW_FUSED : SCONV_DATAFLOW_GMAS;
        df = pl.dataflow;
      }
      sconv_exec_cfg ccfg = cfg;  // autotuned GMaS tiles of this op (Alg. 2)
      if (pl.gather_tile > 0) ccfg.gather_tile = pl.gather_tile;
      if (pl.scatter_tile > 0) ccfg.scatter_tile = pl.scatter_tile;
      layer_forward_dev(ctx, m, w, ccfg, df, io);
      hmark(oi, "conv queued");
      if (pre_cs >= 0 && pre_armed) {
        prelaunch(pre_cs, pre_from, pre_wait);
        pre_cs = -1;
      }
      if (debug_sync()) {
        std::fprintf(stderr, "[sconv] op %d conv K3=%d n_in=%lld n_out=%lld c_in=%d c_out=%d dataflow=%d ...", oi, m.K3,
                     static_cast<long long>(m.n_in), static_cast<long long>(m.n_out), w.c_in, w.c_out, df);
        ctx.sync();
        std::fprintf(stderr, " ok\n");
      }
      out.coordset = it->second.out_cs;
      out.n = m.n_out;
      out.channels = o.c_out;
      out.dtype = act;
      out.ld = o.c_out;
      out.feats = std::move(nb);
      if (pl.out != o.out) tensors.at(o.out).fused_away = true;
      ++convs_issued;
      conv_stats.push_back({m.n_in, m.n_out, m.total, df == SCONV_DATAFLOW_FUSED ? 0 : m.buffer_length, w.c_in, w.c_out,
                            w.k_pad, m.K3, df, pl.res >= 0 ? 1 : 0});
      conv_maps.push_back(&m);
    } else {
      NetTensor& b = tensors.at(o.b);
      if (b.coordset < 0) fail(SCONV_ERR_STATE, "op reads a tensor that was not produced yet");
      if (a.coordset != b.coordset || a.n != b.n) fail(SCONV_ERR_ARG, "add/concat operands need the same coordinates");
      const int64_t n = a.n;
      DevBuf nb;
      if (o.kind == kOpAdd) {
        if (a.channels != b.channels) fail(SCONV_ERR_ARG, "add operands need the same channels");
        if (a.ld != a.channels || b.ld != b.channels) fail(SCONV_ERR_ARG, "add operands must be dense rows");
        // operands may alias the output tensor id (in-place residual): separate allocation
        nb.alloc(std::max<size_t>(2 * static_cast<size_t>(n) * a.channels, 16), st);
        const int64_t total = n * a.channels;
        if (total % 8 == 0) {
          if (act == SCONV_F16)
            ctx.launch("k_add", [&] {
              k_add<__half><<<blocks(total / 8), 256, 0, st>>>(a.feats.get<__half>(), b.feats.get<__half>(),
                                                               nb.get<__half>(), total / 8, o.relu);
            });
          else
            ctx.launch("k_add", [&] {
              k_add<__nv_bfloat16><<<blocks(total / 8), 256, 0, st>>>(
                  a.feats.get<__nv_bfloat16>(), b.feats.get<__nv_bfloat16>(), nb.get<__nv_bfloat16>(), total / 8, o.relu);
            });
        } else if (act == SCONV_F16) {
          ctx.launch("k_add", [&] {
            k_add_scalar<__half><<<blocks(total), 256, 0, st>>>(a.feats.get<__half>(), b.feats.get<__half>(),
                                                                nb.get<__half>(), total, o.relu);
          });
        } else {
          ctx.launch("k_add", [&] {
            k_add_scalar<__nv_bfloat16><<<blocks(total), 256, 0, st>>>(
                a.feats.get<__nv_bfloat16>(), b.feats.get<__nv_bfloat16>(), nb.get<__nv_bfloat16>(), total, o.relu);
          });
        }
        out.channels = a.channels;
      } else {
        const int c = a.channels + b.channels;
        nb.alloc(std::max<size_t>(2 * static_cast<size_t>(n) * c, 16), st);
        if (a.channels % 8 == 0 && b.channels % 8 == 0 && a.ld % 8 == 0 && b.ld % 8 == 0)
          ctx.launch("k_concat", [&] {
            k_concat8<<<blocks(n * c / 8), 256, 0, st>>>(a.feats.get<uint4>(), a.ld / 8, a.channels / 8,
                                                         b.feats.get<uint4>(), b.ld / 8, b.channels / 8, nb.get<uint4>(),
                                                         n);
          });
        else
          ctx.launch("k_concat", [&] {
            k_concat<<<blocks(n * c), 256, 0, st>>>(a.feats.get<uint16_t>(), a.ld, a.channels, b.feats.get<uint16_t>(),
                                                    b.ld, b.channels, nb.get<uint16_t>(), n);
          });
        out.channels = c;
      }
      out.coordset = a.coordset;
      out.n = n;
      out.dtype = act;
      out.ld = out.channels;
      out.feats = std::move(nb);
    }
  }
  if (ms != st) {  // readers of the forward's coordinates (map-stream buffers) use the context stream
    if (cst) {
      SCONV_CUDA(cudaEventRecord(ev_order, cst));
      SCONV_CUDA(cudaStreamWaitEvent(st, ev_order));
    }
    SCONV_CUDA(cudaEventRecord(ev_order, ms));
    SCONV_CUDA(cudaStreamWaitEvent(st, ev_order));
    SCONV_CUDA(cudaEventRecord(ev_order, ls));
    SCONV_CUDA(cudaStreamWaitEvent(st, ev_order));
  }
  // frees enqueued behind this forward's work on the map / layout / coordinate streams, and
  // behind the previous forward's convs (ev_prev: those streams may have started before them)
  if (ms != st)
    for (cudaStream_t s : {ms, ls, cst})
      if (s) SCONV_CUDA(cudaStreamWaitEvent(s, ev_prev));
  old_maps.clear();
  old_coordsets.clear();
  if (in_s >= 0) SCONV_CUDA(cudaEventRecord(in_free[in_s], st));
  SCONV_CUDA(cudaEventRecord(fwd_t1, st));
  fwd_timed = true;
  if (deferred_flags) {  // the copy was queued right after the input's key packing: long done
    SCONV_CUDA(cudaEventSynchronize(ev_flags));
    check_deferred_map_flags(deferred_flags, raw_input);
  }
  if (host_profile) {
    hmark(-1, "forward returns");
    size_t h = 0;
    int op = -1;
    for (size_t i = 0; i < ctx.htrace.size(); ++i) {
      while (h < hops.size() && std::get<1>(hops[h]) <= i) op = std::get<0>(hops[h++]);
      std::fprintf(stderr, "[sconv host] %8.1f us op %d %s\n", ctx.htrace[i].second, op, ctx.htrace[i].first);
    }
  }
  if (!waits.empty()) {  // SCONV_NET_WAIT_PROFILE
    SCONV_CUDA(cudaStreamSynchronize(st));
    double total = 0;
    for (auto& [op, a, b] : waits) {
      float ms_ = 0;
      cudaEventElapsedTime(&ms_, a, b);
      total += ms_;
      if (ms_ > 0.001f)
        std::fprintf(stderr, "[sconv wait] op %d %s %.1f us\n", op % 1000, op >= 1000 ? "layout" : "map", 1e3 * ms_);
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
    std::fprintf(stderr, "[sconv wait] total %.1f us over %zu waits\n", 1e3 * total, waits.size());
  }
}

// Alg. 2 on one conv of a tuning forward: every candidate tile (divisors of C_in for gather,
// C_out for scatter) runs the GMaS dataflow 1 + rounds times on this conv's
// actual map and input; the median of the kernel's CUDA-event times is added
// to the op's per-tile sum over the samples. The other kernel keeps the default tile.
void NetData::tune_conv(Ctx& ctx, int op, MapData& m, const WeightData& w, const LayerIO& io) {
  if (m.n_out == 0) return;
  const bool was = ctx.profiling;
  ctx.resolve_profile();
  ctx.profiling = true;
  DevBuf out;
  out.alloc(static_cast<size_t>(m.n_out) * w.c_out * 2, ctx.stream);
  LayerIO tio = io;
  tio.f_out = out.get();
  tio.res = nullptr;  // the epilogue does not depend on the tile
  auto time_kernel = [&](const char* name, int tg, int ts) {
    sconv_exec_cfg c = cfg;
    c.gather_tile = tg;
    c.scatter_tile = ts;
    std::vector<double> samples;
    for (int r = 0; r <= tune->rounds; ++r) {  // 1 warm-up + R measured
      ctx.last_records.clear();
      layer_forward_dev(ctx, m, w, c, SCONV_DATAFLOW_GMAS, tio);
      ctx.resolve_profile();
      double ms = 0;
      for (auto& rec : ctx.last_records)
        if (rec.first == name) ms += rec.second;
      if (r > 0) samples.push_back(ms);
    }
    std::sort(samples.begin(), samples.end());
    const size_t n = samples.size();
    return n % 2 ? samples[n / 2] : 0.5 * (samples[n / 2 - 1] + samples[n / 2]);
  };
  for (int t : candidate_tiles(w.c_in)) tune->gather_ms[op][t] += time_kernel("k_gather", t, default_tile(w.c_out, false));
  for (int t : candidate_tiles(w.c_out)) tune->scatter_ms[op][t] += time_kernel("k_scatter", default_tile(w.c_in, true), t);
  ctx.last_records.clear();
  ctx.profiling = was;
}

// |M| of lazily built maps (the fused dataflow never needs it): canonical lists on demand, after
// the forward (one sync per unresolved map; statistics / roofline only, never in a timed loop)
void NetData::resolve_stats(Ctx& ctx) {
  for (size_t c = 0; c < conv_stats.size() && c < conv_maps.size(); ++c) {
    if (conv_stats[c][2] >= 0 || !conv_maps[c]) continue;
    ensure_canonical(ctx, *conv_maps[c]);
    conv_stats[c][2] = conv_maps[c]->total;
  }
}

// Per op: how many convs of a forward use the map first built at that op, from the op graph alone
// (the runtime's coordinate-set and map-cache rules replayed symbolically; input sortedness
// decides whether the raw set aliases). Deterministic, so the row-order hint it feeds is the
// same in every forward.
void NetData::plan_map_uses(bool input_sorted) {
  map_uses.assign(ops.size(), 0);
  struct Sym {
    bool keyed, sorted;
  };
  std::vector<Sym> cs{{false, input_sorted}};
  std::vector<int> tcs(num_tensors, -1);
  tcs[input_tensor] = 0;
  std::map<MapKey, std::pair<int, int>> seen;  // key -> (first op, output set)
  std::map<MapKey, int> uses;
  for (int oi = 0; oi < static_cast<int>(ops.size()); ++oi) {
    if (plan[oi].skip) continue;
    const NetOp& o = ops[oi];
    const int a = tcs[o.in];
    if (a < 0) continue;
    if (o.kind != kOpConv) {
      tcs[plan[oi].out] = a;
      continue;
    }
    const int tgt = o.transposed ? tcs[o.target] : -1;
    const MapKey key{a, o.K, o.offset_scale, o.transposed ? 1 : o.out_stride, o.transposed, tgt};
    auto it = seen.find(key);
    if (it == seen.end()) {
      if (!cs[a].keyed && cs[a].sorted) cs[a].keyed = true;
      int out;
      if (o.transposed) {
        out = tgt;
      } else if (o.out_stride == 1 && cs[a].keyed) {
        out = a;
      } else {
        cs.push_back({true, true});
        out = static_cast<int>(cs.size()) - 1;
      }
      it = seen.emplace(key, std::make_pair(oi, out)).first;
    }
    ++uses[key];
    tcs[plan[oi].out] = it->second.second;
  }
  for (const auto& [k, v] : seen) map_uses[v.first] = uses[k];
}

void NetData::finish_tune() {
  auto pick = [](const std::map<int, double>& c) {
    int best = 0;
    double best_ms = 0;
    for (const auto& [t, ms] : c)  // ascending tiles, strict '<': the smallest tile wins ties
      if (best == 0 || ms < best_ms) {
        best = t;
        best_ms = ms;
      }
    return best;
  };
  for (auto& [op, c] : tune->gather_ms) plan.at(op).gather_tile = pick(c);
  for (auto& [op, c] : tune->scatter_ms) plan.at(op).scatter_tile = pick(c);
}

}  // namespace sconvb

// Network driver (SPEC netdef, generalised to the U-Net / ResNet graphs of
// BASELINE configs 2-5): an op list over tensors, executed asynchronously on the context
// stream with a cross-layer kernel-map cache.
//
//   CONV    out = [relu](SC layer(in; K, offset_scale, out_stride, transposed/target))
//   ADD     out = [relu](a + b)           (residual; same coordinates)
//   CONCAT  out = [a | b]                 (U-Net skip; same coordinates)
//
// Coordinates live in "coordinate sets" (sorted packed keys on device). A map is keyed by
// (input coordinate set, K, offset scale, out stride, transposed, target set) and built
// once per forward; the output coordinate set of a stride-1 map on a sorted set aliases it
// (SPEC.md:528 sort reuse), so only the raw input and strided layers ever sort. Map builds
// sync once each (sizes + error flags); GMaS launches never sync.
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "gmas.hpp"
#include "map.hpp"
#include "net.hpp"

namespace sconvb {
namespace {

__global__ void k_add(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out, int64_t n4,
                      int relu) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n4) return;
  const float4 x = reinterpret_cast<const float4*>(a)[i], y = reinterpret_cast<const float4*>(b)[i];
  float4 r = make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
  if (relu) r = make_float4(fmaxf(r.x, 0.f), fmaxf(r.y, 0.f), fmaxf(r.z, 0.f), fmaxf(r.w, 0.f));
  reinterpret_cast<float4*>(out)[i] = r;
}

__global__ void k_add_scalar(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out,
                             int64_t n, int relu) {
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n) return;
  const float r = a[i] + b[i];
  out[i] = relu ? fmaxf(r, 0.f) : r;
}

__global__ void k_concat(const float* __restrict__ a, int ca, const float* __restrict__ b, int cb,
                         float* __restrict__ out, int64_t n) {
  const int c = ca + cb;
  const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
  if (i >= n * c) return;
  const int64_t r = i / c;
  const int ch = static_cast<int>(i - r * c);
  out[i] = ch < ca ? a[r * ca + ch] : b[r * cb + ch - ca];
}

inline unsigned blocks(int64_t n) { return static_cast<unsigned>(std::max<int64_t>(1, (n + 255) / 256)); }

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

void NetData::forward(Ctx& ctx, const MapSource& input, const void* feats, int f_dtype, int f_mem, int c_in) {
  if (f_dtype != SCONV_F32) fail(SCONV_ERR_ARG, "network input features must be fp32");
  const cudaStream_t st = ctx.stream;
  tensors.resize(num_tensors);
  for (auto& t : tensors) t.coordset = -1;
  coordsets.clear();
  maps.clear();
  maps_built = 0;
  conv_stats.clear();
  // coordinate set 0 = the raw input (may be unsorted)
  coordsets.push_back({input.keys, input.n, input.sorted, true});
  raw_input = input;
  NetTensor& tin = tensors[input_tensor];
  tin.coordset = 0;
  tin.n = input.n;
  tin.channels = c_in;
  const size_t in_bytes = sizeof(float) * input.n * c_in;
  tin.feats.reserve(std::max<size_t>(in_bytes, 16), st);
  if (input.n > 0)
    SCONV_CUDA(cudaMemcpyAsync(tin.feats.get(), feats, in_bytes,
                               f_mem == SCONV_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
  for (const NetOp& o : ops) {
    NetTensor& a = tensors.at(o.in);
    if (a.coordset < 0) fail(SCONV_ERR_STATE, "op reads a tensor that was not produced yet");
    NetTensor& out = tensors.at(o.out);
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
        sconv_map_cfg cfg{o.K, o.offset_scale, o.out_stride, o.transposed, block_B, block_C};
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
        auto m = build_map(ctx, P, cfg, o.transposed ? &T : nullptr);
        ++maps_built;
        if (!coordsets[a.coordset].keys && coordsets[a.coordset].sorted)
          coordsets[a.coordset].keys = m->src_keys;  // sorted raw input: its packed keys, same row order
        int out_cs;
        if (o.transposed) {
          out_cs = tgt;
        } else if (o.out_stride == 1 && coordsets[a.coordset].keys) {
          out_cs = a.coordset;  // stride-1 alias
        } else {
          coordsets.push_back({m->q_keys, m->n_out, true, false});
          out_cs = static_cast<int>(coordsets.size()) - 1;
        }
        it = maps.emplace(key, MapEntry{std::move(m), out_cs}).first;
      }
      MapData& m = *it->second.map;
      auto wt = weights.find(o.weight);
      if (wt == weights.end()) fail(SCONV_ERR_STATE, "conv weights not set");
      const WeightData& w = *wt->second;
      if (w.c_in != o.c_in || w.c_out != o.c_out || w.K3 != m.K3) fail(SCONV_ERR_ARG, "weight shape mismatch");
      out.coordset = it->second.out_cs;
      out.n = m.n_out;
      out.channels = o.c_out;
      out.feats.reserve(std::max<size_t>(sizeof(float) * out.n * out.channels, 16), st);
      sconv_exec_cfg c = cfg;
      c.compute_dtype = w.dtype;
      layer_forward(ctx, m, w, a.feats.get(), SCONV_F32, SCONV_MEM_DEVICE, c, out.feats.get(), SCONV_F32,
                    SCONV_MEM_DEVICE, o.relu);
      conv_stats.push_back({m.n_in, m.n_out, m.total, m.buffer_length, w.c_in, w.c_out, w.k_pad, m.K3});
    } else {
      NetTensor& b = tensors.at(o.b);
      if (b.coordset < 0) fail(SCONV_ERR_STATE, "op reads a tensor that was not produced yet");
      if (a.coordset != b.coordset || a.n != b.n) fail(SCONV_ERR_ARG, "add/concat operands need the same coordinates");
      const int64_t n = a.n;
      if (o.kind == kOpAdd) {
        if (a.channels != b.channels) fail(SCONV_ERR_ARG, "add operands need the same channels");
        // operands may alias the output (in-place residual): allocate the output separately
        DevBuf nb;
        nb.alloc(std::max<size_t>(sizeof(float) * n * a.channels, 16), st);
        const int64_t total = n * a.channels;
        if (total % 4 == 0)
          ctx.launch("k_add", [&] {
            k_add<<<blocks(total / 4), 256, 0, st>>>(a.feats.get<float>(), b.feats.get<float>(), nb.get<float>(),
                                                     total / 4, o.relu);
          });
        else
          ctx.launch("k_add", [&] {
            k_add_scalar<<<blocks(total), 256, 0, st>>>(a.feats.get<float>(), b.feats.get<float>(), nb.get<float>(),
                                                        total, o.relu);
          });
        out.channels = a.channels;
        out.coordset = a.coordset;
        out.n = n;
        out.feats = std::move(nb);
      } else {
        DevBuf nb;
        nb.alloc(std::max<size_t>(sizeof(float) * n * (a.channels + b.channels), 16), st);
        ctx.launch("k_concat", [&] {
          k_concat<<<blocks(n * (a.channels + b.channels)), 256, 0, st>>>(
              a.feats.get<float>(), a.channels, b.feats.get<float>(), b.channels, nb.get<float>(), n);
        });
        out.channels = a.channels + b.channels;
        out.coordset = a.coordset;
        out.n = n;
        out.feats = std::move(nb);
      }
    }
  }
}

}  // namespace sconvb

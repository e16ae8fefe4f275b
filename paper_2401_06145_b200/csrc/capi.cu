// C ABI of libsconv_b200 (include/sconv_b200.h): exception-free boundary, context runtime,
// tile autotuner (Alg. 2), synthetic-input generator (SPEC cli gen).
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_set>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"
#include "conv_fused.hpp"
#include "gmas.hpp"
#include "voxelize.hpp"
#include "map.hpp"
#include "net.hpp"

namespace sconvb {

cudaEvent_t Ctx::take_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  SCONV_CUDA(cudaEventCreate(&e));
  return e;
}

void Ctx::resolve_profile() {
  if (pending.empty()) return;
  SCONV_CUDA(cudaEventSynchronize(pending.back().b));
  for (auto& p : pending) {
    float ms = 0.f;
    SCONV_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    auto it = profile.find(p.name);
    if (it == profile.end()) {
      profile_names.push_back(p.name);
      it = profile.emplace(p.name, ProfileEntry{}).first;
    }
    it->second.launches += 1;
    it->second.total_ms += ms;
    last_records.emplace_back(p.name, ms);
    event_pool.push_back(p.a);
    event_pool.push_back(p.b);
  }
  pending.clear();
}

namespace {

std::mutex g_err_mu;
std::string g_err;

template <class Fn>
sconv_status guarded(sconv_ctx* ctx, Fn&& fn) {
  try {
    fn();
    return SCONV_OK;
  } catch (const Error& e) {
    if (ctx) ctx->err = e.what();
    std::lock_guard<std::mutex> l(g_err_mu);
    g_err = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->err = "host allocation failed";
    return SCONV_ERR_OOM;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    std::lock_guard<std::mutex> l(g_err_mu);
    g_err = e.what();
    return SCONV_ERR_STATE;
  }
}

sconv_map_cfg default_map_cfg(int K, int s) {
  sconv_map_cfg c;
  c.kernel_size = K;
  c.offset_scale = s;
  c.out_stride = s;
  c.transposed = 0;
  c.block_B = 256;
  c.block_C = 512;
  c.backend = SCONV_MAP_SORTED;
  return c;
}

sconv_exec_cfg normalize(const sconv_exec_cfg* cfg, int default_dataflow = SCONV_DATAFLOW_GMAS) {
  sconv_exec_cfg c;
  c.policy = SCONV_GROUP_SORTED;
  c.epsilon = 0.25;
  c.max_batch = 16;
  c.gather_tile = 0;
  c.scatter_tile = 0;
  c.compute_dtype = SCONV_F16;
  c.partial_f16 = 0;
  c.dataflow = default_dataflow;
  c.fuse_residual = 1;
  if (cfg) c = *cfg;
  if (c.dataflow < 0) c.dataflow = default_dataflow;
  if (c.dataflow < SCONV_DATAFLOW_GMAS || c.dataflow > SCONV_DATAFLOW_AUTO) fail(SCONV_ERR_ARG, "unknown dataflow");
  if (c.compute_dtype != SCONV_F16 && c.compute_dtype != SCONV_BF16) fail(SCONV_ERR_ARG, "compute dtype must be f16 or bf16");
  return c;
}

sconv_map* wrap(std::unique_ptr<MapData> m) {
  auto* out = new sconv_map;
  static_cast<MapData&>(*out) = std::move(*m);
  return out;
}

// SplitMix64 (reference prng.hpp:19-54), restated for the product's synthetic generator.
struct SplitMix {
  uint64_t s;
  uint64_t next() {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }
  uint64_t below(uint64_t bound) {
    const uint64_t limit = uint64_t{0} - ((uint64_t{0} - bound) % bound);
    for (;;) {
      const uint64_t r = next();
      if (limit == 0 || r < limit) return r % bound;
    }
  }
};
uint64_t stream_seed(uint64_t seed, uint64_t idx) { return seed ^ ((idx + 1) * 0x9E3779B97F4A7C15ull); }

// ---- point-cloud files (".xyz" text, ".mpc" binary) ----
struct File {
  FILE* f = nullptr;
  File(const char* path, const char* mode) : f(path ? std::fopen(path, mode) : nullptr) {
    if (!f) fail(SCONV_ERR_ARG, std::string("cannot open file ") + (path ? path : "(null)"));
  }
  ~File() {
    if (f) std::fclose(f);
  }
};
constexpr int64_t kMpcHeader = 12;  // "MPC1", u32 N, u32 C

uint32_t le_u32(const unsigned char* b) {
  return uint32_t{b[0]} | (uint32_t{b[1]} << 8) | (uint32_t{b[2]} << 16) | (uint32_t{b[3]} << 24);
}

// header of an .mpc file + size check: N, C and the exact file length
void mpc_header(FILE* f, int64_t& n, int64_t& c) {
  unsigned char h[kMpcHeader];
  const size_t got = std::fread(h, 1, kMpcHeader, f);
  if (got < 4 || std::memcmp(h, "MPC1", 4) != 0) fail(SCONV_ERR_ARG, "mpc parse error at offset 0: bad magic");
  if (got < static_cast<size_t>(kMpcHeader))
    fail(SCONV_ERR_ARG, "mpc parse error at offset " + std::to_string(got) + ": truncated header");
  n = le_u32(h + 4);
  c = le_u32(h + 8);
  std::fseek(f, 0, SEEK_END);
  const int64_t size = std::ftell(f);
  const int64_t want = kMpcHeader + 12 * n + 4 * n * c;
  if (size != want)
    fail(SCONV_ERR_ARG, "mpc parse error at offset " + std::to_string(std::min(size, want)) + ": expected " +
                            std::to_string(want) + " bytes, file has " + std::to_string(size));
  std::fseek(f, kMpcHeader, SEEK_SET);
}

// .xyz: one point per line "x y z f1 ... fC"; blank lines and '#' comments skipped. Every
// line must carry the same number of columns (>= 3). Calls row(values) per point.
template <class Row>
void xyz_parse(FILE* f, int64_t& n, int64_t& c, Row&& row) {
  n = 0;
  c = -1;
  std::vector<double> vals;
  std::string line;
  int64_t lineno = 0;
  char buf[4096];
  while (true) {
    line.clear();
    bool got = false;
    while (std::fgets(buf, sizeof(buf), f)) {  // one whole line, however long
      got = true;
      line += buf;
      if (line.back() == '\n') break;
    }
    if (!got) break;
    ++lineno;
    vals.clear();
    const char* p = line.c_str();
    while (true) {
      while (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n') ++p;
      if (!*p || *p == '#') break;
      char* end = nullptr;
      const double v = std::strtod(p, &end);
      if (end == p || (*end && *end != ' ' && *end != '\t' && *end != '\r' && *end != '\n')) {
        const char* e = p;
        while (*e && *e != ' ' && *e != '\t' && *e != '\r' && *e != '\n') ++e;
        fail(SCONV_ERR_ARG, "xyz parse error at line " + std::to_string(lineno) + ": invalid number '" +
                                std::string(p, e) + "'");
      }
      vals.push_back(v);
      p = end;
    }
    if (vals.empty()) continue;
    const int64_t cols = static_cast<int64_t>(vals.size());
    if (cols < 3)
      fail(SCONV_ERR_ARG, "xyz parse error at line " + std::to_string(lineno) + ": expected at least 3 columns, got " +
                              std::to_string(cols));
    if (c < 0) c = cols - 3;
    if (cols != c + 3)
      fail(SCONV_ERR_ARG, "xyz parse error at line " + std::to_string(lineno) + ": expected " + std::to_string(c + 3) +
                              " columns, got " + std::to_string(cols));
    row(n, vals);
    ++n;
  }
  if (c < 0) c = 0;
}

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

}  // namespace
}  // namespace sconvb

using namespace sconvb;

extern "C" {

sconv_status sconv_cloud_file_info(const char* path, int* format, int64_t* n, int64_t* channels) {
  return guarded(nullptr, [&] {
    File fh(path, "rb");
    char magic[4] = {0, 0, 0, 0};
    const size_t got = std::fread(magic, 1, 4, fh.f);
    std::rewind(fh.f);
    int64_t nn = 0, cc = 0;
    const size_t len = std::strlen(path);
    const bool mpc_ext = len >= 4 && std::strcmp(path + len - 4, ".mpc") == 0;
    if (mpc_ext || (got == 4 && std::memcmp(magic, "MPC1", 4) == 0)) {
      mpc_header(fh.f, nn, cc);
      if (format) *format = SCONV_FILE_MPC;
    } else {
      xyz_parse(fh.f, nn, cc, [](int64_t, const std::vector<double>&) {});
      if (format) *format = SCONV_FILE_XYZ;
    }
    if (n) *n = nn;
    if (channels) *channels = cc;
  });
}

sconv_status sconv_mpc_read(const char* path, int32_t* xyz, float* feats, int64_t n, int64_t channels) {
  return guarded(nullptr, [&] {
    File fh(path, "rb");
    int64_t nn = 0, cc = 0;
    mpc_header(fh.f, nn, cc);
    if (nn != n || cc != channels) fail(SCONV_ERR_ARG, "buffer shape does not match the file");
    if (n > 0 && (!xyz || (channels > 0 && !feats))) fail(SCONV_ERR_ARG, "null output buffer");
    if (n > 0 && std::fread(xyz, 12, static_cast<size_t>(n), fh.f) != static_cast<size_t>(n))
      fail(SCONV_ERR_ARG, "mpc parse error at offset 12: short read");
    if (n * channels > 0 &&
        std::fread(feats, 4, static_cast<size_t>(n * channels), fh.f) != static_cast<size_t>(n * channels))
      fail(SCONV_ERR_ARG, "mpc parse error at offset " + std::to_string(kMpcHeader + 12 * n) + ": short read");
  });
}

sconv_status sconv_mpc_write(const char* path, const int32_t* xyz, const float* feats, int64_t n, int64_t channels) {
  return guarded(nullptr, [&] {
    if (n < 0 || channels < 0 || n > UINT32_MAX || channels > UINT32_MAX) fail(SCONV_ERR_ARG, "invalid cloud shape");
    if (n > 0 && (!xyz || (channels > 0 && !feats))) fail(SCONV_ERR_ARG, "null input buffer");
    File fh(path, "wb");
    unsigned char h[kMpcHeader] = {'M', 'P', 'C', '1'};
    for (int b = 0; b < 4; ++b) {
      h[4 + b] = static_cast<unsigned char>((static_cast<uint32_t>(n) >> (8 * b)) & 0xFF);
      h[8 + b] = static_cast<unsigned char>((static_cast<uint32_t>(channels) >> (8 * b)) & 0xFF);
    }
    bool ok = std::fwrite(h, 1, kMpcHeader, fh.f) == static_cast<size_t>(kMpcHeader);
    if (n > 0) ok = ok && std::fwrite(xyz, 12, static_cast<size_t>(n), fh.f) == static_cast<size_t>(n);
    if (n * channels > 0)
      ok = ok && std::fwrite(feats, 4, static_cast<size_t>(n * channels), fh.f) == static_cast<size_t>(n * channels);
    if (!ok) fail(SCONV_ERR_ARG, std::string("write failed: ") + path);
  });
}

sconv_status sconv_xyz_read(const char* path, double* points, float* feats, int64_t n, int64_t channels) {
  return guarded(nullptr, [&] {
    File fh(path, "rb");
    int64_t nn = 0, cc = 0;
    xyz_parse(fh.f, nn, cc, [&](int64_t i, const std::vector<double>& v) {
      if (i >= n || static_cast<int64_t>(v.size()) != channels + 3)
        fail(SCONV_ERR_ARG, "buffer shape does not match the file");
      for (int a = 0; a < 3; ++a) points[3 * i + a] = v[a];
      for (int64_t c = 0; c < channels; ++c) feats[i * channels + c] = static_cast<float>(v[3 + c]);
    });
    if (nn != n) fail(SCONV_ERR_ARG, "buffer shape does not match the file");
  });
}

sconv_status sconv_xyz_write(const char* path, const double* points, const float* feats, int64_t n, int64_t channels) {
  return guarded(nullptr, [&] {
    if (n < 0 || channels < 0) fail(SCONV_ERR_ARG, "invalid cloud shape");
    if (n > 0 && (!points || (channels > 0 && !feats))) fail(SCONV_ERR_ARG, "null input buffer");
    File fh(path, "w");
    bool ok = true;
    for (int64_t i = 0; i < n && ok; ++i) {  // %.17g / %.9g: exact round trips of double / float
      ok = std::fprintf(fh.f, "%.17g %.17g %.17g", points[3 * i], points[3 * i + 1], points[3 * i + 2]) > 0;
      for (int64_t c = 0; c < channels && ok; ++c) ok = std::fprintf(fh.f, " %.9g", double{feats[i * channels + c]}) > 0;
      ok = ok && std::fputc('\n', fh.f) != EOF;
    }
    if (!ok) fail(SCONV_ERR_ARG, std::string("write failed: ") + path);
  });
}

const char* sconv_version(void) { return "sconv_b200 0.1 (sm_100a)"; }

const char* sconv_global_last_error(void) {
  std::lock_guard<std::mutex> l(g_err_mu);
  static thread_local std::string copy;
  copy = g_err;
  return copy.c_str();
}

sconv_status sconv_ctx_create(int device, sconv_ctx** out) {
  if (!out) return SCONV_ERR_ARG;
  *out = nullptr;
  auto* ctx = new sconv_ctx;
  const sconv_status st = guarded(nullptr, [&] {
    ctx->device = device;
    SCONV_CUDA(cudaSetDevice(device));
    SCONV_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
    SCONV_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    cudaMemPool_t pool;
    SCONV_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    SCONV_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    {  // pre-grow the pool: later stream-ordered allocations (three streams in a network
       // forward) are carved from retained memory instead of mapping new physical pages
       // mid-forward (a sporadic multi-ms stall)
      void* warm = nullptr;
      if (cudaMallocAsync(&warm, size_t{4} << 30, ctx->own_stream) == cudaSuccess) {
        cudaFreeAsync(warm, ctx->own_stream);
        cudaStreamSynchronize(ctx->own_stream);
      }
      cudaGetLastError();
    }
    SCONV_CUDA(cudaMalloc(reinterpret_cast<void**>(&ctx->done), 64));
    SCONV_CUDA(cudaMemset(ctx->done, 0, 64));
    SCONV_CUDA(cudaMalloc(reinterpret_cast<void**>(&ctx->lookup_counter), 8));
    SCONV_CUDA(cudaMemset(ctx->lookup_counter, 0, 8));
    const size_t sort_bytes = sizeof(int) * (3 * 65536 + 8);
    SCONV_CUDA(cudaMalloc(reinterpret_cast<void**>(&ctx->sort_state), sort_bytes));
    SCONV_CUDA(cudaMemset(ctx->sort_state, 0, sort_bytes));
    SCONV_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->pinned),
                              Ctx::kPinFlagsBytes + Ctx::kPinReadbackBytes + Ctx::kPinPlanBytes));
  });
  if (st != SCONV_OK) {
    delete ctx;
    return st;
  }
  *out = ctx;
  return SCONV_OK;
}

void sconv_ctx_destroy(sconv_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  {
    // release buffers on the stream before it is destroyed
    ctx->scratch_sort.release();
    ctx->scratch_misc.release();
    ctx->flush_buf.release();
    ctx->gather_buf.release();
    ctx->gemm_out.release();
    ctx->plan_dev.release();
    ctx->fused_counter.release();  // every Ctx-owned DevBuf: freed on the stream before it dies
    ctx->fused_ws.release();
  }
  cudaStreamSynchronize(ctx->stream);
  for (auto& p : ctx->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->done) cudaFree(ctx->done);
  if (ctx->lookup_counter) cudaFree(ctx->lookup_counter);
  if (ctx->sort_state) cudaFree(ctx->sort_state);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

const char* sconv_last_error(const sconv_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

sconv_status sconv_ctx_set_stream(sconv_ctx* ctx, void* s) {
  return guarded(ctx, [&] {
    SCONV_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
  });
}
void* sconv_ctx_stream(const sconv_ctx* ctx) { return ctx->stream; }
sconv_status sconv_ctx_synchronize(sconv_ctx* ctx) {
  return guarded(ctx, [&] {
    ctx->sync();
    ctx->resolve_profile();
  });
}
int64_t sconv_ctx_launch_count(const sconv_ctx* ctx) { return ctx->launches; }
sconv_status sconv_ctx_set_lookup_counting(sconv_ctx* ctx, int enabled) {
  return guarded(ctx, [&] { ctx->count_lookups = enabled != 0; });
}

sconv_status sconv_ctx_lookup_count(sconv_ctx* ctx, unsigned long long* count) {
  return guarded(ctx, [&] {
    if (!count) fail(SCONV_ERR_ARG, "null argument");
    SCONV_CUDA(cudaMemcpyAsync(count, ctx->lookup_counter, 8, cudaMemcpyDeviceToHost, ctx->stream));
    SCONV_CUDA(cudaMemsetAsync(ctx->lookup_counter, 0, 8, ctx->stream));
    ctx->sync();
  });
}

sconv_status sconv_ctx_set_profiling(sconv_ctx* ctx, int enabled) {
  return guarded(ctx, [&] {
    ctx->resolve_profile();
    ctx->profiling = enabled != 0;
  });
}
sconv_status sconv_ctx_set_profile_filter(sconv_ctx* ctx, const char* kernel_label) {
  return guarded(ctx, [&] {
    ctx->resolve_profile();
    ctx->profile_only = kernel_label ? kernel_label : "";
  });
}
int sconv_ctx_profile_count(const sconv_ctx* ctx) { return static_cast<int>(ctx->profile_names.size()); }
sconv_status sconv_ctx_profile_entry(sconv_ctx* ctx, int i, const char** name, int64_t* launches, double* total_ms) {
  return guarded(ctx, [&] {
    ctx->resolve_profile();
    if (i < 0 || i >= static_cast<int>(ctx->profile_names.size())) fail(SCONV_ERR_ARG, "profile index out of range");
    const auto& n = ctx->profile_names[i];
    const auto& e = ctx->profile.at(n);
    if (name) *name = n.c_str();
    if (launches) *launches = e.launches;
    if (total_ms) *total_ms = e.total_ms;
  });
}
sconv_status sconv_ctx_profile_reset(sconv_ctx* ctx) {
  return guarded(ctx, [&] {
    ctx->resolve_profile();
    ctx->profile.clear();
    ctx->profile_names.clear();
    ctx->last_records.clear();
  });
}
sconv_status sconv_ctx_flush_l2(sconv_ctx* ctx, size_t bytes) {
  return guarded(ctx, [&] {
    ctx->flush_buf.reserve(bytes, ctx->stream);
    SCONV_CUDA(cudaMemsetAsync(ctx->flush_buf.get(), ctx->launches & 0xFF, bytes, ctx->stream));
  });
}

sconv_status sconv_device_alloc(sconv_ctx* ctx, size_t bytes, void** out) {
  return guarded(ctx, [&] { SCONV_CUDA(cudaMalloc(out, std::max<size_t>(bytes, 1))); });
}
sconv_status sconv_device_free(sconv_ctx* ctx, void* ptr) {
  return guarded(ctx, [&] {
    SCONV_CUDA(cudaStreamSynchronize(ctx->stream));
    SCONV_CUDA(cudaFree(ptr));
  });
}
sconv_status sconv_memcpy(sconv_ctx* ctx, void* dst, const void* src, size_t bytes, int kind) {
  return guarded(ctx, [&] {
    SCONV_CUDA(cudaMemcpyAsync(dst, src, bytes, static_cast<cudaMemcpyKind>(kind), ctx->stream));
    ctx->sync();
  });
}

sconv_status sconv_map_build(sconv_ctx* ctx, const int32_t* xyz, int64_t n, int mem, int in_sorted,
                             const sconv_map_cfg* cfg, const int32_t* target_xyz, int64_t n_target, int target_mem,
                             sconv_map** out) {
  return guarded(ctx, [&] {
    if (!cfg || !out) fail(SCONV_ERR_ARG, "null argument");
    if (n > 0 && !xyz) fail(SCONV_ERR_ARG, "null coordinates");
    MapSource P;
    P.xyz = xyz;
    P.n = n;
    P.mem = mem;
    P.sorted = in_sorted != 0;
    MapSource T;
    T.xyz = target_xyz;
    T.n = n_target;
    T.mem = target_mem;
    T.sorted = true;
    *out = wrap(build_map(*ctx, P, *cfg, cfg->transposed ? &T : nullptr));
  });
}

sconv_status sconv_map_build_chained(sconv_ctx* ctx, const sconv_map* prev, const sconv_map_cfg* cfg,
                                     const sconv_map* target_of, sconv_map** out) {
  return guarded(ctx, [&] {
    if (!prev || !cfg || !out) fail(SCONV_ERR_ARG, "null argument");
    MapSource P;
    P.keys = prev->q_keys;
    P.n = prev->n_out;
    P.sorted = true;
    MapSource T;
    if (cfg->transposed) {
      if (!target_of) fail(SCONV_ERR_ARG, "transposed layer needs target coordinates");
      if (!target_of->src_identity) fail(SCONV_ERR_ARG, "target map input must be sorted");
      T.keys = target_of->src_keys;
      T.n = target_of->n_in;
      T.sorted = true;
    }
    *out = wrap(build_map(*ctx, P, *cfg, cfg->transposed ? &T : nullptr));
  });
}

sconv_status sconv_map_build_explicit(sconv_ctx* ctx, const int32_t* p_xyz, int64_t n_p, int p_mem, int p_sorted,
                                     const int32_t* q_xyz, int64_t n_q, int q_mem, const int32_t* offsets_xyz,
                                     int n_offsets, int block_B, int block_C, int backend, sconv_map** out) {
  return guarded(ctx, [&] {
    if (!out) fail(SCONV_ERR_ARG, "null argument");
    if ((n_p > 0 && !p_xyz) || (n_q > 0 && !q_xyz)) fail(SCONV_ERR_ARG, "null coordinates");
    if (n_offsets < 1 || !offsets_xyz) fail(SCONV_ERR_ARG, "offset count must be in [1, 4096]");
    if (n_q < 0 || n_q > INT32_MAX / 2) fail(SCONV_ERR_ARG, "point count out of supported range");
    std::vector<int3> offs(static_cast<size_t>(n_offsets));
    for (int k = 0; k < n_offsets; ++k) offs[k] = make_int3(offsets_xyz[3 * k], offsets_xyz[3 * k + 1], offsets_xyz[3 * k + 2]);
    MapSource P;
    P.xyz = p_xyz;
    P.n = n_p;
    P.mem = p_mem;
    P.sorted = p_sorted != 0;
    MapSource T;
    T.xyz = q_xyz;
    T.n = n_q;
    T.mem = q_mem;
    T.sorted = true;
    // kernel_size / scale describe no geometry here (the offsets are explicit); stride 1
    sconv_map_cfg cfg{1, 1, 1, 0, block_B, block_C, backend};
    *out = wrap(build_map(*ctx, P, cfg, &T, false, false, &offs));
  });
}

sconv_status sconv_map_search_counters(sconv_ctx* ctx, const sconv_map* m, sconv_search_counters* c) {
  return guarded(ctx, [&] {
    if (!m || !c) fail(SCONV_ERR_ARG, "null argument");
    *c = sconv_search_counters{};
    c->sorts = static_cast<uint64_t>(m->sorts);
    c->counted = m->counted ? 1 : 0;
    if (m->counted) {
      uint64_t v[4];
      SCONV_CUDA(cudaMemcpyAsync(v, m->counters.get(), sizeof(v), cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      c->backward_comparisons = v[0];
      c->forward_comparisons = v[1];
      c->source_elements_loaded = v[2];
      c->queries_executed = v[3];
    }
  });
}

sconv_status sconv_theoretical_hyperparams(int64_t num_inputs, int64_t num_outputs, int* block_B, int* block_C) {
  return guarded(nullptr, [&] {
  if (num_inputs < 1 || num_outputs < 1) fail(SCONV_ERR_ARG, "point counts must be positive");
  if (!block_B || !block_C) fail(SCONV_ERR_ARG, "null argument");
  // SPEC.md:244-252 (Eq. 4): B = max(1, round(|P|/|Q| log2|Q|)),
  // C = max(1, round(sqrt(|Q| / (|P| log2 B)) B)) with log2 B floored at 1
  const double ratio = static_cast<double>(num_inputs) / static_cast<double>(num_outputs);
  const int B = std::max(1, static_cast<int>(std::lround(ratio * std::log2(static_cast<double>(num_outputs)))));
  const double lb = std::max(1.0, std::log2(static_cast<double>(B)));
  *block_B = B;
  *block_C = std::max(1, static_cast<int>(std::lround(
                             std::sqrt(static_cast<double>(num_outputs) / (static_cast<double>(num_inputs) * lb)) * B)));
  });
}

sconv_status sconv_map_get_info(sconv_ctx* ctx, const sconv_map* m, sconv_map_info* info) {
  return guarded(ctx, [&] {
    if (!m || !info) fail(SCONV_ERR_ARG, "null argument");
    ensure_canonical(*ctx, const_cast<MapData&>(static_cast<const MapData&>(*m)));
    info->num_inputs = m->n_in;
    info->num_outputs = m->n_out;
    info->num_offsets = m->K3;
    info->total_matches = m->total;
    info->buffer_length = m->buffer_length;
    info->groups = m->groups;
    info->padding_overhead = m->padding_overhead;
    info->gather_tile = m->gather_tile;
    info->scatter_tile = m->scatter_tile;
  });
}

sconv_status sconv_map_read(sconv_ctx* ctx, const sconv_map* m, int32_t* out_xyz, int64_t* sizes, int32_t* in_idx,
                            int32_t* out_idx) {
  return guarded(ctx, [&] {
    if (!m) fail(SCONV_ERR_ARG, "null map");
    ensure_canonical(*ctx, const_cast<MapData&>(static_cast<const MapData&>(*m)));
    if (out_xyz && m->n_out > 0) {
      std::vector<uint64_t> keys(m->n_out);
      SCONV_CUDA(cudaMemcpyAsync(keys.data(), m->q_keys_ptr(), keys.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      for (int64_t i = 0; i < m->n_out; ++i) unpack_key(keys[i], out_xyz[3 * i], out_xyz[3 * i + 1], out_xyz[3 * i + 2]);
    }
    if (sizes)
      for (int k = 0; k < m->K3; ++k) sizes[k] = m->sizes[k];
    if (in_idx && m->total > 0)
      SCONV_CUDA(cudaMemcpyAsync(in_idx, m->pair_in.get(), m->total * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (out_idx && m->total > 0)
      SCONV_CUDA(cudaMemcpyAsync(out_idx, m->pair_out.get(), m->total * 4, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  });
}

sconv_status sconv_map_device_views(const sconv_map* m, const uint64_t** out_keys, const int32_t** in_idx,
                                    const int32_t** out_idx) {
  if (!m) return SCONV_ERR_ARG;
  if (out_keys) *out_keys = m->q_keys_ptr();
  if (in_idx) *in_idx = m->pair_in.get<int32_t>();
  if (out_idx) *out_idx = m->pair_out.get<int32_t>();
  return SCONV_OK;
}

void sconv_map_free(sconv_ctx* ctx, sconv_map* m) {
  (void)ctx;
  delete m;
}

sconv_status sconv_weights_create(sconv_ctx* ctx, const float* w, int mem, int num_offsets, int c_in, int c_out,
                                  int dtype, sconv_weights** out) {
  return guarded(ctx, [&] {
    if (!w || !out) fail(SCONV_ERR_ARG, "null argument");
    auto wd = create_weights(*ctx, w, mem, num_offsets, c_in, c_out, dtype);
    auto* o = new sconv_weights;
    static_cast<WeightData&>(*o) = std::move(*wd);
    *out = o;
  });
}
void sconv_weights_free(sconv_ctx* ctx, sconv_weights* w) {
  (void)ctx;
  delete w;
}

sconv_status sconv_layer_forward(sconv_ctx* ctx, sconv_map* map, const sconv_weights* w, const void* f_in,
                                 int f_in_dtype, int f_in_mem, const sconv_exec_cfg* cfg, void* f_out, int f_out_dtype,
                                 int f_out_mem) {
  return guarded(ctx, [&] {
    if (!map || !w) fail(SCONV_ERR_ARG, "null argument");
    if ((map->n_in > 0 && !f_in) || (map->n_out > 0 && !f_out)) fail(SCONV_ERR_ARG, "null feature buffer");
    const sconv_exec_cfg c = normalize(cfg);
    layer_forward(*ctx, *map, *w, f_in, f_in_dtype, f_in_mem, c, f_out, f_out_dtype, f_out_mem);
  });
}

sconv_status sconv_tune_layer(sconv_ctx* ctx, sconv_map* map, const sconv_weights* w, const void* f_in, int f_in_dtype,
                              int rounds, int* gather_tile, int* scatter_tile, double* lat, int* n_lat) {
  return guarded(ctx, [&] {
    if (!map || !w || !f_in) fail(SCONV_ERR_ARG, "null argument");
    if (rounds < 1) fail(SCONV_ERR_ARG, "rounds must be positive");
    const bool was = ctx->profiling;
    ctx->resolve_profile();
    ctx->profiling = true;
    DevBuf out;
    out.alloc(static_cast<size_t>(std::max<int64_t>(1, map->n_out)) * w->c_out * 4, ctx->stream);
    auto time_kernel = [&](const char* name, int tg, int ts) {
      sconv_exec_cfg c = normalize(nullptr);
      c.compute_dtype = w->dtype;
      c.gather_tile = tg;
      c.scatter_tile = ts;
      std::vector<double> samples;
      for (int r = 0; r <= rounds; ++r) {  // 1 warm-up + R measured
        ctx->last_records.clear();
        layer_forward(*ctx, *map, *w, f_in, f_in_dtype, SCONV_MEM_DEVICE, c, out.get(), SCONV_F32, SCONV_MEM_DEVICE);
        ctx->resolve_profile();
        double ms = 0;
        for (auto& rec : ctx->last_records)
          if (rec.first == name) ms += rec.second;
        if (r > 0) samples.push_back(ms);
      }
      return median(samples);
    };
    std::vector<double> all;
    auto pick = [&](const char* name, int channels, bool gather) {
      int best = -1;
      double best_ms = 0;
      for (int t : candidate_tiles(channels)) {
        const double ms = gather ? time_kernel(name, t, default_tile(w->c_out, false))
                                 : time_kernel(name, default_tile(w->c_in, true), t);
        all.push_back(ms);
        if (best < 0 || ms < best_ms) {  // strict: smallest tile wins ties
          best = t;
          best_ms = ms;
        }
      }
      return best;
    };
    const int tg = pick("k_gather", w->c_in, true);
    const int ts = pick("k_scatter", w->c_out, false);
    ctx->profiling = was;
    ctx->tuned[{w->c_in, w->c_out, w->dtype}] = {tg, ts};
    if (gather_tile) *gather_tile = tg;
    if (scatter_tile) *scatter_tile = ts;
    if (n_lat) {
      if (lat)
        for (size_t i = 0; i < all.size() && static_cast<int>(i) < *n_lat; ++i) lat[i] = all[i];
      *n_lat = static_cast<int>(all.size());
    }
  });
}

sconv_status sconv_sc_layer_forward(sconv_ctx* ctx, const int32_t* xyz, int64_t n, int in_sorted, const float* f_in,
                                    int c_in, const float* w, int c_out, int K, int s, const sconv_exec_cfg* cfg,
                                    int32_t* out_xyz, int64_t* n_out, float* f_out) {
  return guarded(ctx, [&] {
    const sconv_exec_cfg c = normalize(cfg);
    if (K < 1 || K % 2 == 0) fail(SCONV_ERR_ARG, "kernel size must be a positive odd integer");
    if (s < 1) fail(SCONV_ERR_ARG, "stride must be positive");
    const sconv_map_cfg mc = default_map_cfg(K, s);
    MapSource P;
    P.xyz = xyz;
    P.n = n;
    P.mem = SCONV_MEM_HOST;
    P.sorted = in_sorted != 0;
    auto m = build_map(*ctx, P, mc, nullptr);
    auto wd = create_weights(*ctx, w, SCONV_MEM_HOST, m->K3, c_in, c_out, c.compute_dtype);
    layer_forward(*ctx, *m, *wd, f_in, SCONV_F32, SCONV_MEM_HOST, c, f_out, SCONV_F32, SCONV_MEM_HOST);
    *n_out = m->n_out;
    if (out_xyz && m->n_out > 0) {
      std::vector<uint64_t> keys(m->n_out);
      SCONV_CUDA(cudaMemcpyAsync(keys.data(), m->q_keys_ptr(), keys.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      for (int64_t i = 0; i < m->n_out; ++i) unpack_key(keys[i], out_xyz[3 * i], out_xyz[3 * i + 1], out_xyz[3 * i + 2]);
    }
  });
}

sconv_status sconv_plan_groups(const int64_t* sizes, int n, int policy, double epsilon, int max_batch, int* order,
                               int* n_order, int* group_begin, int* group_end, int64_t* heights, int* n_groups,
                               int64_t* buffer_offsets, int64_t* buffer_length, double* overhead) {
  return guarded(nullptr, [&] {
    if (n < 0 || (n > 0 && !sizes)) fail(SCONV_ERR_ARG, "invalid sizes");
    const GroupPlan p = group_gemms(std::vector<int64_t>(sizes, sizes + n), policy, epsilon, max_batch);
    *n_order = static_cast<int>(p.order.size());
    for (size_t i = 0; i < p.order.size(); ++i) order[i] = p.order[i];
    *n_groups = static_cast<int>(p.groups.size());
    for (size_t g = 0; g < p.groups.size(); ++g) {
      group_begin[g] = p.groups[g].begin;
      group_end[g] = p.groups[g].end;
      heights[g] = p.groups[g].height;
    }
    for (int k = 0; k < n; ++k) buffer_offsets[k] = p.buffer_offsets[k];
    *buffer_length = p.buffer_length;
    *overhead = p.real_rows > 0 ? static_cast<double>(p.buffer_length - p.real_rows) / p.real_rows : -1.0;
  });
}

sconv_status sconv_net_create(sconv_ctx* ctx, const int32_t* ops, int n_ops, int num_tensors, int input_tensor,
                              int output_tensor, const sconv_exec_cfg* cfg, int block_B, int block_C,
                              sconv_net** out) {
  return guarded(ctx, [&] {
    if (!out || (n_ops > 0 && !ops)) fail(SCONV_ERR_ARG, "null argument");
    auto n = std::make_unique<sconv_net>();
    n->num_tensors = num_tensors;
    n->input_tensor = input_tensor;
    n->output_tensor = output_tensor;
    n->block_B = block_B > 0 ? block_B : 256;
    n->block_C = block_C > 0 ? block_C : 512;
    n->cfg = normalize(cfg, SCONV_DATAFLOW_AUTO);
    if (input_tensor < 0 || input_tensor >= num_tensors || output_tensor < 0 || output_tensor >= num_tensors)
      fail(SCONV_ERR_ARG, "tensor id out of range");
    for (int i = 0; i < n_ops; ++i) {
      const int32_t* r = ops + static_cast<size_t>(i) * kOpFields;
      NetOp o;
      o.kind = r[0];
      o.out = r[1];
      o.in = r[2];
      o.b = r[3];
      o.target = r[3];
      o.K = r[4];
      o.offset_scale = r[5];
      o.out_stride = r[6];
      o.transposed = r[7];
      o.c_in = r[8];
      o.c_out = r[9];
      o.weight = r[10];
      o.relu = r[11];
      n->ops.push_back(o);
    }
    n->check_ops();
    *out = n.release();
  });
}

sconv_status sconv_net_set_weights(sconv_ctx* ctx, sconv_net* net, int weight_id, const float* w, int mem,
                                   int num_offsets, int c_in, int c_out) {
  return guarded(ctx, [&] {
    if (!net || !w) fail(SCONV_ERR_ARG, "null argument");
    net->weights[weight_id] = create_weights(*ctx, w, mem, num_offsets, c_in, c_out, net->cfg.compute_dtype);
  });
}

sconv_status sconv_net_forward(sconv_ctx* ctx, sconv_net* net, const int32_t* xyz, int64_t n, int mem, int in_sorted,
                               const float* feats, int f_mem, int c_in) {
  return guarded(ctx, [&] {
    if (!net || (n > 0 && (!xyz || !feats))) fail(SCONV_ERR_ARG, "null argument");
    MapSource P;
    P.xyz = xyz;
    P.n = n;
    P.mem = mem;
    P.sorted = in_sorted != 0;
    // host inputs must outlive the asynchronous forward: staged on device by the net's input
    // stream (double-buffered), so the copy and the map builds need not wait for the previous
    // forward's convs on the context stream
    if (mem == SCONV_MEM_HOST && n > 0) {
      const int32_t* xd = nullptr;
      const float* fd = nullptr;
      auto& pf = net->prefetch;
      if (pf.slot >= 0 && pf.xyz == xyz && pf.feats == feats && pf.n == n && pf.f_mem == f_mem && pf.c_in == c_in) {
        net->staged_slot = pf.slot;  // copied by sconv_net_prefetch_inputs
        xd = pf.xyz_dev;
        fd = pf.feats_dev;
      } else {
        net->stage_host_inputs(xyz, n, feats, f_mem, c_in, &xd, &fd);
      }
      pf.slot = -1;
      P.xyz = xd;
      P.mem = SCONV_MEM_DEVICE;
      feats = fd;
      f_mem = SCONV_MEM_DEVICE;
    }
    net->forward(*ctx, P, feats, SCONV_F32, f_mem, c_in);
  });
}

sconv_status sconv_net_prefetch_inputs(sconv_ctx* ctx, sconv_net* net, const int32_t* xyz, int64_t n,
                                       const float* feats, int f_mem, int c_in) {
  return guarded(ctx, [&] {
    if (!net || n <= 0 || !xyz || !feats) fail(SCONV_ERR_ARG, "null argument");
    auto& pf = net->prefetch;
    net->stage_host_inputs(xyz, n, feats, f_mem, c_in, &pf.xyz_dev, &pf.feats_dev);
    pf.slot = net->staged_slot;
    net->staged_slot = -1;  // consumed by the matching sconv_net_forward only
    pf.xyz = xyz;
    pf.feats = feats;
    pf.n = n;
    pf.f_mem = f_mem;
    pf.c_in = c_in;
  });
}

sconv_status sconv_net_tensor_info(sconv_ctx* ctx, const sconv_net* net, int tensor, int64_t* n, int* channels,
                                   int* coordset) {
  return guarded(ctx, [&] {
    if (!net || tensor < 0 || tensor >= static_cast<int>(net->tensors.size())) fail(SCONV_ERR_ARG, "bad tensor");
    const NetTensor& t = net->tensors[tensor];
    if (n) *n = t.n;
    if (channels) *channels = t.channels;
    if (coordset) *coordset = t.coordset;
  });
}

sconv_status sconv_net_read_tensor(sconv_ctx* ctx, const sconv_net* net, int tensor, int32_t* xyz, float* feats) {
  return guarded(ctx, [&] {
    if (!net || tensor < 0 || tensor >= static_cast<int>(net->tensors.size())) fail(SCONV_ERR_ARG, "bad tensor");
    const NetTensor& t = net->tensors[tensor];
    if (t.fused_away) fail(SCONV_ERR_STATE, "tensor was folded into a fused residual epilogue");
    if (t.coordset < 0) fail(SCONV_ERR_STATE, "tensor not produced");
    if (feats && t.n > 0) {
      auto* n = const_cast<sconv_net*>(net);
      n->readback.reserve(sizeof(float) * t.n * t.channels, ctx->stream);
      convert_rows(*ctx, t.feats.get(), t.dtype, t.n, t.channels, t.ld, n->readback.get(), SCONV_F32, t.channels);
      SCONV_CUDA(cudaMemcpyAsync(feats, n->readback.get(), sizeof(float) * t.n * t.channels, cudaMemcpyDeviceToHost,
                                 ctx->stream));
    }
    if (xyz && t.n > 0) {
      const CoordSet& cs = net->coordsets[t.coordset];
      if (cs.keys) {
        std::vector<uint64_t> keys(t.n);
        SCONV_CUDA(cudaMemcpyAsync(keys.data(), cs.keys->get(), 8 * t.n, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
        for (int64_t i = 0; i < t.n; ++i) unpack_key(keys[i], xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
      } else {
        SCONV_CUDA(cudaMemcpyAsync(xyz, net->raw_input.xyz, 12 * t.n, cudaMemcpyDeviceToHost, ctx->stream));
      }
    }
    ctx->sync();
  });
}

sconv_status sconv_net_copy_tensor(sconv_ctx* ctx, const sconv_net* net, int tensor, void* dst, int dst_dtype,
                                   int dst_mem) {
  return guarded(ctx, [&] {
    if (!net || tensor < 0 || tensor >= static_cast<int>(net->tensors.size())) fail(SCONV_ERR_ARG, "bad tensor");
    if (dst_dtype != SCONV_F32 && dst_dtype != SCONV_F16 && dst_dtype != SCONV_BF16) fail(SCONV_ERR_ARG, "bad dtype");
    const NetTensor& t = net->tensors[tensor];
    if (t.fused_away) fail(SCONV_ERR_STATE, "tensor was folded into a fused residual epilogue");
    if (t.coordset < 0) fail(SCONV_ERR_STATE, "tensor not produced");
    if (t.n == 0) return;
    const size_t esz = dst_dtype == SCONV_F32 ? 4 : 2;
    const size_t bytes = esz * static_cast<size_t>(t.n) * t.channels;
    if (dst_mem == SCONV_MEM_DEVICE) {
      if (dst_dtype == t.dtype && t.ld == t.channels)
        SCONV_CUDA(cudaMemcpyAsync(dst, t.feats.get(), bytes, cudaMemcpyDeviceToDevice, ctx->stream));
      else
        convert_rows(*ctx, t.feats.get(), t.dtype, t.n, t.channels, t.ld, dst, dst_dtype, t.channels);
      return;  // asynchronous on the context stream
    }
    auto* n = const_cast<sconv_net*>(net);
    n->readback.reserve(bytes, ctx->stream);
    convert_rows(*ctx, t.feats.get(), t.dtype, t.n, t.channels, t.ld, n->readback.get(), dst_dtype, t.channels);
    SCONV_CUDA(cudaMemcpyAsync(dst, n->readback.get(), bytes, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  });
}

sconv_status sconv_net_read_async(sconv_ctx* ctx, sconv_net* net, int tensor, float* feats) {
  return guarded(ctx, [&] {
    if (!net || tensor < 0 || tensor >= static_cast<int>(net->tensors.size())) fail(SCONV_ERR_ARG, "bad tensor");
    const NetTensor& t = net->tensors[tensor];
    if (t.fused_away) fail(SCONV_ERR_STATE, "tensor was folded into a fused residual epilogue");
    if (t.coordset < 0) fail(SCONV_ERR_STATE, "tensor not produced");
    if (t.n == 0) return;
    if (!feats) fail(SCONV_ERR_ARG, "null argument");
    if (!net->copy_stream) {
      SCONV_CUDA(cudaStreamCreateWithFlags(&net->copy_stream, cudaStreamNonBlocking));
      for (int s = 0; s < 2; ++s) {
        SCONV_CUDA(cudaEventCreateWithFlags(&net->rb_ready[s], cudaEventDisableTiming));
        SCONV_CUDA(cudaEventCreateWithFlags(&net->rb_done[s], cudaEventDisableTiming));
      }
    }
    const int s = net->rb_slot;
    net->rb_slot ^= 1;
    const size_t bytes = sizeof(float) * static_cast<size_t>(t.n) * t.channels;
    // the slot's previous copy must have left the staging buffer before it is rewritten (or
    // regrown: the old buffer's free is ordered on the context stream)
    if (net->rb_pending[s]) SCONV_CUDA(cudaStreamWaitEvent(ctx->stream, net->rb_done[s], 0));
    net->rb_async[s].reserve(bytes, ctx->stream);
    convert_rows(*ctx, t.feats.get(), t.dtype, t.n, t.channels, t.ld, net->rb_async[s].get(), SCONV_F32, t.channels);
    SCONV_CUDA(cudaEventRecord(net->rb_ready[s], ctx->stream));
    SCONV_CUDA(cudaStreamWaitEvent(net->copy_stream, net->rb_ready[s], 0));
    // In chunks: the copy engine is FIFO across streams, so a whole-result copy (C2: 45.7 MB =
    // 0.87 ms) holds back the next request's input H2D queued behind it (same box r02ch: C2
    // pipelined e2e 2.26 ms with 2 MB chunks vs 2.40 one copy; r02cl / r02cm: 4 MB 2.27, 2 MB
    // 2.26, 1 MB 2.21, 512 KB 2.17, 256 KB 2.23). Each chunk costs ~3.5 us of engine time, which
    // only shows when the copy is the bottleneck (r02cn, C4: 25 MB per 0.19 ms forward, 0.83 ms
    // with 2 MB chunks vs 1.00 with 512 KB): 512 KB chunks while the copy plus their overhead
    // fits in the last forward's GPU span, else 4 MB. The small map readbacks avoid the engine
    // altogether (map.cu d2h_small). SCONV_RB_CHUNK_KB forces a size.
    static const long forced_kb = [] {
      const char* e = std::getenv("SCONV_RB_CHUNK_KB");
      return e ? std::max(64L, std::atol(e)) : 0L;
    }();
    size_t chunk = size_t{512} << 10;
    if (forced_kb) {
      chunk = static_cast<size_t>(forced_kb) << 10;
    } else if (net->last_fwd_ms >= 0.f) {
      const double copy_ms = static_cast<double>(bytes) / 5.0e7;  // ~50 GB/s pinned D2H (r02cc)
      const double overhead_ms = 0.0035 * static_cast<double>((bytes + chunk - 1) / chunk);
      if (copy_ms + overhead_ms > 0.8 * net->last_fwd_ms) chunk = size_t{4} << 20;
    }
    for (size_t off = 0; off < bytes; off += chunk)
      SCONV_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(feats) + off, net->rb_async[s].get<char>() + off,
                                 std::min(chunk, bytes - off), cudaMemcpyDeviceToHost, net->copy_stream));
    SCONV_CUDA(cudaEventRecord(net->rb_done[s], net->copy_stream));
    net->rb_pending[s] = true;
  });
}

sconv_status sconv_net_read_wait(sconv_ctx* ctx, sconv_net* net) {
  return guarded(ctx, [&] {
    if (!net) fail(SCONV_ERR_ARG, "null argument");
    if (net->copy_stream) SCONV_CUDA(cudaStreamSynchronize(net->copy_stream));
  });
}

sconv_status sconv_net_tensor_device(const sconv_net* net, int tensor, const void** feats, int* dtype, int64_t* ld) {
  if (!net || tensor < 0 || tensor >= static_cast<int>(net->tensors.size()) || !feats) return SCONV_ERR_ARG;
  const NetTensor& t = net->tensors[tensor];
  if (t.fused_away || t.coordset < 0) return SCONV_ERR_STATE;
  *feats = t.feats.get();
  if (dtype) *dtype = t.dtype;
  if (ld) *ld = t.ld;
  return SCONV_OK;
}

sconv_status sconv_net_sort_count(const sconv_net* net, int64_t* sorts) {
  if (!net || !sorts) return SCONV_ERR_ARG;
  *sorts = net->sorts;
  return SCONV_OK;
}

sconv_status sconv_net_stats(const sconv_net* net, int* maps_built, int* convs) {
  if (!net) return SCONV_ERR_ARG;
  if (maps_built) *maps_built = net->maps_built;
  if (convs) {
    int c = 0;
    for (const auto& o : net->ops) c += o.kind == kOpConv;
    *convs = c;
  }
  return SCONV_OK;
}

sconv_status sconv_net_conv_stats(const sconv_net* net, int conv, int64_t* out10) {
  if (!net || !out10 || conv < 0 || conv >= static_cast<int>(net->conv_stats.size())) return SCONV_ERR_ARG;
  for (int i = 0; i < 10; ++i) out10[i] = net->conv_stats[conv][i];
  return SCONV_OK;
}

sconv_status sconv_net_resolve_stats(sconv_ctx* ctx, sconv_net* net) {
  if (!net) return SCONV_ERR_ARG;
  return guarded(ctx, [&] {
    net->resolve_stats(*ctx);
    ctx->sync();
  });
}

sconv_status sconv_net_conv_timings(const sconv_net* net, int op, double* gmas_ms, double* fused_ms) {
  if (!net || op < 0 || op >= static_cast<int>(net->auto_ms.size())) return SCONV_ERR_ARG;
  if (gmas_ms) *gmas_ms = net->auto_ms[op][0];
  if (fused_ms) *fused_ms = net->auto_ms[op][1];
  return SCONV_OK;
}

sconv_status sconv_net_autotune(sconv_ctx* ctx, sconv_net* net, int n_samples, const int32_t* const* xyz,
                                const int64_t* n, const int* sorted, const float* const* feats, int c_in, int rounds,
                                int* tiles_out) {
  return guarded(ctx, [&] {
    if (!net) fail(SCONV_ERR_ARG, "null argument");
    if (n_samples < 1) fail(SCONV_ERR_ARG, "sample must be nonempty");
    if (rounds < 1) fail(SCONV_ERR_ARG, "rounds must be positive");
    if (!xyz || !n || !feats) fail(SCONV_ERR_ARG, "null argument");
    NetTune t;
    t.rounds = rounds;
    struct Reset {
      NetData* net;
      ~Reset() { net->tune = nullptr; }
    } reset{net};
    net->tune = &t;
    for (int i = 0; i < n_samples; ++i) {
      MapSource P;
      P.n = n[i];
      P.sorted = sorted ? sorted[i] != 0 : false;
      DevBuf staged;
      if (P.n > 0) {
        staged.alloc(sizeof(int32_t) * 3 * P.n, ctx->stream);
        SCONV_CUDA(cudaMemcpyAsync(staged.get(), xyz[i], sizeof(int32_t) * 3 * P.n, cudaMemcpyHostToDevice, ctx->stream));
        net->input_xyz = std::move(staged);
        P.xyz = net->input_xyz.get<int32_t>();
        P.mem = SCONV_MEM_DEVICE;
      }
      net->forward(*ctx, P, feats[i], SCONV_F32, SCONV_MEM_HOST, c_in);
      ctx->sync();
    }
    net->finish_tune();
    net->last_tune = t;
    if (tiles_out)
      for (size_t o = 0; o < net->ops.size(); ++o) {
        tiles_out[2 * o] = net->plan.empty() ? 0 : net->plan[o].gather_tile;
        tiles_out[2 * o + 1] = net->plan.empty() ? 0 : net->plan[o].scatter_tile;
      }
  });
}

sconv_status sconv_net_tune_latencies(const sconv_net* net, int op, int* tiles, double* ms, int cap, int* n_gather,
                                      int* n_scatter) {
  if (!net || op < 0) return SCONV_ERR_ARG;
  const NetTune& t = net->last_tune;
  const auto g = t.gather_ms.find(op), s = t.scatter_ms.find(op);
  int i = 0;
  auto put = [&](const std::map<int, double>& c) {
    for (const auto& [tile, v] : c) {
      if (i < cap && tiles) tiles[i] = tile;
      if (i < cap && ms) ms[i] = v;
      ++i;
    }
  };
  if (g != t.gather_ms.end()) put(g->second);
  if (n_gather) *n_gather = g != t.gather_ms.end() ? static_cast<int>(g->second.size()) : 0;
  if (s != t.scatter_ms.end()) put(s->second);
  if (n_scatter) *n_scatter = s != t.scatter_ms.end() ? static_cast<int>(s->second.size()) : 0;
  return SCONV_OK;
}

void sconv_net_free(sconv_ctx* ctx, sconv_net* net) {
  if (ctx) cudaStreamSynchronize(ctx->stream);
  delete net;
}

sconv_status sconv_voxelize(sconv_ctx* ctx, const double* points, int64_t n, int points_mem, const float* feats,
                            int64_t channels, int feats_mem, double resolution, int32_t* out_xyz, float* out_feats,
                            int out_mem, int64_t* n_voxels) {
  return guarded(ctx, [&] {
    if (!n_voxels || (n > 0 && (!points || !out_xyz || (channels > 0 && !out_feats))))
      fail(SCONV_ERR_ARG, "null argument");
    *n_voxels = voxelize(*ctx, points, n, points_mem, feats, channels, feats_mem, resolution, out_xyz, out_feats,
                         out_mem);
  });
}

sconv_status sconv_generate_synthetic(int64_t N, int64_t E, int64_t C, uint64_t seed, int32_t* xyz, float* feats) {
  return guarded(nullptr, [&] {
    if (N < 0 || E < 1 || C < 0) fail(SCONV_ERR_ARG, "invalid synthetic cloud parameters");
    if (static_cast<double>(N) > static_cast<double>(E) * E * E) fail(SCONV_ERR_ARG, "infeasible: N > E^3");
    if (E - 1 > kCoordMax) fail(SCONV_ERR_RANGE, "extent out of coordinate range");
    SplitMix r{stream_seed(seed, 0)};
    std::unordered_set<uint64_t> seen;
    seen.reserve(static_cast<size_t>(N) * 2);
    int64_t got = 0;
    while (got < N) {
      const int32_t x = static_cast<int32_t>(r.below(static_cast<uint64_t>(E)));
      const int32_t y = static_cast<int32_t>(r.below(static_cast<uint64_t>(E)));
      const int32_t z = static_cast<int32_t>(r.below(static_cast<uint64_t>(E)));
      if (!seen.insert(pack_key_unchecked(x, y, z)).second) continue;
      xyz[3 * got] = x;
      xyz[3 * got + 1] = y;
      xyz[3 * got + 2] = z;
      ++got;
    }
    for (int64_t i = 0; i < N * C; ++i) feats[i] = static_cast<float>(r.unit());
  });
}

sconv_status sconv_generate_weights(uint64_t seed, uint64_t stream, int num_offsets, int c_in, int c_out, float* w) {
  return guarded(nullptr, [&] {
    SplitMix r{stream_seed(seed, stream)};
    const int64_t n = int64_t{num_offsets} * c_in * c_out;
    for (int64_t i = 0; i < n; ++i) w[i] = static_cast<float>(-0.1 + 0.2 * r.unit());
  });
}

}  // extern "C"

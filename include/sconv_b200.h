/* sconv_b200 — B200-native sparse-convolution engine (Minuet Map + GMaS), C ABI.
 *
 * Drop-in boundary for the reference's SC-layer API. The reference (arXiv 2401.06145
 * artifact) is a header-only C++20 library in namespace `sconv`; its hot path exists as
 * the types in proj/include/sconv/geometry.hpp plus the SPEC.md operation signatures.
 * Each entry point below names the reference interface it replaces. No exceptions and
 * no C++/torch types cross this boundary: plain pointers, sizes and status codes. The
 * header-only C++ adapter include/sconv_b200.hpp rethrows the reference exception types.
 *
 * Status mapping (reference exception -> status):
 *   std::invalid_argument -> SCONV_ERR_ARG    (geometry.hpp:90,134-136,162,186,189)
 *   std::out_of_range     -> SCONV_ERR_RANGE  (geometry.hpp:53 "coordinate x out of range: v")
 *   std::logic_error      -> SCONV_ERR_STATE  (SPEC.md:327 invariant violations)
 * The message text (sconv_last_error) is identical to the reference's where one exists.
 *
 * Threading: one context per (host thread, device). Calls on a context are serialised
 * on its CUDA stream. Results are deterministic and independent of grid sizes.
 */
#ifndef SCONV_B200_H_
#define SCONV_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SCONV_OK = 0,
  SCONV_ERR_ARG = 1,
  SCONV_ERR_RANGE = 2,
  SCONV_ERR_CUDA = 3,
  SCONV_ERR_OOM = 4,
  SCONV_ERR_STATE = 5
} sconv_status;

typedef enum { SCONV_MEM_HOST = 0, SCONV_MEM_DEVICE = 1 } sconv_mem;
typedef enum { SCONV_F32 = 0, SCONV_F16 = 1, SCONV_BF16 = 2 } sconv_dtype;
typedef enum { SCONV_GROUP_MAP_ORDER = 0, SCONV_GROUP_SORTED = 1 } sconv_group_policy;
/* GMaS dataflow. GMAS: Minuet's gather -> grouped GEMM -> scatter with materialised
 * buffers. FUSED: output-stationary gather -> tcgen05 GEMM -> in-TMEM
 * ascending-k reduction in one kernel; same arithmetic (fp32
 * accumulation of 16-bit operand products, ascending k). AUTO (network driver only):
 * each conv is timed once with both dataflows and the faster is kept (Alg. 2 style). */
typedef enum { SCONV_DATAFLOW_GMAS = 0, SCONV_DATAFLOW_FUSED = 1, SCONV_DATAFLOW_AUTO = 2 } sconv_dataflow;

typedef struct sconv_ctx sconv_ctx;
typedef struct sconv_map sconv_map;
typedef struct sconv_weights sconv_weights;

/* Layer geometry + Map hyperparameters.
 * SPEC-literal sc_layer_forward(cloud, W, K, s, cfg) is
 * {kernel_size=K, offset_scale=s, out_stride=s, transposed=0}. SURVEY §2.2 extensions:
 * even K (t in [0,K-1]), tensor strides (offset_scale != out_stride) and transposed
 * maps (queries = target coordinates, offsets negated). */
typedef struct {
  int kernel_size;  /* K */
  int offset_scale; /* weight offsets = t * offset_scale */
  int out_stride;   /* Eq. 1 stride for the output coordinates (ignored when transposed) */
  int transposed;   /* 1: output coordinates = target, offsets negated */
  int block_B;      /* source block size B (SPEC.md:247 default 256) */
  int block_C;      /* balanced query-block cap C (default 512) */
  int backend;      /* sconv_map_backend: SORTED (Minuet, default) or HASH (SPEC.md:114-160 baseline) */
} sconv_map_cfg;

/* Map backend. SORTED: segmented query sorting + double-traversed binary search (Minuet).
 * HASH: the SPEC's hash-table baseline (capacity = smallest power of two >= 2N, 64-bit
 * Fibonacci multiplicative hash, linear probing) on the GPU. Both produce the
 * identical canonical KernelMap (SPEC.md:367 backend equivalence). */
/* SORTED_SPEC: the same sorted search with the SPEC's literal work decomposition
 * (backward_partition per (offset, source block) -> balance_blocks: ceil(L/C) near-equal ranges
 * -> forward_block_search per range with the block staged in shared memory)
 * and its SearchCounters (sconv_map_search_counters), equal to the oracle's. SORTED is this
 * engine's warp-window redesign of that search (faster; no comparison counters). */
typedef enum { SCONV_MAP_SORTED = 0, SCONV_MAP_HASH = 1, SCONV_MAP_SORTED_SPEC = 2 } sconv_map_backend;

/* GMaS configuration (SPEC.md:359 config{grouping policy, eps, max_batch, tiles}). */
typedef struct {
  int policy;         /* sconv_group_policy, default SORTED */
  double epsilon;     /* padding threshold, default 0.25 */
  int max_batch;      /* max GEMMs per group, default 16 */
  int gather_tile;    /* T_g channels per work item; 0 = autotuned / heuristic */
  int scatter_tile;   /* T_s; 0 = autotuned / heuristic */
  int compute_dtype;  /* GEMM operand type: SCONV_F16 (default) or SCONV_BF16 */
  int partial_f16;    /* 0 (default): per-offset GEMM partials stored as fp32 ("stored as
                         32-bit"); 1: f16 partials when compute is f16 (halves partial traffic; the
                         extra rounding per offset can exceed SURVEY 8(c)'s per-element bound on
                         outputs near zero, so it is opt-in) */
  int dataflow;       /* sconv_dataflow, default GMAS for layers, AUTO for networks */
  int fuse_residual;  /* network driver: fold ADD (+ReLU) into the producing conv's epilogue (default 1) */
} sconv_exec_cfg;

typedef struct {
  int64_t num_inputs;      /* |P| */
  int64_t num_outputs;     /* |Q| */
  int32_t num_offsets;     /* K^3 (or K^3 for even K) */
  int64_t total_matches;   /* |M| */
  int64_t buffer_length;   /* R_pad of the last layer_forward on this map (0 before) */
  int32_t groups;          /* GEMM groups of the last layer_forward */
  double padding_overhead; /* x / y (Fig. 6) of the last layer_forward */
  int32_t gather_tile, scatter_tile;
} sconv_map_info;

/* ---------------- context ---------------- */
sconv_status sconv_ctx_create(int device, sconv_ctx** out);
/* Free every map / weight set / network of the context before destroying it. */
void sconv_ctx_destroy(sconv_ctx* ctx);
const char* sconv_last_error(const sconv_ctx* ctx);
/* Use an existing cudaStream_t (NULL = the context's own stream). */
sconv_status sconv_ctx_set_stream(sconv_ctx* ctx, void* cuda_stream);
void* sconv_ctx_stream(const sconv_ctx* ctx);
sconv_status sconv_ctx_synchronize(sconv_ctx* ctx);
/* Kernel launches issued by this context so far (gpu_launches accounting). */
int64_t sconv_ctx_launch_count(const sconv_ctx* ctx);
/* Per-kernel CUDA-event timing on the context stream (0 = off). */
/* Gather IMT-lookup counter (SPEC.md:332-340 counter; acceptance #6: lookups = (C_in / T) * |M|):
 * while enabled every GMaS gather adds its lookups; sconv_ctx_lookup_count returns the total since
 * the last read and resets it (synchronises the context stream). */
sconv_status sconv_ctx_set_lookup_counting(sconv_ctx* ctx, int enabled);
sconv_status sconv_ctx_lookup_count(sconv_ctx* ctx, unsigned long long* count);
sconv_status sconv_ctx_set_profiling(sconv_ctx* ctx, int enabled);
/* Restrict profiling events to launches with this label (NULL / "" = all). */
sconv_status sconv_ctx_set_profile_filter(sconv_ctx* ctx, const char* kernel_label);
/* Accumulated profile: kernel i -> name, launches, total ms. Returns count. */
int sconv_ctx_profile_count(const sconv_ctx* ctx);
sconv_status sconv_ctx_profile_entry(sconv_ctx* ctx, int i, const char** name, int64_t* launches, double* total_ms);
sconv_status sconv_ctx_profile_reset(sconv_ctx* ctx);
/* Write `bytes` to a scratch buffer (L2 flush between timed iterations). */
sconv_status sconv_ctx_flush_l2(sconv_ctx* ctx, size_t bytes);

/* ---------------- device buffers (for callers without their own allocator) ------ */
sconv_status sconv_device_alloc(sconv_ctx* ctx, size_t bytes, void** out);
sconv_status sconv_device_free(sconv_ctx* ctx, void* ptr);
sconv_status sconv_memcpy(sconv_ctx* ctx, void* dst, const void* src, size_t bytes, int kind /*cudaMemcpyKind*/);

/* ---------------- Map step ----------------
 * Replaces build_kernel_map_sorted(P, Q, offsets, B, C) together with
 * generate_output_coords(P, s) (geometry.hpp:161-178) and weight_offsets(K, s)
 * (geometry.hpp:133-148), as sc_layer_forward composes them.
 * xyz: n x 3 int32 (x,y,z) rows of P in `mem`. in_sorted: P.sorted (SPEC.md:193 sort reuse).
 * target_xyz/n_target: transposed layers only (sorted unique output coordinates).
 * Output coordinates Q are sorted; for stride 1 with sorted P they alias P (geometry.hpp:163).
 * Map indices: j = row of P as given, i = row of Q. */
sconv_status sconv_map_build(sconv_ctx* ctx, const int32_t* xyz, int64_t n, int mem, int in_sorted,
                             const sconv_map_cfg* cfg, const int32_t* target_xyz, int64_t n_target, int target_mem,
                             sconv_map** out);
/* Chain: P = the output coordinates of `prev` (device-resident, sorted; SPEC.md:528 reuse). */
sconv_status sconv_map_build_chained(sconv_ctx* ctx, const sconv_map* prev, const sconv_map_cfg* cfg,
                                     const sconv_map* target_of, sconv_map** out);
/* SPEC-literal build_kernel_map_sorted(P, Q, offsets, B, C): an arbitrary
 * sorted unique query list Q (n_q x 3, "query coordinates must be sorted and unique") and an
 * arbitrary offset list (n_offsets x 3 int32, SPEC: sorted once per layer); P as in
 * sconv_map_build. Map index j = row of P as given, i = row of Q; K3 = n_offsets. backend:
 * sconv_map_backend (SORTED_SPEC fills the comparison counters). */
sconv_status sconv_map_build_explicit(sconv_ctx* ctx, const int32_t* p_xyz, int64_t n_p, int p_mem, int p_sorted,
                                     const int32_t* q_xyz, int64_t n_q, int q_mem, const int32_t* offsets_xyz,
                                     int n_offsets, int block_B, int block_C, int backend, sconv_map** out);
/* SearchCounters of a map build. sorts = coordinate-array sorts the build
 * performed (0 when P was flagged sorted and the stride is 1, acceptance #7).
 * The comparison tallies are filled (counted = 1) by the SORTED_SPEC backend, whose work
 * decomposition is the SPEC's; they equal the oracle's exactly. */
typedef struct {
  uint64_t backward_comparisons;
  uint64_t forward_comparisons;
  uint64_t source_elements_loaded;
  uint64_t queries_executed;
  uint64_t sorts;
  int32_t counted;
} sconv_search_counters;
sconv_status sconv_map_search_counters(sconv_ctx* ctx, const sconv_map* map, sconv_search_counters* out);
/* theoretical_hyperparams(|P|, |Q|) -> (B, C) (Eq. 4): advisory; the runtime
 * defaults stay B = 256, C = 512. Errors: ARG "point counts must be positive". */
sconv_status sconv_theoretical_hyperparams(int64_t num_inputs, int64_t num_outputs, int* block_B, int* block_C);
sconv_status sconv_map_get_info(sconv_ctx* ctx, const sconv_map* map, sconv_map_info* info);
/* KernelMap readback in canonical order (per offset k, sorted by output index i;
 * SPEC.md:109). sizes: num_offsets; in_idx/out_idx: total_matches; out_xyz: num_outputs x 3.
 * Any pointer may be NULL. Host memory. */
sconv_status sconv_map_read(sconv_ctx* ctx, const sconv_map* map, int32_t* out_xyz, int64_t* sizes, int32_t* in_idx,
                            int32_t* out_idx);
/* Device views (valid until sconv_map_free): packed sorted output keys, canonical pairs. */
sconv_status sconv_map_device_views(const sconv_map* map, const uint64_t** out_keys, const int32_t** in_idx,
                                    const int32_t** out_idx);
void sconv_map_free(sconv_ctx* ctx, sconv_map* map);

/* ---------------- weights ----------------
 * WeightSet: num_offsets matrices c_in x c_out, fp32 row-major [k][cin][cout].
 * Stored on device in the GEMM operand type, K-major (transposed) for the tensor cores. */
sconv_status sconv_weights_create(sconv_ctx* ctx, const float* w, int mem, int num_offsets, int c_in, int c_out,
                                  int dtype, sconv_weights** out);
void sconv_weights_free(sconv_ctx* ctx, sconv_weights* w);

/* ---------------- GMaS step ----------------
 * Replaces group_gemms + build_metadata_tables + gather + gemm_execute + scatter
 * as composed by sc_layer_forward. f_in: num_inputs x c_in rows in
 * P order (dtype f_in_dtype, memory f_in_mem). f_out: num_outputs x c_out in Q order. */
sconv_status sconv_layer_forward(sconv_ctx* ctx, sconv_map* map, const sconv_weights* w, const void* f_in,
                                 int f_in_dtype, int f_in_mem, const sconv_exec_cfg* cfg, void* f_out, int f_out_dtype,
                                 int f_out_mem);

/* Alg. 2: profile every divisor tile for gather and scatter on this
 * map (1 warm-up + `rounds`, median of CUDA-event times), keep the argmin (smallest tile
 * on ties) and remember it for layers with the same (c_in, c_out). latencies_ms (optional)
 * receives [gather per candidate..., scatter per candidate...]. */
sconv_status sconv_tune_layer(sconv_ctx* ctx, sconv_map* map, const sconv_weights* w, const void* f_in,
                              int f_in_dtype, int rounds, int* gather_tile, int* scatter_tile,
                              double* latencies_ms, int* n_latencies);

/* One-shot SPEC-literal sc_layer_forward on host buffers:
 * coords + fp32 features in, sorted output coords + fp32 features out. out_xyz must hold
 * n rows (|Q| <= |P|), f_out n x c_out. */
sconv_status sconv_sc_layer_forward(sconv_ctx* ctx, const int32_t* xyz, int64_t n, int in_sorted, const float* f_in,
                                    int c_in, const float* w, int c_out, int K, int s, const sconv_exec_cfg* cfg,
                                    int32_t* out_xyz, int64_t* n_out, float* f_out);

/* GEMM grouping on host (replaces group_gemms + padding_overhead):
 * sizes[n] -> order (non-empty offsets in the chosen order, *n_order entries), groups as
 * [group_begin[g], group_end[g]) over `order` with padded heights[g] (*n_groups), per-offset
 * buffer_offsets[n] (-1 when n_k = 0), *buffer_length, *overhead (x / y; -1 when y = 0).
 * Output arrays hold n entries. */
sconv_status sconv_plan_groups(const int64_t* sizes, int n, int policy, double epsilon, int max_batch, int* order,
                               int* n_order, int* group_begin, int* group_end, int64_t* heights, int* n_groups,
                               int64_t* buffer_offsets, int64_t* buffer_length, double* overhead);

/* ---------------- network driver (SPEC netdef) ----------------
 * An op list over tensor ids, 12 int32 fields per op:
 *   {kind, out, in, b_or_target, K, offset_scale, out_stride, transposed, c_in, c_out, weight_id, relu}
 * kind 1 = CONV (SC layer; transposed convs take the target tensor's coordinates),
 * kind 2 = ADD (out = [relu](in + b)), kind 3 = CONCAT (out = [in | b] along channels).
 * forward_network's sequential chain is the special case of CONV-only ops;
 * U-Net skips / residual blocks (BASELINE configs 2-5) use ADD and CONCAT. Kernel maps are
 * cached per (input coordinates, K, offset scale, stride, transposed, target) within a forward. */
typedef struct sconv_net sconv_net;
sconv_status sconv_net_create(sconv_ctx* ctx, const int32_t* ops, int n_ops, int num_tensors, int input_tensor,
                              int output_tensor, const sconv_exec_cfg* cfg, int block_B, int block_C,
                              sconv_net** out);
/* Weights of CONV ops with this weight_id: fp32 [num_offsets][c_in][c_out] in `mem`. */
sconv_status sconv_net_set_weights(sconv_ctx* ctx, sconv_net* net, int weight_id, const float* w, int mem,
                                   int num_offsets, int c_in, int c_out);
/* Runs the graph on a cloud (xyz n x 3 int32 + fp32 features n x c_in). Asynchronous apart
 * from one sync per distinct kernel map. */
sconv_status sconv_net_forward(sconv_ctx* ctx, sconv_net* net, const int32_t* xyz, int64_t n, int mem, int in_sorted,
                               const float* feats, int f_mem, int c_in);
/* Queues the host->device copy of the NEXT request's host inputs (coordinates n x 3 int32, fp32
 * features n x c_in; f_mem host or device) on the net's input stream now, so that it overlaps
 * the current request's forward; the sconv_net_forward call with the same pointers, n, f_mem
 * and c_in then uses the staged copy (one pending prefetch; the host buffers must not change
 * before that forward). */
sconv_status sconv_net_prefetch_inputs(sconv_ctx* ctx, sconv_net* net, const int32_t* xyz, int64_t n,
                                       const float* feats, int f_mem, int c_in);
sconv_status sconv_net_tensor_info(sconv_ctx* ctx, const sconv_net* net, int tensor, int64_t* n, int* channels,
                                   int* coordset);
/* Host readback: coordinates (n x 3, sorted unless the tensor is the unsorted raw input) and fp32
 * features (activations are stored in the compute dtype and widened on device). A tensor whose
 * producing conv was folded into a residual epilogue (cfg.fuse_residual) returns SCONV_ERR_STATE. */
sconv_status sconv_net_read_tensor(sconv_ctx* ctx, const sconv_net* net, int tensor, int32_t* xyz, float* feats);
/* Device view of a tensor's features: pointer, dtype (sconv_dtype) and row stride in elements
 * (valid until the next forward). */
sconv_status sconv_net_tensor_device(const sconv_net* net, int tensor, const void** feats, int* dtype, int64_t* ld);
/* Copy a tensor's features (n x channels, dense rows) into a caller buffer, converted to
 * dst_dtype (sconv_dtype). Device destination: asynchronous on the context stream (e.g. a
 * per-scene result slot that a scene-sharded runner sends to rank 0 while the next scene
 * runs); host destination: synchronous. */
sconv_status sconv_net_copy_tensor(sconv_ctx* ctx, const sconv_net* net, int tensor, void* dst, int dst_dtype,
                                   int dst_mem);
/* Asynchronous host readback of a tensor's fp32 features (the serving form of
 * sconv_net_read_tensor's feature half): the widening runs on the context stream into one of two
 * net-owned device staging buffers, the device->host copy on the net's own copy stream, so the
 * copy of forward i's result overlaps forward i+1's kernels. `feats` (n x channels fp32, pinned
 * for a truly asynchronous copy) must stay untouched until sconv_net_read_wait returns. */
sconv_status sconv_net_read_async(sconv_ctx* ctx, sconv_net* net, int tensor, float* feats);
/* Blocks until every sconv_net_read_async of this net has landed in host memory. */
sconv_status sconv_net_read_wait(sconv_ctx* ctx, sconv_net* net);
sconv_status sconv_net_stats(const sconv_net* net, int* maps_built, int* convs);
/* Coordinate-array sorts of the last forward: 1 for an unsorted input (0 when flagged sorted)
 * plus one Eq. 1 sort per distinct strided map; stride-1 layers reuse the sorted keys
 * (acceptance #7: a 5-layer stride-1 chain sorts once, strides [1,2,1,2,1]
 * three times). */
sconv_status sconv_net_sort_count(const sconv_net* net, int64_t* sorts);
/* Per CONV op (execution order) of the last forward: {n_in, n_out, |M|, R_pad (0 if fused), c_in, c_out,
 * k_pad, K3, dataflow, residual_folded}. */
sconv_status sconv_net_conv_stats(const sconv_net* net, int conv, int64_t* out10);
/* Fills in |M| (out10[2], -1 for maps built lazily by the forward) of the last forward's convs:
 * builds the canonical lists of those maps (synchronises; statistics only). */
sconv_status sconv_net_resolve_stats(sconv_ctx* ctx, sconv_net* net);
/* AUTO dataflow measurements of the tuning forward for op index `op` (ms; -1 when the op was
 * not tuned): Minuet GMaS vs the fused kernel. */
sconv_status sconv_net_conv_timings(const sconv_net* net, int op, double* gmas_ms, double* fused_ms);
/* autotune_network(layers, dataset sample, R) (Alg. 2): runs the network on each
 * of the n_samples clouds (host xyz n_i x 3 int32, sorted[i], fp32 features n_i x c_in); at every
 * CONV op profiles each candidate gather tile (supported divisors of C_in) and scatter tile
 * (divisors of C_out) of the GMaS dataflow, 1 warm-up + `rounds` measured runs, median of the
 * kernel's CUDA-event times; medians are summed over the samples and the argmin
 * (smallest tile on ties) is kept for the network's later GMaS convs. tiles_out
 * (optional, 2 per op): {T_g, T_s}, 0 for non-CONV ops. Errors: n_samples < 1 -> ARG
 * ("sample must be nonempty"), rounds < 1 -> ARG. Tuning time is outside any benchmark. */
sconv_status sconv_net_autotune(sconv_ctx* ctx, sconv_net* net, int n_samples, const int32_t* const* xyz,
                                const int64_t* n, const int* sorted, const float* const* feats, int c_in, int rounds,
                                int* tiles_out);
/* TunedLayerConfig.latencies of op `op` from the last autotune: summed medians (ms) per candidate,
 * gather candidates then scatter candidates, ascending tiles. tiles/ms hold `cap` entries;
 * *n_gather / *n_scatter receive the candidate counts. */
sconv_status sconv_net_tune_latencies(const sconv_net* net, int op, int* tiles, double* ms, int cap, int* n_gather,
                                      int* n_scatter);
void sconv_net_free(sconv_ctx* ctx, sconv_net* net);

/* ---------------- voxelization (the step before the path) ----------------
 * Replaces voxelize(points, features, resolution) (proj/include/sconv/geometry.hpp:180-255), bit
 * for bit: voxel = floor(p / resolution) in double; duplicates merged by the mean of their
 * feature rows accumulated in double in the reference's canonical order (point coordinates,
 * then feature values); output sorted by packed key. points: n x 3 double; feats: n x channels
 * float (channels may be 0, feats NULL); out_xyz (n x 3) / out_feats (n x channels) sized for
 * n voxels, in out_mem. Errors: "resolution must be positive" (ARG), "voxel index <a> out of
 * range" (RANGE) for the first offending point in input order. */
sconv_status sconv_voxelize(sconv_ctx* ctx, const double* points, int64_t n, int points_mem, const float* feats,
                            int64_t channels, int feats_mem, double resolution, int32_t* out_xyz, float* out_feats,
                            int out_mem, int64_t* n_voxels);

/* ---------------- point-cloud files (SURVEY §8f rank 3 "ingestion") ----------------
 * ".mpc" binary: magic "MPC1", little-endian u32 N, u32 C, N x 3 int32 voxel coordinates, N x C
 * float32 features. ".xyz" text: one point per line "x y z f1 ... fC" (whitespace-separated
 * decimals; blank lines and '#' comments skipped; every line the same column count).
 * sconv_cloud_file_info detects the format (a ".mpc" name or the MPC1 magic) and returns N and C (parses a whole
 * .xyz file); the read calls take buffers of exactly that shape (host memory). Errors are ARG
 * with "mpc parse error at offset <o>: ..." / "xyz parse error at line <l>: ...". An .xyz
 * cloud is float points (voxelize it with sconv_voxelize); an .mpc cloud is already voxels. */
enum sconv_file_format { SCONV_FILE_MPC = 0, SCONV_FILE_XYZ = 1 };
sconv_status sconv_cloud_file_info(const char* path, int* format, int64_t* n, int64_t* channels);
sconv_status sconv_mpc_read(const char* path, int32_t* xyz, float* feats, int64_t n, int64_t channels);
sconv_status sconv_mpc_write(const char* path, const int32_t* xyz, const float* feats, int64_t n, int64_t channels);
sconv_status sconv_xyz_read(const char* path, double* points, float* feats, int64_t n, int64_t channels);
sconv_status sconv_xyz_write(const char* path, const double* points, const float* feats, int64_t n, int64_t channels);

/* ---------------- utilities (cli gen) ----------------
 * N unique coordinates uniform in [0,E)^3 from Rng(stream_seed(seed,0)) (x,y,z order,
 * duplicates rejected), then N x C features U[0,1) from the same stream. Host buffers. */
sconv_status sconv_generate_synthetic(int64_t N, int64_t E, int64_t C, uint64_t seed, int32_t* xyz, float* feats);
/* WeightSet from Rng(stream_seed(seed, stream)), U[-0.1, 0.1], order [k][cin][cout]. */
sconv_status sconv_generate_weights(uint64_t seed, uint64_t stream, int num_offsets, int c_in, int c_out, float* w);
/* Thread-independent last error (for failures before a context exists). */
const char* sconv_global_last_error(void);
const char* sconv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SCONV_B200_H_ */

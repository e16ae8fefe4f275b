// Device-resident kernel map (the product's KernelMap).
#pragma once

#include <functional>
#include <memory>
#include <vector>

#include "ctx.hpp"

namespace sconvb {

struct MapData {
  int64_t n_in = 0, n_out = 0;
  int K3 = 0;
  sconv_map_cfg cfg{};
  // sorted source (P) keys and original indices (null idx = identity, P was sorted)
  std::shared_ptr<DevBuf> src_keys;
  DevBuf src_idx;
  bool src_identity = true;
  // sorted output (Q) keys; aliases src_keys for stride 1 (geometry.hpp:163)
  std::shared_ptr<DevBuf> q_keys;
  DevBuf map_start;  // int32 x (K3 + 1): canonical list starts
  DevBuf pair_in, pair_out;  // int32 x |M|, canonical order (k, then i)
  DevBuf nbr_pos;            // int32 x K3 x n_out: canonical position m of (k, i) or -1
  DevBuf nbr_in;             // int32 x K3 x n_out: input row j of (k, i) or -1 (fused dataflow)
  std::vector<int3> delta;   // search offsets (host copy)
  DevBuf hash_keys, hash_vals;  // hash backend index, kept for inspection
  DevBuf delta_dev;             // explicit offset list (SPEC build_kernel_map_sorted(P, Q, offsets, B, C))
  DevBuf counters;              // SORTED_SPEC backend: u64 {backward, forward, loaded, executed}
  bool counted = false;
  int sorts = 0;                // coordinate sorts this build performed (acceptance #7)
  // Fused-dataflow row order (built lazily, conv_fused.cu prepare_fused_layout): output rows
  // sorted by their neighbour bitmask so a 128-row tile touches few offsets.
  bool fused_ready = false;
  bool permuted = false;     // false: identity order (nbr_perm unused, nbr_in is read directly)
  DevBuf row_perm;           // int32 x n_out: tile row r -> output row
  DevBuf nbr_perm;           // int32 x K3 x n_out: nbr_in[k][row_perm[r]]
  // Fused work items (conv_fused.cu build_fused_items, once per map): each 128-row tile's mask
  // of active offsets and the work items {tile, first offset rank, offset count, part | parts << 8}
  // in descending density; tiles with more active offsets than the per-item cap are split into
  // near-equal offset ranges whose fp32 partials are summed in part order by the last to finish.
  bool items_ready = false;
  DevBuf tile_mask, items, item_ws, n_items, item_counters;
  int64_t max_items = 0, max_ws_slots = 0;
  std::vector<int64_t> sizes;      // n_k (host)
  std::vector<int32_t> starts;     // map_start (host copy)
  int64_t total = 0;
  // Canonical pair lists (scan + emit + one readback sync) are built lazily for network maps:
  // the fused dataflow needs only nbr_in (ensure_canonical() before using sizes/pairs/nbr_pos).
  bool canonical = true;
  bool flags_deferred = false;  // build_map(defer_flags): coordinate checks pending at the caller
  DevBuf pend_nsel;             // coords_only builds: |Q| on the device until finish_coords
  bool identity_pending = false;
  int mask_bits_hint = 0;        // fused row order's key width chosen by the caller (0: default rule)
  bool layout_off_path = false;  // fused row order built beside the convs (network layout stream)  // lazy 1x1 identity map: arrays not yet written (nbr_in[i] = i)
  struct Pending {
    DevBuf counts, offs, tiles, flags;
    int64_t nchunk = 0, grid = 0, ntiles = 0;
    int ngroups = 0, qpl = 0;
    bool flags_init = false;  // k_init_flags ran on `flags`
    int64_t max_pairs = 0;    // pair-list capacity (allocated by the canonical build)
    bool counts_from_nbr = false;  // derived map: chunk counts computed from the table on demand
  } pending;
  // last GMaS stats
  int64_t buffer_length = 0;
  int groups = 0;
  double padding_overhead = 0.0;
  int gather_tile = 0, scatter_tile = 0;

  const uint64_t* src_keys_ptr() const { return src_keys ? src_keys->get<uint64_t>() : nullptr; }
  const uint64_t* q_keys_ptr() const { return q_keys ? q_keys->get<uint64_t>() : nullptr; }
};

// Build from coordinates (host or device) or from a sorted device key array.
struct MapSource {
  const int32_t* xyz = nullptr;  // n x 3
  int mem = SCONV_MEM_HOST;
  bool sorted = false;
  std::shared_ptr<DevBuf> keys;  // alternative: sorted device keys (chained layers)
  int64_t n = 0;
};

// lazy: skip the canonical lists and the end-of-build sync (only for maps over existing sorted
// device keys, whose coordinates were validated when they were first built).
// explicit_offsets: SPEC build_kernel_map_sorted(P, Q, offsets, B, C) with an arbitrary offset
// list and Q = *target (sorted unique queries).
std::unique_ptr<MapData> build_map(Ctx& ctx, const MapSource& P, const sconv_map_cfg& cfg, const MapSource* target,
                                   bool force_wide = false, bool lazy = false,
                                   const std::vector<int3>* explicit_offsets = nullptr, void* defer_flags = nullptr,
                                   bool coords_only = false, const MapSource* strided_q = nullptr,
                                   cudaEvent_t src_ready = nullptr,
                                   const std::function<void(const std::shared_ptr<DevBuf>&)>& on_src_ready = {});
// coords_only: a strided map over existing sorted keys queues only its Eq. 1 output coordinates
// (floor / sort / unique) and returns without a sync (n_out = -1); finish_coords then reads |Q|
// and the flags (one sync on the build's stream; false: the compact-key path overflowed, rebuild
// normally). strided_q: the strided map's Eq. 1 output computed that way (no second sort).
// src_ready: recorded on the build stream once the sorted source keys exist (before the search);
// on_src_ready is called right after that (host), before the search is queued.
bool finish_coords(Ctx& ctx, MapData& m);
// Derived network maps (no search), exact by construction where net.cu uses them:
// derive_down_map: K = 2, stride 2s map of P (on the s-lattice) onto Q = Eq. 1 of P;
// derive_transposed_map: the transposed map (P = fwd's output set, T = fwd's input set) from
// its forward map fwd, pairs swapped.
std::unique_ptr<MapData> derive_down_map(Ctx& ctx, const MapSource& P, const MapSource& Q, const sconv_map_cfg& cfg);
std::unique_ptr<MapData> derive_transposed_map(Ctx& ctx, const MapData& fwd, const MapSource& P, const MapSource& T,
                                               const sconv_map_cfg& cfg);
// defer_flags (pinned host, >= kDeferredFlagsBytes): a map over SORTED raw coordinates (no sort
// fallback exists) skips its flags sync; the flags are copied there asynchronously on the build
// stream and the caller checks them with check_deferred_map_flags once that copy completed
// (networks: at the end of the forward, after every launch is queued).
constexpr size_t kDeferredFlagsBytes = 128;
void check_deferred_map_flags(const void* flags_host, const MapSource& P);
// Builds the canonical pair lists of a lazily built map (no-op otherwise): scan + emit + sync.
void ensure_canonical(Ctx& ctx, MapData& m);

// Weight offsets (reference weight_offsets + SURVEY §2.2 even-K extension), lexicographic.
std::vector<int3> weight_offsets_ext(int K, int scale);

}  // namespace sconvb

struct sconv_map : sconvb::MapData {};

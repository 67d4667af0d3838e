// api.cpp -- host side of the C ABI (include/kvq.h): argument validation, the chunk -> slot map
// with sink / window eviction, K_eff resolution into cache segments, and kernel launches.
// No device memory is allocated here; the caller owns the arena.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <set>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/kvq.h"
#include "../../include/kvq_debug.h"
#include "internal.h"

using namespace kvq;

namespace {

constexpr size_t kAlign = 256;
size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Layout {
  int64_t T_c, T_pad, rows_per_head;  // rows_per_head = slots * T_pad
  size_t codes_bytes, scales_bytes;   // per tensor (K or V), all layers
  size_t off_codes[2], off_scales[2], off_g, off_partials, off_status, off_counters, off_ws, off_apsync, total;
  size_t off_mean, mean_bytes;        // K-smoothing row means [L][H][rows_per_head] fp32 (0 if off)
};

bool valid_cfg(const kvq_config* c) {
  if (!c) return false;
  if (c->num_layers <= 0 || c->num_heads <= 0) return false;
  if (c->head_dim != 64 && c->head_dim != 128) return false;
  if (c->tokens_per_frame <= 0 || c->frames_per_chunk <= 0) return false;
  if (c->sink_frames < 0 || c->window_frames < c->frames_per_chunk) return false;
  if (c->max_chunk_slots <= 0) return false;
  if ((c->scale_mode != 0 && c->scale_mode != 1) || (c->k_smoothing != 0 && c->k_smoothing != 1)) return false;
  int64_t Tc = (int64_t)c->tokens_per_frame * c->frames_per_chunk;
  if (Tc > (1 << 24)) return false;
  return true;
}

Layout make_layout(const kvq_config* c) {
  Layout L{};
  L.T_c = (int64_t)c->tokens_per_frame * c->frames_per_chunk;
  L.T_pad = (L.T_c + kTileKeys - 1) / kTileKeys * kTileKeys;
  L.rows_per_head = (int64_t)c->max_chunk_slots * L.T_pad;
  const int64_t rows = (int64_t)c->num_layers * c->num_heads * L.rows_per_head;
  L.codes_bytes = align_up((size_t)rows * (c->head_dim / 2), kAlign);
  L.scales_bytes = align_up((size_t)rows * (c->head_dim / 16), kAlign);
  size_t off = 0;
  L.off_codes[0] = off; off += L.codes_bytes;
  L.off_codes[1] = off; off += L.codes_bytes;
  L.off_scales[0] = off; off += L.scales_bytes;
  L.off_scales[1] = off; off += L.scales_bytes;
  L.off_g = off; off += align_up((size_t)c->num_layers * c->max_chunk_slots * 2 * sizeof(float), kAlign);
  L.off_partials = off; off += align_up(2 * kNumPartials * sizeof(uint32_t), kAlign);
  L.off_status = off; off += align_up(sizeof(DevStatus), kAlign);
  L.off_counters = off;  // grid-barrier slots of the single-pass quantizer: [CTA][K|V] u64
  off += align_up((size_t)kMaxFusedCtas * kSlotU64 * sizeof(unsigned long long), kAlign);
  L.off_ws = off; off += align_up(attn_ws_bytes(c->head_dim), kAlign);
  L.off_apsync = off; off += align_up(kApSyncWords * sizeof(unsigned long long), kAlign);  // fused append
  L.mean_bytes = c->k_smoothing ? align_up((size_t)rows * sizeof(float), kAlign) : 0;
  L.off_mean = off; off += L.mean_bytes;
  L.total = off;
  return L;
}

struct LayerState {
  int64_t newest = -1;
  std::map<int64_t, int> slot_of;  // resident chunk -> slot
  std::vector<int64_t> chunk_in;   // slot -> chunk (-1 free)
};

}  // namespace

struct kvq_cache {
  kvq_config cfg;
  Layout L;
  uint8_t* arena;
  std::vector<LayerState> layers;
  int64_t shot_start = 0, shot_len = 0;
  bool two_pass_only = false;  // debug: force the amax + quantize two-pass path
};

namespace {

kvq_status cuda_status(cudaError_t e) { return e == cudaSuccess ? KVQ_OK : KVQ_ECUDA; }

extern "C" unsigned long long* kvq_trace_ptr();

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      n = v;
    else
      n = kMaxCtas;
  }
  return n;
}
cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

uint8_t* codes_base(const kvq_cache* c, int t, int layer) {
  return c->arena + c->L.off_codes[t] + (size_t)layer * c->cfg.num_heads * c->L.rows_per_head * (c->cfg.head_dim / 2);
}
uint8_t* scales_base(const kvq_cache* c, int t, int layer) {
  return c->arena + c->L.off_scales[t] + (size_t)layer * c->cfg.num_heads * c->L.rows_per_head * (c->cfg.head_dim / 16);
}
float* g_base(const kvq_cache* c, int layer) {
  return reinterpret_cast<float*>(c->arena + c->L.off_g) + (size_t)layer * c->cfg.max_chunk_slots * 2;
}
// K-smoothing row means of (layer, head 0, slot 0), head-major like the scales; null when off
float* mean_base(const kvq_cache* c, int layer) {
  if (!c->cfg.k_smoothing) return nullptr;
  return reinterpret_cast<float*>(c->arena + c->L.off_mean) + (size_t)layer * c->cfg.num_heads * c->L.rows_per_head;
}
int quant_mode(const kvq_cache* c) {
  return (c->cfg.scale_mode == 1 ? kModeSearch : 0) | (c->cfg.k_smoothing ? kModeSmoothK : 0);
}
DevStatus* status_ptr(const kvq_cache* c) { return reinterpret_cast<DevStatus*>(c->arena + c->L.off_status); }

kvq_status reset_device(kvq_cache* c, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(c->arena, 0, c->L.total, st);
  if (e != cudaSuccess) return KVQ_ECUDA;
  // the grid-barrier slots and the device launch epoch were zeroed with the arena
  DevStatus init{0, 0, ~0ull};
  // status word: code 0, first_bad = max (a small H2D copy from a static host value)
  static DevStatus s_init = init;
  e = cudaMemcpyAsync(status_ptr(c), &s_init, sizeof(DevStatus), cudaMemcpyHostToDevice, st);
  return cuda_status(e);
}

// Frames of K_eff(t) (readings Z9-Z11) -> sorted distinct chunk-local token ranges
// in logical token coordinates.
std::vector<std::pair<int64_t, int64_t>> key_token_ranges(int64_t t, int64_t fc, int64_t tpf, int64_t sink,
                                                          int64_t window, int64_t shot0, int64_t shotn) {
  const int64_t f_end = (t + 1) * fc;
  std::vector<std::pair<int64_t, int64_t>> fr;  // frame intervals
  fr.push_back({0, std::min(sink, f_end)});
  if (shotn > 0) fr.push_back({std::max<int64_t>(shot0, 0), std::min(shot0 + shotn, f_end)});
  fr.push_back({std::max<int64_t>(0, f_end - window), f_end});
  fr.push_back({f_end - fc, f_end});
  std::sort(fr.begin(), fr.end());
  std::vector<std::pair<int64_t, int64_t>> out;
  for (auto& iv : fr) {
    if (iv.second <= iv.first) continue;
    if (!out.empty() && iv.first <= out.back().second) out.back().second = std::max(out.back().second, iv.second);
    else out.push_back(iv);
  }
  for (auto& iv : out) {
    iv.first *= tpf;
    iv.second *= tpf;
  }
  return out;
}

// chunks touched by the ranges
std::set<int64_t> chunks_of(const std::vector<std::pair<int64_t, int64_t>>& r, int64_t Tc) {
  std::set<int64_t> s;
  for (auto& iv : r)
    for (int64_t c = iv.first / Tc; c * Tc < iv.second; ++c) s.insert(c);
  return s;
}

kvq_status resolve_segments(const kvq_cache* c, int layer, const kvq_mask* m, std::vector<AttnSeg>& segs) {
  const LayerState& ls = c->layers[layer];
  auto ranges = key_token_ranges(m->chunk_index, c->cfg.frames_per_chunk, c->cfg.tokens_per_frame, m->sink_frames,
                                 m->window_frames, m->shot_start_frame, m->shot_len_frames);
  const int64_t Tc = c->L.T_c;
  segs.clear();
  for (auto& iv : ranges) {
    int64_t tok = iv.first;
    while (tok < iv.second) {
      const int64_t ch = tok / Tc;
      const int64_t end = std::min(iv.second, (ch + 1) * Tc);
      auto it = ls.slot_of.find(ch);
      if (it == ls.slot_of.end()) return KVQ_ENOCHUNK;
      if ((int)segs.size() >= kMaxSegs) return KVQ_EINVAL;
      segs.push_back(AttnSeg{it->second, (int32_t)(tok - ch * Tc), (int32_t)(end - ch * Tc)});
      tok = end;
    }
  }
  return KVQ_OK;
}

// Slot of (layer, chunk) under the append policy: chunk == newest re-writes its slot (a denoising
// step); chunk == newest + 1 evicts what K_eff of this and later steps can no longer reach (the
// global sink, the bound shot sink and the window ending at the new chunk) and
// takes a slot that is free once those are gone; anything else is KVQ_ENOCHUNK.  Pure: the
// evictions are returned in *evict and applied by commit_slot, after the launch succeeded, so an
// error (KVQ_ECAPACITY, KVQ_ECUDA) leaves the layer's chunk map untouched.
struct SlotPlan {
  int slot = -1;
  std::vector<int64_t> evict;
};
static kvq_status select_slot(const kvq_cache* c, int32_t layer, int64_t chunk, SlotPlan* plan) {
  const LayerState& ls = c->layers[layer];
  plan->slot = -1;
  plan->evict.clear();
  if (ls.newest >= 0 && chunk == ls.newest) {
    plan->slot = ls.slot_of.at(chunk);
  } else if (ls.newest < 0 || chunk == ls.newest + 1) {
    auto keep = chunks_of(key_token_ranges(chunk, c->cfg.frames_per_chunk, 1, c->cfg.sink_frames,
                                           c->cfg.window_frames, c->shot_start, c->shot_len),
                          c->cfg.frames_per_chunk);
    std::vector<char> freed(c->cfg.max_chunk_slots, 0);
    for (auto& kv : ls.slot_of)
      if (!keep.count(kv.first)) {
        plan->evict.push_back(kv.first);
        freed[kv.second] = 1;
      }
    for (int s = 0; s < c->cfg.max_chunk_slots; ++s)
      if (ls.chunk_in[s] < 0 || freed[s]) { plan->slot = s; break; }
    if (plan->slot < 0) return KVQ_ECAPACITY;
  } else {
    return KVQ_ENOCHUNK;
  }
  return KVQ_OK;
}

static void commit_slot(kvq_cache* c, int32_t layer, int64_t chunk, const SlotPlan& plan) {
  LayerState& ls = c->layers[layer];
  for (int64_t e : plan.evict) {
    auto it = ls.slot_of.find(e);
    if (it == ls.slot_of.end()) continue;
    ls.chunk_in[it->second] = -1;
    ls.slot_of.erase(it);
  }
  ls.slot_of[chunk] = plan.slot;
  ls.chunk_in[plan.slot] = chunk;
  ls.newest = chunk;
}

kvq_status append_impl(kvq_cache* c, int32_t layer, int64_t chunk, const void* K, const void* V, kvq_dtype dt,
                       const float* ext_amax, void* stream) {
  if (!c || !K || !V) return KVQ_EINVAL;
  if (layer < 0 || layer >= c->cfg.num_layers || chunk < 0) return KVQ_EINVAL;
  if (dt != KVQ_BF16 && dt != KVQ_FP32) return KVQ_EDTYPE;
  SlotPlan plan;
  const kvq_status ss = select_slot(c, layer, chunk, &plan);
  if (ss != KVQ_OK) return ss;
  const int slot = plan.slot;
  const int H = c->cfg.num_heads, d = c->cfg.head_dim;
  const int64_t rows = c->L.T_c * H;
  cudaStream_t st = S(stream);
  uint32_t* partials = reinterpret_cast<uint32_t*>(c->arena + c->L.off_partials);
  QuantParams p{};
  p.x[0] = K;
  p.x[1] = V;
  p.dtype = dt == KVQ_BF16 ? DT_BF16 : DT_FP32;
  p.rows = (int)rows;
  p.H = H;
  p.d = d;
  for (int t = 0; t < 2; ++t) {
    p.codes[t] = codes_base(c, t, layer) + (size_t)slot * c->L.T_pad * (d / 2);
    p.scales[t] = scales_base(c, t, layer) + (size_t)slot * c->L.T_pad * (d / 16);
  }
  p.head_stride_rows = c->L.rows_per_head;
  p.g_out = g_base(c, layer) + slot * 2;
  p.partials = ext_amax ? nullptr : partials;
  p.ext_amax = ext_amax;
  p.status = status_ptr(c);
  p.trace = kvq_trace_ptr();
  p.mode = quant_mode(c);
  p.mean_out = c->cfg.k_smoothing ? mean_base(c, layer) + (size_t)slot * c->L.T_pad : nullptr;
  p.partials_w = partials;
  // amax supplied (no smoothing): the streaming quantize pass alone (10.7 us on the Wan chunk against
  // 13.0 us for the single-pass kernel, which stages the whole chunk before quantizing).  Otherwise
  // single pass when the chunk fits in aggregate shared memory, else amax pass + quantize pass.
  if (ext_amax && !c->cfg.k_smoothing && !c->two_pass_only) {
    if (launch_quantize2(p, sm_count(), st) != cudaSuccess) return KVQ_ECUDA;
    commit_slot(c, layer, chunk, plan);
    return KVQ_OK;
  }
  cudaError_t e = c->two_pass_only ? cudaErrorNotSupported
                                   : launch_quantize_fused(p, reinterpret_cast<unsigned long long*>(c->arena + c->L.off_counters),
                                                           partials, sm_count(), st);
  if (e == cudaErrorNotSupported) {
    (void)cudaGetLastError();
    if (c->cfg.k_smoothing) {  // K row means (+ K_bar partials), then V's partials
      e = launch_smooth_amax(p, st);
      if (e == cudaSuccess && !ext_amax)
        e = launch_amax(K, V, dt == KVQ_BF16 ? DT_BF16 : DT_FP32, rows * d, partials, status_ptr(c), st, 1);
      if (e != cudaSuccess) return KVQ_ECUDA;
    } else if (!ext_amax) {
      e = launch_amax(K, V, dt == KVQ_BF16 ? DT_BF16 : DT_FP32, rows * d, partials, status_ptr(c), st);
      if (e != cudaSuccess) return KVQ_ECUDA;
    }
    e = launch_quantize2(p, sm_count(), st);
  }
  if (e != cudaSuccess) return KVQ_ECUDA;
  commit_slot(c, layer, chunk, plan);
  return KVQ_OK;
}

}  // namespace

// Dry run of append(chunk) + attend(mask) for the one-call Ulysses step (comm.cpp): every error the
// cache can raise (chunk not appendable, no free slot, a mask chunk not resident after the append's
// evictions, too many key segments) is found here, before the first collective is issued -- a rank
// that failed later would leave its peers blocked in the O all-to-all.
namespace kvq {
kvq_status validate_append_attend(const kvq_cache* c, int32_t layer, int64_t chunk, const kvq_mask* m) {
  if (!c || !m || layer < 0 || layer >= c->cfg.num_layers || chunk < 0 || m->chunk_index < 0) return KVQ_EINVAL;
  if (m->sink_frames < 0 || m->window_frames < 0 || m->shot_len_frames < 0) return KVQ_EINVAL;
  SlotPlan plan;
  kvq_status s = select_slot(c, layer, chunk, &plan);
  if (s != KVQ_OK) return s;
  std::set<int64_t> resident;
  for (auto& kv : c->layers[layer].slot_of) resident.insert(kv.first);
  for (int64_t e : plan.evict) resident.erase(e);
  resident.insert(chunk);
  auto ranges = key_token_ranges(m->chunk_index, c->cfg.frames_per_chunk, c->cfg.tokens_per_frame, m->sink_frames,
                                 m->window_frames, m->shot_start_frame, m->shot_len_frames);
  int nseg = 0;
  const int64_t Tc = c->L.T_c;
  for (auto& iv : ranges)
    for (int64_t ch = iv.first / Tc; ch * Tc < iv.second; ++ch) {
      if (!resident.count(ch)) return KVQ_ENOCHUNK;
      if (++nseg > kMaxSegs) return KVQ_EINVAL;
    }
  return KVQ_OK;
}
}  // namespace kvq

extern "C" {

size_t kvq_cache_bytes(const kvq_config* cfg) {
  if (!valid_cfg(cfg)) return 0;
  return make_layout(cfg).total;
}

kvq_status kvq_cache_create(const kvq_config* cfg, void* dev_arena, size_t arena_bytes, void* stream,
                            kvq_cache** out) {
  if (!out) return KVQ_EINVAL;
  *out = nullptr;
  if (!valid_cfg(cfg)) return (cfg && (cfg->head_dim != 64 && cfg->head_dim != 128)) ? KVQ_ESHAPE : KVQ_EINVAL;
  if (!dev_arena || (reinterpret_cast<uintptr_t>(dev_arena) % kAlign) != 0) return KVQ_EINVAL;
  Layout L = make_layout(cfg);
  if (arena_bytes < L.total) return KVQ_EINVAL;
  kvq_cache* c = new (std::nothrow) kvq_cache();
  if (!c) return KVQ_EINVAL;
  c->cfg = *cfg;
  c->L = L;
  c->arena = static_cast<uint8_t*>(dev_arena);
  c->layers.resize(cfg->num_layers);
  for (auto& ls : c->layers) ls.chunk_in.assign(cfg->max_chunk_slots, -1);
  kvq_status s = reset_device(c, S(stream));
  if (s != KVQ_OK) {
    delete c;
    return s;
  }
  *out = c;
  return KVQ_OK;
}

kvq_status kvq_cache_destroy(kvq_cache* cache) {
  delete cache;
  return KVQ_OK;
}

kvq_status kvq_cache_reset(kvq_cache* c, void* stream) {
  if (!c) return KVQ_EINVAL;
  for (auto& ls : c->layers) {
    ls.newest = -1;
    ls.slot_of.clear();
    ls.chunk_in.assign(c->cfg.max_chunk_slots, -1);
  }
  c->shot_start = c->shot_len = 0;
  return reset_device(c, S(stream));
}

kvq_status kvq_set_shot(kvq_cache* c, int64_t shot_start_frame, int64_t shot_len_frames) {
  if (!c || shot_start_frame < 0 || shot_len_frames < 0) return KVQ_EINVAL;
  c->shot_start = shot_start_frame;
  c->shot_len = shot_len_frames;
  return KVQ_OK;
}

kvq_status kv_quantize_append(kvq_cache* c, int32_t layer, int64_t chunk, const void* K, const void* V,
                              kvq_dtype dt, void* stream) {
  return append_impl(c, layer, chunk, K, V, dt, nullptr, stream);
}

kvq_status kv_quantize_append_amax(kvq_cache* c, int32_t layer, int64_t chunk, const void* K, const void* V,
                                   kvq_dtype dt, const float* dev_amax_kv, void* stream) {
  if (!dev_amax_kv) return KVQ_EINVAL;
  return append_impl(c, layer, chunk, K, V, dt, dev_amax_kv, stream);
}

struct AttnRoute {  // f4 direct: O rows into the owning ranks' O shards (AttnParams::o_peer)
  uint8_t* const* o_peer;
  int P, Ts, H, h0;
};
struct AttnAppend {  // chunk_attention_append: the chunk's K, V quantized inside the attention launch
  const void* K;
  const void* V;
  int dtype, slot;
};
static kvq_status attention_impl(kvq_cache* c, int32_t layer, const void* Q, kvq_dtype q_dtype, const float* q_scale,
                                 const kvq_mask* mask, float softmax_scale, void* O, kvq_dtype out_dtype, void* ws,
                                 size_t ws_bytes, void* stream, const AttnRoute* route = nullptr,
                                 const AttnAppend* app = nullptr);

kvq_status chunk_attention(kvq_cache* c, int32_t layer, const void* Q, kvq_dtype q_dtype, const kvq_mask* mask,
                           float softmax_scale, void* O, kvq_dtype out_dtype, void* stream) {
  if (q_dtype != KVQ_BF16 && q_dtype != KVQ_FP32) return KVQ_EDTYPE;
  return attention_impl(c, layer, Q, q_dtype, nullptr, mask, softmax_scale, O, out_dtype, nullptr, 0, stream);
}

size_t kvq_attention_workspace_bytes(const kvq_cache* c) { return c ? attn_ws_bytes(c->cfg.head_dim) : 0; }

kvq_status chunk_attention_ws(kvq_cache* c, int32_t layer, const void* Q, kvq_dtype q_dtype, const kvq_mask* mask,
                              float softmax_scale, void* O, kvq_dtype out_dtype, void* dev_workspace,
                              size_t workspace_bytes, void* stream) {
  if (q_dtype != KVQ_BF16 && q_dtype != KVQ_FP32) return KVQ_EDTYPE;
  if (!c || !dev_workspace || (reinterpret_cast<uintptr_t>(dev_workspace) % kAlign) != 0) return KVQ_EINVAL;
  if (workspace_bytes < kvq_attention_workspace_bytes(c)) return KVQ_EINVAL;
  return attention_impl(c, layer, Q, q_dtype, nullptr, mask, softmax_scale, O, out_dtype, dev_workspace,
                        workspace_bytes, stream);
}

kvq_status chunk_attention_append(kvq_cache* c, int32_t layer, int64_t chunk_index, const void* K, const void* V,
                                  kvq_dtype in_dtype, const void* Q, kvq_dtype q_dtype, const kvq_mask* mask,
                                  float softmax_scale, void* O, kvq_dtype out_dtype, void* dev_workspace,
                                  size_t workspace_bytes, void* stream) {
  if (!c || !K || !V || !Q || !O || !mask) return KVQ_EINVAL;
  if (in_dtype != KVQ_BF16 && in_dtype != KVQ_FP32) return KVQ_EDTYPE;
  if (q_dtype != KVQ_BF16 && q_dtype != KVQ_FP32) return KVQ_EDTYPE;
  if (out_dtype != KVQ_BF16 && out_dtype != KVQ_FP32) return KVQ_EDTYPE;
  if (mask->chunk_index != chunk_index) return KVQ_EINVAL;  // the call attends the chunk it appends
  if (dev_workspace && ((reinterpret_cast<uintptr_t>(dev_workspace) % kAlign) != 0 ||
                        workspace_bytes < kvq_attention_workspace_bytes(c)))
    return KVQ_EINVAL;
  const kvq_status v = validate_append_attend(c, layer, chunk_index, mask);  // host dry run: nothing launched on error
  if (v != KVQ_OK) return v;
  // fused only where it pays: plain NVFP4 (no 4/6 search, no K-smoothing), bf16 queries, and a key set
  // of which the appended chunk is at most half (the history tiles hide the append); else the two calls
  int64_t n_keys = 0;
  for (auto& iv : key_token_ranges(mask->chunk_index, c->cfg.frames_per_chunk, c->cfg.tokens_per_frame,
                                   mask->sink_frames, mask->window_frames, mask->shot_start_frame, mask->shot_len_frames))
    n_keys += iv.second - iv.first;
  // The fused launch is opt-in (environment KVQ_FUSED_APPEND=1): bit-exact and within tolerance, but
  // measured slower on the Wan layer (998-1031 us against 945 us for the two launches)
  const char* env = std::getenv("KVQ_FUSED_APPEND");
  const bool fuse = env != nullptr && env[0] == '1' && c->cfg.scale_mode == 0 && !c->cfg.k_smoothing &&
                    q_dtype == KVQ_BF16 && !c->two_pass_only && 2 * c->L.T_c <= n_keys;
  if (!fuse) {
    const kvq_status s = kv_quantize_append(c, layer, chunk_index, K, V, in_dtype, stream);
    if (s != KVQ_OK) return s;
    return dev_workspace ? chunk_attention_ws(c, layer, Q, q_dtype, mask, softmax_scale, O, out_dtype, dev_workspace,
                                              workspace_bytes, stream)
                         : chunk_attention(c, layer, Q, q_dtype, mask, softmax_scale, O, out_dtype, stream);
  }
  SlotPlan plan;
  const kvq_status ss = select_slot(c, layer, chunk_index, &plan);
  if (ss != KVQ_OK) return ss;
  commit_slot(c, layer, chunk_index, plan);  // the key set below includes the chunk being appended
  const AttnAppend app{K, V, in_dtype == KVQ_BF16 ? DT_BF16 : DT_FP32, plan.slot};
  return attention_impl(c, layer, Q, q_dtype, nullptr, mask, softmax_scale, O, out_dtype, dev_workspace,
                        workspace_bytes, stream, nullptr, &app);
}

kvq_status chunk_attention_qscaled(kvq_cache* c, int32_t layer, const void* Q_fp16, const float* dev_q_scale,
                                   const kvq_mask* mask, float softmax_scale, void* O, kvq_dtype out_dtype,
                                   void* stream) {
  if (!dev_q_scale) return KVQ_EINVAL;
  return attention_impl(c, layer, Q_fp16, KVQ_FP16, dev_q_scale, mask, softmax_scale, O, out_dtype, nullptr, 0,
                        stream);
}

static kvq_status attention_impl(kvq_cache* c, int32_t layer, const void* Q, kvq_dtype q_dtype, const float* q_scale,
                                 const kvq_mask* mask, float softmax_scale, void* O, kvq_dtype out_dtype, void* ws,
                                 size_t ws_bytes, void* stream, const AttnRoute* route, const AttnAppend* app) {
  (void)ws_bytes;
  if (!c || !Q || !O || !mask) return KVQ_EINVAL;
  if (layer < 0 || layer >= c->cfg.num_layers || mask->chunk_index < 0) return KVQ_EINVAL;
  if (mask->sink_frames < 0 || mask->window_frames < 0 || mask->shot_len_frames < 0) return KVQ_EINVAL;
  if (out_dtype != KVQ_BF16 && out_dtype != KVQ_FP32) return KVQ_EDTYPE;
  AttnParams p{};
  std::vector<AttnSeg> segs;
  kvq_status s = resolve_segments(c, layer, mask, segs);
  if (s != KVQ_OK) return s;
  p.nseg = (int)segs.size();
  std::copy(segs.begin(), segs.end(), p.seg);
  const int d = c->cfg.head_dim;
  p.Q = Q;
  p.q_dtype = q_dtype == KVQ_BF16 ? DT_BF16 : (q_dtype == KVQ_FP16 ? DT_FP16 : DT_FP32);
  p.q_scale = q_scale;
  p.O = O;
  p.out_dtype = out_dtype == KVQ_BF16 ? DT_BF16 : DT_FP32;
  p.mean_k = mean_base(c, layer);
  p.codes_k = codes_base(c, 0, layer);
  p.codes_v = codes_base(c, 1, layer);
  p.scales_k = scales_base(c, 0, layer);
  p.scales_v = scales_base(c, 1, layer);
  p.g = g_base(c, layer);
  p.head_stride_rows = c->L.rows_per_head;
  p.T_pad = (int)c->L.T_pad;
  p.Tq = (int)c->L.T_c;
  p.H = c->cfg.num_heads;
  p.d = d;
  const float sc = softmax_scale > 0.0f ? softmax_scale : 1.0f / std::sqrt((float)d);
  p.scale_log2 = sc * 1.4426950408889634f;
  p.status = status_ptr(c);
  // split-KV partials: the caller's workspace (chunk_attention_ws), else the cache's own
  p.ws = reinterpret_cast<float*>(ws ? static_cast<uint8_t*>(ws) : c->arena + c->L.off_ws);
  p.trace = kvq_trace_ptr();
  p.ws_slots = 2 * kMaxCtas;
  p.max_ctas = std::min(sm_count(), kMaxCtas);
  if (route) {
    for (int r = 0; r < route->P; ++r) p.o_peer[r] = route->o_peer[r];
    p.o_Ts = route->Ts;
    p.o_H = route->H;
    p.o_h0 = route->h0;
  }
  if (app) {
    p.ap_x[0] = app->K;
    p.ap_x[1] = app->V;
    p.ap_dtype = app->dtype;
    p.ap_slot = app->slot;
    for (int t = 0; t < 2; ++t) {
      p.ap_codes[t] = codes_base(c, t, layer) + (size_t)app->slot * c->L.T_pad * (d / 2);
      p.ap_scales[t] = scales_base(c, t, layer) + (size_t)app->slot * c->L.T_pad * (d / 16);
    }
    p.ap_g = g_base(c, layer) + app->slot * 2;
    p.ap_sync = reinterpret_cast<unsigned long long*>(c->arena + c->L.off_apsync);
    return cuda_status(launch_attention_append(p, S(stream)));
  }
  return cuda_status(launch_attention(p, true, S(stream)));
}

kvq_status kv_dequantize(const kvq_cache* c, int32_t layer, int64_t chunk, void* K_out, void* V_out,
                         kvq_dtype out_dtype, void* stream) {
  if (!c || !K_out || !V_out || layer < 0 || layer >= c->cfg.num_layers) return KVQ_EINVAL;
  if (out_dtype != KVQ_BF16 && out_dtype != KVQ_FP32) return KVQ_EDTYPE;
  auto it = c->layers[layer].slot_of.find(chunk);
  if (it == c->layers[layer].slot_of.end()) return KVQ_ENOCHUNK;
  const int slot = it->second, d = c->cfg.head_dim;
  DequantParams p{};
  for (int t = 0; t < 2; ++t) {
    p.codes[t] = codes_base(c, t, layer) + (size_t)slot * c->L.T_pad * (d / 2);
    p.scales[t] = scales_base(c, t, layer) + (size_t)slot * c->L.T_pad * (d / 16);
  }
  p.g = g_base(c, layer) + slot * 2;
  p.head_stride_rows = c->L.rows_per_head;
  p.T = (int)c->L.T_c;
  p.H = c->cfg.num_heads;
  p.d = d;
  p.mean = c->cfg.k_smoothing ? mean_base(c, layer) + (size_t)slot * c->L.T_pad : nullptr;
  p.out[0] = K_out;
  p.out[1] = V_out;
  p.out_dtype = out_dtype == KVQ_BF16 ? DT_BF16 : DT_FP32;
  return cuda_status(launch_dequantize(p, S(stream)));
}

kvq_status kv_export_chunk(const kvq_cache* c, int32_t layer, int64_t chunk, void* codes_k, void* scales_k,
                           float* g_k, void* codes_v, void* scales_v, float* g_v, void* stream) {
  if (!c || layer < 0 || layer >= c->cfg.num_layers) return KVQ_EINVAL;
  if (!codes_k || !scales_k || !g_k || !codes_v || !scales_v || !g_v) return KVQ_EINVAL;
  auto it = c->layers[layer].slot_of.find(chunk);
  if (it == c->layers[layer].slot_of.end()) return KVQ_ENOCHUNK;
  const int slot = it->second, d = c->cfg.head_dim;
  ExportParams p{};
  for (int t = 0; t < 2; ++t) {
    p.codes[t] = codes_base(c, t, layer) + (size_t)slot * c->L.T_pad * (d / 2);
    p.scales[t] = scales_base(c, t, layer) + (size_t)slot * c->L.T_pad * (d / 16);
  }
  p.g = g_base(c, layer) + slot * 2;
  p.head_stride_rows = c->L.rows_per_head;
  p.T = (int)c->L.T_c;
  p.H = c->cfg.num_heads;
  p.d = d;
  p.codes_out[0] = static_cast<uint8_t*>(codes_k);
  p.codes_out[1] = static_cast<uint8_t*>(codes_v);
  p.scales_out[0] = static_cast<uint8_t*>(scales_k);
  p.scales_out[1] = static_cast<uint8_t*>(scales_v);
  p.g_out[0] = g_k;
  p.g_out[1] = g_v;
  return cuda_status(launch_export(p, S(stream)));
}

kvq_status kv_export_kmean(const kvq_cache* c, int32_t layer, int64_t chunk, float* mean_out, void* stream) {
  if (!c || !mean_out || layer < 0 || layer >= c->cfg.num_layers) return KVQ_EINVAL;
  if (!c->cfg.k_smoothing) return KVQ_EINVAL;
  auto it = c->layers[layer].slot_of.find(chunk);
  if (it == c->layers[layer].slot_of.end()) return KVQ_ENOCHUNK;
  const int slot = it->second;
  ExportParams p{};
  p.head_stride_rows = c->L.rows_per_head;
  p.T = (int)c->L.T_c;
  p.H = c->cfg.num_heads;
  p.d = c->cfg.head_dim;
  p.mean = mean_base(c, layer) + (size_t)slot * c->L.T_pad;
  p.mean_out = mean_out;
  return cuda_status(launch_export(p, S(stream)));
}

size_t kvq_resident_bytes(const kvq_cache* c) {
  if (!c) return 0;
  size_t n = 0;
  const size_t rows = (size_t)c->L.T_c * c->cfg.num_heads;
  const size_t per_chunk = 2 * (rows * (c->cfg.head_dim / 2) + rows * (c->cfg.head_dim / 16) + sizeof(float)) +
                           (c->cfg.k_smoothing ? rows * sizeof(float) : 0);  // + K row means
  for (auto& ls : c->layers) n += ls.slot_of.size() * per_chunk;
  return n;
}

int32_t kvq_resident_chunks(const kvq_cache* c, int32_t layer) {
  if (!c || layer < 0 || layer >= c->cfg.num_layers) return -1;
  return (int32_t)c->layers[layer].slot_of.size();
}

kvq_status kv_dequantize_window(const kvq_cache* c, int32_t layer, const kvq_mask* mask, void* K_out, void* V_out,
                                int64_t* n_keys, void* stream) {
  if (!c || !mask || !n_keys || layer < 0 || layer >= c->cfg.num_layers) return KVQ_EINVAL;
  std::vector<AttnSeg> segs;
  kvq_status s = resolve_segments(c, layer, mask, segs);
  if (s != KVQ_OK) return s;
  int64_t n = 0;
  for (auto& sg : segs) n += sg.end - sg.begin;
  *n_keys = n;
  if (!K_out && !V_out) return KVQ_OK;
  if (!K_out || !V_out) return KVQ_EINVAL;
  const int d = c->cfg.head_dim;
  DequantParams p{};
  p.codes[0] = codes_base(c, 0, layer);
  p.codes[1] = codes_base(c, 1, layer);
  p.scales[0] = scales_base(c, 0, layer);
  p.scales[1] = scales_base(c, 1, layer);
  p.g = g_base(c, layer);
  p.mean = mean_base(c, layer);
  p.head_stride_rows = c->L.rows_per_head;
  p.T = (int)c->L.T_pad;
  p.H = c->cfg.num_heads;
  p.d = d;
  p.out_dtype = DT_BF16;
  return cuda_status(launch_dequant_window(p, segs.data(), (int)segs.size(), K_out, V_out, S(stream)));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda at link time)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// [n_keys][H][d] bf16 as a 3-D tensor (d innermost), box {64, 1, 128}: one 128-key x 64-column panel
// of the attention kernel's K-major SW128 tile per copy
static bool kv_tensor_map(CUtensorMap* m, const void* base, int64_t n_keys, int H, int d) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)H, (cuuint64_t)n_keys};
  const cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)H * d * 2};
  const cuuint32_t box[3] = {64, 1, 128}, estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t kvq_bf16kv_workspace_bytes(int32_t d) { return (d == 64 || d == 128) ? attn_ws_bytes(d) : 0; }

kvq_status chunk_attention_bf16kv_ws(const void* Q, const void* K, const void* V, int32_t T_q, int64_t n_keys,
                                     int32_t H, int32_t d, float softmax_scale, void* O, kvq_dtype out_dtype,
                                     void* dev_workspace, size_t workspace_bytes, void* stream) {
  if (!Q || !K || !V || !O || T_q <= 0 || n_keys <= 0 || H <= 0) return KVQ_EINVAL;
  if (d != 64 && d != 128) return KVQ_ESHAPE;
  if (n_keys > INT_MAX) return KVQ_ESHAPE;
  if (out_dtype != KVQ_BF16 && out_dtype != KVQ_FP32) return KVQ_EDTYPE;
  if (dev_workspace && ((reinterpret_cast<uintptr_t>(dev_workspace) % kAlign) != 0 ||
                        workspace_bytes < kvq_bf16kv_workspace_bytes(d)))
    return KVQ_EINVAL;
  AttnParams p{};
  if (!kv_tensor_map(&p.tmap_k, K, n_keys, H, d) || !kv_tensor_map(&p.tmap_v, V, n_keys, H, d)) return KVQ_EINVAL;
  p.Q = Q;
  p.q_dtype = DT_BF16;
  p.O = O;
  p.out_dtype = out_dtype == KVQ_BF16 ? DT_BF16 : DT_FP32;
  p.Kb = K;
  p.Vb = V;
  p.Tq = T_q;
  p.H = H;
  p.d = d;
  p.nseg = 1;
  p.seg[0] = AttnSeg{0, 0, (int32_t)n_keys};
  const float sc = softmax_scale > 0.0f ? softmax_scale : 1.0f / std::sqrt((float)d);
  p.scale_log2 = sc * 1.4426950408889634f;
  if (dev_workspace) {  // persistent grid: whole units in waves (L2 reuse of the bf16 window), stream-K remainder
    p.ws = static_cast<float*>(dev_workspace);
    p.ws_slots = 2 * kMaxCtas;
    p.max_ctas = std::min(sm_count(), kMaxCtas);
    p.hybrid = true;
  }
  return cuda_status(launch_attention(p, false, S(stream)));
}

kvq_status chunk_attention_bf16kv(const void* Q, const void* K, const void* V, int32_t T_q, int64_t n_keys, int32_t H,
                                  int32_t d, float softmax_scale, void* O, kvq_dtype out_dtype, void* stream) {
  return chunk_attention_bf16kv_ws(Q, K, V, T_q, n_keys, H, d, softmax_scale, O, out_dtype, nullptr, 0, stream);
}

kvq_status kvq_get_status(kvq_cache* c, void* stream, int64_t* first_bad_index) {
  if (!c) return KVQ_EINVAL;
  cudaStream_t st = S(stream);
  DevStatus h{};
  if (cudaMemcpyAsync(&h, status_ptr(c), sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess) return KVQ_ECUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return KVQ_ECUDA;
  if (first_bad_index) *first_bad_index = h.first_bad == ~0ull ? -1 : (int64_t)h.first_bad;
  if (h.code != 0) {
    static DevStatus s_init{0, 0, ~0ull};
    if (cudaMemcpyAsync(status_ptr(c), &s_init, sizeof(DevStatus), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return KVQ_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return KVQ_ECUDA;
  }
  return (kvq_status)h.code;
}

const char* kvq_strerror(kvq_status s) {
  switch (s) {
    case KVQ_OK: return "ok";
    case KVQ_EINVAL: return "invalid argument";
    case KVQ_ESHAPE: return "unsupported shape";
    case KVQ_EDTYPE: return "unsupported dtype";
    case KVQ_ENOCHUNK: return "chunk not appendable or not resident";
    case KVQ_ECAPACITY: return "no free cache slot";
    case KVQ_ENONFINITE: return "non-finite input";
    case KVQ_ERANGE: return "value out of range";
    case KVQ_ECUDA: return "CUDA error";
    case KVQ_ENCCL: return "NCCL error";
  }
  return "unknown status";
}

// ----------------------------------------------------------------------------- Ulysses
void kvq_head_partition(int32_t H, int32_t P, int32_t rank, int32_t* h0, int32_t* h1) {
  if (P <= 0 || rank < 0 || rank >= P || H < 0) {
    if (h0) *h0 = 0;
    if (h1) *h1 = 0;
    return;
  }
  const int32_t base = H / P, rem = H % P;
  const int32_t a = rank * base + std::min(rank, rem);
  if (h0) *h0 = a;
  if (h1) *h1 = a + base + (rank < rem ? 1 : 0);
}

static size_t esize(kvq_dtype d) { return d == KVQ_FP32 ? 4 : 2; }

size_t kvq_ulysses_qkv_bytes(int32_t Ts, int32_t H, int32_t d, int32_t P, int32_t dst, kvq_dtype dtype) {
  int32_t h0, h1;
  kvq_head_partition(H, P, dst, &h0, &h1);
  return 3 * (size_t)Ts * (h1 - h0) * d * esize(dtype) + 16;
}

kvq_status kvq_ulysses_pack_qkv(const void* Q, const void* K, const void* V, kvq_dtype dtype, int32_t Ts, int32_t H,
                                int32_t d, int32_t P, void* send_buf, void* dev_scratch, void* stream) {
  if (!Q || !K || !V || !send_buf || !dev_scratch || Ts <= 0 || H <= 0 || P <= 0 || P > 64) return KVQ_EINVAL;
  if (d != 64 && d != 128) return KVQ_ESHAPE;
  if (dtype != KVQ_BF16 && dtype != KVQ_FP32) return KVQ_EDTYPE;
  return cuda_status(launch_ulysses_pack(Q, K, V, dtype == KVQ_BF16 ? DT_BF16 : DT_FP32, Ts, H, d, P,
                                         static_cast<uint8_t*>(send_buf), static_cast<uint32_t*>(dev_scratch),
                                         S(stream)));
}

kvq_status kvq_ulysses_unpack_qkv(const void* recv_buf, kvq_dtype dtype, int32_t Ts, int32_t H_r, int32_t d, int32_t P,
                                  void* Q, void* K, void* V, float* dev_amax_kv, void* stream) {
  if (!recv_buf || !Q || !K || !V || !dev_amax_kv || Ts <= 0 || H_r <= 0 || P <= 0 || P > 64) return KVQ_EINVAL;
  if (d != 64 && d != 128) return KVQ_ESHAPE;
  if (dtype != KVQ_BF16 && dtype != KVQ_FP32) return KVQ_EDTYPE;
  return cuda_status(launch_ulysses_unpack_qkv(static_cast<const uint8_t*>(recv_buf), dtype == KVQ_BF16 ? DT_BF16 : DT_FP32,
                                               Ts, H_r, d, P, Q, K, V, dev_amax_kv, S(stream)));
}

kvq_status kvq_ulysses_unpack_o(const void* recv_buf, kvq_dtype dtype, int32_t Ts, int32_t H, int32_t d, int32_t P,
                                void* O_shard, void* stream) {
  if (!recv_buf || !O_shard || Ts <= 0 || H <= 0 || P <= 0 || P > 64) return KVQ_EINVAL;
  if (d != 64 && d != 128) return KVQ_ESHAPE;
  if (dtype != KVQ_BF16 && dtype != KVQ_FP32) return KVQ_EDTYPE;
  return cuda_status(launch_ulysses_unpack_o(static_cast<const uint8_t*>(recv_buf), dtype == KVQ_BF16 ? DT_BF16 : DT_FP32,
                                             Ts, H, d, P, O_shard, S(stream)));
}

// ---- NVFP4 payload exchange (§8(f) f3)
size_t kvq_ulysses_shard_scratch_bytes(int32_t Ts, int32_t H) {
  return 2 * kNumPartials * sizeof(uint32_t) + 64 + (size_t)Ts * H * sizeof(float);
}

size_t kvq_ulysses_nvfp4_bytes(int32_t Ts, int32_t H, int32_t d, int32_t P, int32_t dst, kvq_dtype q_dtype,
                               int32_t k_smoothing, int32_t q_nvfp4) {
  int32_t h0, h1;
  kvq_head_partition(H, P, dst, &h0, &h1);
  return (size_t)nvfp4_seg_layout(Ts, h1 - h0, d, (int)esize(q_dtype), k_smoothing != 0, q_nvfp4 != 0).total;
}

kvq_status kvq_ulysses_q_amax(const void* Q, kvq_dtype dtype, int32_t Ts, int32_t H, int32_t d, float* dev_amax_q,
                              void* dev_scratch, void* stream) {
  if (!Q || !dev_amax_q || !dev_scratch || Ts <= 0 || H <= 0) return KVQ_EINVAL;
  if (d != 64 && d != 128) return KVQ_ESHAPE;
  if (dtype != KVQ_BF16 && dtype != KVQ_FP32) return KVQ_EDTYPE;
  // amax kernels over (Q, Q): both reduced values are amax(Q); the first is kept
  uint8_t* sc = static_cast<uint8_t*>(dev_scratch);
  QuantParams p{};
  p.x[0] = Q;
  p.x[1] = Q;
  p.dtype = dtype == KVQ_BF16 ? DT_BF16 : DT_FP32;
  p.rows = Ts * H;
  p.H = H;
  p.d = d;
  p.status = reinterpret_cast<DevStatus*>(sc + 2 * kNumPartials * sizeof(uint32_t));
  float* two = reinterpret_cast<float*>(sc + 2 * kNumPartials * sizeof(uint32_t) + 32);
  cudaError_t e = launch_ulysses_shard_amax(p, reinterpret_cast<uint32_t*>(sc), two, S(stream));
  if (e == cudaSuccess) e = cudaMemcpyAsync(dev_amax_q, two, sizeof(float), cudaMemcpyDeviceToDevice, S(stream));
  return cuda_status(e);
}

kvq_status kvq_ulysses_shard_amax(const void* K, const void* V, kvq_dtype dtype, int32_t Ts, int32_t H, int32_t d,
                                  int32_t k_smoothing, float* dev_amax_kv, void* dev_scratch, void* stream) {
  if (!K || !V || !dev_amax_kv || !dev_scratch || Ts <= 0 || H <= 0) return KVQ_EINVAL;
  if (d != 64 && d != 128) return KVQ_ESHAPE;
  if (dtype != KVQ_BF16 && dtype != KVQ_FP32) return KVQ_EDTYPE;
  if (k_smoothing != 0 && k_smoothing != 1) return KVQ_EINVAL;
  uint8_t* sc = static_cast<uint8_t*>(dev_scratch);
  uint32_t* partials = reinterpret_cast<uint32_t*>(sc);
  DevStatus* status = reinterpret_cast<DevStatus*>(sc + 2 * kNumPartials * sizeof(uint32_t));
  QuantParams p{};
  p.x[0] = K;
  p.x[1] = V;
  p.dtype = dtype == KVQ_BF16 ? DT_BF16 : DT_FP32;
  p.rows = Ts * H;
  p.H = H;
  p.d = d;
  p.head_stride_rows = Ts;  // scratch means [H][Ts] (a by-product; the packer recomputes them)
  p.status = status;
  p.mode = k_smoothing ? kModeSmoothK : 0;
  p.mean_out = reinterpret_cast<float*>(sc + 2 * kNumPartials * sizeof(uint32_t) + 64);
  p.partials_w = partials;
  return cuda_status(launch_ulysses_shard_amax(p, partials, dev_amax_kv, S(stream)));
}

kvq_status kvq_ulysses_pack_nvfp4(const void* Q, const void* K, const void* V, kvq_dtype dtype, int32_t Ts, int32_t H,
                                  int32_t d, int32_t P, const float* dev_amax_kv, const float* dev_amax_q,
                                  int32_t scale_mode, int32_t k_smoothing, void* send_buf, void* stream) {
  if (!Q || !K || !V || !dev_amax_kv || !send_buf || Ts <= 0 || H <= 0 || H > 256 || P <= 0 || P > kMaxP)
    return KVQ_EINVAL;
  if (d != 64 && d != 128) return KVQ_ESHAPE;
  if (dtype != KVQ_BF16 && dtype != KVQ_FP32) return KVQ_EDTYPE;
  if ((scale_mode != 0 && scale_mode != 1) || (k_smoothing != 0 && k_smoothing != 1)) return KVQ_EINVAL;
  PackNvfp4Params p{};
  p.x[0] = Q;
  p.x[1] = K;
  p.x[2] = V;
  p.dtype = dtype == KVQ_BF16 ? DT_BF16 : DT_FP32;
  p.Ts = Ts;
  p.H = H;
  p.d = d;
  p.P = P;
  p.mode = (scale_mode == 1 ? kModeSearch : 0) | (k_smoothing ? kModeSmoothK : 0);
  p.amax = dev_amax_kv;
  p.amax_q = dev_amax_q;
  ulysses_partition(H, P, p.h0, p.owner);
  int64_t off = 0;
  for (int r = 0; r < P; ++r) {
    const int Hp = p.h0[r + 1] - p.h0[r];
    const Nvfp4SegLayout L = nvfp4_seg_layout(Ts, Hp, d, (int)esize(dtype), k_smoothing != 0, dev_amax_q != nullptr);
    p.dst[r] = pack_dest_segment(static_cast<uint8_t*>(send_buf) + off, L, Hp);
    off += L.total;
  }
  return cuda_status(launch_ulysses_pack_nvfp4(p, S(stream)));
}

kvq_status kv_append_ulysses_nvfp4(kvq_cache* c, int32_t layer, int64_t chunk_index, const void* recv_buf, int32_t P,
                                   const float* dev_amax_kv, const float* dev_amax_q, void* Q_out, kvq_dtype q_dtype,
                                   float* dev_q_scale, void* stream) {
  if (!c || !recv_buf || !dev_amax_kv || !Q_out || P <= 0 || P > kMaxP) return KVQ_EINVAL;
  if (layer < 0 || layer >= c->cfg.num_layers || chunk_index < 0) return KVQ_EINVAL;
  if (q_dtype != KVQ_BF16 && q_dtype != KVQ_FP32) return KVQ_EDTYPE;
  if ((dev_amax_q == nullptr) != (dev_q_scale == nullptr)) return KVQ_EINVAL;
  if (c->L.T_c % P) return KVQ_ESHAPE;
  SlotPlan plan;
  const kvq_status ss = select_slot(c, layer, chunk_index, &plan);
  if (ss != KVQ_OK) return ss;
  const int slot = plan.slot;
  const int Hr = c->cfg.num_heads, d = c->cfg.head_dim, Ts = (int)(c->L.T_c / P);
  ScatterNvfp4Params p{};
  p.recv = static_cast<const uint8_t*>(recv_buf);
  const bool qn = dev_amax_q != nullptr;
  p.lay = nvfp4_seg_layout(Ts, Hr, d, (int)esize(q_dtype), c->cfg.k_smoothing != 0, qn);
  p.seg = p.lay.total;
  p.Ts = Ts;
  p.Hr = Hr;
  p.d = d;
  p.es = qn ? 2 : (int)esize(q_dtype);  // NVFP4 Q arrives as fp16 dec(c) dec(s)
  p.P = P;
  p.amax_q = dev_amax_q;
  p.q_scale_out = dev_q_scale;
  for (int t = 0; t < 2; ++t) {
    p.codes[t] = codes_base(c, t, layer) + (size_t)slot * c->L.T_pad * (d / 2);
    p.scales[t] = scales_base(c, t, layer) + (size_t)slot * c->L.T_pad * (d / 16);
  }
  p.mean = c->cfg.k_smoothing ? mean_base(c, layer) + (size_t)slot * c->L.T_pad : nullptr;
  p.head_stride_rows = c->L.rows_per_head;
  p.Q = Q_out;
  p.amax = dev_amax_kv;
  p.g_out = g_base(c, layer) + slot * 2;
  p.status = status_ptr(c);
  if (launch_ulysses_scatter_nvfp4(p, S(stream)) != cudaSuccess) return KVQ_ECUDA;
  commit_slot(c, layer, chunk_index, plan);
  return KVQ_OK;
}

// ---- Device-initiated exchange over peer memory (§8(f) f4)
struct PeerWindowLayout {
  int64_t recv, seg, mailbox, arrive, flags, o[2], total;
};
static PeerWindowLayout peer_layout(int32_t T_c, int32_t H, int32_t d, int32_t P, kvq_dtype q_dtype,
                                    int32_t k_smoothing) {
  PeerWindowLayout L{};
  const int Ts = T_c / P, hmax = (H + P - 1) / P;
  auto a128 = [](int64_t x) { return (x + 127) & ~int64_t(127); };
  L.seg = nvfp4_seg_layout(Ts, hmax, d, (int)esize(q_dtype), k_smoothing != 0).total;
  L.recv = 0;
  L.mailbox = a128(P * L.seg);
  L.arrive = L.mailbox + a128(16 * (int64_t)P);
  L.flags = L.arrive + a128(8 * (int64_t)P);
  L.o[0] = L.flags + a128(8 * (int64_t)P);
  L.o[1] = L.o[0] + a128((int64_t)T_c * hmax * d * 2);
  L.total = L.o[1] + a128((int64_t)T_c * hmax * d * 2);
  return L;
}

struct kvq_peer {
  int32_t T_c, H, d, P, rank, scale_mode, k_smoothing;
  kvq_dtype q_dtype;
  PeerWindowLayout L;
  uint8_t* win[kMaxP];
  // f4 direct (kvq_peer_bind_caches): this rank's cache and every rank's cache arena + layout
  kvq_cache* cache = nullptr;
  uint8_t* arena[kMaxP];
  Layout Lr[kMaxP];
  int32_t h0[kMaxP + 1];
};

size_t kvq_peer_window_bytes(int32_t T_c, int32_t H, int32_t d, int32_t P, kvq_dtype q_dtype, int32_t k_smoothing) {
  if (P <= 0 || P > kMaxP || T_c <= 0 || T_c % P) return 0;
  return (size_t)peer_layout(T_c, H, d, P, q_dtype, k_smoothing).total;
}

kvq_status kvq_peer_create(int32_t T_c, int32_t H, int32_t d, int32_t P, int32_t rank, kvq_dtype q_dtype,
                           int32_t scale_mode, int32_t k_smoothing, void* const* windows, kvq_peer** out) {
  if (!windows || !out || P <= 0 || P > kMaxP || rank < 0 || rank >= P || H <= 0 || H > 256 || T_c <= 0)
    return KVQ_EINVAL;
  if (T_c % P) return KVQ_ESHAPE;
  if (d != 64 && d != 128) return KVQ_ESHAPE;
  if (q_dtype != KVQ_BF16 && q_dtype != KVQ_FP32) return KVQ_EDTYPE;
  if ((scale_mode != 0 && scale_mode != 1) || (k_smoothing != 0 && k_smoothing != 1)) return KVQ_EINVAL;
  kvq_peer* pe = new kvq_peer{};
  pe->T_c = T_c;
  pe->H = H;
  pe->d = d;
  pe->P = P;
  pe->rank = rank;
  pe->q_dtype = q_dtype;
  pe->scale_mode = scale_mode;
  pe->k_smoothing = k_smoothing;
  pe->L = peer_layout(T_c, H, d, P, q_dtype, k_smoothing);
  for (int r = 0; r < P; ++r) {
    if (!windows[r]) {
      delete pe;
      return KVQ_EINVAL;
    }
    pe->win[r] = static_cast<uint8_t*>(windows[r]);
  }
  *out = pe;
  return KVQ_OK;
}

kvq_status kvq_peer_destroy(kvq_peer* pe) {
  delete pe;
  return KVQ_OK;
}

kvq_status kvq_peer_o_local(const kvq_peer* pe, int64_t epoch, void** out) {
  if (!pe || !out || epoch <= 0) return KVQ_EINVAL;
  *out = pe->win[pe->rank] + pe->L.o[epoch & 1];
  return KVQ_OK;
}

kvq_status kvq_peer_publish_amax(const kvq_peer* pe, const void* K, const void* V, int64_t epoch, void* dev_scratch,
                                 void* stream) {
  if (!pe || !K || !V || !dev_scratch || epoch <= 0 || epoch >= (int64_t(1) << 32)) return KVQ_EINVAL;
  const int Ts = pe->T_c / pe->P;
  uint8_t* sc = static_cast<uint8_t*>(dev_scratch);
  float* amax = reinterpret_cast<float*>(sc + kvq_ulysses_shard_scratch_bytes(Ts, pe->H));
  kvq_status st = kvq_ulysses_shard_amax(K, V, pe->q_dtype, Ts, pe->H, pe->d, pe->k_smoothing, amax, dev_scratch, stream);
  if (st != KVQ_OK) return st;
  PeerPublishParams pp{};
  pp.amax = amax;
  pp.epoch = (unsigned long long)epoch;
  pp.P = pe->P;
  for (int r = 0; r < pe->P; ++r)
    pp.mailbox[r] = reinterpret_cast<unsigned long long*>(pe->win[r] + pe->L.mailbox) + 2 * pe->rank;
  return cuda_status(launch_peer_publish(pp, S(stream)));
}

kvq_status kvq_peer_pack(const kvq_peer* pe, const void* Q, const void* K, const void* V, int64_t epoch, void* stream) {
  if (!pe || !Q || !K || !V || epoch <= 0 || epoch >= (int64_t(1) << 32)) return KVQ_EINVAL;
  PackNvfp4Params p{};
  p.x[0] = Q;
  p.x[1] = K;
  p.x[2] = V;
  p.dtype = pe->q_dtype == KVQ_BF16 ? DT_BF16 : DT_FP32;
  p.Ts = pe->T_c / pe->P;
  p.H = pe->H;
  p.d = pe->d;
  p.P = pe->P;
  p.mode = (pe->scale_mode == 1 ? kModeSearch : 0) | (pe->k_smoothing ? kModeSmoothK : 0);
  ulysses_partition(pe->H, pe->P, p.h0, p.owner);
  for (int r = 0; r < pe->P; ++r) {
    const int Hp = p.h0[r + 1] - p.h0[r];
    p.dst[r] = pack_dest_segment(pe->win[r] + pe->L.recv + (int64_t)pe->rank * pe->L.seg,
                                 nvfp4_seg_layout(p.Ts, Hp, pe->d, (int)esize(pe->q_dtype), pe->k_smoothing != 0), Hp);
    p.arrive[r] = reinterpret_cast<unsigned long long*>(pe->win[r] + pe->L.arrive) + pe->rank;
  }
  p.mailbox = reinterpret_cast<const unsigned long long*>(pe->win[pe->rank] + pe->L.mailbox);
  p.epoch = (unsigned long long)epoch;
  return cuda_status(launch_ulysses_pack_nvfp4(p, S(stream)));
}

kvq_status kv_append_peer(const kvq_peer* pe, kvq_cache* c, int32_t layer, int64_t chunk_index, int64_t epoch,
                          void* Q_out, void* stream) {
  if (!pe || !c || !Q_out || epoch <= 0) return KVQ_EINVAL;
  if (layer < 0 || layer >= c->cfg.num_layers || chunk_index < 0) return KVQ_EINVAL;
  int32_t h0, h1;
  kvq_head_partition(pe->H, pe->P, pe->rank, &h0, &h1);
  if (c->cfg.num_heads != h1 - h0 || c->cfg.head_dim != pe->d || c->L.T_c != pe->T_c ||
      c->cfg.k_smoothing != pe->k_smoothing || c->cfg.scale_mode != pe->scale_mode)
    return KVQ_ESHAPE;
  SlotPlan plan;
  const kvq_status ss = select_slot(c, layer, chunk_index, &plan);
  if (ss != KVQ_OK) return ss;
  const int slot = plan.slot;
  const int Hr = c->cfg.num_heads, d = c->cfg.head_dim, Ts = (int)(c->L.T_c / pe->P);
  uint8_t* w = pe->win[pe->rank];
  ScatterNvfp4Params p{};
  p.recv = w + pe->L.recv;
  p.lay = nvfp4_seg_layout(Ts, Hr, d, (int)esize(pe->q_dtype), c->cfg.k_smoothing != 0);
  p.seg = pe->L.seg;
  p.Ts = Ts;
  p.Hr = Hr;
  p.d = d;
  p.es = (int)esize(pe->q_dtype);
  p.P = pe->P;
  for (int t = 0; t < 2; ++t) {
    p.codes[t] = codes_base(c, t, layer) + (size_t)slot * c->L.T_pad * (d / 2);
    p.scales[t] = scales_base(c, t, layer) + (size_t)slot * c->L.T_pad * (d / 16);
  }
  p.mean = c->cfg.k_smoothing ? mean_base(c, layer) + (size_t)slot * c->L.T_pad : nullptr;
  p.head_stride_rows = c->L.rows_per_head;
  p.Q = Q_out;
  p.amax = nullptr;
  p.g_out = g_base(c, layer) + slot * 2;
  p.status = status_ptr(c);
  p.arrive = reinterpret_cast<const unsigned long long*>(w + pe->L.arrive);
  p.arrive_target = (unsigned long long)epoch * (unsigned long long)ulysses_pack_grid(Ts, pe->H, d);
  p.mailbox = reinterpret_cast<const unsigned long long*>(w + pe->L.mailbox);
  p.epoch = (unsigned long long)epoch;
  if (launch_ulysses_scatter_nvfp4(p, S(stream)) != cudaSuccess) return KVQ_ECUDA;
  commit_slot(c, layer, chunk_index, plan);
  return KVQ_OK;
}

kvq_status kvq_peer_signal_o(const kvq_peer* pe, int64_t epoch, void* stream) {
  if (!pe || epoch <= 0) return KVQ_EINVAL;
  PeerSignalParams p{};
  p.P = pe->P;
  p.value = (unsigned long long)epoch;
  for (int r = 0; r < pe->P; ++r) p.slot[r] = reinterpret_cast<unsigned long long*>(pe->win[r] + pe->L.flags) + pe->rank;
  return cuda_status(launch_peer_signal(p, S(stream)));
}

kvq_status kvq_peer_pull_o(const kvq_peer* pe, int64_t epoch, void* O_shard, void* stream) {
  if (!pe || !O_shard || epoch <= 0) return KVQ_EINVAL;
  PeerPullParams p{};
  p.flags = reinterpret_cast<const unsigned long long*>(pe->win[pe->rank] + pe->L.flags);
  p.epoch = (unsigned long long)epoch;
  for (int r = 0; r < pe->P; ++r) p.o_src[r] = pe->win[r] + pe->L.o[epoch & 1];
  p.out = static_cast<uint8_t*>(O_shard);
  ulysses_partition(pe->H, pe->P, p.h0, p.owner);
  p.Ts = pe->T_c / pe->P;
  p.H = pe->H;
  p.d = pe->d;
  p.es = 2;  // bf16 O
  p.P = pe->P;
  p.rank = pe->rank;
  return cuda_status(launch_peer_pull_o(p, S(stream)));
}


// ---- f4 direct: stores straight into the owners' cache slots and O shards
kvq_status kvq_peer_bind_caches(kvq_peer* pe, kvq_cache* c, void* const* arenas) {
  if (!pe || !c || !arenas) return KVQ_EINVAL;
  int32_t a, b;
  kvq_head_partition(pe->H, pe->P, pe->rank, &a, &b);
  if (c->cfg.num_heads != b - a || c->cfg.head_dim != pe->d || c->L.T_c != pe->T_c ||
      c->cfg.k_smoothing != pe->k_smoothing || c->cfg.scale_mode != pe->scale_mode)
    return KVQ_ESHAPE;
  if ((int64_t)pe->T_c * (b - a) * pe->d * (int64_t)esize(pe->q_dtype) > pe->L.mailbox) return KVQ_ESHAPE;  // Q_recv fits
  for (int r = 0; r < pe->P; ++r) {
    if (!arenas[r]) return KVQ_EINVAL;
    kvq_head_partition(pe->H, pe->P, r, &pe->h0[r], &pe->h0[r + 1]);
    kvq_config cr = c->cfg;
    cr.num_heads = pe->h0[r + 1] - pe->h0[r];
    pe->Lr[r] = make_layout(&cr);
    pe->arena[r] = static_cast<uint8_t*>(arenas[r]);
  }
  // every kernel of the step is loaded now: under CUDA lazy loading a first launch could otherwise
  // wait for in-flight work while a device-side wait (mailbox / arrivals / O flags) is pending
  if (preload_peer_kernels() != cudaSuccess || preload_quant_kernels() != cudaSuccess ||
      preload_attention_kernels() != cudaSuccess)
    return KVQ_ECUDA;
  pe->cache = c;
  return KVQ_OK;
}

kvq_status kv_append_peer_direct(const kvq_peer* pe, int32_t layer, int64_t chunk_index, const void* Q, const void* K,
                                 const void* V, int64_t epoch, void* stream) {
  if (!pe || !pe->cache || !Q || !K || !V || epoch <= 0 || epoch >= (int64_t(1) << 32)) return KVQ_EINVAL;
  kvq_cache* c = pe->cache;
  if (layer < 0 || layer >= c->cfg.num_layers || chunk_index < 0) return KVQ_EINVAL;
  SlotPlan plan;  // every rank runs the same policy on the same calls: the owners pick this slot too
  const kvq_status ss = select_slot(c, layer, chunk_index, &plan);
  if (ss != KVQ_OK) return ss;
  const int slot = plan.slot, d = pe->d, Ts = pe->T_c / pe->P;
  cudaStream_t st = S(stream);
  uint8_t* w = pe->win[pe->rank];
  PeerWaitParams wm{};  // every shard amax of this epoch is in the mailbox
  wm.words = reinterpret_cast<const unsigned long long*>(w + pe->L.mailbox);
  wm.n = 2 * pe->P;
  wm.stride = 1;
  wm.mode = 0;
  wm.target = (unsigned long long)epoch;
  if (launch_peer_wait(wm, st) != cudaSuccess) return KVQ_ECUDA;
  PackNvfp4Params p{};
  p.x[0] = Q;
  p.x[1] = K;
  p.x[2] = V;
  p.dtype = pe->q_dtype == KVQ_BF16 ? DT_BF16 : DT_FP32;
  p.Ts = Ts;
  p.H = pe->H;
  p.d = d;
  p.P = pe->P;
  p.mode = quant_mode(c);
  ulysses_partition(pe->H, pe->P, p.h0, p.owner);
  const size_t es = esize(pe->q_dtype);
  for (int r = 0; r < pe->P; ++r) {
    const int Hp = pe->h0[r + 1] - pe->h0[r];
    const Layout& Lr = pe->Lr[r];
    const int64_t row0 = (int64_t)slot * Lr.T_pad + (int64_t)pe->rank * Ts;  // first row of this shard in the slot
    const size_t lrows = (size_t)layer * Hp * Lr.rows_per_head;
    PackDest& ds = p.dst[r];
    ds.kc = pe->arena[r] + Lr.off_codes[0] + (lrows + row0) * (d / 2);
    ds.vc = pe->arena[r] + Lr.off_codes[1] + (lrows + row0) * (d / 2);
    ds.ks = pe->arena[r] + Lr.off_scales[0] + (lrows + row0) * (d / 16);
    ds.vs = pe->arena[r] + Lr.off_scales[1] + (lrows + row0) * (d / 16);
    ds.km = pe->k_smoothing ? reinterpret_cast<float*>(pe->arena[r] + Lr.off_mean) + lrows + row0 : nullptr;
    ds.kv_ts = 1;
    ds.kv_hs = Lr.rows_per_head;
    ds.q = pe->win[r] + pe->L.recv + (size_t)pe->rank * Ts * Hp * d * es;  // owner's Q_recv [T_c, Hp, d]
    ds.qs = nullptr;
    ds.q_ts = Hp;
    ds.q_hs = 1;
    p.arrive[r] = reinterpret_cast<unsigned long long*>(pe->win[r] + pe->L.arrive) + pe->rank;
  }
  p.mailbox = reinterpret_cast<const unsigned long long*>(w + pe->L.mailbox);
  p.epoch = (unsigned long long)epoch;
  p.g_out = g_base(c, layer) + slot * 2;
  p.status = status_ptr(c);
  if (launch_ulysses_pack_nvfp4(p, st) != cudaSuccess) return KVQ_ECUDA;
  PeerWaitParams wa{};  // every source's stores into this rank's slot and Q_recv have landed
  wa.words = reinterpret_cast<const unsigned long long*>(w + pe->L.arrive);
  wa.n = pe->P;
  wa.stride = 1;
  wa.mode = 1;
  wa.target = (unsigned long long)epoch * (unsigned long long)ulysses_pack_grid(Ts, pe->H, d);
  if (launch_peer_wait(wa, st) != cudaSuccess) return KVQ_ECUDA;
  commit_slot(c, layer, chunk_index, plan);
  return KVQ_OK;
}

kvq_status chunk_attention_peer(const kvq_peer* pe, int32_t layer, const kvq_mask* mask, float softmax_scale,
                                int64_t epoch, void* dev_workspace, size_t workspace_bytes, void* stream) {
  if (!pe || !pe->cache || !mask || epoch <= 0) return KVQ_EINVAL;
  kvq_cache* c = pe->cache;
  if (dev_workspace && ((reinterpret_cast<uintptr_t>(dev_workspace) % kAlign) != 0 ||
                        workspace_bytes < kvq_attention_workspace_bytes(c)))
    return KVQ_EINVAL;
  uint8_t* o_peer[kMaxP];
  for (int r = 0; r < pe->P; ++r) o_peer[r] = pe->win[r] + pe->L.o[epoch & 1];
  const AttnRoute route{o_peer, pe->P, pe->T_c / pe->P, pe->H, pe->h0[pe->rank]};
  const void* Qr = pe->win[pe->rank] + pe->L.recv;
  const kvq_status s = attention_impl(c, layer, Qr, pe->q_dtype, nullptr, mask, softmax_scale, o_peer[pe->rank],
                                      KVQ_BF16, dev_workspace, workspace_bytes, stream, &route);
  if (s != KVQ_OK) return s;
  return kvq_peer_signal_o(pe, epoch, stream);  // this rank's O rows (attention + combine) have landed
}

kvq_status kvq_peer_wait_o(const kvq_peer* pe, int64_t epoch, void** O_shard, void* stream) {
  if (!pe || epoch <= 0) return KVQ_EINVAL;
  PeerWaitParams wf{};
  wf.words = reinterpret_cast<const unsigned long long*>(pe->win[pe->rank] + pe->L.flags);
  wf.n = pe->P;
  wf.stride = 1;
  wf.mode = 2;
  wf.target = (unsigned long long)epoch;
  if (launch_peer_wait(wf, S(stream)) != cudaSuccess) return KVQ_ECUDA;
  if (O_shard) *O_shard = pe->win[pe->rank] + pe->L.o[epoch & 1];
  return KVQ_OK;
}

kvq_status kvq_cache_get_config(const kvq_cache* c, kvq_config* out) {
  if (!c || !out) return KVQ_EINVAL;
  *out = c->cfg;
  return KVQ_OK;
}

kvq_status kvq_debug_force_two_pass(kvq_cache* c, int32_t on) {
  if (!c) return KVQ_EINVAL;
  c->two_pass_only = on != 0;
  return KVQ_OK;
}

// Debug timeline buffer for chunk_attention (declared in include/kvq_debug.h)
static unsigned long long* g_trace = nullptr;
kvq_status kvq_debug_set_trace(void* dev_buf) {
  g_trace = static_cast<unsigned long long*>(dev_buf);
  return KVQ_OK;
}
unsigned long long* kvq_trace_ptr() { return g_trace; }

// Debug probe entry point (declared in include/kvq_debug.h)
kvq_status kvq_debug_probe(int32_t which, const void* dev_in, void* dev_out, int64_t n, void* stream) {
  if (!dev_in || !dev_out || n < 0 || which < 0 || which > 3) return KVQ_EINVAL;
  return cuda_status(launch_probe(which, dev_in, dev_out, n, S(stream)));
}

}  // extern "C"

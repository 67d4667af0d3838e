// internal.h -- launch interfaces between the host C-ABI layer (api.cpp) and the kernels.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/kvq.h"

namespace kvq {

constexpr int kTileKeys = 128;     // keys per attention tile; slots are padded to a multiple
constexpr int kNumPartials = 592;  // amax partials per tensor (4 x 148 SMs)
constexpr int kMaxFusedCtas = 192;   // single-pass quantizer grid limit
constexpr int kSlotU64 = 16;        // one 128-byte line per barrier slot: K sector [0,4), V sector [4,8) u64
constexpr int kMaxSegs = 48;       // key segments per attention call

enum DType : int { DT_BF16 = 0, DT_FP32 = 1, DT_FP16 = 2 };
// quantizer modes (§8(f)): Four-Over-Six block-scale search for K and V; K-smoothing of K
constexpr int kModeSearch = 1;
constexpr int kModeSmoothK = 2;

// Device status word (in the arena): code (0 = ok), then first bad flat index.
struct DevStatus {
  int32_t code;
  int32_t pad;
  unsigned long long first_bad;
};

struct QuantParams {
  const void* x[2];          // K, V: [rows = T_c*H, d] t-major
  int dtype;                 // DT_BF16 | DT_FP32
  int rows, H, d;
  uint8_t* codes[2];         // slot base for head 0, rows of d/2 bytes
  uint8_t* scales[2];        // slot base for head 0, rows of d/16 bytes
  int64_t head_stride_rows;  // rows between heads (= slots * T_pad)
  float* g_out;              // [2]: K, V tensor scales of this (layer, slot)
  const uint32_t* partials;  // [2][kNumPartials] amax bit patterns, or null
  const float* ext_amax;     // [2] caller-supplied amax (Ulysses), or null
  unsigned long long* trace; // debug timeline (null in production)
  DevStatus* status;
  int mode;                  // kModeSearch | kModeSmoothK bits
  float* mean_out;           // K-smoothing: K row means, slot base for head 0, [H][head_stride_rows]
  uint32_t* partials_w;      // two-pass smoothing: where smooth_amax_kernel writes K's partials
};

struct DequantParams {
  const uint8_t* codes[2];
  const uint8_t* scales[2];
  const float* g;            // [2]
  const float* mean;         // K-smoothing row means (slot base, head-major like scales) or null
  int64_t head_stride_rows;
  int T, H, d;
  void* out[2];              // [T, H, d]
  int out_dtype;             // DT_FP32 | DT_BF16
};

struct ExportParams {
  const uint8_t* codes[2];
  const uint8_t* scales[2];
  const float* g;
  int64_t head_stride_rows;
  int T, H, d;
  uint8_t* codes_out[2];
  uint8_t* scales_out[2];
  float* g_out[2];
  const float* mean;         // K-smoothing row means (slot base) or null
  float* mean_out;           // [T*H] t-major, or null
};

constexpr int kMaxP = 64;  // ranks of a Ulysses group

struct AttnSeg {
  int32_t slot;   // cache slot (bf16kv mode: ignored)
  int32_t begin;  // first key row inside the slot
  int32_t end;    // one past the last key row
};

struct AttnParams {
  const void* Q;             // [Tq, H, d]
  int q_dtype;               // DT_BF16 | DT_FP32
  void* O;                   // [Tq, H, d]
  int out_dtype;             // DT_BF16 | DT_FP32
  // NVFP4 cache (layer base, head 0, slot 0)
  const uint8_t* codes_k;
  const uint8_t* codes_v;
  const uint8_t* scales_k;
  const uint8_t* scales_v;
  const float* g;            // g[slot*2 + {0,1}]
  const float* mean_k;       // K-smoothing row means (layer base, head-major like the codes) or null
  int64_t head_stride_rows;  // slots * T_pad
  int T_pad;                 // rows per slot (multiple of 128)
  // bf16 KV mode: K, V [n_keys, H, d]
  const void* Kb;
  const void* Vb;
  int Tq, H, d;
  float scale_log2;          // softmax_scale * log2(e)
  const float* q_scale;      // NVFP4 Q exchange: Q holds fp16 dec(c) dec(s), scores x g_Q = *q_scale (or null)
  DevStatus* status;         // Q non-finite (KVQ_ENONFINITE) / scores beyond fp32 (KVQ_ERANGE); null: not reported
  // persistent stream-K schedule (filled by launch_attention)
  unsigned long long* trace; // debug timeline of CTA 0 (null in production)
  float* ws;                 // partial-piece workspace (null: one CTA per unit, no partials)
  int ws_slots;              // slots available in ws
  int ws_slot_floats;        // floats per slot: 256 x d (O) + 512 (m, l)
  int max_ctas;              // SM count
  int units, qpairs, grid;
  bool hybrid;               // whole units in waves first, stream-K for the remainder (see Sched)
  int full_units;            // filled by launch_attention
  // f4 direct: O row (t, h) is stored as bf16 into rank r = t / o_Ts's buffer o_peer[r] (a peer
  // pointer, layout [o_Ts, o_H, d]) at row (t - r o_Ts, o_h0 + h); o_peer[0] null = O as usual
  uint8_t* o_peer[kMaxP];
  int o_Ts, o_H, o_h0;
  // Append fused into the attention launch (chunk_attention_append): the three spare warps of every
  // CTA's MMA warpgroup quantize CTA c's share of the chunk's K and V into slot ap_slot (definition
  // R1, quant_core.cuh) while the other warps attend over the history; tiles of ap_slot are read
  // only once every CTA has finished.  ap_sync: [0] launch epoch E, [1 .. 1+kMaxCtas) shard amax
  // of K, [.. +kMaxCtas) of V ((E + 1) << 32 | bits), [.. +kMaxCtas) done tags (= E + 1); tags are
  // E + 1, never 0, so the zeroed arena of a new cache holds no ready-looking word.
  const void* ap_x[2];       // K, V [T_c, H, d] (ap_dtype), or null: no fused append
  int ap_dtype, ap_slot;
  uint8_t* ap_codes[2];      // slot base (head 0) of the codes / scales of K, V
  uint8_t* ap_scales[2];
  float* ap_g;               // [2] g of the slot
  unsigned long long* ap_sync;
  // bf16 KV mode: TMA tensor maps of K and V viewed as [n_keys][H][d] bf16, box {64, 1, 128},
  // 128-byte swizzle (one 128-key x 64-column panel of the K-major SW128 tile per copy)
  CUtensorMap tmap_k, tmap_v;
  int nseg;
  AttnSeg seg[kMaxSegs];
};

constexpr int kMaxCtas = 148;  // workspace sized for one CTA per SM on B200
constexpr int kApSyncWords = 1 + 3 * kMaxCtas;  // AttnParams::ap_sync
inline size_t attn_ws_bytes(int d) { return (size_t)2 * kMaxCtas * (256 * d + 512) * sizeof(float); }

// tsr_begin = 1: V only (K's partials then come from launch_smooth_amax)
cudaError_t launch_smooth_amax(const QuantParams& p, cudaStream_t st);
cudaError_t launch_amax(const void* K, const void* V, int dtype, int64_t n, uint32_t* partials,
                        DevStatus* status, cudaStream_t st, int tsr_begin = 0);
// second pass of the two-launch path (after the amax pass)
cudaError_t launch_quantize2(const QuantParams& p, int sms, cudaStream_t st);
// single-pass cooperative quantize/append; cudaErrorNotSupported when the chunk does not fit
cudaError_t launch_quantize_fused(const QuantParams& p, unsigned long long* counters, uint32_t* partials, int sms,
                                  cudaStream_t st);
cudaError_t launch_dequantize(const DequantParams& p, cudaStream_t st);
cudaError_t launch_export(const ExportParams& p, cudaStream_t st);
cudaError_t launch_attention(const AttnParams& p, bool nvfp4_kv, cudaStream_t st);
cudaError_t launch_attention_append(const AttnParams& p, cudaStream_t st);
cudaError_t launch_dequant_window(const DequantParams& base, const AttnSeg* segs, int nseg, void* Kout,
                                  void* Vout, cudaStream_t st);

// Ulysses exchange kernels
cudaError_t launch_ulysses_pack(const void* Q, const void* K, const void* V, int dtype, int Ts, int H, int d,
                                int P, uint8_t* send, uint32_t* scratch, cudaStream_t st);
cudaError_t launch_ulysses_unpack_qkv(const uint8_t* recv, int dtype, int Ts, int Hr, int d, int P, void* Q,
                                      void* K, void* V, float* amax_kv, cudaStream_t st);
cudaError_t launch_ulysses_unpack_o(const uint8_t* recv, int dtype, int Ts, int H, int d, int P, void* O,
                                    cudaStream_t st);

// NVFP4 payload exchange (§8(f) f3): layout of one destination segment built
// from a source shard of Ts tokens for a destination owning Hp heads, rows (t, h_local) t-major:
// [Q Ts*Hp*d*es][K codes Ts*Hp*d/2][K scales Ts*Hp*d/16][V codes][V scales][K means Ts*Hp*4 if
// smoothing], every part padded to 16 bytes.
struct Nvfp4SegLayout {
  int64_t q, qs, kc, ks, vc, vs, km, total;  // byte offsets within the segment, total size
};
inline int64_t pad16(int64_t x) { return (x + 15) & ~int64_t(15); }
// q_nvfp4: Q travels as NVFP4 too (codes at q, scale bytes at qs; "cast the runtime Q
// to NVFP4"), else as rows of d * es bytes at q
inline Nvfp4SegLayout nvfp4_seg_layout(int Ts, int Hp, int d, int es, bool smooth, bool q_nvfp4 = false) {
  Nvfp4SegLayout L{};
  const int64_t rows = (int64_t)Ts * Hp;
  L.q = 0;
  L.qs = q_nvfp4 ? pad16(rows * d / 2) : pad16(rows * d * es);
  L.kc = q_nvfp4 ? L.qs + pad16(rows * d / 16) : L.qs;
  L.ks = L.kc + pad16(rows * d / 2);
  L.vc = L.ks + pad16(rows * d / 16);
  L.vs = L.vc + pad16(rows * d / 2);
  L.km = L.vs + pad16(rows * d / 16);
  L.total = L.km + (smooth ? pad16(rows * 4) : 0);
  return L;
}
// Where the pack kernel stores destination r's rows (row = (token t of the shard, local head hl)):
// Q rows (d * es bytes, or NVFP4 d/2 + d/16) at index t * q_ts + hl * q_hs, code rows (d/2 bytes),
// scale rows (d/16) and K-smoothing means (fp32) at t * kv_ts + hl * kv_hs.  A staging segment is
// t-major (kv_ts = q_ts = H_r, hs = 1); f4 direct stores into the owner's head-major cache slot
// (kv_ts = 1, kv_hs = rows per head, bases at the slot's row rank * Ts).
struct PackDest {
  uint8_t *q, *qs, *kc, *ks, *vc, *vs;
  float* km;
  int64_t kv_ts, kv_hs, q_ts, q_hs;
};
inline PackDest pack_dest_segment(uint8_t* seg, const Nvfp4SegLayout& L, int Hp) {
  return PackDest{seg + L.q, seg + L.qs, seg + L.kc, seg + L.ks, seg + L.vc, seg + L.vs,
                  reinterpret_cast<float*>(seg + L.km), Hp, 1, Hp, 1};
}
struct PackNvfp4Params {
  const void* x[3];          // Q, K, V shards [Ts, H, d] (dtype)
  int dtype, Ts, H, d, P, mode;
  const float* amax;         // [2] global amax of K (K_bar with smoothing) and V over all ranks
  const float* amax_q;       // global amax of Q: Q travels as NVFP4 (plain R1 encoding); null: as is
  PackDest dst[kMaxP];       // destination r's rows
  int h0[kMaxP + 1];
  uint8_t owner[256];
  // f4 (peer memory): with mailbox set, dst[] are peer pointers over NVLink; the global amax is the
  // max of this rank's mailbox (P epoch-tagged entries, polled), and every CTA bumps each
  // destination's arrival counter for this source (arrive[r], peer pointer) once its stores are done.
  const unsigned long long* mailbox;  // [P][2] (epoch << 32 | amax bits), or null
  unsigned long long* arrive[kMaxP];
  unsigned long long epoch;
  float* g_out;              // f4 direct: [2] g of this rank's own cache slot (from the mailbox), or null
  DevStatus* status;         //   non-finite global amax -> KVQ_ENONFINITE there
};
struct ScatterNvfp4Params {
  const uint8_t* recv;       // P segments of equal size (this rank is every source's destination)
  Nvfp4SegLayout lay;
  int64_t seg;               // segment stride in bytes
  int Ts, Hr, d, es, P;
  uint8_t* codes[2];         // cache slot bases (head 0), head-major rows of d/2 bytes
  uint8_t* scales[2];
  float* mean;               // K-smoothing row means of the slot (head 0) or null
  int64_t head_stride_rows;
  void* Q;                   // out: [P*Ts, Hr, d] (dtype)
  const float* amax;         // [2] global amax -> g of the slot (or null: from the mailbox)
  const float* amax_q;       // NVFP4 Q: its global amax; Q_out then holds fp16 dec(c) dec(s) (exact)
  float* q_scale_out;        //   and *q_scale_out = g_Q = RN32(amax_q / 2688)
  float* g_out;
  DevStatus* status;
  // f4: wait until every source's arrival counter reached `arrive_target` (its stores landed), and
  // take the amax from the mailbox when amax is null
  const unsigned long long* arrive;   // [P] this rank's counters, or null
  unsigned long long arrive_target;
  const unsigned long long* mailbox;  // [P][2]
  unsigned long long epoch;
};
struct PeerSignalParams {
  unsigned long long* slot[kMaxP];   // peer r's flag for this rank (peer pointers)
  unsigned long long value;
  int P;
};
struct PeerPullParams {
  const unsigned long long* flags;   // [P] this rank's flags, wait until all == epoch
  unsigned long long epoch;
  const uint8_t* o_src[kMaxP];       // owner r's O_local [P*Ts, H_r, d] (peer pointers)
  uint8_t* out;                      // this rank's O shard [Ts, H, d]
  int h0[kMaxP + 1];
  uint8_t owner[256];
  int Ts, H, d, es, P, rank;
};
struct PeerPublishParams {
  const float* amax;                 // [2] this rank's shard amax (device)
  unsigned long long* mailbox[kMaxP]; // peer r's mailbox entry pair for this rank (peer pointers)
  unsigned long long epoch;
  int P;
};
// f4: one thread spins (acquire, system scope) until every one of n words at words[i * stride]
// satisfies the mode: 0 = epoch tag (w >> 32) == target, 1 = w >= target, 2 = w == target.  A 1-CTA
// kernel, so the heavy kernels that follow never spin (ranks simulated on one GPU cannot starve).
struct PeerWaitParams {
  const unsigned long long* words;
  int n, stride, mode;
  unsigned long long target;
};
cudaError_t launch_peer_wait(const PeerWaitParams& p, cudaStream_t st);
// module loads of every kernel the f4 direct step launches (no lazy load while a wait is pending)
cudaError_t preload_peer_kernels();
cudaError_t preload_quant_kernels();
cudaError_t preload_attention_kernels();
cudaError_t launch_peer_publish(const PeerPublishParams& p, cudaStream_t st);
cudaError_t launch_peer_signal(const PeerSignalParams& p, cudaStream_t st);
cudaError_t launch_peer_pull_o(const PeerPullParams& p, cudaStream_t st);
int ulysses_pack_grid(int Ts, int H, int d);
cudaError_t launch_ulysses_shard_amax(const QuantParams& p, uint32_t* partials, float* amax_out, cudaStream_t st);
cudaError_t launch_ulysses_pack_nvfp4(const PackNvfp4Params& p, cudaStream_t st);
cudaError_t launch_ulysses_scatter_nvfp4(const ScatterNvfp4Params& p, cudaStream_t st);
void ulysses_partition(int H, int P, int* h0, uint8_t* owner);

// Host-side dry run of kv_*append*(chunk) + chunk_attention(mask) on `cache` (api.cpp): the errors
// either would return, found before the one-call Ulysses step issues its first collective.
kvq_status validate_append_attend(const kvq_cache* c, int32_t layer, int64_t chunk, const kvq_mask* m);

// Debug probes (codec checks against the oracle)
cudaError_t launch_probe(int which, const void* in, void* out, int64_t n, cudaStream_t st);

}  // namespace kvq

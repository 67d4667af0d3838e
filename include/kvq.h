/*
 * kvq.h -- C ABI of the B200-native NVFP4 KV-cache + fused-dequant chunk-attention library
 * (libkvq.so), the hot path of LongLive-2.0's inference infrastructure (arxiv 2605.18739).
 *
 * Citations are lines of the paper's text, PAPER.md (LaTeX of arxiv 2605.18739), with the
 * section / equation they fall in; DESIGN.md §2 lists every reading taken where the paper
 * is silent (Z1..Z19).
 *
 * Conventions (all entry points):
 *  - "dev" pointers are CUDA device pointers OWNED BY THE CALLER (in practice torch tensors);
 *    "host" pointers are ordinary host memory.  The library owns only host metadata.
 *    No entry point allocates device memory.
 *  - Argument errors (bad layer, d not in {64,128}, unknown chunk, ...) are returned
 *    synchronously as a negative kvq_status and NOTHING is launched.
 *  - Data errors found on the device (non-finite input) are asynchronous: they are recorded
 *    in a device status word and reported by kvq_get_status().
 *  - All device work is ordered on the cudaStream_t passed in (passed as void* so the header
 *    needs no CUDA include); nothing synchronizes the host except kvq_get_status().
 *  - A cache has a single writer (kv_quantize_append).  Reads may run concurrently
 *    while no append is in flight: chunk_attention uses a split-KV workspace inside the cache
 *    arena, so calls of it on one cache must be ordered (one stream, or events); calls that run
 *    concurrently on different streams use chunk_attention_ws, each with its own workspace.
 *  - Layouts: an activation tensor [T, H, d] is row-major, row = (t, h), t-major -- the
 *    paper's (T_c H) x d reshape of K_{l,c} (§3.2).
 */
#ifndef KVQ_H_
#define KVQ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KVQ_OK = 0,
  KVQ_EINVAL = -1,      /* bad argument value or null pointer */
  KVQ_ESHAPE = -2,      /* unsupported shape (d not 64/128, T_c not a multiple of 16, ...) */
  KVQ_EDTYPE = -3,      /* unsupported dtype combination */
  KVQ_ENOCHUNK = -4,    /* chunk index is neither newest+1 (append) nor newest (overwrite), or a
                           key chunk needed by the mask is not resident */
  KVQ_ECAPACITY = -5,   /* no free slot: every slot holds a pinned sink / window chunk */
  KVQ_ENONFINITE = -6,  /* (async) non-finite value in an appended K or V tensor */
  KVQ_ERANGE = -7,      /* value outside the representable range */
  KVQ_ECUDA = -8,       /* a CUDA runtime call failed */
  KVQ_ENCCL = -9        /* reserved for the multi-GPU exchange */
} kvq_status;

typedef enum { KVQ_BF16 = 0, KVQ_FP32 = 1, KVQ_FP16 = 2 } kvq_dtype;

/* Cache geometry.  T_c = tokens_per_frame * frames_per_chunk tokens per chunk (PAPER.md:135:
 * "Each chunk contains F_c frames and T_c = F_c L_f latent tokens").  Each chunk occupies one
 * slot of T_pad = round_up(T_c, 128) rows so every 128-key attention tile lies in one chunk
 * (one alpha^FP32 per tile). */
typedef struct {
  int32_t num_layers;
  int32_t num_heads;        /* heads stored by THIS cache (local heads on this rank) */
  int32_t head_dim;         /* d: 64 or 128 */
  int32_t tokens_per_frame; /* L_f, e.g. 1560 */
  int32_t frames_per_chunk; /* F_c, e.g. 3 */
  int32_t sink_frames;      /* S_g of the global sink A_g, pinned, never evicted */
  int32_t window_frames;    /* sliding window W in frames INCLUDING the current chunk (reading Z10) */
  int32_t max_chunk_slots;  /* slots per layer; >= sink chunks + window chunks (+ shot chunks) */
  int32_t scale_mode;       /* 0 = block scale alpha_i(6) = cast_E4M3(max|U_bar|/6);
                               1 = Four-Over-Six search between alpha_i(6) and alpha_i(4) for K and V
                               (Eq. 4o6, applied to KV by PAPER.md:146): the
                               candidate with the lower float32 squared reconstruction error wins,
                               ties to 6 (reading Z21).  Other values: KVQ_EINVAL */
  int32_t k_smoothing;      /* 0 = off; 1 = K-smoothing: keys are stored as
                               K_bar = K - mean_d(K) per (t, h) row (float32 tree-order mean,
                               reading Z20); the fp32 row means are stored with the chunk and
                               restored exactly (K^ = dequant(K_bar) + mean) by kv_dequantize and
                               by chunk_attention (as the rank-1 score term mean_j * sum_u Q_iu).
                               Other values: KVQ_EINVAL */
} kvq_config;

/* Key set of one attention call: K_eff(t) = A_g U A_s U KV_[t-W,t) U {chunk t}, deduplicated
 * (§4.2; reading Z9: the current chunk is attended from the cache). */
typedef struct {
  int64_t chunk_index;       /* t: the chunk whose queries attend */
  int32_t sink_frames;       /* S_g */
  int32_t window_frames;     /* W in frames including the current chunk */
  int64_t shot_start_frame;  /* A_s = (start, len) pointers; len 0 = none */
  int64_t shot_len_frames;
} kvq_mask;

typedef struct kvq_cache kvq_cache; /* opaque; host metadata owned by the library */

/* Device arena bytes for `cfg`: K/V codes (d/2 B per row), K/V E4M3 scales (d/16 B per row),
 * the per-(layer, slot, K|V) FP32 tensor scales, amax partials and the status word.  0 on a
 * bad config. */
size_t kvq_cache_bytes(const kvq_config* cfg);

/* Creates a cache over a caller-owned dev arena of >= kvq_cache_bytes(cfg) bytes, 256-byte
 * aligned.  The arena is zeroed on `stream` (void* cudaStream_t).  *out receives the handle. */
kvq_status kvq_cache_create(const kvq_config* cfg, void* dev_arena, size_t arena_bytes,
                            void* stream, kvq_cache** out);
kvq_status kvq_cache_destroy(kvq_cache* cache);
/* Forget every chunk (new video); zeroes the arena on `stream`. */
kvq_status kvq_cache_reset(kvq_cache* cache, void* stream);
/* Copies the cache's geometry (as passed to kvq_cache_create) into *out (host). */
kvq_status kvq_cache_get_config(const kvq_cache* cache, kvq_config* out);
/* Re-bind the shot-level sink A_s (a prompt switch).  Moves two host
 * pointers only; never touches cache bytes ("zero memory overhead").  Chunks
 * overlapping [start, start+len) frames are pinned against eviction from now on. */
kvq_status kvq_set_shot(kvq_cache* cache, int64_t shot_start_frame, int64_t shot_len_frames);

/* NVFP4-quantize one chunk's K and V of layer `layer` and store them in the cache
 * (§3.2: "reshape to (T_c H) x d and quantize independently with NVFP4";
 * format PAPER.md:81-102 §2.2 Eq. 2, block scale PAPER.md:723-727 App. F).
 * K, V: dev [T_c, H, d] in_dtype (KVQ_BF16 | KVQ_FP32).  Per tensor: g = RN32(amax/2688),
 * per 16-block E4M3 scale s = E4M3(RN32(RN32(bmax/g)/6)), codes E2M1(RN32(x/RN32(dec(s) g)))
 * (reading Z4, definition R1), packed 2 per byte, element 2k in the low nibble.
 * chunk_index == newest+1 appends (evicting chunks outside sinks U window); == newest
 * overwrites (a denoising step re-writes the in-progress chunk); the first append of a layer
 * must be chunk 0 or any index after kvq_cache_reset.  Anything else: KVQ_ENOCHUNK.
 * Stream-ordered; no host synchronization.  Non-finite input: the chunk is left undefined
 * and KVQ_ENONFINITE is reported by kvq_get_status(). */
kvq_status kv_quantize_append(kvq_cache* cache, int32_t layer, int64_t chunk_index,
                              const void* K, const void* V, kvq_dtype in_dtype, void* stream);

/* As kv_quantize_append, but the tensor amax of K and V is supplied by the caller as two
 * floats in device memory (dev_amax_kv[0] = amax(K), [1] = amax(V)) -- used after the
 * Ulysses exchange, where K/V hold only this rank's heads but alpha^FP32 is taken over all
 * heads (reading Z2/Z18). */
kvq_status kv_quantize_append_amax(kvq_cache* cache, int32_t layer, int64_t chunk_index,
                                   const void* K, const void* V, kvq_dtype in_dtype,
                                   const float* dev_amax_kv, void* stream);

/* Chunk attention of chunk t's queries over the quantized cache with dequantization fused
 * into the kernel (§3.2; K_eff PAPER.md:249; attention PAPER.md:187):
 *   O[i,h,:] = softmax_j( Q[i,h,:] . K^[j,h,:] * scale ) V^[j,h,:],  j in K_eff(t)
 * with K^, V^ = dec(code) dec(s) g (Eq. 2).  Q: dev [T_c, H, d] q_dtype (BF16 | FP32);
 * O: dev [T_c, H, d] out_dtype (BF16 = the product, FP32 = parity mode).  softmax_scale <= 0
 * means 1/sqrt(d).  Every key chunk of K_eff must be resident (else KVQ_ENOCHUNK).
 * Range: every finite query value fits the MMA (each Q row is scaled by a power of two into
 * fp16's range before the fp16 tensor-core MMA; exact); scores s = Q.K^ * scale * log2(e) are
 * supported for |s| < 2^12 (fp32 accumulation error grows with |s|, reading Z25).
 * Asynchronous data errors, reported by kvq_get_status with a flat index into Q:
 * KVQ_ENONFINITE for an inf/NaN query element; KVQ_ERANGE when a key tile's largest score of a
 * row reaches 2^12 in magnitude (index = the row's first element).  O is undefined for such rows.
 * Workspace: the cache's own (calls on one cache must be ordered, see the conventions above). */
kvq_status chunk_attention(kvq_cache* cache, int32_t layer, const void* Q, kvq_dtype q_dtype,
                           const kvq_mask* mask, float softmax_scale, void* O,
                           kvq_dtype out_dtype, void* stream);

/* Bytes of the split-KV workspace one chunk_attention_ws call needs (partial O, running max and
 * row sum of the pieces of work units split across CTAs); 0 for a null cache. */
size_t kvq_attention_workspace_bytes(const kvq_cache* cache);

/* chunk_attention with a caller-owned dev workspace (256-byte aligned, >= 
 * kvq_attention_workspace_bytes, else KVQ_EINVAL): calls on different streams may run
 * concurrently if each has its own workspace and no append to the cache is in flight. */
kvq_status chunk_attention_ws(kvq_cache* cache, int32_t layer, const void* Q, kvq_dtype q_dtype,
                              const kvq_mask* mask, float softmax_scale, void* O,
                              kvq_dtype out_dtype, void* dev_workspace, size_t workspace_bytes,
                              void* stream);

/* kv_quantize_append of chunk `chunk_index` followed by chunk_attention of its queries, as ONE
 * launch: the three spare warps of every attention CTA quantize that CTA's share of K and V into
 * the chunk's slot (the same bytes as kv_quantize_append, reading Z4 definition R1) while the other
 * warps attend over the history; each CTA reads the new slot only after every CTA has finished
 * (the tensor amax is exchanged between the co-resident CTAs of a cooperative launch), and a
 * first work piece that would reach the new chunk's tiles early is processed last.  The append's
 * own time would hide behind the history tiles.  MEASURED SLOWER than the two launches on the
 * Wan layer (the combined kernel's register budget costs more than the 14 us append it hides,
 * DESIGN.md §5.1), so it is opt-in: environment KVQ_FUSED_APPEND=1, and only in the plain mode
 * (scale_mode 0, no K-smoothing) with bf16 Q when the appended chunk is at most half of K_eff.
 * Otherwise the call runs kv_quantize_append then chunk_attention(_ws) on the stream.
 * mask->chunk_index must equal chunk_index.  Errors as
 * for those two calls (checked before anything is launched).  dev_workspace: NULL = the cache's
 * own, else as chunk_attention_ws. */
kvq_status chunk_attention_append(kvq_cache* cache, int32_t layer, int64_t chunk_index,
                                  const void* K, const void* V, kvq_dtype in_dtype, const void* Q,
                                  kvq_dtype q_dtype, const kvq_mask* mask, float softmax_scale,
                                  void* O, kvq_dtype out_dtype, void* dev_workspace,
                                  size_t workspace_bytes, void* stream);

/* Checking: dequantize one resident chunk to dev [T_c, H, d]: FP32 = RN32(dec(c) dec(s) g)
 * (Eq. 2), BF16 = RN_bf16 of that.  With k_smoothing, K = RN32(dec(c) dec(s) g + mean)
 * (one rounding). */
kvq_status kv_dequantize(const kvq_cache* cache, int32_t layer, int64_t chunk_index,
                         void* K_out, void* V_out, kvq_dtype out_dtype, void* stream);

/* Canonical bytes of one resident chunk for bit-exact parity, rows (t, h) t-major:
 * codes dev [T_c*H, d/2] u8, scales dev [T_c*H, d/16] u8, g dev fp32[1], for K and V. */
kvq_status kv_export_chunk(const kvq_cache* cache, int32_t layer, int64_t chunk_index,
                           void* codes_k, void* scales_k, float* g_k,
                           void* codes_v, void* scales_v, float* g_v, void* stream);

/* K-smoothing row means of one resident chunk: dev fp32 [T_c*H], rows (t, h) t-major.
 * KVQ_EINVAL when the cache was created with k_smoothing = 0; KVQ_ENOCHUNK if not resident. */
kvq_status kv_export_kmean(const kvq_cache* cache, int32_t layer, int64_t chunk_index,
                           float* mean_out, void* stream);

/* Bytes of resident NVFP4 K/V payload (codes + scales + tensor scales) over all layers'
 * resident chunks -- the footprint report for PAPER.md:146's "close to 3.6x". */
size_t kvq_resident_bytes(const kvq_cache* cache);
/* Number of resident chunks of `layer` (host metadata). */
int32_t kvq_resident_chunks(const kvq_cache* cache, int32_t layer);

/* Bench-only (not the product path): the paper's unfused design -- reconstruct K_eff into a
 * contiguous bf16 buffer dev [n_keys, H, d] (the "customized parallel dequantization kernel",
 * PAPER.md:146) -- and attention over caller-provided bf16 K/V (the same kernel family with
 * no dequantization; BASELINE.json config 4 "NVFP4 vs bf16 KV").  *n_keys (host) receives
 * |K_eff|; pass K_out = V_out = NULL to query it only. */
kvq_status kv_dequantize_window(const kvq_cache* cache, int32_t layer, const kvq_mask* mask,
                                void* K_out, void* V_out, int64_t* n_keys, void* stream);
/* Q: dev [T_q, H, d] bf16; K, V: dev [n_keys, H, d] bf16 (16-byte aligned; every key attended,
 * bidirectional); O: dev [T_q, H, d] out_dtype.  Tiles land by TMA (tensor maps built per call;
 * KVQ_EINVAL if the driver refuses them); P is bf16.  Without a workspace one CTA per
 * (head, 256-query pair). */
kvq_status chunk_attention_bf16kv(const void* Q, const void* K, const void* V, int32_t T_q,
                                  int64_t n_keys, int32_t H, int32_t d, float softmax_scale,
                                  void* O, kvq_dtype out_dtype, void* stream);
/* Bytes of the workspace chunk_attention_bf16kv_ws takes at head dim d (0 for other d). */
size_t kvq_bf16kv_workspace_bytes(int32_t d);
/* chunk_attention_bf16kv on a persistent one-CTA-per-SM grid: whole (head, query pair) units in
 * waves (the CTAs of a wave stream the same heads' key tiles, so the bf16 window is read from
 * HBM about once), the remainder split stream-K with its partials in dev_workspace (256-byte
 * aligned, >= kvq_bf16kv_workspace_bytes(d), else KVQ_EINVAL; NULL = the call above). */
kvq_status chunk_attention_bf16kv_ws(const void* Q, const void* K, const void* V, int32_t T_q,
                                     int64_t n_keys, int32_t H, int32_t d, float softmax_scale,
                                     void* O, kvq_dtype out_dtype, void* dev_workspace,
                                     size_t workspace_bytes, void* stream);

/* Asynchronous data errors: synchronizes `stream`, returns the first recorded error (or
 * KVQ_OK) and the first offending flat element index (K: index into K, V: T_c*H*d + index),
 * then clears it. */
kvq_status kvq_get_status(kvq_cache* cache, void* stream, int64_t* first_bad_index);
const char* kvq_strerror(kvq_status s);

/* ---------------------------------------------------------------------------------------
 * Head-sharded (Ulysses) exchange, PAPER.md:556-564 (App. C) and PAPER.md:640-650 (App. D):
 * z^(p) in R^{L/P x H x d} --All-to-All--> R^{L x H/P x d}; a second All-to-All restores the
 * sequence-sharded layout.  The collective itself is NCCL (torch.distributed); these kernels
 * are the compute around it.  Heads are split contiguously, the first H % P ranks get one more
 * (12 heads on 8 ranks: 2,2,2,2,1,1,1,1). */
void kvq_head_partition(int32_t H, int32_t P, int32_t rank, int32_t* h0, int32_t* h1);

/* Bytes this rank sends to destination `dst` for Q|K|V (= bytes it receives from any source
 * when dst == this rank): 3 * Ts * H_dst * d * esize + 16 (trailer: amax(K), amax(V) of the
 * sender's sequence shard as fp32, then 8 pad bytes). */
size_t kvq_ulysses_qkv_bytes(int32_t Ts, int32_t H, int32_t d, int32_t P, int32_t dst,
                             kvq_dtype dtype);

/* Pack this rank's sequence shard Q, K, V dev [Ts, H, d] into the all-to-allv send buffer:
 * for destination p, one contiguous segment [3][Ts][H_p][d] + trailer, segments in rank
 * order.  Also computes the shard's amax(K), amax(V) into every trailer.
 * dev_scratch: >= 8192 bytes of caller-owned device scratch. */
kvq_status kvq_ulysses_pack_qkv(const void* Q, const void* K, const void* V, kvq_dtype dtype,
                                int32_t Ts, int32_t H, int32_t d, int32_t P, void* send_buf,
                                void* dev_scratch, void* stream);

/* Unpack what this rank (owning H_r heads) received -- P segments [3][Ts][H_r][d] + trailer
 * from sources 0..P-1 -- into contiguous Q, K, V dev [P*Ts, H_r, d] and the global
 * amax_kv dev fp32[2] = max over sources (reading Z18: codes equal the 1-GPU run). */
kvq_status kvq_ulysses_unpack_qkv(const void* recv_buf, kvq_dtype dtype, int32_t Ts,
                                  int32_t H_r, int32_t d, int32_t P, void* Q, void* K, void* V,
                                  float* dev_amax_kv, void* stream);

/* After attention: O_local dev [P*Ts, H_r, d] is sent as P contiguous token blocks (equal
 * splits, no pack needed).  Unpack the received P blocks [Ts][H_p][d] (p = 0..P-1, head
 * counts from kvq_head_partition) into this rank's output shard dev [Ts, H, d]. */
kvq_status kvq_ulysses_unpack_o(const void* recv_buf, kvq_dtype dtype, int32_t Ts, int32_t H,
                                int32_t d, int32_t P, void* O_shard, void* stream);

/* ---------------------------------------------------------------------------------------
 * NVFP4 payload for the exchange (§8(f) f3; App. D: the pre-attention
 * All-to-All "performed entirely in the low-precision space", ~3.6x less K/V volume).  The
 * sender quantizes its sequence shard of K and V with the GLOBAL tensor scales, so what it ships
 * is exactly the cache bytes of the 1-GPU run for those rows (readings Z2/Z18).  Q travels in its
 * input dtype, or -- optionally -- as NVFP4 too (a different attention numerics
 * mode, reading Z24: kvq_ulysses_q_amax, dev_amax_q of kvq_ulysses_pack_nvfp4, and
 * chunk_attention_qscaled).  Sequence:
 *   kvq_ulysses_shard_amax (+ kvq_ulysses_q_amax) -> all-reduce(MAX) of the 2 (3) floats over the
 *   group (NCCL) -> kvq_ulysses_pack_nvfp4 -> all_to_all_single -> kv_append_ulysses_nvfp4 ->
 *   chunk_attention (chunk_attention_qscaled with NVFP4 Q). */

/* Device scratch for kvq_ulysses_shard_amax (partials, status, K-smoothing means). */
size_t kvq_ulysses_shard_scratch_bytes(int32_t Ts, int32_t H);

/* amax of this rank's shard: dev_amax_kv fp32[2] = max |K| (max |K - row mean| with
 * k_smoothing, reading Z20) and max |V| over the shard [Ts, H, d]; non-finite values propagate
 * (the receiving cache reports KVQ_ENONFINITE). */
kvq_status kvq_ulysses_shard_amax(const void* K, const void* V, kvq_dtype dtype, int32_t Ts,
                                  int32_t H, int32_t d, int32_t k_smoothing, float* dev_amax_kv,
                                  void* dev_scratch, void* stream);

/* Bytes of the segment for destination `dst` (= bytes received from every source when dst is
 * this rank): per row (t, h_dst) Q d*esize(q_dtype) (or, with q_nvfp4, d/2 code + d/16 scale
 * bytes), K and V codes d/2 + scales d/16 each (+ a fp32 K mean with k_smoothing), each part
 * padded to 16 bytes. */
size_t kvq_ulysses_nvfp4_bytes(int32_t Ts, int32_t H, int32_t d, int32_t P, int32_t dst,
                               kvq_dtype q_dtype, int32_t k_smoothing, int32_t q_nvfp4);

/* max |Q| of this rank's shard (dev fp32[1]); scratch as for kvq_ulysses_shard_amax. */
kvq_status kvq_ulysses_q_amax(const void* Q, kvq_dtype dtype, int32_t Ts, int32_t H, int32_t d,
                              float* dev_amax_q, void* dev_scratch, void* stream);

/* Quantize + pack this rank's shard (Q, K, V dev [Ts, H, d]) into the all-to-allv send buffer,
 * destination segments in rank order.  dev_amax_kv: the GLOBAL amax (all-reduced) -> g =
 * RN32(amax/2688); scale_mode / k_smoothing must match the receiving caches' config.
 * dev_amax_q: null = Q travels in its dtype; else the GLOBAL amax of Q and Q is cast to NVFP4 too
 * ("we also cast the runtime Q to NVFP4 immediately before the pre-attention
 * All-to-All"; plain R1 encoding) -- a different attention numerics mode (reading Z24). */
kvq_status kvq_ulysses_pack_nvfp4(const void* Q, const void* K, const void* V, kvq_dtype dtype,
                                  int32_t Ts, int32_t H, int32_t d, int32_t P,
                                  const float* dev_amax_kv, const float* dev_amax_q,
                                  int32_t scale_mode, int32_t k_smoothing, void* send_buf,
                                  void* stream);

/* Receiving side: the P received segments (this rank's H_r = cache num_heads heads, Ts = T_c/P
 * tokens each) become chunk `chunk_index` of `layer` under the append policy of
 * kv_quantize_append (same slot / eviction rules, same error codes), g of the slot from
 * dev_amax_kv, and Q_out dev [T_c, H_r, d] receives the chunk's queries: in q_dtype, or, with
 * dev_amax_q (NVFP4 Q; dev_q_scale must then be given too), as fp16 dec(c) dec(s) -- exact --
 * with *dev_q_scale = g_Q; attend with chunk_attention_qscaled. */
kvq_status kv_append_ulysses_nvfp4(kvq_cache* cache, int32_t layer, int64_t chunk_index,
                                   const void* recv_buf, int32_t P, const float* dev_amax_kv,
                                   const float* dev_amax_q, void* Q_out, kvq_dtype q_dtype,
                                   float* dev_q_scale, void* stream);

/* chunk_attention for NVFP4-exchanged queries: Q dev [T_c, H, d] fp16 holding dec(c) dec(s),
 * scores scaled by g_Q = *dev_q_scale (device fp32) on top of softmax_scale. */
kvq_status chunk_attention_qscaled(kvq_cache* cache, int32_t layer, const void* Q_fp16,
                                   const float* dev_q_scale, const kvq_mask* mask,
                                   float softmax_scale, void* O, kvq_dtype out_dtype, void* stream);

/* ---------------------------------------------------------------------------------------
 * Device-initiated exchange over peer memory (§8(f) f4): the NVFP4 exchange above without NCCL.
 * Every rank owns one "window" of kvq_peer_window_bytes (identical layout on all ranks, sized for
 * the largest head share): P receive segments, a mailbox of P shard amaxes, P arrival counters, P
 * O-ready flags and two O_local buffers.  `windows` are the P ranks' window base pointers as seen
 * from this rank -- peer pointers over NVLink/NVSwitch (e.g. torch symmetric memory), or plain
 * device pointers when P ranks are simulated on one GPU.  The caller zeroes every window once.
 * Per step (epoch = 1, 2, 3, ... consecutively, < 2^32), on each rank's stream:
 *   kvq_peer_publish_amax  shard amax -> every peer's mailbox (st.release.sys)
 *   kvq_peer_pack          waits for its mailbox (all P), quantizes its shard with the global scale
 *                          and stores each destination's rows straight into that rank's window,
 *                          then bumps the destination's arrival counter (fence.sys + red.release.sys)
 *   kv_append_peer         waits for all P arrivals, scatters into the cache slot (append policy)
 *   chunk_attention        on the local heads, O into kvq_peer_o_local(epoch)
 *   kvq_peer_signal_o      O-ready flag -> every peer
 *   kvq_peer_pull_o        waits for all P flags, pulls this rank's token rows of every head.
 * Waits are device-side spins: all ranks must run the same sequence of steps. */
typedef struct kvq_peer kvq_peer;
size_t kvq_peer_window_bytes(int32_t T_c, int32_t H, int32_t d, int32_t P, kvq_dtype q_dtype,
                             int32_t k_smoothing);
kvq_status kvq_peer_create(int32_t T_c, int32_t H, int32_t d, int32_t P, int32_t rank,
                           kvq_dtype q_dtype, int32_t scale_mode, int32_t k_smoothing,
                           void* const* windows, kvq_peer** out);
kvq_status kvq_peer_destroy(kvq_peer* peer);
/* O_local dev [T_c, H_rank, d] bf16 of this rank for `epoch` (alternating buffers). */
kvq_status kvq_peer_o_local(const kvq_peer* peer, int64_t epoch, void** out);
/* dev_scratch >= kvq_ulysses_shard_scratch_bytes(T_c/P, H) + 16 bytes. */
kvq_status kvq_peer_publish_amax(const kvq_peer* peer, const void* K_shard, const void* V_shard,
                                 int64_t epoch, void* dev_scratch, void* stream);
kvq_status kvq_peer_pack(const kvq_peer* peer, const void* Q_shard, const void* K_shard,
                         const void* V_shard, int64_t epoch, void* stream);
/* cache: this rank's heads, same d / T_c / modes as the peer config (else KVQ_ESHAPE).
 * Q_out dev [T_c, H_rank, d] (q_dtype). */
kvq_status kv_append_peer(const kvq_peer* peer, kvq_cache* cache, int32_t layer,
                          int64_t chunk_index, int64_t epoch, void* Q_out, void* stream);
kvq_status kvq_peer_signal_o(const kvq_peer* peer, int64_t epoch, void* stream);
/* O_shard dev [T_c/P, H, d] bf16. */
kvq_status kvq_peer_pull_o(const kvq_peer* peer, int64_t epoch, void* O_shard, void* stream);

/* f4 DIRECT (App. D): no staging copies at all.  The
 * pack kernel stores each owner's NVFP4 rows straight into that owner's cache slot (and the
 * bf16/fp32 Q rows into the owner's window), and the attention epilogue (and the split-KV
 * combine) stores every O row straight into the O shard of the rank that owns its tokens.
 * The cache arenas must be peer-accessible: `arenas` are the P ranks' kvq_cache arenas as seen
 * from this rank (torch symmetric memory, or plain pointers for ranks simulated on one GPU);
 * every rank's cache has the same config except num_heads = its head share, and all ranks
 * make the same sequence of calls, so every rank's slot policy picks the same slot.
 * Per step (epoch as above), on each rank's stream:
 *   kvq_peer_publish_amax   (as above)
 *   kv_append_peer_direct   waits (1-CTA kernel) for the mailbox, quantizes this rank's shard
 *                           with the global scale into every owner's slot rows, then waits
 *                           (1-CTA kernel) until all P sources stored into this rank's slot:
 *                           on completion the local cache holds the chunk (and its g)
 *   chunk_attention_peer    attention over the local heads, Q from the window, O rows into
 *                           the owners' O shards over peer memory, then the O-ready signal
 *   kvq_peer_wait_o         waits (1-CTA kernel) for all P signals; *O_shard = this rank's
 *                           O shard [T_c/P, H, d] bf16 inside its window, valid until this
 *                           rank's kvq_peer_publish_amax of epoch + 2.
 * NVFP4 Q (reading Z24) is not offered on this path. */
kvq_status kvq_peer_bind_caches(kvq_peer* peer, kvq_cache* cache, void* const* arenas);
kvq_status kv_append_peer_direct(const kvq_peer* peer, int32_t layer, int64_t chunk_index,
                                 const void* Q_shard, const void* K_shard, const void* V_shard,
                                 int64_t epoch, void* stream);
/* dev_workspace: NULL = the cache's own (see chunk_attention), else as chunk_attention_ws. */
kvq_status chunk_attention_peer(const kvq_peer* peer, int32_t layer, const kvq_mask* mask,
                                float softmax_scale, int64_t epoch, void* dev_workspace,
                                size_t workspace_bytes, void* stream);
kvq_status kvq_peer_wait_o(const kvq_peer* peer, int64_t epoch, void** O_shard, void* stream);

/* ---------------------------------------------------------------------------------------
 * One-call head-sharded chunk step with a library-owned NCCL communicator (
 * PAPER.md:556-564 App. C, App. D).  Same kernels as the calls above, with
 * the collectives issued by the library itself (grouped ncclSend/ncclRecv all-to-allv and an
 * ncclAllReduce(MAX) of the tensor amaxes) on the caller's stream.  NCCL allocates its own
 * device memory inside kvq_comm_create (the one exception to "no entry point allocates");
 * everything else lives in a caller-owned workspace.  Collective calls must be made by every
 * rank of the communicator in the same order (NCCL's rule). */
typedef struct kvq_comm kvq_comm;

/* Exchange payloads: 0 = Q, K, V in the input dtype (+ piggybacked shard amax, reading Z18);
 * 1 = K/V as NVFP4 cache bytes quantized on the sender with the all-reduced amax (f3);
 * 2 = as 1 with NVFP4 Q (reading Z24, different attention numerics). */
enum { KVQ_EXCHANGE_INPUT = 0, KVQ_EXCHANGE_NVFP4 = 1, KVQ_EXCHANGE_NVFP4_Q = 2 };

/* out_128_bytes (host): an ncclUniqueId made on rank 0, to be broadcast to the other ranks. */
kvq_status kvq_get_unique_id(void* out_128_bytes);
/* Joins the communicator (blocking until all nranks joined) on the CURRENT CUDA device. */
kvq_status kvq_comm_create(const void* unique_id, int32_t nranks, int32_t rank, kvq_comm** out);
kvq_status kvq_comm_destroy(kvq_comm* comm);
/* Device workspace bytes for ulysses_chunk_attention on this rank: chunk T_c tokens (T_c % P
 * == 0), H heads in total, exchange mode as above, Q/K/V in in_dtype, O in out_dtype. */
size_t kvq_ulysses_workspace_bytes(int32_t T_c, int32_t H, int32_t d, int32_t P, int32_t rank,
                                   int32_t exchange, kvq_dtype in_dtype, kvq_dtype out_dtype);
/* Binds the total head count H, the exchange mode and a caller-owned dev workspace (256-byte
 * aligned, >= kvq_ulysses_workspace_bytes for the shapes used; KVQ_ECAPACITY at the call
 * otherwise) to the comm. */
kvq_status kvq_comm_configure(kvq_comm* comm, int32_t num_heads, int32_t exchange,
                              void* dev_workspace, size_t workspace_bytes);
/* The chunk step of one rank: Q/K/V_shard dev [T_c/P, H, d] in_dtype (this rank's sequence
 * shard; T_c = P * (T_c/P) must equal the cache's chunk length), cache = this rank's heads
 * [h0, h1) of kvq_head_partition (else KVQ_ESHAPE) -> exchange -> quantize/append chunk
 * `chunk_index` of `layer` -> chunk_attention over `mask` -> exchange of O back ->
 * O_shard dev [T_c/P, H, d] out_dtype.  Codes and scales equal those of a 1-GPU cache of all
 * heads (the amax is global).  KVQ_ENCCL if a collective fails; K-smoothing caches need
 * exchange >= 1 (the shard amax of K is not that of K - mean) -> KVQ_EINVAL otherwise.
 * Every argument and cache-side error (chunk not appendable, no free slot, a mask chunk not
 * resident after the append's evictions) is returned before the first collective is issued, so
 * a rank that fails never leaves its peers blocked in a collective -- provided every rank passes
 * the same layer, chunk_index and mask.  Not supported inside CUDA graph capture: a capture and
 * replay of the world-1 step (NCCL send/recv to self) did not complete on the B200 box; the
 * single-GPU calls (kv_quantize_append, chunk_attention, chunk_attention_append) are capturable
 * and replay-tested. */
kvq_status ulysses_chunk_attention(kvq_comm* comm, kvq_cache* cache, int32_t layer,
                                   int64_t chunk_index, const void* Q_shard, const void* K_shard,
                                   const void* V_shard, kvq_dtype in_dtype, const kvq_mask* mask,
                                   float softmax_scale, void* O_shard, kvq_dtype out_dtype,
                                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KVQ_H_ */

// Library-owned NCCL communicator and the one-call head-sharded chunk step (include/kvq.h,
// "One-call head-sharded chunk step"; App. C: z^(p) in
// R^{L/P x H x d} --All-to-All--> R^{L x H/P x d}, attention on the local heads, a second
// All-to-All back; App. D for the NVFP4 payload).
//
// Host orchestration only: every arithmetic step is one of the library's kernels (pack / unpack /
// shard amax / quantize-append / attention); NCCL moves the bytes (grouped ncclSend/ncclRecv =
// all-to-allv, since 12 heads over 8 ranks are unequal) on the caller's stream.
#include <cstring>
#include <new>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/kvq.h"
#include "internal.h"

struct kvq_comm {
  ncclComm_t nc = nullptr;
  int32_t P = 0, rank = 0;
  int32_t exchange = -1, H = 0;
  uint8_t* ws = nullptr;
  size_t ws_bytes = 0;
};

namespace {

size_t esize(kvq_dtype t) { return t == KVQ_FP32 ? 4 : 2; }
size_t up256(size_t x) { return (x + 255) & ~size_t(255); }
int32_t heads_of(int32_t H, int32_t P, int32_t r) {
  int32_t h0, h1;
  kvq_head_partition(H, P, r, &h0, &h1);
  return h1 - h0;
}

// Workspace regions, each 256-byte aligned; the same function sizes and carves it.
struct Ws {
  size_t send, recv, scratch, q, k, v, amax, qscale, o_local, o_recv, total;
  size_t send_off[65];  // per-destination offsets in the send region
  size_t seg_in;        // bytes received from each source
};

Ws carve(int32_t T_c, int32_t H, int32_t d, int32_t P, int32_t rank, int32_t exchange, kvq_dtype in_dtype,
         kvq_dtype out_dtype, int32_t k_smoothing) {
  Ws w{};
  const int32_t Ts = T_c / P, Hr = heads_of(H, P, rank);
  const bool nv = exchange != KVQ_EXCHANGE_INPUT, qn = exchange == KVQ_EXCHANGE_NVFP4_Q;
  size_t o = 0, s = 0;
  for (int32_t p = 0; p < P; ++p) {
    w.send_off[p] = s;
    s += nv ? kvq_ulysses_nvfp4_bytes(Ts, H, d, P, p, in_dtype, k_smoothing, qn)
            : kvq_ulysses_qkv_bytes(Ts, H, d, P, p, in_dtype);
  }
  w.send_off[P] = s;
  w.seg_in = nv ? kvq_ulysses_nvfp4_bytes(Ts, H, d, P, rank, in_dtype, k_smoothing, qn)
                : kvq_ulysses_qkv_bytes(Ts, H, d, P, rank, in_dtype);
  const size_t act = (size_t)T_c * Hr * d;
  const size_t scratch = nv ? kvq_ulysses_shard_scratch_bytes(Ts, H) : 8192;
  w.send = o; o += up256(s);
  w.recv = o; o += up256(w.seg_in * P);
  w.scratch = o; o += up256(scratch);
  w.q = o; o += up256(act * (qn ? 2 : esize(in_dtype)));
  w.k = o; o += nv ? 0 : up256(act * esize(in_dtype));
  w.v = o; o += nv ? 0 : up256(act * esize(in_dtype));
  w.amax = o; o += 256;
  w.qscale = o; o += 256;
  w.o_local = o; o += up256(act * esize(out_dtype));
  w.o_recv = o; o += up256((size_t)Ts * H * d * esize(out_dtype));
  w.total = o;
  return w;
}

kvq_status nccl_status(ncclResult_t r) { return r == ncclSuccess ? KVQ_OK : KVQ_ENCCL; }

}  // namespace

extern "C" {

kvq_status kvq_get_unique_id(void* out_128_bytes) {
  if (!out_128_bytes) return KVQ_EINVAL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return KVQ_ENCCL;
  std::memcpy(out_128_bytes, &id, sizeof(id));
  return KVQ_OK;
}

kvq_status kvq_comm_create(const void* unique_id, int32_t nranks, int32_t rank, kvq_comm** out) {
  if (!unique_id || !out || nranks <= 0 || nranks > 64 || rank < 0 || rank >= nranks) return KVQ_EINVAL;
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  auto* c = new (std::nothrow) kvq_comm();
  if (!c) return KVQ_EINVAL;
  if (ncclCommInitRank(&c->nc, nranks, id, rank) != ncclSuccess) {
    delete c;
    return KVQ_ENCCL;
  }
  c->P = nranks;
  c->rank = rank;
  *out = c;
  return KVQ_OK;
}

kvq_status kvq_comm_destroy(kvq_comm* c) {
  if (!c) return KVQ_EINVAL;
  const ncclResult_t r = c->nc ? ncclCommDestroy(c->nc) : ncclSuccess;
  delete c;
  return nccl_status(r);
}

size_t kvq_ulysses_workspace_bytes(int32_t T_c, int32_t H, int32_t d, int32_t P, int32_t rank, int32_t exchange,
                                   kvq_dtype in_dtype, kvq_dtype out_dtype) {
  if (T_c <= 0 || H <= 0 || P <= 0 || P > 64 || rank < 0 || rank >= P || T_c % P) return 0;
  if (exchange < KVQ_EXCHANGE_INPUT || exchange > KVQ_EXCHANGE_NVFP4_Q) return 0;
  // sized for K-smoothing (its extra K-mean bytes) so one workspace serves both cache modes
  return carve(T_c, H, d, P, rank, exchange, in_dtype, out_dtype, 1).total;
}

kvq_status kvq_comm_configure(kvq_comm* c, int32_t num_heads, int32_t exchange, void* dev_workspace,
                              size_t workspace_bytes) {
  if (!c || num_heads < c->P || !dev_workspace || (reinterpret_cast<uintptr_t>(dev_workspace) & 255)) return KVQ_EINVAL;
  if (exchange < KVQ_EXCHANGE_INPUT || exchange > KVQ_EXCHANGE_NVFP4_Q) return KVQ_EINVAL;
  c->exchange = exchange;
  c->H = num_heads;
  c->ws = static_cast<uint8_t*>(dev_workspace);
  c->ws_bytes = workspace_bytes;
  return KVQ_OK;
}

kvq_status ulysses_chunk_attention(kvq_comm* c, kvq_cache* cache, int32_t layer, int64_t chunk_index,
                                   const void* Qs, const void* Ks, const void* Vs, kvq_dtype in_dtype,
                                   const kvq_mask* mask, float softmax_scale, void* O_shard, kvq_dtype out_dtype,
                                   void* stream) {
  if (!c || !cache || !Qs || !Ks || !Vs || !mask || !O_shard || c->exchange < 0 || !c->ws) return KVQ_EINVAL;
  if (in_dtype != KVQ_BF16 && in_dtype != KVQ_FP32) return KVQ_EDTYPE;
  if (out_dtype != KVQ_BF16 && out_dtype != KVQ_FP32) return KVQ_EDTYPE;
  kvq_config cfg;
  kvq_status st = kvq_cache_get_config(cache, &cfg);
  if (st != KVQ_OK) return st;
  const int32_t P = c->P, rank = c->rank, d = cfg.head_dim, Hr = cfg.num_heads;
  const int32_t T_c = cfg.tokens_per_frame * cfg.frames_per_chunk;
  if (T_c % P) return KVQ_ESHAPE;
  const int32_t H = c->H, Ts = T_c / P;
  if (Hr != heads_of(H, P, rank)) return KVQ_ESHAPE;
  const int32_t ex = c->exchange;
  const bool nv = ex != KVQ_EXCHANGE_INPUT, qn = ex == KVQ_EXCHANGE_NVFP4_Q;
  if (cfg.k_smoothing && !nv) return KVQ_EINVAL;
  const Ws w = carve(T_c, H, d, P, rank, ex, in_dtype, out_dtype, cfg.k_smoothing);
  if (carve(T_c, H, d, P, rank, ex, in_dtype, out_dtype, 1).total > c->ws_bytes) return KVQ_ECAPACITY;
  uint8_t* ws = c->ws;
  // every cache-side error (slot, eviction, mask residency) is raised here, before the first collective
  if ((st = kvq::validate_append_attend(cache, layer, chunk_index, mask)) != KVQ_OK) return st;
  float* amax = reinterpret_cast<float*>(ws + w.amax);  // [K, V, Q]
  float* qscale = reinterpret_cast<float*>(ws + w.qscale);
  const cudaStream_t cs = static_cast<cudaStream_t>(stream);
  const size_t oes = esize(out_dtype);

  // ---- exchange in: sequence shard [Ts, H, d] -> all T_c tokens of heads [h0, h1)
  if (nv) {
    st = kvq_ulysses_shard_amax(Ks, Vs, in_dtype, Ts, H, d, cfg.k_smoothing, amax, ws + w.scratch, stream);
    if (st != KVQ_OK) return st;
    if (qn && (st = kvq_ulysses_q_amax(Qs, in_dtype, Ts, H, d, amax + 2, ws + w.scratch, stream)) != KVQ_OK) return st;
    st = nccl_status(ncclAllReduce(amax, amax, qn ? 3 : 2, ncclFloat32, ncclMax, c->nc, cs));
    if (st != KVQ_OK) return st;
    st = kvq_ulysses_pack_nvfp4(Qs, Ks, Vs, in_dtype, Ts, H, d, P, amax, qn ? amax + 2 : nullptr, cfg.scale_mode,
                                cfg.k_smoothing, ws + w.send, stream);
  } else {
    st = kvq_ulysses_pack_qkv(Qs, Ks, Vs, in_dtype, Ts, H, d, P, ws + w.send, ws + w.scratch, stream);
  }
  if (st != KVQ_OK) return st;
  ncclGroupStart();
  for (int32_t p = 0; p < P; ++p) {
    ncclSend(ws + w.send + w.send_off[p], w.send_off[p + 1] - w.send_off[p], ncclUint8, p, c->nc, cs);
    ncclRecv(ws + w.recv + (size_t)p * w.seg_in, w.seg_in, ncclUint8, p, c->nc, cs);
  }
  if ((st = nccl_status(ncclGroupEnd())) != KVQ_OK) return st;

  // ---- quantize/append on the local heads, attention
  void* O_local = ws + w.o_local;
  if (nv) {
    st = kv_append_ulysses_nvfp4(cache, layer, chunk_index, ws + w.recv, P, amax, qn ? amax + 2 : nullptr, ws + w.q,
                                 in_dtype, qn ? qscale : nullptr, stream);
    if (st != KVQ_OK) return st;
    st = qn ? chunk_attention_qscaled(cache, layer, ws + w.q, qscale, mask, softmax_scale, O_local, out_dtype, stream)
            : chunk_attention(cache, layer, ws + w.q, in_dtype, mask, softmax_scale, O_local, out_dtype, stream);
  } else {
    st = kvq_ulysses_unpack_qkv(ws + w.recv, in_dtype, Ts, Hr, d, P, ws + w.q, ws + w.k, ws + w.v, amax, stream);
    if (st != KVQ_OK) return st;
    st = kv_quantize_append_amax(cache, layer, chunk_index, ws + w.k, ws + w.v, in_dtype, amax, stream);
    if (st != KVQ_OK) return st;
    st = chunk_attention(cache, layer, ws + w.q, in_dtype, mask, softmax_scale, O_local, out_dtype, stream);
  }
  if (st != KVQ_OK) return st;

  // ---- exchange out: O_local [T_c, H_r, d] as P token blocks -> [Ts, H_p, d] from every p
  const size_t blk = (size_t)Ts * Hr * d * oes;
  ncclGroupStart();
  size_t off = 0;
  for (int32_t p = 0; p < P; ++p) {
    const size_t in_p = (size_t)Ts * heads_of(H, P, p) * d * oes;
    ncclSend(static_cast<uint8_t*>(O_local) + (size_t)p * blk, blk, ncclUint8, p, c->nc, cs);
    ncclRecv(ws + w.o_recv + off, in_p, ncclUint8, p, c->nc, cs);
    off += in_p;
  }
  if ((st = nccl_status(ncclGroupEnd())) != KVQ_OK) return st;
  return kvq_ulysses_unpack_o(ws + w.o_recv, out_dtype, Ts, H, d, P, O_shard, stream);
}

}  // extern "C"

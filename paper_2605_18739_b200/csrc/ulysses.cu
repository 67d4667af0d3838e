// ulysses.cu -- compute around the head-sharded (Ulysses) all-to-all of PAPER.md:556-564
// (App. C): z^(p) in R^{L/P x H x d} -> R^{L x H/P x d} before attention, and back after.
// The collective is NCCL (torch.distributed all_to_all_single over NVLink); these kernels pack
// the per-destination head blocks (with the shard's amax(K), amax(V) piggybacked so every
// owner takes alpha^FP32 over ALL heads -- readings Z2/Z18), unpack the received token blocks,
// and interleave the returned O heads.  All copies are 128-bit and coalesced on both sides.
#include "common.cuh"
#include "internal.h"

namespace kvq {
namespace {

struct PackParams {
  const uint8_t* x[3];
  uint8_t* send;
  const uint32_t* partials;  // [2][kNumPartials] amax of the local K, V shard
  int64_t seg_off[kMaxP];    // byte offset of destination p's segment
  int h0[kMaxP + 1];         // head partition
  uint8_t owner[256];        // head -> destination rank
  int Ts, H, d, es, P;
};

// n / dv for n < 2^24 via a float reciprocal and one-step integer correction (exact)
__device__ __forceinline__ uint32_t div_small_u(uint32_t n, uint32_t dv, float inv) {
  uint32_t q = (uint32_t)__float2int_rz((float)n * inv);
  if (q * dv > n) --q;
  if ((q + 1) * dv <= n) ++q;
  return q;
}

// 32-bit index math throughout (the launchers check byte offsets < 2^31 and rows < 2^24): 16-byte
// chunks per row are a power of two (d * es / 16 in {8, 16, 32}), rows / H by div_small_u
__global__ void __launch_bounds__(256) pack_kernel(const __grid_constant__ PackParams p) {
  const uint32_t cpr = (uint32_t)(p.d * p.es / 16), lc = (uint32_t)(__ffs((int)cpr) - 1);
  const uint32_t per_tensor = (uint32_t)p.Ts * (uint32_t)p.H * cpr;
  const uint32_t total = 3u * per_tensor;
  const float invH = 1.0f / (float)p.H;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t tsr = i >= 2u * per_tensor ? 2u : (i >= per_tensor ? 1u : 0u);
    const uint32_t rem = i - tsr * per_tensor;
    const uint32_t row = rem >> lc, c = rem & (cpr - 1u);
    const uint32_t t = div_small_u(row, (uint32_t)p.H, invH), h = row - t * (uint32_t)p.H;
    const int dst = p.owner[h];
    const int Hp = p.h0[dst + 1] - p.h0[dst];
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.x[tsr] + (size_t)row * (p.d * p.es)) + c);
    uint8_t* o = p.send + p.seg_off[dst] +
                 (size_t)(((tsr * (uint32_t)p.Ts + t) * (uint32_t)Hp + (h - (uint32_t)p.h0[dst])) * (uint32_t)(p.d * p.es));
    reinterpret_cast<uint4*>(o)[c] = v;
  }
  if (blockIdx.x == 0) {  // amax of the local shard -> every destination's trailer
    __shared__ uint32_t red[2][8];
    for (int tsr = 0; tsr < 2; ++tsr) {
      uint32_t m = 0;
      for (int k = threadIdx.x; k < kNumPartials; k += blockDim.x) m = max(m, p.partials[tsr * kNumPartials + k]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      if ((threadIdx.x & 31) == 0) red[tsr][threadIdx.x >> 5] = m;
    }
    __syncthreads();
    if (threadIdx.x < 2 * kMaxP && (threadIdx.x >> 1) < p.P) {
      const int tsr = threadIdx.x & 1, dst = threadIdx.x >> 1;
      uint32_t m = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = max(m, red[tsr][w]);
      const int Hp = p.h0[dst + 1] - p.h0[dst];
      uint32_t* trailer = reinterpret_cast<uint32_t*>(p.send + p.seg_off[dst] + 3 * (int64_t)p.Ts * Hp * p.d * p.es);
      trailer[tsr] = m;
      if (tsr == 0) {
        trailer[2] = 0;
        trailer[3] = 0;
      }
    }
  }
}

__global__ void __launch_bounds__(256) unpack_qkv_kernel(const uint8_t* recv, int Ts, int Hr, int d, int es, int P,
                                                         uint8_t* Q, uint8_t* K, uint8_t* V, float* amax_kv) {
  const int64_t blk = (int64_t)Ts * Hr * d * es;  // bytes of one tensor block from one source
  const int64_t seg = 3 * blk + 16;
  const uint32_t cpb = (uint32_t)(blk / 16);
  // blockIdx.y = (source, tensor) block: no index division at all
  const int src = (int)blockIdx.y / 3, tsr = (int)blockIdx.y - 3 * src;
  uint8_t* out = (tsr == 0 ? Q : (tsr == 1 ? K : V)) + src * blk;
  const uint4* in = reinterpret_cast<const uint4*>(recv + src * seg + tsr * blk);
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < cpb; c += gridDim.x * blockDim.x)
    reinterpret_cast<uint4*>(out)[c] = __ldg(in + c);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x < 2) {  // global amax = max over every source's shard amax
    uint32_t m = 0;
    for (int src = 0; src < P; ++src) m = max(m, reinterpret_cast<const uint32_t*>(recv + src * seg + 3 * blk)[threadIdx.x]);
    amax_kv[threadIdx.x] = __uint_as_float(m);
  }
}

struct UnpackOParams {
  const uint8_t* recv;
  uint8_t* out;
  int64_t src_off[kMaxP];
  int h0[kMaxP + 1];
  uint8_t owner[256];
  int Ts, H, d, es, P;
};

__global__ void __launch_bounds__(256) unpack_o_kernel(const __grid_constant__ UnpackOParams p) {
  const uint32_t cpr = (uint32_t)(p.d * p.es / 16), lc = (uint32_t)(__ffs((int)cpr) - 1);
  const uint32_t total = (uint32_t)p.Ts * (uint32_t)p.H * cpr;
  const float invH = 1.0f / (float)p.H;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t row = i >> lc, c = i & (cpr - 1u);
    const uint32_t t = div_small_u(row, (uint32_t)p.H, invH), h = row - t * (uint32_t)p.H;
    const int src = p.owner[h];
    const int Hp = p.h0[src + 1] - p.h0[src];
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.recv + p.src_off[src] +
                                                         (size_t)((t * (uint32_t)Hp + (h - (uint32_t)p.h0[src])) *
                                                                  (uint32_t)(p.d * p.es))) + c);
    reinterpret_cast<uint4*>(p.out + (size_t)row * (p.d * p.es))[c] = v;
  }
}

// NVFP4 exchange, receiving side: every source segment carries Ts tokens of this rank's Hr heads
// as Q rows, packed K/V codes + scale bytes (+ K means): scatter them into the cache slot
// (head-major rows h * head_stride_rows + src * Ts + t) and Q into [P*Ts, Hr, d]; g of the slot
// from the all-reduced amax (the sender quantized with the same g).
__global__ void __launch_bounds__(256) scatter_nvfp4_kernel(const __grid_constant__ ScatterNvfp4Params p) {
  if (p.arrive) {  // f4: every source's stores into this window have landed
    if (threadIdx.x == 0) {
      for (int s = 0; s < p.P; ++s) {
        unsigned long long a;
        for (;;) {
          asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(a) : "l"(p.arrive + s) : "memory");
          if (a >= p.arrive_target) break;
          __nanosleep(64);
        }
      }
    }
    __syncthreads();
  }
  // blockIdx.y = source; 32-bit index math within a source (chunks per Q / code row are powers of
  // two, rows / Hr by div_small_u; the launcher checks rows < 2^24 and segment bytes < 2^31)
  const uint32_t rows = (uint32_t)p.Ts * (uint32_t)p.Hr;  // per source
  const uint32_t qc = (uint32_t)(p.d * p.es / 16), cc = (uint32_t)(p.d / 2 / 16);  // chunks per Q / code row
  const uint32_t lq = (uint32_t)(__ffs((int)qc) - 1), lcc = (uint32_t)(__ffs((int)cc) - 1);
  const uint32_t per_src = rows * (qc + 2 * cc);
  const float invHr = 1.0f / (float)p.Hr;
  const int src = (int)blockIdx.y;
  const uint8_t* seg = p.recv + (int64_t)src * p.seg;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < per_src; r += gridDim.x * blockDim.x) {
    if (r < rows * qc) {  // Q chunk
      const uint32_t row = r >> lq, c = r & (qc - 1u);
      const uint32_t t = div_small_u(row, (uint32_t)p.Hr, invHr), h = row - t * (uint32_t)p.Hr;
      uint8_t* qdst = (uint8_t*)p.Q + (((int64_t)src * p.Ts + t) * p.Hr + h) * p.d * p.es;
      if (p.amax_q) {  // NVFP4 Q: 8 elements per 16-byte chunk of the fp16 row = dec(c) dec(s), exact
        const uint32_t w = *reinterpret_cast<const uint32_t*>(seg + p.lay.q + (size_t)row * (p.d / 2) + c * 4);
        const uint32_t sb = seg[p.lay.qs + (size_t)row * (p.d / 16) + c / 2];
        uint32_t o[4];
        dequant_word_f16(w, f16x2_from_e4m3x2(sb | (sb << 8)), o);
        reinterpret_cast<uint4*>(qdst)[c] = make_uint4(o[0], o[1], o[2], o[3]);
      } else {
        // __ldcg, not __ldg: with f4 the window is written by peers while this kernel runs (after the
        // acquire above), and the non-coherent path only suits data read-only for the kernel's lifetime
        reinterpret_cast<uint4*>(qdst)[c] = __ldcg(reinterpret_cast<const uint4*>(seg + p.lay.q + (size_t)row * p.d * p.es) + c);
      }
      continue;
    }
    uint32_t k = r - rows * qc;
    const int tsr = k >= rows * cc ? 1 : 0;
    k -= (uint32_t)tsr * rows * cc;
    const uint32_t row = k >> lcc, c = k & (cc - 1u);
    const uint32_t t = div_small_u(row, (uint32_t)p.Hr, invHr), h = row - t * (uint32_t)p.Hr;
    const int64_t orow = (int64_t)h * p.head_stride_rows + (int64_t)src * p.Ts + t;
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(seg + (tsr ? p.lay.vc : p.lay.kc) + (size_t)row * (p.d / 2)) + c);
    reinterpret_cast<uint4*>(p.codes[tsr] + orow * (p.d / 2))[c] = v;
    if (c == 0) {  // the row's scale bytes (d/16) and K mean
      const uint8_t* sc = seg + (tsr ? p.lay.vs : p.lay.ks) + (size_t)row * (p.d / 16);
      uint8_t* dst = p.scales[tsr] + orow * (p.d / 16);
      if (p.d == 128) *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(sc);
      else *reinterpret_cast<uint32_t*>(dst) = *reinterpret_cast<const uint32_t*>(sc);
      if (tsr == 0 && p.mean) p.mean[orow] = reinterpret_cast<const float*>(seg + p.lay.km)[row];
    }
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 2 && p.amax_q) {  // g_Q for the score scale
    const uint32_t qb = __float_as_uint(p.amax_q[0]) & 0x7FFFFFFFu;
    if (qb >= 0x7F800000u) atomicCAS(&p.status->code, 0, -6);
    else *p.q_scale_out = qb == 0 ? 1.0f : __fdiv_rn(__uint_as_float(qb), 2688.0f);
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x < 2) {
    uint32_t mb = 0;
    if (!p.amax)  // f4: the mailbox (complete: the senders read it before storing)
      for (int r = 0; r < p.P; ++r) mb = max(mb, (uint32_t)p.mailbox[2 * r + threadIdx.x] & 0x7FFFFFFFu);
    const uint32_t abits = (p.amax ? __float_as_uint(p.amax[threadIdx.x]) : mb) & 0x7FFFFFFFu;
    if (abits >= 0x7F800000u) {
      atomicCAS(&p.status->code, 0, -6);
    } else {
      const float amax = __uint_as_float(abits);
      p.g_out[threadIdx.x] = amax == 0.0f ? 1.0f : __fdiv_rn(amax, 2688.0f);
    }
  }
}

// f4: one thread waits for n peer-written words (see PeerWaitParams)
__global__ void peer_wait_kernel(const __grid_constant__ PeerWaitParams p) {
  if (threadIdx.x != 0) return;
  for (int i = 0; i < p.n; ++i) {
    for (;;) {
      unsigned long long a;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(a) : "l"(p.words + (int64_t)i * p.stride) : "memory");
      const bool ok = p.mode == 0 ? (a >> 32) == p.target : (p.mode == 1 ? a >= p.target : a == p.target);
      if (ok) break;
      __nanosleep(64);
    }
  }
}

// f4: this rank's shard amax, epoch-tagged, into its entry pair of every peer's mailbox
__global__ void peer_publish_kernel(const __grid_constant__ PeerPublishParams p) {
  const int r = threadIdx.x >> 1, t = threadIdx.x & 1;
  if (r < p.P) {
    const unsigned long long v = (p.epoch << 32) | (__float_as_uint(p.amax[t]) & 0x7FFFFFFFu);
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.mailbox[r] + t), "l"(v) : "memory");
  }
}

// f4: one thread stores `value` (an epoch) into every peer's flag for this rank, after making this
// rank's prior work (stream-ordered kernels) visible system-wide
__global__ void peer_signal_kernel(const __grid_constant__ PeerSignalParams p) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int r = 0; r < p.P; ++r)
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.slot[r]), "l"(p.value) : "memory");
  }
}

// f4: once every owner has signalled this epoch (its attention wrote O_local), pull this rank's token
// rows of every head from the owners' O_local over peer memory (L2-only loads)
__global__ void __launch_bounds__(256) peer_pull_o_kernel(const __grid_constant__ PeerPullParams p) {
  if (threadIdx.x == 0) {
    for (int r = 0; r < p.P; ++r) {
      unsigned long long a;
      for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(a) : "l"(p.flags + r) : "memory");
        if (a == p.epoch) break;
        __nanosleep(64);
      }
    }
  }
  __syncthreads();
  const uint32_t cpr = (uint32_t)(p.d * p.es / 16), lc = (uint32_t)(__ffs((int)cpr) - 1);
  const uint32_t total = (uint32_t)p.Ts * (uint32_t)p.H * cpr;
  const float invH = 1.0f / (float)p.H;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t row = i >> lc, c = i & (cpr - 1u);
    const uint32_t t = div_small_u(row, (uint32_t)p.H, invH), h = row - t * (uint32_t)p.H;
    const int r = p.owner[h];
    const int Hp = p.h0[r + 1] - p.h0[r];
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(p.o_src[r] + (((int64_t)p.rank * p.Ts + t) * Hp + (h - p.h0[r])) *
                                                                           p.d * p.es) + c);
    reinterpret_cast<uint4*>(p.out + (size_t)row * (p.d * p.es))[c] = v;
  }
}

int grid_for(int64_t work) {
  int64_t g = (work + 255) / 256;
  return (int)(g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g));
}

void partition_impl(int H, int P, int* h0, uint8_t* owner) {
  const int base = H / P, rem = H % P;
  h0[0] = 0;
  for (int r = 0; r < P; ++r) h0[r + 1] = h0[r] + base + (r < rem ? 1 : 0);
  for (int r = 0; r < P; ++r)
    for (int h = h0[r]; h < h0[r + 1]; ++h) owner[h] = (uint8_t)r;
}

}  // namespace

void ulysses_partition(int H, int P, int* h0, uint8_t* owner) { partition_impl(H, P, h0, owner); }

cudaError_t preload_peer_kernels() {  // see preload_quant_kernels
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, peer_wait_kernel);
  cudaFuncGetAttributes(&a, peer_publish_kernel);
  cudaFuncGetAttributes(&a, peer_signal_kernel);
  return cudaGetLastError();
}

cudaError_t launch_peer_wait(const PeerWaitParams& p, cudaStream_t st) {
  peer_wait_kernel<<<1, 32, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_peer_publish(const PeerPublishParams& p, cudaStream_t st) {
  peer_publish_kernel<<<1, 2 * kMaxP, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_peer_signal(const PeerSignalParams& p, cudaStream_t st) {
  peer_signal_kernel<<<1, 32, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_peer_pull_o(const PeerPullParams& p, cudaStream_t st) {
  if ((int64_t)p.Ts * p.H * p.d * p.es >= (1ll << 31) || (int64_t)p.Ts * p.H >= (1 << 24)) return cudaErrorInvalidValue;
  peer_pull_o_kernel<<<grid_for((int64_t)p.Ts * p.H * (p.d * p.es / 16)), 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_ulysses_scatter_nvfp4(const ScatterNvfp4Params& p, cudaStream_t st) {
  const int64_t per_src = (int64_t)p.Ts * p.Hr * (p.d * p.es / 16 + p.d / 16);
  if ((int64_t)p.Ts * p.Hr >= (1 << 24) || per_src >= (1ll << 31) || p.P < 1) return cudaErrorInvalidValue;
  int gx = (int)((per_src + 255) / 256);
  const int cap = (148 * 8 + p.P - 1) / p.P;
  gx = gx < 1 ? 1 : (gx > cap ? cap : gx);
  scatter_nvfp4_kernel<<<dim3(gx, p.P), 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_ulysses_pack(const void* Q, const void* K, const void* V, int dtype, int Ts, int H, int d, int P,
                                uint8_t* send, uint32_t* scratch, cudaStream_t st) {
  if (P > kMaxP || H > 256) return cudaErrorInvalidValue;
  const int es = dtype == DT_FP32 ? 4 : 2;
  cudaError_t e = launch_amax(K, V, dtype, (int64_t)Ts * H * d, scratch, reinterpret_cast<DevStatus*>(scratch + 2 * kNumPartials), st);
  if (e != cudaSuccess) return e;
  PackParams p{};
  p.x[0] = (const uint8_t*)Q;
  p.x[1] = (const uint8_t*)K;
  p.x[2] = (const uint8_t*)V;
  p.send = send;
  p.partials = scratch;
  partition_impl(H, P, p.h0, p.owner);
  int64_t off = 0;
  for (int r = 0; r < P; ++r) {
    p.seg_off[r] = off;
    off += 3 * (int64_t)Ts * (p.h0[r + 1] - p.h0[r]) * d * es + 16;
  }
  p.Ts = Ts;
  p.H = H;
  p.d = d;
  p.es = es;
  p.P = P;
  // 32-bit index math in the kernel: every byte offset < 2^31, rows < 2^24
  if (3 * (int64_t)Ts * H * d * es >= (1ll << 31) || (int64_t)Ts * H >= (1 << 24)) return cudaErrorInvalidValue;
  pack_kernel<<<grid_for(3 * (int64_t)Ts * H * d * es / 16), 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_ulysses_unpack_qkv(const uint8_t* recv, int dtype, int Ts, int Hr, int d, int P, void* Q, void* K,
                                      void* V, float* amax_kv, cudaStream_t st) {
  const int es = dtype == DT_FP32 ? 4 : 2;
  const int64_t cpb = (int64_t)Ts * Hr * d * es / 16;
  if (cpb >= (1ll << 31) || P > kMaxP) return cudaErrorInvalidValue;
  int gx = (int)((cpb + 255) / 256);
  const int cap = (148 * 8 + 3 * P - 1) / (3 * P);
  gx = gx < 1 ? 1 : (gx > cap ? cap : gx);
  unpack_qkv_kernel<<<dim3(gx, 3 * P), 256, 0, st>>>(recv, Ts, Hr, d, es, P, (uint8_t*)Q, (uint8_t*)K, (uint8_t*)V,
                                                    amax_kv);
  return cudaGetLastError();
}

cudaError_t launch_ulysses_unpack_o(const uint8_t* recv, int dtype, int Ts, int H, int d, int P, void* O,
                                    cudaStream_t st) {
  if (P > kMaxP || H > 256) return cudaErrorInvalidValue;
  const int es = dtype == DT_FP32 ? 4 : 2;
  UnpackOParams p{};
  p.recv = recv;
  p.out = (uint8_t*)O;
  partition_impl(H, P, p.h0, p.owner);
  int64_t off = 0;
  for (int r = 0; r < P; ++r) {
    p.src_off[r] = off;
    off += (int64_t)Ts * (p.h0[r + 1] - p.h0[r]) * d * es;
  }
  p.Ts = Ts;
  p.H = H;
  p.d = d;
  p.es = es;
  p.P = P;
  if ((int64_t)Ts * H * d * es >= (1ll << 31) || (int64_t)Ts * H >= (1 << 24)) return cudaErrorInvalidValue;
  unpack_o_kernel<<<grid_for((int64_t)Ts * H * d * es / 16), 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace kvq

// quant.cu -- NVFP4 quantize/append, dequantize, export and codec probes (sm_100a).
//
// Quantize/append implements kv_quantize_append (include/kvq.h): PAPER.md:134-139 (§3.2, a KV
// chunk reshaped to (T_c H) x d and quantized independently), the NVFP4 format of PAPER.md:81-102
// (§2.2 Eq. 2; M^FP8 = 448, M^FP4 = 6) and the block scale alpha_i(6) = cast_E4M3(max|U_bar|/6)
// of PAPER.md:723-727 (App. F).  The fp32 operation order is reading Z4's definition R1
// (DESIGN.md §2): every divide / multiply is an IEEE round-to-nearest fp32 operation
// (__fdiv_rn / __fmul_rn; this TU is compiled with -fmad=false -ftz=false -prec-div=true).
//
// Two launches per append (both K and V in each, blockIdx.y = tensor):
//   1. amax_kernel   -- 128-bit coalesced loads, per-CTA max |x| (as bit patterns), non-finite
//                       detection with the first offending index.
//   2. quant_kernel  -- every CTA reduces the partials to the tensor amax, computes
//                       g = RN32(amax/2688); one thread per 16-element block: two/four 128-bit
//                       loads, block max, E4M3 scale, 16 E2M1 codes packed with the hardware
//                       cvt.rn.satfinite.e2m1x2.f32, one 8-byte code store + one scale byte into
//                       the head-major cache slot.  Pass-2 reads hit L2 (the chunk is 28.75 MB).
#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "quant_core.cuh"

namespace kvq {

namespace {

template <int DT>
__global__ void __launch_bounds__(256) amax_kernel(const void* K, const void* V, int64_t n, uint32_t* partials,
                                                   DevStatus* status, int tsr_base) {
  constexpr int kPer = DT == DT_BF16 ? 8 : 4;  // elements per 16-byte vector
  const int tsr = blockIdx.y + tsr_base;
  const uint8_t* x = (const uint8_t*)(tsr ? V : K);
  const int64_t nvec = n / kPer;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t m = 0;
  // 4 independent 128-bit loads in flight per thread per iteration
  for (; i + 3 * stride < nvec; i += 4 * stride) {
    uint4 a = ld_nc_v4(x + 16 * i), b = ld_nc_v4(x + 16 * (i + stride));
    uint4 c = ld_nc_v4(x + 16 * (i + 2 * stride)), d = ld_nc_v4(x + 16 * (i + 3 * stride));
    uint32_t ma = vec_absmax_bits<DT>(a), mb = vec_absmax_bits<DT>(b);
    uint32_t mc = vec_absmax_bits<DT>(c), md = vec_absmax_bits<DT>(d);
    uint32_t mm = max(max(ma, mb), max(mc, md));
    if (mm >= 0x7F800000u) {  // rare: locate the first non-finite element of these vectors
      for (int k = 0; k < 4; ++k) {
        uint4 v = ld_nc_v4(x + 16 * (i + k * stride));
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
        for (int e = 0; e < kPer; ++e) {
          uint32_t bits = DT == DT_BF16 ? ((w[e / 2] >> (16 * (e & 1))) & 0x7FFFu) << 16 : (w[e] & 0x7FFFFFFFu);
          if (bits >= 0x7F800000u) {
            atomicCAS(&status->code, 0, -6);
            atomicMin(&status->first_bad, (unsigned long long)(tsr * n + (i + k * stride) * kPer + e));
          }
        }
      }
    }
    m = max(m, mm);
  }
  for (; i < nvec; i += stride) {
    uint4 a = ld_nc_v4(x + 16 * i);
    uint32_t ma = vec_absmax_bits<DT>(a);
    if (ma >= 0x7F800000u) {
      uint32_t w[4] = {a.x, a.y, a.z, a.w};
      for (int e = 0; e < kPer; ++e) {
        uint32_t bits = DT == DT_BF16 ? ((w[e / 2] >> (16 * (e & 1))) & 0x7FFFu) << 16 : (w[e] & 0x7FFFFFFFu);
        if (bits >= 0x7F800000u) {
          atomicCAS(&status->code, 0, -6);
          atomicMin(&status->first_bad, (unsigned long long)(tsr * n + i * kPer + e));
        }
      }
    }
    m = max(m, ma);
  }
  __shared__ uint32_t red[8];
  m = warp_max_u32(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
    v = warp_max_u32(v);
    if (threadIdx.x == 0) partials[tsr * kNumPartials + blockIdx.x] = v;
  }
}

// Load the 16 elements of one block as fp32 (exact widening of bf16 / fp32).
template <int DT>
KVQ_DEV void load_block16(const uint8_t* src, float (&x)[16]) {
  if (DT == DT_BF16) {
    uint4 a = ld_nc_v4(src), b = ld_nc_v4(src + 16);
    uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x[2 * k] = __uint_as_float(w[k] << 16);
      x[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint4 a = ld_nc_v4(src + 16 * k);
      x[4 * k] = __uint_as_float(a.x);
      x[4 * k + 1] = __uint_as_float(a.y);
      x[4 * k + 2] = __uint_as_float(a.z);
      x[4 * k + 3] = __uint_as_float(a.w);
    }
  }
}

// K-smoothing, reading Z20: the row mean is the float32 sum in a fixed tree
// order times 1/d.  Within a 16-element block: y_k = x_k + x_{k+8}, z_k = y_k + y_{k+4},
// w_k = z_k + z_{k+2}, S = w_0 + w_1 (three FADD2 levels on element pairs, one FADD); across the
// d/16 blocks of a row (held by d/16 consecutive lanes): a butterfly, ((S0+S1)+(S2+S3))+... --
// every lane ends with the same bits because float addition is commutative.
KVQ_DEV float block_sum16(const float (&v)[16]) {
  uint64_t a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = f32x2_pack(v[2 * k], v[2 * k + 1]);
  const uint64_t c0 = fadd2(fadd2(a[0], a[4]), fadd2(a[2], a[6]));
  const uint64_t c1 = fadd2(fadd2(a[1], a[5]), fadd2(a[3], a[7]));
  float lo, hi;
  f32x2_unpack(fadd2(c0, c1), lo, hi);
  return __fadd_rn(lo, hi);
}

template <int KNB>
KVQ_DEV float row_mean(const float (&v)[16]) {
  float s = block_sum16(v);
#pragma unroll
  for (int o = 1; o < KNB; o <<= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  return __fmul_rn(s, 1.0f / (16 * KNB));  // exact: 1/d is a power of two
}

KVQ_DEV void subtract_mean(float (&v)[16], float m) {
  const uint64_t nm2 = f32x2_pack(-m, -m);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint64_t x2 = fadd2(f32x2_pack(v[2 * k], v[2 * k + 1]), nm2);  // RN32(x - m)
    f32x2_unpack(x2, v[2 * k], v[2 * k + 1]);
  }
}

// |x - m| max of a block as float bits; a non-finite mean (some x non-finite) -> +inf bits
KVQ_DEV uint32_t smoothed_absmax_bits(const float (&v)[16], float m) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = v[k];
  subtract_mean(x, m);
  float m0 = 0.0f, m1 = 0.0f;
#pragma unroll
  for (int k = 0; k < 16; k += 4) {
    m0 = fmax3(m0, fabsf(x[k]), fabsf(x[k + 1]));
    m1 = fmax3(m1, fabsf(x[k + 2]), fabsf(x[k + 3]));
  }
  const uint32_t bits = __float_as_uint(fmaxf(m0, m1));
  return fabsf(m) <= 3.402823466e38f ? bits : 0x7F800000u;
}

// bf16 -> fp32 (exact): the low element is w << 16, the high one w & 0xFFFF0000.  KVQ_UNPACK_PRMT of
// the 8 shifts are PRMTs on the ALU pipe, the rest IMAD.U32 on the FMA pipe, to balance the two
// pipes in the quantize loop (whose Markstein quotients are all FMA-pipe work).
// the 16 values of one block from its raw 16-byte words (2 for bf16, 4 for fp32) in registers
template <int DT>
KVQ_DEV void unpack_raw16(const uint4 (&r)[DT == DT_BF16 ? 2 : 4], float (&v)[16]) {
  if (DT == DT_BF16) {
    const uint32_t w[8] = {r[0].x, r[0].y, r[0].z, r[0].w, r[1].x, r[1].y, r[1].z, r[1].w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[2 * k] = __uint_as_float(k < KVQ_UNPACK_PRMT ? bf16lo_prmt(w[k]) : w[k] << 16);
      v[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 x = r[k];
      v[4 * k] = __uint_as_float(x.x); v[4 * k + 1] = __uint_as_float(x.y);
      v[4 * k + 2] = __uint_as_float(x.z); v[4 * k + 3] = __uint_as_float(x.w);
    }
  }
}

// Two-pass path, K with smoothing: per block (thread), row means by lane butterfly, written to the
// head-major mean slot; per-CTA max |K_bar| into partials[0][blockIdx.x] (grid = kNumPartials).
template <int DT, int D>
__global__ void __launch_bounds__(256) smooth_amax_kernel(const __grid_constant__ QuantParams p) {
  constexpr int kNB = D / 16;
  constexpr int kUB = 16 * (DT == DT_BF16 ? 2 : 4);
  const int64_t NU = (int64_t)p.rows * kNB;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t m = 0;
  // warp-uniform trip count: the row butterfly needs every lane
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < NU; base += stride) {
    const int64_t u = base + (threadIdx.x & 31);
    const bool valid = u < NU;
    float v[16];
    if (valid) {
      load_block16<DT>((const uint8_t*)p.x[0] + u * kUB, v);
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = 0.0f;
    }
    const float mean = row_mean<kNB>(v);
    if (valid) {
      m = max(m, smoothed_absmax_bits(v, mean));
      const int64_t row = u / kNB;
      if (u - row * kNB == 0) {
        const int64_t t_tok = row / p.H, h = row - t_tok * p.H;
        p.mean_out[h * p.head_stride_rows + t_tok] = mean;
      }
    }
  }
  __shared__ uint32_t red[8];
  m = warp_max_u32(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
    v = warp_max_u32(v);
    if (threadIdx.x == 0) p.partials_w[blockIdx.x] = v;
  }
}

// ---------------------------------------------------------------------------------------------
// Two-launch path, second pass (chunks too large for the single-pass kernel's shared memory, or
// forced for testing): after amax_kernel (or smooth_amax_kernel) has written per-CTA partials, every
// CTA reduces them to the tensor amax (or takes the caller's, Ulysses) and quantizes its block range
// from global memory (L2-resident after the first pass).  Per-block work as in quant_sp_kernel, with
// the decode scale and its reciprocal computed per block; blocks outside Markstein's range are
// queued and redone with IEEE divisions.
constexpr int kQ2Threads = 512;
#ifndef KVQ_Q2_DEPTH
#define KVQ_Q2_DEPTH 1  // quantize pass: iterations of input loaded ahead per thread (2 measured slower)
#endif
constexpr int kQ2NB = 2;  // blocks per thread per iteration

template <int DT, int D, int MODE>
#ifndef KVQ_Q2_MINB
#define KVQ_Q2_MINB 1  // CTAs per SM of the streaming pass (2: registers capped at 64, measured 12.2 vs 10.7 us)
#endif
__global__ void __launch_bounds__(kQ2Threads, KVQ_Q2_MINB) quant2_kernel(const __grid_constant__ QuantParams p, int upc) {
  constexpr bool SEARCH = (MODE & kModeSearch) != 0;
  constexpr bool SMOOTH = (MODE & kModeSmoothK) != 0;
  constexpr int kNB = D / 16;
  constexpr int kUB = 16 * (DT == DT_BF16 ? 2 : 4);  // bytes per 16-element block
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint32_t s_am[2];
  __shared__ int s_nq;
  const int c = blockIdx.x, tid = threadIdx.x;
  const int64_t NU = (int64_t)p.rows * kNB;
  const int64_t u0 = (int64_t)c * upc;
  const int64_t left = NU - u0;
  const int nu = left <= 0 ? 0 : (left < upc ? (int)left : upc);
  uint32_t* queue = reinterpret_cast<uint32_t*>(sm);  // flagged block indices [upc]
  if (tid < 2) s_am[tid] = 0;
  if (tid == 0) s_nq = 0;
  __syncthreads();
  if (p.ext_amax) {  // caller-supplied amax (Ulysses); with smoothing, of K_bar
    if (tid < 2) s_am[tid] = __float_as_uint(p.ext_amax[tid]) & 0x7FFFFFFFu;
  } else {  // reduce the amax kernels' per-CTA partials
    uint32_t mk = 0, mv = 0;
    for (int k = tid; k < kNumPartials; k += kQ2Threads) {
      mk = max(mk, p.partials[k]);
      mv = max(mv, p.partials[kNumPartials + k]);
    }
    mk = warp_max_u32(mk);
    mv = warp_max_u32(mv);
    if ((tid & 31) == 0) {
      atomicMax(&s_am[0], mk);
      atomicMax(&s_am[1], mv);
    }
  }
  __syncthreads();
  for (int t = 0; t < 2; ++t) {
    const bool smooth_t = SMOOTH && t == 0;
    const uint8_t* s = (const uint8_t*)p.x[t] + u0 * kUB;
    const uint32_t abits = s_am[t];
    if (abits >= 0x7F800000u) {  // non-finite tensor: leave the chunk undefined, report
      if (tid == 0 && c == 0) atomicCAS(&p.status->code, 0, -6);
      for (int i = tid; i < nu * 16; i += kQ2Threads) {  // first offending element of this range
        const uint32_t bits = DT == DT_BF16 ? ((uint32_t)reinterpret_cast<const uint16_t*>(s)[i] & 0x7FFFu) << 16
                                            : reinterpret_cast<const uint32_t*>(s)[i] & 0x7FFFFFFFu;
        if (bits >= 0x7F800000u) atomicMin(&p.status->first_bad, (unsigned long long)(t * NU * 16 + u0 * 16 + i));
      }
      continue;
    }
    const float amax = __uint_as_float(abits);
    const float g = amax == 0.0f ? 1.0f : __fdiv_rn(amax, 2688.0f);
    const float rg = __frcp_rn(g);
    const uint32_t all_exact = g >= 0x1p-60f && g <= 0x1p60f ? 0u : (1u << kQ2NB) - 1;  // Markstein range
    const float invH = 1.0f / (float)p.H;
    if (c == 0 && tid == 0) p.g_out[t] = g;
    uint8_t* codes = p.codes[t];
    uint8_t* scales = p.scales[t];
    // the next iteration's input blocks are loaded into registers before this one is quantized, so
    // each thread keeps a load in flight while it computes (the loop is otherwise latency-bound)
    constexpr int kV4 = kUB / 16;  // 16-byte words per block
    constexpr int kStep = kQ2NB * kQ2Threads;
    uint4 raw[kQ2NB][kV4], raw2[kQ2NB][kV4];  // iterations i + kStep and (depth 2) i + 2 kStep
    auto load_raw = [&](int i0, uint4 (&r)[kQ2NB][kV4]) {
#pragma unroll
      for (int b = 0; b < kQ2NB; ++b) {
        const int ibb = i0 + b * kQ2Threads < nu ? i0 + b * kQ2Threads : i0;
#pragma unroll
        for (int w = 0; w < kV4; ++w) r[b][w] = __ldg(reinterpret_cast<const uint4*>(s + (size_t)ibb * kUB) + w);
      }
    };
    if (tid < nu) load_raw(tid, raw);
    if (KVQ_Q2_DEPTH > 1 && tid + kStep < nu) load_raw(tid + kStep, raw2);
    for (int i = tid; i < nu; i += kStep) {
      int ib[kQ2NB];
      int64_t orow[kQ2NB];
#pragma unroll
      for (int b = 0; b < kQ2NB; ++b) ib[b] = i + b * kQ2Threads < nu ? i + b * kQ2Threads : i;
      float v[kQ2NB][16];
#pragma unroll
      for (int b = 0; b < kQ2NB; ++b) unpack_raw16<DT>(raw[b], v[b]);
      if (KVQ_Q2_DEPTH > 1) {
#pragma unroll
        for (int b = 0; b < kQ2NB; ++b)
#pragma unroll
          for (int w = 0; w < kV4; ++w) raw[b][w] = raw2[b][w];
        if (i + 2 * kStep < nu) load_raw(i + 2 * kStep, raw2);
      } else if (i + kStep < nu) {
        load_raw(i + kStep, raw);
      }
#pragma unroll
      for (int b = 0; b < kQ2NB; ++b) {
        const uint32_t u = (uint32_t)u0 + (uint32_t)ib[b];  // 32-bit index math (rows * d/16 < 2^31)
        const uint32_t row = u / kNB;
        const uint32_t t_tok = div_small(row, (uint32_t)p.H, invH);
        orow[b] = (int64_t)(row - t_tok * (uint32_t)p.H) * p.head_stride_rows + t_tok;
        if (smooth_t) subtract_mean(v[b], p.mean_out[orow[b]]);
      }
      uint32_t sb[kQ2NB], w0[kQ2NB], w1[kQ2NB];
      const uint32_t flags = quantize_blocks_fast<kQ2NB, SEARCH>(v, g, rg, sb, w0, w1) | all_exact;
#pragma unroll
      for (int b = 0; b < kQ2NB; ++b) {
        if (b > 0 && ib[b] == ib[0]) break;
        if (flags & (1u << b)) queue[atomicAdd(&s_nq, 1)] = (uint32_t)ib[b];  // exact recompute below
        const int j = (int)(((uint32_t)u0 + (uint32_t)ib[b]) % kNB);
        *reinterpret_cast<uint2*>(codes + orow[b] * (D / 2) + j * 8) = make_uint2(w0[b], w1[b]);
        scales[orow[b] * kNB + j] = (uint8_t)sb[b];
      }
    }
    __syncthreads();
    // deferred exact path for flagged blocks (out-of-range scales only; one thread per block)
    const int nq = s_nq;
    for (int e = tid; e < nq; e += kQ2Threads) {
      const int ibk = (int)queue[e];
      const uint32_t u = (uint32_t)u0 + (uint32_t)ibk;
      const uint32_t row = u / kNB;
      const int j = (int)(u - row * kNB);
      const uint32_t t_tok = row / (uint32_t)p.H;
      const uint32_t h = row - t_tok * (uint32_t)p.H;
      const int64_t orw = (int64_t)h * p.head_stride_rows + t_tok;
      float v[16];
      unpack_block16<DT>(s + (size_t)ibk * kUB, v);
      if (smooth_t) subtract_mean(v, p.mean_out[orw]);
      uint32_t sbe, a, bb;
      quantize_block16_exact<SEARCH>(v, g, sbe, a, bb);
      *reinterpret_cast<uint2*>(codes + orw * (D / 2) + j * 8) = make_uint2(a, bb);
      scales[orw * kNB + j] = (uint8_t)sbe;
    }
    __syncthreads();
    if (tid == 0) s_nq = 0;
    __syncthreads();  // the reset must land before any thread enqueues a flagged block of the next tensor
  }
}

// ---------------------------------------------------------------------------------------------
// Single-pass quantize/append, pipelined (quant_sp_kernel; the default when the chunk fits in
// aggregate shared memory).  A cooperative grid of one CTA per SM; CTA c owns the contiguous
// block range [u0, u0 + nu) of both K and V (rows t-major, 16-element blocks) and stages it in
// shared memory with TMA bulk copies, so HBM is read exactly once.  The slice of each tensor is cut
// into kSpPieces pieces with their own mbarriers: all K pieces are requested at once, V piece k only
// when K piece k has landed, so the memory system serves K first and V streams in while K is being
// quantized.  Per tensor:
//   A. as pieces land: per-block max |x| (integer max on the bit patterns -- NaN-safe) -> smem, and
//      the slice max -> the CTA's barrier slot (epoch tag << 32 | max bits, one 64-bit store);
//   B. grid barrier: G threads of every CTA poll one slot each until its tag is this launch's; the
//      tensor amax gives g = RN32(amax / 2688) (reading Z1);
//   C. per E4M3 scale byte s a table of (d_b = RN32(dec(s) g), -RN32(1/d_b)) (128 entries, one
//      correctly rounded reciprocal each), then every block: t = RN32(bmax/g), u = RN32(t/6),
//      s = E4M3(u), codes E2M1(RN32(x/d_b)) by Markstein's correction with the
//      tabulated reciprocal -- bit-identical to definition R1 (reading Z4) -- packed and stored
//      head-major into the cache slot.
// Order: A(K) B(K) C(K) A(V) B(V) C(V).  The launch epoch lives on the device (the word after the
// CTA slots): every CTA reads it at start, CTA 0 advances it once the V barrier proves that all
// CTAs have read it -- so a captured graph can replay the same launch any number of times.
#ifndef KVQ_SP_THREADS
#define KVQ_SP_THREADS 512
#endif
#ifndef KVQ_SP_NB
#define KVQ_SP_NB 2
#endif
constexpr int kSpThreads = KVQ_SP_THREADS;
constexpr int kSpNB = KVQ_SP_NB;  // blocks per thread per iteration of the quantize loop
#ifndef KVQ_SP_PIECES
#define KVQ_SP_PIECES 4
#endif
#ifndef KVQ_SP_EXP
#define KVQ_SP_EXP 0      // timing experiments only (wrong results): 1 no stores, 2 no codes, 3 no smem loads, 4 skeleton, 5 no loop
#endif
#ifndef KVQ_SP_SLEEP
#define KVQ_SP_SLEEP 32   // barrier poll back-off (ns)
#endif
constexpr int kSpPieces = KVQ_SP_PIECES;
constexpr int kEpochLine = kMaxFusedCtas - 1;  // barrier line holding the device launch epoch

// 8 codes per word from a 16-element block given d_b and ny = -RN32(1/d_b) (see codes_markstein)
KVQ_DEV void codes_markstein_ny(const float (&v)[16], float db, float ny, uint32_t& w0, uint32_t& w1) {
  const uint64_t ny2 = f32x2_pack(ny, ny), db2 = f32x2_pack(db, db);
  float q[16];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint64_t x2 = f32x2_pack(v[2 * k], v[2 * k + 1]);
    const uint64_t q0 = fmul2(x2, ny2);
    const uint64_t e = ffma2(q0, db2, x2);
    const uint64_t q1 = ffma2(e, ny2, q0);
    f32x2_unpack(q1, q[2 * k], q[2 * k + 1]);
  }
  w0 = e2m1x8(q) ^ 0x88888888u;
  w1 = e2m1x8(q + 8) ^ 0x88888888u;
}

// max |x| of one staged 16-element block as fp32 bits (integer max: +inf/NaN stay >= 0x7F800000)
template <int DT>
KVQ_DEV uint32_t block_absmax_bits(uint32_t addr) {
  if (DT == DT_BF16) {
    const uint4 a = ld_shared_v4(addr), b = ld_shared_v4(addr + 16);
    uint32_t m2 = max_u16x2(a.x & 0x7FFF7FFFu, a.y & 0x7FFF7FFFu, a.z & 0x7FFF7FFFu);
    m2 = max_u16x2(m2, a.w & 0x7FFF7FFFu, b.x & 0x7FFF7FFFu);
    m2 = max_u16x2(m2, b.y & 0x7FFF7FFFu, b.z & 0x7FFF7FFFu);
    m2 = max_u16x2(m2, b.w & 0x7FFF7FFFu, 0u);
    return max((m2 & 0xFFFFu) << 16, m2 & 0xFFFF0000u);
  } else {
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) m = max(m, vec_absmax_bits<DT>(ld_shared_v4(addr + 16 * k)));
    return m;
  }
}

// (t, h) of a cache row, advanced by a fixed number of rows per step without division
struct RowCursor {
  uint32_t t, h;
  KVQ_DEV void advance(uint32_t dq, uint32_t dr, uint32_t H) {
    t += dq;
    h += dr;
    if (h >= H) { h -= H; ++t; }
  }
};

// per-CTA phase timeline (tools/trace_quant.py): compiled in only with -DKVQ_TRACE_BUILD=1
#if KVQ_TRACE_BUILD
#define SPTRACE(ev)                                                                      \
  do {                                                                                   \
    if (p.trace != nullptr && tid == 0 && c < 256) {                                     \
      unsigned long long t_;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
      p.trace[c * 16 + (ev)] = t_;                                                       \
    }                                                                                    \
  } while (0)
#else
#define SPTRACE(ev) \
  do {              \
  } while (0)
#endif

template <int DT, int D, int MODE>
__global__ void __launch_bounds__(kSpThreads, 1)
    quant_sp_kernel(const __grid_constant__ QuantParams p, unsigned long long* slots, int upc) {
  constexpr bool SEARCH = (MODE & kModeSearch) != 0;
  constexpr bool SMOOTH = (MODE & kModeSmoothK) != 0;
  constexpr int kNB = D / 16;
  constexpr int kUB = 16 * (DT == DT_BF16 ? 2 : 4);  // bytes per staged 16-element block
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[2][kSpPieces];
  __shared__ uint32_t red[2][kSpThreads / 32];
  __shared__ uint32_t s_am[2];
  __shared__ float2 tab[2][128];
  __shared__ float s_g[2], s_rg[2];
  __shared__ unsigned long long s_epoch;
  const int c = blockIdx.x, G = gridDim.x, tid = threadIdx.x;
  const int64_t NU = (int64_t)p.rows * kNB;
  const int64_t u0 = (int64_t)c * upc;
  const int nu = NU - u0 <= 0 ? 0 : (NU - u0 < upc ? (int)(NU - u0) : upc);
  const uint32_t slice = (uint32_t)upc * kUB;
  uint32_t* bm = reinterpret_cast<uint32_t*>(sm + 2 * (size_t)slice);  // [2][upc] block max bits
  float* s_mean = reinterpret_cast<float*>(bm + 2 * upc);             // SMOOTH: [upc / kNB] K row means
  int ppc = (nu + kSpPieces - 1) / kSpPieces;
  ppc = (ppc + kNB - 1) / kNB * kNB;  // pieces start on row boundaries
  const bool ext = p.ext_amax != nullptr;
  unsigned long long* epoch_word = slots + (size_t)kEpochLine * kSlotU64;
  auto piece_lo = [&](int k) { return min(k * ppc, nu); };
  auto issue = [&](int t, int k) {
    const int a = piece_lo(k), b = piece_lo(k + 1);
    if (b > a) {
      mbar_arrive_expect_tx(&bar[t][k], (uint32_t)(b - a) * kUB);
      bulk_g2s(sm + t * slice + (size_t)a * kUB, (const uint8_t*)p.x[t] + (u0 + a) * kUB, (uint32_t)(b - a) * kUB,
               &bar[t][k]);
    }
  };
  if (tid == 0) {
    for (int k = 0; k < kSpPieces; ++k) {
      mbar_init(&bar[0][k], 1);
      mbar_init(&bar[1][k], 1);
    }
    fence_mbar_init();
    unsigned long long e = 0;  // requested ahead of the chunk's TMA stream (not queued behind it)
    if (!ext) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(e) : "l"(epoch_word) : "memory");
    for (int k = 0; k < kSpPieces; ++k) issue(0, k);
    s_epoch = e;
  }
  SPTRACE(0);
  __syncthreads();
  const uint32_t tag = (uint32_t)(s_epoch + 1);
  const uint32_t sbase = smem_u32(sm);

  // ---- A(t): per-block max |x| as pieces land -> smem; slice max -> this CTA's slot
  // Threads [wt0, kSpThreads) do the work; with wt0 > 0 (V, single-pass barrier) the first warps
  // meanwhile poll K's barrier slots, so K's barrier resolves while V lands.
  auto phase_a = [&](int t, int wt0) {
    const uint32_t xs = sbase + (uint32_t)t * slice;
    uint32_t* bmt = bm + t * upc;
    const int wtid = tid - wt0, nw = kSpThreads - wt0;
    uint32_t m = 0;
    if (wtid < 0) {  // K barrier pollers (G threads poll one CTA slot each)
      uint32_t mg = 0;
      if (tid < G) {
        unsigned long long a;
        for (;;) {
          asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(slots + (size_t)tid * kSlotU64) : "memory");
          if ((uint32_t)(a >> 32) == tag) break;
          __nanosleep(KVQ_SP_SLEEP);
        }
        mg = (uint32_t)a;
      }
      mg = warp_max_u32(mg);
      if ((tid & 31) == 0) atomicMax(&s_am[0], mg);
    }
#pragma unroll 1
    for (int k = 0; k < kSpPieces && wtid >= 0; ++k) {
      const int a = piece_lo(k), b = piece_lo(k + 1);
      if (b <= a) break;
      mbar_wait(&bar[t][k], 0);
      if (t == 0 && tid == 0) issue(1, k);  // V piece k is requested once K piece k has landed
      if (SMOOTH && t == 0) {
        // row means (fixed fp32 tree order, reading Z20) need the kNB blocks of a row in one warp
        for (int base = a + (tid & ~31); base < b; base += kSpThreads) {
          const int i = base + (tid & 31);
          const bool valid = i < b;
          float v[16];
          if (valid) {
            unpack_block16<DT>(sm + (size_t)i * kUB, v);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = 0.0f;
          }
          const float mean = row_mean<kNB>(v);
          if (valid) {
            const uint32_t mb = smoothed_absmax_bits(v, mean);
            bmt[i] = mb;
            m = max(m, mb);
            if (i % kNB == 0) {
              s_mean[i / kNB] = mean;
              const int64_t row = (u0 + i) / kNB;
              const int64_t t_tok = row / p.H, h = row - t_tok * p.H;
              p.mean_out[h * p.head_stride_rows + t_tok] = mean;
            }
          }
        }
      } else {
        for (int i = a + wtid; i < b; i += nw) {
          const uint32_t mb = block_absmax_bits<DT>(xs + (uint32_t)i * kUB);
          bmt[i] = mb;
          m = max(m, mb);
        }
      }
    }
    SPTRACE(t == 0 ? 1 : 5);
    m = warp_max_u32(m);
    if ((tid & 31) == 0) red[t][tid >> 5] = m;
    __syncthreads();
    if (tid == 0) {
      uint32_t mm = 0;
      for (int w = 0; w < kSpThreads / 32; ++w) mm = max(mm, red[t][w]);
      if (!ext) {
        // the whole 32-byte sector is written (tag|max four times): a sector that is only partly
        // written holds no valid copy in L2, and a poll of it would wait for a DRAM fill
        const unsigned long long val = ((unsigned long long)tag << 32) | mm;
        unsigned long long* sec = slots + (size_t)c * kSlotU64 + 4 * t;
        asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %1};" ::"l"(sec), "l"(val) : "memory");
        asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %1};" ::"l"(sec + 2), "l"(val) : "memory");
      }
      s_am[t] = ext ? (__float_as_uint(p.ext_amax[t]) & 0x7FFFFFFFu) : 0u;
    }
    __syncthreads();
  };
  // ---- B(t): grid barrier on tensor t (G threads poll one CTA slot each)
  unsigned long long vpre = 0;  // V slot loaded ahead (at the start of K's quantization)
  auto phase_b = [&](int t) {
    if (ext) return;
    uint32_t mg = 0;
    if (tid < G) {
      unsigned long long a = t == 1 ? vpre : 0ull;
      while ((uint32_t)(a >> 32) != tag) {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(slots + (size_t)tid * kSlotU64 + 4 * t) : "memory");
        if ((uint32_t)(a >> 32) == tag) break;
        __nanosleep(KVQ_SP_SLEEP);
      }
      mg = (uint32_t)a;
    }
    if ((tid & ~31) < G) {
      mg = warp_max_u32(mg);
      if ((tid & 31) == 0) atomicMax(&s_am[t], mg);
    }
    __syncthreads();
    if (t == 1 && c == 0 && tid == 0)  // every CTA has read the epoch (it published V): advance it
      asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %1};\n st.relaxed.gpu.global.v2.u64 [%2], {%1, %1};"
                   ::"l"(epoch_word), "l"(s_epoch + 1), "l"(epoch_word + 2) : "memory");
    SPTRACE(t == 0 ? 6 : 2);
  };
  // ---- T(t0..t1): g = RN32(amax / 2688) and the decode-scale table per tensor
  auto phase_t = [&](int t0, int nt) {
    if (tid < 128 * nt) {
      const int t = t0 + (tid >> 7), e = tid & 127;
      const uint32_t abits = s_am[t];
      const float amax = __uint_as_float(abits);
      const float g = abits >= 0x7F800000u ? 1.0f : (amax == 0.0f ? 1.0f : __fdiv_rn(amax, 2688.0f));
      const float db = __fmul_rn(e4m3_to_f32((uint32_t)e), g);
      tab[t][e] = make_float2(db, e == 0 ? -1.0f : -__frcp_rn(db));
      if (e == 0) {
        s_g[t] = g;
        s_rg[t] = __frcp_rn(g);
        if (c == 0 && abits < 0x7F800000u) p.g_out[t] = g;
      }
    }
    __syncthreads();
    SPTRACE(8 + t0);
  };
  // ---- C (K, then V): quantize the staged slices (one code copy).
  constexpr uint32_t kRowsStep = kSpThreads / kNB;  // rows advanced per kSpThreads blocks
  const uint32_t H = (uint32_t)p.H, dq = kRowsStep / H, dr = kRowsStep % H;
  const uint32_t hs = (uint32_t)p.head_stride_rows;
  // output row orow = h * hs + t (head-major slot rows; < 2^26, so byte offsets fit in 32 bits)
  const uint32_t ostep = dq + dr * hs, owrap = 1u - H * hs;  // (mod 2^32) when h wraps past H
  const int j = tid % kNB;  // u0 is a multiple of kNB
  uint32_t ch0, orow0;
  {
    const uint32_t row0 = (uint32_t)(u0 + tid) / kNB;
    const uint32_t t0 = row0 / H;
    ch0 = row0 - t0 * H;
    orow0 = ch0 * hs + t0;
  }
  auto phase_c = [&](int t) {
    const bool smooth_t = SMOOTH && t == 0;
    const uint32_t* bmt = bm + t * upc;
    const uint8_t* xs_t = sm + t * slice;
    if (s_am[t] >= 0x7F800000u) {  // non-finite tensor: leave the chunk undefined, report the first index
      if (tid == 0 && c == 0) atomicCAS(&p.status->code, 0, -6);
      for (int i = tid; i < nu * 16; i += kSpThreads) {
        const uint32_t bits = DT == DT_BF16 ? ((uint32_t)reinterpret_cast<const uint16_t*>(xs_t)[i] & 0x7FFFu) << 16
                                            : reinterpret_cast<const uint32_t*>(xs_t)[i] & 0x7FFFFFFFu;
        if (bits >= 0x7F800000u) atomicMin(&p.status->first_bad, (unsigned long long)(t * NU * 16 + u0 * 16 + i));
      }
      return;
    }
    if (t == 0 && !ext && tid < G)  // V's slot, requested now and consumed after K's loop
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(vpre) : "l"(slots + (size_t)tid * kSlotU64 + 4) : "memory");
    const float g = s_g[t], rg = s_rg[t];
    const float2* tb = tab[t];
    uint8_t* codes = p.codes[t];
    uint8_t* scales = p.scales[t];
    uint32_t ch = ch0, orow = orow0;
    // Markstein's conditions (no under/overflow) hold for every block when 2^-55 <= g <= 2^60
    // (d_b >= 2^-9 g >= 2^-64); outside (amax < 2e-13 or > 3e21) every block takes the IEEE path
    if (!(g >= 0x1p-55f && g <= 0x1p60f)) {
#pragma unroll 1
      for (int i = tid; i < nu; i += kSpThreads) {
        const uint32_t row = (uint32_t)(u0 + i) / kNB, tt = row / H, hh = row - tt * H;
        const uint32_t ob = hh * hs + tt;
        float v[16];
        unpack_block16<DT>(xs_t + (size_t)i * kUB, v);
        if (smooth_t) subtract_mean(v, s_mean[i / kNB]);
        uint32_t sb, a0, a1;
        quantize_block16_exact<SEARCH>(v, g, sb, a0, a1);
        *reinterpret_cast<uint2*>(codes + (ob * (uint32_t)(D / 2) + (uint32_t)j * 8u)) = make_uint2(a0, a1);
        scales[ob * (uint32_t)kNB + (uint32_t)j] = (uint8_t)sb;
      }
      return;
    }
    int it_ = 0;
    for (int i = tid; i < (KVQ_SP_EXP == 5 ? 0 : nu); i += kSpNB * kSpThreads, ++it_) {
      if (it_ == 1) SPTRACE(10 + t);
      if (it_ == 2) SPTRACE(12 + t);
      float v[kSpNB][16];
      uint32_t sb[kSpNB], w0[kSpNB], w1[kSpNB], ob[kSpNB];
#pragma unroll
      for (int b = 0; b < kSpNB; ++b) {
        ob[b] = orow;
        ch += dr;
        orow += ostep;
        if (ch >= H) {
          ch -= H;
          orow += owrap;
        }
        const int ib = min(i + b * kSpThreads, nu - 1);
#if KVQ_SP_EXP == 4 || KVQ_SP_EXP == 6  // timing experiment: loop skeleton (cursor, block max load, stores (4))
        w0[b] = bmt[ib];
        w1[b] = w0[b] ^ 0x5555u;
        sb[b] = w0[b] & 0x7F;
        continue;
#endif
#if KVQ_SP_EXP == 7  // timing experiment: codes stores only (no scale-byte stores)
        sb[b] = 0;
#endif
#if KVQ_SP_EXP == 3  // timing experiment: no smem loads
#pragma unroll
        for (int e = 0; e < 16; ++e) v[b][e] = __uint_as_float(0x3F800000u + (uint32_t)(ib * 16 + e));
#else
        unpack_block16<DT>(xs_t + (size_t)ib * kUB, v[b]);
#endif
        if (smooth_t) subtract_mean(v[b], s_mean[ib / kNB]);
        const float bmax = __uint_as_float(bmt[ib]);
        const float tq = div_markstein(bmax, g, rg);
        uint32_t s = scale_byte(div_markstein(tq, 6.0f, 0.16666667163372040f), bmax);  // RN32(1/6)
        const float2 e = tb[s];
#if KVQ_SP_EXP == 2  // timing experiment: no element codes
        w0[b] = __float_as_uint(v[b][0] * e.x + v[b][5]);
        w1[b] = __float_as_uint(v[b][9] * e.y + v[b][15]);
#else
        codes_markstein_ny(v[b], e.x, e.y, w0[b], w1[b]);
#endif
        if (SEARCH) {  // Four-Over-Six: the 4-target scale wins when strictly better
          const uint32_t s4 = scale_byte(__fmul_rn(tq, 0.25f), bmax);
          if (s4 != s) {
            const float2 e4 = tb[s4];
            uint32_t a0, a1;
            codes_markstein_ny(v[b], e4.x, e4.y, a0, a1);
            if (block_sse(v[b], a0, a1, s4, g) < block_sse(v[b], w0[b], w1[b], s, g)) {
              s = s4;
              w0[b] = a0;
              w1[b] = a1;
            }
          }
        }
        const bool z = s == 0;
        w0[b] = z ? 0u : w0[b];
        w1[b] = z ? 0u : w1[b];
        sb[b] = s;
      }
#pragma unroll
      for (int b = 0; b < kSpNB; ++b) {
        if (i + b * kSpThreads < nu && ((KVQ_SP_EXP != 1 && KVQ_SP_EXP != 6) || w0[b] == 0x12345678u)) {
          *reinterpret_cast<uint2*>(codes + (ob[b] * (uint32_t)(D / 2) + (uint32_t)j * 8u)) = make_uint2(w0[b], w1[b]);
          if (KVQ_SP_EXP != 7) scales[ob[b] * (uint32_t)kNB + (uint32_t)j] = (uint8_t)sb[b];
        }
      }
    }
    SPTRACE(t == 0 ? 3 : 7);
  };
  // schedule: A(K), then A(V) on most warps while the first warps poll K's barrier (a barrier takes
  // ~1-2 us to resolve while the chunk's TMA stream is in flight), then (T C) for K with V's slots
  // requested at the start of K's loop, B(V), (T C) for V.  One code copy per phase (loops, not
  // unrolled): the instruction cache stays warm for the second tensor.
  phase_a(0, 0);
  const int npoll = ext ? 0 : (G + 31) & ~31;  // warps that poll K's slots during A(V)
  phase_a(1, npoll);
  if (!ext) SPTRACE(6);
#pragma unroll 1
  for (int t = 0; t < 2; ++t) {
    if (t == 1) phase_b(1);
    phase_t(t, 1);
    phase_c(t);
  }
}

#undef SPTRACE

// ---------------------------------------------------------------------------------------------
// NVFP4 payload for the Ulysses exchange (§8(f) f3; App. D: the all-to-all
// "performed entirely in the low-precision space").  The sender quantizes its sequence shard of K
// and V with the GLOBAL tensor scales (amax all-reduced over the ranks first, readings Z2/Z18), so
// the packed bytes it ships are exactly the bytes the 1-GPU cache holds for those rows: blocks run
// along d inside one (t, h) row, and rows never straddle ranks.  Q travels in its input dtype.

// reduce the per-CTA partials of amax_kernel / smooth_amax_kernel to the shard's [K, V] amax
__global__ void __launch_bounds__(256) reduce_partials_kernel(const uint32_t* partials, float* amax_out) {
  __shared__ uint32_t red[2][8];
  for (int t = 0; t < 2; ++t) {
    uint32_t m = 0;
    for (int k = threadIdx.x; k < kNumPartials; k += blockDim.x) m = max(m, partials[t * kNumPartials + k]);
    m = warp_max_u32(m);
    if ((threadIdx.x & 31) == 0) red[t][threadIdx.x >> 5] = m;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    uint32_t m = 0;
    for (int w = 0; w < 8; ++w) m = max(m, red[threadIdx.x][w]);
    amax_out[threadIdx.x] = __uint_as_float(m);  // bits of max |x| (inf/NaN bits stay non-finite)
  }
}

// One thread per 16-element block of K or V of the shard, blocks (t, h, j) with j fastest, so the
// d/16 blocks of a row sit in consecutive lanes (K-smoothing's row mean is a lane butterfly).
template <int DT, int D, int MODE>
__global__ void __launch_bounds__(256) pack_nvfp4_kernel(const __grid_constant__ PackNvfp4Params p) {
  constexpr bool SEARCH = (MODE & kModeSearch) != 0;
  constexpr bool SMOOTH = (MODE & kModeSmoothK) != 0;
  constexpr int kNB = D / 16;
  constexpr int kUB = 16 * (DT == DT_BF16 ? 2 : 4);
  constexpr int es = DT == DT_BF16 ? 2 : 4;
  const int64_t nblk = (int64_t)p.Ts * p.H * kNB;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool peer = p.mailbox != nullptr;
  __shared__ float s_amax[2];
  if (peer) {  // f4: the global amax = max over this rank's mailbox, once all P entries are this epoch's
    if (threadIdx.x < 2) {
      uint32_t m = 0;
      for (int r = 0; r < p.P; ++r) {
        unsigned long long a;
        for (;;) {
          asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(a) : "l"(p.mailbox + 2 * r + threadIdx.x) : "memory");
          if ((a >> 32) == (p.epoch & 0xFFFFFFFFull)) break;
          __nanosleep(64);
        }
        m = max(m, (uint32_t)a & 0x7FFFFFFFu);
      }
      s_amax[threadIdx.x] = __uint_as_float(m);
    }
    __syncthreads();
    if (p.g_out != nullptr && blockIdx.x == 0 && threadIdx.x < 2) {  // f4 direct: this rank's own slot g
      const uint32_t ab = __float_as_uint(s_amax[threadIdx.x]) & 0x7FFFFFFFu;
      if (ab >= 0x7F800000u) {
        if (p.status) atomicCAS(&p.status->code, 0, -6 /* KVQ_ENONFINITE */);
      } else {
        p.g_out[threadIdx.x] = ab == 0 ? 1.0f : __fdiv_rn(__uint_as_float(ab), 2688.0f);
      }
    }
  }
  // ---- Q rows: NVFP4 (plain R1, the global amax_q) or passed through (16-byte chunks)
  if (p.amax_q) {
    const uint32_t qbits = __float_as_uint(p.amax_q[0]) & 0x7FFFFFFFu;
    if (qbits < 0x7F800000u) {
      const float qa = __uint_as_float(qbits);
      const float g = qa == 0.0f ? 1.0f : __fdiv_rn(qa, 2688.0f);
      const float rg = __frcp_rn(g);
      const bool exact = !(g >= 0x1p-60f && g <= 0x1p60f);
      for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nblk; u += stride) {
        float v[1][16];
        unpack_block16<DT>((const uint8_t*)p.x[0] + u * kUB, v[0]);
        uint32_t sb[1], w0[1], w1[1];
        const uint32_t flags = exact ? 1u : quantize_blocks_fast<1, false>(v, g, rg, sb, w0, w1);
        if (flags) quantize_block16_exact<false>(v[0], g, sb[0], w0[0], w1[0]);
        const int64_t row = u / kNB;
        const int j = (int)(u - row * kNB);
        const int tt = (int)(row / p.H), h = (int)(row - (int64_t)tt * p.H);
        const int r = p.owner[h];
        const PackDest& ds = p.dst[r];
        const int64_t orow = (int64_t)tt * ds.q_ts + (int64_t)(h - p.h0[r]) * ds.q_hs;
        *reinterpret_cast<uint2*>(ds.q + orow * (D / 2) + j * 8) = make_uint2(w0[0], w1[0]);
        ds.qs[orow * kNB + j] = (uint8_t)sb[0];
      }
    }
  } else {
    constexpr int cpr = D * es / 16;
    const int64_t total = (int64_t)p.Ts * p.H * cpr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
      const int64_t row = i / cpr;
      const int cc = (int)(i - row * cpr);
      const int t = (int)(row / p.H), h = (int)(row - (int64_t)t * p.H);
      const int r = p.owner[h];
      const PackDest& ds = p.dst[r];
      const uint4 v = __ldg(reinterpret_cast<const uint4*>((const uint8_t*)p.x[0] + row * D * es) + cc);
      uint8_t* o = ds.q + ((int64_t)t * ds.q_ts + (int64_t)(h - p.h0[r]) * ds.q_hs) * D * es;
      reinterpret_cast<uint4*>(o)[cc] = v;
    }
  }
  // ---- K, V blocks -> codes + scale bytes (+ K row means) in the destination's segment
  for (int t = 0; t < 2; ++t) {
    const bool smooth_t = SMOOTH && t == 0;
    const uint32_t abits = __float_as_uint(peer ? s_amax[t] : p.amax[t]) & 0x7FFFFFFFu;
    if (abits >= 0x7F800000u) continue;  // non-finite: the receiver reports it, bytes undefined
    const float amax = __uint_as_float(abits);
    const float g = amax == 0.0f ? 1.0f : __fdiv_rn(amax, 2688.0f);
    const float rg = __frcp_rn(g);
    const bool exact = !(g >= 0x1p-60f && g <= 0x1p60f);
    const uint8_t* x = (const uint8_t*)p.x[1 + t];
    // warp-uniform trip count (the row butterfly needs every lane)
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < nblk; base += stride) {
      const int64_t u = base + (threadIdx.x & 31);
      const bool valid = u < nblk;
      float v[1][16];
      if (valid) {
        unpack_block16<DT>(x + u * kUB, v[0]);
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) v[0][e] = 0.0f;
      }
      float mean = 0.0f;
      if (smooth_t) {
        mean = row_mean<kNB>(v[0]);
        subtract_mean(v[0], mean);
      }
      if (!valid) continue;
      uint32_t sb[1], w0[1], w1[1];
      const uint32_t flags = exact ? 1u : quantize_blocks_fast<1, SEARCH>(v, g, rg, sb, w0, w1);
      if (flags) quantize_block16_exact<SEARCH>(v[0], g, sb[0], w0[0], w1[0]);
      const int64_t row = u / kNB;
      const int j = (int)(u - row * kNB);
      const int tt = (int)(row / p.H), h = (int)(row - (int64_t)tt * p.H);
      const int r = p.owner[h];
      const PackDest& ds = p.dst[r];
      const int64_t orow = (int64_t)tt * ds.kv_ts + (int64_t)(h - p.h0[r]) * ds.kv_hs;
      *reinterpret_cast<uint2*>((t ? ds.vc : ds.kc) + orow * (D / 2) + j * 8) = make_uint2(w0[0], w1[0]);
      (t ? ds.vs : ds.ks)[orow * kNB + j] = (uint8_t)sb[0];
      if (smooth_t && j == 0) ds.km[orow] = mean;
    }
  }
  if (peer) {  // this CTA's stores are done: make them visible system-wide, then count the arrival
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int r = 0; r < p.P; ++r)
        asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(p.arrive[r]) : "memory");
    }
  }
}

// Eq. 2: x^ = dec(c) dec(s) g.  dec(c) dec(s) is exact in fp32 (<= 7 significant
// bits), so one FMA with g (and the K-smoothing row mean, else -0) rounds the exact value once.
template <int D>
__global__ void __launch_bounds__(256) dequant_kernel(const __grid_constant__ DequantParams p) {
  constexpr int kNB = D / 16;
  const int tsr = blockIdx.y;
  const float g = p.g[tsr];
  const int64_t total = (int64_t)p.T * p.H * kNB;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < total; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = b / kNB;
    const int j = (int)(b - row * kNB);
    const int t = (int)(row / p.H), h = (int)(row - (int64_t)t * p.H);
    const int64_t srow = (int64_t)h * p.head_stride_rows + t;
    const uint2 c = *reinterpret_cast<const uint2*>(p.codes[tsr] + srow * (D / 2) + j * 8);
    const float s = e4m3_to_f32(p.scales[tsr][srow * kNB + j]);
    // K-smoothing restitution (reading Z20); else -0, the additive identity that keeps Eq. 2's
    // sign of zero (code 0x8 -> -0.0, reading Z6)
    const float m = (tsr == 0 && p.mean) ? p.mean[srow] : -0.0f;
    float o[16];
    uint32_t cw[2] = {c.x, c.y};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t h2 = f16x2_from_e2m1x2((cw[k >> 2] >> (8 * (k & 3))) & 0xFF);
      float lo = __half2float(__ushort_as_half((unsigned short)(h2 & 0xFFFF)));
      float hi = __half2float(__ushort_as_half((unsigned short)(h2 >> 16)));
      o[2 * k] = __fmaf_rn(__fmul_rn(lo, s), g, m);      // RN32(dec(c) dec(s) g + mean), one rounding
      o[2 * k + 1] = __fmaf_rn(__fmul_rn(hi, s), g, m);
    }
    if (p.out_dtype == DT_FP32) {
      float4* dst = reinterpret_cast<float4*>((float*)p.out[tsr] + row * D + j * 16);
#pragma unroll
      for (int k = 0; k < 4; ++k) dst[k] = make_float4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
    } else {
      uint32_t w[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        __nv_bfloat162 b2 = __floats2bfloat162_rn(o[2 * k], o[2 * k + 1]);
        w[k] = *reinterpret_cast<uint32_t*>(&b2);
      }
      uint4* dst = reinterpret_cast<uint4*>((__nv_bfloat16*)p.out[tsr] + row * D + j * 16);
      dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
      dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
  }
}

template <int D>
__global__ void __launch_bounds__(256) export_kernel(const __grid_constant__ ExportParams p) {
  constexpr int kNB = D / 16;
  const int tsr = blockIdx.y;
  const bool bytes = p.codes_out[tsr] != nullptr;  // false: K-smoothing means only
  if (bytes && blockIdx.x == 0 && threadIdx.x == 0) *p.g_out[tsr] = p.g[tsr];
  const int64_t total = (int64_t)p.T * p.H * kNB;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < total; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = b / kNB;
    const int j = (int)(b - row * kNB);
    const int t = (int)(row / p.H), h = (int)(row - (int64_t)t * p.H);
    const int64_t srow = (int64_t)h * p.head_stride_rows + t;
    if (bytes) {
      *reinterpret_cast<uint2*>(p.codes_out[tsr] + row * (D / 2) + j * 8) =
          *reinterpret_cast<const uint2*>(p.codes[tsr] + srow * (D / 2) + j * 8);
      p.scales_out[tsr][row * kNB + j] = p.scales[tsr][srow * kNB + j];
    }
    if (tsr == 0 && j == 0 && p.mean && p.mean_out) p.mean_out[row] = p.mean[srow];
  }
}

// The paper's unfused "parallel dequantization kernel": reconstruct K_eff into
// contiguous bf16 [n_keys, H, d] (bench comparison only).  g per segment slot.
struct WinSegs {
  AttnSeg seg[kMaxSegs];
  int64_t off[kMaxSegs + 1];
  int nseg;
};

template <int D>
__global__ void __launch_bounds__(256) dequant_window_kernel(const __grid_constant__ DequantParams p, const float* gtab,
                                                             const WinSegs ws) {
  constexpr int kNB = D / 16;
  const int tsr = blockIdx.y;
  const int64_t nkeys = ws.off[ws.nseg];
  const int64_t total = nkeys * p.H * kNB;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < total; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = b / kNB;
    const int j = (int)(b - row * kNB);
    const int64_t key = row / p.H;
    const int h = (int)(row - key * p.H);
    int s = 0;
    while (s + 1 < ws.nseg && ws.off[s + 1] <= key) ++s;
    const int64_t srow = (int64_t)h * p.head_stride_rows + (int64_t)ws.seg[s].slot * p.T + ws.seg[s].begin +
                         (key - ws.off[s]);
    const float g = gtab[ws.seg[s].slot * 2 + tsr];
    const uint2 c = *reinterpret_cast<const uint2*>(p.codes[tsr] + srow * (D / 2) + j * 8);
    const float sc = e4m3_to_f32(p.scales[tsr][srow * kNB + j]);
    const float m = (tsr == 0 && p.mean) ? p.mean[srow] : -0.0f;  // -0: keeps the sign of zero
    uint32_t cw[2] = {c.x, c.y}, w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t h2 = f16x2_from_e2m1x2((cw[k >> 2] >> (8 * (k & 3))) & 0xFF);
      float lo = __half2float(__ushort_as_half((unsigned short)(h2 & 0xFFFF)));
      float hi = __half2float(__ushort_as_half((unsigned short)(h2 >> 16)));
      __nv_bfloat162 b2 = __floats2bfloat162_rn(__fmaf_rn(__fmul_rn(lo, sc), g, m), __fmaf_rn(__fmul_rn(hi, sc), g, m));
      w[k] = *reinterpret_cast<uint32_t*>(&b2);
    }
    uint4* dst = reinterpret_cast<uint4*>((__nv_bfloat16*)p.out[tsr] + row * D + j * 16);
    dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
    dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
}

// Codec probes: 0 = E2M1 encode (fp32 pairs -> 1 code per element), 1 = E4M3 encode,
// 2 = E2M1 decode (byte -> 2 fp32: low nibble first), 3 = E4M3 decode (byte -> fp32).
__global__ void probe_kernel(int which, const void* in, void* out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (which == 0) {  // n = number of element pairs
      const float* f = (const float*)in;
      uint32_t byte = e2m1x2_from_f32(f[2 * i], f[2 * i + 1]);
      ((uint8_t*)out)[2 * i] = byte & 0xF;
      ((uint8_t*)out)[2 * i + 1] = byte >> 4;
    } else if (which == 1) {
      ((uint8_t*)out)[i] = (uint8_t)e4m3_from_f32(((const float*)in)[i]);
    } else if (which == 2) {
      uint32_t h2 = f16x2_from_e2m1x2(((const uint8_t*)in)[i]);
      ((float*)out)[2 * i] = __half2float(__ushort_as_half((unsigned short)(h2 & 0xFFFF)));
      ((float*)out)[2 * i + 1] = __half2float(__ushort_as_half((unsigned short)(h2 >> 16)));
    } else {
      ((float*)out)[i] = e4m3_to_f32(((const uint8_t*)in)[i]);
    }
  }
}

int grid_for(int64_t work, int per_cta) {
  int64_t g = (work + per_cta - 1) / per_cta;
  return (int)(g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g));
}

}  // namespace

cudaError_t launch_amax(const void* K, const void* V, int dtype, int64_t n, uint32_t* partials, DevStatus* status,
                        cudaStream_t st, int tsr_begin) {
  dim3 grid(kNumPartials, 2 - tsr_begin);
  if (dtype == DT_BF16)
    amax_kernel<DT_BF16><<<grid, 256, 0, st>>>(K, V, n, partials, status, tsr_begin);
  else
    amax_kernel<DT_FP32><<<grid, 256, 0, st>>>(K, V, n, partials, status, tsr_begin);
  return cudaGetLastError();
}

cudaError_t launch_smooth_amax(const QuantParams& p, cudaStream_t st) {
  if (p.dtype == DT_BF16) {
    if (p.d == 128) smooth_amax_kernel<DT_BF16, 128><<<kNumPartials, 256, 0, st>>>(p);
    else smooth_amax_kernel<DT_BF16, 64><<<kNumPartials, 256, 0, st>>>(p);
  } else {
    if (p.d == 128) smooth_amax_kernel<DT_FP32, 128><<<kNumPartials, 256, 0, st>>>(p);
    else smooth_amax_kernel<DT_FP32, 64><<<kNumPartials, 256, 0, st>>>(p);
  }
  return cudaGetLastError();
}

template <int DT, int D, int MODE>
cudaError_t launch_fused_t(const QuantParams& p, unsigned long long* counters, int sms, cudaStream_t st) {
  constexpr int kUB = 16 * (DT == DT_BF16 ? 2 : 4);
  const int64_t NU = (int64_t)p.rows * (D / 16);
  int upc = (int)((NU + sms - 1) / sms);
  if (upc < 64) upc = 64;
  upc = (upc + 7) & ~7;  // 128-byte aligned V slice, slices on row boundaries
  const int G = (int)((NU + upc - 1) / upc);
  // K, V slices + per-block max bits (+ K row means with smoothing)
  const size_t smem = (size_t)2 * upc * kUB + (size_t)2 * upc * sizeof(uint32_t) +
                      ((MODE & kModeSmoothK) ? (size_t)(upc / (D / 16)) * sizeof(float) : 0);
  auto kern = quant_sp_kernel<DT, D, MODE>;
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, kern);
  if (e != cudaSuccess) return e;
  if (smem + fa.sharedSizeBytes > 227 * 1024 || G >= kEpochLine) return cudaErrorNotSupported;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kSpThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: the grid barrier is safe
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // counters -> the barrier slots: [G] lines of kSlotU64 u64 (tag << 32 | amax bits) for K and V,
  // line kEpochLine = the device launch epoch
  return cudaLaunchKernelEx(&cfg, kern, p, counters, upc);
}

// second pass of the two-launch path (after the amax pass): per-block work as in the single-pass kernel
template <int DT, int D, int MODE>
cudaError_t launch_quant2_t(const QuantParams& p, int sms, cudaStream_t st) {
  const int64_t NU = (int64_t)p.rows * (D / 16);
  int64_t G = (int64_t)sms * KVQ_Q2_MINB;
  if ((NU + G - 1) / G > 8192) G = (NU + 8191) / 8192;  // flag queue <= 32 KB of smem
  int upc = (int)((NU + G - 1) / G);
  upc = (upc + 7) & ~7;  // slices start on row boundaries
  G = (NU + upc - 1) / upc;
  const size_t smem = (size_t)upc * sizeof(uint32_t);
  auto kern = quant2_kernel<DT, D, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)G, kQ2Threads, smem, st>>>(p, upc);
  return cudaGetLastError();
}

template <int DT, int D>
cudaError_t quant2_mode(const QuantParams& p, int sms, cudaStream_t st) {
  switch (p.mode & 3) {
    case 0: return launch_quant2_t<DT, D, 0>(p, sms, st);
    case 1: return launch_quant2_t<DT, D, 1>(p, sms, st);
    case 2: return launch_quant2_t<DT, D, 2>(p, sms, st);
    default: return launch_quant2_t<DT, D, 3>(p, sms, st);
  }
}

template <int DT, int D>
cudaError_t fused_mode(const QuantParams& p, unsigned long long* counters, int sms, cudaStream_t st) {
  switch (p.mode & 3) {
    case 0: return launch_fused_t<DT, D, 0>(p, counters, sms, st);
    case 1: return launch_fused_t<DT, D, 1>(p, counters, sms, st);
    case 2: return launch_fused_t<DT, D, 2>(p, counters, sms, st);
    default: return launch_fused_t<DT, D, 3>(p, counters, sms, st);
  }
}

cudaError_t launch_quantize2(const QuantParams& p, int sms, cudaStream_t st) {
  if (p.dtype == DT_BF16)
    return p.d == 128 ? quant2_mode<DT_BF16, 128>(p, sms, st) : quant2_mode<DT_BF16, 64>(p, sms, st);
  return p.d == 128 ? quant2_mode<DT_FP32, 128>(p, sms, st) : quant2_mode<DT_FP32, 64>(p, sms, st);
}

cudaError_t launch_quantize_fused(const QuantParams& p, unsigned long long* counters, uint32_t* partials, int sms,
                                  cudaStream_t st) {
  (void)partials;
  if (p.dtype == DT_BF16)
    return p.d == 128 ? fused_mode<DT_BF16, 128>(p, counters, sms, st) : fused_mode<DT_BF16, 64>(p, counters, sms, st);
  return p.d == 128 ? fused_mode<DT_FP32, 128>(p, counters, sms, st) : fused_mode<DT_FP32, 64>(p, counters, sms, st);
}

cudaError_t launch_dequantize(const DequantParams& p, cudaStream_t st) {
  dim3 grid(grid_for((int64_t)p.T * p.H * (p.d / 16), 256), 2);
  if (p.d == 128) dequant_kernel<128><<<grid, 256, 0, st>>>(p);
  else dequant_kernel<64><<<grid, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_export(const ExportParams& p, cudaStream_t st) {
  dim3 grid(grid_for((int64_t)p.T * p.H * (p.d / 16), 256), 2);
  if (p.d == 128) export_kernel<128><<<grid, 256, 0, st>>>(p);
  else export_kernel<64><<<grid, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_dequant_window(const DequantParams& base, const AttnSeg* segs, int nseg, void* Kout, void* Vout,
                                  cudaStream_t st) {
  // base.T carries T_pad (slot stride in rows); base.g carries the layer's g table
  WinSegs ws{};
  ws.nseg = nseg;
  ws.off[0] = 0;
  for (int s = 0; s < nseg; ++s) {
    ws.seg[s] = segs[s];
    ws.off[s + 1] = ws.off[s] + (segs[s].end - segs[s].begin);
  }
  DequantParams p = base;
  p.out[0] = Kout;
  p.out[1] = Vout;
  dim3 grid(grid_for(ws.off[nseg] * p.H * (p.d / 16), 256), 2);
  if (p.d == 128) dequant_window_kernel<128><<<grid, 256, 0, st>>>(p, base.g, ws);
  else dequant_window_kernel<64><<<grid, 256, 0, st>>>(p, base.g, ws);
  return cudaGetLastError();
}

cudaError_t launch_ulysses_shard_amax(const QuantParams& p, uint32_t* partials, float* amax_out, cudaStream_t st) {
  cudaError_t e;
  if (p.mode & kModeSmoothK) {  // K_bar partials (means to p.mean_out), then V's
    e = launch_smooth_amax(p, st);
    if (e == cudaSuccess) e = launch_amax(p.x[0], p.x[1], p.dtype, (int64_t)p.rows * p.d, partials, p.status, st, 1);
  } else {
    e = launch_amax(p.x[0], p.x[1], p.dtype, (int64_t)p.rows * p.d, partials, p.status, st);
  }
  if (e != cudaSuccess) return e;
  reduce_partials_kernel<<<1, 256, 0, st>>>(partials, amax_out);
  return cudaGetLastError();
}

template <int DT, int D>
cudaError_t pack_nvfp4_mode(const PackNvfp4Params& p, int grid, cudaStream_t st) {
  switch (p.mode & 3) {
    case 0: pack_nvfp4_kernel<DT, D, 0><<<grid, 256, 0, st>>>(p); break;
    case 1: pack_nvfp4_kernel<DT, D, 1><<<grid, 256, 0, st>>>(p); break;
    case 2: pack_nvfp4_kernel<DT, D, 2><<<grid, 256, 0, st>>>(p); break;
    default: pack_nvfp4_kernel<DT, D, 3><<<grid, 256, 0, st>>>(p); break;
  }
  return cudaGetLastError();
}

int ulysses_pack_grid(int Ts, int H, int d) { return grid_for((int64_t)Ts * H * (d / 16), 256); }

cudaError_t launch_ulysses_pack_nvfp4(const PackNvfp4Params& p, cudaStream_t st) {
  const int grid = ulysses_pack_grid(p.Ts, p.H, p.d);
  if (p.dtype == DT_BF16) return p.d == 128 ? pack_nvfp4_mode<DT_BF16, 128>(p, grid, st) : pack_nvfp4_mode<DT_BF16, 64>(p, grid, st);
  return p.d == 128 ? pack_nvfp4_mode<DT_FP32, 128>(p, grid, st) : pack_nvfp4_mode<DT_FP32, 64>(p, grid, st);
}

// Force the module load of every kernel the f4 exchange step launches (cudaFuncGetAttributes loads a
// lazily-loaded kernel): under CUDA lazy loading, the first launch of a kernel may wait for the
// device's in-flight work, which must never happen while a device-side wait is pending.
template <int DT, int D>
static void touch_pack(cudaFuncAttributes* a) {
  cudaFuncGetAttributes(a, pack_nvfp4_kernel<DT, D, 0>);
  cudaFuncGetAttributes(a, pack_nvfp4_kernel<DT, D, 1>);
  cudaFuncGetAttributes(a, pack_nvfp4_kernel<DT, D, 2>);
  cudaFuncGetAttributes(a, pack_nvfp4_kernel<DT, D, 3>);
  cudaFuncGetAttributes(a, smooth_amax_kernel<DT, D>);
}
cudaError_t preload_quant_kernels() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, amax_kernel<DT_BF16>);
  cudaFuncGetAttributes(&a, amax_kernel<DT_FP32>);
  cudaFuncGetAttributes(&a, reduce_partials_kernel);
  touch_pack<DT_BF16, 128>(&a);
  touch_pack<DT_BF16, 64>(&a);
  touch_pack<DT_FP32, 128>(&a);
  touch_pack<DT_FP32, 64>(&a);
  return cudaGetLastError();
}

cudaError_t launch_probe(int which, const void* in, void* out, int64_t n, cudaStream_t st) {
  probe_kernel<<<grid_for(n, 256), 256, 0, st>>>(which, in, out, n);
  return cudaGetLastError();
}

}  // namespace kvq

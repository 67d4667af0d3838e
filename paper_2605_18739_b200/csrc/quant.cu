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
#include "common.cuh"
#include "internal.h"

namespace kvq {

namespace {

KVQ_DEV uint4 ld_nc_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

KVQ_DEV uint32_t warp_max_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// |x| bit pattern of every lane of a 16-byte vector, max-reduced, as an fp32 bit pattern.
template <int DT>
KVQ_DEV uint32_t vec_absmax_bits(uint4 v) {
  if (DT == DT_BF16) {
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      m = max(m, (w[i] & 0x7FFFu) << 16);
      m = max(m, w[i] & 0x7FFF0000u);
    }
    return m;
  } else {
    return max(max(v.x & 0x7FFFFFFFu, v.y & 0x7FFFFFFFu), max(v.z & 0x7FFFFFFFu, v.w & 0x7FFFFFFFu));
  }
}

template <int DT>
__global__ void __launch_bounds__(256) amax_kernel(const void* K, const void* V, int64_t n, uint32_t* partials,
                                                   DevStatus* status) {
  constexpr int kPer = DT == DT_BF16 ? 8 : 4;  // elements per 16-byte vector
  const int tsr = blockIdx.y;
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

template <int DT, int D>
__global__ void __launch_bounds__(256) quant_kernel(const QuantParams p) {
  constexpr int kNB = D / 16;                 // blocks per row
  constexpr int kES = DT == DT_BF16 ? 2 : 4;  // input element bytes
  const int tsr = blockIdx.y;
  __shared__ uint32_t red[8];

  // ---- tensor amax -> g = RN32(amax / (448 * 6)) (reading Z1), amax = 0 -> 1
  uint32_t abits;
  if (p.ext_amax) {
    abits = __float_as_uint(p.ext_amax[tsr]) & 0x7FFFFFFFu;
  } else {
    uint32_t m = 0;
    for (int i = threadIdx.x; i < kNumPartials; i += blockDim.x) m = max(m, p.partials[tsr * kNumPartials + i]);
    m = warp_max_u32(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    m = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) m = max(m, red[w]);
    abits = m;
  }
  if (abits >= 0x7F800000u) {  // non-finite tensor: leave the chunk undefined, report
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(&p.status->code, 0, -6);
    return;
  }
  const float amax = __uint_as_float(abits);
  const float g = amax == 0.0f ? 1.0f : __fdiv_rn(amax, 2688.0f);
  if (blockIdx.x == 0 && threadIdx.x == 0) p.g_out[tsr] = g;

  const uint8_t* x = (const uint8_t*)p.x[tsr];
  uint8_t* codes = p.codes[tsr];
  uint8_t* scales = p.scales[tsr];
  const int64_t total = (int64_t)p.rows * kNB;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < total; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = b / kNB;
    const int j = (int)(b - row * kNB);
    float v[16];
    load_block16<DT>(x + (row * D + j * 16) * kES, v);
    float bmax = 0.0f;
#pragma unroll
    for (int k = 0; k < 16; ++k) bmax = fmaxf(bmax, fabsf(v[k]));
    uint32_t sbyte = 0, w0 = 0, w1 = 0;
    if (bmax > 0.0f) {
      // R1: t = RN32(bmax/g); u = RN32(t/6); s = E4M3_RNE_SAT(u); s = 0 -> 2^-9
      const float t = __fdiv_rn(bmax, g);
      const float u = __fdiv_rn(t, 6.0f);
      sbyte = e4m3_from_f32(u);
      if (sbyte == 0) sbyte = 1;
      // decode scale of Eq. 2: d_b = RN32(dec(s) * g); codes E2M1_RNE_SAT(RN32(x / d_b))
      const float db = __fmul_rn(e4m3_to_f32(sbyte), g);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        w0 |= e2m1x2_from_f32(__fdiv_rn(v[2 * k], db), __fdiv_rn(v[2 * k + 1], db)) << (8 * k);
        w1 |= e2m1x2_from_f32(__fdiv_rn(v[8 + 2 * k], db), __fdiv_rn(v[8 + 2 * k + 1], db)) << (8 * k);
      }
    }  // zero block: scale 0x00, codes 0x00 (reading Z5)
    const int t_tok = (int)(row / p.H);
    const int h = (int)(row - (int64_t)t_tok * p.H);
    const int64_t orow = (int64_t)h * p.head_stride_rows + t_tok;
    *reinterpret_cast<uint2*>(codes + orow * (D / 2) + j * 8) = make_uint2(w0, w1);
    scales[orow * kNB + j] = (uint8_t)sbyte;
  }
}

// Eq. 2: x^ = dec(c) dec(s) g.  dec(c) dec(s) is exact in fp32 (<= 7 significant
// bits), so one __fmul_rn by g gives RN32 of the exact product.
template <int D>
__global__ void __launch_bounds__(256) dequant_kernel(const DequantParams p) {
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
    float o[16];
    uint32_t cw[2] = {c.x, c.y};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t h2 = f16x2_from_e2m1x2((cw[k >> 2] >> (8 * (k & 3))) & 0xFF);
      float lo = __half2float(__ushort_as_half((unsigned short)(h2 & 0xFFFF)));
      float hi = __half2float(__ushort_as_half((unsigned short)(h2 >> 16)));
      o[2 * k] = __fmul_rn(__fmul_rn(lo, s), g);
      o[2 * k + 1] = __fmul_rn(__fmul_rn(hi, s), g);
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
__global__ void __launch_bounds__(256) export_kernel(const ExportParams p) {
  constexpr int kNB = D / 16;
  const int tsr = blockIdx.y;
  if (blockIdx.x == 0 && threadIdx.x == 0) *p.g_out[tsr] = p.g[tsr];
  const int64_t total = (int64_t)p.T * p.H * kNB;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < total; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = b / kNB;
    const int j = (int)(b - row * kNB);
    const int t = (int)(row / p.H), h = (int)(row - (int64_t)t * p.H);
    const int64_t srow = (int64_t)h * p.head_stride_rows + t;
    *reinterpret_cast<uint2*>(p.codes_out[tsr] + row * (D / 2) + j * 8) =
        *reinterpret_cast<const uint2*>(p.codes[tsr] + srow * (D / 2) + j * 8);
    p.scales_out[tsr][row * kNB + j] = p.scales[tsr][srow * kNB + j];
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
__global__ void __launch_bounds__(256) dequant_window_kernel(const DequantParams p, const float* gtab,
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
    uint32_t cw[2] = {c.x, c.y}, w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t h2 = f16x2_from_e2m1x2((cw[k >> 2] >> (8 * (k & 3))) & 0xFF);
      float lo = __half2float(__ushort_as_half((unsigned short)(h2 & 0xFFFF)));
      float hi = __half2float(__ushort_as_half((unsigned short)(h2 >> 16)));
      __nv_bfloat162 b2 = __floats2bfloat162_rn(__fmul_rn(__fmul_rn(lo, sc), g), __fmul_rn(__fmul_rn(hi, sc), g));
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
                        cudaStream_t st) {
  dim3 grid(kNumPartials, 2);
  if (dtype == DT_BF16)
    amax_kernel<DT_BF16><<<grid, 256, 0, st>>>(K, V, n, partials, status);
  else
    amax_kernel<DT_FP32><<<grid, 256, 0, st>>>(K, V, n, partials, status);
  return cudaGetLastError();
}

cudaError_t launch_quantize(const QuantParams& p, cudaStream_t st) {
  const int64_t blocks = (int64_t)p.rows * (p.d / 16);
  dim3 grid(grid_for(blocks, 256), 2);
  if (p.dtype == DT_BF16) {
    if (p.d == 128) quant_kernel<DT_BF16, 128><<<grid, 256, 0, st>>>(p);
    else quant_kernel<DT_BF16, 64><<<grid, 256, 0, st>>>(p);
  } else {
    if (p.d == 128) quant_kernel<DT_FP32, 128><<<grid, 256, 0, st>>>(p);
    else quant_kernel<DT_FP32, 64><<<grid, 256, 0, st>>>(p);
  }
  return cudaGetLastError();
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

cudaError_t launch_probe(int which, const void* in, void* out, int64_t n, cudaStream_t st) {
  probe_kernel<<<grid_for(n, 256), 256, 0, st>>>(which, in, out, n);
  return cudaGetLastError();
}

}  // namespace kvq

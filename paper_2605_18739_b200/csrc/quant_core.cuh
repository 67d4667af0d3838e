// quant_core.cuh -- the NVFP4 block quantizer of definition R1 (reading Z4) as
// inline device functions, shared by quant.cu (the append kernels) and attention.cu (the append fused
// into the attention launch).  Every fp32 operation is an explicit round-to-nearest intrinsic
// (__fmul_rn / __fmaf_rn / __fdiv_rn / __frcp_rn) or a single PTX instruction, so the results do
// not depend on the including TU's -fmad / -prec-div flags: both TUs produce the same bytes.
#pragma once
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
KVQ_DEV uint32_t max_u16x2(uint32_t a, uint32_t b, uint32_t c) {  // VIMNMX3.U16x2
  uint32_t r;
  asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  asm("max.u16x2 %0, %0, %1;" : "+r"(r) : "r"(c));
  return r;
}

template <int DT>
KVQ_DEV uint32_t vec_absmax_bits(uint4 v) {
  if (DT == DT_BF16) {
    // |bf16| bit patterns compare like unsigned 16-bit integers: packed 2-lane max
    const uint32_t m2 = max_u16x2(max_u16x2(v.x & 0x7FFF7FFFu, v.y & 0x7FFF7FFFu, v.z & 0x7FFF7FFFu),
                                  v.w & 0x7FFF7FFFu, 0u);
    return max((m2 & 0xFFFFu) << 16, m2 & 0xFFFF0000u);
  } else {
    return max(max(v.x & 0x7FFFFFFFu, v.y & 0x7FFFFFFFu), max(v.z & 0x7FFFFFFFu, v.w & 0x7FFFFFFFu));
  }
}


// Four E2M1 code bytes (8 elements, element 2k in the low nibble) from four fp32 pairs: ptxas merges
// the four cvt.rn.satfinite.e2m1x2 results into one register (F2FP ... PACK_AB_MERGE_C).
KVQ_DEV uint32_t e2m1x8(const float* q) {
  uint32_t r;
  asm("{ .reg .b8 e0, e1, e2, e3;\n cvt.rn.satfinite.e2m1x2.f32 e0, %2, %1;\n cvt.rn.satfinite.e2m1x2.f32 e1, %4, %3;\n"
      " cvt.rn.satfinite.e2m1x2.f32 e2, %6, %5;\n cvt.rn.satfinite.e2m1x2.f32 e3, %8, %7;\n mov.b32 %0, {e0, e1, e2, e3};\n}"
      : "=r"(r)
      : "f"(q[0]), "f"(q[1]), "f"(q[2]), "f"(q[3]), "f"(q[4]), "f"(q[5]), "f"(q[6]), "f"(q[7]));
  return r;
}

// n / dv for n < 2^24 via a float reciprocal and one-step integer correction (exact)
KVQ_DEV uint32_t div_small(uint32_t n, uint32_t dv, float inv) {
  uint32_t q = (uint32_t)__float2int_rz((float)n * inv);
  if (q * dv > n) --q;
  if ((q + 1) * dv <= n) ++q;
  return q;
}

// RN32(a / b) given rb = RN32(1 / b) (Markstein's theorem; see quantize_blocks_fast).
KVQ_DEV float div_markstein(float a, float b, float rb) {
  const float q0 = __fmul_rn(a, rb);
  return __fmaf_rn(__fmaf_rn(-q0, b, a), rb, q0);
}

// One 16-element block, definition R1 (reading Z4):
//   s = E4M3_RNE_SAT(RN32(RN32(bmax / g) / 6)) (0 -> 2^-9; zero block -> 0x00, codes 0x00),
//   d_b = RN32(dec(s) * g),  c = E2M1_RNE_SAT(RN32(x / d_b)).
// Every quotient is computed without a divide by Markstein's correction: with y = RN32(1/b) (a
// correctly rounded reciprocal) and q0 = RN32(a y) (within 1 ulp of a/b), the residual
// e = a - q0 b is exact under FMA and RN32(q0 + e y) = RN32(a/b) exactly (Muller et al.,
// Handbook of Floating-Point Arithmetic, Markstein's theorem; no overflow/underflow).  So the fast
// path is bit-identical to the definition, not merely close: 1/g is rounded once per CTA, 1/6 is a
// constant, 1/d_b is one rcp.rn per block, and each element costs one FMUL2 + two FFMA2 per pair.
// The element quotients are formed negated (y' = -1/d_b): q0' = x y', e = fma(q0', d_b, x),
// q1' = fma(e, y', q0') = -RN32(x/d_b) including the sign of zero (x = -0 gives q1' = +0), and the
// E2M1 codes of the negation are flipped back with one XOR per 8 codes.  The theorem's range
// conditions hold for 2^-60 <= g <= 2^60 (checked per tensor by the caller) and d_b >= 2^-64
// (checked here: bit b of the return value sends block b through quantize_block16_exact).
KVQ_DEV uint32_t scale_byte(float u, float bmax) {
  uint32_t s = e4m3_from_f32(u);
  if (s == 0) s = 1;              // SPEC.md:191 underflow promotion
  if (!(bmax > 0.0f)) s = 0;      // zero block (reading Z5)
  return s;
}

KVQ_DEV void codes_markstein(const float (&v)[16], float db, uint32_t& w0, uint32_t& w1) {
  const float ny = -__frcp_rn(db);
  const uint64_t ny2 = f32x2_pack(ny, ny), db2 = f32x2_pack(db, db);
  float q[16];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint64_t x2 = f32x2_pack(v[2 * k], v[2 * k + 1]);
    const uint64_t q0 = fmul2(x2, ny2);
    const uint64_t e = ffma2(q0, db2, x2);  // x + q0' d_b = x - q0 d_b, exact
    const uint64_t q1 = ffma2(e, ny2, q0);
    f32x2_unpack(q1, q[2 * k], q[2 * k + 1]);
  }
  w0 = e2m1x8(q) ^ 0x88888888u;
  w1 = e2m1x8(q + 8) ^ 0x88888888u;
}

// Squared reconstruction error of one block under (codes w0 w1, scale byte s) in float32, the
// quantity Four-Over-Six compares (reading Z21): r_i = RN32(x_i - dec(c_i) dec(s) g)
// (dec(c) dec(s) is exact in f16 -- <= 6 significant bits within [2^-10, 2688] -- and the FMA
// rounds once), A / B = FMA chains r_i^2 + acc over the even / odd elements in ascending order
// (one FFMA2 chain on element pairs), E = RN32(A + B).
KVQ_DEV float block_sse(const float (&v)[16], uint32_t w0, uint32_t w1, uint32_t s, float g) {
  const uint32_t s2 = f16x2_from_e4m3x2(s | (s << 8));
  uint32_t o[8];
  dequant_word_f16(w0, s2, *reinterpret_cast<uint32_t(*)[4]>(o));
  dequant_word_f16(w1, s2, *reinterpret_cast<uint32_t(*)[4]>(o + 4));
  const uint64_t ng2 = f32x2_pack(-g, -g);
  uint64_t acc = f32x2_pack(0.0f, 0.0f);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float lo = __half2float(__ushort_as_half((unsigned short)(o[k] & 0xFFFF)));
    const float hi = __half2float(__ushort_as_half((unsigned short)(o[k] >> 16)));
    const uint64_t r = ffma2(f32x2_pack(lo, hi), ng2, f32x2_pack(v[2 * k], v[2 * k + 1]));
    acc = ffma2(r, r, acc);
  }
  float a, b;
  f32x2_unpack(acc, a, b);
  return __fadd_rn(a, b);
}

// NB blocks (independent streams for latency hiding).  SEARCH = Four-Over-Six:
// the 4-target candidate alpha_i(4) = cast_E4M3(RN32(t/4)) (t/4 is an exact scaling) replaces the
// 6-target one when its float32 error is strictly lower (ties to 6).
template <int NB, bool SEARCH>
KVQ_DEV uint32_t quantize_blocks_fast(const float (&v)[NB][16], float g, float rg, uint32_t (&sbyte)[NB],
                                      uint32_t (&w0)[NB], uint32_t (&w1)[NB]) {
  uint32_t flags = 0;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    float m0 = 0.0f, m1 = 0.0f;
#pragma unroll
    for (int k = 0; k < 16; k += 4) {
      m0 = fmax3(m0, fabsf(v[b][k]), fabsf(v[b][k + 1]));
      m1 = fmax3(m1, fabsf(v[b][k + 2]), fabsf(v[b][k + 3]));
    }
    const float bmax = fmaxf(m0, m1);
    const float t = div_markstein(bmax, g, rg);
    uint32_t s = scale_byte(div_markstein(t, 6.0f, 0.16666667163372040f), bmax);  // RN32(1/6)
    const float db = __fmul_rn(e4m3_to_f32(s), g);  // decode scale of Eq. 2
    codes_markstein(v[b], db, w0[b], w1[b]);
    if (s != 0 && !(db >= 0x1p-64f)) flags |= 1u << b;
    if (SEARCH) {
      const uint32_t s4 = scale_byte(__fmul_rn(t, 0.25f), bmax);
      if (s4 != s) {
        const float db4 = __fmul_rn(e4m3_to_f32(s4), g);
        uint32_t a0, a1;
        codes_markstein(v[b], db4, a0, a1);
        if (!(db4 >= 0x1p-64f)) flags |= 1u << b;
        if (block_sse(v[b], a0, a1, s4, g) < block_sse(v[b], w0[b], w1[b], s, g)) {
          s = s4;
          w0[b] = a0;
          w1[b] = a1;
        }
      }
    }
    sbyte[b] = s;
    if (s == 0) w0[b] = w1[b] = 0u;
  }
  return flags;
}

// The definition itself, with IEEE divisions (reading Z4, R1; Four-Over-Six as above): the
// reference path for flagged blocks.
KVQ_DEV void codes_exact(const float (&v)[16], float db, uint32_t& w0, uint32_t& w1) {
  float q[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) q[k] = __fdiv_rn(v[k], db);
  w0 = e2m1x8(q);
  w1 = e2m1x8(q + 8);
}

template <bool SEARCH>
KVQ_DEV void quantize_block16_exact(const float (&v)[16], float g, uint32_t& sbyte, uint32_t& w0, uint32_t& w1) {
  float bmax = 0.0f;
#pragma unroll
  for (int k = 0; k < 16; ++k) bmax = fmaxf(bmax, fabsf(v[k]));
  sbyte = 0;
  w0 = 0;
  w1 = 0;
  if (!(bmax > 0.0f)) return;
  const float t = __fdiv_rn(bmax, g);
  sbyte = scale_byte(__fdiv_rn(t, 6.0f), bmax);
  codes_exact(v, __fmul_rn(e4m3_to_f32(sbyte), g), w0, w1);
  if (SEARCH) {
    const uint32_t s4 = scale_byte(__fdiv_rn(t, 4.0f), bmax);
    if (s4 != sbyte) {
      uint32_t a0, a1;
      codes_exact(v, __fmul_rn(e4m3_to_f32(s4), g), a0, a1);
      if (block_sse(v, a0, a1, s4, g) < block_sse(v, w0, w1, sbyte, g)) {
        sbyte = s4;
        w0 = a0;
        w1 = a1;
      }
    }
  }
}


#ifndef KVQ_UNPACK_PRMT
#define KVQ_UNPACK_PRMT 4
#endif
KVQ_DEV uint32_t bf16lo_prmt(uint32_t w) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(r) : "r"(w));
  return r;
}

template <int DT>
KVQ_DEV void unpack_block16(const uint8_t* src, float (&v)[16]) {  // generic pointer (smem or global)
  if (DT == DT_BF16) {
    const uint4 x0 = *reinterpret_cast<const uint4*>(src), x1 = *reinterpret_cast<const uint4*>(src + 16);
    const uint32_t w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[2 * k] = __uint_as_float(k < KVQ_UNPACK_PRMT ? bf16lo_prmt(w[k]) : w[k] << 16);
      v[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 x = reinterpret_cast<const float4*>(src)[k];
      v[4 * k] = x.x; v[4 * k + 1] = x.y; v[4 * k + 2] = x.z; v[4 * k + 3] = x.w;
    }
  }
}


}  // namespace
}  // namespace kvq

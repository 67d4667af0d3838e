// attention.cu -- chunk attention over the NVFP4 KV cache with dequantization fused into the
// kernel, on tcgen05 tensor cores (sm_100a).
//
// Computes chunk_attention (include/kvq.h): for the current chunk's queries and head h,
//   O = softmax(Q K^T * scale) V over the effective key set K_eff(t)
// (§4.2; the cache of PAPER.md:134-146 §3.2), where K^, V^ are the
// NVFP4 values of Eq. 2.  Dequantization is fused (the paper's separate
// "parallel dequantization kernel", is prior art replaced here).
//
// Numerics: K^' = dec(code) * dec(s) and V^' likewise are EXACT in fp16, so the
// tensor cores see the exact quantized lattice; the FP32 tensor scales g_K, g_V are applied in
// fp32 outside the MMA (g_K in the exponent scale, g_V folded into the running O rescale).
// Q is rounded once to fp16, P is fp16, accumulation is fp32 in TMEM.
//
// Structure (v0 -- correctness first, one CTA per (128-query tile, head), 4 warps, thread i owns
// query row i = TMEM lane i):
//   per 128-key tile: all threads dequantize K/V rows into 128B-swizzled smem (UMMA K-major
//   layout; V's identical bytes are read through an MN-major descriptor) -> one thread issues
//   S = Q K^T (tcgen05.mma kind::f16, M=128 N=128, accumulator in TMEM) -> every thread loads
//   its S row from TMEM, online softmax, writes fp16 P back into TMEM over S -> one thread
//   issues O += P V (A operand from TMEM) -> next tile.  Epilogue O * g_V / l.
#include <cmath>

#include "common.cuh"
#include "internal.h"

namespace kvq {
namespace {

constexpr int kBM = 128;

template <int D>
struct AttnSmem {
  static constexpr int kTile = 128 * D * 2;  // 128 rows x D 16-bit values
  static constexpr int kQ = 0;
  static constexpr int kK = kTile;
  static constexpr int kV = 2 * kTile;
  static constexpr int kBar = 3 * kTile;
  static constexpr int kBytes = kBar + 64 + 1024;  // + barriers + alignment slack
};

// address of 16-byte chunk c (8 consecutive elements along d) of row r in a 128-row tile
KVQ_DEV uint32_t chunk_addr(uint32_t base, int r, int c) { return base + (uint32_t)(c >> 3) * 16384u + sw128_off(r, c & 7); }

// Dequantize one cache row (D values) into the tile: K^' = dec(code) * dec(s), exact in fp16.
template <int D>
KVQ_DEV void dequant_row_to_smem(uint32_t base, int r, const uint8_t* crow, const uint8_t* srow) {
  uint32_t cw[D / 8];
#pragma unroll
  for (int k = 0; k < D / 32; ++k) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(crow) + k);
    cw[4 * k] = v.x; cw[4 * k + 1] = v.y; cw[4 * k + 2] = v.z; cw[4 * k + 3] = v.w;
  }
  uint32_t sw[D / 64 > 0 ? D / 64 : 1];
  if (D == 128) {
    uint2 s2 = __ldg(reinterpret_cast<const uint2*>(srow));
    sw[0] = s2.x; sw[1] = s2.y;
  } else {
    sw[0] = __ldg(reinterpret_cast<const uint32_t*>(srow));
  }
#pragma unroll
  for (int j = 0; j < D / 16; ++j) {
    const uint32_t sb = (sw[j >> 2] >> (8 * (j & 3))) & 0xFFu;
    const uint32_t s2 = f16x2_from_e4m3x2(sb | (sb << 8));
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const uint32_t w = cw[2 * j + half];
      uint32_t o[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) o[b] = hmul2_u32(f16x2_from_e2m1x2((w >> (8 * b)) & 0xFF), s2);
      st_shared_v4(chunk_addr(base, r, 2 * j + half), o[0], o[1], o[2], o[3]);
    }
  }
}

// Copy one bf16 row (D values) into the tile (bf16-KV mode), zeros when !valid.
template <int D>
KVQ_DEV void copy_row_to_smem(uint32_t base, int r, const uint8_t* row, bool valid) {
#pragma unroll
  for (int c = 0; c < D / 8; ++c) {
    uint4 v = valid ? __ldg(reinterpret_cast<const uint4*>(row) + c) : make_uint4(0, 0, 0, 0);
    st_shared_v4(chunk_addr(base, r, c), v.x, v.y, v.z, v.w);
  }
}

KVQ_DEV uint32_t pack_half2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
KVQ_DEV uint32_t pack_bf162(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Q row -> fp16 (or bf16 in bf16-KV mode) into the tile
template <int D, bool MMA_BF16>
KVQ_DEV void load_q_row(uint32_t base, int r, const void* Q, int q_dtype, int64_t row_index, bool valid) {
#pragma unroll
  for (int c = 0; c < D / 8; ++c) {
    uint32_t o[4] = {0, 0, 0, 0};
    if (valid) {
      float f[8];
      if (q_dtype == DT_BF16) {
        uint4 v = __ldg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)Q + row_index * D) + c);
        if (MMA_BF16) {
          o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
        } else {
          uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            f[2 * k] = __uint_as_float(w[k] << 16);
            f[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) o[k] = pack_half2(f[2 * k], f[2 * k + 1]);
        }
      } else {
        const float4* src = reinterpret_cast<const float4*>((const float*)Q + row_index * D) + 2 * c;
        float4 a = __ldg(src), b = __ldg(src + 1);
        f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = MMA_BF16 ? pack_bf162(f[2 * k], f[2 * k + 1]) : pack_half2(f[2 * k], f[2 * k + 1]);
      }
    }
    st_shared_v4(chunk_addr(base, r, c), o[0], o[1], o[2], o[3]);
  }
}

template <int D, bool NVFP4, bool MMA_BF16>
__global__ void __launch_bounds__(128, 1) attn_kernel(const __grid_constant__ AttnParams p) {
  using SM = AttnSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_u32(smem + SM::kQ), sK = smem_u32(smem + SM::kK), sV = smem_u32(smem + SM::kV);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM::kBar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + SM::kBar + 16);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int h = blockIdx.y;
  const int q0 = blockIdx.x * kBM;
  const int H = p.H;

  if (warp == 0) tmem_alloc(tslot, 256);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  {
    const int t = q0 + tid;
    load_q_row<D, MMA_BF16>(sQ, tid, p.Q, p.q_dtype, (int64_t)t * H + h, t < p.Tq);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tO = tmem + 128;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  constexpr uint32_t kIdS = umma_idesc_f16(128, 128, MMA_BF16 ? 1 : 0, 0, 0);
  constexpr uint32_t kIdO = umma_idesc_f16(128, D, MMA_BF16 ? 1 : 0, 0, 1);

  float m_run = -INFINITY, l_run = 0.0f, gv_run = 1.0f;
  uint32_t phase = 0;
  int ntile = 0;

  for (int sgi = 0; sgi < p.nseg; ++sgi) {
    const AttnSeg sg = p.seg[sgi];
    for (int t0 = sg.begin & ~127; t0 < sg.end; t0 += 128) {
      const int lo = max(sg.begin - t0, 0), hi = min(sg.end - t0, 128);
      float gk = 1.0f, gv = 1.0f;
      // ---- K / V tile -> swizzled smem (thread tid owns key row tid of the tile)
      if (NVFP4) {
        const int64_t row = (int64_t)h * p.head_stride_rows + (int64_t)sg.slot * p.T_pad + t0 + tid;
        dequant_row_to_smem<D>(sK, tid, p.codes_k + row * (D / 2), p.scales_k + row * (D / 16));
        dequant_row_to_smem<D>(sV, tid, p.codes_v + row * (D / 2), p.scales_v + row * (D / 16));
        gk = __ldg(p.g + 2 * sg.slot);
        gv = __ldg(p.g + 2 * sg.slot + 1);
      } else {
        const int key = t0 + tid;
        const bool valid = key < sg.end;
        const int64_t off = ((int64_t)key * H + h) * D * 2;
        copy_row_to_smem<D>(sK, tid, (const uint8_t*)p.Kb + (valid ? off : 0), valid);
        copy_row_to_smem<D>(sV, tid, (const uint8_t*)p.Vb + (valid ? off : 0), valid);
      }
      fence_proxy_async_smem();
      __syncthreads();
      // ---- S = Q K^T  (M=128 queries, N=128 keys, K=D), fp32 in TMEM columns [0,128)
      if (tid == 0) {
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (uint32_t)(kk >> 2) * 16384u + (uint32_t)(kk & 3) * 32u;
          umma_ss(tS, umma_desc_sw128(sQ + off, 16, 1024), umma_desc_sw128(sK + off, 16, 1024), kIdS, kk > 0);
        }
        tc_commit(bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1;
      tc_fence_after();

      // ---- online softmax on this thread's row (TMEM lane = tid)
      uint32_t s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) KVQ_TMEM_LD32(tS + lane_off + 32 * c, (s + 32 * c));
      tmem_ld_wait();
      const float cs = gk * p.scale_log2;
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 128; ++j) {
        const float v = (j >= lo && j < hi) ? __uint_as_float(s[j]) * cs : -INFINITY;
        s[j] = __float_as_uint(v);
        mx = fmaxf(mx, v);
      }
      const float m_new = fmaxf(m_run, mx);
      const float alpha = ex2_approx(m_run - m_new);
      float lsum = 0.0f;
#pragma unroll
      for (int k = 0; k < 64; ++k) {
        const float p0 = ex2_approx(__uint_as_float(s[2 * k]) - m_new);
        const float p1 = ex2_approx(__uint_as_float(s[2 * k + 1]) - m_new);
        uint32_t pk;
        if (MMA_BF16) {
          pk = pack_bf162(p0, p1);
          lsum += __uint_as_float(pk << 16) + __uint_as_float(pk & 0xFFFF0000u);
        } else {
          pk = pack_half2(p0, p1);
          __half2 hh = *reinterpret_cast<__half2*>(&pk);
          lsum += __low2float(hh) + __high2float(hh);
        }
        s[k] = pk;
      }
      l_run = l_run * alpha + lsum;
      KVQ_TMEM_ST32(tS + lane_off, s);
      KVQ_TMEM_ST32(tS + lane_off + 32, (s + 32));
      // O is kept in units of the current chunk's g_V: rescale by alpha * g_V,prev / g_V,new
      if (ntile > 0) {
        const float f = alpha * (gv_run / gv);
        if (!__all_sync(0xffffffffu, f == 1.0f)) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            KVQ_TMEM_LD32(tO + lane_off + 32 * c, o);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * f);
            KVQ_TMEM_ST32(tO + lane_off + 32 * c, o);
          }
        }
      }
      gv_run = gv;
      m_run = m_new;
      tmem_st_wait();
      tc_fence_before();
      __syncthreads();
      // ---- O += P V  (A = P from TMEM columns [0,64), B = V^' MN-major in smem)
      if (tid == 0) {
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(tO, tS + 8 * kk, umma_desc_sw128(sV + kk * 2048, 16384, 1024), kIdO, (ntile > 0 || kk > 0) ? 1u : 0u);
        tc_commit(bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1;
      tc_fence_after();
      ntile++;
    }
  }

  // ---- epilogue: O * g_V / l -> [Tq, H, D]
  {
    const int t = q0 + tid;
    const float f = gv_run / l_run;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      KVQ_TMEM_LD32(tO + lane_off + 32 * c, o);
      tmem_ld_wait();
      if (t < p.Tq) {
        const int64_t base = ((int64_t)t * H + h) * D + 32 * c;
        if (p.out_dtype == DT_FP32) {
          float4* dst = reinterpret_cast<float4*>((float*)p.O + base);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            dst[k] = make_float4(__uint_as_float(o[4 * k]) * f, __uint_as_float(o[4 * k + 1]) * f,
                                 __uint_as_float(o[4 * k + 2]) * f, __uint_as_float(o[4 * k + 3]) * f);
        } else {
          uint4* dst = reinterpret_cast<uint4*>((__nv_bfloat16*)p.O + base);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            dst[k] = make_uint4(pack_bf162(__uint_as_float(o[8 * k]) * f, __uint_as_float(o[8 * k + 1]) * f),
                                pack_bf162(__uint_as_float(o[8 * k + 2]) * f, __uint_as_float(o[8 * k + 3]) * f),
                                pack_bf162(__uint_as_float(o[8 * k + 4]) * f, __uint_as_float(o[8 * k + 5]) * f),
                                pack_bf162(__uint_as_float(o[8 * k + 6]) * f, __uint_as_float(o[8 * k + 7]) * f));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

template <int D, bool NVFP4, bool MMA_BF16>
cudaError_t launch_t(const AttnParams& p, cudaStream_t st) {
  auto kern = attn_kernel<D, NVFP4, MMA_BF16>;
  const int smem = AttnSmem<D>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((p.Tq + kBM - 1) / kBM, p.H);
  kern<<<grid, 128, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention(const AttnParams& p, bool nvfp4_kv, cudaStream_t st) {
  if (nvfp4_kv) return p.d == 128 ? launch_t<128, true, false>(p, st) : launch_t<64, true, false>(p, st);
  return p.d == 128 ? launch_t<128, false, true>(p, st) : launch_t<64, false, true>(p, st);
}

}  // namespace kvq

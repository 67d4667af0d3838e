// Issue rate of the quantizer's instruction types on sm_100a: cycles per warp instruction per SM
// sub-partition, 4 warps per sub-partition, 8 independent chains per warp (development aid).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(512, 1) k(uint32_t* out, long long* cyc, int iters) {
  float a[8];
  uint32_t u[8];
  unsigned long long x2[8];
  for (int i = 0; i < 8; ++i) {
    a[i] = 1.0f + threadIdx.x * 1e-3f + i;
    u[i] = threadIdx.x * 7 + i;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x2[i]) : "f"(a[i]), "f"(a[i] * 0.5f));
  }
  const unsigned long long c2 = 0x3F8000003F800000ull;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) {  // 4 merged cvt e2m1x2 (F2FP.SATFINITE.E2M1 ... MERGE_C chain) + 1 LOP3
        uint32_t r;
        asm volatile("{ .reg .b8 e0, e1, e2, e3;\n cvt.rn.satfinite.e2m1x2.f32 e0, %1, %2;\n cvt.rn.satfinite.e2m1x2.f32 e1, %2, %1;\n"
                     " cvt.rn.satfinite.e2m1x2.f32 e2, %1, %1;\n cvt.rn.satfinite.e2m1x2.f32 e3, %2, %2;\n mov.b32 %0, {e0, e1, e2, e3};\n}"
                     : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        u[i] ^= r;
      } else if (OP == 1) {  // FFMA2 self chains
        asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(x2[i]) : "l"(c2));
      } else if (OP == 2) {  // FMUL2 self chains
        asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(x2[i]) : "l"(c2));
      } else if (OP == 3) {  // FFMA scalar
        asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]));
      } else if (OP == 4) {  // LOP3
        asm volatile("lop3.b32 %0, %0, %1, 0xFFFF0000, 0x80;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
      } else if (OP == 5) {  // 1 cvt e4m3x2 + 1 LOP3
        uint16_t r;
        asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        u[i] ^= r;
      } else if (OP == 6) {  // prmt
        asm volatile("prmt.b32 %0, %0, 0, 0x1044;" : "+r"(u[i]));
      } else if (OP == 7) {  // IMAD.U32 style shift (mul.lo by 65536)
        asm volatile("mul.lo.u32 %0, %0, 65536;" : "+r"(u[i]));
      } else if (OP == 8) {  // attention softmax: F2FP.F16.F32.PACK_AB (+ LOP3 to consume it)
        uint32_t r;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        u[i] ^= r;
      } else if (OP == 9) {  // MUFU.EX2
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      } else if (OP == 10) {  // FHADD: fp32 += fp16 lane
        asm volatile("{ .reg .b16 l, h;\n mov.b32 {l, h}, %1;\n add.rn.f32.f16 %0, l, %0;\n}" : "+f"(a[i]) : "r"(u[i]));
      } else if (OP == 11) {  // FMNMX3
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]), "f"(a[(i + 2) & 7]));
      } else if (OP == 12) {  // MUFU.EX2 + F2FP pack (shared pipe?)
        float e;
        uint32_t r;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(a[i]));
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[(i + 3) & 7]), "f"(a[(i + 1) & 7]));
        a[i] = e;
        u[i] ^= r;
      } else if (OP == 13) {  // MUFU.EX2 + FHADD
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        float* b = reinterpret_cast<float*>(&x2[i]);
        asm volatile("{ .reg .b16 l, h;\n mov.b32 {l, h}, %1;\n add.rn.f32.f16 %0, l, %0;\n}" : "+f"(b[0]) : "r"(u[i]));
      } else if (OP == 14) {  // F2FP pack + FHADD x2 (the P pack and the row sum per score pair)
        uint32_t r;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        float* b = reinterpret_cast<float*>(&x2[i]);
        asm volatile("{ .reg .b16 l, h;\n mov.b32 {l, h}, %2;\n add.rn.f32.f16 %0, l, %0;\n add.rn.f32.f16 %1, h, %1;\n}"
                     : "+f"(b[0]), "+f"(b[1]) : "r"(r));
      }
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += __float_as_uint(a[i]) + u[i] + (uint32_t)x2[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, double per) {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  k<OP><<<148, 512>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-26s %.2f cycles per group per SMSP\n", name, (double)c / (iters * 8.0 * 4) / per);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  run<0>("4xF2FP.E2M1+LOP3 (per F2FP)", 4);
  run<1>("FFMA2", 1);
  run<2>("FMUL2", 1);
  run<3>("FFMA", 1);
  run<4>("LOP3", 1);
  run<5>("F2FP.E4M3+LOP3", 1);
  run<6>("PRMT", 1);
  run<7>("IMUL 65536", 1);
  run<8>("F2FP.F16.PACK+LOP3", 1);
  run<9>("MUFU.EX2", 1);
  run<10>("FHADD", 1);
  run<11>("FMNMX3", 1);
  run<12>("MUFU.EX2 + F2FP.F16", 1);
  run<13>("MUFU.EX2 + FHADD", 1);
  run<14>("F2FP.F16 + 2 FHADD", 1);
  return 0;
}

// Microbenchmark 3: unrolled MMA groups with precomputed descriptors (uniform datapath).
#include <cstdio>
#include "../../paper_2605_18739_b200/csrc/common.cuh"
using namespace kvq;

__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile("{ .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
               :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile("{ .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
               :: "r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{ .reg .pred e;\n elect.sync _|e, 0xffffffff;\n selp.u32 %0, 1, 0, e;\n}" : "=r"(pred));
  return pred != 0;
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * 1024 / 16; i += 128) ((uint4*)smem)[i] = make_uint4(0, 0, 0, 0);
  if (tid < 32) tmem_alloc(&tslot, 512);
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t sA = smem_u32(smem), sB = sA + 32768;
  if (tid < 32) {
    const uint64_t dA = umma_desc_sw128(sA, 16, 1024), dB = umma_desc_sw128(sB, 16, 1024);
    const uint64_t dV = umma_desc_sw128(sB, 16384, 1024);
    constexpr uint32_t id128 = umma_idesc_f16(128, 128, 0, 0, 0);
    constexpr uint32_t idmn = umma_idesc_f16(128, 128, 0, 0, 1);
    constexpr uint32_t id256 = umma_idesc_f16(128, 256, 0, 0, 0);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t off = (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          if (MODE == 0) mma_ss(tmem, dA + off, dB + off, id128, (it | kk) ? 1u : 0u);
          if (MODE == 1) mma_ts(tmem + 256, tmem + 8 * kk, dV + (uint64_t)(kk * 2048 >> 4), idmn, (it | kk) ? 1u : 0u);
          if (MODE == 2) mma_ss(tmem, dA + off, dB + off, id256, (it | kk) ? 1u : 0u);
        }
      }
      __syncwarp();
    }
    unsigned long long t1 = clock64();
    if (elect_one()) tc_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    if (tid == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t0; }
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc(tmem, 512);
}

template <int MODE>
void run(const char* name, unsigned long long* d) {
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  for (int iters : {1, 8, 64}) {
    k<MODE><<<148, 128, 140 * 1024>>>(d, iters);
    k<MODE><<<148, 128, 140 * 1024>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    int n = 8 * iters;
    printf("%-26s n=%4d: issue %7llu clk (%.1f/mma), complete %7llu clk (%.1f/mma) %s\n", name, n, h[0], (double)h[0] / n,
           h[1], (double)h[1] / n, e ? cudaGetErrorString(e) : "");
  }
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 2 * 8);
  run<0>("unrolled SS M128 N128", d);
  run<1>("unrolled TS M128 N128", d);
  run<2>("unrolled SS M128 N256", d);
  return 0;
}

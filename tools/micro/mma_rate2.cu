// Microbenchmark 2: tcgen05.mma issued from a converged warp with elect.sync (vs one thread).
#include <cstdio>
#include "../../paper_2605_18739_b200/csrc/common.cuh"
using namespace kvq;

__device__ __forceinline__ void umma_ss_e(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile("{ .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
               :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void umma_ts_e(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile("{ .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
               :: "r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit_e(uint64_t* bar) {
  asm volatile("{ .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}"
               :: "r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(128, 1) k(unsigned long long* out, int nmma, int mode) {
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
    const uint32_t id128 = umma_idesc_f16(128, 128, 0, 0, 0);
    const uint32_t id256 = umma_idesc_f16(128, 256, 0, 0, 0);
    const uint32_t idmn = umma_idesc_f16(128, 128, 0, 0, 1);
    unsigned long long t0 = clock64(), t1 = 0;
    for (int i = 0; i < nmma; ++i) {
      const uint32_t off = (uint32_t)((i & 7) >> 2) * 16384u + (uint32_t)(i & 3) * 32u;
      if (mode == 0) umma_ss_e(tmem, umma_desc_sw128(sA + off, 16, 1024), umma_desc_sw128(sB + off, 16, 1024), id128, i > 0);
      else if (mode == 1) umma_ts_e(tmem + 256, tmem + 8 * (i & 7), umma_desc_sw128(sB + (i & 7) * 2048, 16384, 1024), idmn, i > 0);
      else umma_ss_e(tmem, umma_desc_sw128(sA + off, 16, 1024), umma_desc_sw128(sB + off, 16, 1024), id256, i > 0);
    }
    t1 = clock64();
    commit_e(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    if (tid == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t0; }
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 2 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const char* names[] = {"warp SS M128 N128 K16", "warp TS M128 N128 K16", "warp SS M128 N256 K16"};
  for (int mode = 0; mode < 3; ++mode)
    for (int n : {8, 64, 512}) {
      k<<<148, 128, 140 * 1024>>>(d, n, mode);
      k<<<148, 128, 140 * 1024>>>(d, n, mode);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("%-24s n=%4d: issue %7llu clk (%.1f/mma), complete %7llu clk (%.1f/mma) %s\n", names[mode], n, h[0],
             (double)h[0] / n, h[1], (double)h[1] / n, e ? cudaGetErrorString(e) : "");
    }
  return 0;
}

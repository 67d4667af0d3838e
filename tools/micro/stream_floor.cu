// Streaming floor for the append's traffic: read two 14.38 MB bf16 tensors and write
// 9/32 of that (the NVFP4 bytes), no arithmetic, 16-byte loads, 4 loads in flight per thread; timed as
// bench.py times the append (CUDA graph of 24 launches cycling 6 distinct input pairs, 172 MB > L2,
// L2 flushed before each replay).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 stream_floor.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) stream_kernel(const uint4* __restrict__ a, const uint4* __restrict__ b,
                                                     uint2* __restrict__ out, long n16) {
  // each thread: 4 x 16 B of a and of b per iteration -> one 8-byte store per 16 B read pair (9/32 ratio approx)
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long stride = (long)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 x[4], y[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) { x[k] = __ldcs(a + i + k * stride); y[k] = __ldcs(b + i + k * stride); }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      __stcs(out + i + k * stride, make_uint2(x[k].x ^ y[k].y, x[k].z ^ y[k].w));
  }
  for (; i < n16; i += stride) {
    uint4 x = __ldcs(a + i), y = __ldcs(b + i);
    __stcs(out + i, make_uint2(x.x ^ y.y, x.z ^ y.w));
  }
}

int main() {
  const long n = 4680L * 12 * 128;            // elements per tensor
  const long n16 = n * 2 / 16;                 // 16-byte chunks per tensor
  uint4 *A[6], *B[6];
  uint2* O;
  for (int i = 0; i < 6; ++i) { cudaMalloc(&A[i], n * 2); cudaMalloc(&B[i], n * 2); cudaMemset(A[i], 1, n * 2); cudaMemset(B[i], 2, n * 2); }
  cudaMalloc(&O, n16 * 8);
  char* flush; cudaMalloc(&flush, 256 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int grid_mult : {1, 2, 4}) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < 24; ++r) stream_kernel<<<sms * grid_mult, 512, 0, s>>>(A[r % 6], B[r % 6], O, n16);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    float best = 1e9;
    for (int it = 0; it < 7; ++it) {
      cudaMemsetAsync(flush, it, 256 << 20, s);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (it > 0 && ms < best) best = ms;
    }
    const double us = best * 1e3 / 24, bytes = 2.0 * n * 2 + n16 * 8.0;
    printf("stream floor, grid %d x %d x 512: %.2f us per op, %.1f GB/s (%.2f MB moved)\n", sms, grid_mult, us,
           bytes / us / 1e3, bytes / 1e6);
  }
  return 0;
}

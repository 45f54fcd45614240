// Which warps of a 256-thread CTA share an SM sub-partition (SMSP)? Two warps run a
// DFMA-bound loop, the others exit; the pair that shares an SMSP takes ~2x as long.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/smsp_map.cu -o tools/smsp_map
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, int wa, int wb, double a, double b) {
  const int w = threadIdx.x >> 5;
  if (w != wa && w != wb) return;
  double c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < 20000; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = fma(c[q], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int wb = 1; wb < 8; ++wb) {
    k<<<sms, 256>>>(out, 0, wb, 0.999999, 1e-7);
    cudaEventRecord(e0);
    k<<<sms, 256>>>(out, 0, wb, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("warps 0 + %d: %.3f ms\n", wb, ms);
  }
  return 0;
}

// DMMA / DFMA throughput at the element pass's occupancy (one 256-thread CTA per SM,
// 2 warps per SMSP): how many independent m8n8k4 accumulators a warp needs to keep the
// FP64 pipe busy. nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/dmma_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void k_dmma(double* out, double a) {
  double acc[NACC][2];
#pragma unroll
  for (int q = 0; q < NACC; ++q) acc[q][0] = acc[q][1] = threadIdx.x * 1e-3 + q;
  const double b = a * 0.5;
  for (int it = 0; it < ITERS / NACC; ++it) {
#pragma unroll
    for (int q = 0; q < NACC; ++q) dmma(acc[q][0], acc[q][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < NACC; ++q) s += acc[q][0] + acc[q][1];
  if (s == 1.2345) out[0] = s;
}

template <int NCH>
__global__ void k_dfma(double* out, double a, double b) {
  double c[NCH];
#pragma unroll
  for (int q = 0; q < NCH; ++q) c[q] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < ITERS * 8 / NCH; ++it) {
#pragma unroll
    for (int q = 0; q < NCH; ++q) c[q] = fma(c[q], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < NCH; ++q) s += c[q];
  if (s == 1.2345) out[0] = s;
}

template <typename F>
static float best_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

template <int NACC>
static void run_mma(int sms, double* out, int threads) {
  const float ms = best_ms([&] { k_dmma<NACC><<<sms, threads>>>(out, 0.999999); });
  const double fl = (double)sms * threads / 32.0 * ITERS * 512.0;
  printf("dmma threads %d acc %2d: %.2f TFLOP/s  (%.1f cycles per DMMA per SMSP at 1.965 GHz)\n",
         threads, NACC, fl / ms / 1e9,
         ms * 1e-3 * 1.965e9 / ((double)threads / 128.0 * ITERS));
}

template <int NCH>
static void run_fma(int sms, double* out, int threads) {
  const float ms = best_ms([&] { k_dfma<NCH><<<sms, threads>>>(out, 0.999999, 1e-7); });
  const double fl = (double)sms * threads * ITERS * 8 * 2.0;
  printf("dfma threads %d chains %2d: %.2f TFLOP/s\n", threads, NCH, fl / ms / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  for (int threads : {256, 512, 1024}) {
    run_mma<1>(sms, out, threads);
    run_mma<2>(sms, out, threads);
    run_mma<4>(sms, out, threads);
    run_mma<8>(sms, out, threads);
    run_mma<12>(sms, out, threads);
    run_mma<16>(sms, out, threads);
    run_fma<4>(sms, out, threads);
    run_fma<8>(sms, out, threads);
    run_fma<16>(sms, out, threads);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

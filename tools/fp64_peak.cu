// FP64 peak microbenchmarks on the B200 (SURVEY §8d "measure FP64 peak on the box"):
//   dfma   : DFMA on the FP64 pipe, 8 independent chains per thread
//   dmma   : mma.sync.m8n8k4 f64 (DMMA), 4 independent accumulators per warp
//   mixed  : both in the same warps (do the two pipes overlap?)
//   dadd   : DADD, 8 chains (the split-form pair loop is ~25% DADD)
// Timed with CUDA events over a grid of 148 x 8 blocks, best of 5; clocks read by
// the caller. Output: one JSON object on stdout.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = fma(c[q], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q];
  if (s == 1.2345) out[0] = s;
}

__global__ void k_dadd(double* out, double a) {
  double c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = c[q] + a;
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q];
  if (s == 1.2345) out[0] = s;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, double a) {
  double acc[4][2];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = threadIdx.x * 1e-3 + q;
  const double b = a * 0.5;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int q = 0; q < 4; ++q) dmma(acc[q], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) s += acc[q][0] + acc[q][1];
  if (s == 1.2345) out[0] = s;
}

__global__ void k_mixed(double* out, double a, double b) {
  double acc[4][2], c[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = threadIdx.x * 1e-3 + q;
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int q = 0; q < 4; ++q) dmma(acc[q], a, b);
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = fma(c[q], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) s += acc[q][0] + acc[q][1];
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q];
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

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out;
  CK(cudaMalloc(&out, 8));
  const int blocks = sms * 8, threads = 256;
  const double nthr = (double)blocks * threads;
  const float t_fma = best_ms([&] { k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7); });
  const float t_add = best_ms([&] { k_dadd<<<blocks, threads>>>(out, 1e-7); });
  const float t_mma = best_ms([&] { k_dmma<<<blocks, threads>>>(out, 0.999999); });
  const float t_mix = best_ms([&] { k_mixed<<<blocks, threads>>>(out, 0.999999, 1e-7); });
  CK(cudaGetLastError());
  const double f_fma = nthr * ITERS * 8 * 2.0;                 // flops
  const double i_add = nthr * ITERS * 8;                      // adds
  const double warps = nthr / 32.0;
  const double f_mma = warps * (ITERS / 4) * 4 * 512.0;      // 8x8x4 x2 per mma
  const double f_mix_mma = f_mma, f_mix_fma = nthr * (ITERS / 4) * 8 * 2.0;
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, "
         "\"dfma_tflops\": %.3f, \"dadd_gops\": %.1f, \"dmma_tflops\": %.3f, "
         "\"mixed_tflops\": %.3f, \"mixed_dmma_part_tflops\": %.3f, \"mixed_dfma_part_tflops\": %.3f, "
         "\"ms\": {\"dfma\": %.4f, \"dadd\": %.4f, \"dmma\": %.4f, \"mixed\": %.4f}}\n",
         sms, clk / 1e3, f_fma / t_fma / 1e9, i_add / t_add / 1e6, f_mma / t_mma / 1e9,
         (f_mix_mma + f_mix_fma) / t_mix / 1e9, f_mix_mma / t_mix / 1e9, f_mix_fma / t_mix / 1e9,
         t_fma, t_add, t_mma, t_mix);
  return 0;
}

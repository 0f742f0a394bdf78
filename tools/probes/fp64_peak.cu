// FP64 pipe peak of this B200 (MEASURED_PEAKS.json has HBM and bf16 only):
// independent DFMA / DADD chains per thread, 148 x 4 CTAs of 256 threads,
// CUDA-event timed.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/probes/fp64_peak.cu -o build/fp64_peak ; prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 1 << 14;

__global__ void k_dfma(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dadd(double* out, double a) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = x[c] + a;
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int grid = sms * 4, block = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double ops = (double)grid * block * kIters * kChains;
  float best_fma = 1e30f, best_add = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    float ms;
    cudaEventRecord(e0);
    k_dfma<<<grid, block>>>(out, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_fma) best_fma = ms;
    cudaEventRecord(e0);
    k_dadd<<<grid, block>>>(out, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_add) best_add = ms;
  }
  const double fma_tflops = 2.0 * ops / (best_fma * 1e-3) / 1e12;
  const double add_tops = ops / (best_add * 1e-3) / 1e12;
  printf("{\"fp64_fma_tflops\": %.3f, \"fp64_add_tops\": %.3f, \"sms\": %d, \"max_clock_mhz\": %.0f, "
         "\"fma_per_clk_per_sm_at_max\": %.1f, \"how\": \"%d CTAs x %d threads x %d independent "
         "chains x %d DFMA/DADD, best of 5, CUDA events\"}\n",
         fma_tflops, add_tops, sms, clk / 1e3,
         ops / (best_fma * 1e-3) / (sms * clk * 1e3), grid, block, kChains, kIters);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

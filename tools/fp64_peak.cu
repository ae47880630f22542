// Measured FP64 peak of this GPU (the FP64-bound paths,
// C4 FCN and C5 fused integration, need a measured DFMA peak, not the datasheet).
//
// Eight independent DFMA chains per thread, 256 threads, 148 x 8 CTAs; CUDA events
// around the launch, best of 5.  The SM clock during the run is estimated from
// the longest CTA's clock64() span divided by the event time (oldest-first warp
// scheduling lets early CTAs finish well before the launch does).  Prints one JSON line:
// DFMA/s, TFLOP/s (2 flops per DFMA), DFMA lanes per SM per clock.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o /tmp/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b,
                                              long long* cycles) {
  double x[kChains];
#pragma unroll
  for (int j = 0; j < kChains; ++j) x[j] = threadIdx.x * 1e-3 + j;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kChains; ++j) x[j] = fma(x[j], a, b);
  }
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < kChains; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;  // keeps the chains live
  if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long*>(cycles),
                                  (unsigned long long)(t1 - t0));
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8, threads = 256, iters = 1 << 15;
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<<<blocks, threads>>>(out, iters, 0.9999999, 1e-7, cyc);
  cudaDeviceSynchronize();
  float best = 1e30f;
  long long cycles = 0;
  for (int r = 0; r < 5; ++r) {
    cudaMemset(cyc, 0, 8);
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters, 0.9999999, 1e-7, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) {
      best = ms;
      cudaMemcpy(&cycles, cyc, 8, cudaMemcpyDeviceToHost);
    }
  }
  if (cudaGetLastError() != cudaSuccess) {
    printf("{\"error\": \"launch failed\"}\n");
    return 1;
  }
  const double dfma = (double)blocks * threads * iters * kChains;
  const double s = best * 1e-3;
  // all 8 CTAs per SM are co-resident, so the longest loop spans ~the launch
  const double clk_hz = (double)cycles / s;
  printf("{\"dfma_per_s\": %.4e, \"fp64_tflops\": %.2f, \"sm_clock_mhz_est\": %.0f, "
         "\"dfma_lanes_per_sm_per_clk\": %.1f, \"sms\": %d, \"ms\": %.3f, "
         "\"how\": \"8 independent DFMA chains x 256 threads x %d CTAs x 2^15 iters, best of 5, CUDA events\"}\n",
         dfma / s, 2.0 * dfma / s * 1e-12, clk_hz * 1e-6, dfma / s / clk_hz / sms, sms, best, blocks);
  return 0;
}

// Exhaustive-ish check that the branch-free sqrt / division sequences in
// csrc/hk_device.cuh (cr_sqrt, cr_div) return the IEEE correctly rounded
// result (bit-identical to sqrt.rn.f64 / div.rn.f64) on the operand ranges
// the generator feeds them.  Counts mismatches over N pseudo-random inputs
// per family; exits non-zero on any mismatch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../include -I../paper_1711_05683_b200/csrc verify_cr.cu
#include <cstdio>
#include <cstdint>

#include "hk_device.cuh"

__device__ unsigned long long g_bad[4];
__device__ double g_example[8];

__device__ __forceinline__ double from_bits(uint64_t mant, int exp) {
  return __longlong_as_double((long long)(((uint64_t)(exp + 1023) << 52) | (mant & 0xFFFFFFFFFFFFFull)));
}

__global__ void k_check(uint64_t n, uint64_t seed) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t r1 = hk::mix64(seed + 2 * i), r2 = hk::mix64(seed + 2 * i + 1);
    // family 0: sqrt over exponents [-300, 300] (all mantissas)
    {
      const double x = from_bits(r1, (int)(r2 % 601) - 300);
      const double a = hk::cr_sqrt(x), b = __dsqrt_rn(x);
      if (__double_as_longlong(a) != __double_as_longlong(b)) {
        if (atomicAdd(&g_bad[0], 1ull) == 0) { g_example[0] = x; g_example[1] = a; }
      }
    }
    // family 1: division with quotient exponents in range
    {
      const double x = from_bits(r1, (int)(r2 % 401) - 200);
      const double y = from_bits(r2 >> 3, (int)((r1 >> 40) % 401) - 200);
      const double a = hk::cr_div(x, y), b = __ddiv_rn(x, y);
      if (__double_as_longlong(a) != __double_as_longlong(b)) {
        if (atomicAdd(&g_bad[1], 1ull) == 0) { g_example[2] = x; g_example[3] = y; }
      }
    }
    // family 2: the generator's actual operands: sqrt(lambda) / (2 M), GeV-scale
    {
      const double M = 0.2 + 10.0 * (double)(r1 >> 11) * 0x1.0p-53;
      const double lam = (double)(r2 >> 11) * 0x1.0p-53 * M * M * M * M;
      const double a = hk::cr_div(hk::cr_sqrt(lam), 2.0 * M);
      const double b = __ddiv_rn(__dsqrt_rn(lam), 2.0 * M);
      if (__double_as_longlong(a) != __double_as_longlong(b)) {
        if (atomicAdd(&g_bad[2], 1ull) == 0) { g_example[4] = lam; g_example[5] = M; }
      }
    }
    // family 3: mantissas near all-ones / all-zeros (hard cases for reciprocals)
    {
      const uint64_t m = (r1 & 1) ? (0xFFFFFFFFFFFFFull - (r2 & 0xFFFF)) : (r2 & 0xFFFF);
      const double y = from_bits(m, (int)(r1 >> 58) - 32);
      const double x = from_bits(r2 >> 7, (int)((r1 >> 50) & 31) - 16);
      const double a = hk::cr_div(x, y), b = __ddiv_rn(x, y);
      const double c = hk::cr_sqrt(y), d = __dsqrt_rn(y);
      if (__double_as_longlong(a) != __double_as_longlong(b) ||
          __double_as_longlong(c) != __double_as_longlong(d)) {
        if (atomicAdd(&g_bad[3], 1ull) == 0) { g_example[6] = x; g_example[7] = y; }
      }
    }
  }
}

int main(int argc, char** argv) {
  const unsigned long long n = argc > 1 ? strtoull(argv[1], nullptr, 10) : (1ull << 32);
  unsigned long long zero[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(g_bad, zero, sizeof zero);
  const int chunks = 16;
  for (int c = 0; c < chunks; ++c) k_check<<<148 * 8, 256>>>(n / chunks, 0x1234567ull * (c + 1));
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long bad[4];
  double ex[8];
  cudaMemcpyFromSymbol(bad, g_bad, sizeof bad);
  cudaMemcpyFromSymbol(ex, g_example, sizeof ex);
  std::printf("{\"samples_per_family\": %llu, \"cuda\": \"%s\", \"sqrt_mismatch\": %llu, "
              "\"div_mismatch\": %llu, \"pstar_mismatch\": %llu, \"hard_mismatch\": %llu, "
              "\"examples\": [%.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g]}\n",
              (n / chunks) * chunks, cudaGetErrorString(e), bad[0], bad[1], bad[2], bad[3], ex[0],
              ex[1], ex[2], ex[3], ex[4], ex[5], ex[6], ex[7]);
  return (e == cudaSuccess && !(bad[0] | bad[1] | bad[2] | bad[3])) ? 0 : 1;
}

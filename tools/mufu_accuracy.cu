// Accuracy of the f64 MUFU seeds (rcp.approx.ftz.f64, rsqrt.approx.ftz.f64)
// and of one / two Newton (Goldschmidt) steps from them, measured against
// correctly rounded division / sqrt over 2^26 log-uniform inputs in
// [2^-40, 2^40].  Decides how many refinement steps the momentum path needs
// for the 1e-12 * E parity budget.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_accuracy.cu -o /tmp/mufu
#include <cstdio>
#include <cuda_runtime.h>
#include <cstring>

__device__ unsigned long long g_max[6];  // max relative error bits (as double bits, >= 0)

__device__ void upd(int k, double rel) {
  atomicMax(&g_max[k], (unsigned long long)__double_as_longlong(fabs(rel)));
}

__global__ void k_probe(unsigned long long seed, int per_thread) {
  unsigned long long s = seed + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  for (int i = 0; i < per_thread; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    const double u = (double)(s >> 11) * 0x1.0p-53;
    const double x = exp2(80.0 * u - 40.0);
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double rx = 1.0 / x;
    upd(0, (r - rx) / rx);
    double e = fma(-x, r, 1.0);
    const double r1 = fma(r, e, r);
    upd(1, (r1 - rx) / rx);
    e = fma(-x, r1, 1.0);
    upd(2, (fma(r1, e, r1) - rx) / rx);
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double sx = sqrt(x);
    upd(3, (y * sx - 1.0));
    double sq = x * y, h = 0.5 * y;
    const double rr = fma(-sq, h, 0.5);
    sq = fma(sq, rr, sq);  // one coupled Goldschmidt step
    upd(4, (sq - sx) / sx);
    h = fma(h, rr, h);
    const double d = fma(-sq, sq, x);
    upd(5, (fma(d, h, sq) - sx) / sx);  // + residual correction (fast_sqrt today)
  }
}

int main() {
  cudaMemset(g_max, 0, 0);
  unsigned long long z[6] = {0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbol(g_max, z, sizeof(z));
  k_probe<<<148 * 8, 256>>>(12345, 1 << 8);
  unsigned long long h[6];
  cudaMemcpyFromSymbol(h, g_max, sizeof(h));
  const char* names[6] = {"rcp_seed", "rcp_1step", "rcp_2step", "rsqrt_seed", "sqrt_1step", "sqrt_1step_plus_residual"};
  printf("{");
  for (int k = 0; k < 6; ++k) {
    double v;
    memcpy(&v, &h[k], 8);
    printf("\"%s\": %.3e%s", names[k], v, k < 5 ? ", " : "");
  }
  printf(", \"inputs\": %d, \"err\": \"%s\"}\n", 148 * 8 * 256 * 256, cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// Write-bandwidth ceiling of the generator's store pattern, with no compute.
//
// k_generate<3,REF,vec2> writes 13 fp64 columns: each CTA owns a 4096-row
// chunk, each thread stores 8 x (double2 per column), __stcs streaming
// stores, 2 CTAs/SM.  This kernel reproduces that pattern with a trivial
// value, so its bandwidth is what the generator could reach if its
// arithmetic were free.  Variants:
//   pattern   the generator's shape (2 CTAs/SM via dynamic shared memory)
//   occ       the same stores at full occupancy
//   wb        plain write-back stores (st.global) instead of streaming
//   fill      one column after another, 16 B per thread-store (cudaMemset-like)
// Prints one JSON line per variant (best of 10, CUDA events, 1e8 rows).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/store_pattern.cu -o /tmp/store_pattern
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kCols = 13, kBlock = 256, kChunk = 4096;

template <bool STREAM>
__global__ void __launch_bounds__(kBlock) k_pattern(double* const* cols, long long n) {
  const long long chunks = n / kChunk;
  for (long long c = blockIdx.x; c < chunks; c += gridDim.x) {
#pragma unroll 1
    for (int i = 0; i < kChunk / (2 * kBlock); ++i) {
      const long long r0 = c * kChunk + i * (2 * kBlock) + 2 * threadIdx.x;
      const double v = (double)r0;
#pragma unroll
      for (int j = 0; j < kCols; ++j) {
        double2* p = reinterpret_cast<double2*>(cols[j] + r0);
        const double2 val = make_double2(v + j, v - j);
        if (STREAM)
          __stcs(p, val);
        else
          *p = val;
      }
    }
  }
}

__global__ void k_fill(double2* p, long long n2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x)
    __stcs(p + i, make_double2((double)i, 1.0));
}

struct ColsArg {
  double* p[kCols];
};

int main() {
  const long long n = 100000000LL / kChunk * kChunk;  // whole chunks
  double* base;
  if (cudaMalloc(&base, (size_t)kCols * n * sizeof(double)) != cudaSuccess) return 1;
  double* hcols[kCols];
  for (int j = 0; j < kCols; ++j) hcols[j] = base + (long long)j * n;
  double** dcols;
  cudaMalloc(&dcols, sizeof(hcols));
  cudaMemcpy(dcols, hcols, sizeof(hcols), cudaMemcpyHostToDevice);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned grid = (unsigned)(n / kChunk);
  const size_t smem_2per = 100 * 1024;  // limits residency to 2 CTAs/SM like the generator
  cudaFuncSetAttribute(k_pattern<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_2per);
  cudaFuncSetAttribute(k_pattern<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_2per);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)kCols * n * sizeof(double);
  auto run = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("{\"variant\": \"%s\", \"ms\": %.4f, \"TBps\": %.3f, \"err\": \"%s\"}\n", name, best,
           bytes / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
  run("pattern", [&] { k_pattern<true><<<grid, kBlock, smem_2per>>>(dcols, n); });
  run("occ", [&] { k_pattern<true><<<grid, kBlock>>>(dcols, n); });
  run("wb", [&] { k_pattern<false><<<grid, kBlock, smem_2per>>>(dcols, n); });
  run("fill", [&] { k_fill<<<sms * 8, 512>>>(reinterpret_cast<double2*>(base), (long long)kCols * n / 2); });
  return 0;
}

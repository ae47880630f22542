// Per-command overhead of a resident multi-CTA server (no arithmetic): CTA 0
// polls a host command word, publishes it in device memory, every CTA takes
// a ticket, the last one answers through mapped host memory.  Variants:
// waiter back-off (ns) and payload size read from host memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

struct Cmd {
  unsigned long long seq;
  double payload[15];
};

__device__ __forceinline__ unsigned long long ld_acq_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acq_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_srv(const Cmd* cmd, unsigned long long* gen, unsigned int* ticket, double* dpay,
                      volatile unsigned long long* mail, int iters, int backoff, int npay) {
  __shared__ unsigned long long s_g;
  __shared__ unsigned s_t;
  unsigned long long mine = 0;
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      if (blockIdx.x == 0) {
        unsigned long long s;
        while ((s = ld_acq_sys(&cmd->seq)) == mine) {
        }
        for (int i = 0; i < npay; ++i) dpay[i] = cmd->payload[i];
        __threadfence();
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(gen), "l"(s) : "memory");
      }
      unsigned long long g;
      while ((g = ld_acq_gpu(gen)) == mine)
        if (backoff) __nanosleep(backoff);
      s_g = g;
    }
    __syncthreads();
    mine = s_g;
    if (threadIdx.x == 0) {
      __threadfence();
      s_t = atomicAdd(ticket, 1u);
    }
    __syncthreads();
    if (s_t == gridDim.x - 1 && threadIdx.x == 0) {
      *ticket = 0;
      __threadfence_system();
      mail[0] = mine;
    }
  }
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  Cmd* h_cmd;
  unsigned long long* h_mail;
  cudaHostAlloc(&h_cmd, sizeof(Cmd), cudaHostAllocMapped);
  cudaHostAlloc(&h_mail, 64, cudaHostAllocMapped);
  Cmd* d_cmd;
  unsigned long long* d_mail;
  cudaHostGetDevicePointer(&d_cmd, h_cmd, 0);
  cudaHostGetDevicePointer(&d_mail, h_mail, 0);
  unsigned long long* gen;
  unsigned int* ticket;
  double* dpay;
  cudaMalloc(&gen, 8);
  cudaMalloc(&ticket, 4);
  cudaMalloc(&dpay, 128);
  volatile unsigned long long* vm = h_mail;
  volatile unsigned long long* vc = &h_cmd->seq;
  for (int grid : {1, 148, 592}) {
    for (int backoff : {0, 64, 256}) {
      for (int npay : {0, 8}) {
        cudaMemset(gen, 0, 8);
        cudaMemset(ticket, 0, 4);
        h_cmd->seq = 0;
        h_mail[0] = 0;
        cudaDeviceSynchronize();
        const int iters = 3000;
        k_srv<<<grid, 256>>>(d_cmd, gen, ticket, dpay, d_mail, iters, backoff, npay);
        std::vector<double> t;
        for (unsigned long long s = 1; s <= (unsigned long long)iters; ++s) {
          const double t0 = now_us();
          *vc = s;
          while (vm[0] != s) {
          }
          t.push_back(now_us() - t0);
        }
        cudaDeviceSynchronize();
        std::sort(t.begin(), t.end());
        std::printf("{\"grid\": %d, \"backoff_ns\": %d, \"payload_doubles\": %d, \"median_us\": %.2f}\n", grid,
                    backoff, npay, t[t.size() / 2]);
      }
    }
  }
  return 0;
}

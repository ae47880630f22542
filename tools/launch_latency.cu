// Round-trip latency floor of a synchronous FCN call on this GPU: host
// launches a kernel whose last action is a system-scope write into mapped
// pinned memory, then spins on it (the hk_nll_eval protocol).  Reports the
// median round trip for an empty kernel, and for a persistent kernel that
// waits on a host-written mailbox instead of being launched (the floor a
// resident "FCN server" would have).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

__global__ void k_signal(volatile unsigned long long* mail, unsigned long long seq) {
  if (threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) {
    __threadfence_system();
    mail[0] = seq;
  }
}

// one CTA polls the host command word; on a new sequence number it echoes it
__global__ void k_server(volatile unsigned long long* cmd, volatile unsigned long long* mail, int iters) {
  unsigned long long last = 0;
  for (int i = 0; i < iters; ++i) {
    unsigned long long s;
    do {
      s = cmd[0];
    } while (s == last);
    last = s;
    __threadfence_system();
    mail[0] = s;
  }
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  unsigned long long *h_mail, *d_mail, *h_cmd, *d_cmd;
  cudaHostAlloc(&h_mail, 64, cudaHostAllocMapped);
  cudaHostAlloc(&h_cmd, 64, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&d_mail, h_mail, 0);
  cudaHostGetDevicePointer(&d_cmd, h_cmd, 0);
  h_mail[0] = 0;
  h_cmd[0] = 0;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  volatile unsigned long long* vm = h_mail;
  for (int grid : {1, 592, 2442}) {
    std::vector<double> t;
    for (unsigned long long s = 1; s <= 2000; ++s) {
      const double t0 = now_us();
      k_signal<<<grid, 256, 0, st>>>(d_mail, s);
      while (vm[0] != s) {
      }
      t.push_back(now_us() - t0);
      h_mail[0] = 0;
    }
    std::sort(t.begin(), t.end());
    std::printf("{\"what\": \"launch+signal\", \"grid\": %d, \"median_us\": %.2f, \"p10_us\": %.2f}\n", grid,
                t[t.size() / 2], t[t.size() / 10]);
  }
  cudaDeviceSynchronize();
  const int iters = 2000;
  h_mail[0] = 0;
  k_server<<<1, 32, 0, st>>>(d_cmd, d_mail, iters);
  std::vector<double> t;
  volatile unsigned long long* vc = h_cmd;
  for (unsigned long long s = 1; s <= (unsigned long long)iters; ++s) {
    const double t0 = now_us();
    vc[0] = s;
    while (vm[0] != s) {
    }
    t.push_back(now_us() - t0);
  }
  cudaStreamSynchronize(st);
  std::sort(t.begin(), t.end());
  std::printf("{\"what\": \"resident server round trip\", \"median_us\": %.2f, \"p10_us\": %.2f}\n", t[t.size() / 2],
              t[t.size() / 10]);
  return 0;
}

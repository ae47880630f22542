/* A plain C host of the drop-in boundary: what a cgo / JNI / N-API binding
 * of include/hepkit_cuda.h does, with no Python and no torch.
 *
 *   gcc -std=c99 -O2 examples/c_host.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1711_05683_b200 -lhepkit_cuda -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1711_05683_b200 -o c_host && ./c_host 1000000
 *
 * phsp_generate of B0 -> J/psi K pi into device columns with the fused weight
 * partials, their fixed-order fold (sum w, sum w^2), the same rows generated
 * into host memory, and the library's error contract on a bad call.  Prints
 * one JSON line (tests/test_c_host_gpu.py compares it with the Python API). */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "hepkit_cuda.h"

#define CHECK(call)                                                      \
  do {                                                                   \
    if ((call) != 0) {                                                   \
      char msg[512];                                                     \
      hk_last_error(msg, sizeof msg);                                    \
      fprintf(stderr, "%s failed: %s\n", #call, msg);                    \
      return 1;                                                          \
    }                                                                    \
  } while (0)

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 1000000;
  const double M = 5.27966, m[3] = {3.0969, 0.493677, 0.13957039};
  hk_decay_t d = {0};
  d.n = 3;
  d.moving = 0;
  d.mother_mass = M;
  double sum = 0.0;
  for (int i = 0; i < 3; ++i) { /* numpy's sequential sum and cumsum for three values */
    sum += m[i];
    d.masses[i] = m[i];
    d.csum[i] = sum;
  }
  d.T = M - sum;
  d.mother[0] = M;
  d.m_mother = M;
  hk_key_t key = {1u, 1u, 0u, HK_RNG_REFERENCE, 0};

  /* device columns (weight + 3 x (e, px, py, pz)) and the weight partials */
  double* cols[13];
  for (int c = 0; c < 13; ++c)
    if (cudaMalloc((void**)&cols[c], (size_t)n * sizeof(double)) != cudaSuccess) return 1;
  const int64_t parts = (int64_t)HK_WARP_SLICES * hk_num_chunks(n);
  double *wpart = NULL, *sums = NULL;
  if (cudaMalloc((void**)&wpart, (size_t)(2 * parts) * sizeof(double)) != cudaSuccess) return 1;
  if (cudaMalloc((void**)&sums, 2 * sizeof(double)) != cudaSuccess) return 1;
  CHECK(hk_phsp_generate(&d, &key, 0, n, cols, wpart, NULL));
  CHECK(hk_fold_partials(wpart, parts, 2, sums, NULL));
  double h_sums[2], w_dev[3];
  cudaMemcpy(h_sums, sums, sizeof h_sums, cudaMemcpyDeviceToHost);
  cudaMemcpy(w_dev, cols[0], sizeof w_dev, cudaMemcpyDeviceToHost);

  /* the same rows straight into host memory */
  double* host[13];
  for (int c = 0; c < 13; ++c) host[c] = (double*)malloc((size_t)n * sizeof(double));
  void* stage = NULL;
  const size_t stage_bytes = 64u << 20;
  if (cudaMalloc(&stage, stage_bytes) != cudaSuccess) return 1;
  double h_wsums[2];
  CHECK(hk_phsp_generate_host(&d, &key, 0, n, host, h_wsums, stage, stage_bytes, NULL));
  int same = 1;
  for (int i = 0; i < 3 && i < n; ++i) same &= host[0][i] == w_dev[i];

  /* the error contract: a bad call returns non-zero and names the problem */
  hk_decay_t bad = d;
  bad.n = 1;
  const int rc = hk_phsp_generate(&bad, &key, 0, n, cols, wpart, NULL);
  char msg[256] = {0};
  hk_last_error(msg, sizeof msg);

  printf("{\"abi\": %d, \"n\": %lld, \"sum_w\": %.17g, \"sum_w2\": %.17g, \"host_sum_w\": %.17g, "
         "\"w0\": %.17g, \"w1\": %.17g, \"w2\": %.17g, \"host_equals_device\": %d, \"bad_rc\": %d, "
         "\"bad_msg\": \"%s\"}\n",
         hk_abi_version(), (long long)n, h_sums[0], h_sums[1], h_wsums[0], w_dev[0], w_dev[1], w_dev[2], same, rc,
         msg);
  for (int c = 0; c < 13; ++c) {
    cudaFree(cols[c]);
    free(host[c]);
  }
  cudaFree(wpart);
  cudaFree(sums);
  cudaFree(stage);
  hk_shutdown();
  return 0;
}

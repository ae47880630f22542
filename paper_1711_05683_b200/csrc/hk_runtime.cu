// hk_runtime.cu -- error reporting, device queries and the host-buffer
// generation entry point (generation overlapped with device->host copies).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "hepkit_cuda.h"
#include "hk_host.h"

namespace hk {

namespace {
thread_local char g_err[512] = "";
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* where) {
  set_error("%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
  return HK_ECUDA;
}

int launch_fold(const double* parts, int64_t n, int width, double* out, cudaStream_t st);
int launch_fold_segments(const double* parts, int64_t n_seg, int seg_len, int width, double* out,
                         cudaStream_t st);

// One copy stream + two events per device, created on first use.
struct CopyLane {
  int device = -1;
  cudaStream_t copy = nullptr;
  cudaEvent_t made[2] = {nullptr, nullptr};
  cudaEvent_t freed[2] = {nullptr, nullptr};
};

thread_local CopyLane t_lanes[16];

int copy_lane(CopyLane** out) {
  int dev = 0;
  HK_CUDA(cudaGetDevice(&dev));
  CopyLane& L = t_lanes[dev & 15];
  if (L.device != dev) {
    HK_CUDA(cudaStreamCreateWithFlags(&L.copy, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      HK_CUDA(cudaEventCreateWithFlags(&L.made[b], cudaEventDisableTiming));
      HK_CUDA(cudaEventCreateWithFlags(&L.freed[b], cudaEventDisableTiming));
    }
    L.device = dev;
  }
  *out = &L;
  return HK_OK;
}

// hk_shutdown: destroy this thread's copy streams/events (rebuilt on demand)
void copy_lane_release() {
  for (CopyLane& L : t_lanes) {
    if (L.device < 0) continue;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(L.device);
    cudaStreamDestroy(L.copy);
    for (int b = 0; b < 2; ++b) {
      cudaEventDestroy(L.made[b]);
      cudaEventDestroy(L.freed[b]);
    }
    cudaSetDevice(cur);
    L = CopyLane{};
  }
}

}  // namespace hk

using namespace hk;

extern "C" {

int hk_abi_version(void) { return HK_ABI_VERSION; }

int hk_last_error(char* buf, size_t len) {
  if (!buf || len == 0) return HK_EINVAL;
  std::snprintf(buf, len, "%s", g_err);
  return HK_OK;
}

int hk_device_info(int* n_devices, int* sm_count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (n_devices) *n_devices = n;
  if (sm_count) {
    *sm_count = 0;
    if (n > 0) HK_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, 0));
  }
  return HK_OK;
}

int hk_phsp_generate_host(const hk_decay_t* spec, const hk_key_t* key, uint64_t ev_begin,
                          int64_t ev_count, double* const* h_cols, double* h_wsums,
                          void* d_stage, size_t stage_bytes, void* stream) {
  HK_NVTX("hk_phsp_generate_host");
  HK_REQUIRE(spec && key && h_cols && d_stage, "NULL argument");
  HK_REQUIRE(spec->n >= 2 && spec->n <= HK_MAX_DAUGHTERS, "bad daughter count %d", spec->n);
  HK_REQUIRE(ev_count >= 0, "negative ev_count");
  const int ncols = 4 * spec->n + 1;
  const int64_t chunks = num_chunks(ev_count);
  // stage layout: [partials: 2 doubles per warp-slice][super records: 2 per super]
  //               [sum cell: 2 doubles][2 x piece buffers]
  const size_t head = (size_t)(chunks * 2 * HK_WARP_SLICES + HK_SUPERS * 2 + 2) * sizeof(double);
  HK_REQUIRE(stage_bytes > head, "staging area too small");
  const size_t per_row = (size_t)ncols * sizeof(double);
  int64_t piece = (int64_t)((stage_bytes - head) / (2 * per_row));
  piece = (piece / HK_CHUNK) * HK_CHUNK;
  HK_REQUIRE(piece >= HK_CHUNK || ev_count == 0, "staging area too small for one chunk per buffer");
  if (ev_count == 0) {
    if (h_wsums) h_wsums[0] = h_wsums[1] = 0.0;
    return HK_OK;
  }
  CopyLane* L = nullptr;
  if (int rc = copy_lane(&L)) return rc;
  cudaStream_t st = as_stream(stream);
  double* part = static_cast<double*>(d_stage);
  double* cpart = part + chunks * 2 * HK_WARP_SLICES;
  double* sums = cpart + HK_SUPERS * 2;
  double* buf[2] = {sums + 2, sums + 2 + piece * ncols};
  for (int64_t off = 0, i = 0; off < ev_count; off += piece, ++i) {
    const int b = (int)(i & 1);
    const int64_t cnt = std::min<int64_t>(piece, ev_count - off);
    if (i >= 2) HK_CUDA(cudaStreamWaitEvent(st, L->freed[b], 0));
    double* cols[4 * HK_MAX_DAUGHTERS + 1];
    for (int c = 0; c < ncols; ++c) cols[c] = buf[b] + (int64_t)c * piece;
    if (int rc = hk_phsp_generate(spec, key, ev_begin + (uint64_t)off, cnt, cols,
                                  part + (off / HK_CHUNK) * 2 * HK_WARP_SLICES, stream))
      return rc;
    HK_CUDA(cudaEventRecord(L->made[b], st));
    HK_CUDA(cudaStreamWaitEvent(L->copy, L->made[b], 0));
    for (int c = 0; c < ncols; ++c)
      HK_CUDA(cudaMemcpyAsync(h_cols[c] + off, cols[c], (size_t)cnt * sizeof(double),
                              cudaMemcpyDeviceToHost, L->copy));
    HK_CUDA(cudaEventRecord(L->freed[b], L->copy));
  }
  // the same two-level fold as phsp_weight_moments: slices -> supers -> total
  if (int rc = hk_fold_supers(part, chunks, 0, chunks, HK_WARP_SLICES, 2, 0, HK_SUPERS, cpart, stream))
    return rc;
  if (int rc = launch_fold(cpart, HK_SUPERS, 2, sums, st)) return rc;
  HK_CUDA(cudaStreamSynchronize(L->copy));
  if (h_wsums) {
    HK_CUDA(cudaMemcpyAsync(h_wsums, sums, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  HK_CUDA(cudaStreamSynchronize(st));
  return HK_OK;
}

}  // extern "C"

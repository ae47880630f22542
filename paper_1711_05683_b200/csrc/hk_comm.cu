// hk_comm.cu -- library lifetime (hk_init / hk_shutdown) and the path's one
// collective step, for a C host that drives several GPUs from one process.
//
// The reference's seam is a process pool: `workers` processes each reduce
// their 65 536-row batches to 4096-row chunk partials and the parent folds
// them in chunk order (parallel.py:18-92).  Here devices take the place of
// workers.  Events never move; only partials do -- either summed in place
// (ncclAllReduce, SURVEY.md 8(e) option i) or gathered to every device in
// device order and folded (ncclAllGather, option ii, bitwise invariant to the
// device count).  NCCL is dlopen'ed on hk_init, like NVRTC in hk_jit.cu, so
// the library links without it and the single-GPU paths never touch it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <vector>

#include "hepkit_cuda.h"
#include "hk_host.h"

namespace hk {

void jit_release();        // hk_jit.cu
void fcn_release();        // hk_fcn.cu
void sample_release();     // hk_sample.cu
void copy_lane_release();  // hk_runtime.cu

namespace {

struct Nccl {
  void* so = nullptr;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
};

std::mutex g_mu;
Nccl g_nccl;
std::vector<ncclComm_t> g_comms;

template <class F>
bool bind(void* so, const char* name, F* out) {
  *out = reinterpret_cast<F>(dlsym(so, name));
  return *out != nullptr;
}

// torch's bundled libnccl.so.2 is returned if the process already loaded it
bool load_nccl(Nccl& N) {
  if (N.so) return true;
  for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
    N.so = dlopen(name, RTLD_NOW | RTLD_LOCAL);
    if (N.so) break;
  }
  if (!N.so) return false;
  const bool ok = bind(N.so, "ncclCommInitAll", &N.init_all) && bind(N.so, "ncclCommDestroy", &N.destroy) &&
                  bind(N.so, "ncclAllReduce", &N.all_reduce) && bind(N.so, "ncclAllGather", &N.all_gather) &&
                  bind(N.so, "ncclGroupStart", &N.group_start) && bind(N.so, "ncclGroupEnd", &N.group_end) &&
                  bind(N.so, "ncclGetErrorString", &N.err);
  if (!ok) {
    dlclose(N.so);
    N = Nccl{};
  }
  return ok;
}

int nccl_fail(ncclResult_t r, const char* where) {
  set_error("%s: %s", where, g_nccl.err ? g_nccl.err(r) : "NCCL error");
  return HK_ECUDA;
}

#define HK_NCCL(call)                                         \
  do {                                                        \
    ncclResult_t hk_r_ = (call);                              \
    if (hk_r_ != ncclSuccess) return nccl_fail(hk_r_, #call); \
  } while (0)

void destroy_clique() {
  for (ncclComm_t c : g_comms)
    if (c) g_nccl.destroy(c);
  g_comms.clear();
}

int check_clique(int32_t n_dev, int64_t count) {
  HK_REQUIRE(!g_comms.empty(), "no device clique: call hk_init first");
  HK_REQUIRE(n_dev == (int32_t)g_comms.size(), "clique has %d devices, call passed %d",
             (int)g_comms.size(), n_dev);
  HK_REQUIRE(count >= 0, "negative count");
  return HK_OK;
}

cudaStream_t stream_of(void* const* streams, int g) { return streams ? as_stream(streams[g]) : nullptr; }

}  // namespace
}  // namespace hk

using namespace hk;

extern "C" {

int hk_init(int32_t n_devices) {
  int visible = 0;
  if (cudaGetDeviceCount(&visible) != cudaSuccess) {
    cudaGetLastError();
    visible = 0;
  }
  HK_REQUIRE(n_devices >= 1 && n_devices <= visible, "n_devices %d outside 1..%d visible", n_devices,
             visible);
  std::lock_guard<std::mutex> lock(g_mu);
  if ((int32_t)g_comms.size() == n_devices) return HK_OK;
  if (!load_nccl(g_nccl)) {
    set_error("hk_init: NCCL (libnccl.so.2) not loadable");
    return HK_ECUDA;
  }
  destroy_clique();
  int cur = 0;
  HK_CUDA(cudaGetDevice(&cur));
  std::vector<int> devs(n_devices);
  for (int g = 0; g < n_devices; ++g) devs[g] = g;
  std::vector<ncclComm_t> comms(n_devices, nullptr);
  const ncclResult_t r = g_nccl.init_all(comms.data(), n_devices, devs.data());
  cudaSetDevice(cur);  // ncclCommInitAll may leave another device current
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitAll");
  g_comms = std::move(comms);
  return HK_OK;
}

int hk_shutdown(void) {
  {
    std::lock_guard<std::mutex> lock(g_mu);
    destroy_clique();
  }
  jit_release();
  fcn_release();
  sample_release();
  copy_lane_release();
  return HK_OK;
}

int32_t hk_clique_size(void) {
  std::lock_guard<std::mutex> lock(g_mu);
  return (int32_t)g_comms.size();
}

int hk_allreduce_partials(double* const* d_bufs, int32_t n_dev, int64_t count, void* const* streams) {
  HK_NVTX("hk_allreduce_partials");
  std::lock_guard<std::mutex> lock(g_mu);
  if (int rc = check_clique(n_dev, count)) return rc;
  HK_REQUIRE(d_bufs, "NULL buffer list");
  for (int g = 0; g < n_dev; ++g) HK_REQUIRE(d_bufs[g] || count == 0, "NULL buffer for device %d", g);
  if (count == 0) return HK_OK;
  HK_NCCL(g_nccl.group_start());
  for (int g = 0; g < n_dev; ++g) {
    const ncclResult_t r = g_nccl.all_reduce(d_bufs[g], d_bufs[g], (size_t)count, ncclFloat64, ncclSum,
                                             g_comms[g], stream_of(streams, g));
    if (r != ncclSuccess) {
      g_nccl.group_end();
      return nccl_fail(r, "ncclAllReduce");
    }
  }
  HK_NCCL(g_nccl.group_end());
  return HK_OK;
}

int hk_allgather_partials(const double* const* d_send, double* const* d_recv, int32_t n_dev,
                          int64_t count, void* const* streams) {
  HK_NVTX("hk_allgather_partials");
  std::lock_guard<std::mutex> lock(g_mu);
  if (int rc = check_clique(n_dev, count)) return rc;
  HK_REQUIRE(d_send && d_recv, "NULL buffer list");
  for (int g = 0; g < n_dev; ++g)
    HK_REQUIRE((d_send[g] && d_recv[g]) || count == 0, "NULL buffer for device %d", g);
  if (count == 0) return HK_OK;
  HK_NCCL(g_nccl.group_start());
  for (int g = 0; g < n_dev; ++g) {
    const ncclResult_t r = g_nccl.all_gather(d_send[g], d_recv[g], (size_t)count, ncclFloat64, g_comms[g],
                                             stream_of(streams, g));
    if (r != ncclSuccess) {
      g_nccl.group_end();
      return nccl_fail(r, "ncclAllGather");
    }
  }
  HK_NCCL(g_nccl.group_end());
  return HK_OK;
}

}  // extern "C"

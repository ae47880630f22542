// hk_sample.cu -- accept-reject sampling of a p.d.f. on a box (rng.py:177-242),
// the toy/data synthesis that feeds the FCN.  Compiled with -fmad=false so a
// proposal lo + u * span rounds exactly like the reference's numpy.
//
// Event j owns the counter block (j + key.counter) * 2^16: proposal round t
// consumes counters +t*(d+1) .. +t*(d+1)+d (rng.py:214-219).  A thread walks
// an event's rounds until acceptance, then takes the next event (k_sample),
// so the output is independent of the launch shape, like the reference's
// worker invariance.
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <mutex>

#include "hepkit_cuda.h"
#include "hk_device.cuh"
#include "hk_host.h"

namespace hk {

constexpr int kMaxDim = 8;
constexpr uint64_t kProposalBlock = 1ull << 16;  // rng.py:42
constexpr uint64_t kBatch = 65536;               // parallel.py:21

struct SampleArgs {
  hk_program_t f;
  int32_t dim;
  int32_t max_rounds;
  double lo[kMaxDim];
  double span[kMaxDim];
  double ceiling;
  uint64_t base;
  uint64_t kc;
  uint64_t ev_begin;
  int64_t count;
  double* out[kMaxDim];
  unsigned long long* bad;  // [0] packed (batch, round, row) of a ceiling violation, [1] exhausted row
  unsigned long long* next;  // work-stealing event counter (zeroed before the launch)
};

// One proposal round of event `ev`: returns 1 accepted (point stored), 2 a
// ceiling violation (recorded), 0 rejected.
__device__ __forceinline__ int sample_round(const SampleArgs& a, uint64_t ev, int64_t i, int t) {
  const int d = a.dim;
  const uint64_t c0 = (ev + a.kc) * kProposalBlock + (uint64_t)t * (uint64_t)(d + 1);
  double pts[kMaxDim];
  for (int k = 0; k < d; ++k) pts[k] = a.lo[k] + to_unit(mix64(a.base + (c0 + k) * kGolden) >> 11) * a.span[k];
  const double u = to_unit(mix64(a.base + (c0 + d) * kGolden) >> 11);
  bool div0 = false;
  const double v = run_program(a.f, [&](int col) { return pts[col]; }, &div0);
  if (v > a.ceiling) {
    const unsigned long long key =
        ((unsigned long long)(ev / kBatch) << 40) | ((unsigned long long)t << 24) | (ev % kBatch);
    atomicMin(&a.bad[0], key);
    return 2;
  }
  if (u * a.ceiling < v) {
    for (int k = 0; k < d; ++k) a.out[k][i] = pts[k];
    return 1;
  }
  return 0;
}

// Persistent threads with work stealing: a thread runs proposal rounds of its
// current event and, once the event is accepted (or fails), takes the next
// event index from a device counter (one atomic per warp for all the lanes
// that need work).  With acceptance rate r a lane needs ~1/r rounds, but a
// warp of one-event-per-thread lanes waits for its slowest lane (~3-4x the
// mean at r = 1/8); here lanes stay busy until the events run out.  Each
// event's point depends only on its own counters, so the output is the same
// as one thread per event, whatever the schedule.
__global__ void __launch_bounds__(kBlock) k_sample(const __grid_constant__ SampleArgs a) {
  const int lane = threadIdx.x & 31;
  int64_t i = -1;  // current event (row of the output), -1: needs one
  int t = 0;
  for (;;) {
    const bool need = i < 0;
    const unsigned m = __ballot_sync(0xffffffffu, need);
    if (m) {
      unsigned long long base = 0;
      if (lane == __ffs(m) - 1) base = atomicAdd(a.next, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
      if (need) {
        i = (int64_t)(base + __popc(m & ((1u << lane) - 1u)));
        t = 0;
      }
    }
    const bool live = i < a.count;
    if (!__any_sync(0xffffffffu, live)) break;
    if (live) {
      const uint64_t ev = a.ev_begin + (uint64_t)i;
      const int r = sample_round(a, ev, i, t);
      if (r != 0) {
        i = -1;
      } else if (++t == a.max_rounds) {
        atomicMin(&a.bad[1], (unsigned long long)ev);
        i = -1;
      }
    }
  }
}

// The sampler's event counter, one per (device, stream): calls on one stream
// are serialised, calls on different streams get different counters.
// Zeroed on the stream before every launch; freed by hk_shutdown.
std::mutex g_ctr_mu;
std::map<std::pair<int, cudaStream_t>, unsigned long long*> g_ctr;

unsigned long long* sample_counter(cudaStream_t st) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(g_ctr_mu);
  unsigned long long*& p = g_ctr[{dev, st}];
  if (!p && cudaMalloc(&p, sizeof(unsigned long long)) != cudaSuccess) p = nullptr;
  return p;
}

void sample_release() {
  std::lock_guard<std::mutex> lock(g_ctr_mu);
  for (auto& kv : g_ctr)
    if (kv.second) cudaFree(kv.second);
  g_ctr.clear();
}

int sample_grid() {
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sample, kBlock, 0);
    grid = (sms > 0 ? sms : 148) * (per_sm > 0 ? per_sm : 1);
  }
  return grid;
}

}  // namespace hk

using namespace hk;

extern "C" int hk_sample_pdf(const hk_program_t* f, int32_t dim, const double* lo,
                             const double* span, double ceiling, const hk_key_t* key,
                             uint64_t ev_begin, int64_t count, int32_t max_rounds,
                             double* const* d_out, uint64_t* d_bad, void* stream) {
  HK_NVTX("hk_sample_pdf");
  HK_REQUIRE(f && lo && span && key && d_out && d_bad, "NULL argument");
  HK_REQUIRE(dim >= 1 && dim <= kMaxDim, "dimension %d outside 1..%d", dim, kMaxDim);
  HK_REQUIRE(key->mode == HK_RNG_REFERENCE, "sampling uses the reference stream");
  HK_REQUIRE(count >= 0 && max_rounds >= 1, "bad count/rounds");
  HK_REQUIRE(f->n_ops >= 1 && f->n_ops <= HK_MAX_PROGRAM, "bad program");
  if (count == 0) return HK_OK;
  SampleArgs a;
  std::memset(&a, 0, sizeof(a));
  a.f = *f;
  a.dim = dim;
  a.max_rounds = max_rounds;
  for (int k = 0; k < dim; ++k) {
    HK_REQUIRE(d_out[k], "output column %d NULL", k);
    a.lo[k] = lo[k];
    a.span[k] = span[k];
    a.out[k] = d_out[k];
  }
  a.ceiling = ceiling;
  a.base = key_base(key->seed, key->stream);
  a.kc = key->counter;
  a.ev_begin = ev_begin;
  a.count = count;
  a.bad = reinterpret_cast<unsigned long long*>(d_bad);
  cudaStream_t st = as_stream(stream);
  a.next = sample_counter(st);
  HK_REQUIRE(a.next, "sampler counter allocation failed");
  HK_CUDA(cudaMemsetAsync(a.next, 0, sizeof(unsigned long long), st));
  const int64_t want = (count + kBlock - 1) / kBlock;
  const int g = sample_grid();
  k_sample<<<(unsigned)(want < g ? want : g), kBlock, 0, st>>>(a);
  return check_launch("k_sample");
}

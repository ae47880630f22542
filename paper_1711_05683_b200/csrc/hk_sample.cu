// hk_sample.cu -- accept-reject sampling of a p.d.f. on a box (rng.py:177-242),
// the toy/data synthesis that feeds the FCN.  Compiled with -fmad=false so a
// proposal lo + u * span rounds exactly like the reference's numpy.
//
// Event j owns the counter block (j + key.counter) * 2^16: proposal round t
// consumes counters +t*(d+1) .. +t*(d+1)+d (rng.py:214-219).  One thread per
// event walks its rounds until acceptance, so the output is independent of
// the launch shape, like the reference's worker invariance.
#include <cuda_runtime.h>

#include <cstring>

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
};

__global__ void __launch_bounds__(kBlock) k_sample(const __grid_constant__ SampleArgs a) {
  const int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x;
  if (i >= a.count) return;
  const uint64_t ev = a.ev_begin + (uint64_t)i;
  const uint64_t block0 = (ev + a.kc) * kProposalBlock;
  const int d = a.dim;
  double pts[kMaxDim];
  for (int t = 0; t < a.max_rounds; ++t) {
    const uint64_t c0 = block0 + (uint64_t)t * (uint64_t)(d + 1);
    for (int k = 0; k < d; ++k)
      pts[k] = a.lo[k] + to_unit(mix64(a.base + (c0 + k) * kGolden) >> 11) * a.span[k];
    const double u = to_unit(mix64(a.base + (c0 + d) * kGolden) >> 11);
    bool div0 = false;
    const double v = run_program(a.f, [&](int col) { return pts[col]; }, &div0);
    if (v > a.ceiling) {
      const unsigned long long key =
          ((unsigned long long)(ev / kBatch) << 40) | ((unsigned long long)t << 24) | (ev % kBatch);
      atomicMin(&a.bad[0], key);
      return;
    }
    if (u * a.ceiling < v) {
      for (int k = 0; k < d; ++k) a.out[k][i] = pts[k];
      return;
    }
  }
  atomicMin(&a.bad[1], (unsigned long long)ev);
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
  k_sample<<<(unsigned)((count + kBlock - 1) / kBlock), kBlock, 0, as_stream(stream)>>>(a);
  return check_launch("k_sample");
}

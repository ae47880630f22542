// hk_fcn.cuh -- the FCN's event pass and fold, shared by the hand-specialised
// Gaussian + exponential kernels (hk_fcn.cu), the functor-program interpreter
// kernel (hk_fcn.cu) and the NVRTC-specialised density kernels (hk_jit.cu
// embeds this header), so every variant reduces in the same order:
//
//   per HK_FCN_TILE = 4096-row tile: 16 rows per thread, sum ln d as
//   ln(prod d) (LogProd), a fixed CTA tree -> one partial per tile (per-warp
//   partials without the tile barrier measured slower: the last CTA's fold
//   of 8x the partials costs more than the barrier stalls it removes);
//   the last CTA to finish folds the tile partials in a fixed order,
//   publishes (sum, first bad row, first zero divisor) -- optionally into
//   mapped pinned host memory -- and re-arms the workspace.
//
// nll = sum_k N_k - sum_e ln(sum_k N_k shape_k(x_e) / norm_k)  (fitting.py:175-210)
#pragma once

#include "hk_device.cuh"

namespace hk {

// sum_e ln d_e as ln(prod_e d_e), the product kept as a mantissa in [1, 2^16)
// and an integer binary exponent: one log per 16 events instead of 16, the
// exponent bookkeeping on the integer pipe.  Each product step rounds once
// (<= 2^-53 relative), the same order of error as the per-event logs the
// reference sums; far inside the 1e-10 FCN tolerance.
struct LogProd {
  double m = 1.0;
  int e = 0;

  __device__ __forceinline__ void add(double d) {
    long long b = __double_as_longlong(d);
    int ex = (int)((b >> 52) & 0x7ff);
    if (ex == 0) {  // subnormal (or zero, which the caller flags as bad)
      b = __double_as_longlong(d * 18014398509481984.0);  // * 2^54
      ex = (int)((b >> 52) & 0x7ff) - 54;
    }
    e += ex - 1023;
    m *= __longlong_as_double((b & 0x000FFFFFFFFFFFFFll) | 0x3FF0000000000000ll);
  }

  // add() for a value known to be a normal double (the factored density's s):
  // no subnormal check, same result
  __device__ __forceinline__ void add_normal(double d) {
    const long long b = __double_as_longlong(d);
    e += (int)((b >> 52) & 0x7ff) - 1023;
    m *= __longlong_as_double((b & 0x000FFFFFFFFFFFFFll) | 0x3FF0000000000000ll);
  }

  // move m's binary exponent into e (exact): keeps m in [1, 2) so a thread
  // can multiply any number of events with one log at the end
  __device__ __forceinline__ void renorm() {
    const long long b = __double_as_longlong(m);
    e += (int)((b >> 52) & 0x7ff) - 1023;
    m = __longlong_as_double((b & 0x000FFFFFFFFFFFFFll) | 0x3FF0000000000000ll);
  }

  __device__ __forceinline__ double value() const {
    const double ln2_hi = 6.93147180369123816490e-01;  // 32 significant bits: e * ln2_hi is exact
    const double ln2_lo = 1.90821492927058770002e-10;
    return (e * ln2_hi + log(m)) + e * ln2_lo;
  }
};

// FCN tiles of HK_FCN_TILE = 4096 rows (16 per thread, one log per 16
// events).  2048-row tiles (8.25 waves instead of 4.1 for 1e7 events, less
// tail) measured slower on B200 -- 38.3 vs 36.0 us per kernel -- because the
// extra logs cost more than the tail they remove.
constexpr int kFcnTile = HK_FCN_TILE;
constexpr int kFcnRows = kFcnTile / kBlock;

// One-launch FCN: the same event pass, then the last CTA to finish folds all
// chunk partials in a fixed order (deterministic whichever CTA is last),
// publishes (sum, first bad row) and re-arms the workspace for the next call.
// The first-bad cell holds ~row under atomicMax so that an all-zero
// workspace means "no bad row".
struct FcnWork {
  double* out;               // [0] sum of logs, [1] first bad row, [5] first zero divisor (u64 bits)
  unsigned long long* bad;   // ~row of the first non-positive density, 0 = none
  unsigned int* ticket;      // CTAs finished
  double* part;              // one partial per chunk
  unsigned long long* div0;  // ~row of the first zero divisor, 0 = none (NULL: not tracked)
  // optional zero-copy publication into mapped pinned host memory:
  // host_mail[1..3] = (sum, first bad row, first zero-divisor row), then
  // host_mail[0] = seq (after a system fence)
  volatile unsigned long long* host_mail;
  unsigned long long seq;
  // tile schedule (fcn_schedule): CTA b < full owns tile b (4096 rows); the
  // rows from full * 4096 on are split evenly over tail_ctas more CTAs, so
  // the last wave is short instead of a few full tiles on an idle GPU
  int64_t full, tail_ctas;
  // dynamic tile counter of the persistent (TMA-pipelined) FCN; re-armed to
  // 0 by the last CTA (NULL: not used)
  unsigned long long* next;
  // scan direction: 1 walks the tiles last to first.  The host flips it on
  // every call over the same workspace (fcn_flip), so each pass starts on the
  // tiles the previous pass touched last -- the ones still in L2 -- instead
  // of cycling through a column larger than L2 in LRU order (1e7 events:
  // 8% L2 hits).  Tile partials keep their index, so values do not change.
  int32_t rev;
};

// the tile a CTA's b-th unit covers in this call's scan direction
__device__ __forceinline__ int64_t fcn_tile(const FcnWork& w, int64_t b, int64_t tiles) {
  return w.rev ? tiles - 1 - b : b;
}

__device__ __forceinline__ void fcn_range(const FcnWork& w, int64_t n, int64_t b, int64_t* begin,
                                          int64_t* end) {
  if (b < w.full) {
    *begin = b * kFcnTile;
    *end = *begin + kFcnTile;
    return;
  }
  const int64_t t0 = w.full * kFcnTile, rem = n - t0, j = b - w.full;
  *begin = t0 + rem * j / w.tail_ctas;
  *end = t0 + rem * (j + 1) / w.tail_ctas;
}

// b, z: the first-bad and first-zero-divisor cells, read by the caller after
// every CTA has finished (no other thread touches them any more), so they
// are re-armed with plain stores
__device__ __forceinline__ void fcn_publish(const FcnWork& w, double total, unsigned long long b,
                                            unsigned long long z) {
  if (b) *w.bad = 0ull;
  if (z) *w.div0 = 0ull;
  w.out[0] = total;
  w.out[1] = __longlong_as_double((long long)~b);
  w.out[5] = __longlong_as_double((long long)~z);
  *w.ticket = 0u;
  if (w.next) *w.next = 0ull;
  if (w.host_mail) {
    w.host_mail[1] = (unsigned long long)__double_as_longlong(total);
    w.host_mail[2] = ~b;
    w.host_mail[3] = ~z;
    __threadfence_system();
    w.host_mail[0] = w.seq;
  }
}

__device__ __forceinline__ void fcn_publish(const FcnWork& w, double total) {
  const unsigned long long b = atomicExch(w.bad, 0ull);
  const unsigned long long z = w.div0 ? atomicExch(w.div0, 0ull) : 0ull;
  fcn_publish(w, total, b, z);
}

// Last CTA: fixed-order fold of the `chunks` tile partials, plus `base` (a
// per-call constant the variant hoisted out of the event sum), then publish.
// Called by every thread of every CTA after its tiles are stored.
// 1: the CTA ticket is one atom.add.acq_rel.gpu (a MEMBAR.ALL.GPU + ATOM in
// SASS) instead of fence.sc + atomicAdd, and the last CTA needs no second
// fence (its partial reads are L2 loads after the acquire): one wave of
// tiles 9.4 -> 8.2 us on B200 (profiles/r02_fcn_acqrel_ab.jsonl)
#ifndef HK_FCN_ACQREL
#define HK_FCN_ACQREL 1
#endif
__device__ __forceinline__ void fcn_finish(const FcnWork& w, int64_t chunks, double base = 0.0) {
  // block_sum_store's writer is thread 0: it alone fences before the ticket
  __shared__ unsigned int s_ticket;
  if (threadIdx.x == 0) {
#if HK_FCN_ACQREL
    // one acquire-release RMW instead of two sequentially consistent fences:
    // releases this CTA's partial, and (for the last CTA) acquires every other's
    unsigned int t;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(w.ticket) : "memory");
    s_ticket = t;
#else
    __threadfence();
    s_ticket = atomicAdd(w.ticket, 1u);
#endif
  }
  __syncthreads();
  if (s_ticket != gridDim.x - 1) return;
#if !HK_FCN_ACQREL
  __threadfence();
#endif
  // the problem cells are final now: their loads overlap the partials' reads
  unsigned long long b = 0ull, z = 0ull;
  if (threadIdx.x == 0) {
    b = __ldcg(w.bad);
    if (w.div0) z = __ldcg(w.div0);
  }
  double acc[1] = {0.0};
  for (int64_t i = threadIdx.x; i < chunks; i += kBlock) acc[0] += __ldcg(w.part + i);
  __shared__ double total;
  block_sum_store<1>(acc, &total);
  if (threadIdx.x == 0) fcn_publish(w, total + base, b, z);
}

// The FCN over a density functor dens(row, &div0) -> density (any model: the
// interpreter or a specialised program).  Non-positive / non-finite densities
// (fitting.py:200-205) and zero divisors (functors.py:200-207) are recorded
// as ~row under atomicMax, so the smallest row wins and 0 means none.
// kUnroll (the NVRTC-specialised density): full tiles run their 16 rows
// unrolled, so the compiler issues every row's column loads before the
// arithmetic instead of one load latency per row; the rows, their order and
// every rounding are those of the rolled loop (same values as the
// interpreter's pass).
template <bool kUnroll = false, class Dens>
__device__ __forceinline__ void fcn_density_pass(const FcnWork& w, int64_t n, const Dens& dens) {
  const int64_t chunks = w.full + w.tail_ctas;
  for (int64_t b = blockIdx.x; b < chunks; b += gridDim.x) {
    const int64_t ch = fcn_tile(w, b, chunks);
    int64_t begin, end;
    fcn_range(w, n, ch, &begin, &end);
    unsigned long long bad = 0, zero = 0;
    LogProd lp;
    const auto row = [&](int64_t r) {
      bool z = false;
      const double d = dens(r, z);
      if (z) zero = max(zero, ~(unsigned long long)r);
      if (!(d > 0.0) || !isfinite(d)) bad = max(bad, ~(unsigned long long)r);
      lp.add(d);
    };
    if (kUnroll && end - begin == kFcnTile) {
#pragma unroll
      for (int i = 0; i < kFcnRows; ++i) row(begin + threadIdx.x + (int64_t)i * kBlock);
    } else {
#pragma unroll 1
      for (int i = 0; i < kFcnRows; ++i) {
        const int64_t r = begin + threadIdx.x + (int64_t)i * kBlock;
        if (r < end) row(r);
      }
    }
    double acc[1] = {lp.value()};
    if (bad) atomicMax(w.bad, bad);
    if (zero) atomicMax(w.div0, zero);
    block_sum_store<1>(acc, w.part + ch);
  }
  fcn_finish(w, chunks);
}

// Arguments of the program-driven FCN kernels (interpreter and NVRTC; the
// specialised source mirrors this struct through this header).
struct FcnProgArgs {
  const double* cols[HK_FCN_MAX_OBS];
  int64_t n;
  FcnWork w;
  hk_program_t prog;  // constants (yields, norms, shape parameters) change per call
};

}  // namespace hk

// hk_fcn.cu -- the unbinned extended NLL (FCN) event sum for sm_100a.
//
// nll = sum_k N_k - sum_e ln(sum_k N_k shape_k(x_e) / norm_k)   (fitting.py:175-210)
//
// The host computes the norms (fitting.py:80-89, 103-123) and the
// expected total; this kernel does the data pass: fused p.d.f. evaluation ->
// density -> positivity check -> log -> fixed-order CTA sum per 4096-row
// chunk.  The per-component constants are folded on the host
// (A_k = N_k / (sigma_k sqrt(2 pi) norm_k), 1/sigma_k, -1/tau_k), which moves a
// density by a few ulp -- far inside the 1e-10 FCN tolerance.  For the
// Gaussian + exponential model the density is factored as e^M * s
// (density_factored): one exp per event, one log per 16 events, ~35 FP64
// instructions per event -- FP64-pipe bound, with the 8 B/event column
// usually L2-resident (1e7 events = 80 MB < 126 MB L2).
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include "hepkit_cuda.h"
#include "hk_device.cuh"
#include "hk_fcn.cuh"
#include "hk_host.h"

namespace hk {

struct Coeffs {
  int32_t n_comp;
  int32_t kind[HK_MAX_COMPONENTS];
  double amp[HK_MAX_COMPONENTS];    // gauss: N/(s*sqrt(2pi)*norm); expo: N/norm
  double shift[HK_MAX_COMPONENTS];  // gauss: mean
  double scale[HK_MAX_COMPONENTS];  // gauss: 1/sigma; expo: -1/tau
  // factored Gaussian+exponential path (kFcnFactored): exponents M inside
  // (m_lo, m_hi) give amp_k e^M a normal, finite double for both k; q2, q1,
  // q0: A - B as a quadratic in x - mean
  double m_lo, m_hi;
  double q2, q1, q0;
  // kFcnFast (fast_coeffs): amplitudes over their max c, q = log2(e) (A - B) as
  // a quadratic in x, and base = sum_e B(x_e) + n ln c = b sum(x) + n ln c
  double fa[2], fq[3], base;
  int32_t fast;
};

// One parameter point of the factored Gaussian + exponential density, for
// the multi-point pass (hk_nll_eval_many): the fields the factored and
// reference-order paths read, under Coeffs' names so the same templates
// produce the same bits.
struct FPoint {
  double amp[2], shift[1], scale[2];
  double m_lo, m_hi;
  double q2, q1, q0;
  double fa[2], fq[3], base;  // kFcnFast (all doubles: the session copies it word by word)
};

__host__ __forceinline__ FPoint make_point(const Coeffs& c) {
  FPoint p;
  p.amp[0] = c.amp[0];
  p.amp[1] = c.amp[1];
  p.shift[0] = c.shift[0];
  p.scale[0] = c.scale[0];
  p.scale[1] = c.scale[1];
  p.m_lo = c.m_lo;
  p.m_hi = c.m_hi;
  p.q2 = c.q2;
  p.q1 = c.q1;
  p.q0 = c.q0;
  p.fa[0] = c.fa[0];
  p.fa[1] = c.fa[1];
  p.fq[0] = c.fq[0];
  p.fq[1] = c.fq[1];
  p.fq[2] = c.fq[2];
  p.base = c.base;
  return p;
}

// FCN kernel variants
constexpr int kFcnGeneric = 0;   // any component list
constexpr int kFcnGE = 1;        // Gaussian + exponential, reference op order
constexpr int kFcnFactored = 2;  // Gaussian + exponential, one exp per event
constexpr int kFcnFast = 3;      // kFcnFactored with the data range proved on the host (fast_row)

// exp for the FCN data pass.  libdevice's: a 64-entry shared-memory table
// variant (11 FP64 ops instead of ~17) measured slower on B200 (40.6 vs 36.1 us
// per 1e7 events) -- LDS latency in the dependency chain -- and was dropped.
__device__ __forceinline__ double fcn_exp(double v) { return ::exp(v); }

__device__ __forceinline__ double density(const Coeffs& c, double x) {
  double d = 0.0;
#pragma unroll 1
  for (int k = 0; k < c.n_comp; ++k) {
    double t;
    if (c.kind[k] == HK_SHAPE_GAUSS) {
      const double z = (x - c.shift[k]) * c.scale[k];
      t = c.amp[k] * fcn_exp(-0.5 * z * z);
    } else {
      t = c.amp[k] * fcn_exp(x * c.scale[k]);
    }
    d = k == 0 ? t : d + t;
  }
  return d;
}

// Two-component Gaussian + exponential specialisation (the benchmark model,
// cli.py:316-320 / toymodel.py): no component loop, no kind branches.
template <class C>
__device__ __forceinline__ double density_ge(const C& c, double x) {
  const double z = (x - c.shift[0]) * c.scale[0];
  return c.amp[0] * fcn_exp(-0.5 * z * z) + c.amp[1] * fcn_exp(x * c.scale[1]);
}

// d = a0 e^A + a1 e^B = e^M (a0 e^(A-M) + a1 e^(B-M)), M = max(A, B): one
// exp per event (of min - max <= 0) instead of two.  ln d = M + ln s is then
// summed as sum M + ln(prod s).  Returns false -- the caller falls back to
// density_ge and its positivity check -- unless M is inside the window where
// both reference terms are finite and the larger one is a normal positive
// double, and s is positive and finite: then d > 0 and finite exactly as the
// reference computes it, and only the rounding differs (a few ulp per event).
// The host admits this path only for amps in (1e-250, 1e300) with a finite
// sum, so inside the window t = e^(min-max) is in [0, 1] and s lies in
// [min amp, amp0 + amp1]: positive and finite, no separate check.  A NaN or
// infinite x makes M NaN or infinite and fails the window.
// e^v for v <= 0 on the factored path: 2^(v log2 e) = 2^n 2^f with
// n = rint(v log2 e), f in [-1/2, 1/2] and 2^f a degree-9 polynomial (fitted
// by reweighted least squares; 1.9e-14 relative on the interval), n added to
// the exponent field.  13 FP64 instructions against ~17 for libdevice's exp;
// relative error <= ~1e-13, dominated by the rounding of v log2 e.  Summed
// over 1e7 events that moves ln L by <= 1e-6 absolute, ~1e-14 relative --
// the FCN's budget is 1e-10.  v < -707 returns 0 (the host admits the
// factored path only for amplitude ratios below 1e200, so the dropped term
// is < 1e-100 of the density).
__device__ __forceinline__ double fcn_exp_neg(double v) {
  const double y = v * 1.4426950408889634;          // log2(e)
  const double magic = 6755399441055744.0;          // 1.5 * 2^52: rounds y to an integer
  const double r = y + magic;
  const double f = y - (r - magic);
  double p = 1.0155003747016481e-07;
  p = fma(p, f, 1.3259339489411853e-06);
  p = fma(p, f, 1.5252960462935984e-05);
  p = fma(p, f, 1.5403435240126103e-04);
  p = fma(p, f, 1.3333557659884130e-03);
  p = fma(p, f, 9.6181291916688500e-03);
  p = fma(p, f, 5.5504108668414306e-02);
  p = fma(p, f, 2.4022650695651396e-01);
  p = fma(p, f, 6.9314718055987630e-01);
  p = fma(p, f, 1.0000000000000115e+00);
  const long long n = (long long)__double2loint(r);  // the low word of r is rint(y)
  const double e = __longlong_as_double(__double_as_longlong(p) + (n << 52));
  return v < -707.0 ? 0.0 : e;
}

// The factored density d = e^M s with one exponential per event:
//   A = -z^2/2, z = (x - mean)/sigma; B = -x/tau; M = max(A, B);
//   t = e^-|A - B|; s = amp_big + amp_small t.
// (HK_FCN_EXP_POLY: q = A - B as a quadratic in u = x - mean,
//   (q2 u + q1) u + q0 with q2 = -1/(2 sigma^2), q1 = 1/tau, q0 = mean/tau,
//   M = B + max(q, 0), t = fcn_exp_neg(-|q|).)
// Returns false (the caller falls back to the reference-order density_ge and
// its positivity check) unless M is inside the window where both terms are
// finite normal doubles; a NaN x fails the window.  Against the reference op
// order each event's density moves by a few 1e-13 relative.
//
// Measured on B200 (tools/fcn_kernel_time.py, 1e7 events): the quadratic +
// fcn_exp_neg form (HK_FCN_EXP_POLY) saves ~4 FP64 instructions per event but
// needs more registers -- one-point pass 31.1 vs 32.2 us, the multi-point
// kernel 32.7 vs 28.8 us per point (spills at 64 registers) -- so the
// default is the libdevice form below.
template <class C>
__device__ __forceinline__ bool density_factored(const C& c, double x, double* s, double* M) {
#ifndef HK_FCN_EXP_POLY  // libdevice exp, A and B separately
  const double z = (x - c.shift[0]) * c.scale[0];
  const double A = -0.5 * z * z;
  const double B = x * c.scale[1];
  const bool ga0 = A >= B;
  *M = ga0 ? A : B;
  const double t0 = fcn_exp(ga0 ? B - A : A - B);
  *s = ga0 ? c.amp[0] + c.amp[1] * t0 : c.amp[0] * t0 + c.amp[1];
  return *M > c.m_lo && *M < c.m_hi;
#else
  const double u = x - c.shift[0];
  const double q = fma(fma(c.q2, u, c.q1), u, c.q0);
  const double B = x * c.scale[1];
  const bool ga = q >= 0.0;  // NaN: false, M = B + ... = NaN
  *M = ga ? B + q : B;
  const double t = fcn_exp_neg(ga ? -q : q);
  *s = ga ? fma(c.amp[1], t, c.amp[0]) : fma(c.amp[0], t, c.amp[1]);
  return *M > c.m_lo && *M < c.m_hi;
#endif
}

// 2^f on f in [-1/2, 1/2]: degree-8 polynomial (fitted by reweighted least
// squares; 2.9e-12 relative on the interval evaluated in double).  In the
// constant bank so each DFMA takes its coefficient as an operand (no UMOV).
__constant__ double kExp2Poly[9] = {1.328492507863422e-06,  1.5308981596230215e-05, 0.00015403372425094143,
                                    0.001333345520138187,   0.009618129182690833,   0.05550410935556957,
                                    0.2402265069621877,     0.6931471805476419,     0.9999999999999317};

// 2^y for -1000 <= y <= 60 (the host proves the range, fast_coeffs): 2^n 2^f,
// n = rint(y), f in [-1/2, 1/2], n added to the high word (2^f is normal and
// 2^n in [2^-1000, 2^60], so the result is a normal double, no special path).
// Moves each density by <= 2.9e-12 relative: summed over 1e7 events at most
// 3e-5 of ln L, ~1e-13 relative -- the FCN's budget is 1e-10.
__device__ __forceinline__ double fcn_exp2(double y) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52: rounds y to an integer
  const double r = y + magic;
  const double f = y - (r - magic);
  double p = kExp2Poly[0];
#pragma unroll
  for (int k = 1; k < 9; ++k) p = fma(p, f, kExp2Poly[k]);
  const int n = __double2loint(r);  // the low word of r is rint(y)
  return __hiloint2double(__double2hiint(p) + (n << 20), __double2loint(p));
}

// One event of the kFcnFast FCN.  With A = -((x - mean)/sigma)^2 / 2 and
// B = b x the two reference terms are amp0 e^A and amp1 e^B, so
//   d = c e^B s',  s' = fa1 + fa0 2^q,  q = log2(e) (A - B) = (fq0 x + fq1) x + fq2,
// c = max(amp0, amp1), fa = amp / c.  The host (fast_coeffs) has proved over
// the column's [min, max] that both reference terms are finite normal
// doubles, that the density is positive and that -1000 <= q <= 60, so there
// is no per-event check and no select: s' lies in [1e-15, 1 + 2^60] and a
// product of 16 of them stays a normal double.  ln d = B + ln c + ln s';
// sum_e B = b sum(x) (the column statistic) and n ln c are constants added
// once by the fold (`base`).  Per event 15 FP64 instructions (q, the
// exponential, s', the product); the exponent insert is on the integer pipe.
template <class C>
__device__ __forceinline__ void fast_row(const C& c, double x, double& prod) {
  const double q = fma(fma(c.fq[0], x, c.fq[1]), x, c.fq[2]);
  prod *= fma(c.fa[0], fcn_exp2(q), c.fa[1]);
}

// column loads of the kFcnFast tiles (HK_FCN_LD: 0 __ldg; 1 ld.global.nc
// with an L2 evict_last policy; 2 plain ld.global with evict_last).  The
// evict_last policies measured no gain on B200 (1e7: 20.4 vs 20.3 us; the
// scan order is what keeps the column in L2, fcn_flip):
// profiles/r02_fcn_ld_ab.jsonl, r02_fcn_l2_steady_state.txt
#ifndef HK_FCN_LD
#define HK_FCN_LD 0
#endif
__device__ __forceinline__ double fcn_ldx(const double* p) {
#if HK_FCN_LD == 0
  return __ldg(p);
#else
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  double v;
#if HK_FCN_LD == 1
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
#else
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
#endif
  return v;
#endif
}

// rows of a full tile loaded per batch on the kFcnFast path
#ifndef HK_FCN_FAST_BATCH
#define HK_FCN_FAST_BATCH 16
#endif

// One tile: returns sum ln d over this thread's rows; flags
// d <= 0 / non-finite (fitting.py:200-205) as ~row in *bad (max = first row).
template <int V, class C>
__device__ __forceinline__ void fcn_row(const C& c, double xv, int64_t row, LogProd& lp,
                                       double& msum, unsigned long long* bad) {
  if (V == kFcnFactored) {
    double s, M;
    if (density_factored(c, xv, &s, &M)) {
      lp.add_normal(s);  // s in [min amp, amp0 + amp1]: normal
      msum += M;
      return;
    }
  }
  double d;
  if constexpr (V == kFcnGeneric)
    d = density(c, xv);
  else
    d = density_ge(c, xv);
  if (!(d > 0.0) || !isfinite(d)) *bad = max(*bad, ~(unsigned long long)row);
  lp.add(d);
}

// sum ln d over rows [begin, end) (at most one tile): all 16 loads in flight
// for a full tile, a guarded loop otherwise
// tid: the thread's slot in the tile (threadIdx.x, or a warp-scheduled
// virtual id in the resident session -- same rows, same order)
template <int V, class C>
__device__ __forceinline__ double range_logsum(const double* __restrict__ x, int64_t begin,
                                               int64_t end, const C& c,
                                               unsigned long long* bad, int tid) {
  const int64_t r0 = begin + tid;
  if constexpr (V == kFcnFast) {
    // the product of <= 16 factors s' in [1e-15, 2] stays normal: one log per
    // thread and tile, no exponent bookkeeping
    double prod = 1.0;
    if (end - begin == kFcnTile) {
#pragma unroll
      for (int i0 = 0; i0 < kFcnRows; i0 += HK_FCN_FAST_BATCH) {
        double xv[HK_FCN_FAST_BATCH];
#pragma unroll
        for (int i = 0; i < HK_FCN_FAST_BATCH; ++i) {
#ifdef HK_FCN_PROBE_NOLOAD  // A/B probe only: rows synthesised from the row index
          xv[i] = (double)((r0 + (i0 + i) * kBlock) & 1023) * 0.009765625;
#else
          xv[i] = fcn_ldx(x + r0 + (i0 + i) * kBlock);
#endif
        }
#pragma unroll
        for (int i = 0; i < HK_FCN_FAST_BATCH; ++i) {
#ifdef HK_FCN_PROBE_NOCOMPUTE  // A/B probe only: loads + reductions, no arithmetic
          prod += xv[i];
#else
          fast_row(c, xv[i], prod);
#endif
        }
      }
    } else {
      for (int i = 0; i < kFcnRows; ++i) {
        const int64_t r = r0 + i * kBlock;
        if (r < end) fast_row(c, __ldg(x + r), prod);
      }
    }
    return log(prod);
  }
  LogProd lp;
  double msum = 0.0;
  if (end - begin == kFcnTile) {
    double xv[kFcnRows];
#pragma unroll
    for (int i = 0; i < kFcnRows; ++i) xv[i] = __ldg(x + r0 + i * kBlock);
#pragma unroll
    for (int i = 0; i < kFcnRows; ++i) fcn_row<V>(c, xv[i], r0 + i * kBlock, lp, msum, bad);
  } else {  // the ragged last tile
    for (int i = 0; i < kFcnRows; ++i) {
      const int64_t r = r0 + i * kBlock;
      if (r < end) fcn_row<V>(c, __ldg(x + r), r, lp, msum, bad);
    }
  }
  return V == kFcnFactored ? lp.value() + msum : lp.value();
}

template <int V>
__device__ __forceinline__ double chunk_logsum(const double* __restrict__ x, int64_t n,
                                               const Coeffs& c, int64_t ch,
                                               unsigned long long* bad) {
  const int64_t b = ch * kFcnTile;
  return range_logsum<V>(x, b, b + kFcnTile < n ? b + kFcnTile : n, c, bad, threadIdx.x);
}

template <int V>
__global__ void __launch_bounds__(kBlock) k_nll(const double* __restrict__ x, int64_t n,
                                                const __grid_constant__ Coeffs c,
                                                double* __restrict__ part,
                                                unsigned long long* first_bad) {
  const int64_t chunks = (n + kFcnTile - 1) / kFcnTile;
  for (int64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
    unsigned long long bad = 0;
    double acc[1] = {chunk_logsum<V>(x, n, c, ch, &bad)};
    if (bad) record_bad(first_bad, ~bad);
    block_sum_store<1>(acc, part + ch);
  }
}

// 4 CTAs/SM (64 registers) measured best for the one-launch FCN on B200:
// C-ABI call 47.8 us; 5 CTAs (48 regs + spills) 50.6, 6 CTAs 53.9, 8 CTAs 64.4,
// and an unconstrained (256, 1) bound lets ptxas take 216 registers (82 us).
#ifndef HK_FCN_MIN_BLOCKS
#define HK_FCN_MIN_BLOCKS 4
#endif
// (A persistent one-wave grid -- 592 CTAs over equal contiguous row ranges,
// one log per thread -- measured slower on B200: 53.7 us per call with 4-row
// groups, 60.2 us with 16-row groups and spills, against 44.5 us for tiles.)

template <int V>
__global__ void __launch_bounds__(kBlock, HK_FCN_MIN_BLOCKS) k_nll_fused(const double* __restrict__ x, int64_t n,
                                                      const __grid_constant__ Coeffs c, FcnWork w) {
#ifdef HK_PROBE_EMPTY  // timing probe: launch floor
  return;
#endif
  const int64_t chunks = w.full + w.tail_ctas;
  for (int64_t b = blockIdx.x; b < chunks; b += gridDim.x) {
    const int64_t ch = fcn_tile(w, b, chunks);
    unsigned long long bad = 0;
    int64_t begin, end;
    fcn_range(w, n, ch, &begin, &end);
    double acc[1] = {range_logsum<V>(x, begin, end, c, &bad, threadIdx.x)};
    if (bad) atomicMax(w.bad, bad);
    block_sum_store<1>(acc, w.part + ch);
  }
#ifndef HK_PROBE_NOFINISH  // timing probe: no ticket, fold or publication
  fcn_finish(w, chunks, V == kFcnFast ? c.base : 0.0);
#endif
}

// ----------------------------------------- TMA-pipelined kFcnFast FCN -----
// Persistent CTAs (3 per SM) take 4096-row tiles from a device counter; one
// thread streams each tile (32 KB) into shared memory with a 1-D bulk TMA
// copy (cp.async.bulk, completion on an mbarrier) two tiles ahead, so the
// column's load latency overlaps the previous tiles' arithmetic and the LSU
// issues no global loads.  Per tile the arithmetic, row order and partial
// are range_logsum<kFcnFast>'s (the ragged last tile runs that function), so
// every value is bit-identical to k_nll_fused<kFcnFast>, k_nll_many and the
// session.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n HK_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HK_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

constexpr int kTmaStages = 2;
constexpr int kTmaSmem = kTmaStages * kFcnTile * (int)sizeof(double);  // 64 KB dynamic
// smallest column the persistent TMA FCN takes (shorter: k_nll_fused<kFcnFast>).
// Measured on B200 (tools/gpu_r02_tma.sh, gpurun_out -> profiles/r02_fcn_tma_ab.jsonl),
// kernel us TMA vs k_nll_fused: 5e6 16.6 vs 15.7, 1e7 24.8 vs 22.6 (L2-resident
// column: the launched tiles' 16 loads in flight per thread win), 2e7 47.1 vs
// 48.9, 5e7 88.1 vs 96.1 (HBM-resident: the TMA stream wins by 8%).
#ifndef HK_FCN_TMA_MIN_N
#define HK_FCN_TMA_MIN_N (4096LL * 4096)
#endif
#ifndef HK_FCN_TMA_MIN_BLOCKS
#define HK_FCN_TMA_MIN_BLOCKS 3
#endif

__global__ void __launch_bounds__(kBlock, HK_FCN_TMA_MIN_BLOCKS)
    k_nll_fast_tma(const double* __restrict__ x, int64_t n, const __grid_constant__ Coeffs c, FcnWork w) {
  extern __shared__ __align__(128) double s_x[];  // kTmaStages tiles
  __shared__ __align__(8) uint64_t s_bar[kTmaStages];
  __shared__ long long s_tile[kTmaStages];
  const int64_t full = n / kFcnTile;               // tiles the TMA streams
  const int64_t chunks = (n + kFcnTile - 1) / kFcnTile;
  // thread 0: take the next tile index and start its copy into stage s
  // s_tile: the tile in this call's scan direction, or -1 once the counter
  // has passed the last one
  auto issue = [&](int s) {
    const long long u = (long long)atomicAdd(w.next, 1ull);
    const long long t = u < chunks ? (long long)fcn_tile(w, u, chunks) : -1;
    s_tile[s] = t;
    if (t >= 0 && t < full) tma_load_1d(s_x + s * kFcnTile, x + t * kFcnTile, kFcnTile * sizeof(double), &s_bar[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < kTmaStages; ++s) issue(s);
  }
  __syncthreads();
  uint32_t phase = 0;  // bit s: parity of stage s's next completion
  for (int k = 0;; ++k) {
    const int s = k % kTmaStages;
    const long long t = s_tile[s];
    if (t < 0) break;
    double acc[1];
    if (t < full) {
      mbar_wait(&s_bar[s], (phase >> s) & 1u);
      phase ^= 1u << s;
      const double* xs = s_x + s * kFcnTile + threadIdx.x;
      double prod = 1.0;
#pragma unroll
      for (int i = 0; i < kFcnRows; ++i) fast_row(c, xs[i * kBlock], prod);
      acc[0] = log(prod);
    } else {  // the ragged last tile
      unsigned long long bad = 0;
      acc[0] = range_logsum<kFcnFast>(x, t * kFcnTile, n, c, &bad, threadIdx.x);
    }
    block_sum_store<1>(acc, w.part + t);  // its barriers: every read of stage s is done
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the async-proxy write
      issue(s);
    }
  }
  fcn_finish(w, chunks, c.base);
}

int fast_tma_grid() {
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_nll_fast_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_nll_fast_tma, kBlock, kTmaSmem);
    grid = (sms > 0 ? sms : 148) * (per_sm > 0 ? per_sm : 1);
  }
  return grid;
}

// Reference op order (fitting.py:160-166, functors.py:142-143, :161) with no
// contraction -- used only for the value quoted in the error message.
__global__ void k_density_exact(const double* x, int64_t n, const __grid_constant__ hk_model_t m,
                                double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double xv = x[i];
  double d = 0.0;
  for (int k = 0; k < m.n_comp; ++k) {
    double shape;
    if (m.kind[k] == HK_SHAPE_GAUSS) {
      const double s = m.p1[k];
      const double z = (xv - m.p0[k]) / s;
      shape = exp(__dmul_rn(-0.5 * z, z)) / __dmul_rn(s, 2.5066282746310002);
    } else {
      shape = exp(-xv / m.p0[k]);
    }
    const double t = __dmul_rn(m.yield[k], shape / m.norm[k]);
    d = k == 0 ? t : __dadd_rn(d, t);
  }
  out[i] = d;
}

int launch_fold(const double* parts, int64_t n, int width, double* out, cudaStream_t st);

// pdf_k(x) = shape_k(x)/norm_k without the yield (fitting.py:91-92)
struct PdfCoeffs {
  int32_t kind[4];
  double amp[4], shift[4], scale[4], yield[4];
};

template <int K>
__global__ void __launch_bounds__(kBlock) k_yield(const double* __restrict__ x, int64_t n,
                                                  const __grid_constant__ PdfCoeffs c,
                                                  double* __restrict__ part,
                                                  unsigned long long* first_bad) {
  constexpr int W = K + K * K;
  const int64_t chunks = (n + HK_CHUNK - 1) / HK_CHUNK;
  for (int64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
    double acc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) acc[w] = 0.0;
    // one row's contribution, in row order (the same sums whichever path)
    const auto row = [&](double xv, int64_t r) {
      double p[K], d = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (c.kind[k] == HK_SHAPE_GAUSS) {
          const double z = (xv - c.shift[k]) * c.scale[k];
          p[k] = c.amp[k] * exp(-0.5 * z * z);
        } else {
          p[k] = c.amp[k] * exp(xv * c.scale[k]);
        }
        d += p[k] * c.yield[k];
      }
      // [0]: density not > 0 (fitting.py:418); [1]: also non-finite (splot.py:38)
      if (!(d > 0.0)) record_bad(first_bad, (uint64_t)r);
      if (first_bad && (!(d > 0.0) || !isfinite(d))) record_bad(first_bad + 1, (uint64_t)r);
      const double inv = 1.0 / d;
#pragma unroll
      for (int k = 0; k < K; ++k) p[k] *= inv;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        acc[k] += p[k];
#pragma unroll
        for (int j = 0; j < K; ++j) acc[K + k * K + j] += p[k] * p[j];
      }
    };
    const int64_t r0 = ch * HK_CHUNK + threadIdx.x;
    if (ch * HK_CHUNK + HK_CHUNK <= n) {  // full chunk: every row's load in flight first
      double xv[kRowsPerThread];
#pragma unroll
      for (int i = 0; i < kRowsPerThread; ++i) xv[i] = __ldg(x + r0 + i * kBlock);
#pragma unroll
      for (int i = 0; i < kRowsPerThread; ++i) row(xv[i], r0 + i * kBlock);
    } else {
#pragma unroll 1
      for (int i = 0; i < kRowsPerThread; ++i) {
        const int64_t r = r0 + i * kBlock;
        if (r < n) row(__ldg(x + r), r);
      }
    }
    block_sum_store<W>(acc, part + (int64_t)W * ch);
  }
}

// ---------------------------------------------------- multi-point FCN -----
// K parameter points of the factored Gaussian + exponential model in one
// pass over the data (hk_nll_eval_many): CTA (tile t, group g) evaluates the
// tile for points 4g .. 4g+3 from one register copy of its 16 rows per
// thread, so a Hessian's 51 points (fitting.py:365-386) read the column once
// per group instead of once per call, and the grid is tiles x groups CTAs
// (many waves: no ramp/tail per point).  Per point the arithmetic, the tile
// partials and the fold are those of k_nll_fused (same templates, same
// order), so each value is bit-identical to a single-point hk_nll_eval.
#ifndef HK_FCN_MANY_G
#define HK_FCN_MANY_G 2
#endif
constexpr int kManyG = HK_FCN_MANY_G;
// 3 CTAs/SM (80 registers): the 16 register-resident rows live across the
// four points' passes; at 64 registers they spill
#ifndef HK_FCN_MANY_MIN_BLOCKS
#define HK_FCN_MANY_MIN_BLOCKS 4
#endif

struct ManyArgs {
  const double* x;
  int64_t n;
  int32_t k, groups;
  int64_t tiles, kpad;
  double* part;                  // [tile][kpad]
  double* out;                   // [k] sums
  unsigned long long* bad;       // [k] ~first bad row, 0 = none
  unsigned int* gticket;         // [groups] tiles finished per group
  unsigned int* done;            // groups folded
  volatile unsigned long long* host_mail;
  unsigned long long seq;
  int32_t rev;                   // the first group's scan direction (flipped per call)
  FPoint pt[HK_MAX_POINTS];  // k points, padded with copies of the last to kpad
};

template <int V>
__global__ void __launch_bounds__(kBlock, HK_FCN_MANY_MIN_BLOCKS) k_nll_many(const __grid_constant__ ManyArgs a) {
  __shared__ unsigned int s_t;
  __shared__ double tot[kManyG];
  const int64_t total = a.tiles * a.groups;
  for (int64_t b = blockIdx.x; b < total; b += gridDim.x) {
    const int g = (int)(b / a.tiles);
    // serpentine: group g walks the tiles in the direction opposite to group
    // g - 1 (and to the previous call's last group), so each group's pass
    // starts on the L2-resident end of the column
    const int64_t t = ((g & 1) ^ a.rev) ? a.tiles - 1 - b % a.tiles : b % a.tiles;
    const int64_t begin = t * kFcnTile;
    const int64_t end = begin + kFcnTile < a.n ? begin + kFcnTile : a.n;
    const int64_t r0 = begin + threadIdx.x;
    const bool full = end - begin == kFcnTile;
    // the group's four points advance together, row by row: four independent
    // LogProd / exponent-sum chains per thread (ILP 4); per point the row
    // order -- and so every rounding -- is that of range_logsum
    LogProd lp[kManyG];
    double msum[kManyG];
    unsigned long long bad[kManyG];
#pragma unroll
    for (int j = 0; j < kManyG; ++j) {
      msum[j] = 0.0;
      bad[j] = 0;
    }
    const FPoint* c = a.pt + g * kManyG;  // padded to kpad points on the host
    if constexpr (V == kFcnFast) {
      // per point exactly range_logsum<kFcnFast>'s chain: same values
      double prod[kManyG];
#pragma unroll
      for (int j = 0; j < kManyG; ++j) prod[j] = 1.0;
      if (full) {
        double xv[kFcnRows];
#pragma unroll
        for (int i = 0; i < kFcnRows; ++i) xv[i] = __ldg(a.x + r0 + i * kBlock);
#pragma unroll
        for (int i = 0; i < kFcnRows; ++i) {
#pragma unroll
          for (int j = 0; j < kManyG; ++j) fast_row(c[j], xv[i], prod[j]);
        }
      } else {
        for (int i = 0; i < kFcnRows; ++i) {
          const int64_t r = r0 + i * kBlock;
          if (r >= end) continue;
          const double xr = __ldg(a.x + r);
#pragma unroll
          for (int j = 0; j < kManyG; ++j) fast_row(c[j], xr, prod[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < kManyG; ++j) msum[j] = log(prod[j]);
    } else if (full) {
      double xv[kFcnRows];
#pragma unroll
      for (int i = 0; i < kFcnRows; ++i) xv[i] = __ldg(a.x + r0 + i * kBlock);
#pragma unroll
      for (int i = 0; i < kFcnRows; ++i) {
#pragma unroll
        for (int j = 0; j < kManyG; ++j)
          fcn_row<kFcnFactored>(c[j], xv[i], r0 + i * kBlock, lp[j], msum[j], &bad[j]);
      }
    } else {
      for (int i = 0; i < kFcnRows; ++i) {  // the ragged last tile, as range_logsum
        const int64_t r = r0 + i * kBlock;
        if (r >= end) continue;
        const double xr = __ldg(a.x + r);
#pragma unroll
        for (int j = 0; j < kManyG; ++j) fcn_row<kFcnFactored>(c[j], xr, r, lp[j], msum[j], &bad[j]);
      }
    }
    double acc[kManyG];
#pragma unroll
    for (int j = 0; j < kManyG; ++j) {
      acc[j] = V == kFcnFast ? msum[j] : lp[j].value() + msum[j];
      if (bad[j] && g * kManyG + j < a.k) atomicMax(a.bad + g * kManyG + j, bad[j]);
    }
    block_sum_store<kManyG>(acc, a.part + t * a.kpad + g * kManyG);
    if (threadIdx.x == 0) {
      __threadfence();
      s_t = atomicAdd(a.gticket + g, 1u);
    }
    __syncthreads();
    if (s_t != a.tiles - 1) continue;
    // last tile of group g: fold its points in k_nll_fused's order, publish
    __threadfence();
    double f[kManyG];
#pragma unroll
    for (int j = 0; j < kManyG; ++j) f[j] = 0.0;
    for (int64_t i = threadIdx.x; i < a.tiles; i += kBlock) {
#pragma unroll
      for (int j = 0; j < kManyG; ++j) f[j] += __ldcg(a.part + i * a.kpad + g * kManyG + j);
    }
    block_sum_store<kManyG>(f, tot);
    if (threadIdx.x == 0) {
      for (int j = 0; j < kManyG; ++j) {
        const int p = g * kManyG + j;
        if (p >= a.k) break;
        const unsigned long long bb = atomicExch(a.bad + p, 0ull);
        const double v = tot[j] + (V == kFcnFast ? c[j].base : 0.0);  // fcn_finish's order
        a.out[p] = v;
        if (a.host_mail) {
          a.host_mail[1 + p] = (unsigned long long)__double_as_longlong(v);
          a.host_mail[1 + a.k + p] = ~bb;
        }
      }
      a.gticket[g] = 0u;
      __threadfence_system();
      if (atomicAdd(a.done, 1u) == (unsigned)a.groups - 1) {
        *a.done = 0u;
        __threadfence_system();
        if (a.host_mail) a.host_mail[0] = a.seq;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------ resident FCN session ----
// A minimiser calls the FCN serially (fitting.py:251-340), so each call pays
// a kernel launch plus the launch's ramp (measured on B200: 10.4 us launch +
// mapped-memory signal round trip, tools/launch_latency.cu) on top of the
// ~25 us of arithmetic.  A session keeps one persistent CTA per slot
// (SMs x 4, co-resident by cooperative launch) waiting on a command word in
// mapped host memory: the host writes the parameter point and a sequence
// number; CTA 0 sees it (one PCIe read, ~3.4 us round trip in total),
// publishes it in device memory, every CTA runs the same tiles as
// k_nll_fused (same arithmetic, same partials, same last-CTA fold -- values
// bit-identical to hk_nll_eval) and the last CTA answers through the mailbox.
// The CTAs leave when told to, or after an idle timeout (the host relaunches
// on the next call), so a forgotten session cannot hold the GPU.
// Command page in mapped host memory: kCmdSlots 16-byte slots {seq, word},
// each written by the host with one aligned 16-byte store (atomic on x86
// with AVX), read by lanes 0..10 of CTA 0's first warp with one 16-byte load
// each -- 17 concurrent PCIe reads per poll, and a command is taken only when
// every slot carries the same new seq, so no ordering between the reads is
// needed.  Words: 0 = variant | stop << 8, 1..16 = the FPoint.
constexpr int kCmdSlots = 1 + (int)(sizeof(FPoint) / sizeof(double));  // 17: word 0 + the FPoint
static_assert(kCmdSlots <= 32, "one lane per command slot");
struct alignas(16) CmdSlot {
  unsigned long long seq;
  unsigned long long word;
};
struct ServerCmd {
  CmdSlot slot[kCmdSlots];
};

struct ServerDev {          // device memory
  unsigned long long gen;   // current command seq; ~0 = leave
  unsigned long long done;  // last seq answered
  unsigned long long next;  // dynamic tile counter of the current command
  long long t_seen;         // globaltimer when CTA 0 took the command (diagnostics)
  int32_t variant, _pad;
  FPoint c;
};

struct ServerArgs {
  const double* x;
  int64_t n;
  FcnWork w;                // out/bad/ticket/part of the session workspace; host_mail
  const ServerCmd* cmd;     // device view of the mapped command page
  ServerDev* dev;
  long long idle_ns;
};

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void ld_slot_sys(const CmdSlot* p, unsigned long long* seq, unsigned long long* word) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(*seq), "=l"(*word) : "l"(p) : "memory");
}
__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// CTA 0, warp 0: wait for a complete new command (or the idle timeout), copy
// it to device memory and release it to every CTA through dev->gen.
__device__ __forceinline__ void server_poll(const ServerArgs& a, unsigned long long mine) {
  const int lane = threadIdx.x & 31;
  const long long t0 = global_ns();
  unsigned long long s = 0, word = 0;
  for (;;) {
    if (lane < kCmdSlots) ld_slot_sys(&a.cmd->slot[lane], &s, &word);
    const unsigned long long s0 = __shfl_sync(0xffffffffu, s, 0);
    const bool same = __all_sync(0xffffffffu, lane >= kCmdSlots || s == s0);
    if (same && s0 != mine) {
      s = s0;
      break;
    }
    if (global_ns() - t0 > a.idle_ns) {
      s = ~0ull;
      break;
    }
  }
  const unsigned long long w0 = __shfl_sync(0xffffffffu, word, 0);
  if (s != ~0ull && (w0 >> 8)) s = ~0ull;  // stop
  if (s != ~0ull && lane >= 1 && lane < kCmdSlots) {
    double* c = &a.dev->c.amp[0];           // FPoint: kCmdSlots - 1 consecutive doubles
    c[lane - 1] = __longlong_as_double((long long)word);
  }
  if (lane == 0) {
    if (s != ~0ull) {
      a.dev->variant = (int32_t)(w0 & 0xff);
      a.dev->next = 0ull;
      a.dev->t_seen = global_ns();
    } else {
      a.w.host_mail[6] = 1ull;  // left (idle timeout or stop): the host relaunches before the next command
    }
    __threadfence();
  }
  __syncwarp();
  if (lane == 0) st_release_gpu(&a.dev->gen, s);
}

template <int V>
__device__ __forceinline__ void server_tile(const ServerArgs& a, const FPoint& c, int64_t ch) {
  unsigned long long bad = 0;
  int64_t begin, end;
  fcn_range(a.w, a.n, ch, &begin, &end);
  double acc[1] = {range_logsum<V>(a.x, begin, end, c, &bad, threadIdx.x)};
  if (bad) atomicMax(a.w.bad, bad);
  block_sum_store<1>(acc, a.w.part + ch);
}

template <int V>
__device__ __forceinline__ void server_tiles(const ServerArgs& a, const FPoint& c, int64_t chunks) {
  // dynamic tiles (like a launch's block scheduler): the 74 tiles past
  // 4 x 592 of a 1e7-event set go to the CTAs that finish first (static
  // rounds measured slower); tile ch's partial is the same value whichever
  // CTA computes it.  The next index is fetched while the current tile
  // computes, so the atomic's latency hides.
  __shared__ long long s_tile;
  if (threadIdx.x == 0) s_tile = (long long)atomicAdd(&a.dev->next, 1ull);
  __syncthreads();
  int64_t ch = s_tile;
  while (ch < chunks) {
    __syncthreads();  // every thread has read s_tile
    unsigned long long nxt = 0;
    if (threadIdx.x == 0) nxt = atomicAdd(&a.dev->next, 1ull);
    server_tile<V>(a, c, fcn_tile(a.w, ch, chunks));  // in the pass's scan direction (fcn_flip)
    if (threadIdx.x == 0) s_tile = (long long)nxt;
    __syncthreads();
    ch = s_tile;
  }
}

#ifndef HK_FCN_SERVER_MIN_BLOCKS
#define HK_FCN_SERVER_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kBlock, HK_FCN_SERVER_MIN_BLOCKS) k_fcn_server(const __grid_constant__ ServerArgs a) {
  __shared__ unsigned long long s_gen;
  __shared__ FPoint s_c;
  __shared__ int s_variant;
  unsigned long long mine = a.dev->done;
  const int64_t chunks = a.w.full + a.w.tail_ctas;
  for (;;) {
    if (blockIdx.x == 0 && threadIdx.x < 32) server_poll(a, mine);
    if (threadIdx.x == 0) {
      // waiters back off: a spinning warp would take issue slots from the
      // CTAs still computing on the same SM
      unsigned long long g;
      while ((g = ld_acquire_gpu(&a.dev->gen)) == mine) __nanosleep(32);
      s_gen = g;
      if (g != ~0ull) {
        s_variant = a.dev->variant;
        s_c = a.dev->c;
      }
    }
    __syncthreads();
    const unsigned long long g = s_gen;
    if (g == ~0ull) return;
    mine = g;
    // the coefficients stay in shared memory (operands are LDS'd where the
    // arithmetic needs them): a register copy costs 14 of the 64 registers
    if (s_variant == kFcnFast)
      server_tiles<kFcnFast>(a, s_c, chunks);
    else if (s_variant == kFcnFactored)
      server_tiles<kFcnFactored>(a, s_c, chunks);
    else
      server_tiles<kFcnGE>(a, s_c, chunks);
    // fcn_finish with this command's sequence number
    __shared__ unsigned int s_ticket;
    if (threadIdx.x == 0) {
      __threadfence();
      s_ticket = atomicAdd(a.w.ticket, 1u);
    }
    __syncthreads();
    if (s_ticket == gridDim.x - 1) {
      __threadfence();
      double acc[1] = {0.0};
      for (int64_t i = threadIdx.x; i < chunks; i += kBlock) acc[0] += __ldcg(a.w.part + i);
      __shared__ double total;
      block_sum_store<1>(acc, &total);
      if (threadIdx.x == 0) {
        a.dev->done = g;
        a.w.host_mail[4] = (unsigned long long)a.dev->t_seen;  // device-side span of the command
        a.w.host_mail[5] = (unsigned long long)global_ns();
        FcnWork w = a.w;
        w.seq = g;
        fcn_publish(w, total + (s_variant == kFcnFast ? s_c.base : 0.0));  // fcn_finish's order
      }
    }
    __syncthreads();
  }
}

struct Session {
  int device = -1;
  cudaStream_t stream = nullptr;
  ServerCmd* h_cmd = nullptr;       // mapped
  ServerCmd* d_cmd = nullptr;
  ServerDev* dev = nullptr;
  ServerArgs args{};
  unsigned grid = 0;
  bool running = false;
  bool active = false;  // between hk_fcn_session_start and _stop
  unsigned long long seq = 0;
};
thread_local Session t_session;

// one aligned 16-byte store per slot (SSE2 movdqa: atomic on AVX-capable
// x86 hosts), so the device never sees a slot's seq without its word
void write_slots(ServerCmd* h, const CmdSlot* v) {
  std::atomic_thread_fence(std::memory_order_release);
  for (int k = 0; k < kCmdSlots; ++k) {
#if defined(__SSE2__)
    _mm_store_si128(reinterpret_cast<__m128i*>(&h->slot[k]),
                    _mm_set_epi64x((long long)v[k].word, (long long)v[k].seq));
#else
    __atomic_store(reinterpret_cast<__int128*>(&h->slot[k]), reinterpret_cast<const __int128*>(&v[k]),
                   __ATOMIC_RELEASE);
#endif
  }
  std::atomic_thread_fence(std::memory_order_seq_cst);
}

int session_launch(Session& S) {
  // the next command must be seen as new: gen = done = last answered seq
  ServerDev init{};
  init.gen = init.done = S.seq;
  HK_CUDA(cudaMemcpyAsync(S.dev, &init, sizeof(init), cudaMemcpyHostToDevice, S.stream));
  void* params[] = {&S.args};
  HK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_fcn_server), dim3(S.grid), dim3(kBlock),
                                      params, 0, S.stream));
  S.running = true;
  return HK_OK;
}

// Stop the session's CTAs (if any are running).  The stream, the mapped
// command page and the device control block stay allocated for the next
// session on this thread and device -- cudaHostAlloc / cudaFreeHost cost tens
// of ms and synchronise the device, more than a whole C4 fit's FCN work --
// unless `release` (device change, library shutdown).
int session_stop(Session& S, bool release = false) {
  if (S.device < 0) return HK_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(S.device);
  cudaError_t e = cudaSuccess;
  if (S.running) {
    if (cudaStreamQuery(S.stream) == cudaErrorNotReady) {
      CmdSlot v[kCmdSlots];
      const unsigned long long seq = S.seq + 0x100000000ull;  // any seq the server has not answered
      for (int k = 0; k < kCmdSlots; ++k) {
        v[k].seq = seq;
        v[k].word = k == 0 ? (1ull << 8) : 0ull;
      }
      write_slots(S.h_cmd, v);
    }
    e = cudaStreamSynchronize(S.stream);
    S.running = false;
  }
  S.active = false;
  if (release) {
    cudaStreamDestroy(S.stream);
    cudaFreeHost(S.h_cmd);
    cudaFree(S.dev);
    S = Session{};
  }
  cudaSetDevice(cur);
  if (e != cudaSuccess) return cuda_fail(e, "hk_fcn_session_stop");
  return HK_OK;
}

// kFcnFast admission (see fast_row): the column statistics of hk_model_t
// bound, for every x in [x_min, x_max],
//   A(x) = -((x - mean) / sigma)^2 / 2 (concave), B(x) = b x (b = -1/tau),
//   M(x) = max(A, B) in [min(B(x_min), B(x_max)), max(A(clamp(mean)), B(x_min), B(x_max))],
// and that interval must sit inside kFcnFactored's window (m_lo, m_hi) with a
// margin of 1: then both reference terms are finite normal doubles and the
// density is positive for every event -- exactly the events kFcnFactored
// takes without its fallback, so no per-event check is needed.  Also the
// amplitude ratio must be >= 1e-15 (16-factor products of s' stay normal),
// the rounding of the quadratic q over the range <= 1e-11 (log2 units), and
// -999 <= q <= 59 (fcn_exp2's domain, and s' <= 1 + 2^59).  A model whose
// Gaussian term outgrows the exponential one by more than 2^59 somewhere in
// the range takes kFcnFactored instead.
void fast_coeffs(const hk_model_t* m, int64_t n, Coeffs* c) {
  c->fast = 0;
  if (n <= 0 || !m->has_stats || m->x_count != n) return;
  if (!(c->m_lo < c->m_hi) || c->kind[0] != HK_SHAPE_GAUSS || c->kind[1] != HK_SHAPE_EXPO) return;
  const double xmin = m->x_min, xmax = m->x_max;
  if (!std::isfinite(xmin) || !std::isfinite(xmax) || !(xmin <= xmax) || !std::isfinite(m->x_sum)) return;
  const double mu = c->shift[0], is = c->scale[0], b = c->scale[1];
  const double amax = std::fmax(c->amp[0], c->amp[1]), amin = std::fmin(c->amp[0], c->amp[1]);
  if (!(amin >= 1e-15 * amax)) return;
  const double b_lo = std::fmin(b * xmin, b * xmax), b_hi = std::fmax(b * xmin, b * xmax);
  const double xc = std::fmin(std::fmax(mu, xmin), xmax);
  const double zc = (xc - mu) * is;
  const double a_hi = -0.5 * zc * zc;
  const double m_lo = b_lo, m_hi = std::fmax(a_hi, b_hi);
  if (!(m_lo > c->m_lo + 1.0) || !(m_hi < c->m_hi - 1.0)) return;
  // q(x) = log2(e) (A - B) = a2 x^2 + a1 x + a0 (from q2 u^2 + q1 u + q0, u = x - mean)
  const double log2e = 1.4426950408889634;
  const double a2 = log2e * c->q2;
  const double a1 = log2e * (c->q1 - 2.0 * c->q2 * mu);
  const double a0 = log2e * ((c->q2 * mu - c->q1) * mu + c->q0);
  const double xa = std::fmax(std::fabs(xmin), std::fabs(xmax));
  const double err = 16.0 * 1.1102230246251565e-16 *
                     (std::fabs(a2) * xa * xa + std::fabs(a1) * xa + std::fabs(a0) + 1.0);
  if (!(err <= 1e-11)) return;
  // -999 <= q <= 59 over the range (fcn_exp2's domain): q is concave, so its
  // extremes are at the ends or the vertex
  const double q_lo = std::fmin(a2 * xmin * xmin + a1 * xmin + a0, a2 * xmax * xmax + a1 * xmax + a0);
  const double xv = std::fmin(std::fmax(-a1 / (2.0 * a2), xmin), xmax);
  const double q_hi = std::fmax(a2 * xv * xv + a1 * xv + a0, std::fmax(a2 * xmin * xmin + a1 * xmin + a0,
                                                                      a2 * xmax * xmax + a1 * xmax + a0));
  if (!(q_lo >= -999.0) || !(q_hi <= 59.0)) return;
  c->fq[0] = a2;
  c->fq[1] = a1;
  c->fq[2] = a0;
  c->fa[0] = c->amp[0] / amax;
  c->fa[1] = c->amp[1] / amax;
  c->base = b * m->x_sum + (double)n * std::log(amax);
  c->fast = 1;
}

int make_coeffs(const hk_model_t* m, Coeffs* c, int64_t n = -1) {
  HK_REQUIRE(m != nullptr, "NULL model");
  HK_REQUIRE(m->n_comp >= 1 && m->n_comp <= HK_MAX_COMPONENTS, "component count %d outside 1..%d",
             m->n_comp, HK_MAX_COMPONENTS);
  std::memset(c, 0, sizeof(*c));
  c->n_comp = m->n_comp;
  const double sqrt2pi = 2.5066282746310002;  // functors.py:26
  for (int k = 0; k < m->n_comp; ++k) {
    c->kind[k] = m->kind[k];
    if (m->kind[k] == HK_SHAPE_GAUSS) {
      HK_REQUIRE(m->p1[k] > 0, "component %d: sigma must be positive, got %g", k, m->p1[k]);
      c->amp[k] = m->yield[k] / (m->p1[k] * sqrt2pi * m->norm[k]);
      c->shift[k] = m->p0[k];
      c->scale[k] = 1.0 / m->p1[k];
    } else if (m->kind[k] == HK_SHAPE_EXPO) {
      HK_REQUIRE(m->p0[k] != 0, "component %d: tau must be non-zero", k);
      c->amp[k] = m->yield[k] / m->norm[k];
      c->scale[k] = -1.0 / m->p0[k];
    } else {
      set_error("component %d: unknown shape kind %d", k, m->kind[k]);
      return HK_EUNSUPPORTED;
    }
  }
  // factored-path window: amp_k e^M in [~1e-300, ~1e304] for both k
  c->m_lo = 0.0;
  c->m_hi = -1.0;  // empty: variant kFcnFactored not applicable
  if (m->n_comp == 2 && c->amp[0] > 1e-250 && c->amp[1] > 1e-250 && c->amp[0] < 1e300 &&
      c->amp[1] < 1e300 && std::fmax(c->amp[0], c->amp[1]) < 1e200 * std::fmin(c->amp[0], c->amp[1])) {
    c->m_lo = -690.0 - std::log(std::fmin(c->amp[0], c->amp[1]));
    c->m_hi = 700.0 - std::log(c->amp[0] + c->amp[1]);
  }
  if (m->n_comp == 2 && m->kind[0] == HK_SHAPE_GAUSS && m->kind[1] == HK_SHAPE_EXPO) {
    c->q2 = -0.5 * c->scale[0] * c->scale[0];
    c->q1 = -c->scale[1];
    c->q0 = -c->shift[0] * c->scale[1];
    fast_coeffs(m, n, c);
  }
  return HK_OK;
}

// allow_fast: the caller folds with fcn_finish's base (not hk_nll_partials)
int fcn_variant(const Coeffs& c, bool allow_fast = true) {
  const bool ge = c.n_comp == 2 && c.kind[0] == HK_SHAPE_GAUSS && c.kind[1] == HK_SHAPE_EXPO;
  if (!ge) return kFcnGeneric;
  if (allow_fast && c.fast) return kFcnFast;
  return c.m_lo < c.m_hi ? kFcnFactored : kFcnGE;
}

int launch_nll(const double* d_x, int64_t n, const Coeffs& c, double* part,
               unsigned long long* bad, cudaStream_t st) {
  const unsigned grid = chunk_grid((n + kFcnTile - 1) / kFcnTile);
  switch (fcn_variant(c, false)) {
    case kFcnFactored: k_nll<kFcnFactored><<<grid, kBlock, 0, st>>>(d_x, n, c, part, bad); break;
    case kFcnGE: k_nll<kFcnGE><<<grid, kBlock, 0, st>>>(d_x, n, c, part, bad); break;
    default: k_nll<kFcnGeneric><<<grid, kBlock, 0, st>>>(d_x, n, c, part, bad); break;
  }
  return check_launch("k_nll");
}

// pdf_k coefficients (no yields in amp) for the yield / sPlot kernels
int make_pdf_coeffs(const hk_model_t* model, PdfCoeffs* c) {
  std::memset(c, 0, sizeof(*c));
  const double sqrt2pi = 2.5066282746310002;
  for (int k = 0; k < model->n_comp; ++k) {
    c->kind[k] = model->kind[k];
    c->yield[k] = model->yield[k];
    if (model->kind[k] == HK_SHAPE_GAUSS) {
      HK_REQUIRE(model->p1[k] > 0, "component %d: sigma must be positive", k);
      c->amp[k] = 1.0 / (model->p1[k] * sqrt2pi * model->norm[k]);
      c->shift[k] = model->p0[k];
      c->scale[k] = 1.0 / model->p1[k];
    } else if (model->kind[k] == HK_SHAPE_EXPO) {
      HK_REQUIRE(model->p0[k] != 0, "component %d: tau must be non-zero", k);
      c->amp[k] = 1.0 / model->norm[k];
      c->scale[k] = -1.0 / model->p0[k];
    } else {
      set_error("component %d: unknown shape kind %d", k, model->kind[k]);
      return HK_EUNSUPPORTED;
    }
  }
  return HK_OK;
}

// sWeights (splot.py:90-117): sw_n(e) = sum_j V_nj pdf_j(x_e) / density(x_e)
struct SplotArgs {
  PdfCoeffs c;
  int32_t k;
  double V[16];
  double* out[4];
  unsigned long long* bad;  // density <= 0 or non-finite (splot.py:35-42)
};

__global__ void __launch_bounds__(kBlock) k_splot(const double* __restrict__ x, int64_t n,
                                                  const __grid_constant__ SplotArgs a) {
  const int64_t r = blockIdx.x * (int64_t)kBlock + threadIdx.x;
  if (r >= n) return;
  const double xv = __ldg(x + r);
  double p[4] = {0.0, 0.0, 0.0, 0.0};
  double d = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < a.k) {
      if (a.c.kind[k] == HK_SHAPE_GAUSS) {
        const double z = (xv - a.c.shift[k]) * a.c.scale[k];
        p[k] = a.c.amp[k] * exp(-0.5 * z * z);
      } else {
        p[k] = a.c.amp[k] * exp(xv * a.c.scale[k]);
      }
      d += p[k] * a.c.yield[k];
    }
  }
  if (!(d > 0.0) || !isfinite(d)) record_bad(a.bad, (uint64_t)r);
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (s < a.k) {
      double num = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < a.k) num += p[j] * a.V[s * a.k + j];
      a.out[s][r] = num / d;
    }
  }
}

// Mapped pinned mailbox per (host thread, device) for the FCN entry points:
// [0] sequence number, then the payload -- [1] sum-of-logs bits, [2] first
// bad row, [3] first zero divisor for one point; [1..k] sums and [k+1..2k]
// first bad rows for the k points of hk_nll_eval_many.
constexpr int kMailWords = 1 + 2 * HK_MAX_POINTS;
struct Mailbox {
  volatile unsigned long long* h = nullptr;  // host view
  unsigned long long* d = nullptr;           // device view of the same memory
  unsigned long long seq = 0;
  int device = -1;
};

thread_local Mailbox t_boxes[16];

int mailbox(Mailbox** out) {
  int dev = 0;
  HK_CUDA(cudaGetDevice(&dev));
  Mailbox& m = t_boxes[dev & 15];
  if (m.device != dev) {
    void* p = nullptr;
    HK_CUDA(cudaHostAlloc(&p, kMailWords * sizeof(unsigned long long), cudaHostAllocMapped));
    std::memset(p, 0, kMailWords * sizeof(unsigned long long));
    void* dp = nullptr;
    HK_CUDA(cudaHostGetDevicePointer(&dp, p, 0));
    m.h = static_cast<volatile unsigned long long*>(p);
    m.d = static_cast<unsigned long long*>(dp);
    m.seq = 0;
    m.device = dev;
  }
  *out = &m;
  return HK_OK;
}

// hk_shutdown: free this thread's mailboxes (rebuilt by the next hk_nll_eval)
void fcn_release() {
  session_stop(t_session, true);
  for (Mailbox& m : t_boxes) {
    if (m.device < 0) continue;
    cudaFreeHost(const_cast<unsigned long long*>(m.h));
    m = Mailbox{};
  }
}

// Tile schedule of the one-launch FCN: plain 4096-row tiles.  The spread-tail
// variant (kFcnSpreadTail: whole waves of S = SMs x 4 tiles, then the leftover
// rows split over one wave of short CTAs, 4 x 592 + 592 CTAs for 1e7 events
// instead of 2442 tiles) measured slower on B200 -- C-ABI call 44.6 vs 40.8 us:
// a wave of short CTAs costs about the same latency as the 74-tile tail it
// replaces.  Kept behind the switch for the record.
constexpr bool kFcnSpreadTail = false;

void fcn_schedule(int64_t n, int64_t* full, int64_t* tail_ctas) {
  static int slots = 0;
  if (!slots) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    slots = (sms > 0 ? sms : 148) * HK_FCN_MIN_BLOCKS;
  }
  const int64_t tiles = (n + kFcnTile - 1) / kFcnTile;
  if (!kFcnSpreadTail || tiles <= slots) {  // plain tiles
    *full = n / kFcnTile;
    *tail_ctas = n % kFcnTile ? 1 : 0;
    return;
  }
  *full = (n / kFcnTile / slots) * slots;  // whole waves of whole tiles
  const int64_t rem = n - *full * kFcnTile;
  const int64_t want = (rem + kBlock - 1) / kBlock;
  *tail_ctas = rem == 0 ? 0 : (want < slots ? want : slots);
}

// d_work layout of the one-launch FCN (zero-filled once by the caller,
// re-armed by the kernel): [0] sum of logs, [1] first bad row (u64 bits),
// [2] ~bad-row cell, [3] CTA ticket, [4] ~zero-divisor cell, [5] first zero
// divisor row (u64 bits), [6..7] caller's (hk_nll_combine: [6] = the shard's
// first global row), [8] tile counter (k_nll_fast_tma), [16..] partials.
constexpr int kFcnWorkHead = 16;  // [8] the persistent FCN's tile counter, [9..15] spare

// Scan direction of the next pass over a column of `bytes` behind workspace
// `key` -- a hint only: tile partials keep their index, so values never
// depend on it.  Measured on B200 (profiles/r02_fcn_rev_ab.jsonl, steady
// state, ncu --cache-control none): walking the tiles last to first on
// every call keeps ~35% of an 80 MB column's sectors in L2 (forward: 8%),
// 1e7 events 20.3 -> 18.6 us, 1.3e7 26.9 -> 26.6; for columns past ~0.85 of
// L2 a fixed reverse scan loses (1.5e7: 31.7 vs 28.5 us,
// profiles/r02_fcn_rev_thr.jsonl) and alternating the direction per call
// wins instead.  HK_FCN_REV_MAX_BYTES overrides the threshold.
#ifndef HK_FCN_FLIP
#define HK_FCN_FLIP 1
#endif
int32_t fcn_flip(const void* key, int64_t bytes, int passes = 1) {
  if (!HK_FCN_FLIP) return 0;
  static int64_t rev_max = -1;
  if (rev_max < 0) {
    const char* env = std::getenv("HK_FCN_REV_MAX_BYTES");
    int dev = 0, l2 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    rev_max = env ? std::atoll(env) : (int64_t)(0.85 * (l2 > 0 ? l2 : 0));
  }
  if (bytes <= rev_max) return 1;
  static std::mutex mu;
  static std::unordered_map<const void*, int32_t> dir;
  std::lock_guard<std::mutex> lock(mu);
  if (dir.size() > 4096) dir.clear();
  int32_t& d = dir[key];
  const int32_t cur = d;
  d ^= passes & 1;
  return cur;
}

// mb == NULL: asynchronous call, the result stays in d_work[0, 1, 5]
int fcn_setup(double* d_work, int64_t n, FcnWork* w, Mailbox** mb) {
  w->out = d_work;
  w->bad = reinterpret_cast<unsigned long long*>(d_work + 2);
  w->ticket = reinterpret_cast<unsigned int*>(d_work + 3);
  w->div0 = reinterpret_cast<unsigned long long*>(d_work + 4);
  w->part = d_work + kFcnWorkHead;
  w->next = reinterpret_cast<unsigned long long*>(d_work + 8);
  w->host_mail = nullptr;
  w->seq = 0;
  if (mb) {
    if (int rc = mailbox(mb)) return rc;
    w->host_mail = (*mb)->d;
    w->seq = ++(*mb)->seq;
  }
  fcn_schedule(n, &w->full, &w->tail_ctas);
  w->rev = fcn_flip(d_work, n * (int64_t)sizeof(double));
  return HK_OK;
}

// Rank-order fold of gathered FCN results (hk_nll_combine): one thread.
__global__ void k_nll_combine(const double* g, int world, FcnWork w) {
  if (threadIdx.x != 0) return;
  double total = 0.0;
  unsigned long long bad = ~0ull, zero = ~0ull;
  for (int r = 0; r < world; ++r) {
    const double* v = g + 8 * r;
    total += v[0];
    const unsigned long long off = (unsigned long long)v[6];
    const unsigned long long b = (unsigned long long)__double_as_longlong(v[1]);
    const unsigned long long z = (unsigned long long)__double_as_longlong(v[5]);
    if (b != ~0ull && off + b < bad) bad = off + b;
    if (z != ~0ull && off + z < zero) zero = off + z;
  }
  w.host_mail[1] = (unsigned long long)__double_as_longlong(total);
  w.host_mail[2] = bad;
  w.host_mail[3] = zero;
  __threadfence_system();
  w.host_mail[0] = w.seq;
}

// The last CTA writes the result into mapped host memory and then the
// sequence number; spin on it (no memcpy, no stream sync on the fast path).
// Every 4096 polls the stream is queried so a faulted kernel cannot hang us.
int fcn_wait(Mailbox* mb, unsigned long long seq, cudaStream_t st, const char* what,
             double* h_logsum, uint64_t* h_first_bad, uint64_t* h_first_div0) {
  for (unsigned spins = 1;; ++spins) {
    if (mb->h[0] == seq) break;
    if ((spins & 4095u) == 0) {
      const cudaError_t q = cudaStreamQuery(st);
      if (q == cudaSuccess) {
        if (mb->h[0] == seq) break;
        set_error("%s: kernel finished without publishing its result", what);
        return HK_ECUDA;
      }
      if (q != cudaErrorNotReady) return cuda_fail(q, what);
    }
  }
  // the device fenced (system scope) before writing seq; order our reads
  // of the payload after the seq read (weakly ordered hosts, e.g. Grace)
  std::atomic_thread_fence(std::memory_order_acquire);
  const unsigned long long sum_bits = mb->h[1];
  std::memcpy(h_logsum, &sum_bits, sizeof(double));
  *h_first_bad = mb->h[2];
  if (h_first_div0) *h_first_div0 = mb->h[3];
  return HK_OK;
}

// ------------------------------------------------ program-driven models ---
// The density of any lowered model (hk_density_t) through the interpreter;
// hk_jit.cu specialises the same pass per op structure.
__global__ void __launch_bounds__(kBlock) k_nll_program(const __grid_constant__ FcnProgArgs a) {
  const auto dens = [&](int64_t r, bool& z) -> double {
    return run_program(a.prog, [&](int c) { return __ldg(a.cols[c] + r); }, &z);
  };
  fcn_density_pass(a.w, a.n, dens);
}

int validate_density(const hk_density_t* m) {
  HK_REQUIRE(m != nullptr, "NULL model");
  HK_REQUIRE(m->n_obs >= 1 && m->n_obs <= HK_FCN_MAX_OBS, "observable count %d outside 1..%d",
             m->n_obs, HK_FCN_MAX_OBS);
  HK_REQUIRE(m->n_comp >= 1 && m->n_comp <= HK_MAX_COMPONENTS, "component count %d outside 1..%d",
             m->n_comp, HK_MAX_COMPONENTS);
  if (int rc = validate_program(&m->program, m->n_obs)) return rc;
  for (int k = 0; k < m->n_comp; ++k)
    HK_REQUIRE(m->pdf_slot[k] >= 0 && m->pdf_slot[k] < HK_MAX_SLOTS, "pdf slot %d", m->pdf_slot[k]);
  return HK_OK;
}

struct RatioArgs {
  const double* cols[HK_FCN_MAX_OBS];
  int64_t n;
  hk_density_t m;
  double* part;
  unsigned long long* bad;  // [0] d not > 0, [1] d not > 0 or non-finite, [2] zero divisor
  const double* V;          // sPlot: K x K (device copy in the args below)
};

// per event: p_k (pinned program slots) and d = sum_k N_k p_k (p @ N,
// fitting.py:416 / splot.py:37); flags as documented in the header
template <int K>
__device__ __forceinline__ double ratio_event(const RatioArgs& a, int64_t r, double (&p)[K]) {
  double slots[HK_MAX_SLOTS];
  bool z = false;
  run_program_into(a.m.program, [&](int c) { return __ldg(a.cols[c] + r); }, &z, slots);
  double d = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    p[k] = slots[a.m.pdf_slot[k]];
    d = k == 0 ? p[k] * a.m.yield[k] : d + p[k] * a.m.yield[k];
  }
  if (z) record_bad(a.bad + 2, (uint64_t)r);
  if (!(d > 0.0)) record_bad(a.bad, (uint64_t)r);
  if (!(d > 0.0) || !isfinite(d)) record_bad(a.bad + 1, (uint64_t)r);
  return d;
}

template <int K>
__global__ void __launch_bounds__(kBlock) k_ratio_program(const __grid_constant__ RatioArgs a) {
  constexpr int W = K + K * K;
  const int64_t chunks = (a.n + HK_CHUNK - 1) / HK_CHUNK;
  for (int64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
    double acc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) acc[w] = 0.0;
#pragma unroll 1
    for (int i = 0; i < kRowsPerThread; ++i) {
      const int64_t r = ch * HK_CHUNK + i * kBlock + threadIdx.x;
      if (r >= a.n) continue;
      double p[K];
      const double d = ratio_event<K>(a, r, p);
#pragma unroll
      for (int k = 0; k < K; ++k) p[k] = p[k] / d;  // ratios = p / dens (fitting.py:421)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        acc[k] += p[k];
#pragma unroll
        for (int j = 0; j < K; ++j) acc[K + k * K + j] += p[k] * p[j];
      }
    }
    block_sum_store<W>(acc, a.part + (int64_t)W * ch);
  }
}

struct SplotProgArgs {
  RatioArgs r;
  double V[HK_MAX_COMPONENTS * HK_MAX_COMPONENTS];
  double* out[HK_MAX_COMPONENTS];
};

template <int K>
__global__ void __launch_bounds__(kBlock) k_splot_program(const __grid_constant__ SplotProgArgs a) {
  const int64_t r = blockIdx.x * (int64_t)kBlock + threadIdx.x;
  if (r >= a.r.n) return;
  double p[K];
  const double d = ratio_event<K>(a.r, r, p);
#pragma unroll
  for (int s = 0; s < K; ++s) {
    double num = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) num = j == 0 ? p[j] * a.V[s * K + j] : num + p[j] * a.V[s * K + j];
    a.out[s][r] = num / d;  // (p @ V.T) / dens (splot.py:114)
  }
}

template <template <int> class Kern, class Args>
int launch_by_k(int K, unsigned grid, cudaStream_t st, const Args& a, const char* what);

#define HK_K_CASES(KERN)                                       \
  switch (K) {                                                 \
    case 1: KERN<1><<<grid, kBlock, 0, st>>>(a); break;        \
    case 2: KERN<2><<<grid, kBlock, 0, st>>>(a); break;        \
    case 3: KERN<3><<<grid, kBlock, 0, st>>>(a); break;        \
    case 4: KERN<4><<<grid, kBlock, 0, st>>>(a); break;        \
    case 5: KERN<5><<<grid, kBlock, 0, st>>>(a); break;        \
    case 6: KERN<6><<<grid, kBlock, 0, st>>>(a); break;        \
    case 7: KERN<7><<<grid, kBlock, 0, st>>>(a); break;        \
    default: KERN<8><<<grid, kBlock, 0, st>>>(a); break;       \
  }

int fill_ratio_args(const double* const* d_obs, int64_t n, const hk_density_t* m, RatioArgs* a) {
  if (int rc = validate_density(m)) return rc;
  HK_REQUIRE(n >= 0, "negative n");
  HK_REQUIRE(n == 0 || d_obs, "NULL observables");
  std::memset(a, 0, sizeof(*a));
  for (int c = 0; c < m->n_obs && n > 0; ++c) {
    HK_REQUIRE(d_obs[c], "observable column %d NULL", c);
    a->cols[c] = d_obs[c];
  }
  a->n = n;
  a->m = *m;
  return HK_OK;
}

// ------------------------------------------------- column statistics -----
// hk_column_stats: per 4096-row chunk {min, max, sum, non-finite count} over
// the finite values (min/max by shuffle + shared memory, sum and count by the
// deterministic block_sum_store tree), then one CTA folds the chunks in a
// fixed order.  Read once per data column (fitting.py caches the result).
__device__ __forceinline__ void block_minmax(double& lo, double& hi) {
  __shared__ double s_lo[kBlock / 32], s_hi[kBlock / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    lo = fmin(lo, __shfl_down_sync(0xffffffffu, lo, off));
    hi = fmax(hi, __shfl_down_sync(0xffffffffu, hi, off));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_lo[warp] = lo;
    s_hi[warp] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kBlock / 32; ++i) {
      s_lo[0] = fmin(s_lo[0], s_lo[i]);
      s_hi[0] = fmax(s_hi[0], s_hi[i]);
    }
  }
  __syncthreads();
  lo = s_lo[0];
  hi = s_hi[0];
  __syncthreads();
}

__global__ void __launch_bounds__(kBlock) k_col_stats(const double* __restrict__ x, int64_t n,
                                                     double* __restrict__ part) {
  const int64_t chunks = (n + kFcnTile - 1) / kFcnTile;
  for (int64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    double lo = inf, hi = -inf, acc[2] = {0.0, 0.0};
    for (int i = 0; i < kFcnRows; ++i) {
      const int64_t r = ch * kFcnTile + i * kBlock + threadIdx.x;
      if (r >= n) break;
      const double v = __ldg(x + r);
      if (isfinite(v)) {
        lo = fmin(lo, v);
        hi = fmax(hi, v);
        acc[0] += v;
      } else {
        acc[1] += 1.0;
      }
    }
    block_minmax(lo, hi);
    block_sum_store<2>(acc, part + 4 * ch + 2);
    if (threadIdx.x == 0) {
      part[4 * ch] = lo;
      part[4 * ch + 1] = hi;
    }
  }
}

__global__ void __launch_bounds__(kBlock) k_col_stats_fold(const double* __restrict__ part, int64_t chunks,
                                                          double* __restrict__ out) {
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  double lo = inf, hi = -inf, acc[2] = {0.0, 0.0};
  for (int64_t i = threadIdx.x; i < chunks; i += kBlock) {
    lo = fmin(lo, part[4 * i]);
    hi = fmax(hi, part[4 * i + 1]);
    acc[0] += part[4 * i + 2];
    acc[1] += part[4 * i + 3];
  }
  block_minmax(lo, hi);
  block_sum_store<2>(acc, out + 2);
  if (threadIdx.x == 0) {
    out[0] = lo;
    out[1] = hi;
  }
}

}  // namespace hk

using namespace hk;

extern "C" {

int64_t hk_nll_work_doubles(int64_t n) {
  if (n <= 0) return kFcnWorkHead;
  int64_t full, tail;
  fcn_schedule(n, &full, &tail);
  return kFcnWorkHead + full + tail;
}

int hk_nll_program_eval(const double* const* d_obs, int64_t n, const hk_density_t* model,
                        double* d_work, double* h_logsum, uint64_t* h_first_bad,
                        uint64_t* h_first_div0, void* stream) {
  HK_NVTX("hk_nll_program_eval");
  if (int rc = validate_density(model)) return rc;
  HK_REQUIRE(n > 0, "cannot evaluate an empty data set");
  HK_REQUIRE(d_obs && d_work && (!h_logsum || h_first_bad), "NULL pointer");
  FcnProgArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int c = 0; c < model->n_obs; ++c) {
    HK_REQUIRE(d_obs[c], "observable column %d NULL", c);
    a.cols[c] = d_obs[c];
  }
  a.n = n;
  a.prog = model->program;
  Mailbox* mb = nullptr;
  if (int rc = fcn_setup(d_work, n, &a.w, h_logsum ? &mb : nullptr)) return rc;
  cudaStream_t st = as_stream(stream);
  const unsigned grid = chunk_grid(a.w.full + a.w.tail_ctas);
  const void* jit = nullptr;
  if (int rc = jit_fcn(model->program, n, &jit)) return rc;
  if (jit) {
    void* args[] = {&a};
    HK_CUDA(cudaLaunchKernel(jit, dim3(grid), dim3(kBlock), args, 0, st));
  } else {
    k_nll_program<<<grid, kBlock, 0, st>>>(a);
    if (int rc = check_launch("k_nll_program")) return rc;
  }
  if (!h_logsum) return HK_OK;
  return fcn_wait(mb, a.w.seq, st, "hk_nll_program_eval", h_logsum, h_first_bad, h_first_div0);
}

int hk_nll_combine(const double* d_gathered, int32_t world, double* h_logsum, uint64_t* h_first_bad,
                   uint64_t* h_first_div0, void* stream) {
  HK_NVTX("hk_nll_combine");
  HK_REQUIRE(world >= 1 && d_gathered && h_logsum && h_first_bad, "bad combine arguments");
  Mailbox* mb = nullptr;
  if (int rc = mailbox(&mb)) return rc;
  FcnWork w;
  std::memset(&w, 0, sizeof(w));
  w.host_mail = mb->d;
  w.seq = ++mb->seq;
  cudaStream_t st = as_stream(stream);
  k_nll_combine<<<1, 32, 0, st>>>(d_gathered, world, w);
  if (int rc = check_launch("k_nll_combine")) return rc;
  return fcn_wait(mb, w.seq, st, "hk_nll_combine", h_logsum, h_first_bad, h_first_div0);
}

int hk_ratio_partials_program(const double* const* d_obs, int64_t n, const hk_density_t* model,
                              double* d_partials, uint64_t* d_first_bad, void* stream) {
  HK_NVTX("hk_ratio_partials_program");
  RatioArgs a;
  if (int rc = fill_ratio_args(d_obs, n, model, &a)) return rc;
  if (n == 0) return HK_OK;
  HK_REQUIRE(d_partials && d_first_bad, "NULL pointer");
  a.part = d_partials;
  a.bad = reinterpret_cast<unsigned long long*>(d_first_bad);
  const int K = model->n_comp;
  const unsigned grid = chunk_grid(num_chunks(n));
  cudaStream_t st = as_stream(stream);
  HK_K_CASES(k_ratio_program)
  return check_launch("k_ratio_program");
}

int hk_splot_weights_program(const double* const* d_obs, int64_t n, const hk_density_t* model,
                             const double* V, double* const* d_out, uint64_t* d_first_bad,
                             void* stream) {
  HK_NVTX("hk_splot_weights_program");
  SplotProgArgs a;
  std::memset(&a, 0, sizeof(a));
  if (int rc = fill_ratio_args(d_obs, n, model, &a.r)) return rc;
  const int K = model->n_comp;
  HK_REQUIRE(V && d_out && d_first_bad, "NULL pointer");
  for (int i = 0; i < K * K; ++i) a.V[i] = V[i];
  for (int s = 0; s < K; ++s) {
    HK_REQUIRE(d_out[s] || n == 0, "output column %d NULL", s);
    a.out[s] = d_out[s];
  }
  if (n == 0) return HK_OK;
  a.r.bad = reinterpret_cast<unsigned long long*>(d_first_bad);
  const unsigned grid = (unsigned)((n + kBlock - 1) / kBlock);
  cudaStream_t st = as_stream(stream);
  HK_K_CASES(k_splot_program)
  return check_launch("k_splot_program");
}

int hk_nll_partials(const double* d_x, int64_t n, const hk_model_t* model, double* d_partials,
                    uint64_t* d_first_bad, void* stream) {
  HK_NVTX("hk_nll_partials");
  Coeffs c;
  if (int rc = make_coeffs(model, &c)) return rc;
  HK_REQUIRE(n >= 0, "negative n");
  if (n == 0) return HK_OK;
  HK_REQUIRE(d_x && d_partials, "NULL pointer");
  return launch_nll(d_x, n, c, d_partials, reinterpret_cast<unsigned long long*>(d_first_bad),
                    as_stream(stream));
}

int hk_nll_eval(const double* d_x, int64_t n, const hk_model_t* model, double* d_work,
                double* h_logsum, uint64_t* h_first_bad, void* stream) {
  HK_NVTX("hk_nll_eval");
  Coeffs c;
  if (int rc = make_coeffs(model, &c, n)) return rc;
  HK_REQUIRE(n > 0, "cannot evaluate an empty data set");
  HK_REQUIRE(d_x && d_work && (!h_logsum || h_first_bad), "NULL pointer");
  cudaStream_t st = as_stream(stream);
  FcnWork w;
  Mailbox* mb = nullptr;
  if (int rc = fcn_setup(d_work, n, &w, h_logsum ? &mb : nullptr)) return rc;
  w.div0 = nullptr;  // the closed-form shapes have no divisions to check
  const unsigned grid = chunk_grid(w.full + w.tail_ctas);
  switch (fcn_variant(c)) {
    case kFcnFast:
      if (n >= (int64_t)HK_FCN_TMA_MIN_N) {  // enough tiles to keep every persistent CTA busy
        const int64_t tiles = (n + kFcnTile - 1) / kFcnTile;
        const int g = fast_tma_grid();
        k_nll_fast_tma<<<(unsigned)(tiles < g ? tiles : g), kBlock, kTmaSmem, st>>>(d_x, n, c, w);
      } else {
        k_nll_fused<kFcnFast><<<grid, kBlock, 0, st>>>(d_x, n, c, w);
      }
      break;
    case kFcnFactored: k_nll_fused<kFcnFactored><<<grid, kBlock, 0, st>>>(d_x, n, c, w); break;
    case kFcnGE: k_nll_fused<kFcnGE><<<grid, kBlock, 0, st>>>(d_x, n, c, w); break;
    default: k_nll_fused<kFcnGeneric><<<grid, kBlock, 0, st>>>(d_x, n, c, w); break;
  }
  if (int rc = check_launch("k_nll_fused")) return rc;
  if (!h_logsum) return HK_OK;
  return fcn_wait(mb, w.seq, st, "hk_nll_eval", h_logsum, h_first_bad, nullptr);
}

int64_t hk_nll_many_work_doubles(int64_t n, int32_t k) {
  const int64_t groups = k < 1 ? 1 : (k + kManyG - 1) / kManyG;
  return 256 + (n <= 0 ? 0 : (n + kFcnTile - 1) / kFcnTile) * groups * kManyG;
}

int hk_nll_eval_many(const double* d_x, int64_t n, const hk_model_t* models, int32_t k, double* d_work,
                     double* h_logsums, uint64_t* h_first_bad, void* stream) {
  HK_NVTX("hk_nll_eval_many");
  HK_REQUIRE(k >= 1 && k <= HK_MAX_POINTS, "point count %d outside 1..%d", k, HK_MAX_POINTS);
  HK_REQUIRE(n > 0, "cannot evaluate an empty data set");
  HK_REQUIRE(d_x && d_work && models && h_logsums && h_first_bad, "NULL pointer");
  ManyArgs a;
  std::memset(&a, 0, sizeof(a));
  // one variant for the whole batch, the one each single-point call would
  // take (so every value is bit-identical to hk_nll_eval's); mixed batches
  // run point by point
  bool factored = true;
  int variant = -1;
  for (int p = 0; p < k; ++p) {
    Coeffs c;
    if (int rc = make_coeffs(models + p, &c, n)) return rc;
    const int v = fcn_variant(c);
    if ((v != kFcnFactored && v != kFcnFast) || (variant >= 0 && v != variant)) {
      factored = false;
      break;
    }
    variant = v;
    a.pt[p] = make_point(c);
  }
  for (int p = k; p < ((k + kManyG - 1) / kManyG) * kManyG; ++p) a.pt[p] = a.pt[k - 1];
  if (!factored) {  // other model kinds: one single-point pass per point (same values)
    int64_t full, tail;
    fcn_schedule(n, &full, &tail);
    for (int p = 0; p < k; ++p)
      if (int rc = hk_nll_eval(d_x, n, models + p, d_work, h_logsums + p, h_first_bad + p, stream)) return rc;
    return HK_OK;
  }
  // d_work (zero-filled once, re-armed by the kernel): [0, 64) sums,
  // [64, 128) ~bad cells, [128, 160) group tickets (u32), [160] done (u32),
  // [256 ..) partials [tile][kpad]
  a.x = d_x;
  a.n = n;
  a.k = k;
  a.groups = (k + kManyG - 1) / kManyG;
  a.tiles = (n + kFcnTile - 1) / kFcnTile;
  a.kpad = (int64_t)a.groups * kManyG;
  a.out = d_work;
  a.bad = reinterpret_cast<unsigned long long*>(d_work + 64);
  a.gticket = reinterpret_cast<unsigned int*>(d_work + 128);
  a.done = reinterpret_cast<unsigned int*>(d_work + 160);
  a.part = d_work + 256;
  Mailbox* mb = nullptr;
  if (int rc = mailbox(&mb)) return rc;
  a.host_mail = mb->d;
  a.seq = ++mb->seq;
  a.rev = fcn_flip(d_work, n * (int64_t)sizeof(double), a.groups);
  cudaStream_t st = as_stream(stream);
  if (variant == kFcnFast)
    k_nll_many<kFcnFast><<<chunk_grid(a.tiles * a.groups), kBlock, 0, st>>>(a);
  else
    k_nll_many<kFcnFactored><<<chunk_grid(a.tiles * a.groups), kBlock, 0, st>>>(a);
  if (int rc = check_launch("k_nll_many")) return rc;
  double first = 0.0;
  uint64_t dummy = 0;
  // fcn_wait reads [1], [2]; the payload here is [1 .. 2k]
  if (int rc = fcn_wait(mb, a.seq, st, "hk_nll_eval_many", &first, &dummy, nullptr)) return rc;
  for (int p = 0; p < k; ++p) {
    const unsigned long long bits = mb->h[1 + p];
    std::memcpy(h_logsums + p, &bits, sizeof(double));
    h_first_bad[p] = mb->h[1 + k + p];
  }
  return HK_OK;
}

int hk_fcn_session_start(const double* d_x, int64_t n, double* d_work, int64_t idle_us) {
  HK_REQUIRE(n > 0 && d_x && d_work, "bad session arguments");
  HK_REQUIRE(idle_us > 0, "idle timeout must be positive");
  if (int rc = session_stop(t_session)) return rc;
  Session& S = t_session;
  int dev = 0, sms = 0, per_sm = 0, coop = 0;
  HK_CUDA(cudaGetDevice(&dev));
  if (S.device >= 0 && S.device != dev)
    if (int rc = session_stop(S, true)) return rc;
  HK_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  HK_REQUIRE(coop, "device %d has no cooperative launch", dev);
  HK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  HK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fcn_server, kBlock, 0));
  HK_REQUIRE(per_sm >= 1, "FCN session kernel does not fit an SM");
  if (S.device < 0) {  // first session on this thread: allocate once, reused by later sessions
    HK_CUDA(cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking));
    HK_CUDA(cudaHostAlloc(&S.h_cmd, sizeof(ServerCmd), cudaHostAllocMapped));
    std::memset(S.h_cmd, 0, sizeof(ServerCmd));
    HK_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&S.d_cmd), S.h_cmd, 0));
    HK_CUDA(cudaMalloc(&S.dev, sizeof(ServerDev)));
    S.device = dev;
  }
  S.active = true;
  {  // the page reads "nothing new" to the fresh CTAs: every slot carries the last answered seq
    CmdSlot v[kCmdSlots];
    for (int k = 0; k < kCmdSlots; ++k) {
      v[k].seq = S.seq;
      v[k].word = 0ull;
    }
    write_slots(S.h_cmd, v);
  }
  Mailbox* mb = nullptr;
  if (int rc = mailbox(&mb)) return rc;
  FcnWork w;
  if (int rc = fcn_setup(d_work, n, &w, nullptr)) return rc;
  w.div0 = nullptr;
  w.host_mail = mb->d;
  S.args.x = d_x;
  S.args.n = n;
  S.args.w = w;
  S.args.cmd = S.d_cmd;
  S.args.dev = S.dev;
  S.args.idle_ns = idle_us * 1000;
  S.grid = (unsigned)(sms * per_sm);
  mb->h[6] = 0;
  return session_launch(S);
}

int hk_fcn_session_eval(const hk_model_t* model, double* h_logsum, uint64_t* h_first_bad) {
  HK_NVTX("hk_fcn_session_eval");
  Session& S = t_session;
  HK_REQUIRE(S.active, "no FCN session on this thread (hk_fcn_session_start)");
  HK_REQUIRE(h_logsum && h_first_bad, "NULL pointer");
  Coeffs c;
  if (int rc = make_coeffs(model, &c, S.args.n)) return rc;
  const int variant = fcn_variant(c);
  if (variant == kFcnGeneric) {
    set_error("an FCN session serves the Gaussian + exponential model");
    return HK_EUNSUPPORTED;
  }
  int cur = 0;
  HK_CUDA(cudaGetDevice(&cur));
  HK_REQUIRE(cur == S.device, "FCN session lives on device %d, current device is %d", S.device, cur);
  Mailbox* mb = nullptr;
  if (int rc = mailbox(&mb)) return rc;
  if (mb->h[6]) {  // the CTAs left on their idle timeout: bring them back
    HK_CUDA(cudaStreamSynchronize(S.stream));
    mb->h[6] = 0;
    if (int rc = session_launch(S)) return rc;
  }
  // the mailbox's sequence numbers are per (thread, device): the session's
  // command seq is the mailbox seq the answer will carry
  const unsigned long long seq = ++mb->seq;
  const FPoint pt = make_point(c);
  double words[kCmdSlots - 1];
  std::memcpy(words, &pt, sizeof(pt));
  CmdSlot v[kCmdSlots];
  v[0].seq = seq;
  v[0].word = (unsigned long long)variant;
  for (int k = 1; k < kCmdSlots; ++k) {
    v[k].seq = seq;
    std::memcpy(&v[k].word, &words[k - 1], 8);
  }
  write_slots(S.h_cmd, v);
  for (unsigned spins = 1;; ++spins) {
    if (mb->h[0] == seq) break;
    if ((spins & 4095u) == 0) {
      const cudaError_t e = cudaStreamQuery(S.stream);
      if (e == cudaSuccess) {  // timed out between our check and the command: relaunch
        if (mb->h[0] == seq) break;
        mb->h[6] = 0;
        if (int rc = session_launch(S)) return rc;
      } else if (e != cudaErrorNotReady) {
        return cuda_fail(e, "hk_fcn_session_eval");
      }
    }
  }
  S.seq = seq;  // answered: a relaunch must treat it as done
  std::atomic_thread_fence(std::memory_order_acquire);
  const unsigned long long sum_bits = mb->h[1];
  std::memcpy(h_logsum, &sum_bits, sizeof(double));
  *h_first_bad = mb->h[2];
  return HK_OK;
}

int hk_fcn_session_stop(void) { return session_stop(t_session); }

int64_t hk_fcn_session_device_ns(void) {
  Mailbox* mb = nullptr;
  if (mailbox(&mb)) return -1;
  return (int64_t)(mb->h[5] - mb->h[4]);
}

int hk_yield_partials(const double* d_x, int64_t n, const hk_model_t* model, double* d_partials,
                      uint64_t* d_first_bad, void* stream) {
  HK_NVTX("hk_yield_partials");
  HK_REQUIRE(model && model->n_comp >= 1 && model->n_comp <= 4,
             "yield stationarity supports 1..4 components");
  PdfCoeffs c;
  if (int rc = make_pdf_coeffs(model, &c)) return rc;
  HK_REQUIRE(n >= 0, "negative n");
  if (n == 0) return HK_OK;
  HK_REQUIRE(d_x && d_partials, "NULL pointer");
  const unsigned grid = chunk_grid(num_chunks(n));
  cudaStream_t st = as_stream(stream);
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(d_first_bad);
  switch (model->n_comp) {
    case 1: k_yield<1><<<grid, kBlock, 0, st>>>(d_x, n, c, d_partials, bad); break;
    case 2: k_yield<2><<<grid, kBlock, 0, st>>>(d_x, n, c, d_partials, bad); break;
    case 3: k_yield<3><<<grid, kBlock, 0, st>>>(d_x, n, c, d_partials, bad); break;
    default: k_yield<4><<<grid, kBlock, 0, st>>>(d_x, n, c, d_partials, bad); break;
  }
  return check_launch("k_yield");
}

int hk_splot_weights(const double* d_x, int64_t n, const hk_model_t* model, const double* V,
                     double* const* d_out, uint64_t* d_first_bad, void* stream) {
  HK_NVTX("hk_splot_weights");
  HK_REQUIRE(model && model->n_comp >= 1 && model->n_comp <= 4, "sPlot supports 1..4 species");
  HK_REQUIRE(V && d_out, "NULL pointer");
  SplotArgs a;
  std::memset(&a, 0, sizeof(a));
  if (int rc = make_pdf_coeffs(model, &a.c)) return rc;
  a.k = model->n_comp;
  for (int i = 0; i < a.k * a.k; ++i) a.V[i] = V[i];
  for (int i = 0; i < a.k; ++i) {
    HK_REQUIRE(d_out[i], "output column %d NULL", i);
    a.out[i] = d_out[i];
  }
  a.bad = reinterpret_cast<unsigned long long*>(d_first_bad);
  HK_REQUIRE(n >= 0, "negative n");
  if (n == 0) return HK_OK;
  HK_REQUIRE(d_x, "NULL data");
  k_splot<<<(unsigned)((n + kBlock - 1) / kBlock), kBlock, 0, as_stream(stream)>>>(d_x, n, a);
  return check_launch("k_splot");
}

int64_t hk_column_stats_work_doubles(int64_t n) {
  return 4 * ((n <= 0 ? 0 : (n + kFcnTile - 1) / kFcnTile) + 1);
}

int hk_column_stats(const double* d_x, int64_t n, double* d_work, double* h_out, void* stream) {
  HK_NVTX("hk_column_stats");
  HK_REQUIRE(n > 0 && d_x && d_work && h_out, "bad column-statistics arguments");
  cudaStream_t st = as_stream(stream);
  const int64_t chunks = (n + kFcnTile - 1) / kFcnTile;
  k_col_stats<<<chunk_grid(chunks), kBlock, 0, st>>>(d_x, n, d_work + 4);
  if (int rc = check_launch("k_col_stats")) return rc;
  k_col_stats_fold<<<1, kBlock, 0, st>>>(d_work + 4, chunks, d_work);
  if (int rc = check_launch("k_col_stats_fold")) return rc;
  HK_CUDA(cudaMemcpyAsync(h_out, d_work, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
  HK_CUDA(cudaStreamSynchronize(st));
  return HK_OK;
}

int hk_model_density(const double* d_x, int64_t n, const hk_model_t* model, double* d_out,
                     void* stream) {
  HK_NVTX("hk_model_density");
  Coeffs c;
  if (int rc = make_coeffs(model, &c)) return rc;
  HK_REQUIRE(n >= 0, "negative n");
  if (n == 0) return HK_OK;
  HK_REQUIRE(d_x && d_out, "NULL pointer");
  k_density_exact<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(d_x, n, *model,
                                                                               d_out);
  return check_launch("k_density_exact");
}

}  // extern "C"

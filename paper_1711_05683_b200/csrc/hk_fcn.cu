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
#include <cstring>

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
  // (m_lo, m_hi) give amp_k e^M a normal, finite double for both k
  double m_lo, m_hi;
};

// FCN kernel variants
constexpr int kFcnGeneric = 0;   // any component list
constexpr int kFcnGE = 1;        // Gaussian + exponential, reference op order
constexpr int kFcnFactored = 2;  // Gaussian + exponential, one exp per event

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
__device__ __forceinline__ double density_ge(const Coeffs& c, double x) {
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
__device__ __forceinline__ bool density_factored(const Coeffs& c, double x, double* s, double* M) {
  const double z = (x - c.shift[0]) * c.scale[0];
  const double A = -0.5 * z * z;
  const double B = x * c.scale[1];
  // (fmax(A, B) and exp(-|A - B|) instead of the selects measured slower:
  // 29.8 vs 29.0 us per 1e7 events)
  const bool ga = A >= B;  // NaN: false, M = B = NaN
  *M = ga ? A : B;
  const double t = fcn_exp(ga ? B - A : A - B);
  *s = ga ? c.amp[0] + c.amp[1] * t : c.amp[0] * t + c.amp[1];
  return *M > c.m_lo && *M < c.m_hi;
}

// One tile: returns sum ln d over this thread's rows; flags
// d <= 0 / non-finite (fitting.py:200-205) as ~row in *bad (max = first row).
template <int V>
__device__ __forceinline__ void fcn_row(const Coeffs& c, double xv, int64_t row, LogProd& lp,
                                       double& msum, unsigned long long* bad) {
  if (V == kFcnFactored) {
    double s, M;
    if (density_factored(c, xv, &s, &M)) {
      lp.add_normal(s);  // s in [min amp, amp0 + amp1]: normal
      msum += M;
      return;
    }
  }
  const double d = V == kFcnGeneric ? density(c, xv) : density_ge(c, xv);
  if (!(d > 0.0) || !isfinite(d)) *bad = max(*bad, ~(unsigned long long)row);
  lp.add(d);
}

// sum ln d over rows [begin, end) (at most one tile): all 16 loads in flight
// for a full tile, a guarded loop otherwise
template <int V>
__device__ __forceinline__ double range_logsum(const double* __restrict__ x, int64_t begin,
                                               int64_t end, const Coeffs& c,
                                               unsigned long long* bad) {
  const int64_t r0 = begin + threadIdx.x;
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
  return range_logsum<V>(x, b, b + kFcnTile < n ? b + kFcnTile : n, c, bad);
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
  const int64_t chunks = w.full + w.tail_ctas;
  for (int64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
    unsigned long long bad = 0;
    int64_t begin, end;
    fcn_range(w, n, ch, &begin, &end);
    double acc[1] = {range_logsum<V>(x, begin, end, c, &bad)};
    if (bad) atomicMax(w.bad, bad);
    block_sum_store<1>(acc, w.part + ch);
  }
  fcn_finish(w, chunks);
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
#pragma unroll 1
    for (int i = 0; i < kRowsPerThread; ++i) {
      const int64_t r = ch * HK_CHUNK + i * kBlock + threadIdx.x;
      if (r >= n) continue;
      const double xv = __ldg(x + r);
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
    }
    block_sum_store<W>(acc, part + (int64_t)W * ch);
  }
}

int make_coeffs(const hk_model_t* m, Coeffs* c) {
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
      c->amp[1] < 1e300) {
    c->m_lo = -690.0 - std::log(std::fmin(c->amp[0], c->amp[1]));
    c->m_hi = 700.0 - std::log(c->amp[0] + c->amp[1]);
  }
  return HK_OK;
}

int fcn_variant(const Coeffs& c) {
  const bool ge = c.n_comp == 2 && c.kind[0] == HK_SHAPE_GAUSS && c.kind[1] == HK_SHAPE_EXPO;
  if (!ge) return kFcnGeneric;
  return c.m_lo < c.m_hi ? kFcnFactored : kFcnGE;
}

int launch_nll(const double* d_x, int64_t n, const Coeffs& c, double* part,
               unsigned long long* bad, cudaStream_t st) {
  const unsigned grid = chunk_grid((n + kFcnTile - 1) / kFcnTile);
  switch (fcn_variant(c)) {
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

// Mapped pinned mailbox per (host thread, device) for hk_nll_eval:
// [0] sequence number, [1] sum-of-logs bits, [2] first bad row.
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
    HK_CUDA(cudaHostAlloc(&p, 4 * sizeof(unsigned long long), cudaHostAllocMapped));
    std::memset(p, 0, 4 * sizeof(unsigned long long));
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
// first global row), [8..] partials.
constexpr int kFcnWorkHead = 8;

// mb == NULL: asynchronous call, the result stays in d_work[0, 1, 5]
int fcn_setup(double* d_work, int64_t n, FcnWork* w, Mailbox** mb) {
  w->out = d_work;
  w->bad = reinterpret_cast<unsigned long long*>(d_work + 2);
  w->ticket = reinterpret_cast<unsigned int*>(d_work + 3);
  w->div0 = reinterpret_cast<unsigned long long*>(d_work + 4);
  w->part = d_work + kFcnWorkHead;
  w->host_mail = nullptr;
  w->seq = 0;
  if (mb) {
    if (int rc = mailbox(mb)) return rc;
    w->host_mail = (*mb)->d;
    w->seq = ++(*mb)->seq;
  }
  fcn_schedule(n, &w->full, &w->tail_ctas);
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
  Coeffs c;
  if (int rc = make_coeffs(model, &c)) return rc;
  HK_REQUIRE(n > 0, "cannot evaluate an empty data set");
  HK_REQUIRE(d_x && d_work && (!h_logsum || h_first_bad), "NULL pointer");
  cudaStream_t st = as_stream(stream);
  FcnWork w;
  Mailbox* mb = nullptr;
  if (int rc = fcn_setup(d_work, n, &w, h_logsum ? &mb : nullptr)) return rc;
  w.div0 = nullptr;  // the closed-form shapes have no divisions to check
  const unsigned grid = chunk_grid(w.full + w.tail_ctas);
  switch (fcn_variant(c)) {
    case kFcnFactored: k_nll_fused<kFcnFactored><<<grid, kBlock, 0, st>>>(d_x, n, c, w); break;
    case kFcnGE: k_nll_fused<kFcnGE><<<grid, kBlock, 0, st>>>(d_x, n, c, w); break;
    default: k_nll_fused<kFcnGeneric><<<grid, kBlock, 0, st>>>(d_x, n, c, w); break;
  }
  if (int rc = check_launch("k_nll_fused")) return rc;
  if (!h_logsum) return HK_OK;
  return fcn_wait(mb, w.seq, st, "hk_nll_eval", h_logsum, h_first_bad, nullptr);
}

int hk_yield_partials(const double* d_x, int64_t n, const hk_model_t* model, double* d_partials,
                      uint64_t* d_first_bad, void* stream) {
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

int hk_model_density(const double* d_x, int64_t n, const hk_model_t* model, double* d_out,
                     void* stream) {
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

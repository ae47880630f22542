// hk_integrate.cuh -- fused phsp_generate -> phsp_average (config C5): the
// event stays in registers, only the 5 chunk moments reach HBM.
//
// The chunk loop is written once, over an integrand policy I:
//   PairIntegrand     Dalitz m^2_ij / Breit-Wigner(m^2_ij), recognised on the host
//   ProgramIntegrand  any lowered functor, through the interpreter (run_program)
//   JitIntegrand      any lowered functor as straight-line code, emitted and
//                     NVRTC-compiled at run time by hk_jit.cu, which includes
//                     this header -- so the generator is the same source and,
//                     with -fmad=false on both sides, produces the same bits.
// Rows are visited in one fixed order for every policy -- (r, r + 2048) pairs
// for i = 0..7 -- whether two events run interleaved (ILP 2, full chunks) or
// one at a time, so all three policies give bit-identical chunk moments for
// the same per-event f.
#pragma once

#include "hk_device.cuh"

namespace hk {

// Generator shape, measured on B200 for 1e8 3-body events (tools/bench_gen.py):
//   1 event/iteration, 2 CTAs/SM (<=128 regs) ........ 2.55 ms
//   1 event/iteration, 3 CTAs/SM (<=80 regs) ......... 2.315 ms
//   2 events/iteration, 2 CTAs/SM (<=128 regs) ....... 2.240 ms  <- n <= 4
//   2 events/iteration, 1 CTA/SM ..................... 2.747 ms
// Two independent events per iteration give the scheduler interleavable
// dependency chains (the kernel is issue/FP64-latency bound, "wait" stalls);
// larger final states would spill and keep one event per iteration.
template <int N>
struct GenShape {
  static constexpr int ilp = N <= 4 ? 2 : 1;
  static constexpr int min_blocks = 2;
};

struct IntArgs {
  hk_decay_t d;
  RngParams rp;
  uint64_t ev_begin;
  int64_t count;
  hk_program_t f;
  double* part;  // 5 doubles per chunk
  unsigned long long* div0_bad;
  unsigned long long* nonfinite_bad;
  hk_pair_integrand_t pair;  // kind != HK_PAIR_NONE: f from the fast pair-mass path
};

// daughter q's component c of the register-resident event, q a runtime index
template <int N>
__device__ __forceinline__ double pick(const double (&p)[4 * N], int q, int c) {
  double v = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) v = select_f64(j == q, p[4 * j + c], v);
  return v;
}

// m^2 of daughters i+j with the op order of the reference's pinned integrand
// (test_phasespace.py:196-201), then identity (+0.0) or a Breit-Wigner.
struct PairIntegrand {
  static constexpr bool kIlp2 = true;
  template <int N>
  __device__ __forceinline__ static double eval(const IntArgs& a, double, const double (&p)[4 * N],
                                                uint64_t) {
    const hk_pair_integrand_t& f = a.pair;
    const double e = pick<N>(p, f.i, 0) + pick<N>(p, f.j, 0);
    const double x = pick<N>(p, f.i, 1) + pick<N>(p, f.j, 1);
    const double y = pick<N>(p, f.i, 2) + pick<N>(p, f.j, 2);
    const double z = pick<N>(p, f.i, 3) + pick<N>(p, f.j, 3);
    const double s = e * e - x * x - y * y - z * z;
    if (f.kind == HK_PAIR_BW) {
      const double t = s - f.m0 * f.m0;
      return 1.0 / (t * t + (f.m0 * f.m0) * (f.g0 * f.g0));
    }
    return s + 0.0;
  }
};

// interpreter: columns (weight, p1_e, ...) of the event in a small array
struct ProgramIntegrand {
  static constexpr bool kIlp2 = false;
  template <int N>
  __device__ __forceinline__ static double eval(const IntArgs& a, double w, const double (&p)[4 * N],
                                                uint64_t row) {
    double v[4 * N + 1];
    v[0] = w;
#pragma unroll
    for (int j = 0; j < 4 * N; ++j) v[1 + j] = p[j];
    bool div0 = false;
    const double f = run_program(a.f, [&](int col) { return v[col]; }, &div0);
    if (div0) record_bad(a.div0_bad, row);
    return f;
  }
};

__device__ __forceinline__ void add_moments(double (&acc)[5], double w, double f) {
  const double ww = w * w;
  acc[0] += w;
  acc[1] += w * f;
  acc[2] += ww;
  acc[3] += ww * f;
  acc[4] += ww * f * f;
}

// phsp_generate -> phsp_average (phasespace.py:162-188 then :310-349).
template <int N, int MODE, class I>
__device__ __forceinline__ void integrate_chunks(const IntArgs& a) {
  const int64_t chunks = (a.count + HK_CHUNK - 1) / HK_CHUNK;
  Frame mf{};
  if (a.d.moving) mf = make_frame(a.d.mother[0], a.d.mother[1], a.d.mother[2], a.d.mother[3],
                                  a.d.m_mother);
  const RestHoist h = rest_hoist<N>(a.d);  // per-decay reciprocals, out of the event loop
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (I::kIlp2 && GenShape<N>::ilp == 2 && c * HK_CHUNK + HK_CHUNK <= a.count && !a.d.moving) {
#pragma unroll 1
      for (int i = 0; i < kRowsPerThread / 2; ++i) {  // two events per iteration (ILP 2)
        const uint64_t row0 = a.ev_begin + (uint64_t)(c * HK_CHUNK + i * kBlock + threadIdx.x);
        const uint64_t row1 = row0 + HK_CHUNK / 2;
        double p0[4 * N], p1[4 * N];
        const double w0 = rest_event<N, MODE>(a.d, a.rp, row0, p0, h);
        const double w1 = rest_event<N, MODE>(a.d, a.rp, row1, p1, h);
        const double f0 = I::template eval<N>(a, w0, p0, row0);
        const double f1 = I::template eval<N>(a, w1, p1, row1);
        if (!isfinite(f0)) record_bad(a.nonfinite_bad, row0);
        if (!isfinite(f1)) record_bad(a.nonfinite_bad, row1);
        add_moments(acc, w0, f0);
        add_moments(acc, w1, f1);
      }
      block_sum_store<5>(acc, a.part + 5 * c);
      continue;
    }
#pragma unroll 1
    for (int k = 0; k < kRowsPerThread; ++k) {  // same row order: i-th pair, then its second half
      const int64_t r = c * HK_CHUNK + (k >> 1) * kBlock + (k & 1) * (HK_CHUNK / 2) + threadIdx.x;
      if (r < a.count) {
        const uint64_t row = a.ev_begin + (uint64_t)r;
        double p[4 * N];
        const double w = rest_event<N, MODE>(a.d, a.rp, row, p, h);
        if (a.d.moving) {
#pragma unroll
          for (int j = 0; j < N; ++j) boost_fma(mf, p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
        }
        const double f = I::template eval<N>(a, w, p, row);
        if (!isfinite(f)) record_bad(a.nonfinite_bad, row);
        add_moments(acc, w, f);
      }
    }
    block_sum_store<5>(acc, a.part + 5 * c);
  }
}

}  // namespace hk

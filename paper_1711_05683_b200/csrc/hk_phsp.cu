// hk_phsp.cu -- phase-space generation, decay chains, phase-space averages
// and unweighting for sm_100a.  Compiled with -fmad=false (see hk_device.cuh).
//
// Layout in HBM: one contiguous fp64 column per schema field (phsp_schema,
// phasespace.py:60-64), owned by the caller (torch tensors on the Python side).
// A 4096-row chunk (parallel.py:18) is walked by 256 threads -- one CTA, or
// for the generators two / four smaller CTAs through a virtual thread id --
// in row-strided steps so every column store is a fully coalesced warp
// transaction, and the chunk's moment partial is a fixed-order reduction
// (per-warp slots, or a CTA tree) -- the GPU analogue of the reference's
// chunk partials.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "hepkit_cuda.h"
#include "hk_device.cuh"
#include "hk_host.h"
#include "hk_integrate.cuh"

namespace hk {

namespace cg = cooperative_groups;

constexpr int kMaxCols = 4 * HK_MAX_DAUGHTERS + 1;
constexpr int kFastMaxN = 8;  // templated register-resident kernels for n <= 8

struct GenArgs {
  hk_decay_t d;
  RngParams rp;
  uint64_t ev_begin;
  int64_t count;
  double* cols[kMaxCols];  // all NULL = no store
  double* wpart;           // 2 doubles per warp-slice (HK_WARP_SLICES per chunk) or NULL
  int store;
  int vec2;                // all columns 16-byte aligned: double2 stores (k_generate VEC2)
};

// ------------------------------------------------------------ generation ---
// one event at rest; 2-body decays take the hoisted-constant form (same bits)
template <int N, int MODE>
__device__ __forceinline__ double gen_event(const hk_decay_t& d, const TwoBody& tb, const RestHoist& h,
                                           const RngParams& rp, uint64_t row, double (&p)[4 * N]) {
  if constexpr (N == 2)
    return rest_event2<MODE>(tb, rp, row, p);
  else
    return rest_event<N, MODE>(d, rp, row, p, h);
}

// VEC2: every column pointer is 16-byte aligned, so the two adjacent rows a
// thread owns in the ILP-2 path go out as one 16-byte streaming store per
// column (st.global.cs.v2.f64; a warp writes 512 contiguous bytes).  The row
// mapping -- and so the weight partials -- is the same either way.
//
// T threads per CTA: 256 (one CTA per chunk) or fewer (kBlock / T CTAs per
// chunk, each a slice of it through a virtual thread id, so every warp keeps
// its rows and its weight-partial slot -- identical bits).  The VEC2 3/4-body
// kernels launch T = 128 at 4 CTAs/SM (the same 16 warps and 128 registers as
// 2 x 256): the finer CTA granularity measured 1.1% faster on B200 (1.7755
// vs 1.7957 ms per 1e8, same box); 64 ties, 32 is slower, and 5-6 CTAs/SM
// (102/85 registers) spill and lose.
#ifndef HK_GEN_T
#define HK_GEN_T 128
#endif
#ifndef HK_GEN_T_MINB
#define HK_GEN_T_MINB 4
#endif
template <int N, int MODE, bool VEC2, int T = kBlock>
__global__ void __launch_bounds__(T, T == kBlock ? GenShape<N>::min_blocks : HK_GEN_T_MINB)
    k_generate(const __grid_constant__ GenArgs a) {
  constexpr int kSplit = kBlock / T;  // CTAs per chunk
  const int64_t chunks = (a.count + HK_CHUNK - 1) / HK_CHUNK;
  Frame mf{};
  if (a.d.moving) mf = make_frame(a.d.mother[0], a.d.mother[1], a.d.mother[2], a.d.mother[3],
                                  a.d.m_mother);
  TwoBody tb{};
  if constexpr (N == 2) tb = two_body_consts(a.d);
  const RestHoist h = rest_hoist<N>(a.d);
  for (int64_t u = blockIdx.x; u < chunks * kSplit; u += gridDim.x) {
    const int64_t c = u / kSplit;
    const int vt = (int)(u % kSplit) * T + (int)threadIdx.x;  // thread id within the chunk
    double acc[2] = {0.0, 0.0};
    // full chunks, mother at rest: rows 2t and 2t + 1 of each 512-row block
    // together (ILP 2)
    if (GenShape<N>::ilp == 2 && c * HK_CHUNK + HK_CHUNK <= a.count && !a.d.moving) {
#pragma unroll 1
      for (int i = 0; i < kRowsPerThread / 2; ++i) {
        const int64_t r0 = c * HK_CHUNK + i * (2 * kBlock) + 2 * vt;
        const int64_t r1 = r0 + 1;
        double p0[4 * N], p1[4 * N];
        const double w0 = gen_event<N, MODE>(a.d, tb, h, a.rp, a.ev_begin + (uint64_t)r0, p0);
        const double w1 = gen_event<N, MODE>(a.d, tb, h, a.rp, a.ev_begin + (uint64_t)r1, p1);
        if (a.store) {
          if constexpr (VEC2) {
            __stcs(reinterpret_cast<double2*>(a.cols[0] + r0), make_double2(w0, w1));
#pragma unroll
            for (int j = 0; j < 4 * N; ++j)
              __stcs(reinterpret_cast<double2*>(a.cols[1 + j] + r0), make_double2(p0[j], p1[j]));
          } else {
            __stcs(a.cols[0] + r0, w0);
            __stcs(a.cols[0] + r1, w1);
#pragma unroll
            for (int j = 0; j < 4 * N; ++j) {
              __stcs(a.cols[1 + j] + r0, p0[j]);
              __stcs(a.cols[1 + j] + r1, p1[j]);
            }
          }
        }
        acc[0] += w0;
        acc[1] += w0 * w0;
        acc[0] += w1;
        acc[1] += w1 * w1;
      }
      if (a.wpart) warp_sum_store<2>(acc, a.wpart, c, vt >> 5);
      continue;
    }
#pragma unroll 1
    for (int i = 0; i < kRowsPerThread; ++i) {
      const int64_t r = c * HK_CHUNK + i * kBlock + vt;
      if (r < a.count) {
        double p[4 * N];
        const double w = gen_event<N, MODE>(a.d, tb, h, a.rp, a.ev_begin + (uint64_t)r, p);
        if (a.d.moving) {
#pragma unroll
          for (int j = 0; j < N; ++j) boost_fma(mf, p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
        }
        if (a.store) {
          __stcs(a.cols[0] + r, w);
#pragma unroll
          for (int j = 0; j < 4 * N; ++j) __stcs(a.cols[1 + j] + r, p[j]);
        }
        acc[0] += w;
        acc[1] += w * w;
      }
    }
    if (a.wpart) warp_sum_store<2>(acc, a.wpart, c, vt >> 5);
  }
}

template <int MODE>
__global__ void __launch_bounds__(kBlock) k_generate_rt(const __grid_constant__ GenArgs a) {
  const int64_t chunks = (a.count + HK_CHUNK - 1) / HK_CHUNK;
  const int n = a.d.n;
  Frame mf{};
  if (a.d.moving) mf = make_frame(a.d.mother[0], a.d.mother[1], a.d.mother[2], a.d.mother[3],
                                  a.d.m_mother);
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    double acc[2] = {0.0, 0.0};
    for (int i = 0; i < kRowsPerThread; ++i) {
      const int64_t r = c * HK_CHUNK + i * kBlock + threadIdx.x;
      if (r < a.count) {
        double p[4 * HK_MAX_DAUGHTERS];
        const double w = rest_event_rt<MODE>(a.d, a.rp, a.ev_begin + (uint64_t)r, p);
        if (a.d.moving)
          for (int j = 0; j < n; ++j) boost(mf, p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
        if (a.store) {
          __stcs(a.cols[0] + r, w);
          for (int j = 0; j < 4 * n; ++j) __stcs(a.cols[1 + j] + r, p[j]);
        }
        acc[0] += w;
        acc[1] += w * w;
      }
    }
    if (a.wpart) warp_sum_store<2>(acc, a.wpart, c);
  }
}

// ---------------------------------------------------- fused integration ----
// (chunk loop and integrand policies in hk_integrate.cuh)
template <int N, int MODE, bool PAIR>
__global__ void __launch_bounds__(kBlock, PAIR ? GenShape<N>::min_blocks : 1)
    k_integrate(const __grid_constant__ IntArgs a) {
  if constexpr (PAIR)
    integrate_chunks<N, MODE, PairIntegrand>(a);
  else
    integrate_chunks<N, MODE, ProgramIntegrand>(a);
}

// ------------------------------------------- moments over stored columns ---
struct MomArgs {
  const double* cols[kMaxCols];
  int32_t n_cols;
  int64_t count;
  hk_program_t f;
  double* part;
  unsigned long long* div0_bad;
  unsigned long long* nonfinite_bad;
};

// phsp_average over a stored block (phasespace.py:310-329): f from the
// program over the event's columns, then the five chunk moments.
__global__ void __launch_bounds__(kBlock) k_moments(const __grid_constant__ MomArgs a) {
  const int64_t chunks = (a.count + HK_CHUNK - 1) / HK_CHUNK;
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
    for (int i = 0; i < kRowsPerThread; ++i) {
      const int64_t r = c * HK_CHUNK + i * kBlock + threadIdx.x;
      if (r < a.count) {
        bool div0 = false;
        const double f = run_program(a.f, [&](int col) { return __ldg(a.cols[col] + r); }, &div0);
        if (div0) record_bad(a.div0_bad, (uint64_t)r);
        if (!isfinite(f)) record_bad(a.nonfinite_bad, (uint64_t)r);
        const double w = __ldg(a.cols[0] + r);
        const double ww = w * w;
        acc[0] += w;
        acc[1] += w * f;
        acc[2] += ww;
        acc[3] += ww * f;
        acc[4] += ww * f * f;
      }
    }
    block_sum_store<5>(acc, a.part + 5 * c);
  }
}

static_assert(kJitMaxCols == kMaxCols, "JitArgs column capacity");

inline JitArgs jit_args(const MomArgs& a) {
  JitArgs j;
  std::memset(&j, 0, sizeof(j));
  for (int c = 0; c < a.n_cols; ++c) j.cols[c] = a.cols[c];
  j.count = a.count;
  j.part = a.part;
  j.div0 = a.div0_bad;
  j.nonfin = a.nonfinite_bad;
  return j;
}

__global__ void __launch_bounds__(kBlock) k_map(const __grid_constant__ MomArgs a, double* out) {
  const int64_t r = blockIdx.x * (int64_t)kBlock + threadIdx.x;
  if (r >= a.count) return;
  bool div0 = false;
  out[r] = run_program(a.f, [&](int col) { return __ldg(a.cols[col] + r); }, &div0);
  if (div0) record_bad(a.div0_bad, (uint64_t)r);
}

// --------------------------------------------------------- decay chains ----
struct ChainArgs {
  hk_decay_t sub;
  RngParams rp;
  uint64_t ev_begin;
  int64_t count;
  const double* w_in;
  const double* p4_in[4];
  double* w_out;
  double* sub_cols[4 * HK_MAX_DAUGHTERS];
  unsigned long long* first_bad;
};

// daughter mass from its four columns (phasespace.py:259-260) + check (:261-262)
// sqrt(np.maximum(m2, 0)): the branch-free correctly rounded cr_sqrt over its
// normal domain (every massive daughter), the IEEE routine otherwise.
__device__ __forceinline__ double frame_mass(double fe, double fx, double fy, double fz) {
  const double m2 = fe * fe - fx * fx - fy * fy - fz * fz;
  return m2 > 1e-300 && m2 < 1e300 ? cr_sqrt(m2) : sqrt(max0(m2));
}

// frame_mass for a daughter this kernel generated itself (fused chain): its
// m2 is finite, below M^2 < 1e300, and either >= ~ulp(GeV^2) or <= 0, so
// sqrt_lambda's sign mask + cr_sqrt (sqrt(+0) = +0) is the same correctly
// rounded value with no FP64 compares and no slow-path branch.
__device__ __forceinline__ double gen_frame_mass(double fe, double fx, double fy, double fz) {
  return sqrt_lambda(fe * fe - fx * fx - fy * fy - fz * fz);
}

__device__ __forceinline__ bool mass_mismatch(double fm, double M) {
  const double tol = 1e-9 * (M > 1e-6 ? M : 1e-6);  // MASS_TOLERANCE * max(M, 1e-6)
  return fabs(fm - M) > tol;                         // NaN compares false, as in numpy
}

template <int NS, int MODE>
__global__ void __launch_bounds__(kBlock) k_chain(const __grid_constant__ ChainArgs a) {
  const int64_t chunks = (a.count + HK_CHUNK - 1) / HK_CHUNK;
  TwoBody tb{};
  if constexpr (NS == 2) tb = two_body_consts(a.sub);
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
#pragma unroll 1
    for (int i = 0; i < kRowsPerThread; ++i) {
      const int64_t r = c * HK_CHUNK + i * kBlock + threadIdx.x;
      if (r >= a.count) continue;
      const uint64_t row = a.ev_begin + (uint64_t)r;
      const double fe = __ldg(a.p4_in[0] + r), fx = __ldg(a.p4_in[1] + r);
      const double fy = __ldg(a.p4_in[2] + r), fz = __ldg(a.p4_in[3] + r);
      const double fm = frame_mass(fe, fx, fy, fz);
      if (mass_mismatch(fm, a.sub.mother_mass)) record_bad(a.first_bad, row);
      double q[4 * NS];
      double ws;
      if constexpr (NS == 2)
        ws = rest_event2<MODE>(tb, a.rp, row, q);
      else
        ws = rest_event<NS, MODE>(a.sub, a.rp, row, q);
      const Frame f = make_frame_fast(fe, fx, fy, fz, fm);
#pragma unroll
      for (int s = 0; s < NS; ++s) boost_fma(f, q[4 * s], q[4 * s + 1], q[4 * s + 2], q[4 * s + 3]);
      __stcs(a.w_out + r, __ldg(a.w_in + r) * ws);
#pragma unroll
      for (int j = 0; j < 4 * NS; ++j) __stcs(a.sub_cols[j] + r, q[j]);
    }
  }
}

struct GenChainArgs {
  hk_decay_t d;
  hk_decay_t sub;
  RngParams rp;
  RngParams rp_sub;
  int32_t k;  // 0-based daughter that decays
  uint64_t ev_begin;
  int64_t count;
  double* cols[kMaxCols];  // spliced schema order
  double* wpart;
  unsigned long long* first_bad;
  // fixed-frame path (host-proved, see hk_phsp_generate_chain): the decaying
  // daughter's mass m_k and 1/m_k replace its per-event frame mass
  double fixed_m, fixed_im;
};

// Parent daughters other than the decaying one go to their spliced slots.
// Compile-time recursion over J keeps p[] in registers (a runtime-trip loop
// with a skip made nvcc demote p[] to local memory).
template <int J, int N, int NS>
__device__ __forceinline__ void store_parent_daughters(const GenChainArgs& a, int k,
                                                       const double (&p)[4 * N], int64_t r) {
  if constexpr (J < N) {
    if (J != k) {
      const int slot = 1 + 4 * (J < k ? J : J + NS - 1);
      __stcs(a.cols[slot + 0] + r, p[4 * J + 0]);
      __stcs(a.cols[slot + 1] + r, p[4 * J + 1]);
      __stcs(a.cols[slot + 2] + r, p[4 * J + 2]);
      __stcs(a.cols[slot + 3] + r, p[4 * J + 3]);
    }
    store_parent_daughters<J + 1, N, NS>(a, k, p, r);
  }
}

// Fused phsp_generate + phsp_decay_chain (config C3): only the 4(n-1+n_sub)+1
// final-state columns ever touch HBM.
//
// One fused chain event (generation, decay of daughter k, splice-ordered
// stores); returns the event weight.  Branch-free apart from the moving-mother
// test so two calls interleave; a mass mismatch lowers *bad to the row.
// K >= 0: the decaying daughter as a compile-time index (the hot 3-body
// parent), so its four-vector is a register reference instead of a select chain.
template <int N, int NS, int MODE, int K, bool FIXED>
__device__ __forceinline__ double chain_row(const GenChainArgs& a, const Frame& mf, const TwoBody& tb,
                                            const RestHoist& hp, int64_t r, unsigned long long* bad) {
  const int k = K >= 0 ? K : a.k;
  const uint64_t row = a.ev_begin + (uint64_t)r;
  double p[4 * N];
  const double wp = rest_event<N, MODE>(a.d, a.rp, row, p, hp);
  if (a.d.moving) {
#pragma unroll
    for (int j = 0; j < N; ++j) boost_fma(mf, p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
  }
  // daughter k's four-momentum; selp in asm so the front end cannot turn the
  // select chain back into p[4k] (which demotes p[] to local memory)
  double fe = 0.0, fx = 0.0, fy = 0.0, fz = 0.0;
  if constexpr (K >= 0) {
    fe = p[4 * K];
    fx = p[4 * K + 1];
    fy = p[4 * K + 2];
    fz = p[4 * K + 3];
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const bool sel = j == k;
      fe = select_f64(sel, p[4 * j], fe);
      fx = select_f64(sel, p[4 * j + 1], fx);
      fy = select_f64(sel, p[4 * j + 2], fy);
      fz = select_f64(sel, p[4 * j + 3], fz);
    }
  }
  double q[4 * NS];
  double ws;
  if constexpr (FIXED) {
    // frame mass = m_k (host-proved within the tolerance, no per-event check)
    const MFrame f{fe, fx, fy, fz, a.fixed_im, fast_rcp(fe + a.fixed_m)};
    if constexpr (NS == 2) {
      ws = two_body_boosted<MODE>(tb, a.rp_sub, row, f, q);
    } else {
      ws = rest_event<NS, MODE>(a.sub, a.rp_sub, row, q);
#pragma unroll
      for (int s = 0; s < NS; ++s) boost_m(f, q[4 * s], q[4 * s + 1], q[4 * s + 2], q[4 * s + 3]);
    }
  } else {
    const double fm = gen_frame_mass(fe, fx, fy, fz);
    *bad = mass_mismatch(fm, a.sub.mother_mass) ? min(*bad, (unsigned long long)row) : *bad;
    if constexpr (NS == 2)
      ws = rest_event2<MODE>(tb, a.rp_sub, row, q);  // per-launch constants hoisted, same bits
    else
      ws = rest_event<NS, MODE>(a.sub, a.rp_sub, row, q);
    const Frame f = make_frame_fast(fe, fx, fy, fz, fm);
#pragma unroll
    for (int s = 0; s < NS; ++s) boost_fma(f, q[4 * s], q[4 * s + 1], q[4 * s + 2], q[4 * s + 3]);
  }
  const double w = wp * ws;
  __stcs(a.cols[0] + r, w);
  store_parent_daughters<0, N, NS>(a, k, p, r);
  const int sbase = 1 + 4 * k;
#pragma unroll
  for (int j = 0; j < 4 * NS; ++j) __stcs(a.cols[sbase + j] + r, q[j]);
  return w;
}

// chain kernel shape: events per thread iteration (ILP) and CTAs per SM
#ifndef HK_CHAIN_ILP
#define HK_CHAIN_ILP 2
#endif
#ifndef HK_CHAIN_MINB
#define HK_CHAIN_MINB 2
#endif

// (Adjacent-row pairing with one double2 store per column, as in k_generate,
// measured no faster here -- 4.23 vs 4.20 ms per 1.25e8 C3 events: holding
// both events' 17 outputs for the paired stores spills 64 B at 128 registers.)
// HK_CHAIN_T threads per CTA, kBlock / HK_CHAIN_T CTAs per chunk through a
// virtual thread id (rows and weight slots unchanged), as in k_generate:
// 64 measured 3.576 ms per 1.25e8 C3 events against 3.592 for 256 (same box).
#ifndef HK_CHAIN_T
#define HK_CHAIN_T 64
#endif
template <int N, int NS, int MODE, int K, bool FIXED>
__global__ void __launch_bounds__(HK_CHAIN_T, HK_CHAIN_MINB * (kBlock / HK_CHAIN_T))
    k_generate_chain(const __grid_constant__ GenChainArgs a) {
  constexpr int kSplit = kBlock / HK_CHAIN_T;
  const int64_t chunks = (a.count + HK_CHUNK - 1) / HK_CHUNK;
  Frame mf{};
  if (a.d.moving) mf = make_frame(a.d.mother[0], a.d.mother[1], a.d.mother[2], a.d.mother[3],
                                  a.d.m_mother);
  unsigned long long bad = ~0ull;
  TwoBody tb{};
  if constexpr (NS == 2) tb = two_body_consts(a.sub);
  const RestHoist hp = rest_hoist<N>(a.d);
  for (int64_t u = blockIdx.x; u < chunks * kSplit; u += gridDim.x) {
    const int64_t c = u / kSplit;
    const int vt = (int)(u % kSplit) * HK_CHAIN_T + (int)threadIdx.x;
    double acc[2] = {0.0, 0.0};
    if (HK_CHAIN_ILP == 2 && N + NS <= 5 && c * HK_CHUNK + HK_CHUNK <= a.count) {
#pragma unroll 1
      for (int i = 0; i < kRowsPerThread / 2; ++i) {  // two events per iteration (ILP 2)
        const int64_t r0 = c * HK_CHUNK + i * kBlock + vt;
        const double w0 = chain_row<N, NS, MODE, K, FIXED>(a, mf, tb, hp, r0, &bad);
        const double w1 = chain_row<N, NS, MODE, K, FIXED>(a, mf, tb, hp, r0 + HK_CHUNK / 2, &bad);
        acc[0] += w0;
        acc[1] += w0 * w0;
        acc[0] += w1;
        acc[1] += w1 * w1;
      }
    } else {
#pragma unroll 1
      for (int i = 0; i < kRowsPerThread; ++i) {
        const int64_t r = c * HK_CHUNK + i * kBlock + vt;
        if (r < a.count) {
          const double w = chain_row<N, NS, MODE, K, FIXED>(a, mf, tb, hp, r, &bad);
          acc[0] += w;
          acc[1] += w * w;
        }
      }
    }
    if (a.wpart) warp_sum_store<2>(acc, a.wpart, c, vt >> 5);
  }
  if (bad != ~0ull) record_bad(a.first_bad, bad);
}

// ------------------------------------------------------------ unweighting --
struct UnwArgs {
  const double* w;
  int64_t n;
  double w_max;
  RngParams rp;
  uint64_t ev_begin;
  uint8_t* flags;
  long long* counts;
  unsigned long long* first_bad;
};

__global__ void __launch_bounds__(kBlock) k_unweight_flags(const __grid_constant__ UnwArgs a) {
  const int64_t chunks = (a.n + HK_CHUNK - 1) / HK_CHUNK;
  __shared__ int sm[kBlock / 32];
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    int cnt = 0;
    for (int i = 0; i < kRowsPerThread; ++i) {
      const int64_t r = c * HK_CHUNK + i * kBlock + threadIdx.x;
      if (r < a.n) {
        const uint64_t row = a.ev_begin + (uint64_t)r;
        const double w = __ldg(a.w + r);
        if (w > a.w_max) record_bad(a.first_bad, row);
        // uniform at counter row + key.counter (phasespace.py:226)
        const double u = to_unit(mix64(a.rp.base + (row + a.rp.kc) * kGolden) >> 11);
        const bool acc = u * a.w_max < w;
        a.flags[r] = acc ? 1 : 0;
        cnt += acc ? 1 : 0;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, off);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long s = 0;
      for (int k = 0; k < kBlock / 32; ++k) s += sm[k];
      a.counts[c] = s;
    }
    __syncthreads();
  }
}

// exclusive scan of per-chunk counts by one CTA of 1024 threads
__global__ void __launch_bounds__(1024) k_scan_counts(const long long* in, int64_t n,
                                                      long long* out, long long* total) {
  __shared__ long long sm[1024];
  const int t = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t lo = t * per, hi = lo + per < n ? lo + per : n;
  long long s = 0;
  for (int64_t i = lo; i < hi; ++i) s += in[i];
  sm[t] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // Hillis-Steele inclusive scan
    long long v = t >= off ? sm[t - off] : 0;
    __syncthreads();
    sm[t] += v;
    __syncthreads();
  }
  long long run = t == 0 ? 0 : sm[t - 1];
  for (int64_t i = lo; i < hi; ++i) {
    out[i] = run;
    run += in[i];
  }
  if (t == 1023) *total = sm[1023];
}

#ifndef HK_COMPACT_GROUP
#define HK_COMPACT_GROUP 16  // columns per load group in k_compact (0: one column at a time)
#endif

struct CompactArgs {
  const double* in[kMaxCols];
  double* out[kMaxCols];
  int32_t n_cols;
  int32_t weight_col;
  int64_t n;
  const uint8_t* flags;
  const long long* offsets;
};

// Order-preserving compaction of one 4096-row chunk per CTA iteration, rows
// walked in the kernels' usual 256-row stripes (row c*4096 + i*256 + t), so
// every column load is a coalesced warp transaction and the accepted rows of
// a stripe are stored to consecutive addresses.  A row's destination is the
// chunk's offset + the accepted rows before it in (stripe, warp, lane)
// order: warp ballots per stripe, one 128-entry exclusive scan per chunk.
__global__ void __launch_bounds__(kBlock) k_compact(const __grid_constant__ CompactArgs a) {
  constexpr int kWarps = kBlock / 32;
  const int64_t chunks = (a.n + HK_CHUNK - 1) / HK_CHUNK;
  __shared__ int s_pre[kRowsPerThread * kWarps];  // (stripe, warp) counts, then their exclusive scan
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int64_t c0 = c * HK_CHUNK + threadIdx.x;
    unsigned bits = 0;
#pragma unroll
    for (int i = 0; i < kRowsPerThread; ++i) {
      const int64_t r = c0 + i * kBlock;
      const bool f = r < a.n && a.flags[r];
      bits |= (unsigned)f << i;
      const unsigned m = __ballot_sync(0xffffffffu, f);
      if (lane == 0) s_pre[i * kWarps + warp] = __popc(m);
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 128 counts: 4 consecutive entries per lane
      constexpr int kPer = kRowsPerThread * kWarps / 32;
      int v[kPer], tot = 0;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        v[k] = s_pre[lane * kPer + k];
        tot += v[k];
      }
      int inc = tot;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += y;
      }
      int run = inc - tot;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        s_pre[lane * kPer + k] = run;
        run += v[k];
      }
    }
    __syncthreads();
    const int64_t base = a.offsets[c];
#pragma unroll 1
    for (int i = 0; i < kRowsPerThread; ++i) {
      const bool f = (bits >> i) & 1u;
      const unsigned m = __ballot_sync(0xffffffffu, f);
      if (f) {
        const int64_t dst = base + s_pre[i * kWarps + warp] + __popc(m & lt);
        const int64_t r = c0 + i * kBlock;
#if HK_COMPACT_GROUP > 0
        // a group of columns loaded before any is stored: the outputs may
        // alias the inputs as far as the compiler knows, so a load-store
        // loop would wait one memory latency per column
        for (int g = 0; g < a.n_cols; g += HK_COMPACT_GROUP) {
          double v[HK_COMPACT_GROUP];
#pragma unroll
          for (int k = 0; k < HK_COMPACT_GROUP; ++k) {
            const int col = g + k;
            if (col < a.n_cols) v[k] = col == a.weight_col ? 1.0 : __ldcs(a.in[col] + r);
          }
#pragma unroll
          for (int k = 0; k < HK_COMPACT_GROUP; ++k)
            if (g + k < a.n_cols) a.out[g + k][dst] = v[k];
        }
#else
        for (int col = 0; col < a.n_cols; ++col)
          a.out[col][dst] = col == a.weight_col ? 1.0 : __ldcs(a.in[col] + r);
#endif
      }
    }
    __syncthreads();
  }
}

// -------------------------------------------------------------------- RNG --
__global__ void k_rng(RngParams rp, const uint64_t* ctr, int64_t n, uint64_t* raw, double* uni) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t c = ctr[i] + rp.kc;
  uint64_t bits;
  if (rp.mode == HK_RNG_REFERENCE) {
    const uint64_t r = mix64(rp.base + c * kGolden);
    if (raw) raw[i] = r;
    bits = r >> 11;
  } else {
    const Philox4 o = philox4x32_10_rk((uint32_t)c, (uint32_t)(c >> 32), 0u, kPhiloxTag, rp.rk);
    const uint64_t r = ((uint64_t)o.v[0] << 32) | o.v[1];
    if (raw) raw[i] = r;
    bits = r >> 11;
  }
  if (uni) uni[i] = to_unit(bits);
}

// Raw Philox4x32-10 blocks on (ctr[4], key[2]) rows -- the same device round
// function the production stream uses, exposed for known-answer tests.
__global__ void k_philox_rows(const uint32_t* in6, int64_t n, uint32_t* out4) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* r = in6 + 6 * i;
  const Philox4 o = philox4x32_10(r[0], r[1], r[2], r[3], r[4], r[5]);
  for (int k = 0; k < 4; ++k) out4[4 * i + k] = o.v[k];
}

// ----------------------------------------------------------------- folds ---
// Deterministic fold over one thread-block cluster of kFoldCtas CTAs: global
// thread g sums parts g, g + 8192, ... in order, a fixed shuffle/smem tree
// per CTA, then CTA 0 adds the CTAs' sums in rank order through distributed
// shared memory.  One launch, no global scratch, 8 SMs of load bandwidth;
// same n_parts -> same bits, whatever produced them.
constexpr int kFoldCtas = 8;  // portable cluster size
constexpr int kFoldThreads = 1024;
// widest record folded: the ratio sums of HK_MAX_COMPONENTS species, K + K^2
constexpr int kFoldMaxWidth = HK_MAX_COMPONENTS + HK_MAX_COMPONENTS * HK_MAX_COMPONENTS;

__global__ void __cluster_dims__(kFoldCtas, 1, 1) __launch_bounds__(kFoldThreads)
    k_fold(const double* parts, int64_t n, int width, double* out) {
  __shared__ double sm[32][kFoldMaxWidth];  // [warp][w]
  __shared__ double cta_sum[kFoldMaxWidth];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t g = (int64_t)rank * kFoldThreads + threadIdx.x;
  constexpr int64_t stride = (int64_t)kFoldCtas * kFoldThreads;
  for (int w = 0; w < width; ++w) {
    double s = 0.0;
#pragma unroll 4
    for (int64_t i = g; i < n; i += stride) s += __ldg(parts + i * width + w);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) sm[warp][w] = s;
  }
  __syncthreads();
  if (threadIdx.x < width) {
    double s = sm[0][threadIdx.x];
    for (int k = 1; k < 32; ++k) s += sm[k][threadIdx.x];
    cta_sum[threadIdx.x] = s;
  }
  cl.sync();
  if (rank == 0 && threadIdx.x < width) {
    double s = cta_sum[threadIdx.x];
    for (int r = 1; r < kFoldCtas; ++r) s += cl.map_shared_rank(cta_sum, r)[threadIdx.x];
    out[threadIdx.x] = s;
  }
  cl.sync();  // remote shared memory stays live until CTA 0 has read it
}

int launch_fold(const double* parts, int64_t n, int width, double* out, cudaStream_t st) {
  k_fold<<<kFoldCtas, kFoldThreads, 0, st>>>(parts, n, width, out);
  return check_launch("k_fold");
}

// Per-segment fold in fixed order: out[s][w] = sum_j parts[s * seg_len + j][w],
// j ascending -- e.g. a chunk's 8 warp-slice weight partials into one chunk
// partial, so that only per-chunk records cross GPUs (8x fewer bytes) and the
// global fold sees the same chunk sequence at any GPU count.
__global__ void __launch_bounds__(256) k_fold_segments(const double* __restrict__ parts, int64_t n_seg,
                                                       int seg_len, int width, double* __restrict__ out) {
  const int64_t i = blockIdx.x * 256ll + threadIdx.x;
  if (i >= n_seg * width) return;
  const int64_t s = i / width;
  const int w = (int)(i - s * width);
  const double* p = parts + s * seg_len * width + w;
  double acc = __ldg(p);
  for (int j = 1; j < seg_len; ++j) acc += __ldg(p + (int64_t)j * width);
  out[i] = acc;
}

int launch_fold_segments(const double* parts, int64_t n_seg, int seg_len, int width, double* out,
                         cudaStream_t st) {
  if (n_seg <= 0) return HK_OK;
  const int64_t threads = n_seg * width;
  k_fold_segments<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(parts, n_seg, seg_len, width, out);
  return check_launch("k_fold_segments");
}

// Super-chunk fold (SURVEY.md 8(e) option ii).  The global chunk sequence of
// a run (nch chunks) is cut into HK_SUPERS fixed super-chunks, super s
// covering global chunks [s nch / S, (s+1) nch / S) (floor).  GPU shards are
// whole runs of supers, so every super is folded by exactly one rank from the
// same records in the same order -- whatever the GPU count -- and only
// S x width doubles cross GPUs (40 KB for the 5-wide averages).  One warp per
// super: lane l sums records l, l + 32, ... in order, then a fixed shuffle
// tree.  The local partial array holds recs records (of `width` doubles) per
// chunk for global chunks [c0, c0 + nloc), and this launch writes supers
// [s0, s0 + s_count) (which the caller checks lie inside that range).
__global__ void __launch_bounds__(256) k_fold_supers(const double* __restrict__ parts, int64_t nch,
                                                     int64_t c0, int recs, int width, int n_super,
                                                     int s0, int s_count, double* __restrict__ out) {
  const int sl = (int)((blockIdx.x * 256ll + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (sl >= s_count) return;
  const int64_t s = s0 + sl;
  const int64_t a = (s * nch / n_super - c0) * recs;
  const int64_t b = ((s + 1) * nch / n_super - c0) * recs;
  for (int w = 0; w < width; ++w) {
    double acc = 0.0;
    for (int64_t j = a + lane; j < b; j += 32) acc += __ldg(parts + j * width + w);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
    if (lane == 0) out[(int64_t)sl * width + w] = acc;
  }
}

// ------------------------------------------------------ launch dispatch ----
template <int MODE>
int dispatch_generate(const GenArgs& a, unsigned grid, cudaStream_t st) {
  const unsigned grid_t = chunk_grid(num_chunks(a.count) * (kBlock / HK_GEN_T));
  switch (a.d.n) {
#define HK_GEN_CASE(NN)                                              \
  case NN:                                                           \
    if (NN <= 4 && a.vec2)                                           \
      k_generate<NN, MODE, (NN <= 4), HK_GEN_T>                      \
          <<<grid_t, HK_GEN_T, 0, st>>>(a);                          \
    else                                                             \
      k_generate<NN, MODE, false><<<grid, kBlock, 0, st>>>(a);       \
    break;
    HK_GEN_CASE(2)
    HK_GEN_CASE(3)
    HK_GEN_CASE(4)
    HK_GEN_CASE(5)
    HK_GEN_CASE(6)
    HK_GEN_CASE(7)
    HK_GEN_CASE(8)
#undef HK_GEN_CASE
    default: k_generate_rt<MODE><<<grid, kBlock, 0, st>>>(a); break;
  }
  return check_launch("k_generate");
}

template <int MODE>
int dispatch_integrate(const IntArgs& a, unsigned grid, cudaStream_t st) {
  switch (a.d.n) {
#define HK_INT_CASE(NN)                                                  \
  case NN:                                                               \
    if (a.pair.kind != HK_PAIR_NONE)                                     \
      k_integrate<NN, MODE, true><<<grid, kBlock, 0, st>>>(a);           \
    else                                                                 \
      k_integrate<NN, MODE, false><<<grid, kBlock, 0, st>>>(a);          \
    break;
    HK_INT_CASE(2)
    HK_INT_CASE(3)
    HK_INT_CASE(4)
    HK_INT_CASE(5)
    HK_INT_CASE(6)
    HK_INT_CASE(7)
    HK_INT_CASE(8)
#undef HK_INT_CASE
    default:
      set_error("fused integration supports 2..%d daughters, got %d", kFastMaxN, a.d.n);
      return HK_EUNSUPPORTED;
  }
  return check_launch("k_integrate");
}

template <int MODE>
int dispatch_chain(const ChainArgs& a, unsigned grid, cudaStream_t st) {
  switch (a.sub.n) {
#define HK_CH_CASE(NN) \
  case NN: k_chain<NN, MODE><<<grid, kBlock, 0, st>>>(a); break;
    HK_CH_CASE(2)
    HK_CH_CASE(3)
    HK_CH_CASE(4)
    HK_CH_CASE(5)
    HK_CH_CASE(6)
    HK_CH_CASE(7)
    HK_CH_CASE(8)
#undef HK_CH_CASE
    default:
      set_error("decay chain supports 2..%d sub-daughters, got %d", kFastMaxN, a.sub.n);
      return HK_EUNSUPPORTED;
  }
  return check_launch("k_chain");
}

// (A compile-time decaying-daughter index for 3-body parents -- no select
// chain -- measured no faster on B200: 4.63 vs 4.56 ms per 1.25e8 C3 events.)
template <int N, int NS, int MODE>
void launch_gen_chain(const GenChainArgs& a, unsigned grid, cudaStream_t st) {
  (void)grid;
  const unsigned g = chunk_grid(num_chunks(a.count) * (kBlock / HK_CHAIN_T));
  if (a.fixed_m > 0.0)
    k_generate_chain<N, NS, MODE, -1, true><<<g, HK_CHAIN_T, 0, st>>>(a);
  else
    k_generate_chain<N, NS, MODE, -1, false><<<g, HK_CHAIN_T, 0, st>>>(a);
}

template <int MODE, int N>
int dispatch_gen_chain_sub(const GenChainArgs& a, unsigned grid, cudaStream_t st) {
  switch (a.sub.n) {
    case 2: launch_gen_chain<N, 2, MODE>(a, grid, st); break;
    case 3: launch_gen_chain<N, 3, MODE>(a, grid, st); break;
    case 4: launch_gen_chain<N, 4, MODE>(a, grid, st); break;
    default:
      set_error("fused chain supports 2..4 sub-daughters, got %d", a.sub.n);
      return HK_EUNSUPPORTED;
  }
  return check_launch("k_generate_chain");
}

template <int MODE>
int dispatch_gen_chain(const GenChainArgs& a, unsigned grid, cudaStream_t st) {
  switch (a.d.n) {
    case 2: return dispatch_gen_chain_sub<MODE, 2>(a, grid, st);
    case 3: return dispatch_gen_chain_sub<MODE, 3>(a, grid, st);
    case 4: return dispatch_gen_chain_sub<MODE, 4>(a, grid, st);
    case 5: return dispatch_gen_chain_sub<MODE, 5>(a, grid, st);
    case 6: return dispatch_gen_chain_sub<MODE, 6>(a, grid, st);
    default:
      set_error("fused chain supports 2..6 parent daughters, got %d", a.d.n);
      return HK_EUNSUPPORTED;
  }
}

int validate_decay(const hk_decay_t* d, const char* what) {
  HK_REQUIRE(d != nullptr, "%s: NULL decay", what);
  HK_REQUIRE(d->n >= 2 && d->n <= HK_MAX_DAUGHTERS, "%s: daughter count %d outside 2..%d", what,
             d->n, HK_MAX_DAUGHTERS);
  return HK_OK;
}

int validate_key(const hk_key_t* k, const char* what) {
  HK_REQUIRE(k != nullptr, "%s: NULL key", what);
  HK_REQUIRE(k->mode == HK_RNG_REFERENCE || k->mode == HK_RNG_PHILOX, "%s: bad rng mode %d", what,
             k->mode);
  return HK_OK;
}

int validate_program(const hk_program_t* f, int n_cols) {
  HK_REQUIRE(f != nullptr, "NULL program");
  HK_REQUIRE(f->n_ops >= 1 && f->n_ops <= HK_MAX_PROGRAM, "program length %d", f->n_ops);
  HK_REQUIRE(f->result >= 0 && f->result < HK_MAX_SLOTS, "program result slot %d", f->result);
  for (int i = 0; i < f->n_ops; ++i) {
    HK_REQUIRE(f->op[i] >= HK_OP_COL && f->op[i] <= HK_OP_UDIV, "op %d: bad opcode %d", i,
               f->op[i]);
    HK_REQUIRE(f->dst[i] >= 0 && f->dst[i] < HK_MAX_SLOTS, "op %d: bad dst", i);
    if (f->op[i] == HK_OP_COL) {
      HK_REQUIRE(f->a[i] >= 0 && f->a[i] < n_cols, "op %d: column %d outside 0..%d", i, f->a[i],
                 n_cols - 1);
    } else if (f->op[i] != HK_OP_CONST) {
      HK_REQUIRE(f->a[i] >= 0 && f->a[i] < HK_MAX_SLOTS, "op %d: bad slot a", i);
      HK_REQUIRE(f->b[i] >= 0 && f->b[i] < HK_MAX_SLOTS, "op %d: bad slot b", i);
    }
  }
  return HK_OK;
}

}  // namespace hk

using namespace hk;

extern "C" {

int64_t hk_num_chunks(int64_t ev_count) { return num_chunks(ev_count); }

int hk_rng_raw64(const hk_key_t* key, const uint64_t* d_counters, int64_t n, uint64_t* d_out,
                 void* stream) {
  HK_NVTX("hk_rng_raw64");
  if (int rc = validate_key(key, "hk_rng_raw64")) return rc;
  HK_REQUIRE(n >= 0, "negative n");
  if (n == 0) return HK_OK;
  HK_REQUIRE(d_counters && d_out, "NULL pointer");
  k_rng<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(make_rng(*key), d_counters, n,
                                                                    d_out, nullptr);
  return check_launch("k_rng");
}

int hk_philox4x32_10(const uint32_t* d_ctr_key, int64_t n, uint32_t* d_out, void* stream) {
  HK_REQUIRE(n >= 0, "negative n");
  if (n == 0) return HK_OK;
  HK_REQUIRE(d_ctr_key && d_out, "NULL pointer");
  k_philox_rows<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(d_ctr_key, n, d_out);
  return check_launch("k_philox_rows");
}

int hk_rng_uniform(const hk_key_t* key, const uint64_t* d_counters, int64_t n, double* d_out,
                   void* stream) {
  HK_NVTX("hk_rng_uniform");
  if (int rc = validate_key(key, "hk_rng_uniform")) return rc;
  HK_REQUIRE(n >= 0, "negative n");
  if (n == 0) return HK_OK;
  HK_REQUIRE(d_counters && d_out, "NULL pointer");
  k_rng<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(make_rng(*key), d_counters, n,
                                                                    nullptr, d_out);
  return check_launch("k_rng");
}

int hk_phsp_generate(const hk_decay_t* spec, const hk_key_t* key, uint64_t ev_begin,
                     int64_t ev_count, double* const* d_cols, double* d_wpartials, void* stream) {
  HK_NVTX("hk_phsp_generate");
  if (int rc = validate_decay(spec, "hk_phsp_generate")) return rc;
  if (int rc = validate_key(key, "hk_phsp_generate")) return rc;
  HK_REQUIRE(ev_count >= 0, "negative ev_count");
  if (ev_count == 0) return HK_OK;
  GenArgs a;
  std::memset(&a, 0, sizeof(a));
  a.d = *spec;
  a.rp = make_rng(*key);
  a.ev_begin = ev_begin;
  a.count = ev_count;
  a.wpart = d_wpartials;
  a.store = d_cols != nullptr;
  if (d_cols) {
    a.vec2 = 1;
    for (int j = 0; j < 4 * spec->n + 1; ++j) {
      HK_REQUIRE(d_cols[j] != nullptr, "column %d is NULL", j);
      a.cols[j] = d_cols[j];
      if (reinterpret_cast<uintptr_t>(d_cols[j]) % 16) a.vec2 = 0;
    }
  }
  HK_REQUIRE(a.store || a.wpart, "nothing to write (no columns, no partials)");
  const unsigned grid = chunk_grid(num_chunks(ev_count));
  cudaStream_t st = as_stream(stream);
  return key->mode == HK_RNG_REFERENCE ? dispatch_generate<HK_RNG_REFERENCE>(a, grid, st)
                                       : dispatch_generate<HK_RNG_PHILOX>(a, grid, st);
}

int hk_phsp_decay_chain(const double* d_w_in, const double* const* d_p4_in,
                        const hk_decay_t* sub, const hk_key_t* sub_key, uint64_t ev_begin,
                        int64_t ev_count, double* d_w_out, double* const* d_sub_cols,
                        uint64_t* d_first_bad, void* stream) {
  HK_NVTX("hk_phsp_decay_chain");
  if (int rc = validate_decay(sub, "hk_phsp_decay_chain")) return rc;
  if (int rc = validate_key(sub_key, "hk_phsp_decay_chain")) return rc;
  HK_REQUIRE(ev_count >= 0, "negative ev_count");
  if (ev_count == 0) return HK_OK;
  HK_REQUIRE(d_w_in && d_p4_in && d_w_out && d_sub_cols, "NULL pointer");
  ChainArgs a;
  std::memset(&a, 0, sizeof(a));
  a.sub = *sub;
  a.rp = make_rng(*sub_key);
  a.ev_begin = ev_begin;
  a.count = ev_count;
  a.w_in = d_w_in;
  for (int c = 0; c < 4; ++c) {
    HK_REQUIRE(d_p4_in[c], "input column %d NULL", c);
    a.p4_in[c] = d_p4_in[c];
  }
  a.w_out = d_w_out;
  for (int j = 0; j < 4 * sub->n; ++j) {
    HK_REQUIRE(d_sub_cols[j], "sub column %d NULL", j);
    a.sub_cols[j] = d_sub_cols[j];
  }
  a.first_bad = reinterpret_cast<unsigned long long*>(d_first_bad);
  const unsigned grid = chunk_grid(num_chunks(ev_count));
  cudaStream_t st = as_stream(stream);
  return sub_key->mode == HK_RNG_REFERENCE ? dispatch_chain<HK_RNG_REFERENCE>(a, grid, st)
                                           : dispatch_chain<HK_RNG_PHILOX>(a, grid, st);
}

// When may the fused chain use the decaying daughter's mass m_k as its frame
// mass instead of recomputing sqrt(E^2 - p^2) per event (phasespace.py:259-262)?
// The daughter is generated with mass m_k, so the recomputed mass differs from
// m_k only by the rounding of E^2 - p^2: relative error <= ~8 ulp * gamma^2
// (E^2 and p^2 each carry a few ulp of E^2 = gamma^2 m^2).  Returns m_k (fast
// path) when, over the whole phase space, that error is below 1e-14 (gamma <=
// 4; boosted momenta then move by <~1e-14 * E, the parity budget being 1e-12 * E)
// and m_k is within a quarter of the mismatch tolerance of the sub-decay
// mother mass, so no event can fail the reference's per-event check; else 0
// (the per-event path with the check).
//   gamma bound: E_k <= (M^2 + m_k^2 - (sum of the other masses)^2) / (2M) in the
//   mother frame; a moving mother multiplies gamma by at most 2 gamma_mother.
double fixed_frame_mass(const hk_decay_t& d, int k, const hk_decay_t& sub) {
  const double mk = d.masses[k], M = d.mother_mass;
  if (!(mk > 0.0) || !std::isfinite(mk) || !(M > 0.0) || !std::isfinite(M)) return 0.0;
  const double tol = 1e-9 * (sub.mother_mass > 1e-6 ? sub.mother_mass : 1e-6);
  if (!(std::fabs(mk - sub.mother_mass) <= 0.25 * tol)) return 0.0;
  double others = 0.0;
  for (int j = 0; j < d.n; ++j)
    if (j != k) others += d.masses[j];
  const double e_max = (M * M + mk * mk - others * others) / (2.0 * M);
  double gamma = e_max / mk;
  if (d.moving) gamma *= 2.0 * (d.mother[0] / d.m_mother);  // NaN / inf fail the test below
  if (!(gamma >= 1.0 - 1e-12) || !(gamma <= 4.0)) return 0.0;
  return mk;
}

double hk_chain_fixed_frame_mass(const hk_decay_t* spec, int32_t daughter_index, const hk_decay_t* sub) {
  if (!spec || !sub || daughter_index < 1 || daughter_index > spec->n || spec->n > HK_MAX_DAUGHTERS) return 0.0;
  return fixed_frame_mass(*spec, daughter_index - 1, *sub);
}

int hk_phsp_generate_chain(const hk_decay_t* spec, const hk_key_t* key, int32_t daughter_index,
                           const hk_decay_t* sub, const hk_key_t* sub_key, uint64_t ev_begin,
                           int64_t ev_count, double* const* d_cols, double* d_wpartials,
                           uint64_t* d_first_bad, void* stream) {
  HK_NVTX("hk_phsp_generate_chain");
  if (int rc = validate_decay(spec, "hk_phsp_generate_chain")) return rc;
  if (int rc = validate_decay(sub, "hk_phsp_generate_chain")) return rc;
  if (int rc = validate_key(key, "hk_phsp_generate_chain")) return rc;
  if (int rc = validate_key(sub_key, "hk_phsp_generate_chain")) return rc;
  HK_REQUIRE(key->mode == sub_key->mode, "parent and sub-decay keys must share an rng mode");
  HK_REQUIRE(daughter_index >= 1 && daughter_index <= spec->n, "daughter index %d out of range 1..%d",
             daughter_index, spec->n);
  HK_REQUIRE(ev_count >= 0, "negative ev_count");
  if (ev_count == 0) return HK_OK;
  HK_REQUIRE(d_cols != nullptr, "NULL columns");
  const int ncols = 4 * (spec->n - 1 + sub->n) + 1;
  HK_REQUIRE(ncols <= kMaxCols, "final state too large (%d columns)", ncols);
  GenChainArgs a;
  std::memset(&a, 0, sizeof(a));
  a.d = *spec;
  a.sub = *sub;
  a.rp = make_rng(*key);
  a.rp_sub = make_rng(*sub_key);
  a.k = daughter_index - 1;
  a.ev_begin = ev_begin;
  a.count = ev_count;
  for (int j = 0; j < ncols; ++j) {
    HK_REQUIRE(d_cols[j], "column %d NULL", j);
    a.cols[j] = d_cols[j];
  }
  a.wpart = d_wpartials;
  a.first_bad = reinterpret_cast<unsigned long long*>(d_first_bad);
  a.fixed_m = fixed_frame_mass(*spec, a.k, *sub);
  a.fixed_im = a.fixed_m > 0.0 ? 1.0 / a.fixed_m : 0.0;
  const unsigned grid = chunk_grid(num_chunks(ev_count));
  cudaStream_t st = as_stream(stream);
  return key->mode == HK_RNG_REFERENCE ? dispatch_gen_chain<HK_RNG_REFERENCE>(a, grid, st)
                                       : dispatch_gen_chain<HK_RNG_PHILOX>(a, grid, st);
}

int hk_phsp_moments(const double* const* d_cols, int32_t n_cols, int64_t ev_count,
                    const hk_program_t* f, double* d_partials, uint64_t* d_first_bad,
                    void* stream) {
  HK_NVTX("hk_phsp_moments");
  HK_REQUIRE(d_cols && n_cols >= 1 && n_cols <= kMaxCols, "bad columns (%d)", n_cols);
  if (int rc = validate_program(f, n_cols)) return rc;
  HK_REQUIRE(ev_count >= 0, "negative ev_count");
  if (ev_count == 0) return HK_OK;
  HK_REQUIRE(d_partials, "NULL partials");
  MomArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int c = 0; c < n_cols; ++c) {
    HK_REQUIRE(d_cols[c], "column %d NULL", c);
    a.cols[c] = d_cols[c];
  }
  a.n_cols = n_cols;
  a.count = ev_count;
  a.f = *f;
  a.part = d_partials;
  // d_first_bad[0] = first zero divisor, d_first_bad[1] = first non-finite f
  a.div0_bad = reinterpret_cast<unsigned long long*>(d_first_bad);
  a.nonfinite_bad = d_first_bad ? reinterpret_cast<unsigned long long*>(d_first_bad) + 1 : nullptr;
  const void* jit = nullptr;
  if (int rc = jit_kernel(*f, ev_count, kJitMoments, &jit)) return rc;
  if (jit) {  // specialised straight-line program (hk_jit.cu), bit-identical
    JitArgs j = jit_args(a);
    void* args[] = {&j};
    HK_CUDA(cudaLaunchKernel(jit, dim3(chunk_grid(num_chunks(ev_count))), dim3(kBlock), args, 0,
                             as_stream(stream)));
    return HK_OK;
  }
  k_moments<<<chunk_grid(num_chunks(ev_count)), kBlock, 0, as_stream(stream)>>>(a);
  return check_launch("k_moments");
}

int hk_map_program(const double* const* d_cols, int32_t n_cols, int64_t n, const hk_program_t* f,
                   double* d_out, uint64_t* d_first_bad, void* stream) {
  HK_NVTX("hk_map_program");
  HK_REQUIRE(d_cols && n_cols >= 1 && n_cols <= kMaxCols, "bad columns (%d)", n_cols);
  if (int rc = validate_program(f, n_cols)) return rc;
  HK_REQUIRE(n >= 0, "negative n");
  if (n == 0) return HK_OK;
  HK_REQUIRE(d_out, "NULL output");
  MomArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int c = 0; c < n_cols; ++c) {
    HK_REQUIRE(d_cols[c], "column %d NULL", c);
    a.cols[c] = d_cols[c];
  }
  a.n_cols = n_cols;
  a.count = n;
  a.f = *f;
  a.div0_bad = reinterpret_cast<unsigned long long*>(d_first_bad);
  const void* jit = nullptr;
  if (int rc = jit_kernel(*f, n, kJitMap, &jit)) return rc;
  if (jit) {
    JitArgs j = jit_args(a);
    j.out = d_out;
    void* args[] = {&j};
    HK_CUDA(cudaLaunchKernel(jit, dim3((unsigned)((n + kBlock - 1) / kBlock)), dim3(kBlock), args, 0,
                             as_stream(stream)));
    return HK_OK;
  }
  k_map<<<(unsigned)((n + kBlock - 1) / kBlock), kBlock, 0, as_stream(stream)>>>(a, d_out);
  return check_launch("k_map");
}

int hk_phsp_integrate(const hk_decay_t* spec, const hk_key_t* key, uint64_t ev_begin,
                      int64_t ev_count, const hk_program_t* f, const hk_pair_integrand_t* pair,
                      double* d_partials, uint64_t* d_first_bad, void* stream) {
  HK_NVTX("hk_phsp_integrate");
  if (int rc = validate_decay(spec, "hk_phsp_integrate")) return rc;
  if (int rc = validate_key(key, "hk_phsp_integrate")) return rc;
  const bool fast = pair && pair->kind != HK_PAIR_NONE;
  if (fast) {
    HK_REQUIRE(pair->kind == HK_PAIR_MASS2 || pair->kind == HK_PAIR_BW, "bad pair kind %d",
               pair->kind);
    HK_REQUIRE(pair->i >= 0 && pair->j >= 0 && pair->i < spec->n && pair->j < spec->n,
               "pair (%d, %d) outside the %d daughters", pair->i, pair->j, spec->n);
  } else if (int rc = validate_program(f, 4 * spec->n + 1)) {
    return rc;
  }
  HK_REQUIRE(ev_count >= 0, "negative ev_count");
  if (ev_count == 0) return HK_OK;
  HK_REQUIRE(d_partials, "NULL partials");
  IntArgs a;
  std::memset(&a, 0, sizeof(a));
  a.d = *spec;
  a.rp = make_rng(*key);
  a.ev_begin = ev_begin;
  a.count = ev_count;
  // a recognised pair integrand also arrives with its program (the Python
  // side always lowers it): the specialised kernel serves both
  const bool have_prog = f != nullptr && (!fast || validate_program(f, 4 * spec->n + 1) == HK_OK);
  if (fast) a.pair = *pair;
  if (have_prog) a.f = *f;
  a.part = d_partials;
  a.div0_bad = reinterpret_cast<unsigned long long*>(d_first_bad);
  a.nonfinite_bad = d_first_bad ? reinterpret_cast<unsigned long long*>(d_first_bad) + 1 : nullptr;
  const unsigned grid = chunk_grid(num_chunks(ev_count));
  cudaStream_t st = as_stream(stream);
  if (have_prog && spec->n <= kFastMaxN) {  // specialised generator + straight-line integrand (hk_jit.cu)
    const void* jit = nullptr;
    if (int rc = jit_integrate(*f, spec->n, key->mode, ev_count, &jit)) return rc;
    if (jit) {
      void* args[] = {&a};
      HK_CUDA(cudaLaunchKernel(jit, dim3(grid), dim3(kBlock), args, 0, st));
      return HK_OK;
    }
  }
  return key->mode == HK_RNG_REFERENCE ? dispatch_integrate<HK_RNG_REFERENCE>(a, grid, st)
                                       : dispatch_integrate<HK_RNG_PHILOX>(a, grid, st);
}

int hk_fold_segments(const double* d_partials, int64_t n_segments, int32_t seg_len, int32_t width,
                     double* d_out, void* stream) {
  HK_REQUIRE(width >= 1 && width <= 32 && seg_len >= 1 && seg_len <= 1024, "bad segment shape %d x %d",
             seg_len, width);
  HK_REQUIRE(n_segments >= 0, "negative segment count");
  HK_REQUIRE(n_segments == 0 || (d_partials && d_out), "NULL pointer");
  return launch_fold_segments(d_partials, n_segments, seg_len, width, d_out, as_stream(stream));
}

int hk_fold_supers(const double* d_partials, int64_t n_chunks_total, int64_t chunk_begin,
                   int64_t n_chunks_local, int32_t recs_per_chunk, int32_t width, int32_t s_begin,
                   int32_t s_count, double* d_out, void* stream) {
  HK_NVTX("hk_fold_supers");
  HK_REQUIRE(width >= 1 && width <= kFoldMaxWidth && recs_per_chunk >= 1 && recs_per_chunk <= 1024,
             "bad record shape %d x %d", recs_per_chunk, width);
  HK_REQUIRE(n_chunks_total >= 0 && chunk_begin >= 0 && n_chunks_local >= 0 &&
                 chunk_begin + n_chunks_local <= n_chunks_total,
             "chunk range [%lld, %lld) outside [0, %lld)", (long long)chunk_begin,
             (long long)(chunk_begin + n_chunks_local), (long long)n_chunks_total);
  HK_REQUIRE(s_begin >= 0 && s_count >= 0 && s_begin + s_count <= HK_SUPERS,
             "super range [%d, %d) outside [0, %d)", s_begin, s_begin + s_count, HK_SUPERS);
  if (s_count == 0) return HK_OK;
  // the supers must be exactly the local chunks (a rank folds only its own records)
  const int64_t first = (int64_t)s_begin * n_chunks_total / HK_SUPERS;
  const int64_t last = (int64_t)(s_begin + s_count) * n_chunks_total / HK_SUPERS;
  HK_REQUIRE(first == chunk_begin && last == chunk_begin + n_chunks_local,
             "supers [%d, %d) cover chunks [%lld, %lld), the partials hold [%lld, %lld)", s_begin,
             s_begin + s_count, (long long)first, (long long)last, (long long)chunk_begin,
             (long long)(chunk_begin + n_chunks_local));
  HK_REQUIRE(d_out && (n_chunks_local == 0 || d_partials), "NULL pointer");
  const unsigned grid = (unsigned)((s_count * 32 + 255) / 256);
  k_fold_supers<<<grid, 256, 0, as_stream(stream)>>>(d_partials, n_chunks_total, chunk_begin,
                                                     recs_per_chunk, width, HK_SUPERS, s_begin,
                                                     s_count, d_out);
  return check_launch("k_fold_supers");
}

int hk_fold_partials(const double* d_partials, int64_t n_parts, int32_t width, double* d_out,
                     void* stream) {
  HK_NVTX("hk_fold_partials");
  HK_REQUIRE(width >= 1 && width <= kFoldMaxWidth, "fold width %d outside 1..%d", width, kFoldMaxWidth);
  HK_REQUIRE(n_parts >= 0 && d_out, "bad fold arguments");
  HK_REQUIRE(n_parts == 0 || d_partials, "NULL partials");
  return launch_fold(d_partials, n_parts, width, d_out, as_stream(stream));
}

int hk_unweight_flags(const double* d_w, int64_t n, double w_max, const hk_key_t* key,
                      uint64_t ev_begin, uint8_t* d_flags, int64_t* d_counts,
                      uint64_t* d_first_bad, void* stream) {
  HK_NVTX("hk_unweight_flags");
  if (int rc = validate_key(key, "hk_unweight_flags")) return rc;
  HK_REQUIRE(key->mode == HK_RNG_REFERENCE, "unweighting uses the reference stream");
  HK_REQUIRE(n >= 0, "negative n");
  if (n == 0) return HK_OK;
  HK_REQUIRE(d_w && d_flags && d_counts, "NULL pointer");
  UnwArgs a;
  a.w = d_w;
  a.n = n;
  a.w_max = w_max;
  a.rp = make_rng(*key);
  a.ev_begin = ev_begin;
  a.flags = d_flags;
  a.counts = reinterpret_cast<long long*>(d_counts);
  a.first_bad = reinterpret_cast<unsigned long long*>(d_first_bad);
  k_unweight_flags<<<chunk_grid(num_chunks(n)), kBlock, 0, as_stream(stream)>>>(a);
  return check_launch("k_unweight_flags");
}

int hk_scan_counts(const int64_t* d_counts, int64_t n, int64_t* d_out, int64_t* d_total,
                   void* stream) {
  HK_REQUIRE(n >= 0 && d_total, "bad scan arguments");
  HK_REQUIRE(n == 0 || (d_counts && d_out), "NULL pointer");
  k_scan_counts<<<1, 1024, 0, as_stream(stream)>>>(reinterpret_cast<const long long*>(d_counts), n,
                                                   reinterpret_cast<long long*>(d_out),
                                                   reinterpret_cast<long long*>(d_total));
  return check_launch("k_scan_counts");
}

int hk_compact(const double* const* d_in, int32_t n_cols, int64_t n, const uint8_t* d_flags,
               const int64_t* d_offsets, double* const* d_out, int32_t weight_col, void* stream) {
  HK_NVTX("hk_compact");
  HK_REQUIRE(n_cols >= 1 && n_cols <= kMaxCols, "bad column count %d", n_cols);
  HK_REQUIRE(n >= 0, "negative n");
  if (n == 0) return HK_OK;
  HK_REQUIRE(d_in && d_out && d_flags && d_offsets, "NULL pointer");
  CompactArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int c = 0; c < n_cols; ++c) {
    HK_REQUIRE(d_in[c] && d_out[c], "column %d NULL", c);
    a.in[c] = d_in[c];
    a.out[c] = d_out[c];
  }
  a.n_cols = n_cols;
  a.weight_col = weight_col;
  a.n = n;
  a.flags = d_flags;
  a.offsets = reinterpret_cast<const long long*>(d_offsets);
  k_compact<<<chunk_grid(num_chunks(n)), kBlock, 0, as_stream(stream)>>>(a);
  return check_launch("k_compact");
}

}  // extern "C"

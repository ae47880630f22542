// hk_device.cuh -- device building blocks shared by the sm_100a kernels.
//
// Everything here is per-event register arithmetic on the FP64 pipe (the
// kinematics) and the integer pipe (the counter RNGs); nothing is a dense
// contraction, so there is no tensor-core work in this library.
//
// Parity notes (SURVEY.md 0, 7 "hard parts"):
//  * translation units that include this header are compiled with
//    -fmad=false, so every a*b+c below rounds twice exactly like numpy; the
//    few places that want an FMA spell it out with fma().
//  * CUDA's sqrt and double division are IEEE correctly rounded, so weights
//    (products of breakup momenta) are bit-identical to the reference; only
//    sin/cos differ (<= 1-2 ulp), which moves momentum components by
//    <~1e-16 * E (the parity tolerance is 1e-12 * E_daughter).
#pragma once

#ifndef __CUDACC_RTC__
#include <cstdint>
#endif

#include "hepkit_cuda.h"
#include "hk_math.cuh"

namespace hk {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;  // rng.py:33
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;    // rng.py:34
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;    // rng.py:35
constexpr uint64_t kSalt = 0x6A09E667F3BCC909ull;    // rng.py:36
constexpr double kInv53 = 1.1102230246251565e-16;    // 2^-53, rng.py:39
constexpr double kTwoPi = 6.283185307179586;         // fl(2 * pi), phasespace.py:136
constexpr int kBlock = 256;                          // threads per CTA
constexpr int kRowsPerThread = HK_CHUNK / kBlock;    // 16 rows per thread per chunk

// ---------------------------------------------------------------- RNG ------
// SplitMix64 avalanche finalizer (rng.py:98-102).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}

// base(seed, stream) (rng.py:109-112); inputs already reduced mod 2^64.
__host__ __device__ __forceinline__ uint64_t key_base(uint64_t seed, uint64_t stream) {
  return mix64(seed + kGolden) ^ mix64(stream * kSalt + kGolden);
}

// top 53 bits -> [0, 1), exact (rng.py:125).  One exact DMUL: measured faster
// on B200 than subtracting 53 from the exponent field on the integer pipe
// (six instructions with the zero check; generator 1.964 -> 1.923 ms per
// 1e8), the kernel being issue- rather than FP64-bound.
__device__ __forceinline__ double to_unit(uint64_t bits53) {
  return __ull2double_rn(bits53) * 0x1.0p-53;
}

// 2u and 2u - 1 for u = bits53 * 2^-53: both exact in the first step, so the
// single rounding of the fma equals numpy's 2.0 * u - 1.0 (phasespace.py:135-136)
__device__ __forceinline__ double two_unit(uint64_t bits53) {
  return __ull2double_rn(bits53) * 0x1.0p-52;
}
__device__ __forceinline__ double two_unit_minus_one(uint64_t bits53) {
  return fma(__ull2double_rn(bits53), 0x1.0p-52, -1.0);
}

// Philox4x32-10 (Salmon et al., SC'11); counter = (row lo, row hi, block, tag).
struct Philox4 {
  uint32_t v[4];
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                 uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  Philox4 out;
  out.v[0] = c0;
  out.v[1] = c1;
  out.v[2] = c2;
  out.v[3] = c3;
  return out;
}

// The same rounds with the key schedule precomputed per launch (rk[2r],
// rk[2r + 1] = round r's two key words): the round keys are kernel-parameter
// (constant-bank) operands of the LOP3s, so the 20 key additions and their
// registers leave the per-event code.  Bit-identical to philox4x32_10.
__device__ __forceinline__ Philox4 philox4x32_10_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                    const uint32_t (&rk)[20]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ rk[2 * r], n2 = hi0 ^ c3 ^ rk[2 * r + 1];
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  Philox4 out;
  out.v[0] = c0;
  out.v[1] = c1;
  out.v[2] = c2;
  out.v[3] = c3;
  return out;
}

constexpr uint32_t kPhiloxTag = 0x686b7068u;  // "hkph": separates this use of the key

// Per-launch RNG parameters; both modes are derived from the same hk_key_t.
struct RngParams {
  uint64_t base;  // SplitMix64 key base (reference mode) / Philox key (philox mode)
  uint64_t kc;    // key.counter
  int32_t mode;
  uint32_t rk[20];  // philox mode: the round keys of `base` (philox4x32_10_rk)
};

inline RngParams make_rng(const hk_key_t& k) {
  RngParams r;
  r.base = key_base(k.seed, k.stream);
  r.kc = k.counter;
  r.mode = k.mode;
  uint32_t k0 = (uint32_t)r.base, k1 = (uint32_t)(r.base >> 32);
  for (int i = 0; i < 10; ++i) {
    r.rk[2 * i] = k0;
    r.rk[2 * i + 1] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return r;
}

// The D uniforms of one event as 53-bit integers, so the mass uniforms can be
// ordered on the integer pipe (order of the integers == order of the doubles).
// Reference mode: counter (row + kc) * D + j (phasespace.py:105-109).
template <int D, int MODE>
__device__ __forceinline__ void draw_bits(const RngParams& rp, uint64_t row, uint64_t (&bits)[D]) {
  if (MODE == HK_RNG_REFERENCE) {
    const uint64_t x0 = rp.base + (row + rp.kc) * (uint64_t)D * kGolden;
#pragma unroll
    for (int j = 0; j < D; ++j) bits[j] = mix64(x0 + (uint64_t)j * kGolden) >> 11;
  } else {
    const uint64_t ev = row + rp.kc;
#pragma unroll
    for (int b = 0; b < (D + 1) / 2; ++b) {
      const Philox4 o = philox4x32_10_rk((uint32_t)ev, (uint32_t)(ev >> 32), (uint32_t)b, kPhiloxTag, rp.rk);
      bits[2 * b] = (((uint64_t)o.v[0] << 32) | o.v[1]) >> 11;
      if (2 * b + 1 < D) bits[2 * b + 1] = (((uint64_t)o.v[2] << 32) | o.v[3]) >> 11;
    }
  }
}

// Runtime-D variant for the generic (n > 8) kernels.
template <int MODE>
__device__ __forceinline__ uint64_t draw_bit_rt(const RngParams& rp, uint64_t row, int D, int j) {
  if (MODE == HK_RNG_REFERENCE) {
    return mix64(rp.base + ((row + rp.kc) * (uint64_t)D + (uint64_t)j) * kGolden) >> 11;
  } else {
    const uint64_t ev = row + rp.kc;
    const Philox4 o = philox4x32_10_rk((uint32_t)ev, (uint32_t)(ev >> 32), (uint32_t)(j >> 1), kPhiloxTag, rp.rk);
    return (j & 1) ? ((((uint64_t)o.v[2] << 32) | o.v[3]) >> 11)
                   : ((((uint64_t)o.v[0] << 32) | o.v[1]) >> 11);
  }
}

// ---------------------------------------------------------- kinematics -----
// np.maximum(x, 0.0): NaN propagates, -0.0 kept.
__device__ __forceinline__ double max0(double x) { return (x >= 0.0 || x != x) ? x : 0.0; }


// Boost frame of _boost (phasespace.py:74-81): the per-frame factors are shared
// by every vector boosted into it, which is exact (same operands, same ops).
struct Frame {
  double gamma, bx, by, bz, g2;
};

__device__ __forceinline__ Frame make_frame(double fe, double fx, double fy, double fz,
                                            double fm) {
  Frame f;
  f.gamma = fe / fm;
  f.bx = fx / fe;
  f.by = fy / fe;
  f.bz = fz / fe;
  f.g2 = f.gamma * f.gamma / (f.gamma + 1.0);
  return f;
}

__device__ __forceinline__ void boost(const Frame& f, double& e, double& px, double& py,
                                      double& pz) {
  const double bp = f.bx * px + f.by * py + f.bz * pz;
  const double k = f.g2 * bp + f.gamma * e;
  e = f.gamma * (e + bp);
  px = px + k * f.bx;
  py = py + k * f.by;
  pz = pz + k * f.bz;
}

// ~1 ulp reciprocal: MUFU seed + two Newton steps, no IEEE slow path
// (~5 instructions instead of ~15 for a correctly rounded division).  Used
// only where the parity budget is |dc| <= 1e-12 E (boost factors), never on
// the weight path.  inf -> NaN and 0 -> NaN, which matches what the IEEE
// divisions it replaces produce downstream (inf/inf, 0/0).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// ~1 ulp square root for x >= 0 without the IEEE slow-path branch: MUFU
// rsqrt seed, one Newton step on 1/sqrt, then a residual-corrected product.
// 0, inf and NaN pass through unchanged (as IEEE sqrt returns them); x < 0
// is never passed (callers clamp with max0 or add squares) and subnormal x
// (< 2.2e-308 GeV^2, physically impossible here) would also pass through.
// Used for energies and |sin theta|, never for the breakup momenta that
// make up the weight.
// The f64 rsqrt seed (MUFU.RSQ64H: a ~1e-6 accurate high word, low word 0),
// clamped to <= ~1e300 by one integer min on the high word: positive doubles
// order like their high words, so +inf (x = +0) becomes ~1e300, NaN seeds
// (sign set, negative as int) pass unchanged and positive normal x (seed high
// word < 0x5fd00000) are untouched.  The low word is the raw high word
// instead of 0: a <= 2^-20 relative perturbation of a 1e-6 seed, gone after
// the refinement steps (results bit-identical), and it saves the move that
// zeroes the low register of every seed.
__device__ __forceinline__ double rsqrt_seed_clamp(double y) {
  const int hi = __double2hiint(y);
  return __hiloint2double(min(hi, 0x7e37e43c), hi);
}

__device__ __forceinline__ double fast_sqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // x = 0: the seed is +inf; clamping it makes every step below exact zeros
  // (0 * ~1e300 = 0), so sqrt(0) = 0 without a compare-and-select -- and
  // without fmin's DSETP + 2 FSEL on the contended FP64 pipe.  A NaN x keeps
  // its NaN through x * y.
  y = rsqrt_seed_clamp(y);
  double s = x * y;  // sqrt(x), seed accuracy
  double h = 0.5 * y;  // 1 / (2 sqrt(x))
  const double r = fma(-s, h, 0.5);  // one coupled Goldschmidt step
  s = fma(s, r, s);
  h = fma(h, r, h);
  const double d = fma(-s, s, x);  // residual correction: ~1 ulp
  s = fma(d, h, s);
  return s;  // 0 -> 0 and NaN -> NaN like IEEE sqrt (inputs are finite and >= 0)
}

// Boost frame with one reciprocal for the three beta components and one for
// gamma^2/(gamma+1).  gamma = fe/fm: a reciprocal for fm > 0, the IEEE
// division otherwise, so a massless frame (fm = 0) gives the reference's inf.
__device__ __forceinline__ Frame make_frame_fast(double fe, double fx, double fy, double fz,
                                                 double fm) {
  Frame f;
  // branch-free: fm == +0 selects fe * inf, which is IEEE fe / +0 (inf, -inf
  // or NaN), so the scheduler can interleave across frames
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  f.gamma = fm == 0.0 ? fe * inf : fe * fast_rcp(fm);
  const double r = fast_rcp(fe);
  f.bx = fx * r;
  f.by = fy * r;
  f.bz = fz * r;
  f.g2 = f.gamma * f.gamma * fast_rcp(f.gamma + 1.0);
  return f;
}

// make_frame_fast for a frame whose mass is fixed by the decay: gmul is
// fast_rcp(fm), or +inf for fm == +0 (fe * inf is IEEE fe / +0), selected
// once per launch instead of per event
__device__ __forceinline__ Frame make_frame_fast_r(double fe, double fx, double fy, double fz,
                                                   double gmul) {
  Frame f;
  f.gamma = fe * gmul;
  const double r = fast_rcp(fe);
  f.bx = fx * r;
  f.by = fy * r;
  f.bz = fz * r;
  f.g2 = f.gamma * f.gamma * fast_rcp(f.gamma + 1.0);
  return f;
}

// _boost with the multiply-adds fused (the translation unit has -fmad=false,
// so contraction is opt-in here and nowhere else).
__device__ __forceinline__ void boost_fma(const Frame& f, double& e, double& px, double& py,
                                          double& pz) {
  const double bp = fma(f.bx, px, fma(f.by, py, f.bz * pz));
  const double k = fma(f.g2, bp, f.gamma * e);
  e = f.gamma * (e + bp);
  px = fma(k, f.bx, px);
  py = fma(k, f.by, py);
  pz = fma(k, f.bz, pz);
}

// _boost of a particle at rest (e = m, p = 0): bp = 0 so k = e' = gamma m.
__device__ __forceinline__ void boost_rest(const Frame& f, double m, double& e, double& px,
                                           double& py, double& pz) {
  e = f.gamma * m;
  px = e * f.bx;
  py = e * f.by;
  pz = e * f.bz;
}

// Lorentz boost into the lab of a frame with four-momentum (fe, P) and FIXED
// mass m (im = 1/m, rem = 1/(fe + m)): with beta = P/fe and gamma = fe/m,
//   E' = (fe E + P.p) / m,   p' = p + P ((P.p) / (fe + m) + E) / m,
// the same transformation as _boost (phasespace.py:74-81) with gamma^2/(gamma+1)
// (beta.p) beta rewritten through m -- 10 FP64 instructions per daughter and
// one reciprocal per frame instead of make_frame_fast's three.  Used by the
// fused chain when the host has proved the frame mass is the decay's (see
// hk_phsp_generate_chain); rounding differs from _boost's by a few ulp * E.
struct MFrame {
  double e, px, py, pz, im, rem;
};

// boost_m with the dot product P.p = s supplied by the caller
__device__ __forceinline__ void boost_m_s(const MFrame& f, double s, double& e, double& px, double& py, double& pz) {
  const double c = fma(s, f.rem, e) * f.im;
  e = fma(f.e, e, s) * f.im;
  px = fma(c, f.px, px);
  py = fma(c, f.py, py);
  pz = fma(c, f.pz, pz);
}

__device__ __forceinline__ void boost_m(const MFrame& f, double& e, double& px, double& py, double& pz) {
  const double s = fma(f.px, px, fma(f.py, py, f.pz * pz));
  const double c = fma(s, f.rem, e) * f.im;
  e = fma(f.e, e, s) * f.im;
  px = fma(c, f.px, px);
  py = fma(c, f.py, py);
  pz = fma(c, f.pz, pz);
}

// Branch-free correctly rounded sqrt for positive normal x whose result is
// normal: MUFU rsqrt seed, two Newton steps to y ~ 1/sqrt(x) (error far below
// 2^-53), then Markstein's residual correction s + (x - s^2) y/2.  Verified
// bit-identical to __dsqrt_rn on 2^32 inputs per family on B200
// (tools/verify_cr.cu); used on the weight path so weights stay bit-exact
// without the IEEE routine's slow-path branch.
__device__ __forceinline__ double cr_sqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // x = +0: the +inf seed clamps to ~1e300 (as in fast_sqrt), so every step
  // below is an exact zero and sqrt(+0) = +0
  y = rsqrt_seed_clamp(y);
  double t = x * y;
  y = fma(0.5 * y, fma(-t, y, 1.0), y);
  t = x * y;
  y = fma(0.5 * y, fma(-t, y, 1.0), y);
  const double s = x * y;
  const double d = fma(-s, s, x);
  return fma(d, 0.5 * y, s);
}

// Branch-free correctly rounded a / b for normal operands and quotient:
// q = a * (1/b), then one residual correction q + (a - b q) / b.
__device__ __forceinline__ double cr_div(double a, double b) {
  const double r = fast_rcp(b);
  const double q = a * r;
  const double rem = fma(-b, q, a);
  return fma(rem, r, q);
}

// sqrt(np.maximum(lam, 0)) for the Kallen lambda: correctly rounded for
// lam > 0, 0 for lam <= 0, NaN propagated.  lam = t*t - (4 a2) b2 of GeV-scale
// squares is either 0 or >= ~1e-20 (a multiple of ulp(t*t)), never subnormal,
// so cr_sqrt's normal-range domain covers it.
// np.maximum(lam, 0) as integer ops (no FP64-pipe compares): a set sign bit
// clears both words, so negative lam and -0 become +0 and cr_sqrt gives +0.
// NaN propagates: the FP64 units only produce the positive canonical NaN, and
// lam is formed by subtraction (no negation that could set a NaN's sign).
__device__ __forceinline__ double sqrt_lambda(double lam) {
  const int hi = __double2hiint(lam);
  const int keep = ~(hi >> 31);  // all ones unless the sign bit is set
  return cr_sqrt(__hiloint2double(hi & keep, __double2loint(lam) & keep));
}

// Two-body breakup momentum (phasespace.py:67-71), reference op order; b2 = m*m
// of the fixed daughter.  sqrt and the division are correctly rounded (IEEE
// results, bit-identical), so weights are bit-exact.
__device__ __forceinline__ double pstar(double M, double a, double b2) {
  const double M2 = M * M, a2 = a * a;
  const double t = (M2 - a2) - b2;
  const double lam = t * t - (4.0 * a2) * b2;
  return cr_div(sqrt_lambda(lam), 2.0 * M);
}

// cr_div with the divisor's reciprocal supplied (r = fast_rcp(b), hoisted)
__device__ __forceinline__ double cr_div_r(double a, double b, double r) {
  const double q = a * r;
  const double rem = fma(-b, q, a);
  return fma(rem, r, q);
}

// pstar with 1/(2M) supplied (the last breakup of a decay, M fixed)
__device__ __forceinline__ double pstar_r(double M, double a, double b2, double rcp_2m) {
  const double M2 = M * M, a2 = a * a;
  const double t = (M2 - a2) - b2;
  const double lam = t * t - (4.0 * a2) * b2;
  return cr_div_r(sqrt_lambda(lam), 2.0 * M, rcp_2m);
}

// c ? a : b through PTX selp, opaque to the front end's array-index recovery
__device__ __forceinline__ double select_f64(bool c, double a, double b) {
  double r;
  asm("{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %3, 0;\n\tselp.f64 %0, %1, %2, p;\n\t}"
      : "=d"(r)
      : "d"(a), "d"(b), "r"((int)c));
  return r;
}

// compare-exchange on the integer pipe
__device__ __forceinline__ void cswap(uint64_t& a, uint64_t& b) {
  const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
  a = lo;
  b = hi;
}

// One event of the rest-frame generator (phasespace.py:103-149) for a
// compile-time daughter count N.  p[4j..4j+3] = (e, px, py, pz) of daughter
// j+1; returns the weight (product of breakup momenta, phasespace.py:120-125).
// Per-decay reciprocals of rest_event<N>, hoistable out of the event loop
// (computed with the very operations rest_event would use, so events are
// bit-identical): 1/(2M) of the last breakup (M = inv[N-1] is fixed by the
// decay) and the first cluster frame's gamma multiplier: 1/inv[0], or +inf
// when inv[0] = m1 = 0 (so fe * gmul0 is IEEE fe / +0).
// HK_GEN_MBOOST: the generator's cluster boosts through the cluster's exact
// mass (boost_m) and daughter 1's first boost as the cluster itself
#ifndef HK_GEN_MBOOST
#define HK_GEN_MBOOST 1
#endif

struct RestHoist {
  double rcp_2m_last;
  double gmul0;  // make_frame_fast_r's gamma multiplier of the first cluster frame
  bool m0_zero;  // daughter 1 massless: its first boost is the reference's NaN
};

template <int N>
__device__ __forceinline__ RestHoist rest_hoist(const hk_decay_t& d) {
  RestHoist h;
  h.rcp_2m_last = fast_rcp(2.0 * (d.T + d.csum[N - 1]));
  h.gmul0 = d.csum[0] == 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : fast_rcp(d.csum[0]);
  h.m0_zero = d.csum[0] == 0.0;
  return h;
}

// The event from its D = 3N - 4 drawn uniforms (as 53-bit integers); split from
// the draw so a kernel can draw the next rows while this one computes.
template <int N>
__device__ __forceinline__ double rest_event_bits(const hk_decay_t& d, uint64_t (&bits)[3 * N - 4],
                                                  double (&p)[4 * N], const RestHoist& h) {
  // sorted mass uniforms: odd-even transposition network, integer compares
#pragma unroll
  for (int pass = 0; pass < N - 2; ++pass) {
#pragma unroll
    for (int j = pass & 1; j + 1 < N - 2; j += 2) cswap(bits[j], bits[j + 1]);
  }
  double inv[N];
  inv[0] = d.csum[0];  // 0 * T + csum[0] is exact
#pragma unroll
  for (int k = 1; k < N - 1; ++k) inv[k] = to_unit(bits[k - 1]) * d.T + d.csum[k];
  inv[N - 1] = d.T + d.csum[N - 1];  // 1.0 * T + csum[n-1] (phasespace.py:118)

  double ps[N];
  double w = 1.0;
#pragma unroll
  for (int k = 1; k < N; ++k) {
    // (hoisting the decay-fixed products too -- inv0^2, 4 inv0^2 m1^2, M_last^2
    // -- measured no faster: 1.969 ms either way; ptxas already keeps them)
    ps[k] = k == N - 1 ? pstar_r(inv[k], inv[k - 1], d.masses[k] * d.masses[k], h.rcp_2m_last)
                       : pstar(inv[k], inv[k - 1], d.masses[k] * d.masses[k]);
    w = w * ps[k];
  }

#pragma unroll
  for (int k = 1; k < N; ++k) {
    const double q = ps[k];
    const double cz = two_unit_minus_one(bits[N - 2 + 2 * (k - 1)]);
    // phi = 2 pi u: sincospi(2u) needs no Payne-Hanek reduction and differs
    // from cos(fl(2 pi u)) by at most the rounding of fl(2 pi u) (<= 4.4e-16)
    const double two_u = two_unit(bits[N - 2 + 2 * (k - 1) + 1]);
    // 1 - cz^2 >= 0 exactly (|cz| <= 1), so np.maximum is a no-op here;
    // cancellation-sensitive: no FMA
    const double sz = fast_sqrt(1.0 - cz * cz);
    double sn, cs;
    math::k_sincospi(two_u, &sn, &cs);
    const double nx = sz * cs, ny = sz * sn, nz = cz;
    const double clm = inv[k - 1];
    const double cle = fast_sqrt(q * q + clm * clm);
    const double clx = q * nx, cly = q * ny, clz = q * nz;
#if HK_GEN_MBOOST
    if (k == 1) {
      // daughter 1 starts at rest and is boosted by the cluster it alone makes
      // up (mass inv_0 = m_1): the result is the cluster's own four-momentum,
      // (cle, q n), within a few ulp of the reference's rounding.  m_1 = 0
      // gives the reference's gamma = inf -> NaN daughter (hoisted flag).
      if (h.m0_zero) {
        const double nan = __longlong_as_double(0x7ff8000000000000ll);
        p[0] = nan;
        p[1] = nan;
        p[2] = nan;
        p[3] = nan;
      } else {
        p[0] = cle;
        p[1] = clx;
        p[2] = cly;
        p[3] = clz;
      }
    } else if (__double2hiint(clm) > 0) {  // clm > 0 (clm >= 0 here), tested on the integer pipe
      // the cluster's mass is inv_{k-1} exactly: the fixed-mass boost (one
      // reciprocal per frame for 1/m and one for 1/(E + m), 10 FP64 per daughter)
      const MFrame f{cle, clx, cly, clz, fast_rcp(clm), fast_rcp(cle + clm)};
      if (k == 2 && !h.m0_zero) {
        // daughters 1 and 2 are back to back in the cluster they came from
        // (momenta q n and -q n): P.p is computed once, exactly negated (a
        // massless daughter 1 is the reference's NaN and must not leak into 2)
        const double s0 = fma(f.px, p[1], fma(f.py, p[2], f.pz * p[3]));
        boost_m_s(f, s0, p[0], p[1], p[2], p[3]);
        boost_m_s(f, -s0, p[4], p[5], p[6], p[7]);
      } else {
#pragma unroll
        for (int j = 0; j < k; ++j) boost_m(f, p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
      }
    } else {  // a massless cluster: the reference's gamma = inf arithmetic, exactly
      const Frame f = make_frame_fast(cle, clx, cly, clz, clm);
#pragma unroll
      for (int j = 0; j < k; ++j) boost_fma(f, p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
    }
#else
    const Frame f = k == 1 ? make_frame_fast_r(cle, clx, cly, clz, h.gmul0)
                           : make_frame_fast(cle, clx, cly, clz, clm);
    if (k == 1) {
      boost_rest(f, d.masses[0], p[0], p[1], p[2], p[3]);  // daughter 1 starts at rest
    } else {
#pragma unroll
      for (int j = 0; j < k; ++j) boost_fma(f, p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
    }
#endif
    p[4 * k + 0] = fast_sqrt(q * q + d.masses[k] * d.masses[k]);
    p[4 * k + 1] = -clx;
    p[4 * k + 2] = -cly;
    p[4 * k + 3] = -clz;
  }
  return w;
}

template <int N, int MODE>
__device__ __forceinline__ double rest_event(const hk_decay_t& d, const RngParams& rp,
                                             uint64_t row, double (&p)[4 * N], const RestHoist& h) {
  uint64_t bits[3 * N - 4];  // phasespace.py:84-86
  draw_bits<3 * N - 4, MODE>(rp, row, bits);
  return rest_event_bits<N>(d, bits, p, h);
}

template <int N, int MODE>
__device__ __forceinline__ double rest_event(const hk_decay_t& d, const RngParams& rp,
                                             uint64_t row, double (&p)[4 * N]) {
  return rest_event<N, MODE>(d, rp, row, p, rest_hoist<N>(d));
}

// A 2-body decay at rest has every per-event quantity but the direction
// fixed by the decay: breakup momentum (= the weight), cluster energy, the
// frame's gamma, 1/E and gamma^2/(gamma+1), and daughter 2's energy.
// two_body_consts computes them ONCE per thread with exactly the operations
// of rest_event<2>; rest_event2 then spends per event only the RNG, the
// direction and the boost -- the outputs are bit-identical to rest_event<2>.
// (Used for chain sub-decays such as J/psi -> mu mu.)
struct TwoBody {
  double w, q, r, gamma, g2, e2, m0;
  double e1;  // sqrt(q^2 + m0^2): daughter 0's rest-frame energy (fixed-frame chain path)
};

__device__ __forceinline__ TwoBody two_body_consts(const hk_decay_t& d) {
  TwoBody t;
  const double inv0 = d.csum[0];        // 0 * T + csum[0] is exact
  const double inv1 = d.T + d.csum[1];  // phasespace.py:118
  t.q = pstar(inv1, inv0, d.masses[1] * d.masses[1]);
  t.w = 1.0 * t.q;
  const double cle = fast_sqrt(t.q * t.q + inv0 * inv0);
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  t.gamma = inv0 == 0.0 ? cle * inf : cle * fast_rcp(inv0);
  t.r = fast_rcp(cle);
  t.g2 = t.gamma * t.gamma * fast_rcp(t.gamma + 1.0);
  t.e2 = fast_sqrt(t.q * t.q + d.masses[1] * d.masses[1]);
  t.m0 = d.masses[0];
  t.e1 = cle;
  return t;
}

// Two-body decay in the fixed frame f: daughters (e1, q n) and (e2, -q n) in
// the rest frame (the reference's GENBOD for n = 2 gives daughter 0 as a boost
// of (m0, 0) to (e1, q n), daughter 1 as (e2, -q n)), boosted together: the
// shared P.(q n) is computed once.  Same draws and direction as rest_event2.
template <int MODE>
__device__ __forceinline__ double two_body_boosted(const TwoBody& t, const RngParams& rp, uint64_t row,
                                                   const MFrame& f, double (&p)[8]) {
  uint64_t bits[2];
  draw_bits<2, MODE>(rp, row, bits);
  const double cz = two_unit_minus_one(bits[0]);
  const double two_u = two_unit(bits[1]);
  const double sz = fast_sqrt(1.0 - cz * cz);
  double sn, cs;
  math::k_sincospi(two_u, &sn, &cs);
  const double qs = t.q * sz;
  const double cx = qs * cs, cy = qs * sn, czq = t.q * cz;
  const double s = fma(f.px, cx, fma(f.py, cy, f.pz * czq));
  const double c0 = fma(s, f.rem, t.e1) * f.im;
  const double c1 = fma(-s, f.rem, t.e2) * f.im;
  p[0] = fma(f.e, t.e1, s) * f.im;
  p[1] = fma(c0, f.px, cx);
  p[2] = fma(c0, f.py, cy);
  p[3] = fma(c0, f.pz, czq);
  p[4] = fma(f.e, t.e2, -s) * f.im;
  p[5] = fma(c1, f.px, -cx);
  p[6] = fma(c1, f.py, -cy);
  p[7] = fma(c1, f.pz, -czq);
  return t.w;
}

template <int MODE>
__device__ __forceinline__ double rest_event2(const TwoBody& t, const RngParams& rp, uint64_t row,
                                              double (&p)[8]) {
  uint64_t bits[2];
  draw_bits<2, MODE>(rp, row, bits);
  const double cz = two_unit_minus_one(bits[0]);
  const double two_u = two_unit(bits[1]);
  const double sz = fast_sqrt(1.0 - cz * cz);
  double sn, cs;
  math::k_sincospi(two_u, &sn, &cs);
  const double nx = sz * cs, ny = sz * sn, nz = cz;
  const double clx = t.q * nx, cly = t.q * ny, clz = t.q * nz;
  Frame f;
  f.gamma = t.gamma;
  f.bx = clx * t.r;
  f.by = cly * t.r;
  f.bz = clz * t.r;
  f.g2 = t.g2;
  boost_rest(f, t.m0, p[0], p[1], p[2], p[3]);
  p[4] = t.e2;
  p[5] = -clx;
  p[6] = -cly;
  p[7] = -clz;
  return t.w;
}

// Runtime-n variant (n <= HK_MAX_DAUGHTERS); arrays live in local memory.
template <int MODE>
__device__ double rest_event_rt(const hk_decay_t& d, const RngParams& rp, uint64_t row,
                                double* p) {
  const int n = d.n, D = 3 * n - 4;
  double rno[HK_MAX_DAUGHTERS], inv[HK_MAX_DAUGHTERS], ps[HK_MAX_DAUGHTERS];
  uint64_t sorted[HK_MAX_DAUGHTERS];
  for (int j = 0; j < n - 2; ++j) {  // insertion sort of the mass uniforms
    const uint64_t b = draw_bit_rt<MODE>(rp, row, D, j);
    int i = j;
    while (i > 0 && sorted[i - 1] > b) {
      sorted[i] = sorted[i - 1];
      --i;
    }
    sorted[i] = b;
  }
  for (int k = 1; k < n - 1; ++k) rno[k] = to_unit(sorted[k - 1]);
  inv[0] = d.csum[0];
  for (int k = 1; k < n - 1; ++k) inv[k] = rno[k] * d.T + d.csum[k];
  inv[n - 1] = d.T + d.csum[n - 1];
  double w = 1.0;
  for (int k = 1; k < n; ++k) {
    ps[k] = pstar(inv[k], inv[k - 1], d.masses[k] * d.masses[k]);
    w = w * ps[k];
  }
  p[0] = d.masses[0];
  p[1] = p[2] = p[3] = 0.0;
  for (int k = 1; k < n; ++k) {
    const double q = ps[k];
    const double cz = 2.0 * to_unit(draw_bit_rt<MODE>(rp, row, D, n - 2 + 2 * (k - 1))) - 1.0;
    const double phi = kTwoPi * to_unit(draw_bit_rt<MODE>(rp, row, D, n - 1 + 2 * (k - 1)));
    const double sz = sqrt(max0(1.0 - cz * cz));
    double sn, cs;
    sincos(phi, &sn, &cs);
    const double clm = inv[k - 1];
    const double cle = sqrt(q * q + clm * clm);
    const double clx = q * (sz * cs), cly = q * (sz * sn), clz = q * cz;
    const Frame f = make_frame(cle, clx, cly, clz, clm);
    for (int j = 0; j < k; ++j) boost(f, p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
    p[4 * k + 0] = sqrt(q * q + d.masses[k] * d.masses[k]);
    p[4 * k + 1] = -clx;
    p[4 * k + 2] = -cly;
    p[4 * k + 3] = -clz;
  }
  return w;
}

// -------------------------------------------------------- reductions -------
// Deterministic CTA reduction of W doubles: fixed shuffle tree inside each
// warp, then warps summed in index order by thread w.  Writes out[0..W).
template <int W>
__device__ __forceinline__ void block_sum_store(double (&v)[W], double* out) {
  __shared__ double sm[kBlock / 32][W];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] += __shfl_down_sync(0xffffffffu, v[w], off);
  }
  if (lane == 0) {
#pragma unroll
    for (int w = 0; w < W; ++w) sm[warp][w] = v[w];
  }
  __syncthreads();
  if (threadIdx.x < W) {
    double s = sm[0][threadIdx.x];
#pragma unroll
    for (int i = 1; i < kBlock / 32; ++i) s += sm[i][threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Per-warp partials (no CTA barrier): a fixed shuffle tree inside the warp,
// lane 0 stores W doubles for warp-slice (chunk, warp) at
// out[W * (chunk * HK_WARP_SLICES + warp) ..].  The host folds the slices in
// index order, so the result is as deterministic as a CTA reduction.
template <int W>
__device__ __forceinline__ void warp_sum_store(double (&v)[W], double* out, int64_t chunk,
                                               int warp_in_chunk = -1) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] += __shfl_down_sync(0xffffffffu, v[w], off);
  }
  if ((threadIdx.x & 31) == 0) {
    const int slot = warp_in_chunk >= 0 ? warp_in_chunk : (int)(threadIdx.x >> 5);
    double* dst = out + (int64_t)W * (chunk * HK_WARP_SLICES + slot);
#pragma unroll
    for (int w = 0; w < W; ++w) dst[w] = v[w];
  }
}

__device__ __forceinline__ void record_bad(unsigned long long* first_bad, uint64_t row) {
  if (first_bad) atomicMin(first_bad, (unsigned long long)row);
}

// -------------------------------------------------- functor programs -------
// Interpreter for hk_program_t (host-lowered FunctorExpr + arg_builder DAG).
// Every thread runs the same op stream, so the switch is warp-uniform.
// `load(c)` supplies column c of the current event.  Division by zero sets
// *div0 (functors.py:200-207 raises before evaluating).
// run_program_into leaves every slot in r (multi-output programs keep their
// outputs in pinned slots, functors.compile_program(keep=...)).
template <class Load>
__device__ __forceinline__ void run_program_into(const hk_program_t& P, Load load, bool* div0,
                                                 double (&r)[HK_MAX_SLOTS]) {
  for (int i = 0; i < P.n_ops; ++i) {
    const int op = P.op[i];
    double v;
    switch (op) {
      case HK_OP_COL: v = load(P.a[i]); break;
      case HK_OP_CONST: v = P.cst[i]; break;
      case HK_OP_ADD: v = r[P.a[i]] + r[P.b[i]]; break;
      case HK_OP_SUB: v = r[P.a[i]] - r[P.b[i]]; break;
      case HK_OP_MUL: v = r[P.a[i]] * r[P.b[i]]; break;
      case HK_OP_DIV: {
        const double den = r[P.b[i]];
        if (den == 0.0) *div0 = true;
        v = r[P.a[i]] / den;
        break;
      }
      case HK_OP_NEG: v = -r[P.a[i]]; break;
      case HK_OP_SQRT: v = sqrt(r[P.a[i]]); break;
      case HK_OP_EXP: v = exp(r[P.a[i]]); break;
      case HK_OP_LOG: v = log(r[P.a[i]]); break;
      case HK_OP_GAUSS: {
        const double s = P.cst2[i];
        const double z = (r[P.a[i]] - P.cst[i]) / s;
        v = exp(-0.5 * z * z) / (s * 2.5066282746310002);  // functors.py:26, :142-143
        break;
      }
      case HK_OP_EXPO: v = exp(-r[P.a[i]] / P.cst[i]); break;
      case HK_OP_BW: {
        const double m0 = P.cst[i], g0 = P.cst2[i];
        const double t = r[P.a[i]] - m0 * m0;
        v = 1.0 / (t * t + (m0 * m0) * (g0 * g0));
        break;
      }
      case HK_OP_ADD0: v = r[P.a[i]] + 0.0; break;
      case HK_OP_SQUARE: v = r[P.a[i]] * r[P.a[i]]; break;
      case HK_OP_UDIV: v = r[P.a[i]] / r[P.b[i]]; break;
      default: v = __longlong_as_double(0x7ff8000000000000ll); break;
    }
    r[P.dst[i]] = v;
  }
}

template <class Load>
__device__ __forceinline__ double run_program(const hk_program_t& P, Load load, bool* div0) {
  double r[HK_MAX_SLOTS];
  run_program_into(P, load, div0, r);
  return r[P.result];
}

}  // namespace hk

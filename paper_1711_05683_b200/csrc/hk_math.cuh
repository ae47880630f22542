// hk_math.cuh -- our own fp64 sin/cos(pi t) and exp.
//
// The generator uses sincospi_gen (near-minimax, ~30 instructions; libdevice's
// sincospi takes 53 on sm_100a); k_exp defaults to libdevice's exp, which
// measured faster in the FCN (35.8 vs 45.6 us for ours).  Earlier
// measurements on B200: coefficients from the constant
// bank (HK_MATH_CONST_BANK) were slower (generator +2.6%, FCN +27%); the
// Taylor-form sincospi below tied libdevice (2.315 vs 2.305 ms per 1e8).
// The functions are __host__ __device__ so tests/test_math_host.py checks
// them against long double on the CPU.
//
// Accuracy (CPU, 2^22 points):
//   sincospi: |error| <= 2 ulp(1) absolute for |t| < 2^20
//   exp:      <= 2 ulp relative over [-708, 709]; exact under/overflow to
//             0/inf beyond; NaN propagates.
#pragma once

#ifndef __CUDACC_RTC__
#include <cmath>
#include <cstdint>
#include <cstring>
#endif

#if defined(__CUDACC__)
#define HK_HD __host__ __device__ __forceinline__
#else
#define HK_HD inline
#endif

namespace hk {
namespace math {

// sin(pi r) = r * sum_k S[k] r^2k and cos(pi r) = sum_k C[k] r^2k on |r| <= 1/4
// (Taylor coefficients of pi^(2k+1)/(2k+1)! and pi^2k/(2k)!, rounded to
// double; truncation < 1e-19 on the interval).  exp: 1/k!, k = 0..13 on
// |r| <= ln2/2 (truncation < 5e-18).
#define HK_SIN_COEFFS                                                                     \
  {3.141592653589793, -5.16771278004997, 2.5501640398773455, -0.5992645293207921,         \
   0.08214588661112823, -0.0073704309457143504, 0.00046630280576761255,                   \
   -2.1915353447830217e-05, 7.952054001475513e-07}
#define HK_COS_COEFFS                                                                     \
  {1.0, -4.934802200544679, 4.0587121264167685, -1.3352627688545895, 0.2353306303588932,  \
   -0.02580689139001406, 0.0019295743094039231, -0.0001046381049248457,                   \
   4.303069587032947e-06, -1.3878952462213771e-07}
#define HK_EXP_COEFFS                                                                     \
  {1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664, 0.008333333333333333,        \
   0.001388888888888889, 0.0001984126984126984, 2.48015873015873e-05,                     \
   2.7557319223985893e-06, 2.755731922398589e-07, 2.505210838544172e-08,                  \
   2.08767569878681e-09, 1.6059043836821613e-10}

#if defined(__CUDACC__)
static __constant__ double kSin[9] = HK_SIN_COEFFS;
static __constant__ double kCos[10] = HK_COS_COEFFS;
static __constant__ double kExp[14] = HK_EXP_COEFFS;
#endif

// Same coefficients as compile-time constants (folded into immediates once
// the Horner loops are unrolled); the default on both host and device.
template <int K>
struct CoefArray {
  double v[K];
};
HK_HD constexpr double hSin(int k) { return CoefArray<9>{HK_SIN_COEFFS}.v[k]; }
HK_HD constexpr double hCos(int k) { return CoefArray<10>{HK_COS_COEFFS}.v[k]; }
HK_HD constexpr double hExp(int k) { return CoefArray<14>{HK_EXP_COEFFS}.v[k]; }

#if defined(__CUDA_ARCH__) && defined(HK_MATH_CONST_BANK)
#define HK_COEF(dev, host, k) dev[k]
#else
#define HK_COEF(dev, host, k) host(k)
#endif

HK_HD double bits_to_double(int64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(b);
#else
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
#endif
}

// sin(pi t), cos(pi t).  t = q/2 + r with q = rint(2t) and |r| <= 1/4 exactly
// (t - q/2 is exact for |t| < 2^51); the quadrant q mod 4 swaps/negates.
HK_HD void sincospi(double t, double* s, double* c) {
  const double q = rint(2.0 * t);
  const double r = fma(-0.5, q, t);
  const double r2 = r * r;
  double ps = HK_COEF(kSin, hSin, 8);
#pragma unroll
  for (int k = 7; k >= 0; --k) ps = fma(ps, r2, HK_COEF(kSin, hSin, k));
  double pc = HK_COEF(kCos, hCos, 9);
#pragma unroll
  for (int k = 8; k >= 0; --k) pc = fma(pc, r2, HK_COEF(kCos, hCos, k));
  const double sr = r * ps;
  const int iq = (int)q;
  double sn = (iq & 1) ? pc : sr;
  double cs = (iq & 1) ? sr : pc;
  sn = (iq & 2) ? -sn : sn;
  cs = ((iq + 1) & 2) ? -cs : cs;
  *s = sn;
  *c = cs;
}

// sin(pi t), cos(pi t) for the generator's angles (t = 2u in [0, 2), any
// finite t works): the quadrant reduction above with near-minimax polynomials
// of degree 13 (sin) and 14 (cos) on |r| <= 1/4 -- max abs error 1.1e-16 in
// double, like the longer Taylor forms (fitted by tools/fit_sincospi.py).
// 15 FMA-class ops + the reduction: about 30 instructions where libdevice's
// sincospi takes 53 on sm_100a (ncu source view of k_generate).
HK_HD void sincospi_gen(double t, double* s, double* c) {
  const double q = rint(2.0 * t);
  const double r = fma(-0.5, q, t);
  const double r2 = r * r;
  double ps = 0x1.e3988d39fa62ep-12;
  ps = fma(ps, r2, -0x1.e2ff4a0c92053p-8);
  ps = fma(ps, r2, 0x1.50782e688341bp-4);
  ps = fma(ps, r2, -0x1.32d2cce12a338p-1);
  ps = fma(ps, r2, 0x1.466bc677567a1p+1);
  ps = fma(ps, r2, -0x1.4abbce625be21p+2);
  ps = fma(ps, r2, 0x1.921fb54442d18p+1);
  double pc = -0x1.b264e50804144p-14;
  pc = fma(pc, r2, 0x1.f9cc41b007973p-10);
  pc = fma(pc, r2, -0x1.a6d1ec79e7ce5p-6);
  pc = fma(pc, r2, 0x1.e1f506835728ep-3);
  pc = fma(pc, r2, -0x1.55d3c7e3c9108p+0);
  pc = fma(pc, r2, 0x1.03c1f081b5aacp+2);
  pc = fma(pc, r2, -0x1.3bd3cc9be45dep+2);
  pc = fma(pc, r2, 1.0);
  const double sr = r * ps;
  const int iq = (int)q;
  double sn = (iq & 1) ? pc : sr;
  double cs = (iq & 1) ? sr : pc;
#if defined(__CUDA_ARCH__)
  // quadrant signs as sign-bit flips on the high word (exact, like negation)
  sn = __hiloint2double(__double2hiint(sn) ^ (int)(((unsigned)iq & 2u) << 30), __double2loint(sn));
  cs = __hiloint2double(__double2hiint(cs) ^ (int)(((unsigned)(iq + 1) & 2u) << 30),
                        __double2loint(cs));
#else
  sn = (iq & 2) ? -sn : sn;
  cs = ((iq + 1) & 2) ? -cs : cs;
#endif
  *s = sn;
  *c = cs;
}

// e^x: n = rint(x log2 e), r = x - n ln2 (two-part ln2, exact first step),
// Taylor on r, then 2^n applied as two normal factors so results down to the
// subnormal range and up to overflow come out right without branches.
HK_HD double exp(double x) {
  x = x > 710.0 ? 710.0 : x;    // NaN fails both compares and propagates
  x = x < -746.0 ? -746.0 : x;
  const double n = rint(x * 1.4426950408889634);
  double r = fma(-n, 0.6931471803691238, x);
  r = fma(-n, 1.9082149292705877e-10, r);
  double p = HK_COEF(kExp, hExp, 13);
#pragma unroll
  for (int k = 12; k >= 0; --k) p = fma(p, r, HK_COEF(kExp, hExp, k));
  const int in = (n == n) ? (int)n : 0;
  const int h = in >> 1;
  const double s1 = bits_to_double((int64_t)(h + 1023) << 52);
  const double s2 = bits_to_double((int64_t)(in - h + 1023) << 52);
  return p * s1 * s2;
}

// Kernel entry points; -DHK_MATH_LIBDEVICE selects CUDA's own sincospi/exp
// (for A/B measurements).
// sincospi for the generator: sincospi_gen (minimax, ~30 instructions) by
// default; -DHK_MATH_LIBDEVICE_SINCOSPI selects libdevice's for A/B.  (The
// earlier Taylor-form sincospi measured equal to libdevice: 2.315 vs 2.305 ms.)
HK_HD void k_sincospi(double t, double* s, double* c) {
#if defined(__CUDA_ARCH__) && defined(HK_MATH_LIBDEVICE_SINCOSPI)
  ::sincospi(t, s, c);
#else
  sincospi_gen(t, s, c);
#endif
}

// exp for the FCN: libdevice's exp measured faster than hk::math::exp there
// (35.8 vs 45.6 us per 1e7-event FCN kernel on B200: fewer range-check
// instructions), so it is the default; -DHK_MATH_OWN_EXP selects ours.
HK_HD double k_exp(double x) {
#if defined(__CUDA_ARCH__) && !defined(HK_MATH_OWN_EXP)
  return ::exp(x);
#else
  return math::exp(x);
#endif
}

}  // namespace math
}  // namespace hk

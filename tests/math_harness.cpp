// CPU accuracy check of csrc/hk_math.cuh (the same source the kernels use),
// against long double references.  Prints max errors in ulps as JSON.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "hk_math.cuh"

static double ulp(double x) { return std::nextafter(std::fabs(x), INFINITY) - std::fabs(x); }

int main(int argc, char** argv) {
  std::mt19937_64 rng(12345);
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  const long double PI = 3.141592653589793238462643383279502884L;
  double max_sc = 0, max_exp = 0, max_gen = 0;
  const int N = argc > 1 ? std::atoi(argv[1]) : (1 << 24);
  for (int i = 0; i < N; ++i) {
    // t = 2u exactly as the generator forms it, plus a sweep of wider t
    double t = (i & 1) ? 2.0 * (double)(rng() >> 11) * 0x1.0p-53 : (u01(rng) - 0.5) * 2048.0;
    double s, c;
    hk::math::sincospi(t, &s, &c);
    long double tl = t;
    long double rs = sinl(PI * tl), rc = cosl(PI * tl);
    double es = (double)fabsl((long double)s - rs) / ulp(1.0);
    double ec = (double)fabsl((long double)c - rc) / ulp(1.0);
    if (es > max_sc) max_sc = es;
    if (ec > max_sc) max_sc = ec;
    double gs, gc;   // the generator's minimax variant
    hk::math::sincospi_gen(t, &gs, &gc);
    double gse = (double)fabsl((long double)gs - rs) / ulp(1.0);
    double gce = (double)fabsl((long double)gc - rc) / ulp(1.0);
    if (gse > max_gen) max_gen = gse;
    if (gce > max_gen) max_gen = gce;
    double x = (u01(rng) - 0.5) * 1416.0;   // [-708, 708]
    if (i % 7 == 0) x = (u01(rng) - 0.5) * 20.0;
    double e = hk::math::exp(x);
    long double re = expl((long double)x);
    double ee = (double)(fabsl((long double)e - re) / (long double)ulp((double)re));
    if (ee > max_exp) max_exp = ee;
  }
  // special values
  bool ok = hk::math::exp(-800.0) == 0.0 && std::isinf(hk::math::exp(800.0)) &&
            std::isnan(hk::math::exp(NAN)) && hk::math::exp(0.0) == 1.0;
  double sub = hk::math::exp(-740.0);
  double rsub = (double)expl(-740.0L);
  ok = ok && std::fabs(sub - rsub) <= 2 * 4.9406564584124654e-324;
  std::printf("{\"sincospi_max_abs_err_ulp1\": %.3f, \"sincospi_gen_max_abs_err_ulp1\": %.3f, "
              "\"exp_max_rel_err_ulp\": %.3f, \"special_ok\": %s}\n",
              max_sc, max_gen, max_exp, ok ? "true" : "false");
  return 0;
}

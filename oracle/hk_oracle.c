/*
 * hk_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, scalar, CPU restatement of the reference (`hepkit`) hot path, used
 * as the parity oracle for the CUDA kernels and as the `cpu_baseline` /
 * `--impl reference` leg of bench.py.  Nothing in the product package links or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py may.
 *
 * Compile with -ffp-contract=off (see oracle/Makefile): the reference is numpy,
 * which never fuses a*b+c, and the Kallen lambda / 1-cz^2 expressions are
 * cancellation-sensitive, so any FMA contraction breaks bit-parity.
 * libm (glibc) sin/cos/sqrt are bit-identical to numpy's float64 ufuncs here,
 * so the generator reproduces the reference bit for bit (pinned against
 * the tests/golden fixtures, produced by tests/golden/make_golden.py from the
 * reference itself).
 *
 * Reference citations (all under /root/reference/pkg/src/hepkit/):
 *   SplitMix64 finalizer ........ rng.py:98-102   (_mix64)
 *   key base .................... rng.py:109-112  (_base)
 *   raw / uniform ............... rng.py:115-125  (raw64, uniform_array)
 *   draws per event ............. phasespace.py:84-86
 *   breakup momentum ............ phasespace.py:67-71 (_pdk_array)
 *   boost ....................... phasespace.py:74-81 (_boost)
 *   rest-frame generator ........ phasespace.py:89-159
 *   mother boost ................ phasespace.py:181-187
 *   decay chain ................. phasespace.py:237-288
 *   unweight accept ............. phasespace.py:225-227
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define HKO_GOLDEN 0x9E3779B97F4A7C15ULL
#define HKO_MIX1 0xBF58476D1CE4E5B9ULL
#define HKO_MIX2 0x94D049BB133111EBULL
#define HKO_SALT 0x6A09E667F3BCC909ULL
#define HKO_MAXN 64

static const double kTwoPi = 6.283185307179586; /* fl(2.0 * math.pi) */
static const double kInv53 = 1.1102230246251565e-16; /* 2**-53 */

uint64_t hko_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * HKO_MIX1;
  z = (z ^ (z >> 27)) * HKO_MIX2;
  return z ^ (z >> 31);
}

uint64_t hko_base(uint64_t seed, uint64_t stream) {
  return hko_mix64(seed + HKO_GOLDEN) ^ hko_mix64(stream * HKO_SALT + HKO_GOLDEN);
}

static inline double u01(uint64_t base, uint64_t c) {
  return (double)(hko_mix64(base + c * HKO_GOLDEN) >> 11) * kInv53;
}

/*
 * Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy
 * as 1, 2, 3", SC'11; Random123 philox4x32 with R = 10): the production stream
 * of the CUDA path (not a reference stream; north_star subsystem 2).  Round:
 * (c0, c1, c2, c3) -> (hi(M1 c2) ^ c1 ^ k0, lo(M1 c2), hi(M0 c0) ^ c3 ^ k1,
 * lo(M0 c0)), M0 = 0xD2511F53, M1 = 0xCD9E8D57; key bumped by the Weyl
 * constants (0x9E3779B9, 0xBB67AE85) between rounds.  Pinned against the
 * Random123 known-answer vectors in tests/test_oracle_golden.py.
 */
void hko_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* rows x (ctr[4], key[2]) -> rows x 4 words */
void hko_philox_rows(const uint32_t* in6, int64_t n, uint32_t* out4) {
  for (int64_t i = 0; i < n; ++i) hko_philox4x32_10(in6 + 6 * i, in6 + 6 * i + 4, out4 + 4 * i);
}

#define HKO_RNG_REFERENCE 0
#define HKO_RNG_PHILOX 1
#define HKO_PHILOX_TAG 0x686b7068u /* "hkph" */

/* The CUDA path's Philox stream mapping (csrc/hk_device.cuh draw_bits): draw
 * j of event ev (key counter included) is word pair j & 1 of the block
 * philox(ctr = (ev lo, ev hi, j >> 1, tag), key = (base lo, base hi)). */
static inline uint64_t philox_bits(uint64_t base, uint64_t ev, uint64_t j) {
  uint32_t ctr[4] = {(uint32_t)ev, (uint32_t)(ev >> 32), (uint32_t)(j >> 1), HKO_PHILOX_TAG};
  uint32_t key[2] = {(uint32_t)base, (uint32_t)(base >> 32)}, o[4];
  hko_philox4x32_10(ctr, key, o);
  return (j & 1) ? (((uint64_t)o[2] << 32) | o[3]) : (((uint64_t)o[0] << 32) | o[1]);
}

/* uniform draw j of event evk (= event + key.counter) with D draws per event */
typedef struct {
  int mode;
  uint64_t base;
} rng_t;

static inline double draw(const rng_t* r, uint64_t evk, uint64_t D, uint64_t j) {
  if (r->mode == HKO_RNG_PHILOX) return (double)(philox_bits(r->base, evk, j) >> 11) * kInv53;
  return u01(r->base, evk * D + j);
}

/* raw64 in the Philox mode (hk_rng_raw64): counter c -> block (c lo, c hi, 0, tag), words 0-1 */
void hko_philox_raw64(uint64_t base, uint64_t kc, const uint64_t* counters, int64_t n, uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = philox_bits(base, counters[i] + kc, 0);
}

/* raw64(key, counters): out[i] = mix(base + (counters[i] + kc) * G) */
void hko_raw64(uint64_t base, uint64_t kc, const uint64_t* counters, int64_t n,
               uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = hko_mix64(base + (counters[i] + kc) * HKO_GOLDEN);
}

void hko_uniform(uint64_t base, uint64_t kc, const uint64_t* counters, int64_t n,
                 double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = u01(base, counters[i] + kc);
}

/* np.maximum(x, 0.0): NaN propagates, -0.0 is kept (it compares >= 0). */
static inline double max0(double x) { return (x >= 0.0 || x != x) ? x : 0.0; }

static inline double pstar(double M, double a, double b) {
  double M2 = M * M, a2 = a * a, b2 = b * b;
  double t = (M2 - a2) - b2;
  double lam = t * t - (4.0 * a2) * b2;
  return sqrt(max0(lam)) / (2.0 * M);
}

typedef struct {
  double gamma, bx, by, bz, g2;
} frame_t;

static inline frame_t make_frame(double fe, double fx, double fy, double fz, double fm) {
  frame_t f;
  f.gamma = fe / fm;
  f.bx = fx / fe;
  f.by = fy / fe;
  f.bz = fz / fe;
  f.g2 = f.gamma * f.gamma / (f.gamma + 1.0);
  return f;
}

static inline void apply_frame(const frame_t* f, double* v /* e,px,py,pz */) {
  double bp = f->bx * v[1] + f->by * v[2] + f->bz * v[3];
  double k = f->g2 * bp + f->gamma * v[0];
  v[0] = f->gamma * (v[0] + bp);
  v[1] = v[1] + k * f->bx;
  v[2] = v[2] + k * f->by;
  v[3] = v[3] + k * f->bz;
}

/* One event in the rest frame: returns weight, fills p[4*n]. */
static double rest_frame_event(int n, const double* m, double T, const double* csum,
                               const rng_t* rng, uint64_t evk, double* p) {
  const uint64_t D = (uint64_t)(3 * n - 4);
  double rno[HKO_MAXN], inv[HKO_MAXN], ps[HKO_MAXN];
  rno[0] = 0.0;
  rno[n - 1] = 1.0;
  for (int j = 0; j < n - 2; ++j) {  /* insertion sort == np.sort order */
    double u = draw(rng, evk, D, (uint64_t)j);
    int i = j;
    while (i > 0 && rno[i] > u) {
      rno[i + 1] = rno[i];
      --i;
    }
    rno[i + 1] = u;
  }
  for (int k = 0; k < n; ++k) inv[k] = rno[k] * T + csum[k];
  double w = 1.0;
  for (int k = 1; k < n; ++k) {
    ps[k] = pstar(inv[k], inv[k - 1], m[k]);
    w = w * ps[k];
  }
  for (int j = 0; j < 4 * n; ++j) p[j] = 0.0;
  p[0] = m[0];
  for (int k = 1; k < n; ++k) {
    double q = ps[k];
    uint64_t ca = (uint64_t)(n - 2 + 2 * (k - 1));
    double cz = 2.0 * draw(rng, evk, D, ca) - 1.0;
    double phi = kTwoPi * draw(rng, evk, D, ca + 1);
    double s2 = 1.0 - cz * cz;
    double sz = sqrt(max0(s2));
    double nx = sz * cos(phi), ny = sz * sin(phi), nz = cz;
    double clm = inv[k - 1];
    double cle = sqrt(q * q + clm * clm);
    double clx = q * nx, cly = q * ny, clz = q * nz;
    frame_t f = make_frame(cle, clx, cly, clz, clm);
    for (int j = 0; j < k; ++j) apply_frame(&f, p + 4 * j);
    p[4 * k + 0] = sqrt(q * q + m[k] * m[k]);
    p[4 * k + 1] = -clx;
    p[4 * k + 2] = -cly;
    p[4 * k + 3] = -clz;
  }
  return w;
}


/* Minimal static-partition parallel-for over [0, n) on pthreads (no OpenMP in
 * this toolchain).  Each row is a pure function of its index, so the split
 * never changes a bit of the output. */
typedef void (*hko_body_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct {
  hko_body_fn fn;
  void* ctx;
  int64_t lo, hi;
} hko_slice_t;

static void* hko_slice_main(void* arg) {
  hko_slice_t* s = (hko_slice_t*)arg;
  s->fn(s->ctx, s->lo, s->hi);
  return NULL;
}

static void hko_parallel_for(int64_t n, int threads, hko_body_fn fn, void* ctx) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (threads == 1 || n < 4096) {
    fn(ctx, 0, n);
    return;
  }
  pthread_t tid[256];
  hko_slice_t sl[256];
  int64_t per = (n + threads - 1) / threads;
  int used = 0;
  for (int t = 0; t < threads; ++t) {
    int64_t lo = (int64_t)t * per, hi = lo + per < n ? lo + per : n;
    if (lo >= hi) break;
    sl[t].fn = fn; sl[t].ctx = ctx; sl[t].lo = lo; sl[t].hi = hi;
    if (t == 0) continue;
    pthread_create(&tid[t], NULL, hko_slice_main, &sl[t]);
    used = t;
  }
  fn(ctx, sl[0].lo, sl[0].hi);
  for (int t = 1; t <= used; ++t) pthread_join(tid[t], NULL);
}

/*
 * Rows [ev_begin, ev_begin + ev_count) of phsp_generate (phasespace.py:162-188).
 * cols[0] = weight, cols[1 + 4j + c] = daughter j component c; each points at
 * ev_count doubles.  T and csum come from numpy on the host (phasespace.py:96-97)
 * so their rounding matches the reference exactly.
 */
typedef struct {
  int n, moving;
  const double *masses, *csum;
  double T;
  frame_t mf;
  rng_t rng;
  uint64_t kc, ev_begin;
  double* const* cols;
} gen_ctx_t;

static void gen_body(void* vctx, int64_t lo, int64_t hi) {
  const gen_ctx_t* c = (const gen_ctx_t*)vctx;
  double p[4 * HKO_MAXN];
  for (int64_t i = lo; i < hi; ++i) {
    uint64_t ev = c->ev_begin + (uint64_t)i;
    double w = rest_frame_event(c->n, c->masses, c->T, c->csum, &c->rng, ev + c->kc, p);
    if (c->moving)
      for (int j = 0; j < c->n; ++j) apply_frame(&c->mf, p + 4 * j);
    c->cols[0][i] = w;
    for (int j = 0; j < 4 * c->n; ++j) c->cols[1 + j][i] = p[j];
  }
}

int hko_generate(int n, const double* masses, double T, const double* csum, int moving,
                 const double* mother, double m_mother, uint64_t base, uint64_t kc,
                 uint64_t ev_begin, int64_t ev_count, double* const* cols, int threads,
                 int rng_mode) {
  if (n < 2 || n > HKO_MAXN) return 1;
  gen_ctx_t c;
  c.n = n; c.moving = moving; c.masses = masses; c.csum = csum; c.T = T;
  if (moving) c.mf = make_frame(mother[0], mother[1], mother[2], mother[3], m_mother);
  c.rng.mode = rng_mode; c.rng.base = base; c.kc = kc; c.ev_begin = ev_begin;
  c.cols = cols;
  hko_parallel_for(ev_count, threads, gen_body, &c);
  return 0;
}

/*
 * phsp_decay_chain (phasespace.py:237-288) for rows [ev_begin, ev_begin+count):
 * in_w/in_p4[4] are the parent weight and daughter-k columns; writes out_w and
 * 4*n_sub sub-daughter columns.  Returns -1 on success, else the first row
 * (relative to ev_begin) whose daughter mass fails the check.
 */
typedef struct {
  const double* in_w;
  const double* const* in_p4;
  int n_sub;
  const double *sub_masses, *csum;
  double T;
  rng_t rng;
  uint64_t kc, ev_begin;
  double* out_w;
  double* const* out_cols;
} chain_ctx_t;

static void chain_body(void* vctx, int64_t lo, int64_t hi) {
  const chain_ctx_t* c = (const chain_ctx_t*)vctx;
  double p[4 * HKO_MAXN];
  for (int64_t i = lo; i < hi; ++i) {
    uint64_t ev = c->ev_begin + (uint64_t)i;
    double fe = c->in_p4[0][i], fx = c->in_p4[1][i], fy = c->in_p4[2][i], fz = c->in_p4[3][i];
    double m2 = fe * fe - fx * fx - fy * fy - fz * fz;
    double fm = sqrt(max0(m2));
    double w = rest_frame_event(c->n_sub, c->sub_masses, c->T, c->csum, &c->rng, ev + c->kc, p);
    frame_t f = make_frame(fe, fx, fy, fz, fm);
    for (int j = 0; j < c->n_sub; ++j) apply_frame(&f, p + 4 * j);
    c->out_w[i] = c->in_w[i] * w;
    for (int j = 0; j < 4 * c->n_sub; ++j) c->out_cols[j][i] = p[j];
  }
}

int64_t hko_decay_chain(const double* in_w, const double* const* in_p4, int n_sub,
                        const double* sub_masses, double M_sub, double T, const double* csum,
                        uint64_t base, uint64_t kc, uint64_t ev_begin, int64_t ev_count,
                        double* out_w, double* const* out_cols, int threads, int rng_mode) {
  if (n_sub < 2 || n_sub > HKO_MAXN) return -2;
  const double tol = 1e-9 * (M_sub > 1e-6 ? M_sub : 1e-6);
  for (int64_t i = 0; i < ev_count; ++i) {
    double fe = in_p4[0][i], fx = in_p4[1][i], fy = in_p4[2][i], fz = in_p4[3][i];
    double m2 = fe * fe - fx * fx - fy * fy - fz * fz;
    double fm = sqrt(max0(m2));
    if (fabs(fm - M_sub) > tol) return i; /* NaN passes, as in numpy */
  }
  chain_ctx_t c;
  c.in_w = in_w; c.in_p4 = in_p4; c.n_sub = n_sub; c.sub_masses = sub_masses; c.csum = csum;
  c.T = T; c.rng.mode = rng_mode; c.rng.base = base; c.kc = kc; c.ev_begin = ev_begin;
  c.out_w = out_w; c.out_cols = out_cols;
  hko_parallel_for(ev_count, threads, chain_body, &c);
  return -1;
}

/* phsp_unweight accept flags (phasespace.py:225-227): u_i * w_max < w_i. */
void hko_unweight_flags(const double* w, int64_t n, double w_max, uint64_t base, uint64_t kc,
                        uint64_t ev_begin, uint8_t* accept) {
  for (int64_t i = 0; i < n; ++i)
    accept[i] = (u01(base, ev_begin + (uint64_t)i + kc) * w_max < w[i]) ? 1 : 0;
}

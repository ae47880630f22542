/*
 * hepkit_cuda.h -- C ABI of libhepkit_cuda.so, the B200 (sm_100a) hot path of
 * the reference's event-parallel map/reduce (arXiv:1711.05683 -> `hepkit`).
 *
 * The reference has no FFI: its seam is the public Python API whose bodies all
 * go through parallel.run_batches (parallel.py:56-71).  Each entry point below
 * replaces the *body* of one such function; the Python package
 * paper_1711_05683_b200 keeps the reference names/signatures/exceptions and
 * calls these through ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - plain C types only; every array argument is a raw pointer + a size;
 *    "d_" pointers are device (HBM) addresses, "h_" pointers host addresses;
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *  - calls are asynchronous on `stream` unless documented otherwise;
 *  - return value: HK_OK (0) or an HK_E* code; hk_last_error() gives text.
 *  - event ("row") indices are 64-bit and global: row r of a run draws the RNG
 *    counters (r + key.counter) * D + j (phasespace.py:105-109), so any window
 *    [ev_begin, ev_begin + ev_count) -- a GPU shard, say -- is bit-identical to
 *    the same rows of a one-shot run.
 *  - reductions produce one partial per HK_CHUNK rows (parallel.py:18) in a
 *    fixed in-block tree order, then hk_fold_partials folds them in a fixed
 *    tree; results are deterministic and independent of the launch grid.
 */
#ifndef HEPKIT_CUDA_H
#define HEPKIT_CUDA_H

#ifndef __CUDACC_RTC__ /* NVRTC (hk_jit.cu) supplies the fixed-width types */
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define HK_ABI_VERSION 1

/* status codes */
#define HK_OK 0
#define HK_EINVAL 1       /* bad argument (sizes, pointers, arity) */
#define HK_ECUDA 2        /* CUDA runtime error (see hk_last_error) */
#define HK_EDOMAIN 3      /* per-event domain failure; first bad row reported */
#define HK_EUNSUPPORTED 4 /* configuration outside the compiled kernels */

#define HK_CHUNK 4096        /* rows per reduction partial (parallel.py:18) */
#define HK_WARP_SLICES 8     /* per-warp weight partials per chunk (generation kernels) */
#define HK_SUPERS 1024       /* fixed super-chunks per run: the multi-GPU exchange grid (hk_fold_supers) */
#define HK_MAX_DAUGHTERS 16  /* templated fast path covers n <= 8 */
#define HK_MAX_PROGRAM 256   /* ops per device functor program */
#define HK_MAX_SLOTS 32      /* virtual registers per program */
#define HK_MAX_COMPONENTS 8  /* p.d.f. components per extended model */
#define HK_NO_BAD_ROW UINT64_MAX

/* RNG selection: the reference SplitMix64 stream (rng.py:98-125), bit-exact,
 * or the production Philox4x32-10 stream (SPEC.md:343 allows any
 * counter-based bijection). */
#define HK_RNG_REFERENCE 0
#define HK_RNG_PHILOX 1

/* RngKey (rng.py:45-62); all fields already reduced mod 2^64 (rng.py:105). */
typedef struct hk_key {
  uint64_t seed;
  uint64_t stream;
  uint64_t counter;
  int32_t mode; /* HK_RNG_* */
  int32_t _pad;
} hk_key_t;

/* DecaySpec (phasespace.py:36-57) plus the mother four-vector of
 * phsp_generate (phasespace.py:162-188).  T and csum are computed on the host
 * with numpy (phasespace.py:94-97) so their rounding is the reference's. */
typedef struct hk_decay {
  int32_t n;      /* daughters, 2..HK_MAX_DAUGHTERS */
  int32_t moving; /* boost every daughter by the mother (phasespace.py:181) */
  double mother_mass;
  double T;
  double masses[HK_MAX_DAUGHTERS];
  double csum[HK_MAX_DAUGHTERS];
  double mother[4]; /* e, px, py, pz */
  double m_mother;  /* invariant_mass(mother) (phasespace.py:175) */
} hk_decay_t;

/* Device functor program: an SSA register program lowered on the host from a
 * FunctorExpr tree (functors.py:79-249) composed with a traced arg_builder.
 * Each op writes slot dst[i] from slots a[i], b[i]. */
enum hk_opcode {
  HK_OP_COL = 0,    /* dst = column[a]  (0 = weight, 1 + 4(j-1) + c = p_j comp c) */
  HK_OP_CONST = 1,  /* dst = cst[i] */
  HK_OP_ADD = 2,    /* dst = a + b */
  HK_OP_SUB = 3,    /* dst = a - b */
  HK_OP_MUL = 4,    /* dst = a * b */
  HK_OP_DIV = 5,    /* dst = a / b; b == 0 is a domain error (_BinaryOp "/", functors.py:200-207) */
  HK_OP_NEG = 6,    /* dst = -a */
  HK_OP_SQRT = 7,   /* dst = sqrt(a) */
  HK_OP_EXP = 8,    /* dst = exp(a) */
  HK_OP_LOG = 9,    /* dst = log(a) */
  HK_OP_GAUSS = 10, /* dst = exp(-0.5 z z)/(s sqrt(2pi)), z=(a-cst[i])/cst2[i] (functors.py:137-143) */
  HK_OP_EXPO = 11,  /* dst = exp(-a / cst[i]) (functors.py:157-161) */
  HK_OP_BW = 12,    /* dst = 1/((a - m0^2)^2 + m0^2 g0^2), m0=cst[i], g0=cst2[i] */
  HK_OP_ADD0 = 13,  /* dst = a + 0.0 (Coordinate, functors.py:248-249) */
  HK_OP_SQUARE = 14, /* dst = a * a */
  HK_OP_UDIV = 15    /* dst = a / b, unchecked: numpy division inside a traced closure or
                        arg_builder, or a shape body (IEEE inf/nan, no EvaluationError) */
};

typedef struct hk_program {
  int32_t n_ops;
  int32_t result; /* slot holding the value */
  int32_t op[HK_MAX_PROGRAM];
  int32_t dst[HK_MAX_PROGRAM];
  int32_t a[HK_MAX_PROGRAM];
  int32_t b[HK_MAX_PROGRAM];
  double cst[HK_MAX_PROGRAM];
  double cst2[HK_MAX_PROGRAM];
} hk_program_t;

/* ExtendedModel (fitting.py:126-166) lowered for the FCN: per component the
 * yield N_k (a Parameter value), the host-computed norm_k (fitting.py:80-89)
 * and the shape kind/parameters. */
#define HK_SHAPE_GAUSS 0 /* p0 = mean, p1 = sigma */
#define HK_SHAPE_EXPO 1  /* p0 = tau */
typedef struct hk_model {
  int32_t n_comp;
  int32_t _pad;
  int32_t kind[HK_MAX_COMPONENTS];
  double yield[HK_MAX_COMPONENTS];
  double norm[HK_MAX_COMPONENTS];
  double p0[HK_MAX_COMPONENTS];
  double p1[HK_MAX_COMPONENTS];
  /* optional statistics of the observable column the FCN will read
   * (hk_column_stats; has_stats = 0: none).  With them the host can prove,
   * for the whole data range, that no event's density is non-positive or
   * non-finite, and the Gaussian + exponential FCN drops its per-event
   * checks and hoists sum_e B(x_e) = -sum(x) / tau out of the event loop.
   * x_count must equal the n of the call or the statistics are ignored. */
  int32_t has_stats;
  int32_t _pad2;
  int64_t x_count;
  double x_min, x_max, x_sum;
} hk_model_t;

/* ---------------------------------------------------------------- runtime */
int hk_abi_version(void);
/* Copy the last error message of this thread into buf (NUL-terminated). */
int hk_last_error(char* buf, size_t len);
/* Number of CUDA devices visible; sets *sm_count to device 0's SM count. */
int hk_device_info(int* n_devices, int* sm_count);
/* Number of 4096-row chunk partials for ev_count rows. */
int64_t hk_num_chunks(int64_t ev_count);

/* ------------------------------------------------- lifetime + collectives
 * For a C host that drives several GPUs from ONE process -- the analogue of
 * the reference's `workers` pool (parallel.py:18-92), with devices in place
 * of processes.  The Python drop-in does not use these: it runs one process
 * per GPU and exchanges the same partials with torch.distributed (parallel.py
 * in this package).  NCCL (libnccl.so.2) is dlopen'ed by hk_init, so the
 * library has no link-time NCCL dependency.
 *
 * hk_init(n): one NCCL communicator per device 0..n-1 (ncclCommInitAll), a
 * clique the two collectives below run over; n = 1 is valid (a one-rank
 * clique).  HK_EINVAL when n exceeds the visible devices, HK_ECUDA when NCCL
 * is unavailable.  Calling it again with another n rebuilds the clique.
 * hk_shutdown(): destroys the clique and releases the library's cached state
 * (NVRTC-specialised modules, this thread's mapped FCN mailboxes and copy
 * streams).  The library stays usable; those caches rebuild on demand. */
int hk_init(int32_t n_devices);
int hk_shutdown(void);
/* Devices in the current clique (0 before hk_init / after hk_shutdown). */
int32_t hk_clique_size(void);

/* In-place sum of `count` doubles across the clique: d_bufs[g] lives on
 * device g, streams[g] is device g's stream (NULL = legacy default).  Returns
 * after the work is enqueued (stream-ordered, like a kernel launch).  A sum
 * over devices is deterministic for a fixed clique size but not invariant to
 * it; use hk_allgather_partials + hk_fold_partials for bitwise device-count
 * invariance (SURVEY.md 8(e) option ii). */
int hk_allreduce_partials(double* const* d_bufs, int32_t n_dev, int64_t count,
                          void* const* streams);
/* Every device receives all devices' partials in device order:
 * d_recv[g][h * count + i] = d_send[h][i].  d_recv[g] holds n_dev * count
 * doubles.  When the devices hold consecutive, equal-length runs of chunk
 * partials (shards split on HK_CHUNK boundaries), folding d_recv[g] in order
 * (hk_fold_partials) gives every device the same total, bit-identical to the
 * one-device fold of the whole chunk sequence. */
int hk_allgather_partials(const double* const* d_send, double* const* d_recv, int32_t n_dev,
                          int64_t count, void* const* streams);

/* -------------------------------------------------------------------- RNG */
/* rng.py:115-120 raw64 / :123-125 uniform_array at key.counter + d_counters[i].
 * Mode HK_RNG_PHILOX is not a reference stream (uniform only, for tests). */
int hk_rng_raw64(const hk_key_t* key, const uint64_t* d_counters, int64_t n, uint64_t* d_out,
                 void* stream);
int hk_rng_uniform(const hk_key_t* key, const uint64_t* d_counters, int64_t n, double* d_out,
                   void* stream);

/* Raw Philox4x32-10 (Salmon et al., SC'11; Random123 philox4x32, R = 10), the
 * round function of the production stream: row i of d_ctr_key is
 * (ctr0..ctr3, key0, key1) as uint32, row i of d_out the 4 output words.  For
 * known-answer tests of the device implementation.  The production stream
 * maps draw j of event e (key.counter added) to words 2(j & 1), 2(j & 1) + 1
 * of block ctr = (e lo, e hi, j >> 1, 0x686b7068), key = base(seed, stream). */
int hk_philox4x32_10(const uint32_t* d_ctr_key, int64_t n, uint32_t* d_out, void* stream);

/* ------------------------------------------------------------- generation */
/* phsp_generate (phasespace.py:162-188) for rows [ev_begin, ev_begin+ev_count):
 * writes 4n+1 columns, d_cols[0] = weight, d_cols[1+4j+c] = daughter j+1,
 * component c (e, px, py, pz) (phsp_schema, phasespace.py:60-64).
 * d_wpartials (optional, NULL to skip): (sum w, sum w^2) per warp-slice --
 * HK_WARP_SLICES slices per 4096-row chunk, 2 * HK_WARP_SLICES * chunks
 * doubles -- the weight-integration moments fused into the same pass without
 * a CTA barrier; fold them with hk_fold_partials(n_parts = slices, width 2). */
int hk_phsp_generate(const hk_decay_t* spec, const hk_key_t* key, uint64_t ev_begin,
                     int64_t ev_count, double* const* d_cols, double* d_wpartials, void* stream);

/* Same rows written to HOST memory (h_cols[4n+1], pinned for full speed):
 * generation into a double-buffered device staging area (d_stage, stage_bytes)
 * overlapped with device->host copies on a second stream.  Synchronous.
 * h_wsums (optional): 2 doubles, folded (sum w, sum w^2). */
int hk_phsp_generate_host(const hk_decay_t* spec, const hk_key_t* key, uint64_t ev_begin,
                          int64_t ev_count, double* const* h_cols, double* h_wsums,
                          void* d_stage, size_t stage_bytes, void* stream);

/* phsp_decay_chain (phasespace.py:237-288), standalone on an existing block:
 * reads parent weight d_w_in and the daughter's four columns d_p4_in[4];
 * writes d_w_out and 4*n_sub sub-daughter columns d_sub_cols (the caller
 * splices them into the schema).  Rows failing the mass check
 * (phasespace.py:259-268) are reported through *d_first_bad (atomicMin;
 * initialise to HK_NO_BAD_ROW). */
int hk_phsp_decay_chain(const double* d_w_in, const double* const* d_p4_in,
                        const hk_decay_t* sub, const hk_key_t* sub_key, uint64_t ev_begin,
                        int64_t ev_count, double* d_w_out, double* const* d_sub_cols,
                        uint64_t* d_first_bad, void* stream);

/* Fused generate + decay_chain (config C3): parent spec/key generate, daughter
 * `daughter_index` (1-based) decays by sub/sub_key, output in the spliced
 * schema order (4*(n-1+n_sub)+1 columns). */
int hk_phsp_generate_chain(const hk_decay_t* spec, const hk_key_t* key, int32_t daughter_index,
                           const hk_decay_t* sub, const hk_key_t* sub_key, uint64_t ev_begin,
                           int64_t ev_count, double* const* d_cols, double* d_wpartials,
                           uint64_t* d_first_bad, void* stream);

/* Statistics of one fp64 column for hk_model_t: h_out = {min, max, sum,
 * number of non-finite values} over the finite values (sum in a fixed
 * chunk-then-tree order: deterministic).  d_work: hk_column_stats_work_doubles(n)
 * doubles of device scratch.  Synchronous on `stream`. */
int64_t hk_column_stats_work_doubles(int64_t n);
int hk_column_stats(const double* d_x, int64_t n, double* d_work, double* h_out, void* stream);

/* The frame mass hk_phsp_generate_chain uses for the decaying daughter
 * instead of recomputing sqrt(E^2 - p^2) per event (phasespace.py:259-262):
 * m_k when the host proves no event can fail the mass check and the
 * recomputed mass moves boosted momenta by < 1e-14 E (then *d_first_bad is
 * never written and the caller need not read it back), else 0.0 (per-event
 * mass and check).  Pure host function. */
double hk_chain_fixed_frame_mass(const hk_decay_t* spec, int32_t daughter_index, const hk_decay_t* sub);

/* --------------------------------------------------------------- averages */
/* phsp_average moments (phasespace.py:310-329) over stored columns: per chunk
 * 5 doubles (sum w, sum w f, sum w^2, sum w^2 f, sum w^2 f^2), f = program.
 * Non-finite f (phasespace.py:314-316) or a zero divisor is reported via
 * *d_first_bad. */
int hk_phsp_moments(const double* const* d_cols, int32_t n_cols, int64_t ev_count,
                    const hk_program_t* f, double* d_partials, uint64_t* d_first_bad,
                    void* stream);

/* map_evaluate (functors.py:288-318): d_out[i] = program(columns at row i).
 * Zero divisors -> d_first_bad (may be NULL). */
int hk_map_program(const double* const* d_cols, int32_t n_cols, int64_t n, const hk_program_t* f,
                   double* d_out, uint64_t* d_first_bad, void* stream);

/* Runtime specialisation of functor programs, the GPU analogue of Hydra's
 * compile-time functor instantiation: hk_phsp_moments / hk_map_program emit
 * the program as straight-line CUDA, compile it with NVRTC for sm_100a
 * (no FMA contraction, same rounding as the interpreter: results are
 * bit-identical) and cache the cubin per program.  mode 0 = always interpret,
 * 1 = always specialise (HK_ECUDA if NVRTC is unavailable), 2 = auto
 * (specialise when >= HK_JIT_MIN_ROWS rows or already compiled; default, the
 * HK_JIT environment variable "0"/"1"/"auto" sets the initial mode).
 * Returns the previous mode, or -1 for a bad mode. */
#define HK_JIT_MIN_ROWS (1LL << 22)
int hk_set_jit_mode(int32_t mode);
/* programs specialised so far in this process (cache entries) */
int64_t hk_jit_count(void);
/* The CUDA source emitted for a program (into buf, NUL-terminated, at most
 * cap bytes); returns the full length, -1 for a bad program/target.
 * n_daughters = 0: the stored-block module (hk_phsp_moments / hk_map_program);
 * 2..8: the fused generate+integrate module (hk_phsp_integrate) for that
 * final state and rng_mode (HK_RNG_*). */
int64_t hk_jit_source(const hk_program_t* f, int32_t n_daughters, int32_t rng_mode, char* buf,
                      int64_t cap);
/* NVRTC-compile that module for sm_100a without loading it (needs no GPU);
 * *cubin_bytes = cubin size. */
int hk_jit_compile(const hk_program_t* f, int32_t n_daughters, int32_t rng_mode, int64_t* cubin_bytes);

/* Dalitz-plane integrands with a specialised (non-interpreted) device path:
 * s = m^2 of daughters i+j (0-based) in the op order of the reference's
 * pinned integrand (test_phasespace.py:196-201); f = s + 0.0 (identity) or a
 * Breit-Wigner 1/((s - m0^2)^2 + m0^2 g0^2).  The host recognises these
 * structurally in a lowered expression. */
#define HK_PAIR_NONE 0
#define HK_PAIR_MASS2 1
#define HK_PAIR_BW 2
typedef struct hk_pair_integrand {
  int32_t kind;
  int32_t i;
  int32_t j;
  int32_t _pad;
  double m0;
  double g0;
} hk_pair_integrand_t;

/* Fused generate -> f -> moments with no event store (config C5).  f is the
 * program, or `pair` (non-NULL, kind != HK_PAIR_NONE) selects the fast path. */
int hk_phsp_integrate(const hk_decay_t* spec, const hk_key_t* key, uint64_t ev_begin,
                      int64_t ev_count, const hk_program_t* f, const hk_pair_integrand_t* pair,
                      double* d_partials, uint64_t* d_first_bad, void* stream);

/* Fixed-order fold of each segment of seg_len consecutive partials (width
 * doubles each) into one: d_out[s * width + w] = sum over j ascending of
 * d_partials[(s * seg_len + j) * width + w].  Used to turn a chunk's
 * HK_WARP_SLICES weight partials into one chunk partial before partials cross
 * GPUs, so the global fold sees the same chunk sequence at any GPU count. */
int hk_fold_segments(const double* d_partials, int64_t n_segments, int32_t seg_len, int32_t width,
                     double* d_out, void* stream);

/* Super-chunk fold, the GPU-count-invariant exchange unit (SURVEY.md 8(e)
 * option ii; replaces the ordered fold of parallel.py:74-92 across devices).
 * A run's n_chunks_total 4096-row chunks are cut into HK_SUPERS fixed
 * super-chunks: super s covers global chunks [s*N/S, (s+1)*N/S) (floor).
 * d_partials holds recs_per_chunk records of `width` doubles per chunk for
 * global chunks [chunk_begin, chunk_begin + n_chunks_local) -- which must be
 * exactly supers [s_begin, s_begin + s_count) -- and d_out receives one
 * record per super (s_count * width doubles), each the fixed-order sum of its
 * records.  A GPU shard made of whole supers folds them locally; the
 * HK_SUPERS records (40 KB at width 5) are all-gathered and hk_fold_partials
 * folds them identically on every device, so totals are bitwise independent
 * of the device count (1/2/4/8 divide HK_SUPERS). */
#define HK_SUPERS 1024
int hk_fold_supers(const double* d_partials, int64_t n_chunks_total, int64_t chunk_begin,
                   int64_t n_chunks_local, int32_t recs_per_chunk, int32_t width, int32_t s_begin,
                   int32_t s_count, double* d_out, void* stream);

/* Deterministic fold of n_parts partials of `width` (<= 72: K + K^2 for 8 components) doubles each
 * (parallel.py:86-92 semantics, fixed tree order) into d_out[width]. */
int hk_fold_partials(const double* d_partials, int64_t n_parts, int32_t width, double* d_out,
                     void* stream);

/* ------------------------------------------------------------------- FCN */
/* The FCN reduces per HK_FCN_TILE rows (a divisor of HK_CHUNK, so chunk-
 * aligned shards stay tile-aligned): ceil(n / HK_FCN_TILE) partials. */
#define HK_FCN_TILE 4096

/* Extended NLL event sum (fitting.py:197-207): per tile sum_e ln density(x_e);
 * density <= 0 or non-finite -> *d_first_bad (fitting.py:200-205). */
int hk_nll_partials(const double* d_x, int64_t n, const hk_model_t* model, double* d_partials,
                    uint64_t* d_first_bad, void* stream);

/* The FCN of ANY traceable model (fitting.py:160-166 with any FunctorExpr
 * shape -- closures, compositions, sums/products -- and any observable
 * arity): the density is a lowered functor program whose constants (yields,
 * host norms, shape parameters) sit in program.cst and change per call while
 * the op structure stays fixed.  pdf_slot[k] holds pdf_k = shape_k / norm_k and
 * program.result the density sum_k N_k pdf_k in the reference's order after the
 * program runs; HK_OP_COL c reads observable column c. */
#define HK_FCN_MAX_OBS 8
typedef struct hk_density {
  int32_t n_obs;  /* observable columns, 1..HK_FCN_MAX_OBS */
  int32_t n_comp; /* components K, 1..HK_MAX_COMPONENTS */
  int32_t pdf_slot[HK_MAX_COMPONENTS];
  double yield[HK_MAX_COMPONENTS]; /* N_k (the ratio sums' density p @ N, fitting.py:416) */
  hk_program_t program;
} hk_density_t;

/* hk_nll_eval for an hk_density_t over d_obs[n_obs] columns: same workspace,
 * schedule and fold; *h_first_div0 = first row with a zero divisor
 * (functors.py:200-207) or HK_NO_BAD_ROW.  The program runs through the
 * interpreter or, per the hk_set_jit_mode policy, an NVRTC-specialised kernel
 * compiled once per op structure (constants stay kernel arguments). */
int hk_nll_program_eval(const double* const* d_obs, int64_t n, const hk_density_t* model,
                        double* d_work, double* h_logsum, uint64_t* h_first_bad,
                        uint64_t* h_first_div0, void* stream);

/* Both FCN entry points are asynchronous when h_logsum is NULL: the result
 * stays on the device in d_work[0] (sum of logs), d_work[1] (first bad row,
 * u64 bits) and d_work[5] (first zero divisor, u64 bits).  That is the
 * row-sharded multi-GPU FCN's step 1; step 2 all-gathers d_work[0..7] of every
 * rank (the caller stores its shard's first global row as a double in
 * d_work[6]) with one stream-ordered NCCL collective, and step 3 is: */

/* Rank-order fold of world gathered 8-double FCN records (d_gathered[8 r ..]):
 * *h_logsum = sum over r in order of [0]; *h_first_bad / *h_first_div0 = the
 * smallest global row ([6] + local row) over ranks, or HK_NO_BAD_ROW.  One
 * kernel that publishes into the mapped mailbox: the sharded FCN has a single
 * host synchronisation per evaluation.  Synchronous. */
int hk_nll_combine(const double* d_gathered, int32_t world, double* h_logsum, uint64_t* h_first_bad,
                   uint64_t* h_first_div0, void* stream);

/* Yield-stationarity / sPlot sums for an hk_density_t (any shape, K <= 8 per pass; the host
 * covers more components with passes whose slot 0 is the density at yield 1, fitting.py
 * _ratio_sums_passes):
 * per chunk K values sum_e r_k and K*K values sum_e r_k r_j, r_k = pdf_k / d,
 * d = sum_k N_k pdf_k; d_first_bad[0]: d not > 0; [1]: d not > 0 or
 * non-finite; [2]: first zero divisor (all initialised to HK_NO_BAD_ROW). */
int hk_ratio_partials_program(const double* const* d_obs, int64_t n, const hk_density_t* model,
                              double* d_partials, uint64_t* d_first_bad, void* stream);

/* sWeights for an hk_density_t (K <= 8): d_out[s][i] = sum_j V[s*K+j] pdf_j / d. */
int hk_splot_weights_program(const double* const* d_obs, int64_t n, const hk_density_t* model,
                             const double* V, double* const* d_out, uint64_t* d_first_bad,
                             void* stream);

/* One FCN evaluation end to end.  Synchronous.  *h_logsum = sum_e ln density;
 * *h_first_bad = first failing row or HK_NO_BAD_ROW.  One kernel launch (the
 * last CTA folds the tile partials in a fixed order and publishes the result
 * into mapped pinned host memory, which the caller's thread polls).  d_work
 * needs hk_nll_work_doubles(n) doubles, ZERO-FILLED before its first use;
 * the kernel re-arms it for the next call.  Rows are scheduled as whole
 * waves of HK_FCN_TILE-row tiles plus the leftover spread over one wave, so
 * the sum's grouping (not its value beyond rounding) depends on the SM count. */
int hk_nll_eval(const double* d_x, int64_t n, const hk_model_t* model, double* d_work,
                double* h_logsum, uint64_t* h_first_bad, void* stream);
/* The FCN at k parameter points in one pass over the data (the numeric
 * Hessian's 2n^2+1 points, a simplex's initial vertices -- fitting.py:251-395
 * call the FCN serially): h_logsums[p], h_first_bad[p] as hk_nll_eval would
 * return for models[p], bit for bit.  The factored Gaussian + exponential
 * model runs as one kernel (CTA = 4096-row tile x group of 4 points); other
 * models run one hk_nll_eval per point.  d_work: hk_nll_many_work_doubles(n,
 * k) doubles, zero-filled before first use.  Synchronous. */
#define HK_MAX_POINTS 64
int hk_nll_eval_many(const double* d_x, int64_t n, const hk_model_t* models, int32_t k, double* d_work,
                     double* h_logsums, uint64_t* h_first_bad, void* stream);
int64_t hk_nll_many_work_doubles(int64_t n, int32_t k);

/* Resident FCN session (a minimiser's serial FCN calls, fitting.py:251-340,
 * without a kernel launch per call): hk_fcn_session_start binds the data
 * column and a zero-filled hk_nll_work_doubles(n) workspace and launches
 * persistent CTAs (one per SM slot, cooperative launch) on a library stream;
 * hk_fcn_session_eval(model) posts the parameter point into mapped host
 * memory and waits for the answer -- the same value as hk_nll_eval, bit for
 * bit.  Gaussian + exponential models only (HK_EUNSUPPORTED otherwise).  The
 * CTAs occupy the GPU: other kernels wait until hk_fcn_session_stop, or until
 * idle_us without a command passes (the next eval relaunches them).  One
 * session per host thread, on the device current at start. */
int hk_fcn_session_start(const double* d_x, int64_t n, double* d_work, int64_t idle_us);
int hk_fcn_session_eval(const hk_model_t* model, double* h_logsum, uint64_t* h_first_bad);
int hk_fcn_session_stop(void);
/* diagnostics: device-side ns from command pickup to answer, last session eval */
int64_t hk_fcn_session_device_ns(void);

/* workspace size of hk_nll_eval / hk_nll_program_eval for n rows (8 + one
 * partial per scheduled CTA) */
int64_t hk_nll_work_doubles(int64_t n);

/* Yield-stationarity sums (fitting.py:401-434) and the sWeights matrix
 * accumulation (splot.py:45-87) for K <= 4 components: per chunk K values
 * sum_e r_k and K*K values sum_e r_k r_j, r_k = pdf_k(x)/density(x),
 * pdf_k = shape_k/norm_k.  Width K + K*K doubles per chunk.
 * d_first_bad[0]: first row with density not > 0 (NaN included,
 * fitting.py:418-420); d_first_bad[1]: same or non-finite (splot.py:38). */
int hk_yield_partials(const double* d_x, int64_t n, const hk_model_t* model, double* d_partials,
                      uint64_t* d_first_bad, void* stream);

/* sWeights table (splot.py:90-117): d_out[s][i] = sum_j V[s*K+j] pdf_j(x_i) / density(x_i)
 * for K <= 4 species; V is a host K*K row-major matrix.  Non-positive or
 * non-finite density -> *d_first_bad. */
int hk_splot_weights(const double* d_x, int64_t n, const hk_model_t* model, const double* V,
                     double* const* d_out, uint64_t* d_first_bad, void* stream);

/* density(x) for n values (the value the error message quotes). */
int hk_model_density(const double* d_x, int64_t n, const hk_model_t* model, double* d_out,
                     void* stream);

/* ------------------------------------------------------------- sampling */
/* sample_pdf (rng.py:177-242): rows [ev_begin, ev_begin+count) of an
 * accept-reject sample of program f on the box lo + [0, span)^dim.
 * d_bad[0]: packed (batch << 40 | round << 24 | row % 65536) of the first
 * proposal above `ceiling` (CeilingError); d_bad[1]: first row with no
 * acceptance in max_rounds.  Both initialised to HK_NO_BAD_ROW. */
int hk_sample_pdf(const hk_program_t* f, int32_t dim, const double* lo, const double* span,
                  double ceiling, const hk_key_t* key, uint64_t ev_begin, int64_t count,
                  int32_t max_rounds, double* const* d_out, uint64_t* d_bad, void* stream);

/* ----------------------------------------------------------- unweighting */
/* phsp_unweight accept test (phasespace.py:225-227): u_i * w_max < w_i with
 * u_i at key.counter + ev_begin + i.  Writes d_flags (uint8), per-chunk
 * accept counts into d_counts (int64 per chunk) and reports w > w_max rows
 * via *d_first_bad (phasespace.py:217-221). */
int hk_unweight_flags(const double* d_w, int64_t n, double w_max, const hk_key_t* key,
                      uint64_t ev_begin, uint8_t* d_flags, int64_t* d_counts,
                      uint64_t* d_first_bad, void* stream);

/* Order-preserving compaction of n_cols columns by d_flags given the exclusive
 * prefix of per-chunk counts d_offsets (int64 per chunk); accepted rows of
 * d_in[c] land in d_out[c]; weight column index `weight_col` (or -1) is set to 1.0
 * (phasespace.py:230-234). */
int hk_compact(const double* const* d_in, int32_t n_cols, int64_t n, const uint8_t* d_flags,
               const int64_t* d_offsets, double* const* d_out, int32_t weight_col, void* stream);

/* Exclusive scan of n int64 values (per-chunk counts) -> d_out; total -> d_total. */
int hk_scan_counts(const int64_t* d_counts, int64_t n, int64_t* d_out, int64_t* d_total,
                   void* stream);

/* ------------------------------------------------------------------- CSV */
/* The body of ColumnStore.write_csv (store.py:181-204) for real64 columns:
 * rows [0, n_rows) of the n_cols device columns as text, each value exactly
 * Python's f"{v:.17g}" (correctly rounded 17 significant digits; nan, inf,
 * -inf, -0), ',' between columns, '\n' after every row -- no header.
 * d_scratch: hk_csv_scratch_bytes(n_rows, n_cols) bytes; d_out: at least
 * n_rows * n_cols * 25 bytes.  Synchronous: *h_len = bytes of text written. */
int64_t hk_csv_scratch_bytes(int64_t n_rows, int32_t n_cols);
int hk_format_csv(const double* const* d_cols, int32_t n_cols, int64_t n_rows, void* d_scratch,
                  char* d_out, int64_t out_cap, int64_t* h_len, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HEPKIT_CUDA_H */

// hk_jit.cu -- runtime specialisation of functor programs.
//
// Hydra instantiates the user's functor into the kernel at C++ compile time.
// The Python API receives functors at run time, so the device path lowers
// them to an hk_program_t (functors.py:lower) which the interpreter in
// hk_device.cuh runs op by op.  The interpreter is instruction-bound
// (warp-uniform dispatch + local-memory slots, ~20 instructions per op); for
// big blocks this file emits the program as straight-line CUDA, compiles it
// with NVRTC for sm_100a and caches the cubin per program, so the average
// over a stored block runs at HBM speed.
//
// Bit-identity with the interpreter: every operation is written with the
// explicit round-to-nearest intrinsics in the interpreter's order, NVRTC runs
// with --fmad=false (the interpreter's TU is built with -fmad=false), exp/log
// come from the same libdevice, and the chunk moments use the same per-thread
// order and the same block tree as k_moments / block_sum_store<5>.
// tests/test_jit_gpu.py checks interpreter == specialised bitwise.
//
// NVRTC is dlopen'ed on first use, so the library keeps no link-time
// dependency on it (the CPU ABI tests load the .so without a CUDA driver).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "hepkit_cuda.h"
#include "hk_host.h"

namespace hk {

namespace {

// ------------------------------------------------------------ NVRTC access --
struct Nvrtc {
  bool tried = false;
  void* so = nullptr;
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcGetErrorString) err = nullptr;
};

template <class F>
bool sym(void* so, const char* name, F* out) {
  *out = reinterpret_cast<F>(dlsym(so, name));
  return *out != nullptr;
}

// The toolkit's own NVRTC first (same libdevice as nvcc built the
// interpreter with), then whatever the loader finds.
bool load_nvrtc(Nvrtc& N) {
  if (N.tried) return N.so != nullptr;
  N.tried = true;
  const char* names[] = {"/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12", "libnvrtc.so"};
  for (const char* n : names) {
    N.so = dlopen(n, RTLD_NOW | RTLD_LOCAL);
    if (N.so) break;
  }
  if (!N.so) return false;
  bool ok = sym(N.so, "nvrtcCreateProgram", &N.create) && sym(N.so, "nvrtcCompileProgram", &N.compile) &&
            sym(N.so, "nvrtcGetCUBINSize", &N.cubin_size) && sym(N.so, "nvrtcGetCUBIN", &N.cubin) &&
            sym(N.so, "nvrtcGetProgramLogSize", &N.log_size) && sym(N.so, "nvrtcGetProgramLog", &N.log) &&
            sym(N.so, "nvrtcDestroyProgram", &N.destroy) && sym(N.so, "nvrtcGetErrorString", &N.err);
  if (!ok) {
    dlclose(N.so);
    N.so = nullptr;
  }
  return ok;
}

// -------------------------------------------------------------- code emit --
std::string hex_const(double v) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  char buf[64];
  std::snprintf(buf, sizeof(buf), "__longlong_as_double(0x%016llxll)", (unsigned long long)bits);
  return buf;
}

// Straight-line program: one const double per op, slots renamed to the op
// that last wrote them (the program is in execution order).  Column c reads
// HBM (stored block) or the register-resident event (fused: c = 0 is the
// weight w, c = 1 + 4 j + k is p[4 j + k]).  Zero divisors set d0.
// params: constants come from the kernel arguments (a.prog.cst[i]) instead of
// being baked in -- the FCN module, compiled once per op structure.
// params (the FCN module): constants are kernel arguments, and an unchecked
// division by a value computed from constants only (a p.d.f. norm, a shape's
// sigma) becomes a product with its reciprocal -- loop-invariant, so the
// compiler computes it once per thread.  Each such quotient moves by <= 1
// ulp, far inside the FCN's 1e-10 budget; the value an error message quotes
// comes from the map module, which keeps every division exact.
std::string emit_body(const hk_program_t& P, bool fused, bool params = false) {
  std::string s;
  int slot_of[HK_MAX_SLOTS];
  for (int& x : slot_of) x = -1;
  bool cst_only[HK_MAX_PROGRAM] = {};
  auto v = [&](int slot) -> std::string {
    return slot_of[slot] < 0 ? std::string("0.0") : "v" + std::to_string(slot_of[slot]);
  };
  for (int i = 0; i < P.n_ops; ++i) {
    const bool leaf = P.op[i] == HK_OP_COL || P.op[i] == HK_OP_CONST;
    const std::string A = leaf ? "" : v(P.a[i]);
    const std::string B = leaf ? "" : v(P.b[i]);
    const std::string c1 = params ? "a.prog.cst[" + std::to_string(i) + "]" : hex_const(P.cst[i]);
    const std::string c2 = params ? "a.prog.cst2[" + std::to_string(i) + "]" : hex_const(P.cst2[i]);
    std::string e;
    switch (P.op[i]) {
      case HK_OP_COL:
        if (fused)
          e = P.a[i] == 0 ? std::string("w") : "p[" + std::to_string(P.a[i] - 1) + "]";
        else
          e = "__ldg(a.cols[" + std::to_string(P.a[i]) + "] + r)";
        break;
      case HK_OP_CONST: e = c1; break;
      case HK_OP_ADD: e = "__dadd_rn(" + A + ", " + B + ")"; break;
      case HK_OP_SUB: e = "__dsub_rn(" + A + ", " + B + ")"; break;
      case HK_OP_MUL: e = "__dmul_rn(" + A + ", " + B + ")"; break;
      case HK_OP_DIV:
        s += "  if (" + B + " == 0.0) d0 = true;\n";
        e = "__ddiv_rn(" + A + ", " + B + ")";
        break;
      case HK_OP_NEG: e = "-" + A; break;
      case HK_OP_SQRT: e = "__dsqrt_rn(" + A + ")"; break;
      case HK_OP_EXP: e = "exp(" + A + ")"; break;
      case HK_OP_LOG: e = "log(" + A + ")"; break;
      case HK_OP_GAUSS:  // exp(-0.5 z z) / (s sqrt(2 pi)), z = (a - mu) / s
        e = "__ddiv_rn(exp(__dmul_rn(__dmul_rn(-0.5, __ddiv_rn(__dsub_rn(" + A + ", " + c1 + "), " + c2 +
            ")), __ddiv_rn(__dsub_rn(" + A + ", " + c1 + "), " + c2 + "))), __dmul_rn(" + c2 +
            ", 2.5066282746310002))";
        break;
      case HK_OP_EXPO: e = "exp(__ddiv_rn(-" + A + ", " + c1 + "))"; break;
      case HK_OP_BW:  // 1 / ((a - m0^2)^2 + m0^2 g0^2)
        e = "__ddiv_rn(1.0, __dadd_rn(__dmul_rn(__dsub_rn(" + A + ", __dmul_rn(" + c1 + ", " + c1 +
            ")), __dsub_rn(" + A + ", __dmul_rn(" + c1 + ", " + c1 + "))), __dmul_rn(__dmul_rn(" + c1 +
            ", " + c1 + "), __dmul_rn(" + c2 + ", " + c2 + "))))";
        break;
      case HK_OP_ADD0: e = "__dadd_rn(" + A + ", 0.0)"; break;
      case HK_OP_SQUARE: e = "__dmul_rn(" + A + ", " + A + ")"; break;
      case HK_OP_UDIV:
        if (params && slot_of[P.b[i]] >= 0 && cst_only[slot_of[P.b[i]]])
          e = "__dmul_rn(" + A + ", __drcp_rn(" + B + "))";
        else
          e = "__ddiv_rn(" + A + ", " + B + ")";
        break;
      default: e = "__longlong_as_double(0x7ff8000000000000ll)"; break;
    }
    const bool binary = P.op[i] == HK_OP_ADD || P.op[i] == HK_OP_SUB || P.op[i] == HK_OP_MUL ||
                        P.op[i] == HK_OP_UDIV;
    const bool unary = P.op[i] == HK_OP_NEG || P.op[i] == HK_OP_SQUARE || P.op[i] == HK_OP_ADD0;
    const auto konst = [&](int slot) { return slot_of[slot] >= 0 && cst_only[slot_of[slot]]; };
    cst_only[i] = P.op[i] == HK_OP_CONST || (binary && konst(P.a[i]) && konst(P.b[i])) ||
                  (unary && konst(P.a[i]));
    s += "  const double v" + std::to_string(i) + " = " + e + ";\n";
    slot_of[P.dst[i]] = i;
  }
  s += "  return " + v(P.result) + ";\n";
  return s;
}

// ---- stored-block module: chunk moments + per-row map over HBM columns ----
const char* kStoredPrelude = R"(
typedef unsigned long long u64;
struct JitArgs {
  const double* cols[HK_JIT_MAX_COLS];
  long long count;
  double* part;
  u64* div0;
  u64* nonfin;
  double* out;
};
)";

// Chunk moments: the per-thread order and block tree of k_moments /
// block_sum_store<5> (hk_phsp.cu, hk_device.cuh).
const char* kStoredKernels = R"(
__device__ __forceinline__ void hk_row_moments(const JitArgs& a, long long r, double (&acc)[5]) {
  bool d0 = false;
  const double f = hk_f(a, r, d0);
  if (d0 && a.div0) atomicMin(a.div0, (u64)r);
  if (!isfinite(f) && a.nonfin) atomicMin(a.nonfin, (u64)r);
  const double w = __ldg(a.cols[0] + r);
  const double ww = __dmul_rn(w, w);
  acc[0] = __dadd_rn(acc[0], w);
  acc[1] = __dadd_rn(acc[1], __dmul_rn(w, f));
  acc[2] = __dadd_rn(acc[2], ww);
  acc[3] = __dadd_rn(acc[3], __dmul_rn(ww, f));
  acc[4] = __dadd_rn(acc[4], __dmul_rn(__dmul_rn(ww, f), f));
}

extern "C" __global__ void __launch_bounds__(256) hk_jit_moments(const __grid_constant__ JitArgs a) {
  __shared__ double sm[8][5];
  const long long chunks = (a.count + 4095) / 4096;
  for (long long c = blockIdx.x; c < chunks; c += gridDim.x) {
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    // full chunk: no guards, two rows' loads in flight.  Measured on B200 for
    // <m12^2> over 1e8 stored rows: unroll 1 / 2 / 4 / 8 = 1.31 / 1.16 /
    // 1.27 / 1.37 ms (more unrolling costs resident warps)
    if (c * 4096 + 4096 <= a.count) {
#pragma unroll 2
      for (int i = 0; i < 16; ++i) hk_row_moments(a, c * 4096 + i * 256 + threadIdx.x, acc);
    } else {
#pragma unroll 1
      for (int i = 0; i < 16; ++i) {
        const long long r = c * 4096 + i * 256 + threadIdx.x;
        if (r < a.count) hk_row_moments(a, r, acc);
      }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
      for (int w = 0; w < 5; ++w) acc[w] = __dadd_rn(acc[w], __shfl_down_sync(0xffffffffu, acc[w], off));
    }
    if (lane == 0) {
#pragma unroll
      for (int w = 0; w < 5; ++w) sm[warp][w] = acc[w];
    }
    __syncthreads();
    if (threadIdx.x < 5) {
      double s = sm[0][threadIdx.x];
#pragma unroll
      for (int i = 1; i < 8; ++i) s = __dadd_rn(s, sm[i][threadIdx.x]);
      a.part[5 * c + threadIdx.x] = s;
    }
    __syncthreads();
  }
}

extern "C" __global__ void __launch_bounds__(256) hk_jit_map(const __grid_constant__ JitArgs a) {
  const long long r = blockIdx.x * 256LL + threadIdx.x;
  if (r >= a.count) return;
  bool d0 = false;
  a.out[r] = hk_f(a, r, d0);
  if (d0 && a.div0) atomicMin(a.div0, (u64)r);
}
)";

// ---- fused module: the generator of hk_integrate.cuh with the program inlined
// (LP64 fixed-width types: NVRTC has no libc headers)
const char* kFusedPrelude = R"(
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef short int16_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long int64_t;
typedef unsigned long uint64_t;
typedef unsigned long size_t;
#define UINT64_MAX 0xffffffffffffffffUL
#include "hk_integrate.cuh"
)";

struct EmbeddedHeader {
  const char* name;
  const char* text;
};
const EmbeddedHeader kHeaders[] = {
#include "build/hk_embed.inc"
};
constexpr int kNumHeaders = sizeof(kHeaders) / sizeof(kHeaders[0]);

// n == -1: the FCN module (hk_fcn.cuh fcn_density_pass with the density
// program inlined, constants from the arguments)
const char* kFcnPrelude = R"(
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef short int16_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long int64_t;
typedef unsigned long uint64_t;
typedef unsigned long size_t;
#define UINT64_MAX 0xffffffffffffffffUL
#include "hk_fcn.cuh"
)";

// n == 0: stored-block module; n > 0: fused generate+integrate for n daughters
std::string full_source(const hk_program_t& P, int n, int mode) {
  if (n < 0)
    return std::string(kFcnPrelude) +
           "struct HkDensity {\n"
           "  const hk::FcnProgArgs& a;\n"
           "  __device__ __forceinline__ double operator()(long long r, bool& d0) const {\n" +
           emit_body(P, false, true) +
           "  }\n"
           "};\n"
           "extern \"C\" __global__ void __launch_bounds__(256)\n"
           "    hk_jit_nll(const __grid_constant__ hk::FcnProgArgs a) {\n"
           "  hk::fcn_density_pass<true>(a.w, a.n, HkDensity{a});\n"
           "}\n";
  if (n == 0)
    return "#define HK_JIT_MAX_COLS " + std::to_string(kJitMaxCols) + "\n" + kStoredPrelude +
           "__device__ __forceinline__ double hk_f(const JitArgs& a, long long r, bool& d0) {\n" +
           emit_body(P, false) + "}\n" + kStoredKernels;
  const std::string N = std::to_string(n), M = std::to_string(mode);
  return std::string(kFusedPrelude) +
         "namespace hk {\n"
         "struct JitIntegrand {\n"
         "  static constexpr bool kIlp2 = true;\n"
         "  template <int N>\n"
         "  __device__ __forceinline__ static double eval(const IntArgs& a, double w,\n"
         "                                                const double (&p)[4 * N], uint64_t row) {\n"
         "    bool d0 = false;\n"
         "    const double f = [&]() {\n" +
         emit_body(P, true) +
         "    }();\n"
         "    if (d0) record_bad(a.div0_bad, row);\n"
         "    return f;\n"
         "  }\n"
         "};\n"
         "}  // namespace hk\n"
         "extern \"C\" __global__ void __launch_bounds__(256, hk::GenShape<" + N + ">::min_blocks)\n"
         "    hk_jit_integrate(const __grid_constant__ hk::IntArgs a) {\n"
         "  hk::integrate_chunks<" + N + ", " + M + ", hk::JitIntegrand>(a);\n"
         "}\n";
}

struct Entry {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern[2] = {nullptr, nullptr};
};

std::mutex g_mu;
std::unordered_map<std::string, Entry> g_cache;
Nvrtc g_nvrtc;
int g_mode = -1;

int initial_mode() {
  const char* e = std::getenv("HK_JIT");
  if (!e || !*e || !std::strcmp(e, "auto")) return 2;
  if (!std::strcmp(e, "0")) return 0;
  if (!std::strcmp(e, "1")) return 1;
  return 2;
}

std::string cache_key(const hk_program_t& P, int n, int mode) {
  std::string k;
  k.reserve(16 + P.n_ops * 32);
  auto put = [&](const void* p, size_t b) { k.append(reinterpret_cast<const char*>(p), b); };
  put(&n, 4);
  put(&mode, 4);
  put(&P.n_ops, 4);
  put(&P.result, 4);
  for (int i = 0; i < P.n_ops; ++i) {
    put(&P.op[i], 4);
    put(&P.dst[i], 4);
    put(&P.a[i], 4);
    put(&P.b[i], 4);
    if (n >= 0) {  // the FCN module (n = -1) reads its constants at run time
      put(&P.cst[i], 8);
      put(&P.cst2[i], 8);
    }
  }
  return k;
}

// NVRTC -> sm_100a cubin (no device needed)
int compile_cubin(const hk_program_t& P, int n, int mode, std::vector<char>* cubin) {
  if (!load_nvrtc(g_nvrtc)) {
    set_error("functor specialisation: NVRTC (libnvrtc.so.12) not loadable");
    return HK_ECUDA;
  }
  Nvrtc& N = g_nvrtc;
  const std::string src = full_source(P, n, mode);
  const char* names[kNumHeaders];
  const char* texts[kNumHeaders];
  for (int h = 0; h < kNumHeaders; ++h) {
    names[h] = kHeaders[h].name;
    texts[h] = kHeaders[h].text;
  }
  nvrtcProgram prog;
  nvrtcResult rc = N.create(&prog, src.c_str(), "hk_functor.cu", kNumHeaders, texts, names);
  if (rc != NVRTC_SUCCESS) {
    set_error("nvrtcCreateProgram: %s", N.err(rc));
    return HK_ECUDA;
  }
  // -default-device: the headers' unannotated inline helpers become device code
  const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--std=c++17", "-lineinfo",
                        "-default-device"};
  rc = N.compile(prog, 5, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t len = 0;
    N.log_size(prog, &len);
    std::vector<char> log(len + 1, 0);
    N.log(prog, log.data());
    set_error("functor specialisation failed: %s: %.380s", N.err(rc), log.data());
    N.destroy(&prog);
    return HK_ECUDA;
  }
  size_t len = 0;
  N.cubin_size(prog, &len);
  cubin->resize(len);
  N.cubin(prog, cubin->data());
  N.destroy(&prog);
  return HK_OK;
}

int compile_entry(const hk_program_t& P, int n, int mode, Entry* out) {
  std::vector<char> cubin;
  if (int rc = compile_cubin(P, n, mode, &cubin)) return rc;
  HK_CUDA(cudaLibraryLoadData(&out->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  if (n < 0) {
    HK_CUDA(cudaLibraryGetKernel(&out->kern[0], out->lib, "hk_jit_nll"));
  } else if (n == 0) {
    HK_CUDA(cudaLibraryGetKernel(&out->kern[kJitMoments], out->lib, "hk_jit_moments"));
    HK_CUDA(cudaLibraryGetKernel(&out->kern[kJitMap], out->lib, "hk_jit_map"));
  } else {
    HK_CUDA(cudaLibraryGetKernel(&out->kern[0], out->lib, "hk_jit_integrate"));
  }
  return HK_OK;
}

int lookup(const hk_program_t& P, int n, int mode, int64_t rows, int slot, const void** fn) {
  *fn = nullptr;
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_mode < 0) g_mode = initial_mode();
  if (g_mode == 0) return HK_OK;
  const std::string key = cache_key(P, n, mode);
  auto it = g_cache.find(key);
  if (it == g_cache.end()) {
    if (g_mode == 2 && rows < HK_JIT_MIN_ROWS) return HK_OK;  // small: the interpreter is cheaper
    Entry e;
    if (int rc = compile_entry(P, n, mode, &e)) {
      if (g_mode == 1) return rc;
      g_mode = 0;  // auto: NVRTC unusable here, stay on the (GPU) interpreter
      return HK_OK;
    }
    it = g_cache.emplace(key, e).first;
  }
  *fn = reinterpret_cast<const void*>(it->second.kern[slot]);
  return HK_OK;
}

}  // namespace

int jit_kernel(const hk_program_t& P, int64_t rows, int kind, const void** fn) {
  return lookup(P, 0, 0, rows, kind, fn);
}

int jit_integrate(const hk_program_t& P, int n, int mode, int64_t rows, const void** fn) {
  return lookup(P, n, mode, rows, 0, fn);
}

int jit_fcn(const hk_program_t& P, int64_t rows, const void** fn) {
  return lookup(P, -1, 0, rows, 0, fn);
}

// hk_shutdown: unload every specialised module (no launch may be in flight)
void jit_release() {
  std::lock_guard<std::mutex> lock(g_mu);
  for (auto& kv : g_cache)
    if (kv.second.lib) cudaLibraryUnload(kv.second.lib);
  g_cache.clear();
}

}  // namespace hk

using namespace hk;

extern "C" {

int hk_set_jit_mode(int32_t mode) {
  if (mode < 0 || mode > 2) {
    set_error("jit mode %d not in 0..2", mode);
    return -1;
  }
  std::lock_guard<std::mutex> lock(g_mu);
  const int prev = g_mode < 0 ? initial_mode() : g_mode;
  g_mode = mode;
  return prev;
}

int64_t hk_jit_source(const hk_program_t* f, int32_t n_daughters, int32_t rng_mode, char* buf,
                      int64_t cap) {
  if (!f || f->n_ops < 1 || f->n_ops > HK_MAX_PROGRAM || n_daughters < -1 || n_daughters > 8 ||
      n_daughters == 1 || rng_mode < 0 || rng_mode > 1) {
    set_error("bad program / target");
    return -1;
  }
  const std::string src = full_source(*f, n_daughters, rng_mode);
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>((size_t)cap - 1, src.size());
    std::memcpy(buf, src.data(), n);
    buf[n] = 0;
  }
  return (int64_t)src.size();
}

int hk_jit_compile(const hk_program_t* f, int32_t n_daughters, int32_t rng_mode, int64_t* cubin_bytes) {
  HK_NVTX("hk_jit_compile");
  HK_REQUIRE(f && f->n_ops >= 1 && f->n_ops <= HK_MAX_PROGRAM, "bad program");
  HK_REQUIRE(n_daughters == -1 || n_daughters == 0 || (n_daughters >= 2 && n_daughters <= 8),
             "n_daughters %d", n_daughters);
  HK_REQUIRE(rng_mode == HK_RNG_REFERENCE || rng_mode == HK_RNG_PHILOX, "rng mode %d", rng_mode);
  std::vector<char> cubin;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    if (int rc = compile_cubin(*f, n_daughters, rng_mode, &cubin)) return rc;
  }
  if (cubin_bytes) *cubin_bytes = (int64_t)cubin.size();
  return HK_OK;
}

int64_t hk_jit_count(void) {
  std::lock_guard<std::mutex> lock(g_mu);
  return (int64_t)g_cache.size();
}

}  // extern "C"

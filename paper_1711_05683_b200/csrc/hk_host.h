// hk_host.h -- host-side helpers shared by the C-ABI translation units:
// per-thread error text, CUDA status checks, launch-shape helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>

#include "hepkit_cuda.h"

// NVTX ranges (header-only NVTX v3: no link dependency; a no-op unless a
// profiler injects its tool library): every compute entry point of the C ABI
// opens one named after itself, so nsys / ncu --nvtx timelines show the
// reference-facing calls around their kernels.
#include <nvtx3/nvToolsExt.h>

namespace hk {

struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define HK_NVTX(name) ::hk::NvtxRange hk_nvtx_range_(name)

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* where);

inline int check_launch(const char* where) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HK_OK : cuda_fail(e, where);
}

inline int64_t num_chunks(int64_t n) { return n <= 0 ? 0 : (n + HK_CHUNK - 1) / HK_CHUNK; }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Grid for chunk-per-CTA kernels.  One CTA per 4096-row chunk; the hardware
// block scheduler load-balances the waves.  gridDim.x is capped and kernels
// grid-stride over chunks beyond the cap.
inline unsigned chunk_grid(int64_t chunks) {
  const int64_t cap = int64_t(1) << 30;
  return (unsigned)(chunks < 1 ? 1 : (chunks > cap ? cap : chunks));
}

// hk_jit.cu: specialised functor kernels.  JitArgs is mirrored field for
// field by the NVRTC-compiled source.
constexpr int kJitMaxCols = 4 * HK_MAX_DAUGHTERS + 1;
constexpr int kJitMoments = 0;
constexpr int kJitMap = 1;
struct JitArgs {
  const double* cols[kJitMaxCols];
  long long count;
  double* part;
  unsigned long long* div0;
  unsigned long long* nonfin;
  double* out;
};
// *fn = specialised kernel for the program (kind kJitMoments / kJitMap), or
// nullptr when the interpreter should run (mode / size policy).
int jit_kernel(const hk_program_t& P, int64_t rows, int kind, const void** fn);
// same for the fused generate+integrate kernel (n daughters, RNG mode)
int jit_integrate(const hk_program_t& P, int n, int mode, int64_t rows, const void** fn);
// the program-driven FCN pass (hk_fcn.cuh fcn_density_pass) with the density
// program inlined; constants are read from the kernel's FcnProgArgs, so one
// module serves every parameter point of a model structure
int jit_fcn(const hk_program_t& P, int64_t rows, const void** fn);

// hk_phsp.cu: structural check of a program reading n_cols columns
int validate_program(const hk_program_t* f, int n_cols);

}  // namespace hk

#define HK_REQUIRE(cond, ...)       \
  do {                              \
    if (!(cond)) {                  \
      ::hk::set_error(__VA_ARGS__); \
      return HK_EINVAL;             \
    }                               \
  } while (0)

#define HK_CUDA(call)                                                  \
  do {                                                                 \
    cudaError_t hk_e_ = (call);                                        \
    if (hk_e_ != cudaSuccess) return ::hk::cuda_fail(hk_e_, #call);    \
  } while (0)

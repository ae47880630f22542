// hk_csv.cu -- CSV text of real64 columns on the GPU,
// the body of ColumnStore.write_csv (store.py:181-204): every value as
// Python's f"{v:.17g}" (17 significant digits, correctly rounded, so values
// round-trip), ',' between columns, '\n' after each row.
//
// Per value: exact decimal conversion -- Q = round_half_even(v * 10^(16-X)),
// 10^16 <= Q < 10^17, X the decimal exponent -- then Python's 'g' layout
// (fixed for -4 <= X < 17, else d.ddde+XX; trailing zeros stripped; nan,
// inf, -inf, -0).  Exactness: values in [1e-3, ~1e17) take a 128-bit path
// (m * 10^k fits in 117 bits, the binary point is a shift); everything else
// (tiny, huge, subnormal) takes a multi-limb path.  Both round on the exact
// remainder, so the digits equal CPython's dtoa for every double
// (tests/test_csv_gpu.py compares against f"{v:.17g}" on random bit patterns).
//
// Four launches per call: values -> fixed 24-byte slots + lengths; row
// lengths + block scan; scan of block totals; pack rows into one compact
// buffer.  Integer work on the INT pipes; bound by the pack's byte stores and
// by PCIe once the text leaves the GPU.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "hepkit_cuda.h"
#include "hk_host.h"

namespace hk {
namespace csv {

constexpr int kSlot = 24;  // "-1.2345678901234567e-308" is 24 characters
constexpr int kBlockRows = 256;

__constant__ uint64_t kPow10[20] = {1ull,
                                    10ull,
                                    100ull,
                                    1000ull,
                                    10000ull,
                                    100000ull,
                                    1000000ull,
                                    10000000ull,
                                    100000000ull,
                                    1000000000ull,
                                    10000000000ull,
                                    100000000000ull,
                                    1000000000000ull,
                                    10000000000000ull,
                                    100000000000000ull,
                                    1000000000000000ull,
                                    10000000000000000ull,
                                    100000000000000000ull,
                                    1000000000000000000ull,
                                    10000000000000000000ull};

// ---------------------------------------------------------- multi-limb ----
// little-endian 32-bit limbs; 40 limbs = 1280 bits covers m * 10^340 and
// m * 2^971 (the extremes of the double range)
struct Big {
  uint32_t w[40];
  int n;
};

__device__ __forceinline__ void big_set(Big& b, uint64_t v) {
  b.w[0] = (uint32_t)v;
  b.w[1] = (uint32_t)(v >> 32);
  b.n = b.w[1] ? 2 : 1;
}

__device__ __forceinline__ void big_mul_small(Big& b, uint32_t x) {
  uint64_t carry = 0;
  for (int i = 0; i < b.n; ++i) {
    const uint64_t t = (uint64_t)b.w[i] * x + carry;
    b.w[i] = (uint32_t)t;
    carry = t >> 32;
  }
  if (carry) b.w[b.n++] = (uint32_t)carry;
}

__device__ __forceinline__ void big_shl(Big& b, int s) {
  const int limbs = s >> 5, bits = s & 31;
  if (bits) {
    uint32_t carry = 0;
    for (int i = 0; i < b.n; ++i) {
      const uint32_t v = b.w[i];
      b.w[i] = (v << bits) | carry;
      carry = v >> (32 - bits);
    }
    if (carry) b.w[b.n++] = carry;
  }
  if (limbs) {
    for (int i = b.n - 1; i >= 0; --i) b.w[i + limbs] = b.w[i];
    for (int i = 0; i < limbs; ++i) b.w[i] = 0;
    b.n += limbs;
  }
}

// b = floor(b / d), returns b mod d
__device__ __forceinline__ uint32_t big_divmod(Big& b, uint32_t d) {
  uint64_t rem = 0;
  for (int i = b.n - 1; i >= 0; --i) {
    const uint64_t cur = (rem << 32) | b.w[i];
    b.w[i] = (uint32_t)(cur / d);
    rem = cur % d;
  }
  while (b.n > 1 && b.w[b.n - 1] == 0) --b.n;
  return (uint32_t)rem;
}

__device__ __forceinline__ uint32_t big_bit(const Big& b, int i) {
  return (i >> 5) < b.n ? (b.w[i >> 5] >> (i & 31)) & 1u : 0u;
}

__device__ __forceinline__ bool big_any_below(const Big& b, int t) {  // any bit < t
  const int full = t >> 5;
  for (int i = 0; i < full && i < b.n; ++i)
    if (b.w[i]) return true;
  if ((t & 31) && full < b.n) return (b.w[full] & ((1u << (t & 31)) - 1u)) != 0;
  return false;
}

__device__ __forceinline__ uint64_t big_bits_from(const Big& b, int t) {  // floor(b / 2^t), < 2^64
  uint64_t q = 0;
  for (int k = 0; k < 64; k += 32) {
    const int bit = t + k, li = bit >> 5, sh = bit & 31;
    uint64_t part = li < b.n ? (uint64_t)(b.w[li] >> sh) : 0;
    if (sh && li + 1 < b.n) part |= (uint64_t)b.w[li + 1] << (32 - sh);
    q |= (part & 0xffffffffull) << k;
  }
  return q;
}

// round_half_even(m * 2^q * 10^k), exact; the result is < 2^64 for the k
// the caller asks for (about 17-18 digits)
__device__ uint64_t round_scaled(uint64_t m, int q, int k) {
  if (k >= 0 && k <= 19 && q >= -127 && q <= 10) {  // 128-bit path: m * 10^k < 2^117
    const unsigned __int128 P = (unsigned __int128)m * kPow10[k];
    if (q >= 0) return (uint64_t)(P << q);
    const int t = -q;
    const uint64_t Q = (uint64_t)(P >> t);
    const unsigned __int128 rem = P & ((((unsigned __int128)1) << t) - 1);
    const unsigned __int128 half = ((unsigned __int128)1) << (t - 1);
    return Q + ((rem > half || (rem == half && (Q & 1))) ? 1 : 0);
  }
  Big b;
  big_set(b, m);
  if (k >= 0) {
    int kk = k;
    for (; kk >= 9; kk -= 9) big_mul_small(b, 1000000000u);
    if (kk) big_mul_small(b, (uint32_t)kPow10[kk]);
    if (q >= 0) {
      big_shl(b, q);
      return big_bits_from(b, 0);
    }
    const int t = -q;
    const uint64_t Q = big_bits_from(b, t);
    const uint32_t a = big_bit(b, t - 1);
    const bool sticky = big_any_below(b, t - 1);
    return Q + ((a && (sticky || (Q & 1))) ? 1 : 0);
  }
  // k < 0: divide m * 2^q (q >= 0 here: |v| >= 1e17 > 2^53) by 10^j, the
  // least significant group first so the last remainder is the leading one
  if (q > 0) big_shl(b, q);
  const int j = -k;
  bool sticky = false;
  uint32_t a = 0, d = 1;
  int rest = j;
  if (j % 9) {
    d = (uint32_t)kPow10[j % 9];
    a = big_divmod(b, d);
    rest -= j % 9;
  }
  for (; rest > 0; rest -= 9) {
    sticky = sticky || a != 0;
    d = 1000000000u;
    a = big_divmod(b, d);
  }
  const uint64_t Q = big_bits_from(b, 0);
  const uint32_t half = d / 2;  // d = 10^i, even
  return Q + ((a > half || (a == half && (sticky || (Q & 1)))) ? 1 : 0);
}

// |v| = Q * 10^(X-16), 10^16 <= Q < 10^17, Q correctly rounded (half even)
__device__ void dec17(double av, uint64_t* Qo, int* Xo) {
  const uint64_t bits = (uint64_t)__double_as_longlong(av);
  const int be = (int)((bits >> 52) & 0x7ff);
  const uint64_t frac = bits & 0x000fffffffffffffull;
  const uint64_t m = be ? (frac | 0x0010000000000000ull) : frac;
  const int q = be ? be - 1075 : -1074;
  int X = (int)floor(log10(av));
  for (int it = 0; it < 4; ++it) {
    const uint64_t Q = round_scaled(m, q, 16 - X);
    if (Q >= kPow10[17]) {
      ++X;  // estimate one low, or rounding carried to 10^17
    } else if (Q < kPow10[16]) {
      --X;
    } else {
      *Qo = Q;
      *Xo = X;
      return;
    }
  }
  *Qo = kPow10[16];  // unreachable for finite nonzero doubles
  *Xo = X;
}

// f"{v:.17g}" into out (no terminator); returns the length (<= 24)
__device__ int format_g17(double v, char* out) {
  const uint64_t bits = (uint64_t)__double_as_longlong(v);
  const bool neg = bits >> 63;
  int n = 0;
  if (isnan(v)) {
    out[0] = 'n', out[1] = 'a', out[2] = 'n';
    return 3;
  }
  if (neg) out[n++] = '-';
  if (isinf(v)) {
    out[n] = 'i', out[n + 1] = 'n', out[n + 2] = 'f';
    return n + 3;
  }
  if (v == 0.0) {
    out[n++] = '0';
    return n;
  }
  uint64_t Q;
  int X;
  dec17(fabs(v), &Q, &X);
  char dg[17];
#pragma unroll
  for (int i = 16; i >= 0; --i) {
    dg[i] = (char)('0' + Q % 10);
    Q /= 10;
  }
  int nd = 17;
  while (nd > 1 && dg[nd - 1] == '0') --nd;
  if (X >= -4 && X < 17) {
    if (X >= 0) {
      for (int i = 0; i <= X; ++i) out[n++] = i < nd ? dg[i] : '0';
      if (nd > X + 1) {
        out[n++] = '.';
        for (int i = X + 1; i < nd; ++i) out[n++] = dg[i];
      }
    } else {
      out[n++] = '0';
      out[n++] = '.';
      for (int i = 0; i < -X - 1; ++i) out[n++] = '0';
      for (int i = 0; i < nd; ++i) out[n++] = dg[i];
    }
  } else {
    out[n++] = dg[0];
    if (nd > 1) {
      out[n++] = '.';
      for (int i = 1; i < nd; ++i) out[n++] = dg[i];
    }
    out[n++] = 'e';
    out[n++] = X < 0 ? '-' : '+';
    const int ax = X < 0 ? -X : X;
    if (ax >= 100) out[n++] = (char)('0' + ax / 100);
    out[n++] = (char)('0' + (ax / 10) % 10);
    out[n++] = (char)('0' + ax % 10);
  }
  return n;
}

struct CsvArgs {
  const double* cols[4 * HK_MAX_DAUGHTERS + 1];
  int32_t n_cols;
  int64_t n_rows;
  char* slots;         // n_rows * n_cols * kSlot
  uint8_t* lens;       // n_rows * n_cols
  int64_t* row_off;    // n_rows: offset of the row inside its block
  int64_t* block_tot;  // blocks: total bytes of the block, then (scanned) its offset
  char* out;
};

// one thread per value; column-major index so each warp reads one column
__global__ void __launch_bounds__(256) k_csv_values(const __grid_constant__ CsvArgs a) {
  const int64_t total = a.n_rows * a.n_cols;
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
    const int c = (int)(i / a.n_rows);
    const int64_t r = i - (int64_t)c * a.n_rows;
    char buf[kSlot];
    const int len = format_g17(__ldg(a.cols[c] + r), buf);
    const int64_t slot = r * a.n_cols + c;
    char* dst = a.slots + slot * kSlot;
#pragma unroll
    for (int k = 0; k < kSlot; ++k) dst[k] = k < len ? buf[k] : 0;
    a.lens[slot] = (uint8_t)len;
  }
}

// row length = sum of value lengths + n_cols separators (commas + newline);
// exclusive scan inside each 256-row block
__global__ void __launch_bounds__(kBlockRows) k_csv_rows(const __grid_constant__ CsvArgs a) {
  __shared__ int64_t warp_tot[kBlockRows / 32];
  const int64_t r = blockIdx.x * (int64_t)kBlockRows + threadIdx.x;
  int64_t len = 0;
  if (r < a.n_rows) {
    len = a.n_cols;
    for (int c = 0; c < a.n_cols; ++c) len += a.lens[r * a.n_cols + c];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t incl = len;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int64_t t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  int64_t before = 0;
  for (int w = 0; w < warp; ++w) before += warp_tot[w];
  if (r < a.n_rows) a.row_off[r] = before + incl - len;
  if (threadIdx.x == kBlockRows - 1) {
    int64_t tot = 0;
    for (int w = 0; w < kBlockRows / 32; ++w) tot += warp_tot[w];
    a.block_tot[blockIdx.x] = tot;
  }
}

// exclusive scan of the block totals by one CTA; *total = bytes of text
__global__ void __launch_bounds__(1024) k_csv_scan(int64_t* tot, int64_t nb, int64_t* total) {
  __shared__ int64_t sm[1024];
  const int t = threadIdx.x;
  const int64_t per = (nb + 1023) / 1024;
  const int64_t b0 = t * per, b1 = b0 + per < nb ? b0 + per : nb;
  int64_t s = 0;
  for (int64_t b = b0; b < b1; ++b) s += tot[b];
  sm[t] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int64_t v = t >= off ? sm[t - off] : 0;
    __syncthreads();
    sm[t] += v;
    __syncthreads();
  }
  int64_t run = sm[t] - s;
  for (int64_t b = b0; b < b1; ++b) {
    const int64_t v = tot[b];
    tot[b] = run;
    run += v;
  }
  if (t == 1023) *total = sm[1023];
}

// one warp per row: lanes copy the row's slots into its place in the text
__global__ void __launch_bounds__(256) k_csv_pack(const __grid_constant__ CsvArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * 8;
  for (int64_t r = blockIdx.x * 8ll + (threadIdx.x >> 5); r < a.n_rows; r += warps) {
    char* dst = a.out + a.block_tot[r / kBlockRows] + a.row_off[r];
    const uint8_t* L = a.lens + r * a.n_cols;
    const char* S = a.slots + r * a.n_cols * (int64_t)kSlot;
    int pos = 0;
    for (int c = 0; c < a.n_cols; ++c) {
      const int len = L[c];
      if (lane < len) dst[pos + lane] = S[c * kSlot + lane];
      if (lane == 0) dst[pos + len] = c + 1 < a.n_cols ? ',' : '\n';
      pos += len + 1;
    }
  }
}

}  // namespace csv
}  // namespace hk

using namespace hk;
using namespace hk::csv;

extern "C" {

int64_t hk_csv_scratch_bytes(int64_t n_rows, int32_t n_cols) {
  if (n_rows <= 0 || n_cols <= 0) return 0;
  const int64_t blocks = (n_rows + kBlockRows - 1) / kBlockRows;
  const int64_t vals = n_rows * n_cols;
  auto up = [](int64_t b) { return (b + 255) & ~(int64_t)255; };
  return up(vals * kSlot) + up(vals) + up(n_rows * 8) + up(blocks * 8) + up(8);
}

int hk_format_csv(const double* const* d_cols, int32_t n_cols, int64_t n_rows, void* d_scratch,
                  char* d_out, int64_t out_cap, int64_t* h_len, void* stream) {
  HK_NVTX("hk_format_csv");
  HK_REQUIRE(d_cols && n_cols >= 1 && n_cols <= 4 * HK_MAX_DAUGHTERS + 1, "bad columns (%d)", n_cols);
  HK_REQUIRE(n_rows >= 0 && h_len, "bad arguments");
  *h_len = 0;
  if (n_rows == 0) return HK_OK;
  HK_REQUIRE(d_scratch && d_out, "NULL scratch/output");
  HK_REQUIRE(out_cap >= n_rows * n_cols * (kSlot + 1), "output capacity %lld < %lld", (long long)out_cap,
             (long long)(n_rows * n_cols * (kSlot + 1)));
  CsvArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int c = 0; c < n_cols; ++c) {
    HK_REQUIRE(d_cols[c], "column %d NULL", c);
    a.cols[c] = d_cols[c];
  }
  a.n_cols = n_cols;
  a.n_rows = n_rows;
  const int64_t blocks = (n_rows + kBlockRows - 1) / kBlockRows;
  const int64_t vals = n_rows * n_cols;
  auto up = [](int64_t b) { return (b + 255) & ~(int64_t)255; };
  char* p = static_cast<char*>(d_scratch);
  a.slots = p;
  p += up(vals * kSlot);
  a.lens = reinterpret_cast<uint8_t*>(p);
  p += up(vals);
  a.row_off = reinterpret_cast<int64_t*>(p);
  p += up(n_rows * 8);
  a.block_tot = reinterpret_cast<int64_t*>(p);
  p += up(blocks * 8);
  int64_t* d_total = reinterpret_cast<int64_t*>(p);
  a.out = d_out;
  cudaStream_t st = as_stream(stream);
  const int64_t vgrid = (vals + 255) / 256;
  k_csv_values<<<(unsigned)(vgrid < (1 << 30) ? vgrid : (1 << 30)), 256, 0, st>>>(a);
  k_csv_rows<<<(unsigned)blocks, kBlockRows, 0, st>>>(a);
  k_csv_scan<<<1, 1024, 0, st>>>(a.block_tot, blocks, d_total);
  const int64_t pgrid = (n_rows + 7) / 8;
  k_csv_pack<<<(unsigned)(pgrid < (1 << 30) ? pgrid : (1 << 30)), 256, 0, st>>>(a);
  if (int rc = check_launch("k_csv")) return rc;
  HK_CUDA(cudaMemcpyAsync(h_len, d_total, 8, cudaMemcpyDeviceToHost, st));
  HK_CUDA(cudaStreamSynchronize(st));
  return HK_OK;
}

}  // extern "C"

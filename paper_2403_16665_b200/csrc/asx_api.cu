// asx_api.cu — C ABI of libasx.so (declared in include/asx.h).
//
// Host side of the drop-in boundary: plan validation mirrors the reference
// (core.py:95-105 validate_pair, fastpath.py:85-110 plan), tables are built
// on device at plan time, execute only launches kernels on the caller's
// stream (no allocation, no host sync).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "../../include/asx.h"
#include "asx_direct_tc.cuh"
#ifndef ASX_DTC_PAIR
#define ASX_DTC_PAIR 0
#endif
#if ASX_DTC_PAIR
#include "asx_direct_tc2.cuh"
#endif
#include "asx_dispatch.cuh"

using namespace asx;
using namespace asx_host;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  cudaGetLastError();  // clear sticky-free errors
  return fail(e == cudaErrorMemoryAllocation ? ASX_ERR_OOM : ASX_ERR_CUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                      \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}
bool is_pow2(int64_t v) { return v >= 1 && (v & (v - 1)) == 0; }
int log2i(int64_t v) {
  int r = 0;
  while ((int64_t(1) << r) < v) ++r;
  return r;
}
int bit_length(int64_t v) {
  int r = 0;
  while (v) {
    ++r;
    v >>= 1;
  }
  return r;
}

constexpr int kMaxP_c64 = 16384;
constexpr int kMaxP_c128 = 8192;
constexpr int64_t kDtcMaxN = 1024;


}  // namespace

struct asx_plan_s {
  int64_t n = 0, m = 0, a = 1, d = 1;
  int dtype = ASX_C128, real_input = 0, method = ASX_AUTO, device = 0;
  int P = 0;
  int64_t r = 1, fold = 1;
  int64_t m_ref = 0;
  int depth = -1, leaf = ASX_LEAF_NONE;
  int64_t pred_mults = -1, pred_adds = -1;
  // device tables
  void* tables = nullptr;
  size_t table_bytes = 0;
  size_t off_twP = 0, off_twA = 0, off_chirp = 0, off_H = 0, off_W = 0;
  size_t off_afl = 0;
  int dtc = 0;            // direct form on the tensor cores: 1 k_direct_tc (M = 128), 2 k_direct_tc2 (M = 256, CTA pairs)
  size_t off_vimg = 0;    // its fp16 operand image (bytes from tables)
  int lfA = 0;
  int tw_elems = 0;  // shared-memory twiddle elements (twP [+ twA])
  // large chirp path (P > one CTA): four-step P = P1 x P2 through workspace A
  int large = 0;
  int large_fft = 0;  // the α-FFT through the same four-step kernels (P = N > one CTA), one residue per launch pair
  int64_t P1 = 0, P2 = 0;
  int64_t group = 1;  // signals per four-step launch set (the plan workspace holds group x P elements)
  int lfBig = 0;
  int row_local = 0;  // complex128 P2 = 8192: rows on k_large_rows_local, Ht stored permuted
  size_t off_twP1 = 0, off_twBig = 0, off_A = 0;
  LaunchEnv env;
  // execute_host resources
  std::mutex host_mtx;
  // four-step workspace per stream: the plan's own buffer serves the first
  // stream that executes, further streams get their own (asx_execute stays
  // reentrant across streams, including the host path's stream ring)
  std::mutex ws_mtx;
  cudaStream_t ws_owner = nullptr;
  bool ws_owned = false;
  std::vector<std::pair<cudaStream_t, void*>> ws_extra;
  static constexpr int kLanes = 3;
  cudaStream_t lane[kLanes] = {nullptr, nullptr, nullptr};
  void* din[kLanes] = {nullptr, nullptr, nullptr};
  void* dout[kLanes] = {nullptr, nullptr, nullptr};
  int64_t lane_rows = 0;
};

namespace {

size_t celem(int dtype) { return dtype == ASX_C64 ? sizeof(float2) : sizeof(double2); }
size_t in_elem(const asx_plan_s* p) {
  size_t re = p->dtype == ASX_C64 ? sizeof(float) : sizeof(double);
  return p->real_input ? re : 2 * re;
}

// --------------------------- kernel dispatch --------------------------------

// Team shape per (precision, FFT size): R values per thread, NT = P/R
// threads per transform, TPB transforms per CTA.  Chosen so the data fits the
// register budget at the CTA size (no spills, see build/ptxas.log).
#ifndef ASX_R_BIG_C64
#define ASX_R_BIG_C64 16  // values per thread for c64 P >= 4096
#endif
#ifndef ASX_R_16K_C64
#define ASX_R_16K_C64 16  // values per thread for c64 P == 16384
#endif
#ifndef ASX_R_4K_C128
#define ASX_R_4K_C128 8  // values per thread for c128 P == 4096
#endif
int two_level_lf(int64_t L) { return (log2i(L) + 1) / 2; }

// Builds [fine(F) | coarse(ceil(L/F))] for W_L at dst.
void fill_two_level(void* dst, int64_t L, int lf, int dbl, cudaStream_t st) {
  const int64_t F = int64_t(1) << lf;
  const int64_t coarse = (L + F - 1) / F;
  const size_t es = dbl ? sizeof(double2) : sizeof(float2);
  k_fill_roots<<<(unsigned)std::min<int64_t>((F + 255) / 256, 4096), 256, 0, st>>>(dst, F, 1, (uint64_t)L, dbl);
  k_fill_roots<<<(unsigned)std::min<int64_t>((coarse + 255) / 256, 4096), 256, 0, st>>>(
      static_cast<char*>(dst) + F * es, coarse, (uint64_t)F, (uint64_t)L, dbl);
}
int64_t two_level_size(int64_t L, int lf) {
  const int64_t F = int64_t(1) << lf;
  return F + (L + F - 1) / F;
}

struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    ok = (cudaSetDevice(dev) == cudaSuccess);
    if (!ok) cudaGetLastError();
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int64_t next_pow2(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

void fill_kparams(const asx_plan_s* p, KParams& kp) {
  std::memset(&kp, 0, sizeof(kp));
  kp.n = p->n;
  kp.m = p->m;
  kp.r = p->r;
  kp.fold = p->fold;
  kp.real_in = p->real_input;
  kp.lfA = p->lfA;
  char* base = static_cast<char*>(p->tables);
  kp.twP = base + p->off_twP;
  kp.twA = base + p->off_twA;
  kp.chirp = base + p->off_chirp;
  kp.H = base + p->off_H;
  kp.W = base + p->off_W;
  kp.tw_elems = p->tw_elems;
  kp.chirp_len = std::max(p->n, p->m);
  kp.afl = p->off_afl ? base + p->off_afl : nullptr;
}

void* large_workspace(asx_plan_s* p, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(p->ws_mtx);
  void* own = static_cast<char*>(p->tables) + p->off_A;
  if (!p->ws_owned || p->ws_owner == st) {
    p->ws_owned = true;
    p->ws_owner = st;
    return own;
  }
  for (auto& kv : p->ws_extra)
    if (kv.first == st) return kv.second;
  void* w = nullptr;
  if (cudaMalloc(&w, celem(p->dtype) * size_t(p->P) * size_t(p->group)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  p->ws_extra.emplace_back(st, w);
  return w;
}

// k_direct_tc reads rows as float4 and writes them as float4
bool dtc_aligned(const void* x, int64_t xs, const void* X, int64_t Xs) {
  return (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 && xs % 2 == 0 &&
         Xs % 2 == 0;
}

int launch_execute(asx_plan_s* p, const void* x, int64_t xs, void* X, int64_t Xs, int64_t batch,
                   cudaStream_t st) {
  if (batch == 0 || p->m == 0) return ASX_OK;
  if (batch > 0x7fffffffLL) return fail(ASX_ERR_INVALID, "batch must be < 2^31 per call");
  KParams kp;
  fill_kparams(p, kp);
  kp.x = x;
  kp.xs = xs;
  kp.X = X;
  kp.Xs = Xs;
  kp.batch = batch;
  cudaError_t e = cudaSuccess;
  if (p->method == ASX_DIRECT && batch <= kDirectSmallBatch) {
    const unsigned grid = (unsigned)((p->m + 1) / 2);  // 4 warps per bin, 2 bins per CTA
    if (p->dtype == ASX_C64)
      k_direct_small<float><<<grid, 256, 0, st>>>(kp);
    else
      k_direct_small<double><<<grid, 256, 0, st>>>(kp);
    e = cudaGetLastError();
#if ASX_DTC_PAIR
  } else if (p->method == ASX_DIRECT && p->dtc == 2 && dtc_aligned(x, xs, X, Xs) && p->env.sms >= 2) {
    dtc2::Params dp;
    dp.x = static_cast<const float*>(x);
    dp.xs = xs;
    dp.X = static_cast<float*>(X);
    dp.Xs = Xs;
    dp.batch = batch;
    dp.n = (int)p->n;
    dp.wimg = static_cast<const unsigned char*>(p->tables) + p->off_vimg;
    const int64_t tiles = (batch + dtc2::TS - 1) / dtc2::TS;
    const int grid = 2 * (int)std::min<int64_t>(tiles, p->env.sms / 2);
    dtc2::k_direct_tc2<<<grid, dtc2::NTHREADS, dtc2::SMEM_BYTES, st>>>(dp);
    g_last_launch.grid = grid;
    g_last_launch.block = dtc2::NTHREADS;
    g_last_launch.smem = dtc2::SMEM_BYTES;
    g_last_launch.staged = 1;
    g_last_launch.tmem = 10;
    e = cudaGetLastError();
#endif
  } else if (p->method == ASX_DIRECT && p->dtc && dtc_aligned(x, xs, X, Xs)) {
    dtc::Params dp;
    dp.x = static_cast<const float*>(x);
    dp.xs = xs;
    dp.X = static_cast<float*>(X);
    dp.Xs = Xs;
    dp.batch = batch;
    dp.n = (int)p->n;
    dp.m = (int)p->m;
    dp.wimg = static_cast<const unsigned char*>(p->tables) + p->off_vimg;
    const int64_t tiles = (batch + dtc::TS - 1) / dtc::TS;
    const int grid = (int)std::min<int64_t>(tiles, p->env.sms);
    dtc::k_direct_tc<<<grid, dtc::NTHREADS, dtc::SMEM_BYTES, st>>>(dp);
    g_last_launch.grid = grid;
    g_last_launch.block = dtc::NTHREADS;
    g_last_launch.smem = dtc::SMEM_BYTES;
    g_last_launch.staged = 1;
    g_last_launch.tmem = 8;
    e = cudaGetLastError();
  } else if (p->method == ASX_DIRECT) {
    const int64_t gy = (batch + 63) / 64, gx = (p->m + 63) / 64;
    if (gy > 65535) {
      // grid.y limit: walk the batch in slabs of 65535*64 signals
      const int64_t slab = 65535LL * 64;
      for (int64_t b0 = 0; b0 < batch; b0 += slab) {
        KParams k2 = kp;
        k2.x = static_cast<const char*>(x) + b0 * xs * in_elem(p);
        k2.X = static_cast<char*>(X) + b0 * Xs * celem(p->dtype);
        k2.batch = std::min(slab, batch - b0);
        dim3 grid((unsigned)gx, (unsigned)((k2.batch + 63) / 64));
        if (p->dtype == ASX_C64)
          k_direct<float><<<grid, 256, 0, st>>>(k2);
        else
          k_direct<double><<<grid, 256, 0, st>>>(k2);
      }
    } else {
      dim3 grid((unsigned)gx, (unsigned)gy);
      if (p->dtype == ASX_C64)
        k_direct<float><<<grid, 256, 0, st>>>(kp);
      else
        k_direct<double><<<grid, 256, 0, st>>>(kp);
    }
    e = cudaGetLastError();
  } else if (p->large) {
    char* base = static_cast<char*>(p->tables);
    LParams lp;
    std::memset(&lp, 0, sizeof(lp));
    lp.real_in = p->real_input;
    lp.n = p->n;
    lp.m = p->m;
    lp.chirp = base + p->off_chirp;
    lp.A = large_workspace(p, st);
    if (!lp.A) return fail(ASX_ERR_OOM, "four-step workspace allocation failed");
    lp.Ht = base + p->off_H;
    lp.twP1 = base + p->off_twP1;
    lp.twP2 = base + p->off_twP;
    lp.twBig = base + p->off_twBig;
    lp.lfBig = p->lfBig;
    lp.P = p->P;
    lp.P2 = p->P2;
    const int dbl = p->dtype == ASX_C128;
    const size_t ie = in_elem(p), oe = celem(p->dtype);
    lp.xs = xs;
    lp.Xs = Xs;
    // the batch in groups of p->group signals, one launch set per group
    for (int64_t b = 0; b < batch && e == cudaSuccess; b += p->group) {
      lp.nsig = std::min(p->group, batch - b);
      lp.x = static_cast<const char*>(x) + (size_t)b * xs * ie;
      lp.X = static_cast<char*>(X) + (size_t)b * Xs * oe;
      if (p->large_fft) {
        // α-FFT: one (columns, rows) launch pair per output residue c < min(r, M)
        lp.P = p->n;
        lp.r = p->r;
        const int64_t nres = std::min<int64_t>(p->r, p->m);
        for (int64_t c = 0; c < nres && e == cudaSuccess; ++c) {
          lp.c = c;
          e = launch_large(dbl, p->P1, COL_AFFT, 0, 0, lp, st);
          if (e == cudaSuccess) e = launch_large(dbl, p->P1, 0, ROW_AFFT, 1, lp, st);
        }
      } else {
        e = launch_large(dbl, p->P1, COL_FWD_SIGNAL, 0, 0, lp, st);
        if (e == cudaSuccess) e = launch_large(dbl, p->P1, 0, p->row_local ? ROW_MAIN_LOCAL : ROW_MAIN, 1, lp, st);
        if (e == cudaSuccess) e = launch_large(dbl, p->P1, COL_INV_OUT, 0, 0, lp, st);
      }
    }
  } else {
    const size_t ie = in_elem(p);
    kp.staged = ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && ((size_t)xs * ie) % 16 == 0 &&
                 ((size_t)p->n * ie) % 16 == 0 && (batch == 1 || xs >= p->n))
                    ? 1
                    : 0;
    if (p->dtype == ASX_C64 && p->method == ASX_FFT)
      e = launch_afft_io32(p->P, kp, batch, st, p->env);  // FP64 recursion, complex64 in/out
    else if (p->dtype == ASX_C64)
      e = launch_by_size<float>(p->method, p->P, kp, batch, st, p->env);
    else
      e = launch_by_size<double>(p->method, p->P, kp, batch, st, p->env);
  }
  if (e != cudaSuccess) return cuda_fail(e, "asx_execute launch");
  return ASX_OK;
}

}  // namespace

// ================================ C ABI =====================================

extern "C" {

int asx_version(void) { return ASX_ABI_VERSION; }

const char* asx_strerror(int status) {
  switch (status) {
    case ASX_OK: return "ok";
    case ASX_ERR_INVALID: return "invalid argument";
    case ASX_ERR_INCOMPATIBLE: return "density factor incompatible with signal length (alpha*N not an integer)";
    case ASX_ERR_UNSUPPORTED: return "unsupported size for this method";
    case ASX_ERR_CUDA: return "CUDA error";
    case ASX_ERR_OOM: return "device out of memory";
    default: return "unknown status";
  }
}

const char* asx_last_error(void) { return g_last_error.c_str(); }

int asx_last_launch(int* grid, int* block, int* smem_bytes, int* staged) {
  if (grid) *grid = g_last_launch.grid;
  if (block) *block = g_last_launch.block;
  if (smem_bytes) *smem_bytes = g_last_launch.smem;
  if (staged) *staged = g_last_launch.staged | (g_last_launch.tmem << 1);
  return ASX_OK;
}

int asx_plan_create(asx_plan_t* out, int64_t n, int64_t a_num, int64_t a_den, int64_t m, int dtype,
                    int real_input, int method, int device) {
  if (!out) return fail(ASX_ERR_INVALID, "plan pointer is NULL");
  *out = nullptr;
  if (n < 1) return fail(ASX_ERR_INVALID, "signal length must be >= 1, got " + std::to_string(n));
  if (a_num < 1 || a_den < 1)
    return fail(ASX_ERR_INVALID, "density factor must be positive, got " + std::to_string(a_num) + "/" +
                                     std::to_string(a_den));
  if (dtype != ASX_C64 && dtype != ASX_C128) return fail(ASX_ERR_INVALID, "dtype must be ASX_C64 or ASX_C128");
  if (method < ASX_AUTO || method > ASX_CHIRP) return fail(ASX_ERR_INVALID, "unknown method");
  const int64_t g = gcd64(a_num, a_den);
  const int64_t a = a_num / g, d = a_den / g;  // α = a/d ; reference α_ref = d/a
  // Reference full-spectrum size (core.py:95-105 with DenseFactor(d, a)).
  const bool integral = ((n * d) % a) == 0;
  const int64_t m_ref = integral ? (n * d) / a : 0;
  if (m <= 0) {
    if (!integral)
      return fail(ASX_ERR_INCOMPATIBLE, "density factor " + std::to_string(d) + "/" + std::to_string(a) +
                                            " is incompatible with N=" + std::to_string(n) + ": alpha*N = " +
                                            std::to_string(n * d) + "/" + std::to_string(a) +
                                            " is not an integer");
    m = m_ref;
  }
  if (d > (int64_t(1) << 20) || a > (int64_t(1) << 20) || n > (int64_t(1) << 26))
    return fail(ASX_ERR_UNSUPPORTED, "alpha terms or N beyond the exact-reduction range");

  const int maxP = dtype == ASX_C64 ? kMaxP_c64 : kMaxP_c128;
  // α-FFT applicability (reference plan(): power-of-two N and alpha*N,
  // fastpath.py:97-101; generalised to any integer density r = d (a == 1),
  // or integer decimation fold = a with N/a a power of two (d == 1)).
  // The recursion always runs in FP64 (complex64 plans convert on load and
  // store): its error grows with the signal norm, and in FP32 it misses the
  // complex64 bound on signals whose energy lies outside the M-bin window
  // (config 4: 2.6e-5 against 2e-5), so the inner size is
  // capped at the FP64 engine's maxP for both dtypes.
  const int maxP_fft = kMaxP_c128;
  bool fft_ok = false, fft_large = false;
  int64_t fft_r = 1, fft_fold = 1, fft_P = 0;
  if (a == 1 && is_pow2(n) && n <= maxP_fft) {
    fft_ok = true;
    fft_r = d;
    fft_P = n;
  } else if (a == 1 && is_pow2(n) && is_pow2(d) && n > maxP_fft && n / maxP_fft <= 1024 && dtype == ASX_C128 &&
             m <= d * n) {
    // past one CTA: the four-step α-FFT (asx_large.cuh), complex128, power-of-two
    // r as the reference's plan() requires (fastpath.py:97-101), bins m < r N
    fft_ok = fft_large = true;
    fft_r = d;
    fft_P = n;
  } else if (d == 1 && n % a == 0 && is_pow2(n / a) && (n / a) <= maxP_fft) {
    fft_ok = true;
    fft_fold = a;
    fft_P = n / a;
  }
  // P >= N + M - 1 (linear convolution) and P >= 2N (the chirp kernel treats
  // the upper half of its FFT input as compile-time zero padding)
  const int64_t chirp_P = next_pow2(std::max(n + m - 1, 2 * n));
  // one CTA per transform up to maxP; beyond, the four-step path P = P1 x maxP
  const bool chirp_large = chirp_P > maxP && chirp_P / maxP <= 1024;
  const bool chirp_ok = chirp_P <= maxP || chirp_large;

  auto lg = [](int64_t v) { return (double)std::max(1, log2i(v)); };
  const double cost_direct_cuda = 8.0 * (double)n * (double)m * 0.5;
  // FP64 recursion: twice the FP32 cost for complex64 plans (B200 DFMA = FFMA / 2)
  const double cost_fft = fft_ok ? (dtype == ASX_C64 ? 2.0 : 1.0) *
                                       ((double)fft_r * (5.0 * fft_P * lg(fft_P) + 8.0 * fft_P) +
                                        (double)fft_fold * fft_P * 2.0)
                                 : 1e300;
  // direct form on the tensor cores (k_direct_tc): complex64 complex input,
  // N a multiple of the 32-sample K chunk, M = 128 or 256 bins (Re and Im of
  // the tile fill the 512 TMEM columns).  Cost in the same units, calibrated
  // on config 3 (N = M = 256: 0.375 ms against the chirp path's 0.470 ms).
  const char* no_dtc = std::getenv("ASX_NO_DTC");
  // N is capped at 1024: the tensor core's fp32 accumulation does not round
  // to nearest, so its error grows with the number of accumulate steps
  // (6 N / 16 per output); on coherent tone signals it measured 2.6e-5 of
  // max|X| at N = 2048 (over the 2e-5 bound) and stays below it up to 1024
  // (tests/test_gpu_direct_tc.py::test_long_signals_at_the_cap).  Longer
  // signals go to chirp-z.  The fp16 W image (8 M N bytes) stays <= 2 MiB.
  const bool dtc_ok = dtype == ASX_C64 && !real_input && n % 32 == 0 && n <= kDtcMaxN && (m == 128 || m == 256) &&
                      !(no_dtc && no_dtc[0] == '1');
  const double cost_direct = dtc_ok ? 0.75 * (double)n * (double)m : cost_direct_cuda;
  const double cost_chirp = chirp_ok ? 2.0 * 5.0 * chirp_P * lg(chirp_P) + 24.0 * chirp_P : 1e300;

  int chosen = method;
  if (method == ASX_AUTO) {
    chosen = ASX_DIRECT;
    double best = cost_direct;
    if (cost_fft < best) {
      best = cost_fft;
      chosen = ASX_FFT;
    }
    if (cost_chirp < best) {
      best = cost_chirp;
      chosen = ASX_CHIRP;
    }
  } else if (method == ASX_FFT && !fft_ok) {
    return fail(ASX_ERR_UNSUPPORTED,
                "fast path needs power-of-two N and an integer density (alpha = 1/r) or a power-of-two "
                "decimation (alpha = q, N/q a power of two), N <= " +
                    std::to_string(maxP_fft) + "; got N=" + std::to_string(n) + ", alpha=" + std::to_string(a) + "/" +
                    std::to_string(d) + "; use the naive transform for this pair");
  } else if (method == ASX_CHIRP && !chirp_ok) {
    return fail(ASX_ERR_UNSUPPORTED, "chirp path needs N+M-1 <= " + std::to_string(maxP * 1024) + " for this dtype");
  }
  if (chosen == ASX_DIRECT && (n * m > (int64_t(1) << 31)))
    return fail(ASX_ERR_UNSUPPORTED, "direct W matrix beyond 2^31 entries; use method fft/chirp");

  asx_plan_s* p = new (std::nothrow) asx_plan_s();
  if (!p) return fail(ASX_ERR_OOM, "host allocation failed");
  p->n = n;
  p->m = m;
  p->a = a;
  p->d = d;
  p->dtype = dtype;
  p->real_input = real_input ? 1 : 0;
  p->method = chosen;
  p->device = device;
  p->m_ref = m_ref;
  if (integral) {
    p->depth = bit_length(std::min(n, m_ref)) - 1;  // fastpath.py:102
    p->leaf = (d >= a) ? ASX_LEAF_SINGLE_SAMPLE : ASX_LEAF_BLOCK_SUM;  // fastpath.py:103
    p->pred_mults = (m_ref / 2) * p->depth;                              // fastpath.py:113-121
    p->pred_adds = m_ref * p->depth + (m_ref < n ? n - m_ref : 0);       // fastpath.py:124-127
  }

  DeviceGuard guard(device);
  if (!guard.ok) {
    delete p;
    return fail(ASX_ERR_CUDA, "cannot select CUDA device " + std::to_string(device) + " (no GPU?)");
  }
  {
    const char* no_tm = std::getenv("ASX_NO_TMEM");
    p->env.use_tmem = (no_tm && no_tm[0] == '1') ? 0 : 1;
    const char* no_loc = std::getenv("ASX_NO_LOCAL");
    p->env.use_local = (no_loc && no_loc[0] == '1') ? 0 : 1;
    const char* no_split = std::getenv("ASX_NO_SPLIT");
    p->env.use_split = (no_split && no_split[0] == '1') ? 0 : 1;
    const char* no_afl = std::getenv("ASX_NO_AFFT_LOCAL");
    p->env.use_afl = (no_afl && no_afl[0] == '1') ? 0 : 1;
    const char* no_r32 = std::getenv("ASX_NO_R32");
    p->env.use_r32 = (no_r32 && no_r32[0] == '1') ? 0 : 1;
    const char* no_rs = std::getenv("ASX_NO_RSPLIT");
    p->env.use_rsplit = (no_rs && no_rs[0] == '1') ? 0 : 1;
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && v > 0) p->env.sms = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) == cudaSuccess && v > 0)
      p->env.smem_optin = (size_t)v;
    cudaGetLastError();
  }
  // tables in the arithmetic precision: FP64 for every α-FFT plan
  const int dbl = dtype == ASX_C128 || chosen == ASX_FFT;
  const size_t es = dbl ? sizeof(double2) : sizeof(float2);
  // ---- table layout ----
  size_t elems = 0;
  int64_t twP_sz = 0, twA_sz = 0, chirp_sz = 0, H_sz = 0, W_sz = 0;
  if (chosen == ASX_FFT) {
    p->P = (int)fft_P;
    p->r = fft_r;
    p->fold = fft_fold;
  }
  int64_t twP1_sz = 0, twBig_sz = 0, A_sz = 0;
  if (chosen == ASX_FFT && fft_large) {
    p->large = p->large_fft = 1;
    p->P2 = maxP_fft;
    p->P1 = n / maxP_fft;
  }
  // must equal TwSplit<P>::LF (asx_engine.cuh)
  auto lf_of_P = [](int P) {
    const int LP = log2i(P);
    return (LP + 1) / 2;
  };
  if (chosen == ASX_FFT || chosen == ASX_CHIRP) {
    if (chosen == ASX_CHIRP) p->P = (int)chirp_P;
    twP_sz = two_level_size(p->P, lf_of_P(p->P));
  }
  if (p->large_fft) {
    twP_sz = two_level_size(p->P2, lf_of_P((int)p->P2));  // row FFT table W_P2
    twP1_sz = two_level_size(p->P1, lf_of_P((int)p->P1));
    p->lfBig = two_level_lf(p->r * n);
    twBig_sz = two_level_size(p->r * n, p->lfBig);  // W_{rN}: α pre-twiddle and four-step twiddle
    A_sz = n;
  }
  // four-step workspace: group x P elements, group = the signals one launch
  // set transforms (512 MiB of workspace, at least one signal)
  if (chosen == ASX_FFT && p->r > 1 && !p->large_fft) {
    p->lfA = two_level_lf(p->r * p->P);
    twA_sz = two_level_size(p->r * p->P, p->lfA);
  }
  if (chosen == ASX_CHIRP) {
    chirp_sz = std::max(n, m);
    H_sz = p->P;
  }
  if (chosen == ASX_CHIRP && chirp_large) {
    p->large = 1;
    p->P2 = maxP;
    p->P1 = chirp_P / maxP;
    twP_sz = two_level_size(p->P2, lf_of_P((int)p->P2));  // row FFT table W_P2
    twP1_sz = two_level_size(p->P1, lf_of_P((int)p->P1));
    p->lfBig = two_level_lf(chirp_P);
    twBig_sz = two_level_size(chirp_P, p->lfBig);
    A_sz = chirp_P;  // four-step workspace (x group, below)
  }
  if (p->large) {
    const size_t per = (dbl ? sizeof(double2) : sizeof(float2)) * (size_t)A_sz;
    p->group = std::max<int64_t>(1, std::min<int64_t>(4096, (int64_t)((512ull << 20) / per)));
    A_sz *= p->group;
  }
  if (chosen == ASX_DIRECT) W_sz = m * n;
  if (chosen == ASX_DIRECT && dtc_ok) {
    // the CTA-pair kernel (k_direct_tc2) measured 0.39 ms on config 3 against
    // 0.375 ms for k_direct_tc: built only in `make variant
    // VFLAGS=-DASX_DTC_PAIR=1` for further tuning, not in the shipped library
    p->dtc = (ASX_DTC_PAIR && m == 256) ? 2 : 1;
    W_sz = 2 * m * n;  // complex W (small-batch / misaligned launches) + the fp16 Wr/Wi hi/lo image (8 m n bytes)
  }
  const bool afl = chosen == ASX_FFT && dtype == ASX_C128 && p->P == AfftLocal::P && p->r == 2 && p->fold == 1;
  const int64_t afl_sz = afl ? AfftLocal::IMG_ELEMS : 0;
  p->tw_elems = (int)twA_sz;  // shared-memory table: α pre-twiddle only
  auto align = [](size_t v) { return (v + 31) & ~size_t(31); };
  p->off_twP = 0;
  elems = align(twP_sz);
  p->off_twA = elems * es;
  elems += align(twA_sz);
  p->off_chirp = elems * es;
  elems += align(chirp_sz);
  p->off_H = elems * es;
  elems += align(H_sz);
  p->off_W = elems * es;
  p->off_vimg = p->off_W + size_t(m * n) * es;
  elems += align(W_sz);
  p->off_twP1 = elems * es;
  elems += align(twP1_sz);
  p->off_twBig = elems * es;
  elems += align(twBig_sz);
  p->off_A = elems * es;
  elems += align(A_sz);
  p->off_afl = afl_sz ? elems * es : 0;
  elems += align(afl_sz);
  p->table_bytes = std::max<size_t>(elems * es, 64);

  cudaError_t e = cudaMalloc(&p->tables, p->table_bytes);
  if (e != cudaSuccess) {
    delete p;
    return cuda_fail(e, "cudaMalloc(plan tables)");
  }
  cudaStream_t st = nullptr;
  e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    cudaFree(p->tables);
    delete p;
    return cuda_fail(e, "cudaStreamCreate");
  }
  char* base = static_cast<char*>(p->tables);
  if (twP_sz) fill_two_level(base + p->off_twP, p->large ? p->P2 : p->P, lf_of_P(p->large ? (int)p->P2 : p->P), dbl, st);
  if (twP1_sz) fill_two_level(base + p->off_twP1, p->P1, lf_of_P((int)p->P1), dbl, st);
  if (twBig_sz) fill_two_level(base + p->off_twBig, p->large_fft ? p->r * n : chirp_P, p->lfBig, dbl, st);
  if (twA_sz) fill_two_level(base + p->off_twA, p->r * p->P, p->lfA, dbl, st);
  if (afl_sz) k_afl_image<<<(unsigned)((afl_sz + 255) / 256), 256, 0, st>>>(reinterpret_cast<double2*>(base + p->off_afl));
  double2* wP_d = nullptr;
  if (chosen == ASX_CHIRP) {
    const uint64_t L2 = 2ull * (uint64_t)d * (uint64_t)n;
    k_fill_chirp<<<(unsigned)std::min<int64_t>((chirp_sz + 255) / 256, 4096), 256, 0, st>>>(
        base + p->off_chirp, chirp_sz, (uint64_t)a, L2, dbl);
    if (p->large) {
      // H = FFT(h)/P with the same four-step kernels: h -> A (columns), rows -> Ht
      void* hbuf = nullptr;
      e = cudaMallocAsync(&hbuf, es * chirp_P, st);
      if (e == cudaSuccess) {
        if (dbl)
          k_fill_h<double><<<4096, 256, 0, st>>>(hbuf, base + p->off_chirp, chirp_P, n, m);
        else
          k_fill_h<float><<<4096, 256, 0, st>>>(hbuf, base + p->off_chirp, chirp_P, n, m);
        LParams lp;
        std::memset(&lp, 0, sizeof(lp));
        lp.n = n;
        lp.m = m;
        lp.h = hbuf;
        lp.A = base + p->off_A;
        lp.Hout = base + p->off_H;
        lp.twP1 = base + p->off_twP1;
        lp.twP2 = base + p->off_twP;
        lp.twBig = base + p->off_twBig;
        lp.lfBig = p->lfBig;
        lp.scale = 1.0 / (double)chirp_P;
        lp.P = chirp_P;
        lp.P2 = p->P2;
        lp.nsig = 1;
        e = launch_large(dbl, p->P1, COL_FWD_TABLE, 0, 0, lp, st);
        if (e == cudaSuccess) e = launch_large(dbl, p->P1, 0, ROW_SPECTRUM, 1, lp, st);
        p->row_local = (dbl && p->P2 == ChirpLocal128::P && p->env.use_local && p->env.use_tmem) ? 1 : 0;
        if (e == cudaSuccess && p->row_local) {
          // Ht rows in k_large_rows_local's per-thread spectrum order (hbuf is free again)
          k_permute_ht<<<4096, 256, 0, st>>>(static_cast<double2*>(hbuf),
                                             reinterpret_cast<const double2*>(base + p->off_H), p->P1);
          e = cudaMemcpyAsync(base + p->off_H, hbuf, es * chirp_P, cudaMemcpyDeviceToDevice, st);
        }
        cudaFreeAsync(hbuf, st);
      }
    } else if ((e = cudaMallocAsync(reinterpret_cast<void**>(&wP_d), 3 * sizeof(double2) * p->P, st)) ==
               cudaSuccess) {
      // H = FFT(h)/P in FP64: log2 P radix-2 Stockham levels against the exact W_P table
      double2 *src = wP_d + p->P, *dst = wP_d + 2 * p->P;
      k_fill_roots<<<(p->P + 255) / 256, 256, 0, st>>>(wP_d, p->P, 1, (uint64_t)p->P, 1);
      k_chirp_kernel_fp64<<<(p->P + 255) / 256, 256, 0, st>>>(src, p->P, n, m, (uint64_t)a, L2);
      for (int s = 1; s < p->P; s <<= 1) {
        k_stockham2_level<<<(p->P / 2 + 255) / 256, 256, 0, st>>>(src, dst, p->P, s, wP_d);
        std::swap(src, dst);
      }
      k_store_scaled<<<(p->P + 255) / 256, 256, 0, st>>>(base + p->off_H, p->P, src, dbl);
      cudaFreeAsync(wP_d, st);
    }
  }
  if (chosen == ASX_DIRECT) {
    const uint64_t L = (uint64_t)d * (uint64_t)n;
    const int64_t total = m * n;
    k_dft_matrix<<<(unsigned)std::min<int64_t>((total + 255) / 256, 65535), 256, 0, st>>>(
        base + p->off_W, m, n, (uint64_t)a, L, dbl);
#if ASX_DTC_PAIR
    if (p->dtc == 2) {
      dtc2::k_direct_tc2_image<<<(unsigned)std::min<int64_t>((total + 255) / 256, 65535), 256, 0, st>>>(
          reinterpret_cast<unsigned char*>(base + p->off_vimg), (int)n, (uint64_t)a, L);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(dtc2::k_direct_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, dtc2::SMEM_BYTES);
    } else
#endif
    if (p->dtc) {
      dtc::k_direct_tc_image<<<(unsigned)std::min<int64_t>((total + 255) / 256, 65535), 256, 0, st>>>(
          reinterpret_cast<unsigned char*>(base + p->off_vimg), (int)n, (int)m, (uint64_t)a, L);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(dtc::k_direct_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, dtc::SMEM_BYTES);
    }
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (e != cudaSuccess) {
    cudaFree(p->tables);
    delete p;
    return cuda_fail(e, "plan table build");
  }
  *out = p;
  return ASX_OK;
}

int asx_plan_destroy(asx_plan_t p) {
  if (!p) return ASX_OK;
  {
    DeviceGuard guard(p->device);
    for (int i = 0; i < asx_plan_s::kLanes; ++i) {
      if (p->lane[i]) cudaStreamDestroy(p->lane[i]);
      if (p->din[i]) cudaFree(p->din[i]);
      if (p->dout[i]) cudaFree(p->dout[i]);
    }
    for (auto& kv : p->ws_extra) cudaFree(kv.second);
    if (p->tables) cudaFree(p->tables);
  }
  delete p;
  return ASX_OK;
}

int asx_plan_query(asx_plan_t p, asx_plan_info* info) {
  if (!p || !info) return fail(ASX_ERR_INVALID, "NULL plan or info");
  std::memset(info, 0, sizeof(*info));
  info->n = p->n;
  info->m = p->m;
  info->a_num = p->a;
  info->a_den = p->d;
  info->m_ref = p->m_ref;
  info->depth = p->depth;
  info->leaf = p->leaf;
  info->method = p->method;
  info->dtype = p->dtype;
  info->real_input = p->real_input;
  info->fft_size = p->P;
  info->predicted_mults = p->pred_mults;
  info->predicted_adds = p->pred_adds;
  info->workspace_bytes = (int64_t)p->table_bytes;
  info->kernels_per_execute = p->large_fft ? (int32_t)(2 * std::min<int64_t>(p->r, p->m)) : p->large ? 3 : 1;
  info->batch_group = p->large ? p->group : 0;
  info->device = p->device;
  return ASX_OK;
}

int asx_execute(asx_plan_t p, const void* x, int64_t x_stride, void* X, int64_t X_stride, int64_t batch,
                void* stream) {
  if (!p) return fail(ASX_ERR_INVALID, "NULL plan");
  if (batch < 0) return fail(ASX_ERR_INVALID, "batch must be >= 0");
  if (batch > 0 && (!x || !X)) return fail(ASX_ERR_INVALID, "NULL data pointer");
  if (x_stride < p->n && batch > 1) return fail(ASX_ERR_INVALID, "x_stride smaller than n");
  if (X_stride < p->m && batch > 1) return fail(ASX_ERR_INVALID, "X_stride smaller than m");
  DeviceGuard guard(p->device);
  if (!guard.ok) return fail(ASX_ERR_CUDA, "cannot select CUDA device");
  return launch_execute(p, x, x_stride, X, X_stride, batch, static_cast<cudaStream_t>(stream));
}

int asx_execute_host(asx_plan_t p, const void* x, int64_t x_stride, void* X, int64_t X_stride, int64_t batch,
                     int64_t chunk) {
  if (!p) return fail(ASX_ERR_INVALID, "NULL plan");
  if (batch < 0) return fail(ASX_ERR_INVALID, "batch must be >= 0");
  if (batch == 0) return ASX_OK;
  if (!x || !X) return fail(ASX_ERR_INVALID, "NULL data pointer");
  if (x_stride < p->n || X_stride < p->m) return fail(ASX_ERR_INVALID, "row stride smaller than row length");
  std::lock_guard<std::mutex> lk(p->host_mtx);
  DeviceGuard guard(p->device);
  if (!guard.ok) return fail(ASX_ERR_CUDA, "cannot select CUDA device");
  const size_t ib = in_elem(p), ob = celem(p->dtype);
  const size_t in_row = (size_t)p->n * ib, out_row = (size_t)p->m * ob;
  // default: ~128 MiB of in+out per chunk, with chunk sizes ramping up from
  // 1/8 at the start and back down at the end, so the pipeline fill (first
  // H2D alone) and drain (last D2H alone) are short while the steady state
  // amortises the per-copy DMA setup (scripts/e2e_chunks.py)
  const bool ramp = chunk <= 0;
  if (ramp) chunk = std::max<int64_t>(1, (int64_t)((128ull << 20) / std::max(in_row + out_row, (size_t)1)));
  chunk = std::min(chunk, batch);
  std::vector<int64_t> sizes;
  {
    int64_t left = batch;
    if (ramp)
      for (int64_t s = std::max<int64_t>(1, chunk / 8); s < chunk && left > 0; s *= 2) {
        sizes.push_back(std::min(s, left));
        left -= sizes.back();
      }
    const int64_t smin = ramp ? std::max<int64_t>(1, chunk / 8) : chunk;
    while (left > 0) {
      int64_t s = chunk;
      if (ramp && left < 2 * chunk) s = std::max(smin, (left + 1) / 2);
      sizes.push_back(std::min(s, left));
      left -= sizes.back();
    }
  }
  if (chunk > p->lane_rows) {
    for (int i = 0; i < asx_plan_s::kLanes; ++i) {
      if (p->din[i]) cudaFree(p->din[i]);
      if (p->dout[i]) cudaFree(p->dout[i]);
      p->din[i] = p->dout[i] = nullptr;
    }
    p->lane_rows = 0;
    for (int i = 0; i < asx_plan_s::kLanes; ++i) {
      if (!p->lane[i]) CK(cudaStreamCreateWithFlags(&p->lane[i], cudaStreamNonBlocking));
      CK(cudaMalloc(&p->din[i], chunk * in_row));
      CK(cudaMalloc(&p->dout[i], chunk * out_row));
    }
    p->lane_rows = chunk;
  }
  int k = 0;
  int64_t b0 = 0;
  for (size_t c = 0; c < sizes.size(); b0 += sizes[c], ++c, k = (k + 1) % asx_plan_s::kLanes) {
    const int64_t rows = sizes[c];
    cudaStream_t st = p->lane[k];
    const char* src = static_cast<const char*>(x) + (size_t)b0 * x_stride * ib;
    char* dst = static_cast<char*>(X) + (size_t)b0 * X_stride * ob;
    if ((size_t)x_stride * ib == in_row)
      CK(cudaMemcpyAsync(p->din[k], src, rows * in_row, cudaMemcpyHostToDevice, st));
    else
      CK(cudaMemcpy2DAsync(p->din[k], in_row, src, (size_t)x_stride * ib, in_row, rows, cudaMemcpyHostToDevice,
                           st));
    int rc = launch_execute(p, p->din[k], p->n, p->dout[k], p->m, rows, st);
    if (rc != ASX_OK) return rc;
    if ((size_t)X_stride * ob == out_row)
      CK(cudaMemcpyAsync(dst, p->dout[k], rows * out_row, cudaMemcpyDeviceToHost, st));
    else
      CK(cudaMemcpy2DAsync(dst, (size_t)X_stride * ob, p->dout[k], out_row, out_row, rows, cudaMemcpyDeviceToHost,
                           st));
  }
  for (int i = 0; i < asx_plan_s::kLanes; ++i) CK(cudaStreamSynchronize(p->lane[i]));
  return ASX_OK;
}

int asx_dft_matrix(int64_t n, int64_t a_num, int64_t a_den, int64_t m_rows, int dtype, void* W, void* stream) {
  if (n < 1 || a_num < 1 || a_den < 1 || m_rows < 0) return fail(ASX_ERR_INVALID, "bad dft_matrix arguments");
  if (dtype != ASX_C64 && dtype != ASX_C128) return fail(ASX_ERR_INVALID, "bad dtype");
  if (m_rows == 0) return ASX_OK;
  if (!W) return fail(ASX_ERR_INVALID, "NULL output");
  const int64_t g = gcd64(a_num, a_den);
  const int64_t a = a_num / g, d = a_den / g;
  const int64_t total = m_rows * n;
  k_dft_matrix<<<(unsigned)std::min<int64_t>((total + 255) / 256, 65535), 256, 0,
                 static_cast<cudaStream_t>(stream)>>>(W, m_rows, n, (uint64_t)a, (uint64_t)(d * n),
                                                      dtype == ASX_C128);
  CK(cudaGetLastError());
  return ASX_OK;
}

int asx_combine(const void* y, const void* z, const void* tw, void* out, int64_t rows, int64_t half, int dtype,
                void* stream) {
  if (rows < 0 || half < 0) return fail(ASX_ERR_INVALID, "bad combine shape");
  if (rows * half == 0) return ASX_OK;
  if (!y || !z || !tw || !out) return fail(ASX_ERR_INVALID, "NULL pointer");
  const int64_t total = rows * half;
  const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 65535);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == ASX_C64)
    k_combine<float><<<blocks, 256, 0, st>>>(y, z, tw, out, rows, half);
  else if (dtype == ASX_C128)
    k_combine<double><<<blocks, 256, 0, st>>>(y, z, tw, out, rows, half);
  else
    return fail(ASX_ERR_INVALID, "bad dtype");
  CK(cudaGetLastError());
  return ASX_OK;
}

int asx_block_sum(const void* x, void* out, int64_t rows, int64_t len, int dtype, void* stream) {
  if (rows < 0 || len < 0) return fail(ASX_ERR_INVALID, "bad block_sum shape");
  if (rows == 0) return ASX_OK;
  if (!x || !out) return fail(ASX_ERR_INVALID, "NULL pointer");
  if (rows > 0x7fffffffLL) return fail(ASX_ERR_INVALID, "too many rows");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == ASX_C64)
    k_block_sum<float><<<(unsigned)rows, 256, 0, st>>>(x, out, rows, len);
  else if (dtype == ASX_C128)
    k_block_sum<double><<<(unsigned)rows, 256, 0, st>>>(x, out, rows, len);
  else
    return fail(ASX_ERR_INVALID, "bad dtype");
  CK(cudaGetLastError());
  return ASX_OK;
}

}  // extern "C"

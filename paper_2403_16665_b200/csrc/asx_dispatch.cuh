// asx_dispatch.cuh — launch configuration and kernel dispatch, shared by the
// translation units that instantiate the kernels (asx_launch_f32.cu,
// asx_launch_f64.cu, asx_launch_misc.cu) and the C ABI (asx_api.cu), so the
// sm_100a kernels compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "../../include/asx.h"
#include "asx_afft_local.cuh"
#include "asx_chirp_local.cuh"
#include "asx_chirp_local128.cuh"
#include "asx_chirp_r32.cuh"
#include "asx_large.cuh"

namespace asx_host {
using namespace asx;

struct LaunchEnv {
  int sms = 148;
  size_t smem_optin = 227 * 1024;
  int use_tmem = 1;  // chirp tables in tensor memory (env ASX_NO_TMEM=1 disables, for A/B runs)
  int use_local = 1; // P = 16384 complex64 chirp on k_chirp_local (env ASX_NO_LOCAL=1 disables)
  int use_split = 1; // α-FFT residues split over two teams sharing a staged row (env ASX_NO_SPLIT=1 disables)
  int use_afl = 1;   // complex128 N = 4096, α = 1/2 α-FFT on k_afft_local (env ASX_NO_AFFT_LOCAL=1 disables)
  int use_rsplit = 1; // small α-FFT batches: one team per (signal, residue) (env ASX_NO_RSPLIT=1 disables)
  int use_r32 = 1;   // P = 16384 complex64 chirp at 32 values per thread, k_chirp_r32 (env ASX_NO_R32=1 disables)
};

// Shape of the most recent launch on this thread (asx_last_launch, for
// benchmarks / tests that report occupancy decisions).
struct LastLaunch {
  int grid = 0, block = 0, smem = 0, staged = 0, tmem = 0;
};
extern thread_local LastLaunch g_last_launch;

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
#ifndef ASX_R_512_C64
#define ASX_R_512_C64 16  // values per thread for c64 P == 512: one warp per transform
#endif
#ifndef ASX_KR_C128_4K
#define ASX_KR_C128_4K 1
#endif
#ifndef ASX_KR_C64_8K
#define ASX_KR_C64_8K 1
#endif
#ifndef ASX_MT_C64
#define ASX_MT_C64 1024  // threads per SM the register budget targets (c64)
#endif
#ifndef ASX_MT_C128
#define ASX_MT_C128 512  // threads per SM the register budget targets (c128)
#endif
#ifndef ASX_MT_C128_4K
#define ASX_MT_C128_4K 1024  // the same for c128 P == 4096 (two CTAs per SM: config 1a 0.262 -> 0.242 ms)
#endif
template <int P, typename Real> struct Cfg {
  static constexpr bool DBL = sizeof(Real) == 8;
  static constexpr int R = (P <= 32)                 ? P
                           : (P == 512 && !DBL) ? ASX_R_512_C64
                           : (P <= 2048)        ? 8
                           : DBL         ? (P == 4096 ? ASX_R_4K_C128 : 16)
                                         : (P == 16384 ? ASX_R_16K_C64 : ASX_R_BIG_C64);
  static constexpr int NT = P / R;
  static constexpr int TPB = (NT == 1) ? 64 : (NT >= 256 ? 1 : 256 / NT);
  static constexpr int MT = DBL ? (P == 4096 ? ASX_MT_C128_4K : ASX_MT_C128) : ASX_MT_C64;
  static constexpr int MINB = (MT / (NT * TPB)) > 1 ? (MT / (NT * TPB)) : 1;
  // α-FFT residues transformed together per thread (ILP for the latency-bound FP64 case)
  static constexpr int KR = (DBL && P == 4096) ? ASX_KR_C128_4K : ((!DBL && P == 8192) ? ASX_KR_C64_8K : 1);
};

template <typename KernelT>
cudaError_t prep_smem(KernelT kern, size_t smem) {
  if (smem > 48 * 1024) return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return cudaSuccess;
}

// IO: element type of the signals / bins when it differs from the arithmetic
// type (complex64 α-FFT plans: IO = float, Real = double).
template <typename Real, int P, int KIND, typename IO = Real>
cudaError_t launch_persist(KParams kp, int64_t batch, cudaStream_t st, const LaunchEnv& env) {
  using G = Cfg<P, Real>;
  constexpr bool SAME_IO = sizeof(IO) == sizeof(Real);
  constexpr int KR = KIND == KIND_AFFT ? G::KR : 1;
  constexpr bool DBUF = persist_dbuf<Real, P, G::NT, KIND>();
  using L = PersistLayout<Real, P, G::NT, G::TPB, false, KR, DBUF>;
  if (batch == 0) return cudaSuccess;
  const size_t row_bytes = size_t(kp.n) * (kp.real_in ? sizeof(IO) : 2 * sizeof(IO));
  auto kern = k_fft_persist<Real, P, G::NT, G::TPB, KIND, G::MINB, false, KR, false, false, IO>;
  // one-time opt-in to the full shared-memory carve-out for this kernel
  static thread_local int attr_set_for = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_set_for != dev) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)env.smem_optin);
    if (e != cudaSuccess) return e;
    attr_set_for = dev;
  }
  // occupancy with / without the TMA staging buffer (cached per smem size);
  // staging is used only when it does not cost resident CTAs.
  struct Occ {
    size_t smem = 0;
    int per_sm = 0;
  };
  static thread_local Occ cache[2];
  auto occ = [&](int stg, size_t sm) -> int {
    if (sm > env.smem_optin) return 0;
    Occ& c = cache[stg];
    if (c.smem != sm) {
      int v = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, G::NT * G::TPB, sm) != cudaSuccess) {
        cudaGetLastError();
        v = 0;
      }
      c.smem = sm;
      c.per_sm = v;
    }
    return c.per_sm;
  };
  if (G::NT == 1) kp.staged = 0;
  if constexpr (SAME_IO && KIND == KIND_AFFT && G::NT == 512 && sizeof(Real) == 4 &&
                size_t(P) * 2 * sizeof(Real) <= 65536) {
    // two 512-thread teams per CTA split one signal's residues, one TMA-staged row
    // (complex64 P = 8192: config 4 alpha-FFT 19.2 -> 17.5 ms; complex128 P = 4096
    // measured slower than two independent CTAs per SM: 0.260 vs 0.242 ms)
    using LS = PersistLayout<Real, P, G::NT, 2, false, 1, DBUF, 1>;
    auto ks = k_fft_persist<Real, P, G::NT, 2, KIND_AFFT, 1, false, 1, true>;
    const size_t smem_s = LS::total(row_bytes, true, kp.tw_elems);
    if (env.use_split && kp.r >= 2 && kp.staged && smem_s <= env.smem_optin) {
      static thread_local int sp_attr_for = -1;
      int dev_s = 0;
      cudaGetDevice(&dev_s);
      if (sp_attr_for != dev_s) {
        cudaError_t e = cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)env.smem_optin);
        if (e != cudaSuccess) return e;
        sp_attr_for = dev_s;
      }
      const int64_t grid_s = std::min<int64_t>(batch, env.sms);
      kp.batch = batch;
      ks<<<(unsigned)grid_s, 2 * G::NT, smem_s, st>>>(kp);
      g_last_launch.tmem = 3;
      g_last_launch.grid = (int)grid_s;
      g_last_launch.block = 2 * G::NT;
      g_last_launch.smem = (int)smem_s;
      g_last_launch.staged = kp.staged;
      return cudaGetLastError();
    }
  }
  if constexpr (SAME_IO && KIND == KIND_AFFT && sizeof(Real) == 8 && P == AfftLocal::P) {
    // group-local α-FFT kernel (asx_afft_local.cuh): one CTA (two residue teams) per SM
    if (env.use_afl && kp.r == 2 && kp.fold == 1 && !kp.real_in && kp.n == P && kp.m <= P && kp.staged &&
        kp.afl && batch < (int64_t(1) << 31) && AfftLocal::SMEM <= env.smem_optin) {
      auto ka = k_afft_local<double>;
      static thread_local int afl_attr_for = -1;
      int dev_a = 0;
      cudaGetDevice(&dev_a);
      if (afl_attr_for != dev_a) {
        cudaError_t e = cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AfftLocal::SMEM);
        if (e != cudaSuccess) return e;
        afl_attr_for = dev_a;
      }
      const int64_t grid_a = std::min<int64_t>(batch, env.sms);
      kp.batch = batch;
      ka<<<(unsigned)grid_a, AfftLocal::NTH, AfftLocal::SMEM, st>>>(kp);
      g_last_launch.tmem = 4;
      g_last_launch.grid = (int)grid_a;
      g_last_launch.block = AfftLocal::NTH;
      g_last_launch.smem = (int)AfftLocal::SMEM;
      g_last_launch.staged = 1;
      return cudaGetLastError();
    }
  }
  if constexpr (KIND == KIND_CHIRP && sizeof(Real) == 8 && P == ChirpLocal128::P) {
    // complex128 group-local chirp kernel (asx_chirp_local128.cuh): one CTA per SM
    if (env.use_local && env.use_tmem && 2 * kp.m <= P && 2 * kp.n <= P && batch < (int64_t(1) << 31)) {
      using CL = ChirpLocal128;
      auto kl = k_chirp_local128<double>;
      size_t smem_l = CL::total(row_bytes, kp.staged != 0);
      if (smem_l > env.smem_optin) {
        kp.staged = 0;
        smem_l = CL::total(row_bytes, false);
      }
      static thread_local int cl_attr_for = -1;
      int dev_l = 0;
      cudaGetDevice(&dev_l);
      if (cl_attr_for != dev_l) {
        cudaError_t e = cudaFuncSetAttribute(kl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)env.smem_optin);
        if (e != cudaSuccess) return e;
        cl_attr_for = dev_l;
      }
      const int64_t grid_l = std::min<int64_t>(batch, env.sms);
      kp.batch = batch;
      kl<<<(unsigned)grid_l, CL::NT, smem_l, st>>>(kp);
      g_last_launch.tmem = 6;
      g_last_launch.grid = (int)grid_l;
      g_last_launch.block = CL::NT;
      g_last_launch.smem = (int)smem_l;
      g_last_launch.staged = kp.staged;
      return cudaGetLastError();
    }
  }
  if constexpr (KIND == KIND_CHIRP && sizeof(Real) == 4 && P == ChirpR32::P) {
    // 32 values per thread, 4 exchanges per signal (asx_chirp_r32.cuh): one CTA per SM
    if (env.use_r32 && env.use_local && env.use_tmem && 2 * kp.m <= P && 2 * kp.n <= P &&
        batch < (int64_t(1) << 31)) {
      using CR = ChirpR32;
      auto kr = k_chirp_r32<float>;
      size_t smem_r = CR::total(row_bytes, kp.staged != 0);
      if (smem_r > env.smem_optin) {
        kp.staged = 0;
        smem_r = CR::total(row_bytes, false);
      }
      static thread_local int cr_attr_for = -1;
      int dev_r = 0;
      cudaGetDevice(&dev_r);
      if (cr_attr_for != dev_r) {
        cudaError_t e = cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)env.smem_optin);
        if (e != cudaSuccess) return e;
        cr_attr_for = dev_r;
      }
      const int64_t grid_r = std::min<int64_t>(batch, env.sms);
      kp.batch = batch;
      kr<<<(unsigned)grid_r, CR::NT, smem_r, st>>>(kp);
      g_last_launch.tmem = 14;
      g_last_launch.grid = (int)grid_r;
      g_last_launch.block = CR::NT;
      g_last_launch.smem = (int)smem_r;
      g_last_launch.staged = kp.staged;
      return cudaGetLastError();
    }
  }
  if constexpr (KIND == KIND_CHIRP && sizeof(Real) == 4 && P == ChirpLocal::P) {
    // group-local exchange kernel (asx_chirp_local.cuh): one CTA per SM
    if (env.use_local && env.use_tmem && 2 * kp.m <= P && 2 * kp.n <= P && batch < (int64_t(1) << 31)) {
      using CL = ChirpLocal;
      auto kl = k_chirp_local<float>;
      size_t smem_l = CL::total<typename CT<Real>::T>(row_bytes, kp.staged != 0);
      if (smem_l > env.smem_optin) {
        kp.staged = 0;
        smem_l = CL::total<typename CT<Real>::T>(row_bytes, false);
      }
      static thread_local int cl_attr_for = -1;
      int dev_l = 0;
      cudaGetDevice(&dev_l);
      if (cl_attr_for != dev_l) {
        cudaError_t e = cudaFuncSetAttribute(kl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)env.smem_optin);
        if (e != cudaSuccess) return e;
        cl_attr_for = dev_l;
      }
      const int64_t grid_l = std::min<int64_t>(batch, env.sms);
      kp.batch = batch;
      kl<<<(unsigned)grid_l, CL::NT, smem_l, st>>>(kp);
      g_last_launch.tmem = 2;
      g_last_launch.grid = (int)grid_l;
      g_last_launch.block = CL::NT;
      g_last_launch.smem = (int)smem_l;
      g_last_launch.staged = kp.staged;
      return cudaGetLastError();
    }
  }
  const size_t smem_u = L::total(row_bytes, false, kp.tw_elems);
  const int occ_u = occ(0, smem_u);
  size_t smem = smem_u;
  int per_sm = occ_u;
  if (kp.staged) {
    const size_t smem_s = L::total(row_bytes, true, kp.tw_elems);
    const int occ_s = occ(1, smem_s);
    if (occ_s >= occ_u && occ_s > 0) {
      smem = smem_s;
      per_sm = occ_s;
    } else {
      kp.staged = 0;
    }
  }
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  bool rsplit = false;
  int64_t units = batch;
  if constexpr (KIND == KIND_AFFT && KR == 1) {
    // fewer signals than resident teams: one (signal, residue) pair per team
    // instead of one signal, so a single signal's r residues run in parallel
    if (env.use_rsplit && kp.r > 1 && batch < int64_t(env.sms) * per_sm * G::TPB && batch * kp.r < (int64_t(1) << 31)) {
      rsplit = true;
      units = batch * kp.r;
    }
  }
  const int64_t need = (units + G::TPB - 1) / G::TPB;
  const int64_t grid = std::min<int64_t>(need, int64_t(env.sms) * per_sm);
  kp.batch = batch;
  int tm_used = 0;
  if constexpr (KIND == KIND_CHIRP && G::NT > 1 &&
                TmemCfg<Real, G::NT * G::TPB, G::R, Fft<Real, P, G::NT, ASX_TWTAB_MAX, true>::TSEED_COLS>::OK) {
    using TMC = TmemCfg<Real, G::NT * G::TPB, G::R, Fft<Real, P, G::NT, ASX_TWTAB_MAX, true>::TSEED_COLS>;
    using LT = PersistLayout<Real, P, G::NT, G::TPB, true, 1, DBUF>;
    if (env.use_tmem && per_sm * TMC::NCOLS <= 512 && 2 * kp.m <= P &&
        LT::total(row_bytes, kp.staged != 0, kp.tw_elems) <= smem) {
      auto kern_tm = k_fft_persist<Real, P, G::NT, G::TPB, KIND, G::MINB, true>;
      static thread_local int tm_attr_for = -1;
      if (tm_attr_for != dev) {
        cudaError_t e = cudaFuncSetAttribute(kern_tm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)env.smem_optin);
        if (e != cudaSuccess) return e;
        tm_attr_for = dev;
      }
      kern_tm<<<(unsigned)grid, G::NT * G::TPB, smem, st>>>(kp);
      tm_used = 1;
    }
  }
  if constexpr (KIND == KIND_AFFT && KR == 1) {
    if (rsplit) {
      auto kern_rs = k_fft_persist<Real, P, G::NT, G::TPB, KIND, G::MINB, false, KR, false, true, IO>;
      static thread_local int rs_attr_for = -1;
      if (rs_attr_for != dev) {
        cudaError_t e = cudaFuncSetAttribute(kern_rs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)env.smem_optin);
        if (e != cudaSuccess) return e;
        rs_attr_for = dev;
      }
      kern_rs<<<(unsigned)grid, G::NT * G::TPB, smem, st>>>(kp);
      tm_used = -1;
    }
  }
  if (!tm_used) kern<<<(unsigned)grid, G::NT * G::TPB, smem, st>>>(kp);
  if (tm_used < 0) tm_used = 0;
  g_last_launch.tmem = tm_used;
  g_last_launch.grid = (int)grid;
  g_last_launch.block = G::NT * G::TPB;
  g_last_launch.smem = (int)smem;
  g_last_launch.staged = kp.staged;
  return cudaGetLastError();
}

template <typename Real>
cudaError_t launch_by_size(int which, int P, const KParams& kp, int64_t batch, cudaStream_t st,
                           const LaunchEnv& env) {
  switch (P) {
#define ASX_CASE(S)                                                               \
  case S:                                                                         \
    return which == ASX_FFT ? launch_persist<Real, S, KIND_AFFT>(kp, batch, st, env) \
                            : launch_persist<Real, S, KIND_CHIRP>(kp, batch, st, env);
    ASX_CASE(1)
    ASX_CASE(2)
    ASX_CASE(4)
    ASX_CASE(8)
    ASX_CASE(16)
    ASX_CASE(32)
    ASX_CASE(64)
    ASX_CASE(128)
    ASX_CASE(256)
    ASX_CASE(512)
    ASX_CASE(1024)
    ASX_CASE(2048)
    ASX_CASE(4096)
    ASX_CASE(8192)
#undef ASX_CASE
    case 16384:
      if constexpr (sizeof(Real) == 4)
        return which == ASX_FFT ? launch_persist<Real, 16384, KIND_AFFT>(kp, batch, st, env)
                                : launch_persist<Real, 16384, KIND_CHIRP>(kp, batch, st, env);
      return cudaErrorInvalidValue;
    default:
      return cudaErrorInvalidValue;
  }
}

template <typename Real, int P1>
cudaError_t launch_cols(int mode, const LParams& lp, cudaStream_t st) {
  using G = ColCfg<Real, P1>;
  const int64_t tiles = (lp.P2 / kColTile) * std::max<int64_t>(lp.nsig, 1);
  cudaError_t e = cudaSuccess;
  auto go = [&](auto kern) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    // persistent: as many CTAs as fit on the device at once
    int per_sm = 0, sms = 148, dev = 0;
    if (e == cudaSuccess && (cudaGetDevice(&dev) != cudaSuccess ||
                             cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
                             cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::NT * kColTile, G::SMEM) !=
                                 cudaSuccess))
      cudaGetLastError();
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, int64_t(sms) * std::max(per_sm, 1));
    if (e == cudaSuccess) kern<<<grid, G::NT * kColTile, G::SMEM, st>>>(lp);
  };
  if (mode == COL_AFFT)
    go(k_large_cols<Real, P1, G::NT, COL_AFFT>);
  else if (mode == COL_FWD_SIGNAL)
    go(k_large_cols<Real, P1, G::NT, COL_FWD_SIGNAL>);
  else if (mode == COL_FWD_TABLE)
    go(k_large_cols<Real, P1, G::NT, COL_FWD_TABLE>);
  else
    go(k_large_cols<Real, P1, G::NT, COL_INV_OUT>);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <typename Real>
cudaError_t launch_cols_p1(int64_t P1, int mode, const LParams& lp, cudaStream_t st) {
  switch (P1) {
#define ASX_COL(S) \
  case S:          \
    return launch_cols<Real, S>(mode, lp, st);
    ASX_COL(2)
    ASX_COL(4)
    ASX_COL(8)
    ASX_COL(16)
    ASX_COL(32)
    ASX_COL(64)
    ASX_COL(128)
    ASX_COL(256)
    ASX_COL(512)
    ASX_COL(1024)
#undef ASX_COL
    default:
      return cudaErrorInvalidValue;
  }
}

template <typename Real>
cudaError_t launch_rows(int mode, int64_t P1, const LParams& lp, cudaStream_t st) {
  constexpr int P2 = sizeof(Real) == 4 ? 16384 : 8192;
  using G = Cfg<P2, Real>;
  using E = Fft<Real, P2, G::NT>;
  const size_t smem = size_t(E::SMEM_ELEMS + E::TAB_ELEMS + 2) * sizeof(typename CT<Real>::T) + 16;
  cudaError_t e = cudaSuccess;
  auto go = [&](auto kern) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      cudaGetLastError();
    if (e == cudaSuccess) kern<<<(unsigned)std::min<int64_t>(P1 * std::max<int64_t>(lp.nsig, 1), sms), G::NT, smem, st>>>(lp);
  };
  if constexpr (sizeof(Real) == 8) {
    if (mode == ROW_MAIN_LOCAL) {
      auto kern = k_large_rows_local<double>;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RowsLocal::SMEM);
      int sms = 148, dev = 0;
      if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        cudaGetLastError();
      if (e == cudaSuccess)
        kern<<<(unsigned)std::min<int64_t>(P1 * std::max<int64_t>(lp.nsig, 1), sms), ChirpLocal128::NT, RowsLocal::SMEM,
               st>>>(lp);
      if (e != cudaSuccess) return e;
      return cudaGetLastError();
    }
  }
  if (mode == ROW_AFFT)
    go(k_large_rows<Real, P2, G::NT, ROW_AFFT>);
  else if (mode == ROW_SPECTRUM)
    go(k_large_rows<Real, P2, G::NT, ROW_SPECTRUM>);
  else
    go(k_large_rows<Real, P2, G::NT, ROW_MAIN>);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_large(int dbl, int64_t P1, int mode_cols, int mode_rows, int which, const LParams& lp,
                         cudaStream_t st);

// complex64 α-FFT plans: the FP64 recursion with complex64 loads / stores
// (asx_launch_mixed.cu)
cudaError_t launch_afft_io32(int P, const KParams& kp, int64_t batch, cudaStream_t st, const LaunchEnv& env);

extern template cudaError_t launch_by_size<float>(int, int, const KParams&, int64_t, cudaStream_t, const LaunchEnv&);
extern template cudaError_t launch_by_size<double>(int, int, const KParams&, int64_t, cudaStream_t, const LaunchEnv&);
extern template cudaError_t launch_cols_p1<float>(int64_t, int, const LParams&, cudaStream_t);
extern template cudaError_t launch_cols_p1<double>(int64_t, int, const LParams&, cudaStream_t);
extern template cudaError_t launch_rows<float>(int, int64_t, const LParams&, cudaStream_t);
extern template cudaError_t launch_rows<double>(int, int64_t, const LParams&, cudaStream_t);

}  // namespace asx_host

// asx_chirp_local.cuh — chirp-z convolution for P = 16384 (complex64) with
// group-local exchanges: the config-4 hot kernel (BASELINE config 4:
// N = M = 8192, α = 1/8).
//
// Same mathematics as k_fft_persist<KIND_CHIRP> (the α-DFT as the chirp-z
// convolution X_m = c_m Σ_n (x_n c_n) conj(c_{m-n}), fastpath.py:162-181 /
// oracle.py:50-67 restated), but the P-point forward FFT is decimation in
// FREQUENCY and the inverse its exact transpose (decimation in time on the
// digit-reversed spectrum), so the spectrum is never reordered and most data
// exchanges stay inside small thread groups:
//
//   P1  radix-16 DIF over x[t + 1024 i] (the io layout, no exchange), twiddle
//       W_16384^{t k1}                          -> 16 sub-problems of 1024
//   G1  global exchange (CTA barrier): sub-problem k1 -> threads 64 k1 ..
//   P2  radix-4 DIF (4 groups/thread), twiddle W_1024^{n' k2} (exact table)
//   L1  exchange inside the 2-warp group (named barrier)
//   P3  radix-16 DIF, twiddle W_256^{n'' k3}    -> 16-point sub-problems
//   L2  exchange inside the half-warp (__syncwarp)
//   P4  radix-16 DIF, no twiddle                -> Y[f], f = k1 + 16 k2 + 64 k3 + 1024 k4
//   × H[f] (tensor memory, stored in this per-thread order), conj
//   Q1..Q4 = P4ᵀ..P1ᵀ on the same thread/data mapping (twiddle, then butterfly,
//   then the inverse exchange), ending in the io layout: X[t + 1024 i].
//
// Per signal: 2 CTA-wide exchanges instead of 6, 2 group-local, 2 warp-local;
// warps drift apart inside the local phases so butterflies (FP32 pipe) and
// exchanges (shared-memory pipe) of different groups overlap.
#pragma once

#include "asx_kernels.cuh"

namespace asx {

struct ChirpLocal {
  static constexpr int P = 16384, NT = 1024, R = 16;
  static constexpr int L2S = 18;        // L2 row stride: 16-byte aligned rows, conflict-free columns
  static constexpr int SUB = 288;       // one 256-element sub-block (+32 pad: L2's 18-stride rows fit)
  static constexpr int REG = 4 * SUB;   // one 1024-point sub-problem
  static constexpr int XB = 16 * REG;   // exchange buffer (complex elements)
  static constexpr int T2N = 3 * 256;   // W_1024^{n' k2}, k2 = 1..3, n' < 256
  static constexpr int T3S = 18;        // T3 row stride: 16-byte aligned rows, conflict-free 128-bit reads
  static constexpr int T3N = 16 * T3S;  // row n'' < 16: W_256^{n'' k3} at column k3 (exact; chain variant: seeds)
  static constexpr int CPT = 64;        // TMEM columns per thread: H 32 | chirp 16 | P1 twiddles 16
  // position of element n (< 1024) of a sub-problem inside its region
  __host__ __device__ static constexpr int pos(int n) { return n + (n >> 8) * (SUB - 256); }
  template <typename C>
  __host__ __device__ static size_t stage_off() { return align_up(size_t(XB) * sizeof(C), 128); }
  template <typename C>
  __host__ __device__ static size_t tab_off(size_t row_bytes, bool staged) {
    return stage_off<C>() + (staged ? align_up(row_bytes, 128) : 0);
  }
  template <typename C>
  __host__ __device__ static size_t bar_off(size_t row_bytes, bool staged) {
    return align_up(tab_off<C>(row_bytes, staged) + size_t(T2N + T3N) * sizeof(C), 16);
  }
  template <typename C>
  __host__ __device__ static size_t total(size_t row_bytes, bool staged) {
    return bar_off<C>(row_bytes, staged) + 2 * sizeof(uint64_t) + 16;  // stage mbar, WAR mbar, TMEM slot
  }
};

template <typename C>
__device__ __forceinline__ C exact_w(int e, int L) {  // W_L^e rounded once from FP64
  double sn, cs;
  sincospi(2.0 * double(e) / double(L), &sn, &cs);
  using Rl = decltype(C{}.x);
  return mk(Rl(cs), Rl(-sn));
}

// Complex product whose components carry the exact residual of one of their
// two products (FMA error-free transformation): nearly correctly rounded.
template <typename C>
__device__ __forceinline__ C cmul_acc(C a, C b) {
  using Real = decltype(a.x);
  const Real p1 = a.x * b.x, e1 = fma(a.x, b.x, -p1);
  const Real p2 = a.x * b.y, e2 = fma(a.x, b.y, -p2);
  return mk(fma(-a.y, b.y, p1) + e1, fma(a.y, b.x, p2) + e2);
}

// u[r] *= w^r (r < 16) from exact w, w^2, w^3 and exact seeds w^{4a}
// (w = {w1, w2, w3, s1, s2, s3, -, -}): every applied twiddle is one
// compensated product of exactly rounded values.
template <typename C>
__device__ __forceinline__ void tw16_apply(C (&u)[16], const C (&w)[8]) {
  u[1] = cmul(u[1], w[0]);
  u[2] = cmul(u[2], w[1]);
  u[3] = cmul(u[3], w[2]);
#pragma unroll
  for (int a = 1; a < 4; ++a) {
    const C w4a = w[2 + a];
    u[4 * a] = cmul(u[4 * a], w4a);
    u[4 * a + 1] = cmul(u[4 * a + 1], cmul_acc(w4a, w[0]));
    u[4 * a + 2] = cmul(u[4 * a + 2], cmul_acc(w4a, w[1]));
    u[4 * a + 3] = cmul(u[4 * a + 3], cmul_acc(w4a, w[2]));
  }
}

// two adjacent complex64 values as one 16-byte shared-memory access
__device__ __forceinline__ void ld_pair(const float2* a, float2& x, float2& y) {
  const float4 w = *reinterpret_cast<const float4*>(a);
  x = make_float2(w.x, w.y);
  y = make_float2(w.z, w.w);
}
__device__ __forceinline__ void st_pair(float2* a, float2 x, float2 y) {
  *reinterpret_cast<float4*>(a) = make_float4(x.x, x.y, y.x, y.y);
}

__device__ __forceinline__ void group_bar(int id) {
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}

// Timing diagnostics (variant builds only, -DASX_CL_TIMELINE=<iteration>): warp
// leaders of CTA 0 stamp clock64() at the phase boundaries of two consecutive
// signals into the row AFTER the last output row (the caller allocates it).
#ifdef ASX_CL_TIMELINE
#define CL_TL(i)                                                                                  \
  do {                                                                                            \
    if (blockIdx.x == 0 && (t & 31) == 0 && (it == ASX_CL_TIMELINE || it == ASX_CL_TIMELINE + 1)) \
      tl[((it - ASX_CL_TIMELINE) * 32 + warp) * 32 + (i)] = clock64();                            \
  } while (0)
#else
#define CL_TL(i)
#endif

template <typename Real>
__global__ void __launch_bounds__(1024, 1) k_chirp_local(KParams p) {
  using C = typename CT<Real>::T;
  using L = ChirpLocal;
  static_assert(sizeof(C) == 8, "TMEM column layout assumes complex64");
  constexpr int WPC = 2, CPC = 4;  // words per complex, complex per 8-column TMEM access
  extern __shared__ __align__(128) unsigned char smraw[];
  C* xb = reinterpret_cast<C*>(smraw);
  const int t = threadIdx.x, warp = t >> 5;
  const int gk = t >> 6;           // P2/Q3: sub-problem k1 of this thread's group
  const int tau = t & 63;          // P2/Q3: n' = 2 tau + (g & 1) + 128 (g >> 1) (adjacent pairs)
  const int k2 = tau >> 4;         // P3..Q2: sub-block
  const int n16 = t & 15;          // P3/Q2: n''; P4/Q1: k3
  const int gbar = 1 + (t >> 7);   // named barrier of this 4-warp pair of groups
  const bool staged = p.staged != 0;
  const size_t row_bytes = size_t(p.n) * (p.real_in ? sizeof(Real) : sizeof(C));
  unsigned char* stage = smraw + L::stage_off<C>();
  C* T2 = reinterpret_cast<C*>(smraw + L::tab_off<C>(row_bytes, staged));
  C* T3 = T2 + L::T2N;
  uint64_t* stbar = reinterpret_cast<uint64_t*>(smraw + L::bar_off<C>(row_bytes, staged));
  uint64_t* war = stbar + 1;
  uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(stbar + 2);

  for (int e = t; e < L::T2N; e += L::NT) T2[e] = exact_w<C>((e & 255) * (e / 256 + 1), 1024);
  for (int e = t; e < L::T3N; e += L::NT) {
    const int row = e / L::T3S, col = e % L::T3S;  // n'', k3
    T3[e] = exact_w<C>(col < 16 ? row * col : 0, 256);
  }
  if (t == 0) {
    mbar_init(stbar, 1);
    mbar_init(war, L::NT / 32);
    fence_mbar_init();
  }
  const int stride = int(gridDim.x);
  int u = int(blockIdx.x);
  const int batch = int(p.batch);
  const int iters = (batch + stride - 1) / stride;
  const C* chirp = reinterpret_cast<const C*>(p.chirp);
  const C* H = reinterpret_cast<const C*>(p.H);

  // tensor memory: H in this thread's spectrum order, the chirp, P1 seeds
  if (warp == 0) tmem_alloc(&tmem_slot, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = tmem_slot + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * L::CPT);
  {
    const int fbase = gk + 16 * k2 + 64 * n16;  // f = fbase + 1024 k4
#pragma unroll
    for (int j0 = 0; j0 < 16; j0 += CPC) {
      uint32_t wh[8], wc[8];
#pragma unroll
      for (int k = 0; k < CPC; ++k) {
        c_to_words(__ldg(H + fbase + 1024 * (j0 + k)), &wh[k * WPC]);
        const int idx = t + 1024 * (j0 + k);
        c_to_words((j0 + k < 8 && idx < p.chirp_len) ? __ldg(chirp + idx) : mk(Real(0), Real(0)), &wc[k * WPC]);
      }
      tmem_st8(tbase + j0 * WPC, wh);
      if (j0 < 8) tmem_st8(tbase + 32 + j0 * WPC, wc);
    }
    // P1 / Q4 twiddles of W = W_16384^t: {W, W^2, W^3, W^4, W^8, W^12} (exactly rounded)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t ws[8];
#pragma unroll
      for (int k = 0; k < CPC; ++k) {
        const int i = 4 * h + k;
        const int e = i < 3 ? (i + 1) * t : (i < 6 ? 4 * (i - 2) * t : 0);
        c_to_words(exact_w<C>(e & (L::P - 1), L::P), &ws[k * WPC]);
      }
      tmem_st8(tbase + 48 + 8 * h, ws);
    }
    tmem_wait_st();
  }
  __syncthreads();
  if (staged && t == 0 && u < batch) {
    mbar_expect_tx(stbar, (uint32_t)row_bytes);
    tma_load_1d(stage, static_cast<const unsigned char*>(p.x) + int64_t(u) * p.xs * (row_bytes / p.n),
                (uint32_t)row_bytes, stbar);
  }
  uint32_t phase = 0, xcnt = 0;
  auto ld_tm = [&](int col, C (&out)[CPC]) {
    uint32_t w[8];
    tmem_ld8(tbase + col, w);
#pragma unroll
    for (int k = 0; k < CPC; ++k) out[k] = words_to_c(&w[k * WPC], (C*)nullptr);
  };
  auto tw_p1 = [&](C (&w)[8]) {
    ld_tm(48, reinterpret_cast<C(&)[CPC]>(w[0]));
    ld_tm(56, reinterpret_cast<C(&)[CPC]>(w[4]));
  };
  // P3 / Q2: u[k3] *= W_256^{n'' k3} from the exact shared table (or chains)
  auto tw_p3 = [&](C (&u3)[16]) {
    const C* row = T3 + L::T3S * n16;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      C w0, w1;
      ld_pair(row + 2 * q, w0, w1);
      if (q > 0) u3[2 * q] = cmul(u3[2 * q], w0);
      u3[2 * q + 1] = cmul(u3[2 * q + 1], w1);
    }
  };

  // twiddle tables are prefetched into registers right after an exchange
  // write (the data registers are free then), i.e. inside the barrier shadow
  auto ld_t2 = [&](C (&w)[12]) {  // W_1024^{n' k2}, n' = 2 tau + (g & 1) + 128 (g >> 1), k2 = 1..3
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 1; j < 4; ++j)
        ld_pair(T2 + (j - 1) * 256 + 2 * tau + 128 * h, w[3 * (2 * h) + j - 1], w[3 * (2 * h + 1) + j - 1]);
  };
  auto ld_t3 = [&](C (&w)[15]) {  // W_256^{n'' k3}, k3 = 1..15
#pragma unroll
    for (int r = 1; r < 16; ++r) w[r - 1] = T3[(r - 1) * 16 + n16];
  };
  const bool fast_in = staged && !p.real_in && p.n >= L::P / 2;  // uniform over the CTA
  const bool fast_out = p.m >= L::P / 2;
  C* const rg = xb + gk * L::REG;             // this group's region
  C* const sb = rg + k2 * L::SUB;             // this half-warp's sub-block
#ifdef ASX_CL_TIMELINE
  unsigned long long* const tl = reinterpret_cast<unsigned long long*>(reinterpret_cast<C*>(p.X) + int64_t(p.batch) * p.Xs);
#endif

#pragma unroll 1
  for (int it = 0; it < iters; ++it, u += stride) {
    const bool live = u < batch;
    const int64_t row_off = int64_t(u) * p.xs;
    C v[16];
    CL_TL(0);
    if (staged && live) {
      mbar_wait(stbar, phase);
      phase ^= 1;
    }
    CL_TL(1);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = mk(Real(0), Real(0));
#pragma unroll
    for (int j0 = 0; j0 < 8; j0 += CPC) {
      C cw[CPC];
      ld_tm(32 + j0 * WPC, cw);
      if (fast_in && live) {  // full complex row staged in shared memory: no per-element checks
#pragma unroll
        for (int k = 0; k < CPC; ++k) v[j0 + k] = cmul(reinterpret_cast<const C*>(stage)[t + 1024 * (j0 + k)], cw[k]);
      } else {
#pragma unroll
        for (int k = 0; k < CPC; ++k) {
          const int nn = t + 1024 * (j0 + k);
          if (live && nn < p.n) v[j0 + k] = cmul(load_row<C>(stage, p.x, row_off, nn, p.real_in, staged), cw[k]);
        }
      }
    }
    CL_TL(2);
    // ---- P1: radix-16 DIF over x[t + 1024 i] (upper half zero), twiddle W_16384^{t k1}
    dft_reg<16>(v);
    {
      C w[8];
      tw_p1(w);
      tw16_apply(v, w);
    }
    CL_TL(3);
    // ---- G1: y_k1[t] -> region k1 (WAR: previous signal's Q4 reads)
    if (xcnt) mbar_wait(war, (xcnt - 1) & 1);
    CL_TL(4);
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) xb[k1 * L::REG + L::pos(t)] = v[k1];
    C tw2[12];
    ld_t2(tw2);
    CL_TL(5);
    __syncthreads();  // G1 RAW; also: every thread has consumed the staged row
    CL_TL(6);
    if (staged && t == 0 && u + stride < batch) {
      fence_proxy_async();
      mbar_expect_tx(stbar, (uint32_t)row_bytes);
      tma_load_1d(stage, static_cast<const unsigned char*>(p.x) + int64_t(u + stride) * p.xs * (row_bytes / p.n),
                  (uint32_t)row_bytes, stbar);
    }
    // ---- P2: radix-4 DIF over y_k[n' + 256 i'], n' = 2 tau + (g & 1) + 128 (g >> 1); twiddle W_1024^{n' k2}
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < 4; ++i) ld_pair(rg + 2 * tau + 128 * h + L::SUB * i, v[4 * (2 * h) + i], v[4 * (2 * h + 1) + i]);
    CL_TL(7);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      dft_reg<4>(reinterpret_cast<C(&)[4]>(v[4 * g]));
#pragma unroll
      for (int j = 1; j < 4; ++j) v[4 * g + j] = cmul(v[4 * g + j], tw2[3 * g + j - 1]);
    }
    // no WAR barrier: each thread overwrites exactly the slots it read
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < 4; ++j) st_pair(rg + j * L::SUB + 2 * tau + 128 * h, v[4 * (2 * h) + j], v[4 * (2 * h + 1) + j]);
    CL_TL(8);
    group_bar(gbar);  // RAW
    CL_TL(9);
    // ---- P3: radix-16 DIF over z_{k,k2}[n'' + 16 i'']; twiddle W_256^{n'' k3}
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = sb[n16 + 16 * i];
    CL_TL(10);
    dft_reg<16>(v);
    tw_p3(v);
    CL_TL(11);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) sb[L::L2S * j + n16] = v[j];
    __syncwarp();
    // ---- P4: radix-16 DIF over n'' (no twiddle) -> Y[f], f = gk + 16 k2 + 64 n16 + 1024 k4
    {
      const float4* row = reinterpret_cast<const float4*>(sb + L::L2S * n16);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 w = row[q];
        v[2 * q] = mk(Real(w.x), Real(w.y));
        v[2 * q + 1] = mk(Real(w.z), Real(w.w));
      }
    }
    CL_TL(12);
    dft_reg<16>(v);
#pragma unroll
    for (int j0 = 0; j0 < 16; j0 += CPC) {
      C hw[CPC];
      ld_tm(j0 * WPC, hw);
#pragma unroll
      for (int k = 0; k < CPC; ++k) v[j0 + k] = cconj(cmul(v[j0 + k], hw[k]));
    }
    // ---- inverse = conj(DFT(conj(.))), DFT as the transposed passes Q1..Q4
    CL_TL(13);
    dft_reg<16>(v);  // Q1 = P4^T
    CL_TL(14);
    __syncwarp();
    {
      float4* row = reinterpret_cast<float4*>(sb + L::L2S * n16);
#pragma unroll
      for (int q = 0; q < 8; ++q) row[q] = make_float4(v[2 * q].x, v[2 * q].y, v[2 * q + 1].x, v[2 * q + 1].y);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = sb[L::L2S * j + n16];
    CL_TL(15);
    tw_p3(v);  // Q2 = P3^T
    dft_reg<16>(v);
    CL_TL(16);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 16; ++i) sb[n16 + 16 * i] = v[i];
    ld_t2(tw2);
    CL_TL(17);
    group_bar(gbar);  // RAW
    CL_TL(18);
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < 4; ++j) ld_pair(rg + j * L::SUB + 2 * tau + 128 * h, v[4 * (2 * h) + j], v[4 * (2 * h + 1) + j]);
    CL_TL(19);
#pragma unroll
    for (int g = 0; g < 4; ++g) {  // Q3 = P2^T
#pragma unroll
      for (int j = 1; j < 4; ++j) v[4 * g + j] = cmul(v[4 * g + j], tw2[3 * g + j - 1]);
      dft_reg<4>(reinterpret_cast<C(&)[4]>(v[4 * g]));
    }
    // no WAR barrier: each thread overwrites exactly the slots it read
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < 4; ++i) st_pair(rg + 2 * tau + 128 * h + L::SUB * i, v[4 * (2 * h) + i], v[4 * (2 * h + 1) + i]);
    C tw1[8];
    tw_p1(tw1);
    CL_TL(20);
    __syncthreads();
    CL_TL(21);
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) v[k1] = xb[k1 * L::REG + L::pos(t)];
    __syncwarp();
    CL_TL(22);
    if ((t & 31) == 0) mbar_arrive(war);
    ++xcnt;
    tw16_apply(v, tw1);
    dft_reg<16>(v);
    CL_TL(23);
    {
      C* X = reinterpret_cast<C*>(p.X) + int64_t(u) * p.Xs;
#pragma unroll
      for (int j0 = 0; j0 < 8; j0 += CPC) {
        C cw[CPC];
        ld_tm(32 + j0 * WPC, cw);
        if (fast_out && live) {
#pragma unroll
          for (int k = 0; k < CPC; ++k) X[t + 1024 * (j0 + k)] = cmul(cconj(v[j0 + k]), cw[k]);
        } else {
#pragma unroll
          for (int k = 0; k < CPC; ++k) {
            const int mm = t + 1024 * (j0 + k);
            if (live && mm < p.m) X[mm] = cmul(cconj(v[j0 + k]), cw[k]);
          }
        }
      }
    }
    CL_TL(24);
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(tmem_slot, 512);
}

}  // namespace asx

// asx_chirp_r32.cuh — chirp-z α-DFT for P = 16384 (complex64, N, M <= 8192)
// at 32 values per thread: the config-4 hot kernel (BASELINE config 4:
// N = M = 8192, α = 1/8).
//
// Same mathematics as k_chirp_local (the α-DFT as the chirp-z convolution
// X_m = c_m Σ_n (x_n c_n) conj(c_{m-n}), fastpath.py:162-181 / oracle.py:50-67
// restated) and the same forward-DIF / transposed-inverse scheme, but
// factored P = 32 · 16 · 32 over 512 threads x 32 values (128 registers)
// instead of 16 · 4 · 16 · 16 over 1024 threads x 16 values: three passes per
// transform, so a signal crosses shared memory 4 times instead of 6 (one
// CTA-wide and one warp-local exchange per transform).  k_chirp_local is
// co-limited by the shared-memory data pipe (80 % busy: its 6 exchanges are
// 12.3 k of 16.9 k wavefronts per signal) and by issue (73 %); this kernel
// moves 10.2 k wavefronts per signal with the same arithmetic.
//
//   P1  radix-32 DIF over a[t + 512 i] (i >= 16 zero: the first level is
//       16 constant twiddles, then two radix-16), × W_16384^{t k1}
//   G1  CTA-wide exchange: sub-problems 2j, 2j + 1 (512 points each) -> warp j
//   P2  per sub-problem: radix-16 DIF over y[lane + 32 i'], × W_512^{lane k2}
//   L1  32 x 32 transpose inside the warp: problem q = 16 s + k2 -> lane q
//   P3  radix-32 (no twiddle) -> Y[f], f = k1 + 32 k2 + 512 f''; × H[f]; conj
//   Q1 .. Q3 = P3ᵀ, P2ᵀ, P1ᵀ on the same thread <-> data map (twiddle, then
//   butterfly, then the inverse exchange), ending in the io layout
//   X[t + 512 i], i < 16 (the last level of P1ᵀ keeps only those).
//
// Tensor memory per thread: H in this thread's spectrum order (64 columns),
// the chirp (32), the exact P1 twiddles W and W^2, W^4 .. W^30 (32); the odd
// powers W^{2j+1} are one compensated product of two exact values.
#pragma once

#include "asx_chirp_local.cuh"

#ifndef ASX_R32_ACCMODE
#define ASX_R32_ACCMODE 2  // tw_const ACC mode of the selected passes (1 all constants, 2 two-constant twiddles only)
#endif
#ifndef ASX_R32_ACC
#define ASX_R32_ACC 2  // butterfly constants with their rounding residual: bit 0 radix-32 passes, 1 first / last level of P1 / Q3, 2 radix-16 passes
#endif

#ifndef ASX_R32_PLAINTW
#define ASX_R32_PLAINTW 1  // P1 / Q3 odd-power twiddles W^{2j} W as plain FP32 products (0: compensated products, +2.8 % time, 1.63e-5 instead of 1.69e-5 on config 4)
#endif

#ifndef ASX_R32_DIT
#define ASX_R32_DIT 2  // in-register DFTs in the FMA-fused decimation-in-time form: 1 exact differences, 2 differences as 2a - sum
#endif

namespace asx {

#if ASX_R32_DIT
#define R32_DFT16(x) dft_reg_dit<16, ASX_R32_DIT == 2>(x)
#define R32_DFT32(x) dft_reg_dit<32, ASX_R32_DIT == 2>(x)
#else
#define R32_DFT16(x) dft_reg<16, ((ASX_R32_ACC >> 2) & 1) * ASX_R32_ACCMODE>(x)
#define R32_DFT32(x) dft_reg<32, (ASX_R32_ACC & 1) * ASX_R32_ACCMODE>(x)
#endif

#if ASX_R32_PLAINTW
#define R32_TWMUL cmul
#else
#define R32_TWMUL cmul_acc
#endif

struct ChirpR32 {
  static constexpr int P = 16384, NT = 512;
  static constexpr int RS = 34;          // L1 row stride: 16-byte aligned rows, conflict-free both ways
  static constexpr int REGW = 32 * RS;   // one warp's region: two 512-point sub-problems / the 32 x 32 transpose
  static constexpr int XB = 16 * REGW;   // exchange buffer (complex64 elements)
  static constexpr int T5N = 16 * 32;    // W_512^{lane k2}, [k2][lane]
  static constexpr int CPT = 128;        // TMEM columns per thread: H 64 | chirp 32 | P1 twiddles 32
  __host__ __device__ static size_t stage_off() { return align_up(size_t(XB) * sizeof(float2), 128); }
  __host__ __device__ static size_t tab_off(size_t row_bytes, bool staged) {
    return stage_off() + (staged ? align_up(row_bytes, 128) : 0);
  }
  __host__ __device__ static size_t bar_off(size_t row_bytes, bool staged) {
    return align_up(tab_off(row_bytes, staged) + size_t(T5N) * sizeof(float2), 16);
  }
  __host__ __device__ static size_t total(size_t row_bytes, bool staged) {
    return bar_off(row_bytes, staged) + 2 * sizeof(uint64_t) + 16;  // stage mbar, WAR mbar, TMEM slot
  }
};

template <typename Real>
__global__ void __launch_bounds__(512, 1) k_chirp_r32(KParams p) {
  static_assert(sizeof(Real) == 4, "complex64 kernel");
  using C = float2;
  using L = ChirpR32;
  extern __shared__ __align__(128) unsigned char smraw[];
  C* const xb = reinterpret_cast<C*>(smraw);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const bool staged = p.staged != 0;
  const size_t row_bytes = size_t(p.n) * (p.real_in ? sizeof(Real) : sizeof(C));
  unsigned char* const stage = smraw + L::stage_off();
  C* const T5 = reinterpret_cast<C*>(smraw + L::tab_off(row_bytes, staged));
  uint64_t* const stbar = reinterpret_cast<uint64_t*>(smraw + L::bar_off(row_bytes, staged));
  uint64_t* const war = stbar + 1;
  uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(stbar + 2);

  for (int e = t; e < L::T5N; e += L::NT) T5[e] = exact_w<C>((e & 31) * (e >> 5), 512);
  const int stride = int(gridDim.x);
  int u = int(blockIdx.x);
  const int batch = int(p.batch);
  const int iters = (batch + stride - 1) / stride;
  if (t == 0) {
    mbar_init(stbar, 1);
    mbar_init(war, L::NT / 32);
    fence_mbar_init();
    if (staged && u < batch) {
      mbar_expect_tx(stbar, (uint32_t)row_bytes);
      tma_load_1d(stage, static_cast<const unsigned char*>(p.x) + int64_t(u) * p.xs * (row_bytes / p.n),
                  (uint32_t)row_bytes, stbar);
    }
  }
  const C* chirp = reinterpret_cast<const C*>(p.chirp);
  const C* H = reinterpret_cast<const C*>(p.H);
  if (warp == 0) tmem_alloc(&tmem_slot, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = tmem_slot + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * L::CPT);
  {
    // H in this thread's spectrum order f = k1 + 32 k2 + 512 f'' (k1 = 2 warp + (lane >> 4), k2 = lane & 15)
    const int fbase = 2 * warp + (lane >> 4) + 32 * (lane & 15);
#pragma unroll
    for (int f0 = 0; f0 < 32; f0 += 4) {
      uint32_t w8[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) c_to_words(__ldg(H + fbase + 512 * (f0 + k)), &w8[2 * k]);
      tmem_st8(tbase + 2 * f0, w8);
    }
    // chirp[t + 512 i], i < 16 (input and output rows share the io layout)
#pragma unroll
    for (int i0 = 0; i0 < 16; i0 += 4) {
      uint32_t w8[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int idx = t + 512 * (i0 + k);
        c_to_words(idx < p.chirp_len ? __ldg(chirp + idx) : mk(0.0f, 0.0f), &w8[2 * k]);
      }
      tmem_st8(tbase + 64 + 2 * i0, w8);
    }
    // exact W^e, W = W_16384^t, e = 1, 2, 4, 6, .., 30 (slot 0: W; slot j: W^{2j})
#pragma unroll
    for (int q0 = 0; q0 < 16; q0 += 4) {
      uint32_t w8[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int q = q0 + k;
        const int e = q == 0 ? 1 : 2 * q;
        c_to_words(exact_w<C>((e * t) & (L::P - 1), L::P), &w8[2 * k]);
      }
      tmem_st8(tbase + 96 + 2 * q0, w8);
    }
    tmem_wait_st();
  }
  __syncthreads();

  auto ld_tm = [&](uint32_t col, C (&out)[4]) {
    uint32_t wd[8];
    tmem_ld8(tbase + col, wd);
#pragma unroll
    for (int k = 0; k < 4; ++k) out[k] = words_to_c(&wd[2 * k], (C*)nullptr);
  };
  // P1 / Q3: element k1 (lo[j] = 2j, hi[j] = 2j + 1) *= W^{k1}: the even powers are exact
  // (tensor memory), the odd ones W^{2j} W one product of two exact values
  auto tw_p1 = [&](C (&v)[32]) {
    C s[4];
    ld_tm(96, s);  // W, W^2, W^4, W^6
    const C w1 = s[0];
    v[16] = cmul(v[16], w1);
#pragma unroll
    for (int j = 1; j < 4; ++j) {
      v[j] = cmul(v[j], s[j]);
      v[16 + j] = cmul(v[16 + j], R32_TWMUL(s[j], w1));
    }
#pragma unroll
    for (int j0 = 4; j0 < 16; j0 += 4) {
      ld_tm(96 + 2 * j0, s);  // W^{2 j0} .. W^{2 j0 + 6}
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[j0 + k] = cmul(v[j0 + k], s[k]);
        v[16 + j0 + k] = cmul(v[16 + j0 + k], R32_TWMUL(s[k], w1));
      }
    }
  };
  // P2 / Q2 twiddles W_512^{lane k2}, k2 = 1 .. 15 (the same for both sub-problems)
  auto tw_p2 = [&](C (&v)[32]) {
#pragma unroll
    for (int k2 = 1; k2 < 16; ++k2) {
      const C w = T5[32 * k2 + lane];
      v[k2] = cmul(v[k2], w);
      v[16 + k2] = cmul(v[16 + k2], w);
    }
  };
  const bool fast_in = staged && !p.real_in && p.n >= L::P / 2;  // uniform over the CTA
  const bool fast_out = p.m >= L::P / 2;
  C* const rgw = xb + warp * L::REGW;  // this warp's region
  uint32_t phase = 0, xcnt = 0;

#pragma unroll 1
  for (int it = 0; it < iters; ++it, u += stride) {
    const bool live = u < batch;
    const int64_t row_off = int64_t(u) * p.xs;
    C v[32];  // lo = v[0..15], hi = v[16..31]
    if (staged && live) {
      mbar_wait(stbar, phase);
      phase ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = mk(0.0f, 0.0f);
#pragma unroll
    for (int i0 = 0; i0 < 16; i0 += 4) {
      C cw[4];
      ld_tm(64 + 2 * i0, cw);
      if (fast_in && live) {  // full complex row staged in shared memory: no per-element checks
#pragma unroll
        for (int k = 0; k < 4; ++k) v[i0 + k] = cmul(reinterpret_cast<const C*>(stage)[t + 512 * (i0 + k)], cw[k]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int nn = t + 512 * (i0 + k);
          if (live && nn < p.n) v[i0 + k] = cmul(load_row<C>(stage, p.x, row_off, nn, p.real_in, staged), cw[k]);
        }
      }
    }
    // ---- P1: radix-32 DIF over i with a[t + 512 i] = 0 for i >= 16: first level (a, a W_32^i), two radix-16
#pragma unroll
    for (int i = 0; i < 16; ++i) v[16 + i] = tw_const<32, ((ASX_R32_ACC >> 1) & 1) * ASX_R32_ACCMODE>(v[i], i);
    R32_DFT16(reinterpret_cast<C(&)[16]>(v[0]));
    R32_DFT16(reinterpret_cast<C(&)[16]>(v[16]));
    // WAR on the exchange buffer (the previous signal's Q3 reads, long done by now); waited for here so
    // that the stores below can be scheduled into the twiddle products
    if (xcnt) mbar_wait(war, (xcnt - 1) & 1);
    tw_p1(v);
    // ---- G1: sub-problems 2j (lo[j]) and 2j + 1 (hi[j]) -> warp j's region
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      xb[j * L::REGW + t] = v[j];
      xb[j * L::REGW + 512 + t] = v[16 + j];
    }
    __syncthreads();  // G1 RAW; every thread has consumed the staged row
    if (staged && t == 0 && u + stride < batch) {
      fence_proxy_async();
      mbar_expect_tx(stbar, (uint32_t)row_bytes);
      tma_load_1d(stage, static_cast<const unsigned char*>(p.x) + int64_t(u + stride) * p.xs * (row_bytes / p.n),
                  (uint32_t)row_bytes, stbar);
    }
    // ---- P2: per sub-problem s, radix-16 DIF over y[lane + 32 i'], × W_512^{lane k2}
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] = rgw[lane + 32 * i];
      v[16 + i] = rgw[512 + lane + 32 * i];
    }
    R32_DFT16(reinterpret_cast<C(&)[16]>(v[0]));
    R32_DFT16(reinterpret_cast<C(&)[16]>(v[16]));
    tw_p2(v);
    __syncwarp();
    // ---- L1 (warp): problem q = 16 s + k2, point lane -> lane q
#pragma unroll
    for (int q = 0; q < 32; ++q) rgw[L::RS * q + lane] = v[q];
    __syncwarp();
    {
      const float4* row = reinterpret_cast<const float4*>(rgw + L::RS * lane);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float4 f = row[q];
        v[2 * q] = mk(f.x, f.y);
        v[2 * q + 1] = mk(f.z, f.w);
      }
    }
    // ---- P3: radix-32 over the lane index -> Y[f]; × H[f]; conj
    R32_DFT32(v);
#pragma unroll
    for (int f0 = 0; f0 < 32; f0 += 4) {
      C hw[4];
      ld_tm(2 * f0, hw);
#pragma unroll
      for (int k = 0; k < 4; ++k) v[f0 + k] = cconj(cmul(v[f0 + k], hw[k]));
    }
    // ---- inverse = conj(DFT(conj(.))): Q1 = P3ᵀ
    R32_DFT32(v);
    __syncwarp();
    {
      float4* row = reinterpret_cast<float4*>(rgw + L::RS * lane);  // L1ᵀ: the slots this thread read
#pragma unroll
      for (int q = 0; q < 16; ++q) row[q] = make_float4(v[2 * q].x, v[2 * q].y, v[2 * q + 1].x, v[2 * q + 1].y);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = rgw[L::RS * q + lane];
    // ---- Q2 = P2ᵀ
    tw_p2(v);
    R32_DFT16(reinterpret_cast<C(&)[16]>(v[0]));
    R32_DFT16(reinterpret_cast<C(&)[16]>(v[16]));
    __syncwarp();  // every lane has read the transpose before the sub-problems are written back
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      rgw[lane + 32 * i] = v[i];
      rgw[512 + lane + 32 * i] = v[16 + i];
    }
    __syncthreads();  // G1ᵀ RAW
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j] = xb[j * L::REGW + t];
      v[16 + j] = xb[j * L::REGW + 512 + t];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(war);
    ++xcnt;
    // ---- Q3 = P1ᵀ: × W^{k1}, two radix-16, last level X_i = E_i + W_32^i O_i kept for i < 16
    tw_p1(v);
    R32_DFT16(reinterpret_cast<C(&)[16]>(v[0]));
    R32_DFT16(reinterpret_cast<C(&)[16]>(v[16]));
    {
      C* X = reinterpret_cast<C*>(p.X) + int64_t(u) * p.Xs;
#pragma unroll
      for (int i0 = 0; i0 < 16; i0 += 4) {
        C cw[4];
        ld_tm(64 + 2 * i0, cw);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = i0 + k, mm = t + 512 * i;
          const C y = cadd(v[i], tw_const<32, ((ASX_R32_ACC >> 1) & 1) * ASX_R32_ACCMODE>(v[16 + i], i));
          if (live && (fast_out || mm < p.m)) X[mm] = cmul(cconj(y), cw[k]);
        }
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(tmem_slot, 512);
}

}  // namespace asx

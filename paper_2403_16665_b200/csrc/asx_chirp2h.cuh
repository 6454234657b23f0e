// asx_chirp2h.cuh — chirp-z α-DFT with the P-point cyclic convolution split
// into even/odd halves, so two independent CTAs fit on one SM.
//
// With P = 2Q >= 2N (the plan guarantees the zero padding) and M <= Q:
//   FFT_P(y)[2k]   = FFT_Q(y)[k]                 (y[k+Q] = 0)
//   FFT_P(y)[2k+1] = FFT_Q(y[k] W_P^k)[k]
//   G = FFT_P(conj(Y H/P)):  G[n] = E'[n] + W_P^n O'[n],  n < Q,
//     E' = FFT_Q(conj(Y_even H_even/P)),  O' = FFT_Q(conj(Y_odd H_odd/P))
//   X[m] = conj(G[m]) chirp[m] = conj(E'[m]) chirp[m] + conj(O'[m]) chirpWc[m],
//     chirpWc[m] = conj(W_P^m) chirp[m],  chirpW[k] = W_P^k chirp[k]  (plan tables).
// Per signal: four Q-point FFTs (the same op count as two P-point ones), the
// even half's result E' parked in a per-CTA L2 scratch row between the
// halves (written and re-read by the same thread: no synchronisation).
// Resources per CTA: Q registers-worth of data, one Q-point exchange buffer,
// half the SM's TMEM (H_even/H_odd of this thread) — two CTAs per SM, whose
// FP, shared-memory and latency phases interleave freely.
#pragma once

#include "asx_kernels.cuh"

namespace asx {

#ifndef ASX_C2H_TAB
#define ASX_C2H_TAB 64  // the two-halves kernel serves passes with Ns <= 64 from shared tables
#endif

template <typename Real, int Q, int NT>
struct Chirp2hCfg {
  using E = Fft<Real, Q, NT, ASX_C2H_TAB>;
  using C = typename CT<Real>::T;
  static constexpr int R = E::R;
  static constexpr int WPC = sizeof(C) / 4;
  static constexpr int CPT = 2 * R * WPC;  // TMEM columns per thread: H_even, H_odd
  static constexpr int NEED = (NT / 128) * CPT;
  static constexpr int NCOLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr int CPC = 8 / WPC;  // complex per 8-column TMEM access
  static constexpr size_t SMEM = align_up((size_t(E::SMEM_ELEMS) + E::TAB_ELEMS) * sizeof(C), 16) + 32;
};

template <typename Real, int Q, int NT>
__global__ void __launch_bounds__(NT, 2) k_chirp2h(KParams p, void* scratch_base, const void* chirpW,
                                                   const void* chirpWc) {
  using G = Chirp2hCfg<Real, Q, NT>;
  using E = typename G::E;
  using C = typename CT<Real>::T;
  constexpr int R = G::R;
  static_assert(NT % 128 == 0 && G::NEED <= 256, "two CTAs per SM must share TMEM");
  extern __shared__ __align__(128) unsigned char smraw[];
  C* fbuf = reinterpret_cast<C*>(smraw);
  C* tab = fbuf + E::SMEM_ELEMS;
  uint64_t* war = reinterpret_cast<uint64_t*>(smraw + G::SMEM - 32);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smraw + G::SMEM - 16);
  const int t = threadIdx.x;
  const int warp = t >> 5;

  const typename E::TwRegs tr = E::make_tw(t, reinterpret_cast<const C*>(p.twP), tab, t, NT);
  typename E::XSync xs;
  E::xs_init(xs, war, NT);
  if (warp == 0) tmem_alloc(tmem_slot, G::NCOLS);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *tmem_slot + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * G::CPT);
  const C* H = reinterpret_cast<const C*>(p.H);
  // TMEM: H_even[j] = H[2(t + NT j)] at columns [0, R*WPC), H_odd after it
#pragma unroll
  for (int j0 = 0; j0 < R; j0 += G::CPC) {
    uint32_t we[8], wo[8];
#pragma unroll
    for (int k = 0; k < G::CPC; ++k) {
      const int idx = 2 * (t + NT * (j0 + k));
      c_to_words(__ldg(H + idx), &we[k * G::WPC]);
      c_to_words(__ldg(H + idx + 1), &wo[k * G::WPC]);
    }
    tmem_st8(tbase + j0 * G::WPC, we);
    tmem_st8(tbase + (R + j0) * G::WPC, wo);
  }
  tmem_wait_st();

  const C* chirp = reinterpret_cast<const C*>(p.chirp);
  const C* cw = reinterpret_cast<const C*>(chirpW);
  const C* cwc = reinterpret_cast<const C*>(chirpWc);
  C* scratch = reinterpret_cast<C*>(scratch_base) + size_t(blockIdx.x) * Q;
  const int batch = int(p.batch);

#pragma unroll 1
  for (int u = blockIdx.x; u < batch; u += gridDim.x) {
    const int64_t row_off = int64_t(u) * p.xs;
    C v[R];
    // four Q-point transforms per signal, one FFT body: stage s -> half s/2,
    // forward (s even) or inverse (s odd) transform of that half
#pragma unroll 1
    for (int s = 0; s < 4; ++s) {
      const int half = s >> 1;
      if ((s & 1) == 0) {
        const C* tabin = half == 0 ? chirp : cw;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int k = t + NT * j;
          C val = mk(Real(0), Real(0));
          if (k < p.n) val = cmul(load_in<C>(p.x, row_off + k, p.real_in), __ldg(tabin + k));
          v[j] = val;
          if ((j & 3) == 3) reg_fence();
        }
      }
      E::run(v, fbuf, t, tr, xs);
      if ((s & 1) == 0) {
#pragma unroll
        for (int j0 = 0; j0 < R; j0 += G::CPC) {
          uint32_t w[8];
          tmem_ld8(tbase + (half * R + j0) * G::WPC, w);
#pragma unroll
          for (int k = 0; k < G::CPC; ++k)
            v[j0 + k] = cconj(cmul(v[j0 + k], words_to_c(&w[k * G::WPC], (C*)nullptr)));
        }
      } else if (half == 0) {
#pragma unroll
        for (int j = 0; j < R; ++j) scratch[t + NT * j] = v[j];  // E' (this thread's own slots)
      } else {
        C* X = reinterpret_cast<C*>(p.X) + int64_t(u) * p.Xs;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int m = t + NT * j;
          if (m < p.m) {
            const C e = scratch[m];
            X[m] = cadd(cmul(cconj(e), __ldg(chirp + m)), cmul(cconj(v[j]), __ldg(cwc + m)));
          }
          if ((j & 1) == 1) reg_fence();
        }
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(*tmem_slot, G::NCOLS);
}

// chirpW[k] = W_P^k chirp[k] (k < n), chirpWc[k] = conj(W_P^k) chirp[k] (k < m),
// evaluated in FP64 from the exactly reduced phases.
static __global__ void k_fill_chirp_tw(void* cw, void* cwc, int64_t n, int64_t m, uint64_t a, uint64_t L2, uint64_t P,
                                int dbl) {
  const int64_t cnt = n > m ? n : m;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < cnt; k += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t kk = mulmod((uint64_t)k, (uint64_t)k, L2);
    const uint64_t j = mulmod(kk, a, L2);
    double s1, c1, s2, c2;
    sincospi(2.0 * (double)j / (double)L2, &s1, &c1);          // chirp = (c1, -s1)
    sincospi(2.0 * (double)(k % P) / (double)P, &s2, &c2);      // W_P^k = (c2, -s2)
    // chirp * W = (c1 c2 - s1 s2, -(s1 c2 + c1 s2)) ; chirp * conj(W) = (c1 c2 + s1 s2, c1 s2 - s1 c2)
    if (k < n) store_c(cw, k, c1 * c2 - s1 * s2, -(s1 * c2 + c1 * s2), dbl);
    if (k < m) store_c(cwc, k, c1 * c2 + s1 * s2, c1 * s2 - s1 * c2, dbl);
  }
}

}  // namespace asx

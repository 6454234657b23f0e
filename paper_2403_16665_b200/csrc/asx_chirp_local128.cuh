// asx_chirp_local128.cuh — chirp-z α-DFT for P = 8192 complex128 with
// group-local exchanges (BASELINE config 1b: N = M = 4096, α = 1/10, and any
// complex128 chirp plan with 2N, 2M <= 8192).
//
// The same mathematics and the same forward-DIF / transposed-inverse scheme
// as k_chirp_local (asx_chirp_local.cuh), re-factored for
// 16-byte elements at 512 threads x 16 values (one signal per SM):
//
//   P1  radix-16 DIF over y[t + 512 i] (upper half zero), × W_8192^{t k1}
//   G1  CTA-wide exchange: sub-problem k1 (512 points) -> warp k1
//   P2  8 radix-2 DIF butterflies per thread over (n', n' + 256),
//       × W_512^{n'} on the odd half                -> two 256-point halves
//   L1  exchange inside the warp (every thread rewrites the slots it read)
//   P3  radix-16 DIF over n'' = l + 16 i'' in the half-warp, × W_256^{l k3}
//   L2  exchange inside the half-warp (padded 17)
//   P4  radix-16 -> Y[f], f = k1 + 16 k2 + 32 k3 + 512 k4;  × H[f]; conj
//   Q1..Q4 = P4ᵀ..P1ᵀ on the same thread <-> data map, ending in the io layout
//
// Per signal: 2 CTA-wide exchanges (the Stockham engine needs 6 at P = 8192,
// R = 16: passes 2 x 16 x 16 x 16), 4 warp-local ones.  Tensor memory holds
// per thread H (16 values in this thread's spectrum order), the chirp
// (8 values) and the exact P1 / P2 twiddle seeds: 124 of 128 columns.
#pragma once

#include "asx_chirp_local.cuh"
#include "asx_large.cuh"

#ifndef ASX_CL128_SHFL
#define ASX_CL128_SHFL 1  // L1 / L1ᵀ as lane-pair shuffles instead of a shared-memory round trip
#endif

namespace asx {

struct ChirpLocal128 {
  static constexpr int P = 8192, NT = 512;
  static constexpr int SUBR = 272;        // one 256-point half (+16 pad: the L2 layout l + 17 k3 fits)
  static constexpr int REG = 2 * SUBR;    // one 512-point sub-problem (warp region)
  static constexpr int XB = 16 * REG;     // exchange buffer (complex128 elements)
  static constexpr int T3S = 17;          // T3 row stride: conflict-free 16 B reads
  static constexpr int T3N = 16 * T3S;    // W_256^{l k3}, row l, column k3
  static constexpr int CPT = 128;         // TMEM columns per thread: H 64 | chirp 32 | P1 seeds 24 | W_512^j 4
  __host__ __device__ static constexpr int pos(int n) { return n + (n >> 8) * (SUBR - 256); }  // n < 512
  __host__ __device__ static size_t stage_off() { return align_up(size_t(XB) * sizeof(double2), 128); }
  __host__ __device__ static size_t tab_off(size_t row_bytes, bool staged) {
    return stage_off() + (staged ? align_up(row_bytes, 128) : 0);
  }
  __host__ __device__ static size_t bar_off(size_t row_bytes, bool staged) {
    return align_up(tab_off(row_bytes, staged) + size_t(T3N) * sizeof(double2), 16);
  }
  __host__ __device__ static size_t total(size_t row_bytes, bool staged) {
    return bar_off(row_bytes, staged) + 2 * sizeof(uint64_t) + 16;  // stage mbar, WAR mbar, TMEM slot
  }
};

// 4 consecutive complex128 values (16 TMEM columns) of this thread's lane
__device__ __forceinline__ void tm_ld4c(uint32_t taddr, double2 (&out)[4]) {
  uint32_t w[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
        "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int k = 0; k < 4; ++k) out[k] = words_to_c(&w[4 * k], (double2*)nullptr);
}

template <typename Real>
__global__ void __launch_bounds__(512, 1) k_chirp_local128(KParams p) {
  static_assert(sizeof(Real) == 8, "complex128 kernel");
  using C = double2;
  using L = ChirpLocal128;
  extern __shared__ __align__(128) unsigned char smraw[];
  C* xb = reinterpret_cast<C*>(smraw);
  const int t = threadIdx.x, warp = t >> 5, j = t & 31, h = j >> 4, l = j & 15;
  const bool staged = p.staged != 0;
  const size_t row_bytes = size_t(p.n) * (p.real_in ? sizeof(Real) : sizeof(C));
  unsigned char* stage = smraw + L::stage_off();
  C* T3 = reinterpret_cast<C*>(smraw + L::tab_off(row_bytes, staged));
  uint64_t* stbar = reinterpret_cast<uint64_t*>(smraw + L::bar_off(row_bytes, staged));
  uint64_t* war = stbar + 1;
  uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(stbar + 2);

  for (int e = t; e < L::T3N; e += L::NT) {
    const int row = e / L::T3S, col = e % L::T3S;  // l, k3
    T3[e] = exact_w<C>(col < 16 ? row * col : 0, 256);
  }
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
    // H in this thread's spectrum order f = k1 + 16 k2 + 32 k3 + 512 k4 (k1 = warp, k2 = h, k3 = l)
    const int fbase = warp + 16 * h + 32 * l;
#pragma unroll
    for (int k0 = 0; k0 < 16; k0 += 2) {
      uint32_t w8[8];
      c_to_words(__ldg(H + fbase + 512 * k0), &w8[0]);
      c_to_words(__ldg(H + fbase + 512 * (k0 + 1)), &w8[4]);
      tmem_st8(tbase + 4 * k0, w8);
    }
    // chirp[t + 512 i], i < 8 (input and output rows share the io layout)
#pragma unroll
    for (int i0 = 0; i0 < 8; i0 += 2) {
      uint32_t w8[8];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int idx = t + 512 * (i0 + k);
        c_to_words(idx < p.chirp_len ? __ldg(chirp + idx) : mk(0.0, 0.0), &w8[4 * k]);
      }
      tmem_st8(tbase + 64 + 4 * i0, w8);
    }
    // exact W_8192^{e t} for e = 1, 2, 3, 4, 8, 12 and W_512^j
    const int es[8] = {1, 2, 3, 4, 8, 12, 0, 0};
#pragma unroll
    for (int q0 = 0; q0 < 8; q0 += 2) {
      uint32_t w8[8];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int q = q0 + k;
        const C w = q < 6 ? exact_w<C>((es[q] * t) & (L::P - 1), L::P) : (q == 6 ? exact_w<C>(j, 512) : mk(1.0, 0.0));
        c_to_words(w, &w8[4 * k]);
      }
      tmem_st8(tbase + 96 + 4 * q0, w8);
    }
    tmem_wait_st();
  }
  __syncthreads();

  // P1 / Q4: u[r] *= W^{t r} from exact W, W^2, W^3 and seeds W^4, W^8, W^12
  auto tw_p1 = [&](C (&v)[16]) {
    C w[8];
    tm_ld4c(tbase + 96, reinterpret_cast<C(&)[4]>(w[0]));
    tm_ld4c(tbase + 112, reinterpret_cast<C(&)[4]>(w[4]));
    v[1] = cmul(v[1], w[0]);
    v[2] = cmul(v[2], w[1]);
    v[3] = cmul(v[3], w[2]);
#pragma unroll
    for (int a = 1; a < 4; ++a) {
      const C w4a = w[2 + a];
      v[4 * a] = cmul(v[4 * a], w4a);
      v[4 * a + 1] = cmul(v[4 * a + 1], cmul(w4a, w[0]));
      v[4 * a + 2] = cmul(v[4 * a + 2], cmul(w4a, w[1]));
      v[4 * a + 3] = cmul(v[4 * a + 3], cmul(w4a, w[2]));
    }
  };
  // P2 / Q3 twiddle of pair q: W_512^{j + 32 q} = W_512^j W_16^q
  auto w512 = [&]() {
    C w[4];
    tm_ld4c(tbase + 112, w);
    return w[2];
  };
  // P3 / Q2: v[k3] *= W_256^{l k3}
  auto tw_p3 = [&](C (&v)[16]) {
    const C* row = T3 + L::T3S * l;
#pragma unroll
    for (int k3 = 1; k3 < 16; ++k3) v[k3] = cmul(v[k3], row[k3]);
  };
  const bool fast_in = staged && !p.real_in && p.n >= L::P / 2;
  const bool fast_out = p.m >= L::P / 2;
  C* const rg = xb + warp * L::REG;  // this warp's sub-problem region
  C* const sr = rg + h * L::SUBR;    // this half-warp's 256-point half
  uint32_t phase = 0, xcnt = 0;

#pragma unroll 1
  for (int it = 0; it < iters; ++it, u += stride) {
    const bool live = u < batch;
    const int64_t row_off = int64_t(u) * p.xs;
    C v[16];
    if (staged && live) {
      mbar_wait(stbar, phase);
      phase ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = mk(0.0, 0.0);
#pragma unroll
    for (int i0 = 0; i0 < 8; i0 += 4) {
      C cw[4];
      tm_ld4c(tbase + 64 + 4 * i0, cw);
      if (fast_in && live) {
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
    // ---- P1: radix-16 DIF (upper half zero), × W_8192^{t k1}
    ASX_DFT16_F64(v);
    tw_p1(v);
    // ---- G1: y_k1[t] -> region k1 (WAR: the previous signal's Q4 reads)
    if (xcnt) mbar_wait(war, (xcnt - 1) & 1);
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) xb[k1 * L::REG + L::pos(t)] = v[k1];
    __syncthreads();  // G1 RAW; every thread has consumed the staged row
    if (staged && t == 0 && u + stride < batch) {
      fence_proxy_async();
      mbar_expect_tx(stbar, (uint32_t)row_bytes);
      tma_load_1d(stage, static_cast<const unsigned char*>(p.x) + int64_t(u + stride) * p.xs * (row_bytes / p.n),
                  (uint32_t)row_bytes, stbar);
    }
    // ---- P2: (a, b) = (y[n'], y[n' + 256]), n' = j + 32 q -> (a + b, (a - b) W_512^{n'})
    if (ASX_CL128_SHFL) {
      // L1 as a lane-pair swap: n' = l + 16 (h + 2q), so lane (h, l) already holds
      // the i'' = h + 2q half of both 256-point halves; it keeps half k2 = h and
      // trades the other with lane l + 16 (h ^ 1)
      const C wj = w512();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const C a = rg[j + 32 * q], b = rg[L::SUBR + j + 32 * q];
        const C A = cadd(a, b), B = tw_const<16>(cmul(csub(a, b), wj), q);
        const C snd = h ? A : B;
        const C rcv = mk(__shfl_xor_sync(0xffffffffu, snd.x, 16), __shfl_xor_sync(0xffffffffu, snd.y, 16));
        v[2 * q] = h ? rcv : A;
        v[2 * q + 1] = h ? B : rcv;
      }
    } else {
      const C wj = w512();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const C a = rg[j + 32 * q], b = rg[L::SUBR + j + 32 * q];
        v[q] = cadd(a, b);
        v[8 + q] = tw_const<16>(cmul(csub(a, b), wj), q);
      }
      // ---- L1: half k2 -> half-warp k2 (each thread rewrites the slots it read)
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        rg[j + 32 * q] = v[q];
        rg[L::SUBR + j + 32 * q] = v[8 + q];
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = sr[l + 16 * i];
    }
    // ---- P3: radix-16 DIF over n'' = l + 16 i'', × W_256^{l k3}
    ASX_DFT16_F64(v);
    tw_p3(v);
    __syncwarp();
    // ---- L2 (half-warp): (l, k3) -> thread k3
#pragma unroll
    for (int k3 = 0; k3 < 16; ++k3) sr[l + 17 * k3] = v[k3];
    __syncwarp();
#pragma unroll
    for (int n = 0; n < 16; ++n) v[n] = sr[n + 17 * l];
    // ---- P4: radix-16 -> Y[f], × H[f], conj
    ASX_DFT16_F64(v);
#pragma unroll
    for (int k0 = 0; k0 < 16; k0 += 4) {
      C hw[4];
      tm_ld4c(tbase + 4 * k0, hw);
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k0 + k] = cconj(cmul(v[k0 + k], hw[k]));
    }
    // ---- inverse = conj(DFT(conj(.))): Q1 = P4ᵀ
    ASX_DFT16_F64(v);
#pragma unroll
    for (int n = 0; n < 16; ++n) sr[n + 17 * l] = v[n];  // L2ᵀ: the slots this thread read
    __syncwarp();
#pragma unroll
    for (int k3 = 0; k3 < 16; ++k3) v[k3] = sr[l + 17 * k3];
    // ---- Q2 = P3ᵀ
    tw_p3(v);
    ASX_DFT16_F64(v);
    if (ASX_CL128_SHFL) {
      // ---- L1ᵀ (lane-pair swap) and Q3 = P2ᵀ: (A, B) -> (A + W B, A - W B) at (n', n' + 256);
      // the shuffles order every lane's Q2 reads before the writes below
      const C wj = w512();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const C snd = h ? v[2 * q] : v[2 * q + 1];
        const C rcv = mk(__shfl_xor_sync(0xffffffffu, snd.x, 16), __shfl_xor_sync(0xffffffffu, snd.y, 16));
        const C A = h ? rcv : v[2 * q];
        const C WB = tw_const<16>(cmul(h ? v[2 * q + 1] : rcv, wj), q);
        rg[j + 32 * q] = cadd(A, WB);
        rg[L::SUBR + j + 32 * q] = csub(A, WB);
      }
    } else {
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i) sr[l + 16 * i] = v[i];  // L1ᵀ
      __syncwarp();
      // ---- Q3 = P2ᵀ: (A, B) -> (A + W B, A - W B) back to (n', n' + 256)
      const C wj = w512();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const C A = rg[j + 32 * q];
        const C WB = tw_const<16>(cmul(rg[L::SUBR + j + 32 * q], wj), q);
        rg[j + 32 * q] = cadd(A, WB);
        rg[L::SUBR + j + 32 * q] = csub(A, WB);
      }
    }
    __syncthreads();  // G1ᵀ RAW
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) v[k1] = xb[k1 * L::REG + L::pos(t)];
    __syncwarp();
    if ((t & 31) == 0) mbar_arrive(war);
    ++xcnt;
    // ---- Q4 = P1ᵀ: × W_8192^{t k1}, radix-16 -> X[t + 512 i], i < 8
    tw_p1(v);
    ASX_DFT16_F64(v);
    {
      C* X = reinterpret_cast<C*>(p.X) + int64_t(u) * p.Xs;
#pragma unroll
      for (int i0 = 0; i0 < 8; i0 += 4) {
        C cw[4];
        tm_ld4c(tbase + 64 + 4 * i0, cw);
        if (fast_out && live) {
#pragma unroll
          for (int k = 0; k < 4; ++k) X[t + 512 * (i0 + k)] = cmul(cconj(v[i0 + k]), cw[k]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int mm = t + 512 * (i0 + k);
            if (live && mm < p.m) X[mm] = cmul(cconj(v[i0 + k]), cw[k]);
          }
        }
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(tmem_slot, 512);
}



// ---------------------------------------------------------------------------
// k_large_rows_local: the four-step path's fused row pass (asx_large.cuh KB,
// BASELINE config 2: P = 2^23 = 1024 rows x 8192) on the same group-local
// structure: per row k1, forward FFT_8192 (P1 .. P4, DIF) -> × Ht[k1][f] in
// the per-thread spectrum order (the plan stores Ht permuted that way,
// k_permute_ht) -> conj -> the transposed chain Q1 .. Q4 -> × W_P^{k1 c} back
// into the row.  Persistent over rows, the next row of A and of Ht prefetched
// into L2.  2 CTA-wide exchanges per row instead of the engine's 6.
// ---------------------------------------------------------------------------
#ifndef ASX_ROWS_HT_EARLY
#define ASX_ROWS_HT_EARLY 1
#endif
struct RowsLocal {
  using L = ChirpLocal128;
  static constexpr size_t T3_OFF = align_up(size_t(L::XB) * sizeof(double2), 128);
  static constexpr size_t BAR_OFF = align_up(T3_OFF + size_t(L::T3N) * sizeof(double2), 16);
  static constexpr size_t SMEM = BAR_OFF + sizeof(uint64_t) + 16;  // WAR mbar, TMEM slot
  // position of spectrum bin f's value in the permuted Ht row: thread
  // t = 32 k1' + 16 k2 + k3 holds f = k1' + 16 k2 + 32 k3 + 512 k4 at t + 512 k4
  __host__ __device__ static constexpr int perm_src(int slot) {
    return ((slot & 511) >> 5) + 16 * ((slot >> 4) & 1) + 32 * (slot & 15) + 512 * (slot >> 9);
  }
};

// dst[r][slot] = src[r][perm_src(slot)] for r < rows (plan time)
static __global__ void k_permute_ht(double2* __restrict__ dst, const double2* __restrict__ src, int64_t rows) {
  const int64_t total = rows * 8192;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i >> 13;
    const int slot = int(i & 8191);
    dst[i] = src[(r << 13) + RowsLocal::perm_src(slot)];
  }
}

template <typename Real>
__global__ void __launch_bounds__(512, 1) k_large_rows_local(LParams p) {
  static_assert(sizeof(Real) == 8, "complex128 kernel");
  using C = double2;
  using L = ChirpLocal128;
  using RL = RowsLocal;
  extern __shared__ __align__(128) unsigned char smraw[];
  C* xb = reinterpret_cast<C*>(smraw);
  C* T3 = reinterpret_cast<C*>(smraw + RL::T3_OFF);
  uint64_t* war = reinterpret_cast<uint64_t*>(smraw + RL::BAR_OFF);
  uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(war + 1);
  const int t = threadIdx.x, warp = t >> 5, j = t & 31, h = j >> 4, l = j & 15;
  const int rows = int(p.P / L::P);
  const int64_t urows = int64_t(rows) * p.nsig;  // the group's workspaces are one [nsig * rows][P2] matrix
  const uint64_t Pmask = uint64_t(p.P - 1);
  for (int e = t; e < L::T3N; e += L::NT) {
    const int row = e / L::T3S, col = e % L::T3S;
    T3[e] = exact_w<C>(col < 16 ? row * col : 0, 256);
  }
  if (t == 0) {
    mbar_init(war, L::NT / 32);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tmem_slot, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = tmem_slot + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * L::CPT);
  {
    const int es[8] = {1, 2, 3, 4, 8, 12, 0, 0};
#pragma unroll
    for (int q0 = 0; q0 < 8; q0 += 2) {
      uint32_t w8[8];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int q = q0 + k;
        const C w = q < 6 ? exact_w<C>((es[q] * t) & (L::P - 1), L::P) : (q == 6 ? exact_w<C>(j, 512) : mk(1.0, 0.0));
        c_to_words(w, &w8[4 * k]);
      }
      tmem_st8(tbase + 96 + 4 * q0, w8);
    }
    tmem_wait_st();
  }
  __syncthreads();
  auto tw_p1 = [&](C (&v)[16]) {
    C w[8];
    tm_ld4c(tbase + 96, reinterpret_cast<C(&)[4]>(w[0]));
    tm_ld4c(tbase + 112, reinterpret_cast<C(&)[4]>(w[4]));
    v[1] = cmul(v[1], w[0]);
    v[2] = cmul(v[2], w[1]);
    v[3] = cmul(v[3], w[2]);
#pragma unroll
    for (int a = 1; a < 4; ++a) {
      const C w4a = w[2 + a];
      v[4 * a] = cmul(v[4 * a], w4a);
      v[4 * a + 1] = cmul(v[4 * a + 1], cmul(w4a, w[0]));
      v[4 * a + 2] = cmul(v[4 * a + 2], cmul(w4a, w[1]));
      v[4 * a + 3] = cmul(v[4 * a + 3], cmul(w4a, w[2]));
    }
  };
  auto w512 = [&]() {
    C w[4];
    tm_ld4c(tbase + 112, w);
    return w[2];
  };
  auto tw_p3 = [&](C (&v)[16]) {
    const C* row = T3 + L::T3S * l;
#pragma unroll
    for (int k3 = 1; k3 < 16; ++k3) v[k3] = cmul(v[k3], row[k3]);
  };
  C* const rg = xb + warp * L::REG;
  C* const sr = rg + h * L::SUBR;
  const C* Ht = reinterpret_cast<const C*>(p.Ht);
  const C* twb = reinterpret_cast<const C*>(p.twBig);
  uint32_t xcnt = 0;
#pragma unroll 1
  for (int64_t ur = blockIdx.x; ur < urows; ur += gridDim.x) {
    const int k1 = int(ur % rows);
    if (t == 0 && ur + int64_t(gridDim.x) < urows) {
      const int64_t nr = ur + int64_t(gridDim.x);
      prefetch_l2_bulk(reinterpret_cast<const C*>(p.A) + nr * L::P, uint32_t(L::P * sizeof(C)));
      const int64_t nxt = int64_t(nr % rows) * L::P;
      prefetch_l2_bulk(Ht + nxt, uint32_t(L::P * sizeof(C)));
    }
    C* row = reinterpret_cast<C*>(p.A) + ur * L::P;
    C v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = row[t + 512 * i];
    // ---- P1: radix-16 DIF, × W_8192^{t k1'}
    ASX_DFT16_F64(v);
    tw_p1(v);
    if (xcnt) mbar_wait(war, (xcnt - 1) & 1);
#pragma unroll
    for (int k = 0; k < 16; ++k) xb[k * L::REG + L::pos(t)] = v[k];
    __syncthreads();  // G1 RAW
    // ---- P2 + L1 (lane-pair swap)
    {
      const C wj = w512();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const C a = rg[j + 32 * q], b = rg[L::SUBR + j + 32 * q];
        const C A = cadd(a, b), B = tw_const<16>(cmul(csub(a, b), wj), q);
        const C snd = h ? A : B;
        const C rcv = mk(__shfl_xor_sync(0xffffffffu, snd.x, 16), __shfl_xor_sync(0xffffffffu, snd.y, 16));
        v[2 * q] = h ? rcv : A;
        v[2 * q + 1] = h ? B : rcv;
      }
    }
    // ---- P3, L2, P4
    ASX_DFT16_F64(v);
    tw_p3(v);
    __syncwarp();
#pragma unroll
    for (int k3 = 0; k3 < 16; ++k3) sr[l + 17 * k3] = v[k3];
    __syncwarp();
#pragma unroll
    for (int n = 0; n < 16; ++n) v[n] = sr[n + 17 * l];
    // ---- × Ht (permuted row: this thread's bins are contiguous across the CTA), conj; the first half of the
    // spectrum values is requested before P4's butterflies so its L2 latency runs under them
    {
      const C* hr = Ht + int64_t(k1) * L::P + t;
      C hw[8];
#if ASX_ROWS_HT_EARLY
#pragma unroll
      for (int k = 0; k < 8; ++k) hw[k] = __ldg(hr + 512 * k);
      reg_fence();
#endif
      ASX_DFT16_F64(v);
#pragma unroll
      for (int k0 = 0; k0 < 16; k0 += 8) {
        if (k0 || !ASX_ROWS_HT_EARLY) {
#pragma unroll
          for (int k = 0; k < 8; ++k) hw[k] = __ldg(hr + 512 * (k0 + k));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k0 + k] = cconj(cmul(v[k0 + k], hw[k]));
      }
    }
    // ---- Q1, L2ᵀ, Q2
    ASX_DFT16_F64(v);
#pragma unroll
    for (int n = 0; n < 16; ++n) sr[n + 17 * l] = v[n];
    __syncwarp();
#pragma unroll
    for (int k3 = 0; k3 < 16; ++k3) v[k3] = sr[l + 17 * k3];
    tw_p3(v);
    ASX_DFT16_F64(v);
    // ---- L1ᵀ (lane-pair swap) + Q3
    {
      const C wj = w512();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const C snd = h ? v[2 * q] : v[2 * q + 1];
        const C rcv = mk(__shfl_xor_sync(0xffffffffu, snd.x, 16), __shfl_xor_sync(0xffffffffu, snd.y, 16));
        const C A = h ? rcv : v[2 * q];
        const C WB = tw_const<16>(cmul(h ? v[2 * q + 1] : rcv, wj), q);
        rg[j + 32 * q] = cadd(A, WB);
        rg[L::SUBR + j + 32 * q] = csub(A, WB);
      }
    }
    __syncthreads();  // G1ᵀ RAW
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = xb[k * L::REG + L::pos(t)];
    __syncwarp();
    if ((t & 31) == 0) mbar_arrive(war);
    ++xcnt;
    // ---- Q4 = P1ᵀ -> B[k1][c], c = t + 512 i, times W_P^{k1 c}
    tw_p1(v);
    ASX_DFT16_F64(v);
#if ASX_COL_TWCHAIN
    tw_chain_apply<C, 16>(v, twb, uint64_t(k1) * uint64_t(t), uint64_t(k1) * 512u, Pmask, p.lfBig);
#pragma unroll
    for (int i = 0; i < 16; ++i) row[t + 512 * i] = v[i];
#else
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint64_t c = uint64_t(t + 512 * i);
      row[t + 512 * i] = cmul(v[i], tw_big(twb, (uint64_t(k1) * c) & Pmask, p.lfBig));
      if ((i % ASX_FENCE_CHUNK) == ASX_FENCE_CHUNK - 1) reg_fence();
    }
#endif
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(tmem_slot, 512);
}

}  // namespace asx
